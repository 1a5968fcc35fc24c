"""Decomposed-box host logic on CPU (no GPU): the rank layout, the
migration exchange over torch.distributed gloo with world_size 2 and 4, and
the in-process exchange -- driven by a MODEL domain that steps its particles
with the CPU oracle (test infrastructure) instead of libmpcd.

What this pins: cell ownership + one migration per step reproduces the
whole-box step bit for bit (the serial oracle, itself pinned to the
reference), for slab and pencil rank grids, through the same
``DistExchange`` / ``LocalExchange`` / runner code the CUDA backends use.
"""

import os
import socket

import numpy as np
import pytest
import torch

import oracle
import paper_2212_11878_b200 as mp
from paper_2212_11878_b200 import distributed as D

REC = np.dtype([("x", "<f8"), ("y", "<f8"), ("z", "<f8"), ("id", "<u4"), ("pad", "<u4"),
                ("vx", "<f8"), ("vy", "<f8"), ("vz", "<f8"), ("m", "<f8")])
assert REC.itemsize == D.RECORD_BYTES


def owner_cells(layout, positions, step, seed, a):
    """Global cell coordinates of each particle in step `step`'s shifted grid
    (the oracle's binning) and the owning rank."""
    off = oracle.grid_shift(step, seed, a)
    G = np.asarray(layout.global_dims)
    cells = oracle.build_linked_cells(positions, a, off, G, wrap=(True, True, True))[0]
    gx, rem = np.divmod(cells, G[1] * G[2])
    gy, gz = np.divmod(rem, G[2])
    return layout.owner_of_cells(gx, gy, gz)


class ModelDomain:
    """The Domain interface of distributed.py over numpy + the oracle."""

    def __init__(self, params, layout, rank, send_capacity=1 << 14):
        self.params, self.layout, self.rank = params, layout, rank
        self.send_capacity = send_capacity
        self.cs, self.sn = float(np.cos(params.alpha)), float(np.sin(params.alpha))
        self.ids = np.empty(0, np.int64)
        self.pos = np.empty((0, 3))
        self.vel = np.empty((0, 3))
        self.k = 0

    def _keep_own(self, ids, pos, vel, step):
        own = owner_cells(self.layout, pos, step, self.params.seed, self.params.cell_size)
        m = own == self.rank
        order = np.argsort(ids[m], kind="stable")
        self.ids, self.pos, self.vel = ids[m][order], pos[m][order], vel[m][order]

    def upload(self, p):
        self._keep_own(np.arange(p.n, dtype=np.int64), p.positions, p.velocities, 0)

    def init_device(self, n, var):
        raise NotImplementedError

    def step(self, k, flags):
        P = self.layout.n_ranks
        r = oracle.serial_step(self.pos, self.vel, np.ones(len(self.ids)),
                               self.layout.global_dims, self.params.cell_size, self.params.dt,
                               self.cs, self.sn, self.params.seed, k)
        self.post_vel = r.velocities
        dest = owner_cells(self.layout, r.positions, k + 1, self.params.seed,
                           self.params.cell_size) if len(self.ids) else np.empty(0, np.int64)
        self.send = np.zeros((P, self.send_capacity), REC)
        self.send_n = np.zeros(P, np.int64)
        for d in range(P):
            if d == self.rank:
                continue
            sel = np.nonzero(dest == d)[0]
            self.send_n[d] = sel.size
            rec = self.send[d, : min(sel.size, self.send_capacity)]
            sel = sel[: rec.size]
            rec["x"], rec["y"], rec["z"] = r.positions[sel].T
            rec["id"] = self.ids[sel]
            rec["vx"], rec["vy"], rec["vz"] = r.velocities[sel].T
            rec["m"] = 1.0
        stay = dest == self.rank
        self.collided, self.migrated = len(self.ids), int((~stay).sum())
        self.ids, self.pos, self.vel = self.ids[stay], r.positions[stay], r.velocities[stay]
        self.k = k + 1

    def send_counts(self):
        return torch.from_numpy(self.send_n.copy())

    def send_view(self, dest, count):
        return torch.from_numpy(self.send[dest, :count].view(np.uint8).reshape(-1).copy())

    def recv_buffer(self, n):
        return torch.empty(n * D.RECORD_BYTES, dtype=torch.uint8)

    def absorb(self, recv, n_recv, n_sent):
        if n_recv:
            rec = recv[: n_recv * D.RECORD_BYTES].numpy().view(REC)
            ids = np.concatenate([self.ids, rec["id"].astype(np.int64)])
            pos = np.concatenate([self.pos, np.stack([rec["x"], rec["y"], rec["z"]], 1)])
            vel = np.concatenate([self.vel, np.stack([rec["vx"], rec["vy"], rec["vz"]], 1)])
            own = owner_cells(self.layout, pos, self.k, self.params.seed, self.params.cell_size)
            assert np.all(own == self.rank), "received a particle of another rank"
            order = np.argsort(ids, kind="stable")
            self.ids, self.pos, self.vel = ids[order], pos[order], vel[order]

    def diag(self):
        d = oracle.diag(self.post_vel, np.ones(len(self.post_vel)))
        return np.array([*d[:3], d[3], d[4], 0.0, self.collided, self.k - 1, self.migrated])

    def read_com(self):
        raise NotImplementedError

    def download(self):
        return self.ids.copy(), mp.ParticleSet(self.pos.copy(), self.vel.copy(),
                                               np.ones(len(self.ids)))

    def close(self):
        pass


def serial_reference(params, n_steps):
    p = mp.init_system(params)
    pos, vel = p.positions, p.velocities
    cs, sn = float(np.cos(params.alpha)), float(np.sin(params.alpha))
    for k in range(n_steps):
        r = oracle.serial_step(pos, vel, np.ones(p.n), params.dims, params.cell_size, params.dt,
                               cs, sn, params.seed, k)
        pos, vel = r.positions, r.velocities
    return pos, vel


# ------------------------------------------------------------------ layout --
def test_layout_matches_reference_rank_numbering():
    lay = D.DomainLayout((8, 4, 6), (2, 2, 3))
    assert lay.n_ranks == 12 and lay.local_dims == (4, 2, 2)
    for r in range(12):
        ry, rz = 2, 3  # decomposition.py:56-61
        want = (r // (ry * rz), (r // rz) % ry, r % rz)
        assert lay.coords(r) == want
        assert lay.origin(r) == tuple(w * L for w, L in zip(want, (4, 2, 2)))
        o = lay.origin(r)
        assert int(lay.owner_of_cells(o[0], o[1], o[2])) == r
        assert int(lay.owner_of_cells(o[0] + 3, o[1] + 1, o[2] + 1)) == r
    with pytest.raises(mp.TopologyError):
        D.DomainLayout((8, 8, 8), (3, 1, 1))


def test_default_send_capacity_covers_a_face():
    lay = D.DomainLayout((512, 256, 256), (2, 1, 1))
    cap = D.default_send_capacity(lay, 10.0)
    # ~1/3 of a cell layer crosses each face per step; both faces go to the
    # one neighbour at P = 2
    assert cap >= 10 * 256 * 256


# -------------------------------------------------- in-process exchange ---
def _run_local(params, n_steps):
    lay = D.DomainLayout.from_params(params)
    doms = [ModelDomain(params, lay, r) for r in range(lay.n_ranks)]
    p = mp.init_system(params)
    for d in doms:
        d.upload(p)
    assert sum(len(d.ids) for d in doms) == p.n
    runner = D._DomainRunner(params, doms, D.LocalExchange(), capture_drift=False,
                             capture_com=False)
    crossings = 0
    for k in range(n_steps):
        diag = runner.run_step(k)
        crossings += diag["crossings"]
        assert diag["n"] == p.n
    return runner.collect(), crossings


@pytest.mark.parametrize("rank_dims", [(2, 1, 1), (2, 2, 1), (1, 2, 2)])
def test_local_exchange_matches_serial_bitwise(rank_dims):
    params = mp.SimParams(edge_length=8, seed=3, rank_dims=rank_dims)
    (ids, p), crossings = _run_local(params, 4)
    pos, vel = serial_reference(params, 4)
    assert np.array_equal(ids, np.arange(params.n_particles))
    assert np.array_equal(p.positions, pos)
    assert np.array_equal(p.velocities, vel)
    assert crossings > 0


def test_local_exchange_overflow_raises():
    params = mp.SimParams(edge_length=8, seed=3, rank_dims=(2, 1, 1))
    lay = D.DomainLayout.from_params(params)
    doms = [ModelDomain(params, lay, r, send_capacity=4) for r in range(2)]
    p = mp.init_system(params)
    for d in doms:
        d.upload(p)
    runner = D._DomainRunner(params, doms, D.LocalExchange(), capture_drift=False,
                             capture_com=False)
    with pytest.raises(mp.MpcdError, match="overflow"):
        runner.run_step(0)


# ------------------------------------------------ gloo, world_size 2 / 4 ---
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, rank_dims, n_steps, out_dir):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        params = mp.SimParams(edge_length=8, seed=5, rank_dims=rank_dims)
        runner = D.NcclRunner(params, domain_factory=lambda pr, lay, r: ModelDomain(pr, lay, r))
        diags = [runner.run_step(k) for k in range(n_steps)]
        ids, p = runner.collect()
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), ids=ids, pos=p.positions,
                 vel=p.velocities, n=[d["n"] for d in diags],
                 crossings=[d["crossings"] for d in diags],
                 mom=np.array([d["momentum"] for d in diags]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("rank_dims", [(2, 1, 1), (2, 2, 1)])
def test_gloo_ranks_match_serial_bitwise(tmp_path, rank_dims):
    import torch.multiprocessing as tmp_mp

    world = int(np.prod(rank_dims))
    n_steps = 3
    tmp_mp.spawn(_gloo_worker, args=(world, _free_port(), rank_dims, n_steps, str(tmp_path)),
                 nprocs=world, join=True)
    params = mp.SimParams(edge_length=8, seed=5)
    pos, vel = serial_reference(params, n_steps)
    outs = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    for o in outs:  # every rank collects the same global, id-ordered state
        assert np.array_equal(o["ids"], np.arange(params.n_particles))
        assert np.array_equal(o["pos"], pos)
        assert np.array_equal(o["vel"], vel)
        assert list(o["n"]) == [params.n_particles] * n_steps
        assert np.array_equal(o["crossings"], outs[0]["crossings"])
        assert np.all(o["crossings"] > 0)
    # diagnostics are merged in rank order: identical on every rank
    assert all(np.array_equal(o["mom"], outs[0]["mom"]) for o in outs)
    assert np.allclose(outs[0]["mom"], 0.0, atol=1e-10)
