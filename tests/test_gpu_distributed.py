"""GPU parity of the decomposed box: every domain layout
must reproduce the whole-box engine bit for bit -- positions, velocities,
com captures -- because a rank owns whole shifted cells and keys their axes
by the global cell id.  Mirrors the reference's own parallel-vs-serial tests
(test_engine.py:119-135: 1 rank bitwise == serial; N ranks within 1e-10),
with the stronger bitwise bar.

Run on a B200: python -m pytest tests -m gpu
"""

import os
import socket

import numpy as np
import pytest

import paper_2212_11878_b200 as mp
from paper_2212_11878_b200 import distributed as D

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def run(params, backend, n_steps, **kw):
    with mp.Simulation(params, backend=backend, **kw) as sim:
        diags = [sim.step() for _ in range(n_steps)]
        ids, p = sim.collect()
        coms = list(sim.com_captures)
        drift = list(sim.drift_history)
    return ids, p, diags, coms, drift


@pytest.mark.parametrize("dims,rank_dims", [
    ((16, 16, 16), (2, 1, 1)),
    ((16, 16, 16), (4, 1, 1)),
    ((16, 16, 16), (2, 2, 1)),
    ((16, 16, 16), (1, 2, 2)),
    ((16, 16, 16), (2, 2, 2)),
    ((24, 16, 8), (4, 2, 1)),   # non-cubic, pencil (the config-5 shape in small)
    ((8, 8, 8), (8, 1, 1)),     # one-cell slabs: most particles change owner every step
    ((4, 4, 4), (2, 2, 4)),     # 1-2 cells per domain axis, 16 domains
])
@pytest.mark.parametrize("migration", ["fused", "exchange"])
def test_sequential_domains_bitwise_equal_whole_box(dims, rank_dims, migration):
    base = mp.SimParams(edge_length=dims[0], edge_lengths=dims, seed=11)
    dec = mp.SimParams(edge_length=dims[0], edge_lengths=dims, seed=11, rank_dims=rank_dims)
    ids_a, pa, da, ca, _ = run(base, "cuda", 6, capture_com=True)
    ids_b, pb, db, cb, _ = run(dec, "sequential", 6, capture_com=True, migration=migration)
    assert np.array_equal(ids_a, ids_b)
    assert np.array_equal(pa.positions, pb.positions)
    assert np.array_equal(pa.velocities, pb.velocities)
    for (ia, va), (ib, vb) in zip(ca, cb):
        assert np.array_equal(ia, ib) and np.array_equal(va, vb)
    for x, y in zip(da, db):
        assert x["n"] == y["n"]
        assert np.allclose(x["momentum"], y["momentum"], atol=1e-9)
        assert abs(x["energy"] - y["energy"]) <= 1e-10 * x["energy"]
        assert x["mass"] == y["mass"]
    assert sum(d["crossings"] for d in db) > 0


def test_one_domain_nccl_equals_cuda():
    """test_engine.py:129-135: one rank of the parallel path == serial, bitwise."""
    import torch.distributed as dist

    params = mp.SimParams(edge_length=12, seed=2)
    ids_a, pa, _, _, _ = run(params, "cuda", 5)
    os.environ["MASTER_PORT"] = str(_free_port())
    D.init_distributed("nccl")
    try:
        ids_b, pb, db, _, _ = run(params, "nccl", 5)
    finally:
        dist.destroy_process_group()
    assert np.array_equal(pa.positions, pb.positions)
    assert np.array_equal(pa.velocities, pb.velocities)
    assert all(d["crossings"] == 0 for d in db)


@pytest.mark.parametrize("prng", ["splitmix", "pcg32", "minstd", "sfc64"])
def test_device_init_domains_equal_whole_box(prng):
    dims = (32, 32, 32)
    base = mp.SimParams(edge_length=32, seed=7, prng=prng)
    dec = mp.SimParams(edge_length=32, seed=7, prng=prng, rank_dims=(4, 1, 1))
    ids_a, pa, _, _, drift_a = run(base, "cuda", 4, init="device", capture_drift=True)
    ids_b, pb, _, _, drift_b = run(dec, "sequential", 4, init="device", capture_drift=True)
    assert np.array_equal(ids_a, ids_b)
    assert np.array_equal(pa.positions, pb.positions)
    assert np.array_equal(pa.velocities, pb.velocities)
    assert np.allclose(drift_a, drift_b, rtol=0, atol=1e-12)
    del dims


def test_migration_overflow_raises():
    params = mp.SimParams(edge_length=16, seed=1, rank_dims=(2, 1, 1))
    from paper_2212_11878_b200.distributed import SequentialRunner
    r = SequentialRunner(params, send_capacity=8, migration="exchange")
    try:
        with pytest.raises(mp.MpcdError, match="overflow"):
            r.run_step(0)
    finally:
        r.close()


def test_domain_rejects_bad_topology():
    from paper_2212_11878_b200.engine import EngineContext
    ctx = EngineContext((8, 8, 8), 1.0, 0.1, 1.0, 0, "splitmix", 6000, mass_value=1.0)
    try:
        with pytest.raises(mp.TopologyError):
            ctx.set_domain((24, 8, 8), (2, 1, 1), 0)  # 24 != 2 * 8
        with pytest.raises(mp.TopologyError):
            ctx.set_domain((16, 8, 8), (2, 1, 1), 2)  # rank out of range
    finally:
        ctx.close()


# ------------------------------------- two processes on one GPU (gloo) ---
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir, migration):
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        params = mp.SimParams(edge_length=16, seed=4, rank_dims=(world, 1, 1))
        with mp.Simulation(params, backend="nccl", capture_com=True,
                           migration=migration) as sim:
            diags = [sim.step() for _ in range(4)]
            ids, p = sim.collect()
            ci, cv = sim.com_captures[-1]
            used = sim.runner.migration
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), ids=ids, pos=p.positions,
                 vel=p.velocities, ci=ci, cv=cv, crossings=[d["crossings"] for d in diags],
                 used=used)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("migration", ["fused", "exchange"])
def test_two_processes_gloo_equal_whole_box(tmp_path, migration):
    """Two processes sharing one GPU: fused = k_step writes into the other
    process's regions through CUDA IPC handles; exchange = gloo host-staged."""
    import torch.multiprocessing as tmp_mp

    tmp_mp.spawn(_worker, args=(2, _free_port(), str(tmp_path), migration), nprocs=2,
                 join=True)
    params = mp.SimParams(edge_length=16, seed=4)
    ids, p, _, coms, _ = run(params, "cuda", 4, capture_com=True)
    for r in range(2):
        o = np.load(tmp_path / f"r{r}.npz")
        assert np.array_equal(o["ids"], ids)
        assert np.array_equal(o["pos"], p.positions)
        assert np.array_equal(o["vel"], p.velocities)
        assert np.array_equal(o["ci"], coms[-1][0]) and np.array_equal(o["cv"], coms[-1][1])
        assert np.all(o["crossings"] > 0)
        assert str(o["used"]) == migration


@pytest.mark.parametrize("scheme", ["halo", "migration"])
def test_equivalence_check_serial_vs_decomposed_is_exact(scheme):
    """Acceptance criterion 3 of the reference (cross-scheme equivalence,
    test_acceptance.py:63-85, bound 1e-10): here the deviations are zero."""
    params = mp.SimParams(edge_length=12, seed=8)
    rep = mp.equivalence_check(params, (1, 1, 1), (2, 2, 1), "serial", scheme, 5,
                               capture_com=True)
    assert rep.n_steps == 5
    assert rep.max_position_dev == 0.0
    assert rep.max_velocity_dev == 0.0
    assert rep.max_com_dev == 0.0


@pytest.mark.parametrize("migration", ["fused", "exchange"])
def test_dense_cluster_across_domain_boundary(migration):
    """Clustered particles straddling a slab boundary: cells far above their
    capacity (overflow lists, k_step_dense) on both sides, and -- fused --
    overflow appends into the other domain's lists.  Must equal the whole box
    and the oracle."""
    import oracle

    rs = np.random.default_rng(12)
    n = 8000
    pos = np.concatenate([rs.uniform([7.4, 3.1, 3.1], [8.6, 3.9, 3.9], size=(6000, 3)),
                          rs.uniform(0, 16, size=(2000, 3))])
    vel = rs.normal(size=(n, 3)) * 3.0
    p = mp.ParticleSet(pos, vel, np.ones(n))
    base = mp.SimParams(edge_length=16, seed=5, mean_density=n / 4096)
    dec = mp.SimParams(edge_length=16, seed=5, mean_density=n / 4096, rank_dims=(2, 1, 1))
    with mp.Simulation(base, backend="cuda") as whole, \
            mp.Simulation(dec, backend="sequential", migration=migration) as parts:
        whole.runner.ctx.upload(p.positions, p.velocities, None, None, 0)
        for d in parts.runner.domains:
            d.upload(p)
        cs, sn = float(np.cos(base.alpha)), float(np.sin(base.alpha))
        ref_pos, ref_vel = pos, vel
        for k in range(4):
            whole.step()
            parts.step()
            r = oracle.serial_step(ref_pos, ref_vel, np.ones(n), 16, 1.0, base.dt, cs, sn,
                                   base.seed, k)
            ref_pos, ref_vel = r.positions, r.velocities
            (ia, pa), (ib, pb) = whole.collect(), parts.collect()
            assert np.array_equal(pa.positions, ref_pos) and np.array_equal(pa.velocities, ref_vel)
            assert np.array_equal(ia, ib)
            assert np.array_equal(pa.positions, pb.positions), k
            assert np.array_equal(pa.velocities, pb.velocities), k


@pytest.mark.parametrize("tag", ["halo", "migr"])
@pytest.mark.parametrize("migration", ["fused", "exchange"])
def test_matches_reference_parallel_runs(tag, migration):
    """Against the reference's OWN rank-parallel step (golden parallel_L8.npz,
    its "sequential" runner, halo scheme on (2,2,1) and migration scheme on
    (2,1,1)): within the reference's bound of 1e-10 (test_engine.py:119-126),
    and bitwise equal to the reference's serial run of the same config."""
    from conftest import golden

    g = golden("parallel_L8.npz")
    rank_dims = tuple(int(x) for x in g[f"{tag}_rank_dims"])
    params = mp.SimParams(edge_length=8, seed=3, rank_dims=rank_dims,
                          scheme="halo" if tag == "halo" else "migration")
    with mp.Simulation(params, backend="sequential", capture_com=True,
                       migration=migration) as sim:
        for k in range(int(g["steps"])):
            sim.step()
            ids, p = sim.collect()
            assert np.array_equal(ids, g[f"{tag}_ids{k}"])
            d = np.abs(p.positions - g[f"{tag}_pos{k}"])
            assert np.minimum(d, 8.0 - d).max() <= 1e-10
            assert np.abs(p.velocities - g[f"{tag}_vel{k}"]).max() <= 1e-10
            assert np.array_equal(p.positions, g[f"serial_pos{k}"])
            assert np.array_equal(p.velocities, g[f"serial_vel{k}"])
            ci, cv = sim.com_captures[-1]
            assert np.array_equal(ci, g[f"{tag}_comids{k}"])
            assert np.abs(cv - g[f"{tag}_com{k}"]).max() <= 1e-10


@pytest.mark.parametrize("migration", ["fused", "exchange"])
def test_non_unit_cell_size_and_prng_domains(migration):
    """cell_size != 1 (IEEE division in the binning), a short dt, a 3 x 1 x 2
    rank grid and the pcg32 generator: still the whole box bit for bit."""
    kw = dict(edge_length=12, cell_size=0.5, dt=0.05, seed=21, prng="pcg32")
    ids_a, pa, _, ca, _ = run(mp.SimParams(**kw), "cuda", 5, capture_com=True)
    ids_b, pb, _, cb, _ = run(mp.SimParams(rank_dims=(3, 1, 2), **kw), "sequential", 5,
                              capture_com=True, migration=migration)
    assert np.array_equal(ids_a, ids_b)
    assert np.array_equal(pa.positions, pb.positions)
    assert np.array_equal(pa.velocities, pb.velocities)
    assert np.array_equal(ca[-1][0], cb[-1][0]) and np.array_equal(ca[-1][1], cb[-1][1])


@pytest.mark.parametrize("prng", ["splitmix", "minstd", "pcg32", "sfc64"])
def test_config2_64cubed_domains_equal_whole_box(prng):
    """BASELINE config 2 (64^3 x 10 = 2.6 M particles) on a 2 x 2 x 2 domain
    grid with fused migration, every PRNG: the whole box bit for bit."""
    base = mp.SimParams(edge_length=64, seed=0, prng=prng)
    dec = mp.SimParams(edge_length=64, seed=0, prng=prng, rank_dims=(2, 2, 2))
    ids_a, pa, da, _, _ = run(base, "cuda", 3, init="device")
    ids_b, pb, db, _, _ = run(dec, "sequential", 3, init="device")
    assert np.array_equal(ids_a, ids_b)
    assert np.array_equal(pa.positions, pb.positions)
    assert np.array_equal(pa.velocities, pb.velocities)
    assert all(d["crossings"] > 0 for d in db)


def test_benchmark_report_cases_and_matrix(tmp_path):
    """mpcdsim.bench on the GPU backends (the reference's test_bench_cli.py:43-104)."""
    from paper_2212_11878_b200 import bench

    params = mp.SimParams(edge_length=8, mean_density=4.0, rank_dims=(2, 1, 1), n_steps=3)
    rec = bench.run_benchmark_case(params, steps=3, warmup=1)
    assert rec.L == 8 and rec.ranks == 2 and rec.steps == 3
    assert rec.particles == params.n_particles and rec.seconds > 0.0
    assert rec.bytes_per_step > 0.0 and rec.msgs_per_step > 0.0
    assert rec.max_drift < 1e-11 and rec.error == ""
    one = bench.run_benchmark_case(mp.SimParams(edge_length=8, mean_density=4.0), steps=2,
                                   warmup=1)
    assert one.ranks == 1 and one.bytes_per_step == 0.0
    with pytest.raises(mp.ConfigError):
        bench.run_benchmark_case(params, steps=0, warmup=1)
    seen = []
    recs = bench.run_benchmark_matrix(sizes=(8,), rank_counts=(1, 2, 3), steps=2, warmup=1,
                                      density=4.0,
                                      progress=lambda L, s, r: seen.append((L, s, r)))
    assert seen == [(8, "halo", 1), (8, "halo", 2), (8, "halo", 3)]
    assert recs[0].error == "" and recs[1].error == ""
    assert "ConfigError" in recs[2].error and recs[2].seconds == 0.0
    path = tmp_path / "b.csv"
    bench.emit_report(recs, str(path))
    assert bench.read_report(str(path)) == recs


def test_process_backend_alias_runs_the_domains_in_process():
    """The reference's "process" backend name (one worker per rank there)
    runs the same decomposition in this process here."""
    params = mp.SimParams(edge_length=8, seed=6, rank_dims=(2, 1, 1))
    ids_a, pa, _, _, _ = run(mp.SimParams(edge_length=8, seed=6), "cuda", 3)
    ids_b, pb, _, _, _ = run(params, mp.BACKEND_PROCESS, 3)
    assert np.array_equal(pa.positions, pb.positions)
    assert np.array_equal(pa.velocities, pb.velocities)


def test_full_size_two_domains_fused_equal_whole_box():
    """BASELINE config 3 size (256^3 cells, 167.8 M particles) as two fused
    slab domains on this GPU: hundreds of thousands of particles migrate
    every step, and the state equals the whole box bit for bit."""
    import torch

    kw = dict(edge_length=256, seed=2)
    with mp.Simulation(mp.SimParams(**kw), backend="cuda", init="device") as whole:
        whole.advance(3)
        ids_a, pa = whole.collect()
    torch.cuda.empty_cache()
    with mp.Simulation(mp.SimParams(rank_dims=(2, 1, 1), **kw), backend="sequential",
                       init="device") as parts:
        diags = [parts.step() for _ in range(3)]
        ids_b, pb = parts.collect()
    torch.cuda.empty_cache()
    assert np.array_equal(ids_a, ids_b)
    assert np.array_equal(pa.positions, pb.positions)
    assert np.array_equal(pa.velocities, pb.velocities)
    assert all(d["crossings"] > 100_000 for d in diags)


# -------------------------------- two NCCL ranks on two distinct GPUs ---
def _nccl_worker(rank, world, port, out_dir, L, steps, migration):
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(rank)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        params = mp.SimParams(edge_length=L, seed=13, rank_dims=(world, 1, 1))
        with mp.Simulation(params, backend="nccl", init="device", capture_com=True,
                           migration=migration) as sim:
            diags = [sim.step() for _ in range(steps)]
            # this rank's own particles only (no all-gather of the whole box)
            (_, ids, p), = sim.runner._local_sets()
            used = sim.runner.migration
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), ids=ids, pos=p.positions,
                 vel=p.velocities, crossings=[d["crossings"] for d in diags], used=used)
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(not __import__("torch").cuda.is_available()
                    or __import__("torch").cuda.device_count() < 2,
                    reason="needs two GPUs (NCCL ranks on distinct devices)")
@pytest.mark.parametrize("L,steps", [(64, 5), (256, 3)])
@pytest.mark.parametrize("migration", ["fused", "exchange"])
def test_two_gpus_nccl_equal_whole_box(tmp_path, L, steps, migration):
    """Two NCCL ranks on two distinct GPUs (slab (2,1,1)): the fused migration
    writes over NVLink peer memory with system-scope slot claims and an NCCL
    all-reduce step fence; the exchange moves send buffers with NCCL
    point-to-point.  Either way the collected state equals the whole box on
    one GPU bit for bit (reference contract: engine.py:190-272,
    test_engine.py:119-135, bound 1e-10 there; bitwise here)."""
    import torch
    import torch.multiprocessing as tmp_mp

    tmp_mp.spawn(_nccl_worker, args=(2, _free_port(), str(tmp_path), L, steps, migration),
                 nprocs=2, join=True)
    torch.cuda.set_device(0)
    with mp.Simulation(mp.SimParams(edge_length=L, seed=13), backend="cuda",
                       init="device") as whole:
        for _ in range(steps):
            whole.step()
        ids, p = whole.collect()
    torch.cuda.empty_cache()
    parts = [np.load(tmp_path / f"r{r}.npz") for r in range(2)]
    got_ids = np.concatenate([o["ids"] for o in parts])
    order = np.argsort(got_ids, kind="stable")
    assert np.array_equal(got_ids[order], ids)
    pos = np.concatenate([o["pos"].reshape(-1, 3) for o in parts])[order]
    vel = np.concatenate([o["vel"].reshape(-1, 3) for o in parts])[order]
    assert np.array_equal(pos, p.positions)
    assert np.array_equal(vel, p.velocities)
    for o in parts:
        assert str(o["used"]) == migration
        assert np.all(o["crossings"] > 0)


def test_ids_above_2_31_rank_with_unsigned_compares():
    """Global ids above 2^31 - 1 (a system of more than 2^31 particles, e.g.
    BASELINE config 5's 2.7 G) switch k_step's in-cell ranking from the
    sign-bit compare to the unsigned compare.  Ids 3e9 + i order like i, so
    the decomposed box must equal the whole box (ids i) bit for bit."""
    from paper_2212_11878_b200.distributed import SequentialRunner

    base = mp.SimParams(edge_length=16, seed=31)
    ids_w, p_w, _, _, _ = run(base, "cuda", 3)
    p0 = mp.init_system(base)
    big = np.int64(3_000_000_000) + np.arange(p0.n, dtype=np.int64)
    r = SequentialRunner(mp.SimParams(edge_length=16, seed=31, rank_dims=(2, 1, 1)))
    try:
        for d in r.domains:  # every domain takes the whole box's rows and keeps its own
            d.ctx.upload(p0.positions, p0.velocities, None, big, 0)
        for k in range(3):
            r.run_step(k)
        ids, p = r.collect()
    finally:
        r.close()
    assert np.array_equal(ids, big)
    assert np.array_equal(p.positions, p_w.positions)
    assert np.array_equal(p.velocities, p_w.velocities)


def _geometry_worker(rank, world, port, out_dir):
    import warnings

    import torch
    import torch.distributed as dist

    from paper_2212_11878_b200.distributed import (CudaDomain, DistExchange, DomainLayout,
                                                   _DomainRunner, connect_fused)
    torch.cuda.set_device(0)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        params = mp.SimParams(edge_length=16, seed=7, rank_dims=(world, 1, 1))
        layout = DomainLayout.from_params(params)
        # rank 1 sizes its context larger: its cell capacity (and overflow
        # list) differ from rank 0's, so the fused connection must refuse
        cap = 30_000 if rank == 0 else 200_000
        dom = CudaDomain(params, layout, rank, capacity=cap)
        exch = DistExchange()
        with warnings.catch_warnings(record=True) as w:
            warnings.simplefilter("always")
            fused = connect_fused(dom, exch)
        dom.upload(mp.init_system(mp.SimParams(edge_length=16, seed=7)))
        runner = _DomainRunner(params, [dom], exch, capture_drift=False, capture_com=False,
                               fused=fused)
        for k in range(3):
            runner.run_step(k)
        ids, p = runner.collect()
        np.savez(os.path.join(out_dir, f"g{rank}.npz"), ids=ids, pos=p.positions,
                 vel=p.velocities, fused=fused, warned=any("fused" in str(x.message) for x in w))
        runner.close()
    finally:
        dist.destroy_process_group()


def test_fused_connection_refuses_unequal_geometry(tmp_path):
    """Two ranks whose contexts differ in slots per cell: mpcd_connect_peers
    rejects the connection (a peer would address the other's regions with
    the wrong stride), connect_fused warns and every rank falls back to the
    exchange, and the result is still the whole box bit for bit."""
    import torch.multiprocessing as tmp_mp

    tmp_mp.spawn(_geometry_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    ids, p, _, _, _ = run(mp.SimParams(edge_length=16, seed=7), "cuda", 3)
    for r in range(2):
        o = np.load(tmp_path / f"g{r}.npz")
        assert not bool(o["fused"]) and bool(o["warned"])
        assert np.array_equal(o["ids"], ids)
        assert np.array_equal(o["pos"], p.positions)
        assert np.array_equal(o["vel"], p.velocities)
