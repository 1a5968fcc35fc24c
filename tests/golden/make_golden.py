"""Generate golden vectors from the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``mpcdsim`` from ``/root/reference/pkg/src`` (read-only, never
copied) and writes small ``.npz`` fixtures next to this script.  Nothing on
the GPU box reads ``/root/reference``: the tests only read these fixtures.

Fixtures
--------
rng.npz         key_state / uniform_at / gaussian_at / grid shifts / axes
collision.npz   build_linked_cells, segment_moments, finalize_com,
                rotate_velocities, wrap_coordinates, stream_and_wrap cases
serial_small.npz  full per-step state of serial_collision_step runs
                (L=4 seed 7, L=6 seed 1, L=4 random masses, L=5 dt=8 boost)
config1_L16.npz   BASELINE config 1 (16^3, 10/cell, 130 deg, seed 42):
                initial state + per-step SHA-256 of the reference state,
                cells, counts, permutation for 100 steps, diagnostics
config2_L64.npz   64^3 seed 0: hash of the initial state and of 3 steps
init_device.npz   init_system (particles.py:101-127) at 64^3 seed 0 and
                16^3 x 12.5 seed 3: SHA-256 of the positions, every 1009th
                velocity row, the subtracted mean (mean_init_velocity) --
                pins the device init (positions bit-exact, velocities to
                libm-vs-numpy ulps)
bench_report.csv  the reference's emit_report of fixed records (+ .summary.txt)
                and rank_dims_for(1..64) (bench_rank_dims.npy)
decomposition.npz rank grids (neighbour tables, borders, coordinates),
                base-3 side codes of random and border positions
parallel_L8.npz   the reference's own rank-parallel step (backend
                "sequential": halo scheme on (2,2,1), migration scheme on
                (2,1,1)), per-step state and com capture, and the serial run
                of the same config
"""

from __future__ import annotations

import hashlib
import math
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.dont_write_bytecode = True
sys.path.insert(0, REF_SRC)

import mpcdsim  # noqa: E402
from mpcdsim import collision, engine, particles, rng  # noqa: E402
from mpcdsim.params import SimParams  # noqa: E402


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def make_rng():
    rs = np.random.default_rng(1234)
    M = (1 << 64) - 1
    keys = [(0, 0, 0, 0), (M, M, M, M), (42, 7, 1, 123), (1, 0, 0, 0), (0, 1, 0, 0),
            (0, 0, 1, 0), (0, 0, 0, 1), (5, 2, 1, 2 ** 40), (2 ** 63, 3, 2, 99)]
    keys += [tuple(int(x) for x in rs.integers(0, 2 ** 63, size=4)) for _ in range(55)]
    ks_in = np.array(keys, dtype=np.uint64)
    ks_out = np.array([int(rng.key_state(*k)) for k in keys], dtype=np.uint64)
    ua_state = ks_out[:16]
    ua_idx = np.array([0, 1, 2, 3, 7, 100, 2 ** 32, 2 ** 63 - 1, M - 1, 12345, 6, 5, 4, 9, 8, 11],
                      dtype=np.uint64)
    ua_out = np.array([float(rng.uniform_at(s, np.uint64(i))) for s, i in zip(ua_state, ua_idx)])
    gstate = rng.key_state(11, 0, rng.Purpose.INIT, 0)
    gauss = rng.gaussian_at(gstate, np.arange(1000, dtype=np.uint64))
    shift_seeds = np.array([0, 17, 42, 2 ** 63 + 5], dtype=np.uint64)
    shifts = np.array([[collision.sample_grid_shift(s, int(seed), 1.0).offset for s in range(100)]
                       for seed in shift_seeds])
    shifts_a25 = np.array([collision.sample_grid_shift(s, 9, 2.5).offset for s in range(50)])
    axes_ids = np.arange(4096, dtype=np.int64)
    axes = collision.sample_rotation_axes(7, axes_ids, 42)
    axes_sparse_ids = np.array([3, 17, 99, 2 ** 40, 2 ** 62 + 11], dtype=np.int64)
    axes_sparse = collision.sample_rotation_axes(5, axes_sparse_ids, 11)
    su = rng.sample_uniform(rng.RngKey(seed=42, step=7, purpose=rng.Purpose.AXIS, cell_id=123), 64)
    np.savez_compressed(
        os.path.join(HERE, "rng.npz"), ks_in=ks_in, ks_out=ks_out, ua_state=ua_state, ua_idx=ua_idx,
        ua_out=ua_out, gauss=gauss, shift_seeds=shift_seeds, shifts=shifts, shifts_a25=shifts_a25,
        axes_ids=axes_ids, axes=axes, axes_sparse_ids=axes_sparse_ids, axes_sparse=axes_sparse,
        sample_uniform=su)


def make_collision():
    out = {}
    rs = np.random.default_rng(99)
    cases = []
    # (name, positions, cell_size, gmin, gmax, wrap)
    cases.append(("A", rs.uniform(0.0, 4.0, size=(500, 3)), 1.0, np.zeros(3), np.full(3, 4.0),
                  (False, False, False)))
    cases.append(("B", np.array([[-0.3, 3.9, 8.2], [7.9, 0.0, -7.9]]), 1.0, np.zeros(3),
                  np.full(3, 8.0), (True, True, True)))
    cases.append(("C", rs.uniform(0.0, 8.0, size=(20000, 3)), 1.0, np.array([-0.3, 0.2, 0.45]),
                  np.array([7.7, 8.2, 8.45]), (True, True, True)))
    cases.append(("D", rs.uniform([-1.2, -3.0, -1.4], [6.7, 9.0, 7.4], size=(3000, 3)), 0.5, np.array([-1.25, -1.0, -1.5]),
                  np.array([6.75, 7.0, 7.5]), (False, True, False)))
    # dense: ~375 particles per cell (pairwise recursion > 128)
    cases.append(("E", rs.uniform(0.0, 2.0, size=(3000, 3)), 1.0, np.zeros(3), np.full(3, 2.0),
                  (True, True, True)))
    # exact cell faces and tiny negatives
    face = np.array([[0.0, 1.0, 2.0], [1.0 - 2 ** -53, 2.0 - 2 ** -52, 3.0], [-1e-17, 0.5, 3.999999],
                     [3.0, 3.0, 3.0], [np.nextafter(0.0, 1.0), 1e-300, 2.5]])
    cases.append(("F", face, 1.0, np.zeros(3), np.full(3, 4.0), (True, True, True)))
    for name, pos, a, gmin, gmax, wrap in cases:
        lc = collision.build_linked_cells(pos, a, gmin, gmax, wrap=wrap)
        out[f"{name}_pos"] = pos
        out[f"{name}_a"] = np.float64(a)
        out[f"{name}_gmin"] = gmin
        out[f"{name}_dims"] = lc.dims
        out[f"{name}_wrap"] = np.array(wrap, dtype=np.int32)
        out[f"{name}_cells"] = lc.cells
        out[f"{name}_counts"] = lc.bin_count
        out[f"{name}_offsets"] = lc.bin_offset
        out[f"{name}_perm"] = lc.permutation
        vel = rs.normal(size=pos.shape) * 10 ** rs.uniform(-2, 2, size=pos.shape)
        mass = rs.uniform(0.5, 2.0, size=pos.shape[0])
        mom = collision.segment_moments(lc, vel, mass)
        out[f"{name}_vel"] = vel
        out[f"{name}_mass"] = mass
        out[f"{name}_moments"] = mom
        out[f"{name}_com"] = collision.finalize_com(collision.CellMomentField(mom))
    # binning errors (index, axis)
    err_pos = np.array([[0.5, 0.5, 0.5], [0.5, 2.5, 0.5], [3.0, 0.5, -0.2], [0.1, 0.2, 0.3]])
    try:
        collision.build_linked_cells(err_pos, 1.0, np.zeros(3), np.full(3, 2.0))
    except mpcdsim.BinningError as e:
        out["err_pos"] = err_pos
        out["err_info"] = np.array([e.particle_index, e.dimension])
    # rotation
    n = 5000
    vel = rs.normal(size=(n, 3))
    com = rs.normal(size=(n, 3))
    axes = rs.normal(size=(n, 3))
    axes /= np.linalg.norm(axes, axis=1, keepdims=True)
    for tag, alpha in (("r1", 1.1), ("r130", math.radians(130.0)), ("rq", np.pi / 2)):
        out[f"{tag}_alpha"] = np.float64(alpha)
        out[f"{tag}_cos"] = np.float64(np.cos(alpha))
        out[f"{tag}_sin"] = np.float64(np.sin(alpha))
        out[f"{tag}_out"] = collision.rotate_velocities(vel, com, axes, alpha)
    out["rot_vel"], out["rot_com"], out["rot_axes"] = vel, com, axes
    # wrap + stream
    wx = np.concatenate([np.array([-0.5, 8.5, 17.0, -16.25, -1e-17, 8.0, 0.0, -0.0, 1e-300,
                                   np.nextafter(8.0, 0.0), -8.0, 16.0, -24.0 - 1e-13]),
                         rs.uniform(-30.0, 40.0, size=2000)])
    out["wrap_x"] = wx
    out["wrap_out"] = particles.wrap_coordinates(wx, 8.0)
    sp = rs.uniform(0.0, 8.0, size=(3000, 3))
    sv = rs.normal(size=(3000, 3)) * 5
    ps = particles.stream_and_wrap(particles.ParticleSet(sp, sv, np.ones(3000)), 0.7, 8.0)
    out["stream_pos"], out["stream_vel"], out["stream_out"] = sp, sv, ps.positions
    np.savez_compressed(os.path.join(HERE, "collision.npz"), **out)


def _run_serial(params, p0, steps, tag, out):
    """Record every intermediate of serial_collision_step for `steps` steps."""
    p = p0
    out[f"{tag}_L"] = np.int64(params.edge_length)
    out[f"{tag}_seed"] = np.int64(params.seed)
    out[f"{tag}_dt"] = np.float64(params.dt)
    out[f"{tag}_a"] = np.float64(params.cell_size)
    out[f"{tag}_cos"] = np.float64(np.cos(params.alpha))
    out[f"{tag}_sin"] = np.float64(np.sin(params.alpha))
    out[f"{tag}_alpha"] = np.float64(params.alpha)
    out[f"{tag}_steps"] = np.int64(steps)
    out[f"{tag}_pos0"], out[f"{tag}_vel0"], out[f"{tag}_mass"] = p.positions, p.velocities, p.masses
    for k in range(steps):
        off = collision.sample_grid_shift(k, params.seed, params.cell_size).offset
        box = params.box_length
        lc = collision.build_linked_cells(p.positions, params.cell_size, off, off + box,
                                          wrap=(True, True, True))
        mom = collision.segment_moments(lc, p.velocities, p.masses)
        p, drift, (occ, com) = engine.serial_collision_step(p, params, k, want_drift=True,
                                                             want_com=True)
        out[f"{tag}_cells{k}"] = lc.cells
        out[f"{tag}_counts{k}"] = lc.bin_count
        out[f"{tag}_perm{k}"] = lc.permutation
        out[f"{tag}_mom{k}"] = mom
        out[f"{tag}_occ{k}"] = occ
        out[f"{tag}_com{k}"] = com
        out[f"{tag}_drift{k}"] = np.float64(drift)
        out[f"{tag}_pos{k + 1}"] = p.positions
        out[f"{tag}_vel{k + 1}"] = p.velocities


def make_serial_small():
    out = {}
    pa = SimParams(edge_length=4, seed=7)
    _run_serial(pa, particles.init_system(pa), 6, "L4", out)
    pb = SimParams(edge_length=6, seed=1, mean_density=5.0)
    _run_serial(pb, particles.init_system(pb), 6, "L6", out)
    pc = SimParams(edge_length=4, seed=3, alpha=1.1, dt=0.37)
    base = particles.init_system(pc)
    rs = np.random.default_rng(5)
    massive = particles.ParticleSet(base.positions, base.velocities,
                                    rs.uniform(0.5, 2.0, size=base.n))
    _run_serial(pc, massive, 5, "M4", out)
    pd = SimParams(edge_length=5, seed=3, dt=8.0)
    _run_serial(pd, particles.init_system(pd), 4, "B5", out)
    np.savez_compressed(os.path.join(HERE, "serial_small.npz"), **out)


def make_config1():
    params = SimParams(edge_length=16, mean_density=10.0, dt=0.1, alpha=math.radians(130.0),
                       seed=42, n_steps=100)
    sim = engine.Simulation(params, backend="serial", capture_drift=True)
    ids, p0 = sim.collect()
    out = dict(pos0=p0.positions, vel0=p0.velocities, L=np.int64(16), seed=np.int64(42),
               dt=np.float64(0.1), cos=np.float64(np.cos(params.alpha)),
               sin=np.float64(np.sin(params.alpha)), steps=np.int64(100))
    out["init_sha"] = np.array(sha(p0.positions, p0.velocities))
    state_sha, bin_sha, diag = [], [], []
    p = p0
    for k in range(100):
        off = collision.sample_grid_shift(k, params.seed, params.cell_size).offset
        lc = collision.build_linked_cells(p.positions, 1.0, off, off + params.box_length,
                                          wrap=(True, True, True))
        bin_sha.append(sha(lc.cells, lc.bin_count, lc.permutation))
        d = sim.step()
        _, p = sim.collect()
        state_sha.append(sha(p.positions, p.velocities))
        diag.append(np.concatenate([d["momentum"], [d["energy"], d["mass"], d["max_cell_drift"]]]))
    out["state_sha"] = np.array(state_sha)
    out["bin_sha"] = np.array(bin_sha)
    out["diag"] = np.array(diag)
    out["pos_final"], out["vel_final"] = p.positions, p.velocities
    np.savez_compressed(os.path.join(HERE, "config1_L16.npz"), **out)


def make_config2(steps=3):
    params = SimParams(edge_length=64, seed=0)
    p = particles.init_system(params)
    out = dict(L=np.int64(64), seed=np.int64(0), dt=np.float64(params.dt),
               cos=np.float64(np.cos(params.alpha)), sin=np.float64(np.sin(params.alpha)),
               steps=np.int64(steps))
    out["init_sha"] = np.array(sha(p.positions, p.velocities))
    state_sha, bin_sha = [], []
    for k in range(steps):
        off = collision.sample_grid_shift(k, params.seed, params.cell_size).offset
        lc = collision.build_linked_cells(p.positions, 1.0, off, off + params.box_length,
                                          wrap=(True, True, True))
        bin_sha.append(sha(lc.cells, lc.bin_count, lc.permutation))
        p, _, _ = engine.serial_collision_step(p, params, k)
        state_sha.append(sha(p.positions, p.velocities))
    out["state_sha"] = np.array(state_sha)
    out["bin_sha"] = np.array(bin_sha)
    np.savez_compressed(os.path.join(HERE, "config2_L64.npz"), **out)


def make_init_device():
    out = {}
    for tag, params in (("L64", SimParams(edge_length=64, seed=0)),
                        ("L16", SimParams(edge_length=16, seed=3, mean_density=12.5))):
        p = particles.init_system(params)
        out[f"{tag}_L"] = np.int64(params.edge_length)
        out[f"{tag}_seed"] = np.int64(params.seed)
        out[f"{tag}_density"] = np.float64(params.mean_density)
        out[f"{tag}_n"] = np.int64(p.n)
        out[f"{tag}_pos_sha"] = np.array(sha(p.positions))
        out[f"{tag}_vel_rows"] = p.velocities[::1009].copy()
        out[f"{tag}_pos_rows"] = p.positions[::1009].copy()
        out[f"{tag}_mean"] = particles.mean_init_velocity(params)
    # an explicit key: the reference still subtracts the (seed, step 0) mean
    params = SimParams(edge_length=6, seed=5)
    for step in (0, 3):
        p = particles.init_system(params, key=rng.RngKey(seed=5, step=step))
        out[f"key_step{step}_sha"] = np.array(sha(p.positions, p.velocities))
    np.savez_compressed(os.path.join(HERE, "init_device.npz"), **out)


def make_bench_report():
    from mpcdsim import bench
    recs = [bench.BenchRecord(L=16, ranks=1, scheme="halo", steps=3, seconds=0.1 + 1e-17,
                              particles=40960, bytes_per_step=0.0, msgs_per_step=0.0,
                              max_drift=1.3e-17),
            bench.BenchRecord(L=16, ranks=2, scheme="halo", steps=3, seconds=0.07,
                              particles=40960, bytes_per_step=2.0 ** 20 / 3,
                              msgs_per_step=2.0, max_drift=2.2e-16),
            bench.BenchRecord(L=16, ranks=3, scheme="migration", steps=3, seconds=0.0,
                              particles=0, bytes_per_step=0.0, msgs_per_step=0.0,
                              max_drift=0.0, error="ConfigError: rank_dims entry 3 does not "
                              "divide 16, \"quoted\""),
            bench.BenchRecord(L=32, ranks=1, scheme="halo", steps=20, seconds=1.2345678901234,
                              particles=327680, bytes_per_step=0.0, msgs_per_step=0.0,
                              max_drift=3.5e-15),
            bench.BenchRecord(L=32, ranks=8, scheme="halo", steps=20, seconds=0.2,
                              particles=327680, bytes_per_step=123456.5, msgs_per_step=7.5,
                              max_drift=1e-300)]
    bench.emit_report(recs, os.path.join(HERE, "bench_report.csv"))
    np.save(os.path.join(HERE, "bench_rank_dims.npy"),
            np.array([bench.rank_dims_for(n) for n in range(1, 65)], dtype=np.int64))


def make_parallel(steps=5):
    """The reference's multi-rank path (engine.py:190-391 through
    runners.SequentialRunner) and its serial run, for the decomposed-box
    parity tests (its own bound vs serial: 1e-10, test_engine.py:119-126)."""
    out = {}
    cases = {"halo": ((2, 2, 1), "halo"), "migr": ((2, 1, 1), "migration")}
    for tag, (rank_dims, scheme) in cases.items():
        params = SimParams(edge_length=8, seed=3, rank_dims=rank_dims, scheme=scheme)
        sim = engine.Simulation(params, backend="sequential", capture_com=True)
        for k in range(steps):
            sim.step()
            ids, p = sim.collect()
            out[f"{tag}_ids{k}"] = ids
            out[f"{tag}_pos{k}"] = p.positions
            out[f"{tag}_vel{k}"] = p.velocities
            ci, cv = sim.com_captures[-1]
            out[f"{tag}_comids{k}"] = ci
            out[f"{tag}_com{k}"] = cv
        sim.close()
        out[f"{tag}_rank_dims"] = np.array(rank_dims)
    params = SimParams(edge_length=8, seed=3)
    sim = engine.Simulation(params, backend="serial", capture_com=True)
    for k in range(steps):
        sim.step()
        ids, p = sim.collect()
        out[f"serial_pos{k}"] = p.positions
        out[f"serial_vel{k}"] = p.velocities
    out["steps"] = np.array(steps)
    np.savez_compressed(os.path.join(HERE, "parallel_L8.npz"), **out)


def make_decomposition():
    from mpcdsim import decomposition as dec

    out = {}
    rs = np.random.default_rng(99)
    cases = [(8, 1.0, (2, 2, 2)), (12, 0.5, (3, 2, 1)), (6, 2.0, (1, 3, 2)), (4, 1.0, (1, 1, 1))]
    for i, (L, a, rd) in enumerate(cases):
        g = dec.build_decomposition(L, a, rd)
        out[f"c{i}_own"] = g.own_cells
        out[f"c{i}_table"] = g.neighbor_table
        out[f"c{i}_borders"] = np.array([g.dom_borders(r) for r in range(g.n_ranks)])
        out[f"c{i}_coords"] = np.array([g.rank_coords(r) for r in range(g.n_ranks)])
        gc = rs.integers(-2 * L, 3 * L, size=(50, 3))
        out[f"c{i}_gc"] = gc
        out[f"c{i}_flat"] = g.global_flat_cells(gc)
        box = L * a
        pos = rs.uniform(-0.2 * box, 1.2 * box, size=(400, 3))
        pos[:40] = np.round(pos[:40] / (a * g.own_cells)) * (a * g.own_cells)  # on borders
        out[f"c{i}_pos"] = pos
        out[f"c{i}_codes"] = np.array([dec.classify_base3(pos, g.dom_borders(r))
                                       for r in range(g.n_ranks)])
    out["digits"] = dec.code_digits(np.arange(27))
    out["reflect"] = np.array([dec.reflect_code(c) for c in range(27)])
    np.savez_compressed(os.path.join(HERE, "decomposition.npz"), **out)


if __name__ == "__main__":
    print("numpy", np.__version__, "reference", REF_SRC)
    make_rng()
    make_collision()
    make_serial_small()
    make_config1()
    make_config2()
    make_init_device()
    make_bench_report()
    make_parallel()
    make_decomposition()
    with open(os.path.join(HERE, "PROVENANCE.txt"), "w") as f:
        f.write(f"generated by tests/golden/make_golden.py from {REF_SRC}\n")
        f.write(f"numpy {np.__version__}, python {sys.version.split()[0]}\n")
    for fn in sorted(os.listdir(HERE)):
        print(fn, os.path.getsize(os.path.join(HERE, fn)))
