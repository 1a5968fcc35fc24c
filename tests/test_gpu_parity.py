"""GPU parity: every stage and the full step vs the reference's golden
vectors (bit-exact) and vs the CPU oracle on seeded inputs.

Run on a B200: python -m pytest tests -m gpu
"""

import hashlib
import os

import numpy as np
import pytest

import oracle
import paper_2212_11878_b200 as mp
from paper_2212_11878_b200 import engine

pytestmark = pytest.mark.gpu


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


# ---------------------------------------------------------------- stages ---
def test_grid_shift_and_axes_match_reference(g_rng):
    for seed, rows in zip(g_rng["shift_seeds"], g_rng["shifts"]):
        got = np.array([mp.sample_grid_shift(s, int(seed)).offset for s in range(rows.shape[0])])
        assert np.array_equal(got, rows)
    got = np.array([mp.sample_grid_shift(s, 9, 2.5).offset for s in range(50)])
    assert np.array_equal(got, g_rng["shifts_a25"])
    assert np.array_equal(mp.sample_rotation_axes(7, g_rng["axes_ids"], 42), g_rng["axes"])
    assert np.array_equal(mp.sample_rotation_axes(5, g_rng["axes_sparse_ids"], 11),
                          g_rng["axes_sparse"])
    su = mp.sample_uniform(mp.RngKey(seed=42, step=7, purpose=mp.Purpose.AXIS, cell_id=123), 64)
    assert np.array_equal(su, g_rng["sample_uniform"])


@pytest.mark.parametrize("kind", ["minstd", "pcg32", "sfc64"])
def test_keyed_prng_streams_match_oracle(kind):
    key = mp.RngKey(seed=42, step=3, purpose=mp.Purpose.AXIS, cell_id=77)
    got = mp.sample_uniform(key, 1000, prng=kind)
    want = oracle.sample_uniform(kind, 42, 3, oracle.AXIS, 77, 1000)
    assert np.array_equal(got, want)
    ids = np.arange(5000)
    assert np.array_equal(mp.sample_rotation_axes(9, ids, 42, prng=kind),
                          oracle.rotation_axes(9, ids, 42, prng=kind))
    for s in range(20):
        assert np.array_equal(mp.sample_grid_shift(s, 42, 1.0, kind).offset,
                              oracle.grid_shift(s, 42, 1.0, kind))


@pytest.mark.parametrize("case", list("ABCDEF"))
def test_binning_and_moments_match_reference(g_collision, case):
    g = g_collision
    dims = g[f"{case}_dims"]
    a = float(g[f"{case}_a"])
    gmin = g[f"{case}_gmin"]
    lc = mp.build_linked_cells(g[f"{case}_pos"], a, gmin, gmin + dims * a, wrap=g[f"{case}_wrap"])
    assert np.array_equal(lc.cells, g[f"{case}_cells"])
    assert np.array_equal(lc.bin_count, g[f"{case}_counts"])
    assert np.array_equal(lc.bin_offset, g[f"{case}_offsets"])
    assert np.array_equal(lc.permutation, g[f"{case}_perm"])
    mom = mp.segment_moments(lc, g[f"{case}_vel"], g[f"{case}_mass"])
    assert np.array_equal(mom, g[f"{case}_moments"])
    assert np.array_equal(mp.finalize_com(mp.CellMomentField(mom)), g[f"{case}_com"])
    alt = mp.linked_cells_from_indices(lc.cells, dims, gmin, gmin + dims * a, a, lc.wrap)
    assert np.array_equal(alt.permutation, lc.permutation)


def test_binning_error_matches_reference(g_collision):
    with pytest.raises(mp.BinningError) as info:
        mp.build_linked_cells(g_collision["err_pos"], 1.0, np.zeros(3), np.full(3, 2.0))
    assert [info.value.particle_index, info.value.dimension] == list(g_collision["err_info"])
    with pytest.raises(mp.BinningError):
        mp.linked_cells_from_indices(np.array([0, 8]), (2, 2, 2), np.zeros(3), np.full(3, 2.0),
                                     1.0, (False,) * 3)


@pytest.mark.parametrize("tag", ["r1", "r130", "rq"])
def test_rotation_matches_reference(g_collision, tag):
    g = g_collision
    got = mp.rotate_velocities(g["rot_vel"], g["rot_com"], g["rot_axes"], float(g[f"{tag}_alpha"]))
    assert np.array_equal(got, g[f"{tag}_out"])


def test_wrap_and_stream_match_reference(g_collision):
    g = g_collision
    got = mp.wrap_coordinates(g["wrap_x"], 8.0)
    assert np.array_equal(got, g["wrap_out"])
    assert np.array_equal(np.signbit(got), np.signbit(g["wrap_out"]))
    p = mp.ParticleSet(g["stream_pos"], g["stream_vel"], np.ones(3000))
    assert np.array_equal(mp.stream_and_wrap(p, 0.7, 8.0).positions, g["stream_out"])


def test_drift_metric_values():
    before = np.array([[1.0, 0.0, 0.0, 2.0], [0.0, 0.0, 0.0, 0.0]])
    assert mp.cell_momentum_drift(before, before) == 0.0
    bumped = before.copy()
    bumped[0, 0] += 0.5
    assert mp.cell_momentum_drift(before, bumped) == pytest.approx(0.25)
    assert mp.cell_momentum_drift(np.zeros((4, 4)), np.zeros((4, 4))) == 0.0


# -------------------------------------------------------- the full step ---
@pytest.mark.parametrize("tag", ["L4", "L6", "M4", "B5"])
def test_pure_step_matches_reference(g_serial, tag):
    """serial_collision_step (GPU) == reference, every intermediate, bitwise."""
    g = g_serial
    params = mp.SimParams(edge_length=int(g[f"{tag}_L"]), seed=int(g[f"{tag}_seed"]),
                          dt=float(g[f"{tag}_dt"]), alpha=float(g[f"{tag}_alpha"]))
    assert float(np.cos(params.alpha)) == float(g[f"{tag}_cos"])
    p = mp.ParticleSet(g[f"{tag}_pos0"], g[f"{tag}_vel0"], g[f"{tag}_mass"])
    for k in range(int(g[f"{tag}_steps"])):
        p, drift, (occ, com) = mp.serial_collision_step(p, params, k, want_drift=True,
                                                        want_com=True)
        assert np.array_equal(p.positions, g[f"{tag}_pos{k + 1}"]), k
        assert np.array_equal(p.velocities, g[f"{tag}_vel{k + 1}"]), k
        assert np.array_equal(occ, g[f"{tag}_occ{k}"])
        assert np.array_equal(com, g[f"{tag}_com{k}"])
        assert drift == pytest.approx(float(g[f"{tag}_drift{k}"]), rel=1e-6, abs=1e-15)


def _sim_from_state(params, pos, vel, **kw):
    sim = mp.Simulation(params, backend="cuda", **kw)
    sim.runner.ctx.upload(pos, vel, None, None, 0)
    return sim


def test_config1_engine_100_steps_bitexact(g_config1):
    """BASELINE config 1 through the resident engine: binning (cells, counts,
    permutation) and state hashes equal the reference at every step."""
    g = g_config1
    params = mp.SimParams(edge_length=16, seed=int(g["seed"]), dt=float(g["dt"]))
    assert float(np.cos(params.alpha)) == float(g["cos"])
    sim = _sim_from_state(params, g["pos0"], g["vel0"], capture_drift=True)
    ctx = sim.runner.ctx
    try:
        for k in range(int(g["steps"])):
            cells, counts, offsets, perm = ctx.read_binning()
            assert sha(cells, counts, perm) == str(g["bin_sha"][k]), k
            d = sim.step()
            ids, p = sim.collect()
            assert np.array_equal(ids, np.arange(p.n))
            assert sha(p.positions, p.velocities) == str(g["state_sha"][k]), k
            ref = g["diag"][k]
            assert np.allclose(d["momentum"], ref[:3], atol=1e-10)
            assert d["energy"] == pytest.approx(ref[3], rel=1e-12)
            assert d["mass"] == ref[4]
            assert d["max_cell_drift"] == pytest.approx(ref[5], rel=1e-3, abs=1e-15)
        assert np.array_equal(p.positions, g["pos_final"])
    finally:
        sim.close()


def test_host_init_matches_reference(g_config1):
    p = mp.init_system(mp.SimParams(edge_length=16, seed=42))
    assert sha(p.positions, p.velocities) == str(g_config1["init_sha"])


def _oracle_run(pos, vel, mass, dims, params, steps, start=0):
    cs, sn = float(np.cos(params.alpha)), float(np.sin(params.alpha))
    for k in range(start, start + steps):
        r = oracle.serial_step(pos, vel, mass, dims, params.cell_size, params.dt, cs, sn,
                               params.seed, k, prng=params.prng)
        pos, vel = r.positions, r.velocities
    return pos, vel


@pytest.mark.parametrize("prng", ["splitmix", "minstd", "pcg32", "sfc64"])
def test_engine_64cubed_matches_oracle(prng):
    """Config 2: 64^3 x 10 (2.6M particles), each PRNG, 4 steps bitwise."""
    params = mp.SimParams(edge_length=64, seed=1, prng=prng)
    sim = mp.Simulation(params, backend="cuda", init="device")
    try:
        ids, p0 = sim.collect()
        sim.run(4)
        ids, p = sim.collect()
    finally:
        sim.close()
    pos, vel = _oracle_run(p0.positions, p0.velocities, np.ones(p0.n), 64, params, 4)
    assert np.array_equal(p.positions, pos)
    assert np.array_equal(p.velocities, vel)


def test_config2_reference_hashes():
    """64^3 seed 0 against the reference's own trajectory hashes."""
    from conftest import golden
    g = golden("config2_L64.npz")
    params = mp.SimParams(edge_length=64, seed=0)
    p = mp.init_system(params)
    if sha(p.positions, p.velocities) != str(g["init_sha"]):
        pytest.skip("host numpy transcendental results differ from the fixture host")
    sim = _sim_from_state(params, p.positions, p.velocities)
    try:
        for k in range(int(g["steps"])):
            cells, counts, offsets, perm = sim.runner.ctx.read_binning()
            assert sha(cells, counts, perm) == str(g["bin_sha"][k])
            sim.step()
            _, q = sim.collect()
            assert sha(q.positions, q.velocities) == str(g["state_sha"][k])
    finally:
        sim.close()


def test_noncubic_box_matches_oracle():
    params = mp.SimParams(edge_length=24, edge_lengths=(24, 16, 8), seed=5)
    sim = mp.Simulation(params, backend="cuda")
    try:
        _, p0 = sim.collect()
        sim.run(5)
        _, p = sim.collect()
    finally:
        sim.close()
    pos, vel = _oracle_run(p0.positions, p0.velocities, np.ones(p0.n), [24, 16, 8], params, 5)
    assert np.array_equal(p.positions, pos) and np.array_equal(p.velocities, vel)


def test_dense_cells_overflow_path():
    """Tiles far above the shared-memory capacity (clustered particles)."""
    rs = np.random.default_rng(3)
    n = 6000
    pos = np.concatenate([rs.uniform(2.0, 2.9, size=(5000, 3)), rs.uniform(0, 8, size=(1000, 3))])
    vel = rs.normal(size=(n, 3))
    params = mp.SimParams(edge_length=8, seed=9, mean_density=n / 512)
    p = mp.ParticleSet(pos, vel, np.ones(n))
    ref_pos, ref_vel = pos, vel
    for k in range(4):
        p, drift, _ = mp.serial_collision_step(p, params, k, want_drift=True)
        ref_pos, ref_vel = _oracle_run(ref_pos, ref_vel, np.ones(n), 8, params, 1, start=k)
        assert np.array_equal(p.positions, ref_pos) and np.array_equal(p.velocities, ref_vel), k
        assert drift < 1e-12


def test_empty_and_tiny_systems():
    params = mp.SimParams(edge_length=4, seed=1)
    p = mp.ParticleSet.empty()
    out, drift, com = mp.serial_collision_step(p, params, 0, want_drift=True, want_com=True)
    assert out.n == 0 and drift == 0.0 and com[0].size == 0
    one = mp.ParticleSet(np.array([[0.5, 1.5, 3.99]]), np.array([[1.0, -2.0, 0.5]]), np.ones(1))
    out, _, _ = mp.serial_collision_step(one, params, 3)
    ref_pos, ref_vel = _oracle_run(one.positions, one.velocities, np.ones(1), 4, params, 1, 3)
    assert np.array_equal(out.positions, ref_pos) and np.array_equal(out.velocities, ref_vel)


def test_conservation_and_determinism():
    params = mp.SimParams(edge_length=16, seed=3)
    a = mp.Simulation(params, backend="cuda", capture_drift=True)
    b = mp.Simulation(params, backend="cuda", capture_drift=True)
    try:
        r0 = a.conservation_report()
        a.run(50)
        b.run(50)
        r1 = a.conservation_report()
        assert r1.n_particles == r0.n_particles and r1.total_mass == r0.total_mass
        assert np.abs(r1.total_momentum - r0.total_momentum).max() < 1e-10
        assert abs(r1.kinetic_energy - r0.kinetic_energy) < 1e-9 * r0.kinetic_energy
        assert max(a.drift_history) < 1e-10
        ia, pa = a.collect()
        ib, pb = b.collect()
        assert np.array_equal(pa.positions, pb.positions)
        assert np.array_equal(pa.velocities, pb.velocities)
        assert [d["momentum"].tobytes() for d in a.diagnostics] == \
               [d["momentum"].tobytes() for d in b.diagnostics]
    finally:
        a.close()
        b.close()


def test_galilean_boost():
    """Acceptance criterion 8 (test_acceptance.py:251-268) on the GPU step."""
    w = np.array([1.0, 2.0, 3.0])
    params = mp.SimParams(edge_length=8, dt=8.0, seed=3)
    base = mp.init_system(params)
    boosted = mp.ParticleSet(base.positions.copy(), base.velocities + w, base.masses.copy())
    for step in range(20):
        base, _, _ = mp.serial_collision_step(base, params, step)
        boosted, _, _ = mp.serial_collision_step(boosted, params, step)
    assert np.abs(boosted.velocities - w - base.velocities).max() < 1e-9


def test_advance_equals_step_loop():
    params = mp.SimParams(edge_length=12, seed=8)
    a = mp.Simulation(params, backend="cuda")
    b = mp.Simulation(params, backend="cuda")
    try:
        a.run(7)
        b.advance(7)
        _, pa = a.collect()
        _, pb = b.collect()
        assert np.array_equal(pa.positions, pb.positions)
        assert np.array_equal(pa.velocities, pb.velocities)
    finally:
        a.close()
        b.close()


def test_pure_step_pinned_buffers_equal_pageable():
    """mpcd_step_host reads/writes pinned host rows in place (zero-copy) and
    stages pageable ones: both must give the oracle's step bit for bit."""
    import torch

    params = mp.SimParams(edge_length=12, seed=21)
    p = mp.init_system(params)
    n = p.n
    ctx = engine.EngineContext(params.dims, 1.0, params.dt, params.alpha, params.seed,
                               "splitmix", n, mass_value=1.0)
    try:
        pos_t = torch.empty((n, 3), dtype=torch.float64, pin_memory=True)
        vel_t = torch.empty((n, 3), dtype=torch.float64, pin_memory=True)
        pin_pos, pin_vel = pos_t.numpy(), vel_t.numpy()
        pin_pos[:] = p.positions
        pin_vel[:] = p.velocities
        pag_pos, pag_vel = p.positions.copy(), p.velocities.copy()
        ref_pos, ref_vel = p.positions, p.velocities
        cs, sn = float(np.cos(params.alpha)), float(np.sin(params.alpha))
        for k in range(3):
            ctx.step_host(pin_pos, pin_vel, None, k, False)
            ctx.step_host(pag_pos, pag_vel, None, k, False)
            r = oracle.serial_step(ref_pos, ref_vel, np.ones(n), 12, 1.0, params.dt, cs, sn,
                                   params.seed, k)
            ref_pos, ref_vel = r.positions, r.velocities
            assert np.array_equal(pin_pos, ref_pos) and np.array_equal(pin_vel, ref_vel)
            assert np.array_equal(pag_pos, ref_pos) and np.array_equal(pag_vel, ref_vel)
    finally:
        ctx.close()


def test_determinism_at_256cubed():
    """BASELINE config 3 scale (167.8 M particles, overflow cells and dense
    tiles included): two runs give bitwise-identical diagnostics and state
    hashes, although slot order inside the cell regions is atomic arrival
    order."""
    import torch

    params = mp.SimParams(edge_length=256, seed=3)
    out = []
    for _ in range(2):
        ctx = engine.EngineContext(params.dims, 1.0, params.dt, params.alpha, params.seed,
                                   "splitmix", params.n_particles, mass_value=1.0)
        try:
            ctx.init_device(params.n_particles, 1.0, 0)
            ctx.run(0, 4)
            d = ctx.read_diag()
            diag = (tuple(d.momentum), d.energy, d.mass, d.n)
            ids, p = ctx.download(id_order=True)
            out.append((diag, sha(p.positions[::997], p.velocities[::997]), ids[::997].sum()))
            del ids, p
        finally:
            ctx.close()
            torch.cuda.empty_cache()
    assert out[0] == out[1]
    assert out[0][0][3] == params.n_particles


def test_full_size_step_bitexact_vs_oracle():
    """BASELINE config 3 at full size (256^3 cells, 167.8 M particles): one
    engine step from a device-initialised state equals the oracle's step of
    the same state bit for bit (positions, velocities; id order)."""
    import os

    import torch

    params = mp.SimParams(edge_length=256, seed=0)
    n = params.n_particles
    ctx = engine.EngineContext(params.dims, 1.0, params.dt, params.alpha, params.seed,
                               "splitmix", n, mass_value=1.0)
    try:
        ctx.init_device(n, 1.0, 0)
        ids0, p0 = ctx.download(id_order=True)
        assert np.array_equal(ids0, np.arange(n))
        del ids0
        ctx.step(0)
        ids1, p1 = ctx.download(id_order=True)
    finally:
        ctx.close()
        torch.cuda.empty_cache()
    oracle.set_threads(os.cpu_count() or 1)
    cs, sn = float(np.cos(params.alpha)), float(np.sin(params.alpha))
    r = oracle.serial_step(p0.positions, p0.velocities, np.ones(n), 256, 1.0, params.dt, cs, sn,
                           params.seed, 0)
    assert np.array_equal(p1.positions, r.positions)
    assert np.array_equal(p1.velocities, r.velocities)


def _ulp(x):
    x = np.abs(np.asarray(x, dtype=np.float64))
    return np.spacing(np.maximum(x, np.finfo(np.float64).tiny))


@pytest.mark.parametrize("tag", ["L16", "L64"])
def test_device_init_matches_reference_init_system(tag):
    """mpcd_init_device vs the reference's init_system (particles.py:101-127):
    positions bit-exact (53-bit counter hash x box); velocities within 4 ulp
    of the particle's Box-Muller radius r = sqrt(-2 log(1 - u1)) (floored at 1).
    A draw r cos(2 pi u2) is the product of r (log, sqrt) and a cosine, whose
    device (CUDA libdevice) and numpy results may each differ by an ulp; the
    product's error is therefore ~ulp(r) |cos| + r ulp(cos) <= 2 ulp(r) plus
    its own rounding, however small |v| is.  The subtracted mean (a
    fixed-order device sum vs numpy's chunked pairwise sum) differs by a few
    ulp of itself (~1e-18).  r is recomputed here from the same counters."""
    from conftest import golden
    g = golden("init_device.npz")
    L, seed, n = int(g[f"{tag}_L"]), int(g[f"{tag}_seed"]), int(g[f"{tag}_n"])
    params = mp.SimParams(edge_length=L, seed=seed, mean_density=float(g[f"{tag}_density"]))
    assert params.n_particles == n
    ctx = engine.EngineContext(params.dims, 1.0, params.dt, params.alpha, params.seed,
                               "splitmix", n, mass_value=1.0)
    try:
        ctx.init_device(n, 1.0, 0)
        ids, p = ctx.download(id_order=True)
    finally:
        ctx.close()
    assert np.array_equal(ids, np.arange(n))
    assert sha(p.positions) == str(g[f"{tag}_pos_sha"])
    assert np.array_equal(p.positions[::1009], g[f"{tag}_pos_rows"])
    ref = g[f"{tag}_vel_rows"]
    dev = np.abs(p.velocities[::1009] - ref)
    from paper_2212_11878_b200 import rng as R
    state = R.key_state(seed, 0, R.Purpose.INIT, 0)
    rows = np.arange(n)[::1009].astype(np.uint64)
    cols = np.uint64(3 * n) + (np.uint64(3) * rows[:, None] + np.arange(3, dtype=np.uint64))
    u1 = R.uniform_at(state, cols * np.uint64(2))
    radius = np.sqrt(-2.0 * np.log(1.0 - u1))
    assert np.all(np.abs(ref) <= radius + 1e-2)  # these draws, minus the O(n^-1/2) mean
    tol = 4.0 * _ulp(np.maximum(radius, 1.0))
    stats = (f"max |dv| {dev.max():.3e}, identical {np.mean(dev == 0.0):.3f}, "
             f"max |dv|/ulp(v) {(dev / _ulp(ref)).max():.1f}")
    assert np.all(dev <= tol), stats
    assert np.mean(dev == 0.0) > 0.5, stats
    # the host init is numpy itself: bitwise
    assert sha(mp.init_system(params).positions) == str(g[f"{tag}_pos_sha"])


def test_config1_pcg32_100_steps_vs_oracle(g_config1):
    """BASELINE config 1 literally: 16^3 x 10, 130 deg, prng="pcg32", seed 42,
    100 steps through the resident engine; binning (cells, counts,
    permutation) and state equal the oracle's at every step."""
    params = mp.SimParams(edge_length=16, seed=42, prng="pcg32")
    pos, vel = g_config1["pos0"], g_config1["vel0"]
    n = pos.shape[0]
    cs, sn = float(np.cos(params.alpha)), float(np.sin(params.alpha))
    sim = _sim_from_state(params, pos, vel, capture_drift=True)
    ctx = sim.runner.ctx
    try:
        for k in range(100):
            cells, counts, offsets, perm = ctx.read_binning()
            r = oracle.serial_step(pos, vel, np.ones(n), 16, 1.0, params.dt, cs, sn, params.seed,
                                   k, prng="pcg32", want_drift=True, want_detail=True)
            assert np.array_equal(cells, r.cells), k
            assert np.array_equal(counts, r.counts), k
            assert np.array_equal(perm, r.perm), k
            d = sim.step()
            ids, p = sim.collect()
            pos, vel = r.positions, r.velocities
            assert np.array_equal(p.positions, pos), k
            assert np.array_equal(p.velocities, vel), k
            assert d["max_cell_drift"] == pytest.approx(r.drift, rel=1e-6, abs=1e-15)
    finally:
        sim.close()


def test_public_pure_step_zero_copy_chain():
    """serial_collision_step returns its rows in pooled page-locked blocks and
    reads such rows in place next call; the input is never modified, and a
    chain of calls equals the oracle bit for bit (engine.py:415-455)."""
    from paper_2212_11878_b200 import _dev

    params = mp.SimParams(edge_length=12, seed=21)
    p0 = mp.init_system(params)
    keep = p0.copy()
    assert not _dev.is_pinned(p0.positions)
    q = p0
    ref_pos, ref_vel = p0.positions, p0.velocities
    cs, sn = float(np.cos(params.alpha)), float(np.sin(params.alpha))
    for k in range(4):
        q, _, _ = mp.serial_collision_step(q, params, k)
        assert _dev.is_pinned(q.positions) and _dev.is_pinned(q.velocities)
        r = oracle.serial_step(ref_pos, ref_vel, np.ones(p0.n), 12, 1.0, params.dt, cs, sn,
                               params.seed, k)
        ref_pos, ref_vel = r.positions, r.velocities
        assert np.array_equal(q.positions, ref_pos) and np.array_equal(q.velocities, ref_vel), k
    assert np.array_equal(p0.positions, keep.positions)
    assert np.array_equal(p0.velocities, keep.velocities)
    # random masses: the staged (non-uniform) path through the same call
    m = np.random.default_rng(2).uniform(0.5, 2.0, size=p0.n)
    pm = mp.ParticleSet(p0.positions, p0.velocities, m)
    out, _, _ = mp.serial_collision_step(pm, params, 0)
    r = oracle.serial_step(p0.positions, p0.velocities, m, 12, 1.0, params.dt, cs, sn,
                           params.seed, 0)
    assert np.array_equal(out.positions, r.positions)
    assert np.array_equal(out.velocities, r.velocities)


def test_public_pure_step_pipelined_transfers():
    """Above 2 Mi rows the pure function moves pinned rows by chunked DMA (8 Mi
    rows per chunk, each binned / produced by a kernel on arrival) and checks
    the masses on a worker thread while the GPU steps with the first mass as
    its guess.  104^3 x 10 = 11.2 M rows: a full chunk plus a partial one;
    uniform masses, then non-uniform ones (the guess fails and the
    per-particle-mass path runs): the oracle's steps bit for bit."""
    params = mp.SimParams(edge_length=104, seed=5)
    p0 = mp.init_system(params)
    n = p0.n
    assert n > (1 << 23)
    oracle.set_threads(os.cpu_count() or 1)
    cs, sn = float(np.cos(params.alpha)), float(np.sin(params.alpha))
    q = p0
    ref_pos, ref_vel = p0.positions, p0.velocities
    for k in range(2):
        q, _, _ = mp.serial_collision_step(q, params, k)
        r = oracle.serial_step(ref_pos, ref_vel, np.ones(n), 104, 1.0, params.dt, cs, sn,
                               params.seed, k)
        ref_pos, ref_vel = r.positions, r.velocities
        assert np.array_equal(q.positions, ref_pos) and np.array_equal(q.velocities, ref_vel), k
    m = np.ones(n)
    m[n - 3] = 1.5  # the first mass is a wrong guess only at the very end
    out, _, _ = mp.serial_collision_step(mp.ParticleSet(p0.positions, p0.velocities, m),
                                         params, 0)
    r = oracle.serial_step(p0.positions, p0.velocities, m, 104, 1.0, params.dt, cs, sn,
                           params.seed, 0)
    assert np.array_equal(out.positions, r.positions)
    assert np.array_equal(out.velocities, r.velocities)


@pytest.mark.parametrize("mass", [2.5, 0.3])
def test_uniform_nonunit_mass_matches_oracle(mass):
    """Uniform masses other than 1 take the uniform-mass kernel with the
    mass staged as a column (its reduceat is not simply k): a chain of pure
    steps, with the drift diagnostic, equals the oracle bit for bit
    (engine.py:415-455; collision.py:190-214 for the mass-weighted com)."""
    params = mp.SimParams(edge_length=12, seed=33)
    p0 = mp.init_system(params)
    m = np.full(p0.n, mass)
    cs, sn = float(np.cos(params.alpha)), float(np.sin(params.alpha))
    q = mp.ParticleSet(p0.positions, p0.velocities, m)
    ref_pos, ref_vel = p0.positions, p0.velocities
    for k in range(3):
        q, drift, _ = mp.serial_collision_step(q, params, k, want_drift=True)
        r = oracle.serial_step(ref_pos, ref_vel, m, 12, 1.0, params.dt, cs, sn, params.seed, k,
                               want_drift=True)
        ref_pos, ref_vel = r.positions, r.velocities
        assert np.array_equal(q.positions, ref_pos) and np.array_equal(q.velocities, ref_vel), k
        assert drift == pytest.approx(r.drift, rel=1e-9, abs=1e-15)
