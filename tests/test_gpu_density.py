"""Densities and clusters the reference accepts (params.py:61-62: any
mean_density > 0; collision.py:93-109 bins any occupancy), engine vs the CPU
oracle bit for bit.

The tile size of k_step follows the density (16, 8 or 4 cells per tile, see
mpcd_ctx_create); tiles that still do not fit (overflowing cells, clusters)
take the dense-tile path.  These tests cover each geometry, the dense path
at scale (overflow buckets, HBM staging) and its capacity error.

Run on a B200: python -m pytest tests -m gpu
"""

import os

import numpy as np
import pytest

import oracle
import paper_2212_11878_b200 as mp
from paper_2212_11878_b200 import engine

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    oracle.set_threads(os.cpu_count() or 1)


def _oracle_steps(pos, vel, mass, dims, params, first, steps):
    cs, sn = float(np.cos(params.alpha)), float(np.sin(params.alpha))
    for k in range(first, first + steps):
        r = oracle.serial_step(pos, vel, mass, dims, params.cell_size, params.dt, cs, sn,
                               params.seed, k, prng=params.prng)
        pos, vel = r.positions, r.velocities
    return pos, vel


def expected_tile_cells(density, max_cells=32):
    """mpcd_ctx_create's rule: the largest multiple of 4 cells whose padded
    tile fits the 256 staging slots with 2.5 standard deviations to spare."""
    import math
    for tc in range(max_cells, 4, -4):
        if tc * (density + 1.5) + 2.5 * math.sqrt(tc * density) <= 256:
            return tc
    return 4


@pytest.mark.parametrize("L", [64, 128])
@pytest.mark.parametrize("density", [4, 15, 20, 30])
def test_density_matches_oracle(L, density):
    """64^3 and 128^3 boxes (128^3 x 30 = 62.9 M particles) at 4-30 particles
    per cell: resident engine == oracle after 3 steps, bitwise."""
    import torch

    params = mp.SimParams(edge_length=L, seed=11 + density, mean_density=density)
    sim = mp.Simulation(params, backend="cuda", init="device", capture_drift=True)
    try:
        assert sim.runner.ctx.tile_cells == expected_tile_cells(density)
        ids0, p0 = sim.collect()
        assert ids0.size == params.n_particles
        steps = 3 if L == 64 else 2
        sim.run(steps)
        d = sim.diagnostics[-1]
        assert d["n"] == params.n_particles
        assert max(sim.drift_history) < 1e-10
        ids, p = sim.collect()
    finally:
        sim.close()
        torch.cuda.empty_cache()
    pos, vel = _oracle_steps(p0.positions, p0.velocities, np.ones(p0.n), L, params, 0, steps)
    assert np.array_equal(ids, ids0)
    assert np.array_equal(p.positions, pos)
    assert np.array_equal(p.velocities, vel)


@pytest.mark.parametrize("tc", ["32", "20", "16", "12", "8", "4"])
def test_tile_geometry_does_not_change_results(tc, monkeypatch):
    """Any tile size gives the same trajectory (the geometry is a schedule,
    not part of the numerics): forced 32/20/16/12/8/4-cell tiles at 10 per
    cell (32 and 20 send many tiles to the dense kernel)."""
    monkeypatch.setenv("MPCD_TILE_CELLS", tc)
    params = mp.SimParams(edge_length=32, seed=4)
    sim = mp.Simulation(params, backend="cuda", init="device")
    try:
        assert sim.runner.ctx.tile_cells == int(tc)
        _, p0 = sim.collect()
        sim.run(4)
        _, p = sim.collect()
    finally:
        sim.close()
    pos, vel = _oracle_steps(p0.positions, p0.velocities, np.ones(p0.n), 32, params, 0, 4)
    assert np.array_equal(p.positions, pos) and np.array_equal(p.velocities, vel)


def test_very_high_density_dense_path():
    """60 per cell: cells above the fast path's 64 padded slots, so nearly
    every tile takes the dense kernel (shared-memory staging)."""
    params = mp.SimParams(edge_length=24, seed=2, mean_density=60)
    sim = mp.Simulation(params, backend="cuda", init="device")
    try:
        _, p0 = sim.collect()
        sim.run(3)
        _, p = sim.collect()
    finally:
        sim.close()
    pos, vel = _oracle_steps(p0.positions, p0.velocities, np.ones(p0.n), 24, params, 0, 3)
    assert np.array_equal(p.positions, pos) and np.array_equal(p.velocities, vel)


def _blob_state(L, n, frac, sigma, seed):
    rs = np.random.default_rng(seed)
    nb = int(n * frac)
    centre = np.array([0.37, 0.52, 0.61]) * L
    blob = np.mod(centre + rs.normal(scale=sigma, size=(nb, 3)), float(L))
    rest = rs.uniform(0.0, float(L), size=(n - nb, 3))
    pos = np.concatenate([blob, rest])
    pos[pos >= L] = 0.0
    vel = rs.normal(size=(n, 3))
    return pos, vel


def test_blob_128cubed_matches_oracle():
    """128^3 x 10 with 10 % of the particles (2.1 M) in one Gaussian blob
    (sigma 3 cells, ~5000 particles in the central cells): overflowing cells,
    dense tiles staged in HBM, overflow buckets -- bitwise vs the oracle,
    with the diagnostics conserved."""
    import torch

    L = 128
    params = mp.SimParams(edge_length=L, seed=31)
    n = params.n_particles
    pos, vel = _blob_state(L, n, 0.10, 3.0, 5)
    vel -= vel.mean(axis=0)
    sim = mp.Simulation(params, backend="cuda", init="device", capture_drift=True)
    try:
        sim.runner.ctx.upload(pos, vel, None, None, 0)
        sim.run(2)
        d = sim.diagnostics[-1]
        assert d["n"] == n
        assert np.abs(d["momentum"]).max() < 1e-6
        ids, p = sim.collect()
    finally:
        sim.close()
        torch.cuda.empty_cache()
    rpos, rvel = _oracle_steps(pos, vel, np.ones(n), L, params, 0, 2)
    assert np.array_equal(ids, np.arange(n))
    assert np.array_equal(p.positions, rpos)
    assert np.array_equal(p.velocities, rvel)


def test_blob_deterministic_diagnostics():
    """Dense tiles arrive in the queue in any order; the diagnostics are
    reduced per tile in tile order, so two runs agree bit for bit."""
    L = 48
    params = mp.SimParams(edge_length=L, seed=8)
    pos, vel = _blob_state(L, params.n_particles, 0.15, 2.0, 9)
    out = []
    for _ in range(2):
        sim = mp.Simulation(params, backend="cuda", init="device", capture_drift=True)
        try:
            sim.runner.ctx.upload(pos, vel, None, None, 0)
            sim.run(3)
            out.append([(d["momentum"].tobytes(), d["energy"], d["max_cell_drift"])
                        for d in sim.diagnostics])
        finally:
            sim.close()
    assert out[0] == out[1]


def test_pure_step_blob_matches_oracle():
    """serial_collision_step (the reference's pure function) on clustered input."""
    L = 16
    params = mp.SimParams(edge_length=L, seed=12, mean_density=12)
    n = params.n_particles
    pos, vel = _blob_state(L, n, 0.5, 0.8, 2)
    p = mp.ParticleSet(pos, vel, np.ones(n))
    rpos, rvel = pos, vel
    for k in range(3):
        p, drift, _ = mp.serial_collision_step(p, params, k, want_drift=True)
        rpos, rvel = _oracle_steps(rpos, rvel, np.ones(n), L, params, k, 1)
        assert np.array_equal(p.positions, rpos) and np.array_equal(p.velocities, rvel), k
        assert drift < 1e-10


def test_cluster_beyond_capacity_fails_loudly():
    """Every particle in one cell (2 M particles, far beyond the overflow
    lists' n/4 entries) is MPCD_ERR_CAPACITY, and the context refuses to
    step until the state is uploaded again -- never silent corruption."""
    L = 64
    n = 1 << 21
    ctx = engine.EngineContext((L, L, L), 1.0, 0.1, np.radians(130.0), 1, "splitmix", n,
                               mass_value=1.0)
    try:
        vel = np.random.default_rng(0).normal(size=(n, 3))
        with pytest.raises(mp.MpcdError):
            ctx.upload(np.full((n, 3), 3.5), vel, None, None, 0)
        with pytest.raises(mp.MpcdError):
            ctx.step(0)
        ok = np.random.default_rng(1).uniform(0, L, size=(n, 3))
        ctx.upload(ok, vel, None, None, 0)
        ctx.step(0)
        assert ctx.read_diag().n == n
    finally:
        ctx.close()


def test_upload_rejects_bad_ids():
    """ids outside 0..n-1 (or repeated) on a whole-box context are a
    ConfigError, not an out-of-bounds device write at download."""
    n = 64
    ctx = engine.EngineContext((4, 4, 4), 1.0, 0.1, 1.0, 1, "splitmix", n, mass_value=1.0)
    try:
        rs = np.random.default_rng(0)
        pos, vel = rs.uniform(0, 4, size=(n, 3)), rs.normal(size=(n, 3))
        for bad in (np.arange(n) + 1, np.zeros(n, np.int64), np.arange(n) - 1):
            with pytest.raises(mp.ConfigError):
                ctx.upload(pos, vel, None, bad, 0)
        perm = rs.permutation(n)
        ctx.upload(pos, vel, None, perm, 0)
        ids, p = ctx.download(id_order=True)
        assert np.array_equal(ids, np.arange(n))
        assert np.array_equal(p.positions[perm], pos)
    finally:
        ctx.close()


def test_cell_beyond_dense_ranking_limit_fails_loudly():
    """70,000 particles in one cell (above k_step_dense's 65,536 ranking
    limit, mpcd_step.cuh kDenseMaxCell): MPCD_ERR_CAPACITY rather than an
    O(k^2) stall; a sane state steps again after a fresh upload."""
    n = 70_000
    L = 16
    ctx = engine.EngineContext((L, L, L), 1.0, 0.1, np.radians(130.0), 1, "splitmix", 4 * n,
                               mass_value=1.0)
    try:
        vel = np.random.default_rng(0).normal(size=(n, 3))
        with pytest.raises(mp.MpcdError, match="ranking limit"):
            ctx.upload(np.full((n, 3), 3.5), vel, None, None, 0)
            ctx.step(0)
            ctx.read_diag()
        ok = np.random.default_rng(1).uniform(0, L, size=(n, 3))
        ctx.upload(ok, vel, None, None, 0)
        ctx.step(0)
        assert ctx.read_diag().n == n
    finally:
        ctx.close()
