"""Host-side logic of the package (no GPU): parameters, the numpy mirror of
the keyed RNG, initial conditions, errors -- against the reference's golden
vectors and the reference's own test expectations (test_particles.py,
test_rng.py, params.py)."""

import hashlib
import math

import numpy as np
import pytest

import paper_2212_11878_b200 as mp
from paper_2212_11878_b200 import rng


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def test_key_state_and_uniform_match_reference(g_rng):
    for k, want in zip(g_rng["ks_in"], g_rng["ks_out"]):
        assert int(rng.key_state(*(int(x) for x in k))) == int(want)
    for s, i, want in zip(g_rng["ua_state"], g_rng["ua_idx"], g_rng["ua_out"]):
        assert float(rng.uniform_at(np.uint64(s), np.uint64(i))) == want
    got = rng.gaussian_at(rng.key_state(11, 0, rng.Purpose.INIT, 0), np.arange(1000, dtype=np.uint64))
    assert np.array_equal(got, g_rng["gauss"])


def test_vector_keys_match_scalar():
    cells = np.array([0, 1, 99, 2 ** 40], dtype=np.int64)
    states = rng.key_state(5, 2, rng.Purpose.AXIS, cells)
    for i, c in enumerate(cells):
        assert states[i] == rng.key_state(5, 2, rng.Purpose.AXIS, int(c))


def test_rng_key_validation():
    with pytest.raises(ValueError):
        mp.RngKey(seed=-1)
    with pytest.raises(ValueError):
        mp.RngKey(seed=2 ** 64)


def test_init_system_bitexact_with_reference(g_config1, g_serial):
    p = mp.init_system(mp.SimParams(edge_length=16, seed=42))
    assert sha(p.positions, p.velocities) == str(g_config1["init_sha"])
    q = mp.init_system(mp.SimParams(edge_length=4, seed=7))
    assert np.array_equal(q.positions, g_serial["L4_pos0"])
    assert np.array_equal(q.velocities, g_serial["L4_vel0"])


def test_init_properties():
    params = mp.SimParams(edge_length=4, mean_density=7.0)
    p = mp.init_system(params)
    assert p.n == params.n_particles == round(4 ** 3 * 7.0)
    assert np.all(p.positions >= 0.0) and np.all(p.positions < params.box_length)
    assert np.all(p.masses == 1.0)
    p6 = mp.init_system(mp.SimParams(edge_length=6))
    assert np.abs(mp.total_momentum(p6)).max() < 1e-10 * p6.n
    p1 = mp.init_system(mp.SimParams(edge_length=8), velocity_variance=1.0)
    p4 = mp.init_system(mp.SimParams(edge_length=8), velocity_variance=4.0)
    assert np.allclose(p4.velocities, 2.0 * p1.velocities)


@pytest.mark.parametrize("rank_dims", [(2, 1, 1), (2, 2, 2), (4, 2, 1)])
def test_owned_slice_matches_full_init(rank_dims):
    params = mp.SimParams(edge_length=4, mean_density=6.0, rank_dims=rank_dims)
    full = mp.init_system(params)
    box = params.box_length
    seen = 0
    for rx in range(rank_dims[0]):
        for ry in range(rank_dims[1]):
            for rz in range(rank_dims[2]):
                lower = np.array([rx, ry, rz]) * box / np.array(rank_dims)
                upper = lower + box / np.array(rank_dims)
                ids, owned = mp.init_owned_slice(params, lower, upper)
                mask = np.all((full.positions >= lower) & (full.positions < upper), axis=1)
                assert np.array_equal(ids, np.nonzero(mask)[0])
                assert np.array_equal(owned.positions, full.positions[mask])
                assert np.array_equal(owned.velocities, full.velocities[mask])
                seen += owned.n
    assert seen == full.n


def test_params_validation_matches_reference():
    with pytest.raises(mp.ConfigError):
        mp.SimParams(edge_length=0)
    with pytest.raises(mp.ConfigError):
        mp.SimParams(edge_length=4, alpha=4.0)
    with pytest.raises(mp.ConfigError):
        mp.SimParams(edge_length=4, dt=0.0)
    with pytest.raises(mp.ConfigError):
        mp.SimParams(edge_length=6, rank_dims=(4, 1, 1))
    with pytest.raises(mp.ConfigError):
        mp.SimParams(edge_length=4, scheme="nope")
    with pytest.raises(mp.ConfigError):
        mp.SimParams(edge_length=4, prng="mt19937")
    p = mp.SimParams(edge_length=4)
    assert p.n_cells == 64 and p.n_particles == 640 and p.box_length == 4.0
    assert p.alpha == math.radians(130.0)


def test_noncubic_extension():
    p = mp.SimParams(edge_length=8, edge_lengths=(8, 4, 2), rank_dims=(2, 1, 1))
    assert p.dims == (8, 4, 2) and p.n_cells == 64 and p.box_lengths == (8.0, 4.0, 2.0)
    with pytest.raises(mp.ConfigError):
        _ = p.box_length
    with pytest.raises(mp.ConfigError):
        mp.SimParams(edge_length=8, edge_lengths=(8, 3, 2), rank_dims=(1, 2, 1))
    q = mp.init_system(p)
    assert np.all(q.positions < np.array(p.box_lengths))


def test_particle_set_validation():
    with pytest.raises(ValueError):
        mp.ParticleSet(np.zeros((3, 3)), np.zeros((2, 3)), np.ones(3))
    e = mp.ParticleSet.empty()
    assert e.n == 0 and mp.kinetic_energy(e) == 0.0 and mp.total_mass(e) == 0.0


def test_errors_hierarchy():
    e = mp.BinningError("x", particle_index=3, dimension=1)
    assert isinstance(e, mp.MpcdError) and e.particle_index == 3 and e.dimension == 1
    assert issubclass(mp.TopologyError, mp.MpcdError)


def test_cuda_backend_needs_gpu_loudly():
    """No CPU fallback: without a GPU the engine refuses to run."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(mp.MpcdError):
        mp.Simulation(mp.SimParams(edge_length=4), backend="cuda")
    with pytest.raises(mp.ConfigError):
        mp.Simulation(mp.SimParams(edge_length=4), backend="threads")


def test_bench_reference_arm_runs_on_cpu():
    """bench.py --impl reference (the oracle on the host cores) prints the
    contract's JSON line without a GPU."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference",
                          "--steps", "2", "--warmup", "1", "--cpu-sample-L", "8"],
                         capture_output=True, text=True, timeout=300, check=True).stdout
    line = json.loads(out.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["metric"] == "MPCD particle-steps/sec" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_init_system_explicit_key_matches_reference():
    """init_system(params, key) subtracts the (params.seed, step 0) mean, as
    the reference does (particles.py:101-127), for any key step."""
    import hashlib

    from conftest import golden
    g = golden("init_device.npz")
    params = mp.SimParams(edge_length=6, seed=5)
    for step in (0, 3):
        p = mp.init_system(params, key=mp.RngKey(seed=5, step=step))
        h = hashlib.sha256()
        for a in (p.positions, p.velocities):
            h.update(np.ascontiguousarray(a).tobytes())
        assert h.hexdigest() == str(g[f"key_step{step}_sha"]), step


def test_lazy_policy_and_scheme_a_warn_as_aliases():
    """policy='lazy' and scheme='migration' run the cell-ownership
    decomposition: documented aliases that warn, never silently accepted."""
    import warnings

    from paper_2212_11878_b200 import engine
    dec = mp.SimParams(edge_length=8, rank_dims=(2, 1, 1), scheme="migration")
    with pytest.warns(mp.DecompositionAliasWarning) as rec:
        engine._warn_aliases(dec, "lazy")
    assert len(rec) == 2
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        engine._warn_aliases(mp.SimParams(edge_length=8, rank_dims=(2, 1, 1)), "immediate")
        engine._warn_aliases(mp.SimParams(edge_length=8, scheme="migration"), "lazy")
