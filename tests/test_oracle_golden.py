"""Pin the CPU oracle against golden vectors produced by the reference itself.

The fixtures come from tests/golden/make_golden.py, which imports the
reference mpcdsim package.  Every comparison here is bit-exact
(np.array_equal), except the tolerance-level diagnostics.
"""

import hashlib

import numpy as np
import pytest

import oracle


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


# ----------------------------------------------------------------------- RNG --
def test_key_state_matches_reference(g_rng):
    for k, want in zip(g_rng["ks_in"], g_rng["ks_out"]):
        assert oracle.key_state(*(int(x) for x in k)) == int(want)


def test_uniform_at_matches_reference(g_rng):
    for s, i, want in zip(g_rng["ua_state"], g_rng["ua_idx"], g_rng["ua_out"]):
        assert oracle.uniform_at(int(s), int(i)) == want


def test_sample_uniform_matches_reference(g_rng):
    got = oracle.sample_uniform("splitmix", 42, 7, oracle.AXIS, 123, 64)
    assert np.array_equal(got, g_rng["sample_uniform"])


def test_grid_shift_matches_reference(g_rng):
    for seed, rows in zip(g_rng["shift_seeds"], g_rng["shifts"]):
        got = np.array([oracle.grid_shift(s, int(seed)) for s in range(rows.shape[0])])
        assert np.array_equal(got, rows)
    got = np.array([oracle.grid_shift(s, 9, 2.5) for s in range(50)])
    assert np.array_equal(got, g_rng["shifts_a25"])


def test_rotation_axes_match_reference(g_rng):
    assert np.array_equal(oracle.rotation_axes(7, g_rng["axes_ids"], 42), g_rng["axes"])
    assert np.array_equal(oracle.rotation_axes(5, g_rng["axes_sparse_ids"], 11),
                          g_rng["axes_sparse"])


# ------------------------------------------------------- canonical PRNG KATs --
def test_minstd_kat():
    # std::minstd_rand (a=48271, m=2^31-1), default seed 1: 10000th output
    out = oracle.prng_raw("minstd", 1, count=10000)
    assert int(out[-1]) == 399268537


def test_pcg32_kat():
    # pcg32 (XSH-RR 64/32) pcg32_srandom(42, 54) demo output
    out = oracle.prng_raw("pcg32", 42, 54, count=6)
    want = [0xA15C02B7, 0x7B47F409, 0xBA1D3330, 0x83D2F293, 0xBFA4784B, 0xCBED606E]
    assert [int(x) for x in out] == want


def test_sfc64_matches_numpy():
    bg = np.random.SFC64(0)
    st = bg.state
    st["state"]["state"] = np.array([1, 2, 3, 1], dtype=np.uint64)
    bg.state = st
    want = bg.random_raw(1000)
    got = oracle.prng_raw("sfc64", 1, 2, 3, 1, count=1000)
    assert np.array_equal(got, want)
    assert [int(x) for x in got[:3]] == [0x4, 0x1F, 0x1B000042]


@pytest.mark.parametrize("kind", ["minstd", "pcg32", "sfc64"])
def test_keyed_streams_uniform_and_distinct(kind):
    a = oracle.sample_uniform(kind, 42, 0, oracle.AXIS, 5, 20000)
    b = oracle.sample_uniform(kind, 42, 0, oracle.AXIS, 6, 20000)
    assert np.all((a >= 0) & (a < 1))
    assert abs(a.mean() - 0.5) < 0.01 and abs(a.var() - 1 / 12) < 0.005
    assert abs(np.corrcoef(a, b)[0, 1]) < 0.05
    ax = oracle.rotation_axes(3, np.arange(500), 42, prng=kind)
    assert np.allclose(np.linalg.norm(ax, axis=1), 1.0, atol=1e-12)


# ----------------------------------------------------------------- binning --
@pytest.mark.parametrize("case", list("ABCDEF"))
def test_binning_matches_reference(g_collision, case):
    g = g_collision
    cells, counts, offsets, perm = oracle.build_linked_cells(
        g[f"{case}_pos"], float(g[f"{case}_a"]), g[f"{case}_gmin"], g[f"{case}_dims"],
        g[f"{case}_wrap"])
    assert np.array_equal(cells, g[f"{case}_cells"])
    assert np.array_equal(counts, g[f"{case}_counts"])
    assert np.array_equal(offsets, g[f"{case}_offsets"])
    assert np.array_equal(perm, g[f"{case}_perm"])


def test_binning_error_matches_reference(g_collision):
    with pytest.raises(ValueError) as info:
        oracle.build_linked_cells(g_collision["err_pos"], 1.0, np.zeros(3), [2, 2, 2])
    assert list(info.value.args) == [int(x) for x in g_collision["err_info"]]


@pytest.mark.parametrize("case", list("ABCDEF"))
def test_moments_and_com_match_reference(g_collision, case):
    g = g_collision
    mom = oracle.segment_moments(g[f"{case}_perm"], g[f"{case}_counts"], g[f"{case}_offsets"],
                                 g[f"{case}_vel"], g[f"{case}_mass"])
    assert np.array_equal(mom, g[f"{case}_moments"])
    assert np.array_equal(oracle.finalize_com(mom), g[f"{case}_com"])


@pytest.mark.parametrize("tag", ["r1", "r130", "rq"])
def test_rotation_matches_reference(g_collision, tag):
    g = g_collision
    got = oracle.rotate_velocities(g["rot_vel"], g["rot_com"], g["rot_axes"],
                                   float(g[f"{tag}_cos"]), float(g[f"{tag}_sin"]))
    assert np.array_equal(got, g[f"{tag}_out"])


def test_wrap_and_stream_match_reference(g_collision):
    g = g_collision
    got = oracle.wrap_coordinates(g["wrap_x"], 8.0)
    assert np.array_equal(got, g["wrap_out"])
    assert np.array_equal(np.signbit(got), np.signbit(g["wrap_out"]))
    got = oracle.stream_and_wrap(g["stream_pos"], g["stream_vel"], 0.7, 8.0)
    assert np.array_equal(got, g["stream_out"])


# --------------------------------------------------------------- full step --
@pytest.mark.parametrize("tag", ["L4", "L6", "M4", "B5"])
def test_serial_step_matches_reference(g_serial, tag):
    g = g_serial
    L = int(g[f"{tag}_L"])
    pos, vel, mass = g[f"{tag}_pos0"], g[f"{tag}_vel0"], g[f"{tag}_mass"]
    for k in range(int(g[f"{tag}_steps"])):
        r = oracle.serial_step(pos, vel, mass, L, float(g[f"{tag}_a"]), float(g[f"{tag}_dt"]),
                               float(g[f"{tag}_cos"]), float(g[f"{tag}_sin"]),
                               int(g[f"{tag}_seed"]), k, want_drift=True, want_detail=True)
        assert np.array_equal(r.cells, g[f"{tag}_cells{k}"])
        assert np.array_equal(r.counts, g[f"{tag}_counts{k}"])
        assert np.array_equal(r.perm, g[f"{tag}_perm{k}"])
        occ = g[f"{tag}_occ{k}"]
        assert np.array_equal(np.nonzero(r.counts)[0], occ)
        assert np.array_equal(r.com[occ], g[f"{tag}_com{k}"])
        assert np.array_equal(r.positions, g[f"{tag}_pos{k + 1}"])
        assert np.array_equal(r.velocities, g[f"{tag}_vel{k + 1}"])
        assert r.drift == pytest.approx(float(g[f"{tag}_drift{k}"]), rel=1e-6, abs=1e-15)
        pos, vel = r.positions, r.velocities


def test_config1_100_steps_bitexact(g_config1):
    """BASELINE config 1: 16^3 x 10, 130 deg, seed 42, 100 steps."""
    g = g_config1
    pos, vel = g["pos0"], g["vel0"]
    assert sha(pos, vel) == str(g["init_sha"])
    mass = np.ones(pos.shape[0])
    for k in range(int(g["steps"])):
        r = oracle.serial_step(pos, vel, mass, 16, 1.0, float(g["dt"]), float(g["cos"]),
                               float(g["sin"]), int(g["seed"]), k, want_detail=True)
        assert sha(r.cells, r.counts, r.perm) == str(g["bin_sha"][k]), k
        assert sha(r.positions, r.velocities) == str(g["state_sha"][k]), k
        d = oracle.diag(r.velocities, mass)
        assert np.allclose(d[:3], g["diag"][k, :3], atol=1e-10)
        assert d[3] == pytest.approx(g["diag"][k, 3], rel=1e-12)
        assert d[4] == g["diag"][k, 4]
        pos, vel = r.positions, r.velocities
    assert np.array_equal(pos, g["pos_final"]) and np.array_equal(vel, g["vel_final"])
