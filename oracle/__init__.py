"""CPU oracle for the MPCD/SRD hot path -- TEST INFRASTRUCTURE ONLY.

ctypes bindings over ``oracle/libmpcd_oracle.so`` (built from
``oracle/mpcd_oracle.c`` by ``oracle/Makefile``), a plain-C restatement of the
reference package ``mpcdsim`` (``/root/reference/pkg/src/mpcdsim``) that is bit
exact with it under numpy 2.3.5's operation order.  Pinned against golden
vectors produced by the reference itself (``tests/golden/make_golden.py``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this package, and only as the checker / the timed CPU
baseline.  The product (``paper_2212_11878_b200``) never imports it.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmpcd_oracle.so")

PRNG_IDS = {"splitmix": 0, "minstd": 1, "pcg32": 2, "sfc64": 3}
SHIFT, AXIS, INIT = 0, 1, 2

_lib = None

_d = C.POINTER(C.c_double)
_i64 = C.POINTER(C.c_int64)
_u64 = C.POINTER(C.c_uint64)
_i32 = C.POINTER(C.c_int32)


def build() -> str:
    """Compile the oracle shared library (make -C oracle)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.orc_key_state.restype = C.c_uint64
        L.orc_key_state.argtypes = [C.c_uint64] * 4
        L.orc_uniform_at.restype = C.c_double
        L.orc_uniform_at.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_prng_raw.argtypes = [C.c_int] + [C.c_uint64] * 4 + [C.c_int64, _u64]
        L.orc_sample_uniform.argtypes = [C.c_int] + [C.c_uint64] * 4 + [C.c_int64, _d]
        L.orc_grid_shift.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_double, _d]
        L.orc_rotation_axes.restype = C.c_int
        L.orc_rotation_axes.argtypes = [C.c_int, C.c_uint64, C.c_uint64, _i64, C.c_int64, _d]
        L.orc_wrap.argtypes = [C.c_int64, _d, C.c_double, _d]
        L.orc_build_linked_cells.restype = C.c_int
        L.orc_build_linked_cells.argtypes = [_d, C.c_int64, C.c_double, _d, _i64, _i32,
                                             _i64, _i64, _i64, _i64, _i64]
        L.orc_linked_cells_from_indices.restype = C.c_int
        L.orc_linked_cells_from_indices.argtypes = [_i64, C.c_int64, C.c_int64, _i64, _i64, _i64]
        L.orc_segment_moments.argtypes = [C.c_int64, C.c_int64, _i64, _i64, _i64, _d, _d, _d]
        L.orc_finalize_com.argtypes = [C.c_int64, _d, _d]
        L.orc_rotate.argtypes = [C.c_int64, _d, _d, _d, C.c_double, C.c_double, _d]
        L.orc_rotate_cells.argtypes = [C.c_int64, _i64, _d, _d, _d, C.c_double, C.c_double, _d]
        L.orc_stream_wrap.argtypes = [C.c_int64, _d, _d, C.c_double, _d, _d]
        L.orc_cell_drift.restype = C.c_double
        L.orc_cell_drift.argtypes = [C.c_int64, _d, _d]
        L.orc_diag.argtypes = [C.c_int64, _d, _d, _d]
        L.orc_serial_step.restype = C.c_int
        L.orc_serial_step.argtypes = [C.c_int64, _d, _d, _d, _i64, C.c_double, C.c_double,
                                      C.c_double, C.c_double, C.c_uint64, C.c_uint64, C.c_int,
                                      C.c_int, _d, _d, _i64, _i64, _i64]
        L.orc_init_system.argtypes = [C.c_int64, _d, C.c_uint64, C.c_double, _d, _d]
        L.orc_set_threads.restype = C.c_int
        L.orc_set_threads.argtypes = [C.c_int]
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t) if a is not None else None


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a if shape is None else a.reshape(shape)


def set_threads(t: int) -> int:
    return lib().orc_set_threads(int(t))


# ------------------------------------------------------------------- RNG ----
def key_state(seed, step, purpose, cell) -> int:
    m = (1 << 64) - 1
    return int(lib().orc_key_state(seed & m, step & m, purpose & m, cell & m))


def uniform_at(state, index) -> float:
    return float(lib().orc_uniform_at(state, index))


def prng_raw(kind: str, s0=0, s1=0, s2=0, s3=0, count=1) -> np.ndarray:
    out = np.empty(count, dtype=np.uint64)
    lib().orc_prng_raw(PRNG_IDS[kind], s0, s1, s2, s3, count, _p(out, _u64))
    return out


def sample_uniform(kind, seed, step, purpose, cell, count) -> np.ndarray:
    out = np.empty(count)
    lib().orc_sample_uniform(PRNG_IDS[kind], seed, step, purpose, cell, count, _p(out, _d))
    return out


def grid_shift(step, seed, a=1.0, prng="splitmix") -> np.ndarray:
    out = np.empty(3)
    lib().orc_grid_shift(PRNG_IDS[prng], seed, step, a, _p(out, _d))
    return out


def rotation_axes(step, cell_ids, seed, prng="splitmix") -> np.ndarray:
    ids = np.ascontiguousarray(np.atleast_1d(cell_ids), dtype=np.int64)
    out = np.empty((ids.shape[0], 3))
    rc = lib().orc_rotation_axes(PRNG_IDS[prng], seed, step, _p(ids, _i64), ids.shape[0], _p(out, _d))
    if rc:
        raise RuntimeError("axis rejection sampling failed to terminate")
    return out


# ------------------------------------------------------------ collision ----
def wrap_coordinates(x, box) -> np.ndarray:
    x = _f64(x)
    out = np.empty_like(x)
    lib().orc_wrap(x.size, _p(x, _d), box, _p(out, _d))
    return out


def build_linked_cells(positions, cell_size, grid_min, dims, wrap=(False, False, False)):
    """Returns (cells, counts, offsets, perm) or raises ValueError(index, dim)."""
    pos = _f64(positions, (-1, 3))
    n = pos.shape[0]
    gmin = _f64(grid_min)
    dims = np.ascontiguousarray(dims, dtype=np.int64)
    wr = np.ascontiguousarray(wrap, dtype=np.int32)
    nc = int(np.prod(dims))
    cells = np.empty(n, np.int64)
    counts = np.empty(nc, np.int64)
    offsets = np.empty(nc, np.int64)
    perm = np.empty(n, np.int64)
    err = np.zeros(2, np.int64)
    rc = lib().orc_build_linked_cells(_p(pos, _d), n, cell_size, _p(gmin, _d), _p(dims, _i64),
                                      _p(wr, _i32), _p(cells, _i64), _p(counts, _i64),
                                      _p(offsets, _i64), _p(perm, _i64), _p(err, _i64))
    if rc:
        raise ValueError(int(err[0]), int(err[1]))
    return cells, counts, offsets, perm


def structure_from_indices(cells, n_cells):
    cells = np.ascontiguousarray(cells, dtype=np.int64)
    counts = np.empty(n_cells, np.int64)
    offsets = np.empty(n_cells, np.int64)
    perm = np.empty(cells.shape[0], np.int64)
    rc = lib().orc_linked_cells_from_indices(_p(cells, _i64), cells.shape[0], n_cells,
                                             _p(counts, _i64), _p(offsets, _i64), _p(perm, _i64))
    if rc:
        raise ValueError("flat cell index out of range")
    return counts, offsets, perm


def segment_moments(perm, counts, offsets, velocities, masses) -> np.ndarray:
    perm = np.ascontiguousarray(perm, dtype=np.int64)
    counts = np.ascontiguousarray(counts, dtype=np.int64)
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    v = _f64(velocities, (-1, 3))
    m = _f64(masses)
    out = np.empty((counts.shape[0], 4))
    lib().orc_segment_moments(v.shape[0], counts.shape[0], _p(perm, _i64), _p(counts, _i64),
                              _p(offsets, _i64), _p(v, _d), _p(m, _d), _p(out, _d))
    return out


def finalize_com(moments) -> np.ndarray:
    mom = _f64(moments, (-1, 4))
    out = np.empty((mom.shape[0], 3))
    lib().orc_finalize_com(mom.shape[0], _p(mom, _d), _p(out, _d))
    return out


def rotate_velocities(velocities, com_pp, axis_pp, cos_a, sin_a) -> np.ndarray:
    v = _f64(velocities, (-1, 3))
    c = _f64(com_pp, (-1, 3))
    a = _f64(axis_pp, (-1, 3))
    out = np.empty_like(v)
    lib().orc_rotate(v.shape[0], _p(v, _d), _p(c, _d), _p(a, _d), cos_a, sin_a, _p(out, _d))
    return out


def stream_and_wrap(positions, velocities, dt, box) -> np.ndarray:
    p = _f64(positions, (-1, 3))
    v = _f64(velocities, (-1, 3))
    b = _f64(np.broadcast_to(np.asarray(box, dtype=np.float64), (3,)))
    out = np.empty_like(p)
    lib().orc_stream_wrap(p.shape[0], _p(p, _d), _p(v, _d), dt, _p(b, _d), _p(out, _d))
    return out


def cell_drift(before, after) -> float:
    b = _f64(before, (-1, 4))
    a = _f64(after, (-1, 4))
    return float(lib().orc_cell_drift(b.shape[0], _p(b, _d), _p(a, _d)))


def diag(velocities, masses) -> np.ndarray:
    v = _f64(velocities, (-1, 3))
    m = _f64(masses)
    out = np.empty(5)
    lib().orc_diag(v.shape[0], _p(v, _d), _p(m, _d), _p(out, _d))
    return out


class StepResult:
    def __init__(self, **kw):
        self.__dict__.update(kw)


def serial_step(positions, velocities, masses, dims, cell_size, dt, cos_a, sin_a, seed, step,
                prng="splitmix", want_drift=False, want_detail=False) -> StepResult:
    """engine.py:415-455 on copies of the inputs (id order preserved)."""
    pos = _f64(positions, (-1, 3)).copy()
    vel = _f64(velocities, (-1, 3)).copy()
    m = _f64(masses)
    dims = np.ascontiguousarray(np.broadcast_to(np.asarray(dims), (3,)), dtype=np.int64)
    n = pos.shape[0]
    nc = int(np.prod(dims))
    drift = np.zeros(1)
    com = np.empty((nc, 3)) if want_detail else None
    counts = np.empty(nc, np.int64) if want_detail else None
    perm = np.empty(n, np.int64) if want_detail else None
    cells = np.empty(n, np.int64) if want_detail else None
    rc = lib().orc_serial_step(n, _p(pos, _d), _p(vel, _d), _p(m, _d), _p(dims, _i64), cell_size,
                               dt, cos_a, sin_a, seed, step, PRNG_IDS[prng], int(want_drift),
                               _p(drift, _d), _p(com, _d), _p(counts, _i64), _p(perm, _i64),
                               _p(cells, _i64))
    if rc:
        raise RuntimeError("axis rejection sampling failed to terminate")
    return StepResult(positions=pos, velocities=vel, drift=float(drift[0]) if want_drift else None,
                      com=com, counts=counts, perm=perm, cells=cells)


def init_system(dims, density, seed, cell_size=1.0, variance=1.0):
    """Baseline-only init (positions exact; velocities libm, ~1 ulp of numpy)."""
    dims = np.broadcast_to(np.asarray(dims, dtype=np.int64), (3,))
    n = int(round(int(np.prod(dims)) * density))
    box = np.ascontiguousarray(dims * cell_size, dtype=np.float64)
    pos = np.empty((n, 3))
    vel = np.empty((n, 3))
    lib().orc_init_system(n, _p(box, _d), seed, variance, _p(pos, _d), _p(vel, _d))
    return pos, vel, np.ones(n)
