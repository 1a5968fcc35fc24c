"""Shifted collision grid on the GPU, stage by stage.

Same names, arguments, return types and exceptions as the reference module
(collision.py:1-344); every numeric stage runs as a libmpcd kernel
(csrc/mpcd_stages.cu) with bit-exact reference results.  The time-step
engine (engine.py) fuses these stages; this module exists so stage-level
parity can be tested function by function and so user code calling the
reference's stage functions keeps working.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _dev, _lib
from .errors import BinningError, ConfigError
from .rng import RngKey

_MAX_AXIS_TRIALS = 128


@dataclass(frozen=True)
class GridShift:
    """Per-step random translation of the collision grid (collision.py:25-29)."""

    offset: np.ndarray


def sample_grid_shift(step: int, seed: int, cell_size: float = 1.0,
                      prng: str = "splitmix") -> GridShift:
    """collision.py:32-36 -- evaluated by libmpcd's host build of the kernel code."""
    out = (C.c_double * 3)()
    _lib.load().mpcd_grid_shift(_lib.PRNGS[prng], int(seed) & ((1 << 64) - 1),
                                int(step) & ((1 << 64) - 1), float(cell_size), out)
    return GridShift(offset=np.array(out[:], dtype=np.float64))


def sample_keyed_stream(key: RngKey, count: int, prng: str = "splitmix") -> np.ndarray:
    out = _dev.empty((max(int(count), 0),))
    _lib.check(_lib.load().mpcd_stage_sample_uniform(
        _lib.PRNGS[prng], int(key.seed), int(key.step), int(key.purpose), int(key.cell_id),
        int(count), _dev.ptr(out), _dev.stream()))
    return np.atleast_1d(_dev.to_host(out))


@dataclass
class LinkedCellList:
    """Cell binning of a particle batch over a local grid (collision.py:39-80)."""

    grid_min: np.ndarray
    grid_max: np.ndarray
    cell_size: float
    dims: np.ndarray
    wrap: np.ndarray
    bin_count: np.ndarray
    bin_offset: np.ndarray
    permutation: np.ndarray
    cells: np.ndarray

    @property
    def n_cells(self) -> int:
        return int(self.dims[0] * self.dims[1] * self.dims[2])

    @property
    def n(self) -> int:
        return self.cells.shape[0]


def _dims_from_bounds(grid_min, grid_max, cell_size) -> np.ndarray:
    span = (np.asarray(grid_max, dtype=np.float64) - grid_min) / cell_size
    dims = np.rint(span).astype(np.int64)
    if np.any(np.abs(span - dims) > 1e-9) or np.any(dims < 1):
        raise ConfigError("grid bounds must span a positive whole number of cells")
    return dims


def build_linked_cells(positions, cell_size, grid_min, grid_max,
                       wrap=(False, False, False)) -> LinkedCellList:
    """Bin particles into the local grid (collision.py:112-147) on the GPU.

    Cell = floor((x - grid_min) / cell_size) per axis, modulo the axis size
    on wrapped axes; on bounded axes an out-of-grid particle raises
    BinningError naming the first offending particle of the first axis.
    """
    pos = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
    gmin = np.ascontiguousarray(grid_min, dtype=np.float64)
    gmax = np.asarray(grid_max, dtype=np.float64)
    wr = np.ascontiguousarray(np.asarray(wrap, dtype=bool).astype(np.int32))
    dims = _dims_from_bounds(gmin, gmax, cell_size)
    n = pos.shape[0]
    nc = int(np.prod(dims))
    dpos = _dev.to_dev(pos)
    cells = _dev.empty((n,), np.int64)
    counts = _dev.empty((nc,), np.int64)
    offsets = _dev.empty((nc,), np.int64)
    perm = _dev.empty((n,), np.int64)
    err = np.zeros(2, dtype=np.int64)
    dims_c = np.ascontiguousarray(dims, dtype=np.int64)
    rc = _lib.load().mpcd_stage_build_linked_cells(
        _dev.ptr(dpos), n, float(cell_size), gmin.ctypes.data_as(_lib._d),
        dims_c.ctypes.data_as(_lib._i64), wr.ctypes.data_as(_lib._i32), _dev.ptr(cells),
        _dev.ptr(counts), _dev.ptr(offsets), _dev.ptr(perm), err.ctypes.data_as(_lib._i64),
        _dev.stream())
    if rc == _lib.ERR_BINNING:
        i, d = int(err[0]), int(err[1])
        raise BinningError(
            f"particle {i} at {pos[i].tolist()} lies outside the grid along axis {d}",
            particle_index=i, dimension=d)
    _lib.check(rc)
    return LinkedCellList(grid_min=gmin, grid_max=gmax, cell_size=float(cell_size), dims=dims,
                          wrap=np.asarray(wrap, dtype=bool), bin_count=_dev.to_host(counts),
                          bin_offset=_dev.to_host(offsets), permutation=_dev.to_host(perm),
                          cells=_dev.to_host(cells))


def linked_cells_from_indices(flat, dims, grid_min, grid_max, cell_size, wrap) -> LinkedCellList:
    """collision.py:150-163: structure from precomputed flat indices."""
    dims = np.asarray(dims, dtype=np.int64)
    flat = np.ascontiguousarray(flat, dtype=np.int64)
    nc = int(np.prod(dims))
    n = flat.shape[0]
    dflat = _dev.to_dev(flat, np.int64)
    counts = _dev.empty((nc,), np.int64)
    offsets = _dev.empty((nc,), np.int64)
    perm = _dev.empty((n,), np.int64)
    rc = _lib.load().mpcd_stage_structure_from_cells(_dev.ptr(dflat), n, nc, _dev.ptr(counts),
                                                      _dev.ptr(offsets), _dev.ptr(perm),
                                                      _dev.stream())
    if rc == _lib.ERR_BINNING:
        raise BinningError("flat cell index out of range")
    _lib.check(rc)
    return LinkedCellList(grid_min=np.asarray(grid_min, dtype=np.float64),
                          grid_max=np.asarray(grid_max, dtype=np.float64),
                          cell_size=float(cell_size), dims=dims,
                          wrap=np.asarray(wrap, dtype=bool), bin_count=_dev.to_host(counts),
                          bin_offset=_dev.to_host(offsets), permutation=_dev.to_host(perm),
                          cells=flat)


@dataclass
class CellMomentField:
    """Per-cell accumulator: columns 0-2 momentum, column 3 mass."""

    moments: np.ndarray

    @property
    def momentum(self) -> np.ndarray:
        return self.moments[:, :3]

    @property
    def mass(self) -> np.ndarray:
        return self.moments[:, 3]


def segment_moments(cells: LinkedCellList, velocities, masses) -> np.ndarray:
    """collision.py:190-206 on the GPU, numpy reduceat association."""
    nc = cells.n_cells
    n = cells.n
    if n == 0:
        return np.zeros((nc, 4))
    out = _dev.empty((nc, 4))
    # keep every device temporary referenced until the kernel has run
    perm = _dev.to_dev(cells.permutation, np.int64)
    cnt = _dev.to_dev(cells.bin_count, np.int64)
    off = _dev.to_dev(cells.bin_offset, np.int64)
    vel = _dev.to_dev(np.asarray(velocities).reshape(-1, 3))
    m = _dev.to_dev(masses)
    _lib.check(_lib.load().mpcd_stage_segment_moments(
        _dev.ptr(perm), _dev.ptr(cnt), _dev.ptr(off), nc, _dev.ptr(vel), _dev.ptr(m), n,
        _dev.ptr(out), _dev.stream()))
    return _dev.to_host(out)


def accumulate_cell_moments(cells: LinkedCellList, velocities, masses) -> CellMomentField:
    return CellMomentField(segment_moments(cells, np.asarray(velocities), np.asarray(masses)))


def finalize_com(field: CellMomentField) -> np.ndarray:
    """collision.py:209-214: com = p / m where m > 0, else 0."""
    mom = np.ascontiguousarray(field.moments, dtype=np.float64)
    nc = mom.shape[0]
    if nc == 0:
        return np.zeros((0, 3))
    out = _dev.empty((nc, 3))
    dmom = _dev.to_dev(mom)
    _lib.check(_lib.load().mpcd_stage_finalize_com(_dev.ptr(dmom), nc, _dev.ptr(out),
                                                   _dev.stream()))
    return _dev.to_host(out)


def sample_rotation_axes(step: int, cell_ids, seed: int, prng: str = "splitmix") -> np.ndarray:
    """collision.py:217-250: one Marsaglia unit axis per global cell id."""
    ids = np.ascontiguousarray(np.atleast_1d(np.asarray(cell_ids, dtype=np.int64)))
    k = ids.shape[0]
    if k == 0:
        return np.empty((0, 3))
    out = _dev.empty((k, 3))
    dids = _dev.to_dev(ids, np.int64)
    _lib.check(_lib.load().mpcd_stage_rotation_axes(
        _lib.PRNGS[prng], int(seed) & ((1 << 64) - 1), int(step), _dev.ptr(dids), k,
        _dev.ptr(out), _dev.stream()))
    return _dev.to_host(out)


def sample_rotation_axis(step: int, global_cell_id: int, seed: int) -> np.ndarray:
    return sample_rotation_axes(step, np.array([global_cell_id]), seed)[0]


@dataclass
class RotationPlan:
    """Dense per-cell rotation axes plus the shared angle (collision.py:257-266)."""

    axes: np.ndarray
    alpha: float


def build_rotation_plan(step, seed, alpha, global_cell_ids, occupied,
                        prng: str = "splitmix") -> RotationPlan:
    """collision.py:269-286: axes for occupied cells, zeros elsewhere."""
    ids = np.asarray(global_cell_ids)
    occupied = np.asarray(occupied, dtype=bool)
    axes = np.zeros((ids.shape[0], 3))
    if occupied.any():
        axes[occupied] = sample_rotation_axes(step, ids[occupied], seed, prng)
    return RotationPlan(axes=axes, alpha=float(alpha))


def _cos_sin(alpha):
    # the reference multiplies by np.cos(alpha) / np.sin(alpha) (collision.py:304-305)
    return float(np.cos(alpha)), float(np.sin(alpha))


def rotate_velocities(velocities, com_per_particle, axis_per_particle, alpha) -> np.ndarray:
    """collision.py:289-306: Rodrigues rotation about per-particle axes (GPU)."""
    v = np.ascontiguousarray(velocities, dtype=np.float64).reshape(-1, 3)
    n = v.shape[0]
    if n == 0:
        return v.copy()
    cs, sn = _cos_sin(alpha)
    out = _dev.empty((n, 3))
    dv = _dev.to_dev(v)
    dc = _dev.to_dev(np.broadcast_to(com_per_particle, (n, 3)))
    da = _dev.to_dev(np.broadcast_to(axis_per_particle, (n, 3)))
    _lib.check(_lib.load().mpcd_stage_rotate(_dev.ptr(dv), _dev.ptr(dc), _dev.ptr(da), n, cs, sn,
                                             _dev.ptr(out), _dev.stream()))
    return _dev.to_host(out)


def rotate_cell_velocities(cells: LinkedCellList, velocities, com, plan: RotationPlan) -> np.ndarray:
    """collision.py:309-324: each particle rotated with its cell's com/axis."""
    if cells.n == 0:
        return np.asarray(velocities, dtype=np.float64).copy()
    cs, sn = _cos_sin(plan.alpha)
    n = cells.n
    out = _dev.empty((n, 3))
    dcells = _dev.to_dev(cells.cells, np.int64)
    dv = _dev.to_dev(np.asarray(velocities).reshape(-1, 3))
    dcom = _dev.to_dev(com)
    dax = _dev.to_dev(plan.axes)
    _lib.check(_lib.load().mpcd_stage_rotate_cells(_dev.ptr(dcells), _dev.ptr(dv), _dev.ptr(dcom),
                                                   _dev.ptr(dax), n, cs, sn, _dev.ptr(out),
                                                   _dev.stream()))
    return _dev.to_host(out)


def cell_momentum_drift(before: np.ndarray, after: np.ndarray) -> float:
    """collision.py:327-344 (GPU reduction)."""
    b = np.ascontiguousarray(before, dtype=np.float64)
    a = np.ascontiguousarray(after, dtype=np.float64)
    out = (C.c_double * 1)()
    db, da = _dev.to_dev(b), _dev.to_dev(a)
    _lib.check(_lib.load().mpcd_stage_cell_drift(_dev.ptr(db), _dev.ptr(da), b.shape[0], out,
                                                 _dev.stream()))
    return float(out[0])
