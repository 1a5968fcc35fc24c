"""ctypes binding of libmpcd.so (include/mpcd.h).

The shared library is built in-tree by ``paper_2212_11878_b200._build`` (or
``__graft_entry__.build()``).  There is no fallback: if the library is missing
every entry point raises MpcdError immediately.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import BinningError, ConfigError, MpcdError, TopologyError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmpcd.so")

OK, ERR_CONFIG, ERR_BINNING, ERR_TOPOLOGY, ERR_RNG, ERR_CUDA, ERR_CAPACITY = range(7)
STEP_WANT_DRIFT = 1
STEP_WANT_COM = 2
PRNGS = {"splitmix": 0, "minstd": 1, "pcg32": 2, "sfc64": 3}

_d = C.POINTER(C.c_double)
_i64 = C.POINTER(C.c_int64)
_i32 = C.POINTER(C.c_int32)
_vp = C.c_void_p


class MpcdConfig(C.Structure):
    _fields_ = [
        ("dims", C.c_int64 * 3),
        ("cell_size", C.c_double),
        ("dt", C.c_double),
        ("cos_alpha", C.c_double),
        ("sin_alpha", C.c_double),
        ("seed", C.c_uint64),
        ("prng", C.c_int32),
        ("device", C.c_int32),
        ("capacity", C.c_int64),
        ("uniform_mass", C.c_int32),
        ("mass_value", C.c_double),
    ]


class MpcdDiag(C.Structure):
    _fields_ = [
        ("momentum", C.c_double * 3),
        ("energy", C.c_double),
        ("mass", C.c_double),
        ("max_cell_drift", C.c_double),
        ("n", C.c_int64),
        ("step", C.c_int64),
        ("migrated", C.c_int64),
    ]


class MpcdDomain(C.Structure):
    _fields_ = [
        ("global_dims", C.c_int64 * 3),
        ("rank_dims", C.c_int32 * 3),
        ("rank", C.c_int32),
        ("send_capacity", C.c_int64),
    ]


class MpcdExchange(C.Structure):
    _fields_ = [
        ("send", C.c_void_p),
        ("send_n", C.c_void_p),
        ("send_capacity", C.c_int64),
        ("n_ranks", C.c_int32),
        ("record_bytes", C.c_int32),
    ]


# name -> (restype, argtypes); mirrors include/mpcd.h one to one
SIGNATURES = {
    "mpcd_version": (C.c_char_p, []),
    "mpcd_last_error": (C.c_char_p, []),
    "mpcd_ctx_create": (C.c_int, [C.POINTER(MpcdConfig), C.POINTER(_vp)]),
    "mpcd_ctx_destroy": (C.c_int, [_vp]),
    "mpcd_upload": (C.c_int, [_vp, _d, _d, _d, _i64, C.c_int64, C.c_int64, _vp]),
    "mpcd_download": (C.c_int, [_vp, _d, _d, _d, _i64, C.c_int32, _vp]),
    "mpcd_count": (C.c_int64, [_vp]),
    "mpcd_cell_capacity": (C.c_int64, [_vp]),
    "mpcd_tile_cells": (C.c_int32, [_vp]),
    "mpcd_current_step": (C.c_int64, [_vp]),
    "mpcd_step": (C.c_int, [_vp, C.c_int64, C.c_int32, _vp]),
    "mpcd_run": (C.c_int, [_vp, C.c_int64, C.c_int64, C.c_int32, _vp]),
    "mpcd_read_diag": (C.c_int, [_vp, C.POINTER(MpcdDiag), _vp]),
    "mpcd_read_com": (C.c_int, [_vp, _i64, _d, _i64, _vp]),
    "mpcd_read_binning": (C.c_int, [_vp, _i64, _i64, _i64, _i64, _vp]),
    "mpcd_step_host": (C.c_int, [_vp, _d, _d, _d, C.c_int64, C.c_int64, C.c_int32, _d, _vp]),
    "mpcd_step_rows": (C.c_int, [_vp, _d, _d, _d, C.c_int64, C.c_int64, C.c_int32, _d, _d, _d,
                                 _vp]),
    "mpcd_host_alloc": (C.c_int, [C.c_int64, C.POINTER(C.c_void_p)]),
    "mpcd_host_free": (C.c_int, [_vp]),
    "mpcd_host_is_pinned": (C.c_int, [_vp]),
    "mpcd_init_device": (C.c_int, [_vp, C.c_int64, C.c_double, C.c_int64, _vp]),
    "mpcd_ctx_set_domain": (C.c_int, [_vp, C.POINTER(MpcdDomain)]),
    "mpcd_exchange_buffers": (C.c_int, [_vp, C.POINTER(MpcdExchange)]),
    "mpcd_absorb": (C.c_int, [_vp, _vp, C.c_int64, C.c_int64, _vp]),
    "mpcd_ipc_handles": (C.c_int, [_vp, _vp, _i64]),
    "mpcd_connect_peers": (C.c_int, [_vp, _vp, C.c_int32]),
    "mpcd_connect_local": (C.c_int, [C.POINTER(_vp), C.c_int32]),
    "mpcd_profile": (C.c_int, [_vp, C.c_int32]),
    "mpcd_read_profile": (C.c_int, [_vp, _d, _i64]),
    "mpcd_key_state": (C.c_uint64, [C.c_uint64] * 4),
    "mpcd_uniform_at": (C.c_double, [C.c_uint64, C.c_uint64]),
    "mpcd_grid_shift": (None, [C.c_int32, C.c_uint64, C.c_uint64, C.c_double, _d]),
    "mpcd_stage_sample_uniform": (C.c_int, [C.c_int32, C.c_uint64, C.c_uint64, C.c_uint64,
                                            C.c_uint64, C.c_int64, _vp, _vp]),
    "mpcd_stage_build_linked_cells": (C.c_int, [_vp, C.c_int64, C.c_double, _d, _i64, _i32, _vp,
                                                _vp, _vp, _vp, _i64, _vp]),
    "mpcd_stage_structure_from_cells": (C.c_int, [_vp, C.c_int64, C.c_int64, _vp, _vp, _vp, _vp]),
    "mpcd_stage_segment_moments": (C.c_int, [_vp, _vp, _vp, C.c_int64, _vp, _vp, C.c_int64, _vp,
                                             _vp]),
    "mpcd_stage_finalize_com": (C.c_int, [_vp, C.c_int64, _vp, _vp]),
    "mpcd_stage_rotation_axes": (C.c_int, [C.c_int32, C.c_uint64, C.c_int64, _vp, C.c_int64, _vp,
                                           _vp]),
    "mpcd_stage_rotate": (C.c_int, [_vp, _vp, _vp, C.c_int64, C.c_double, C.c_double, _vp, _vp]),
    "mpcd_stage_rotate_cells": (C.c_int, [_vp, _vp, _vp, _vp, C.c_int64, C.c_double, C.c_double,
                                          _vp, _vp]),
    "mpcd_stage_wrap": (C.c_int, [_vp, C.c_int64, C.c_double, _vp, _vp]),
    "mpcd_stage_stream_wrap": (C.c_int, [_vp, _vp, C.c_int64, C.c_double, _d, _vp, _vp]),
    "mpcd_stage_cell_drift": (C.c_int, [_vp, _vp, C.c_int64, _d, _vp]),
}

_lib = None


def load():
    """Load libmpcd.so, raising MpcdError if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("MPCD_LIB", LIB_PATH)  # tuning variants (tools/tune.py)
    if not os.path.exists(path):
        raise MpcdError(
            f"CUDA extension not built: {path} is missing. Run "
            "`python -c 'import __graft_entry__ as g; g.build()'` (nvcc, sm_100a).")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, err_info=None):
    """Map an mpcd_status to the reference's exception types (errors.py)."""
    if rc == OK:
        return
    msg = load().mpcd_last_error().decode(errors="replace")
    if rc == ERR_CONFIG:
        raise ConfigError(msg)
    if rc == ERR_BINNING:
        if err_info is not None:
            raise BinningError(msg, particle_index=int(err_info[0]), dimension=int(err_info[1]))
        raise BinningError(msg)
    if rc == ERR_TOPOLOGY:
        raise TopologyError(msg)
    if rc == ERR_RNG:
        raise RuntimeError("axis rejection sampling failed to terminate")
    raise MpcdError(f"libmpcd error {rc}: {msg}")
