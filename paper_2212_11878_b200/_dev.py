"""Device plumbing via PyTorch: buffers, the current stream, host<->device.

PyTorch is only the allocator / stream provider here; every computation is a
libmpcd kernel.  Without a CUDA device these helpers raise MpcdError (there
is no CPU path).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from .errors import MpcdError

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as _t
        _torch = _t
    if not _torch.cuda.is_available():
        raise MpcdError("a CUDA device is required (libmpcd has no CPU path)")
    return _torch


def device():
    t = torch()
    return t.device("cuda", t.cuda.current_device())


def device_index() -> int:
    return torch().cuda.current_device()


def stream():
    """Raw cudaStream_t of torch's current stream."""
    return C.c_void_p(torch().cuda.current_stream().cuda_stream)


def to_dev(a, dtype=np.float64):
    t = torch()
    arr = np.ascontiguousarray(a, dtype=dtype)
    return t.from_numpy(arr).to(device())


def empty(shape, dtype=np.float64):
    t = torch()
    tdt = {np.float64: t.float64, np.int64: t.int64, np.int32: t.int32}[np.dtype(dtype).type]
    return t.empty(shape, dtype=tdt, device=device())


def ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None and t.numel() else C.c_void_p(0)


def to_host(t) -> np.ndarray:
    return t.cpu().numpy()
