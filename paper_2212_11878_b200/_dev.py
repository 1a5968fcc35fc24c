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


# ------------------------------------------------- page-locked host rows ---
class _PinnedBlock:
    """Page-locked host memory behind one numpy array (its ``base``); the
    block goes back to the pool when the array is released."""

    def __init__(self, pool, addr: int, nbytes: int, shape, typestr: str):
        self._pool = pool
        self._addr = addr
        self._nbytes = nbytes
        self.__array_interface__ = {"data": (addr, False), "shape": tuple(shape),
                                    "typestr": typestr, "version": 3}

    def __del__(self):
        try:
            self._pool._give_back(self._addr, self._nbytes)
        except Exception:  # interpreter shutdown
            pass


class PinnedPool:
    """Reusable page-locked (mpcd_host_alloc) blocks, keyed by exact size.

    The pure-function boundary returns its rows in these arrays, so that the
    next call reads them over PCIe in place (no staging copy), and a step
    loop ``p = serial_collision_step(p, ...)`` recycles the same few blocks.
    At most ``keep`` free blocks per size are kept; the rest are freed.
    """

    def __init__(self, keep: int = 4):
        import threading
        self._free: dict = {}
        self._keep = keep
        self._lock = threading.Lock()

    def empty(self, shape, dtype=np.float64) -> np.ndarray:
        dt = np.dtype(dtype)
        nbytes = int(np.prod(shape)) * dt.itemsize
        if nbytes == 0:
            return np.empty(shape, dtype=dt)
        with self._lock:
            stack = self._free.get(nbytes)
            addr = stack.pop() if stack else None
        if addr is None:
            from . import _lib
            out = C.c_void_p()
            _lib.check(_lib.load().mpcd_host_alloc(nbytes, C.byref(out)))
            addr = out.value
        block = _PinnedBlock(self, addr, nbytes, shape, dt.str)
        return np.asarray(block)

    def _give_back(self, addr: int, nbytes: int):
        with self._lock:
            stack = self._free.setdefault(nbytes, [])
            if len(stack) < self._keep:
                stack.append(addr)
                return
        from . import _lib
        _lib.load().mpcd_host_free(C.c_void_p(addr))

    def clear(self):
        from . import _lib
        with self._lock:
            blocks = [a for stack in self._free.values() for a in stack]
            self._free.clear()
        for a in blocks:
            _lib.load().mpcd_host_free(C.c_void_p(a))


pinned = PinnedPool()


def is_pinned(a: np.ndarray) -> bool:
    from . import _lib
    return a.size > 0 and bool(_lib.load().mpcd_host_is_pinned(C.c_void_p(a.ctypes.data)))


def pinned_rows(a) -> np.ndarray:
    """``a`` as C-contiguous float64 in page-locked memory: ``a`` itself when
    it already is, else a pooled copy (multi-threaded host copy)."""
    arr = np.asarray(a)
    if arr.dtype == np.float64 and arr.flags.c_contiguous and (arr.size == 0 or is_pinned(arr)):
        return arr
    out = pinned.empty(arr.shape, np.float64)
    if arr.size:
        t = torch()
        t.from_numpy(out).copy_(t.from_numpy(np.ascontiguousarray(arr)).to(t.float64))
    return out
