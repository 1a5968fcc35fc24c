"""A/B timing of libmpcd builds on one box: alternating rounds of K steps of
a device-initialised box per library, CUDA events on one stream.  Only the
round-1 C ABI is used, so builds from any commit compare.

    python tools/ab_time.py LIB_A.so LIB_B.so:ENV=VAL,ENV2=VAL [--L 256] [--steps 20]

A spec's ENV=VAL settings are exported while that library runs.
"""

import argparse
import ctypes as C
import json
import math
import os

import torch


class Cfg(C.Structure):
    _fields_ = [("dims", C.c_int64 * 3), ("cell_size", C.c_double), ("dt", C.c_double),
                ("cos_alpha", C.c_double), ("sin_alpha", C.c_double), ("seed", C.c_uint64),
                ("prng", C.c_int32), ("device", C.c_int32), ("capacity", C.c_int64),
                ("uniform_mass", C.c_int32), ("mass_value", C.c_double)]


class Diag(C.Structure):
    _fields_ = [("momentum", C.c_double * 3), ("energy", C.c_double), ("mass", C.c_double),
                ("max_cell_drift", C.c_double), ("n", C.c_int64), ("step", C.c_int64),
                ("migrated", C.c_int64)]


def make(lib_path, L, density):
    lib = C.CDLL(lib_path)
    lib.mpcd_ctx_create.argtypes = [C.POINTER(Cfg), C.POINTER(C.c_void_p)]
    lib.mpcd_init_device.argtypes = [C.c_void_p, C.c_int64, C.c_double, C.c_int64, C.c_void_p]
    lib.mpcd_run.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int32, C.c_void_p]
    lib.mpcd_read_diag.argtypes = [C.c_void_p, C.POINTER(Diag), C.c_void_p]
    lib.mpcd_ctx_destroy.argtypes = [C.c_void_p]
    lib.mpcd_last_error.restype = C.c_char_p
    cfg = Cfg()
    for d in range(3):
        cfg.dims[d] = L
    a = math.radians(130.0)
    cfg.cell_size, cfg.dt, cfg.cos_alpha, cfg.sin_alpha = 1.0, 0.1, math.cos(a), math.sin(a)
    cfg.seed, cfg.prng, cfg.device = 0, 0, 0
    n = round(L ** 3 * density)
    cfg.capacity, cfg.uniform_mass, cfg.mass_value = n, 1, 1.0
    h = C.c_void_p()
    assert lib.mpcd_ctx_create(C.byref(cfg), C.byref(h)) == 0, lib.mpcd_last_error()
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    assert lib.mpcd_init_device(h, n, 1.0, 0, st) == 0, lib.mpcd_last_error()
    return lib, h, n, st


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="+")
    ap.add_argument("--L", type=int, default=256)
    ap.add_argument("--density", type=float, default=10.0)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--hash", type=int, default=1, help="compare the final state across libs")
    ap.add_argument("--split", type=int, default=1, help="per-kernel ms: k_step, dense, diag")
    a = ap.parse_args()
    torch.cuda.init()
    res = {p: [] for p in a.libs}
    hashes = {}
    splits = {}
    diags = {}
    step0 = {p: 0 for p in a.libs}
    for r in range(a.rounds):
        for p in a.libs:
            path, _, envs = p.partition(":")
            saved = dict(os.environ)
            for kv in filter(None, envs.split(",")):
                k, _, v = kv.partition("=")
                os.environ[k] = v
            lib, h, n, st = make(path, a.L, a.density)
            assert lib.mpcd_run(h, 0, 3, 0, st) == 0, lib.mpcd_last_error()
            if a.split:  # per-kernel CUDA events inside mpcd_step (an extra timed run)
                lib.mpcd_profile.argtypes = [C.c_void_p, C.c_int32]
                lib.mpcd_read_profile.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
                lib.mpcd_profile(h, 1)
                assert lib.mpcd_run(h, 3, 5, 0, st) == 0, lib.mpcd_last_error()
                ms = (C.c_double * 5)()
                ns = C.c_int64(0)
                lib.mpcd_read_profile(h, ms, C.byref(ns))
                lib.mpcd_profile(h, 0)
                splits.setdefault(p, [round(ms[i] / max(ns.value, 1), 3) for i in range(3)])
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            assert lib.mpcd_run(h, 3, a.steps, 0, st) == 0, lib.mpcd_last_error()
            e1.record()
            torch.cuda.synchronize()
            d = Diag()
            assert lib.mpcd_read_diag(h, C.byref(d), st) == 0
            assert d.n == n
            res[p].append(e0.elapsed_time(e1) / a.steps)
            if r == 0 and a.hash:  # state after 3 + steps steps, id order: must agree across libs
                import hashlib

                import numpy as np
                pos = np.empty((n, 3)); vel = np.empty((n, 3))
                lib.mpcd_download.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                              C.c_void_p, C.c_int32, C.c_void_p]
                assert lib.mpcd_download(h, pos.ctypes.data, vel.ctypes.data, None, None, 1, st) == 0
                torch.cuda.synchronize()
                hashes[p] = hashlib.sha256(pos.tobytes() + vel.tobytes()).hexdigest()[:16]
                diags[p] = [float(d.momentum[0]).hex(), float(d.energy).hex()]
            lib.mpcd_ctx_destroy(h)
            torch.cuda.empty_cache()
            os.environ.clear()
            os.environ.update(saved)
    for p in a.libs:
        v = res[p]
        print(json.dumps({"lib": p, "ms_per_step": sorted(v), "best": min(v),
                          "gps": n / min(v) / 1e6, "state": hashes.get(p),
                          "k_step/dense/diag": splits.get(p), "diag": diags.get(p)}))
    if a.hash and len(set(hashes.values())) > 1:
        print("STATE MISMATCH across libs:", hashes)


if __name__ == "__main__":
    main()
