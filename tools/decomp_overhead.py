"""Cost of the decomposition on one GPU: the whole 256^3 box against the same
box as (2,1,1) domains (fused migration, and the staged exchange), all in
this process.  Prints ms/step for each (CUDA events, K steps after W).

    python tools/decomp_overhead.py [L] [K]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2212_11878_b200 as mp  # noqa: E402
from paper_2212_11878_b200.distributed import SequentialRunner  # noqa: E402
from paper_2212_11878_b200.engine import CudaRunner  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 256
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
W = 3


def timed(advance):
    for k in range(W):
        advance(k)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for k in range(W, W + K):
        advance(k)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / K


r = CudaRunner(mp.SimParams(edge_length=L, seed=0), capture_drift=False, capture_com=False,
               init="device")
print(f"whole box {L}^3: {timed(lambda k: r.ctx.step(k)):.3f} ms/step")
r.close()
torch.cuda.empty_cache()
for mig in ("fused", "exchange"):
    r = SequentialRunner(mp.SimParams(edge_length=L, seed=0, rank_dims=(2, 1, 1)), init="device",
                         migration=mig)
    ms = timed(lambda k: r.advance(k, 0))
    d = r.run_step(W + K)
    print(f"(2,1,1) domains, {mig}: {ms:.3f} ms/step, {d['crossings']} particles migrate/step")
    r.close()
    torch.cuda.empty_cache()

# per-kernel split of the fused domains (CUDA events inside mpcd_step)
import ctypes as C  # noqa: E402

from paper_2212_11878_b200 import _lib  # noqa: E402

r = SequentialRunner(mp.SimParams(edge_length=L, seed=0, rank_dims=(2, 1, 1)), init="device")
lib = _lib.load()
for k in range(W):
    r.advance(k, 0)
for d in r.domains:
    lib.mpcd_profile(d.ctx.handle, 1)
for k in range(W, W + 10):
    r.advance(k, 0)
for d in r.domains:
    ms = (C.c_double * 5)()
    ns = C.c_int64(0)
    lib.mpcd_read_profile(d.ctx.handle, ms, C.byref(ns))
    print(f"domain {d.rank}: k_step {ms[0] / ns.value:.3f} ms, dense {ms[1] / ns.value:.3f}, "
          f"diag {ms[2] / ns.value:.3f} per step")
r.close()

# Weak-scaling form (BASELINE config 4 per GPU): a (2L) x L x L box as two
# (2,1,1) domains of L^3 each, fused migration; each domain's k_step against
# the whole L^3 box's k_step (same cells and particles per kernel).
if os.environ.get("WEAK", "0") == "1":
    r = SequentialRunner(mp.SimParams(edge_length=2 * L, edge_lengths=(2 * L, L, L), seed=0,
                                      rank_dims=(2, 1, 1)),
                         init="device")
    for k in range(W):
        r.advance(k, 0)
    for d in r.domains:
        lib.mpcd_profile(d.ctx.handle, 1)
    for k in range(W, W + 10):
        r.advance(k, 0)
    d0 = r.run_step(W + 10)
    for d in r.domains:
        ms = (C.c_double * 5)()
        ns = C.c_int64(0)
        lib.mpcd_read_profile(d.ctx.handle, ms, C.byref(ns))
        print(f"weak: domain {d.rank} of (2L,L,L), L={L}: k_step {ms[0] / ns.value:.3f} ms, "
              f"dense {ms[1] / ns.value:.3f}, diag {ms[2] / ns.value:.3f} per step; "
              f"{d0['crossings']} particles migrate/step")
    r.close()
