"""Cost of the decomposition on one GPU.

Default: the whole L^3 box against the same box as (2,1,1) domains (fused
migration, and the staged exchange), all in this process, plus the
per-kernel split of the fused domains.

WEAK=1 adds the weak-scaling form (BASELINE config 4 per GPU): a (2L) x L x L
box as two (2,1,1) domains of L^3 cells each, fused migration; each domain's
k_step is compared with the whole L^3 box's k_step (same cells and particles
per kernel).  ONLY_WEAK=1 runs the whole box's k_step and the weak form only.

    [WEAK=1|ONLY_WEAK=1] python tools/decomp_overhead.py [L] [K]
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2212_11878_b200 as mp  # noqa: E402
from paper_2212_11878_b200 import _lib  # noqa: E402
from paper_2212_11878_b200.distributed import SequentialRunner  # noqa: E402
from paper_2212_11878_b200.engine import CudaRunner  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 256
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
W = 3
ONLY_WEAK = os.environ.get("ONLY_WEAK", "0") == "1"
lib = _lib.load()


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


def kernel_split(ctxs, advance, steps=10):
    """Per-context k_step / dense / diag ms per step (CUDA events inside mpcd_step)."""
    for k in range(W):
        advance(k)
    for c in ctxs:
        lib.mpcd_profile(c.handle, 1)
    for k in range(W, W + steps):
        advance(k)
    out = []
    for c in ctxs:
        ms = (C.c_double * 5)()
        ns = C.c_int64(0)
        lib.mpcd_read_profile(c.handle, ms, C.byref(ns))
        out.append([ms[i] / ns.value for i in range(3)])
    return out


r = CudaRunner(mp.SimParams(edge_length=L, seed=0), capture_drift=False, capture_com=False,
               init="device")
if ONLY_WEAK:
    (ks, dn, dg), = kernel_split([r.ctx], lambda k: r.ctx.step(k))
    print(f"whole box {L}^3: k_step {ks:.3f} ms, dense {dn:.3f}, diag {dg:.3f} per step")
else:
    print(f"whole box {L}^3: {timed(lambda k: r.ctx.step(k)):.3f} ms/step")
r.close()
torch.cuda.empty_cache()

if not ONLY_WEAK:
    for mig in ("fused", "exchange"):
        r = SequentialRunner(mp.SimParams(edge_length=L, seed=0, rank_dims=(2, 1, 1)),
                             init="device", migration=mig)
        ms = timed(lambda k: r.advance(k, 0))
        d = r.run_step(W + K)
        print(f"(2,1,1) domains, {mig}: {ms:.3f} ms/step, {d['crossings']} particles migrate/step")
        r.close()
        torch.cuda.empty_cache()
    r = SequentialRunner(mp.SimParams(edge_length=L, seed=0, rank_dims=(2, 1, 1)), init="device")
    for d, (ks, dn, dg) in zip(r.domains, kernel_split([d.ctx for d in r.domains],
                                                       lambda k: r.advance(k, 0))):
        print(f"domain {d.rank}: k_step {ks:.3f} ms, dense {dn:.3f}, diag {dg:.3f} per step")
    r.close()
    torch.cuda.empty_cache()

if ONLY_WEAK or os.environ.get("WEAK", "0") == "1":
    r = SequentialRunner(mp.SimParams(edge_length=2 * L, edge_lengths=(2 * L, L, L), seed=0,
                                      rank_dims=(2, 1, 1)), init="device")
    split = kernel_split([d.ctx for d in r.domains], lambda k: r.advance(k, 0))
    d0 = r.run_step(W + 10)
    for d, (ks, dn, dg) in zip(r.domains, split):
        print(f"weak: domain {d.rank} of (2L,L,L), L={L}: k_step {ks:.3f} ms, dense {dn:.3f}, "
              f"diag {dg:.3f} per step; {d0['crossings']} particles migrate/step")
    r.close()
