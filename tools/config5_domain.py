"""One GPU's share of BASELINE config 5 at full size: rank 0 of the (4, 2, 1)
pencil decomposition of the 1024 x 512 x 512 box (2.68 G particles), i.e. a
256 x 256 x 512-cell domain holding ~335 M particles, initialised on the
device from the whole box's particle stream and stepped alone.  Leavers go
to the exchange send buffers and are not re-inserted (no peers here), so the
domain loses ~0.2 % of its particles per step; the per-step kernel time is
what a rank of the 8-GPU strong-scaling run spends before its migration.

    python tools/config5_domain.py [steps]
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2212_11878_b200 as mp  # noqa: E402
from paper_2212_11878_b200 import _lib  # noqa: E402
from paper_2212_11878_b200.distributed import CudaDomain, DomainLayout  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
params = mp.SimParams(edge_length=1024, edge_lengths=(1024, 512, 512), seed=0,
                      rank_dims=(4, 2, 1))
layout = DomainLayout.from_params(params)
n_local = params.n_particles // layout.n_ranks
# capacity: the mean share + 6 sigma + the leavers of a step; send buffers of
# 1 M records per destination (a step moves ~0.45 M across a 256 x 512 face)
dom = CudaDomain(params, layout, 0, send_capacity=1 << 20,
                 capacity=int(n_local + 6 * n_local ** 0.5 + (1 << 22)))
free0, total = torch.cuda.mem_get_info()
dom.init_device(params.n_particles, 1.0)
torch.cuda.synchronize()
n0 = dom.ctx.n
free, total = torch.cuda.mem_get_info()
lib = _lib.load()
lib.mpcd_profile(dom.ctx.handle, 1)
prev = [0.0, 0.0, 0.0]
ms = (C.c_double * 5)()
ns = C.c_int64(0)
for k in range(steps):
    dom.step(k, 0)
    sent = int(dom.send_counts().sum().item())
    dom.absorb(None, 0, sent)
    lib.mpcd_read_profile(dom.ctx.handle, ms, C.byref(ns))
    print(f"step {k}: k_step {ms[0] - prev[0]:.3f} ms, dense {ms[1] - prev[1]:.3f} ms, "
          f"sent {sent}, resident {dom.ctx.n}", flush=True)
    prev = [ms[0], ms[1], ms[2]]
    if k == 0:  # the first step touches every page of the regions: not steady state
        lib.mpcd_profile(dom.ctx.handle, 0)
        lib.mpcd_profile(dom.ctx.handle, 1)
        prev = [0.0, 0.0, 0.0]
        n0 = dom.ctx.n
n1 = dom.ctx.n
per = {k: ms[i] / ns.value for i, k in enumerate(("k_step", "dense", "diag"))}
print(json.dumps({
    "domain_cells": list(layout.local_dims), "particles_start": n0, "particles_end": n1,
    "steps_averaged": steps - 1, "kernel_ms_per_step": per,
    "particle_steps_per_s_domain": n0 / (per["k_step"] + per["dense"] + per["diag"]) * 1e3,
    "device_memory_used_gb": (total - free) / 1e9, "device_memory_total_gb": total / 1e9}))
dom.close()
