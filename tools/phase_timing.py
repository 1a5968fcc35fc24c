"""Per-phase cycle split of k_step's consumer warps (tuning build with
-DMPCD_TIMING, see tools/build_variants.py):

    MPCD_LIB=build/variants/timing.so python tools/phase_timing.py [L]
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2212_11878_b200 import _lib  # noqa: E402
from paper_2212_11878_b200.engine import EngineContext  # noqa: E402
from paper_2212_11878_b200.params import SimParams  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 256
p = SimParams(edge_length=L, seed=0)
ctx = EngineContext(p.dims, 1.0, p.dt, p.alpha, 0, "splitmix", p.n_particles, mass_value=1.0)
ctx.init_device(p.n_particles, 1.0, 0)
ctx.run(0, 3)
torch.cuda.synchronize()
lib = _lib.load()
buf = (C.c_ulonglong * 12)()
lib.mpcd_debug_phase_cycles(buf, 1)
steps = 5
ctx.run(3, steps)
torch.cuda.synchronize()
lib.mpcd_debug_phase_cycles(buf, 1)
v = list(buf)
tiles = v[9]  # consumer-warp tile visits
names = ["", "ids", "rank+stage", "moments+com", "rotate/stream/claims", "conservation sums",
         "claims' atomics return", "stores + drift", "wait for the tile (full)", ""]
tot = sum(v[1:9])
print(f"L={L}: {tiles} warp-tile visits over {steps} steps")
for k in range(1, 9):
    print(f"  {names[k]:22s} {v[k] / max(tiles, 1):9.1f} cycles/warp-tile  {100 * v[k] / tot:5.1f} %")

tiles_p = tiles / 4  # one producer per 4 consumer warps
print(f"  producer: waiting for a free buffer {v[10] / max(tiles_p, 1):9.1f} cycles/tile, "
      f"preparing {v[11] / max(tiles_p, 1):9.1f} cycles/tile "
      f"({100 * v[10] / max(v[10] + v[11], 1):.1f} % waiting)")
