"""PCIe rates on this box: DMA (cudaMemcpyAsync, pinned) vs the engine's
zero-copy upload / download of the pure-function path, 256^3 x 10 rows."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

n = 167_772_160
nbytes = n * 3 * 8
h = torch.empty(n * 3, dtype=torch.float64, pin_memory=True)
d = torch.empty(n * 3, dtype=torch.float64, device="cuda")
for name, src, dst in (("H2D", h, d), ("D2H", d, h)):
    dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(3):
        dst.copy_(src, non_blocking=True)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 3
    print(f"DMA {name}: {nbytes / ms / 1e6:.1f} GB/s ({ms:.1f} ms per 4.03 GB)")
# both directions at once (separate streams)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
h2 = torch.empty(n * 3, dtype=torch.float64, pin_memory=True)
d2 = torch.empty(n * 3, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
with torch.cuda.stream(s1):
    d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2):
    h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"DMA H2D + D2H concurrently: {2 * nbytes / dt / 1e9:.1f} GB/s total")
del d, d2, h2
torch.cuda.empty_cache()

from paper_2212_11878_b200 import ParticleSet, SimParams, serial_collision_step  # noqa: E402
from paper_2212_11878_b200 import engine  # noqa: E402

params = SimParams(edge_length=256, seed=0)
rs = np.random.default_rng(0)
p = ParticleSet(rs.uniform(0, 256, size=(n, 3)), rs.normal(size=(n, 3)), np.ones(n))
p, _, _ = serial_collision_step(p, params, 0)
torch.cuda.synchronize()
ctx = engine._pure_context(params, n) if hasattr(engine, "_pure_context") else None
t0 = time.perf_counter()
for k in range(3):
    p, _, _ = serial_collision_step(p, params, 1 + k)
dt = (time.perf_counter() - t0) / 3
print(f"serial_collision_step: {dt * 1e3:.1f} ms per step, {n / dt / 1e9:.3f} G particle-steps/s")
t0 = time.perf_counter()
for _ in range(3):
    engine._uniform_mass(np.ascontiguousarray(p.masses, dtype=np.float64))
print(f"_uniform_mass host scan: {(time.perf_counter() - t0) / 3 * 1e3:.1f} ms")
ctx = engine._context_for(params, n, 1.0)
from paper_2212_11878_b200 import _dev  # noqa: E402
po, vo = _dev.pinned.empty((n, 3)), _dev.pinned.empty((n, 3))
torch.cuda.synchronize()
t0 = time.perf_counter()
for k in range(3):
    ctx.step_rows(p.positions, p.velocities, None, po, vo, 10 + k, False, False)
print(f"step_rows (upload + step + download): {(time.perf_counter() - t0) / 3 * 1e3:.1f} ms")
lib = ctx._lib
torch.cuda.synchronize()
t0 = time.perf_counter()
ctx.upload(p.positions, p.velocities, None, None, 0)
torch.cuda.synchronize()
print(f"upload (zero-copy binning from pinned rows): {(time.perf_counter() - t0) * 1e3:.1f} ms")
