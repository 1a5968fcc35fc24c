"""ms/step of the resident engine across particle densities (device init,
CUDA events around ctx.run), with the tile geometry each density picks and
the share of tiles that went to the dense-tile path.

    python tools/density_sweep.py [--out profiles/r02_density_sweep.json]
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2212_11878_b200 as mp  # noqa: E402
from paper_2212_11878_b200 import _dev, engine  # noqa: E402


def time_case(L, density, steps=10, warmup=3, tile=None):
    if tile:
        os.environ["MPCD_TILE_CELLS"] = str(tile)
    else:
        os.environ.pop("MPCD_TILE_CELLS", None)
    params = mp.SimParams(edge_length=L, seed=1, mean_density=density)
    n = params.n_particles
    ctx = engine.EngineContext(params.dims, 1.0, params.dt, params.alpha, params.seed,
                               "splitmix", n, mass_value=1.0)
    try:
        ctx.init_device(n, 1.0, 0)
        ctx.run(0, warmup)
        ctx.read_diag()
        st = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        ctx.run(warmup, steps)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        d = ctx.read_diag()
        assert d.n == n
        # profile one more step for the kernel split
        ctx._lib.mpcd_profile(ctx.handle, 1)
        ctx.step(warmup + steps)
        prof = (mp._lib.C.c_double * 8)()
        cnt = mp._lib.C.c_int64()
        ctx._lib.mpcd_read_profile(ctx.handle, prof, mp._lib.C.byref(cnt))
        ctx._lib.mpcd_profile(ctx.handle, 0)
        return dict(L=L, density=density, n=n, tile_cells=ctx.tile_cells,
                    cell_capacity=ctx.cell_capacity, ms_per_step=ms,
                    g_particle_steps_per_s=n / ms / 1e6,
                    kernel_ms=dict(k_step=prof[0], dense_path=prof[1], diag=prof[2]))
    finally:
        ctx.close()
        torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    _dev.torch()
    cases = [(128, d) for d in (4, 10, 15, 20, 30, 60)]
    if not a.quick:
        cases += [(256, d) for d in (4, 10, 15)]
    rows = []
    for L, d in cases:
        r = time_case(L, d)
        rows.append(r)
        print(json.dumps(r), flush=True)
    # the tile geometry at the densities around the switch points
    if not a.quick:
        for L, d in ((128, 10), (128, 12), (128, 15), (128, 20), (128, 30)):
            for tc in (16, 8, 4):
                r = time_case(L, d, tile=tc)
                r["forced"] = True
                rows.append(r)
                print(json.dumps(r), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(dict(device=torch.cuda.get_device_name(0), rows=rows), f, indent=1)


if __name__ == "__main__":
    main()
