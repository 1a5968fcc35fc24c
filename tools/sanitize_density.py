"""Small dense/cluster cases for compute-sanitizer (memcheck / racecheck):
densities 4-60 on a 16^3 box, a blob that overflows cells and stages dense
tiles in HBM, and the pure-function path.

    compute-sanitizer --tool memcheck python tools/sanitize_density.py
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2212_11878_b200 as mp  # noqa: E402
from paper_2212_11878_b200 import engine  # noqa: E402


def main():
    for density in (4, 15, 20, 30, 60):
        params = mp.SimParams(edge_length=16, seed=density, mean_density=density)
        with mp.Simulation(params, backend="cuda", init="device", capture_drift=True) as sim:
            sim.run(3)
            assert sim.diagnostics[-1]["n"] == params.n_particles
            print("density", density, "tile", sim.runner.ctx.tile_cells, "ok", flush=True)
    # blob: overflowing cells + a dense tile larger than the shared-memory staging
    L = 16
    n = 40960
    rs = np.random.default_rng(1)
    pos = np.concatenate([np.mod(8.3 + rs.normal(scale=0.7, size=(12000, 3)), L),
                          rs.uniform(0, L, size=(n - 12000, 3))])
    pos[pos >= L] = 0.0
    vel = rs.normal(size=(n, 3))
    ctx = engine.EngineContext((L, L, L), 1.0, 0.1, np.radians(130.0), 3, "splitmix", n,
                               mass_value=1.0)
    try:
        ctx.upload(pos, vel, None, None, 0)
        ctx.run(0, 3, 1)
        d = ctx.read_diag()
        assert d.n == n
        print("blob ok", d.momentum[:], flush=True)
    finally:
        ctx.close()
    p = mp.ParticleSet(pos, vel, np.ones(n))
    params = mp.SimParams(edge_length=L, seed=3)
    for k in range(2):
        p, drift, com = mp.serial_collision_step(p, params, k, want_drift=True, want_com=True)
    print("pure step ok", drift, flush=True)


if __name__ == "__main__":
    main()
