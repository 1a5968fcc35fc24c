#!/usr/bin/env python
"""MPCD/SRD time-step benchmark (BASELINE.json metric: particle-steps/s and
fraction of the HBM roofline).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--L 256]

One "step" is one full SRD step (collide + stream + re-bin) of the whole
workload.  Default workload: BASELINE config 3, a 256^3-cell periodic box at
10 particles/cell (167,772,160 particles), alpha = 130 deg, dt = 0.1, seed 0,
the reference's splitmix keyed RNG.  The particle state (17.4 GB with its
double buffer) is far larger than L2, so no flush is needed between steps.

`value` is timed with CUDA events around K back-to-back steps on the
engine's stream (state resident in HBM).  `e2e` times the reference's public
pure function serial_collision_step(p, params, k) chained on host rows: the
rows go host -> device and back every step.  `--impl reference` times the
reference algorithm on the host cores (the oracle, oracle/, its bit-exact C
restatement, all host threads) on the same workload, and the reference
package's own benchmark (baseline/_ref) on a 64^3 box beside it.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MPCD particle-steps/sec"
UNIT = "particle-steps/s"
PPC = 10.0

# Roofline numerator: SURVEY.md 8(d)'s per-unit
# algorithmic bytes of the MPCD step, B_alg = 216 B per particle + 28 B per
# cell -- the compulsory traffic of the sort-based step the survey models --
# times the particles and cells one k_step launch processes.  Reported beside
# it: this design's own bytes (a particle is two 32-byte records, read once
# from its cell region and written once into its next-step cell: 128 B; per
# cell read + zero its count and one atomic on the next count: 16 B) and the
# compulsory floor B_min (read + write x, v once: 96 B).
KERNELS = ("k_step", "k_step_dense", "k_diag")  # mpcd_read_profile slots 0..2
# k_step, k_dense_prep, k_ovf_bucket, k_step_dense, k_diag_partial,
# k_diag_finalize (+ k_place_xrecs, the absorb of received particles, in a
# decomposed box with the exchange migration)
LAUNCHES_PER_STEP = 6
BYTES_PER_N = {"k_step": 128, "k_step_dense": 0, "k_diag": 0}   # this design
BYTES_PER_C = {"k_step": 16, "k_step_dense": 0, "k_diag": 0}
SURVEY_B_ALG_N, SURVEY_B_ALG_C = 216, 28  # B_alg = 216 n + 28 C
B_MIN_N = 96                              # compulsory: read + write x, v once


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--L", type=int, default=256, help="cells per box edge (per GPU)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-sample-L", type=int, default=128,
                    help="cells per edge of the CPU (oracle) sample box")
    ap.add_argument("--cpu-sample-steps", type=int, default=15,
                    help="timed oracle steps of the cpu_baseline sample (~10 s of host work)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--config", type=int, default=4, choices=(4, 5),
                    help="N > 1: 4 = (256 N) x 256 x 256 slabs (weak), 5 = 1024 x 512 x 512 "
                         "pencils (strong, 8 GPUs)")
    ap.add_argument("--migration", default="fused", choices=("fused", "exchange"),
                    help="N > 1: particle migration inside k_step over peer memory, or "
                         "through send buffers + NCCL point-to-point")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region.

    A reader thread collects the samples; __enter__ returns once the first
    sample arrived, so nvidia-smi's start-up does not eat the timed region.
    The summary uses the samples taken under load (utilization >= 50 %)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,"
              "utilization.gpu")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.rows = []

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 10:
                self.rows.append(parts)

    def __enter__(self):
        import threading

        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return self
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        t0 = time.time()
        while not self.rows and time.time() - t0 < 5.0 and self.proc.poll() is None:
            time.sleep(0.01)
        self.rows.clear()  # idle samples before the timed region
        return self

    def __exit__(self, *exc):
        if self.proc is None:
            return False
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=5)
        return False

    def summary(self):
        rows = list(self.rows)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        loaded = [r for r in rows if r[9].replace(".", "").isdigit() and float(r[9]) >= 50.0]
        use = loaded or rows
        sm = [float(r[1]) for r in use if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({n for r in use for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows), "samples_under_load": len(loaded)}


class NvmlClockSampler:
    """SM clocks and clock-event (throttle) reasons polled through NVML every
    ~2 ms by a thread during the timed region, so even a 20-step region of
    ~130 ms yields tens of samples (nvidia-smi's 50 ms loop yielded 2).
    Falls back to ClockSampler (nvidia-smi) when NVML is unavailable."""

    # nvmlClocksEventReason* bits (nvml.h)
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
            "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index, period=0.002):
        self.index = index
        self.period = period
        self.rows = []
        self.ok = False
        self.fallback = None

    def _handle(self, nv):
        import torch

        try:  # the NVML device of this CUDA ordinal (CUDA_VISIBLE_DEVICES may remap)
            uuid = str(torch.cuda.get_device_properties(self.index).uuid)
            if not uuid.startswith("GPU-"):
                uuid = "GPU-" + uuid
            return nv.nvmlDeviceGetHandleByUUID(uuid.encode())
        except Exception:  # noqa: BLE001
            return nv.nvmlDeviceGetHandleByIndex(self.index)

    def _poll(self):
        nv, h = self.nv, self.h
        while not self.stop:
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h) \
                    if hasattr(nv, "nvmlDeviceGetCurrentClocksEventReasons") \
                    else nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.rows.append((sm, rs))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __enter__(self):
        import threading

        try:
            import pynvml as nv

            nv.nvmlInit()
            self.nv = nv
            self.h = self._handle(nv)
            self.max_sm = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self.ok = True
        except Exception:  # noqa: BLE001 -- no NVML: nvidia-smi
            self.fallback = ClockSampler(self.index).__enter__()
            return self
        self.stop = False
        self.thread = threading.Thread(target=self._poll, daemon=True)
        self.thread.start()
        return self

    def __exit__(self, *exc):
        if self.fallback is not None:
            return self.fallback.__exit__(*exc)
        if self.ok:
            self.stop = True
            self.thread.join(timeout=5)
        return False

    def summary(self):
        if self.fallback is not None:
            return self.fallback.summary()
        rows = list(self.rows)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_sm if self.ok else None,
                    "reasons": ["unsampled"]}
        reasons = sorted({n for _, rs in rows for n, b in self.BITS.items() if rs & b})
        return {"sm_mhz": statistics.median(sm for sm, _ in rows), "sm_max_mhz": self.max_sm,
                "reasons": reasons, "samples": len(rows), "samples_under_load": len(rows),
                "sampler": f"NVML every {self.period * 1e3:g} ms during the timed region"}


def dist_setup(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_baseline(L, steps, seed):
    """The oracle (reference algorithm restated in C) on a bounded sample."""
    import numpy as np

    import oracle

    threads = oracle.set_threads(os.cpu_count() or 1)
    pos, vel, mass = oracle.init_system(L, PPC, seed)
    cs, sn = float(np.cos(np.radians(130.0))), float(np.sin(np.radians(130.0)))
    oracle.serial_step(pos, vel, mass, L, 1.0, 0.1, cs, sn, seed, 0)  # warm-up
    t0 = time.perf_counter()
    for k in range(1, steps + 1):
        r = oracle.serial_step(pos, vel, mass, L, 1.0, 0.1, cs, sn, seed, k)
        pos, vel = r.positions, r.velocities
    dt = time.perf_counter() - t0
    n = pos.shape[0]
    return {"value": n * steps / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"oracle/mpcd_oracle.c serial step, {L}^3 cells x {PPC:g} ({n} particles), "
                      f"{steps} steps after 1 warm-up, {threads} OpenMP threads, "
                      f"{dt / steps:.3f} s/step"}


def reference_package_cases(seed):
    """The reference package's own benchmark (mpcdsim.bench.run_benchmark_case,
    reference bench.py:77-122) on this host, when baseline/_ref holds its
    offline install: the serial backend (1 core) and the process backend
    (forked ranks, halo scheme) on a 64^3 box.  Secondary numbers beside the
    oracle port; None when the package is not installed."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "mpcdsim")):
        return None
    import math

    sys.path.insert(0, ref)
    try:
        from mpcdsim import bench as rbench
        from mpcdsim.params import SimParams as RParams
    finally:
        sys.path.remove(ref)
    cpus = os.cpu_count() or 1
    ranks = 1
    while ranks * 2 <= min(cpus, 64):
        ranks *= 2
    out = {}
    # serial on 1 core at 16^3 and 64^3, process on all cores;
    # the process backend runs at 64^3 and 128^3 (256^3 needs ~46 GB of host
    # RAM and minutes per step in numpy, beyond the reference arm's budget)
    cases = (("serial_16", "serial", 1, 16), ("serial_64", "serial", 1, 64),
             ("process_64", "process", ranks, 64), ("process_128", "process", ranks, 128))
    for name, backend, nranks, L in cases:
        params = RParams(edge_length=L, mean_density=PPC, dt=0.1, alpha=math.radians(130.0),
                         seed=seed, n_steps=3, rank_dims=rbench.rank_dims_for(nranks))
        t0 = time.perf_counter()
        rec = rbench.run_benchmark_case(params, steps=2, warmup=1, backend=backend)
        wall = time.perf_counter() - t0
        out[name] = {"value": rec.particles * rec.steps / rec.seconds, "unit": UNIT,
                     "cores": nranks, "backend": backend, "ranks": list(params.rank_dims),
                     "seconds_per_step": rec.seconds / rec.steps, "wall_s": wall,
                     "sample": f"{L}^3 x 10 ({L ** 3 * 10:,} particles), 1 warm-up + 2 timed "
                               "steps, mpcdsim.bench.run_benchmark_case"}
    return out


def run_reference(args):
    """The reference's CPU implementation of the step on this host's cores
    (the oracle: the reference algorithm restated in C, bit-exact with it,
    all host threads) on the SAME workload as our arm -- args.L^3 cells x 10
    -- with warm-up capped at 2 steps and the timed steps capped at ~120 s of
    host work (the metric is a rate).  The reference package's own benchmark
    runs beside it when installed (reference_package_cases)."""
    ws, rank, _ = dist_setup(args)
    if rank != 0:
        return
    L = args.L
    import numpy as np

    import oracle

    threads = oracle.set_threads(os.cpu_count() or 1)
    pos, vel, mass = oracle.init_system(L, PPC, args.seed)
    n = pos.shape[0]
    cs, sn = float(np.cos(np.radians(130.0))), float(np.sin(np.radians(130.0)))
    warm = min(args.warmup, 2)
    t_warm = None
    for k in range(warm):
        t0 = time.perf_counter()
        r = oracle.serial_step(pos, vel, mass, L, 1.0, 0.1, cs, sn, args.seed, k)
        t_warm = time.perf_counter() - t0
        pos, vel = r.positions, r.velocities
    timed = args.steps
    if t_warm:
        timed = max(1, min(args.steps, int(120.0 / t_warm)))
    t0 = time.perf_counter()
    for k in range(warm, warm + timed):
        r = oracle.serial_step(pos, vel, mass, L, 1.0, 0.1, cs, sn, args.seed, k)
        pos, vel = r.positions, r.velocities
    dt = time.perf_counter() - t0
    del pos, vel, r
    value = n * timed / dt
    sample = (f"{L}^3 cells x 10 ({n} particles) per step -- the benchmark workload itself -- "
              f"{warm} warm-up + {timed} timed steps of the {args.steps} asked (capped at ~120 s "
              f"of host work), {threads} OpenMP threads, oracle/mpcd_oracle.c (the reference "
              "algorithm restated in C, bit-exact with the reference package)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / timed, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (oracle init_system)",
        "config": config_of(args, ws, workload_params(args, ws)),
        "layout": f"CPU reference on the host: {L}^3 cells x 10 per timed step "
                  f"({timed} timed steps)" + ("" if ws == 1 else
                  f"; the GPU arm's per-GPU share of the {ws}-GPU box is {L}^3 cells x 10"),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    try:
        line["reference_package"] = reference_package_cases(args.seed)
    except Exception as exc:  # noqa: BLE001 -- secondary numbers only
        line["reference_package"] = {"error": f"{type(exc).__name__}: {exc}"}
    print(json.dumps(line), flush=True)


def run_ours(args):
    import numpy as np
    import torch

    ws, rank, local = dist_setup(args)
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        # MPCD_BENCH_BACKEND=gloo: host-staged exchange, lets several ranks
        # share one GPU (a functional check of this path, not a bench number)
        backend = os.environ.get("MPCD_BENCH_BACKEND", "nccl")
        kw = {"device_id": torch.device("cuda", local)} if backend == "nccl" else {}
        dist.init_process_group(backend, **kw)
    from paper_2212_11878_b200 import _lib
    from paper_2212_11878_b200.engine import EngineContext
    from paper_2212_11878_b200.params import SimParams

    L = args.L
    stream = torch.cuda.current_stream()
    if ws == 1:
        # BASELINE config 3: one 256^3 periodic box, no collective
        params = SimParams(edge_length=L, seed=args.seed)
        n = params.n_particles
        ctx = EngineContext(params.dims, params.cell_size, params.dt, params.alpha, params.seed,
                            params.prng, n, mass_value=1.0)
        ctx.init_device(n, 1.0, 0)
        n_total = n
        fused = False

        def run_steps(first, count):
            ctx.run(first, count)  # no host synchronisation between steps
    else:
        # BASELINE config 4: (L*ws) x L x L box, slab-decomposed, L^3 cells per
        # GPU.  Fused migration: k_step writes leaving particles into the
        # neighbour's cells over NVLink peer memory, a one-element NCCL
        # all-reduce fences each step (falls back to the NCCL exchange if
        # peer memory cannot be opened).
        from paper_2212_11878_b200.distributed import (CudaDomain, DistExchange, DomainLayout,
                                                       _DomainRunner, connect_fused)
        if args.config == 5:
            # BASELINE config 5: 1024 x 512 x 512 cells (2.7 G particles) strong
            # scaling, pencil decomposition (8 GPUs: 4 x 2 x 1)
            dims = (1024, 512, 512)
            rank_dims = {8: (4, 2, 1), 16: (4, 2, 2)}.get(ws)
            if rank_dims is None:
                raise SystemExit("config 5 needs 8 GPUs (1.1 TB of cell regions)")
        else:
            dims, rank_dims = (L * ws, L, L), (ws, 1, 1)
        params = SimParams(edge_length=dims[0], edge_lengths=dims, seed=args.seed,
                           rank_dims=rank_dims)
        layout = DomainLayout.from_params(params)
        dom = CudaDomain(params, layout, rank)
        exch = DistExchange()
        fused = args.migration == "fused" and connect_fused(dom, exch)
        dom.init_device(params.n_particles, 1.0)
        if fused:  # every rank's init precedes any rank's first step
            exch.fence()
        ctx = dom.ctx
        runner_md = _DomainRunner(params, [dom], exch, capture_drift=False, capture_com=False,
                                  fused=fused)
        n_total = params.n_particles
        n = n_total // ws

        def run_steps(first, count):
            for k in range(first, first + count):
                runner_md.advance(k, 0)
    C = L ** 3 if ws == 1 else int(np.prod(layout.local_dims))  # cells per GPU
    run_steps(0, args.warmup)
    torch.cuda.synchronize()

    def barrier():
        if ws > 1:
            torch.distributed.barrier()

    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    with NvmlClockSampler(local) as clocks:
        barrier()
        torch.cuda.synchronize()
        start.record(stream)
        run_steps(args.warmup, args.steps)
        end.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = start.elapsed_time(end) / args.steps
    if ws > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    value = n_total / (ms * 1e-3)
    d = ctx.read_diag()

    # per-kernel timing (CUDA events on the engine stream), separate pass
    import ctypes as C_
    lib = _lib.load()
    lib.mpcd_profile(ctx.handle, 1)
    prof_steps = max(3, min(args.steps, 10))
    run_steps(args.warmup + args.steps, prof_steps)
    kms = (C_.c_double * 5)()
    nst = C_.c_int64(0)
    _lib.check(lib.mpcd_read_profile(ctx.handle, kms, C_.byref(nst)))
    lib.mpcd_profile(ctx.handle, 0)
    per_kernel = {k: kms[i] / max(nst.value, 1) for i, k in enumerate(KERNELS)}
    top = max(per_kernel, key=per_kernel.get)
    alg = {k: BYTES_PER_N[k] * n + BYTES_PER_C[k] * C for k in KERNELS}  # design bytes
    peak, peak_src = peaks()
    survey_launch = SURVEY_B_ALG_N * n + SURVEY_B_ALG_C * C  # k_step does the whole step
    achieved = survey_launch / (per_kernel[top] * 1e-3) / 1e9
    design_achieved = alg[top] / (per_kernel[top] * 1e-3) / 1e9
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tfile):
        try:
            with open(tfile) as f:
                tr = json.load(f)
            if tr.get("L") == L and top in tr.get("kernels", {}):
                traffic = tr["kernels"][top]
        except Exception:
            traffic = None
    step_bytes = sum(alg.values())
    survey_bytes = SURVEY_B_ALG_N * n + SURVEY_B_ALG_C * C
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if ws > 1 and args.config == 5 else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (device init_system: uniform positions, N(0,1) velocities minus "
                "their mean, unit masses)",
        "config": config_of(args, ws, params),
        "layout": {"parallelism": "single domain" if ws == 1 else
                   f"{'slab' if params.rank_dims[1:] == (1, 1) else 'pencil'} decomposition "
                   f"{tuple(params.rank_dims)} of a {'x'.join(map(str, params.dims))} box, "
                   "particle migration every step: " +
                   ("fused into k_step over peer memory, " +
                    ("gloo barrier step fence (host-staged check mode)" if exch.host_staged
                     else "NCCL all-reduce step fence")
                    if fused else "send buffers + point-to-point exchange")},
        "roofline": {"bound": "hbm", "kernel": top, "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "algorithmic_bytes_per_launch": survey_launch,
                     "bytes_model": "SURVEY.md 8(d): 216 B/particle + 28 B/cell",
                     "design_bytes_per_launch": alg[top],
                     "design_achieved": design_achieved, "design_frac": design_achieved / peak,
                     "b_min_frac": B_MIN_N * n / (per_kernel[top] * 1e-3) / 1e9 / peak,
                     "traffic_source": "profiles/ncu_traffic.json (ncu --set full, "
                                       "dram__bytes_read.sum + dram__bytes_write.sum)",
                     "avg_launch_ms": per_kernel[top], "peak_source": peak_src,
                     # the DRAM bytes ncu measured for one launch, over this run's
                     # launch time: the fraction of the copy peak the kernel
                     # actually moves (the survey-byte `frac` counts bytes this
                     # one-pass design never moves)
                     "dram_frac": (traffic / (per_kernel[top] * 1e-3) / 1e9 / peak)
                     if traffic else None},
        "roofline_step": {
            "bytes_per_step": step_bytes, "achieved": step_bytes / (ms * 1e-3) / 1e9,
            "frac": step_bytes / (ms * 1e-3) / 1e9 / peak,
            "survey_b_alg_frac": survey_bytes / (ms * 1e-3) / 1e9 / peak,
            "b_min_frac": B_MIN_N * n / (ms * 1e-3) / 1e9 / peak,
            "kernel_ms": per_kernel},
        "gpu_launches": args.steps * (LAUNCHES_PER_STEP + (1 if ws > 1 and not fused else 0)),
        "diag_last": {"momentum": list(d.momentum), "energy": d.energy, "mass": d.mass,
                      "collided": int(d.n), "migrated": int(d.migrated)},
    }
    line["clocks"] = clocks.summary()
    if ws > 1:
        # the migration over NVLink (fused) or NCCL (exchange): every particle
        # that changes owner moves its two 32-byte records once
        mig = [int(d.migrated)]
        t = torch.tensor(mig, device="cuda", dtype=torch.int64)
        torch.distributed.all_reduce(t)
        line["migration"] = {"particles_per_step": int(t.item()),
                             "bytes_per_step": 64 * int(t.item()),
                             "bytes_per_gpu_per_step": 64 * int(d.migrated),
                             "path": "NVLink peer stores inside k_step" if fused
                             else "NCCL point-to-point"}
    if ws == 1 and not args.no_e2e:
        line["e2e"], line["e2e_stateful"] = e2e(args, params, ctx)
    elif ws > 1 and not args.no_e2e:
        line["e2e"] = e2e_decomposed(args, params, dom, exch, fused)
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.cpu_sample_L, args.cpu_sample_steps, args.seed)
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if ws > 1:
        torch.distributed.destroy_process_group()


def workload_params(args, ws):
    """The SimParams of the workload both arms describe (config 3 at N = 1,
    config 4 / 5 at N > 1)."""
    from paper_2212_11878_b200.params import SimParams

    L = args.L
    if ws == 1:
        return SimParams(edge_length=L, seed=args.seed)
    if args.config == 5:
        dims = (1024, 512, 512)
        rank_dims = {8: (4, 2, 1), 16: (4, 2, 2)}.get(ws)
        if rank_dims is None:
            raise SystemExit("config 5 needs 8 GPUs (1.1 TB of cell regions)")
    else:
        dims, rank_dims = (L * ws, L, L), (ws, 1, 1)
    return SimParams(edge_length=dims[0], edge_lengths=dims, seed=args.seed, rank_dims=rank_dims)


def config_of(args, ws, params):
    """`config` of the JSON line: identical for our arm and the reference arm
    (the driver compares them); how each arm runs it is reported outside."""
    cells = params.dims[0] * params.dims[1] * params.dims[2]
    state_gb = params.n_particles // ws * 64 / 1e9  # two 32-byte records per particle
    return {"workload": workload_text(args, ws, params), "cells_per_gpu": cells // ws,
            "particles_per_gpu": params.n_particles // ws,
            "l2": f"inputs larger than L2: {state_gb:.1f} GB of particle records per GPU "
                  ">> 126 MB L2, read once per step; no flush"}


def workload_text(args, ws, params):
    if ws == 1:
        L = args.L
        dims = f"{L}x{L}x{L}"
        which = "BASELINE config 3" if args.L == 256 else "custom size"
        return (f"{dims} cells x 10 particles/cell periodic SRD box ({which}), 130 deg, dt 0.1, "
                "splitmix keyed RNG")
    dims = "x".join(map(str, params.dims))
    if args.config == 5:
        return (f"{dims} cells x 10 particles/cell (BASELINE config 5, strong scaling over "
                f"{ws} GPUs), 130 deg, dt 0.1, splitmix keyed RNG")
    return (f"{args.L}^3 cells x 10 particles/cell per GPU, {dims} box (BASELINE config 4, weak "
            "scaling), 130 deg, dt 0.1, splitmix keyed RNG")


def e2e_decomposed(args, params, dom, exch, fused):
    """Simulation.step() of the nccl backend (NcclRunner.run_step): step,
    migration, per-rank diagnostics read back and merged on every rank."""
    import torch

    from paper_2212_11878_b200.distributed import _DomainRunner

    runner = _DomainRunner(params, [dom], exch, capture_drift=False, capture_com=False,
                           fused=fused)
    first = int(dom.ctx._lib.mpcd_current_step(dom.ctx.handle))  # a domain steps consecutively
    runner.run_step(first)
    torch.cuda.synchronize()
    torch.distributed.barrier()
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    for k in range(args.steps):
        runner.run_step(first + 1 + k)
    e.record()
    torch.cuda.synchronize()
    t = torch.tensor([s.elapsed_time(e) * 1e-3], device="cuda")
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return {"value": params.n_particles * args.steps / float(t.item()), "unit": UNIT,
            "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 8 * 9,
            "api": "Simulation(backend='nccl').step(): state resident, per-rank diagnostics "
                   "read back and merged every step (no pure-function form for a decomposed box)"}


def e2e(args, params, ctx):
    """End to end through the public API, K steps each:

    * ``e2e``: the reference's pure function ``serial_collision_step(p,
      params, k)`` (engine.py:415-455) chained ``p = step(p)`` on host rows --
      every step bins the caller's (n,3) rows from host memory over PCIe,
      steps, and writes the new rows back to host memory (page-locked rows
      from the API's own pool, read and written in place by the kernels);
    * ``e2e_stateful``: ``Simulation.step()`` with the state resident in HBM
      and the diagnostics read back every step.

    The bench's own context is closed before the pure-function leg, which
    builds its own (the API's cached context)."""
    import numpy as np
    import torch

    from paper_2212_11878_b200 import ParticleSet, serial_collision_step

    n = params.n_particles
    K = args.e2e_steps
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    # stateful: Simulation.step() == mpcd_step + mpcd_read_diag (diag + flags D2H)
    first = int(ctx._lib.mpcd_current_step(ctx.handle))
    torch.cuda.synchronize()
    s.record()
    for k in range(args.steps):
        ctx.step(first + k)
        ctx.read_diag()
    e.record()
    torch.cuda.synchronize()
    t2 = s.elapsed_time(e) * 1e-3
    stateful = {"value": n * args.steps / t2, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 72 + 64,
                "api": "Simulation.step() (state resident, diagnostics read back every step)"}
    ids, p = ctx.download(id_order=True)
    del ids
    ctx.close()
    torch.cuda.empty_cache()
    step0 = 1000
    p, _, _ = serial_collision_step(p, params, step0)  # warm-up: context, pool, pageable input
    torch.cuda.synchronize()
    s.record()
    for k in range(K):
        p, _, _ = serial_collision_step(p, params, step0 + 1 + k)
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e) * 1e-3
    assert isinstance(p, ParticleSet) and p.n == n and np.isfinite(p.positions[-1]).all()
    pure = {"value": n * K / t, "unit": UNIT, "h2d_bytes_per_step": 48 * n,
            "d2h_bytes_per_step": 48 * n + 72 + 2 * 64,
            "api": "serial_collision_step(ParticleSet, params, step) -- the reference's pure "
                   "function -- chained p = step(p) on host (n,3) float64 rows (the API's pooled "
                   "page-locked rows)", "steps": K}
    return pure, stateful


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
