"""Scaling benchmark over a (size, ranks) matrix, in the reference's CSV
format (mpcdsim/bench.py:1-243).

Same names, arguments, columns and error behaviour as the reference.
`backend` selects this package's backends:

- one rank: ``"cuda"``;
- several: ``"sequential"`` (every domain on this GPU), or ``"nccl"`` under
  torchrun.

The reference counts its in-process Transport's messages. Here the traffic
columns count what actually moves between domains each step:

- `bytes_per_step` is the migrated particles times the 64-byte record;
- `msgs_per_step` is the number of domains that sent particles. With the
  fused migration each such domain writes straight into its neighbours'
  cells.

There are no moment messages: a cell is never split between domains
(DESIGN.md section 6).
"""

from __future__ import annotations

import csv
import time
from dataclasses import dataclass, fields

import numpy as np

from .engine import BACKEND_CUDA, BACKEND_SEQUENTIAL, Simulation
from .errors import ConfigError, MpcdError
from .params import SCHEME_HALO, SimParams

DEFAULT_SIZES = (16, 32, 64)
DEFAULT_RANK_COUNTS = (1, 2, 4, 8)
DEFAULT_WARMUP = 5
RECORD_BYTES = 64

CSV_COLUMNS = ("L", "ranks", "scheme", "steps", "seconds", "particles", "bytes_per_step",
               "msgs_per_step", "max_drift", "error")


@dataclass
class BenchRecord:
    L: int
    ranks: int
    scheme: str
    steps: int
    seconds: float
    particles: int
    bytes_per_step: float
    msgs_per_step: float
    max_drift: float
    error: str = ""


def rank_dims_for(n_ranks: int) -> tuple:
    """Near-cubic 3-d factorisation of a rank count (bench.py:53-74): prime
    factors, largest first, each to the currently smallest dimension."""
    if n_ranks < 1:
        raise ConfigError("rank count must be positive")
    factors = []
    n, d = n_ranks, 2
    while d * d <= n:
        while n % d == 0:
            factors.append(d)
            n //= d
        d += 1
    if n > 1:
        factors.append(n)
    dims = [1, 1, 1]
    for f in sorted(factors, reverse=True):
        dims[int(np.argmin(dims))] *= f
    dims.sort(reverse=True)
    return (dims[0], dims[1], dims[2])


def run_benchmark_case(params: SimParams, *, steps: int, warmup: int = DEFAULT_WARMUP,
                       backend: str = BACKEND_SEQUENTIAL) -> BenchRecord:
    """Time `steps` steps after `warmup` unmeasured ones (bench.py:77-122)."""
    if steps < 1:
        raise ConfigError("bench needs at least one measured step")
    if params.n_ranks == 1:
        backend = BACKEND_CUDA
    sim = Simulation(params, backend=backend)
    try:
        sim.run(warmup)
        p_ref = sim.conservation_report().total_momentum
        max_drift = 0.0
        seconds = 0.0
        moved = 0
        senders = 0
        for _ in range(steps):
            t0 = time.perf_counter()
            diag = sim.step()  # synchronises: the diagnostics are read back
            seconds += time.perf_counter() - t0
            moved += int(diag.get("crossings", 0))
            senders += int(diag.get("sending_domains", 0))
            mom = sim.conservation_report().total_momentum
            max_drift = max(max_drift, float(np.max(np.abs(mom - p_ref))))
        return BenchRecord(L=params.edge_length, ranks=params.n_ranks, scheme=params.scheme,
                           steps=steps, seconds=seconds, particles=params.n_particles,
                           bytes_per_step=moved * RECORD_BYTES / steps,
                           msgs_per_step=senders / steps, max_drift=max_drift)
    finally:
        sim.close()


def run_benchmark_matrix(sizes=DEFAULT_SIZES, rank_counts=DEFAULT_RANK_COUNTS,
                         schemes=(SCHEME_HALO,), *, steps: int = 20,
                         warmup: int = DEFAULT_WARMUP, density: float = 10.0,
                         cell_size: float = 1.0, dt: float = 0.1, alpha_degrees: float = 130.0,
                         halo_width: int = 1, seed: int = 0, backend: str = BACKEND_SEQUENTIAL,
                         progress=None) -> list:
    """Every (size, scheme, ranks) case; a failing case becomes an error row
    and the matrix goes on (bench.py:125-182)."""
    records = []
    for L in sizes:
        for scheme in schemes:
            for ranks in rank_counts:
                if progress is not None:
                    progress(L, scheme, ranks)
                try:
                    params = SimParams(edge_length=L, cell_size=cell_size, mean_density=density,
                                       dt=dt, alpha=np.radians(alpha_degrees),
                                       halo_width=halo_width, seed=seed, n_steps=steps,
                                       scheme=scheme, rank_dims=rank_dims_for(ranks))
                    records.append(run_benchmark_case(params, steps=steps, warmup=warmup,
                                                      backend=backend))
                except Exception as exc:  # keep the matrix going
                    records.append(BenchRecord(L=L, ranks=ranks, scheme=scheme, steps=steps,
                                               seconds=0.0, particles=0, bytes_per_step=0.0,
                                               msgs_per_step=0.0, max_drift=0.0,
                                               error=f"{type(exc).__name__}: {exc}"))
    return records


def _cell_text(value) -> str:
    return repr(value) if isinstance(value, float) else str(value)


def emit_report(records: list, path: str) -> None:
    """The CSV plus a human-readable speedup summary (bench.py:191-222)."""
    if not records:
        raise MpcdError("benchmark produced no records")
    with open(path, "w", newline="") as fh:
        writer = csv.writer(fh)
        writer.writerow(CSV_COLUMNS)
        for rec in records:
            writer.writerow([_cell_text(getattr(rec, name)) for name in CSV_COLUMNS])
    with open(path + ".summary.txt", "w") as fh:
        base = {}
        for rec in records:
            if rec.ranks == 1 and not rec.error and rec.seconds > 0:
                base[(rec.L, rec.scheme)] = rec.seconds
        for rec in records:
            if rec.error:
                fh.write(f"L={rec.L} scheme={rec.scheme} ranks={rec.ranks} FAILED: {rec.error}\n")
                continue
            line = (f"L={rec.L} scheme={rec.scheme} ranks={rec.ranks} seconds={rec.seconds:.3f}"
                    f" bytes/step={rec.bytes_per_step:.0f} msgs/step={rec.msgs_per_step:.1f}")
            ref = base.get((rec.L, rec.scheme))
            if ref is not None and rec.seconds > 0:
                line += f" speedup={ref / rec.seconds:.2f}"
            fh.write(line + "\n")


def read_report(path: str) -> list:
    """Records back from a CSV written by emit_report, floats exact (repr)
    (bench.py:225-243)."""
    types = {f.name: f.type for f in fields(BenchRecord)}
    out = []
    with open(path, newline="") as fh:
        reader = csv.DictReader(fh)
        if tuple(reader.fieldnames or ()) != CSV_COLUMNS:
            raise MpcdError(f"unexpected benchmark columns in {path}")
        for row in reader:
            kw = {}
            for name in CSV_COLUMNS:
                typ, raw = types[name], row[name]
                if typ in (int, "int"):
                    kw[name] = int(raw)
                elif typ in (float, "float"):
                    kw[name] = float(raw)
                else:
                    kw[name] = raw
            out.append(BenchRecord(**kw))
    return out
