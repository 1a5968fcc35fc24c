"""The reference's scaling-benchmark report on the
GPU backends.

Drop-in surface of ``mpcdsim.bench`` (reference bench.py:1-243): the names
``BenchRecord``, ``CSV_COLUMNS``, ``rank_dims_for``, ``run_benchmark_case``,
``run_benchmark_matrix``, ``emit_report`` and ``read_report``, with the same
arguments, the same CSV file (header + one row per case, floats written with
``repr`` so they read back exactly) and the same ``<path>.summary.txt`` lines.

What differs is what is timed and counted:

* a case runs on ``"cuda"`` (one domain) or, for several ranks, on
  ``"sequential"`` (every domain on this GPU) or ``"nccl"`` (torchrun);
  each measured step is bracketed by CUDA events on the engine's stream;
* the traffic columns count the particle migration, the only inter-domain
  traffic of the cell-ownership decomposition:
  ``bytes_per_step`` = migrated particles x the 64-byte record, and
  ``msgs_per_step`` = domains that sent particles.  No cell is ever split,
  so there are no moment messages.
"""

from __future__ import annotations

import csv
import heapq
import itertools
from dataclasses import astuple, dataclass, fields

import numpy as np

from . import _dev
from .engine import BACKEND_CUDA, BACKEND_SEQUENTIAL, Simulation
from .errors import ConfigError, MpcdError
from .params import SCHEME_HALO, SimParams

DEFAULT_SIZES = (16, 32, 64)
DEFAULT_RANK_COUNTS = (1, 2, 4, 8)
DEFAULT_WARMUP = 5
RECORD_BYTES = 64  # one migrated particle: two 32-byte records

CSV_COLUMNS = ("L", "ranks", "scheme", "steps", "seconds", "particles", "bytes_per_step",
               "msgs_per_step", "max_drift", "error")


@dataclass
class BenchRecord:
    """One (size, scheme, ranks) case; ``error`` is empty unless it failed."""

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

    @classmethod
    def failed(cls, L: int, ranks: int, scheme: str, steps: int, exc: BaseException):
        return cls(L, ranks, scheme, steps, 0.0, 0, 0.0, 0.0, 0.0,
                   f"{type(exc).__name__}: {exc}")


# ------------------------------------------------------------- ranks ---
def _prime_factors(n: int):
    p = 2
    while p * p <= n:
        while n % p == 0:
            yield p
            n //= p
        p += 1 if p == 2 else 2
    if n > 1:
        yield n


def rank_dims_for(n_ranks: int) -> tuple:
    """Near-cubic (x, y, z) rank grid for ``n_ranks`` (descending).

    The reference's rule (bench.py:53-74): hand the prime factors out,
    largest first, each to the axis that is currently smallest (the first
    such axis on ties).  A heap of (extent, axis) does the bookkeeping.
    """
    if n_ranks < 1:
        raise ConfigError("rank count must be positive")
    heap = [(1, axis) for axis in range(3)]
    for f in sorted(_prime_factors(n_ranks), reverse=True):
        extent, axis = heapq.heappop(heap)
        heapq.heappush(heap, (extent * f, axis))
    return tuple(sorted((extent for extent, _ in heap), reverse=True))


# ------------------------------------------------------------ timing ---
class _StepClock:
    """CUDA events around each measured step on the engine's stream."""

    def __init__(self):
        torch = _dev.torch()
        self._torch = torch
        self._pairs = []

    def time(self, fn):
        torch = self._torch
        stream = torch.cuda.current_stream()
        start = torch.cuda.Event(enable_timing=True)
        stop = torch.cuda.Event(enable_timing=True)
        start.record(stream)
        out = fn()
        stop.record(stream)
        self._pairs.append((start, stop))
        return out

    def seconds(self) -> float:
        self._torch.cuda.synchronize()
        return sum(a.elapsed_time(b) for a, b in self._pairs) / 1e3


def run_benchmark_case(params: SimParams, *, steps: int, warmup: int = DEFAULT_WARMUP,
                       backend: str = BACKEND_SEQUENTIAL) -> BenchRecord:
    """Warm up, then time ``steps`` steps of one configuration
    (reference bench.py:77-122).  ``max_drift`` is the largest deviation of
    the total momentum from its post-warm-up value over the measured steps."""
    if steps < 1:
        raise ConfigError("bench needs at least one measured step")
    chosen = BACKEND_CUDA if params.n_ranks == 1 else backend
    with Simulation(params, backend=chosen) as sim:
        for _ in range(warmup):
            sim.step()
        momentum0 = np.asarray(sim.conservation_report().total_momentum, dtype=np.float64)
        clock = _StepClock()
        migrated = senders = 0
        drift = 0.0
        for _ in range(steps):
            diag = clock.time(sim.step)
            migrated += int(diag.get("crossings", 0))
            senders += int(diag.get("sending_domains", 0))
            now = np.asarray(sim.conservation_report().total_momentum, dtype=np.float64)
            drift = max(drift, float(np.abs(now - momentum0).max()))
        return BenchRecord(L=params.edge_length, ranks=params.n_ranks, scheme=params.scheme,
                           steps=steps, seconds=clock.seconds(),
                           particles=params.n_particles,
                           bytes_per_step=RECORD_BYTES * migrated / steps,
                           msgs_per_step=senders / steps, max_drift=drift)


def run_benchmark_matrix(sizes=DEFAULT_SIZES, rank_counts=DEFAULT_RANK_COUNTS,
                         schemes=(SCHEME_HALO,), *, steps: int = 20,
                         warmup: int = DEFAULT_WARMUP, density: float = 10.0,
                         cell_size: float = 1.0, dt: float = 0.1, alpha_degrees: float = 130.0,
                         halo_width: int = 1, seed: int = 0, backend: str = BACKEND_SEQUENTIAL,
                         progress=None) -> list:
    """Every (size, scheme, ranks) case in that nesting order; a case that
    raises becomes an error record and the matrix carries on
    (reference bench.py:125-182)."""
    out = []
    for L, scheme, ranks in itertools.product(sizes, schemes, rank_counts):
        if progress is not None:
            progress(L, scheme, ranks)
        try:
            params = SimParams(edge_length=L, cell_size=cell_size, mean_density=density, dt=dt,
                               alpha=float(np.radians(alpha_degrees)), halo_width=halo_width,
                               seed=seed, n_steps=steps, scheme=scheme,
                               rank_dims=rank_dims_for(ranks))
            out.append(run_benchmark_case(params, steps=steps, warmup=warmup, backend=backend))
        except Exception as exc:  # noqa: BLE001 -- recorded, not raised
            out.append(BenchRecord.failed(L, ranks, scheme, steps, exc))
    return out


# ------------------------------------------------------------ report ---
_COLUMN_TYPES = {f.name: f.type for f in fields(BenchRecord)}
_PARSERS = {"int": int, "float": float, "str": str, int: int, float: float, str: str}


def _encode(value) -> str:
    # repr for floats: the CSV must read back bit for bit
    return repr(value) if isinstance(value, float) else str(value)


def _summary_lines(records):
    serial = {(r.L, r.scheme): r.seconds for r in records
              if r.ranks == 1 and not r.error and r.seconds > 0}
    for r in records:
        head = f"L={r.L} scheme={r.scheme} ranks={r.ranks}"
        if r.error:
            yield f"{head} FAILED: {r.error}"
            continue
        text = (f"{head} seconds={r.seconds:.3f} bytes/step={r.bytes_per_step:.0f} "
                f"msgs/step={r.msgs_per_step:.1f}")
        one = serial.get((r.L, r.scheme))
        if one is not None and r.seconds > 0:
            text += f" speedup={one / r.seconds:.2f}"
        yield text


def emit_report(records: list, path: str) -> None:
    """``path``: the CSV; ``path + ".summary.txt"``: one line per case with
    the speed-up over the same size's one-rank case (bench.py:191-222)."""
    if not records:
        raise MpcdError("benchmark produced no records")
    order = [CSV_COLUMNS.index(f.name) for f in fields(BenchRecord)]
    with open(path, "w", newline="") as fh:
        out = csv.writer(fh)
        out.writerow(CSV_COLUMNS)
        for rec in records:
            cells = [""] * len(CSV_COLUMNS)
            for pos, value in zip(order, astuple(rec)):
                cells[pos] = _encode(value)
            out.writerow(cells)
    with open(path + ".summary.txt", "w") as fh:
        fh.writelines(line + "\n" for line in _summary_lines(records))


def read_report(path: str) -> list:
    """The records of a CSV written by ``emit_report`` (bench.py:225-243);
    any other header is an MpcdError."""
    with open(path, newline="") as fh:
        rows = csv.reader(fh)
        header = tuple(next(rows, ()))
        if header != CSV_COLUMNS:
            raise MpcdError(f"unexpected benchmark columns in {path}")
        parse = [_PARSERS[_COLUMN_TYPES[name]] for name in header]
        return [BenchRecord(**{name: conv(cell) for name, conv, cell in zip(header, parse, row)})
                for row in rows]
