"""Decomposed box: slab / pencil domains over several GPUs (backend "nccl",
one process per GPU) or all in one process on one GPU (backend
"sequential", the reference's in-process runner).

Reference: the parallel step of ``mpcdsim`` (engine.py:190-272 for the halo
scheme, runners.py:73-348 for the runners, exchange.py:225-506 for the moment
reduction and particle migration, decomposition.py:20-146 for the rank grid).

B200 design.  Rank r owns the cells of its block of each
step's SHIFTED grid and every particle in them.  A cell is therefore never
split between ranks and needs no moment exchange: each rank collides whole
cells exactly as the one-domain kernel does, with the rotation axis keyed by
the global cell id, so the trajectory is bit-identical to the whole-box step
(and to the reference's serial path).  The one exchange per step is particle
migration: ``k_step`` writes each particle whose next-step cell belongs to
another rank into a per-destination send buffer; the runner exchanges counts
(one all_gather of the P x P count matrix), then the records (grouped
point-to-point), and ``mpcd_absorb`` bins the received ones.

Two migration modes:

* ``"fused"`` (default, the B200 path): after the domains connect their
  region / count / overflow allocations (CUDA IPC handles between
  processes, direct pointers within one), ``k_step`` itself writes each
  leaving particle into its new owner's next-step cell -- slot claimed by an
  atomic on the owner's count, record stored over NVLink peer memory.  A step
  is one kernel per rank plus a one-element all-reduce enqueued on the stream
  as the step fence; no send buffers, no host synchronisation, no absorb.
* ``"exchange"``: the particles go to per-destination send buffers; the
  runner all-gathers the count matrix and moves the records with grouped
  point-to-point sends (NCCL, or gloo host-staged), and ``mpcd_absorb`` bins
  them.  Also the fallback when peer memory cannot be opened.

The exchange is written against a small ``Domain`` interface (``step``,
``send_counts``, ``send_view``, ``absorb``, ``diag``) so the same host logic
drives the CUDA domains and, in the CPU test-suite, a model domain.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

from . import _dev, _lib
from .errors import ConfigError, MpcdError, TopologyError
from .params import SimParams
from .particles import ParticleSet, init_system

RECORD_BYTES = 64  # x y z id|pad vx vy vz m (include/mpcd.h, mpcd_exchange)
MIGRATIONS = ("fused", "exchange")


# ------------------------------------------------------------------ layout --
@dataclass(frozen=True)
class DomainLayout:
    """Uniform blocks of a global cell grid (decomposition.py:20-83).

    rank = (bx * Ry + by) * Rz + bz, as the reference's DomainGrid numbers
    its ranks (DomainGrid.rank_coords / rank_of_coords, decomposition.py:56-66);
    rank r owns cells [b * L, (b + 1) * L) per axis (own_cell_lo, :68-69).
    """

    global_dims: tuple
    rank_dims: tuple

    def __post_init__(self):
        for G, R in zip(self.global_dims, self.rank_dims):
            if R < 1 or G % R:
                raise TopologyError(f"rank_dims {self.rank_dims} must divide the cell grid "
                                    f"{self.global_dims}")

    @classmethod
    def from_params(cls, params: SimParams) -> "DomainLayout":
        return cls(tuple(int(x) for x in params.dims), tuple(int(x) for x in params.rank_dims))

    @property
    def n_ranks(self) -> int:
        return int(np.prod(self.rank_dims))

    @property
    def local_dims(self) -> tuple:
        return tuple(G // R for G, R in zip(self.global_dims, self.rank_dims))

    def coords(self, rank: int) -> tuple:
        Rx, Ry, Rz = self.rank_dims
        return (rank // (Ry * Rz), (rank // Rz) % Ry, rank % Rz)

    def origin(self, rank: int) -> tuple:
        return tuple(b * L for b, L in zip(self.coords(rank), self.local_dims))

    def owner_of_cells(self, gx, gy, gz):
        """Rank owning global cell coordinates (arrays)."""
        lx, ly, lz = self.local_dims
        _, Ry, Rz = self.rank_dims
        return (np.asarray(gx) // lx * Ry + np.asarray(gy) // ly) * Rz + np.asarray(gz) // lz


def default_send_capacity(layout: DomainLayout, mean_density: float) -> int:
    """Records per destination: 8 cell layers of the largest block face at
    the mean density (a step moves ~1/3 of one layer across a face), at least
    64 Ki.  Overflow is detected and raised, never silent."""
    lx, ly, lz = layout.local_dims
    face = max(ly * lz, lx * lz, lx * ly)
    return int(max(1 << 16, 8 * face * mean_density))


# --------------------------------------------------------------- exchange --
def _check_overflow(counts: np.ndarray, cap: int):
    """Every rank checks the same all-gathered matrix, so all raise together."""
    if counts.size and np.any(np.diag(counts)):
        r = int(np.argmax(np.diag(counts)))
        raise TopologyError(f"rank {r} routed particles to itself")
    if counts.size and int(counts.max()) > cap:
        src, dst = np.unravel_index(int(np.argmax(counts)), counts.shape)
        raise MpcdError(f"migration buffer overflow: rank {src} sends {int(counts.max())} "
                        f"particles to rank {dst}, capacity {cap} (raise send_capacity)")


class LocalExchange:
    """Every domain in this process: the records move by device copies."""

    def fence(self):
        pass  # one stream: domain steps run in order

    def exchange(self, domains) -> list:
        import torch

        P = len(domains)
        counts = torch.stack([d.send_counts() for d in domains]).cpu().numpy().astype(np.int64)
        _check_overflow(counts, min(d.send_capacity for d in domains))
        sent = []
        for dst in range(P):
            parts = [domains[src].send_view(dst, int(counts[src, dst]))
                     for src in range(P) if counts[src, dst] > 0]
            recv = torch.cat(parts) if parts else None
            domains[dst].absorb(recv, int(counts[:, dst].sum()), int(counts[dst].sum()))
            sent.append(int(counts[dst].sum()))
        return sent


class DistExchange:
    """One domain per process over torch.distributed.

    NCCL: counts and records move device to device (NVLink).  gloo (CPU
    tests, or several processes sharing one GPU): the same protocol staged
    through host tensors.
    """

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.host_staged = dist.get_backend(group) != "nccl"
        self._token = None

    def fence(self):
        """Step fence of the fused migration: every rank's step k completes
        before any rank's step k+1 starts.  NCCL: a one-element all-reduce on
        the current stream (device-side ordering, no host wait); gloo: the
        host waits for the device, then a barrier."""
        import torch

        if self.host_staged:
            torch.cuda.synchronize()
            self.dist.barrier(group=self.group)
            return
        if self._token is None:
            self._token = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.dist.all_reduce(self._token, group=self.group)

    def _stage(self, t):
        return t.cpu() if self.host_staged else t

    def exchange(self, domains) -> list:
        import torch

        (dom,) = domains
        dist = self.dist
        P = self.world
        mine = self._stage(dom.send_counts().to(torch.int64))
        rows = [torch.empty_like(mine) for _ in range(P)]
        dist.all_gather(rows, mine, group=self.group)
        counts = torch.stack(rows).cpu().numpy()  # [src, dst]
        _check_overflow(counts, dom.send_capacity)
        me = self.rank
        n_recv = int(counts[:, me].sum())
        n_sent = int(counts[me].sum())
        recv_dev = dom.recv_buffer(n_recv)
        recv = (torch.empty(n_recv * RECORD_BYTES, dtype=torch.uint8) if self.host_staged
                else recv_dev)
        ops = []
        off = 0
        for peer in range(P):
            c = int(counts[peer, me])
            if c and peer != me:
                ops.append(dist.P2POp(dist.irecv, recv[off:off + c * RECORD_BYTES], peer,
                                      group=self.group))
                off += c * RECORD_BYTES
        for peer in range(P):
            c = int(counts[me, peer])
            if c and peer != me:
                ops.append(dist.P2POp(dist.isend, self._stage(dom.send_view(peer, c)), peer,
                                      group=self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        if self.host_staged and n_recv:
            recv_dev[: n_recv * RECORD_BYTES].copy_(recv.to(recv_dev.device))
        dom.absorb(recv_dev[: n_recv * RECORD_BYTES] if n_recv else None, n_recv, n_sent)
        return [n_sent]

    def gather_objects(self, obj) -> list:
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out


# ------------------------------------------------------------- CUDA domain --
class _DeviceBytes:
    """__cuda_array_interface__ view of device memory owned by libmpcd."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1",
                                         "data": (int(ptr), False), "version": 3}


class CudaDomain:
    """One libmpcd context set up as domain `rank` of `layout`."""

    def __init__(self, params: SimParams, layout: DomainLayout, rank: int, *,
                 send_capacity: int = 0, capacity: int | None = None):
        from .engine import EngineContext

        torch = _dev.torch()
        self.rank = rank
        self.layout = layout
        n_local = params.n_particles / layout.n_ranks
        if capacity is None:  # mean share + 6 sigma + the migration margin
            capacity = int(n_local + 6 * np.sqrt(max(n_local, 1.0)) + 4096 +
                           2 * default_send_capacity(layout, params.mean_density))
        self.ctx = EngineContext(layout.local_dims, params.cell_size, params.dt, params.alpha,
                                 params.seed, params.prng, capacity, mass_value=1.0)
        cap = send_capacity or default_send_capacity(layout, params.mean_density)
        ex = self.ctx.set_domain(layout.global_dims, layout.rank_dims, rank, cap)
        self.send_capacity = int(ex.send_capacity)
        P = layout.n_ranks
        dev = _dev.device()
        self._send = torch.as_tensor(
            _DeviceBytes(ex.send, P * self.send_capacity * RECORD_BYTES), device=dev
        ).view(P, self.send_capacity * RECORD_BYTES)
        self._send_n = torch.as_tensor(_DeviceBytes(ex.send_n, P * 8), device=dev).view(torch.int64)
        self._recv = torch.empty(0, dtype=torch.uint8, device=dev)

    # Domain interface
    def step(self, k: int, flags: int):
        self.ctx.step(k, flags)

    def send_counts(self):
        return self._send_n

    def send_view(self, dest: int, count: int):
        return self._send[dest, : count * RECORD_BYTES]

    def recv_buffer(self, n: int):
        torch = _dev.torch()
        need = n * RECORD_BYTES
        if self._recv.numel() < need:
            self._recv = torch.empty(max(need, 2 * self._recv.numel()), dtype=torch.uint8,
                                     device=self._recv.device)
        return self._recv

    def absorb(self, recv, n_recv: int, n_sent: int):
        ptr = recv.data_ptr() if (recv is not None and n_recv) else 0
        self.ctx.absorb(ptr, n_recv, n_sent)
        self._keep = recv  # alive until the absorb kernel has run (same stream)

    def diag(self):
        d = self.ctx.read_diag()
        return np.array([*d.momentum, d.energy, d.mass, d.max_cell_drift, d.n, d.step,
                         d.migrated])

    def read_com(self):
        return self.ctx.read_com()

    def download(self):
        return self.ctx.download(id_order=False)

    def upload(self, p: ParticleSet):
        self.ctx.upload(p.positions, p.velocities, None, None, 0)

    def init_device(self, n: int, velocity_variance: float):
        self.ctx.init_device(n, velocity_variance, 0)

    def close(self):
        self.ctx.close()


# ----------------------------------------------------------------- runners --
def _merge(diags: list, crossings: int) -> dict:
    """Per-rank diagnostics combined in rank order (runners.py:27-56)."""
    out = {"n": 0, "momentum": np.zeros(3), "energy": 0.0, "mass": 0.0,
           "crossings": int(crossings)}  # particles that changed domain
    for d in diags:
        out["n"] += int(d[6])
        out["momentum"] = out["momentum"] + d[0:3]
        out["energy"] += float(d[3])
        out["mass"] += float(d[4])
    return out


def _sorted_by_id(ids, pos, vel, mass):
    order = np.argsort(ids, kind="stable")
    return ids[order], ParticleSet(pos[order], vel[order], mass[order])


class _DomainRunner:
    """Runner duck type of the reference (runners.py:73-155) over domains."""

    def __init__(self, params: SimParams, domains: list, exchange, *, capture_drift: bool,
                 capture_com: bool, fused: bool = False):
        self.params = params
        self.domains = domains
        self.exchange = exchange
        self.fused = fused
        self.capture_drift = capture_drift
        self.capture_com = capture_com
        self.transport = None
        self._last = None

    def _flags(self):
        return (_lib.STEP_WANT_DRIFT if self.capture_drift else 0) | \
            (_lib.STEP_WANT_COM if self.capture_com else 0)

    def advance(self, k: int, flags: int | None = None) -> int:
        """One step of every local domain plus the migration; returns the
        particles this process sent (no diagnostics read)."""
        f = self._flags() if flags is None else flags
        for d in self.domains:
            d.step(k, f)
        if self.fused:  # the particles already moved inside k_step
            self.exchange.fence()
            return 0
        return sum(self.exchange.exchange(self.domains))

    def _gather(self, obj):
        if isinstance(self.exchange, DistExchange):
            return self.exchange.gather_objects(obj)
        return [obj]

    def run_step(self, step: int) -> dict:
        self.advance(step)
        local = [(d.rank, d.diag(), d.read_com() if self.capture_com else None)
                 for d in self.domains]
        parts = sorted((x for g in self._gather(local) for x in g), key=lambda x: x[0])
        diag = _merge([p[1] for p in parts], int(sum(p[1][8] for p in parts)))
        diag["sending_domains"] = int(sum(1 for p in parts if p[1][8] > 0))
        if self.capture_drift:
            diag["max_cell_drift"] = max(float(p[1][5]) for p in parts)
        if self.capture_com:
            ids = np.concatenate([p[2][0] for p in parts])
            com = np.concatenate([p[2][1] for p in parts]).reshape(-1, 3)
            order = np.argsort(ids, kind="stable")
            diag["com_capture"] = (ids[order], com[order])
        self._last = diag
        return diag

    def _local_sets(self):
        return [(d.rank, *d.download()) for d in self.domains]

    def particle_sets(self):
        sets = [x for group in self._gather(self._local_sets()) for x in group]
        sets.sort(key=lambda x: x[0])
        return [(ids, p) for _, ids, p in sets]

    def collect(self):
        sets = self.particle_sets()
        ids = np.concatenate([s[0] for s in sets])
        pos = np.concatenate([s[1].positions for s in sets]).reshape(-1, 3)
        vel = np.concatenate([s[1].velocities for s in sets]).reshape(-1, 3)
        mass = np.concatenate([s[1].masses for s in sets])
        return _sorted_by_id(ids, pos, vel, mass)

    def reduce_conservation(self):
        if self._last is None:
            from .particles import kinetic_energy, total_mass, total_momentum
            _, p = self.collect()
            return p.n, total_momentum(p), kinetic_energy(p), total_mass(p)
        d = self._last
        return int(d["n"]), np.array(d["momentum"]), float(d["energy"]), float(d["mass"])

    def close(self):
        for d in self.domains:
            d.close()


def _initialise(domains: list, params: SimParams, velocity_variance: float, init: str):
    if init == "device":
        for d in domains:
            d.init_device(params.n_particles, velocity_variance)
    elif init == "host":
        p = init_system(params, velocity_variance=velocity_variance)
        for d in domains:  # each keeps the particles of its cells
            d.upload(p)
    else:
        raise ConfigError(f"unknown init {init!r}")


class SequentialRunner(_DomainRunner):
    """All domains of the decomposed box in this process, on the current GPU
    (the reference's SequentialRunner, runners.py:73-155)."""

    def __init__(self, params: SimParams, *, policy: str = "immediate",
                 capture_drift: bool = False, capture_com: bool = False,
                 velocity_variance: float = 1.0, init: str = "host", send_capacity: int = 0,
                 migration: str = "fused"):
        # `policy` (immediate / lazy migration, engine.py:134-146) trades halo
        # width against migration traffic in the reference; with cell
        # ownership every step migrates exactly the particles that change
        # owner, so both policies run the same exchange.
        layout = DomainLayout.from_params(params)
        if migration not in MIGRATIONS:
            raise ConfigError(f"migration must be one of {MIGRATIONS}")
        domains = [CudaDomain(params, layout, r, send_capacity=send_capacity)
                   for r in range(layout.n_ranks)]
        fused = migration == "fused"
        if fused:
            from .engine import EngineContext
            EngineContext.connect_local([d.ctx for d in domains])
        _initialise(domains, params, velocity_variance, init)
        super().__init__(params, domains, LocalExchange(), capture_drift=capture_drift,
                         capture_com=capture_com, fused=fused)
        self.layout = layout


def init_distributed(backend: str = "nccl"):
    """Join the torchrun process group (MASTER_ADDR/PORT, RANK, WORLD_SIZE)
    and bind this process to its GPU (LOCAL_RANK)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        if torch.cuda.is_available():
            ndev = torch.cuda.device_count()
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % ndev)
        kw = {}
        if backend == "nccl":
            kw["device_id"] = torch.device("cuda", torch.cuda.current_device())
        dist.init_process_group(backend, **kw)
    return dist


class NcclRunner(_DomainRunner):
    """One domain per process (torchrun, one process per GPU); migration over
    NCCL (or gloo, host-staged, when that is the process group's backend).
    World size must equal params.n_ranks.  `domain_factory(params, layout,
    rank)` replaces the CUDA domain (the CPU test-suite's model domain)."""

    def __init__(self, params: SimParams, *, policy: str = "immediate",
                 capture_drift: bool = False, capture_com: bool = False,
                 velocity_variance: float = 1.0, init: str = "host", send_capacity: int = 0,
                 group=None, domain_factory=None, migration: str = "fused"):
        import torch.distributed as dist

        if migration not in MIGRATIONS:
            raise ConfigError(f"migration must be one of {MIGRATIONS}")
        layout = DomainLayout.from_params(params)
        if not dist.is_initialized():
            init_distributed("nccl")
        world = dist.get_world_size(group)
        if world != layout.n_ranks:
            raise ConfigError(f"backend nccl runs one domain per process: rank_dims "
                              f"{params.rank_dims} needs {layout.n_ranks} processes, got {world}")
        rank = dist.get_rank(group)
        exchange = DistExchange(group)
        if domain_factory is None:
            domains = [CudaDomain(params, layout, rank, send_capacity=send_capacity)]
            fused = migration == "fused" and connect_fused(domains[0], exchange)
        else:
            domains = [domain_factory(params, layout, rank)]
            fused = False
        _initialise(domains, params, velocity_variance, init)
        if fused:  # every rank's init (counts zeroed) precedes any rank's first step
            exchange.fence()
        super().__init__(params, domains, exchange, capture_drift=capture_drift,
                         capture_com=capture_com, fused=fused)
        self.layout = layout
        self.migration = "fused" if fused else "exchange"


def connect_fused(dom: "CudaDomain", exchange: DistExchange) -> bool:
    """Open every other rank's regions (CUDA IPC) for the fused migration.
    All ranks agree: if any rank fails, all fall back to the exchange."""
    import torch

    err = None
    # every peer's device must be reachable from this one (NVLink / P2P)
    me = torch.cuda.current_device()
    devices = exchange.gather_objects(me)
    unreachable = [d for d in devices
                   if d != me and not torch.cuda.can_device_access_peer(me, d)]
    if unreachable:
        err = f"device {me} cannot access peer device(s) {sorted(set(unreachable))}"
    try:
        handles = dom.ctx.ipc_handles() if err is None else b""
    except Exception as e:  # noqa: BLE001 - reported, then the fallback
        err, handles = repr(e), b""
    allh = exchange.gather_objects(handles)
    if err is None and all(allh):
        try:
            dom.ctx.connect_peers(b"".join(allh), exchange.world)
        except Exception as e:  # noqa: BLE001
            err = repr(e)
    errs = [e for e in exchange.gather_objects(err) if e]
    if errs:
        import warnings
        warnings.warn(f"fused migration unavailable ({errs[0]}); using the exchange path")
        return False
    return True
