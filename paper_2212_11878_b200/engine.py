"""Time-step front end: ``Simulation`` and the pure-function step on the GPU.

Mirrors the reference's engine.py API (Simulation, serial_collision_step,
ConservationReport, equivalence_check, step_serial/step_parallel) with GPU
backends registered in the same backend dispatch (engine.py:524-542):

* ``"cuda"`` -- one GPU, the whole box (serial-equivalent; bit-exact with
  the reference's serial path).  ``"serial"`` is accepted as an alias so
  reference call sites run unmodified.
* ``"nccl"`` -- slab/pencil domain decomposition over several GPUs, one
  process per GPU (see ``distributed.py``).
* ``"sequential"`` -- the same decomposition with every domain in this
  process on one GPU (the reference's in-process ``sequential`` backend).
"""

from __future__ import annotations

import ctypes as C
import warnings
from dataclasses import dataclass, field, replace

import numpy as np

from . import _dev, _lib
from .collision import GridShift, sample_grid_shift
from .errors import ConfigError, MpcdError
from .params import SCHEME_MIGRATION, SimParams
from .particles import ParticleSet, init_system

BACKEND_CUDA = "cuda"
BACKEND_NCCL = "nccl"
BACKEND_SERIAL = "serial"  # alias of "cuda" (the single-domain path)
BACKEND_SEQUENTIAL = "sequential"  # decomposed box, every domain in this process
# the reference's one-worker-process-per-rank backend: here the same domains
# run in this process on this GPU ("nccl" is the one-process-per-GPU form)
BACKEND_PROCESS = "process"
BACKENDS = (BACKEND_CUDA, BACKEND_NCCL, BACKEND_SERIAL, BACKEND_SEQUENTIAL, BACKEND_PROCESS)
POLICY_IMMEDIATE = "immediate"
POLICY_LAZY = "lazy"
POLICIES = (POLICY_IMMEDIATE, POLICY_LAZY)


def _cos_sin(alpha):
    return float(np.cos(alpha)), float(np.sin(alpha))


class EngineContext:
    """Owns one libmpcd context (device state of one domain)."""

    def __init__(self, dims, cell_size, dt, alpha, seed, prng, capacity, mass_value=None,
                 device=None):
        lib = _lib.load()
        _dev.torch()  # fail loudly without a GPU
        cfg = _lib.MpcdConfig()
        for d in range(3):
            cfg.dims[d] = int(dims[d])
        cfg.cell_size = float(cell_size)
        cfg.dt = float(dt)
        cfg.cos_alpha, cfg.sin_alpha = _cos_sin(alpha)
        cfg.seed = int(seed) & ((1 << 64) - 1)
        cfg.prng = _lib.PRNGS[prng]
        cfg.device = int(_dev.device_index() if device is None else device)
        cfg.capacity = int(capacity)
        cfg.uniform_mass = 1 if mass_value is not None else 0
        cfg.mass_value = float(mass_value) if mass_value is not None else 0.0
        self.cfg = cfg
        self.capacity = int(capacity)
        self.dims = tuple(int(x) for x in dims)
        self.n_cells = self.dims[0] * self.dims[1] * self.dims[2]
        self.uniform_mass = mass_value is not None
        handle = C.c_void_p()
        _lib.check(lib.mpcd_ctx_create(C.byref(cfg), C.byref(handle)))
        self.handle = handle
        self._lib = lib

    def close(self):
        if self.handle:
            self._lib.mpcd_ctx_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def n(self) -> int:
        return int(self._lib.mpcd_count(self.handle))

    @property
    def tile_cells(self) -> int:
        """Cells per k_step tile (16, 8 or 4: follows capacity / cells)."""
        return int(self._lib.mpcd_tile_cells(self.handle))

    @property
    def cell_capacity(self) -> int:
        return int(self._lib.mpcd_cell_capacity(self.handle))

    def upload(self, positions, velocities, masses, ids, step: int):
        pos = np.ascontiguousarray(positions, dtype=np.float64)
        vel = np.ascontiguousarray(velocities, dtype=np.float64)
        m = None if self.uniform_mass else np.ascontiguousarray(masses, dtype=np.float64)
        idv = None if ids is None else np.ascontiguousarray(ids, dtype=np.int64)
        n = pos.shape[0]
        _lib.check(self._lib.mpcd_upload(
            self.handle, pos.ctypes.data_as(_lib._d), vel.ctypes.data_as(_lib._d),
            m.ctypes.data_as(_lib._d) if m is not None else None,
            idv.ctypes.data_as(_lib._i64) if idv is not None else None, n, int(step),
            _dev.stream()))

    def init_device(self, n: int, velocity_variance: float, step: int):
        _lib.check(self._lib.mpcd_init_device(self.handle, int(n), float(velocity_variance),
                                              int(step), _dev.stream()))

    def download(self, id_order: bool):
        n = self.n
        pos = np.empty((n, 3))
        vel = np.empty((n, 3))
        mass = np.empty(n)
        ids = np.empty(n, dtype=np.int64)
        _lib.check(self._lib.mpcd_download(
            self.handle, pos.ctypes.data_as(_lib._d), vel.ctypes.data_as(_lib._d),
            mass.ctypes.data_as(_lib._d), ids.ctypes.data_as(_lib._i64), 1 if id_order else 0,
            _dev.stream()))
        return ids, ParticleSet(pos, vel, mass)

    def step(self, step: int, flags: int = 0):
        _lib.check(self._lib.mpcd_step(self.handle, int(step), int(flags), _dev.stream()))

    def run(self, first_step: int, n_steps: int, flags: int = 0):
        _lib.check(self._lib.mpcd_run(self.handle, int(first_step), int(n_steps), int(flags),
                                      _dev.stream()))

    def read_diag(self) -> _lib.MpcdDiag:
        d = _lib.MpcdDiag()
        _lib.check(self._lib.mpcd_read_diag(self.handle, C.byref(d), _dev.stream()))
        return d

    def read_com(self):
        k = C.c_int64(0)
        _lib.check(self._lib.mpcd_read_com(self.handle, None, None, C.byref(k), _dev.stream()))
        ids = np.empty(k.value, dtype=np.int64)
        com = np.empty((k.value, 3))
        _lib.check(self._lib.mpcd_read_com(self.handle, ids.ctypes.data_as(_lib._i64),
                                           com.ctypes.data_as(_lib._d), C.byref(k),
                                           _dev.stream()))
        return ids, com

    def read_binning(self):
        n, nc = self.n, self.n_cells
        cells = np.empty(n, dtype=np.int64)
        counts = np.empty(nc, dtype=np.int64)
        offsets = np.empty(nc, dtype=np.int64)
        perm = np.empty(n, dtype=np.int64)
        _lib.check(self._lib.mpcd_read_binning(
            self.handle, cells.ctypes.data_as(_lib._i64), counts.ctypes.data_as(_lib._i64),
            offsets.ctypes.data_as(_lib._i64), perm.ctypes.data_as(_lib._i64), _dev.stream()))
        return cells, counts, offsets, perm

    # ------------------------------------------------ decomposed box ---
    def set_domain(self, global_dims, rank_dims, rank: int, send_capacity: int = 0):
        dom = _lib.MpcdDomain()
        for d in range(3):
            dom.global_dims[d] = int(global_dims[d])
            dom.rank_dims[d] = int(rank_dims[d])
        dom.rank = int(rank)
        dom.send_capacity = int(send_capacity)
        _lib.check(self._lib.mpcd_ctx_set_domain(self.handle, C.byref(dom)))
        ex = _lib.MpcdExchange()
        _lib.check(self._lib.mpcd_exchange_buffers(self.handle, C.byref(ex)))
        self.exchange_info = ex
        return ex

    def ipc_handles(self) -> bytes:
        """CUDA IPC handles of this context's regions, counts and overflow lists."""
        n = C.c_int64(0)
        _lib.check(self._lib.mpcd_ipc_handles(self.handle, None, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        _lib.check(self._lib.mpcd_ipc_handles(self.handle, buf, C.byref(n)))
        return buf.raw[: n.value]

    def connect_peers(self, all_handles: bytes, n_ranks: int):
        """Fused migration over peer memory opened from every rank's handles."""
        buf = C.create_string_buffer(all_handles, len(all_handles))
        _lib.check(self._lib.mpcd_connect_peers(self.handle, buf, int(n_ranks)))

    @staticmethod
    def connect_local(ctxs):
        """Fused migration between the domains of this process (ctxs[rank])."""
        lib = _lib.load()
        arr = (C.c_void_p * len(ctxs))(*[c.handle.value for c in ctxs])
        _lib.check(lib.mpcd_connect_local(arr, len(ctxs)))

    def absorb(self, recv_ptr: int, n_recv: int, n_sent: int):
        _lib.check(self._lib.mpcd_absorb(self.handle, C.c_void_p(int(recv_ptr) or None),
                                         int(n_recv), int(n_sent), _dev.stream()))

    def step_rows(self, pos_in, vel_in, masses, pos_out, vel_out, step: int, want_drift: bool,
                  want_com: bool = False):
        """serial_collision_step rows: (n,3) inputs -> (n,3) outputs (host)."""
        n = pos_in.shape[0]
        drift = C.c_double(0.0)
        m = None if self.uniform_mass else np.ascontiguousarray(masses, dtype=np.float64)
        _lib.check(self._lib.mpcd_step_rows(
            self.handle, pos_in.ctypes.data_as(_lib._d), vel_in.ctypes.data_as(_lib._d),
            m.ctypes.data_as(_lib._d) if m is not None else None, n, int(step),
            (_lib.STEP_WANT_DRIFT if want_drift else 0) | (_lib.STEP_WANT_COM if want_com else 0),
            pos_out.ctypes.data_as(_lib._d), vel_out.ctypes.data_as(_lib._d), C.byref(drift),
            _dev.stream()))
        return drift.value

    def step_host(self, positions, velocities, masses, step: int, want_drift: bool,
                  want_com: bool = False):
        """serial_collision_step on host buffers (overwritten in place)."""
        n = positions.shape[0]
        drift = C.c_double(0.0)
        m = None if self.uniform_mass else np.ascontiguousarray(masses, dtype=np.float64)
        _lib.check(self._lib.mpcd_step_host(
            self.handle, positions.ctypes.data_as(_lib._d), velocities.ctypes.data_as(_lib._d),
            m.ctypes.data_as(_lib._d) if m is not None else None, n, int(step),
            (_lib.STEP_WANT_DRIFT if want_drift else 0) | (_lib.STEP_WANT_COM if want_com else 0),
            C.byref(drift), _dev.stream()))
        return drift.value


# ------------------------------------------------------- pure function ---
_ctx_cache: dict = {}


def _context_for(params: SimParams, n: int, mass_value):
    key = (params.dims, params.cell_size, params.dt, params.alpha, params.seed, params.prng,
           mass_value, _dev.device_index())
    ctx = _ctx_cache.get(key)
    if ctx is None or ctx.capacity < n:
        if ctx is not None:
            ctx.close()
        if len(_ctx_cache) >= 4:
            for k in list(_ctx_cache):
                _ctx_cache.pop(k).close()
        ctx = EngineContext(params.dims, params.cell_size, params.dt, params.alpha, params.seed,
                            params.prng, max(n, 1), mass_value)
        _ctx_cache[key] = ctx
    return ctx


def _uniform_mass(masses: np.ndarray):
    """The common mass when every particle has it, else None (a parallel
    host scan: the pure function checks its input on every call)."""
    if masses.size == 0:
        return 1.0
    m0 = float(masses[0])
    if masses.size < (1 << 20):
        return m0 if bool(np.all(masses == m0)) else None
    t = _dev.torch()
    return m0 if bool(t.from_numpy(masses).eq(m0).all()) else None


def serial_collision_step(p: ParticleSet, params: SimParams, step: int, *,
                          want_drift: bool = False, want_com: bool = False):
    """One full step of the whole box on the GPU (engine.py:415-455).

    Same contract as the reference: returns (ParticleSet, drift | None,
    (occupied_ids, com) | None) with rows in the input order; the input is
    not modified.  The returned rows live in pooled page-locked host memory
    (``_dev.pinned``): the kernels bin them straight from there on the next
    call and write the next rows straight into another pooled block, so a
    step loop moves each row over PCIe once per direction and copies nothing
    on the host.  Pageable inputs are copied into a pooled block first.
    """
    masses = np.ascontiguousarray(p.masses, dtype=np.float64)
    pos_in = _dev.pinned_rows(p.positions)
    vel_in = _dev.pinned_rows(p.velocities)
    pos_out = _dev.pinned.empty((p.n, 3))
    vel_out = _dev.pinned.empty((p.n, 3))
    if masses.size >= (1 << 20):
        # Large inputs: the host scan that proves the masses uniform (33 ms at
        # 167 M particles) runs on a worker thread while the GPU steps with
        # the first mass as the guess (ctypes and torch release the GIL); a
        # non-uniform input then takes the per-particle-mass path again.
        guess = float(masses[0])
        pending = _scan_pool().submit(_uniform_mass, masses)
        ctx = _context_for(params, p.n, guess)
        drift = ctx.step_rows(pos_in, vel_in, None, pos_out, vel_out, step, want_drift, want_com)
        m0 = pending.result()
        if m0 is None or m0 != guess:
            ctx = _context_for(params, p.n, m0)
            m_in = None if m0 is not None else _dev.pinned_rows(masses)
            drift = ctx.step_rows(pos_in, vel_in, m_in, pos_out, vel_out, step, want_drift,
                                  want_com)
    else:
        m0 = _uniform_mass(masses)
        ctx = _context_for(params, p.n, m0)
        m_in = None if m0 is not None else _dev.pinned_rows(masses)
        drift = ctx.step_rows(pos_in, vel_in, m_in, pos_out, vel_out, step, want_drift, want_com)
    com = ctx.read_com() if want_com else None
    return ParticleSet(pos_out, vel_out, p.masses), (drift if want_drift else None), com


_SCAN_POOL = None


def _scan_pool():
    global _SCAN_POOL
    if _SCAN_POOL is None:
        import concurrent.futures as cf
        _SCAN_POOL = cf.ThreadPoolExecutor(max_workers=1, thread_name_prefix="mpcd-mass-scan")
    return _SCAN_POOL


# -------------------------------------------------------------- reports ---
@dataclass(frozen=True)
class ConservationReport:
    """Whole-system sums of the last step (reference engine.py:463-477):
    the same fields, and the same MpcdError for a non-finite value."""

    total_momentum: np.ndarray
    kinetic_energy: float
    total_mass: float
    max_cell_drift: float
    n_particles: int

    def __post_init__(self):
        scalars = np.array([self.kinetic_energy, self.total_mass, self.max_cell_drift],
                           dtype=np.float64)
        vec = np.asarray(self.total_momentum, dtype=np.float64).reshape(-1)
        if not (np.isfinite(vec).all() and np.isfinite(scalars).all()):
            raise MpcdError("conservation report contains non-finite values")


def conservation_report(sim: "Simulation") -> ConservationReport:
    return sim.conservation_report()


class CudaRunner:
    """Single-GPU runner: the whole periodic box in one engine context."""

    def __init__(self, params: SimParams, *, capture_drift: bool, capture_com: bool,
                 velocity_variance: float = 1.0, init: str = "host"):
        if params.n_ranks != 1:
            raise ConfigError("the cuda backend runs one domain: rank_dims must be (1,1,1)")
        self.params = params
        self.capture_drift = capture_drift
        self.capture_com = capture_com
        n = params.n_particles
        self.ctx = EngineContext(params.dims, params.cell_size, params.dt, params.alpha,
                                 params.seed, params.prng, max(n, 1), mass_value=1.0)
        if init == "device":
            self.ctx.init_device(n, velocity_variance, 0)
        elif init == "host":
            p = init_system(params, velocity_variance=velocity_variance)
            self.ctx.upload(p.positions, p.velocities, None, None, 0)
        else:
            raise ConfigError(f"unknown init {init!r}")
        self.transport = None
        self._last = None

    def run_step(self, step: int) -> dict:
        flags = (_lib.STEP_WANT_DRIFT if self.capture_drift else 0) | \
            (_lib.STEP_WANT_COM if self.capture_com else 0)
        self.ctx.step(step, flags)
        d = self.ctx.read_diag()
        self._last = d
        diag = {
            "n": int(d.n),
            "momentum": np.array(d.momentum[:]),
            "energy": float(d.energy),
            "mass": float(d.mass),
            "crossings": 0,
        }
        if self.capture_drift:
            diag["max_cell_drift"] = float(d.max_cell_drift)
        if self.capture_com:
            diag["com_capture"] = self.ctx.read_com()
        return diag

    def collect(self):
        return self.ctx.download(id_order=True)

    def particle_sets(self):
        return [self.ctx.download(id_order=False)]

    def reduce_conservation(self):
        if self._last is None:
            ids, p = self.ctx.download(id_order=False)
            from .particles import kinetic_energy, total_mass, total_momentum
            return p.n, total_momentum(p), kinetic_energy(p), total_mass(p)
        d = self._last
        return int(d.n), np.array(d.momentum[:]), float(d.energy), float(d.mass)

    def close(self):
        self.ctx.close()


class DecompositionAliasWarning(UserWarning):
    """A reference decomposition option that this engine runs as an alias."""


def _warn_aliases(params: SimParams, policy: str):
    """Scheme A (engine.py:280-391) and the lazy policy (engine.py:134-146)
    exist in the reference to limit split cells and halo traffic.  This
    engine owns whole cells of the shifted grid, so no
    cell is ever split: every scheme and policy runs the same decomposition,
    with trajectories bitwise equal to the whole box."""
    if params.n_ranks == 1:
        return
    if policy == POLICY_LAZY:
        warnings.warn("policy='lazy' is an alias here: cell ownership migrates exactly the "
                      "particles that change owner each step, with no guard band (the "
                      "reference's lazy policy, engine.py:134-146, widens the halo instead)",
                      DecompositionAliasWarning, stacklevel=3)
    if params.scheme == SCHEME_MIGRATION:
        warnings.warn("scheme='migration' (scheme A) runs the same cell-ownership "
                      "decomposition as 'halo': no cell is split, so there are no halo "
                      "moments to exchange (engine.py:280-391)",
                      DecompositionAliasWarning, stacklevel=3)


class Simulation:
    """A configured run: initialization, stepping, and collection (engine.py:494-641)."""

    def __init__(self, params: SimParams, *, backend: str = BACKEND_CUDA,
                 policy: str = POLICY_IMMEDIATE, capture_drift: bool = False,
                 capture_com: bool = False, velocity_variance: float = 1.0,
                 init: str = "host", migration: str = "fused"):
        if policy not in POLICIES:
            raise ConfigError(f"migration policy must be one of {POLICIES}")
        self.params = params
        self.backend_name = backend
        self.step_index = 0
        self.current_shift: GridShift | None = None
        self.diagnostics: list[dict] = []
        self.com_captures: list = []
        self.drift_history: list[float] = []
        self.capture_drift = capture_drift
        self.capture_com = capture_com
        if backend in (BACKEND_CUDA, BACKEND_SERIAL):
            if params.n_ranks != 1:
                raise ConfigError(f"{backend} backend requires rank_dims=(1,1,1)")
            self._runner = CudaRunner(params, capture_drift=capture_drift,
                                      capture_com=capture_com,
                                      velocity_variance=velocity_variance, init=init)
        elif backend in (BACKEND_NCCL, BACKEND_SEQUENTIAL, BACKEND_PROCESS):
            from .distributed import NcclRunner, SequentialRunner
            _warn_aliases(params, policy)
            cls = NcclRunner if backend == BACKEND_NCCL else SequentialRunner
            self._runner = cls(params, policy=policy, capture_drift=capture_drift,
                               capture_com=capture_com, velocity_variance=velocity_variance,
                               init=init, migration=migration)
        else:
            raise ConfigError(f"unknown backend {backend!r}")

    @property
    def runner(self):
        return self._runner

    @property
    def comm_records(self):
        t = getattr(self._runner, "transport", None)
        return [] if t is None else t.records

    def step(self) -> dict:
        k = self.step_index
        self.current_shift = sample_grid_shift(k, self.params.seed, self.params.cell_size,
                                               self.params.prng)
        diag = self._runner.run_step(k)
        diag["step"] = k
        if self.capture_drift:
            self.drift_history.append(diag.get("max_cell_drift", 0.0))
        if self.capture_com:
            self.com_captures.append(diag.pop("com_capture"))
        self.diagnostics.append(diag)
        self.step_index += 1
        return diag

    def run(self, n_steps: int | None = None) -> "Simulation":
        count = self.params.n_steps if n_steps is None else n_steps
        for _ in range(count):
            self.step()
        return self

    def advance(self, n_steps: int) -> "Simulation":
        """n steps without per-step host synchronisation.

        The first n - 1 steps run back to back on the device (their
        diagnostics are not read); the last is an ordinary ``step()``, so
        ``diagnostics``, ``drift_history``, ``com_captures``,
        ``current_shift`` and ``conservation_report()`` describe it."""
        if n_steps <= 0:
            return self
        runner = self._runner
        if not isinstance(runner, CudaRunner):
            return self.run(n_steps)
        if n_steps > 1:
            runner.ctx.run(self.step_index, n_steps - 1, 0)
            self.step_index += n_steps - 1
        self.step()
        return self

    def collect(self):
        """Global state ordered by particle id (engine.py:599-607)."""
        return self._runner.collect()

    def particle_sets(self):
        return self._runner.particle_sets()

    def conservation_report(self) -> ConservationReport:
        n, mom, en, mass = self._runner.reduce_conservation()
        drift = self.drift_history[-1] if self.drift_history else 0.0
        return ConservationReport(total_momentum=mom, kinetic_energy=en, total_mass=mass,
                                  max_cell_drift=drift, n_particles=n)

    def close(self):
        if self._runner is not None:
            self._runner.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False


def step_serial(sim: Simulation) -> Simulation:
    if sim.backend_name not in (BACKEND_SERIAL, BACKEND_CUDA):
        raise ConfigError("step_serial requires a single-domain (cuda) simulation")
    sim.step()
    return sim


def step_parallel(sim: Simulation, scheme: str | None = None) -> Simulation:
    if sim.backend_name in (BACKEND_SERIAL, BACKEND_CUDA):
        raise ConfigError("step_parallel requires a decomposed (nccl) simulation")
    if scheme is not None and scheme != sim.params.scheme:
        raise ConfigError(f"simulation was built for scheme {sim.params.scheme!r}")
    sim.step()
    return sim


@dataclass
class EquivalenceReport:
    n_steps: int
    per_step_position: list = field(default_factory=list)
    per_step_velocity: list = field(default_factory=list)
    per_step_com: list = field(default_factory=list)

    @property
    def max_position_dev(self) -> float:
        return max(self.per_step_position, default=0.0)

    @property
    def max_velocity_dev(self) -> float:
        return max(self.per_step_velocity, default=0.0)

    @property
    def max_com_dev(self) -> float:
        return max(self.per_step_com, default=0.0)


def _min_image_dev(pa, pb, box) -> float:
    d = np.abs(pa - pb)
    d = np.minimum(d, np.asarray(box) - d)
    return float(d.max()) if d.size else 0.0


def _build_for_check(params, rank_dims, scheme, capture_com, backend):
    if scheme == "serial":
        return Simulation(replace(params, rank_dims=(1, 1, 1)), backend=BACKEND_CUDA,
                          capture_com=capture_com)
    return Simulation(replace(params, rank_dims=tuple(rank_dims), scheme=scheme),
                      backend=backend, capture_com=capture_com)


def equivalence_check(config: SimParams, ranks_a, ranks_b, scheme_a: str, scheme_b: str,
                      n_steps: int, *, capture_com: bool = False,
                      backend: str = BACKEND_SEQUENTIAL) -> EquivalenceReport:
    """Run two settings of one physical config in lockstep (engine.py:703-748).

    The reference's default backend is its in-process "sequential" runner;
    here "sequential" runs the decomposed box's domains in-process on one GPU.
    """
    box = config.box_lengths
    report = EquivalenceReport(n_steps=n_steps)
    sim_a = _build_for_check(config, ranks_a, scheme_a, capture_com, backend)
    sim_b = _build_for_check(config, ranks_b, scheme_b, capture_com, backend)
    try:
        for _ in range(n_steps):
            sim_a.step()
            sim_b.step()
            ids_a, pa = sim_a.collect()
            ids_b, pb = sim_b.collect()
            if not np.array_equal(ids_a, ids_b):
                raise MpcdError("particle id sets diverged between runs")
            report.per_step_position.append(_min_image_dev(pa.positions, pb.positions, box))
            dv = np.abs(pa.velocities - pb.velocities)
            report.per_step_velocity.append(float(dv.max()) if dv.size else 0.0)
            if capture_com:
                ca_ids, ca = sim_a.com_captures[-1]
                cb_ids, cb = sim_b.com_captures[-1]
                if not np.array_equal(ca_ids, cb_ids):
                    raise MpcdError("occupied cell sets diverged between runs")
                dc = np.abs(ca - cb)
                report.per_step_com.append(float(dc.max()) if dc.size else 0.0)
    finally:
        sim_a.close()
        sim_b.close()
    return report
