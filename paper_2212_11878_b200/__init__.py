"""B200-native MPCD / stochastic rotation dynamics engine.

A drop-in for the time-step loop of the reference package ``mpcdsim``
(arXiv:2212.11878 companion code): same public names, arguments and
exceptions, with the hot path -- grid shift, binning + counting sort,
per-cell reductions, random-axis rotation, streaming -- as hand-written
sm_100a CUDA kernels in ``libmpcd.so`` (C ABI: include/mpcd.h).

Backends: ``"cuda"`` (one GPU, bit-exact with the reference's serial path;
``"serial"`` is an alias) and ``"nccl"`` (slab/pencil decomposition, one
process per GPU).
"""

from .collision import (
    CellMomentField,
    GridShift,
    LinkedCellList,
    RotationPlan,
    accumulate_cell_moments,
    build_linked_cells,
    build_rotation_plan,
    cell_momentum_drift,
    finalize_com,
    linked_cells_from_indices,
    rotate_cell_velocities,
    rotate_velocities,
    sample_grid_shift,
    sample_rotation_axes,
    sample_rotation_axis,
    segment_moments,
)
from .decomposition import (
    CODE_STAY,
    DomainGrid,
    build_decomposition,
    classify_base3,
    code_digits,
    neighbor_rank,
    reflect_code,
)
from .engine import (
    BACKEND_CUDA,
    BACKEND_NCCL,
    BACKEND_PROCESS,
    BACKEND_SEQUENTIAL,
    BACKEND_SERIAL,
    POLICY_IMMEDIATE,
    POLICY_LAZY,
    ConservationReport,
    DecompositionAliasWarning,
    EquivalenceReport,
    Simulation,
    conservation_report,
    equivalence_check,
    serial_collision_step,
    step_parallel,
    step_serial,
)
from .errors import BinningError, ConfigError, MpcdError, TopologyError
from .params import PRNGS, SCHEME_HALO, SCHEME_MIGRATION, SimParams
from .particles import (
    ParticleSet,
    init_owned_slice,
    init_system,
    kinetic_energy,
    stream_and_wrap,
    total_mass,
    total_momentum,
    wrap_coordinates,
)
from .rng import Purpose, RngKey, gaussian_at, key_state, sample_uniform, uniform_at

__version__ = "0.1.0"
