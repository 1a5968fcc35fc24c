/*
 * mpcd.h -- C ABI of the B200-native MPCD/SRD time-step engine (libmpcd.so).
 *
 * Plain C types only (no torch, no C++).  Two layers:
 *
 *  1. Engine context (mpcd_ctx_*): particle state resident in HBM across
 *     steps in fixed-capacity collision-cell regions.  One step is one
 *     persistent kernel (collide + stream + write each particle into its
 *     next-step cell) plus a dense-tile kernel and a diagnostics reduction
 *     (DESIGN.md section 3).  Replaces the
 *     reference's per-step entry point
 *         Simulation.step()                 engine.py:555-591
 *         serial_collision_step(p, params, step, want_drift, want_com)
 *                                           engine.py:415-455
 *     and the runner duck type run_step/collect/particle_sets/
 *     reduce_conservation (runners.py:113-155).
 *
 *  2. Stage entry points (mpcd_stage_*): one kernel per reference function of
 *     collision.py / particles.py, on caller-owned DEVICE buffers in the
 *     reference layouts ((n,3) float64 C-order, int64 indices).  They exist so
 *     the reference's own unit tests (test_collision.py, test_particles.py)
 *     can run against the GPU stage by stage.
 *
 * Every call returns an mpcd_status; mpcd_last_error() gives the message of
 * the calling thread's last failure.  `stream` is a cudaStream_t (NULL = the
 * legacy default stream).  Device pointers must be 8-byte aligned.
 */
#ifndef MPCD_H_
#define MPCD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* errors.py:4-22 mapping (host shim raises the matching mpcdsim exception) */
typedef enum {
  MPCD_OK = 0,
  MPCD_ERR_CONFIG = 1,   /* ConfigError          errors.py:8-9   */
  MPCD_ERR_BINNING = 2,  /* BinningError(index, dim) errors.py:16-22 */
  MPCD_ERR_TOPOLOGY = 3, /* TopologyError        errors.py:12-13 */
  MPCD_ERR_RNG = 4,      /* RuntimeError: axis rejection did not terminate (collision.py:248-249) */
  MPCD_ERR_CUDA = 5,
  MPCD_ERR_CAPACITY = 6  /* more particles than the context holds */
} mpcd_status;

/* SimParams.prng extension: splitmix is the reference's keyed generator
 * (rng.py); the others are canonical generators seeded from its key
 * (absent from the reference). */
typedef enum {
  MPCD_PRNG_SPLITMIX = 0,
  MPCD_PRNG_MINSTD = 1,
  MPCD_PRNG_PCG32 = 2,
  MPCD_PRNG_SFC64 = 3
} mpcd_prng;

enum {
  MPCD_STEP_WANT_DRIFT = 1, /* capture_drift: per-cell momentum drift (engine.py:447-449) */
  MPCD_STEP_WANT_COM = 2    /* capture_com: keep com of occupied cells (engine.py:451-453) */
};

/* SimParams (params.py:44-53) as the engine needs it.  dims are the cells per
 * axis (cubic boxes: all equal to edge_length; non-cubic is the BASELINE
 * configs 4/5 extension). */
typedef struct {
  int64_t dims[3];
  double cell_size;
  double dt;
  double cos_alpha; /* np.cos(alpha) from the host, as the reference computes it */
  double sin_alpha; /* np.sin(alpha) */
  uint64_t seed;
  int32_t prng;     /* mpcd_prng */
  int32_t device;   /* CUDA ordinal */
  int64_t capacity; /* max resident particles (< 2^32) */
  int32_t uniform_mass; /* 1: every mass == mass_value, not stored per particle */
  double mass_value;
} mpcd_config;

/* Per-step diagnostics (engine.py:569-589, particles.py:168-181). */
typedef struct {
  double momentum[3];
  double energy;
  double mass;
  double max_cell_drift; /* valid when the step had MPCD_STEP_WANT_DRIFT */
  int64_t n;             /* particles this context collided in the step */
  int64_t step;          /* index of the step these describe */
  int64_t migrated;      /* of them, particles that moved to another domain */
} mpcd_diag;

typedef struct mpcd_ctx mpcd_ctx;

const char* mpcd_version(void);
const char* mpcd_last_error(void);

/* ---------------------------------------------------------------- engine */
int mpcd_ctx_create(const mpcd_config* cfg, mpcd_ctx** out);
int mpcd_ctx_destroy(mpcd_ctx* ctx);

/* Load n particles from HOST arrays in the reference layout: pos/vel (n,3)
 * float64 C-order, mass (n) float64 (ignored when uniform_mass), ids (n)
 * int64 (NULL = 0..n-1).  The state is then binned for step `step`.  Ids
 * must lie in [0, 2^32); a whole-box context requires a permutation of
 * 0..n-1 (else MPCD_ERR_CONFIG). */
int mpcd_upload(mpcd_ctx* ctx, const double* pos, const double* vel, const double* mass,
                const int64_t* ids, int64_t n, int64_t step, void* stream);

/* Copy the state to HOST arrays.  id_order=1 returns rows ordered by
 * particle id (Simulation.collect(), engine.py:599-607); id_order=0 returns
 * the engine's storage order (particle_sets()).  Any pointer may be NULL. */
int mpcd_download(mpcd_ctx* ctx, double* pos, double* vel, double* mass, int64_t* ids,
                  int32_t id_order, void* stream);

int64_t mpcd_count(const mpcd_ctx* ctx);
/* Record slots per cell region (fixed-capacity cell layout). */
int64_t mpcd_cell_capacity(const mpcd_ctx* ctx);
/* Cells per k_step tile (16, 8 or 4), chosen from capacity / cells so that
 * tiles too full for shared-memory staging stay rare at any density. */
int32_t mpcd_tile_cells(const mpcd_ctx* ctx);
int64_t mpcd_current_step(const mpcd_ctx* ctx);

/* One collision + streaming step with index `step` (the reference's
 * Simulation.step() with step_index == step).  Asynchronous on `stream`;
 * diagnostics stay on the device until mpcd_read_diag. */
int mpcd_step(mpcd_ctx* ctx, int64_t step, int32_t flags, void* stream);

/* n_steps consecutive steps first_step, first_step+1, ... without host
 * synchronisation (diagnostics of the last step are kept). */
int mpcd_run(mpcd_ctx* ctx, int64_t first_step, int64_t n_steps, int32_t flags, void* stream);

/* Diagnostics of the most recent step (synchronises `stream`). */
int mpcd_read_diag(mpcd_ctx* ctx, mpcd_diag* out, void* stream);

/* com capture of the most recent step: occupied cell ids (ascending) and
 * their com velocities (k,3).  Pass NULL buffers to get k in *n_occupied. */
int mpcd_read_com(mpcd_ctx* ctx, int64_t* cell_ids, double* com, int64_t* n_occupied,
                  void* stream);

/* The binning of the state for the step about to run, as the reference's
 * LinkedCellList (collision.py:39-80): cells (n, per particle id), bin_count
 * and bin_offset (ncells), permutation (n) in particle-id space (stable
 * argsort of cells over id order).  Requires ids == 0..n-1. */
int mpcd_read_binning(mpcd_ctx* ctx, int64_t* cells, int64_t* bin_count, int64_t* bin_offset,
                      int64_t* permutation, void* stream);

/* Pure-function boundary serial_collision_step (engine.py:415-455) on HOST
 * buffers: pos/vel (n,3) are read and overwritten in id order.  drift may be
 * NULL.  Uses ctx's device workspace (capacity >= n). */
int mpcd_step_host(mpcd_ctx* ctx, double* pos, double* vel, const double* mass, int64_t n,
                   int64_t step, int32_t flags, double* drift, void* stream);

/* Out-of-place form of mpcd_step_host: reads pos_in/vel_in, writes the
 * stepped rows (input order) to pos_out/vel_out (which may alias the
 * inputs).  Page-locked buffers (mpcd_host_alloc, cudaHostAlloc/Register)
 * move by DMA in 8 Mi-row chunks on a copy stream, each chunk binned (input)
 * or produced (output) by a kernel while the next is in flight; below 2 Mi
 * rows the kernels read and write them in place over PCIe.  Pageable
 * buffers are staged through device memory.  Returns after the output rows
 * are on the host. */
int mpcd_step_rows(mpcd_ctx* ctx, const double* pos_in, const double* vel_in, const double* mass,
                   int64_t n, int64_t step, int32_t flags, double* pos_out, double* vel_out,
                   double* drift, void* stream);

/* Page-locked, device-mapped host memory for the pure-function boundary's
 * rows (the host shim pools these blocks), and whether a host pointer is
 * page-locked (1) or pageable (0). */
int mpcd_host_alloc(int64_t bytes, void** out);
int mpcd_host_free(void* ptr);
int mpcd_host_is_pinned(const void* ptr);

/* Device init (particles.py:101-127 positions bit-exact; velocities are
 * Box-Muller with device log/cos, equal to numpy's only within ~1 ulp). */
int mpcd_init_device(mpcd_ctx* ctx, int64_t n, double velocity_variance, int64_t step,
                     void* stream);

/* Per-kernel CUDA-event timing of subsequent mpcd_step/mpcd_run calls
 * (enable=0 stops and clears).  mpcd_read_profile synchronises and returns
 * the summed milliseconds per kernel slot, MPCD_PROFILE_SLOTS entries:
 * [0] k_step (the tile kernel), [1] k_step_dense, [2] diagnostics
 * reduction (k_diag_partial + k_diag_finalize), [3], [4] reserved (0). */
#define MPCD_PROFILE_SLOTS 5
int mpcd_profile(mpcd_ctx* ctx, int32_t enable);
int mpcd_read_profile(mpcd_ctx* ctx, double* ms, int64_t* n_steps);

/* ---------------------------------------------- decomposed box (backend nccl)
 * The reference's parallel path splits the box over a rank grid
 * (decomposition.py:20-146, SimParams.rank_dims) and runs per-rank phases
 * with halo moment exchange and particle migration (engine.py:190-272,
 * exchange.py:225-506).  Here a rank owns the cells of its block of the
 * SHIFTED grid of each step and every particle in them, so a cell is never
 * split between ranks: no moment exchange, and the trajectory is
 * bit-identical to the whole-box step.  After mpcd_step the particles whose
 * next-step cell belongs to another rank sit in per-destination send
 * buffers; the caller moves them (NCCL / gloo / device copies) and hands the
 * received ones to mpcd_absorb before the next step.
 *
 * The context's cfg.dims are the domain's cells; global_dims = rank_dims *
 * dims; rank = (bx * rank_dims[1] + by) * rank_dims[2] + bz owns cells
 * [b * dims, (b + 1) * dims) per axis.  After set_domain, mpcd_upload and
 * mpcd_init_device take the WHOLE box's particles and keep this domain's. */
typedef struct {
  int64_t global_dims[3];
  int32_t rank_dims[3];
  int32_t rank;
  int64_t send_capacity; /* records per destination rank; 0 = default */
} mpcd_domain;

/* Send side of the exchange (device pointers owned by the context).
 * send + (d * send_capacity + i) * record_bytes is the i-th record for rank
 * d, i < send_n[d] after mpcd_step (send_n[d] > send_capacity means the
 * buffer overflowed and the step is lost: MPCD_ERR_CAPACITY for the caller).
 * Record: double x, y, z; uint32 id, pad; double vx, vy, vz, m (64 bytes). */
typedef struct {
  void* send;
  unsigned long long* send_n;
  int64_t send_capacity;
  int32_t n_ranks;
  int32_t record_bytes;
} mpcd_exchange;

int mpcd_ctx_set_domain(mpcd_ctx* ctx, const mpcd_domain* dom);
int mpcd_exchange_buffers(mpcd_ctx* ctx, mpcd_exchange* out);
/* Bin n_recv received DEVICE records for the next step, account for the
 * n_sent this domain gave away, and clear send_n. */
int mpcd_absorb(mpcd_ctx* ctx, const void* recs, int64_t n_recv, int64_t n_sent, void* stream);

/* Fused migration (the B200 path): instead of send buffers, k_step writes a
 * leaving particle straight into its new owner's next-step cell region --
 * slot claimed by an atomic on the owner's count, record stored -- over peer
 * memory (NVLink P2P stores and atomics between GPUs of a node).  After
 * connecting, mpcd_step alone advances the domain; no mpcd_absorb.  The
 * caller fences every step across ranks (e.g. a one-element NCCL all-reduce
 * enqueued on the stream after mpcd_step): all ranks' step k must complete
 * before any rank's step k+1 reads its cells.
 *
 * mpcd_ipc_handles exports this context's region / count / overflow
 * allocations as CUDA IPC handles (*nbytes bytes; out = NULL asks the size);
 * mpcd_connect_peers takes every rank's handles concatenated in rank order
 * and opens the others'.  Each rank's blob ends with its domain geometry
 * (cells, slots per cell, overflow capacity); connecting requires equal
 * geometry on every rank (else MPCD_ERR_TOPOLOGY, nothing opened: use the
 * exchange).  Domains of one process (one GPU or several)
 * connect directly with mpcd_connect_local(ctxs[rank], n). */
int mpcd_ipc_handles(mpcd_ctx* ctx, void* out, int64_t* nbytes);
int mpcd_connect_peers(mpcd_ctx* ctx, const void* all_handles, int32_t n_ranks);
int mpcd_connect_local(mpcd_ctx* const* ctxs, int32_t n);

/* ------------------------------------------------------ host RNG helpers */
uint64_t mpcd_key_state(uint64_t seed, uint64_t step, uint64_t purpose, uint64_t cell);
double mpcd_uniform_at(uint64_t state, uint64_t index);
void mpcd_grid_shift(int32_t prng, uint64_t seed, uint64_t step, double cell_size, double out[3]);

/* ---------------------------------------------- stage entry points (device) */
/* rng.sample_uniform / uniform_at stream (rng.py:84-110) */
int mpcd_stage_sample_uniform(int32_t prng, uint64_t seed, uint64_t step, uint64_t purpose,
                              uint64_t cell, int64_t count, double* out, void* stream);
/* collision.build_linked_cells (collision.py:112-147).  err (host, 2) gets
 * {particle_index, dimension} on MPCD_ERR_BINNING. */
int mpcd_stage_build_linked_cells(const double* pos, int64_t n, double cell_size,
                                  const double grid_min[3], const int64_t dims[3],
                                  const int32_t wrap[3], int64_t* cells, int64_t* bin_count,
                                  int64_t* bin_offset, int64_t* permutation, int64_t err[2],
                                  void* stream);
/* collision.linked_cells_from_indices structure (collision.py:150-163) */
int mpcd_stage_structure_from_cells(const int64_t* cells, int64_t n, int64_t n_cells,
                                    int64_t* bin_count, int64_t* bin_offset,
                                    int64_t* permutation, void* stream);
/* collision.segment_moments (collision.py:190-206) -> (n_cells,4) */
int mpcd_stage_segment_moments(const int64_t* permutation, const int64_t* bin_count,
                               const int64_t* bin_offset, int64_t n_cells, const double* vel,
                               const double* mass, int64_t n, double* moments, void* stream);
/* collision.finalize_com (collision.py:209-214) */
int mpcd_stage_finalize_com(const double* moments, int64_t n_cells, double* com, void* stream);
/* collision.sample_rotation_axes (collision.py:217-250) */
int mpcd_stage_rotation_axes(int32_t prng, uint64_t seed, int64_t step, const int64_t* cell_ids,
                             int64_t k, double* axes, void* stream);
/* collision.rotate_velocities (collision.py:289-306), per-particle com/axis */
int mpcd_stage_rotate(const double* vel, const double* com_pp, const double* axis_pp, int64_t n,
                      double cos_alpha, double sin_alpha, double* out, void* stream);
/* collision.rotate_cell_velocities (collision.py:309-324) */
int mpcd_stage_rotate_cells(const int64_t* cells, const double* vel, const double* com,
                            const double* axes, int64_t n, double cos_alpha, double sin_alpha,
                            double* out, void* stream);
/* particles.wrap_coordinates (particles.py:52-59), elementwise */
int mpcd_stage_wrap(const double* x, int64_t count, double box, double* out, void* stream);
/* particles.stream_and_wrap (particles.py:62-67), per-axis box */
int mpcd_stage_stream_wrap(const double* pos, const double* vel, int64_t n, double dt,
                           const double box[3], double* out, void* stream);
/* collision.cell_momentum_drift (collision.py:327-344) -> *out (host) */
int mpcd_stage_cell_drift(const double* before, const double* after, int64_t n_cells,
                          double* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MPCD_H_ */
