// mpcd_engine.cu -- the B200 SRD engine context and its C ABI (include/mpcd.h).
//
// State in HBM: fixed-capacity cell regions (mpcd_step.cuh) double-buffered
// between "this step's binning" and "the next step's binning", the per-cell
// counts of both, and the overflow lists.  One step (engine.py:415-455 for
// the whole box) is
//
//   k_step         persistent, warp-specialised: a producer warp stages each
//                  16-cell tile with TMA bulk copies and draws its keyed
//                  Marsaglia axes; each of 4 consumer warps takes 4 cells:
//                  rank by id inside each cell (the reference's stable
//                  argsort over id order), reduce (m v, m) in numpy's
//                  reduceat association, com = p / m, Rodrigues rotation,
//                  stream + wrap, next-step cell; the particle is written into
//                  that cell's region (slot from an atomic on its count) --
//                  or, in a decomposed box, into another rank's send buffer
//                  or (fused migration) straight into that rank's region;
//                  conservation / drift partials per CTA.
//   k_step_dense   the rare tiles with a full cell (overflow) or too many rows.
//   k_diag_*       fixed-order reduction of the CTA partials.
//
// Algorithmic bytes per particle-step: read 64 + write 64 (records) and, per
// cell, read + zero its count and one atomic on the next count.  See
// DESIGN.md section 3.
#include <string.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include "mpcd_internal.h"
#include "mpcd_step.cuh"
#include "mpcd_launch.cuh"

namespace mpcd {

// -------------------------------------------------------- binning helpers --
__device__ __forceinline__ uint32_t flat_cell(double x, double y, double z, double o0, double o1,
                                              double o2, double a, int unit, int64_t L0,
                                              int64_t L1, int64_t L2) {
  const int64_t ix = pymod(cell_coord(x, o0, a, unit), L0);
  const int64_t iy = pymod(cell_coord(y, o1, a, unit), L1);
  const int64_t iz = pymod(cell_coord(z, o2, a, unit), L2);
  return (uint32_t)((ix * L1 + iy) * L2 + iz);
}

struct PlaceArgs {
  Recs reg;
  // multi-domain: keep only the particles whose cell lies in [org, org + L)
  // of the global G grid (strict: any other is a routing error, flags[3])
  int multi, strict;
  int64_t G0, G1, G2, org0, org1, org2;
  uint32_t* count;
  Recs ovf;
  uint32_t* ovf_cell;
  uint32_t* ovf_n;
  uint32_t ovf_cap;
  uint32_t cap;
  uint32_t* flags;
  double o0, o1, o2, a;
  int unit;
  int64_t L0, L1, L2;
};

// Returns 1 when the particle was placed in this domain.
__device__ __forceinline__ int place_one(const PlaceArgs& P, double x, double y, double z,
                                         uint32_t id, double vx, double vy, double vz, double m) {
  uint32_t c;
  if (P.multi) {
    const int64_t lx = pymod(cell_coord(x, P.o0, P.a, P.unit), P.G0) - P.org0;
    const int64_t ly = pymod(cell_coord(y, P.o1, P.a, P.unit), P.G1) - P.org1;
    const int64_t lz = pymod(cell_coord(z, P.o2, P.a, P.unit), P.G2) - P.org2;
    if ((uint64_t)lx >= (uint64_t)P.L0 || (uint64_t)ly >= (uint64_t)P.L1 ||
        (uint64_t)lz >= (uint64_t)P.L2) {
      if (P.strict) atomicOr(&P.flags[3], 1u);
      return 0;
    }
    c = (uint32_t)((lx * P.L1 + ly) * P.L2 + lz);
  } else {
    c = flat_cell(x, y, z, P.o0, P.o1, P.o2, P.a, P.unit, P.L0, P.L1, P.L2);
  }
  const uint32_t s = atomicAdd(&P.count[c], 1u);
  if (s < P.cap) {
    store_rec(P.reg, (uint64_t)c * P.cap + s, x, y, z, id, vx, vy, vz, m);
  } else {
    const uint32_t o = atomicAdd(P.ovf_n, 1u);
    if (o < P.ovf_cap) {
      store_rec(P.ovf, o, x, y, z, id, vx, vy, vz, m);
      P.ovf_cell[o] = c;
    } else {
      atomicOr(&P.flags[2], 1u);
    }
  }
  return 1;
}

__device__ __forceinline__ void add_placed(const PlaceArgs& P, uint32_t* placed, uint32_t k) {
  if (placed && k) atomicAdd(placed, k);
}

// bin host rows ((n,3) positions/velocities) for step k
// (n,3) rows are read as whole contiguous chunks (kRowBlock rows per block
// iteration, staged in shared memory), so that the same kernel reads mapped
// pinned HOST memory over PCIe at full efficiency: the pure-function path
// bins its input straight from the caller's buffers (no H2D copy pass).
constexpr int kRowBlock = 256;

__device__ __forceinline__ void load_rows3(double* dst, const double* src, int64_t r0, int rows) {
  const int64_t base = 3 * r0;
  const int cnt = 3 * rows;
  for (int j = threadIdx.x; j < cnt; j += blockDim.x) dst[j] = src[base + j];
}

// row0: the rows are rows row0 .. row0 + n - 1 of the caller's arrays (their
// ids when `ids` is null); a pipelined upload bins one staged chunk at a time
__global__ void __launch_bounds__(kRowBlock) k_place_rows(const double* pos, const double* vel,
                                                          const double* mass, const int64_t* ids,
                                                          int64_t n, double m0, PlaceArgs P,
                                                          uint32_t* placed, int64_t row0 = 0) {
  __shared__ double sp[3 * kRowBlock], sv[3 * kRowBlock];
  uint32_t k = 0;
  for (int64_t r0 = (int64_t)blockIdx.x * kRowBlock; r0 < n; r0 += (int64_t)gridDim.x * kRowBlock) {
    const int rows = (int)min((int64_t)kRowBlock, n - r0);
    __syncthreads();
    load_rows3(sp, pos, r0, rows);
    load_rows3(sv, vel, r0, rows);
    __syncthreads();
    const int t = threadIdx.x;
    if (t < rows) {
      const int64_t i = r0 + t;
      k += place_one(P, sp[3 * t], sp[3 * t + 1], sp[3 * t + 2],
                     ids ? (uint32_t)ids[i] : (uint32_t)(row0 + i), sv[3 * t], sv[3 * t + 1],
                     sv[3 * t + 2], mass ? mass[i] : m0);
    }
  }
  add_placed(P, placed, k);
}

// insert particles received from other domains (64-byte records)
__global__ void k_place_xrecs(const XRec* r, int64_t n, PlaceArgs P) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const XRec q = r[i];
    place_one(P, q.p.x, q.p.y, q.p.z, q.p.id, q.v.vx, q.v.vy, q.v.vz, q.v.m);
  }
}

// bin flat records (rows 0..n-1 of a record array) for step k
__global__ void k_place_flat(Recs flat, int64_t n, PlaceArgs P) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const PRec p = flat.p[i];
    const VRec v = flat.v[i];
    place_one(P, p.x, p.y, p.z, p.id, v.vx, v.vy, v.vz, v.m);
  }
}

// particles resident in region set b: sum of min(count, cap) + overflow entries
__global__ void k_count_resident(const uint32_t* count, int64_t C, uint32_t cap,
                                 const uint32_t* ovf_n, uint32_t ovf_cap,
                                 unsigned long long* out) {
  unsigned long long s = 0;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < C;
       c += (int64_t)gridDim.x * blockDim.x)
    s += min(count[c], cap);
  if (blockIdx.x == 0 && threadIdx.x == 0) s += min(*ovf_n, ovf_cap);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

__global__ void k_clamp_counts(const uint32_t* count, int64_t C, uint32_t cap, uint32_t* out) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < C;
       c += (int64_t)gridDim.x * blockDim.x)
    out[c] = min(count[c], cap);
}

// Binned state -> flat records.  Region rows go to offs[c] + slot (cell-major
// storage order), overflow entries follow in list order; with by_id the
// destination row is the particle id instead.
__global__ void k_flatten(Recs reg, const uint32_t* count, int64_t C, uint32_t cap,
                          const uint32_t* offs, Recs ovf, uint32_t n_ovf, uint32_t n_reg,
                          int by_id, Recs flat) {
  const int64_t total = C * (int64_t)cap;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total + n_ovf;
       q += (int64_t)gridDim.x * blockDim.x) {
    PRec p;
    VRec v;
    uint64_t dst;
    if (q < total) {
      const int64_t c = q / cap;
      const uint32_t s = (uint32_t)(q - c * cap);
      if (s >= min(count[c], cap)) continue;
      p = reg.p[q];
      v = reg.v[q];
      dst = by_id ? p.id : (uint64_t)offs[c] + s;
    } else {
      const uint32_t o = (uint32_t)(q - total);
      p = ovf.p[o];
      v = ovf.v[o];
      dst = by_id ? p.id : (uint64_t)n_reg + o;
    }
    flat.p[dst] = p;
    flat.v[dst] = v;
  }
}

// flat records -> host row layout
// flat records -> (n,3) rows written as contiguous chunks (device or mapped
// pinned host memory: the pure-function path writes the caller's buffers
// directly, no D2H copy pass)
__global__ void __launch_bounds__(kRowBlock) k_flat_to_rows_chunked(Recs flat, int64_t n,
                                                                    double* pos, double* vel) {
  __shared__ double sp[3 * kRowBlock], sv[3 * kRowBlock];
  for (int64_t r0 = (int64_t)blockIdx.x * kRowBlock; r0 < n; r0 += (int64_t)gridDim.x * kRowBlock) {
    const int rows = (int)min((int64_t)kRowBlock, n - r0);
    const int t = threadIdx.x;
    __syncthreads();
    if (t < rows) {
      const PRec p = flat.p[r0 + t];
      const VRec v = flat.v[r0 + t];
      sp[3 * t] = p.x; sp[3 * t + 1] = p.y; sp[3 * t + 2] = p.z;
      sv[3 * t] = v.vx; sv[3 * t + 1] = v.vy; sv[3 * t + 2] = v.vz;
    }
    __syncthreads();
    for (int j = t; j < 3 * rows; j += blockDim.x) {
      pos[3 * r0 + j] = sp[j];
      vel[3 * r0 + j] = sv[j];
    }
  }
}

__global__ void k_flat_to_rows(Recs flat, int64_t n, double* pos, double* vel, double* mass,
                               int64_t* ids, int uniform_mass, double m0) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const PRec p = flat.p[i];
    const VRec v = flat.v[i];
    if (pos) { pos[3 * i] = p.x; pos[3 * i + 1] = p.y; pos[3 * i + 2] = p.z; }
    if (vel) { vel[3 * i] = v.vx; vel[3 * i + 1] = v.vy; vel[3 * i + 2] = v.vz; }
    if (mass) mass[i] = uniform_mass ? m0 : v.m;
    if (ids) ids[i] = (int64_t)p.id;
  }
}

// LinkedCellList of the binning in id space: cells[id], and the permutation
// (each cell's ids ascending at its bin_offset).
__global__ void k_binning_debug(Recs reg, const uint32_t* count, int64_t C, uint32_t cap,
                                Recs ovf, const uint32_t* ovf_cell, uint32_t n_ovf,
                                const int64_t* offs, int64_t* cells, int64_t* perm) {
  const int64_t total = C * (int64_t)cap;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total + n_ovf;
       q += (int64_t)gridDim.x * blockDim.x) {
    int64_t c;
    uint32_t me;
    if (q < total) {
      c = q / cap;
      if ((uint32_t)(q - c * cap) >= min(count[c], cap)) continue;
      me = reg.p[q].id;
    } else {
      c = ovf_cell[q - total];
      me = ovf.p[q - total].id;
    }
    uint32_t rank = 0;
    const uint32_t k = min(count[c], cap);
    for (uint32_t s = 0; s < k; ++s) rank += (reg.p[(uint64_t)c * cap + s].id < me) ? 1u : 0u;
    if (count[c] > cap)
      for (uint32_t o = 0; o < n_ovf; ++o)
        if (ovf_cell[o] == (uint32_t)c && ovf.p[o].id < me) ++rank;
    if (cells) cells[me] = c;
    if (perm) perm[offs[c] + rank] = (int64_t)me;
  }
}

__global__ void k_widen_counts(const uint32_t* count, int64_t C, int64_t* out) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < C;
       c += (int64_t)gridDim.x * blockDim.x)
    out[c] = (int64_t)count[c];
}

// particles.py:101-127 on the device: positions exact (integer hash * box),
// velocities through device log/cos (numpy agrees to ~1 ulp only).  Two
// passes over the particle ids, so nothing is staged: k_init_sum reduces the
// velocities (fixed grid and order: every domain of a decomposed box gets the
// same mean bits), k_init_place regenerates each particle, removes the mean
// (particles.py mean_init_velocity) and bins it for the first step -- in a
// decomposed box only the particles of this domain's cells.
constexpr int kInitBlocks = 148 * 8;

__device__ __forceinline__ void init_velocity(uint64_t state, int64_t n, int64_t i, double sigma,
                                              double v[3]) {
  const double two_pi = 2.0 * 3.141592653589793;
  for (int d = 0; d < 3; ++d) {
    const uint64_t g = (uint64_t)(3 * n + 3 * i + d);
    const double u1 = uniform_at(state, 2 * g), u2 = uniform_at(state, 2 * g + 1);
    v[d] = sqrt(-2.0 * log(1.0 - u1)) * cos(two_pi * u2) * sigma;
  }
}

__global__ void __launch_bounds__(256) k_init_sum(int64_t n, uint64_t state, double sigma,
                                                  double* vsum_partials) {
  __shared__ double s_sum[3][256];
  double acc[3] = {0, 0, 0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v[3];
    init_velocity(state, n, i, sigma, v);
    for (int d = 0; d < 3; ++d) acc[d] += v[d];
  }
  for (int d = 0; d < 3; ++d) s_sum[d][threadIdx.x] = acc[d];
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w)
      for (int d = 0; d < 3; ++d) s_sum[d][threadIdx.x] += s_sum[d][threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int d = 0; d < 3; ++d) vsum_partials[blockIdx.x * 3 + d] = s_sum[d][0];
}

__global__ void __launch_bounds__(256) k_init_place(int64_t n, uint64_t state, double b0,
                                                    double b1, double b2, double sigma,
                                                    double m0, const double* vsum_partials,
                                                    int nblocks, PlaceArgs P,
                                                    uint32_t* placed) {
  __shared__ double mean[3];
  if (threadIdx.x < 3) {
    double acc = 0.0;
    for (int b = 0; b < nblocks; ++b) acc += vsum_partials[b * 3 + threadIdx.x];
    mean[threadIdx.x] = n ? acc / (double)n : 0.0;
  }
  __syncthreads();
  uint32_t k = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v[3];
    init_velocity(state, n, i, sigma, v);
    k += place_one(P, uniform_at(state, (uint64_t)(3 * i)) * b0,
                   uniform_at(state, (uint64_t)(3 * i + 1)) * b1,
                   uniform_at(state, (uint64_t)(3 * i + 2)) * b2, (uint32_t)i, v[0] - mean[0],
                   v[1] - mean[1], v[2] - mean[2], m0);
  }
  add_placed(P, placed, k);
}

}  // namespace mpcd

// =============================================================== context ==
using namespace mpcd;

struct mpcd_ctx {
  mpcd_config cfg;
  int64_t C = 0, ntiles = 0, n = 0;
  // every id of the (global) system is below this: set by upload / device
  // init, which take the whole box's particles on every domain
  int64_t id_bound = 0;
  // pipelined host transfers (pinned host rows): a copy stream, two staging
  // chunks, and the events that hand each chunk between the two streams
  cudaStream_t copy_st = nullptr;
  cudaEvent_t xfer_ev[4] = {nullptr, nullptr, nullptr, nullptr};
  double* xfer_buf = nullptr;
  uint32_t cap = 0, ovf_cap = 0, scratch_cap = 0;
  int tc = kTC;            // cells per tile of k_step (chosen from the density)
  uint32_t np_smem = 0;    // dense-tile particles staged in shared memory
  bool poisoned = false;   // particles were lost (capacity): steps refuse
  int dev = 0;
  void* slab[2] = {nullptr, nullptr};
  Recs reg[2];
  uint32_t* count[2] = {nullptr, nullptr};
  void* ovf_slab[2] = {nullptr, nullptr};
  Recs ovf[2];
  uint32_t* ovf_cell[2] = {nullptr, nullptr};
  // [0..3] flags, [4,5] ovf_n, [6] scratch_n, [7] placed, [8] overflow
  // bucket allocator, [9] dense staging exhausted, [10] a cell above the
  // dense kernel's ranking limit
  uint32_t* small = nullptr;
  uint32_t* dense = nullptr;
  uint32_t* dense_bits = nullptr;
  uint32_t* cell_aux = nullptr;
  uint32_t* ovf_sorted = nullptr;
  uint32_t* scratch_id = nullptr;
  uint32_t* scratch_src = nullptr;
  double* scratch_val = nullptr;
  double* partials = nullptr;
  double* level1 = nullptr;
  double* diag = nullptr;
  double* com_cap = nullptr;  // allocated on the first capture_com step
  unsigned long long* drift_bits = nullptr;
  ScanState scan;
  int cur = 0;
  // state: binned in reg[cur] (for cur_step) or flat rows in reg[flat]
  bool binned = false;
  int flat = -1;
  int64_t cur_step = 0;
  bool have_diag = false;
  bool last_com = false;
  int64_t last_step = -1;
  bool prof = false;
  std::vector<cudaEvent_t> prof_events;
  // multi-domain (mpcd_ctx_set_domain): cfg.dims are this domain's cells
  bool multi = false;
  mpcd_domain dom{};
  int64_t org[3] = {0, 0, 0};
  XRec* send = nullptr;
  unsigned long long* send_n = nullptr;
  // fused migration (mpcd_connect_peers / mpcd_connect_local)
  bool p2p = false;
  bool n_stale = false;      // c->n unknown on the host since the last fused step
  PeerBufs* d_peers = nullptr;
  std::vector<void*> ipc_opened;
};

namespace {

constexpr int kProfSlots = 3;  // step, step_dense, diagnostics

uint32_t* flags_of(mpcd_ctx* c) { return c->small; }
uint32_t* ovf_n_of(mpcd_ctx* c, int b) { return c->small + 4 + b; }
uint32_t* scratch_n_of(mpcd_ctx* c) { return c->small + 6; }
uint32_t* placed_of(mpcd_ctx* c) { return c->small + 7; }
constexpr int kSmallWords = 16;

// partials rows: k_step's CTAs first, then one row per tile of k_step_dense
constexpr int64_t kMainRows = 4096;

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

Recs carve(void* slab, uint64_t rows) {
  Recs r;
  r.p = static_cast<PRec*>(slab);
  r.v = reinterpret_cast<VRec*>(static_cast<char*>(slab) + sizeof(PRec) * rows);
  return r;
}

// Cells per k_step tile: the largest multiple of kNCW (one consumer-warp
// share each) up to kTC whose padded tile (cells padded to 4 slots, ~1.5 per
// cell) stays within the kMaxPT staging slots with 2.5 standard deviations
// to spare -- so that dense tiles stay rare (measured: a few per mille of
// the tiles cost far less than the lane utilisation a smaller tile loses).
// 16 cells at 10 particles per cell; 8 from ~17; 4 from ~27.
// MPCD_TILE_CELLS overrides it (tuning and tests).
int tile_cells(double density) {
  if (const char* e = getenv("MPCD_TILE_CELLS")) {
    const int v = atoi(e);
    if (v >= kNCW && v <= kTC && v % kNCW == 0) return v;
  }
  for (int tc = kTC; tc > kNCW; tc -= kNCW)
    if (tc * (density + 1.5) + 2.5 * sqrt(tc * density) <= (double)kMaxPT) return tc;
  return kNCW;
}

// Poisson-tail default: the smallest multiple of 8 with an expected number of
// overflowing cells per step below ~1 (cap = 32 at 10 particles per cell).
uint32_t default_cap(double density, int64_t C) {
  if (density <= 0.0) density = 1.0;
  for (uint32_t cap = 16; cap < 4096; cap += 8) {
    // P(N > cap) for N ~ Poisson(density), by summing the pmf up to cap
    double term = exp(-density), cdf = term;
    for (uint32_t k = 1; k <= cap; ++k) {
      term *= density / k;
      cdf += term;
    }
    if ((1.0 - cdf) * (double)C < 1.0) return cap;
  }
  return 4096;
}

PlaceArgs place_args(mpcd_ctx* c, int b, int64_t step) {
  PlaceArgs P;
  const mpcd_config& g = c->cfg;
  P.reg = c->reg[b];
  P.count = c->count[b];
  P.ovf = c->ovf[b];
  P.ovf_cell = c->ovf_cell[b];
  P.ovf_n = ovf_n_of(c, b);
  P.ovf_cap = c->ovf_cap;
  P.cap = c->cap;
  P.flags = flags_of(c);
  double off[3];
  grid_shift(g.prng, g.seed, (uint64_t)step, g.cell_size, off);
  P.o0 = off[0]; P.o1 = off[1]; P.o2 = off[2];
  P.a = g.cell_size;
  P.unit = g.cell_size == 1.0;
  P.L0 = g.dims[0]; P.L1 = g.dims[1]; P.L2 = g.dims[2];
  P.multi = c->multi ? 1 : 0;
  P.strict = 0;
  P.G0 = c->multi ? c->dom.global_dims[0] : g.dims[0];
  P.G1 = c->multi ? c->dom.global_dims[1] : g.dims[1];
  P.G2 = c->multi ? c->dom.global_dims[2] : g.dims[2];
  P.org0 = c->org[0]; P.org1 = c->org[1]; P.org2 = c->org[2];
  return P;
}

// Device-usable address of a caller buffer: pinned (page-locked, UVA-mapped)
// host memory and device memory are read / written by the kernels in place;
// pageable host memory gives nullptr (the caller stages it).
template <class T>
T* mapped(T* p) {
  if (!p) return nullptr;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (a.type == cudaMemoryTypeHost && a.devicePointer) return static_cast<T*>(a.devicePointer);
  if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) return p;
  return nullptr;
}

// Particle ids are stored as u32; a whole-box context also writes row `id`
// of an n-row array when it downloads in id order, so its ids must be a
// permutation of 0..n-1 (a decomposed domain holds a subset of the global
// ids and sorts them on the host instead).
int validate_ids(const int64_t* ids, int64_t n, bool permutation, int64_t* bound) {
  std::vector<int64_t> copy;
  const int64_t* h = ids;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, ids) != cudaSuccess) {
    cudaGetLastError();
  } else if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) {
    copy.resize(n);
    MPCD_CUDA(cudaMemcpy(copy.data(), ids, sizeof(int64_t) * n, cudaMemcpyDefault));
    h = copy.data();
  }
  std::vector<uint8_t> seen(permutation ? n : 0, 0);
  int64_t top = -1;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t id = h[i];
    top = std::max(top, id);
    if (id < 0 || id >= (1LL << 32))
      return fail(MPCD_ERR_CONFIG, "particle id %lld (row %lld) outside [0, 2^32)", (long long)id,
                  (long long)i);
    if (permutation) {
      if (id >= n || seen[id])
        return fail(MPCD_ERR_CONFIG, "ids of a whole-box context must be a permutation of "
                    "0..n-1 (row %lld has id %lld)", (long long)i, (long long)id);
      seen[id] = 1;
    }
  }
  *bound = top + 1;
  return MPCD_OK;
}

// Refresh c->n after fused steps (peers added and removed particles).
int refresh_n(mpcd_ctx* c, cudaStream_t st) {
  if (!c->n_stale) return MPCD_OK;
  unsigned long long* d = nullptr;
  unsigned long long h = 0;
  MPCD_CUDA(cudaMallocAsync(&d, sizeof(*d), st));
  MPCD_CUDA(cudaMemsetAsync(d, 0, sizeof(*d), st));
  k_count_resident<<<grid_for(c->C, 256), 256, 0, st>>>(c->count[c->cur], c->C, c->cap,
                                                       ovf_n_of(c, c->cur), c->ovf_cap, d);
  MPCD_LAUNCH_CHECK();
  MPCD_CUDA(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, st));
  MPCD_CUDA(cudaFreeAsync(d, st));
  MPCD_CUDA(cudaStreamSynchronize(st));
  c->n = (int64_t)h;
  c->n_stale = false;
  return MPCD_OK;
}

// particles placed by the last filtered placement (multi-domain upload/init)
int read_placed(mpcd_ctx* c, cudaStream_t st, int64_t* out) {
  uint32_t h = 0;
  MPCD_CUDA(cudaMemcpyAsync(&h, placed_of(c), 4, cudaMemcpyDeviceToHost, st));
  MPCD_CUDA(cudaStreamSynchronize(st));
  *out = h;
  return MPCD_OK;
}

// Flatten the binned state of reg[cur] into rows of reg[cur ^ 1] (cell-major
// storage order, or by id).
int flatten(mpcd_ctx* c, bool by_id, cudaStream_t st) {
  const int b = c->cur;
  uint32_t n_ovf = 0, h_ovf = 0;
  MPCD_CUDA(cudaMemcpyAsync(&h_ovf, ovf_n_of(c, b), 4, cudaMemcpyDeviceToHost, st));
  MPCD_CUDA(cudaStreamSynchronize(st));
  n_ovf = std::min(h_ovf, c->ovf_cap);
  uint32_t* offs = nullptr;
  uint32_t n_reg = (uint32_t)c->n - n_ovf;
  if (!by_id) {
    MPCD_CUDA(cudaMallocAsync(&offs, sizeof(uint32_t) * 2 * c->C, st));
    k_clamp_counts<<<grid_for(c->C, 256), 256, 0, st>>>(c->count[b], c->C, c->cap, offs + c->C);
    MPCD_LAUNCH_CHECK();
    int rc = scan_u32(c->scan, offs + c->C, offs, nullptr, c->C, false, st);
    if (rc) return rc;
  }
  const int64_t work = c->C * (int64_t)c->cap + n_ovf;
  k_flatten<<<grid_for(work, 256), 256, 0, st>>>(c->reg[b], c->count[b], c->C, c->cap, offs,
                                                 c->ovf[b], n_ovf, n_reg, by_id ? 1 : 0,
                                                 c->reg[b ^ 1]);
  MPCD_LAUNCH_CHECK();
  if (offs) MPCD_CUDA(cudaFreeAsync(offs, st));
  // the binned copy is retired: zero its counts / overflow
  MPCD_CUDA(cudaMemsetAsync(c->count[b], 0, sizeof(uint32_t) * c->C, st));
  MPCD_CUDA(cudaMemsetAsync(ovf_n_of(c, b), 0, 4, st));
  c->binned = false;
  c->flat = b ^ 1;
  return MPCD_OK;
}

// Bin the flat rows of reg[flat] for step `step` into reg[flat ^ 1].
int place_flat(mpcd_ctx* c, int64_t step, cudaStream_t st) {
  const int b = c->flat ^ 1;
  if (c->n > 0) {
    PlaceArgs P = place_args(c, b, step);
    P.strict = 1;  // every resident particle is this domain's
    k_place_flat<<<grid_for(c->n, 256), 256, 0, st>>>(c->reg[c->flat], c->n, P);
    MPCD_LAUNCH_CHECK();
  }
  c->cur = b;
  c->binned = true;
  c->flat = -1;
  c->cur_step = step;
  return MPCD_OK;
}

int ensure_binned(mpcd_ctx* c, int64_t step, cudaStream_t st) {
  if (c->binned && c->cur_step == step) return MPCD_OK;
  if (c->binned) {
    int rc = flatten(c, false, st);
    if (rc) return rc;
  }
  return place_flat(c, step, st);
}

int check_flags(mpcd_ctx* c, cudaStream_t st) {
  uint32_t fl[kSmallWords];
  MPCD_CUDA(cudaMemcpyAsync(fl, flags_of(c), sizeof(fl), cudaMemcpyDeviceToHost, st));
  MPCD_CUDA(cudaStreamSynchronize(st));
  if (fl[1] || fl[2] || fl[3] || fl[9] || fl[10]) {
    cudaMemsetAsync(flags_of(c) + 1, 0, 3 * sizeof(uint32_t), st);
    cudaMemsetAsync(flags_of(c) + 9, 0, 2 * sizeof(uint32_t), st);
    if (fl[1]) return fail(MPCD_ERR_RNG, "axis rejection sampling failed to terminate");
    if (fl[3])
      return fail(MPCD_ERR_TOPOLOGY, "a particle given to domain %d lies outside its cells",
                  (int)c->dom.rank);
    c->poisoned = true;  // particles were dropped: the state is no longer the system
    if (fl[10])
      return fail(MPCD_ERR_CAPACITY, "a cell holds more than %u particles (the dense-tile "
                                     "kernel's ranking limit); particles were lost",
                  (unsigned)kDenseMaxCell);
    if (fl[9])
      return fail(MPCD_ERR_CAPACITY, "a cluster of full tiles exceeds the dense-tile staging "
                                     "capacity (%u particles); particles were lost",
                  c->scratch_cap);
    return fail(MPCD_ERR_CAPACITY, "overflow list full: more particles in full cells than the "
                                   "context's overflow capacity %u; particles were lost",
                c->ovf_cap);
  }
  return MPCD_OK;
}

StepArgs step_args(mpcd_ctx* c, int64_t step, bool by_id) {
  StepArgs A;
  const mpcd_config& g = c->cfg;
  const int b = c->cur;
  A.in = c->reg[b];
  A.out = c->reg[b ^ 1];
  A.count_in = c->count[b];
  A.count_out = c->count[b ^ 1];
  A.ovf_in = c->ovf[b];
  A.ovf_out = c->ovf[b ^ 1];
  A.ovf_cell_in = c->ovf_cell[b];
  A.ovf_cell_out = c->ovf_cell[b ^ 1];
  A.ovf_n_in = ovf_n_of(c, b);
  A.ovf_n_out = ovf_n_of(c, b ^ 1);
  A.ovf_cap = c->ovf_cap;
  A.cap = c->cap;
  A.partials = c->partials;
  A.com_cap = c->com_cap;
  A.drift_bits = c->drift_bits;
  A.flags = flags_of(c);
  A.dense = c->dense;
  A.dense_bits = c->dense_bits;
  A.cell_aux = c->cell_aux;
  A.ovf_sorted = c->ovf_sorted;
  A.scratch_n = scratch_n_of(c);
  A.scratch_id = c->scratch_id;
  A.scratch_val = c->scratch_val;
  A.scratch_src = c->scratch_src;
  A.scratch_cap = c->scratch_cap;
  A.np_smem = c->np_smem;
  // ranks by the sign of a 32-bit difference need every id below 2^31 - 1:
  // a whole-box context's ids are a permutation of 0..n-1, n <= capacity;
  // a domain's are the global system's (bound set by upload / device init)
  A.ids31 = (c->multi ? c->id_bound : g.capacity) <= (int64_t)kIds31Bound ? 1 : 0;
  A.tc = c->tc;
  A.cw = c->tc / kNCW;
  A.L0 = (int)g.dims[0]; A.L1 = (int)g.dims[1]; A.L2 = (int)g.dims[2];
  A.C = c->C;
  A.a = g.cell_size;
  A.dt = g.dt;
  A.cs = g.cos_alpha;
  A.sn = g.sin_alpha;
  A.box0 = (double)g.dims[0] * g.cell_size;
  A.box1 = (double)g.dims[1] * g.cell_size;
  A.box2 = (double)g.dims[2] * g.cell_size;
  double off[3];
  grid_shift(g.prng, g.seed, (uint64_t)(step + 1), g.cell_size, off);
  A.off_next0 = off[0]; A.off_next1 = off[1]; A.off_next2 = off[2];
  A.seed = g.seed;
  A.step = (uint64_t)step;
  A.prng = g.prng;
  A.axis_prefix = key_prefix(g.seed, (uint64_t)step, kAxis);
  A.m0 = g.mass_value;
  A.dense_row0 = kMainRows;
  (void)by_id;
  A.peers = c->p2p ? c->d_peers : nullptr;
  A.n_ranks = c->multi ? (int)((int64_t)c->dom.rank_dims[0] * c->dom.rank_dims[1] *
                               c->dom.rank_dims[2])
                       : 1;
  A.out_set = b ^ 1;
  if (c->multi) {
    A.G0 = (int)c->dom.global_dims[0]; A.G1 = (int)c->dom.global_dims[1];
    A.G2 = (int)c->dom.global_dims[2];
    A.o0 = (int)c->org[0]; A.o1 = (int)c->org[1]; A.o2 = (int)c->org[2];
    A.R1 = c->dom.rank_dims[1]; A.R2 = c->dom.rank_dims[2];
    A.box0 = (double)A.G0 * g.cell_size;
    A.box1 = (double)A.G1 * g.cell_size;
    A.box2 = (double)A.G2 * g.cell_size;
    A.send = c->send;
    A.send_n = c->send_n;
    A.send_cap = (uint32_t)c->dom.send_capacity;
  } else {
    A.G0 = A.L0; A.G1 = A.L1; A.G2 = A.L2;
    A.o0 = A.o1 = A.o2 = 0;
    A.R1 = A.R2 = 1;
    A.send = nullptr;
    A.send_n = nullptr;
    A.send_cap = 0;
  }
  return A;
}

// The k_step / k_step_dense variants are compiled in four translation units,
// one per step mode (mpcd_step_<mode>.cu, built in parallel).
int64_t launch_step_kernel(const StepArgs& A, int64_t nt, Variant v, int which, cudaStream_t st) {
  switch (v.mode) {
    case kById: return launch_mode_byid(A, nt, v, which, st);
    case kMulti: return launch_mode_multi(A, nt, v, which, st);
    case kFused: return launch_mode_fused(A, nt, v, which, st);
    default: return launch_mode_binned(A, nt, v, which, st);
  }
}

int launch_step(mpcd_ctx* c, int64_t step, int flags, bool by_id, cudaStream_t st) {
  if (c->poisoned)
    return fail(MPCD_ERR_CAPACITY, "the context lost particles in an earlier step (capacity "
                "exceeded); upload or initialise the state again");
  if (c->multi && !(c->binned && c->cur_step == step))
    return fail(MPCD_ERR_CONFIG, "a decomposed domain steps consecutively: it holds the "
                "particles of step %lld's cells, not of step %lld's",
                (long long)c->cur_step, (long long)step);
  int rc = ensure_binned(c, step, st);
  if (rc) return rc;
  const bool com = (flags & MPCD_STEP_WANT_COM) != 0;
  if (com && !c->com_cap) MPCD_CUDA(cudaMalloc(&c->com_cap, sizeof(double) * 4 * c->C));
  StepArgs A = step_args(c, step, by_id);
  cudaEvent_t* ev = nullptr;
  if (c->prof) {
    const size_t base = c->prof_events.size();
    c->prof_events.resize(base + kProfSlots + 1);
    ev = c->prof_events.data() + base;
    for (int i = 0; i <= kProfSlots; ++i) MPCD_CUDA(cudaEventCreate(&ev[i]));
    MPCD_CUDA(cudaEventRecord(ev[0], st));
  }
  const Variant v{c->cfg.cell_size == 1.0, c->cfg.uniform_mass != 0,
                  (flags & MPCD_STEP_WANT_DRIFT) != 0, com,
                  by_id ? kById : (c->multi ? (c->p2p ? kFused : kMulti) : kBinned)};
  const int64_t grid = launch_step_kernel(A, c->ntiles, v, 0, st);
  MPCD_LAUNCH_CHECK();
  if (grid > kMainRows) return fail(MPCD_ERR_CUDA, "step grid %lld exceeds its partials rows",
                                    (long long)grid);
  if (ev) MPCD_CUDA(cudaEventRecord(ev[1], st));
  // the dense-tile path: overflow buckets, then the dense-tile kernel (each
  // exits at once when k_step queued no tile)
  k_dense_prep<<<grid_for(c->ntiles, 256, kDenseGrid), 256, 0, st>>>(A);
  k_ovf_bucket<<<(unsigned)kDenseGrid, 256, 0, st>>>(A);
  launch_step_kernel(A, c->ntiles, v, 1, st);
  MPCD_LAUNCH_CHECK();
  if (ev) MPCD_CUDA(cudaEventRecord(ev[2], st));
  k_diag_partial<<<kDiagBlocks, 256, 0, st>>>(c->partials, grid, kMainRows, c->ntiles,
                                              c->dense_bits, flags_of(c), c->level1);
  MPCD_LAUNCH_CHECK();
  k_diag_finalize<<<1, 32, 0, st>>>(c->level1, kDiagBlocks, c->drift_bits, c->diag, step,
                                    flags_of(c), ovf_n_of(c, c->cur), scratch_n_of(c));
  MPCD_LAUNCH_CHECK();
  if (ev) MPCD_CUDA(cudaEventRecord(ev[3], st));
  if (by_id) {
    c->binned = false;
    c->flat = c->cur ^ 1;
  } else {
    c->cur ^= 1;
    c->binned = true;
    c->cur_step = step + 1;
  }
  c->have_diag = true;
  c->last_com = com;
  c->last_step = step;
  if (c->p2p) c->n_stale = true;  // particles arrived from / left to peers
  return MPCD_OK;
}

int download_rows(mpcd_ctx* c, double* pos, double* vel, double* mass, int64_t* ids,
                  int32_t id_order, void* stream) {
  cudaStream_t st = as_stream(stream);
  {
    int rc = refresh_n(c, st);
    if (rc) return rc;
  }
  const int64_t n = c->n;
  if (n == 0) return MPCD_OK;
  Recs rows;
  Recs tmp_recs;
  void* tmp_slab = nullptr;
  if (c->binned) {
    // flatten into a scratch record array (the state stays binned)
    MPCD_CUDA(cudaMallocAsync(&tmp_slab, (size_t)n * 64, st));
    tmp_recs = carve(tmp_slab, n);
    const int b = c->cur;
    uint32_t h_ovf = 0;
    MPCD_CUDA(cudaMemcpyAsync(&h_ovf, ovf_n_of(c, b), 4, cudaMemcpyDeviceToHost, st));
    MPCD_CUDA(cudaStreamSynchronize(st));
    const uint32_t n_ovf = std::min(h_ovf, c->ovf_cap);
    uint32_t* offs = nullptr;
    if (!id_order) {
      MPCD_CUDA(cudaMallocAsync(&offs, sizeof(uint32_t) * 2 * c->C, st));
      k_clamp_counts<<<grid_for(c->C, 256), 256, 0, st>>>(c->count[b], c->C, c->cap, offs + c->C);
      int rc = scan_u32(c->scan, offs + c->C, offs, nullptr, c->C, false, st);
      if (rc) return rc;
    }
    const int64_t work = c->C * (int64_t)c->cap + n_ovf;
    k_flatten<<<grid_for(work, 256), 256, 0, st>>>(c->reg[b], c->count[b], c->C, c->cap, offs,
                                                   c->ovf[b], n_ovf, (uint32_t)(n - n_ovf),
                                                   id_order ? 1 : 0, tmp_recs);
    MPCD_LAUNCH_CHECK();
    if (offs) MPCD_CUDA(cudaFreeAsync(offs, st));
    rows = tmp_recs;
  } else {
    rows = c->reg[c->flat];  // flat rows are in id order already
  }
  double* tmp = nullptr;
  MPCD_CUDA(cudaMallocAsync(&tmp, (size_t)n * 8 * 8, st));
  double* dpos = tmp;
  double* dvel = tmp + 3 * n;
  double* dmass = tmp + 6 * n;
  int64_t* dids = reinterpret_cast<int64_t*>(tmp + 7 * n);
  k_flat_to_rows<<<grid_for(n, 256), 256, 0, st>>>(rows, n, pos ? dpos : nullptr,
                                                   vel ? dvel : nullptr, mass ? dmass : nullptr,
                                                   ids ? dids : nullptr, c->cfg.uniform_mass,
                                                   c->cfg.mass_value);
  MPCD_LAUNCH_CHECK();
  if (pos) MPCD_CUDA(cudaMemcpyAsync(pos, dpos, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, st));
  if (vel) MPCD_CUDA(cudaMemcpyAsync(vel, dvel, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, st));
  if (mass) MPCD_CUDA(cudaMemcpyAsync(mass, dmass, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  if (ids) MPCD_CUDA(cudaMemcpyAsync(ids, dids, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, st));
  MPCD_CUDA(cudaFreeAsync(tmp, st));
  if (tmp_slab) MPCD_CUDA(cudaFreeAsync(tmp_slab, st));
  MPCD_CUDA(cudaStreamSynchronize(st));
  return MPCD_OK;
}


// Multi-domain download: storage order, then rows sorted by (global) id on
// the host when id_order is asked for.
int download_multi(mpcd_ctx* c, double* pos, double* vel, double* mass, int64_t* ids,
                   int32_t id_order, void* stream) {
  int rc0 = refresh_n(c, as_stream(stream));
  if (rc0) return rc0;
  const int64_t n = c->n;
  std::vector<double> hp(3 * n), hv(3 * n), hm(n);
  std::vector<int64_t> hi(n);
  int rc = download_rows(c, hp.data(), hv.data(), hm.data(), hi.data(), 0, stream);
  if (rc) return rc;
  std::vector<int64_t> order(n);
  for (int64_t i = 0; i < n; ++i) order[i] = i;
  if (id_order)
    std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return hi[a] < hi[b]; });
  for (int64_t r = 0; r < n; ++r) {
    const int64_t i = order[r];
    if (pos) for (int d = 0; d < 3; ++d) pos[3 * r + d] = hp[3 * i + d];
    if (vel) for (int d = 0; d < 3; ++d) vel[3 * r + d] = hv[3 * i + d];
    if (mass) mass[r] = hm[i];
    if (ids) ids[r] = hi[i];
  }
  return MPCD_OK;
}


}  // namespace

extern "C" {

int mpcd_ctx_create(const mpcd_config* cfg, mpcd_ctx** out) {
  clear_error();
  if (!cfg || !out) return fail(MPCD_ERR_CONFIG, "null argument");
  for (int d = 0; d < 3; ++d)
    if (cfg->dims[d] < 1 || cfg->dims[d] >= (1LL << 31))
      return fail(MPCD_ERR_CONFIG, "dims must be positive and < 2^31");
  const int64_t C = cfg->dims[0] * cfg->dims[1] * cfg->dims[2];
  if (C >= (1LL << 32)) return fail(MPCD_ERR_CONFIG, "more than 2^32 cells per context");
  if (!(cfg->cell_size > 0.0)) return fail(MPCD_ERR_CONFIG, "cell_size must be positive");
  if (cfg->capacity < 0 || cfg->capacity >= (1LL << 32) - 1)
    return fail(MPCD_ERR_CONFIG, "capacity must be in [0, 2^32-1)");
  if (cfg->prng < 0 || cfg->prng > 3) return fail(MPCD_ERR_CONFIG, "unknown prng %d", cfg->prng);
  DeviceGuard dg(cfg->device);
  {  // staging buffers of upload/download come from the stream-ordered pool:
     // keep what is freed instead of returning it to the OS at every sync
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, cfg->device) == cudaSuccess) {
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  mpcd_ctx* c = new mpcd_ctx();
  c->cfg = *cfg;
  c->dev = cfg->device;
  c->C = C;
  const int64_t cap_n = std::max<int64_t>(cfg->capacity, 1);
  const double density = (double)cap_n / (double)C;
  c->tc = tile_cells(density);
  c->ntiles = (C + c->tc - 1) / c->tc;
  // dense tiles of up to ~3x the expected tile population stage in shared
  // memory; larger ones (clusters) in HBM
  c->np_smem = (uint32_t)std::min<double>(4096.0, std::max<double>(1024.0, 3.0 * c->tc * density));
  uint32_t cap = default_cap((double)cap_n / (double)C, C);
  // flat rows 0..n-1 must fit in one region array
  cap = std::max<uint32_t>(cap, (uint32_t)((cap_n + C - 1) / C));
  c->cap = cap;
  // Clusters: the overflow lists (particles beyond their cell's cap) and the
  // HBM staging of oversized dense tiles take up to 1/4 and 1/2 of the
  // particles when HBM allows (1/16 and 1/8 at least); a cluster beyond that
  // fails loudly with MPCD_ERR_CAPACITY.
  {
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    const double regions = 2.0 * (double)C * cap * 64.0;
    const double spare = (double)free_b - regions - 4.0 * (1ull << 30);
    int shift = 2;  // n / 4 overflow entries, n / 2 staged rows
    // per particle of overflow capacity (n >> shift entries): 2 lists x (64 B
    // record + 4 B cell) + 4 B bucket index; of staging (n >> (shift - 1)
    // rows): 40 B
    while (shift < 4 && spare < (double)cap_n * (140.0 / (1 << shift) + 40.0 / (1 << (shift - 1))))
      ++shift;
    c->ovf_cap = (uint32_t)std::min<int64_t>(cap_n, std::max<int64_t>(cap_n >> shift, 1 << 16));
    c->scratch_cap =
        (uint32_t)std::min<int64_t>(cap_n, std::max<int64_t>(cap_n >> (shift - 1), 1 << 20));
    // densities where a typical tile exceeds the shared-memory staging
    // (hundreds of particles per cell): every tile may stage in HBM
    if (c->tc * density >= 0.5 * c->np_smem) c->scratch_cap = (uint32_t)cap_n;
  }
  auto cleanup = [&](int rc) {
    mpcd_ctx_destroy(c);
    return rc;
  };
  const uint64_t rows = (uint64_t)C * cap;
  for (int b = 0; b < 2; ++b) {
    if (cudaMalloc(&c->slab[b], rows * (sizeof(PRec) + sizeof(VRec))) != cudaSuccess)
      return cleanup(fail(MPCD_ERR_CUDA, "cudaMalloc of %llu region bytes failed",
                          (unsigned long long)(rows * 64)));
    c->reg[b] = carve(c->slab[b], rows);
    if (cudaMalloc(&c->count[b], sizeof(uint32_t) * C) != cudaSuccess ||
        cudaMalloc(&c->ovf_slab[b], (uint64_t)c->ovf_cap * 64) != cudaSuccess ||
        cudaMalloc(&c->ovf_cell[b], sizeof(uint32_t) * c->ovf_cap) != cudaSuccess)
      return cleanup(fail(MPCD_ERR_CUDA, "cudaMalloc of counts / overflow failed"));
    c->ovf[b] = carve(c->ovf_slab[b], c->ovf_cap);
    cudaMemset(c->count[b], 0, sizeof(uint32_t) * C);
  }
  if (cudaMalloc(&c->small, sizeof(uint32_t) * kSmallWords) != cudaSuccess ||
      cudaMalloc(&c->dense, sizeof(uint32_t) * c->ntiles) != cudaSuccess ||
      cudaMalloc(&c->dense_bits, sizeof(uint32_t) * ((c->ntiles + 31) / 32)) != cudaSuccess ||
      cudaMalloc(&c->cell_aux, sizeof(uint32_t) * C) != cudaSuccess ||
      cudaMalloc(&c->ovf_sorted, sizeof(uint32_t) * c->ovf_cap) != cudaSuccess ||
      cudaMalloc(&c->scratch_id, sizeof(uint32_t) * c->scratch_cap) != cudaSuccess ||
      cudaMalloc(&c->scratch_src, sizeof(uint32_t) * c->scratch_cap) != cudaSuccess ||
      cudaMalloc(&c->scratch_val, sizeof(double) * 4 * c->scratch_cap) != cudaSuccess ||
      cudaMalloc(&c->partials, sizeof(double) * 8 * (c->ntiles + kMainRows)) != cudaSuccess ||
      cudaMalloc(&c->level1, sizeof(double) * kDiagCols * kDiagBlocks) != cudaSuccess ||
      cudaMalloc(&c->diag, sizeof(double) * 16) != cudaSuccess ||
      cudaMalloc(&c->drift_bits, sizeof(unsigned long long)) != cudaSuccess)
    return cleanup(fail(MPCD_ERR_CUDA, "cudaMalloc of per-tile arrays failed"));
  cudaMemset(c->small, 0, sizeof(uint32_t) * kSmallWords);
  cudaMemset(c->dense_bits, 0, sizeof(uint32_t) * ((c->ntiles + 31) / 32));
  cudaMemset(c->diag, 0, sizeof(double) * 16);
  cudaMemset(c->drift_bits, 0, sizeof(unsigned long long));
  int rc = c->scan.init(C);
  if (rc) return cleanup(rc);
  if (cudaDeviceSynchronize() != cudaSuccess)
    return cleanup(fail(MPCD_ERR_CUDA, "context init failed: %s",
                        cudaGetErrorString(cudaGetLastError())));
  *out = c;
  return MPCD_OK;
}

int mpcd_ctx_destroy(mpcd_ctx* c) {
  if (!c) return MPCD_OK;
  DeviceGuard dg(c->dev);
  for (int b = 0; b < 2; ++b) {
    if (c->slab[b]) cudaFree(c->slab[b]);
    if (c->count[b]) cudaFree(c->count[b]);
    if (c->ovf_slab[b]) cudaFree(c->ovf_slab[b]);
    if (c->ovf_cell[b]) cudaFree(c->ovf_cell[b]);
  }
  void* ptrs[] = {c->small, c->dense, c->dense_bits, c->cell_aux, c->ovf_sorted,
                  c->scratch_id, c->scratch_src, c->scratch_val,
                  c->partials, c->level1, c->diag, c->com_cap, c->drift_bits};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (cudaEvent_t e : c->prof_events) cudaEventDestroy(e);
  for (cudaEvent_t e : c->xfer_ev)
    if (e) cudaEventDestroy(e);
  if (c->copy_st) cudaStreamDestroy(c->copy_st);
  if (c->xfer_buf) cudaFree(c->xfer_buf);
  if (c->send) cudaFree(c->send);
  if (c->send_n) cudaFree(c->send_n);
  if (c->d_peers) cudaFree(c->d_peers);
  for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
  c->scan.release();
  delete c;
  return MPCD_OK;
}

int64_t mpcd_count(const mpcd_ctx* c) {
  if (!c) return -1;
  if (c->n_stale) {  // after fused steps: count on the device (synchronises the null stream)
    DeviceGuard dg(c->dev);
    if (refresh_n(const_cast<mpcd_ctx*>(c), nullptr)) return -1;
  }
  return c->n;
}
int64_t mpcd_current_step(const mpcd_ctx* c) { return c ? c->cur_step : -1; }
int64_t mpcd_cell_capacity(const mpcd_ctx* c) { return c ? (int64_t)c->cap : -1; }
int32_t mpcd_tile_cells(const mpcd_ctx* c) { return c ? (int32_t)c->tc : -1; }

// ------------------------------------------- pipelined host transfers ---
// Pinned host rows move by DMA (cudaMemcpyAsync on a copy stream) in chunks,
// each binned (upload) or produced (download) by a kernel on the compute
// stream while the next chunk is in flight: PCIe runs at the copy engines'
// rate (55-57 GB/s on a B200 box) instead of the SMs' zero-copy rate
// (~51 GB/s), and the kernels hide behind the copies.
constexpr int64_t kXferRows = int64_t(1) << 23;  // rows per chunk (8 Mi: 448 MB pos+vel+mass)

bool host_pinned(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

int xfer_setup(mpcd_ctx* c) {
  if (!c->copy_st) MPCD_CUDA(cudaStreamCreateWithFlags(&c->copy_st, cudaStreamNonBlocking));
  for (cudaEvent_t& e : c->xfer_ev)
    if (!e) MPCD_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  if (!c->xfer_buf) MPCD_CUDA(cudaMalloc(&c->xfer_buf, sizeof(double) * 7 * 2 * kXferRows));
  return MPCD_OK;
}

// rows [0, n) of pinned host pos/vel(/mass) -> binned into region set b
int upload_pipelined(mpcd_ctx* c, const double* pos, const double* vel, const double* mass,
                     int64_t n, int64_t step, int b, cudaStream_t st) {
  int rc = xfer_setup(c);
  if (rc) return rc;
  cudaEvent_t* copied = c->xfer_ev;      // [0], [1]: chunk in staging slot s has landed
  cudaEvent_t* consumed = c->xfer_ev + 2;  // [2], [3]: slot s is free again
  // the copies may start only after the compute stream's earlier work
  MPCD_CUDA(cudaEventRecord(consumed[0], st));
  MPCD_CUDA(cudaEventRecord(consumed[1], st));
  int i = 0;
  for (int64_t r0 = 0; r0 < n; r0 += kXferRows, ++i) {
    const int s = i & 1;
    const int64_t rows = std::min(kXferRows, n - r0);
    double* sp = c->xfer_buf + (size_t)s * 7 * kXferRows;
    double* sv = sp + 3 * kXferRows;
    double* sm = sp + 6 * kXferRows;
    MPCD_CUDA(cudaStreamWaitEvent(c->copy_st, consumed[s], 0));
    MPCD_CUDA(cudaMemcpyAsync(sp, pos + 3 * r0, sizeof(double) * 3 * rows,
                              cudaMemcpyHostToDevice, c->copy_st));
    MPCD_CUDA(cudaMemcpyAsync(sv, vel + 3 * r0, sizeof(double) * 3 * rows,
                              cudaMemcpyHostToDevice, c->copy_st));
    if (mass)
      MPCD_CUDA(cudaMemcpyAsync(sm, mass + r0, sizeof(double) * rows, cudaMemcpyHostToDevice,
                                c->copy_st));
    MPCD_CUDA(cudaEventRecord(copied[s], c->copy_st));
    MPCD_CUDA(cudaStreamWaitEvent(st, copied[s], 0));
    k_place_rows<<<grid_for(rows, kRowBlock), kRowBlock, 0, st>>>(
        sp, sv, mass ? sm : nullptr, nullptr, rows, c->cfg.mass_value, place_args(c, b, step),
        nullptr, r0);
    MPCD_LAUNCH_CHECK();
    MPCD_CUDA(cudaEventRecord(consumed[s], st));
  }
  return MPCD_OK;
}

// flat id-ordered records -> rows [0, n) of pinned host pos/vel
int download_pipelined(mpcd_ctx* c, Recs flat, int64_t n, double* pos, double* vel,
                       cudaStream_t st) {
  int rc = xfer_setup(c);
  if (rc) return rc;
  cudaEvent_t* produced = c->xfer_ev;      // staging slot s holds rows to copy out
  cudaEvent_t* drained = c->xfer_ev + 2;   // slot s has been copied out
  MPCD_CUDA(cudaEventRecord(drained[0], st));
  MPCD_CUDA(cudaEventRecord(drained[1], st));
  int i = 0;
  for (int64_t r0 = 0; r0 < n; r0 += kXferRows, ++i) {
    const int s = i & 1;
    const int64_t rows = std::min(kXferRows, n - r0);
    double* sp = c->xfer_buf + (size_t)s * 7 * kXferRows;
    double* sv = sp + 3 * kXferRows;
    MPCD_CUDA(cudaStreamWaitEvent(st, drained[s], 0));
    Recs part{flat.p + r0, flat.v + r0};
    k_flat_to_rows_chunked<<<grid_for(rows, kRowBlock), kRowBlock, 0, st>>>(part, rows, sp, sv);
    MPCD_LAUNCH_CHECK();
    MPCD_CUDA(cudaEventRecord(produced[s], st));
    MPCD_CUDA(cudaStreamWaitEvent(c->copy_st, produced[s], 0));
    MPCD_CUDA(cudaMemcpyAsync(pos + 3 * r0, sp, sizeof(double) * 3 * rows,
                              cudaMemcpyDeviceToHost, c->copy_st));
    MPCD_CUDA(cudaMemcpyAsync(vel + 3 * r0, sv, sizeof(double) * 3 * rows,
                              cudaMemcpyDeviceToHost, c->copy_st));
    MPCD_CUDA(cudaEventRecord(drained[s], c->copy_st));
  }
  // the caller's stream (and its synchronisation) covers the last copies
  MPCD_CUDA(cudaStreamWaitEvent(st, drained[0], 0));
  MPCD_CUDA(cudaStreamWaitEvent(st, drained[1], 0));
  return MPCD_OK;
}

int mpcd_upload(mpcd_ctx* c, const double* pos, const double* vel, const double* mass,
                const int64_t* ids, int64_t n, int64_t step, void* stream) {
  clear_error();
  if (!c) return fail(MPCD_ERR_CONFIG, "null context");
  if (n < 0 || (!c->multi && n > c->cfg.capacity) || n >= (1LL << 32))
    return fail(MPCD_ERR_CAPACITY, "%lld particles exceed capacity %lld", (long long)n,
                (long long)c->cfg.capacity);
  if (n > 0 && (!pos || !vel)) return fail(MPCD_ERR_CONFIG, "positions/velocities required");
  if (n > 0 && !c->cfg.uniform_mass && !mass) return fail(MPCD_ERR_CONFIG, "masses required");
  DeviceGuard dg(c->dev);
  cudaStream_t st = as_stream(stream);
  int64_t bound = n;
  if (ids && n > 0) {
    int rc = validate_ids(ids, n, !c->multi, &bound);
    if (rc) return rc;
  }
  c->id_bound = bound;
  // retire whatever is resident
  for (int b = 0; b < 2; ++b) {
    MPCD_CUDA(cudaMemsetAsync(c->count[b], 0, sizeof(uint32_t) * c->C, st));
    MPCD_CUDA(cudaMemsetAsync(ovf_n_of(c, b), 0, 4, st));
  }
  c->n = n;
  const int b = 0;
  if (c->multi) MPCD_CUDA(cudaMemsetAsync(placed_of(c), 0, 4, st));
  const double* zpos = mapped(pos);
  const double* zvel = mapped(vel);
  const double* zmass = c->cfg.uniform_mass ? nullptr : mapped(mass);
  const int64_t* zids = mapped(ids);
  const bool dma = n >= kXferRows / 4 && !ids && !c->multi && host_pinned(pos) &&
                   host_pinned(vel) && (c->cfg.uniform_mass || host_pinned(mass));
  if (dma) {  // pinned host rows, large: chunked DMA, each chunk binned on arrival
    int rc = upload_pipelined(c, pos, vel, c->cfg.uniform_mass ? nullptr : mass, n, step, b, st);
    if (rc) return rc;
  } else if (n > 0 && zpos && zvel && (c->cfg.uniform_mass || zmass) && (!ids || zids)) {
    // pinned host (or device) rows: bin them straight from the caller's buffers
    k_place_rows<<<grid_for(n, kRowBlock), kRowBlock, 0, st>>>(
        zpos, zvel, zmass, zids, n, c->cfg.mass_value, place_args(c, b, step),
        c->multi ? placed_of(c) : nullptr);
    MPCD_LAUNCH_CHECK();
  } else if (n > 0) {
    double* tmp = nullptr;
    const size_t bytes = (size_t)n * 8 * (3 + 3 + 1 + 1);
    MPCD_CUDA(cudaMallocAsync(&tmp, bytes, st));
    double* dpos = tmp;
    double* dvel = tmp + 3 * n;
    double* dmass = tmp + 6 * n;
    int64_t* dids = reinterpret_cast<int64_t*>(tmp + 7 * n);
    MPCD_CUDA(cudaMemcpyAsync(dpos, pos, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, st));
    MPCD_CUDA(cudaMemcpyAsync(dvel, vel, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, st));
    if (!c->cfg.uniform_mass)
      MPCD_CUDA(cudaMemcpyAsync(dmass, mass, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    if (ids) MPCD_CUDA(cudaMemcpyAsync(dids, ids, sizeof(int64_t) * n, cudaMemcpyHostToDevice, st));
    k_place_rows<<<grid_for(n, kRowBlock), kRowBlock, 0, st>>>(
        dpos, dvel, c->cfg.uniform_mass ? nullptr : dmass, ids ? dids : nullptr, n,
        c->cfg.mass_value, place_args(c, b, step), c->multi ? placed_of(c) : nullptr);
    MPCD_LAUNCH_CHECK();
    MPCD_CUDA(cudaFreeAsync(tmp, st));
  }
  if (c->multi) {  // the rows of other domains were dropped
    int rc = read_placed(c, st, &c->n);
    if (rc) return rc;
    if (c->n > c->cfg.capacity)
      return fail(MPCD_ERR_CAPACITY, "domain %d holds %lld particles, capacity %lld",
                  (int)c->dom.rank, (long long)c->n, (long long)c->cfg.capacity);
  }
  c->cur = b;
  c->binned = true;
  c->flat = -1;
  c->cur_step = step;
  c->have_diag = false;
  c->poisoned = false;
  return check_flags(c, st);
}

int mpcd_download(mpcd_ctx* c, double* pos, double* vel, double* mass, int64_t* ids,
                  int32_t id_order, void* stream) {
  clear_error();
  if (!c) return fail(MPCD_ERR_CONFIG, "null context");
  DeviceGuard dg(c->dev);
  if (c->multi) return download_multi(c, pos, vel, mass, ids, id_order, stream);
  return download_rows(c, pos, vel, mass, ids, id_order, stream);
}

int mpcd_step(mpcd_ctx* c, int64_t step, int32_t flags, void* stream) {
  clear_error();
  if (!c) return fail(MPCD_ERR_CONFIG, "null context");
  if (step < 0) return fail(MPCD_ERR_CONFIG, "step must be non-negative");
  DeviceGuard dg(c->dev);
  return launch_step(c, step, flags, false, as_stream(stream));
}

int mpcd_run(mpcd_ctx* c, int64_t first_step, int64_t n_steps, int32_t flags, void* stream) {
  clear_error();
  if (!c) return fail(MPCD_ERR_CONFIG, "null context");
  if (c->multi && n_steps > 1)
    return fail(MPCD_ERR_CONFIG, "a decomposed domain exchanges leavers between steps: use "
                                 "mpcd_step + mpcd_absorb");
  DeviceGuard dg(c->dev);
  for (int64_t k = 0; k < n_steps; ++k) {
    int rc = launch_step(c, first_step + k, flags, false, as_stream(stream));
    if (rc) return rc;
  }
  // capacity / RNG failures of any step of the run surface here (one sync)
  return n_steps > 0 ? check_flags(c, as_stream(stream)) : MPCD_OK;
}

int mpcd_read_diag(mpcd_ctx* c, mpcd_diag* out, void* stream) {
  clear_error();
  if (!c || !out) return fail(MPCD_ERR_CONFIG, "null argument");
  DeviceGuard dg(c->dev);
  cudaStream_t st = as_stream(stream);
  double h[9];
  MPCD_CUDA(cudaMemcpyAsync(h, c->diag, sizeof(h), cudaMemcpyDeviceToHost, st));
  int rc = check_flags(c, st);  // synchronises
  if (rc) return rc;
  out->momentum[0] = h[0]; out->momentum[1] = h[1]; out->momentum[2] = h[2];
  out->energy = h[3];
  out->mass = h[4];
  out->max_cell_drift = h[5];
  out->n = (int64_t)h[6];
  out->step = c->have_diag ? (int64_t)h[7] : -1;
  out->migrated = (int64_t)h[8];
  return MPCD_OK;
}

int mpcd_read_com(mpcd_ctx* c, int64_t* cell_ids, double* com, int64_t* n_occupied, void* stream) {
  clear_error();
  if (!c || !n_occupied) return fail(MPCD_ERR_CONFIG, "null argument");
  if (!c->have_diag || !c->last_com || !c->com_cap)
    return fail(MPCD_ERR_CONFIG, "the last step did not capture com (MPCD_STEP_WANT_COM)");
  DeviceGuard dg(c->dev);
  cudaStream_t st = as_stream(stream);
  std::vector<double> cx(4 * c->C);
  MPCD_CUDA(cudaMemcpyAsync(cx.data(), c->com_cap, sizeof(double) * 4 * c->C,
                            cudaMemcpyDeviceToHost, st));
  MPCD_CUDA(cudaStreamSynchronize(st));
  // (global cell id, local cell) of the occupied cells, ascending by global id
  std::vector<std::pair<int64_t, int64_t>> occ;
  const int64_t* L = c->cfg.dims;
  const int64_t* G = c->multi ? c->dom.global_dims : c->cfg.dims;
  for (int64_t cc = 0; cc < c->C; ++cc) {
    if (cx[4 * cc + 3] > 0.0) {
      const int64_t lz = cc % L[2], ly = (cc / L[2]) % L[1], lx = cc / (L[1] * L[2]);
      const int64_t g = ((lx + c->org[0]) * G[1] + (ly + c->org[1])) * G[2] + (lz + c->org[2]);
      occ.emplace_back(g, cc);
    }
  }
  if (c->multi) std::sort(occ.begin(), occ.end());
  const int64_t k = (int64_t)occ.size();
  for (int64_t j = 0; j < k; ++j) {
    if (cell_ids) cell_ids[j] = occ[j].first;
    if (com) for (int d = 0; d < 3; ++d) com[3 * j + d] = cx[4 * occ[j].second + d];
  }
  *n_occupied = k;
  return MPCD_OK;
}

int mpcd_read_binning(mpcd_ctx* c, int64_t* cells, int64_t* bin_count, int64_t* bin_offset,
                      int64_t* permutation, void* stream) {
  clear_error();
  if (!c) return fail(MPCD_ERR_CONFIG, "null context");
  if (c->multi) return fail(MPCD_ERR_CONFIG, "read_binning is for a whole-box context");
  DeviceGuard dg(c->dev);
  cudaStream_t st = as_stream(stream);
  int rc = ensure_binned(c, c->cur_step, st);
  if (rc) return rc;
  const int64_t n = c->n, C = c->C;
  const int b = c->cur;
  uint32_t h_ovf = 0;
  MPCD_CUDA(cudaMemcpyAsync(&h_ovf, ovf_n_of(c, b), 4, cudaMemcpyDeviceToHost, st));
  MPCD_CUDA(cudaStreamSynchronize(st));
  const uint32_t n_ovf = std::min(h_ovf, c->ovf_cap);
  int64_t* tmp = nullptr;
  MPCD_CUDA(cudaMallocAsync(&tmp, sizeof(int64_t) * (2 * n + 2 * C + 1), st));
  int64_t* dcells = tmp;
  int64_t* dperm = tmp + n;
  int64_t* dcnt = tmp + 2 * n;
  int64_t* doff = tmp + 2 * n + C;
  k_widen_counts<<<grid_for(C, 256), 256, 0, st>>>(c->count[b], C, dcnt);
  MPCD_LAUNCH_CHECK();
  rc = scan_u32(c->scan, c->count[b], nullptr, doff, C, false, st);
  if (rc) return rc;
  if (n > 0) {
    const int64_t work = C * (int64_t)c->cap + n_ovf;
    k_binning_debug<<<grid_for(work, 256), 256, 0, st>>>(c->reg[b], c->count[b], C, c->cap,
                                                         c->ovf[b], c->ovf_cell[b], n_ovf, doff,
                                                         dcells, dperm);
    MPCD_LAUNCH_CHECK();
  }
  if (cells && n) MPCD_CUDA(cudaMemcpyAsync(cells, dcells, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, st));
  if (permutation && n) MPCD_CUDA(cudaMemcpyAsync(permutation, dperm, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, st));
  if (bin_count) MPCD_CUDA(cudaMemcpyAsync(bin_count, dcnt, sizeof(int64_t) * C, cudaMemcpyDeviceToHost, st));
  if (bin_offset) MPCD_CUDA(cudaMemcpyAsync(bin_offset, doff, sizeof(int64_t) * C, cudaMemcpyDeviceToHost, st));
  MPCD_CUDA(cudaFreeAsync(tmp, st));
  MPCD_CUDA(cudaStreamSynchronize(st));
  return MPCD_OK;
}

int mpcd_step_rows(mpcd_ctx* c, const double* pos_in, const double* vel_in, const double* mass,
                   int64_t n, int64_t step, int32_t flags, double* pos_out, double* vel_out,
                   double* drift, void* stream) {
  clear_error();
  if (!c) return fail(MPCD_ERR_CONFIG, "null context");
  if (c->multi) return fail(MPCD_ERR_CONFIG, "step_host is for a whole-box context");
  if (n > 0 && (!pos_out || !vel_out)) return fail(MPCD_ERR_CONFIG, "output rows required");
  int rc = mpcd_upload(c, pos_in, vel_in, mass, nullptr, n, step, stream);
  if (rc) return rc;
  DeviceGuard dg(c->dev);
  cudaStream_t st = as_stream(stream);
  rc = launch_step(c, step, flags, true, st);
  if (rc) return rc;
  double* zpos = mapped(pos_out);
  double* zvel = mapped(vel_out);
  if (n >= kXferRows / 4 && host_pinned(pos_out) && host_pinned(vel_out)) {
    // large pinned host rows: chunked, DMA-copied out as each chunk is produced
    rc = download_pipelined(c, c->reg[c->flat], n, pos_out, vel_out, st);
    if (rc) return rc;
  } else if (n > 0 && zpos && zvel) {  // by-id rows straight into the caller's pinned buffers
    k_flat_to_rows_chunked<<<grid_for(n, kRowBlock), kRowBlock, 0, st>>>(c->reg[c->flat], n,
                                                                         zpos, zvel);
    MPCD_LAUNCH_CHECK();
  } else if (n > 0) {  // by-id rows: row i == particle i
    double* tmp = nullptr;
    MPCD_CUDA(cudaMallocAsync(&tmp, sizeof(double) * 6 * n, st));
    k_flat_to_rows_chunked<<<grid_for(n, kRowBlock), kRowBlock, 0, st>>>(c->reg[c->flat], n, tmp,
                                                                         tmp + 3 * n);
    MPCD_LAUNCH_CHECK();
    MPCD_CUDA(cudaMemcpyAsync(pos_out, tmp, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, st));
    MPCD_CUDA(cudaMemcpyAsync(vel_out, tmp + 3 * n, sizeof(double) * 3 * n,
                              cudaMemcpyDeviceToHost, st));
    MPCD_CUDA(cudaFreeAsync(tmp, st));
  }
  mpcd_diag d;
  rc = mpcd_read_diag(c, &d, stream);
  if (rc) return rc;
  if (drift) *drift = d.max_cell_drift;
  return MPCD_OK;
}

int mpcd_step_host(mpcd_ctx* c, double* pos, double* vel, const double* mass, int64_t n,
                   int64_t step, int32_t flags, double* drift, void* stream) {
  return mpcd_step_rows(c, pos, vel, mass, n, step, flags, pos, vel, drift, stream);
}

int mpcd_host_alloc(int64_t bytes, void** out) {
  clear_error();
  if (!out || bytes < 0) return fail(MPCD_ERR_CONFIG, "bad argument");
  *out = nullptr;
  if (bytes == 0) return MPCD_OK;
  MPCD_CUDA(cudaHostAlloc(out, (size_t)bytes, cudaHostAllocPortable | cudaHostAllocMapped));
  return MPCD_OK;
}

int mpcd_host_free(void* ptr) {
  clear_error();
  if (ptr) MPCD_CUDA(cudaFreeHost(ptr));
  return MPCD_OK;
}

int mpcd_host_is_pinned(const void* ptr) {
  if (!ptr) return 0;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return a.type == cudaMemoryTypeHost ? 1 : 0;
}

int mpcd_init_device(mpcd_ctx* c, int64_t n, double velocity_variance, int64_t step, void* stream) {
  clear_error();
  if (!c) return fail(MPCD_ERR_CONFIG, "null context");
  if (n < 0 || (!c->multi && n > c->cfg.capacity) || n >= (1LL << 32))
    return fail(MPCD_ERR_CAPACITY, "n exceeds capacity");
  if (!c->cfg.uniform_mass) return fail(MPCD_ERR_CONFIG, "device init needs uniform_mass");
  DeviceGuard dg(c->dev);
  cudaStream_t st = as_stream(stream);
  for (int b = 0; b < 2; ++b) {
    MPCD_CUDA(cudaMemsetAsync(c->count[b], 0, sizeof(uint32_t) * c->C, st));
    MPCD_CUDA(cudaMemsetAsync(ovf_n_of(c, b), 0, 4, st));
  }
  MPCD_CUDA(cudaMemsetAsync(placed_of(c), 0, 4, st));
  c->id_bound = n;
  const int b = 0;
  if (n > 0) {
    double* part = nullptr;
    MPCD_CUDA(cudaMallocAsync(&part, sizeof(double) * 3 * kInitBlocks, st));
    const mpcd_config& g = c->cfg;
    const int64_t* G = c->multi ? c->dom.global_dims : g.dims;
    const uint64_t state = key_state(g.seed, 0, kInit, 0);
    const double sigma = sqrt(velocity_variance);
    k_init_sum<<<kInitBlocks, 256, 0, st>>>(n, state, sigma, part);
    MPCD_LAUNCH_CHECK();
    k_init_place<<<kInitBlocks, 256, 0, st>>>(n, state, G[0] * g.cell_size, G[1] * g.cell_size,
                                              G[2] * g.cell_size, sigma, g.mass_value, part,
                                              kInitBlocks, place_args(c, b, step), placed_of(c));
    MPCD_LAUNCH_CHECK();
    MPCD_CUDA(cudaFreeAsync(part, st));
  }
  int rc = read_placed(c, st, &c->n);
  if (rc) return rc;
  if (c->n > c->cfg.capacity)
    return fail(MPCD_ERR_CAPACITY, "domain holds %lld particles, capacity %lld",
                (long long)c->n, (long long)c->cfg.capacity);
  c->cur = b;
  c->binned = true;
  c->flat = -1;
  c->cur_step = step;
  c->have_diag = false;
  c->poisoned = false;
  return check_flags(c, st);
}

int mpcd_ctx_set_domain(mpcd_ctx* c, const mpcd_domain* dom) {
  clear_error();
  if (!c || !dom) return fail(MPCD_ERR_CONFIG, "null argument");
  int64_t P = 1;
  for (int d = 0; d < 3; ++d) {
    if (dom->rank_dims[d] < 1) return fail(MPCD_ERR_TOPOLOGY, "rank_dims must be positive");
    if (dom->global_dims[d] != c->cfg.dims[d] * dom->rank_dims[d])
      return fail(MPCD_ERR_TOPOLOGY,
                  "global_dims[%d] = %lld is not rank_dims * the context's dims (%lld * %d)", d,
                  (long long)dom->global_dims[d], (long long)c->cfg.dims[d], dom->rank_dims[d]);
    if (dom->global_dims[d] >= (1LL << 31)) return fail(MPCD_ERR_CONFIG, "global dims too large");
    P *= dom->rank_dims[d];
  }
  if (dom->rank < 0 || dom->rank >= P) return fail(MPCD_ERR_TOPOLOGY, "rank out of range");
  DeviceGuard dg(c->dev);
  if (c->send) cudaFree(c->send);
  if (c->send_n) cudaFree(c->send_n);
  c->send = nullptr;
  c->send_n = nullptr;
  c->dom = *dom;
  const int r = dom->rank;
  const int bz = r % dom->rank_dims[2], by = (r / dom->rank_dims[2]) % dom->rank_dims[1];
  const int bx = r / (dom->rank_dims[1] * dom->rank_dims[2]);
  c->org[0] = bx * c->cfg.dims[0];
  c->org[1] = by * c->cfg.dims[1];
  c->org[2] = bz * c->cfg.dims[2];
  int64_t cap = dom->send_capacity;
  if (cap <= 0) cap = std::max<int64_t>(1 << 16, c->cfg.capacity / 16);
  if (cap >= (1LL << 32)) cap = (1LL << 32) - 1;
  c->dom.send_capacity = cap;
  if (cudaMalloc(&c->send, (size_t)P * cap * sizeof(XRec)) != cudaSuccess ||
      cudaMalloc(&c->send_n, sizeof(unsigned long long) * P) != cudaSuccess)
    return fail(MPCD_ERR_CUDA, "cudaMalloc of %lld send records failed", (long long)(P * cap));
  MPCD_CUDA(cudaMemset(c->send_n, 0, sizeof(unsigned long long) * P));
  c->multi = true;
  c->n = 0;
  c->binned = false;
  c->flat = -1;
  c->have_diag = false;
  MPCD_CUDA(cudaDeviceSynchronize());
  return MPCD_OK;
}

int mpcd_exchange_buffers(mpcd_ctx* c, mpcd_exchange* out) {
  clear_error();
  if (!c || !out) return fail(MPCD_ERR_CONFIG, "null argument");
  if (!c->multi) return fail(MPCD_ERR_CONFIG, "not a decomposed domain (mpcd_ctx_set_domain)");
  out->send = c->send;
  out->send_n = c->send_n;
  out->send_capacity = c->dom.send_capacity;
  out->n_ranks = c->dom.rank_dims[0] * c->dom.rank_dims[1] * c->dom.rank_dims[2];
  out->record_bytes = (int32_t)sizeof(XRec);
  return MPCD_OK;
}

int mpcd_absorb(mpcd_ctx* c, const void* recs, int64_t n_recv, int64_t n_sent, void* stream) {
  clear_error();
  if (!c) return fail(MPCD_ERR_CONFIG, "null context");
  if (!c->multi) return fail(MPCD_ERR_CONFIG, "not a decomposed domain (mpcd_ctx_set_domain)");
  if (!c->binned) return fail(MPCD_ERR_CONFIG, "absorb follows mpcd_step");
  if (n_recv < 0 || n_sent < 0 || n_sent > c->n || (n_recv > 0 && !recs))
    return fail(MPCD_ERR_CONFIG, "bad absorb counts");
  if (c->n - n_sent + n_recv > c->cfg.capacity)
    return fail(MPCD_ERR_CAPACITY, "domain %d would hold %lld particles, capacity %lld",
                (int)c->dom.rank, (long long)(c->n - n_sent + n_recv),
                (long long)c->cfg.capacity);
  DeviceGuard dg(c->dev);
  cudaStream_t st = as_stream(stream);
  if (n_recv > 0) {
    PlaceArgs P = place_args(c, c->cur, c->cur_step);
    P.strict = 1;
    k_place_xrecs<<<grid_for(n_recv, 256), 256, 0, st>>>(static_cast<const XRec*>(recs), n_recv, P);
    MPCD_LAUNCH_CHECK();
  }
  const int64_t P = c->dom.rank_dims[0] * c->dom.rank_dims[1] * c->dom.rank_dims[2];
  MPCD_CUDA(cudaMemsetAsync(c->send_n, 0, sizeof(unsigned long long) * P, st));
  c->n += n_recv - n_sent;
  return MPCD_OK;
}

// ---------------------------------------------------- fused migration ---
namespace {
constexpr int kIpcAllocs = 9;  // slab[2], count[2], ovf_slab[2], ovf_cell[2], small

PeerBufs local_bufs(mpcd_ctx* c) {
  PeerBufs P;
  for (int b = 0; b < 2; ++b) {
    P.reg[b] = c->reg[b];
    P.count[b] = c->count[b];
    P.ovf[b] = c->ovf[b];
    P.ovf_cell[b] = c->ovf_cell[b];
  }
  P.small = c->small;
  return P;
}

int install_peers(mpcd_ctx* c, const std::vector<PeerBufs>& tab) {
  const int64_t P = (int64_t)c->dom.rank_dims[0] * c->dom.rank_dims[1] * c->dom.rank_dims[2];
  if ((int64_t)tab.size() != P) return fail(MPCD_ERR_TOPOLOGY, "peer table has %d of %lld ranks",
                                            (int)tab.size(), (long long)P);
  if (P > kMaxPeers)  // k_step keeps the peers' pointers in shared memory
    return fail(MPCD_ERR_TOPOLOGY, "fused migration connects at most %d ranks (%lld here): "
                "use the exchange", kMaxPeers, (long long)P);
  if (c->d_peers) cudaFree(c->d_peers);
  MPCD_CUDA(cudaMalloc(&c->d_peers, sizeof(PeerBufs) * P));
  MPCD_CUDA(cudaMemcpy(c->d_peers, tab.data(), sizeof(PeerBufs) * P, cudaMemcpyHostToDevice));
  c->p2p = true;
  return MPCD_OK;
}
}  // namespace

// Each rank's blob: its allocations' IPC handles, then the geometry a peer
// addresses them with (cells, slots per cell, overflow capacity).  A peer's
// k_step indexes the owner's regions and overflow list with its own values,
// so connecting requires equal geometry (the overflow capacity follows the
// free device memory at context creation and could differ between GPUs).
struct IpcGeometry {
  int64_t C, cap, ovf_cap;
};
constexpr int64_t kIpcBlob = kIpcAllocs * (int64_t)sizeof(cudaIpcMemHandle_t) +
                             (int64_t)sizeof(IpcGeometry);

int mpcd_ipc_handles(mpcd_ctx* c, void* out, int64_t* nbytes) {
  clear_error();
  if (!c || !nbytes) return fail(MPCD_ERR_CONFIG, "null argument");
  const int64_t need = kIpcBlob;
  if (!out) {
    *nbytes = need;
    return MPCD_OK;
  }
  if (*nbytes < need) return fail(MPCD_ERR_CONFIG, "handle buffer needs %lld bytes", (long long)need);
  DeviceGuard dg(c->dev);
  void* allocs[kIpcAllocs] = {c->slab[0], c->slab[1], c->count[0], c->count[1], c->ovf_slab[0],
                              c->ovf_slab[1], c->ovf_cell[0], c->ovf_cell[1], c->small};
  cudaIpcMemHandle_t* h = static_cast<cudaIpcMemHandle_t*>(out);
  for (int i = 0; i < kIpcAllocs; ++i) MPCD_CUDA(cudaIpcGetMemHandle(&h[i], allocs[i]));
  const IpcGeometry g{c->C, (int64_t)c->cap, (int64_t)c->ovf_cap};
  memcpy(h + kIpcAllocs, &g, sizeof(g));
  *nbytes = need;
  return MPCD_OK;
}

int mpcd_connect_peers(mpcd_ctx* c, const void* all, int32_t n_ranks) {
  clear_error();
  if (!c || !all) return fail(MPCD_ERR_CONFIG, "null argument");
  if (!c->multi) return fail(MPCD_ERR_CONFIG, "not a decomposed domain (mpcd_ctx_set_domain)");
  DeviceGuard dg(c->dev);
  const char* blobs = static_cast<const char*>(all);
  const uint64_t rows = (uint64_t)c->C * c->cap, orows = c->ovf_cap;
  for (int r = 0; r < n_ranks; ++r) {  // equal geometry first: nothing opened on failure
    IpcGeometry g;
    memcpy(&g, blobs + r * kIpcBlob + kIpcAllocs * sizeof(cudaIpcMemHandle_t), sizeof(g));
    if (g.C != c->C || g.cap != (int64_t)c->cap || g.ovf_cap != (int64_t)c->ovf_cap)
      return fail(MPCD_ERR_TOPOLOGY,
                  "rank %d's domain differs (cells %lld, cap %lld, overflow %lld; here %lld, "
                  "%u, %u): fused migration needs equal geometry",
                  r, (long long)g.C, (long long)g.cap, (long long)g.ovf_cap, (long long)c->C,
                  c->cap, c->ovf_cap);
  }
  std::vector<PeerBufs> tab(n_ranks);
  for (int r = 0; r < n_ranks; ++r) {
    if (r == c->dom.rank) {
      tab[r] = local_bufs(c);
      continue;
    }
    const cudaIpcMemHandle_t* h = reinterpret_cast<const cudaIpcMemHandle_t*>(blobs + r * kIpcBlob);
    void* p[kIpcAllocs];
    for (int i = 0; i < kIpcAllocs; ++i) {
      MPCD_CUDA(cudaIpcOpenMemHandle(&p[i], h[i], cudaIpcMemLazyEnablePeerAccess));
      c->ipc_opened.push_back(p[i]);
    }
    // every rank has the same cells per domain, cap and overflow capacity
    PeerBufs& P = tab[r];
    for (int b = 0; b < 2; ++b) {
      P.reg[b] = carve(p[b], rows);
      P.count[b] = static_cast<uint32_t*>(p[2 + b]);
      P.ovf[b] = carve(p[4 + b], orows);
      P.ovf_cell[b] = static_cast<uint32_t*>(p[6 + b]);
    }
    P.small = static_cast<uint32_t*>(p[8]);
  }
  return install_peers(c, tab);
}

int mpcd_connect_local(mpcd_ctx* const* ctxs, int32_t n) {
  clear_error();
  if (!ctxs || n < 1) return fail(MPCD_ERR_CONFIG, "null argument");
  std::vector<PeerBufs> tab(n);
  for (int r = 0; r < n; ++r) {
    if (!ctxs[r] || !ctxs[r]->multi || ctxs[r]->dom.rank != r)
      return fail(MPCD_ERR_TOPOLOGY, "context %d is not domain %d of the box", r, r);
    if (ctxs[r]->C != ctxs[0]->C || ctxs[r]->cap != ctxs[0]->cap ||
        ctxs[r]->ovf_cap != ctxs[0]->ovf_cap || ctxs[r]->dev != ctxs[0]->dev)
      return fail(MPCD_ERR_TOPOLOGY, "domains differ in cells, capacities or device");
    tab[r] = local_bufs(ctxs[r]);
  }
  for (int r = 0; r < n; ++r) {
    DeviceGuard dg(ctxs[r]->dev);
    int rc = install_peers(ctxs[r], tab);
    if (rc) return rc;
  }
  return MPCD_OK;
}

int mpcd_profile(mpcd_ctx* c, int32_t enable) {
  clear_error();
  if (!c) return fail(MPCD_ERR_CONFIG, "null context");
  DeviceGuard dg(c->dev);
  for (cudaEvent_t e : c->prof_events) cudaEventDestroy(e);
  for (cudaEvent_t e : c->xfer_ev)
    if (e) cudaEventDestroy(e);
  if (c->copy_st) cudaStreamDestroy(c->copy_st);
  if (c->xfer_buf) cudaFree(c->xfer_buf);
  c->prof_events.clear();
  c->prof = enable != 0;
  return MPCD_OK;
}

int mpcd_read_profile(mpcd_ctx* c, double* ms, int64_t* n_steps) {
  clear_error();
  if (!c || !ms) return fail(MPCD_ERR_CONFIG, "null argument");
  DeviceGuard dg(c->dev);
  for (int i = 0; i < MPCD_PROFILE_SLOTS; ++i) ms[i] = 0.0;
  const size_t per = kProfSlots + 1;
  const size_t steps = c->prof_events.size() / per;
  if (steps) MPCD_CUDA(cudaEventSynchronize(c->prof_events.back()));
  for (size_t s = 0; s < steps; ++s) {
    cudaEvent_t* e = c->prof_events.data() + s * per;
    for (int i = 0; i < kProfSlots; ++i) {
      float tt = 0.f;
      MPCD_CUDA(cudaEventElapsedTime(&tt, e[i], e[i + 1]));
      ms[i] += tt;
    }
  }
  if (n_steps) *n_steps = (int64_t)steps;
  return MPCD_OK;
}

uint64_t mpcd_key_state(uint64_t seed, uint64_t step, uint64_t purpose, uint64_t cell) {
  return key_state(seed, step, purpose, cell);
}
double mpcd_uniform_at(uint64_t state, uint64_t index) { return uniform_at(state, index); }
void mpcd_grid_shift(int32_t prng, uint64_t seed, uint64_t step, double cell_size, double out[3]) {
  grid_shift(prng, seed, step, cell_size, out);
}

}  // extern "C"
