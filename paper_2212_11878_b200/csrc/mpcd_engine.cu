// mpcd_engine.cu -- the B200 SRD time step (engine.py:415-455 semantics).
//
// State in HBM (SoA, double-buffered): x y z vx vy vz [m] (f64), id (u32),
// sorted by collision cell of the NEXT step to run, plus `ends` (u32 per
// cell: inclusive prefix of that binning).  One step k is
//
//   A  k_collide_count   per tile of TC cells: stage ids, rank every particle
//                        by id inside its cell (the reference permutation is
//                        the stable argsort over id order, collision.py:98),
//                        sum (m v, m) in numpy's reduceat association,
//                        com = p/m, Marsaglia axis from the keyed RNG keyed by
//                        global cell id, rotate, stream + wrap, bin for step
//                        k+1 -> histogram; per-cell com/axis -> HBM; post-
//                        collision sums -> drift + conservation partials.
//   S  scan              exclusive prefix of the k+1 histogram -> cursor.
//   B  k_collide_scatter recompute v', x' from the stored com/axis (bit-
//                        identical) and scatter each particle to its slot in
//                        the k+1 order (warp-aggregated cursor atomics).
//   F  k_diag_finalize   fixed-order reduction of the tile partials.
//
// Algorithmic bytes per particle-step (uniform mass, ppc = 10): A reads
// id+v+x (52), B reads id+v+x (52) and writes them (52); per cell A reads
// ends (4) and writes com+axis (48), S reads/writes/zeroes counts (12), B
// reads ends+com/axis (52).  See DESIGN.md section 3.
#include <algorithm>
#include <vector>

#include "mpcd_internal.h"

namespace mpcd {

struct SoA {
  double *x, *y, *z, *vx, *vy, *vz, *m;
  uint32_t* id;
};

struct StepArgs {
  SoA in, out;
  const uint32_t* ends;  // binning of step k (inclusive prefix per cell)
  uint32_t* counts;      // histogram of step k+1 (zeroed by the scan)
  uint32_t* cursor;      // exclusive prefix of counts -> ends of step k+1
  double* comax;         // per cell: com[3], axis[3]
  double* partials;      // per tile: px py pz sum(m v^2) mass
  unsigned long long* drift_bits;
  uint32_t* flags;       // [0] overflow tiles, [1] rng failure
  uint32_t* overflow;    // tile list
  int64_t L0, L1, L2, C;
  double a, dt, cs, sn, box0, box1, box2;
  double off_next0, off_next1, off_next2;
  uint64_t seed, step;
  int prng;
  int unit_a;
  int uniform_mass;
  double m0;
  int want_drift;
  int by_id;  // pure-function mode: scatter to row `id`, no next binning
};

// ------------------------------------------------------------------ tiles --
constexpr int kTC = 32;        // cells per tile
constexpr int kNTA = 128;      // threads of the collide-count CTA
constexpr int kPPT = 4;        // particles per thread held in registers
constexpr int kMaxP = kNTA * kPPT;
constexpr int kNTB = 256;      // threads of the collide-scatter CTA
constexpr int kUnrollB = 2;

__device__ __forceinline__ uint32_t next_cell(const StepArgs& A, double x, double y, double z) {
  const bool unit = A.unit_a != 0;
  int64_t ix = pymod(cell_coord(x, A.off_next0, A.a, unit), A.L0);
  int64_t iy = pymod(cell_coord(y, A.off_next1, A.a, unit), A.L1);
  int64_t iz = pymod(cell_coord(z, A.off_next2, A.a, unit), A.L2);
  return (uint32_t)((ix * A.L1 + iy) * A.L2 + iz);
}

// Position of particle `i` (absolute index) among the tile's cells: first lc
// with end[lc] > i, where s_end[lc + 1] is the end of cell lc.
__device__ __forceinline__ int find_cell(const uint32_t* s_end, int nc, uint32_t i) {
  int lo = 0, hi = nc - 1;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (s_end[mid + 1] > i) hi = mid; else lo = mid + 1;
  }
  return lo;
}

__device__ __forceinline__ void atomic_max_pos_double(unsigned long long* p, double v) {
  // non-negative doubles order like their bit patterns
  atomicMax(p, (unsigned long long)__double_as_longlong(v));
}

// collision.py:327-344 for one cell (tolerance-level diagnostic)
__device__ __forceinline__ double cell_drift(const double* pre, const double* post) {
  double d0 = post[0] - pre[0], d1 = post[1] - pre[1], d2 = post[2] - pre[2];
  double dp = sqrt(((0.0 + d0 * d0) + d1 * d1) + d2 * d2);
  double nb = sqrt(((0.0 + pre[0] * pre[0]) + pre[1] * pre[1]) + pre[2] * pre[2]);
  double na = sqrt(((0.0 + post[0] * post[0]) + post[1] * post[1]) + post[2] * post[2]);
  double scale = fmax(fmax(nb, na), pre[3]);
  return dp / fmax(scale, 1e-300);
}

// Per-tile tail shared by both collide-count variants: partial sums in
// fixed cell order (deterministic) and the drift maximum.
__device__ __forceinline__ void tile_epilogue(const StepArgs& A, int64_t tile, int nc,
                                              const uint32_t* s_end, const double* s_mom,
                                              const double* s_post) {
  const int t = threadIdx.x;
  if (t < 5) {
    double s = 0.0;
    for (int lc = 0; lc < nc; ++lc) s += (t < 4) ? s_post[lc * 4 + t] : s_mom[lc * 4 + 3];
    A.partials[tile * 8 + t] = s;
  }
  if (A.want_drift && t >= 32 && t < 64) {
    double worst = 0.0;
    for (int lc = t - 32; lc < nc; lc += 32)
      if (s_mom[lc * 4 + 3] > 0.0) worst = fmax(worst, cell_drift(s_mom + lc * 4, s_post + lc * 4));
    for (int o = 16; o > 0; o >>= 1) worst = fmax(worst, __shfl_xor_sync(0xffffffffu, worst, o));
    if (t == 32 && worst > 0.0) atomic_max_pos_double(A.drift_bits, worst);
  }
}

// Phase 4: com (collision.py:209-214) and axis (collision.py:217-250) per
// occupied cell; global cell id == flat id in the single-domain engine.
__device__ __forceinline__ void cell_com_axis(const StepArgs& A, int64_t c0, int nc,
                                              const uint32_t* s_end, const double* s_mom,
                                              double* s_cx) {
  for (int lc = threadIdx.x; lc < nc; lc += blockDim.x) {
    double mass = s_mom[lc * 4 + 3];
    double v[6];
    for (int d = 0; d < 3; ++d) v[d] = (mass > 0.0) ? s_mom[lc * 4 + d] / mass : 0.0;
    v[3] = v[4] = v[5] = 0.0;
    if (s_end[lc + 1] > s_end[lc]) {
      if (!rotation_axis(A.prng, A.seed, A.step, (uint64_t)(c0 + lc), v + 3)) atomicOr(&A.flags[1], 1u);
    }
    double* g = A.comax + (c0 + lc) * 6;
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      s_cx[lc * 6 + q] = v[q];
      g[q] = v[q];
    }
  }
}

// ------------------------------------------------- pass A (fast, in smem) --
__global__ void __launch_bounds__(kNTA) k_collide_count(const StepArgs A) {
  __shared__ uint32_t s_end[kTC + 1];
  __shared__ uint32_t s_id[kMaxP];
  __shared__ double s_val[kMaxP * 4];
  __shared__ double s_mom[kTC * 4];
  __shared__ double s_post[kTC * 4];
  __shared__ double s_cx[kTC * 6];
  const int t = threadIdx.x;
  const int64_t tile = blockIdx.x;
  const int64_t c0 = tile * kTC;
  const int nc = (int)min((int64_t)kTC, A.C - c0);
  if (t <= nc) s_end[t] = (t == 0) ? (c0 == 0 ? 0u : A.ends[c0 - 1]) : A.ends[c0 + t - 1];
  __syncthreads();
  const uint32_t p0 = s_end[0];
  const int np = (int)(s_end[nc] - p0);
  if (np > kMaxP) {  // rare dense tile: the global-staging kernel handles it
    if (t == 0) A.overflow[atomicAdd(&A.flags[0], 1u)] = (uint32_t)tile;
    return;
  }

  // phase 1: every input of the tile is loaded once, up front (MLP)
  double px[kPPT], py[kPPT], pz[kPPT], vx[kPPT], vy[kPPT], vz[kPPT], mm[kPPT];
  uint32_t pid[kPPT];
  int lcell[kPPT], slot[kPPT];
#pragma unroll
  for (int r = 0; r < kPPT; ++r) {
    const int j = r * kNTA + t;
    if (j < np) {
      const uint32_t i = p0 + j;
      pid[r] = A.in.id[i];
      vx[r] = A.in.vx[i]; vy[r] = A.in.vy[i]; vz[r] = A.in.vz[i];
      px[r] = A.in.x[i]; py[r] = A.in.y[i]; pz[r] = A.in.z[i];
      mm[r] = A.uniform_mass ? A.m0 : A.in.m[i];
      lcell[r] = find_cell(s_end, nc, i);
      s_id[j] = pid[r];
    }
  }
  __syncthreads();

  // phase 2: rank by id inside the cell -> slot; stage (m v, m) in slot order
#pragma unroll
  for (int r = 0; r < kPPT; ++r) {
    const int j = r * kNTA + t;
    if (j < np) {
      const int lc = lcell[r];
      const int lo = (int)(s_end[lc] - p0), hi = (int)(s_end[lc + 1] - p0);
      int rank = 0;
      for (int q = lo; q < hi; ++q) rank += (s_id[q] < pid[r]) ? 1 : 0;
      slot[r] = lo + rank;
      double* sv = s_val + slot[r] * 4;
      sv[0] = mm[r] * vx[r]; sv[1] = mm[r] * vy[r]; sv[2] = mm[r] * vz[r]; sv[3] = mm[r];
    }
  }
  __syncthreads();

  // phase 3: per-cell moments in reduceat order (collision.py:190-206)
  for (int task = t; task < nc * 4; task += kNTA) {
    const int lc = task >> 2, comp = task & 3;
    const int lo = (int)(s_end[lc] - p0), k = (int)(s_end[lc + 1] - s_end[lc]);
    s_mom[task] = k ? reduceat(s_val + lo * 4 + comp, k, 4) : 0.0;
  }
  __syncthreads();

  // phase 4: com + axis
  cell_com_axis(A, c0, nc, s_end, s_mom, s_cx);
  __syncthreads();

  // phase 5: rotate, stream + wrap, bin for k+1; stage post-collision values
#pragma unroll
  for (int r = 0; r < kPPT; ++r) {
    const int j = r * kNTA + t;
    if (j < np) {
      const double* cx = s_cx + lcell[r] * 6;
      double v[3] = {vx[r], vy[r], vz[r]}, w[3];
      rotate(v, cx, cx + 3, A.cs, A.sn, w);
      if (!A.by_id) {
        double nx = wrap(px[r] + w[0] * A.dt, A.box0);
        double ny = wrap(py[r] + w[1] * A.dt, A.box1);
        double nz = wrap(pz[r] + w[2] * A.dt, A.box2);
        atomicAdd(&A.counts[next_cell(A, nx, ny, nz)], 1u);
      }
      double* sv = s_val + slot[r] * 4;
      const double m = mm[r];
      sv[0] = m * w[0]; sv[1] = m * w[1]; sv[2] = m * w[2];
      sv[3] = m * (((0.0 + w[0] * w[0]) + w[1] * w[1]) + w[2] * w[2]);
    }
  }
  __syncthreads();

  // phase 6: post-collision sums (drift check, conservation partials)
  for (int task = t; task < nc * 4; task += kNTA) {
    const int lc = task >> 2, comp = task & 3;
    const int lo = (int)(s_end[lc] - p0), k = (int)(s_end[lc + 1] - s_end[lc]);
    s_post[task] = k ? reduceat(s_val + lo * 4 + comp, k, 4) : 0.0;
  }
  __syncthreads();
  tile_epilogue(A, tile, nc, s_end, s_mom, s_post);
}

// --------------------------------------- pass A (dense tiles, HBM staging) --
// Same phases with the staging arrays in the (not yet written) destination
// buffer rows [p0, p0 + np) of this tile, and nothing held in registers.
// Ranking is O(k^2) per cell; it only runs for tiles above kMaxP particles.
__global__ void __launch_bounds__(kNTA) k_collide_count_dense(const StepArgs A) {
  __shared__ uint32_t s_end[kTC + 1];
  __shared__ double s_mom[kTC * 4];
  __shared__ double s_post[kTC * 4];
  __shared__ double s_cx[kTC * 6];
  const int t = threadIdx.x;
  const uint32_t n_over = *(volatile uint32_t*)&A.flags[0];
  for (uint32_t e = blockIdx.x; e < n_over; e += gridDim.x) {
    const int64_t tile = A.overflow[e];
    const int64_t c0 = tile * kTC;
    const int nc = (int)min((int64_t)kTC, A.C - c0);
    __syncthreads();
    if (t <= nc) s_end[t] = (t == 0) ? (c0 == 0 ? 0u : A.ends[c0 - 1]) : A.ends[c0 + t - 1];
    __syncthreads();
    const uint32_t p0 = s_end[0];
    const int64_t np = s_end[nc] - p0;
    uint32_t* g_id = A.out.id + p0;
    double* g_val[4] = {A.out.x + p0, A.out.y + p0, A.out.z + p0, A.out.vx + p0};
    for (int64_t j = t; j < np; j += kNTA) g_id[j] = A.in.id[p0 + j];
    __syncthreads();
    auto slot_of = [&](int64_t j, int& lc_out) -> int64_t {
      const uint32_t i = p0 + (uint32_t)j;
      const int lc = find_cell(s_end, nc, i);
      const int64_t lo = s_end[lc] - p0, hi = s_end[lc + 1] - p0;
      const uint32_t me = g_id[j];
      int64_t rank = 0;
      for (int64_t q = lo; q < hi; ++q) rank += (g_id[q] < me) ? 1 : 0;
      lc_out = lc;
      return lo + rank;
    };
    for (int64_t j = t; j < np; j += kNTA) {
      int lc;
      const int64_t s = slot_of(j, lc);
      const uint32_t i = p0 + (uint32_t)j;
      const double m = A.uniform_mass ? A.m0 : A.in.m[i];
      g_val[0][s] = m * A.in.vx[i]; g_val[1][s] = m * A.in.vy[i]; g_val[2][s] = m * A.in.vz[i];
      g_val[3][s] = m;
    }
    __syncthreads();
    for (int task = t; task < nc * 4; task += kNTA) {
      const int lc = task >> 2, comp = task & 3;
      const int64_t lo = s_end[lc] - p0, k = s_end[lc + 1] - s_end[lc];
      s_mom[task] = k ? reduceat(g_val[comp] + lo, k, 1) : 0.0;
    }
    __syncthreads();
    cell_com_axis(A, c0, nc, s_end, s_mom, s_cx);
    __syncthreads();
    for (int64_t j = t; j < np; j += kNTA) {
      int lc;
      const int64_t s = slot_of(j, lc);
      const uint32_t i = p0 + (uint32_t)j;
      const double m = A.uniform_mass ? A.m0 : A.in.m[i];
      const double* cx = s_cx + lc * 6;
      double v[3] = {A.in.vx[i], A.in.vy[i], A.in.vz[i]}, w[3];
      rotate(v, cx, cx + 3, A.cs, A.sn, w);
      if (!A.by_id) {
        double nx = wrap(A.in.x[i] + w[0] * A.dt, A.box0);
        double ny = wrap(A.in.y[i] + w[1] * A.dt, A.box1);
        double nz = wrap(A.in.z[i] + w[2] * A.dt, A.box2);
        atomicAdd(&A.counts[next_cell(A, nx, ny, nz)], 1u);
      }
      // the pre-collision staging of slot s is no longer needed: overwrite
      g_val[0][s] = m * w[0]; g_val[1][s] = m * w[1]; g_val[2][s] = m * w[2];
      g_val[3][s] = m * (((0.0 + w[0] * w[0]) + w[1] * w[1]) + w[2] * w[2]);
    }
    __syncthreads();
    for (int task = t; task < nc * 4; task += kNTA) {
      const int lc = task >> 2, comp = task & 3;
      const int64_t lo = s_end[lc] - p0, k = s_end[lc + 1] - s_end[lc];
      s_post[task] = k ? reduceat(g_val[comp] + lo, k, 1) : 0.0;
    }
    __syncthreads();
    tile_epilogue(A, tile, nc, s_end, s_mom, s_post);
  }
}

// ----------------------------------------------------- pass B (scatter) ----
__global__ void __launch_bounds__(kNTB) k_collide_scatter(const StepArgs A) {
  __shared__ uint32_t s_end[kTC + 1];
  __shared__ double s_cx[kTC * 6];
  const int t = threadIdx.x, lane = t & 31;
  const int64_t tile = blockIdx.x;
  const int64_t c0 = tile * kTC;
  const int nc = (int)min((int64_t)kTC, A.C - c0);
  if (t <= nc) s_end[t] = (t == 0) ? (c0 == 0 ? 0u : A.ends[c0 - 1]) : A.ends[c0 + t - 1];
  for (int q = t; q < nc * 6; q += kNTB) s_cx[q] = A.comax[c0 * 6 + q];
  __syncthreads();
  const uint32_t p0 = s_end[0];
  const int np = (int)(s_end[nc] - p0);
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int base = 0; base < np; base += kNTB * kUnrollB) {
    double px[kUnrollB], py[kUnrollB], pz[kUnrollB], vx[kUnrollB], vy[kUnrollB], vz[kUnrollB],
        mm[kUnrollB];
    uint32_t pid[kUnrollB];
    int lcell[kUnrollB];
#pragma unroll
    for (int u = 0; u < kUnrollB; ++u) {
      const int j = base + u * kNTB + t;
      if (j < np) {
        const uint32_t i = p0 + j;
        pid[u] = A.in.id[i];
        vx[u] = A.in.vx[i]; vy[u] = A.in.vy[i]; vz[u] = A.in.vz[i];
        px[u] = A.in.x[i]; py[u] = A.in.y[i]; pz[u] = A.in.z[i];
        mm[u] = A.uniform_mass ? A.m0 : A.in.m[i];
        lcell[u] = find_cell(s_end, nc, i);
      }
    }
#pragma unroll
    for (int u = 0; u < kUnrollB; ++u) {
      const int j = base + u * kNTB + t;
      const bool active = j < np;
      double w[3] = {0, 0, 0}, nx = 0, ny = 0, nz = 0;
      uint32_t dst = 0;
      if (active) {
        const double* cx = s_cx + lcell[u] * 6;
        double v[3] = {vx[u], vy[u], vz[u]};
        rotate(v, cx, cx + 3, A.cs, A.sn, w);
        nx = wrap(px[u] + w[0] * A.dt, A.box0);
        ny = wrap(py[u] + w[1] * A.dt, A.box1);
        nz = wrap(pz[u] + w[2] * A.dt, A.box2);
      }
      if (A.by_id) {
        dst = pid[u];
      } else {
        const uint32_t key = active ? next_cell(A, nx, ny, nz) : 0u;
        const unsigned act = __ballot_sync(0xffffffffu, active);
        if (active) {
          const unsigned grp = __match_any_sync(act, key);
          const int leader = __ffs(grp) - 1;
          uint32_t b = 0;
          if (lane == leader) b = atomicAdd(&A.cursor[key], (uint32_t)__popc(grp));
          b = __shfl_sync(grp, b, leader);
          dst = b + (uint32_t)__popc(grp & lt_mask);
        }
      }
      if (active) {
        A.out.x[dst] = nx; A.out.y[dst] = ny; A.out.z[dst] = nz;
        A.out.vx[dst] = w[0]; A.out.vy[dst] = w[1]; A.out.vz[dst] = w[2];
        A.out.id[dst] = pid[u];
        if (!A.uniform_mass) A.out.m[dst] = mm[u];
      }
    }
  }
}

// ---------------------------------------------------- diagnostics reduce --
__global__ void __launch_bounds__(1024) k_diag_finalize(const double* partials, int64_t ntiles,
                                                       unsigned long long* drift_bits,
                                                       double* out, int64_t n, int64_t step) {
  __shared__ double s[5][1024];
  const int t = threadIdx.x;
  double acc[5] = {0, 0, 0, 0, 0};
  const int64_t chunk = (ntiles + 1023) / 1024;
  const int64_t lo = t * chunk, hi = min(ntiles, lo + chunk);
  for (int64_t i = lo; i < hi; ++i)
    for (int c = 0; c < 5; ++c) acc[c] += partials[i * 8 + c];
  for (int c = 0; c < 5; ++c) s[c][t] = acc[c];
  __syncthreads();
  for (int w = 512; w > 0; w >>= 1) {
    if (t < w)
      for (int c = 0; c < 5; ++c) s[c][t] += s[c][t + w];
    __syncthreads();
  }
  if (t == 0) {
    out[0] = s[0][0]; out[1] = s[1][0]; out[2] = s[2][0];
    out[3] = 0.5 * s[3][0];
    out[4] = s[4][0];
    out[5] = __longlong_as_double((long long)*drift_bits);
    out[6] = (double)n;
    out[7] = (double)step;
    *drift_bits = 0ULL;
  }
}

// ------------------------------------------------ rebin / upload helpers --
// Histogram of the cells of step `k` over an unsorted SoA state.
__global__ void k_count_soa(SoA s, int64_t n, double o0, double o1, double o2, double a, int unit,
                            int64_t L0, int64_t L1, int64_t L2, uint32_t* counts) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t ix = pymod(cell_coord(s.x[i], o0, a, unit), L0);
    int64_t iy = pymod(cell_coord(s.y[i], o1, a, unit), L1);
    int64_t iz = pymod(cell_coord(s.z[i], o2, a, unit), L2);
    atomicAdd(&counts[(ix * L1 + iy) * L2 + iz], 1u);
  }
}

__global__ void k_scatter_soa(SoA in, SoA out, int64_t n, double o0, double o1, double o2,
                              double a, int unit, int64_t L0, int64_t L1, int64_t L2,
                              uint32_t* cursor, int uniform_mass) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t ix = pymod(cell_coord(in.x[i], o0, a, unit), L0);
    int64_t iy = pymod(cell_coord(in.y[i], o1, a, unit), L1);
    int64_t iz = pymod(cell_coord(in.z[i], o2, a, unit), L2);
    uint32_t d = atomicAdd(&cursor[(ix * L1 + iy) * L2 + iz], 1u);
    out.x[d] = in.x[i]; out.y[d] = in.y[i]; out.z[d] = in.z[i];
    out.vx[d] = in.vx[i]; out.vy[d] = in.vy[i]; out.vz[d] = in.vz[i];
    out.id[d] = in.id[i];
    if (!uniform_mass) out.m[d] = in.m[i];
  }
}

// (n,3) AoS host layout <-> SoA
__global__ void k_aos_to_soa(const double* pos, const double* vel, const double* mass,
                             const int64_t* ids, int64_t n, SoA out, int uniform_mass) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    out.x[i] = pos[3 * i]; out.y[i] = pos[3 * i + 1]; out.z[i] = pos[3 * i + 2];
    out.vx[i] = vel[3 * i]; out.vy[i] = vel[3 * i + 1]; out.vz[i] = vel[3 * i + 2];
    out.id[i] = ids ? (uint32_t)ids[i] : (uint32_t)i;
    if (!uniform_mass) out.m[i] = mass[i];
  }
}

__global__ void k_soa_to_aos(SoA in, int64_t n, int by_id, double* pos, double* vel, double* mass,
                             int64_t* ids, int uniform_mass, double m0) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = by_id ? (int64_t)in.id[i] : i;
    if (pos) { pos[3 * r] = in.x[i]; pos[3 * r + 1] = in.y[i]; pos[3 * r + 2] = in.z[i]; }
    if (vel) { vel[3 * r] = in.vx[i]; vel[3 * r + 1] = in.vy[i]; vel[3 * r + 2] = in.vz[i]; }
    if (mass) mass[r] = uniform_mass ? m0 : in.m[i];
    if (ids) ids[r] = (int64_t)in.id[i];
  }
}

// LinkedCellList of the current binning in particle-id space.
__global__ void k_binning_debug(const uint32_t* ends, int64_t C, const uint32_t* id, int64_t n,
                                int64_t* cells, int64_t* perm) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = C - 1;  // first cell with ends[c] > j
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (ends[mid] > (uint32_t)j) hi = mid; else lo = mid + 1;
    }
    const int64_t c = lo;
    const uint32_t s = c ? ends[c - 1] : 0u, e = ends[c];
    const uint32_t me = id[j];
    uint32_t rank = 0;
    for (uint32_t q = s; q < e; ++q) rank += (id[q] < me) ? 1u : 0u;
    if (cells) cells[me] = c;
    if (perm) perm[s + rank] = (int64_t)me;
  }
}

__global__ void k_ends_to_counts(const uint32_t* ends, int64_t C, int64_t* counts, int64_t* offs) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < C;
       c += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t s = c ? ends[c - 1] : 0u;
    if (counts) counts[c] = (int64_t)(ends[c] - s);
    if (offs) offs[c] = (int64_t)s;
  }
}

// particles.py:101-127 on the device: positions are exact (integer hash *
// box); velocities use device log/cos (numpy agrees to ~1 ulp only).
__global__ void k_init_device(SoA out, int64_t n, uint64_t state, double b0, double b1, double b2,
                              double sigma, double* vsum_partials) {
  __shared__ double s_sum[3][256];
  double acc[3] = {0, 0, 0};
  const double two_pi = 2.0 * 3.141592653589793;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    out.x[i] = uniform_at(state, (uint64_t)(3 * i)) * b0;
    out.y[i] = uniform_at(state, (uint64_t)(3 * i + 1)) * b1;
    out.z[i] = uniform_at(state, (uint64_t)(3 * i + 2)) * b2;
    double v[3];
    for (int d = 0; d < 3; ++d) {
      const uint64_t g = (uint64_t)(3 * n + 3 * i + d);
      const double u1 = uniform_at(state, 2 * g), u2 = uniform_at(state, 2 * g + 1);
      v[d] = sqrt(-2.0 * log(1.0 - u1)) * cos(two_pi * u2) * sigma;
      acc[d] += v[d];
    }
    out.vx[i] = v[0]; out.vy[i] = v[1]; out.vz[i] = v[2];
    out.id[i] = (uint32_t)i;
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

__global__ void k_init_remove_mean(SoA s, int64_t n, const double* vsum_partials, int nblocks) {
  __shared__ double mean[3];
  if (threadIdx.x < 3) {
    double acc = 0.0;
    for (int b = 0; b < nblocks; ++b) acc += vsum_partials[b * 3 + threadIdx.x];
    mean[threadIdx.x] = n ? acc / (double)n : 0.0;
  }
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    s.vx[i] -= mean[0]; s.vy[i] -= mean[1]; s.vz[i] -= mean[2];
  }
}

}  // namespace mpcd

// =============================================================== context ==
using namespace mpcd;

struct mpcd_ctx {
  mpcd_config cfg;
  int64_t C = 0, ntiles = 0, n = 0;
  int dev = 0;
  void* slab[2] = {nullptr, nullptr};
  SoA buf[2];
  int cur = 0;
  uint32_t* ends[2] = {nullptr, nullptr};
  int ecur = 0;
  uint32_t* counts = nullptr;
  double* comax = nullptr;
  double* partials = nullptr;
  double* diag = nullptr;
  unsigned long long* drift_bits = nullptr;
  uint32_t* flags = nullptr;
  uint32_t* overflow = nullptr;
  ScanState scan;
  int64_t cur_step = 0;   // binning of the state is for this step
  bool binned = false;
  bool have_diag = false;
  int64_t last_step = -1;
  int last_flags = 0;
  // optional per-kernel CUDA-event timing of mpcd_step (mpcd_profile)
  bool prof = false;
  std::vector<cudaEvent_t> prof_events;  // kProfSlots + 1 per profiled step
};

namespace {

constexpr int kProfSlots = 5;  // collide_count, dense, scan, collide_scatter, finalize

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

SoA carve(void* slab, int64_t cap, bool with_mass) {
  SoA s;
  double* d = static_cast<double*>(slab);
  s.x = d; s.y = d + cap; s.z = d + 2 * cap;
  s.vx = d + 3 * cap; s.vy = d + 4 * cap; s.vz = d + 5 * cap;
  s.m = with_mass ? d + 6 * cap : nullptr;
  s.id = reinterpret_cast<uint32_t*>(d + (with_mass ? 7 : 6) * cap);
  return s;
}

StepArgs make_args(mpcd_ctx* c, int64_t step, int flags) {
  StepArgs A;
  const mpcd_config& g = c->cfg;
  A.in = c->buf[c->cur];
  A.out = c->buf[c->cur ^ 1];
  A.ends = c->ends[c->ecur];
  A.counts = c->counts;
  A.cursor = c->ends[c->ecur ^ 1];
  A.comax = c->comax;
  A.partials = c->partials;
  A.drift_bits = c->drift_bits;
  A.flags = c->flags;
  A.overflow = c->overflow;
  A.L0 = g.dims[0]; A.L1 = g.dims[1]; A.L2 = g.dims[2];
  A.C = c->C;
  A.a = g.cell_size;
  A.unit_a = g.cell_size == 1.0;
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
  A.uniform_mass = g.uniform_mass;
  A.m0 = g.mass_value;
  A.want_drift = (flags & MPCD_STEP_WANT_DRIFT) ? 1 : 0;
  A.by_id = 0;
  return A;
}

// Sort the resident (unsorted or differently binned) state for step `step`:
// histogram, scan, scatter into the other buffer.
int rebin(mpcd_ctx* c, int64_t step, cudaStream_t st) {
  const mpcd_config& g = c->cfg;
  double off[3];
  grid_shift(g.prng, g.seed, (uint64_t)step, g.cell_size, off);
  const int unit = g.cell_size == 1.0;
  if (c->n > 0) {
    unsigned grid = grid_for(c->n, 256);
    k_count_soa<<<grid, 256, 0, st>>>(c->buf[c->cur], c->n, off[0], off[1], off[2], g.cell_size,
                                      unit, g.dims[0], g.dims[1], g.dims[2], c->counts);
    MPCD_LAUNCH_CHECK();
  }
  int rc = scan_u32(c->scan, c->counts, c->ends[c->ecur ^ 1], nullptr, c->C, true, st);
  if (rc) return rc;
  if (c->n > 0) {
    unsigned grid = grid_for(c->n, 256);
    k_scatter_soa<<<grid, 256, 0, st>>>(c->buf[c->cur], c->buf[c->cur ^ 1], c->n, off[0], off[1],
                                        off[2], g.cell_size, unit, g.dims[0], g.dims[1], g.dims[2],
                                        c->ends[c->ecur ^ 1], g.uniform_mass);
    MPCD_LAUNCH_CHECK();
  }
  c->cur ^= 1;
  c->ecur ^= 1;
  c->cur_step = step;
  c->binned = true;
  return MPCD_OK;
}

int launch_step(mpcd_ctx* c, int64_t step, int flags, bool by_id, cudaStream_t st) {
  if (!c->binned || c->cur_step != step) {
    int rc = rebin(c, step, st);
    if (rc) return rc;
  }
  StepArgs A = make_args(c, step, flags);
  A.by_id = by_id ? 1 : 0;
  const unsigned tiles = (unsigned)c->ntiles;
  cudaEvent_t* ev = nullptr;
  if (c->prof) {
    const size_t base = c->prof_events.size();
    c->prof_events.resize(base + kProfSlots + 1);
    ev = c->prof_events.data() + base;
    for (int i = 0; i <= kProfSlots; ++i) MPCD_CUDA(cudaEventCreate(&ev[i]));
    MPCD_CUDA(cudaEventRecord(ev[0], st));
  }
  auto mark = [&](int i) -> int {
    if (ev) MPCD_CUDA(cudaEventRecord(ev[i], st));
    return MPCD_OK;
  };
  k_collide_count<<<tiles, kNTA, 0, st>>>(A);
  MPCD_LAUNCH_CHECK();
  if (mark(1)) return MPCD_ERR_CUDA;
  k_collide_count_dense<<<std::min<int64_t>(c->ntiles, 592), kNTA, 0, st>>>(A);
  MPCD_LAUNCH_CHECK();
  if (mark(2)) return MPCD_ERR_CUDA;
  if (!by_id) {
    int rc = scan_u32(c->scan, c->counts, c->ends[c->ecur ^ 1], nullptr, c->C, true, st);
    if (rc) return rc;
  }
  if (mark(3)) return MPCD_ERR_CUDA;
  k_collide_scatter<<<tiles, kNTB, 0, st>>>(A);
  MPCD_LAUNCH_CHECK();
  if (mark(4)) return MPCD_ERR_CUDA;
  MPCD_CUDA(cudaMemsetAsync(c->flags, 0, sizeof(uint32_t), st));  // overflow count
  k_diag_finalize<<<1, 1024, 0, st>>>(c->partials, c->ntiles, c->drift_bits, c->diag, c->n, step);
  MPCD_LAUNCH_CHECK();
  if (mark(5)) return MPCD_ERR_CUDA;
  c->cur ^= 1;
  if (by_id) {
    c->binned = false;
  } else {
    c->ecur ^= 1;
    c->cur_step = step + 1;
  }
  c->have_diag = true;
  c->last_step = step;
  c->last_flags = flags;
  return MPCD_OK;
}

}  // namespace

extern "C" {

int mpcd_ctx_create(const mpcd_config* cfg, mpcd_ctx** out) {
  clear_error();
  if (!cfg || !out) return fail(MPCD_ERR_CONFIG, "null argument");
  for (int d = 0; d < 3; ++d)
    if (cfg->dims[d] < 1) return fail(MPCD_ERR_CONFIG, "dims must be positive");
  const int64_t C = cfg->dims[0] * cfg->dims[1] * cfg->dims[2];
  if (C >= (1LL << 32)) return fail(MPCD_ERR_CONFIG, "more than 2^32 cells per context");
  if (!(cfg->cell_size > 0.0)) return fail(MPCD_ERR_CONFIG, "cell_size must be positive");
  if (cfg->capacity < 0 || cfg->capacity >= (1LL << 32) - 1)
    return fail(MPCD_ERR_CONFIG, "capacity must be in [0, 2^32-1)");
  if (cfg->prng < 0 || cfg->prng > 3) return fail(MPCD_ERR_CONFIG, "unknown prng %d", cfg->prng);
  DeviceGuard dg(cfg->device);
  mpcd_ctx* c = new mpcd_ctx();
  c->cfg = *cfg;
  c->dev = cfg->device;
  c->C = C;
  c->ntiles = (C + kTC - 1) / kTC;
  const int64_t cap = std::max<int64_t>(cfg->capacity, 1);
  const bool with_mass = !cfg->uniform_mass;
  const size_t slab_bytes = (size_t)cap * (with_mass ? 7 : 6) * 8 + (size_t)cap * 4 + 256;
  auto cleanup = [&](int rc) {
    mpcd_ctx_destroy(c);
    return rc;
  };
  for (int b = 0; b < 2; ++b) {
    if (cudaMalloc(&c->slab[b], slab_bytes) != cudaSuccess)
      return cleanup(fail(MPCD_ERR_CUDA, "cudaMalloc of %zu bytes failed", slab_bytes));
    c->buf[b] = carve(c->slab[b], cap, with_mass);
  }
  for (int b = 0; b < 2; ++b)
    if (cudaMalloc(&c->ends[b], sizeof(uint32_t) * C) != cudaSuccess)
      return cleanup(fail(MPCD_ERR_CUDA, "cudaMalloc ends failed"));
  if (cudaMalloc(&c->counts, sizeof(uint32_t) * C) != cudaSuccess ||
      cudaMalloc(&c->comax, sizeof(double) * 6 * C) != cudaSuccess ||
      cudaMalloc(&c->partials, sizeof(double) * 8 * c->ntiles) != cudaSuccess ||
      cudaMalloc(&c->diag, sizeof(double) * 8) != cudaSuccess ||
      cudaMalloc(&c->drift_bits, sizeof(unsigned long long)) != cudaSuccess ||
      cudaMalloc(&c->flags, sizeof(uint32_t) * 4) != cudaSuccess ||
      cudaMalloc(&c->overflow, sizeof(uint32_t) * c->ntiles) != cudaSuccess)
    return cleanup(fail(MPCD_ERR_CUDA, "cudaMalloc of per-cell arrays failed"));
  cudaMemset(c->counts, 0, sizeof(uint32_t) * C);
  cudaMemset(c->ends[0], 0, sizeof(uint32_t) * C);
  cudaMemset(c->ends[1], 0, sizeof(uint32_t) * C);
  cudaMemset(c->comax, 0, sizeof(double) * 6 * C);
  cudaMemset(c->diag, 0, sizeof(double) * 8);
  cudaMemset(c->drift_bits, 0, sizeof(unsigned long long));
  cudaMemset(c->flags, 0, sizeof(uint32_t) * 4);
  int rc = c->scan.init(C);
  if (rc) return cleanup(rc);
  if (cudaDeviceSynchronize() != cudaSuccess)
    return cleanup(fail(MPCD_ERR_CUDA, "context init failed: %s", cudaGetErrorString(cudaGetLastError())));
  *out = c;
  return MPCD_OK;
}

int mpcd_ctx_destroy(mpcd_ctx* c) {
  if (!c) return MPCD_OK;
  DeviceGuard dg(c->dev);
  for (int b = 0; b < 2; ++b) {
    if (c->slab[b]) cudaFree(c->slab[b]);
    if (c->ends[b]) cudaFree(c->ends[b]);
  }
  if (c->counts) cudaFree(c->counts);
  if (c->comax) cudaFree(c->comax);
  if (c->partials) cudaFree(c->partials);
  if (c->diag) cudaFree(c->diag);
  if (c->drift_bits) cudaFree(c->drift_bits);
  if (c->flags) cudaFree(c->flags);
  if (c->overflow) cudaFree(c->overflow);
  for (cudaEvent_t e : c->prof_events) cudaEventDestroy(e);
  c->scan.release();
  delete c;
  return MPCD_OK;
}

int64_t mpcd_count(const mpcd_ctx* c) { return c ? c->n : -1; }
int64_t mpcd_current_step(const mpcd_ctx* c) { return c ? c->cur_step : -1; }

int mpcd_upload(mpcd_ctx* c, const double* pos, const double* vel, const double* mass,
                const int64_t* ids, int64_t n, int64_t step, void* stream) {
  clear_error();
  if (!c) return fail(MPCD_ERR_CONFIG, "null context");
  if (n < 0 || n > c->cfg.capacity)
    return fail(MPCD_ERR_CAPACITY, "%lld particles exceed capacity %lld", (long long)n,
                (long long)c->cfg.capacity);
  if (n > 0 && (!pos || !vel)) return fail(MPCD_ERR_CONFIG, "positions/velocities required");
  if (n > 0 && !c->cfg.uniform_mass && !mass) return fail(MPCD_ERR_CONFIG, "masses required");
  DeviceGuard dg(c->dev);
  cudaStream_t st = as_stream(stream);
  c->n = n;
  if (n > 0) {
    // stage the host AoS rows in the destination slab, then transpose
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
    k_aos_to_soa<<<grid_for(n, 256), 256, 0, st>>>(dpos, dvel, dmass, ids ? dids : nullptr, n,
                                                   c->buf[c->cur], c->cfg.uniform_mass);
    MPCD_LAUNCH_CHECK();
    MPCD_CUDA(cudaFreeAsync(tmp, st));
  }
  c->binned = false;
  c->have_diag = false;
  return rebin(c, step, st);
}

int mpcd_download(mpcd_ctx* c, double* pos, double* vel, double* mass, int64_t* ids,
                  int32_t id_order, void* stream) {
  clear_error();
  if (!c) return fail(MPCD_ERR_CONFIG, "null context");
  DeviceGuard dg(c->dev);
  cudaStream_t st = as_stream(stream);
  const int64_t n = c->n;
  if (n == 0) return MPCD_OK;
  double* tmp = nullptr;
  const size_t bytes = (size_t)n * 8 * 8;
  MPCD_CUDA(cudaMallocAsync(&tmp, bytes, st));
  double* dpos = tmp;
  double* dvel = tmp + 3 * n;
  double* dmass = tmp + 6 * n;
  int64_t* dids = reinterpret_cast<int64_t*>(tmp + 7 * n);
  k_soa_to_aos<<<grid_for(n, 256), 256, 0, st>>>(c->buf[c->cur], n, id_order ? 1 : 0,
                                                 pos ? dpos : nullptr, vel ? dvel : nullptr,
                                                 mass ? dmass : nullptr, ids ? dids : nullptr,
                                                 c->cfg.uniform_mass, c->cfg.mass_value);
  MPCD_LAUNCH_CHECK();
  if (pos) MPCD_CUDA(cudaMemcpyAsync(pos, dpos, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, st));
  if (vel) MPCD_CUDA(cudaMemcpyAsync(vel, dvel, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, st));
  if (mass) MPCD_CUDA(cudaMemcpyAsync(mass, dmass, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  if (ids) MPCD_CUDA(cudaMemcpyAsync(ids, dids, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, st));
  MPCD_CUDA(cudaFreeAsync(tmp, st));
  MPCD_CUDA(cudaStreamSynchronize(st));
  return MPCD_OK;
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
  DeviceGuard dg(c->dev);
  for (int64_t k = 0; k < n_steps; ++k) {
    int rc = launch_step(c, first_step + k, flags, false, as_stream(stream));
    if (rc) return rc;
  }
  return MPCD_OK;
}

int mpcd_read_diag(mpcd_ctx* c, mpcd_diag* out, void* stream) {
  clear_error();
  if (!c || !out) return fail(MPCD_ERR_CONFIG, "null argument");
  DeviceGuard dg(c->dev);
  cudaStream_t st = as_stream(stream);
  double h[8];
  uint32_t fl[4];
  MPCD_CUDA(cudaMemcpyAsync(h, c->diag, sizeof(h), cudaMemcpyDeviceToHost, st));
  MPCD_CUDA(cudaMemcpyAsync(fl, c->flags, sizeof(fl), cudaMemcpyDeviceToHost, st));
  MPCD_CUDA(cudaStreamSynchronize(st));
  if (fl[1]) {
    cudaMemsetAsync(c->flags + 1, 0, sizeof(uint32_t), st);
    return fail(MPCD_ERR_RNG, "axis rejection sampling failed to terminate");
  }
  out->momentum[0] = h[0]; out->momentum[1] = h[1]; out->momentum[2] = h[2];
  out->energy = h[3];
  out->mass = h[4];
  out->max_cell_drift = h[5];
  out->n = (int64_t)h[6];
  out->step = c->have_diag ? (int64_t)h[7] : -1;
  return MPCD_OK;
}

int mpcd_read_com(mpcd_ctx* c, int64_t* cell_ids, double* com, int64_t* n_occupied, void* stream) {
  clear_error();
  if (!c || !n_occupied) return fail(MPCD_ERR_CONFIG, "null argument");
  if (!c->have_diag) return fail(MPCD_ERR_CONFIG, "no step has run");
  DeviceGuard dg(c->dev);
  cudaStream_t st = as_stream(stream);
  // the binning used by the last step: the ends array not current any more
  // (after a by_id step the binning array was not advanced)
  const uint32_t* prev = c->binned ? c->ends[c->ecur ^ 1] : c->ends[c->ecur];
  std::vector<uint32_t> ends(c->C);
  MPCD_CUDA(cudaMemcpyAsync(ends.data(), prev, sizeof(uint32_t) * c->C, cudaMemcpyDeviceToHost, st));
  std::vector<double> cx;
  if (com) {
    cx.resize(6 * c->C);
    MPCD_CUDA(cudaMemcpyAsync(cx.data(), c->comax, sizeof(double) * 6 * c->C, cudaMemcpyDeviceToHost, st));
  }
  MPCD_CUDA(cudaStreamSynchronize(st));
  int64_t k = 0;
  uint32_t s = 0;
  for (int64_t cc = 0; cc < c->C; ++cc) {
    if (ends[cc] > s) {
      if (cell_ids) cell_ids[k] = cc;
      if (com) for (int d = 0; d < 3; ++d) com[3 * k + d] = cx[6 * cc + d];
      ++k;
    }
    s = ends[cc];
  }
  *n_occupied = k;
  return MPCD_OK;
}

int mpcd_read_binning(mpcd_ctx* c, int64_t* cells, int64_t* bin_count, int64_t* bin_offset,
                      int64_t* permutation, void* stream) {
  clear_error();
  if (!c) return fail(MPCD_ERR_CONFIG, "null context");
  DeviceGuard dg(c->dev);
  cudaStream_t st = as_stream(stream);
  if (!c->binned) {
    int rc = rebin(c, c->cur_step, st);
    if (rc) return rc;
  }
  const int64_t n = c->n, C = c->C;
  int64_t* tmp = nullptr;
  MPCD_CUDA(cudaMallocAsync(&tmp, sizeof(int64_t) * (2 * n + 2 * C + 1), st));
  int64_t* dcells = tmp;
  int64_t* dperm = tmp + n;
  int64_t* dcnt = tmp + 2 * n;
  int64_t* doff = tmp + 2 * n + C;
  if (n > 0) {
    k_binning_debug<<<grid_for(n, 256), 256, 0, st>>>(c->ends[c->ecur], C, c->buf[c->cur].id, n,
                                                     dcells, dperm);
    MPCD_LAUNCH_CHECK();
  }
  k_ends_to_counts<<<grid_for(C, 256), 256, 0, st>>>(c->ends[c->ecur], C, dcnt, doff);
  MPCD_LAUNCH_CHECK();
  if (cells && n) MPCD_CUDA(cudaMemcpyAsync(cells, dcells, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, st));
  if (permutation && n) MPCD_CUDA(cudaMemcpyAsync(permutation, dperm, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, st));
  if (bin_count) MPCD_CUDA(cudaMemcpyAsync(bin_count, dcnt, sizeof(int64_t) * C, cudaMemcpyDeviceToHost, st));
  if (bin_offset) MPCD_CUDA(cudaMemcpyAsync(bin_offset, doff, sizeof(int64_t) * C, cudaMemcpyDeviceToHost, st));
  MPCD_CUDA(cudaFreeAsync(tmp, st));
  MPCD_CUDA(cudaStreamSynchronize(st));
  return MPCD_OK;
}

int mpcd_step_host(mpcd_ctx* c, double* pos, double* vel, const double* mass, int64_t n,
                   int64_t step, int32_t flags, double* drift, void* stream) {
  clear_error();
  if (!c) return fail(MPCD_ERR_CONFIG, "null context");
  int rc = mpcd_upload(c, pos, vel, mass, nullptr, n, step, stream);
  if (rc) return rc;
  DeviceGuard dg(c->dev);
  cudaStream_t st = as_stream(stream);
  rc = launch_step(c, step, flags, true, st);
  if (rc) return rc;
  // by-id scatter: storage row == particle id, copy straight out
  if (n > 0) {
    double* tmp = nullptr;
    MPCD_CUDA(cudaMallocAsync(&tmp, sizeof(double) * 6 * n, st));
    k_soa_to_aos<<<grid_for(n, 256), 256, 0, st>>>(c->buf[c->cur], n, 0, tmp, tmp + 3 * n, nullptr,
                                                   nullptr, 1, 0.0);
    MPCD_LAUNCH_CHECK();
    MPCD_CUDA(cudaMemcpyAsync(pos, tmp, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, st));
    MPCD_CUDA(cudaMemcpyAsync(vel, tmp + 3 * n, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, st));
    MPCD_CUDA(cudaFreeAsync(tmp, st));
  }
  mpcd_diag d;
  rc = mpcd_read_diag(c, &d, stream);
  if (rc) return rc;
  if (drift) *drift = d.max_cell_drift;
  return MPCD_OK;
}

int mpcd_init_device(mpcd_ctx* c, int64_t n, double velocity_variance, int64_t step, void* stream) {
  clear_error();
  if (!c) return fail(MPCD_ERR_CONFIG, "null context");
  if (n < 0 || n > c->cfg.capacity) return fail(MPCD_ERR_CAPACITY, "n exceeds capacity");
  if (!c->cfg.uniform_mass) return fail(MPCD_ERR_CONFIG, "device init needs uniform_mass");
  DeviceGuard dg(c->dev);
  cudaStream_t st = as_stream(stream);
  c->n = n;
  if (n > 0) {
    const int blocks = 148 * 8;
    double* part = nullptr;
    MPCD_CUDA(cudaMallocAsync(&part, sizeof(double) * 3 * blocks, st));
    const mpcd_config& g = c->cfg;
    k_init_device<<<blocks, 256, 0, st>>>(c->buf[c->cur], n, key_state(g.seed, 0, kInit, 0),
                                          g.dims[0] * g.cell_size, g.dims[1] * g.cell_size,
                                          g.dims[2] * g.cell_size, sqrt(velocity_variance), part);
    MPCD_LAUNCH_CHECK();
    k_init_remove_mean<<<blocks, 256, 0, st>>>(c->buf[c->cur], n, part, blocks);
    MPCD_LAUNCH_CHECK();
    MPCD_CUDA(cudaFreeAsync(part, st));
  }
  c->binned = false;
  c->have_diag = false;
  return rebin(c, step, st);
}

int mpcd_profile(mpcd_ctx* c, int32_t enable) {
  clear_error();
  if (!c) return fail(MPCD_ERR_CONFIG, "null context");
  DeviceGuard dg(c->dev);
  for (cudaEvent_t e : c->prof_events) cudaEventDestroy(e);
  c->prof_events.clear();
  c->prof = enable != 0;
  return MPCD_OK;
}

int mpcd_read_profile(mpcd_ctx* c, double* ms, int64_t* n_steps) {
  clear_error();
  if (!c || !ms) return fail(MPCD_ERR_CONFIG, "null argument");
  DeviceGuard dg(c->dev);
  for (int i = 0; i < kProfSlots; ++i) ms[i] = 0.0;
  const size_t per = kProfSlots + 1;
  const size_t steps = c->prof_events.size() / per;
  if (steps) MPCD_CUDA(cudaEventSynchronize(c->prof_events.back()));
  for (size_t s = 0; s < steps; ++s)
    for (int i = 0; i < kProfSlots; ++i) {
      float t = 0.f;
      MPCD_CUDA(cudaEventElapsedTime(&t, c->prof_events[s * per + i], c->prof_events[s * per + i + 1]));
      ms[i] += t;
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
