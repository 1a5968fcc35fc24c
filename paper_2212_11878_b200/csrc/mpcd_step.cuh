// mpcd_step.cuh -- the one-kernel SRD step over fixed-capacity cell regions
// (included once, by mpcd_engine.cu).
//
// Layout: every collision cell c of the step's grid owns
// `cap` record slots [c*cap, (c+1)*cap) of each record array; count[c] says
// how many are filled.  A cell that receives more than cap particles keeps
// the first cap in its region and the rest in an overflow list (record +
// cell), which the dense-tile kernel gathers next step.  With 180 GB of HBM
// the regions cost ~3x the state (cap = 32 at 10 particles/cell) and buy a
// single pass per step: read the tile's particles, collide, stream, and
// write each particle straight into its next-step cell, its slot claimed by
// an atomic on that cell's next count.  No scan, no second pass.
//
// Compile-time specialisation: UNIT (cell_size == 1: (x - off)/a is exact
// without the division), UMASS (uniform mass, the record's mass slot is
// unused), DRIFT (capture_drift: per-cell post-collision moments in numpy
// order), COM (capture_com: com rows to HBM), BYID (pure-function mode:
// write row `id` of a flat array, no next binning).
#pragma once

namespace mpcd {

// Particle = two sector-aligned 32-byte records; every store of the step
// writes whole 32 B sectors.
struct __align__(16) PRec {
  double x, y, z;
  uint32_t id, pad;
};
struct __align__(16) VRec {
  double vx, vy, vz, m;
};
struct Recs {
  PRec* p;
  VRec* v;
};

__device__ __forceinline__ double id_bits(uint32_t id) {
  return __longlong_as_double((long long)(unsigned long long)id);
}
__device__ __forceinline__ uint32_t bits_id(double d) {
  return (uint32_t)(unsigned long long)__double_as_longlong(d);
}
__device__ __forceinline__ double2 ld2cs(const void* p) {  // read-once stream
  return __ldcs(reinterpret_cast<const double2*>(p));
}
__device__ __forceinline__ void st2(void* p, double a, double b) {
  *reinterpret_cast<double2*>(p) = make_double2(a, b);
}
__device__ __forceinline__ void store_rec(const Recs& s, uint64_t dst, double x, double y,
                                          double z, uint32_t id, double vx, double vy, double vz,
                                          double m) {
  PRec* pr = s.p + dst;
  VRec* vr = s.v + dst;
  st2(&pr->x, x, y);
  st2(&pr->z, z, id_bits(id));
  st2(&vr->vx, vx, vy);
  st2(&vr->vz, vz, m);
}

struct StepArgs {
  Recs in, out;               // regions of this step / of the next step
  uint32_t* count_in;         // per cell of this step (zeroed once consumed)
  uint32_t* count_out;        // per cell of the next step (zero on entry)
  Recs ovf_in, ovf_out;       // overflow records
  uint32_t* ovf_cell_in;
  uint32_t* ovf_cell_out;
  uint32_t* ovf_n_in;         // entries in ovf_in
  uint32_t* ovf_n_out;        // claimed entries in ovf_out
  uint32_t ovf_cap;
  uint32_t cap;               // slots per cell
  double* partials;           // per tile: px py pz sum(m v^2) mass
  double* com_cap;            // COM: per cell com[3], count
  unsigned long long* drift_bits;
  uint32_t* flags;            // [0] dense tiles, [1] rng failure, [2] overflow list full
  uint32_t* dense;            // dense tile list
  uint32_t* scratch_n;        // dense-kernel staging allocator
  uint32_t* scratch_id;       // dense-kernel staging (n entries)
  double* scratch_val;        // dense-kernel staging (4 n doubles)
  uint32_t* scratch_src;      // dense-kernel: source slot of each staged row
  int L0, L1, L2;
  int64_t C;
  double a, dt, cs, sn, box0, box1, box2;
  double off_next0, off_next1, off_next2;
  uint64_t seed, step;
  int prng;
  double m0;
};

constexpr int kTC = 32;         // cells per tile (one warp owns the per-cell work)
constexpr int kNT = 256;        // threads of the step CTA
constexpr int kPPT = 3;         // staged particles per thread
constexpr int kMaxP = kNT * kPPT;  // padded staging slots per tile
constexpr uint32_t kSentinel = 0xFFFFFFFFu;

// ------------------------------------------------------------ cell index --
__device__ __noinline__ int cell_coord_slow(double t, int L) {
  return (int)pymod(__double2ll_rd(t), (int64_t)L);
}

template <bool UNIT>
__device__ __forceinline__ int cell_coord32(double x, double off, double a, int L) {
  double t = x - off;
  if (!UNIT) t = t / a;  // IEEE division, as collision.py:132
  const int c = __double2int_rd(t);
  if ((unsigned)c < (unsigned)L) return c;
  if (c == -1) return L - 1;
  if (c == L) return 0;
  return cell_coord_slow(t, L);
}

template <bool UNIT>
__device__ __forceinline__ uint32_t next_cell(const StepArgs& A, double x, double y, double z) {
  const unsigned ix = cell_coord32<UNIT>(x, A.off_next0, A.a, A.L0);
  const unsigned iy = cell_coord32<UNIT>(y, A.off_next1, A.a, A.L1);
  const unsigned iz = cell_coord32<UNIT>(z, A.off_next2, A.a, A.L2);
  return (ix * (unsigned)A.L1 + iy) * (unsigned)A.L2 + iz;
}

__device__ __noinline__ double wrap_slow(double x, double box) { return wrap(x, box); }

// particles.py:52-67 fast path (positions move less than a box per step)
__device__ __forceinline__ double wrap_fast(double x, double box) {
  if (x >= 0.0 && x < box) return x + 0.0;
  if (x < 0.0 && x >= -box) {
    const double m = x + box;
    return (m == box) ? 0.0 : m;
  }
  if (x >= box && x < 2.0 * box) return x - box;
  return wrap_slow(x, box);
}

// numpy pairwise leaf, compile-time stride, 32-bit indices
template <int S>
__device__ __forceinline__ double pw_leaf(const double* t, int n) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res += t[i * S];
    return res;
  }
  double r0 = t[0], r1 = t[S], r2 = t[2 * S], r3 = t[3 * S];
  double r4 = t[4 * S], r5 = t[5 * S], r6 = t[6 * S], r7 = t[7 * S];
  int i = 8;
  const int full = n - (n & 7);
  for (; i < full; i += 8) {
    const double* q = t + i * S;
    r0 += q[0]; r1 += q[S]; r2 += q[2 * S]; r3 += q[3 * S];
    r4 += q[4 * S]; r5 += q[5 * S]; r6 += q[6 * S]; r7 += q[7 * S];
  }
  double res = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7));
  for (; i < n; ++i) res += t[i * S];
  return res;
}

// np.add.reduceat of one column over k rows of stride S
template <int S>
__device__ __forceinline__ double reduceat_col(const double* t, int k) {
  if (k <= 0) return 0.0;
  if (k == 1) return t[0];
  if (k <= 129) return t[0] + pw_leaf<S>(t + S, k - 1);
  return t[0] + pairwise_sum(t + S, (int64_t)(k - 1), (int64_t)S);
}

__device__ __forceinline__ void atomic_max_pos_double(unsigned long long* p, double v) {
  atomicMax(p, (unsigned long long)__double_as_longlong(v));  // v >= 0
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

// Slot claims in the next binning, batched so that every atomic of a thread
// is in flight before any result is used.  One atomic per distinct
// destination cell per warp (match_any aggregation).
__device__ __forceinline__ void claim_slot(const StepArgs& A, bool active, uint32_t key,
                                           unsigned& grp, uint32_t& base) {
  const unsigned act = __ballot_sync(0xffffffffu, active);
  grp = 0u;
  base = 0u;
  if (active) {
    grp = __match_any_sync(act, key);
    if ((int)(threadIdx.x & 31) == __ffs(grp) - 1)
      base = atomicAdd(&A.count_out[key], (uint32_t)__popc(grp));
  }
}

// Store one collided particle into its claimed slot (or the overflow list).
__device__ __forceinline__ void finish_slot(const StepArgs& A, uint32_t key, unsigned grp,
                                            uint32_t base, const double* o, uint32_t id,
                                            double m) {
  const int lane = threadIdx.x & 31;
  base = __shfl_sync(grp, base, __ffs(grp) - 1);
  const uint32_t slot = base + (uint32_t)__popc(grp & ((1u << lane) - 1u));
  if (slot < A.cap) {
    store_rec(A.out, (uint64_t)key * A.cap + slot, o[0], o[1], o[2], id, o[3], o[4], o[5], m);
  } else {  // full cell: overflow list (gathered by the dense kernel next step)
    const uint32_t q = atomicAdd(A.ovf_n_out, 1u);
    if (q < A.ovf_cap) {
      store_rec(A.ovf_out, q, o[0], o[1], o[2], id, o[3], o[4], o[5], m);
      A.ovf_cell_out[q] = key;
    } else {
      atomicOr(&A.flags[2], 1u);
    }
  }
}

// Unbatched variant for the dense kernel.
template <bool UNIT, bool BYID>
__device__ __forceinline__ void emit(const StepArgs& A, bool active, double nx, double ny,
                                     double nz, uint32_t id, const double* w, double m) {
  const double o[6] = {nx, ny, nz, w[0], w[1], w[2]};
  if (BYID) {
    if (active) store_rec(A.out, id, nx, ny, nz, id, w[0], w[1], w[2], m);
    return;
  }
  const uint32_t key = active ? next_cell<UNIT>(A, nx, ny, nz) : 0u;
  unsigned grp;
  uint32_t base;
  claim_slot(A, active, key, grp, base);
  if (active) finish_slot(A, key, grp, base, o, id, m);
}

// ------------------------------------------------------- the step kernel --
template <bool UNIT, bool UMASS, bool DRIFT, bool COM, bool BYID>
__global__ void __launch_bounds__(kNT, 3) k_step(const StepArgs A) {
  __shared__ uint32_t s_cnt[kTC];
  __shared__ uint32_t s_off[kTC + 1];  // padded (multiple-of-4) segment starts
  __shared__ __align__(16) uint32_t s_id[kMaxP];
  __shared__ uint8_t s_cell[kMaxP];
  __shared__ __align__(16) double s_val[kMaxP * 4];
  __shared__ double s_mom[kTC * 4];
  __shared__ double s_post[DRIFT ? kTC * 4 : 1];
  __shared__ double s_cx[kTC * 6];
  __shared__ double s_red[(kNT / 32) * 4];
  __shared__ int s_dense;
  const int t = threadIdx.x, lane = t & 31;
  const int64_t tile = blockIdx.x;
  const int64_t c0 = tile * kTC;
  const int nc = (int)min((int64_t)kTC, A.C - c0);

  // phase 0 (warp 0): counts, padded segment offsets, dense-tile test
  if (t < 32) {
    const uint32_t cnt = (lane < nc) ? A.count_in[c0 + lane] : 0u;
    const uint32_t k = min(cnt, A.cap);
    uint32_t incl = (k + 3u) & ~3u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    s_cnt[lane] = cnt;
    s_off[lane + 1] = incl;
    if (lane == 0) s_off[0] = 0;
    const bool over = __any_sync(0xffffffffu, cnt > A.cap);
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    if (lane == 0) s_dense = (over || total > (uint32_t)kMaxP) ? 1 : 0;
  }
  __syncthreads();
  if (s_dense) {  // rare: the dense kernel handles this tile
    if (t == 0) A.dense[atomicAdd(&A.flags[0], 1u)] = (uint32_t)tile;
    return;
  }
  const int npad = (int)s_off[nc];
  if (t < nc) {
    // slot -> cell table; sentinel ids in the padding (they never rank below)
    const uint32_t lo = s_off[t], k = s_cnt[t], hi = s_off[t + 1];
    for (uint32_t j = lo; j < hi; ++j) s_cell[j] = (uint8_t)t;
    for (uint32_t j = lo + k; j < hi; ++j) s_id[j] = kSentinel;
    A.count_in[c0 + t] = 0u;  // consumed: this array is the count_out of step k+1
  }
  __syncthreads();

  // phase 1: issue the loads of (z, id) and the velocity record of every
  // particle; warp 0 draws the cells' rotation axes while they are in flight
  double vx[kPPT], vy[kPPT], vz[kPPT], pz[kPPT], mm[kPPT];
  uint32_t pid[kPPT];
  int lcell[kPPT];
  uint64_t src[kPPT];
#pragma unroll
  for (int r = 0; r < kPPT; ++r) {
    const int j = r * kNT + t;
    pid[r] = kSentinel;
    lcell[r] = 0;
    if (j < npad) {
      const int lc = s_cell[j];
      const uint32_t s = (uint32_t)j - s_off[lc];
      lcell[r] = lc;
      if (s < s_cnt[lc]) {
        src[r] = (uint64_t)(c0 + lc) * A.cap + s;
        const double2 zi = ld2cs(&A.in.p[src[r]].z);
        const double2 v01 = ld2cs(&A.in.v[src[r]].vx);
        const double2 v2m = ld2cs(&A.in.v[src[r]].vz);
        pz[r] = zi.x;
        pid[r] = bits_id(zi.y);
        vx[r] = v01.x; vy[r] = v01.y; vz[r] = v2m.x;
        mm[r] = UMASS ? A.m0 : v2m.y;
      }
    }
  }
  if (t < nc) {  // collision.py:217-250, keyed by the global cell id
    double* ax = s_cx + t * 6 + 3;
    ax[0] = ax[1] = ax[2] = 0.0;
    if (s_cnt[t] > 0u && !rotation_axis(A.prng, A.seed, A.step, (uint64_t)(c0 + t), ax))
      atomicOr(&A.flags[1], 1u);
  }
#pragma unroll
  for (int r = 0; r < kPPT; ++r)
    if (pid[r] != kSentinel) s_id[r * kNT + t] = pid[r];
  __syncthreads();

  // phase 2: rank by id inside the cell (4-wide over the padded segment);
  // stage (m v, m) in rank order -- the reference permutation is the stable
  // argsort over id order (collision.py:98)
  int slot[kPPT];
#pragma unroll
  for (int r = 0; r < kPPT; ++r) {
    slot[r] = 0;
    if (pid[r] != kSentinel) {
      const int lc = lcell[r];
      const int lo = (int)s_off[lc], hi = (int)s_off[lc + 1];
      const uint32_t me = pid[r];
      int rank = 0;
      for (int q = lo; q < hi; q += 4) {
        const uint4 w = *reinterpret_cast<const uint4*>(s_id + q);
        rank += (int)(w.x < me) + (int)(w.y < me) + (int)(w.z < me) + (int)(w.w < me);
      }
      slot[r] = lo + rank;
      double2* sv = reinterpret_cast<double2*>(s_val + slot[r] * 4);
      sv[0] = make_double2(mm[r] * vx[r], mm[r] * vy[r]);
      sv[1] = make_double2(mm[r] * vz[r], mm[r]);
    }
  }
  __syncthreads();

  // phase 3: per-cell moments, numpy reduceat association (collision.py:190-206)
  for (int task = t; task < nc * 4; task += kNT) {
    const int lc = task >> 2, comp = task & 3;
    s_mom[task] = reduceat_col<4>(s_val + s_off[lc] * 4 + comp, (int)min(s_cnt[lc], A.cap));
  }
  __syncthreads();

  // phase 4: com = p / m (collision.py:209-214)
  if (t < nc) {
    const double mass = s_mom[t * 4 + 3];
    double* cx = s_cx + t * 6;
    for (int d = 0; d < 3; ++d) cx[d] = (mass > 0.0) ? s_mom[t * 4 + d] / mass : 0.0;
    if (COM) {
      double* g = A.com_cap + (c0 + t) * 4;
      g[0] = cx[0]; g[1] = cx[1]; g[2] = cx[2]; g[3] = (double)s_cnt[t];
    }
  }
  __syncthreads();

  // phase 5: rotate (collision.py:289-306), stream + wrap (particles.py:62-67),
  // next-step cell; claim every slot, then store; stage post-collision rows
  double o[kPPT][6];
  uint32_t key[kPPT];
#pragma unroll
  for (int r = 0; r < kPPT; ++r) {
    key[r] = 0u;
    if (pid[r] != kSentinel) {
      const double* cx = s_cx + lcell[r] * 6;
      double v[3] = {vx[r], vy[r], vz[r]}, w[3];
      rotate(v, cx, cx + 3, A.cs, A.sn, w);
      const double2 xy = ld2cs(&A.in.p[src[r]].x);  // same sector as (z, id): L2 hit
      o[r][0] = wrap_fast(xy.x + w[0] * A.dt, A.box0);
      o[r][1] = wrap_fast(xy.y + w[1] * A.dt, A.box1);
      o[r][2] = wrap_fast(pz[r] + w[2] * A.dt, A.box2);
      o[r][3] = w[0]; o[r][4] = w[1]; o[r][5] = w[2];
      key[r] = BYID ? pid[r] : next_cell<UNIT>(A, o[r][0], o[r][1], o[r][2]);
      const double m = mm[r];
      double2* sv = reinterpret_cast<double2*>(s_val + slot[r] * 4);
      sv[0] = make_double2(m * w[0], m * w[1]);
      sv[1] = make_double2(m * w[2], m * (((0.0 + w[0] * w[0]) + w[1] * w[1]) + w[2] * w[2]));
    }
  }
  if (BYID) {
#pragma unroll
    for (int r = 0; r < kPPT; ++r)
      if (pid[r] != kSentinel)
        store_rec(A.out, pid[r], o[r][0], o[r][1], o[r][2], pid[r], o[r][3], o[r][4], o[r][5],
                  UMASS ? A.m0 : mm[r]);
  } else {
    unsigned grp[kPPT];
    uint32_t base[kPPT];
#pragma unroll
    for (int r = 0; r < kPPT; ++r) {
      grp[r] = 0u;
      base[r] = 0u;
      if (r * kNT < npad)  // warp-uniform: every lane takes part in the ballot
        claim_slot(A, pid[r] != kSentinel, key[r], grp[r], base[r]);
    }
#pragma unroll
    for (int r = 0; r < kPPT; ++r)
      if (pid[r] != kSentinel)
        finish_slot(A, key[r], grp[r], base[r], o[r], pid[r], UMASS ? A.m0 : mm[r]);
  }
  __syncthreads();

  // phase 6: tile partials (fixed order: deterministic) and drift
  if (DRIFT) {
    for (int task = t; task < nc * 4; task += kNT) {
      const int lc = task >> 2, comp = task & 3;
      s_post[task] = reduceat_col<4>(s_val + s_off[lc] * 4 + comp, (int)min(s_cnt[lc], A.cap));
    }
    __syncthreads();
    if (t < 5) {
      double s = 0.0;
      for (int lc = 0; lc < nc; ++lc) s += (t < 4) ? s_post[lc * 4 + t] : s_mom[lc * 4 + 3];
      A.partials[tile * 8 + t] = s;
    }
    if (t >= 32 && t < 64) {
      double worst = 0.0;
      for (int lc = t - 32; lc < nc; lc += 32)
        if (s_mom[lc * 4 + 3] > 0.0) worst = fmax(worst, cell_drift(s_mom + lc * 4, s_post + lc * 4));
      for (int off = 16; off > 0; off >>= 1)
        worst = fmax(worst, __shfl_xor_sync(0xffffffffu, worst, off));
      if (t == 32 && worst > 0.0) atomic_max_pos_double(A.drift_bits, worst);
    }
  } else {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int lc = t >> 5; lc < nc; lc += kNT / 32) {  // warp w: cells w, w + 8, ...
      const int lo = (int)s_off[lc], k = (int)min(s_cnt[lc], A.cap);
      for (int j = lo + lane; j < lo + k; j += 32)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q] += s_val[j * 4 + q];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      for (int off = 16; off > 0; off >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], off);
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < 4; ++q) s_red[(t >> 5) * 4 + q] = acc[q];
    __syncthreads();
    if (t < 4) {
      double s = 0.0;
      for (int w = 0; w < kNT / 32; ++w) s += s_red[w * 4 + t];
      A.partials[tile * 8 + t] = s;
    } else if (t == 4) {
      double s = 0.0;
      for (int lc = 0; lc < nc; ++lc) s += s_mom[lc * 4 + 3];
      A.partials[tile * 8 + 4] = s;
    }
  }
}

// ----------------------------------------------------- dense-tile kernel --
// Tiles with a cell above `cap` or more than kMaxP padded rows.  Gathers each
// cell's region slots plus its overflow entries into HBM staging, then the
// same phases with plain loops; ranking is O(k^2) per cell.  One CTA per
// queued tile (grid-strided); staging ranges come from a bump allocator.
template <bool UNIT, bool UMASS, bool DRIFT, bool COM, bool BYID>
__global__ void __launch_bounds__(kNT) k_step_dense(const StepArgs A) {
  __shared__ uint32_t s_cnt[kTC];
  __shared__ uint32_t s_off[kTC + 1];
  __shared__ uint32_t s_fill[kTC];
  __shared__ uint32_t s_base;
  __shared__ double s_mom[kTC * 4];
  __shared__ double s_post[kTC * 4];
  __shared__ double s_cx[kTC * 6];
  const int t = threadIdx.x;
  const uint32_t n_dense = *(volatile uint32_t*)&A.flags[0];
  const uint32_t n_ovf = min(*(volatile uint32_t*)A.ovf_n_in, A.ovf_cap);
  for (uint32_t e = blockIdx.x; e < n_dense; e += gridDim.x) {
    const int64_t tile = A.dense[e];
    const int64_t c0 = tile * kTC;
    const int nc = (int)min((int64_t)kTC, A.C - c0);
    __syncthreads();
    if (t == 0) {
      uint32_t acc = 0;
      for (int lc = 0; lc < kTC; ++lc) {
        const uint32_t cnt = lc < nc ? A.count_in[c0 + lc] : 0u;
        s_cnt[lc] = cnt;
        s_off[lc] = acc;
        s_fill[lc] = min(cnt, A.cap);
        acc += cnt;
      }
      s_off[kTC] = acc;
      s_base = atomicAdd(A.scratch_n, acc);
    }
    __syncthreads();
    const uint32_t np = s_off[kTC];
    uint32_t* g_id = A.scratch_id + s_base;
    uint32_t* g_src = A.scratch_src + s_base;  // region slot, or 0x80000000|overflow index
    double* g_val = A.scratch_val + 4 * (uint64_t)s_base;
    // gather: region slots in order, then overflow entries (claimed in order)
    for (int lc = 0; lc < nc; ++lc)
      for (uint32_t s = t; s < min(s_cnt[lc], A.cap); s += kNT) {
        g_id[s_off[lc] + s] = A.in.p[(uint64_t)(c0 + lc) * A.cap + s].id;
        g_src[s_off[lc] + s] = s;
      }
    for (uint32_t o = t; o < n_ovf; o += kNT) {
      const uint32_t c = A.ovf_cell_in[o];
      if (c >= (uint64_t)c0 && c < (uint64_t)(c0 + nc)) {
        const int lc = (int)(c - c0);
        const uint32_t at = s_off[lc] + atomicAdd(&s_fill[lc], 1u);
        g_id[at] = A.ovf_in.p[o].id;
        g_src[at] = 0x80000000u | o;
      }
    }
    __syncthreads();
    auto cell_of = [&](uint32_t j) {
      int lo = 0, hi = nc - 1;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (s_off[mid + 1] > j) hi = mid; else lo = mid + 1;
      }
      return lo;
    };
    auto rec_p = [&](uint32_t j, int lc) -> const PRec& {
      const uint32_t s = g_src[j];
      return (s & 0x80000000u) ? A.ovf_in.p[s & 0x7FFFFFFFu] : A.in.p[(uint64_t)(c0 + lc) * A.cap + s];
    };
    auto rec_v = [&](uint32_t j, int lc) -> const VRec& {
      const uint32_t s = g_src[j];
      return (s & 0x80000000u) ? A.ovf_in.v[s & 0x7FFFFFFFu] : A.in.v[(uint64_t)(c0 + lc) * A.cap + s];
    };
    auto rank_of = [&](uint32_t j, int lc) {
      const uint32_t me = g_id[j];
      uint32_t rank = 0;
      for (uint32_t q = s_off[lc]; q < s_off[lc + 1]; ++q) rank += (g_id[q] < me) ? 1u : 0u;
      return s_off[lc] + rank;
    };
    // staged rows live after the tile's np ids/srcs in g_val (4 per row)
    for (uint32_t j = t; j < np; j += kNT) {
      const int lc = cell_of(j);
      const uint32_t s = rank_of(j, lc);
      const VRec& v = rec_v(j, lc);
      const double m = UMASS ? A.m0 : v.m;
      g_val[4 * s] = m * v.vx; g_val[4 * s + 1] = m * v.vy; g_val[4 * s + 2] = m * v.vz;
      g_val[4 * s + 3] = m;
    }
    __syncthreads();
    for (int task = t; task < nc * 4; task += kNT) {
      const int lc = task >> 2, comp = task & 3;
      s_mom[task] =
          s_cnt[lc] ? reduceat(g_val + 4 * (uint64_t)s_off[lc] + comp, (int64_t)s_cnt[lc], 4) : 0.0;
    }
    __syncthreads();
    if (t < nc) {
      const double mass = s_mom[t * 4 + 3];
      double* cx = s_cx + t * 6;
      for (int d = 0; d < 3; ++d) cx[d] = (mass > 0.0) ? s_mom[t * 4 + d] / mass : 0.0;
      cx[3] = cx[4] = cx[5] = 0.0;
      if (s_cnt[t] > 0u && !rotation_axis(A.prng, A.seed, A.step, (uint64_t)(c0 + t), cx + 3))
        atomicOr(&A.flags[1], 1u);
      if (COM) {
        double* g = A.com_cap + (c0 + t) * 4;
        g[0] = cx[0]; g[1] = cx[1]; g[2] = cx[2]; g[3] = (double)s_cnt[t];
      }
    }
    __syncthreads();
    for (uint32_t base = 0; base < np; base += kNT) {
      const uint32_t j = base + t;
      const bool active = j < np;
      double w[3] = {0.0, 0.0, 0.0}, nx = 0.0, ny = 0.0, nz = 0.0, m = 0.0;
      uint32_t id = 0;
      if (active) {
        const int lc = cell_of(j);
        const uint32_t s = rank_of(j, lc);
        const PRec p = rec_p(j, lc);
        const VRec v = rec_v(j, lc);
        m = UMASS ? A.m0 : v.m;
        id = p.id;
        const double* cx = s_cx + lc * 6;
        double vv[3] = {v.vx, v.vy, v.vz};
        rotate(vv, cx, cx + 3, A.cs, A.sn, w);
        nx = wrap(p.x + w[0] * A.dt, A.box0);
        ny = wrap(p.y + w[1] * A.dt, A.box1);
        nz = wrap(p.z + w[2] * A.dt, A.box2);
        // pre-collision rows of slot s are no longer needed: post rows
        g_val[4 * s] = m * w[0]; g_val[4 * s + 1] = m * w[1]; g_val[4 * s + 2] = m * w[2];
        g_val[4 * s + 3] = m * (((0.0 + w[0] * w[0]) + w[1] * w[1]) + w[2] * w[2]);
      }
      emit<UNIT, BYID>(A, active, nx, ny, nz, id, w, UMASS ? A.m0 : m);
    }
    __syncthreads();
    for (int task = t; task < nc * 4; task += kNT) {
      const int lc = task >> 2, comp = task & 3;
      s_post[task] = s_cnt[lc] ? reduceat(g_val + 4 * (uint64_t)s_off[lc] + comp, (int64_t)s_cnt[lc], 4) : 0.0;
    }
    __syncthreads();
    if (t < 5) {
      double s = 0.0;
      for (int lc = 0; lc < nc; ++lc) s += (t < 4) ? s_post[lc * 4 + t] : s_mom[lc * 4 + 3];
      A.partials[tile * 8 + t] = s;
    }
    if (DRIFT && t >= 32 && t < 64) {
      double worst = 0.0;
      for (int lc = t - 32; lc < nc; lc += 32)
        if (s_mom[lc * 4 + 3] > 0.0) worst = fmax(worst, cell_drift(s_mom + lc * 4, s_post + lc * 4));
      for (int o = 16; o > 0; o >>= 1) worst = fmax(worst, __shfl_xor_sync(0xffffffffu, worst, o));
      if (t == 32 && worst > 0.0) atomic_max_pos_double(A.drift_bits, worst);
    }
    if (t < nc) A.count_in[c0 + t] = 0u;
  }
}

// ---------------------------------------------------- diagnostics reduce --
constexpr int kDiagBlocks = 592;

__global__ void __launch_bounds__(256) k_diag_partial(const double* partials, int64_t ntiles,
                                                     double* level1) {
  __shared__ double s[5][256];
  const int t = threadIdx.x;
  const int64_t per = (ntiles + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * per, hi = min(ntiles, lo + per);
  double acc[5] = {0, 0, 0, 0, 0};
  for (int64_t i = lo + t; i < hi; i += 256)
#pragma unroll
    for (int c = 0; c < 5; ++c) acc[c] += partials[i * 8 + c];
#pragma unroll
  for (int c = 0; c < 5; ++c) s[c][t] = acc[c];
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (t < w)
#pragma unroll
      for (int c = 0; c < 5; ++c) s[c][t] += s[c][t + w];
    __syncthreads();
  }
  if (t < 5) level1[blockIdx.x * 5 + t] = s[t][0];
}

// Final fixed-order sum; also retires the step's transient counters.
__global__ void __launch_bounds__(32) k_diag_finalize(const double* level1, int nblocks,
                                                     unsigned long long* drift_bits, double* out,
                                                     int64_t n, int64_t step, uint32_t* flags,
                                                     uint32_t* ovf_n_consumed,
                                                     uint32_t* scratch_n) {
  const int t = threadIdx.x;
  if (t < 5) {
    double s = 0.0;
    for (int b = 0; b < nblocks; ++b) s += level1[b * 5 + t];
    out[t] = (t == 3) ? 0.5 * s : s;
  }
  if (t == 0) {
    out[5] = __longlong_as_double((long long)*drift_bits);
    out[6] = (double)n;
    out[7] = (double)step;
    *drift_bits = 0ULL;
    flags[0] = 0u;         // dense-tile list consumed
    *ovf_n_consumed = 0u;  // this step's input overflow list consumed
    *scratch_n = 0u;
  }
}

}  // namespace mpcd
