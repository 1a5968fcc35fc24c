// mpcd_step.cuh -- the one-kernel SRD step over fixed-capacity cell regions
// (included by mpcd_engine.cu, which launches the non-template kernels, and by
// the four mpcd_step_<mode>.cu units, which instantiate the step variants).
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
// order), COM (capture_com: com rows to HBM), MODE: kBinned (one domain),
// kById (pure-function mode: write row `id` of a flat array, no next
// binning), kMulti (one domain of a decomposed box: leavers are written to
// per-rank send buffers instead of a local cell) or kFused (the same, leavers
// written straight into their owner's cells over peer memory).  Each mode
// compiles only its own leaver path, which keeps the hot loop's code small.
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
// A particle bound for another domain: both records back to back (64 B)
struct __align__(16) XRec {
  PRec p;
  VRec v;
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
// Record stores stream past L2 (evict-first): the step writes ~11 GB of
// records at 256^3 that are only read back next step from DRAM, and must not
// evict the next-step count array whose slot atomics sit on the critical path.
#ifndef MPCD_STCS
#define MPCD_STCS 1
#endif
__device__ __forceinline__ void st2(void* p, double a, double b) {
  if (MPCD_STCS)
    __stcs(reinterpret_cast<double2*>(p), make_double2(a, b));
  else
    *reinterpret_cast<double2*>(p) = make_double2(a, b);
}
// Next-step counts carry an evict-last hint: their slot atomics are on the
// critical path of every particle.  Measured 1 % faster than no hint,
// although the atomics' L2 miss ratio (about 45 %, at every box size) is the
// same either way (profiles/r01_k_step.md, v8).
#ifndef MPCD_PREFETCH_COUNTS
#define MPCD_PREFETCH_COUNTS 0  // measured slower (7.55 vs 7.40 ms): off
#endif
#ifndef MPCD_EARLYCLAIM
#define MPCD_EARLYCLAIM 1
#endif
#ifndef MPCD_BRANCHLESS4
#define MPCD_BRANCHLESS4 1
#endif
#ifndef MPCD_SOA
#define MPCD_SOA 1  // warp staging as columns (see consume_cells)
#endif
#ifndef MPCD_P2FLAT
#define MPCD_P2FLAT 0
#endif
#ifndef MPCD_FUSED_OOL
#define MPCD_FUSED_OOL 1  // fused migration: leavers claim + store in one out-of-line call
#endif
#ifndef MPCD_RANKU
#define MPCD_RANKU 3  // id groups of the rank loop unrolled (0: the do-while loop)
#endif
#ifndef MPCD_RANKORD
#define MPCD_RANKORD 1
#endif
#ifndef MPCD_CNT_EVICT_LAST
#define MPCD_CNT_EVICT_LAST 1
#endif
// producer: slot -> cell table written four slots per store
#ifndef MPCD_CELLW
#define MPCD_CELLW 1
#endif
// producer: two lanes per cell draw Marsaglia trials (tiles of <= 16 cells)
#ifndef MPCD_AXPAIR
#define MPCD_AXPAIR 1
#endif
// consumers: XOR-swizzled 16-byte halves of the 32-byte rows (bank conflicts)
// (measured slower on B200: the kernel's time follows its instruction count,
// and the swizzles' selects / column index math cost more issue slots than
// the bank conflicts they remove -- profiles/r02_k_step.md)
// producer: draw the next tile's axes into registers before waiting for a
// free buffer (the draw's latency hides in the wait)
#ifndef MPCD_EARLYAX
#define MPCD_EARLYAX 1
#endif
#ifndef MPCD_SWZ_W
#define MPCD_SWZ_W 0
#endif
#ifndef MPCD_SWZ_T
#define MPCD_SWZ_T 0
#endif
// MPCD_POLNV: the policy asm is not volatile (no side effects, no inputs),
// so the compiler computes it once instead of at every claim
#ifndef MPCD_POLNV
#define MPCD_POLNV 1
#endif
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
#if MPCD_POLNV
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
#else
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
#endif
  return pol;
}
// SYS: system scope, for the words that other GPUs claim in too (fused
// migration: a peer's k_step adds to this domain's counts over NVLink, and
// device-scope atomics of two GPUs are not atomic with respect to each other)
#ifndef MPCD_ABL_DEVSCOPE
#define MPCD_ABL_DEVSCOPE 0  // timing ablation only: device-scope local claims in fused mode
#endif
template <bool SYS = false>
__device__ __forceinline__ uint32_t count_claim(uint32_t* p, uint32_t v) {
  if (SYS && !MPCD_ABL_DEVSCOPE) return atomicAdd_system(p, v);
  if (!MPCD_CNT_EVICT_LAST) return atomicAdd(p, v);
  uint32_t old;
  asm volatile("atom.global.add.L2::cache_hint.u32 %0, [%1], %2, %3;"
               : "=r"(old)
               : "l"(p), "r"(v), "l"(policy_evict_last())
               : "memory");
  return old;
}
__device__ __forceinline__ void count_zero(uint32_t* p) {
  if (!MPCD_CNT_EVICT_LAST) {
    *p = 0u;
    return;
  }
  asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(p), "r"(0u),
               "l"(policy_evict_last())
               : "memory");
}

// One 32-byte record with a single 256-bit store (sm_100: STG.256), streaming.
#ifndef MPCD_ST256
#define MPCD_ST256 1
#endif
__device__ __forceinline__ void st4(void* p, double a, double b, double c, double d) {
  asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c),
               "d"(d)
               : "memory");
}

__device__ __forceinline__ void store_rec(const Recs& s, uint64_t dst, double x, double y,
                                          double z, uint32_t id, double vx, double vy, double vz,
                                          double m) {
  PRec* pr = s.p + dst;
  VRec* vr = s.v + dst;
  if (MPCD_ST256) {
    st4(pr, x, y, z, id_bits(id));
    st4(vr, vx, vy, vz, m);
    return;
  }
  st2(&pr->x, x, y);
  st2(&pr->z, z, id_bits(id));
  st2(&vr->vx, vx, vy);
  st2(&vr->vz, vz, m);
}

// The next-step buffers of every rank of a decomposed box, as this device
// addresses them (its own, or peer memory opened from another process's CUDA
// IPC handles, or another context of this process): the fused migration of
// k_step writes a leaving particle straight into its new owner's cell region.
// Index [b] = region set b (all ranks flip in lockstep).
struct PeerBufs {
  Recs reg[2];
  uint32_t* count[2];
  Recs ovf[2];
  uint32_t* ovf_cell[2];
  uint32_t* small;  // [2] overflow-list-full flag, [4 + b] overflow entries of set b
};

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
  // [0] dense tiles, [1] rng failure, [2] overflow list full, [3] routing
  // error, [8] overflow bucket allocator, [9] dense staging exhausted,
  // [10] a cell above kDenseMaxCell
  uint32_t* flags;
  uint32_t* dense;            // dense tile list (arrival order)
  uint32_t* dense_bits;       // one bit per tile: queued for k_step_dense
  uint32_t* cell_aux;         // per cell: its overflow bucket in ovf_sorted
  uint32_t* ovf_sorted;       // overflow entries bucketed by cell
  uint32_t* scratch_n;        // dense-kernel staging allocator (tiles above np_smem)
  uint32_t* scratch_id;       // dense-kernel staging (scratch_cap entries)
  double* scratch_val;        // dense-kernel staging (4 scratch_cap doubles)
  uint32_t* scratch_src;      // dense-kernel: source slot of each staged row
  uint32_t scratch_cap;
  uint32_t np_smem;           // particles of a dense tile staged in shared memory
  int ids31;                  // every id < kIds31Bound: sign-bit ranking
  int tc, cw;                 // cells per tile, cells per consumer warp (tc / 4)
  int L0, L1, L2;
  int64_t C;
  double a, dt, cs, sn, box0, box1, box2;
  double off_next0, off_next1, off_next2;
  uint64_t seed, step;
  uint64_t axis_prefix;       // key_prefix(seed, step, AXIS)
  int prng;
  double m0;
  int64_t dense_row0;         // partials row of dense tile t: dense_row0 + t
  // multi-domain (MODE == kMulti): this context owns the cells [o, o + L) of
  // a global G0 x G1 x G2 grid split into uniform blocks; rank of a block =
  // (bx * R1 + by) * R2 + bz.  Leavers go to send[dest * send_cap + slot].
  int G0, G1, G2;
  int o0, o1, o2;
  int R1, R2;
  XRec* send;
  unsigned long long* send_n;  // claimed per destination (may exceed send_cap)
  uint32_t send_cap;
  const PeerBufs* peers;       // non-null: fused migration over peer memory
  int n_ranks;                 // fused: ranks of the decomposed box (<= kMaxPeers)
  int out_set;                 // region set the step writes (the same on every rank)
};

// Step kernel modes: binned single domain, by-id pure function, multi-domain
constexpr int kBinned = 0, kById = 1, kMulti = 2, kFused = 3;
__host__ __device__ constexpr bool decomposed(int mode) { return mode >= kMulti; }

// Global (whole-box) id of local cell c: the key of its rotation axis
// (engine.py:82-92, 225-227 key axes by the global cell id).
template <int MODE>
__device__ __forceinline__ uint64_t global_cell_id(const StepArgs& A, int64_t c) {
  if (!decomposed(MODE)) return (uint64_t)c;
  // 32-bit division: a context holds fewer than 2^32 cells (mpcd_ctx_create)
  const uint32_t cc = (uint32_t)c, l2 = (uint32_t)A.L2, l1 = (uint32_t)A.L1;
  const uint32_t t = cc / l2, lz = cc - t * l2;
  const uint32_t lx = t / l1, ly = t - lx * l1;
  return ((uint64_t)(lx + A.o0) * (uint64_t)A.G1 + (uint64_t)(ly + A.o1)) * (uint64_t)A.G2 +
         (uint64_t)(lz + A.o2);
}

#ifndef MPCD_TC
#define MPCD_TC 32
#endif
#ifndef MPCD_MAXPT
#define MPCD_MAXPT 256
#endif
#ifndef MPCD_MINB
#define MPCD_MINB 4
#endif
constexpr int kTC = MPCD_TC;    // most cells per tile (one producer lane per cell, <= 32)
constexpr int kNT = 256;        // threads of the dense-tile CTA
constexpr uint32_t kSentinel = 0xFFFFFFFFu;
// Ids below 2^31 - 1 rank by the sign bit of a 32-bit difference (one add +
// one shift-add per compare instead of a compare + select + add); the
// padding then carries kSentinel31, which never counts as smaller.
constexpr uint32_t kIds31Bound = 0x7FFFFFFFu;
constexpr uint32_t kSentinel31 = 0x7FFFFFFFu;
constexpr int kPadBit = 0x80;  // slot-table flag of a padding slot
constexpr int kDiagCols = 7;  // partial columns: px py pz sum(m v^2) mass collided migrated

// ------------------------------------------------------------ cell index --
static __device__ __noinline__ int cell_coord_slow(double t, int L) {
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

// floor(t) mod L for t = (x - off) / a with x in [0, box) (a wrapped
// position) and |off| <= a/2: floor(t) is in [-1, L], mapped without a
// branch.  Anything else (NaN / inf from a corrupt state) leaves the result
// >= L, which cell_coord_fix sends through the exact general path.
template <bool UNIT>
__device__ __forceinline__ unsigned cell_coord_u(double x, double off, double a, int L, double& t) {
  t = x - off;
  if (!UNIT) t = t / a;  // IEEE division, as collision.py:132
  const int c = __double2int_rd(t);
  const unsigned u = (unsigned)(c < 0 ? c + L : c);  // -1 -> L - 1
  return u == (unsigned)L ? 0u : u;                  // L -> 0
}
__device__ __forceinline__ unsigned cell_coord_fix(unsigned u, double t, int L) {
  return u < (unsigned)L ? u : (unsigned)cell_coord_slow(t, L);
}

#ifndef MPCD_ONEBRANCH
#define MPCD_ONEBRANCH 1
#endif
template <bool UNIT>
__device__ __forceinline__ uint32_t next_cell(const StepArgs& A, double x, double y, double z) {
  if (MPCD_ONEBRANCH) {  // one rarely taken branch for the three axes
    double tx, ty, tz;
    unsigned ix = cell_coord_u<UNIT>(x, A.off_next0, A.a, A.L0, tx);
    unsigned iy = cell_coord_u<UNIT>(y, A.off_next1, A.a, A.L1, ty);
    unsigned iz = cell_coord_u<UNIT>(z, A.off_next2, A.a, A.L2, tz);
    if ((ix >= (unsigned)A.L0) | (iy >= (unsigned)A.L1) | (iz >= (unsigned)A.L2)) {
      ix = cell_coord_fix(ix, tx, A.L0);
      iy = cell_coord_fix(iy, ty, A.L1);
      iz = cell_coord_fix(iz, tz, A.L2);
    }
    return (ix * (unsigned)A.L1 + iy) * (unsigned)A.L2 + iz;
  }
  const unsigned ix = cell_coord32<UNIT>(x, A.off_next0, A.a, A.L0);
  const unsigned iy = cell_coord32<UNIT>(y, A.off_next1, A.a, A.L1);
  const unsigned iz = cell_coord32<UNIT>(z, A.off_next2, A.a, A.L2);
  return (ix * (unsigned)A.L1 + iy) * (unsigned)A.L2 + iz;
}

// A leaver's owner and its cell in the owner's numbering (uniform blocks:
// global mod block), packed (dest << 32 | key).  Out of line: the divisions
// are rare and would otherwise bloat every inlined copy of the hot loop.
static __device__ __noinline__ uint64_t foreign_target(int gx, int gy, int gz, int L0, int L1, int L2,
                                                int R1, int R2) {
  const int dest = ((gx / L0) * R1 + gy / L1) * R2 + gz / L2;
  const uint32_t key = ((uint32_t)(gx % L0) * (uint32_t)L1 + (uint32_t)(gy % L1)) * (uint32_t)L2 +
                       (uint32_t)(gz % L2);
  return ((uint64_t)(uint32_t)dest << 32) | key;
}

// Fused migration of one leaver: claim a slot in its owner's next-step cell
// and store it there over peer memory (or the owner's overflow list).  Out
// of line, scalar arguments only (no address of the kernel's parameters).
static __device__ __noinline__ void fused_put(const PeerBufs* peers, int b, uint32_t cap,
                                       uint32_t ovf_cap, int dest, uint32_t key, double x,
                                       double y, double z, uint32_t id, double vx, double vy,
                                       double vz, double m) {
  const PeerBufs& P = peers[dest];
  const uint32_t slot = atomicAdd_system(&P.count[b][key], 1u);
  // two 16-byte stores per record here: ptxas mis-assembles the 256-bit
  // inline-asm store inside a called (non-inlined) function
  auto put = [&](const Recs& r, uint64_t dst) {
    st2(&r.p[dst].x, x, y);
    st2(&r.p[dst].z, z, id_bits(id));
    st2(&r.v[dst].vx, vx, vy);
    st2(&r.v[dst].vz, vz, m);
  };
  if (slot < cap) {
    put(P.reg[b], (uint64_t)key * cap + slot);
  } else {  // the owner's cell is full: its overflow list
    const uint32_t q = atomicAdd_system(&P.small[4 + b], 1u);
    if (q < ovf_cap) {
      put(P.ovf[b], q);
      P.ovf_cell[b][q] = key;
    } else {
      atomicOr_system(&P.small[2], 1u);
    }
  }
}

// A fused leaver whose owner's cell is full (claimed slot >= cap): the
// owner's overflow list.  Out of line (rare).
static __device__ __noinline__ void fused_overflow(const PeerBufs* peers, int b,
                                                   uint32_t ovf_cap, int dest, uint32_t key,
                                                   double x, double y, double z, uint32_t id,
                                                   double vx, double vy, double vz, double m) {
  const PeerBufs& P = peers[dest];
  const uint32_t q = atomicAdd_system(&P.small[4 + b], 1u);
  if (q < ovf_cap) {
    st2(&P.ovf[b].p[q].x, x, y);
    st2(&P.ovf[b].p[q].z, z, id_bits(id));
    st2(&P.ovf[b].v[q].vx, vx, vy);
    st2(&P.ovf[b].v[q].vz, vz, m);
    P.ovf_cell[b][q] = key;
  } else {
    atomicOr_system(&P.small[2], 1u);
  }
}

// Multi-domain: the next-step cell in global coordinates (the serial
// formula, so binning is bit-identical to one domain); true and the local
// key when this domain owns it, else false and the owning rank.
template <bool UNIT>
__device__ __forceinline__ bool next_cell_multi(const StepArgs& A, double x, double y, double z,
                                                uint32_t& key, int& dest) {
  int gx, gy, gz;
  if (MPCD_ONEBRANCH) {
    double tx, ty, tz;
    unsigned ux = cell_coord_u<UNIT>(x, A.off_next0, A.a, A.G0, tx);
    unsigned uy = cell_coord_u<UNIT>(y, A.off_next1, A.a, A.G1, ty);
    unsigned uz = cell_coord_u<UNIT>(z, A.off_next2, A.a, A.G2, tz);
    if ((ux >= (unsigned)A.G0) | (uy >= (unsigned)A.G1) | (uz >= (unsigned)A.G2)) {
      ux = cell_coord_fix(ux, tx, A.G0);
      uy = cell_coord_fix(uy, ty, A.G1);
      uz = cell_coord_fix(uz, tz, A.G2);
    }
    gx = (int)ux;
    gy = (int)uy;
    gz = (int)uz;
  } else {
    gx = cell_coord32<UNIT>(x, A.off_next0, A.a, A.G0);
    gy = cell_coord32<UNIT>(y, A.off_next1, A.a, A.G1);
    gz = cell_coord32<UNIT>(z, A.off_next2, A.a, A.G2);
  }
  const unsigned lx = (unsigned)(gx - A.o0), ly = (unsigned)(gy - A.o1), lz = (unsigned)(gz - A.o2);
  if (__builtin_expect((lx < (unsigned)A.L0) & (ly < (unsigned)A.L1) & (lz < (unsigned)A.L2), 1)) {
    key = (lx * (unsigned)A.L1 + ly) * (unsigned)A.L2 + lz;
    return true;
  }
  const uint64_t t = foreign_target(gx, gy, gz, A.L0, A.L1, A.L2, A.R1, A.R2);
  dest = (int)(t >> 32);
  key = (uint32_t)t;
  return false;
}

static __device__ __noinline__ double wrap_slow(double x, double box) { return wrap(x, box); }

// particles.py:52-67 fast path (positions move less than a box per step)
__device__ __forceinline__ double wrap_fast(double x, double box) {
  // x in [+0, box): one unsigned compare of the bit patterns (box > 0, so
  // -0.0, negatives and NaN all compare above); x is then its own remainder,
  // already +0-signed (np.mod's copysign(0, box))
  if ((unsigned long long)__double_as_longlong(x) < (unsigned long long)__double_as_longlong(box))
    return x;
  if (x < 0.0 && x >= -box) {
    const double m = x + box;
    return (m == box) ? 0.0 : m;
  }
  if (x >= box && x < 2.0 * box) return x - box;
  return wrap_slow(x, box);
}

// Three coordinates with one rarely taken branch: x in [+0, box) is its own
// remainder (the bit-pattern compare of wrap_fast); any other value takes
// wrap_fast's full ladder.
__device__ __forceinline__ void wrap3(double& x, double& y, double& z, double bx, double by,
                                      double bz) {
  typedef unsigned long long u64;
  const bool fx = (u64)__double_as_longlong(x) < (u64)__double_as_longlong(bx);
  const bool fy = (u64)__double_as_longlong(y) < (u64)__double_as_longlong(by);
  const bool fz = (u64)__double_as_longlong(z) < (u64)__double_as_longlong(bz);
  if (!(fx & fy & fz)) {
    x = wrap_fast(x, bx);
    y = wrap_fast(y, by);
    z = wrap_fast(z, bz);
  }
}

// numpy pairwise leaf, compile-time stride, 32-bit indices
template <int S>
__device__ __forceinline__ double pw_leaf(const double* t, int n) {
  if (n < 16) {  // the common cell sizes, predicated instead of looped (same association)
    if (n < 8) {
      double res = 0.0;
#pragma unroll
      for (int i = 0; i < 7; ++i)
        if (i < n) res += t[i * S];
      return res;
    }
    double res = ((t[0] + t[S]) + (t[2 * S] + t[3 * S])) +
                 ((t[4 * S] + t[5 * S]) + (t[6 * S] + t[7 * S]));
#pragma unroll
    for (int i = 8; i < 15; ++i)
      if (i < n) res += t[i * S];
    return res;
  }
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
// Slot claims: one atomic per particle (MPCD_NOAGG=1, measured faster on
// B200 than warp aggregation with match_any: the atomics' L2 throughput is
// ample and the aggregation's MATCH / shuffle latency sat on the critical path)
#ifndef MPCD_NOAGG
#define MPCD_NOAGG 1
#endif
template <bool SYS>
__device__ __forceinline__ void claim_slot(const StepArgs& A, bool active, uint32_t key,
                                           unsigned& grp, uint32_t& base) {
  grp = 0u;
  base = 0u;
  if (MPCD_NOAGG) {  // one atomic per particle: the slot itself
#ifdef MPCD_ABL_NOATOM  // timing ablation only (wrong results): no claim round trip
    if (active) {  // the counts stay right (no-return reduction), the slot is made up
      atomicAdd(&A.count_out[key], 1u);
      base = (key ^ threadIdx.x) & 7u;
    }
    return;
#endif
    if (active) base = count_claim<SYS>(&A.count_out[key], 1u);
    return;
  }
  const unsigned act = __ballot_sync(0xffffffffu, active);
  if (active) {
    grp = __match_any_sync(act, key);
    if ((int)(threadIdx.x & 31) == __ffs(grp) - 1)
      base = count_claim<SYS>(&A.count_out[key], (uint32_t)__popc(grp));
  }
}

// Store one collided particle into its claimed slot (or the overflow list).
template <bool SYS>
__device__ __forceinline__ void finish_slot(const StepArgs& A, uint32_t key, unsigned grp,
                                            uint32_t base, const double* o, uint32_t id,
                                            double m) {
  const int lane = threadIdx.x & 31;
  uint32_t slot = base;
  if (!MPCD_NOAGG) {
    base = __shfl_sync(grp, base, __ffs(grp) - 1);
    slot = base + (uint32_t)__popc(grp & ((1u << lane) - 1u));
  }
  if (slot < A.cap) {
#ifdef MPCD_ABL_NOSTORE  // timing ablation only (wrong results): no record stores
    if (slot == 0xFFFFFFF0u)
#endif
    store_rec(A.out, (uint64_t)key * A.cap + slot, o[0], o[1], o[2], id, o[3], o[4], o[5], m);
  } else {  // full cell: overflow list (gathered by the dense kernel next step)
    const uint32_t q = SYS ? atomicAdd_system(A.ovf_n_out, 1u) : atomicAdd(A.ovf_n_out, 1u);
    if (q < A.ovf_cap) {
      store_rec(A.ovf_out, q, o[0], o[1], o[2], id, o[3], o[4], o[5], m);
      A.ovf_cell_out[q] = key;
    } else if (SYS) {
      atomicOr_system(&A.flags[2], 1u);
    } else {
      atomicOr(&A.flags[2], 1u);
    }
  }
}

// Multi-domain leavers: one atomic per destination rank per warp; a
// destination's count may run past send_cap (the host sees it and fails).
// Must be reached by the whole warp.
template <bool FUSED>
__device__ __forceinline__ void send_foreign(const StepArgs& A, bool active, int dest,
                                             uint32_t key, const double* o, uint32_t id,
                                             double m, double& migrated) {
  if (FUSED) {  // claim a slot in the owner's next-step cell, store there
    if (!active) return;
    migrated += 1.0;
    fused_put(A.peers, A.out_set, A.cap, A.ovf_cap, dest, key, o[0], o[1], o[2], id, o[3], o[4],
              o[5], m);
    return;
  }
  const unsigned act = __ballot_sync(0xffffffffu, active);
  if (!active) return;
  migrated += 1.0;
  const int lane = threadIdx.x & 31;
  const unsigned grp = __match_any_sync(act, dest);
  const int leader = __ffs(grp) - 1;
  unsigned long long base = 0ull;
  if (lane == leader) base = atomicAdd(&A.send_n[dest], (unsigned long long)__popc(grp));
  base = __shfl_sync(grp, base, leader);
  const unsigned long long slot = base + (unsigned long long)__popc(grp & ((1u << lane) - 1u));
  if (slot < A.send_cap) {
    XRec* x = A.send + (uint64_t)dest * A.send_cap + slot;
    st2(&x->p.x, o[0], o[1]);
    st2(&x->p.z, o[2], id_bits(id));
    st2(&x->v.vx, o[3], o[4]);
    st2(&x->v.vz, o[5], m);
  }
}

// Unbatched variant for the dense kernel.
template <bool UNIT, int MODE>
__device__ __forceinline__ void emit(const StepArgs& A, bool active, double nx, double ny,
                                     double nz, uint32_t id, const double* w, double m,
                                     double& migrated) {
  const double o[6] = {nx, ny, nz, w[0], w[1], w[2]};
  if (MODE == kById) {
    if (active) store_rec(A.out, id, nx, ny, nz, id, w[0], w[1], w[2], m);
    return;
  }
  uint32_t key = 0u;
  bool local = active;
  if (decomposed(MODE)) {
    int dest = 0;
    if (active) local = next_cell_multi<UNIT>(A, nx, ny, nz, key, dest);
    send_foreign<MODE == kFused>(A, active && !local, dest, key, o, id, m, migrated);
  } else if (active) {
    key = next_cell<UNIT>(A, nx, ny, nz);
  }
  unsigned grp;
  uint32_t base;
  claim_slot<MODE == kFused>(A, local, key, grp, base);
  if (local) finish_slot<MODE == kFused>(A, key, grp, base, o, id, m);
}

// ----------------------------------------------- shared-memory row access --
// The two 16-byte halves of a 32-byte row.  (Swizzling the half order by
// row to avoid the 2-way bank conflict of the 32-byte stride was measured
// slower on B200: the selects cost more issue slots than the conflicts.)
__device__ __forceinline__ void lds_row32(const void* base, int row, double2& lo, double2& hi) {
  const double2* p = reinterpret_cast<const double2*>(base) + 2 * row;
  lo = p[0];
  hi = p[1];
}
__device__ __forceinline__ void sts_row32(void* base, int row, double2 lo, double2 hi) {
  double2* p = reinterpret_cast<double2*>(base) + 2 * row;
  p[0] = lo;
  p[1] = hi;
}

// 32-byte rows read by consecutive lanes: rows r and r + 4 share a bank
// group, so eight lanes reading the same half of eight rows conflict 2-way.
// Swizzled rows (the warp-private staging W.val) keep half h of row r at
// 16 * (h ^ sw(r)) with sw(r) = (r >> 2) & 1, so the same access reaches all
// eight bank groups; a column element (r, c) is double c ^ 2 sw(r) of row r.
__device__ __forceinline__ int row_sw(int row) { return MPCD_SWZ_W ? (row >> 2) & 1 : 0; }
__device__ __forceinline__ void lds_row32w(const double* base, int row, double2& lo, double2& hi) {
  const double2* p = reinterpret_cast<const double2*>(base) + 2 * row;
  const int h = row_sw(row);
  lo = p[h];
  hi = p[h ^ 1];
}
__device__ __forceinline__ void sts_row32w(double* base, int row, double2 lo, double2 hi) {
  double2* p = reinterpret_cast<double2*>(base) + 2 * row;
  const int h = row_sw(row);
  p[h] = lo;
  p[h ^ 1] = hi;
}
// Rows laid out by the copy engine (the tile buffer, unswizzled): lanes with
// sw(r) = 1 load the high half first, which spreads the eight lanes of each
// access over all bank groups; the halves are put back in place by selects.
__device__ __forceinline__ void lds_row32t(const void* base, int row, double2& lo, double2& hi) {
  const double2* p = reinterpret_cast<const double2*>(base) + 2 * row;
  if (!MPCD_SWZ_T) {
    lo = p[0];
    hi = p[1];
    return;
  }
  const bool h = (row >> 2) & 1;
  const double2 a = p[h ? 1 : 0], b = p[h ? 0 : 1];
  lo.x = h ? b.x : a.x;
  lo.y = h ? b.y : a.y;
  hi.x = h ? a.x : b.x;
  hi.y = h ? a.y : b.y;
}

// numpy pairwise leaf over column c of swizzled rows row0 + 0 .. n - 1 (the
// association of pw_leaf, n < 129)
__device__ __forceinline__ double pw_leaf_w(const double* base, int row0, int c, int n) {
  auto at = [&](int i) {
    const int r = row0 + i;
    return base[r * 4 + (c ^ (row_sw(r) << 1))];
  };
  if (n < 16) {
    if (n < 8) {
      double res = 0.0;
#pragma unroll
      for (int i = 0; i < 7; ++i)
        if (i < n) res += at(i);
      return res;
    }
    double res = ((at(0) + at(1)) + (at(2) + at(3))) + ((at(4) + at(5)) + (at(6) + at(7)));
#pragma unroll
    for (int i = 8; i < 15; ++i)
      if (i < n) res += at(i);
    return res;
  }
  double r0 = at(0), r1 = at(1), r2 = at(2), r3 = at(3);
  double r4 = at(4), r5 = at(5), r6 = at(6), r7 = at(7);
  int i = 8;
  const int full = n - (n & 7);
  for (; i < full; i += 8) {
    r0 += at(i); r1 += at(i + 1); r2 += at(i + 2); r3 += at(i + 3);
    r4 += at(i + 4); r5 += at(i + 5); r6 += at(i + 6); r7 += at(i + 7);
  }
  double res = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7));
  for (; i < n; ++i) res += at(i);
  return res;
}
// np.add.reduceat of column c over the k swizzled rows from row0 (k <= kSlotsW)
__device__ __forceinline__ double reduceat_wcol(const double* base, int row0, int c, int k) {
  if (!MPCD_SWZ_W) {  // immediate offsets; k <= kSlotsW < 130: one pairwise leaf
    const double* t = base + row0 * 4 + c;
    if (k <= 0) return 0.0;
    if (k == 1) return t[0];
    return t[0] + pw_leaf<4>(t + 4, k - 1);
  }
  if (k <= 0) return 0.0;
  const double first = base[row0 * 4 + (c ^ (row_sw(row0) << 1))];
  if (k == 1) return first;
  return first + pw_leaf_w(base, row0 + 1, c, k - 1);
}

// ------------------------------------------------------------ TMA helpers --
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "MPCD_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra MPCD_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// 1-D bulk copy global -> shared (TMA), completion counted on `bar`
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

#ifdef MPCD_TIMING
static __device__ unsigned long long g_phase_cycles[10];
// producer warps: [0] cycles waiting for a free buffer, [1] cycles preparing tiles
static __device__ unsigned long long g_prod_cycles[2];
// per-warp shared accumulators (S.tim), flushed once per warp at kernel end
#define MPCD_PROBE(k)                                                              \
  do {                                                                             \
    const long long now_ = clock64();                                              \
    if ((k) > 0 && (threadIdx.x & 31) == 0)                                        \
      S.tim[threadIdx.x >> 5][(k)] += (unsigned long long)(now_ - probe_t_);       \
    probe_t_ = now_;                                                               \
  } while (0)
#else
#define MPCD_PROBE(k) do {} while (0)
#endif

// ------------------------------------------------------- the step kernel --
// Persistent and warp-specialised.  CTA b walks tiles b, b + G, ...  The
// producer warp prepares tiles ahead of the consumers: reads the tile's
// counts, lays out its records in shared memory (each cell padded to a
// multiple of 4 slots), writes the slot -> cell table, issues one
// cp.async.bulk (TMA) per cell and record array, zeroes the consumed counts
// and draws the cells' rotation axes.  Each consumer warp owns A.cw <= kCW = 8 cells
// of the tile and runs every phase on them alone -- rank, moments, com,
// rotation, stream, next-cell claims and stores -- synchronised only by
// __syncwarp, in warp-private shared scratch; so consumer warps never wait
// for each other.  Two tile buffers with full / empty mbarriers (empty
// counts one arrival per consumer warp).
constexpr int kMaxPT = MPCD_MAXPT;     // padded record slots per tile in shared memory
#ifndef MPCD_CW
#define MPCD_CW 8
#endif
constexpr int kCW = MPCD_CW;           // cells per consumer warp
constexpr int kNCW = kTC / kCW;        // consumer warps
constexpr int kNC = kNCW * 32;         // consumer threads
constexpr int kNTW = kNC + 32;         // + one producer warp
#ifndef MPCD_ROWSW
#define MPCD_ROWSW 2
#endif
constexpr int kRowsW = MPCD_ROWSW;     // slot rows per consumer lane
constexpr int kSlotsW = 32 * kRowsW;   // padded slots one consumer warp can hold
static_assert(kTC % kCW == 0 && kTC <= 32, "tile = whole consumer warps, one producer lane per cell");

struct TileBuf {
  PRec p[kMaxPT];
  VRec v[kMaxPT];
  double ax[kTC * 4];  // axis of each cell, padded to 4 doubles (two 16-byte loads)
  uint32_t cnt[kTC];
  uint32_t off[kTC + 1];
  uint8_t cell[kMaxPT];
  int skip;  // past the end, or a dense tile (queued for k_step_dense)
};

// Warp-private scratch.  Staged rows of cell q (0..3 inside the warp) live
// at rows [lo_q + q, hi_q + q) of val: the one-row skew per cell puts the four
// cells' moment columns in different bank groups.
struct __align__(16) WarpScratch {
  double val[(kSlotsW + kCW) * 4];  // (m v, m) rows in rank order; post rows later
  uint32_t id[kSlotsW];             // ids in slot order, sentinel in padding
  double mom[kCW * 4];
  double com[kCW * 4];  // com of each cell, padded to 4 doubles
};

#ifndef MPCD_STAGES
#define MPCD_STAGES 2
#endif
constexpr int kStages = MPCD_STAGES;  // tile buffers in flight per CTA

// Fused migration: the next-step count / record arrays of every rank, for
// the region set this step writes (copied from A.peers at kernel start), so
// a leaver's claim and store pick their target with a select, in line.
// Only the fused kernel carries it: 48 KB of shared memory per CTA is the
// most that keeps the 200 KB carve-out (56 KB of L1), and a larger carve-out
// measured 7 % slower.  More ranks than kMaxPeers use the exchange.
constexpr int kMaxPeers = 16;
struct PeerTable {
  uint32_t* count[kMaxPeers];
  PRec* p[kMaxPeers];
  VRec* v[kMaxPeers];
};
struct NoPeerTable {};

template <bool DRIFT, bool PEERS = false>
struct StepSmem {
  TileBuf buf[kStages];
  WarpScratch w[kNCW];
  typename std::conditional<PEERS, PeerTable, NoPeerTable>::type peer;
  double post[DRIFT ? kTC * 4 : 1];
  double red[kNCW * kDiagCols];
#ifdef MPCD_SMEM_PAD  // tuning: extra shared memory per CTA (carve-out / L1 experiments)
  unsigned char pad_[MPCD_SMEM_PAD];
#endif
#ifdef MPCD_TIMING
  unsigned long long tim[kNCW][10];
#endif
  uint64_t full[kStages], empty[kStages];
};

__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kNC) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Early release of a tile buffer (MPCD_EARLYREL): after the last pass's
// phase 4 instead of after its stores; not with the drift diagnostic (reads
// the tile's offsets later) or the exchange mode (flushes parked tile slots)
#ifndef MPCD_EARLYREL
#define MPCD_EARLYREL 1
#endif
template <bool DRIFT, int MODE>
constexpr bool kEarlyRel = MPCD_EARLYREL && !DRIFT && MODE != kMulti;

// Tile geometry: FIX = 16 compiles the 16-cell tile of ~10 particles per
// cell (the common density) into the kernel; FIX = 0 reads A.tc / A.cw (any
// multiple of kNCW up to kTC).  The compile-time form is ~1.5 % faster.
#define TILE_CELLS(A) (FIX ? FIX : (A).tc)
#define WARP_CELLS(A) (FIX ? FIX / kNCW : (A).cw)

template <int FIX>
__device__ __forceinline__ uint32_t tile_count(const StepArgs& A, int64_t tl, int64_t ntiles) {
  const int lane = threadIdx.x & 31;
  const int64_t c = tl * TILE_CELLS(A) + lane;
  return (lane < TILE_CELLS(A) && tl < ntiles && c < A.C) ? __ldcg(A.count_in + c) : 0u;
}

// A tile's rotation axes drawn ahead into registers (tiles of <= 16 cells,
// the reference's counter generator): lane pair (2 c, 2 c + 1) draws cell c;
// `write` marks the lane that stores B.ax[c] (the winning lane of the pair,
// or lane 2 c for an empty cell, whose axis stays zero).
struct AxisReg {
  double a0, a1, a2;
  bool write;
};

template <int MODE, int FIX>
__device__ __forceinline__ AxisReg draw_axes_early(const StepArgs& A, int64_t tl,
                                                   int64_t ntiles, uint32_t cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t c0 = tl * TILE_CELLS(A);
  const int nc = tl < ntiles ? (int)min((int64_t)TILE_CELLS(A), A.C - c0) : 0;
  const int cell = lane >> 1, s = lane & 1;
  const uint32_t ccnt = __shfl_sync(0xffffffffu, cnt, cell);
  bool done = !(cell < nc && ccnt > 0u);
  AxisReg r{0.0, 0.0, 0.0, s == 0 && cell < TILE_CELLS(A)};
  const uint64_t key = done ? 0ull : key_from_prefix(A.axis_prefix, global_cell_id<MODE>(A, c0 + cell));
  for (int i = 0; i < kMaxAxisTrials / 2; ++i) {
    if (!__any_sync(0xffffffffu, !done)) break;
    double x = 0.0, y = 0.0, rsq = 1.0;
    if (!done) {
      const uint64_t t = 2ull * (uint64_t)(2 * i + s);
      x = 2.0 * uniform_at(key, t) - 1.0;
      y = 2.0 * uniform_at(key, t + 1ull) - 1.0;
      rsq = x * x + y * y;
    }
    const unsigned acc = __ballot_sync(0xffffffffu, !done && rsq < 1.0);
    const unsigned pair = (acc >> (lane & ~1)) & 3u;
    if (!done && pair) {
      r.write = s == ((pair & 1u) ? 0 : 1);  // the earlier accepted trial of the pair
      if (r.write) {
        const double root = sqrt(1.0 - rsq);
        r.a0 = (2.0 * x) * root;
        r.a1 = (2.0 * y) * root;
        r.a2 = 1.0 - 2.0 * rsq;
      }
      done = true;
    }
  }
  if (!done && s == 0) atomicOr(&A.flags[1], 1u);  // 128 trials rejected
  return r;
}

// Producer warp: lay out tile `tl` in `B` from its counts (one per lane),
// start its copies, draw its axes.  Completes two arrivals on `full` (one
// with the byte count, one once the generic writes are done).
// The tile's layout from its counts (one per lane): computed before the
// producer waits for a free buffer.  Also queues a dense tile and zeroes the
// counts of a staged one (global memory only).
struct TilePlan {
  uint32_t k, excl, incl, total, sum;
  int nc;
  bool skip;
};

template <int MODE, int FIX>
__device__ __forceinline__ TilePlan plan_tile(const StepArgs& A, int64_t tl, int64_t ntiles,
                                              uint32_t cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t c0 = tl * TILE_CELLS(A);
  TilePlan P;
  P.nc = tl < ntiles ? (int)min((int64_t)TILE_CELLS(A), A.C - c0) : 0;
  P.k = min(cnt, A.cap);
  const uint32_t pad = (P.k + 3u) & ~3u;
  uint32_t incl = pad;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  P.incl = incl;
  P.excl = incl - pad;
  // a consumer warp pass holds at most kSlotsW padded slots
  const bool over = __any_sync(0xffffffffu, cnt > A.cap || pad > (uint32_t)kSlotsW);
  P.total = __shfl_sync(0xffffffffu, incl, 31);
  P.skip = tl >= ntiles || over || P.total > (uint32_t)kMaxPT;
  uint32_t sum = 2u * P.k * (uint32_t)sizeof(PRec);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  P.sum = sum;
  if (lane == 0 && P.skip && tl < ntiles) {  // queued for k_step_dense
    A.dense[atomicAdd(&A.flags[0], 1u)] = (uint32_t)tl;
    atomicOr(&A.dense_bits[tl >> 5], 1u << (tl & 31));
  }
  // consumed: the count_out of step k+1 (a dense tile's are read and zeroed
  // by k_step_dense)
  if (!P.skip && lane < P.nc) count_zero(&A.count_in[c0 + lane]);
  return P;
}

template <int MODE, int FIX>
__device__ __forceinline__ void prepare_tile(const StepArgs& A, TileBuf& B, uint64_t* full,
                                             int64_t tl, int64_t ntiles, uint32_t cnt,
                                             uint64_t pol, const TilePlan& P,
                                             const AxisReg* pre = nullptr) {
  const int lane = threadIdx.x & 31;
  const int64_t c0 = tl * TILE_CELLS(A);
  const int nc = P.nc;
  const uint32_t k = P.k, excl = P.excl, incl = P.incl;
  const bool skip = P.skip;
  if (lane < kTC) {
    B.cnt[lane] = cnt;
    B.off[lane + 1] = incl;
  }
  if (lane == 0) {
    B.off[0] = 0;
    B.skip = skip ? 1 : 0;
  }
  if (skip) {
    __syncwarp();
    if (lane == 0) {
      mbar_arrive_expect(full, 0u);
      mbar_arrive(full);
    }
    return;
  }
  const uint32_t bytes = k * (uint32_t)sizeof(PRec);
  if (lane == 0) {
    fence_proxy_async();  // the consumers' generic reads of B precede the async writes
    mbar_arrive_expect(full, P.sum);
  }
  __syncwarp();
  if (k) {
    const uint64_t src = (uint64_t)(c0 + lane) * A.cap;
    bulk_load(B.p + excl, A.in.p + src, bytes, full, pol);
    bulk_load(B.v + excl, A.in.v + src, bytes, full, pol);
  }
#if MPCD_PREFETCH_COUNTS
  // The tile's particles claim slots in next-step cells within one cell of
  // their own: pull those count lines into L2 now, a tile ahead of the
  // claims (9 (x, y) rows x the tile's z-range +- 1, two 128 B lines each).
  if (lane < 18 && nc > 0) {
    const int64_t zyx = c0 / A.L2;  // x * L1 + y of the tile (tiles do not cross z rows)
    const int z0 = (int)(c0 - zyx * A.L2);
    const int x = (int)(zyx / A.L1), y = (int)(zyx - (int64_t)x * A.L1);
    const int r = lane >> 1;
    int xn = x + r / 3 - 1, yn = y + r % 3 - 1;
    xn = xn < 0 ? xn + A.L0 : (xn >= A.L0 ? xn - A.L0 : xn);
    yn = yn < 0 ? yn + A.L1 : (yn >= A.L1 ? yn - A.L1 : yn);
    const int zn = (lane & 1) ? min(z0 + nc, A.L2 - 1) : max(z0 - 1, 0);
    const uint32_t* q = A.count_out + ((int64_t)xn * A.L1 + yn) * A.L2 + zn;
    asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(q));
  }
#endif
  // slot -> cell, bit 7 set on a padding slot
#if MPCD_CELLW
  // four slots per 32-bit store (a cell's padded run starts and ends on a
  // multiple of 4 slots)
  for (uint32_t j = excl; j < incl; j += 4) {
    const uint32_t real = k - min(k, j - excl);  // real slots from j on
    const uint32_t pad = real >= 4u ? 0u : (0x80808080u << (8u * real));
    *reinterpret_cast<uint32_t*>(B.cell + j) = ((uint32_t)lane * 0x01010101u) | pad;
  }
#else
  for (uint32_t j = excl; j < incl; ++j) B.cell[j] = (uint8_t)(lane | (j - excl < k ? 0 : kPadBit));
#endif
  // rotation axes (collision.py:217-250), keyed by the global cell id
#ifdef MPCD_ABL_NOAXIS  // timing ablation only (wrong results): a fixed axis
  if (lane < kTC) {
    double* ax = B.ax + lane * 4;
    ax[0] = 0.0; ax[1] = 0.6; ax[2] = 0.8;
  }
  if (0)
#endif
  if (pre) {  // drawn before the buffer was free (draw_axes_early)
    if (pre->write) {
      double* ax = B.ax + (lane >> 1) * 4;
      ax[0] = pre->a0;
      ax[1] = pre->a1;
      ax[2] = pre->a2;
    }
  } else
#if MPCD_AXPAIR
  if (A.prng == kSplitmix) {
    // two lanes per cell draw Marsaglia trials 2i and 2i + 1 at once (the
    // counter generator needs no sequential state); the first accepted
    // trial in trial order wins, exactly as the one-lane loop.  16 cells
    // per round of the warp.
   for (int cg = 0; cg < TILE_CELLS(A); cg += 16) {
    const int cell = cg + (lane >> 1), s = lane & 1;
    const uint32_t ccnt = __shfl_sync(0xffffffffu, cnt, cell & 31);
    bool done = !(cell < TILE_CELLS(A) && ccnt > 0u);
    const uint64_t key = done ? 0ull : key_from_prefix(A.axis_prefix, global_cell_id<MODE>(A, c0 + cell));
    double* ax = B.ax + cell * 4;
    if (s == 0 && cell < TILE_CELLS(A)) ax[0] = ax[1] = ax[2] = 0.0;
    __syncwarp();  // the zeros precede a partner lane's axis
    for (int i = 0; i < kMaxAxisTrials / 2; ++i) {
      if (!__any_sync(0xffffffffu, !done)) break;
      double x = 0.0, y = 0.0, rsq = 1.0;
      if (!done) {
        const uint64_t t = 2ull * (uint64_t)(2 * i + s);
        x = 2.0 * uniform_at(key, t) - 1.0;
        y = 2.0 * uniform_at(key, t + 1ull) - 1.0;
        rsq = x * x + y * y;
      }
      const unsigned acc = __ballot_sync(0xffffffffu, !done && rsq < 1.0);
      const unsigned pair = (acc >> (lane & ~1)) & 3u;
      if (!done && pair) {
        if (s == ((pair & 1u) ? 0 : 1)) {  // the earlier accepted trial of the pair
          const double root = sqrt(1.0 - rsq);
          ax[0] = (2.0 * x) * root;
          ax[1] = (2.0 * y) * root;
          ax[2] = 1.0 - 2.0 * rsq;
        }
        done = true;
      }
    }
    if (!done && s == 0) atomicOr(&A.flags[1], 1u);  // 128 trials rejected
   }
  } else
#endif
  if (lane < kTC) {
    double* ax = B.ax + lane * 4;
    ax[0] = ax[1] = ax[2] = 0.0;
    if (cnt > 0u && !rotation_axis_pre(A.prng, A.axis_prefix, global_cell_id<MODE>(A, c0 + lane), ax))
      atomicOr(&A.flags[1], 1u);
  }
  __syncwarp();
  if (lane == 0) mbar_arrive(full);  // release: layout, table and axes written
}


// One consumer warp's cells of one tile: every phase, R slot rows per lane.
template <int R, bool UNIT, bool UMASS, bool DRIFT, bool COM, int MODE, int VS, class Smem>
__device__ __forceinline__ void consume_cells(const StepArgs& A, Smem& S, TileBuf& T,
                                              WarpScratch& W, int64_t c0, int cw0,
                                              int ncw, int j0, int j1, double* acc,
                                              uint32_t& ncoll, uint64_t* rel = nullptr) {
  constexpr bool BYID = MODE == kById;
  // Rank order (MPCD_RANKORD): phase 4 visits each cell's particles in rank
  // order, so a lane's post-collision sums are its own rank positions -- the
  // conservation sums come from registers, with no post rows staged and read
  // back (the exchange mode keeps the slot order: it parks leavers in W.id).
  constexpr bool RO = MPCD_RANKORD && MODE != kMulti;
  // MPCD_SOA: the staging as four columns of stride VS (VS = 4 mod 16 for
  // 16-cell tiles: a moment lane group's 16 reads hit 16 bank pairs); the
  // unit-mass pre-collision mass column is not staged (its reduceat is k)
  // (columns measured 0.5 % faster for the whole box and 1.5 % slower for
  // the fused kernel: the fused kernel keeps the rows)
  constexpr bool SOA = MPCD_SOA && MODE != kFused;
  static_assert(4 * VS <= (kSlotsW + kCW) * 4 && VS >= kSlotsW + 4,
                "four staging columns of VS rows fit W.val and hold a pass's skewed rows");
  auto stage4 = [&](int row, double a, double b, double c, double d) {
    if (SOA) {
      W.val[row] = a; W.val[VS + row] = b; W.val[2 * VS + row] = c; W.val[3 * VS + row] = d;
    } else {
      sts_row32w(W.val, row, make_double2(a, b), make_double2(c, d));
    }
  };
  auto stage_moment = [&](int row0, int comp, int k) -> double {
    if (SOA) {  // k <= kSlotsW < 130: one pairwise leaf, immediate offsets
      const double* t = W.val + comp * VS + row0;
      if (k <= 0) return 0.0;
      if (k == 1) return t[0];
      return t[0] + pw_leaf<1>(t + 1, k - 1);
    }
    return reduceat_wcol(W.val, row0, comp, k);
  };
  const int lane = threadIdx.x & 31;
#ifdef MPCD_TIMING
  long long probe_t_ = 0;
#endif
  MPCD_PROBE(0);

  // phase 1: ids in slot order (sentinel in the padding), warp-local rows
  int lq[R];  // cell of the row inside the warp (0..3)
  bool real[R];
  uint32_t myid[R];  // the row's id (kept: phase 2 ranks it)
  const uint32_t pad_id = A.ids31 ? kSentinel31 : kSentinel;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int jl = lane + 32 * r, j = j0 + jl;
    real[r] = false;
    lq[r] = 0;
    myid[r] = pad_id;
    if (j < j1) {
      const int cj = T.cell[j];
      lq[r] = (cj & ~kPadBit) - cw0;
      real[r] = !(cj & kPadBit);
      if (real[r]) myid[r] = T.p[j].id;
      W.id[jl] = myid[r];
    }
  }
  __syncwarp();
  MPCD_PROBE(1);

  // phase 2: rank by id inside the cell, 4-wide over the padded segment;
  // stage (m v, m) in rank order -- the reference permutation is the stable
  // argsort over id order (collision.py:98)
  int row[R];  // skewed staging row of the particle
#pragma unroll
  for (int r = 0; r < R; ++r) {
    row[r] = 0;
    // MPCD_P2FLAT: every lane of a row the pass reaches runs the ranking
    // (warp-uniform test; a padding lane ranks the sentinel, k, and stores
    // nothing), so the phase has no divergent region
    if (MPCD_P2FLAT ? j0 + 32 * r < j1 : real[r]) {
      const int jl = lane + 32 * r;
      const int q = lq[r];
      const int lo = (int)T.off[cw0 + q] - j0, hi = (int)T.off[cw0 + q + 1] - j0;
      const uint32_t me = myid[r];
      uint32_t rank = 0;
#ifdef MPCD_ABL_NORANK  // timing ablation only (wrong results): slot order
      rank = (uint32_t)(jl - lo);
      if (0)
#endif
      if (A.ids31) {
        // a real row's cell has at least one group of four: do-while over a
        // pointer (no index arithmetic or entry test per group)
        const uint4* q = reinterpret_cast<const uint4*>(W.id + lo);
        const uint4* const qe = reinterpret_cast<const uint4*>(W.id + hi);
#if MPCD_RANKU
        // the first MPCD_RANKU groups unrolled, loads issued together; groups
        // past the cell read neighbouring scratch and are masked out
        const int ng = (hi - lo) >> 2;
#pragma unroll
        for (int g = 0; g < MPCD_RANKU; ++g) {
          const uint4 w = q[g];
          const uint32_t c = ((w.x - me) >> 31) + ((w.y - me) >> 31) + ((w.z - me) >> 31) +
                             ((w.w - me) >> 31);
          rank += g < ng ? c : 0u;
        }
        q += MPCD_RANKU;
        if (__builtin_expect(ng > MPCD_RANKU, 0))
#endif
#pragma unroll 1
        do {
          const uint4 w = *q++;
          // both below 2^31: w < me is the sign bit of w - me
          rank += ((w.x - me) >> 31) + ((w.y - me) >> 31) + ((w.z - me) >> 31) +
                  ((w.w - me) >> 31);
        } while (q < qe);
      } else {
#pragma unroll 1
        for (int s = lo; s < hi; s += 4) {
          const uint4 w = *reinterpret_cast<const uint4*>(W.id + s);
          rank += (w.x < me) + (w.y < me) + (w.z < me) + (w.w < me);
        }
      }
      row[r] = lo + (int)rank + q;
      double2 v01, v23;  // vx vy | vz m
      lds_row32t(T.v, j0 + jl, v01, v23);
      const double m = UMASS ? A.m0 : v23.y;
      if (!MPCD_P2FLAT || real[r]) {
        if (UMASS && A.m0 == 1.0) {  // unit masses: m v == v exactly, no multiplies
          if (SOA) {  // the mass column's reduceat is k (phase 3)
            W.val[row[r]] = v01.x; W.val[VS + row[r]] = v01.y; W.val[2 * VS + row[r]] = v23.x;
          } else {
            stage4(row[r], v01.x, v01.y, v23.x, 1.0);
          }
        } else {
          stage4(row[r], m * v01.x, m * v01.y, m * v23.x, m);
        }
      }
    }
  }
  __syncwarp();
  if constexpr (RO) {
    // the rank order's slot map: staging row -> slot of the pass (the ids in
    // W.id are no longer read; phase 4 visits the particles in rank order)
    uint8_t* map = reinterpret_cast<uint8_t*>(W.id);
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (real[r]) map[row[r]] = (uint8_t)(lane + 32 * r);
  }
  MPCD_PROBE(2);

  // phase 3: per-cell moments, numpy reduceat association (collision.py:190-206);
  // four lanes per cell, com = p / m (collision.py:209-214) from the group's
  // mass lane by shuffle
  {
    const int q = lane >> 2, comp = lane & 3;
    const bool mine = lane < 4 * kCW && q < ncw;
    double mom = 0.0;
    if (mine) {
      const int lc = cw0 + q;
      mom = stage_moment((int)T.off[lc] - j0 + q, comp, (int)T.cnt[lc]);
      // unit masses, SoA: k ones sum to k exactly in any association
      if (SOA && UMASS && comp == 3 && A.m0 == 1.0) mom = (double)T.cnt[lc];
    }
    const double mass = __shfl_sync(0xffffffffu, mom, lane | 3);
    if (mine) {
      W.mom[lane] = mom;
      const double c = (comp < 3) ? ((mass > 0.0) ? mom / mass : 0.0)
                                  : (double)T.cnt[cw0 + q];
      if (comp < 3) W.com[q * 4 + comp] = c;
      else {
        acc[4] += mass;
        ncoll += T.cnt[cw0 + q];  // particles collided
      }
      if (COM) A.com_cap[(c0 + cw0 + q) * 4 + comp] = c;
    }
  }
  __syncwarp();
  MPCD_PROBE(3);

  // phase 4: rotate (collision.py:289-306), stream + wrap (particles.py:62-67),
  // next-step cell; claim every slot, then store; stage post-collision rows
  double o[R][6];
  uint32_t key[R];
  double mm[R];
  uint32_t pid[R];
  bool stay[R];  // decomposed: the next cell is this domain's
  int dest[R];
  unsigned leavers = 0u;  // decomposed: bit r, row r's particle goes to another domain
  unsigned grp[R];
  uint32_t base[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    key[r] = 0u;
    stay[r] = real[r];
    dest[r] = 0;
#if MPCD_BRANCHLESS4
    // padding lanes compute on a real slot of the pass (slot j0) and store
    // nothing: no divergent region, so the rows' chains can interleave
    {
      // rank order: the slot of this rank position's particle (slot map)
      const int j = !real[r] ? j0
                    : RO ? j0 + (int)reinterpret_cast<const uint8_t*>(W.id)[lane + 32 * r + lq[r]]
                         : j0 + lane + 32 * r;
#else
    if (real[r]) {
      const int j = j0 + lane + 32 * r;
#endif
      double2 p01, p23, v01, v23;  // x y | z id, vx vy | vz m
      lds_row32t(T.p, j, p01, p23);
      lds_row32t(T.v, j, v01, v23);
      double2 c01, c2, a01, a2;
      lds_row32(W.com + lq[r] * 4, 0, c01, c2);
      lds_row32(T.ax + (cw0 + lq[r]) * 4, 0, a01, a2);
      const double cx[3] = {c01.x, c01.y, c2.x}, ax[3] = {a01.x, a01.y, a2.x};
      double v[3] = {v01.x, v01.y, v23.x}, w[3];
      rotate(v, cx, ax, A.cs, A.sn, w);
      if (MPCD_ONEBRANCH) {
        o[r][0] = p01.x + w[0] * A.dt;
        o[r][1] = p01.y + w[1] * A.dt;
        o[r][2] = p23.x + w[2] * A.dt;
        wrap3(o[r][0], o[r][1], o[r][2], A.box0, A.box1, A.box2);
      } else {
        o[r][0] = wrap_fast(p01.x + w[0] * A.dt, A.box0);
        o[r][1] = wrap_fast(p01.y + w[1] * A.dt, A.box1);
        o[r][2] = wrap_fast(p23.x + w[2] * A.dt, A.box2);
      }
      o[r][3] = w[0]; o[r][4] = w[1]; o[r][5] = w[2];
      pid[r] = bits_id(p23.y);
      mm[r] = UMASS ? A.m0 : v23.y;
      if (decomposed(MODE))
        stay[r] = next_cell_multi<UNIT>(A, o[r][0], o[r][1], o[r][2], key[r], dest[r]) && real[r];
      else
        key[r] = BYID ? pid[r] : next_cell<UNIT>(A, o[r][0], o[r][1], o[r][2]);
#if MPCD_EARLYCLAIM && MPCD_BRANCHLESS4
      // claim as soon as the key is known: the atomic's round trip overlaps
      // the staging below and the next row's whole chain
      grp[r] = 0u;
      base[r] = 0u;
      if constexpr (MODE == kFused) {
        // local or remote, one system-scope claim per particle: the
        // owner's next-step count, picked with a select
        if (MPCD_FUSED_OOL) {  // leavers claim in fused_put, out of line
          if (stay[r]) base[r] = count_claim<true>(A.count_out + key[r], 1u);
        } else if (real[r]) {
          uint32_t* cnt = A.count_out;
          if (__builtin_expect(!stay[r], 0)) cnt = S.peer.count[dest[r]];
          base[r] = count_claim<true>(cnt + key[r], 1u);
        }
      } else if (!BYID && j0 + 32 * r < j1) {
        claim_slot<false>(A, stay[r], key[r], grp[r], base[r]);
      }
#endif
      const double m = mm[r];
      const double ke = (w[0] * w[0] + w[1] * w[1]) + w[2] * w[2];  // diagnostics only
      if (RO) {
        // this lane's rank position: phase 5's sums straight from registers
        // (same values, same per-lane order); post rows only for the drift
        if (real[r]) {
          const bool unit = UMASS && A.m0 == 1.0;
          const double s0 = unit ? w[0] : m * w[0], s1 = unit ? w[1] : m * w[1];
          const double s2 = unit ? w[2] : m * w[2], s3 = unit ? ke : m * ke;
          acc[0] += s0; acc[1] += s1; acc[2] += s2; acc[3] += s3;
          if (DRIFT)
            stage4(lane + 32 * r + lq[r], s0, s1, s2, s3);
        }
      } else if (real[r]) {
        if (UMASS && A.m0 == 1.0)
          stage4(row[r], w[0], w[1], w[2], ke);
        else
          stage4(row[r], m * w[0], m * w[1], m * w[2], m * ke);
      }
      if (MODE == kMulti && real[r] && !stay[r]) {
        // a leaver: park its record in its own tile slot (dest in the pad
        // word) and its owner-local cell in W.id; flushed after the pass, so
        // the hot loop carries no copy of the sending code
        sts_row32(T.p, j, make_double2(o[r][0], o[r][1]),
                  make_double2(o[r][2], __longlong_as_double(
                                            (long long)(((uint64_t)(uint32_t)dest[r] << 32) |
                                                        pid[r]))));
        sts_row32(T.v, j, make_double2(o[r][3], o[r][4]), make_double2(o[r][5], m));
        W.id[lane + 32 * r] = key[r];
        leavers |= 1u << r;
      }
    }
  }
  if (BYID) {
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (real[r])
        store_rec(A.out, pid[r], o[r][0], o[r][1], o[r][2], pid[r], o[r][3], o[r][4], o[r][5],
                  mm[r]);
  } else if (!(MPCD_EARLYCLAIM && MPCD_BRANCHLESS4)) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      grp[r] = 0u;
      base[r] = 0u;
      if (j0 + 32 * r < j1)  // warp-uniform: every lane takes part in the ballot
        claim_slot<MODE == kFused>(A, stay[r], key[r], grp[r], base[r]);
    }
  }
  __syncwarp();
  // the tile's last pass: nothing below reads the tile buffer (stores take
  // registers), so the producer may refill it while the claims return
  if (kEarlyRel<DRIFT, MODE> && rel != nullptr && lane == 0) mbar_arrive(rel);
  MPCD_PROBE(4);

  // phase 5: conservation sums over the staged post rows, each lane its
  // rank positions (fixed: deterministic) -- while the slot claims are in
  // flight.  Position jl of cell q holds rank jl - lo_q, a real particle
  // exactly when real[r].
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if (!RO && real[r]) {
      const int jl = lane + 32 * r;
      double2 a, c;
      if (SOA) {
        const int p = jl + lq[r];
        a = make_double2(W.val[p], W.val[VS + p]);
        c = make_double2(W.val[2 * VS + p], W.val[3 * VS + p]);
      } else {
        lds_row32w(W.val, jl + lq[r], a, c);
      }
      acc[0] += a.x; acc[1] += a.y; acc[2] += c.x; acc[3] += c.y;
    }
  }
  MPCD_PROBE(5);
#ifdef MPCD_TIMING
  {  // wait for the claims alone
    uint32_t dep = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) dep += base[r];
    if (dep == 0xFFFFFFFFu) acc[0] += 1.0;
  }
  MPCD_PROBE(6);
#endif
  if constexpr (MODE == kFused) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (stay[r]) {
        finish_slot<true>(A, key[r], 0u, base[r], o[r], pid[r], mm[r]);
      } else if (__builtin_expect(real[r], 0)) {  // a leaver: into its owner's cell, over peer memory
        acc[6] += 1.0;
        if (MPCD_FUSED_OOL) {
          fused_put(A.peers, A.out_set, A.cap, A.ovf_cap, dest[r], key[r], o[r][0], o[r][1],
                    o[r][2], pid[r], o[r][3], o[r][4], o[r][5], mm[r]);
        } else if (__builtin_expect(base[r] < A.cap, 1)) {
          const Recs dst{S.peer.p[dest[r]], S.peer.v[dest[r]]};
          store_rec(dst, (uint64_t)key[r] * A.cap + base[r], o[r][0], o[r][1], o[r][2], pid[r],
                    o[r][3], o[r][4], o[r][5], mm[r]);
        } else {
          fused_overflow(A.peers, A.out_set, A.ovf_cap, dest[r], key[r], o[r][0], o[r][1],
                         o[r][2], pid[r], o[r][3], o[r][4], o[r][5], mm[r]);
        }
      }
    }
  } else if (!BYID) {
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (stay[r]) finish_slot<false>(A, key[r], grp[r], base[r], o[r], pid[r], mm[r]);
  }
  if (MODE == kMulti && __any_sync(0xffffffffu, leavers != 0u)) {
    // the pass's leavers, from their parked slots: one copy of the sending
    // code, run only by passes that have any
#pragma unroll 1
    for (int r = 0; r < R; ++r) {
      const bool go = (leavers >> r) & 1u;
      double q[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0}, m = 0.0;
      uint32_t id = 0u, k = 0u;
      int to = 0;
      if (go) {
        double2 p01, p23, v01, v23;
        lds_row32(T.p, j0 + lane + 32 * r, p01, p23);
        lds_row32(T.v, j0 + lane + 32 * r, v01, v23);
        const uint64_t bits = (uint64_t)__double_as_longlong(p23.y);
        q[0] = p01.x; q[1] = p01.y; q[2] = p23.x; q[3] = v01.x; q[4] = v01.y; q[5] = v23.x;
        m = v23.y;
        id = (uint32_t)bits;
        to = (int)(bits >> 32);
        k = W.id[lane + 32 * r];
      }
      send_foreign<MODE == kFused>(A, go, to, k, q, id, m, acc[6]);
    }
    fence_proxy_async();  // the parked slots' generic writes precede the next TMA fill
  }
  if (DRIFT) {
    const int q = lane >> 2, comp = lane & 3;
    double post = 0.0;
    if (lane < 4 * kCW && q < ncw) {
      const int lc = cw0 + q;
      post = stage_moment((int)T.off[lc] - j0 + q, comp, (int)T.cnt[lc]);
    }
    double* P = S.post + cw0 * 4;  // this pass's cells only
    if (lane < 4 * ncw) P[lane] = post;
    __syncwarp();
    double worst = 0.0;
    if (lane < ncw && W.mom[lane * 4 + 3] > 0.0)
      worst = cell_drift(W.mom + lane * 4, P + lane * 4);
    for (int off = 16; off > 0; off >>= 1)
      worst = fmax(worst, __shfl_xor_sync(0xffffffffu, worst, off));
    if (lane == 0 && worst > 0.0) atomic_max_pos_double(A.drift_bits, worst);
  }
  MPCD_PROBE(7);
}

template <bool UNIT, bool UMASS, bool DRIFT, bool COM, int MODE, int FIX>
__global__ void __launch_bounds__(kNTW, MPCD_MINB) k_step(const StepArgs A, int64_t ntiles) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  using Smem = StepSmem<DRIFT, MODE == kFused>;
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t G = gridDim.x;
#ifdef MPCD_TIMING
  if (t < kNCW * 10) (&S.tim[0][0])[t] = 0ull;
#endif
  if (t == 0) {
    for (int b = 0; b < kStages; ++b) {
      mbar_init(&S.full[b], 2);
      mbar_init(&S.empty[b], kNCW);
    }
    fence_mbar_init();
  }
  if constexpr (MODE == kFused) {
    if (t < A.n_ranks) {
      const PeerBufs& P = A.peers[t];
      S.peer.count[t] = P.count[A.out_set];
      S.peer.p[t] = P.reg[A.out_set].p;
      S.peer.v[t] = P.reg[A.out_set].v;
    }
  }
  __syncthreads();

  if (warp == kNCW) {  // -------------------------------------- producer
    // the records' TMA loads at evict-normal priority; measured slower:
    // evict-first by 1.2 %, evict-last by 0.9 %, evict-first at fraction 0.5
    // by 0.1 %; evict-unchanged is the same
    const uint64_t pol = policy_evict_normal();
    int64_t tile = blockIdx.x;
    uint32_t cnt = tile_count<FIX>(A, tile, ntiles);
    // buffer b of round `ph` (the parity of i / kStages), kept incrementally:
    // no 64-bit division per tile
    int b = 0;
    uint32_t ph = 0u;
#ifdef MPCD_TIMING
    unsigned long long pw = 0ull, pp = 0ull;
#endif
    for (int64_t i = 0; tile < ntiles; ++i, tile += G) {
      const uint32_t cnt_next = tile_count<FIX>(A, tile + G, ntiles);  // in flight meanwhile
#ifdef MPCD_TIMING
      const long long q0 = clock64();
#endif
      // everything that does not touch the buffer happens before waiting for it
      const TilePlan plan = plan_tile<MODE, FIX>(A, tile, ntiles, cnt);
      const bool early = MPCD_EARLYAX && A.prng == kSplitmix && TILE_CELLS(A) <= 16 && !plan.skip;
      AxisReg ar{0.0, 0.0, 0.0, false};
      if (early) ar = draw_axes_early<MODE, FIX>(A, tile, ntiles, cnt);
      if (i >= kStages) mbar_wait(&S.empty[b], ph ^ 1u);
#ifdef MPCD_TIMING
      const long long q1 = clock64();
#endif
      prepare_tile<MODE, FIX>(A, S.buf[b], &S.full[b], tile, ntiles, cnt, pol, plan,
                              early ? &ar : nullptr);
#ifdef MPCD_TIMING
      pw += (unsigned long long)(q1 - q0);
      pp += (unsigned long long)(clock64() - q1);
#endif
      cnt = cnt_next;
      if (++b == kStages) {
        b = 0;
        ph ^= 1u;
      }
    }
#ifdef MPCD_TIMING
    if (lane == 0) {
      atomicAdd(&g_prod_cycles[0], pw);
      atomicAdd(&g_prod_cycles[1], pp);
    }
#endif
    return;
  }

  // ------------------------------------------------------------ consumers
  WarpScratch& W = S.w[warp];
  const int cw0 = warp * WARP_CELLS(A);  // this warp's first cell of every tile
  // px py pz sum(m v^2) mass, particles collided, particles sent to other ranks
  double acc[kDiagCols] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  uint32_t ncoll = 0u;  // particles collided by this thread's cell lanes (acc[5])
  int64_t tile = blockIdx.x;
  int b = 0;
  uint32_t ph = 0u;
  for (int64_t i = 0; tile < ntiles; ++i, tile += G, b = (b + 1 == kStages) ? 0 : b + 1,
               ph ^= (b == 0) ? 1u : 0u) {
    TileBuf& T = S.buf[b];
#ifdef MPCD_TIMING
    const long long tw0 = clock64();
#endif
    mbar_wait(&S.full[b], ph);
#ifdef MPCD_TIMING
    if (lane == 0) S.tim[warp][8] += (unsigned long long)(clock64() - tw0);
    if (lane == 0) S.tim[warp][9] += 1ull;
#endif
    const int64_t c0 = tile * TILE_CELLS(A);
    int ncw = WARP_CELLS(A);
    if (c0 + TILE_CELLS(A) > A.C)  // the box's last, partial tile
      ncw = (int)max((int64_t)0, min((int64_t)ncw, A.C - c0 - cw0));
    if (T.skip) ncw = 0;
    if (ncw == 0) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.empty[b]);
      continue;
    }
    // The warp's cells in passes of at most kSlotsW padded slots: one pass
    // almost always, two for the fullest quarter tiles (a cell never holds
    // more than kSlotsW: the producer sends such tiles to k_step_dense).
    const int gend = cw0 + ncw;
    const bool one = T.off[gend] - T.off[cw0] <= (uint32_t)kSlotsW;
    for (int g0 = cw0; g0 < gend;) {
      int g1 = gend;
      if (!one) {
        g1 = g0 + 1;
        while (g1 < gend && T.off[g1 + 1] - T.off[g0] <= (uint32_t)kSlotsW) ++g1;
      }
      const int t1 = (int)T.off[g1];
      consume_cells<kRowsW, UNIT, UMASS, DRIFT, COM, MODE, (FIX == 16 ? 68 : 72)>(
          A, S, T, W, c0, g0, g1 - g0, (int)T.off[g0], t1, acc, ncoll,
          g1 == gend ? &S.empty[b] : nullptr);
      __syncwarp();  // W is rewritten by the next pass
      g0 = g1;
    }
    // the tile buffer is free for the producer (released early, see consume_cells)
    if (!kEarlyRel<DRIFT, MODE> && lane == 0) mbar_arrive(&S.empty[b]);
  }
#ifdef MPCD_TIMING
  if (lane < 10) atomicAdd(&g_phase_cycles[lane], S.tim[warp][lane]);
#endif
  // fused migration: this thread's stores into peers' regions become visible
  // system-wide before the step fence (the all-reduce that follows the step)
  if (A.peers) __threadfence_system();
  // CTA partials: fixed-order block reduction of the per-thread sums
  acc[5] = (double)ncoll;
#pragma unroll
  for (int q = 0; q < kDiagCols; ++q)
    for (int off = 16; off > 0; off >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], off);
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < kDiagCols; ++q) S.red[warp * kDiagCols + q] = acc[q];
  consumer_sync();
  if (t < kDiagCols) {
    double s = 0.0;
    for (int w = 0; w < kNCW; ++w) s += S.red[w * kDiagCols + t];
    A.partials[(int64_t)blockIdx.x * 8 + t] = s;
  }
}

// ----------------------------------------------------- dense-tile kernel --
// Tiles that k_step cannot stage: a cell above `cap` (its extra particles sit
// in the overflow list), a cell of more than kSlotsW padded rows, or more than
// kMaxPT padded rows in the tile.  These are rare at the density a context's
// tile size was chosen for (mpcd_ctx_create); this is the general path for
// clusters and for densities above ~40 particles per cell.  Work is O(n)
// apart from the in-cell ranking (O(k^2 / threads) per cell of k particles):
//
//   k_dense_prep   per queued tile, reserve each overflowing cell's bucket in
//                  ovf_sorted (cell_aux[c] = its first position);
//   k_ovf_bucket   each overflow entry into its cell's bucket;
//   k_step_dense   one CTA per queued tile: gather the tile's particles (region
//                  slots + bucket) into shared memory (or, above np_smem, into
//                  HBM staging from a bounded allocator), rank by id, the same
//                  phases as k_step, one partials row per tile.
//
// Every overflow entry belongs to a queued tile: a cell above cap makes its
// tile dense.  Results never depend on the (arrival) order of the queue: the
// diagnostics rows are per tile and reduced in tile order (k_diag_partial).
#ifndef MPCD_STEP_VARIANTS_ONLY
__global__ void __launch_bounds__(256) k_dense_prep(const StepArgs A) {
  const uint32_t n_dense = *(volatile uint32_t*)&A.flags[0];
  const uint32_t n_ovf = min(*(volatile uint32_t*)A.ovf_n_in, A.ovf_cap);
  if (n_ovf == 0) return;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < n_dense;
       e += gridDim.x * blockDim.x) {
    const int64_t c0 = (int64_t)A.dense[e] * A.tc;
    const int nc = (int)min((int64_t)A.tc, A.C - c0);
    uint32_t tot = 0;
    for (int lc = 0; lc < nc; ++lc) {
      const uint32_t cnt = A.count_in[c0 + lc];
      tot += cnt > A.cap ? cnt - A.cap : 0u;
    }
    if (!tot) continue;
    uint32_t base = atomicAdd(&A.flags[8], tot);
    for (int lc = 0; lc < nc; ++lc) {
      const uint32_t cnt = A.count_in[c0 + lc];
      if (cnt > A.cap) {
        A.cell_aux[c0 + lc] = base;
        base += cnt - A.cap;
      }
    }
  }
}

__global__ void __launch_bounds__(256) k_ovf_bucket(const StepArgs A) {
  if (*(volatile uint32_t*)&A.flags[0] == 0u) return;
  const uint32_t n_ovf = min(*(volatile uint32_t*)A.ovf_n_in, A.ovf_cap);
  for (uint32_t o = blockIdx.x * blockDim.x + threadIdx.x; o < n_ovf; o += gridDim.x * blockDim.x) {
    const uint32_t c = A.ovf_cell_in[o];
    if ((int64_t)c >= A.C) continue;
    const uint32_t pos = atomicAdd(&A.cell_aux[c], 1u);
    if (pos < A.ovf_cap) A.ovf_sorted[pos] = o;
  }
}

#endif  // MPCD_STEP_VARIANTS_ONLY

// Largest cell occupancy the dense-tile kernel ranks (k^2 / 256 compares per
// CTA: ~16 M at the limit); a step that meets a bigger cell fails with
// MPCD_ERR_CAPACITY.  65536 particles in one cell is 6500x the mean density
// of the benchmark configurations.
constexpr uint32_t kDenseMaxCell = 65536;

// Bytes of dynamic shared memory k_step_dense stages `np` particles in.
__host__ __device__ constexpr size_t dense_smem_bytes(uint32_t np) {
  return (size_t)np * (4 * sizeof(double) + 2 * sizeof(uint32_t));
}

template <bool UNIT, bool UMASS, bool DRIFT, bool COM, int MODE>
__global__ void __launch_bounds__(kNT) k_step_dense(const StepArgs A) {
  extern __shared__ __align__(16) unsigned char dsm[];
  double* const sm_val = reinterpret_cast<double*>(dsm);
  uint32_t* const sm_id = reinterpret_cast<uint32_t*>(sm_val + 4 * (size_t)A.np_smem);
  uint32_t* const sm_src = sm_id + A.np_smem;
  __shared__ uint32_t s_cnt[kTC];
  __shared__ uint32_t s_off[kTC + 1];
  __shared__ uint32_t s_nreg[kTC];
  __shared__ uint32_t s_obeg[kTC];
  __shared__ uint32_t s_base;
  __shared__ int s_mode;  // 0 shared-memory staging, 1 HBM staging, -1 no room
  __shared__ double s_mom[kTC * 4];
  __shared__ double s_post[kTC * 4];
  __shared__ double s_cx[kTC * 6];
  __shared__ double s_mig[kNT / 32];
  const int t = threadIdx.x;
  const uint32_t n_dense = *(volatile uint32_t*)&A.flags[0];
  const uint32_t n_ovf = min(*(volatile uint32_t*)A.ovf_n_in, A.ovf_cap);
  for (uint32_t e = blockIdx.x; e < n_dense; e += gridDim.x) {
    const int64_t tile = A.dense[e];
    const int64_t c0 = tile * A.tc;
    const int nc = (int)min((int64_t)A.tc, A.C - c0);
    __syncthreads();
    if (t == 0) {
      uint32_t acc = 0;
      for (int lc = 0; lc < kTC; ++lc) {
        const uint32_t cnt = lc < nc ? A.count_in[c0 + lc] : 0u;
        s_cnt[lc] = cnt;
        s_off[lc] = acc;
        s_nreg[lc] = min(cnt, A.cap);
        // bucket end (k_ovf_bucket advanced it) minus this cell's entries
        s_obeg[lc] = cnt > A.cap ? A.cell_aux[c0 + lc] - (cnt - A.cap) : 0u;
        acc += cnt;
      }
      s_off[kTC] = acc;
      s_mode = 0;
      s_base = 0;
      uint32_t biggest = 0;
      for (int lc = 0; lc < nc; ++lc) biggest = max(biggest, s_cnt[lc]);
      if (biggest > kDenseMaxCell) {
        // the in-cell ranking is O(k^2 / threads): refuse rather than stall
        s_mode = -1;
        atomicOr(&A.flags[10], 1u);
      } else if (acc > A.np_smem) {
        const uint32_t b = atomicAdd(A.scratch_n, acc);
        if ((uint64_t)b + acc <= (uint64_t)A.scratch_cap) {
          s_mode = 1;
          s_base = b;
        } else {
          s_mode = -1;
          atomicOr(&A.flags[9], 1u);  // MPCD_ERR_CAPACITY: the particles are lost
        }
      }
    }
    __syncthreads();
    const uint32_t np = s_off[kTC];
    if (s_mode < 0) {
      if (t < nc) A.count_in[c0 + t] = 0u;
      continue;
    }
    uint32_t* const g_id = s_mode ? A.scratch_id + s_base : sm_id;
    uint32_t* const g_src = s_mode ? A.scratch_src + s_base : sm_src;  // slot, or 0x80000000|entry
    double* const g_val = s_mode ? A.scratch_val + 4 * (uint64_t)s_base : sm_val;
    // gather: region slots, then the cell's overflow bucket
    for (int lc = 0; lc < nc; ++lc) {
      const uint32_t nreg = s_nreg[lc], nall = s_cnt[lc];
      for (uint32_t s = t; s < nall; s += kNT) {
        uint32_t id = kSentinel, src = 0x80000000u;
        if (s < nreg) {
          id = A.in.p[(uint64_t)(c0 + lc) * A.cap + s].id;
          src = s;
        } else {
          const uint32_t pos = s_obeg[lc] + (s - nreg);
          const uint32_t o = pos < A.ovf_cap ? A.ovf_sorted[pos] : 0xFFFFFFFFu;
          if (o < n_ovf) {  // (else: entries were dropped, flags[2] already set)
            id = A.ovf_in.p[o].id;
            src = 0x80000000u | o;
          }
        }
        g_id[s_off[lc] + s] = id;
        g_src[s_off[lc] + s] = src;
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
      return (s & 0x80000000u) ? A.ovf_in.p[min(s & 0x7FFFFFFFu, A.ovf_cap - 1u)]
                               : A.in.p[(uint64_t)(c0 + lc) * A.cap + s];
    };
    auto rec_v = [&](uint32_t j, int lc) -> const VRec& {
      const uint32_t s = g_src[j];
      return (s & 0x80000000u) ? A.ovf_in.v[min(s & 0x7FFFFFFFu, A.ovf_cap - 1u)]
                               : A.in.v[(uint64_t)(c0 + lc) * A.cap + s];
    };
    // rank by id inside the cell (ids are unique): the stable argsort order
    auto rank_of = [&](uint32_t j, int lc) {
      const uint32_t me = g_id[j];
      uint32_t rank = 0;
      for (uint32_t q = s_off[lc]; q < s_off[lc + 1]; ++q) rank += (g_id[q] < me) ? 1u : 0u;
      return s_off[lc] + rank;
    };
    // pre-collision (m v, m) rows in rank order
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
      if (s_cnt[t] > 0u && !rotation_axis_pre(A.prng, A.axis_prefix, global_cell_id<MODE>(A, c0 + t), cx + 3))
        atomicOr(&A.flags[1], 1u);
      if (COM) {
        double* g = A.com_cap + (c0 + t) * 4;
        g[0] = cx[0]; g[1] = cx[1]; g[2] = cx[2]; g[3] = (double)s_cnt[t];
      }
    }
    __syncthreads();
    // each rank-order row is rewritten with its post-collision row below;
    // the ranks come from the ids, which stay, so the loop is race-free
    double dmig = 0.0;
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
        g_val[4 * s] = m * w[0]; g_val[4 * s + 1] = m * w[1]; g_val[4 * s + 2] = m * w[2];
        g_val[4 * s + 3] = m * (((0.0 + w[0] * w[0]) + w[1] * w[1]) + w[2] * w[2]);
      }
      emit<UNIT, MODE>(A, active, nx, ny, nz, id, w, UMASS ? A.m0 : m, dmig);
    }
    __syncthreads();
    for (int task = t; task < nc * 4; task += kNT) {
      const int lc = task >> 2, comp = task & 3;
      s_post[task] = s_cnt[lc] ? reduceat(g_val + 4 * (uint64_t)s_off[lc] + comp, (int64_t)s_cnt[lc], 4) : 0.0;
    }
    for (int o = 16; o > 0; o >>= 1) dmig += __shfl_xor_sync(0xffffffffu, dmig, o);
    if ((t & 31) == 0) s_mig[t >> 5] = dmig;
    __syncthreads();
    // this tile's partials row: px py pz sum(m v^2) mass collided migrated
    if (t < kDiagCols) {
      double s = 0.0;
      if (t < 6) {
        for (int lc = 0; lc < nc; ++lc)
          s += (t < 4) ? s_post[lc * 4 + t] : (t == 4 ? s_mom[lc * 4 + 3] : (double)s_cnt[lc]);
      } else {
        for (int w = 0; w < kNT / 32; ++w) s += s_mig[w];
      }
      A.partials[(A.dense_row0 + tile) * 8 + t] = s;
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
  if (A.peers) __threadfence_system();
}

// ---------------------------------------------------- diagnostics reduce --
constexpr int kDiagBlocks = 592;

#ifndef MPCD_STEP_VARIANTS_ONLY
// Level 1 of the fixed-order diagnostics reduction: block b sums its share of
// k_step's per-CTA rows [0, main_rows) and then, when tiles went to the dense
// kernel, the rows of the queued tiles in its share of the tile range, in
// tile order (their queue bits are cleared on the way).
__global__ void __launch_bounds__(256) k_diag_partial(const double* partials, int64_t main_rows,
                                                     int64_t dense_row0, int64_t ntiles,
                                                     uint32_t* dense_bits, const uint32_t* flags,
                                                     double* level1) {
  __shared__ double s[kDiagCols][256];
  const int t = threadIdx.x;
  double acc[kDiagCols] = {0, 0, 0, 0, 0, 0, 0};
  {
    const int64_t per = (main_rows + gridDim.x - 1) / gridDim.x;
    const int64_t lo = blockIdx.x * per, hi = min(main_rows, lo + per);
    for (int64_t i = lo + t; i < hi; i += 256)
#pragma unroll
      for (int c = 0; c < kDiagCols; ++c) acc[c] += partials[i * 8 + c];
  }
  if (*(volatile const uint32_t*)&flags[0] != 0u) {
    const int64_t words = (ntiles + 31) / 32;
    const int64_t per = (words + gridDim.x - 1) / gridDim.x;
    const int64_t lo = blockIdx.x * per, hi = min(words, lo + per);
    for (int64_t w = lo + t; w < hi; w += 256) {
      uint32_t bits = dense_bits[w];
      if (!bits) continue;
      dense_bits[w] = 0u;
      while (bits) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1u;
        const double* row = partials + (dense_row0 + w * 32 + b) * 8;
#pragma unroll
        for (int c = 0; c < kDiagCols; ++c) acc[c] += row[c];
      }
    }
  }
#pragma unroll
  for (int c = 0; c < kDiagCols; ++c) s[c][t] = acc[c];
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (t < w)
#pragma unroll
      for (int c = 0; c < kDiagCols; ++c) s[c][t] += s[c][t + w];
    __syncthreads();
  }
  if (t < kDiagCols) level1[blockIdx.x * kDiagCols + t] = s[t][0];
}

// Final fixed-order sum (strided lanes, then a shuffle tree); also retires the
// step's transient counters.  out: px py pz energy mass drift n step migrated.
__global__ void __launch_bounds__(32) k_diag_finalize(const double* level1, int nblocks,
                                                     unsigned long long* drift_bits, double* out,
                                                     int64_t step, uint32_t* flags,
                                                     uint32_t* ovf_n_consumed,
                                                     uint32_t* scratch_n) {
  const int t = threadIdx.x;
  double col[kDiagCols];
#pragma unroll
  for (int c = 0; c < kDiagCols; ++c) {
    double s = 0.0;
    for (int b = t; b < nblocks; b += 32) s += level1[b * kDiagCols + c];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    col[c] = s;
  }
  if (t == 0) {
    out[0] = col[0];
    out[1] = col[1];
    out[2] = col[2];
    out[3] = 0.5 * col[3];
    out[4] = col[4];
    out[5] = __longlong_as_double((long long)*drift_bits);
    out[6] = col[5];
    out[7] = (double)step;
    out[8] = col[6];
    *drift_bits = 0ULL;
    flags[0] = 0u;         // dense-tile list consumed
    *ovf_n_consumed = 0u;  // this step's input overflow list consumed
    *scratch_n = 0u;
    flags[8] = 0u;  // overflow bucket allocator
  }
}

#endif  // MPCD_STEP_VARIANTS_ONLY

}  // namespace mpcd
