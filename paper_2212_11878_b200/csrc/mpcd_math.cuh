// mpcd_math.cuh -- host+device numerics of one SRD step, in the reference's
// exact IEEE-754 operation order.
//
// Every function here is __host__ __device__ so the library's host entry
// points (grid shift, key_state) and its kernels share one definition.  The
// translation units that include it MUST be compiled with -fmad=false
// (device) and -ffp-contract=off (host): the reference (numpy) never fuses
// a*b+c, so neither may we.  tests/test_build.py checks the SASS for DFMA.
#pragma once
#include <stdint.h>
#include <math.h>

#ifdef __CUDACC__
#define MPCD_HD __host__ __device__ __forceinline__
#else
#define MPCD_HD inline
#endif

namespace mpcd {

// rng.py:20-24
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t kMulA = 0xBF58476D1CE4E5B9ULL;
constexpr uint64_t kMulB = 0x94D049BB133111EBULL;
constexpr uint64_t kSeq = 0x2545F4914F6CDD1DULL;
constexpr double kInv53 = 1.0 / 9007199254740992.0;  // 2^-53
constexpr int kMaxAxisTrials = 128;                  // collision.py:22

enum Purpose : uint64_t { kShift = 0, kAxis = 1, kInit = 2 };  // rng.py:28-33
enum Prng : int { kSplitmix = 0, kMinstd = 1, kPcg32 = 2, kSfc64 = 3 };

// rng.py:50-54
MPCD_HD uint64_t mix64(uint64_t x) {
  x = (x ^ (x >> 30)) * kMulA;
  x = (x ^ (x >> 27)) * kMulB;
  return x ^ (x >> 31);
}

// rng.py:57-58, 67-77
MPCD_HD uint64_t key_state(uint64_t seed, uint64_t step, uint64_t purpose, uint64_t cell) {
  uint64_t s = mix64(seed * kSeq + kGolden);
  s = mix64(s ^ (step * kSeq + kGolden));
  s = mix64(s ^ (purpose * kSeq + kGolden));
  return mix64(s ^ (cell * kSeq + kGolden));
}

// rng.py:84-92: 53 high bits of one finalizer round, times 2^-53 (exact)
MPCD_HD double uniform_at(uint64_t state, uint64_t index) {
  return (double)(mix64(state ^ ((index + 1ULL) * kSeq)) >> 11) * kInv53;
}

// Key state after absorbing (seed, step, purpose): the last absorb
// (rng.py:76) is the only per-cell part, so kernels receive this prefix.
MPCD_HD uint64_t key_prefix(uint64_t seed, uint64_t step, uint64_t purpose) {
  uint64_t s = mix64(seed * kSeq + kGolden);
  s = mix64(s ^ (step * kSeq + kGolden));
  return mix64(s ^ (purpose * kSeq + kGolden));
}
MPCD_HD uint64_t key_from_prefix(uint64_t prefix, uint64_t cell) {
  return mix64(prefix ^ (cell * kSeq + kGolden));
}

// A keyed stream of doubles in [0,1), one type per generator (compile-time,
// so no other generator's code is ever predicated in).  KIND == kSplitmix is
// the reference's counter generator (draw j == uniform_at(key, j)); the
// sequential generators (not in the reference) are
// seeded from the same key and consumed in draw order, so draw j plays the
// role of counter j.
template <int KIND>
struct KStream {
  uint64_t s0, s1, s2, s3;

  MPCD_HD explicit KStream(uint64_t key) : s0(key), s1(0), s2(0), s3(0) {
    if (KIND == kMinstd) {
      s0 = 1ULL + key % 2147483646ULL;  // x0 in [1, m-1]
    } else if (KIND == kPcg32) {        // pcg32_srandom_r(key, 54)
      s0 = 0;
      s1 = (54ULL << 1) | 1ULL;
      pcg_next();
      s0 += key;
      pcg_next();
    } else if (KIND == kSfc64) {  // a = b = c = key, counter = 1, 12 discards
      s1 = key;
      s2 = key;
      s3 = 1;
      for (int i = 0; i < 12; ++i) sfc_next();
    }
  }
  // Park-Miller with Carta's reduction: p < 2^47, p mod (2^31-1) exactly
  MPCD_HD uint32_t minstd_next() {
    uint64_t p = s0 * 48271ULL;
    uint64_t r = (p & 0x7FFFFFFFULL) + (p >> 31);
    if (r >= 0x7FFFFFFFULL) r -= 0x7FFFFFFFULL;
    s0 = r;
    return (uint32_t)r;
  }
  MPCD_HD uint32_t pcg_next() {
    uint64_t old = s0;
    s0 = old * 6364136223846793005ULL + s1;
    uint32_t xs = (uint32_t)(((old >> 18) ^ old) >> 27);
    uint32_t rot = (uint32_t)(old >> 59);
    return (xs >> rot) | (xs << ((32u - rot) & 31u));
  }
  MPCD_HD uint64_t sfc_next() {
    uint64_t t = s0 + s1 + s3;
    s3 += 1;
    s0 = s1 ^ (s1 >> 11);
    s1 = s2 + (s2 << 3);
    s2 = ((s2 << 24) | (s2 >> 40)) + t;
    return t;
  }
  MPCD_HD double next() {
    if (KIND == kMinstd) {
      uint64_t hi = (uint64_t)(minstd_next() - 1u) >> 4;  // 27 bits
      uint64_t lo = (uint64_t)(minstd_next() - 1u) >> 5;  // 26 bits
      return (double)((hi << 26) | lo) * kInv53;
    } else if (KIND == kPcg32) {
      uint64_t hi = pcg_next() >> 5;
      uint64_t lo = pcg_next() >> 6;
      return (double)((hi << 26) | lo) * kInv53;
    } else if (KIND == kSfc64) {
      return (double)(sfc_next() >> 11) * kInv53;
    } else {
      return uniform_at(s0, s1++);
    }
  }
};

// Runtime-kind stream for host helpers and the stage API (not hot).
struct Stream {
  int kind;
  KStream<kSplitmix> a;
  KStream<kMinstd> b;
  KStream<kPcg32> c;
  KStream<kSfc64> d;
  MPCD_HD Stream(int k, uint64_t key)
      : kind(k),
        a(key),
        b(k == kMinstd ? key : 1ULL),
        c(k == kPcg32 ? key : 0ULL),
        d(k == kSfc64 ? key : 0ULL) {}
  MPCD_HD double next() {
    switch (kind) {
      case kMinstd: return b.next();
      case kPcg32: return c.next();
      case kSfc64: return d.next();
      default: return a.next();
    }
  }
};

// collision.py:32-36
MPCD_HD void grid_shift(int kind, uint64_t seed, uint64_t step, double a, double off[3]) {
  Stream g(kind, key_state(seed, step, kShift, 0));
  for (int d = 0; d < 3; ++d) off[d] = (g.next() - 0.5) * a;
}

// collision.py:217-250 for one cell: Marsaglia rejection, first accepted
// trial wins.  Returns false if 128 trials all failed (reference raises).
template <int KIND>
MPCD_HD bool rotation_axis_k(uint64_t key, double ax[3]) {
  KStream<KIND> g(key);
  for (int t = 0; t < kMaxAxisTrials; ++t) {
    double x = 2.0 * g.next() - 1.0;
    double y = 2.0 * g.next() - 1.0;
    double rsq = x * x + y * y;
    if (rsq < 1.0) {
      double root = sqrt(1.0 - rsq);
      ax[0] = (2.0 * x) * root;
      ax[1] = (2.0 * y) * root;
      ax[2] = 1.0 - 2.0 * rsq;
      return true;
    }
  }
  ax[0] = ax[1] = ax[2] = 0.0;
  return false;
}

// The axis of `cell` from the per-step prefix (key_prefix(seed, step, kAxis));
// the generator branch is uniform across a launch.
MPCD_HD bool rotation_axis_pre(int kind, uint64_t prefix, uint64_t cell, double ax[3]) {
  const uint64_t key = key_from_prefix(prefix, cell);
  switch (kind) {
    case kMinstd: return rotation_axis_k<kMinstd>(key, ax);
    case kPcg32: return rotation_axis_k<kPcg32>(key, ax);
    case kSfc64: return rotation_axis_k<kSfc64>(key, ax);
    default: return rotation_axis_k<kSplitmix>(key, ax);
  }
}

MPCD_HD bool rotation_axis(int kind, uint64_t seed, uint64_t step, uint64_t cell, double ax[3]) {
  return rotation_axis_pre(kind, key_prefix(seed, step, kAxis), cell, ax);
}

// collision.py:289-306 (Rodrigues), numpy order:
//   dot = ((0 + u0 a0) + u1 a1) + u2 a2         (np.sum(axis=1))
//   c   = (a1 p2 - a2 p1, a2 p0 - a0 p2, a0 p1 - a1 p0)   (np.cross)
//   v'  = ((com + u_par) + u_perp cos) + c sin
MPCD_HD void rotate(const double v[3], const double com[3], const double ax[3], double cs,
                    double sn, double out[3]) {
  double u0 = v[0] - com[0], u1 = v[1] - com[1], u2 = v[2] - com[2];
  double dot = ((0.0 + u0 * ax[0]) + u1 * ax[1]) + u2 * ax[2];
  double q0 = dot * ax[0], q1 = dot * ax[1], q2 = dot * ax[2];
  double w0 = u0 - q0, w1 = u1 - q1, w2 = u2 - q2;
  double c0 = ax[1] * w2 - ax[2] * w1;
  double c1 = ax[2] * w0 - ax[0] * w2;
  double c2 = ax[0] * w1 - ax[1] * w0;
  out[0] = ((com[0] + q0) + w0 * cs) + c0 * sn;
  out[1] = ((com[1] + q1) + w1 * cs) + c1 * sn;
  out[2] = ((com[2] + q2) + w2 * cs) + c2 * sn;
}

// np.mod(x, box) (npy_divmod: fmod, +box if the sign differs, +0 for a zero
// remainder) followed by particles.py:58-59's snap of == box to 0.0.  The
// common ranges avoid fmod: x in [0,box) is its own remainder (x + 0.0 turns
// -0.0 into +0.0 like copysign(0, box)); x in [-box,0) gives x + box;
// x in [box, 2 box) gives x - box exactly (Sterbenz).
MPCD_HD double wrap(double x, double box) {
  double m;
  if (x >= 0.0 && x < box) {
    m = x + 0.0;
  } else if (x < 0.0 && x >= -box) {
    m = x + box;
  } else if (x >= box && x < 2.0 * box) {
    m = x - box;
  } else {
    m = fmod(x, box);
    if (m != 0.0) {
      if ((box < 0.0) != (m < 0.0)) m += box;
    } else {
      m = copysign(0.0, box);
    }
  }
  return (m == box) ? 0.0 : m;
}

// Python-style non-negative integer modulo (numpy int64 % positive dims)
MPCD_HD int64_t pymod(int64_t v, int64_t d) {
  if ((uint64_t)v < (uint64_t)d) return v;
  int64_t r = v % d;
  return r < 0 ? r + d : r;
}

// floor((x - gmin) / a) as int64 (collision.py:132).  Division by a == 1.0
// is the identity in IEEE arithmetic, so `unit` skips it with equal bits.
MPCD_HD int64_t cell_coord(double x, double gmin, double a, bool unit) {
  double t = x - gmin;
  if (!unit) t = t / a;
#ifdef __CUDA_ARCH__
  return __double2ll_rd(t);
#else
  return (int64_t)floor(t);
#endif
}

// numpy pairwise_sum (numpy/_core/src/umath/loops_utils.h.src) over
// t[0], t[s], ..., t[(n-1) s]: below 8 terms a running sum from 0.0; up to
// 128 terms 8 strided accumulators, a fixed tree, then the tail; above 128
// the halves split at n/2 - (n/2)%8.
template <typename Ptr>
MPCD_HD double pairwise_leaf(Ptr t, int64_t n, int64_t s) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res += t[i * s];
    return res;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = t[j * s];
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8)
    for (int j = 0; j < 8; ++j) r[j] += t[(i + j) * s];
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; ++i) res += t[i * s];
  return res;
}

// The recursion above 128 terms runs on an explicit stack (post-order);
// the split points depend only on n, so the association is numpy's.
template <typename Ptr>
MPCD_HD double pairwise_sum(Ptr t, int64_t n, int64_t s) {
  if (n <= 128) return pairwise_leaf(t, n, s);
  struct Frame {
    int64_t off, n;
    double left;
    int state;
  };
  Frame st[48];
  int sp = 0;
  st[0] = Frame{0, n, 0.0, 0};
  double ret = 0.0;
  while (sp >= 0) {
    Frame& f = st[sp];
    if (f.n <= 128) {
      ret = pairwise_leaf(t + f.off * s, f.n, s);
      --sp;
      continue;
    }
    int64_t n2 = f.n / 2;
    n2 -= n2 % 8;
    if (f.state == 0) {
      f.state = 1;
      st[sp + 1] = Frame{f.off, n2, 0.0, 0};
      ++sp;
    } else if (f.state == 1) {
      f.left = ret;
      f.state = 2;
      st[sp + 1] = Frame{f.off + n2, f.n - n2, 0.0, 0};
      ++sp;
    } else {
      ret = f.left + ret;
      --sp;
    }
  }
  return ret;
}

// np.add.reduceat row semantics: seg[0] + pairwise_sum(seg[1:])
template <typename Ptr>
MPCD_HD double reduceat(Ptr t, int64_t k, int64_t s) {
  double out = t[0];
  if (k > 1) out = out + pairwise_sum(t + s, k - 1, s);
  return out;
}

}  // namespace mpcd
