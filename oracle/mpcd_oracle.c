/*
 * mpcd_oracle.c -- CPU restatement of the reference MPCD/SRD time step.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the
 * B200 engine in paper_2212_11878_b200/.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it, and only
 * as the checker or the timed CPU baseline -- never as the product path.
 *
 * It restates the reference Python/numpy package `mpcdsim`
 * (/root/reference/pkg/src/mpcdsim) in plain scalar C with the exact IEEE-754
 * operation order numpy 2.3.5 uses, so that it reproduces the reference
 * bit for bit (pinned against golden vectors generated from the reference
 * itself: tests/golden/make_golden.py, tests/test_oracle_golden.py).
 *
 * Numerics contract:
 *   - compile with -ffp-contract=off (no FMA contraction);
 *   - IEEE division and sqrt; floor; numpy float mod semantics;
 *   - np.add.reduceat association: seg[0] + pairwise_sum(seg[1:]) with
 *     numpy's 8-accumulator / 128-block pairwise kernel;
 *   - np.sum(axis=1) of 3 terms: ((0 + t0) + t1) + t2;
 *   - cos(alpha), sin(alpha) are inputs (the reference takes them from numpy).
 *
 * The keyed generators minstd / pcg32 / sfc64 do not exist in the reference
 * (SURVEY.md section 0.2); they follow their canonical published definitions
 * and the keyed-seeding protocol stated in DESIGN.md section 5.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------------------------------------------------------- RNG ---- */
/* rng.py:20-24 */
#define ORC_GOLDEN 0x9E3779B97F4A7C15ULL
#define ORC_MULT_A 0xBF58476D1CE4E5B9ULL
#define ORC_MULT_B 0x94D049BB133111EBULL
#define ORC_SEQ 0x2545F4914F6CDD1DULL

enum { ORC_SPLITMIX = 0, ORC_MINSTD = 1, ORC_PCG32 = 2, ORC_SFC64 = 3 };
enum { ORC_SHIFT = 0, ORC_AXIS = 1, ORC_INIT = 2 }; /* rng.py:28-33 */

/* rng.py:50-54 splitmix64 finalizer */
static inline uint64_t orc_mix64(uint64_t x) {
  x = (x ^ (x >> 30)) * ORC_MULT_A;
  x = (x ^ (x >> 27)) * ORC_MULT_B;
  return x ^ (x >> 31);
}

/* rng.py:67-77 */
uint64_t orc_key_state(uint64_t seed, uint64_t step, uint64_t purpose, uint64_t cell) {
  uint64_t s = orc_mix64(seed * ORC_SEQ + ORC_GOLDEN);
  s = orc_mix64(s ^ (step * ORC_SEQ + ORC_GOLDEN));
  s = orc_mix64(s ^ (purpose * ORC_SEQ + ORC_GOLDEN));
  s = orc_mix64(s ^ (cell * ORC_SEQ + ORC_GOLDEN));
  return s;
}

/* rng.py:84-92: (mix(state ^ ((i+1)*SEQ)) >> 11) * 2^-53 */
double orc_uniform_at(uint64_t state, uint64_t index) {
  uint64_t h = orc_mix64(state ^ ((index + 1ULL) * ORC_SEQ));
  return (double)(h >> 11) * (1.0 / 9007199254740992.0);
}

/* Sequential keyed stream: draw j of the stream keyed by `state`. */
typedef struct {
  int kind;
  uint64_t state;   /* splitmix: key; minstd: x; pcg32: state; sfc64: a */
  uint64_t b, c, w; /* pcg32: inc in b; sfc64: b, c, counter */
  uint64_t draw;    /* splitmix counter */
} orc_stream;

static inline uint32_t orc_minstd_step(orc_stream* g) {
  g->state = (g->state * 48271ULL) % 2147483647ULL;
  return (uint32_t)g->state;
}
static inline uint32_t orc_pcg32_step(orc_stream* g) {
  uint64_t old = g->state;
  g->state = old * 6364136223846793005ULL + g->b;
  uint32_t xs = (uint32_t)(((old >> 18) ^ old) >> 27);
  uint32_t rot = (uint32_t)(old >> 59);
  return (xs >> rot) | (xs << ((-rot) & 31u));
}
static inline uint64_t orc_sfc64_step(orc_stream* g) {
  uint64_t a = g->state, b = g->b, c = g->c, w = g->w;
  uint64_t tmp = a + b + w;
  g->w = w + 1;
  g->state = b ^ (b >> 11);
  g->b = c + (c << 3);
  g->c = ((c << 24) | (c >> 40)) + tmp;
  return tmp;
}

static void orc_stream_init(orc_stream* g, int kind, uint64_t key) {
  memset(g, 0, sizeof(*g));
  g->kind = kind;
  if (kind == ORC_MINSTD) {
    g->state = 1ULL + key % 2147483646ULL;
  } else if (kind == ORC_PCG32) { /* pcg32_srandom_r(key, 54) */
    g->state = 0;
    g->b = (54ULL << 1) | 1ULL;
    orc_pcg32_step(g);
    g->state += key;
    orc_pcg32_step(g);
  } else if (kind == ORC_SFC64) { /* a = b = c = key, counter = 1, 12 discards */
    g->state = key;
    g->b = key;
    g->c = key;
    g->w = 1;
    for (int i = 0; i < 12; ++i) orc_sfc64_step(g);
  } else {
    g->state = key;
    g->draw = 0;
  }
}

static double orc_stream_next(orc_stream* g) {
  switch (g->kind) {
    case ORC_MINSTD: {
      uint64_t hi = (uint64_t)(orc_minstd_step(g) - 1u) >> 4;
      uint64_t lo = (uint64_t)(orc_minstd_step(g) - 1u) >> 5;
      return (double)((hi << 26) | lo) * (1.0 / 9007199254740992.0);
    }
    case ORC_PCG32: {
      uint64_t hi = orc_pcg32_step(g) >> 5;
      uint64_t lo = orc_pcg32_step(g) >> 6;
      return (double)((hi << 26) | lo) * (1.0 / 9007199254740992.0);
    }
    case ORC_SFC64:
      return (double)(orc_sfc64_step(g) >> 11) * (1.0 / 9007199254740992.0);
    default:
      return orc_uniform_at(g->state, g->draw++);
  }
}

/* Raw generator outputs from an explicit state (known-answer tests). */
void orc_prng_raw(int kind, uint64_t s0, uint64_t s1, uint64_t s2, uint64_t s3,
                  int64_t count, uint64_t* out) {
  orc_stream g;
  memset(&g, 0, sizeof(g));
  g.kind = kind;
  if (kind == ORC_MINSTD) {
    g.state = s0;
    for (int64_t i = 0; i < count; ++i) out[i] = orc_minstd_step(&g);
  } else if (kind == ORC_PCG32) { /* pcg32_srandom_r(s0, s1) */
    g.b = (s1 << 1) | 1ULL;
    orc_pcg32_step(&g);
    g.state += s0;
    orc_pcg32_step(&g);
    for (int64_t i = 0; i < count; ++i) out[i] = orc_pcg32_step(&g);
  } else if (kind == ORC_SFC64) {
    g.state = s0; g.b = s1; g.c = s2; g.w = s3;
    for (int64_t i = 0; i < count; ++i) out[i] = orc_sfc64_step(&g);
  } else {
    for (int64_t i = 0; i < count; ++i) out[i] = orc_mix64(s0 ^ (((uint64_t)i + 1ULL) * ORC_SEQ));
  }
}

/* First `count` doubles of the stream keyed by (seed, step, purpose, cell). */
void orc_sample_uniform(int kind, uint64_t seed, uint64_t step, uint64_t purpose,
                        uint64_t cell, int64_t count, double* out) {
  orc_stream g;
  orc_stream_init(&g, kind, orc_key_state(seed, step, purpose, cell));
  for (int64_t i = 0; i < count; ++i) out[i] = orc_stream_next(&g);
}

/* collision.py:32-36 */
void orc_grid_shift(int kind, uint64_t seed, uint64_t step, double a, double out[3]) {
  orc_stream g;
  orc_stream_init(&g, kind, orc_key_state(seed, step, ORC_SHIFT, 0));
  for (int d = 0; d < 3; ++d) out[d] = (orc_stream_next(&g) - 0.5) * a;
}

/* collision.py:217-250 (one cell): Marsaglia, <= 128 trials. */
static int orc_axis_one(int kind, uint64_t seed, uint64_t step, uint64_t cell, double ax[3]) {
  orc_stream g;
  orc_stream_init(&g, kind, orc_key_state(seed, step, ORC_AXIS, cell));
  for (int t = 0; t < 128; ++t) {
    double u1 = orc_stream_next(&g);
    double u2 = orc_stream_next(&g);
    double x = 2.0 * u1 - 1.0;
    double y = 2.0 * u2 - 1.0;
    double xx = x * x, yy = y * y;
    double rsq = xx + yy;
    if (rsq < 1.0) {
      double root = sqrt(1.0 - rsq);
      ax[0] = (2.0 * x) * root;
      ax[1] = (2.0 * y) * root;
      ax[2] = 1.0 - 2.0 * rsq;
      return 0;
    }
  }
  return 1;
}

int orc_rotation_axes(int kind, uint64_t seed, uint64_t step, const int64_t* cell_ids,
                      int64_t k, double* axes) {
  int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
  for (int64_t i = 0; i < k; ++i) bad |= orc_axis_one(kind, seed, step, (uint64_t)cell_ids[i], axes + 3 * i);
  return bad;
}

/* ----------------------------------------------------------- numerics ---- */
/* numpy npy_divmod remainder (np.mod for float64) + particles.py:52-59 snap */
static inline double orc_wrap1(double x, double box) {
  double m = fmod(x, box);
  if (m != 0.0) {
    if ((box < 0.0) != (m < 0.0)) m += box;
  } else {
    m = copysign(0.0, box);
  }
  return (m == box) ? 0.0 : m;
}

void orc_wrap(int64_t n, const double* x, double box, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = orc_wrap1(x[i], box);
}

/* numpy pairwise_sum (loops_utils.h.src) over t[0..n) with stride */
static double orc_pairwise(const double* t, int64_t n, int64_t stride) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res += t[i * stride];
    return res;
  } else if (n <= 128) {
    double r[8];
    int64_t i;
    for (int j = 0; j < 8; ++j) r[j] = t[j * stride];
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += t[(i + j) * stride];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += t[i * stride];
    return res;
  } else {
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return orc_pairwise(t, n2, stride) + orc_pairwise(t + n2 * stride, n - n2, stride);
  }
}

/* np.add.reduceat row semantics: seg[0] + pairwise(seg[1:]) */
static inline double orc_reduceat_col(const double* seg, int64_t k, int64_t stride) {
  double out = seg[0];
  if (k > 1) out = out + orc_pairwise(seg + stride, k - 1, stride);
  return out;
}

/* ------------------------------------------------------------ binning ---- */
static inline int64_t orc_pymod(int64_t a, int64_t d) {
  int64_t r = a % d;
  return r < 0 ? r + d : r;
}

/* collision.py:93-109 structure: bincount, exclusive cumsum, stable argsort */
static void orc_structure(const int64_t* cells, int64_t n, int64_t ncells, int64_t* counts,
                          int64_t* offsets, int64_t* perm) {
  memset(counts, 0, sizeof(int64_t) * (size_t)ncells);
  for (int64_t i = 0; i < n; ++i) counts[cells[i]]++;
  int64_t acc = 0;
  for (int64_t c = 0; c < ncells; ++c) {
    offsets[c] = acc;
    acc += counts[c];
  }
  int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ncells ? ncells : 1));
  memcpy(cur, offsets, sizeof(int64_t) * (size_t)ncells);
  for (int64_t i = 0; i < n; ++i) perm[cur[cells[i]]++] = i; /* stable */
  free(cur);
}

/* collision.py:112-147.  Returns 0, or 1 with err_info = {particle, axis}. */
int orc_build_linked_cells(const double* pos, int64_t n, double a, const double gmin[3],
                           const int64_t dims[3], const int32_t wrap[3], int64_t* cells,
                           int64_t* counts, int64_t* offsets, int64_t* perm, int64_t* err_info) {
  int64_t ncells = dims[0] * dims[1] * dims[2];
  int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(3 * (n ? n : 1)));
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)
    for (int d = 0; d < 3; ++d) idx[3 * i + d] = (int64_t)floor((pos[3 * i + d] - gmin[d]) / a);
  for (int d = 0; d < 3; ++d) {
    if (wrap[d]) {
      for (int64_t i = 0; i < n; ++i) idx[3 * i + d] = orc_pymod(idx[3 * i + d], dims[d]);
    } else {
      for (int64_t i = 0; i < n; ++i) {
        int64_t v = idx[3 * i + d];
        if (v < 0 || v >= dims[d]) {
          err_info[0] = i;
          err_info[1] = d;
          free(idx);
          return 1;
        }
      }
    }
  }
  for (int64_t i = 0; i < n; ++i)
    cells[i] = (idx[3 * i] * dims[1] + idx[3 * i + 1]) * dims[2] + idx[3 * i + 2];
  free(idx);
  orc_structure(cells, n, ncells, counts, offsets, perm);
  return 0;
}

/* collision.py:150-163 */
int orc_linked_cells_from_indices(const int64_t* cells, int64_t n, int64_t ncells, int64_t* counts,
                                  int64_t* offsets, int64_t* perm) {
  for (int64_t i = 0; i < n; ++i)
    if (cells[i] < 0 || cells[i] >= ncells) return 1;
  orc_structure(cells, n, ncells, counts, offsets, perm);
  return 0;
}

/* ------------------------------------------------------------ moments ---- */
/* collision.py:190-206: rows (m*v0, m*v1, m*v2, m) gathered in permutation
 * order, reduceat over occupied bins; zeros for empty cells. */
void orc_segment_moments(int64_t n, int64_t ncells, const int64_t* perm, const int64_t* counts,
                         const int64_t* offsets, const double* vel, const double* mass,
                         double* out) {
  (void)n;
#pragma omp parallel
  {
    int64_t cap = 64;
    double* buf = (double*)malloc(sizeof(double) * 4 * (size_t)cap);
#pragma omp for schedule(dynamic, 4096)
    for (int64_t c = 0; c < ncells; ++c) {
      int64_t k = counts[c];
      double* o = out + 4 * c;
      if (k == 0) {
        o[0] = o[1] = o[2] = o[3] = 0.0;
        continue;
      }
      if (k > cap) {
        cap = k;
        buf = (double*)realloc(buf, sizeof(double) * 4 * (size_t)cap);
      }
      const int64_t* seg = perm + offsets[c];
      for (int64_t j = 0; j < k; ++j) {
        int64_t p = seg[j];
        double m = mass[p];
        buf[4 * j + 0] = m * vel[3 * p + 0];
        buf[4 * j + 1] = m * vel[3 * p + 1];
        buf[4 * j + 2] = m * vel[3 * p + 2];
        buf[4 * j + 3] = m;
      }
      for (int col = 0; col < 4; ++col) o[col] = orc_reduceat_col(buf + col, k, 4);
    }
    free(buf);
  }
}

/* collision.py:209-214 */
void orc_finalize_com(int64_t ncells, const double* mom, double* com) {
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < ncells; ++c) {
    double m = mom[4 * c + 3];
    for (int d = 0; d < 3; ++d) com[3 * c + d] = (m > 0.0) ? mom[4 * c + d] / m : 0.0;
  }
}

/* ----------------------------------------------------------- rotation ---- */
/* collision.py:289-306 (Rodrigues, numpy operation order) */
static inline void orc_rotate1(const double* v, const double* com, const double* ax, double cs,
                               double sn, double* out) {
  double u0 = v[0] - com[0], u1 = v[1] - com[1], u2 = v[2] - com[2];
  double p0 = u0 * ax[0], p1 = u1 * ax[1], p2 = u2 * ax[2];
  double dot = ((0.0 + p0) + p1) + p2;
  double q0 = dot * ax[0], q1 = dot * ax[1], q2 = dot * ax[2];
  double w0 = u0 - q0, w1 = u1 - q1, w2 = u2 - q2;
  double c0 = ax[1] * w2 - ax[2] * w1;
  double c1 = ax[2] * w0 - ax[0] * w2;
  double c2 = ax[0] * w1 - ax[1] * w0;
  out[0] = ((com[0] + q0) + w0 * cs) + c0 * sn;
  out[1] = ((com[1] + q1) + w1 * cs) + c1 * sn;
  out[2] = ((com[2] + q2) + w2 * cs) + c2 * sn;
}

void orc_rotate(int64_t n, const double* vel, const double* com_pp, const double* axis_pp,
                double cs, double sn, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) orc_rotate1(vel + 3 * i, com_pp + 3 * i, axis_pp + 3 * i, cs, sn, out + 3 * i);
}

/* collision.py:309-324 */
void orc_rotate_cells(int64_t n, const int64_t* cells, const double* vel, const double* com,
                      const double* axes, double cs, double sn, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    int64_t c = cells[i];
    orc_rotate1(vel + 3 * i, com + 3 * c, axes + 3 * c, cs, sn, out + 3 * i);
  }
}

/* particles.py:62-67 with a per-axis box (the cubic case has box[d] equal) */
void orc_stream_wrap(int64_t n, const double* pos, const double* vel, double dt, const double box[3],
                     double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)
    for (int d = 0; d < 3; ++d) {
      double s = vel[3 * i + d] * dt;
      out[3 * i + d] = orc_wrap1(pos[3 * i + d] + s, box[d]);
    }
}

/* collision.py:327-344 (tolerance-level diagnostic) */
double orc_cell_drift(int64_t ncells, const double* before, const double* after) {
  double worst = 0.0;
  int any = 0;
  for (int64_t c = 0; c < ncells; ++c) {
    const double* b = before + 4 * c;
    const double* a = after + 4 * c;
    if (!(b[3] > 0.0)) continue;
    any = 1;
    double d0 = a[0] - b[0], d1 = a[1] - b[1], d2 = a[2] - b[2];
    double dp = sqrt(((0.0 + d0 * d0) + d1 * d1) + d2 * d2);
    double nb = sqrt(((0.0 + b[0] * b[0]) + b[1] * b[1]) + b[2] * b[2]);
    double na = sqrt(((0.0 + a[0] * a[0]) + a[1] * a[1]) + a[2] * a[2]);
    double scale = nb > na ? nb : na;
    if (b[3] > scale) scale = b[3];
    if (scale < 1e-300) scale = 1e-300;
    double r = dp / scale;
    if (r > worst) worst = r;
  }
  return any ? worst : 0.0;
}

/* particles.py:168-181 (tolerance-level): momentum(3), energy, mass */
void orc_diag(int64_t n, const double* vel, const double* mass, double out[5]) {
  double px = 0, py = 0, pz = 0, e = 0, m = 0;
  for (int64_t i = 0; i < n; ++i) {
    double mi = mass[i];
    const double* v = vel + 3 * i;
    px += mi * v[0];
    py += mi * v[1];
    pz += mi * v[2];
    e += mi * (((0.0 + v[0] * v[0]) + v[1] * v[1]) + v[2] * v[2]);
    m += mi;
  }
  out[0] = px; out[1] = py; out[2] = pz; out[3] = 0.5 * e; out[4] = m;
}

/* -------------------------------------------------------- serial step ---- */
/*
 * engine.py:415-455 serial_collision_step, in place on (n,3) C-order arrays.
 * dims = cells per axis (cubic: all equal; per-axis is the non-cubic
 * extension).  Optional outputs: drift (want_drift), com (ncells*3),
 * counts (ncells), perm (n), cells (n).  Returns 0, or 2 if an axis draw
 * failed to terminate.
 */
int orc_serial_step(int64_t n, double* pos, double* vel, const double* mass, const int64_t dims[3],
                    double a, double dt, double cs, double sn, uint64_t seed, uint64_t step,
                    int kind, int want_drift, double* drift_out, double* com_out,
                    int64_t* counts_out, int64_t* perm_out, int64_t* cells_out) {
  int64_t ncells = dims[0] * dims[1] * dims[2];
  double off[3], box[3];
  orc_grid_shift(kind, seed, step, a, off);
  for (int d = 0; d < 3; ++d) box[d] = (double)dims[d] * a;
  int64_t* cells = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
  int64_t* counts = (int64_t*)malloc(sizeof(int64_t) * (size_t)ncells);
  int64_t* offsets = (int64_t*)malloc(sizeof(int64_t) * (size_t)ncells);
  int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
  double* mom = (double*)malloc(sizeof(double) * 4 * (size_t)ncells);
  double* com = (double*)malloc(sizeof(double) * 3 * (size_t)ncells);
  double* axes = (double*)calloc(3 * (size_t)ncells, sizeof(double));
  double* rot = (double*)malloc(sizeof(double) * 3 * (size_t)(n ? n : 1));
  int rc = 0;

  /* build_linked_cells(pos, a, off, off + box, wrap=(T,T,T)) */
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    int64_t ix = orc_pymod((int64_t)floor((pos[3 * i + 0] - off[0]) / a), dims[0]);
    int64_t iy = orc_pymod((int64_t)floor((pos[3 * i + 1] - off[1]) / a), dims[1]);
    int64_t iz = orc_pymod((int64_t)floor((pos[3 * i + 2] - off[2]) / a), dims[2]);
    cells[i] = (ix * dims[1] + iy) * dims[2] + iz;
  }
  orc_structure(cells, n, ncells, counts, offsets, perm);
  orc_segment_moments(n, ncells, perm, counts, offsets, vel, mass, mom);
  orc_finalize_com(ncells, mom, com);
  /* build_rotation_plan over occupied cells; global id == local flat id */
  int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
  for (int64_t c = 0; c < ncells; ++c)
    if (counts[c] > 0) bad |= orc_axis_one(kind, seed, step, (uint64_t)c, axes + 3 * c);
  if (bad) rc = 2;
  orc_rotate_cells(n, cells, vel, com, axes, cs, sn, rot);
  if (want_drift && drift_out) {
    double* post = (double*)malloc(sizeof(double) * 4 * (size_t)ncells);
    orc_segment_moments(n, ncells, perm, counts, offsets, rot, mass, post);
    *drift_out = orc_cell_drift(ncells, mom, post);
    free(post);
  }
  if (com_out) memcpy(com_out, com, sizeof(double) * 3 * (size_t)ncells);
  if (counts_out) memcpy(counts_out, counts, sizeof(int64_t) * (size_t)ncells);
  if (perm_out) memcpy(perm_out, perm, sizeof(int64_t) * (size_t)n);
  if (cells_out) memcpy(cells_out, cells, sizeof(int64_t) * (size_t)n);
  /* stream_and_wrap */
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)
    for (int d = 0; d < 3; ++d) {
      double s = rot[3 * i + d] * dt;
      pos[3 * i + d] = orc_wrap1(pos[3 * i + d] + s, box[d]);
      vel[3 * i + d] = rot[3 * i + d];
    }
  free(cells); free(counts); free(offsets); free(perm);
  free(mom); free(com); free(axes); free(rot);
  return rc;
}

/* particles.py:101-127 init_system for the CPU-baseline sample only: positions
 * are bit-exact (integer hash times box); velocities use libm log/cos, which
 * agree with numpy only to within an ulp. */
void orc_init_system(int64_t n, const double box[3], uint64_t seed, double variance, double* pos,
                     double* vel) {
  uint64_t st = orc_key_state(seed, 0, ORC_INIT, 0);
  double sigma = sqrt(variance);
  const double two_pi = 2.0 * 3.141592653589793;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)
    for (int d = 0; d < 3; ++d) {
      pos[3 * i + d] = orc_uniform_at(st, (uint64_t)(3 * i + d)) * box[d];
      uint64_t g = (uint64_t)(3 * n + 3 * i + d);
      double u1 = orc_uniform_at(st, 2 * g), u2 = orc_uniform_at(st, 2 * g + 1);
      vel[3 * i + d] = sqrt(-2.0 * log(1.0 - u1)) * cos(two_pi * u2) * sigma;
    }
  double mean[3] = {0, 0, 0};
  for (int64_t i = 0; i < n; ++i)
    for (int d = 0; d < 3; ++d) mean[d] += vel[3 * i + d];
  for (int d = 0; d < 3; ++d) mean[d] = n ? mean[d] / (double)n : 0.0;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)
    for (int d = 0; d < 3; ++d) vel[3 * i + d] -= mean[d];
}

int orc_set_threads(int t) {
#ifdef _OPENMP
  if (t > 0) omp_set_num_threads(t);
  return omp_get_max_threads();
#else
  (void)t;
  return 1;
#endif
}
