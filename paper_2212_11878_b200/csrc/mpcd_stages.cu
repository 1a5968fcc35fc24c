// mpcd_stages.cu -- one kernel per reference function of collision.py /
// particles.py, on caller-owned device buffers in the reference layouts.
// These are the stage-level drop-in boundary; the
// engine (mpcd_engine.cu) fuses the same math for the time step.
#include <string.h>

#include <vector>

#include "mpcd_internal.h"

namespace mpcd {
namespace {

// rng.sample_uniform: the keyed stream is sequential for the non-reference
// generators, so one thread walks it (counts in the API are small).
__global__ void k_sample_uniform(int prng, uint64_t key, int64_t count, double* out) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  Stream g(prng, key);
  for (int64_t i = 0; i < count; ++i) out[i] = g.next();
}

__global__ void k_sample_uniform_counter(uint64_t key, int64_t count, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = uniform_at(key, (uint64_t)i);
}

// collision.py:132-146: per-axis floor index, wrap or range check, flatten.
__global__ void k_bin_cells(const double* pos, int64_t n, double a, int unit, double g0, double g1,
                            double g2, int64_t L0, int64_t L1, int64_t L2, int w0, int w1, int w2,
                            int64_t* cells, unsigned long long* bad /*3*/, uint32_t* counts) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t ix = cell_coord(pos[3 * i], g0, a, unit);
    int64_t iy = cell_coord(pos[3 * i + 1], g1, a, unit);
    int64_t iz = cell_coord(pos[3 * i + 2], g2, a, unit);
    bool ok = true;
    if (w0) ix = pymod(ix, L0); else if (ix < 0 || ix >= L0) { atomicMin(&bad[0], (unsigned long long)i); ok = false; }
    if (w1) iy = pymod(iy, L1); else if (iy < 0 || iy >= L1) { atomicMin(&bad[1], (unsigned long long)i); ok = false; }
    if (w2) iz = pymod(iz, L2); else if (iz < 0 || iz >= L2) { atomicMin(&bad[2], (unsigned long long)i); ok = false; }
    if (ok) {
      const int64_t c = (ix * L1 + iy) * L2 + iz;
      cells[i] = c;
      atomicAdd(&counts[c], 1u);
    }
  }
}

__global__ void k_count_cells(const int64_t* cells, int64_t n, int64_t nc, uint32_t* counts,
                              unsigned long long* bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = cells[i];
    if (c < 0 || c >= nc) atomicMin(bad, (unsigned long long)i);
    else atomicAdd(&counts[c], 1u);
  }
}

__global__ void k_widen(const uint32_t* in, int64_t* out, int64_t count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int64_t)in[i];
}

// unstable scatter of particle indices into their cell segments
__global__ void k_scatter_idx(const int64_t* cells, int64_t n, const int64_t* offsets,
                              uint32_t* cursor, int64_t* tmp_perm) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = cells[i];
    tmp_perm[offsets[c] + atomicAdd(&cursor[c], 1u)] = i;
  }
}

// Canonicalise each segment to ascending particle index: that is exactly
// np.argsort(kind="stable") (collision.py:98).
__global__ void k_segment_rank(const int64_t* cells, const int64_t* offsets, const int64_t* counts,
                               const int64_t* tmp_perm, int64_t n, int64_t* perm) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t me = tmp_perm[j];
    const int64_t c = cells[me];
    const int64_t s = offsets[c], e = s + counts[c];
    int64_t rank = 0;
    for (int64_t q = s; q < e; ++q) rank += (tmp_perm[q] < me) ? 1 : 0;
    perm[s + rank] = me;
  }
}

// rows (m v0, m v1, m v2, m) gathered through the permutation
struct Gather {
  const int64_t* perm;
  const double* vel;
  const double* mass;
  int comp;
  __device__ double operator[](int64_t i) const {
    const int64_t p = perm[i];
    const double m = mass[p];
    return comp < 3 ? m * vel[3 * p + comp] : m;
  }
  __device__ Gather operator+(int64_t o) const { return Gather{perm + o, vel, mass, comp}; }
};

__global__ void k_segment_moments(const int64_t* perm, const int64_t* counts,
                                  const int64_t* offsets, int64_t nc, const double* vel,
                                  const double* mass, double* out) {
  for (int64_t task = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; task < 4 * nc;
       task += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = task >> 2;
    const int comp = (int)(task & 3);
    const int64_t k = counts[c];
    out[task] = k ? reduceat(Gather{perm + offsets[c], vel, mass, comp}, k, 1) : 0.0;
  }
}

__global__ void k_finalize_com(const double* mom, int64_t nc, double* com) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nc;
       c += (int64_t)gridDim.x * blockDim.x) {
    const double m = mom[4 * c + 3];
    for (int d = 0; d < 3; ++d) com[3 * c + d] = (m > 0.0) ? mom[4 * c + d] / m : 0.0;
  }
}

__global__ void k_axes(int prng, uint64_t seed, uint64_t step, const int64_t* ids, int64_t k,
                       double* axes, uint32_t* fail_flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
       i += (int64_t)gridDim.x * blockDim.x)
    if (!rotation_axis(prng, seed, step, (uint64_t)ids[i], axes + 3 * i)) atomicOr(fail_flag, 1u);
}

__global__ void k_rotate(const double* vel, const double* com, const double* ax, int64_t n,
                         double cs, double sn, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    rotate(vel + 3 * i, com + 3 * i, ax + 3 * i, cs, sn, out + 3 * i);
}

__global__ void k_rotate_cells(const int64_t* cells, const double* vel, const double* com,
                               const double* ax, int64_t n, double cs, double sn, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = cells[i];
    rotate(vel + 3 * i, com + 3 * c, ax + 3 * c, cs, sn, out + 3 * i);
  }
}

__global__ void k_wrap(const double* x, int64_t count, double box, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = wrap(x[i], box);
}

__global__ void k_stream_wrap(const double* pos, const double* vel, int64_t n, double dt,
                              double b0, double b1, double b2, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    out[3 * i] = wrap(pos[3 * i] + vel[3 * i] * dt, b0);
    out[3 * i + 1] = wrap(pos[3 * i + 1] + vel[3 * i + 1] * dt, b1);
    out[3 * i + 2] = wrap(pos[3 * i + 2] + vel[3 * i + 2] * dt, b2);
  }
}

__global__ void k_cell_drift(const double* before, const double* after, int64_t nc,
                             unsigned long long* out_bits, uint32_t* any) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nc;
       c += (int64_t)gridDim.x * blockDim.x) {
    const double* b = before + 4 * c;
    const double* a = after + 4 * c;
    if (!(b[3] > 0.0)) continue;
    atomicOr(any, 1u);
    double d0 = a[0] - b[0], d1 = a[1] - b[1], d2 = a[2] - b[2];
    double dp = sqrt(((0.0 + d0 * d0) + d1 * d1) + d2 * d2);
    double nb = sqrt(((0.0 + b[0] * b[0]) + b[1] * b[1]) + b[2] * b[2]);
    double na = sqrt(((0.0 + a[0] * a[0]) + a[1] * a[1]) + a[2] * a[2]);
    double scale = fmax(fmax(nb, na), b[3]);
    atomicMax(out_bits, (unsigned long long)__double_as_longlong(dp / fmax(scale, 1e-300)));
  }
}

// Stable structure (counts, offsets, permutation) from flat cell indices.
int structure(const int64_t* cells, int64_t n, int64_t nc, int64_t* counts64, int64_t* offsets,
              int64_t* perm, cudaStream_t st, uint32_t* counts32, bool counted) {
  ScanState scan;
  int rc = scan.init(nc);
  if (rc) return rc;
  if (!counted) {
    unsigned long long* bad = nullptr;
    MPCD_CUDA(cudaMallocAsync(&bad, sizeof(unsigned long long), st));
    MPCD_CUDA(cudaMemsetAsync(bad, 0xFF, sizeof(unsigned long long), st));
    if (n > 0) k_count_cells<<<grid_for(n, 256), 256, 0, st>>>(cells, n, nc, counts32, bad);
    unsigned long long hbad = 0;
    MPCD_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(hbad), cudaMemcpyDeviceToHost, st));
    MPCD_CUDA(cudaFreeAsync(bad, st));
    MPCD_CUDA(cudaStreamSynchronize(st));
    if (hbad != ~0ULL) {
      scan.release();
      return fail(MPCD_ERR_BINNING, "flat cell index out of range");
    }
  }
  k_widen<<<grid_for(nc, 256), 256, 0, st>>>(counts32, counts64, nc);
  rc = scan_u32(scan, counts32, nullptr, offsets, nc, true, st);
  if (rc) { scan.release(); return rc; }
  if (n > 0) {
    int64_t* tmp = nullptr;
    MPCD_CUDA(cudaMallocAsync(&tmp, sizeof(int64_t) * n, st));
    // counts32 was zeroed by the scan: reuse it as the cursor
    k_scatter_idx<<<grid_for(n, 256), 256, 0, st>>>(cells, n, offsets, counts32, tmp);
    k_segment_rank<<<grid_for(n, 256), 256, 0, st>>>(cells, offsets, counts64, tmp, n, perm);
    MPCD_CUDA(cudaFreeAsync(tmp, st));
  }
  MPCD_LAUNCH_CHECK();
  MPCD_CUDA(cudaStreamSynchronize(st));
  scan.release();
  return MPCD_OK;
}

}  // namespace
}  // namespace mpcd

using namespace mpcd;

extern "C" {

int mpcd_stage_sample_uniform(int32_t prng, uint64_t seed, uint64_t step, uint64_t purpose,
                              uint64_t cell, int64_t count, double* out, void* stream) {
  clear_error();
  if (count <= 0) return MPCD_OK;
  const uint64_t key = key_state(seed, step, purpose, cell);
  if (prng == kSplitmix)
    k_sample_uniform_counter<<<grid_for(count, 256), 256, 0, as_stream(stream)>>>(key, count, out);
  else
    k_sample_uniform<<<1, 1, 0, as_stream(stream)>>>(prng, key, count, out);
  MPCD_LAUNCH_CHECK();
  return MPCD_OK;
}

int mpcd_stage_build_linked_cells(const double* pos, int64_t n, double cell_size,
                                  const double grid_min[3], const int64_t dims[3],
                                  const int32_t wrap[3], int64_t* cells, int64_t* bin_count,
                                  int64_t* bin_offset, int64_t* permutation, int64_t err[2],
                                  void* stream) {
  clear_error();
  cudaStream_t st = as_stream(stream);
  const int64_t nc = dims[0] * dims[1] * dims[2];
  if (nc < 1 || nc >= (1LL << 32)) return fail(MPCD_ERR_CONFIG, "bad grid dims");
  uint32_t* counts32 = nullptr;
  unsigned long long* bad = nullptr;
  MPCD_CUDA(cudaMallocAsync(&counts32, sizeof(uint32_t) * nc, st));
  MPCD_CUDA(cudaMemsetAsync(counts32, 0, sizeof(uint32_t) * nc, st));
  MPCD_CUDA(cudaMallocAsync(&bad, 3 * sizeof(unsigned long long), st));
  MPCD_CUDA(cudaMemsetAsync(bad, 0xFF, 3 * sizeof(unsigned long long), st));
  if (n > 0) {
    k_bin_cells<<<grid_for(n, 256), 256, 0, st>>>(
        pos, n, cell_size, cell_size == 1.0, grid_min[0], grid_min[1], grid_min[2], dims[0],
        dims[1], dims[2], wrap[0], wrap[1], wrap[2], cells, bad, counts32);
    MPCD_LAUNCH_CHECK();
  }
  unsigned long long hbad[3];
  MPCD_CUDA(cudaMemcpyAsync(hbad, bad, sizeof(hbad), cudaMemcpyDeviceToHost, st));
  MPCD_CUDA(cudaFreeAsync(bad, st));
  MPCD_CUDA(cudaStreamSynchronize(st));
  for (int d = 0; d < 3; ++d) {
    if (hbad[d] != ~0ULL) {  // first failing axis, first particle on it
      if (err) { err[0] = (int64_t)hbad[d]; err[1] = d; }
      cudaFreeAsync(counts32, st);
      return fail(MPCD_ERR_BINNING, "particle %llu lies outside the grid along axis %d", hbad[d], d);
    }
  }
  int rc = structure(cells, n, nc, bin_count, bin_offset, permutation, st, counts32, true);
  cudaFreeAsync(counts32, st);
  return rc;
}

int mpcd_stage_structure_from_cells(const int64_t* cells, int64_t n, int64_t n_cells,
                                    int64_t* bin_count, int64_t* bin_offset,
                                    int64_t* permutation, void* stream) {
  clear_error();
  cudaStream_t st = as_stream(stream);
  if (n_cells < 1 || n_cells >= (1LL << 32)) return fail(MPCD_ERR_CONFIG, "bad cell count");
  uint32_t* counts32 = nullptr;
  MPCD_CUDA(cudaMallocAsync(&counts32, sizeof(uint32_t) * n_cells, st));
  MPCD_CUDA(cudaMemsetAsync(counts32, 0, sizeof(uint32_t) * n_cells, st));
  int rc = structure(cells, n, n_cells, bin_count, bin_offset, permutation, st, counts32, false);
  cudaFreeAsync(counts32, st);
  cudaStreamSynchronize(st);
  return rc;
}

int mpcd_stage_segment_moments(const int64_t* permutation, const int64_t* bin_count,
                               const int64_t* bin_offset, int64_t n_cells, const double* vel,
                               const double* mass, int64_t n, double* moments, void* stream) {
  clear_error();
  (void)n;
  if (n_cells <= 0) return MPCD_OK;
  k_segment_moments<<<grid_for(4 * n_cells, 128), 128, 0, as_stream(stream)>>>(
      permutation, bin_count, bin_offset, n_cells, vel, mass, moments);
  MPCD_LAUNCH_CHECK();
  return MPCD_OK;
}

int mpcd_stage_finalize_com(const double* moments, int64_t n_cells, double* com, void* stream) {
  clear_error();
  if (n_cells <= 0) return MPCD_OK;
  k_finalize_com<<<grid_for(n_cells, 256), 256, 0, as_stream(stream)>>>(moments, n_cells, com);
  MPCD_LAUNCH_CHECK();
  return MPCD_OK;
}

int mpcd_stage_rotation_axes(int32_t prng, uint64_t seed, int64_t step, const int64_t* cell_ids,
                             int64_t k, double* axes, void* stream) {
  clear_error();
  if (k <= 0) return MPCD_OK;
  cudaStream_t st = as_stream(stream);
  uint32_t* flag = nullptr;
  MPCD_CUDA(cudaMallocAsync(&flag, sizeof(uint32_t), st));
  MPCD_CUDA(cudaMemsetAsync(flag, 0, sizeof(uint32_t), st));
  k_axes<<<grid_for(k, 128), 128, 0, st>>>(prng, seed, (uint64_t)step, cell_ids, k, axes, flag);
  MPCD_LAUNCH_CHECK();
  uint32_t h = 0;
  MPCD_CUDA(cudaMemcpyAsync(&h, flag, sizeof(h), cudaMemcpyDeviceToHost, st));
  MPCD_CUDA(cudaFreeAsync(flag, st));
  MPCD_CUDA(cudaStreamSynchronize(st));
  if (h) return fail(MPCD_ERR_RNG, "axis rejection sampling failed to terminate");
  return MPCD_OK;
}

int mpcd_stage_rotate(const double* vel, const double* com_pp, const double* axis_pp, int64_t n,
                      double cos_alpha, double sin_alpha, double* out, void* stream) {
  clear_error();
  if (n <= 0) return MPCD_OK;
  k_rotate<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(vel, com_pp, axis_pp, n, cos_alpha,
                                                           sin_alpha, out);
  MPCD_LAUNCH_CHECK();
  return MPCD_OK;
}

int mpcd_stage_rotate_cells(const int64_t* cells, const double* vel, const double* com,
                            const double* axes, int64_t n, double cos_alpha, double sin_alpha,
                            double* out, void* stream) {
  clear_error();
  if (n <= 0) return MPCD_OK;
  k_rotate_cells<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(cells, vel, com, axes, n,
                                                                 cos_alpha, sin_alpha, out);
  MPCD_LAUNCH_CHECK();
  return MPCD_OK;
}

int mpcd_stage_wrap(const double* x, int64_t count, double box, double* out, void* stream) {
  clear_error();
  if (count <= 0) return MPCD_OK;
  k_wrap<<<grid_for(count, 256), 256, 0, as_stream(stream)>>>(x, count, box, out);
  MPCD_LAUNCH_CHECK();
  return MPCD_OK;
}

int mpcd_stage_stream_wrap(const double* pos, const double* vel, int64_t n, double dt,
                           const double box[3], double* out, void* stream) {
  clear_error();
  if (n <= 0) return MPCD_OK;
  k_stream_wrap<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(pos, vel, n, dt, box[0], box[1],
                                                                box[2], out);
  MPCD_LAUNCH_CHECK();
  return MPCD_OK;
}

int mpcd_stage_cell_drift(const double* before, const double* after, int64_t n_cells, double* out,
                          void* stream) {
  clear_error();
  cudaStream_t st = as_stream(stream);
  *out = 0.0;
  if (n_cells <= 0) return MPCD_OK;
  void* tmp = nullptr;
  MPCD_CUDA(cudaMallocAsync(&tmp, 16, st));
  MPCD_CUDA(cudaMemsetAsync(tmp, 0, 16, st));
  unsigned long long* bits = static_cast<unsigned long long*>(tmp);
  uint32_t* any = reinterpret_cast<uint32_t*>(bits + 1);
  k_cell_drift<<<grid_for(n_cells, 256), 256, 0, st>>>(before, after, n_cells, bits, any);
  MPCD_LAUNCH_CHECK();
  unsigned long long h[2];
  MPCD_CUDA(cudaMemcpyAsync(h, tmp, 16, cudaMemcpyDeviceToHost, st));
  MPCD_CUDA(cudaFreeAsync(tmp, st));
  MPCD_CUDA(cudaStreamSynchronize(st));
  double v;
  memcpy(&v, &h[0], sizeof(v));
  *out = v;
  return MPCD_OK;
}

}  // extern "C"
