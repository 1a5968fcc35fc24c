// mpcd_scan.cu -- exclusive prefix sum of per-cell counts (the reference's
// np.cumsum of bin_count, collision.py:96-97) in one pass over HBM.
//
// Decoupled look-back: each CTA takes a 4096-element tile by ticket, scans it
// in registers + warp shuffles, publishes its aggregate, and lane-parallel
// looks back over predecessors' (epoch | status | value) words.  The epoch in
// each flag word makes the flag array reusable without a memset per call.
// Traffic: read 4 B + write 4 B (+4 B zeroing, engine only) per cell.
#include <stdarg.h>
#include <string>

#include "mpcd_internal.h"

namespace mpcd {

namespace {
thread_local std::string g_error;
}

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_error = buf;
  return code;
}

void clear_error() { g_error.clear(); }

const char* last_error() { return g_error.c_str(); }

constexpr uint64_t kStatusAgg = 1, kStatusIncl = 2;

__device__ __forceinline__ uint64_t flag_word(uint64_t epoch, uint64_t status, uint32_t v) {
  return (epoch << 34) | (status << 32) | (uint64_t)v;
}

template <typename OutT>
__global__ void __launch_bounds__(kScanThreads) k_scan(uint32_t* __restrict__ in,
                                                       OutT* __restrict__ out, int64_t count,
                                                       int zero_input, uint64_t* flags,
                                                       unsigned long long* counter, uint64_t epoch,
                                                       unsigned long long ticket_base) {
  __shared__ int64_t s_tile;
  __shared__ uint32_t s_warp[kScanThreads / 32];
  __shared__ uint32_t s_prefix;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  if (t == 0) s_tile = (int64_t)(atomicAdd(counter, 1ULL) - ticket_base);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t base = tile * kScanTile + (int64_t)t * kScanItems;

  uint32_t v[kScanItems];
  if (base + kScanItems <= count) {
    const uint4* p = reinterpret_cast<const uint4*>(in + base);
#pragma unroll
    for (int q = 0; q < kScanItems / 4; ++q) {
      uint4 w = p[q];
      v[4 * q] = w.x; v[4 * q + 1] = w.y; v[4 * q + 2] = w.z; v[4 * q + 3] = w.w;
    }
    if (zero_input) {
      uint4* pz = reinterpret_cast<uint4*>(in + base);
#pragma unroll
      for (int q = 0; q < kScanItems / 4; ++q) pz[q] = make_uint4(0, 0, 0, 0);
    }
  } else {
#pragma unroll
    for (int q = 0; q < kScanItems; ++q) {
      int64_t i = base + q;
      v[q] = (i < count) ? in[i] : 0u;
      if (zero_input && i < count) in[i] = 0u;
    }
  }
  uint32_t sum = 0;
#pragma unroll
  for (int q = 0; q < kScanItems; ++q) sum += v[q];
  // inclusive warp scan of per-thread sums
  uint32_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  uint32_t warp_excl = 0, total = 0;
#pragma unroll
  for (int w = 0; w < kScanThreads / 32; ++w) {
    uint32_t x = s_warp[w];
    if (w < warp) warp_excl += x;
    total += x;
  }
  uint32_t thread_excl = warp_excl + incl - sum;

  // publish + look back (warp 0)
  if (warp == 0) {
    volatile uint64_t* vf = flags;
    if (tile == 0) {
      if (lane == 0) {
        vf[0] = flag_word(epoch, kStatusIncl, total);
        s_prefix = 0;
      }
    } else {
      if (lane == 0) vf[tile] = flag_word(epoch, kStatusAgg, total);
      uint32_t excl = 0;
      int64_t idx = tile - 1;
      while (true) {
        int64_t j = idx - lane;
        uint64_t f;
        if (j >= 0) {
          do {
            f = vf[j];
          } while ((f >> 34) != epoch || ((f >> 32) & 3) == 0);
        } else {
          f = flag_word(epoch, kStatusIncl, 0);
        }
        uint32_t status = (uint32_t)((f >> 32) & 3);
        uint32_t val = (uint32_t)f;
        unsigned incl_mask = __ballot_sync(0xffffffffu, status == kStatusIncl);
        if (incl_mask) {
          int first = __ffs(incl_mask) - 1;
          uint32_t contrib = (lane <= first) ? val : 0u;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) contrib += __shfl_xor_sync(0xffffffffu, contrib, o);
          excl += contrib;
          break;
        }
        uint32_t contrib = val;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) contrib += __shfl_xor_sync(0xffffffffu, contrib, o);
        excl += contrib;
        idx -= 32;
      }
      if (lane == 0) {
        vf[tile] = flag_word(epoch, kStatusIncl, excl + total);
        s_prefix = excl;
      }
    }
  }
  __syncthreads();
  uint32_t run = s_prefix + thread_excl;
  if (base + kScanItems <= count && sizeof(OutT) == 4) {
    uint4* p = reinterpret_cast<uint4*>(out + base);
#pragma unroll
    for (int q = 0; q < kScanItems / 4; ++q) {
      uint4 w;
      w.x = run; run += v[4 * q];
      w.y = run; run += v[4 * q + 1];
      w.z = run; run += v[4 * q + 2];
      w.w = run; run += v[4 * q + 3];
      p[q] = w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < kScanItems; ++q) {
      int64_t i = base + q;
      if (i < count) out[i] = (OutT)run;
      run += v[q];
    }
  }
}

int ScanState::init(int64_t max_elems) {
  max_tiles = (max_elems + kScanTile - 1) / kScanTile;
  if (max_tiles < 1) max_tiles = 1;
  MPCD_CUDA(cudaMalloc(&tile_flags, sizeof(uint64_t) * max_tiles));
  MPCD_CUDA(cudaMemset(tile_flags, 0, sizeof(uint64_t) * max_tiles));
  MPCD_CUDA(cudaMalloc(&counter, sizeof(unsigned long long)));
  MPCD_CUDA(cudaMemset(counter, 0, sizeof(unsigned long long)));
  epoch = 0;
  return MPCD_OK;
}

void ScanState::release() {
  if (tile_flags) cudaFree(tile_flags);
  if (counter) cudaFree(counter);
  tile_flags = nullptr;
  counter = nullptr;
}

int scan_u32(ScanState& st, uint32_t* in, uint32_t* out_u32, int64_t* out_i64, int64_t count,
             bool zero_input, cudaStream_t stream) {
  if (count <= 0) return MPCD_OK;
  int64_t ntiles = (count + kScanTile - 1) / kScanTile;
  if (ntiles > st.max_tiles) return fail(MPCD_ERR_CAPACITY, "scan of %lld exceeds capacity", (long long)count);
  // Every launched CTA takes exactly one ticket, so the ticket counter
  // advances by ntiles per call (stream order); the epoch (monotonic, 30 bits)
  // invalidates the previous call's flag words without a memset.
  st.epoch += 1;
  unsigned long long base = st.ticket;
  st.ticket += (unsigned long long)ntiles;
  if (out_u32)
    k_scan<uint32_t><<<(unsigned)ntiles, kScanThreads, 0, stream>>>(
        in, out_u32, count, zero_input ? 1 : 0, st.tile_flags, st.counter, st.epoch, base);
  else
    k_scan<int64_t><<<(unsigned)ntiles, kScanThreads, 0, stream>>>(
        in, out_i64, count, zero_input ? 1 : 0, st.tile_flags, st.counter, st.epoch, base);
  MPCD_LAUNCH_CHECK();
  return MPCD_OK;
}

}  // namespace mpcd

extern "C" const char* mpcd_last_error(void) { return mpcd::last_error(); }
extern "C" const char* mpcd_version(void) { return "mpcd-b200 0.1.0 (sm_100a)"; }
