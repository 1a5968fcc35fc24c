// mpcd_internal.h -- shared helpers of libmpcd (error state, scan, launch).
#pragma once
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>

#include <type_traits>

#include "mpcd.h"
#include "mpcd_math.cuh"

namespace mpcd {

int fail(int code, const char* fmt, ...);
void clear_error();

#define MPCD_CUDA(call)                                                                      \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      return ::mpcd::fail(MPCD_ERR_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_),   \
                          __FILE__, __LINE__);                                               \
  } while (0)

#define MPCD_LAUNCH_CHECK() MPCD_CUDA(cudaGetLastError())

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline unsigned grid_for(int64_t n, int block, int64_t cap = 148LL * 64) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

// Single-pass exclusive scan (decoupled look-back) of a u32 array whose total
// fits in 32 bits.  `zero_input` clears the input after reading it (the
// engine's histogram is reused next step).  OutT is uint32_t or int64_t.
struct ScanState {
  uint64_t* tile_flags = nullptr;       // one 64-bit word per tile
  unsigned long long* counter = nullptr;  // dynamic tile ticket
  int64_t max_tiles = 0;
  uint64_t epoch = 0;                   // last epoch used (flags carry it)
  unsigned long long ticket = 0;        // device counter value before the next call
  int init(int64_t max_elems);
  void release();
};

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;

int scan_u32(ScanState& st, uint32_t* in, uint32_t* out_u32, int64_t* out_i64, int64_t count,
             bool zero_input, cudaStream_t stream);

}  // namespace mpcd
