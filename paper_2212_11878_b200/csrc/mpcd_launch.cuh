// mpcd_launch.cuh -- host-side launch of the step kernels' compile-time
// variants.  Included by mpcd_engine.cu (declarations) and by the four
// mpcd_step_<mode>.cu translation units, each of which instantiates the
// 16 (UNIT, UMASS, DRIFT, COM) variants of one step mode.
#pragma once

#include <map>
#include <mutex>
#include <utility>

namespace mpcd {

// 64 compile-time variants, chosen at run time
struct Variant {
  bool unit, umass, drift, com;
  int mode;
};

int64_t launch_mode_binned(const StepArgs& A, int64_t nt, Variant v, int which, cudaStream_t st);
int64_t launch_mode_byid(const StepArgs& A, int64_t nt, Variant v, int which, cudaStream_t st);
int64_t launch_mode_multi(const StepArgs& A, int64_t nt, Variant v, int which, cudaStream_t st);
int64_t launch_mode_fused(const StepArgs& A, int64_t nt, Variant v, int which, cudaStream_t st);

constexpr int64_t kDenseGrid = 592;
#ifndef MPCD_FIXTC
#define MPCD_FIXTC 16
#endif

#ifdef MPCD_STEP_VARIANTS_ONLY
namespace {
// Resident CTAs per device for a persistent kernel, cached per (kernel, device).
int64_t resident_ctas(const void* kernel, int block, size_t smem) {
  static std::map<std::pair<const void*, int>, int64_t> cache;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  int dev = 0;
  cudaGetDevice(&dev);
  auto key = std::make_pair(kernel, dev);
  auto it = cache.find(key);
  if (it == cache.end()) {
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem);
    it = cache.emplace(key, (int64_t)std::max(per_sm, 1) * sms).first;
  }
  return it->second;
}

// Opt a kernel in to `smem` bytes of dynamic shared memory (once per size).
void allow_smem(const void* kernel, size_t smem) {
  static std::map<std::pair<const void*, int>, size_t> done;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  int dev = 0;
  cudaGetDevice(&dev);
  size_t& have = done[std::make_pair(kernel, dev)];
  if (have >= smem) return;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  have = smem;
}

// which == 0: the persistent tile kernel (returns its grid); which == 1: the
// dense-tile kernel (exits at once when k_step queued no tile).
template <bool UNIT, bool UMASS, bool DRIFT, bool COM, int MODE>
int64_t launch_variant(const StepArgs& A, int64_t ntiles, int which, cudaStream_t st) {
  if (which == 0) {
    // the common geometry (16 cells at ~10 particles per cell) compiled in,
    // any other read at run time
    auto kern = A.tc == MPCD_FIXTC ? k_step<UNIT, UMASS, DRIFT, COM, MODE, MPCD_FIXTC>
                                   : k_step<UNIT, UMASS, DRIFT, COM, MODE, 0>;
    const size_t smem = sizeof(StepSmem<DRIFT, MODE == kFused>);
    const int64_t grid =
        std::max<int64_t>(1, std::min<int64_t>(ntiles, resident_ctas((const void*)kern, kNTW, smem)));
    kern<<<(unsigned)grid, kNTW, smem, st>>>(A, ntiles);
    return grid;
  }
  auto dk = k_step_dense<UNIT, UMASS, DRIFT, COM, MODE>;
  const size_t dsmem = dense_smem_bytes(A.np_smem);
  allow_smem((const void*)dk, dsmem);
  dk<<<(unsigned)kDenseGrid, kNT, dsmem, st>>>(A);
  return kDenseGrid;
}

}  // namespace

template <int MODE>
int64_t launch_mode_t(const StepArgs& A, int64_t nt, Variant v, int which, cudaStream_t st) {
#ifdef MPCD_ONLY_MAIN
  // tuning builds (tools/build_variants.py): the unit-mass variant of the
  // binned and fused modes alone
  if constexpr (MODE == kBinned || MODE == kFused)
    return launch_variant<true, true, false, false, MODE>(A, nt, which, st);
  else return -1;
#else
#define MPCD_V(U, M, D, C) \
  if (v.unit == U && v.umass == M && v.drift == D && v.com == C) \
    return launch_variant<U, M, D, C, MODE>(A, nt, which, st);
  MPCD_V(true, true, false, false) MPCD_V(true, true, false, true)
  MPCD_V(true, true, true, false) MPCD_V(true, true, true, true)
  MPCD_V(true, false, false, false) MPCD_V(true, false, false, true)
  MPCD_V(true, false, true, false) MPCD_V(true, false, true, true)
  MPCD_V(false, true, false, false) MPCD_V(false, true, false, true)
  MPCD_V(false, true, true, false) MPCD_V(false, true, true, true)
  MPCD_V(false, false, false, false) MPCD_V(false, false, false, true)
  MPCD_V(false, false, true, false)
#undef MPCD_V
  return launch_variant<false, false, true, true, MODE>(A, nt, which, st);
#endif
}
#endif  // MPCD_STEP_VARIANTS_ONLY

}  // namespace mpcd
