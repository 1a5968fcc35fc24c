// mpcd_step_binned.cu -- the k_step / k_step_dense variants of step mode
// kBinned (one of four translation units compiled in parallel; see
// mpcd_launch.cuh).
#define MPCD_STEP_VARIANTS_ONLY 1
#include "mpcd_internal.h"
#include "mpcd_step.cuh"
#include "mpcd_launch.cuh"

namespace mpcd {

int64_t launch_mode_binned(const StepArgs& A, int64_t nt, Variant v, int which, cudaStream_t st) {
  return launch_mode_t<kBinned>(A, nt, v, which, st);
}

}  // namespace mpcd

#ifdef MPCD_TIMING
// Tuning builds only (-DMPCD_TIMING): per-phase clock64 sums of the k_step
// consumer warps of this translation unit's kernels (tools/phase_timing.py).
extern "C" int mpcd_debug_phase_cycles(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, mpcd::g_phase_cycles, sizeof(unsigned long long) * 10) !=
      cudaSuccess ||
      cudaMemcpyFromSymbol(out + 10, mpcd::g_prod_cycles, sizeof(unsigned long long) * 2) !=
      cudaSuccess)
    return MPCD_ERR_CUDA;
  if (reset) {
    unsigned long long z[10] = {0};
    cudaMemcpyToSymbol(mpcd::g_phase_cycles, z, sizeof(z));
    cudaMemcpyToSymbol(mpcd::g_prod_cycles, z, 2 * sizeof(unsigned long long));
  }
  return MPCD_OK;
}
#endif
