// mpcd_step_fused.cu -- the k_step / k_step_dense variants of step mode
// kFused (one of four translation units compiled in parallel; see
// mpcd_launch.cuh).
#define MPCD_STEP_VARIANTS_ONLY 1
#include "mpcd_internal.h"
#include "mpcd_step.cuh"
#include "mpcd_launch.cuh"

namespace mpcd {

int64_t launch_mode_fused(const StepArgs& A, int64_t nt, Variant v, int which, cudaStream_t st) {
  return launch_mode_t<kFused>(A, nt, v, which, st);
}

}  // namespace mpcd
