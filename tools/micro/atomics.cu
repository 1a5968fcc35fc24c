// Micro-benchmark: throughput of the slot-claim pattern of k_step on B200.
// 167.8 M atomicAdd on a 16.8 M-entry u32 count array (10 per cell), with
// the result used (ATOM) or not (RED), cell order clustered like k_step's
// (a warp's lanes hit ~3 consecutive cells) or hashed (random cells).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atomics atomics.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

template <bool RET, bool HASH>
__global__ void k(uint32_t* cnt, uint32_t C, uint64_t n, uint32_t* sink) {
  uint32_t acc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c = HASH ? hash32((uint32_t)i) % C : (uint32_t)(i / 10) % C;
    if (RET) acc += atomicAdd(&cnt[c], 1u);
    else atomicAdd(&cnt[c], 1u);
  }
  if (RET && acc == 0xFFFFFFFFu) *sink = acc;
}

template <bool RET, bool HASH>
float run(uint32_t* cnt, uint32_t C, uint64_t n, uint32_t* sink) {
  cudaMemset(cnt, 0, sizeof(uint32_t) * C);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  k<RET, HASH><<<148 * 16, 256>>>(cnt, C, n, sink);
  cudaEventRecord(a);
  k<RET, HASH><<<148 * 16, 256>>>(cnt, C, n, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0; cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  const uint32_t C = 1u << 24;
  const uint64_t n = 10ull * C;
  uint32_t *cnt, *sink;
  cudaMalloc(&cnt, sizeof(uint32_t) * C);
  cudaMalloc(&sink, 4);
  printf("clustered ATOM %.3f ms\n", run<true, false>(cnt, C, n, sink));
  printf("clustered RED  %.3f ms\n", run<false, false>(cnt, C, n, sink));
  printf("hashed    ATOM %.3f ms\n", run<true, true>(cnt, C, n, sink));
  printf("hashed    RED  %.3f ms\n", run<false, true>(cnt, C, n, sink));
  printf("(%llu atomics on %u counters)\n", (unsigned long long)n, C);
  return 0;
}
