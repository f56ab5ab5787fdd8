// k_intpeak.cu — INT32 issue-rate microbenchmark (roofline denominator for
// the integer-bound enumeration path: "measure B200 INT32
// issue peak with a microbenchmark on the box").  Each thread runs 8
// independent chains of dependent IADD3/LOP3-class operations; the grid is
// 148 SMs x 4 CTAs x 512 threads so every SMSP has >= 16 warps in flight.
#include <cuda_runtime.h>
#include <cstdint>
#include "gvo_kernels.h"

namespace gvo {

constexpr int kIters = 4096;

__global__ void __launch_bounds__(512) k_int_peak(uint32_t seed, uint32_t* sink) {
  uint32_t a0 = threadIdx.x ^ seed, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  uint32_t a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
#pragma unroll 16
  for (int i = 0; i < kIters; ++i) {
    // 2 int ops per chain per iteration (add, xor) -> 16 per iteration
    a0 = (a0 + 0x9e3779b9u) ^ a1; a1 = (a1 + 0x7f4a7c15u) ^ a2;
    a2 = (a2 + 0x85ebca6bu) ^ a3; a3 = (a3 + 0xc2b2ae35u) ^ a4;
    a4 = (a4 + 0x27d4eb2fu) ^ a5; a5 = (a5 + 0x165667b1u) ^ a6;
    a6 = (a6 + 0xd3a2646cu) ^ a7; a7 = (a7 + 0xfd7046c5u) ^ a0;
  }
  const uint32_t r = a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7;
  if (r == 0x12345678u) sink[0] = r;
}

int launch_int_peak(int n_sm, cudaStream_t st, double* ops_per_s) {
  uint32_t* sink = nullptr;
  if (cudaMalloc(&sink, 4) != cudaSuccess) return 1;
  const int blocks = n_sm * 4, threads = 512;
  k_int_peak<<<blocks, threads, 0, st>>>(1u, sink);  // warm-up
  cudaEvent_t b, e;
  cudaEventCreate(&b);
  cudaEventCreate(&e);
  cudaEventRecord(b, st);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) k_int_peak<<<blocks, threads, 0, st>>>(2u + r, sink);
  cudaEventRecord(e, st);
  cudaEventSynchronize(e);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, b, e);
  cudaEventDestroy(b);
  cudaEventDestroy(e);
  cudaFree(sink);
  const double ops = (double)reps * blocks * threads * (double)kIters * 16.0;
  *ops_per_s = ops / (ms * 1e-3);
  return cudaGetLastError() != cudaSuccess;
}

}  // namespace gvo
