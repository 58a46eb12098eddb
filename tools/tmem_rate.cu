// TMEM -> register load bandwidth probe: W warps (W/4 per lane quadrant) each issuing
// tcgen05.ld.sync.aligned.32x32b.x32 (4 KB per warp-instruction) NL times per wait, repeated.
// Reports bytes per SM clock.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2508_15881_b200/csrc tools/tmem_rate.cu -o tools/tmem_rate
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include "sm100.cuh"

using namespace tpla::sm100;

constexpr int kIters = 256;

template <int NL>
__global__ void ld_kernel(long long* cyc, float* sink) {
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tmem_base;
  const uint32_t lane_base = tb + (uint32_t((warp & 3) * 32) << 16);
  float acc = 0.f;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
    uint32_t v[NL][32];
#pragma unroll
    for (int q = 0; q < NL; ++q) tmem_ld32(lane_base + ((q * 32 + (warp >> 2) * 64) & 511), v[q]);
    tmem_ld_wait();
#pragma unroll
    for (int q = 0; q < NL; ++q) acc += __uint_as_float(v[q][q]);
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(tb);
}

template <int NL>
void run(int warps) {
  long long* d;
  float* sink;
  cudaMalloc(&d, 148 * sizeof(long long));
  cudaMalloc(&sink, 148 * 1024 * sizeof(float));
  ld_kernel<NL><<<148, warps * 32>>>(d, sink);
  ld_kernel<NL><<<148, warps * 32>>>(d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  const double bytes = double(warps) * kIters * NL * 4096;
  printf("warps %2d, %d x ld32 per wait: %7.1f B/clk/SM  (%.0f cyc per iteration)\n", warps, NL, bytes / avg, avg / kIters);
  cudaFree(d);
  cudaFree(sink);
}

int main() {
  run<1>(4);
  run<2>(4);
  run<2>(8);
  run<4>(8);
  run<2>(16);
  printf("TMEM OK\n");
  return 0;
}
