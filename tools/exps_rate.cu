// Throughput of K3's softmax exponential loop (the PP `exps` body: FFMA2 scale-subtract, ex2 on
// MUFU with a 1-in-kPoly share of pairs on the FMA-pipe cubic, FADD2 row sums, bf16x2 packs) for
// W warps per SMSP: cycles per 128-element row per warp.  Does one warp saturate the MUFU?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2508_15881_b200/csrc tools/exps_rate.cu -o tools/exps_rate
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "sm100.cuh"
using namespace tpla::sm100;

template <int kPoly>
__device__ __forceinline__ float exps128(const float* x, float m, uint32_t (&pw)[64]) {
  const uint64_t sc2 = f2_pack(0.1f, 0.1f), nm2 = f2_pack(-m, -m);
  uint64_t l01 = f2_pack(0.f, 0.f), l23 = f2_pack(0.f, 0.f);
#pragma unroll
  for (int j = 0; j < 64; j += 2) {
    float y0, y1, y2, y3;
    f2_unpack(ffma2(f2_pack(x[2 * j], x[2 * j + 1]), sc2, nm2), y0, y1);
    f2_unpack(ffma2(f2_pack(x[2 * j + 2], x[2 * j + 3]), sc2, nm2), y2, y3);
    const float p0 = ex2(y0), p1 = ex2(y1);
    float p2, p3;
    if (kPoly > 0 && (j / 2) % kPoly == 0) {
      ex2_poly2<true>(y2, y3, p2, p3);
    } else {
      p2 = ex2(y2);
      p3 = ex2(y3);
    }
    l01 = fadd2(l01, f2_pack(p0, p1));
    l23 = fadd2(l23, f2_pack(p2, p3));
    pw[j] = pack_bf16x2(p0, p1);
    pw[j + 1] = pack_bf16x2(p2, p3);
  }
  float a0, a1, a2, a3;
  f2_unpack(l01, a0, a1);
  f2_unpack(l23, a2, a3);
  return (a0 + a1) + (a2 + a3);
}

template <int kPoly>
__global__ void rate(float* out, long long* cyc, int iters) {
  float x[128];
#pragma unroll
  for (int i = 0; i < 128; ++i) x[i] = -0.01f * ((threadIdx.x + i) & 63);
  float acc = 0.f;
  uint32_t pk = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t pw[64];
    acc += exps128<kPoly>(x, acc * 1e-9f, pw);
#pragma unroll
    for (int i = 0; i < 64; ++i) pk ^= pw[i];
    x[it & 127] += 1e-7f * acc;
  }
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + pk;
  if (threadIdx.x % 32 == 0) cyc[blockIdx.x * 32 + threadIdx.x / 32] = t1 - t0;
}

template <int kPoly>
void run(int warps_per_smsp) {
  const int threads = 128 * warps_per_smsp, iters = 200;
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * threads * 4);
  cudaMalloc(&cyc, 148 * 32 * 8);
  rate<kPoly><<<148, threads>>>(out, cyc, iters);
  rate<kPoly><<<148, threads>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  long long h[32];
  cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
  double c = double(h[0]) / iters;
  // per SMSP: warps_per_smsp warps each did iters rows of 128 elements (32 lanes)
  printf("poly 1/%d, %d warp(s)/SMSP: %.0f cycles per row-iteration per warp -> %.0f cycles per 4096-exp tile per SMSP"
         " (%.2f exp/clk/SMSP)\n", kPoly ? 8 * kPoly / 2 : 0, warps_per_smsp, c, c / warps_per_smsp,
         4096.0 * warps_per_smsp / c);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {1, 2, 3, 4}) run<0>(w);
  for (int w : {1, 2, 3, 4}) run<2>(w);
  for (int w : {1, 2, 3}) run<4>(w);
  cudaError_t e = cudaGetLastError();
  printf("%s\n", e == cudaSuccess ? "EXPS OK" : cudaGetErrorString(e));
  return 0;
}
