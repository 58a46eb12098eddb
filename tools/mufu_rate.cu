// MUFU.EX2 throughput probe: ex2.approx.ftz.f32 per clock per SM (and FFMA for reference),
// 148 CTAs x W warps, 8 independent chains per thread.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tools/mufu_rate.cu -o tools/mufu_rate
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

constexpr int kIters = 4096;

template <int OP>
__global__ void rate_kernel(float* out, long long* cyc) {
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
      else if (OP == 1) asm volatile("fma.rn.f32 %0, %0, 0.999, -0.001;" : "+f"(v[i]));
      else if (OP == 2) {   // ex2.approx.f16x2: two exponentials per instruction
        uint32_t u = __float_as_uint(v[i]);
        asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(u));
        v[i] = __uint_as_float(u);
      } else if (OP == 4) { // cvt.rn.bf16x2.f32 (F2FP.BF16.F32.PACK_AB): is it on the MUFU pipe?
        uint32_t u;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u) : "f"(v[i]), "f"(v[(i + 1) & 7]));
        v[i] = __uint_as_float(u) * 0.5f;
      } else if (OP == 5) { // one ex2 + one cvt per element (the softmax's mix)
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
        uint32_t u;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u) : "f"(v[i]), "f"(v[(i + 3) & 7]));
        v[(i + 5) & 7] += __uint_as_float(u);
      } else if (OP == 6) { // fmax only
        asm volatile("max.f32 %0, %0, %1;" : "+f"(v[i]) : "f"(v[(i + 1) & 7]));
      } else {              // ex2.approx.ftz.bf16x2
        uint32_t u = __float_as_uint(v[i]);
        asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(u));
        v[i] = __uint_as_float(u);
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int threads) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * threads * sizeof(float));
  cudaMalloc(&cyc, 148 * sizeof(long long));
  rate_kernel<OP><<<148, threads>>>(out, cyc);
  rate_kernel<OP><<<148, threads>>>(out, cyc);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  const double ops = double(threads) * kIters * 8;
  printf("%-10s threads %4d: %6.2f ops/clk/SM\n", name, threads, ops / avg);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int t : {128, 256, 512, 1024}) run<0>("ex2", t);
  for (int t : {128, 256, 1024}) run<1>("ffma", t);
  for (int t : {256, 1024}) run<2>("ex2.f16x2 (instr)", t);
  for (int t : {256, 1024}) run<3>("ex2.bf16x2 (instr)", t);
  for (int t : {256, 1024}) run<4>("cvt.bf16x2 (instr)", t);
  for (int t : {256, 1024}) run<5>("ex2+cvt (pairs)", t);
  for (int t : {256, 1024}) run<6>("fmax", t);
  printf("MUFU OK\n");
  return 0;
}
