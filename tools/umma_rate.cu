// Throughput probe of tcgen05.mma kind::f16 shapes (one CTA per SM, one elected issuer):
// cycles per MMA instruction and the implied dense bf16 rate for the shapes K3 uses and the
// alternatives (A from smem = SS, A from TMEM = TS; N = 64 / 128 / 256).  Operand contents are
// irrelevant (zeros); the point is the issue/execute rate of back-to-back MMAs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2508_15881_b200/csrc tools/umma_rate.cu -o /tmp/umma_rate
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include "sm100.cuh"

using namespace tpla::sm100;

constexpr int kIters = 4096;

template <int N, bool TS, bool B_MN>
__global__ void rate_kernel(long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tmem_base;
  if (warp == 1) {
    constexpr uint32_t idesc = idesc_bf16(128, N, false, B_MN);
    constexpr uint32_t hi = desc_sw128_hi(1024);
    const uint64_t da = make_desc(smem_addr(smem), 16, hi);
    const uint64_t db = make_desc(smem_addr(smem + 16384), B_MN ? 8192 : 16, hi);
    long long t0 = 0;
    if (elect_one()) {
      t0 = clock64();
      for (int it = 0; it < kIters; ++it) {
        const uint32_t d = tb;   // one accumulator chain, as in a GEMM k-loop
        if (TS) mma_ts(d, tb + 256 + (it & 3) * 8, db + uint64_t((it & 3) * 2), idesc, 1u);
        else mma_ss(d, da + uint64_t((it & 3) * 2), db + uint64_t((it & 3) * 2), idesc, 1u);
      }
      mma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    if (elect_one()) cyc[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(tb);
}

template <int N, bool TS, bool B_MN>
void run(const char* name, int n_cta) {
  long long* d;
  cudaMalloc(&d, n_cta * sizeof(long long));
  auto k = rate_kernel<N, TS, B_MN>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024 + 1024);
  k<<<n_cta, 128, 66 * 1024 + 1024>>>(d);   // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<n_cta, 128, 66 * 1024 + 1024>>>(d);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(err)); exit(1); }
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[148];
  cudaMemcpy(h, d, n_cta * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < n_cta; ++i) avg += h[i];
  avg /= n_cta;
  const double flops = 2.0 * 128 * N * 16 * kIters * n_cta;
  printf("%-22s N=%3d  %6.1f cyc/mma (floor %3d)  %7.1f TFLOP/s (event %.1f us)\n", name, N, avg / kIters,
         128 * N / 256, flops / (ms * 1e-3) / 1e12, ms * 1e3);
  cudaFree(d);
}


// K3-like per-tile issue sequence: QK = NQ TS (K-major, N=64) + 4 SS (N=64) into S, commit;
// PV = 4 TS (MN-major, N=NPV) into O, COMMITS commits.  Reports cycles per tile.
template <int NQ, int NPV, int COMMITS, int FENCE = 0, int NQN = 64, int NPVK = 4, int BG = 0>
__global__ void tile_kernel(long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tmem_base;
  constexpr int kTiles = 512;
  if (warp == 1) {
    constexpr uint32_t id_qk = idesc_bf16(128, NQN, false, false);
    constexpr uint32_t id_pv = idesc_bf16(128, NPV, false, true);
    constexpr uint32_t hi = desc_sw128_hi(1024);
    const uint64_t da = make_desc(smem_addr(smem), 16, hi);
    const uint64_t db = make_desc(smem_addr(smem + 16384), 16, hi);
    const uint64_t dv = make_desc(smem_addr(smem + 16384), 8192, hi);
    long long t0 = 0;
    if (elect_one()) {
      t0 = clock64();
      for (int it = 0; it < kTiles; ++it) {
        const uint32_t s_t = tb + 256 + (it & 1) * (NQN == 64 ? 64 : 0);   // S buffer(s) (cols 256..383)
        if (FENCE & 1) tc_fence_after();
        if (FENCE & 4) { mbar_wait(&bar[3], 1); tc_fence_after(); }   // completed-phase wait (returns at once)
        if (FENCE & 8) mbar_wait(&bar[3], 1);
        for (int kk = 0; kk < NQ; ++kk) mma_ts(s_t, tb + 384 + (kk & 7) * 8, db + uint64_t(kk * 2), id_qk, kk > 0);
        for (int kk = 0; kk < 4; ++kk) mma_ss(s_t, da + uint64_t(kk * 2), db + uint64_t(kk * 2), id_qk, 1u);
        if (COMMITS > 0) mma_commit(&bar[0]);
        if (FENCE & 2) tc_fence_after();
        for (int kk = 0; kk < NPVK; ++kk) mma_ts(tb, tb + 448 + (kk & 3) * 8, dv + uint64_t((kk & 3) * 128), id_pv, 1u);
        if (COMMITS > 1) { mma_commit(&bar[1]); mma_commit(&bar[2]); }
      }
      mma_commit(&bar[3]);     // completes after every MMA issued before it
    }
    __syncwarp();
    mbar_wait(&bar[3], 0);
    if (elect_one()) cyc[blockIdx.x] = (clock64() - t0) / kTiles;
  } else if (BG && warp >= 2) {
    // background: MUFU (BG=1) or FFMA (BG=2) streams on the other warps for ~the same duration
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = -0.001f * (threadIdx.x + i);
    for (int it = 0; it < kTiles * (NQN == 64 ? 2 : 4); ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (BG == 1) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
        else asm volatile("fma.rn.f32 %0, %0, 0.999, -0.001;" : "+f"(v[i]));
      }
    }
    if (v[0] == 1234.f) cyc[0] = 0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(tb);
}

template <int NQ, int NPV, int COMMITS, int FENCE = 0, int NQN = 64, int NPVK = 4, int BG = 0>
void run_tile(const char* name) {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  auto k = tile_kernel<NQ, NPV, COMMITS, FENCE, NQN, NPVK, BG>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024 + 1024);
  k<<<148, BG ? 384 : 128, 66 * 1024 + 1024>>>(d);
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(err)); exit(1); }
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  printf("%-34s %6.0f cyc/tile (floor %d)\n", name, avg / 148, NQ * NQN / 2 + 4 * (NQN == 64 ? 48 : NQN / 2) + NPVK * (128 * NPV / 256));
  cudaFree(d);
}

// Faithful K3 (W_lat = 64, 128-token tile) TMEM dataflow: O cols [0,64), Q' [64,96), S0 [128,256),
// S1 [256,384).  Issue order QK(g) -> S[g&1] (A = Q' TMEM, + SS rope), then PV(g-1) with
// A = P(g-1) aliased in S[(g-1)&1] (RAW on the TMEM written by QK(g-1)), accumulate into O.
template <int ALIAS>
__global__ void k3flow_kernel(long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tmem_base;
  constexpr int kTiles = 512;
  if (warp == 1) {
    constexpr uint32_t id_qk = idesc_bf16(128, 128, false, false);
    constexpr uint32_t id_pv = idesc_bf16(128, 64, false, true);
    constexpr uint32_t hi = desc_sw128_hi(1024);
    const uint64_t da = make_desc(smem_addr(smem), 16, hi);
    const uint64_t db = make_desc(smem_addr(smem + 16384), 16, hi);
    const uint64_t dv = make_desc(smem_addr(smem + 16384), 16384, hi);
    long long t0 = 0;
    if (elect_one()) {
      t0 = clock64();
      for (int g = 0; g <= kTiles; ++g) {
        if (g < kTiles) {
          const uint32_t s_t = tb + 128 + (g & 1) * 128;
          for (int kk = 0; kk < 4; ++kk) mma_ts(s_t, tb + 64 + kk * 8, db + uint64_t(kk * 2), id_qk, kk > 0);
          for (int kk = 0; kk < 4; ++kk) mma_ss(s_t, da + uint64_t(kk * 2), db + uint64_t(kk * 2), id_qk, 1u);
        }
        if (g > 0) {
          const uint32_t p_t = ALIAS ? tb + 128 + ((g - 1) & 1) * 128 : tb + 448;
          for (int kk = 0; kk < 8; ++kk) mma_ts(tb, p_t + kk * 8, dv + uint64_t(kk * 128), id_pv, 1u);
        }
      }
      mma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    if (elect_one()) cyc[blockIdx.x] = (clock64() - t0) / kTiles;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(tb);
}

template <int ALIAS>
void run_k3flow(const char* name) {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  auto k = k3flow_kernel<ALIAS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024 + 1024);
  k<<<148, 128, 66 * 1024 + 1024>>>(d);
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(err)); exit(1); }
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  printf("%-34s %6.0f cyc/tile (floor 768)\n", name, avg / 148);
  cudaFree(d);
}

// Does a commit fire while its issuing thread is blocked in an mbarrier wait?  Warp 1 issues 8
// MMAs (~512 cycles) + commit(barA), then waits on barB, which warp 2 arrives DELAY cycles after
// the start; warp 3 records when it observes barA.
template <int DELAY>
__global__ void commit_kernel(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t barA, barB;
  __shared__ uint32_t tmem_base;
  __shared__ long long t_start;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&barA, 1); mbar_init(&barB, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tmem_base;
  if (threadIdx.x == 0) t_start = clock64();
  __syncthreads();
  const long long t0 = t_start;
  if (warp == 1) {
    constexpr uint32_t id_qk = idesc_bf16(128, 128, false, false);
    constexpr uint32_t hi = desc_sw128_hi(1024);
    const uint64_t da = make_desc(smem_addr(smem), 16, hi);
    const uint64_t db = make_desc(smem_addr(smem + 16384), 16, hi);
    if (elect_one()) {
      for (int kk = 0; kk < 4; ++kk) mma_ts(tb + 128, tb + 64 + kk * 8, db + uint64_t(kk * 2), id_qk, kk > 0);
      for (int kk = 0; kk < 4; ++kk) mma_ss(tb + 128, da + uint64_t(kk * 2), db + uint64_t(kk * 2), id_qk, 1u);
      mma_commit(&barA);
      out[blockIdx.x * 4 + 0] = clock64() - t0;
    }
    __syncwarp();
    mbar_wait(&barB, 0);
    if (lane == 0) out[blockIdx.x * 4 + 1] = clock64() - t0;
  } else if (warp == 2) {
    while (clock64() - t0 < DELAY) { }
    if (lane == 0) mbar_arrive(&barB);
  } else if (warp == 3) {
    mbar_wait(&barA, 0);
    if (lane == 0) out[blockIdx.x * 4 + 2] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(tb);
}

template <int DELAY>
void run_commit() {
  long long* d;
  cudaMalloc(&d, 148 * 4 * sizeof(long long));
  auto k = commit_kernel<DELAY>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024 + 1024);
  k<<<148, 128, 66 * 1024 + 1024>>>(d);
  k<<<148, 128, 66 * 1024 + 1024>>>(d);
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) { printf("commit: %s\n", cudaGetErrorString(err)); exit(1); }
  long long h[148 * 4];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("commit probe DELAY %6d: issued %5lld  barA seen %5lld  barB seen %5lld (cycles, CTA 0)\n", DELAY, h[0], h[2], h[1]);
  cudaFree(d);
}

int main() {
  int n = 148;
  run<64, false, false>("SS K-major", n);
  run<64, true, false>("TS K-major", n);
  run<128, false, false>("SS K-major", n);
  run<128, true, false>("TS K-major", n);
  run<256, false, false>("SS K-major", n);
  run<256, true, false>("TS K-major", n);
  run<256, true, true>("TS MN-major (PV)", n);
  run<128, true, true>("TS MN-major", n);
  run<64, true, false>("TS K-major 1 CTA", 1);
  run<256, true, true>("TS MN-major 1 CTA", 1);
  run_tile<4, 64, 0>("tile c3-like, no commits");
  run_tile<4, 64, 1>("tile c3-like, 1 commit");
  run_tile<4, 64, 2>("tile c3-like, 3 commits");
  run_tile<16, 256, 0>("tile c1-like, no commits");
  run_tile<16, 256, 2>("tile c1-like, 3 commits");
  run_tile<4, 64, 2, 1>("tile c3-like, fence before QK");
  run_tile<4, 64, 2, 3>("tile c3-like, fence before QK+PV");
  run_tile<4, 64, 2, 4>("tile c3-like, mbar wait+fence");
  run_tile<16, 256, 2, 3>("tile c1-like, fence before QK+PV");
  run_tile<4, 64, 2, 8>("tile c3-like, mbar wait only");
  run_tile<16, 256, 2, 4>("tile c1-like, mbar wait+fence");
  run_tile<16, 256, 2, 8>("tile c1-like, mbar wait only");
  run_tile<4, 64, 2, 0, 128, 8>("tile c3 TT=128");
  run_tile<4, 64, 2, 4, 128, 8>("tile c3 TT=128, mbar wait+fence");
  run_tile<4, 64, 2, 0, 128, 8, 1>("tile c3 TT=128 + MUFU load");
  run_tile<4, 64, 2, 0, 128, 8, 2>("tile c3 TT=128 + FFMA load");
  run_tile<16, 256, 2, 0, 64, 4, 1>("tile c1 + MUFU load");
  run_k3flow<0>("k3 flow, P separate");
  run_k3flow<1>("k3 flow, P aliased in S");
  run_commit<0>();
  run_commit<3000>();
  run_commit<20000>();
  printf("RATE OK\n");
  return 0;
}
