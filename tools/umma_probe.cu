// Probe of the sm_100a primitives used by K3 (built and run on the B200 by hand):
//   1. SS  MMA  M128 N64  K64   A smem K-major SW128 (manual swizzle), B smem K-major SW128 (TMA)
//   2. TS  MMA  M128 N64  K64   A in TMEM (tcgen05.st, bf16 pairs per column), B as in 1
//   3. TS  MMA  M128 N256 K16   A in TMEM, B smem MN-major SW128: 4 TMA boxes of [16 rows x 64 cols]
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2508_15881_b200/csrc tools/umma_probe.cu -o /tmp/umma_probe
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "sm100.cuh"

using namespace tpla::sm100;

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e = (x);                                                              \
    if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1); } \
  } while (0)

static uint16_t f2b(float f) { uint32_t u; memcpy(&u, &f, 4); return uint16_t((u + 0x7FFF + ((u >> 16) & 1)) >> 16); }
static float b2f(uint16_t b) { uint32_t u = uint32_t(b) << 16; float f; memcpy(&f, &u, 4); return f; }

// A: [128][64] bf16 row-major (global). Bk: [64][64] (N x K) row-major. V: [16][256] (K x N) row-major.
__global__ void probe_kernel(const uint16_t* A, const __grid_constant__ CUtensorMap mapB,
                             const __grid_constant__ CUtensorMap mapV, float* D1, float* D2, float* D3) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;               // 128 rows x 128 B = 16 KB
  uint8_t* sB = smem + 16384;       // 64 rows x 128 B = 8 KB
  uint8_t* sV = smem + 24576;       // 4 boxes x 16 rows x 128 B = 8 KB
  __shared__ uint64_t bar_tma, bar_mma;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // A -> smem, K-major SW128 (chunk c of row r at c ^ (r & 7))
  for (int i = tid; i < 128 * 8; i += blockDim.x) {
    int r = i >> 3, c = i & 7;
    *reinterpret_cast<uint4*>(sA + r * 128 + ((c ^ (r & 7)) << 4)) = *reinterpret_cast<const uint4*>(A + r * 64 + c * 8);
  }
  fence_proxy_async_smem();
  if (tid == 0) {
    mbar_init(&bar_tma, 1);
    mbar_init(&bar_mma, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tmem_base;

  if (tid == 0) {
    mbar_arrive_expect_tx(&bar_tma, 8192 + 8192);
    tma_load_2d(sB, &mapB, 0, 0, &bar_tma, kEvictNormal);
    for (int j = 0; j < 4; ++j) tma_load_2d(sV + j * 2048, &mapV, j * 64, 0, &bar_tma, kEvictNormal);
  }
  // A -> TMEM columns [384, 416): thread t (warp quadrant) writes row t, 32 columns = 64 bf16
  {
    uint32_t r[32];
    int row = (warp & 3) * 32 + lane;
    for (int c = 0; c < 32; ++c) r[c] = *reinterpret_cast<const uint32_t*>(A + row * 64 + 2 * c);
    if (warp < 4) tmem_st32(tb + ((warp & 3) * 32u << 16) + 384, r);
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  mbar_wait(&bar_tma, 0);

  if (tid == 0) {
    const uint32_t id64 = idesc_bf16(128, 64, false, false);
    const uint32_t id256 = idesc_bf16(128, 256, false, true);
    for (int k = 0; k < 4; ++k)   // 1: SS into cols [0,64)
      mma_ss(tb + 0, desc_kmajor_sw128(smem_addr(sA) + 32 * k), desc_kmajor_sw128(smem_addr(sB) + 32 * k), id64, k > 0);
    for (int k = 0; k < 4; ++k)   // 2: TS into cols [64,128)
      mma_ts(tb + 64, tb + 384 + 8 * k, desc_kmajor_sw128(smem_addr(sB) + 32 * k), id64, k > 0);
    // 3: TS, A = first 16 K of the TMEM A (cols 384..391), B = V MN-major (LBO = box stride 2048 B)
    mma_ts(tb + 128, tb + 384, desc_mnmajor_sw128(smem_addr(sV), 2048), id256, 0);
    mma_commit(&bar_mma);
  }
  mbar_wait(&bar_mma, 0);
  tc_fence_after();
  if (warp < 4) {
    int row = warp * 32 + lane;
    uint32_t r[32];
    for (int c0 = 0; c0 < 64; c0 += 32) {
      tmem_ld32(tb + ((warp * 32u) << 16) + c0, r);
      tmem_ld_wait();
      for (int c = 0; c < 32; ++c) D1[row * 64 + c0 + c] = __uint_as_float(r[c]);
      tmem_ld32(tb + ((warp * 32u) << 16) + 64 + c0, r);
      tmem_ld_wait();
      for (int c = 0; c < 32; ++c) D2[row * 64 + c0 + c] = __uint_as_float(r[c]);
    }
    for (int c0 = 0; c0 < 256; c0 += 32) {
      tmem_ld32(tb + ((warp * 32u) << 16) + 128 + c0, r);
      tmem_ld_wait();
      for (int c = 0; c < 32; ++c) D3[row * 256 + c0 + c] = __uint_as_float(r[c]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tb);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static CUtensorMap make_map(EncodeFn enc, void* base, uint64_t cols, uint64_t rows, uint32_t box_c, uint32_t box_r) {
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {box_c, box_r};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", r); exit(1); }
  return m;
}

int main() {
  std::vector<uint16_t> A(128 * 64), Bk(64 * 64), V(16 * 256);
  srand(1);
  auto rnd = [] { return (rand() / float(RAND_MAX)) * 2.f - 1.f; };
  for (auto& x : A) x = f2b(rnd());
  for (auto& x : Bk) x = f2b(rnd());
  for (auto& x : V) x = f2b(rnd());
  uint16_t *dA, *dB, *dV;
  float *D1, *D2, *D3;
  CK(cudaMalloc(&dA, A.size() * 2)); CK(cudaMalloc(&dB, Bk.size() * 2)); CK(cudaMalloc(&dV, V.size() * 2));
  CK(cudaMalloc(&D1, 128 * 64 * 4)); CK(cudaMalloc(&D2, 128 * 64 * 4)); CK(cudaMalloc(&D3, 128 * 256 * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, Bk.data(), Bk.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dV, V.data(), V.size() * 2, cudaMemcpyHostToDevice));
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  EncodeFn enc = reinterpret_cast<EncodeFn>(fn);
  CUtensorMap mB = make_map(enc, dB, 64, 64, 64, 64);
  CUtensorMap mV = make_map(enc, dV, 256, 16, 64, 16);
  CK(cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
  probe_kernel<<<1, 128, 64 * 1024>>>(dA, mB, mV, D1, D2, D3);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<float> h1(128 * 64), h2(128 * 64), h3(128 * 256);
  CK(cudaMemcpy(h1.data(), D1, h1.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h2.data(), D2, h2.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h3.data(), D3, h3.size() * 4, cudaMemcpyDeviceToHost));
  double e1 = 0, e2 = 0, e3 = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 64; ++n) {
      double ref = 0;
      for (int k = 0; k < 64; ++k) ref += double(b2f(A[m * 64 + k])) * b2f(Bk[n * 64 + k]);
      e1 = fmax(e1, fabs(ref - h1[m * 64 + n]));
      e2 = fmax(e2, fabs(ref - h2[m * 64 + n]));
    }
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 256; ++n) {
      double ref = 0;
      for (int k = 0; k < 16; ++k) ref += double(b2f(A[m * 64 + k])) * b2f(V[k * 256 + n]);
      e3 = fmax(e3, fabs(ref - h3[m * 256 + n]));
    }
  printf("SS K-major        max abs err %.3e  (D[0][0] %f)\n", e1, h1[0]);
  printf("TS K-major        max abs err %.3e\n", e2);
  printf("TS MN-major N=256 max abs err %.3e\n", e3);
  bool ok = e1 < 1e-3 && e2 < 1e-3 && e3 < 1e-3;
  printf(ok ? "PROBE OK\n" : "PROBE FAIL\n");
  return ok ? 0 : 1;
}
