// K9 — the prefill's dense GEMMs: the per-head key / value up-projections k = ĉ W^UK_h,
// v = ĉ W^UV_h and the output projection y = concat_h O_h W^O over all L prompt rows.
//
//   out[t, n] = Σ_k X[t, k] · Wt[n, k]        X: [L, K] bf16 activations (row stride ld_x),
//                                             Wt: blocked K-major weights [ceil(N/128)][K/64][128][64]
//
// One CTA per [256 weight rows x 256 tokens] output tile, the whole K loop: two M = 128 MMAs (the two
// weight row tiles, swap-AB: D[128 x 256] fp32 each, the 512 TMEM columns) share each [256 x 64]
// activation box, so a k-step moves 64 KB (two 16 KB weight blocks + the box) for 8.4 MFLOP — with one
// row tile per CTA (48 KB for 4.2 MFLOP) the kernel was bound by the L2 -> SM operand traffic
// (measured ~512 TFLOP/s).  TMA streams the operands through a 3-stage mbarrier ring; one thread
// issues tcgen05.mma; the epilogue (8 warps: TMEM lane quadrant x row tile, thread = weight row)
// writes out[t, n] token column by token column, 128 contiguous bytes per warp (fp32 y, =/+=, and/or
// a bf16 copy).  Unlike the decode's weight-stream K5 (split-K over a huge K, a few rows), nothing is
// split over K here: no partials, no reduce pass.  CTAs sharing a weight tile run back to back
// (token tile fastest), so each weight block comes from HBM once and from L2 for the rest.
//
// Warp roles (384 threads): w0 TMA, w1 MMA, w2 TMEM allocator, w4-w11 epilogue.
#include <cuda.h>
#include <stdlib.h>

#include "common.cuh"
#include "internal.h"
#include "sm100.cuh"

namespace tpla {
namespace {

using namespace sm100;

constexpr int kM = 128, kN = 256, kK = 64;      // kN: the largest token tile (runtime a.tn <= kN, 32 | tn)
constexpr int kMT = 2;                        // weight row tiles per CTA (MMA M = 128 each)
constexpr int kWBytes = kM * 128;             // 16 KB per row tile
constexpr int kXBytes = kN * 128;             // 32 KB
constexpr int kStage = kMT * kWBytes + kXBytes;
constexpr int kStages = 3;
constexpr int kSmem = 1024 + kStages * kStage;

struct G9Args {
  float* y;           // [L, N] fp32 or null
  uint16_t* out;      // [L, N] bf16 or null
  int N, L, k_steps, n_tt, n_rt, accumulate;
  int tn;             // tokens per tile (MMA N): chosen per launch against the wave quantisation
};

__global__ void __launch_bounds__(384, 1)
gemm_tn_kernel(const __grid_constant__ CUtensorMap mw, const __grid_constant__ CUtensorMap mx,
               const __grid_constant__ CUtensorMap my, const __grid_constant__ CUtensorMap mo, G9Args a) {
  pdl_trigger();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[kStages], empty[kStages], acc_full;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rp = int(blockIdx.x) / a.n_tt, tt = int(blockIdx.x) % a.n_tt;   // row-tile pair, token tile
  const int n_mt = min(kMT, a.n_rt - rp * kMT);                            // (the last pair may be single)
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mw);
    tma_prefetch_desc(&mx);
    for (int i = 0; i < kStages; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    mbar_init(&acc_full, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<kMT * kN>(&tmem_base);
  pdl_wait();                                   // X (and y) come from the predecessors
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tmem_base;

  if (warp == 0) {
    if (elect_one()) {
      for (int ks = 0; ks < a.k_steps; ++ks) {
        const int st = ks % kStages;
        mbar_wait(&empty[st], ((ks / kStages) & 1) ^ 1);
        uint8_t* dst = smem + st * kStage;
        mbar_arrive_expect_tx(&full[st], n_mt * kWBytes + a.tn * 128);
        for (int m = 0; m < n_mt; ++m)
          tma_load_2d(dst + m * kWBytes, &mw, 0, ((rp * kMT + m) * a.k_steps + ks) * kM, &full[st], kEvictNormal);
        tma_load_2d(dst + kMT * kWBytes, &mx, ks * kK, tt * a.tn, &full[st], kEvictNormal);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    const uint32_t idesc = idesc_bf16(kM, a.tn, false, false);
    constexpr uint32_t hi_k = desc_sw128_hi(1024);
    const uint32_t s0 = smem_addr(smem);
    for (int ks = 0; ks < a.k_steps; ++ks) {
      const int st = ks % kStages;
      mbar_wait(&full[st], (ks / kStages) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint64_t db = make_desc(s0 + st * kStage + kMT * kWBytes, 16, hi_k);
        for (int m = 0; m < n_mt; ++m) {
          const uint64_t da = make_desc(s0 + st * kStage + m * kWBytes, 16, hi_k);
#pragma unroll
          for (int kk = 0; kk < kK / 16; ++kk)
            mma_ss(tb + m * kN, da + uint64_t(kk * 2), db + uint64_t(kk * 2), idesc, (ks == 0 && kk == 0) ? 0u : 1u);
        }
        mma_commit(&empty[st]);
        if (ks + 1 == a.k_steps) mma_commit(&acc_full);
      }
      __syncwarp();
    }
  } else if (warp >= 4 && (warp - 4) / 4 < n_mt) {
    const int q4 = warp & 3, m = (warp - 4) / 4;   // TMEM lane quadrant, row tile of the pair
    const int n = (rp * kMT + m) * kM + q4 * 32 + lane;   // weight row = output feature
    const uint32_t lane_base = tb + m * kN + (uint32_t(q4 * 32) << 16);
    mbar_wait(&acc_full, 0);
    tc_fence_after();
    // Through shared memory and TMA: per 32-token chunk the warp stages its [32 tokens x 32 features]
    // block (fp32 and / or bf16; the ring is free once acc_full fired) and one lane stores it with
    // cp.async.bulk.tensor (or reduce-adds it into y); out-of-range rows / columns are clipped by the
    // tensor maps.  (Per-thread 4-byte stores, three memory instructions per element with the
    // accumulate, made the epilogue as long as a K = 512 main loop.)
    const int wi = warp - 4;                     // 0..7
    float* stg = reinterpret_cast<float*>(smem) + wi * 2 * 1024;               // 2 x [32 x 32] fp32
    uint16_t* stg16 = reinterpret_cast<uint16_t*>(smem + 8 * 2 * 4096) + wi * 2 * 1024;   // 2 x [32 x 32] bf16
    const int n0 = (rp * kMT + m) * kM + q4 * 32;
#pragma unroll 1
    for (int c = 0; c < a.tn / 32; ++c) {
      uint32_t d[32];
      tmem_ld32(lane_base + 32 * c, d);
      tmem_ld_wait();
      if (lane == 0) bulk_wait_read<1>();        // this chunk's staging buffer (used two chunks ago) is read
      __syncwarp();
      float* bf = stg + (c & 1) * 1024;
      uint16_t* bh = stg16 + (c & 1) * 1024;
#pragma unroll
      for (int j = 0; j < 32; ++j) {             // row j = token, column lane = feature: conflict-free
        if (a.y) bf[j * 32 + lane] = __uint_as_float(d[j]);
        if (a.out && !(a.y && a.accumulate)) bh[j * 32 + lane] = f2bf(__uint_as_float(d[j]));
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        const int t0 = tt * a.tn + 32 * c;
        if (a.y) {
          if (a.accumulate) tma_reduce_add_2d(&my, n0, t0, bf);
          else tma_store_2d(&my, n0, t0, bf);
        }
        if (a.out && !(a.y && a.accumulate)) tma_store_2d(&mo, n0, t0, bh);
        bulk_commit();
      }
    }
    if (lane == 0) bulk_wait<0>();
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<kMT * kN>(tb);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

bool map2d(CUtensorMap* m, const void* base, long cols, long rows, long ld, int box_r, int box_c = kK,
           CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, int esize = 2,
           CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  }
  if (!fn) return false;
  cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(ld) * esize};
  cuuint32_t box[2] = {cuuint32_t(box_c), cuuint32_t(box_r)};
  cuuint32_t es[2] = {1, 1};
  return fn(m, dt, 2, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int sm_count9() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace

bool gemm_tn_supported(int N, int K) { return N >= 1 && K >= kK && K % kK == 0; }

// Token tile: the grid is (row-tile pairs) x (token tiles), one CTA per SM, so its time is set by the
// rounds ceil(tiles / #SMs) of one tile each.  A tile costs about (tokens + 96) token-units (the 96:
// epilogue and pipeline fill, fitted to the A/B below); pick the width (multiple of 32, >= 128) that
// minimises rounds x cost, larger on ties.  Measured (tools/prefill_bench.py, K9 per device, forced
// widths 256 / 224 / 192 / 160 / 128): 4K 518 / 478 / 527 / 503 / 638 µs, 1K 133 / 150 / 214 / 199 / 192;
// the rule picks 224 for the W^O GEMM at 4K (448 tiles of 256 = 4 rounds for 3.03 of work -> 532 of
// 224) and at 1K, 256 for the k / v up-projections.  TPLA_K9_TN forces one width (A/B).
static int pick_tn(int n_rp, int L) {
  static const int forced = getenv("TPLA_K9_TN") ? atoi(getenv("TPLA_K9_TN")) : 0;
  if (forced >= 32 && forced <= kN && forced % 32 == 0) return forced;
  const int sms = sm_count9();
  int best = kN;
  long best_cost = -1;
  for (int tn = kN; tn >= 128; tn -= 32) {
    const long tiles = long(n_rp) * ((L + tn - 1) / tn);
    const long cost = (tiles + sms - 1) / sms * (tn + 96);
    if (best_cost < 0 || cost < best_cost) { best_cost = cost; best = tn; }
  }
  return best;
}

cudaError_t launch_gemm_tn(const uint16_t* Wt, const uint16_t* X, long ld_x, int N, int K, int L, float* y,
                           bool accumulate, uint16_t* out, cudaStream_t s) {
  const int n_rt = (N + kM - 1) / kM, n_rp = (n_rt + kMT - 1) / kMT;
  const int tn = pick_tn(n_rp, L), n_tt = (L + tn - 1) / tn;
  if (y && accumulate && out) return cudaErrorInvalidValue;   // (the bf16 copy of an accumulated y: not here)
  CUtensorMap mw, mx, my{}, mo{};
  if (!map2d(&mw, Wt, kK, long(n_rt) * (K / kK) * kM, kK, kM) || !map2d(&mx, X, K, L, ld_x, tn))
    return cudaErrorInvalidValue;
  if (y && !map2d(&my, y, N, L, N, 32, 32, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, CU_TENSOR_MAP_SWIZZLE_NONE))
    return cudaErrorInvalidValue;
  if (out && !map2d(&mo, out, N, L, N, 32, 32, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, CU_TENSOR_MAP_SWIZZLE_NONE))
    return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  G9Args a{y, out, N, L, K / kK, n_tt, n_rt, accumulate ? 1 : 0, tn};
  KernelScope ks("K9_prefill_gemm", s);
  return launch_k(gemm_tn_kernel, n_rp * n_tt, 384, kSmem, s, mw, mx, my, mo, a);
}

}  // namespace tpla
