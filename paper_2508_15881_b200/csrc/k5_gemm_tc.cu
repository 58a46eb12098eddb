// K5b (Blackwell-native) — the W^O up-projection  Õ_j[b, n] = Σ_k v[b, k] · W^O_j[n, k]
// as a persistent, weight-streaming tcgen05 GEMM.
//
// M = batch is small (B <= 256) and W^O_j (D x H_loc·d_h bf16, 235 MB for DeepSeek-V3 at g = 2)
// is read exactly once, so the kernel is an HBM stream: TMA moves [128 weight rows x 64 k]
// tiles (SWIZZLE_128B) plus the matching [B x 64] slice of v through a deep mbarrier ring,
// and one elected thread issues tcgen05.mma with the WEIGHT rows as the MMA M dimension
// (swap-AB: D[128 x Bp] fp32 in TMEM), so the tensor pipe is idle most of the time.
// Work split: the (row tile, k-step) list is cut into equal contiguous ranges, one per CTA;
// a range is one or two row-tile segments whose partial sums go to a workspace buffer, and a
// small deterministic reduce kernel adds a row tile's (contiguous) segments into y (and writes
// the bf16 output when no all-reduce follows).  The first ring stages' weight blocks are
// requested before the PDL wait, under the previous kernel's tail.
//
// Warp roles (256 threads): w0 TMA, w1 MMA, w2 TMEM allocator, w4-w7 epilogue (TMEM lanes).
#include <cuda.h>
#include <nccl.h>
#include <nccl_device.h>

#include <algorithm>

#include "common.cuh"
#include "internal.h"
#include "sm100.cuh"

namespace tpla {
namespace {

using namespace sm100;

constexpr int kBK = 64;     // k per stage (one 128-byte swizzled row)
constexpr int kTM = 128;    // weight rows per tile (MMA M)

struct GArgs {
  float* part;        // [max_segs, B, 128] partial sums
  int32_t* meta;      // [n_tiles, 2] first / last segment id of each row tile
  int N, K, B, n_tiles, k_steps;
  int k_total, k0;    // K-slice: W^O k-steps [k0, k0 + k_steps) of k_total (v holds only the slice's columns)
};

template <int NP>
struct GCfg {
  static constexpr int A_BYTES = kTM * 128;            // 16 KB
  static constexpr int B_BYTES = NP * 128;
  static constexpr int STAGE = A_BYTES + B_BYTES;
#ifndef TPLA_K5_SMEM_KB
#define TPLA_K5_SMEM_KB 200
#endif
// Ring depth: at most 6 stages (A/B, tools/gpu_ab_k.sh: 6 / 8 / 10 / 11 stages of 20 KB at B <= 32 —
// K5 43.5 / 44.0 / 45.5 / 45.5 us per c1 step, 42.0 / 42.1 / 44.9 / 45.5 at batch 1; ncu cold 40.5 us
// at 8 against 43.0 at 10: ~120 KB in flight per SM already covers the HBM latency)
#ifndef TPLA_K5_MAX_NST
#define TPLA_K5_MAX_NST 6
#endif
  static constexpr int NST = std::min(TPLA_K5_MAX_NST, (TPLA_K5_SMEM_KB * 1024) / STAGE);
  static constexpr int SMEM = 1024 + NST * STAGE;
  static constexpr int TMEM_COLS = 2 * NP < 32 ? 32 : 2 * NP;
};

template <int NP>
__global__ void __launch_bounds__(256, 1)
skinny_tc_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, GArgs a) {
  pdl_trigger();
  using C = GCfg<NP>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[C::NST], empty[C::NST], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base;
  __shared__ int s_seg_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int U = a.n_tiles * a.k_steps;                 // < 2^31 / #SMs (checked on the host)
  const int c = blockIdx.x, n_cta = gridDim.x;
  const int lo = c * U / n_cta, hi = (c + 1) * U / n_cta;
  if (warp == 3) {
    // segments before this CTA (a range [l, h) touches row tiles l/ks .. (h-1)/ks), lane-parallel
    int n = 0;
    for (int cc = lane; cc < c; cc += 32) {
      const int l = cc * U / n_cta, h = (cc + 1) * U / n_cta;
      if (l < h) n += (h - 1) / a.k_steps - l / a.k_steps + 1;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
    if (lane == 0) s_seg_base = n;
  }

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mapA);
    tma_prefetch_desc(&mapB);
    for (int i = 0; i < C::NST; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&acc_full[i], 1); mbar_init(&acc_empty[i], 128); }
    fence_barrier_init();
    // W^O does not depend on the predecessors: fill the ring's weight halves now, under the
    // previous kernel's tail (PDL); the v halves follow after the wait
    for (int i = 0; i < C::NST && lo + i < hi; ++i) {
      const int u = lo + i;
      mbar_arrive_expect_tx(&full[i], C::STAGE);
      const int rt0 = u / a.k_steps, ks0 = u % a.k_steps;
      tma_load_2d(smem + i * C::STAGE, &mapA, 0, (rt0 * a.k_total + a.k0 + ks0) * kTM, &full[i], kEvictFirst);
    }
  }
  if (warp == 2) tmem_alloc<C::TMEM_COLS>(&tmem_base);
  pdl_wait();   // v (and y) come from the predecessors
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tmem_base;
  const int seg_base = s_seg_base;

  if (warp == 0) {
    // ---- TMA producer
    int g = 0, rt = lo / a.k_steps, ks = lo % a.k_steps;
    for (int u = lo; u < hi; ++u, ++g) {
      const int st = g % C::NST;
      if (g >= C::NST) mbar_wait(&empty[st], ((g / C::NST) & 1) ^ 1);
      if (elect_one()) {
        uint8_t* dst = smem + st * C::STAGE;
        if (g >= C::NST) {   // (the first NST weight blocks were issued before the PDL wait)
          mbar_arrive_expect_tx(&full[st], C::STAGE);
          // weights (blocked layout: tile (rt, ks) is one contiguous 16 KB block), read once
          tma_load_2d(dst, &mapA, 0, (rt * a.k_total + a.k0 + ks) * kTM, &full[st], kEvictFirst);
        }
        tma_load_2d(dst + C::A_BYTES, &mapB, ks * kBK, 0, &full[st], kEvictNormal);   // v: re-read per tile
      }
      __syncwarp();
      if (++ks == a.k_steps) { ks = 0; ++rt; }
    }
  } else if (warp == 1) {
    // ---- MMA issuer: D[128 x NP] (+)= W tile [128 x 64] x v tileᵀ [64 x NP]
    constexpr uint32_t idesc = idesc_bf16(kTM, NP, false, false);
    constexpr uint32_t hi_k = desc_sw128_hi(1024);
    const uint32_t s0 = smem_addr(smem);
    int g = 0, seg = 0;
    for (int u = lo; u < hi; ++seg) {
      const int seg_end = min(hi, (u / a.k_steps + 1) * a.k_steps);
      const int ab = seg & 1;
      mbar_wait(&acc_empty[ab], ((seg >> 1) & 1) ^ 1);
      tc_fence_after();
      for (int v = u; v < seg_end; ++v, ++g) {
        const int st = g % C::NST;
        mbar_wait(&full[st], (g / C::NST) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t da = make_desc(s0 + st * C::STAGE, 16, hi_k);
          const uint64_t db = make_desc(s0 + st * C::STAGE + C::A_BYTES, 16, hi_k);
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk)
            mma_ss(tb + ab * NP, da + uint64_t(kk * 2), db + uint64_t(kk * 2), idesc, (v == u && kk == 0) ? 0u : 1u);
          mma_commit(&empty[st]);
          if (v + 1 == seg_end) mma_commit(&acc_full[ab]);
        }
        __syncwarp();
      }
      u = seg_end;
    }
  } else if (warp >= 4) {
    // ---- epilogue: TMEM -> partial [seg, b, row]
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;
    const uint32_t lane_base = tb + (uint32_t(q4 * 32) << 16);
    int seg = 0;
    for (int u = lo; u < hi; ++seg) {
      const int rt = u / a.k_steps;
      const int seg_end = min(hi, (rt + 1) * a.k_steps);
      const int ab = seg & 1;
      mbar_wait(&acc_full[ab], (seg >> 1) & 1);
      tc_fence_after();
      const int seg_id = seg_base + seg;
      float* out = a.part + (long)seg_id * a.B * kTM + r;
#pragma unroll 1
      for (int c0 = 0; c0 < NP; c0 += 32) {
        uint32_t d[32];
        tmem_ld32(lane_base + ab * NP + c0, d);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (c0 + j < a.B) out[(long)(c0 + j) * kTM] = __uint_as_float(d[j]);
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[ab]);
      if (r == 0) {
        if (u == long(rt) * a.k_steps) a.meta[2 * rt] = seg_id;
        if (seg_end == long(rt + 1) * a.k_steps) a.meta[2 * rt + 1] = seg_id;
      }
      u = seg_end;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<C::TMEM_COLS>(tb);
}

// y[b, n] = (accumulate ? y[b, n] : 0) + Σ_{seg of tile n/128} part[seg, b, n % 128]   (fixed order);
// out (optional): the bf16 copy of y (the final cast, when no all-reduce follows)
__global__ void reduce_seg_kernel(const float* __restrict__ part, const int32_t* __restrict__ meta, int N, int B,
                                  float* __restrict__ y, int accumulate, uint16_t* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (i >= (long)B * N) return;
  const int b = int(i / N), n = int(i % N), rt = n / kTM;
  float acc = accumulate ? y[i] : 0.f;
  for (int s = meta[2 * rt]; s <= meta[2 * rt + 1]; ++s) acc += part[((long)s * B + b) * kTM + (n % kTM)];
  y[i] = acc;
  if (out) out[i] = f2bf(acc);
}

// The same reduce fused with the one-shot all-reduce over the symmetric buffer (FusedAr, SURVEY f2(i);
// O = AllReduce(Σ_r Õ_r)): (1) this rank's rows of the launch -> its half of the buffer (the half
// chosen by the barrier epoch: a rank can be one call ahead of a peer, never two); (2) the CTA meets
// the same CTA index of every peer (LSA barrier, release / acquire at system scope); (3) every element of
// the CTA's slice summed over the ranks — multimem.ld_reduce through the NVLS multicast address, or
// peer loads over NVLink in rank order — into y and the bf16 output.  Fixed geometry: kArCtas CTAs,
// so a CTA's slice is the same set of elements on every rank.
__global__ void __launch_bounds__(256) reduce_seg_ar_kernel(const float* __restrict__ part,
                                                            const int32_t* __restrict__ meta, int N, int B,
                                                            float* __restrict__ y, int accumulate,
                                                            uint16_t* __restrict__ out, ncclDevComm dc,
                                                            ncclWindow_t win, size_t half_elems, long row0,
                                                            int multimem) {
  pdl_trigger();
  pdl_wait();
  ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamTagLsa(), blockIdx.x, multimem != 0);
  const uint32_t step = multimem ? uint32_t(dc.lsaSize) : 1u;          // epoch advance per barrier
  const size_t base = ((bar.epoch / step) & 1u) * half_elems + size_t(row0) * N;
  float* mine = static_cast<float*>(ncclGetLocalPointer(win, 0)) + base;
  const long n = (long)B * N;
  for (long i = blockIdx.x * 256L + threadIdx.x; i < n; i += 256L * gridDim.x) {
    const int b = int(i / N), nn = int(i % N), rt = nn / kTM;
    float acc = accumulate ? y[i] : 0.f;
    for (int s = meta[2 * rt]; s <= meta[2 * rt + 1]; ++s) acc += part[((long)s * B + b) * kTM + (nn % kTM)];
    mine[i] = acc;
  }
  bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
  if (multimem) {
    const float* mc = static_cast<const float*>(ncclGetLsaMultimemPointer(win, 0, dc)) + base;
    for (long i = blockIdx.x * 256L + threadIdx.x; i < n; i += 256L * gridDim.x) {
      float t;
      asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(t) : "l"(mc + i) : "memory");
      y[i] = t;
      if (out) out[i] = f2bf(t);
    }
  } else {
    for (long i = blockIdx.x * 256L + threadIdx.x; i < n; i += 256L * gridDim.x) {
      float t = 0.f;
      for (int p = 0; p < dc.lsaSize; ++p)                             // fixed rank order: deterministic
        t += static_cast<const float*>(ncclGetLsaPointer(win, 0, p))[base + i];
      y[i] = t;
      if (out) out[i] = f2bf(t);
    }
  }
  // (no second barrier: this half is written again two calls later, and this CTA index of every peer
  // must have arrived at the next call's barrier — after these reads — before that)
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  }
  return fn;
}

bool make_map(CUtensorMap* m, const void* base, long cols, long rows, int box_c, int box_r, long ld = 0) {
  EncodeFn enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(ld > 0 ? ld : cols) * 2};
  cuuint32_t box[2] = {cuuint32_t(box_c), cuuint32_t(box_r)};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int NP>
cudaError_t launch_np(const CUtensorMap& mA, const CUtensorMap& mB, const GArgs& a, int n_cta, cudaStream_t s) {
  using C = GCfg<NP>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(skinny_tc_kernel<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  KernelScope ks("K5_W_O_tc", s);
  return launch_k(skinny_tc_kernel<NP>, n_cta, 256, C::SMEM, s, mA, mB, a);
}

}  // namespace

bool wo_tc_supported(int N, int K, int B) {
  const long units = long((N + kTM - 1) / kTM) * (K / kBK);
  return K % kBK == 0 && B >= 1 && B <= 256 && N >= 1 && units * 1024 < (1L << 31);   // c*U fits an int
}

int wo_tc_ctas(int N, int K) {   // (K: the columns this launch reduces over)
  const long units = long((N + kTM - 1) / kTM) * (K / kBK);
  return int(std::max(1L, std::min<long>(sm_count(), units)));
}

size_t wo_tc_part_bytes(int N, int K, int B) {
  const int n_tiles = (N + kTM - 1) / kTM;
  return size_t(wo_tc_ctas(N, K) + n_tiles) * B * kTM * 4 + size_t(n_tiles) * 2 * 4 + 256;
}

cudaError_t launch_wo_tc(const uint16_t* Wt, const uint16_t* v, int N, int K, int B, void* part_ws, float* y,
                         bool accumulate, uint16_t* out_bf16, cudaStream_t s, int k_begin, int k_len, long v_ld,
                         const FusedAr* ar, long ar_row0) {
  if (k_len <= 0) k_len = K;
  const int n_tiles = (N + kTM - 1) / kTM;
  const int NP = B <= 32 ? 32 : B <= 64 ? 64 : B <= 128 ? 128 : 256;
  CUtensorMap mA, mB;
  // A: the blocked weights viewed as [n_tiles * k_steps * 128 rows, 64 cols]
  if (!make_map(&mA, Wt, kBK, long(n_tiles) * (K / kBK) * kTM, kBK, kTM) || !make_map(&mB, v, k_len, B, kBK, NP, v_ld))
    return cudaErrorInvalidValue;
  GArgs a;
  a.part = static_cast<float*>(part_ws);
  const int n_cta = wo_tc_ctas(N, k_len);
  a.meta = reinterpret_cast<int32_t*>(static_cast<char*>(part_ws) + size_t(n_cta + n_tiles) * B * kTM * 4);
  a.N = N; a.K = K; a.B = B; a.n_tiles = n_tiles; a.k_steps = k_len / kBK;
  a.k_total = K / kBK; a.k0 = k_begin / kBK;
  cudaError_t e;
  switch (NP) {
    case 32: e = launch_np<32>(mA, mB, a, n_cta, s); break;
    case 64: e = launch_np<64>(mA, mB, a, n_cta, s); break;
    case 128: e = launch_np<128>(mA, mB, a, n_cta, s); break;
    default: e = launch_np<256>(mA, mB, a, n_cta, s); break;
  }
  if (e != cudaSuccess) return e;
  const long n = long(B) * N;
  if (ar) {
    KernelScope ks("K5_reduce_allreduce", s);
    return launch_k(reduce_seg_ar_kernel, kArCtas, 256, 0, s, a.part, a.meta, N, B, y, accumulate ? 1 : 0, out_bf16,
                    *static_cast<const ncclDevComm*>(ar->dev_comm), static_cast<ncclWindow_t>(ar->window),
                    ar->half_elems, ar_row0, ar->multimem);
  }
  KernelScope ks("K5_reduce", s);
  return launch_k(reduce_seg_kernel, int((n + 255) / 256), 256, 0, s, a.part, a.meta, N, B, y, accumulate ? 1 : 0,
                  out_bf16);
}

}  // namespace tpla
