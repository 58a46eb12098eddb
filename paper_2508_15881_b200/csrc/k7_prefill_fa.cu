// K8 — causal prefill attention of MLA in its non-absorbed form (§5.1 PD
// separation P:421, §4.5 / §5.4.2: prefill is compute-bound, so MLA's prefill
// runs with the heads split over the devices and the latent NOT sliced; its rows go to the TPLA
// decode cache with the full RMS).
//
// Per head h of this device (Eq. isolate_rope):
//   s[i, t] = sm_scale (q_h[i] · k_h[t] + q^PE_h[i] · k^PE[t]),  t <= i (causal),   k_h = ĉ W^UK_h
//   O_h[i]  = Σ_t softmax(s[i, :])_t v_h[t],                                          v_h = ĉ W^UV_h
// with the head dimension 128 (+ 64 RoPE) instead of the absorbed 512 (+ 64): ~3.4x fewer FLOPs
// than attending to the latent directly (f1).
//
// Persistent CTAs over (128-query tile, head) work items, longest first; queries are the MMA M
// dimension.  Per 128-key tile:
//   QK  S[128 x 128] fp32 (TMEM) = Q [128 x 192] (smem) x [K ‖ k^PE] tileᵀ (smem, K-major)   tcgen05 SS
//   softmax: 8 warps (two per TMEM lane quadrant, 64 columns each, thread = query row), exact row max
//            (half maxima exchanged through smem), lazily raised
//            running max (O rescaled in TMEM only when it grows by > 2^8), P bf16 over S's columns
//   PV  O[128 x 128] (TMEM) += P (TMEM) x V tile (smem, MN-major)                          tcgen05 TS
// Q, K, k^PE and V tiles arrive by TMA (SWIZZLE_128B, 128-row x 64-column boxes); two K/V stages and
// two S buffers let QK(j + 1) run on the tensor pipe while the softmax works on tile j.  The
// diagonal tile is masked per row; tiles past it are never loaded (causal).  CTAs are issued
// longest-first (the last query tiles attend to the most keys).
//
// Warp roles (384 threads): w0 TMA (Q, K ring), w1 MMA issuer, w2 TMEM allocator, w3 TMA (V ring),
// w4-w11 softmax + epilogue.
#include <cuda.h>
#include <math.h>

#include <algorithm>

#include "common.cuh"
#include "internal.h"
#include "sm100.cuh"

namespace tpla {
namespace {

// Polynomial exp2 share of the softmax: iterations c (step 2) with (c & kPolyMask) == 0 compute two of
// their four exponentials on the FMA pipe — 6: 1 in 8 (default), 2: 1 in 4, 0: 1 in 2, -1: none.
#ifndef TPLA_K8_POLY_MASK
#define TPLA_K8_POLY_MASK 6
#endif
constexpr int kPolyMask = TPLA_K8_POLY_MASK;

using namespace sm100;

constexpr int kT = 128;               // queries per CTA = keys per tile
constexpr int kBox = kT * 128;        // one [128 rows x 64 cols] bf16 box, 16 KB
constexpr int kQBytes = 3 * kBox;     // q (2 boxes) + q^PE (1 box)
constexpr int kKBytes = 3 * kBox;     // K (2 boxes) + k^PE (1): a K-ring stage
constexpr int kVBytes = 2 * kBox;     // V (2 boxes): a V-ring stage
constexpr int kStages = 2;            // per ring
constexpr int kSmem = 1024 + kQBytes + kStages * (kKBytes + kVBytes);
constexpr int kThreads = 384;
constexpr float kRescale = 8.0f;      // log2 units (p <= 2^8 between running-max raises)
// TMEM columns: S0, S1 (128 each), O (128)
constexpr int kS0 = 0, kO = 256, kTmemCols = 512;

struct FaArgs {
  uint16_t* o;          // [L, H * 128] bf16
  int L, H, n_qt;
  int q_head0;          // head index of this device's head 0 in the q arrays
  float scale_log2;
};

// work item i -> (query tile, head): head-major, so the ~148 items in flight at any time cover only a
// few heads and their K / V tiles (2 MB per head at 4K tokens) stay in L2 (query-tile-major order made
// every CTA stream a different head's K / V from HBM); within a head the longest query tiles first
__device__ __forceinline__ void item_of(const FaArgs& a, int i, int& qt, int& h) {
  h = i / a.n_qt;
  qt = a.n_qt - 1 - i % a.n_qt;
}

// Persistent: CTA c takes work items c, c + G, c + 2G, ... (G = gridDim.x); the ring, S buffers and
// their barrier phases run on over a CTA-global key-tile counter J, so one item's epilogue overlaps the
// next item's first QKs: the next Q is loaded once the last QK of the item completed (q_free), and the
// first PV of the next item (which overwrites O) waits for the epilogue's O loads (o_free).
__global__ void __launch_bounds__(kThreads, 1)
attn_fwd_causal_kernel(const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mqp,
                       const __grid_constant__ CUtensorMap mk, const __grid_constant__ CUtensorMap mkp,
                       const __grid_constant__ CUtensorMap mv, FaArgs a) {
  pdl_trigger();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* s_q = smem;
  uint8_t* s_k = smem + kQBytes;                 // K ring: [K ‖ k^PE] tiles, freed when their QK completes
  uint8_t* s_v = s_k + kStages * kKBytes;        // V ring: freed when the tile's PV completes
  __shared__ uint64_t q_full, q_free, o_free, k_full[kStages], k_empty[kStages], v_full[kStages], v_empty[kStages];
  __shared__ uint64_t s_full[2], p_full[2], pv_done[2];
  __shared__ uint32_t tmem_base;
  __shared__ float red_max[2][2][128];           // [J & 1][half][row] half-row maxima
  __shared__ float red_l[2][128];                // [half][row] half-row sums at an item's end
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_items = a.n_qt * a.H, G = int(gridDim.x);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mq); tma_prefetch_desc(&mqp); tma_prefetch_desc(&mk); tma_prefetch_desc(&mkp);
    tma_prefetch_desc(&mv);
    mbar_init(&q_full, 1);
    mbar_init(&q_free, 1);
    mbar_init(&o_free, 8);
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&k_full[i], 1); mbar_init(&k_empty[i], 1); mbar_init(&v_full[i], 1); mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) { mbar_init(&s_full[i], 1); mbar_init(&p_full[i], 8); mbar_init(&pv_done[i], 1); }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<kTmemCols>(&tmem_base);
  pdl_wait();                                   // K / V (the up-projection GEMMs) come from the predecessors
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tmem_base;

  if (warp == 0 || warp == 3) {
    // ---------------------------------------------------------------- TMA producers: w0 Q + K ring, w3 V ring
    // (two rings: the K tile of QK(J + 2) can land while PV(J) still holds V(J) — with one K/V stage
    // released only by the PV, each QK waited for its tile's load latency, trace / ncu: tensor 32 %)
    if (elect_one()) {
      int J = 0;
      for (int it = 0, i = blockIdx.x; i < n_items; ++it, i += G) {
        int qt, h;
        item_of(a, i, qt, h);
        if (warp == 0) {
          if (it > 0) mbar_wait(&q_free, (it - 1) & 1);   // the previous item's QKs are complete
          mbar_arrive_expect_tx(&q_full, kQBytes);
          const int qc = (a.q_head0 + h) * 128, qpc = (a.q_head0 + h) * 64;
          tma_load_2d(s_q, &mq, qc, qt * kT, &q_full, kEvictFirst);
          tma_load_2d(s_q + kBox, &mq, qc + 64, qt * kT, &q_full, kEvictFirst);
          tma_load_2d(s_q + 2 * kBox, &mqp, qpc, qt * kT, &q_full, kEvictFirst);
        }
        for (int j = 0; j <= qt; ++j, ++J) {           // key tiles 0..qt (causal)
          const int st = J % kStages, t0 = j * kT, kc = h * 128;
          if (warp == 0) {
            mbar_wait(&k_empty[st], ((J / kStages) & 1) ^ 1);
            uint8_t* dst = s_k + st * kKBytes;
            mbar_arrive_expect_tx(&k_full[st], kKBytes);
            tma_load_2d(dst, &mk, kc, t0, &k_full[st], kEvictNormal);            // K: re-read by every query tile
            tma_load_2d(dst + kBox, &mk, kc + 64, t0, &k_full[st], kEvictNormal);
            tma_load_2d(dst + 2 * kBox, &mkp, 0, t0, &k_full[st], kEvictNormal);   // k^PE (shared by the heads)
          } else {
            mbar_wait(&v_empty[st], ((J / kStages) & 1) ^ 1);
            uint8_t* dst = s_v + st * kVBytes;
            mbar_arrive_expect_tx(&v_full[st], kVBytes);
            tma_load_2d(dst, &mv, kc, t0, &v_full[st], kEvictNormal);
            tma_load_2d(dst + kBox, &mv, kc + 64, t0, &v_full[st], kEvictNormal);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer: QK(J), then PV(J - 1)
    constexpr uint32_t id_qk = idesc_bf16(128, kT, false, false);
    constexpr uint32_t id_pv = idesc_bf16(128, 128, false, true);
    constexpr uint32_t hi_k = desc_sw128_hi(1024);
    const uint32_t q_addr = smem_addr(s_q), k0 = smem_addr(s_k), v0 = smem_addr(s_v);
    auto issue_pv = [&](int J, bool first) {
      const int st = J % kStages;
      mbar_wait(&p_full[J & 1], (J >> 1) & 1);
      mbar_wait(&v_full[st], (J / kStages) & 1);
      tc_fence_after();
      if (elect_one()) {
        // V: two 64-column MN-major atoms one box apart; 16 keys (2 KB) per k-step
        const uint64_t v_desc = make_desc(v0 + st * kVBytes, kBox, hi_k);
        const uint32_t p_tmem = tb + kS0 + (J & 1) * kT;
#pragma unroll
        for (int kk = 0; kk < kT / 16; ++kk)
          mma_ts(tb + kO, p_tmem + kk * 8, v_desc + uint64_t(kk * (2048 >> 4)), id_pv, (first && kk == 0) ? 0u : 1u);
        mma_commit(&v_empty[st]);
        mma_commit(&pv_done[J & 1]);
      }
      __syncwarp();
    };
    int J = 0;
    for (int it = 0, i = blockIdx.x; i < n_items; ++it, i += G) {
      int qt, h;
      item_of(a, i, qt, h);
      mbar_wait(&q_full, it & 1);
      const int J0 = J;
      for (int j = 0; j <= qt; ++j, ++J) {
        const int st = J % kStages;
        mbar_wait(&k_full[st], (J / kStages) & 1);
        if (J >= 2) mbar_wait(&pv_done[J & 1], ((J - 2) >> 1) & 1);   // S buffer (= P of tile J - 2) free
        tc_fence_after();
        if (elect_one()) {
          const uint64_t kd = make_desc(k0 + st * kKBytes, 16, hi_k);
          const uint64_t qd = make_desc(q_addr, 16, hi_k);
          const uint32_t s_tmem = tb + kS0 + (J & 1) * kT;
#pragma unroll
          for (int kk = 0; kk < 12; ++kk) {        // 192 = q (128) ‖ q^PE (64): box kk/4, +32 B per k-step
            const uint64_t off = uint64_t(((kk >> 2) * kBox + (kk & 3) * 32) >> 4);
            mma_ss(s_tmem, qd + off, kd + off, id_qk, kk > 0 ? 1u : 0u);
          }
          mma_commit(&s_full[J & 1]);
          mma_commit(&k_empty[st]);                // the K stage is free once this QK completed
          if (j == qt) mma_commit(&q_free);        // Q may be replaced once this QK completed
        }
        __syncwarp();
        if (j >= 1) issue_pv(J - 1, J - 1 == J0);
        else if (it > 0) mbar_wait(&o_free, (it - 1) & 1);   // the previous item's O has been read
      }
      issue_pv(J - 1, J - 1 == J0);
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- softmax + epilogue
    // Two warps per TMEM lane quadrant (warps 4+q and 8+q share SMSP q): warp `half` owns S columns
    // [64 half, 64 half + 64) of every tile and O columns [64 half, ..); they exchange their half-row
    // maxima through shared memory (named barrier per quadrant) so both take the same rescale
    // decisions.  One warp alone reached ~2.8 of the SMSP's 4 exp/clk (tools/exps_rate), two ~3.7.
    const int q4 = warp & 3, half = (warp - 4) >> 2;
    const int r = q4 * 32 + lane;                  // query row of the tile = TMEM lane
    const uint32_t lane_base = tb + (uint32_t(q4 * 32) << 16);
    const uint32_t pair_bar = 1 + q4;
    const float sc = a.scale_log2;
    int J = 0;
    for (int it = 0, i = blockIdx.x; i < n_items; ++it, i += G) {
      int qt, h;
      item_of(a, i, qt, h);
      const int qi = qt * kT + r;                  // this row's token index
      float m_run = -INFINITY, l = 0.f;
      for (int j = 0; j <= qt; ++j, ++J) {
        mbar_wait(&s_full[J & 1], (J >> 1) & 1);
        tc_fence_after();
        uint32_t sv[2][32];
        const uint32_t s_addr = lane_base + kS0 + (J & 1) * kT;
        tmem_ld32(s_addr + 64 * half, sv[0]);
        tmem_ld32(s_addr + 64 * half + 32, sv[1]);
        tmem_ld_wait();
        float* x = reinterpret_cast<float*>(&sv[0][0]);
        if (j == qt) {                               // the diagonal tile: key t <= query i (t, i < L)
          const int lim = min(qi, a.L - 1) - j * kT - 64 * half;
#pragma unroll
          for (int c = 0; c < 64; ++c) x[c] = c <= lim ? x[c] : -INFINITY;
        }
        float m0 = x[0], m1 = x[1], m2 = x[2], m3 = x[3];
#pragma unroll
        for (int c = 4; c < 64; c += 4) {
          m0 = fmaxf(m0, x[c]); m1 = fmaxf(m1, x[c + 1]); m2 = fmaxf(m2, x[c + 2]); m3 = fmaxf(m3, x[c + 3]);
        }
        float mx = fmaxf(fmaxf(m0, m1), fmaxf(m2, m3));
        red_max[J & 1][half][r] = mx;
        named_bar_sync(pair_bar, 64);
        mx = fmaxf(mx, red_max[J & 1][half ^ 1][r]) * sc;
        const float m_new = mx > m_run + kRescale ? mx : m_run;
        const bool grow = j > 0 && m_new != m_run;
        if (__any_sync(0xffffffffu, grow)) {         // O holds PV(J - 1) and earlier at m_run: this half
          const float f = grow ? ex2(m_run - m_new) : 1.f;
          mbar_wait(&pv_done[(J - 1) & 1], ((J - 1) >> 1) & 1);
          tc_fence_after();
#pragma unroll 1
          for (int c0 = 64 * half; c0 < 64 * half + 64; c0 += 32) {
            uint32_t ov[32];
            tmem_ld32(lane_base + kO + c0, ov);
            tmem_ld_wait();
#pragma unroll
            for (int c = 0; c < 32; ++c) ov[c] = __float_as_uint(__uint_as_float(ov[c]) * f);
            tmem_st32(lane_base + kO + c0, ov);
          }
          l *= f;
        }
        m_run = m_new;
        const float neg_m = m_run == -INFINITY ? 0.f : -m_run;
        const uint64_t sc2 = f2_pack(sc, sc), nm2 = f2_pack(neg_m, neg_m);
        uint64_t l01 = f2_pack(0.f, 0.f), l23 = f2_pack(0.f, 0.f);
        uint32_t pw[32];
#pragma unroll
        for (int c = 0; c < 32; c += 2) {
          float y0, y1, y2, y3;
          f2_unpack(ffma2(f2_pack(x[2 * c], x[2 * c + 1]), sc2, nm2), y0, y1);
          f2_unpack(ffma2(f2_pack(x[2 * c + 2], x[2 * c + 3]), sc2, nm2), y2, y3);
          const float p0 = ex2(y0), p1 = ex2(y1);
          float p2, p3;
          if (kPolyMask >= 0 && (c & kPolyMask) == 0) {
            ex2_poly2(y2, y3, p2, p3);               // 1 in 8 on the FMA pipe (arguments <= 8)
          } else {
            p2 = ex2(y2);
            p3 = ex2(y3);
          }
          l01 = fadd2(l01, f2_pack(p0, p1));
          l23 = fadd2(l23, f2_pack(p2, p3));
          pw[c] = pack_bf16x2(p0, p1);
          pw[c + 1] = pack_bf16x2(p2, p3);
        }
        float a0, a1, a2, a3;
        f2_unpack(l01, a0, a1);
        f2_unpack(l23, a2, a3);
        l += (a0 + a1) + (a2 + a3);
        // P (bf16 pairs) of this half: packed columns [32 half, 32 half + 32) of S (logits consumed)
        tmem_st32(s_addr + 32 * half, pw);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[J & 1]);
      }
      // ---- epilogue: O / l -> bf16 [L, H * 128] (this half's 64 columns), then O is free
      red_l[half][r] = l;
      mbar_wait(&pv_done[(J - 1) & 1], ((J - 1) >> 1) & 1);
      tc_fence_after();
      named_bar_sync(pair_bar, 64);
      const float lt = l + red_l[half ^ 1][r];
      const float inv = lt > 0.f ? 1.f / lt : 0.f;
      uint16_t* orow = a.o + (long)qi * a.H * 128 + h * 128;
#pragma unroll 1
      for (int c0 = 64 * half; c0 < 64 * half + 64; c0 += 32) {
        uint32_t ov[32];
        tmem_ld32(lane_base + kO + c0, ov);
        tmem_ld_wait();
        if (qi < a.L) {
#pragma unroll
          for (int c = 0; c < 32; c += 8) {
            uint4 u;
            u.x = pack_bf16(__uint_as_float(ov[c]) * inv, __uint_as_float(ov[c + 1]) * inv);
            u.y = pack_bf16(__uint_as_float(ov[c + 2]) * inv, __uint_as_float(ov[c + 3]) * inv);
            u.z = pack_bf16(__uint_as_float(ov[c + 4]) * inv, __uint_as_float(ov[c + 5]) * inv);
            u.w = pack_bf16(__uint_as_float(ov[c + 6]) * inv, __uint_as_float(ov[c + 7]) * inv);
            *reinterpret_cast<uint4*>(orow + c0 + c) = u;
          }
        }
      }
      named_bar_sync(pair_bar, 64);                 // red_l free again
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_free);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<kTmemCols>(tb);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode() {
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

// [rows x cols] bf16 with row stride ld elements; 128-row x 64-column boxes, SWIZZLE_128B (OOB rows read 0)
bool map2d(CUtensorMap* m, const void* base, long cols, long rows, long ld) {
  EncodeFn enc = encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(ld) * 2};
  cuuint32_t box[2] = {64, kT};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// one warp per row: ĉ = c / sqrt(|c|^2 / d_c + eps), bf16 pairs (d_c even)
__global__ void prefill_rmsnorm_kernel(const uint32_t* __restrict__ c, int L, int d_c, float eps,
                                       uint32_t* __restrict__ out) {
  pdl_trigger();
  const int row = blockIdx.x * 4 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  const int np = d_c / 2;
  float ss = 0.f;
  if (row < L)
    for (int p = lane; p < np; p += 32) {
      const uint32_t v = c[(long)row * np + p];
      ss += bf16_lo(v) * bf16_lo(v) + bf16_hi(v) * bf16_hi(v);
    }
  ss = warp_sum(ss);
  const float r = rsqrtf(ss / d_c + eps);
  pdl_wait();                                     // first store (the previous prefill may still read ĉ)
  if (row < L)
    for (int p = lane; p < np; p += 32) {
      const uint32_t v = c[(long)row * np + p];
      out[(long)row * np + p] = pack_bf16(bf16_lo(v) * r, bf16_hi(v) * r);
    }
}

}  // namespace

cudaError_t launch_prefill_rmsnorm(const uint16_t* c_kv, int L, int d_c, float eps, uint16_t* c_hat, cudaStream_t s) {
  KernelScope ks("K8_prefill_rmsnorm", s);
  return launch_k(prefill_rmsnorm_kernel, (L + 3) / 4, 128, 0, s, reinterpret_cast<const uint32_t*>(c_kv), L, d_c, eps,
                  reinterpret_cast<uint32_t*>(c_hat));
}

cudaError_t launch_attn_fwd_causal(const uint16_t* q_nope, const uint16_t* q_pe, int h_q, int q_head0,
                                   const uint16_t* K, const uint16_t* V, int H, const uint16_t* k_pe, long kpe_ld,
                                   int L, float sm_scale, uint16_t* O, cudaStream_t s) {
  CUtensorMap mq, mqp, mk, mkp, mv;
  if (!map2d(&mq, q_nope, long(h_q) * 128, L, long(h_q) * 128) || !map2d(&mqp, q_pe, long(h_q) * 64, L, long(h_q) * 64) ||
      !map2d(&mk, K, long(H) * 128, L, long(H) * 128) || !map2d(&mkp, k_pe, 64, L, kpe_ld) ||
      !map2d(&mv, V, long(H) * 128, L, long(H) * 128))
    return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_causal_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  FaArgs a;
  a.o = O;
  a.L = L;
  a.H = H;
  a.n_qt = (L + kT - 1) / kT;
  a.q_head0 = q_head0;
  a.scale_log2 = sm_scale * 1.4426950408889634f;
  int sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = std::max(1, std::min(a.n_qt * H, sms > 0 ? sms : 148));
  KernelScope ks("K8_prefill_fa", s);
  return launch_k(attn_fwd_causal_kernel, grid, kThreads, kSmem, s, mq, mqp, mk, mkp, mv, a);
}

}  // namespace tpla
