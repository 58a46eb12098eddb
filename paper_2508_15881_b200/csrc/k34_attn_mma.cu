// K3 (v0, legacy tensor path) — per-shard split-K flash decoding; K4 — split-K combine.
//
// One CTA per work unit (sequence b, token chunk).  Heads are the M dimension (16 per warp),
// the device's cache row [ĉ_j ‖ k^PE] is the K dimension of QKᵀ and its latent part the N
// dimension of PV (Eq. tpla_softmax_one_device):
//   s_t = sm_scale · ([Q'_j ‖ q^PE] · [ĉ_{j,t} ‖ k^PE_t])          (μ_j already in Q'_j)
//   online softmax over THIS shard's tokens only — no cross-device max/sum
//   O_j += p_t ĉ_{j,t}
// Each unit emits an unnormalised partial (O, m, l); K4 merges the units of a sequence.
//
// This is the mma.sync (HMMA) baseline: 64-token tiles double-buffered with cp.async into
// padded shared memory, ldmatrix fragments, FA2-style register softmax.
#include <math.h>

#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace tpla {
namespace {

constexpr int TILE = 64;

struct AttnArgs {
  const uint16_t* q_lat;   // [B, H_loc, W_lat]
  const uint16_t* q_pe;    // [B, h_q, d_r]
  const uint16_t* cache;
  const int32_t* block_table;
  const int32_t* seq_lens;
  float* o_part;           // [B*n_split, H_loc, W_lat]
  float* ml_part;          // [B*n_split, H_loc, 2]
  int h_loc, h_q, head_begin, page_size, max_pages, row_stride, n_split, chunk;
  float scale_log2;        // sm_scale * log2(e)
};

template <int W_LAT, int D_R>
__global__ void __launch_bounds__(256, 1) attn_mma_kernel(AttnArgs a) {
  pdl_trigger();
  pdl_wait();
  constexpr int W = W_LAT + D_R;
  constexpr int WP = W + 8;                 // padded row: odd number of 16-byte chunks -> no ldmatrix conflicts
  constexpr int KSTEPS = W / 16;
  constexpr int NT_O = W_LAT / 8;           // n8 tiles of the output
  extern __shared__ __align__(128) uint16_t smem[];
  const int nwarps = blockDim.x >> 5;
  const int H_pad = nwarps * 16;
  uint16_t* sQ = smem;                      // [H_pad][WP]
  uint16_t* sKV = smem + H_pad * WP;        // [2][TILE][WP]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int split = blockIdx.x, b = blockIdx.y;
  const int unit = b * a.n_split + split;
  const int S = a.seq_lens[b];
  const int t_begin = split * a.chunk;
  const int t_end = min(S, t_begin + a.chunk);

  // ---- stage Q = [Q'_j ‖ q^PE] for this sequence
  for (int c = tid; c < H_pad * (W / 8); c += blockDim.x) {
    int h = c / (W / 8), ch = c % (W / 8);
    int col = ch * 8;
    const uint16_t* src;
    bool ok = h < a.h_loc;
    if (col < W_LAT) src = a.q_lat + ((long)b * a.h_loc + h) * W_LAT + col;
    else src = a.q_pe + ((long)b * a.h_q + a.head_begin + h) * D_R + (col - W_LAT);
    cp_async16(sQ + h * WP + col, ok ? src : a.q_lat, ok);
  }
  cp_async_commit();

  auto load_tile = [&](int t0, int buf) {
    uint16_t* dst = sKV + buf * TILE * WP;
    const int page = a.block_table[(long)b * a.max_pages + t0 / a.page_size];
    const uint16_t* src = a.cache + ((long)page * a.page_size + (t0 % a.page_size)) * a.row_stride;
    for (int c = tid; c < TILE * (W / 8); c += blockDim.x) {
      int r = c / (W / 8), ch = c % (W / 8);
      bool ok = t0 + r < t_end;
      cp_async16(dst + r * WP + ch * 8, ok ? src + (long)r * a.row_stride + ch * 8 : src, ok);
    }
  };

  float o[NT_O][4];
#pragma unroll
  for (int i = 0; i < NT_O; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};

  const int ntiles = t_end > t_begin ? (t_end - t_begin + TILE - 1) / TILE : 0;
  if (ntiles > 0) load_tile(t_begin, 0);
  cp_async_commit();

  for (int it = 0; it < ntiles; ++it) {
    const int t0 = t_begin + it * TILE;
    if (it + 1 < ntiles) load_tile(t0 + TILE, (it + 1) & 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const uint16_t* kv = sKV + (it & 1) * TILE * WP;

    // S = Q Kᵀ : 16 heads x 64 tokens per warp
    float s[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < KSTEPS; ++ks) {
      uint32_t af[4];
      ldmatrix_x4(af[0], af[1], af[2], af[3],
                  smem_u32(sQ + (warp * 16 + (lane & 15)) * WP + ks * 16 + ((lane >> 4) << 3)));
#pragma unroll
      for (int nj = 0; nj < 4; ++nj) {
        uint32_t b0, b1, b2, b3;
        int r = nj * 16 + (lane & 7) + ((lane >> 4) << 3);
        int col = ks * 16 + (((lane >> 3) & 1) << 3);
        ldmatrix_x4(b0, b1, b2, b3, smem_u32(kv + r * WP + col));
        uint32_t bb0[2] = {b0, b1}, bb1[2] = {b2, b3};
        mma_bf16_16816(s[2 * nj], af, bb0);
        mma_bf16_16816(s[2 * nj + 1], af, bb1);
      }
    }
    // mask + online softmax (log2 domain)
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        int t = t0 + j * 8 + (lane & 3) * 2 + (q & 1);
        float v = (t < t_end) ? s[j][q] * a.scale_log2 : -INFINITY;
        s[j][q] = v;
        mx[q >> 1] = fmaxf(mx[q >> 1], v);
      }
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      mx[hh] = fmaxf(mx[hh], __shfl_xor_sync(0xffffffffu, mx[hh], 1));
      mx[hh] = fmaxf(mx[hh], __shfl_xor_sync(0xffffffffu, mx[hh], 2));
    }
    float alpha[2], mnew[2];
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      mnew[hh] = fmaxf(m_r[hh], mx[hh]);          // finite: every tile has >= 1 valid token
      alpha[hh] = exp2f(m_r[hh] - mnew[hh]);      // exp2(-inf) = 0 on the first tile
      m_r[hh] = mnew[hh];
      l_r[hh] *= alpha[hh];
    }
    uint32_t pf[4][4];                             // P as A fragments (4 k16 steps over tokens)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float p0 = exp2f(s[j][0] - mnew[0]), p1 = exp2f(s[j][1] - mnew[0]);
      float p2 = exp2f(s[j][2] - mnew[1]), p3 = exp2f(s[j][3] - mnew[1]);
      l_r[0] += p0 + p1;
      l_r[1] += p2 + p3;
      pf[j >> 1][(j & 1) * 2 + 0] = pack_bf16(p0, p1);
      pf[j >> 1][(j & 1) * 2 + 1] = pack_bf16(p2, p3);
    }
#pragma unroll
    for (int i = 0; i < NT_O; ++i) {
      o[i][0] *= alpha[0]; o[i][1] *= alpha[0];
      o[i][2] *= alpha[1]; o[i][3] *= alpha[1];
    }
    // O += P V, V = latent columns of the tile
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t pa[4] = {pf[kk][0], pf[kk][1], pf[kk][2], pf[kk][3]};
#pragma unroll
      for (int nj = 0; nj < NT_O / 2; ++nj) {
        uint32_t b0, b1, b2, b3;
        int r = kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
        int col = nj * 16 + ((lane >> 4) << 3);
        ldmatrix_x4_trans(b0, b1, b2, b3, smem_u32(kv + r * WP + col));
        uint32_t bb0[2] = {b0, b1}, bb1[2] = {b2, b3};
        mma_bf16_16816(o[2 * nj], pa, bb0);
        mma_bf16_16816(o[2 * nj + 1], pa, bb1);
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();

  // partial results
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    l_r[hh] += __shfl_xor_sync(0xffffffffu, l_r[hh], 1);
    l_r[hh] += __shfl_xor_sync(0xffffffffu, l_r[hh], 2);
  }
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    int h = warp * 16 + (lane >> 2) + hh * 8;
    if (h >= a.h_loc) continue;
    float* op = a.o_part + ((long)unit * a.h_loc + h) * W_LAT;
#pragma unroll
    for (int i = 0; i < NT_O; ++i)
      *reinterpret_cast<float2*>(op + i * 8 + (lane & 3) * 2) = make_float2(o[i][2 * hh], o[i][2 * hh + 1]);
    if ((lane & 3) == 0) {
      float* ml = a.ml_part + ((long)unit * a.h_loc + h) * 2;
      ml[0] = m_r[hh];
      ml[1] = l_r[hh];
    }
  }
}

template <int W_LAT, int D_R>
cudaError_t launch_attn_t(const AttnArgs& a, int B, cudaStream_t s) {
  constexpr int WP = W_LAT + D_R + 8;
  int nwarps = (a.h_loc + 15) / 16;
  size_t smem = size_t(nwarps * 16 + 2 * TILE) * WP * 2;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_mma_kernel<W_LAT, D_R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  dim3 grid(a.n_split, B);
  KernelScope ks("K3_attn_mma", s);
  return launch_k(attn_mma_kernel<W_LAT, D_R>, grid, nwarps * 32, smem, s, a);
}

// K4: O = Σ_s 2^{m_s - M} O_s / Σ_s 2^{m_s - M} l_s
__global__ void combine_kernel(const float* __restrict__ o_part, const float* __restrict__ ml_part, int n_split,
                               int h_loc, int w_lat, uint16_t* __restrict__ o_bf16, float* __restrict__ o_f32,
                               float* __restrict__ lse) {
  pdl_trigger();
  pdl_wait();
  const int h = blockIdx.x, b = blockIdx.y;
  const long base = (long)b * n_split;
  float M = -INFINITY;
  for (int s = 0; s < n_split; ++s) M = fmaxf(M, ml_part[((base + s) * h_loc + h) * 2]);
  float L = 0.f;
  for (int s = 0; s < n_split; ++s) {
    const float* ml = ml_part + ((base + s) * h_loc + h) * 2;
    if (ml[1] > 0.f) L += exp2f(ml[0] - M) * ml[1];
  }
  const float inv = 1.f / L;
  for (int c = threadIdx.x * 4; c < w_lat; c += blockDim.x * 4) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < n_split; ++s) {
      const float* ml = ml_part + ((base + s) * h_loc + h) * 2;
      if (!(ml[1] > 0.f)) continue;            // empty split: weight 0 (reading R17)
      float w = exp2f(ml[0] - M);
      float4 v = *reinterpret_cast<const float4*>(o_part + ((base + s) * h_loc + h) * w_lat + c);
      acc.x += w * v.x; acc.y += w * v.y; acc.z += w * v.z; acc.w += w * v.w;
    }
    acc.x *= inv; acc.y *= inv; acc.z *= inv; acc.w *= inv;
    const long off = ((long)b * h_loc + h) * w_lat + c;
    if (o_f32) *reinterpret_cast<float4*>(o_f32 + off) = acc;
    if (o_bf16) {
      uint2 u;
      u.x = pack_bf16(acc.x, acc.y);
      u.y = pack_bf16(acc.z, acc.w);
      *reinterpret_cast<uint2*>(o_bf16 + off) = u;
    }
  }
  if (lse && threadIdx.x == 0) lse[(long)b * h_loc + h] = (M + log2f(L)) * 0.69314718055994531f;
}

}  // namespace

cudaError_t launch_decode_attn(const Geom& g, const tpla_cache& cache, const uint16_t* q_lat, const uint16_t* q_pe,
                               const int32_t* seq_lens, int B, const SplitPlan& sp, float* o_part, float* ml_part,
                               cudaStream_t s) {
  AttnArgs a;
  a.q_lat = q_lat; a.q_pe = q_pe; a.cache = static_cast<const uint16_t*>(cache.base);
  a.block_table = cache.block_table; a.seq_lens = seq_lens; a.o_part = o_part; a.ml_part = ml_part;
  a.h_loc = g.h_loc; a.h_q = g.h_q; a.head_begin = g.head_begin; a.page_size = cache.page_size;
  a.max_pages = cache.max_pages_per_seq; a.row_stride = cache.row_stride; a.n_split = sp.n_split; a.chunk = sp.chunk;
  a.scale_log2 = g.sm_scale * 1.4426950408889634f;
  const int key = g.w_lat * 1000 + g.d_r;
  switch (key) {
    case 32 * 1000 + 16: return launch_attn_t<32, 16>(a, B, s);
    case 64 * 1000 + 16: return launch_attn_t<64, 16>(a, B, s);
    case 32 * 1000 + 64: return launch_attn_t<32, 64>(a, B, s);
    case 64 * 1000 + 64: return launch_attn_t<64, 64>(a, B, s);
    case 128 * 1000 + 64: return launch_attn_t<128, 64>(a, B, s);
    case 256 * 1000 + 64: return launch_attn_t<256, 64>(a, B, s);
  }
  return cudaErrorNotSupported;
}

cudaError_t launch_combine(const Geom& g, int B, const SplitPlan& sp, const float* o_part, const float* ml_part,
                           uint16_t* o_bf16, float* o_f32, float* lse, cudaStream_t s) {
  dim3 grid(g.h_loc, B);
  int threads = std::min(64, std::max(32, g.w_lat / 4));
  KernelScope ks("K4_combine", s);
  return launch_k(combine_kernel, grid, threads, 0, s, o_part, ml_part, sp.n_split, g.h_loc, g.w_lat, o_bf16,
                  o_f32, lse);
}

}  // namespace tpla
