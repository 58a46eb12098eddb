// K4 + K5a fused — split-K combine of the persistent K3's segment partials and the per-head
// W^UV product, for one head per CTA:
//   O_j[b, h, :] = Σ_s 2^{m_s - M} O_s / Σ_s 2^{m_s - M} l_s          (flash-decoding merge)
//   v[b, h, :]   = O_j[b, h, :] · W^UV'_j[h]ᵀ                         (W^VO kept factored)
// The combined rows never leave shared memory (bf16 A tile), W^UV'_j[h] is staged with
// cp.async, and the [B x W_lat] x [W_lat x d_h] product runs on mma.sync (it is ~1 MFLOP per
// head: the kernel is bound by reading the partials and the 64 KB weight slice).
#include <math.h>

#include "common.cuh"
#include "internal.h"

namespace tpla {
namespace {

constexpr int kMB = 16;     // batch rows per CTA (grid = heads x ceil(B/16))
constexpr int kThreads = 32 * kMB;   // one warp per row: the merge is load-latency bound, so every
                                     // row's segment loads are in flight at once

struct FArgs {
  const float* o_part;      // [segs, H_loc, W_lat]
  const float* ml_part;     // [segs, H_loc, 2]
  const int32_t* meta;      // [B, 2] first / last segment of each sequence
  const uint16_t* W_UV;     // [H_loc, d_h, W_lat]
  uint16_t* v;              // [B * n_q, H_loc * d_h]
  int B, h_loc, w_lat, d_h;
  int n_q;                  // query tokens per sequence: output row b' = b * n_q + i, partial row i * H_loc + h
  float* v_acc;             // or null: fp32 v written (v_acc_add: added) instead of v, in v_chunks
  int v_acc_add, v_chunks;  // column chunks [v_chunks][B * n_q][H_loc * d_h / v_chunks]
};

__global__ void __launch_bounds__(kThreads) combine_wuv_kernel(FArgs a) {
  pdl_trigger();
  extern __shared__ __align__(128) uint16_t smem[];
  __shared__ float s_w[kMB][32];                    // per-row segment weights 2^(m_s - M)
  const int h = blockIdx.x;
  const int WP = a.w_lat + 8;                       // padded rows: conflict-free ldmatrix
  uint16_t* sW = smem;                              // [d_h][WP]
  uint16_t* sA = smem + a.d_h * WP;                 // [kMB][WP]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // W^UV'_j[h] -> smem (does not depend on the predecessor: issue before the PDL wait)
  const uint16_t* wsrc = a.W_UV + (long)h * a.d_h * a.w_lat;
  const int chunks = a.d_h * (a.w_lat / 8);
  for (int c = tid; c < chunks; c += kThreads) {
    const int r = c / (a.w_lat / 8), ch = c % (a.w_lat / 8);
    cp_async16(sW + r * WP + ch * 8, wsrc + (long)r * a.w_lat + ch * 8, true);
  }
  cp_async_commit();
  pdl_wait();

  const int n_warps_n = a.d_h / 32;                 // warps along d_h (32 columns each)
  {
    const int m0 = blockIdx.y * kMB;
    // ---- combine: warp w merges rows b = m0 + w, m0 + w + 8, ...
    const int n_rows = a.n_q * a.h_loc;             // partial rows per segment
    for (int bi = warp; bi < kMB; bi += kThreads / 32) {
      const int bq = m0 + bi;                       // output row (sequence b, token i)
      const int b = bq / a.n_q, prow = (bq % a.n_q) * a.h_loc + h;
      uint16_t* arow = sA + bi * WP;
      if (bq >= a.B * a.n_q) {
        for (int c = lane * 8; c < a.w_lat; c += 256) *reinterpret_cast<uint4*>(arow + c) = make_uint4(0, 0, 0, 0);
        continue;
      }
      const int s0 = a.meta[2 * b], s1 = a.meta[2 * b + 1];
      float M = -INFINITY;
      for (int s = s0 + lane; s <= s1; s += 32) M = fmaxf(M, a.ml_part[((long)s * n_rows + prow) * 2]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
      float L = 0.f;
      for (int s = s0 + lane; s <= s1; s += 32) {
        const float* ml = a.ml_part + ((long)s * n_rows + prow) * 2;
        const float w = exp2f(ml[0] - M);
        if (s - s0 < 32) s_w[warp][s - s0] = w;         // first 32 segment weights, for the merge
        L += w * ml[1];
      }
      __syncwarp();
      L = warp_sum(L);
      const float inv = 1.f / L;
      for (int c = lane * 8; c < a.w_lat; c += 256) {
        float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll 8
        for (int s = s0; s <= s1; ++s) {
          // (lanes past W_lat have left this loop: no warp-collective ops in here)
          const float wgt = s - s0 < 32 ? s_w[warp][s - s0] : exp2f(a.ml_part[((long)s * n_rows + prow) * 2] - M);
          const float4* src = reinterpret_cast<const float4*>(a.o_part + ((long)s * n_rows + prow) * a.w_lat + c);
          const float4 x0 = src[0], x1 = src[1];
          acc[0] += wgt * x0.x; acc[1] += wgt * x0.y; acc[2] += wgt * x0.z; acc[3] += wgt * x0.w;
          acc[4] += wgt * x1.x; acc[5] += wgt * x1.y; acc[6] += wgt * x1.z; acc[7] += wgt * x1.w;
        }
        uint4 u;
        u.x = pack_bf16(acc[0] * inv, acc[1] * inv);
        u.y = pack_bf16(acc[2] * inv, acc[3] * inv);
        u.z = pack_bf16(acc[4] * inv, acc[5] * inv);
        u.w = pack_bf16(acc[6] * inv, acc[7] * inv);
        *reinterpret_cast<uint4*>(arow + c) = u;
      }
    }
    cp_async_wait<0>();
    __syncthreads();
    // ---- v[m0.., h, :] = A [32 x W_lat] · W^UVᵀ: warp (mw, nw) owns rows 16*mw.. and columns 32*nw..
    for (int task = warp; task < n_warps_n; task += kThreads / 32) {
      const int mw = 0, nw = task;
      float acc[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
      for (int k0 = 0; k0 < a.w_lat; k0 += 16) {
        uint32_t af[4];
        ldmatrix_x4(af[0], af[1], af[2], af[3],
                    smem_u32(sA + (mw * 16 + (lane & 15)) * WP + k0 + ((lane >> 4) << 3)));
#pragma unroll
        for (int nj = 0; nj < 2; ++nj) {
          uint32_t b0, b1, b2, b3;
          const int r = nw * 32 + nj * 16 + (lane & 7) + ((lane >> 4) << 3);
          ldmatrix_x4(b0, b1, b2, b3, smem_u32(sW + r * WP + k0 + (((lane >> 3) & 1) << 3)));
          uint32_t bb0[2] = {b0, b1}, bb1[2] = {b2, b3};
          mma_bf16_16816(acc[2 * nj], af, bb0);
          mma_bf16_16816(acc[2 * nj + 1], af, bb1);
        }
      }
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int b = m0 + mw * 16 + (lane >> 2) + hh * 8;
          const int e = nw * 32 + ni * 8 + (lane & 3) * 2;
          if (b < a.B * a.n_q) {
            if (a.v_acc) {                          // (each element has exactly one writer: no atomics)
              const int kc = a.h_loc * a.d_h / a.v_chunks, c = h * a.d_h + e;   // (kc even: e, c even)
              const long idx = (long(c / kc) * a.B * a.n_q + b) * kc + c % kc;
              float2 o = make_float2(acc[ni][2 * hh], acc[ni][2 * hh + 1]);
              if (a.v_acc_add) {
                const float2 p = *reinterpret_cast<const float2*>(a.v_acc + idx);
                o.x += p.x;
                o.y += p.y;
              }
              *reinterpret_cast<float2*>(a.v_acc + idx) = o;
            } else {
              const long idx = (long)b * a.h_loc * a.d_h + h * a.d_h + e;
              *reinterpret_cast<uint32_t*>(a.v + idx) = pack_bf16(acc[ni][2 * hh], acc[ni][2 * hh + 1]);
            }
          }
        }
    }
    __syncthreads();
  }
}

}  // namespace

bool combine_wuv_supported(const Geom& g) { return g.d_h % 32 == 0 && g.w_lat % 64 == 0 && g.w_lat <= 512; }

cudaError_t launch_combine_wuv(const Geom& g, int B, int n_q, const float* o_part, const float* ml_part,
                               const int32_t* meta, const uint16_t* W_UV, uint16_t* v, cudaStream_t s,
                               float* v_acc, bool v_acc_add, int v_chunks) {
  FArgs a{o_part, ml_part, meta, W_UV, v, B, g.h_loc, g.w_lat, g.d_h, n_q, v_acc, v_acc_add ? 1 : 0, v_chunks};
  const size_t smem = size_t(g.d_h + kMB) * (g.w_lat + 8) * 2;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(combine_wuv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  KernelScope ks("K45_combine_W_UV", s);
  return launch_k(combine_wuv_kernel, dim3(g.h_loc, (B * n_q + kMB - 1) / kMB), kThreads, smem, s, a);
}

}  // namespace tpla
