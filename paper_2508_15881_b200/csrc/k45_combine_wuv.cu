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
constexpr int kSegBatch = 4;        // segments (O row + (m, l)) in flight per lane

struct FArgs {
  const uint16_t* o_part;   // fp16 [segs, n_q * H_loc, W_lat]: normalised partials O_s / l_s
  const float* ml_part;     // [segs, H_loc, 2]
  const int32_t* meta;      // [B, 2] first / last segment of each sequence
  const uint16_t* W_UV;     // [H_loc, d_h, W_lat]
  uint16_t* v;              // [B * n_q, H_loc * d_h]
  int B, h_loc, w_lat, d_h;
  int n_q;                  // query tokens per sequence: output row b' = b * n_q + i, partial row i * H_loc + h
  float* v_acc;             // or null: fp32 v written (v_acc_add: added) instead of v, in v_chunks
  int v_acc_add, v_chunks;  // column chunks [v_chunks][B * n_q][H_loc * d_h / v_chunks]
};

__global__ void __launch_bounds__(kThreads, 2) combine_wuv_kernel(FArgs a) {
  pdl_trigger();
  extern __shared__ __align__(128) uint16_t smem[];
  __shared__ float s_ml[kMB][2];                   // per-warp (M, L) of a split row (wpr > 1)
  const int h = blockIdx.x;
  const int WP = a.w_lat + 8;                       // padded rows: conflict-free ldmatrix
  uint16_t* sW = smem;                              // [d_h][WP]
  uint16_t* sA = smem + a.d_h * WP;                 // [kMB][WP]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // W^UV'_j[h] -> smem (does not depend on the predecessor: issue before the PDL wait)
  const uint16_t* wsrc = a.W_UV + (long)h * a.d_h * a.w_lat;
  // (16-byte chunks per weight row: a power of two for every W_lat = d_c / g, so shifts instead of
  // integer divisions — the division loop had been ~30 % of the kernel's instructions, ncu source)
  const int cpr = a.w_lat / 8, chunks = a.d_h * cpr;
  if ((cpr & (cpr - 1)) == 0) {
    const int sh = __ffs(cpr) - 1;
    for (int c = tid; c < chunks; c += kThreads) {
      const int r = c >> sh, ch = c & (cpr - 1);
      cp_async16(sW + r * WP + ch * 8, wsrc + (long)r * a.w_lat + ch * 8, true);
    }
  } else {
    for (int c = tid; c < chunks; c += kThreads) {
      const int r = c / cpr, ch = c % cpr;
      cp_async16(sW + r * WP + ch * 8, wsrc + (long)r * a.w_lat + ch * 8, true);
    }
  }
  cp_async_commit();
  pdl_wait();

  {
    const int m0 = blockIdx.y * kMB;
    // ---- combine.  The CTA's R_c rows share the 16 warps: wpr = 16 / pow2ceil(R_c) warps per row (one
    // at B >= 16; all 16 for a single sequence, whose K3 segments number up to the grid size).  A row of
    // W_lat fp32 is split over lpr lanes of 8 columns (two passes at W_lat = 512); the 32 / lpr lane
    // groups of each of the row's wpr warps take every NG-th segment, NG = wpr * 32 / lpr, in batches of
    // kSegBatch independent loads (the merge is bound by load latency).  Groups merge by shuffles in a
    // warp, then (wpr > 1) through shared memory.
    const int n_rows = a.n_q * a.h_loc;             // partial rows per segment
    const int lpr = a.w_lat / 8 < 32 ? a.w_lat / 8 : 32, sp = 32 / lpr;
    const int sub = lane / lpr, cl = lane % lpr;
    const int R_c = min(kMB, a.B * a.n_q - m0);
    int rp = 1;
    while (rp < R_c) rp <<= 1;
    const int wpr = kMB / rp, bi = warp / wpr, part = warp % wpr, NG = wpr * sp, G = part * sp + sub;
    float* scr = reinterpret_cast<float*>(sA + kMB * WP);   // [16 warps][W_lat] fp32 (wpr > 1)
    for (int r = R_c + warp; r < kMB; r += kThreads / 32)    // rows past B * n_q: zero A rows
      for (int c = lane * 8; c < a.w_lat; c += 256) *reinterpret_cast<uint4*>(sA + r * WP + c) = make_uint4(0, 0, 0, 0);
    if (bi < R_c) {
      const int bq = m0 + bi;                       // output row (sequence b, token i)
      const int b = bq / a.n_q, prow = (bq % a.n_q) * a.h_loc + h;
      uint16_t* arow = sA + bi * WP;
      const int s0 = a.meta[2 * b], s1 = a.meta[2 * b + 1];
      // Online merge (running max, as in the attention itself): a segment's (m, l) and its O row are
      // loaded together, so one batch of kSegBatch segments is one round trip.
      const float2* mlp = reinterpret_cast<const float2*>(a.ml_part);
      for (int c0 = 0; c0 < a.w_lat; c0 += lpr * 8) {
        const int c = c0 + cl * 8;
        float M = -INFINITY, L = 0.f;
        float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        for (int sb = s0 + G; sb <= s1; sb += kSegBatch * NG) {
          uint4 x[kSegBatch];                         // 8 fp16 of Ô_s = O_s / l_s
          float2 ml[kSegBatch];
#pragma unroll
          for (int i = 0; i < kSegBatch; ++i) {       // past s1: reload s1 (no divergent loads), weight 0
            const int sg = sb + i * NG, sc = sg <= s1 ? sg : s1;
            x[i] = *reinterpret_cast<const uint4*>(a.o_part + ((long)sc * n_rows + prow) * a.w_lat + c);
            ml[i] = mlp[(long)sc * n_rows + prow];
          }
          float Mn = M;
#pragma unroll
          for (int i = 0; i < kSegBatch; ++i)
            if (sb + i * NG <= s1) Mn = fmaxf(Mn, ml[i].x);
          const float r = exp2f(M - Mn);              // (M = -inf on the first batch: 0; Mn is finite)
          L *= r;
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[e] *= r;
#pragma unroll
          for (int i = 0; i < kSegBatch; ++i) {
            const float wl = (sb + i * NG <= s1 ? exp2f(ml[i].x - Mn) : 0.f) * ml[i].y;   // 2^(m_s - M) l_s
            L += wl;
            acc[0] += wl * f16_lo(x[i].x); acc[1] += wl * f16_hi(x[i].x);
            acc[2] += wl * f16_lo(x[i].y); acc[3] += wl * f16_hi(x[i].y);
            acc[4] += wl * f16_lo(x[i].z); acc[5] += wl * f16_hi(x[i].z);
            acc[6] += wl * f16_lo(x[i].w); acc[7] += wl * f16_hi(x[i].w);
          }
          M = Mn;
        }
        if (sp > 1) {                                 // merge the lane groups of this warp
          float Mg = M;
#pragma unroll
          for (int o = lpr; o < 32; o <<= 1) Mg = fmaxf(Mg, __shfl_xor_sync(0xffffffffu, Mg, o));
          const float f = M == -INFINITY ? 0.f : exp2f(M - Mg);   // (a group without segments)
          L *= f;
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[e] *= f;
#pragma unroll
          for (int o = lpr; o < 32; o <<= 1) {
            L += __shfl_xor_sync(0xffffffffu, L, o);
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], o);
          }
          M = Mg;
        }
        if (wpr > 1) {                                // this warp's share, unnormalised, for the row's merge
          if (sub == 0) {
            float4* d = reinterpret_cast<float4*>(scr + warp * a.w_lat + c);
            d[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
            d[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
          }
          if (lane == 0) { s_ml[warp][0] = M; s_ml[warp][1] = L; }
          continue;
        }
        const float inv = 1.f / L;
        if (sub == 0) {
          uint4 u;
          u.x = pack_bf16(acc[0] * inv, acc[1] * inv);
          u.y = pack_bf16(acc[2] * inv, acc[3] * inv);
          u.z = pack_bf16(acc[4] * inv, acc[5] * inv);
          u.w = pack_bf16(acc[6] * inv, acc[7] * inv);
          *reinterpret_cast<uint4*>(arow + c) = u;
        }
      }
    }
    if (wpr > 1) {                                    // (CTA-uniform) merge the row's wpr warps, in warp order
      __syncthreads();
      if (bi < R_c && part == 0) {
        float Mg = -INFINITY;
        for (int p = 0; p < wpr; ++p) Mg = fmaxf(Mg, s_ml[warp + p][0]);
        // lane p < wpr: warp p's weight 2^(M_p - M), broadcast by shuffles below
        const float Mp = lane < wpr ? s_ml[warp + lane][0] : -INFINITY;
        const float fl = Mp == -INFINITY ? 0.f : exp2f(Mp - Mg);
        const float L = warp_sum(lane < wpr ? fl * s_ml[warp + lane][1] : 0.f);
        const float inv = 1.f / L;
        float4 o[4];                                  // columns lane * 4 + 128 j (W_lat <= 512)
#pragma unroll
        for (int j = 0; j < 4; ++j) o[j] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int p = 0; p < wpr; ++p) {
          const float fp = __shfl_sync(0xffffffffu, fl, p);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int c = lane * 4 + 128 * j;
            if (c < a.w_lat) {
              const float4 x = *reinterpret_cast<const float4*>(scr + (warp + p) * a.w_lat + c);
              o[j].x += fp * x.x; o[j].y += fp * x.y; o[j].z += fp * x.z; o[j].w += fp * x.w;
            }
          }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int c = lane * 4 + 128 * j;
          if (c < a.w_lat)
            *reinterpret_cast<uint2*>(sA + bi * WP + c) = make_uint2(pack_bf16(o[j].x * inv, o[j].y * inv),
                                                                     pack_bf16(o[j].z * inv, o[j].w * inv));
        }
      }
    }
    cp_async_wait<0>();
    __syncthreads();
    // ---- v[m0.., h, :] = A [16 x W_lat] · W^UVᵀ: warp w owns the 8 columns 8w.. (m16n8k16, full K)
    for (int nw = warp; nw < a.d_h / 8; nw += kThreads / 32) {
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      const uint16_t* brow = sW + (nw * 8 + (lane & 7)) * WP + (((lane >> 3) & 1) << 3);
      const uint16_t* arow = sA + (lane & 15) * WP + ((lane >> 4) << 3);
#pragma unroll 4
      for (int k0 = 0; k0 < a.w_lat; k0 += 16) {
        uint32_t af[4], bf[2];
        ldmatrix_x4(af[0], af[1], af[2], af[3], smem_u32(arow + k0));
        ldmatrix_x2(bf[0], bf[1], smem_u32(brow + k0));
        mma_bf16_16816(acc, af, bf);
      }
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int b = m0 + (lane >> 2) + hh * 8;
        const int e = nw * 8 + (lane & 3) * 2;
        if (b < a.B * a.n_q) {
          if (a.v_acc) {                            // (each element has exactly one writer: no atomics)
            const int kc = a.h_loc * a.d_h / a.v_chunks, c = h * a.d_h + e;   // (kc even: e, c even)
            const int cq = (kc & (kc - 1)) == 0 ? c >> (__ffs(kc) - 1) : c / kc;
            const long idx = (long(cq) * a.B * a.n_q + b) * kc + (c - cq * kc);
            float2 o = make_float2(acc[2 * hh], acc[2 * hh + 1]);
            if (a.v_acc_add) {
              const float2 p = *reinterpret_cast<const float2*>(a.v_acc + idx);
              o.x += p.x;
              o.y += p.y;
            }
            *reinterpret_cast<float2*>(a.v_acc + idx) = o;
          } else {
            const long idx = (long)b * a.h_loc * a.d_h + h * a.d_h + e;
            *reinterpret_cast<uint32_t*>(a.v + idx) = pack_bf16(acc[2 * hh], acc[2 * hh + 1]);
          }
        }
      }
    }
  }
}

}  // namespace

bool combine_wuv_supported(const Geom& g) { return g.d_h % 8 == 0 && g.w_lat % 64 == 0 && g.w_lat <= 512; }

cudaError_t launch_combine_wuv(const Geom& g, int B, int n_q, const uint16_t* o_part, const float* ml_part,
                               const int32_t* meta, const uint16_t* W_UV, uint16_t* v, cudaStream_t s,
                               float* v_acc, bool v_acc_add, int v_chunks) {
  FArgs a{o_part, ml_part, meta, W_UV, v, B, g.h_loc, g.w_lat, g.d_h, n_q, v_acc, v_acc_add ? 1 : 0, v_chunks};
  const size_t smem = size_t(g.d_h + kMB) * (g.w_lat + 8) * 2 + size_t(kMB) * g.w_lat * 4;
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
