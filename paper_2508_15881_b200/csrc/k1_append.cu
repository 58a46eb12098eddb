// K1 — cache write (tpla_append_kv / tpla_prefill_mla).
//
// Per appended token (§4.1, §4.3):
//   c' = c U                      U = D H_{d_c}/sqrt(d_c) (FWHT) | PCA columns | I
//   r  = sqrt(alpha_j/d_c ||c'_j||^2 + eps)   (SLICED, Condition 1 chain P:205-209)
//      | sqrt(||c||^2/d_c + eps)               (EXACT, orthogonal U preserves the norm)
//   row = [bf16(c'_j / r) ‖ k^PE]  at (seq, pos) through the page table (k^PE replicated)
//
// One warp per row.  Lane l holds elements e = l*E + i (E = d_c/32) so the FWHT runs as
// log2(E) in-register butterfly stages plus 5 shfl.xor stages; the device's slice is a
// contiguous range of lanes and leaves as 16-byte stores.  Bound: latency (one row per
// sequence per decode step) — see DESIGN.md.
#include "common.cuh"
#include "internal.h"

namespace tpla {
namespace {

constexpr int kMaxNormSlices = 8;

struct AppendArgs {
  const uint16_t* c_kv;
  const uint16_t* k_pe;
  const int32_t* seq_idx;
  const int32_t* pos;
  const float* xform;
  uint16_t* base;
  const int32_t* block_table;
  int32_t* n_dropped;
  long num_pages;
  int n, d_c, d_r, w_lat, lat_begin, page_size, max_pages, row_stride, batch;
  int xform_kind, rms_mode;
  float alpha, eps;
  // "norm only": a g = 1 row normalised per slice — n_norm slices of d_c / n_norm
  // coordinates, slice s divided by sqrt(alpha_s / d_c ||c'_s||^2 + eps); 0 = off
  int n_norm;
  float alpha_s[kMaxNormSlices];
};

template <int E>
__device__ __forceinline__ void append_row(const AppendArgs& a);

template <int E>
__global__ void __launch_bounds__(128) append_kernel(AppendArgs a) {
  pdl_trigger();
  append_row<E>(a);   // loads and math under the predecessor's tail; waits before its first store
  pdl_wait();         // (threads without a row: keep completion transitive)
}

template <int E>
__device__ __forceinline__ void append_row(const AppendArgs& a) {
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (row >= a.n) return;
  const int seq = a.seq_idx[row];
  const int p = a.pos[row];
  int page = -1;
  if (seq >= 0 && seq < a.batch && p >= 0 && p < a.max_pages * a.page_size)
    page = a.block_table[(long)seq * a.max_pages + p / a.page_size];
  if (page < 0 || page >= a.num_pages) {
    pdl_wait();
    if (lane == 0 && a.n_dropped) atomicAdd(a.n_dropped, 1);
    return;
  }
  uint16_t* dst = a.base + ((long)page * a.page_size + (p % a.page_size)) * a.row_stride;
  const uint16_t* src = a.c_kv + (long)row * a.d_c;

  float x[E];
  if constexpr (E >= 8) {
#pragma unroll
    for (int v = 0; v < E / 8; ++v) {
      uint4 u = *reinterpret_cast<const uint4*>(src + lane * E + v * 8);
      uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) { x[v * 8 + 2 * q] = bf16_lo(w[q]); x[v * 8 + 2 * q + 1] = bf16_hi(w[q]); }
    }
  } else {
#pragma unroll
    for (int i = 0; i < E; ++i) x[i] = bf16f(src[lane * E + i]);
  }

  // full-row energy (= energy of c U for orthogonal U) for EXACT
  float ss_full = 0.f;
#pragma unroll
  for (int i = 0; i < E; ++i) ss_full += x[i] * x[i];
  ss_full = warp_sum(ss_full);

  const int W = a.w_lat;
  if (a.xform_kind == TPLA_XFORM_PCA) {
    // c'_j[l] = sum_i c_i U[i, lat_begin + l]; xform holds U[:, lat range] as [d_c, W_lat]
    extern __shared__ float sh[];
    float* c = sh + (threadIdx.x >> 5) * a.d_c;
#pragma unroll
    for (int i = 0; i < E; ++i) c[lane * E + i] = x[i];
    __syncwarp();
    // pass 1: slice energy; pass 2 recomputes the projection (keeps registers independent of W)
    float ss = 0.f;
    float ssn[kMaxNormSlices];                    // norm only: per-slice energies
#pragma unroll
    for (int q = 0; q < kMaxNormSlices; ++q) ssn[q] = 0.f;
    const int wn = a.n_norm > 0 ? W / a.n_norm : W;
    for (int l = lane; l < W; l += 32) {
      float acc = 0.f;
      for (int i = 0; i < a.d_c; ++i) acc = fmaf(c[i], a.xform[(long)i * W + l], acc);
      ss += acc * acc;
#pragma unroll
      for (int q = 0; q < kMaxNormSlices; ++q)
        if (q == l / wn) ssn[q] += acc * acc;
    }
    ss = warp_sum(ss);
    float rn[kMaxNormSlices];
#pragma unroll
    for (int q = 0; q < kMaxNormSlices; ++q)
      rn[q] = q < a.n_norm ? rsqrtf(a.alpha_s[q] / a.d_c * warp_sum(ssn[q]) + a.eps) : 1.f;
    float r;
    if (a.rms_mode == TPLA_RMS_SLICED) r = rsqrtf(a.alpha / a.d_c * ss + a.eps);
    else if (a.rms_mode == TPLA_RMS_EXACT) r = rsqrtf(ss_full / a.d_c + a.eps);
    else r = 1.f;
    pdl_wait();   // first store: the previous step's K3 may still read this row's 64-row box
    for (int l = lane; l < W; l += 32) {
      float acc = 0.f;
      for (int i = 0; i < a.d_c; ++i) acc = fmaf(c[i], a.xform[(long)i * W + l], acc);
      float rr = r;
#pragma unroll
      for (int q = 0; q < kMaxNormSlices; ++q)
        if (a.n_norm > 0 && q == l / wn) rr = rn[q];
      dst[l] = f2bf(acc * rr);
    }
  } else {
    if (a.xform_kind == TPLA_XFORM_HADAMARD) {
#pragma unroll
      for (int i = 0; i < E; ++i) x[i] *= a.xform[lane * E + i];      // D (left signs, reading R7)
#pragma unroll
      for (int h = 1; h < E; h <<= 1) {                               // in-lane butterflies
#pragma unroll
        for (int i = 0; i < E; ++i)
          if ((i & h) == 0) { float u = x[i], v = x[i + h]; x[i] = u + v; x[i + h] = u - v; }
      }
#pragma unroll
      for (int m = 1; m < 32; m <<= 1) {                              // cross-lane butterflies
        const bool upper = lane & m;
#pragma unroll
        for (int i = 0; i < E; ++i) {
          float y = __shfl_xor_sync(0xffffffffu, x[i], m);
          x[i] = upper ? (y - x[i]) : (x[i] + y);
        }
      }
      const float s = rsqrtf((float)a.d_c);
#pragma unroll
      for (int i = 0; i < E; ++i) x[i] *= s;
    }
    const int e0 = lane * E;
    const bool mine = e0 >= a.lat_begin && e0 < a.lat_begin + W;     // slice = whole lanes (g <= 32)
    float ss = 0.f;
    if (mine) {
#pragma unroll
      for (int i = 0; i < E; ++i) ss += x[i] * x[i];
    }
    float r;
    if (a.n_norm > 0) {                           // norm only: each slice's lanes reduce among themselves
      const int lanes = 32 / a.n_norm;            // (a power of two: aligned xor groups)
      for (int m = 1; m < lanes; m <<= 1) ss += __shfl_xor_sync(0xffffffffu, ss, m);
      r = rsqrtf(a.alpha_s[lane / lanes] / a.d_c * ss + a.eps);
    } else {
      ss = warp_sum(ss);
      if (a.rms_mode == TPLA_RMS_SLICED) r = rsqrtf(a.alpha / a.d_c * ss + a.eps);
      else if (a.rms_mode == TPLA_RMS_EXACT) r = rsqrtf(ss_full / a.d_c + a.eps);
      else r = 1.f;
    }
    pdl_wait();   // first store: the previous step's K3 may still read this row's 64-row box
    if (mine) {
      uint16_t* o = dst + (e0 - a.lat_begin);
      if constexpr (E >= 8) {
#pragma unroll
        for (int v = 0; v < E / 8; ++v) {
          uint4 u;
          u.x = pack_bf16(x[v * 8 + 0] * r, x[v * 8 + 1] * r);
          u.y = pack_bf16(x[v * 8 + 2] * r, x[v * 8 + 3] * r);
          u.z = pack_bf16(x[v * 8 + 4] * r, x[v * 8 + 5] * r);
          u.w = pack_bf16(x[v * 8 + 6] * r, x[v * 8 + 7] * r);
          *reinterpret_cast<uint4*>(o + v * 8) = u;
        }
      } else {
#pragma unroll
        for (int i = 0; i < E; ++i) o[i] = f2bf(x[i] * r);
      }
    }
  }
  // replicated RoPE key and zero padding up to the row stride
  const uint16_t* kp = a.k_pe + (long)row * a.d_r;
  for (int c = lane; c < a.row_stride - W; c += 32) dst[W + c] = (c < a.d_r) ? kp[c] : uint16_t(0);
}

template <int E>
cudaError_t launch_E(const AppendArgs& a, cudaStream_t s) {
  int blocks = (a.n + 3) / 4;
  size_t smem = (a.xform_kind == TPLA_XFORM_PCA) ? size_t(4) * a.d_c * sizeof(float) : 0;
  KernelScope ks("K1_append_kv", s);
  return launch_k(append_kernel<E>, blocks, 128, smem, s, a);
}

}  // namespace

cudaError_t launch_append_kv(const Geom& g, int xform_kind, const float* xform, float alpha_j,
                             const tpla_cache& cache, const uint16_t* c_kv, const uint16_t* k_pe,
                             const int32_t* seq_idx, const int32_t* pos, int n, int rms_mode,
                             int32_t* n_dropped, cudaStream_t s, int n_norm, const float* alpha_s) {
  AppendArgs a;
  a.n_norm = n_norm;
  for (int q = 0; q < kMaxNormSlices; ++q) a.alpha_s[q] = (n_norm > 0 && q < n_norm) ? alpha_s[q] : 1.f;
  a.c_kv = c_kv; a.k_pe = k_pe; a.seq_idx = seq_idx; a.pos = pos; a.xform = xform;
  a.base = static_cast<uint16_t*>(cache.base); a.block_table = cache.block_table; a.n_dropped = n_dropped;
  a.num_pages = cache.num_pages; a.n = n; a.d_c = g.d_c; a.d_r = g.d_r; a.w_lat = g.w_lat;
  a.lat_begin = g.lat_begin; a.page_size = cache.page_size; a.max_pages = cache.max_pages_per_seq;
  a.row_stride = cache.row_stride; a.batch = cache.batch; a.xform_kind = xform_kind; a.rms_mode = rms_mode;
  a.alpha = alpha_j; a.eps = g.eps;
  switch (g.d_c / 32) {
    case 1: return launch_E<1>(a, s);
    case 2: return launch_E<2>(a, s);
    case 4: return launch_E<4>(a, s);
    case 8: return launch_E<8>(a, s);
    case 16: return launch_E<16>(a, s);
    case 32: return launch_E<32>(a, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace tpla
