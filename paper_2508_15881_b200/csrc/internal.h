// Internal interface between the C-ABI layer (tpla_abi.cpp) and the CUDA kernels.
// Not installed; the public surface is include/tpla.h.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>

#include "../../include/tpla.h"

namespace tpla {

extern std::atomic<int64_t> g_launches;
extern std::atomic<int> g_profile_on;
extern thread_local bool g_no_pdl_next;   // next launch without PDL (common.cuh)

// Wraps one kernel launch: counts it (tpla_launch_count) and, when profiling is enabled
// (tpla_profile_enable), brackets it with CUDA events on the launching stream.
struct KernelScope {
  KernelScope(const char* name, cudaStream_t s);
  ~KernelScope();
  int slot = -1;
  cudaStream_t stream;
  const char* name_;
};

// Resolved per-device problem geometry (validated).
struct Geom {
  int h_q, d_c, d_r, d_h, D;
  int k, g, rank;
  int h_loc, w_lat, W;          // W = w_lat + d_r
  int head_begin, lat_begin;
  float eps, sm_scale;
};

// Split-K work decomposition of K3.
struct SplitPlan {
  int n_split;      // splits per sequence
  int chunk;        // tokens per split (multiple of 64)
};

// Workspace layout of tpla_decode (byte offsets, all 256-aligned).
struct WsLayout {
  size_t q_lat;     // bf16 [B, H_loc, W_lat]   (Q'_j)
  size_t o_part;    // split-K partials: fp32 [B*n_split, H_loc, W_lat] (mma.sync K3), fp16 [segs, ...] (tcgen05 K3)
  size_t ml_part;   // fp32 [B*n_split, H_loc, 2] (m, l)
  size_t o_lat;     // bf16 [B, H_loc, W_lat]   (combined O_j)
  size_t v;         // bf16 [B, H_loc*d_h]
  size_t y_part;    // fp32 [kslices, B, D]
  size_t meta;      // int32 [B, 2] (persistent K3: first segment id, count)
  size_t plan;      // int32 K3p schedule (attn_plan_bytes)
  size_t wo_part;   // persistent W^O GEMM partials + segment map
  size_t total;
  int kslices;
  int n_cta;        // persistent K3 grid
};

SplitPlan choose_split(int B, int max_seq_len);
WsLayout ws_layout(const Geom& g, int B, int n_q, int max_seq_len);

// ---- kernels (each returns cudaGetLastError() after launch) ----
// n_norm > 0: "norm only" rows: the g = 1 row normalised per slice (n_norm slices, alpha_s host)
cudaError_t launch_append_kv(const Geom& g, int xform_kind, const float* xform, float alpha_j,
                             const tpla_cache& cache, const uint16_t* c_kv, const uint16_t* k_pe,
                             const int32_t* seq_idx, const int32_t* pos, int n, int rms_mode,
                             int32_t* n_dropped, cudaStream_t s, int n_norm = 0, const float* alpha_s = nullptr);

// out[b, h, r] = sum_c W[h, r, c] * x[b, h, c]     (K2 with R=W_lat,C=d_h; K5a with R=d_h,C=W_lat)
// x has row stride x_head_stride elements between heads and x_batch_stride between batches.
// inputs_from_host: x/W are not written by the preceding kernel (PDL: overlap it, wait at the end)
cudaError_t launch_head_gemv(const char* name, const uint16_t* W, const uint16_t* x, long x_batch_stride, int H,
                             int R, int C, int B, uint16_t* out_bf16, bool inputs_from_host, cudaStream_t s);

cudaError_t launch_decode_attn(const Geom& g, const tpla_cache& cache, const uint16_t* q_lat,
                               const uint16_t* q_pe, const int32_t* seq_lens, int B, const SplitPlan& sp,
                               float* o_part, float* ml_part, cudaStream_t s);

cudaError_t launch_combine(const Geom& g, int B, const SplitPlan& sp, const float* o_part, const float* ml_part,
                           uint16_t* o_bf16, float* o_f32, float* lse, cudaStream_t s);

// Blackwell-native K3 (tcgen05/TMEM/TMA, persistent) and its segment combine.
bool tc_attention_supported(const Geom& g, int B);
// persistent K3 grid in logical CTAs (a logical CTA is a cluster of two for W_lat = 512)
int tc_num_ctas(const Geom& g, int B, int max_seq_len);
// n_q query tokens per sequence (multi-token decode): MMA rows = n_q * H_loc <= 128
// K3p: the persistent K3's schedule (every CTA's tile range, segment base, first 32 box rows), computed
// by one CTA from seq_lens and the block table ahead of K2; `plan`: attn_plan_bytes(n_cta, B) bytes
size_t attn_plan_bytes(int n_cta, int B);
cudaError_t launch_attn_plan(const Geom& g, const tpla_cache& cache, const int32_t* seq_lens, int B, int n_cta,
                             int32_t* plan, cudaStream_t s);
// K3p + K2 fused (one launch): the schedule as launch_attn_plan, and Q'_j = W^UK'_j q (TMA-staged
// per (head, 32 rows)); q_nope [R, h_q*d_h] all heads, W_UK [H_loc, W_lat, d_h], q_lat [R, H_loc, W_lat]
bool pre_attn_supported(const Geom& g);
cudaError_t launch_pre_attn(const Geom& g, const tpla_cache& cache, const int32_t* seq_lens, int B, int n_cta,
                            int32_t* plan, const uint16_t* W_UK, const uint16_t* q_nope, int R, uint16_t* q_lat,
                            cudaStream_t s);
cudaError_t launch_decode_attn_tc(const Geom& g, const tpla_cache& cache, const uint16_t* q_lat, const uint16_t* q_pe,
                                  const int32_t* seq_lens, int B, int n_q, int n_cta, const int32_t* plan,
                                  uint16_t* o_part, float* ml_part, int32_t* meta, cudaStream_t s);
// (o_part of the persistent K3: fp16 [segs, n_q * H_loc, W_lat] normalised partials O_s / l_s; ml_part (m_s, l_s))
cudaError_t launch_combine_seg(const Geom& g, int B, const uint16_t* o_part, const float* ml_part, const int32_t* meta,
                               uint16_t* o_bf16, float* o_f32, float* lse, cudaStream_t s);

// K4 + K5a fused (persistent-K3 partials): v[b, h, :] = combine(partials)[b, h, :] · W^UV'_j[h]ᵀ
bool combine_wuv_supported(const Geom& g);
// v_acc != null: write (accumulate: add) v in fp32 there instead of bf16 v, column-chunk-major with
// v_chunks chunks: element (row b, col c) at ((c / kc) * B*n_q + b) * kc + c % kc, kc = H_loc*d_h / v_chunks
cudaError_t launch_combine_wuv(const Geom& g, int B, int n_q, const uint16_t* o_part, const float* ml_part,
                               const int32_t* meta, const uint16_t* W_UV, uint16_t* v, cudaStream_t s,
                               float* v_acc = nullptr, bool v_acc_add = false, int v_chunks = 1);

// y_part[ks, b, n] = sum_{k in slice ks} Wt[n, k] * v[b, k]; Wt [N, K] bf16, v [B, K] bf16.
cudaError_t launch_skinny_gemm(const uint16_t* Wt, const uint16_t* v, int N, int K, int B, int kslices,
                               float* y_part, cudaStream_t s);

// Blackwell-native W^O up-projection (tcgen05 + TMA, persistent split-K) with its segment reduce:
// y[b, n] (=|+=) Σ_k v[b, k] Wt[n, k].  part_ws: wo_tc_part_bytes(N, K, B) bytes of workspace.
bool wo_tc_supported(int N, int K, int B);
// W^O is stored blocked [ceil(D/128)][K/64][128][64] when 64 | K (the tcgen05 path), else [D, K]
inline bool wo_blocked(int K) { return K % 64 == 0; }
size_t wo_tc_part_bytes(int N, int K, int B);
// out_bf16 (optional): also write bf16(y) (the step's output when no all-reduce follows)
// [k_begin, k_begin + k_len): a 64-multiple slice of W^O's K rows (k_len 0 = all); v is then [B, k_len],
// the slice's columns only (a rank projecting its share of a v summed over the latent group)
// v_ld: v's row stride in elements (0: k_len, dense rows).  ar (optional): fuse the all-reduce into the
// segment reduce (FusedAr below); ar_row0: the first row of this launch in the symmetric buffer.
struct FusedAr;
cudaError_t launch_wo_tc(const uint16_t* Wt, const uint16_t* v, int N, int K, int B, void* part_ws, float* y,
                         bool accumulate, uint16_t* out_bf16, cudaStream_t s, int k_begin = 0, int k_len = 0,
                         long v_ld = 0, const FusedAr* ar = nullptr, long ar_row0 = 0);

// Fused W^O epilogue + one-shot all-reduce: the segment reduce of K5 writes this rank's
// Õ rows into a symmetric buffer (an NCCL window), every reduce CTA meets the same CTA of every peer at
// an LSA barrier, then sums the k ranks' rows — through the NVLS multicast address (multimem.ld_reduce)
// when the communicator has one, else by peer loads in rank order — into y (fp32) and the bf16 output.
// The buffer is double-buffered by the barrier epoch (a rank can be at most one call ahead of a peer).
constexpr int kArCtas = 128;          // reduce CTAs = LSA barriers of the device communicator
struct FusedAr {
  void* dev_comm;                     // ncclDevComm (host copy, passed by value to the kernel)
  void* window;                       // ncclWindow_t
  size_t half_elems;                  // fp32 elements per buffer half
  int multimem;                       // use the NVLS multicast address
};

// K8: causal prefill attention, non-absorbed MLA (k7_prefill_fa.cu).  q_nope [L, h_q*128] and q_pe
// [L, h_q*64] hold all heads (this device's head 0 is q_head0); K, V, O [L, H*128] bf16; k_pe rows of
// 64 with row stride kpe_ld elements.
cudaError_t launch_attn_fwd_causal(const uint16_t* q_nope, const uint16_t* q_pe, int h_q, int q_head0,
                                   const uint16_t* K, const uint16_t* V, int H, const uint16_t* k_pe, long kpe_ld,
                                   int L, float sm_scale, uint16_t* O, cudaStream_t s);
// K9: out[t, n] = Σ_k X[t, k] Wt[n, k] for t < L (X row stride ld_x; Wt blocked like W^O): fp32 y (=, or
// += with accumulate) and/or bf16 out, either may be null.  One CTA per [128 x 256] tile, full K.
bool gemm_tn_supported(int N, int K);
cudaError_t launch_gemm_tn(const uint16_t* Wt, const uint16_t* X, long ld_x, int N, int K, int L, float* y,
                           bool accumulate, uint16_t* out, cudaStream_t s);
// ĉ = c / sqrt(|c|^2 / d_c + eps) per row (the full RMS; gamma lives in the up-projection weights)
cudaError_t launch_prefill_rmsnorm(const uint16_t* c_kv, int L, int d_c, float eps, uint16_t* c_hat, cudaStream_t s);

// K6: page-table rows + lengths of the prefill pseudo-sequences (k6_prefill.cu)
cudaError_t launch_prefix_table(const int32_t* block_table, int seq, int max_pages, int n_full, int n_q, int r0,
                                int n_rows, int32_t* table, int32_t* lens, cudaStream_t s);

// y[b, n] (=|+=) sum_ks y_part[ks, b, n]
cudaError_t launch_reduce_slices(const float* y_part, int kslices, int B, int N, float* y, bool accumulate,
                                 cudaStream_t s);

cudaError_t launch_cast_bf16(const float* y, long n, uint16_t* out, cudaStream_t s, const char* name = "C1_cast_bf16");
// out = bf16(Σ_i src[i]) over n elements (n % 4 == 0), the sources added in list order (n_src <= 16)
constexpr int kMaxSumSrc = 16;
cudaError_t launch_sum_cast_bf16(const float* const* src, int n_src, long n, uint16_t* out, cudaStream_t s,
                                 const char* name = "K5_v_sum_cast");

}  // namespace tpla
