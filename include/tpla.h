/*
 * tpla.h — C ABI of libtpla.so, the B200 (sm_100a) decode hot path of
 * Tensor-Parallel Latent Attention (TPLA, arXiv 2508.15881).
 *
 * Citations: "P:n" = line n of the paper text, with its section.
 *
 * The path, per layer, per decode step, on each device (rank r of k):
 *   tpla_append_kv   K1  transform + (sliced) RMSNorm + slice + bf16 store  §4.1/§4.3
 *   tpla_decode      K2  Q'_j = q W^UK'_j^T (mu_j folded)                     §3.3/§4.2
 *                    K3  per-shard split-K flash decoding over [ĉ_j ‖ k^PE]  §4, Eq. tpla_softmax_one_device
 *                    K4  split-K combine
 *                    K5  Õ_j = O_j W^UV'_j W^O_rows                           §4; W^VO factored P:114
 *                    C1  O = AllReduce(Σ Õ_j)  (NCCL, sum, fp32)              §4
 *
 * Conventions (all entry points):
 *  - Every tensor argument is a plain pointer.  "device" pointers are CUDA
 *    device memory owned by the caller (the Python side allocates them with
 *    PyTorch); "host" pointers are ordinary host memory.  The library never
 *    allocates device memory on the decode path: scratch comes from the caller's
 *    workspace, sized by tpla_decode_workspace_bytes().  The only object the
 *    library owns is tpla_comm (an NCCL communicator).
 *  - bf16 tensors are passed as their 16-bit patterns (uint16).  Row-major,
 *    densely packed, 16-byte aligned base addresses, unless stated otherwise.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    All device work is asynchronous on that stream, NCCL included, so a whole
 *    decode step can be captured in a CUDA graph.
 *  - Every call returns a tpla_status.  Arguments are validated BEFORE any
 *    launch; on failure nothing is launched and tpla_last_error() (thread-local)
 *    explains.  Asynchronous CUDA faults are reported by the next call that
 *    synchronises (tpla_sync) as TPLA_ERR_CUDA.  No C++ exception crosses the ABI.
 */
#ifndef TPLA_H_
#define TPLA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t tpla_status;
enum {
  TPLA_OK = 0,
  TPLA_ERR_INVALID_ARG = 1,   /* NULL pointer, bad enum, misaligned pointer            */
  TPLA_ERR_SHAPE = 2,         /* dimension outside what the kernels support            */
  TPLA_ERR_DIVISIBILITY = 3,  /* g ∤ k, g ∤ d_c, (k/g) ∤ h_q, d_c not a power of two    */
  TPLA_ERR_CAPACITY = 4,      /* workspace too small, position beyond the page table    */
  TPLA_ERR_CUDA = 5,          /* CUDA runtime error (launch or asynchronous fault)      */
  TPLA_ERR_NCCL = 6,          /* NCCL unavailable or failed                             */
  TPLA_ERR_UNSUPPORTED = 7    /* valid request this build does not implement            */
};

/* Orthogonal transform U applied to the latent before slicing (§4.3). */
enum {
  TPLA_XFORM_IDENTITY = 0,  /* U = I ("Original" split, Fig. 3)                        */
  TPLA_XFORM_HADAMARD = 1,  /* U = D H_{d_c} / sqrt(d_c), D = diag(±1) from splitmix64 */
  TPLA_XFORM_PCA = 2        /* U = eigenvectors of the calibration second moment     */
};

/* How a cached row is normalised (§4.1). */
enum {
  TPLA_RMS_SLICED = 0,  /* sqrt(alpha_j/d_c ||(cU)_j||^2 + eps): the device's slice only */
  TPLA_RMS_EXACT = 1,   /* sqrt(||c||^2/d_c + eps): full-row RMS, PD-separated prefill  */
  TPLA_RMS_NONE = 2     /* no normalisation: layout tests (row = bf16 copy of (cU)_j)           */
};

/* tpla_decode flags */
enum {
  TPLA_DECODE_ACCUMULATE = 1,  /* y += Õ_j instead of y = Õ_j (single-GPU k-shard emulation)          */
  /* tpla_decode_v in two calls on the same workspace (a scheduler may issue the first early, on
   * another stream): STAGE_PRE = K3p + K2 only (the schedule and Q'_j), STAGE_ATTN = K3 + K4/K5a only
   * (requires the STAGE_PRE call with the same inputs to have completed).  Neither bit: both. */
  TPLA_DECODE_STAGE_PRE = 2,
  TPLA_DECODE_STAGE_ATTN = 4
};

/* Model + deployment.  Semantics: PAPER.md §3.1/§3.3 symbols; k devices, g latent groups (§4.4). */
typedef struct tpla_config {
  int32_t h_q;      /* query heads                                         */
  int32_t d_c;      /* latent width (4 d_h in the paper), power of 2 */
  int32_t d_r;      /* decoupled RoPE width, even                          */
  int32_t d_h;      /* head dim                                            */
  int32_t D;        /* hidden size                                         */
  int32_t k;        /* devices in the tensor-parallel group                */
  int32_t g;        /* latent groups; g | k, g | d_c, (k/g) | h_q          */
  int32_t rank;     /* this device, 0 <= rank < k                          */
  float eps;        /* RMSNorm epsilon                             */
  float sm_scale;   /* logit scale, one scalar for NoPE and RoPE   */
} tpla_config;

/* This device's share (group-major: shard j = rank / (k/g), head block i = rank % (k/g)). */
typedef struct tpla_device_plan {
  int32_t rank, shard, head_block;
  int32_t head_begin, head_end;   /* [i·H_loc, (i+1)·H_loc)                        */
  int32_t lat_begin, lat_end;     /* [j·W_lat, (j+1)·W_lat) of the TRANSFORMED basis */
  int32_t row_width;              /* W = W_lat + d_r (latent slice ‖ k^PE)  */
  int32_t h_loc, w_lat;
} tpla_device_plan;

/* Converted, device-resident weights of one device (caller-allocated device buffers). */
typedef struct tpla_weights {
  void* W_UK;         /* bf16 [H_loc, W_lat, d_h]: mu_j · (U^T W_γ W^UK)[lat rows, head h cols]   */
  void* W_UV;         /* bf16 [H_loc, d_h, W_lat]: (U^T W_γ W^UV)[lat rows, head h cols]^T         */
  void* W_O;          /* bf16 (W^O[head rows of block i, :])^T, K = H_loc·d_h: if 64 | K blocked
                         [ceil(D/128)][K/64][128][64] (rows >= D zero), else [D, K]               */
  void* xform;        /* fp32: HADAMARD [d_c] signs ±1; PCA [d_c, W_lat] = U[:, lat range]; else NULL */
  int32_t xform_kind; /* TPLA_XFORM_*                                                              */
  float alpha_j;      /* Condition 1 constant of this shard                     */
  float mu_j;         /* Condition 2 constant; already folded into W_UK             */
} tpla_weights;

/* Paged latent cache of one device: bf16 [num_pages, page_size, row_stride]; a token's row
 * holds [ĉ_j (W_lat) ‖ k^PE (d_r)] in columns [0, W) and zero padding up to row_stride.
 * Token t of sequence b lives in page block_table[b·max_pages_per_seq + t / page_size],
 * row t % page_size.  page_size is a multiple of 64; row_stride a multiple of 64 ≥ W.
 * Decode reads whole 64-row groups: rows of a sequence's last 64-row group beyond its length
 * are multiplied by a zero probability, so they must hold finite values (allocate pages
 * zero-filled, as the Python runtime does); their contents never reach the output. */
typedef struct tpla_cache {
  void* base;                  /* device bf16                                  */
  const int32_t* block_table;  /* device int32 [batch, max_pages_per_seq]      */
  int64_t num_pages;
  int32_t page_size;
  int32_t max_pages_per_seq;
  int32_t row_stride;          /* elements                                     */
  int32_t batch;               /* rows of block_table                          */
} tpla_cache;

typedef struct tpla_comm tpla_comm; /* opaque: NCCL communicator over the k devices */

/* ---- host-only helpers (no device work) ---------------------------------------- */

const char* tpla_version(void);
/* Thread-local message for the last non-OK status of this thread ("" if none). */
const char* tpla_last_error(void);
/* Number of kernels this library has launched in this process (monotone counter). */
int64_t tpla_launch_count(void);

/* Device plan of cfg->rank.  Pure integer arithmetic. */
tpla_status tpla_make_plan(const tpla_config* cfg, tpla_device_plan* out);

/* Hadamard sign diagonal D: out[i] = -1 if bit 63 of splitmix64 output i is set, else +1.
 * out: host fp32 [d]. */
tpla_status tpla_hadamard_signs(uint64_t seed, int32_t d, float* out);

/* PCA constants: alpha_j = Σ_all λ / Σ_{slice j} λ, λ in descending order.
 * lambda: host fp64 [d_c]; alpha_out: host fp32 [g]. */
tpla_status tpla_pca_alpha(const double* lambda, int32_t d_c, int32_t g, float* alpha_out);

/* Byte sizes of the four device buffers of tpla_weights for cfg->rank (xform = 0 for IDENTITY). */
tpla_status tpla_weights_bytes(const tpla_config* cfg, int32_t xform_kind, size_t* W_UK, size_t* W_UV,
                               size_t* W_O, size_t* xform);

/* ---- offline conversion ------------------------------- */

/* Absorb γ and U into W^UK/W^UV (W^UKV_new = U^T W_γ W^UKV), take this device's latent rows
 * and head block, fold mu_j into the W^UK slice, lay W^UV and W^O out K-major, round to bf16
 * (RNE) and copy into the caller's device buffers out->W_UK, W_UV, W_O, xform (already set).
 * Arithmetic in fp64 on the host.
 *   sign_seed  HADAMARD: seed of D;  U_pca  PCA: host fp32 [d_c, d_c] row-major, column c = c-th
 *   eigenvector (descending eigenvalue), else NULL;  alpha, mu: host fp32 [g];
 *   W_UK, W_UV: host bf16 [d_c, h_q·d_h]; gamma: host bf16 [d_c]; W_O: host bf16 [h_q·d_h, D].
 * Synchronous (returns after the copies completed on `stream`). */
tpla_status tpla_convert_weights(const tpla_config* cfg, int32_t xform_kind, uint64_t sign_seed,
                                 const float* U_pca, const float* alpha, const float* mu,
                                 const uint16_t* W_UK, const uint16_t* W_UV, const uint16_t* gamma,
                                 const uint16_t* W_O, tpla_weights* out, void* stream);

/* ---- K1: cache write ------------------------------------------------------------- */

/* Append n latent rows.  Row r: c' = c_kv[r]·U; keep (c')_j; normalise per rms_mode; store
 * bf16(ĉ_j) ‖ k_pe[r] at (seq_idx[r], pos[r]) through the page table.
 *   c_kv: device bf16 [n, d_c] raw (pre-RMSNorm) latents; k_pe: device bf16 [n, d_r] post-RoPE;
 *   seq_idx, pos: device int32 [n].  Out-of-range (seq, pos) rows are skipped by the kernel and
 *   counted in *n_dropped if n_dropped (device int32) is non-NULL. */
tpla_status tpla_append_kv(const tpla_config* cfg, const tpla_weights* w, const tpla_cache* cache,
                           const void* c_kv, const void* k_pe, const int32_t* seq_idx, const int32_t* pos,
                           int32_t n, int32_t rms_mode, int32_t* n_dropped, void* stream);

/* PD-separated prefill: the prompt rows are written to this device's
 * cache with the EXACT (unsliced) RMS, so decode reuses the MLA prefill cache.  q must be NULL:
 * the causal prefill attention is tpla_prefill_attention (returns TPLA_ERR_UNSUPPORTED otherwise). */
/* "Norm only" rows (Fig. 3 "TPLA (norm only)"): the ablation where the
 * RMSNorm is sliced but the softmax is not.  On one device holding the whole latent (cfg.g = 1), each
 * row c' = c U is cut into n_slices (1, 2, 4, 8) slices of d_c / n_slices coordinates and slice s is
 * divided by its own sliced RMS sqrt(alpha[s] / d_c ||c'_s||^2 + eps) (Condition 1 chain);
 * decoding these rows with the g = 1 kernels and mu = 1 sums the partial logits of the slices before
 * ONE softmax — exactly the all-gather-the-logits variant of P:469 (oracle tpla_decode_exact_logits).
 * alpha: host [n_slices].  Otherwise as tpla_append_kv. */
tpla_status tpla_append_kv_norm_only(const tpla_config* cfg, const tpla_weights* w, const tpla_cache* cache,
                                     const void* c_kv, const void* k_pe, const int32_t* seq_idx, const int32_t* pos,
                                     int32_t n, int32_t n_slices, const float* alpha, int32_t* n_dropped,
                                     void* stream);
tpla_status tpla_prefill_mla(const tpla_config* cfg, const tpla_weights* w, const tpla_cache* cache,
                             const void* c_kv, const void* k_pe, const int32_t* seq_idx, const int32_t* pos,
                             int32_t n, const void* q, void* stream);

/* ---- K2..K5 + C1: decode ---------------------------------------------------------- */

/* Workspace bytes for tpla_decode / tpla_decode_attention with batch B and at most
 * max_seq_len cached tokens per sequence. */
tpla_status tpla_decode_workspace_bytes(const tpla_config* cfg, int32_t B, int32_t max_seq_len, size_t* bytes);

/* One decode step of this device (K2, K3, K4, K5) + the all-reduce (C1).
 *   q_nope: device bf16 [B, h_q, d_h] and q_pe: device bf16 [B, h_q, d_r] hold ALL heads (the
 *   device reads its head block); seq_lens: device int32 [B], 1 <= seq_lens[b] <= max_seq_len,
 *   the number of cached tokens (the current token already appended);
 *   y: device fp32 [B, D]: receives Õ_j (or += with TPLA_DECODE_ACCUMULATE), then, if comm != NULL,
 *   is all-reduced in place (sum over the k devices);  out: device bf16 [B, D] or NULL:
 *   bf16(y) after the all-reduce.  A process may hold m of the k ranks: it calls tpla_decode once
 *   per held rank with TPLA_DECODE_ACCUMULATE after the first and passes comm (world = k/m
 *   processes) only on the last call, so the all-reduce sums every rank exactly once.
 *   Ordering: the kernels use programmatic dependent launch; K3 reads seq_lens and the block table
 *   BEFORE waiting for its predecessor kernels (its schedule overlaps their tail), so the caller's
 *   writes to those two arrays must be complete when the call is enqueued (a copy, or a kernel
 *   that does not trigger its dependents early).  Every other input may come from the preceding
 *   kernels of the stream (e.g. tpla_append_kv of the same step). */
tpla_status tpla_decode(const tpla_config* cfg, const tpla_weights* w, const tpla_cache* cache,
                        const void* q_nope, const void* q_pe, const int32_t* seq_lens, int32_t B,
                        int32_t max_seq_len, void* ws, size_t ws_bytes, float* y, void* out, int32_t flags,
                        tpla_comm* comm, void* stream);

/* Multi-token decode (speculative / MTP decoding): n_q query tokens per sequence,
 * already appended to the cache, decoded in one step.  Token i of sequence b sits at position
 * seq_lens[b] - n_q + i and attends to the first seq_lens[b] - n_q + 1 + i cached tokens (causal
 * among the new tokens); otherwise exactly tpla_decode per token.  The heads of all
 * n_q tokens share the tensor-core M dimension: requires the tcgen05 path and n_q * H_loc <= 128
 * (else TPLA_ERR_UNSUPPORTED), and seq_lens[b] >= n_q (not checked: device data).
 *   q_nope: device bf16 [B, n_q, h_q, d_h];  q_pe: device bf16 [B, n_q, h_q, d_r];
 *   y: device fp32 [B * n_q, D] (row b * n_q + i);  out: device bf16 [B * n_q, D] or NULL;
 *   ws: tpla_decode_workspace_bytes_mtp(cfg, B, n_q, max_seq_len) bytes.  tpla_decode = n_q 1. */
tpla_status tpla_decode_workspace_bytes_mtp(const tpla_config* cfg, int32_t B, int32_t n_q, int32_t max_seq_len,
                                            size_t* bytes);

/* Causal prefill attention of one prompt.  The prompt's
 * L rows must already be in this device's cache as sequence `seq`, positions 0..L-1 (written by
 * tpla_prefill_mla: EXACT rows).  Every prompt token t attends to rows 0..t with this
 * device's shard softmax (g = 1: plain MLA with the heads split over k devices — the PD-separated
 * prefill; g > 1: TPLA prefill over the latent shard, the paper's comparison), then W^UV, W^O and the
 * all-reduce over comm exactly as tpla_decode.
 * Computed as the multi-token decode (tpla_decode_mtp) over pseudo-sequences that share the
 * prompt's pages: pseudo-sequence j holds n_q = 128 / H_loc consecutive prompt tokens as its newest
 * tokens, with causal per-row limits; chunks of <= 256 prompt rows per decode call.
 *   q_nope [L, h_q, d_h], q_pe [L, h_q, d_r] bf16 (device, post-RoPE); y [L, D] fp32 (= or +=
 *   with TPLA_DECODE_ACCUMULATE), out [L, D] bf16 or NULL; ws: tpla_prefill_workspace_bytes.
 *   Needs the tcgen05 attention path (d_r = 64, W_lat in {64, 128, 256, 512}).  Errors as tpla_decode. */
tpla_status tpla_prefill_workspace_bytes(const tpla_config* cfg, int32_t L, int32_t max_pages_per_seq, size_t* bytes);
tpla_status tpla_prefill_attention(const tpla_config* cfg, const tpla_weights* w, const tpla_cache* cache,
                                   const void* q_nope, const void* q_pe, int32_t seq, int32_t L, void* ws,
                                   size_t ws_bytes, float* y, void* out, int32_t flags, tpla_comm* comm, void* stream);

/* MLA prefill in its NON-absorbed form (PD separation P:421):
 * prefill is compute-bound, so it runs as MLA with the heads split over the k prefill devices and
 * the latent unsliced (cfg: g = 1; rank r holds heads [r·h_q/k, (r+1)·h_q/k)), on keys and values
 * up-projected per head (head dimension d_h + d_r = 192 for QK, d_h = 128 for PV, against 576 / 512
 * for the absorbed decode form):  ĉ = RMSNorm(c^KV) with the full RMS (γ lives in the
 * weights), k_h = ĉ W^UK_h, v_h = ĉ W^UV_h, s = sm_scale (q_h k_hᵀ + q^PE_h k^PEᵀ) causal, O_h =
 * softmax(s) v_h (Eq. isolate_rope), y = concat_h O_h · W^O[rows of the heads]
 * (+ all-reduce over comm).  The decode cache rows of the prompt are written separately by
 * tpla_prefill_mla (EXACT rows in the TPLA basis), which TPLA decode then reads.
 *   tpla_prefill_weights: per device, bf16 blocked [N/128][K/64][128][64] (K-major rows, rows past
 *     N zero): W_UK / W_UV with N = H·d_h output features (h-major), K = d_c latent rows
 *     (W_γ W^UK[:, heads], original basis); W_O with N = D, K = H·d_h (W^O[head rows]ᵀ).
 *   tpla_convert_prefill_weights: host bf16 W_UK, W_UV [d_c, h_q·d_h], gamma [d_c], W_O [h_q·d_h, D]
 *     (fp64 on the host, bf16 RNE) into caller-allocated buffers of tpla_prefill_weights_bytes.
 *   tpla_prefill_mla_forward: c_kv [L, d_c] raw pre-norm latents, k_pe [L, d_r] post-RoPE,
 *     q_nope [L, h_q, d_h], q_pe [L, h_q, d_r] (all heads; the device takes its block), device bf16;
 *     y [L, D] fp32 (= or += with TPLA_DECODE_ACCUMULATE); out [L, D] bf16 or NULL; ws:
 *     tpla_prefill_mla_workspace_bytes(cfg, L).  Needs g = 1, d_h = 128, d_r = 64, 64 | d_c,
 *     64 | h_q·d_h / k (else TPLA_ERR_UNSUPPORTED).  Errors as tpla_decode. */
typedef struct tpla_prefill_weights {
  void* W_UK;
  void* W_UV;
  void* W_O;
} tpla_prefill_weights;
tpla_status tpla_prefill_weights_bytes(const tpla_config* cfg, size_t* W_UK, size_t* W_UV, size_t* W_O);
tpla_status tpla_convert_prefill_weights(const tpla_config* cfg, const uint16_t* W_UK, const uint16_t* W_UV,
                                         const uint16_t* gamma, const uint16_t* W_O, tpla_prefill_weights* out,
                                         void* stream);
tpla_status tpla_prefill_mla_workspace_bytes(const tpla_config* cfg, int32_t L, size_t* bytes);
tpla_status tpla_prefill_mla_forward(const tpla_config* cfg, const tpla_prefill_weights* w, const void* c_kv,
                                     const void* k_pe, const void* q_nope, const void* q_pe, int32_t L, void* ws,
                                     size_t ws_bytes, float* y, void* out, int32_t flags, tpla_comm* comm,
                                     void* stream);

/* Up-projection shared by a latent group.  The g devices j of head block i hold
 * the same W^O rows, so Õ_i = Σ_j v_j W^O_i = (Σ_j v_j) W^O_i: the group may sum its
 * v_j = O_j W^UV'_j first and read W^O once instead of g times.  Co-located devices add into one v_acc;
 * devices in different processes reduce-scatter it over its column chunks and each projects its
 * chunk's K-slice of W^O (1/n_chunks of the rows), then the usual all-reduce of y.
 * v_acc layout: fp32, column-chunk-major [n_chunks][B * n_q][K / n_chunks], K = H_loc * d_h, i.e.
 * element (row, col) at ((col / kc) * B*n_q + row) * kc + col % kc, kc = K / n_chunks (64 * n_chunks | K).
 *   tpla_decode_v:    K2, K3, K4+K5a of this device into v_acc (= v_j, or += with TPLA_DECODE_ACCUMULATE).
 *                     Needs the tcgen05 attention path; same inputs and workspace as tpla_decode_mtp.
 *                     TPLA_DECODE_STAGE_PRE / _ATTN split it into its query stage and attention stage.
 *   tpla_project_out: with group_comm (world n_chunks, rank chunk): in-place ncclReduceScatter of v_acc
 *                     (sum over the group; chunk `chunk` lands in place), then for every caller
 *                     y [R, D] fp32 (=, or += with TPLA_DECODE_ACCUMULATE) = bf16(v_acc chunk) ·
 *                     W^O[chunk's K rows]; then the all-reduce of y over comm (if given) and the bf16
 *                     out [R, D] (or NULL).  Without group_comm the chunk must already hold the group
 *                     sum.  ws: a decode workspace for at least R = B * n_q rows.  Errors as tpla_decode. */
tpla_status tpla_decode_v(const tpla_config* cfg, const tpla_weights* w, const tpla_cache* cache, const void* q_nope,
                          const void* q_pe, const int32_t* seq_lens, int32_t B, int32_t n_q, int32_t max_seq_len,
                          void* ws, size_t ws_bytes, float* v_acc, int32_t n_chunks, int32_t flags, void* stream);
tpla_status tpla_project_out(const tpla_config* cfg, const tpla_weights* w, float* v_acc, int32_t R, int32_t n_chunks,
                             int32_t chunk, void* ws, size_t ws_bytes, float* y, void* out, int32_t flags,
                             tpla_comm* group_comm, tpla_comm* comm, void* stream);
/* tpla_project_out_sum: tpla_project_out for a latent group whose g ranks live in THIS process and
 * wrote SEPARATE accumulators (tpla_decode_v without TPLA_DECODE_ACCUMULATE, each on its own
 * stream, so their attention runs concurrently): v = bf16(Σ_i v_list[i] chunk), summed in list order
 * (deterministic), then as tpla_project_out without group_comm.  v_list: n_v (1..16) device pointers
 * of the same [n_chunks][R][K / n_chunks] fp32 layout.  The sum Σ_j v_j W^O = (Σ_j v_j) W^O is the
 * group-shared up-projection.  Errors as tpla_project_out. */
tpla_status tpla_project_out_sum(const tpla_config* cfg, const tpla_weights* w, const float* const* v_list, int32_t n_v,
                                 int32_t R, int32_t n_chunks, int32_t chunk, void* ws, size_t ws_bytes, float* y,
                                 void* out, int32_t flags, tpla_comm* comm, void* stream);
tpla_status tpla_decode_mtp(const tpla_config* cfg, const tpla_weights* w, const tpla_cache* cache,
                            const void* q_nope, const void* q_pe, const int32_t* seq_lens, int32_t B, int32_t n_q,
                            int32_t max_seq_len, void* ws, size_t ws_bytes, float* y, void* out, int32_t flags,
                            tpla_comm* comm, void* stream);

/* K3 + K4 only (attention of one shard, Eq. tpla_softmax_one_device without W^VO):
 *   q_lat: device bf16 [B, H_loc, W_lat] (= Q'_j, mu_j included); q_pe: device bf16 [B, h_q, d_r]
 *   (all heads); O: device fp32 [B, H_loc, W_lat] = Σ_t p_t ĉ_{j,t};  lse: device fp32 [B, H_loc]
 *   or NULL: log Σ_t exp(s_t) (natural log, s_t including sm_scale).  O = lse = NULL skips K4 (the
 *   partials stay in the workspace).  On the tcgen05 path K3's schedule kernel K3p runs first. */
tpla_status tpla_decode_attention(const tpla_config* cfg, const tpla_cache* cache, const void* q_lat,
                                  const void* q_pe, const int32_t* seq_lens, int32_t B, int32_t max_seq_len,
                                  void* ws, size_t ws_bytes, float* O, float* lse, void* stream);

/* ---- C1: communicator -------------------------------------------------------------- */

/* 128-byte NCCL unique id for rank 0 to broadcast (e.g. over a torch.distributed group). */
tpla_status tpla_comm_unique_id(void* out128);
/* Join the k-device communicator (blocking until all ranks join).  The current CUDA device
 * must already be this rank's GPU. */
tpla_status tpla_comm_init(tpla_comm** out, const void* unique_id128, int32_t world, int32_t rank);
/* Fused W^O epilogue + one-shot all-reduce (O = AllReduce(Σ_r Õ_r)):
 * allocates a symmetric buffer of 2 · max_elems fp32 (ncclMemAlloc), registers it as an NCCL window
 * (NCCL_WIN_COLL_SYMMETRIC) and creates a device communicator with LSA barriers (and the NVLS
 * multicast address when the system has one).  COLLECTIVE: every rank of the communicator calls it.
 * Afterwards the K5 segment reduce of tpla_decode / tpla_decode_mtp / tpla_project_out calls on this
 * communicator whose R·D <= max_elems writes the rank's Õ rows into the buffer, meets the peers at an
 * LSA barrier and sums the ranks itself (multimem.ld_reduce through the switch, else peer loads over
 * NVLink in rank order) — no separate ncclAllReduce or cast launch.  TPLA_FUSED_AR=0 disables it per
 * process, =unicast forbids the multicast.  TPLA_ERR_UNSUPPORTED if the loaded NCCL has no device API
 * matching the headers (NCCL 2.28).  tpla_comm_fused_allreduce_mode: 0 off, 1 peer loads, 2 multicast. */
/* tpla_decode_attention with flags.  TPLA_ATTN_REUSE_PLAN: no K3p — K3 reuses the schedule that a
 * completed tpla_decode_attention on the same workspace left there (same cfg, cache, seq_lens contents,
 * B and max_seq_len; the caller guarantees it), so O = lse = NULL runs K3 ALONE (to time the attention
 * kernel by itself).  Requires the tcgen05 K3 (TPLA_ERR_UNSUPPORTED otherwise). */
enum { TPLA_ATTN_REUSE_PLAN = 1 };
tpla_status tpla_decode_attention_ex(const tpla_config* cfg, const tpla_cache* cache, const void* q_lat,
                                     const void* q_pe, const int32_t* seq_lens, int32_t B, int32_t max_seq_len,
                                     void* ws, size_t ws_bytes, float* O, float* lse, int32_t flags, void* stream);
/* Which attention kernel tpla_decode / tpla_decode_v / tpla_decode_attention run for this shape
 * (validated first; a status < 0 is -(tpla_status) of the failed validation): 1 = the tcgen05
 * persistent K3 (d_r = 64, W_lat in {64, 128, 256, 512}, B <= 512), 0 = the mma.sync K3 that serves
 * every other shape (or TPLA_ATTN=mma).  TPLA_REQUIRE_TC=1 in the environment turns the fallback into
 * TPLA_ERR_UNSUPPORTED for the decode calls. */
int32_t tpla_decode_kernel_path(const tpla_config* cfg, int32_t B);
tpla_status tpla_comm_enable_fused_allreduce(tpla_comm* comm, int64_t max_elems);
int32_t tpla_comm_fused_allreduce_mode(const tpla_comm* comm);
tpla_status tpla_comm_destroy(tpla_comm* comm);

/* Synchronise `stream` and report any asynchronous CUDA fault. */
tpla_status tpla_sync(void* stream);

/* ---- measurement: per-kernel device time --------------------------------------------- */

/* on = 1: every kernel launch of this library is bracketed by two CUDA events recorded on its
 * launching stream (no device work is added; under stream capture they become event nodes);
 * on = 2: only the decode-attention kernel (K3) is bracketed; on = 0: off. */
tpla_status tpla_profile_enable(int32_t on);
/* Wait for the recorded events and accumulate their elapsed times per kernel name. */
tpla_status tpla_profile_collect(void);
/* Number of distinct kernel names accumulated so far. */
int32_t tpla_profile_count(void);
/* Entry i: name (host buffer of 64 bytes), total milliseconds, number of launches. */
tpla_status tpla_profile_get(int32_t i, char* name64, double* total_ms, int64_t* launches);
/* Drop all accumulated and pending records. */
tpla_status tpla_profile_reset(void);

#ifdef __cplusplus
}
#endif
#endif /* TPLA_H_ */
