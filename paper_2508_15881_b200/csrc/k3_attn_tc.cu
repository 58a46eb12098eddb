// K3 (v1, Blackwell-native) — persistent split-K flash decoding of one TPLA shard on the
// 5th-generation tensor cores, and its K4 combine.
//
// What it computes (Eq. tpla_softmax_one_device; RoPE part P:238-242):
//   s_t = [Q'_j ‖ q^PE] · [ĉ_{j,t} ‖ k^PE_t]          (μ_j already folded into Q'_j)
//   p_t = softmax over this shard's own tokens (sm_scale applied; no cross-device max/sum)
//   O_j = Σ_t p_t ĉ_{j,t}
//
// Mapping: heads are the MMA M dimension (128 TMEM lanes, one head per lane).
// Per tile of TT tokens (TT = 128 when W_lat <= 128, else 64):
//   QK  S[128 x TT]   = Q'_j (TMEM, A operand, K = W_lat)  x  ĉ tileᵀ (smem, K-major)     tcgen05 TS
//                     + q^PE (smem, A, K = 64)             x  k^PE tileᵀ (smem, K-major)   tcgen05 SS
//   softmax on 8 warps (thread = head row, two warps per TMEM lane quadrant splitting the
//   columns), exp2 with a lazily-raised running max (the O accumulator is rescaled only when the
//   max grows by more than 2^8), P written back to TMEM as bf16 over its own S columns
//   PV  O[128 x W_lat] += P (TMEM, A, K = TT tokens)       x  ĉ tile (smem, MN-major)      tcgen05 TS
// The cache tile [TT tokens x (W_lat + 64)] arrives by TMA (SWIZZLE_128B, 64-row x 64-column
// boxes) into a 4-8 stage mbarrier ring; the same smem bytes serve as the K-major B operand of
// QK and the MN-major B operand of PV, so every cache byte crosses HBM -> SMEM once.
//
// Work split: persistent grid (<= #SMs CTAs).  The flattened (sequence, tile) list is cut into
// equal contiguous work ranges, one per CTA; a range is a few segments (one per sequence it
// touches).  Each segment leaves an unnormalised partial (O, m, l); K45 merges a sequence's
// segments, whose ids are contiguous.
//
// Warp roles (384 threads): w0 TMA producer, w1 MMA issuer, w2 TMEM allocator, w3 sequence
// scan, w4-w11 softmax + Q loader + epilogue (warp w owns TMEM lanes 32*(w%4)..).
#include <cuda.h>
#include <math.h>

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include "common.cuh"
#include "internal.h"
#include "sm100.cuh"

namespace tpla {
namespace {

using namespace sm100;

constexpr int kSub = 64;          // cache rows per TMA box (page_size is a multiple of 64)
constexpr int kThreads = 384;    // w0 TMA, w1 MMA, w2 TMEM alloc, w3 schedule, w4-w11 softmax
constexpr int kMaxB = 512;        // sequences per launch supported by the smem schedule
constexpr int kMaxCta = 256;      // persistent grid bound (<= #SMs in practice)
constexpr int kPlanStride = 8;    // ints per CTA entry of the K3p plan
constexpr float kRescaleThreshold = 8.0f;   // log2 units: p <= 2^8 between max updates
// Every kPolyEvery-th group of 4 exponentials computes 2 of them with ex2_poly2 on the FMA pipe
// (0 = none).  Measured (tools/gpu_ab.sh, round 2): at W_lat <= 128 a 1-in-8 share (kPolyEvery 4)
// is the best of 0 / 1-in-8 / 1-in-4 / 1-in-2 (h8 K3 63.2 vs 63.6 us at 1-in-4, 71.4 at 1-in-2: the
// loop is bound by one warp's issue, not by the MUFU, tools/exps_rate); at W_lat = 256 none helps.
#ifdef TPLA_POLY_EVERY
template <int W_LAT> constexpr int kPolyEvery = TPLA_POLY_EVERY;
#else
template <int W_LAT> constexpr int kPolyEvery = W_LAT <= 128 ? 4 : 0;
#endif

struct TcArgs {
  const uint16_t* q_lat;       // [B, H_loc, W_lat]
  const uint16_t* q_pe;        // [B, h_q, d_r]
  const int32_t* block_table;  // [B, max_pages]
  const int32_t* seq_lens;     // [B]
  const int32_t* plan;         // K3p's schedule (plan_ints): per-CTA ranges, first box rows, cum, slen
  uint16_t* o_part;            // fp16 [max_segs, H_loc, W_lat]: the segment's O / l (normalised)
  float* ml_part;              // [max_segs, H_loc, 2]: (m, l)
  int32_t* meta;               // [B, 2]: first segment id, segment count
  int B, h_loc, h_q, head_begin, page_size, max_pages;
  int n_q;                     // query tokens per sequence (multi-token decode): MMA rows = n_q * h_loc
  int cap;                     // max_pages * page_size: lengths beyond the page table are clamped
  float scale_log2;
  long long* trace;            // MODE 2 (diagnostic): clock64 stamps of CTA trace_cta, [4][kTrace]
  int trace_cta;
};
constexpr int kTrace = 128;
constexpr int kSlots = 23;        // trace slots: qk_issue, pv_issue, s_ready, p_done, qk_issued, pv_issued,
                                  // then p_done of each softmax warp 4..11, then the producer's TMA issue,
                                  // then warp 4's softmax phases: S loaded, max exchanged, exps done,
                                  // MMA warp waits (19-21, non-PAIR), slot 22: tile landed (kv_full
                                  // observed by the otherwise idle warp 3)
// startup events of the traced CTA (clock64): 0 kernel entry, 1 after pdl_wait, 2 schedule done,
// 3 producer lookups resolved, 4 first TMA issued, 5 Q loaded (warp 4), 6 MMA saw q_ready,
// 7 MMA saw kv_full(0)
#define EV(i)                                                                            \
  do {                                                                                   \
    if ((MODE & 2) && blockIdx.x == a.trace_cta) a.trace[kSlots * kTrace + 4 * kMaxCta + (i)] = clock64(); \
  } while (0)
#define TRACE(slot, gg)                                                                  \
  do {                                                                                   \
    if ((MODE & 2) && blockIdx.x == a.trace_cta && (gg) < kTrace) a.trace[(slot) * kTrace + (gg)] = clock64(); \
  } while (0)

#ifndef TPLA_SEQ_COST_TOKENS
#define TPLA_SEQ_COST_TOKENS 0      // 0: the measured per-width default (Cfg::SEQ_COST)
#endif

template <int W_LAT>
struct Cfg {
  // PAIR (W_lat = 512: g = 1, plain MLA): O [128 x 512] fp32 alone would fill TMEM, so a cluster of
  // two CTAs splits the latent: CTA r holds Q'[:, 256r:256r+256], streams latent columns
  // [256r, 256r+256) (+ the RoPE part), computes partial logits, swaps them with its peer through
  // distributed shared memory (st.async into the peer's buffer) and sums them — exact logits,
  // the softmax is then identical in both — and accumulates O[:, 256r:256r+256].
  static constexpr bool PAIR = W_LAT == 512;
  static constexpr int WL = PAIR ? 256 : W_LAT;       // latent columns this CTA handles
  // Tokens per tile: 128 when the TMEM budget allows it (O, Q' and two 128-column S buffers),
  // else 64.  Per tile the MMA warp waits on two mbarriers and the softmax warps synchronise
  // once; at W_lat <= 128 the MMA work per 64-token tile is too short to hide those (measured),
  // so the larger tile halves the synchronisation per byte.
  static constexpr int TT = WL <= 128 ? 128 : 64;
  // PP (ping-pong softmax, TT = 128): the two warps of a TMEM lane quadrant take alternate tiles
  // with whole rows each, instead of splitting every tile's columns and exchanging row maxima.
  // They share one SMSP (warps w and w+4); out of phase, one warp's loads, stores and barrier
  // waits overlap the other's exponentials (see the PP branch of the softmax).
#ifdef TPLA_NO_PP
  static constexpr bool PP = false;
#else
  static constexpr bool PP = !PAIR && TT == 128;
#endif
  // S (= P) buffers in TMEM.  Three when they fit (W_lat = 64: O 64 + Q' 32 + 3 x 128 = 480
  // columns): QK then runs two tiles ahead of PV, so S(g+1) is ready when the softmax finishes
  // tile g (with two buffers the softmax waited ~470 cycles per tile for it, measured).
  static constexpr int NSB = W_LAT == 64 ? 3 : 2;
  static constexpr int LAG = NSB - 1;                 // PV issued LAG tiles behind QK
  // SPLIT: QK and PV issued by two warps (w1, w2) with their own loops.  Measured A/B: W_lat = 64
  // (h8, c3) 1.5-2 % faster; W_lat = 256 (c1) 5 % slower (its PV / QK waits interleave better in
  // one loop); W_lat = 128 neutral.  Not for the CTA pair.
#ifdef TPLA_K3_NO_SPLIT
  static constexpr bool SPLIT = false;
#else
  static constexpr bool SPLIT = !PAIR && W_LAT == 64;
#endif
  static constexpr int SUB = TT / kSub;               // TMA boxes per column group per tile
  static constexpr int CH = TT / 2;                   // S columns per softmax warp
  // Per-sequence header cost of the schedule, in tiles: a CTA whose range starts a second
  // segment pays its epilogue, the next Q load and the pipeline refill.  Measured with the trace's
  // per-CTA end times (h8, c1): at 512 tokens the two-segment CTAs ended 3-4 us after the others
  // (every one of the slowest eight had two segments).  A/B of the in-step K3 time over 512 / 768 /
  // 1024 / 1536 tokens: 1024 best at W_lat 64 / 256 (h8 -3.5 %, c1 -4 %, c3 -3 %), 512 at W_lat 128.
  // Re-fitted at the end of round 2 (per-CTA end times of the trace against tiles and segment count:
  // an extra segment costs ~6 tiles at h8 and ~6-8 at c1 once the partials are fp16) and A/B'd: 512
  // tokens at W_lat 256 (c1 K3 243.5 -> 240.5 us per step), 768 at W_lat 64 (h8 476.3 -> 474.9).
  static constexpr int SEQ_COST = (TPLA_SEQ_COST_TOKENS > 0 ? TPLA_SEQ_COST_TOKENS
                                   : W_LAT == 128 || W_LAT == 256 ? 512 : W_LAT == 64 ? 768 : 1024) / TT;
  static constexpr int W = WL + 64;
  static constexpr int NBOX = W / 64;                 // 64-column groups per tile (latent part + RoPE)
  static constexpr int SUB_BYTES = kSub * 128;        // one TMA box: 64 rows x 128 B
  static constexpr int BOX_BYTES = TT * 128;          // one column group of the tile (TT rows)
  static constexpr int STAGE_BYTES = NBOX * BOX_BYTES;
  static constexpr int QPE_BYTES = 128 * 128;         // q^PE A operand [128 rows x 64] bf16
  static constexpr int XCH_BYTES = PAIR ? 2 * 8 * 32 * CH * 4 : 0;   // PAIR: peer's partial logits + ours to send
  // Ring depth, A/B over 3-6 stages (tools/gpu_ab_k.sh): 4 x 40 KB at W_lat = 256 (c1 K3 244.0 ->
  // 242.6 us per step, against the 5 that fit), 5 x 32 KB at W_lat <= 128 (h8 499.5 -> 496.0, c3
  // 847 -> 843, against 6; 4 is slower there, 3 slower everywhere); the CTA pair keeps what fits.
#ifndef TPLA_K3_MAX_NST
#define TPLA_K3_MAX_NST (PAIR ? 8 : W_LAT == 256 ? 4 : 5)
#endif
  static constexpr int NST = std::min(TPLA_K3_MAX_NST, (220 * 1024 - QPE_BYTES - XCH_BYTES) / STAGE_BYTES);
  static constexpr int SMEM = 1024 + QPE_BYTES + XCH_BYTES + NST * STAGE_BYTES;
  // TMEM columns
  static constexpr int O_COL = 0;
  static constexpr int Q_COL = WL;                    // WL/2 columns of packed bf16
  static constexpr int S_COL0 = (WL + WL / 2 + 63) / 64 * 64;
  static constexpr int S_COLS = S_COL0 + NSB * TT;
  static constexpr int TMEM_COLS = S_COLS <= 256 ? 256 : 512;
  static_assert(S_COLS <= 512, "TMEM budget");
};

struct Sched {
  int lo, hi;          // tile range [lo, hi) in the flattened list
  int b_first, b_last;
  int seg_base;
};

// Work split with a fixed cost per sequence start: sequence b occupies kSeqCost work units of
// "header" (its Q load, pipeline refill and the previous segment's epilogue) followed by one
// unit per tile, so a CTA whose range crosses a sequence boundary gets fewer tiles.  tile_of maps
// a work position to the first tile at or after it.
template <int kSeqCost>
__device__ __forceinline__ int tile_of(const int* cum, int B, long w) {
  int lo = 0, hi = B + 1;                       // first b with cum[b] + kSeqCost*b > w
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if ((long)cum[mid] + (long)kSeqCost * mid <= w) lo = mid + 1; else hi = mid;
  }
  const int b = lo - 1;
  const long off = w - ((long)cum[b] + (long)kSeqCost * b) - kSeqCost;
  long t = cum[b] + (off > 0 ? off : 0);
  if (b < B && t > cum[b + 1]) t = cum[b + 1];
  return int(t);
}

__device__ __forceinline__ int upper_bound_cum(const int* cum, int n, int x) {  // first i with cum[i] > x
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (cum[mid] <= x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// ---------------------------------------------------------------- K3p: the persistent schedule
// Plan layout (int32, plan_ints(n_cta, B)): [n_cta][kPlanStride] = (lo, hi, b_first, b_last, seg_base),
// then cum[B + 1], slen[B], then the first 32 box rows of every CTA [n_cta][32].
struct PlanArgs {
  const int32_t* seq_lens;
  const int32_t* block_table;
  int32_t* plan;
  int B, n_cta, cap, page_size, max_pages;
};

__device__ __forceinline__ int block_excl_scan(int x, int* wsum, int& total) {   // 512 threads
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    int w = lane < 16 ? wsum[lane] : 0, wi = w;
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < 16) wsum[16 + lane] = wi - w;          // exclusive warp offsets
    if (lane == 15) wsum[32] = wi;
  }
  __syncthreads();
  total = wsum[32];
  const int r = wsum[16 + warp] + inc - x;
  __syncthreads();                                   // (wsum reusable)
  return r;
}

// K3p: CTA 0 computes every K3 CTA's schedule entry (the flattened (sequence, tile) list cut into
// equal work ranges with a per-sequence header cost, tile_of; each CTA's first segment id by a block
// scan) and copies the sequence scan; CTAs 1.. each resolve the first 32 box rows of 8 K3 CTAs through
// the page table, one lookup per thread (each recomputes the scan: B <= 512 lengths, one per thread).
// (One CTA doing all 148 x 32 lookups took ~16 us, measured: its dependent loads did not overlap.)
// Reads only caller inputs: runs under the predecessor's tail and waits only before its stores.
constexpr int kPlanThreads = 512;
constexpr int kPlanRowCtas = kPlanThreads / 32;           // K3 CTAs whose rows one plan CTA resolves

template <int W_LAT>
__device__ __forceinline__ void plan_body(const PlanArgs& p, int cta) {   // cta: this CTA's index in K3p's grid
  using C = Cfg<W_LAT>;
  __shared__ int cum[kMaxB + 1], slen[kMaxB], lo_arr[kMaxCta + 1], wsum[40];
  const int tid = threadIdx.x;
  const int len = tid < p.B ? min(p.seq_lens[tid], p.cap) : 0;
  const int nt = (len + C::TT - 1) / C::TT;
  int total;
  const int ex = block_excl_scan(nt, wsum, total);
  if (tid < p.B) { cum[tid] = ex; slen[tid] = len; }
  if (tid == 0) cum[p.B] = total;
  __syncthreads();
  const int n = p.n_cta;
  const long Wt = long(total) + long(C::SEQ_COST) * p.B;            // total work units
  if (cta == 0) {
    for (int cc = tid; cc <= n; cc += kPlanThreads) lo_arr[cc] = tile_of<C::SEQ_COST>(cum, p.B, cc * Wt / n);
    __syncthreads();
    int lo = 0, hi = 0, bf = 0, bl = -1;
    if (tid < n) {
      lo = lo_arr[tid];
      hi = lo_arr[tid + 1];
      if (lo < hi) {
        bf = upper_bound_cum(cum, p.B + 1, lo) - 1;
        bl = upper_bound_cum(cum, p.B + 1, hi - 1) - 1;
      }
    }
    int n_seg_total;
    const int seg_base = block_excl_scan(tid < n ? bl - bf + 1 : 0, wsum, n_seg_total);
    pdl_wait();   // first store: the previous launch's K3 read this plan (write-after-read)
    if (tid < n) {
      int32_t* e = p.plan + tid * kPlanStride;
      e[0] = lo; e[1] = hi; e[2] = bf; e[3] = bl; e[4] = seg_base;
    }
    int32_t* pc = p.plan + n * kPlanStride;
    for (int i = tid; i <= p.B; i += kPlanThreads) pc[i] = cum[i];
    for (int i = tid; i < p.B; i += kPlanThreads) pc[p.B + 1 + i] = slen[i];
    return;
  }
  // first 32 box rows of K3 CTAs [c0, c0 + kPlanRowCtas)
  const int c0 = (cta - 1) * kPlanRowCtas, cc = c0 + tid / 32, u = tid & 31;
  int row = 0;
  if (cc < n) {
    const int lo = tile_of<C::SEQ_COST>(cum, p.B, cc * Wt / n), hi = tile_of<C::SEQ_COST>(cum, p.B, (cc + 1) * Wt / n);
    const int tt = lo + u / C::SUB;
    if (tt < hi) {
      const int bb = upper_bound_cum(cum, p.B + 1, tt) - 1;
      const int tok0 = (tt - cum[bb]) * C::TT;
      int tok = tok0 + (u % C::SUB) * kSub;
      if (tok >= slen[bb]) tok = tok0;
      row = p.block_table[(long)bb * p.max_pages + tok / p.page_size] * p.page_size + tok % p.page_size;
    }
  }
  pdl_wait();
  if (cc < n) p.plan[n * kPlanStride + 2 * p.B + 1 + cc * 32 + u] = row;
}

template <int W_LAT>
__global__ void __launch_bounds__(kPlanThreads) attn_plan_kernel(PlanArgs p) {
  pdl_trigger();
  plan_body<W_LAT>(p, blockIdx.x);
}

inline int plan_ctas(int n_cta) { return 1 + (n_cta + kPlanRowCtas - 1) / kPlanRowCtas; }

#include "k2_absorb.cuh"

// K3p + K2 in one launch (the two are independent: K3p reads seq_lens / the block table, K2 the
// queries and W^UK'): the first plan_ctas(n_cta) CTAs compute K3's schedule, the others one
// (head, 32-row tile) of Q'_j each.  One launch and one PDL hop fewer ahead of K3.
template <int W_LAT>
__global__ void __launch_bounds__(kPlanThreads) pre_attn_kernel(const __grid_constant__ CUtensorMap wmap,
                                                                const __grid_constant__ CUtensorMap qmap, PlanArgs p,
                                                                absorb::Args a, int n_plan) {
  pdl_trigger();
  if (int(blockIdx.x) < n_plan) {
    plan_body<W_LAT>(p, blockIdx.x);
    return;
  }
  extern __shared__ __align__(1024) uint8_t pre_smem[];
  __shared__ uint64_t bar;
  absorb::body(&wmap, &qmap, a, blockIdx.x - n_plan, pre_smem, &bar);
}

// MODE 0: the kernel.  MODE 1 (diagnostic, TPLA_K3_MODE=stream): the TMA ring alone — every
// tile is released as soon as it lands, no MMA/softmax — to measure the cache streaming rate.
// Bit 16 (nosm, PP only): the softmax warps pass every tile straight through (MMA + ring alone).
// Bit 32 (nomma): the MMA warp commits without issuing MMAs (softmax + ring alone).
// MODE bit 2 (trace): per-tile clock64 stamps.  Bit 8 (nold): softmax without its TMEM
// loads/stores.  Bit 4 (notma): no cache loads (stale smem), to time MMA + softmax alone.  Diagnostic modes
// compute garbage; they exist to isolate the pipeline's limiter.
template <int W_LAT, int MODE>
__global__ void __launch_bounds__(kThreads, 1)
attn_tc_kernel(const __grid_constant__ CUtensorMap tmap, TcArgs a) {
  pdl_trigger();
  if (threadIdx.x == 0) EV(0);
  using C = Cfg<W_LAT>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* s_qpe = smem;
  float* s_xch = reinterpret_cast<float*>(smem + C::QPE_BYTES);   // PAIR: recv [8 warps][CH/4][32 lanes] float4,
                                                                   // then the send staging buffer (same shape)
  uint8_t* s_kv = smem + C::QPE_BYTES + C::XCH_BYTES;
  __shared__ uint64_t kv_full[C::NST], kv_empty[C::NST];
  __shared__ uint64_t s_full[C::NSB], p_full[C::NSB], pv_done[C::NSB], q_ready;
  __shared__ uint32_t tmem_base;
  __shared__ int cum[kMaxB + 1];
  __shared__ int slen[kMaxB];            // min(seq_len, capacity) per sequence
  __shared__ int s_rows[32];             // the first 32 box rows of the range (K3p)
  __shared__ int s_sched[5];             // this CTA's plan entry: lo, hi, b_first, b_last, seg_base
  __shared__ float red_max[C::NSB][2][128];   // [S buffer][half][row] partial row maxima
  __shared__ float red_l[2][128];        // [half][row] partial row sums at a segment end
  __shared__ float red_m[2][128];        // PP: [set][row] the max each set's sums are expressed in
  __shared__ float m_row[128];           // PP: the row's running max after the last finalised tile
  __shared__ uint64_t x_full[8], x_ok[8]; // PAIR, per softmax warp: peer's logits landed / peer read ours

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // PAIR: CTAs 2c and 2c+1 form a cluster and share logical work range c
  const int c = C::PAIR ? blockIdx.x >> 1 : blockIdx.x, n_cta = C::PAIR ? gridDim.x >> 1 : gridDim.x;
  const uint32_t crank = C::PAIR ? cluster_ctarank() : 0;            // latent half of this CTA

  // ---------------------------------------------------------------- setup
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap);
    for (int i = 0; i < C::NST; ++i) { mbar_init(&kv_full[i], 1); mbar_init(&kv_empty[i], 1); }
    for (int i = 0; i < C::NSB; ++i) { mbar_init(&s_full[i], 1); mbar_init(&p_full[i], C::PP ? 4 : 8); mbar_init(&pv_done[i], 1); }
    mbar_init(&q_ready, 8);      // p_full / q_ready: one arrival per softmax warp (elected lane)
    if (C::PAIR)
      for (int i = 0; i < 8; ++i) { mbar_init(&x_full[i], 1); mbar_init(&x_ok[i], 1); }
    fence_barrier_init();
  }
  if (C::PAIR) cluster_sync();   // the peer's barriers are initialised before any remote operation
  if (warp == 2) tmem_alloc<C::TMEM_COLS>(&tmem_base);
  // The schedule (every CTA's tile range, segment ids, its first 32 box rows) was computed by K3p
  // ahead of K2 (attn_plan_kernel): a CTA reads its entry and starts streaming.  (Computed here, the
  // sequence scan, the range starts and the first page-table lookups took ~10 K cycles per CTA
  // before the first TMA — measured, trace mode — with the SMs' HBM streams idle.)
  if (threadIdx.x == 0) EV(1);
  // Softmax warps' row geometry (warps >= 4; harmless elsewhere).  Multi-token decode (n_q > 1,
  // SURVEY f3): row r = (token i, head h).
  const int q4 = warp & 3;
  const int half = (warp - 4) >> 2;                     // 0 or 1 for the softmax warps
  const int r = q4 * 32 + lane;                         // head row = TMEM lane
  const int n_rows = a.n_q * a.h_loc;
  const bool row_ok = r < n_rows;
  const int tok_i = row_ok ? r / a.h_loc : 0, head_h = row_ok ? r % a.h_loc : 0;
  // Q'_j row (bf16 pairs, this warp's columns) and the q^PE chunks 4*half .. 4*half+3 of sequence bb
  // into registers; q_store (softmax branch) moves them to TMEM / smem.
  constexpr int QC = C::WL / 2;                         // packed columns of Q'_j
  constexpr int QH = QC / 2 >= 32 ? QC / 2 : 32;        // columns per warp (W_LAT=64: one warp does all)
  const int q_cbegin = QC / 2 >= 32 ? half * QH : 0;
  const bool q_loads = QC / 2 >= 32 || half == 0;
  struct QRegs { uint4 pe[4]; uint4 q[QH / 4]; };
  auto q_fetch = [&](int bb, QRegs& v) {
    const uint4* pe = reinterpret_cast<const uint4*>(
        a.q_pe + (((long)bb * a.n_q + tok_i) * a.h_q + a.head_begin + head_h) * 64);
#pragma unroll
    for (int c = 0; c < 4; ++c) v.pe[c] = row_ok ? pe[4 * half + c] : make_uint4(0, 0, 0, 0);
    const uint4* src = reinterpret_cast<const uint4*>(
        a.q_lat + (((long)bb * a.n_q + tok_i) * a.h_loc + head_h) * W_LAT + crank * C::WL);
#pragma unroll
    for (int v4 = 0; v4 < QH / 4; ++v4)
      v.q[v4] = row_ok && q_loads ? src[q_cbegin / 4 + v4] : make_uint4(0, 0, 0, 0);
  };
  // One ring stage (tile g of the range): its TT/64 boxes per 64-column group, rows from the
  // producer's batch of 32 resolved box rows.
  auto issue_stage = [&](int g, int rows_batch) {
    int row[C::SUB];
#pragma unroll
    for (int r = 0; r < C::SUB; ++r) row[r] = __shfl_sync(0xffffffffu, rows_batch, (g * C::SUB + r) & 31);
    const int st = g % C::NST;
    if (elect_one()) {
      TRACE(14, g);
      if (g == 0) EV(4);
      uint8_t* dst = s_kv + st * C::STAGE_BYTES;
      if (MODE & 4) {
        mbar_arrive(&kv_full[st]);      // diagnostic: no HBM traffic, stale smem contents
      } else {
        mbar_arrive_expect_tx(&kv_full[st], C::STAGE_BYTES);
#pragma unroll
        for (int j = 0; j < C::NBOX; ++j)
#pragma unroll
          for (int r = 0; r < C::SUB; ++r)
            tma_load_2d(dst + j * C::BOX_BYTES + r * C::SUB_BYTES, &tmap,
                        j < C::NBOX - 1 ? int(crank) * C::WL + j * 64 : W_LAT, row[r], &kv_full[st], kEvictFirst);
      }
    }
    __syncwarp();
  };
  pdl_wait();          // the plan (K3p), Q' (K2) and the appended rows (K1) come from the predecessors
  // Warp 3 (otherwise idle) fills the first ring stages straight after the wait: the range and the
  // first 32 box rows (resolved by K3p) are read in one round trip, concurrently with the CTA's plan
  // loads by the other warps (the producer, issuing after those, waited for a second dependent round
  // trip: ~2400 cycles of an h8 CTA's ~6400-cycle start, trace mode).  The empty ring needs no
  // kv_empty waits; the producer continues at stage n_early.
  // The softmax warps fetch the first segment's Q'_j / q^PE (plan entry, then the rows) before that
  // burst of cache loads reaches HBM (named barrier kQBar: queued behind it, the fetch took ~7 K
  // cycles and became the start's critical path, trace mode).
  static_assert(C::NST * C::SUB < 32, "the early stages come from the first batch of box rows");
  constexpr uint32_t kQBar = 13;                        // 8 softmax warps + warp 3
  QRegs q0;
  bool q0_ok = false;
  if (warp == 3) {
    const int32_t* pl = a.plan;
    const int rows_first = pl[n_cta * kPlanStride + 2 * a.B + 1 + c * 32 + lane];
    const int lo0 = pl[c * kPlanStride], hi0 = pl[c * kPlanStride + 1];
    const int n_early = max(0, min(C::NST, hi0 - lo0));
    named_bar_sync(kQBar, 288);
    if (lane == 0) EV(2);
    for (int g = 0; g < n_early; ++g) issue_stage(g, rows_first);
    s_rows[lane] = rows_first;                          // the producer's first batch (a reload would queue
                                                        // behind the burst: ~8 K cycles, the ring drained)
  } else if (warp >= 4) {
    const int32_t* pl = a.plan;
    const int b0 = pl[c * kPlanStride + 2], b1 = pl[c * kPlanStride + 3];
    q0_ok = b0 <= b1;
    if (q0_ok) q_fetch(b0, q0);
    named_bar_arrive(kQBar, 288);
  }
  if (warp != 3) {
    const int32_t* pl = a.plan;
    const int off_cum = n_cta * kPlanStride, off_slen = off_cum + a.B + 1;
    const int i0 = tid < 96 ? tid : tid - 32;           // every thread but warp 3's
    for (int i = i0; i <= a.B; i += kThreads - 32) cum[i] = pl[off_cum + i];
    for (int i = i0; i < a.B; i += kThreads - 32) slen[i] = pl[off_slen + i];
    if (tid < 5) s_sched[tid] = pl[c * kPlanStride + tid];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) EV(11);
  if ((MODE & 2) && tid == 0) {
    a.trace[kSlots * kTrace + 2 * c] = globaltimer();
    a.trace[kSlots * kTrace + 2 * kMaxCta + 2 * c] = clock64();
  }
  const uint32_t tb = tmem_base;
  Sched S;
  S.lo = s_sched[0];
  S.hi = s_sched[1];
  S.b_first = s_sched[2];
  S.b_last = s_sched[3];
  S.seg_base = s_sched[4];

  if (warp == 0) {
    // ============================================================ TMA producer (converged warp, one issuer)
    // Tile t of the flattened list -> cache rows of its TT/64 boxes (a 64-row box never
    // straddles a page: page_size % 64 == 0).  The page-table lookups are dependent global loads;
    // done one tile at a time they paced the producer at ~800 cycles per tile (measured: the
    // W = 128 shapes were producer-bound).  Each lane resolves one of the next 32 boxes, a batch
    // ahead, so the lookup latency is paid once per 32 boxes and hidden behind the previous batch.
    // Boxes wholly past the sequence end re-load the tile's first box (masked in the softmax).
    auto lookup = [&](int u) {                         // u = box index within this CTA's range
      const int tt = S.lo + u / C::SUB;
      if (tt >= S.hi) return 0;
      const int bb = upper_bound_cum(cum, a.B + 1, tt) - 1;
      const int tok0 = (tt - cum[bb]) * C::TT;
      int tok = tok0 + (u % C::SUB) * kSub;
      if (tok >= slen[bb]) tok = tok0;
      return a.block_table[(long)bb * a.max_pages + tok / a.page_size] * a.page_size + tok % a.page_size;
    };
    const int n_early = max(0, min(C::NST, S.hi - S.lo));   // stages warp 3 issued
    int rows_cur = s_rows[lane];                       // K3p resolved the first 32 (warp 3 read them)
    int rows_next = lookup(32 + lane);                 // (in flight while the first batch streams)
    if (lane == 0) EV(3);
    for (int t = S.lo + n_early, g = n_early; t < S.hi; ++t, ++g) {
      const int u0 = g * C::SUB;                       // SUB divides 32: a tile never spans batches
      if (u0 > 0 && (u0 & 31) == 0) {
        rows_cur = rows_next;
        rows_next = lookup(u0 + 32 + lane);
      }
      mbar_wait(&kv_empty[g % C::NST], ((g / C::NST) & 1) ^ 1);
      issue_stage(g, rows_cur);
    }
  } else if (MODE == 1 && warp == 1) {
    int g = 0;
    for (int b = S.b_first; b <= S.b_last; ++b)
      for (int t = max(S.lo, cum[b]); t < min(S.hi, cum[b + 1]); ++t, ++g) {
        mbar_wait(&kv_full[g % C::NST], (g / C::NST) & 1);
        if (elect_one()) mbar_arrive(&kv_empty[g % C::NST]);
        __syncwarp();
      }
  } else if (MODE == 1) {
    if (warp == 4 && lane == 0) {   // keep K4's segment map valid (values are meaningless)
      int seg = 0;
      for (int b = S.b_first; b <= S.b_last; ++b, ++seg) {
        if (max(S.lo, cum[b]) == cum[b]) a.meta[2 * b] = S.seg_base + seg;
        if (min(S.hi, cum[b + 1]) == cum[b + 1]) a.meta[2 * b + 1] = S.seg_base + seg;
      }
    }
  } else if ((MODE & 2) && warp == 3) {
    // trace only: observe when each tile lands (the MMA warp sees kv_full only when it gets to it)
    if (blockIdx.x == a.trace_cta)
      for (int g = 0; g < S.hi - S.lo && g < kTrace; ++g) {
        while (!mbar_try_wait(&kv_full[g % C::NST], (g / C::NST) & 1)) {
        }
        if (lane == 0) TRACE(22, g);
      }
  } else if (C::SPLIT && (warp == 1 || warp == 2)) {
    // ============================================================ MMA issuers, split: w1 QK, w2 PV
    // One issuing warp spent ~1340 cycles per 128-token tile on its waits, elects and descriptor
    // setup (trace, W_lat = 64) for 768 cycles of tensor work.  Two independent loops halve the
    // steps each warp takes per tile; their ordering constraints become mbarrier waits:
    //   QK(g) needs its tile (kv_full), its segment's Q' (q_ready) and S buffer g % NSB free: the
    //         PV of tile g - NSB complete (pv_done, committed by the PV warp);
    //   PV(g) needs P(g) (p_full; implies QK(g) complete, and for a segment's first PV that the
    //         previous segment's epilogue has read O).  Its commits release the ring stage
    //         (both MMAs of the tile have read it) and signal pv_done.
    // (tcgen05.commit tracks the issuing thread's own MMAs: each warp commits what it issued.)
    constexpr uint32_t id_qk = idesc_bf16(128, C::TT, false, false);
    constexpr uint32_t id_pv = idesc_bf16(128, C::WL, false, true);
    constexpr uint32_t hi_k = desc_sw128_hi(1024);           // K-major: SBO = 1024 B (8-row groups)
    const uint32_t kv0 = smem_addr(s_kv);
    int g = 0, seg = 0;
    if (warp == 1) {
      const uint64_t qpe_desc = make_desc(smem_addr(s_qpe), 16, hi_k);
      for (int b = S.b_first; b <= S.b_last; ++b, ++seg) {
        const int t0 = max(S.lo, cum[b]), t1 = min(S.hi, cum[b + 1]);
        mbar_wait(&q_ready, seg & 1);
        if (seg == 0 && lane == 0) EV(6);
        for (int t = t0; t < t1; ++t, ++g) {
          const int st = g % C::NST, sb = g % C::NSB;
          if (lane == 0) TRACE(19, g);
          mbar_wait(&kv_full[st], (g / C::NST) & 1);
          if (g >= C::NSB) mbar_wait(&pv_done[sb], ((g / C::NSB) & 1) ^ 1);   // PV(g - NSB) complete
          if (lane == 0) TRACE(20, g);
          if (g == 0 && lane == 0) EV(7);
          tc_fence_after();
          if (elect_one()) {
            TRACE(0, g);
            const uint64_t kv_desc = make_desc(kv0 + st * C::STAGE_BYTES, 16, hi_k);
            const uint32_t s_tmem = tb + C::S_COL0 + sb * C::TT;
#pragma unroll
            for (int kk = 0; kk < C::WL / 16; ++kk)
              if (!(MODE & 32))
                mma_ts(s_tmem, tb + C::Q_COL + kk * 8,
                       kv_desc + uint64_t(((kk >> 2) * C::BOX_BYTES + (kk & 3) * 32) >> 4), id_qk, kk > 0 ? 1u : 0u);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              if (!(MODE & 32))
                mma_ss(s_tmem, qpe_desc + uint64_t(kk * 2),
                       kv_desc + uint64_t(((C::NBOX - 1) * C::BOX_BYTES + kk * 32) >> 4), id_qk, 1u);
            mma_commit(&s_full[sb]);
            TRACE(4, g);
          }
          __syncwarp();
        }
      }
    } else {
      for (int b = S.b_first; b <= S.b_last; ++b) {
        const int t0 = max(S.lo, cum[b]), t1 = min(S.hi, cum[b + 1]);
        for (int t = t0; t < t1; ++t, ++g) {
          const int st = g % C::NST, sb = g % C::NSB;
          if (lane == 0) TRACE(21, g);
          mbar_wait(&p_full[sb], (g / C::NSB) & 1);
          tc_fence_after();
          if (elect_one()) {
            TRACE(1, g);
            const uint64_t v_desc = make_desc(kv0 + st * C::STAGE_BYTES, C::BOX_BYTES, hi_k);
            const uint32_t p_tmem = tb + C::S_COL0 + sb * C::TT;
#pragma unroll
            for (int kk = 0; kk < C::TT / 16; ++kk)
              if (!(MODE & 32))
                mma_ts(tb + C::O_COL, p_tmem + kk * 8, v_desc + uint64_t(kk * (2048 >> 4)), id_pv,
                       (t == t0 && kk == 0) ? 0u : 1u);
            mma_commit(&kv_empty[st]);
            mma_commit(&pv_done[sb]);
            TRACE(5, g);
          }
          __syncwarp();
        }
      }
    }
  } else if (warp == 1) {
    // ============================================================ MMA issuer (converged warp, one issuer)
    constexpr uint32_t id_qk = idesc_bf16(128, C::TT, false, false);
    constexpr uint32_t id_pv = idesc_bf16(128, C::WL, false, true);
    constexpr uint32_t hi_k = desc_sw128_hi(1024);           // K-major: SBO = 1024 B (8-row groups)
    const uint64_t qpe_desc = make_desc(smem_addr(s_qpe), 16, hi_k);
    const uint32_t kv0 = smem_addr(s_kv);
    int g = 0, seg = 0;
    auto issue_pv = [&](int gp, bool first_pv) {
      const int st = gp % C::NST;
      if (!C::PAIR && lane == 0) TRACE(21, gp);
      mbar_wait(&p_full[gp % C::NSB], (gp / C::NSB) & 1);
      tc_fence_after();
      if (elect_one()) {
        TRACE(1, gp);
        // V = latent boxes of the tile, MN-major: 64-column atoms one box (8 KB) apart
        const uint64_t v_desc = make_desc(kv0 + st * C::STAGE_BYTES, C::BOX_BYTES, hi_k);
        const uint32_t p_tmem = tb + C::S_COL0 + (gp % C::NSB) * C::TT;
#pragma unroll
        for (int kk = 0; kk < C::TT / 16; ++kk)      // 16 tokens (2 KB of rows) per step
          if (!(MODE & 32))
            mma_ts(tb + C::O_COL, p_tmem + kk * 8, v_desc + uint64_t(kk * (2048 >> 4)), id_pv,
                   (first_pv && kk == 0) ? 0u : 1u);
        mma_commit(&kv_empty[st]);
        mma_commit(&pv_done[gp % C::NSB]);
        TRACE(5, gp);
      }
      __syncwarp();
    };
    for (int b = S.b_first; b <= S.b_last; ++b, ++seg) {
      const int t0 = max(S.lo, cum[b]), t1 = min(S.hi, cum[b + 1]);
      const int g0 = g;
      mbar_wait(&q_ready, seg & 1);
      if (seg == 0 && lane == 0) EV(6);
      tc_fence_after();
      for (int t = t0; t < t1; ++t, ++g) {
        const int st = g % C::NST;
        if (!C::PAIR && lane == 0) TRACE(19, g);
        mbar_wait(&kv_full[st], (g / C::NST) & 1);
        if (!C::PAIR && lane == 0) TRACE(20, g);
        if (g == 0 && lane == 0) EV(7);
        tc_fence_after();
        if (elect_one()) {
          TRACE(0, g);
          const uint64_t kv_desc = make_desc(kv0 + st * C::STAGE_BYTES, 16, hi_k);
          const uint32_t s_tmem = tb + C::S_COL0 + (g % C::NSB) * C::TT;
#pragma unroll
          for (int kk = 0; kk < C::WL / 16; ++kk)     // Q'_j (TMEM) x ĉ tileᵀ: box kk/4, +32 B per k-step
            if (!(MODE & 32))
              mma_ts(s_tmem, tb + C::Q_COL + kk * 8,
                     kv_desc + uint64_t(((kk >> 2) * C::BOX_BYTES + (kk & 3) * 32) >> 4), id_qk, kk > 0 ? 1u : 0u);
          // q^PE x k^PE tileᵀ (last box), 4 k-steps of 16; PAIR: each rank takes two of them, so the
          // partial logits carry half of the RoPE term each and the two QKs take equal time
#pragma unroll
          for (int kk = (C::PAIR ? 2 * int(crank) : 0); kk < (C::PAIR ? 2 * int(crank) + 2 : 4); ++kk)
            if (!(MODE & 32))
              mma_ss(s_tmem, qpe_desc + uint64_t(kk * 2),
                     kv_desc + uint64_t(((C::NBOX - 1) * C::BOX_BYTES + kk * 32) >> 4), id_qk, 1u);
          mma_commit(&s_full[g % C::NSB]);
          TRACE(4, g);
        }
        __syncwarp();
        if (t - t0 >= C::LAG) issue_pv(g - C::LAG, g - C::LAG == g0);
      }
      for (int gp = max(g0, g - C::LAG); gp < g; ++gp) issue_pv(gp, gp == g0);
    }
  } else if (warp >= 4) {
    // ============================================================ softmax / Q loader / epilogue
    // Two warps per TMEM lane quadrant: warp 4+q handles S columns [0,32) (tokens 0-31 of the
    // tile), warp 8+q columns [32,64), for the same 32 head rows; they exchange their partial
    // row maxima through shared memory so both take the same rescale decisions.
    const uint32_t lane_base = tb + (uint32_t(q4 * 32) << 16);
    // Multi-token decode: token i of sequence b sits at position S_b - n_q + i and attends to the
    // first S_b - n_q + 1 + i cached tokens (causal among the new tokens, already in the cache).
    const bool q_active = q4 * 32 < n_rows;             // warp-uniform: this quadrant holds rows
    const int len_adj = tok_i + 1 - a.n_q;              // this row's visible length = S_b + len_adj
    const float sc = a.scale_log2;
    const uint32_t pair_bar = 1 + q4;                   // named barrier of the two warps of a quadrant
    // Q'_j row -> TMEM (A operand, bf16 pairs per 32-bit column), half of it per warp;
    // q^PE row -> swizzled smem (chunks 4*half .. 4*half+3); then signal the MMA warp
    auto q_store = [&](const QRegs& v, int bb) {
        if (q_loads) {
#pragma unroll
          for (int c0 = 0; c0 < QH; c0 += 32) {
            uint32_t w[32];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const uint4 u = v.q[c0 / 4 + k];
              w[4 * k] = u.x; w[4 * k + 1] = u.y; w[4 * k + 2] = u.z; w[4 * k + 3] = u.w;
            }
            tmem_st32(lane_base + C::Q_COL + q_cbegin + c0, w);
          }
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int ch = 4 * half + c;
          *reinterpret_cast<uint4*>(s_qpe + r * 128 + ((ch ^ (r & 7)) << 4)) = v.pe[c];
        }
        fence_proxy_async_smem();
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&q_ready);
        if (warp == 4 && lane == 0 && bb == S.b_first) EV(5);
    };
    // (the loads are all issued before the Q' TMEM stores, which are asm volatile with a memory
    // clobber: loads placed after them would wait for a second round trip)
    auto load_q = [&](int bb) {
        QRegs v;
        q_fetch(bb, v);
        q_store(v, bb);
    };
    if constexpr (C::PP) {
    // ---- ping-pong softmax (TT = 128).  Warp set `half` takes the tiles with g % 2 == half, whole
    // 128-column rows.  A tile's exponentials use a provisional running max read from m_row
    // (the max the previous tile's warp published) — no max pass; the tiles are then finalised in
    // order (named barriers between the two warps of the quadrant): if the provisional max turns
    // out stale, or a row's tile sum leaves [0, 2^20] (p may exceed 2^20 only when the max grew:
    // the lazy-rescale condition, with inf/NaN caught by the same test), the tile's logits (still
    // in TMEM: P is stored only after finalising) are reloaded and redone with the exact rule.
    // The first tile of a segment takes its exact row max.
    const uint32_t fin_mine = 5 + 2 * q4 + half, fin_other = 5 + 2 * q4 + (half ^ 1);
    constexpr float kLim = 1048576.f;                   // 2^20
    volatile float* mrow = m_row;
    auto row_max = [&](const float* x) {
      float m0 = x[0], m1 = x[1], m2 = x[2], m3 = x[3];
#pragma unroll
      for (int j = 4; j < C::TT; j += 4) {
        m0 = fmaxf(m0, x[j]); m1 = fmaxf(m1, x[j + 1]); m2 = fmaxf(m2, x[j + 2]); m3 = fmaxf(m3, x[j + 3]);
      }
      return fmaxf(fmaxf(m0, m1), fmaxf(m2, m3));
    };
    // p = 2^(x·sc − m) for the row's 128 columns -> bf16 pairs pw, and the row's tile sum
    auto exps = [&](const float* x, float m, uint32_t (&pw)[C::TT / 2]) {
      const float neg_m = m == -INFINITY ? 0.f : -m;    // (a row with nothing visible: p = 0)
      const uint64_t sc2 = f2_pack(sc, sc), nm2 = f2_pack(neg_m, neg_m);
      uint64_t l01 = f2_pack(0.f, 0.f), l23 = f2_pack(0.f, 0.f);
#pragma unroll
      for (int j = 0; j < C::TT / 2; j += 2) {
        float y0, y1, y2, y3;
        f2_unpack(ffma2(f2_pack(x[2 * j], x[2 * j + 1]), sc2, nm2), y0, y1);
        f2_unpack(ffma2(f2_pack(x[2 * j + 2], x[2 * j + 3]), sc2, nm2), y2, y3);
        const float p0 = ex2(y0), p1 = ex2(y1);
        float p2, p3;
        if (kPolyEvery<W_LAT> > 0 && (j / 2) % kPolyEvery<W_LAT> == 0) {
          ex2_poly2<true>(y2, y3, p2, p3);
        } else {
          p2 = ex2(y2);
          p3 = ex2(y3);
        }
        l01 = fadd2(l01, f2_pack(p0, p1));
        l23 = fadd2(l23, f2_pack(p2, p3));
        pw[j] = pack_bf16x2(p0, p1);
        pw[j + 1] = pack_bf16x2(p2, p3);
      }
      float a0, a1, a2, a3;
      f2_unpack(l01, a0, a1);
      f2_unpack(l23, a2, a3);
      return (a0 + a1) + (a2 + a3);
    };
    int g = 0, seg = 0;
    if (q0_ok) q_store(q0, S.b_first);               // fetched in the prologue
    for (int b = S.b_first; b <= S.b_last; ++b, ++seg) {
      const int t0 = max(S.lo, cum[b]), t1 = min(S.hi, cum[b + 1]);
      const int S_b = slen[b] + len_adj;                 // this row's visible length
      float m_w = -INFINITY;                             // the max this warp's sum l_w is expressed in
      float l_w = 0.f;
      for (int t = t0; t < t1; ++t, ++g) {
        if ((g & 1) != half) continue;
        const int sb = g % C::NSB;
        if (q4 == 0 && lane == 0) TRACE(18, g);
        mbar_wait(&s_full[sb], (g / C::NSB) & 1);
        if (q4 == 0 && lane == 0) TRACE(2, g);
        if (!q_active || (MODE & 16)) {                  // no head rows here: P stays 0 (S rows are 0)
          if (lane == 0) mbar_arrive(&p_full[sb]);
          continue;
        }
        tc_fence_after();
        const uint32_t s_addr = lane_base + C::S_COL0 + sb * C::TT;
        uint32_t sv[C::TT / 32][32];
        float* x = reinterpret_cast<float*>(&sv[0][0]);
        const int nvalid = S_b - (t - cum[b]) * C::TT;   // (per row when n_q > 1)
        auto load_s = [&]() {
#pragma unroll
          for (int q = 0; q < C::TT / 32; ++q) tmem_ld32(s_addr + 32 * q, sv[q]);
          tmem_ld_wait();
          if (nvalid < C::TT) {                          // ragged last tile of the sequence
#pragma unroll
            for (int j = 0; j < C::TT; ++j) x[j] = j < nvalid ? x[j] : -INFINITY;
          }
        };
        load_s();
        if (q4 == 0 && lane == 0) TRACE(15, g);
        const float m_prov = t == t0 ? row_max(x) * sc : mrow[r];   // sc > 0: max commutes with scaling
        uint32_t pw[C::TT / 2];
        float ts = exps(x, m_prov, pw);
        if (q4 == 0 && lane == 0) TRACE(16, g);
        // ---- finalise in tile order: tile g-1 (the other warp) has published its final max
        if (t > t0) named_bar_sync(fin_other, 64);
        if (q4 == 0 && lane == 0) TRACE(17, g);
        const float m_prev = t > t0 ? mrow[r] : -INFINITY;
        const bool redo = !(ts <= kLim) || (t > t0 && m_prov != m_prev);
        float m_fin = m_prov;
        if (__any_sync(0xffffffffu, redo)) {             // rare: reload the logits, exact rule
          load_s();
          const float mx = row_max(x) * sc;
          if (redo) m_fin = mx > m_prev + kRescaleThreshold ? mx : m_prev;
          ts = exps(x, m_fin, pw);
        }
        // O holds PV(g-1) and earlier at m_prev: rescale the rows whose max grew (warp-collective)
        const bool grow = t > t0 && m_fin != m_prev;
        if (__any_sync(0xffffffffu, grow)) {
          const float f = grow ? ex2(m_prev - m_fin) : 1.f;
          mbar_wait(&pv_done[(g - 1) % C::NSB], ((g - 1) / C::NSB) & 1);
          tc_fence_after();
#pragma unroll 1
          for (int c0 = 0; c0 < C::WL; c0 += 32) {
            uint32_t ov[32];
            tmem_ld32(lane_base + C::O_COL + c0, ov);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) ov[j] = __float_as_uint(__uint_as_float(ov[j]) * f);
            tmem_st32(lane_base + C::O_COL + c0, ov);
          }
        }
        mrow[r] = m_fin;
        if (m_fin != m_w) {                              // this warp's sum follows the row's max
          l_w = m_w == -INFINITY ? 0.f : l_w * ex2(m_w - m_fin);
          m_w = m_fin;
        }
        l_w += ts;
        // P (bf16 pairs) over columns [0, TT/2) of S(g)
#pragma unroll
        for (int q = 0; q < C::TT / 64; ++q) {
          uint32_t (&pq)[32] = *reinterpret_cast<uint32_t(*)[32]>(&pw[32 * q]);
          tmem_st32(s_addr + 32 * q, pq);
        }
        tmem_st_wait();
        tc_fence_before();
        if (q4 == 0 && lane == 0) TRACE(3, g);
        if (lane == 0) TRACE(6 + warp - 4, g);
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[sb]);
        if (t + 1 < t1) {                                // the other warp finalises tile g+1 next
#ifndef TPLA_K3_NO_FENCE
          __threadfence_block();
#endif
          named_bar_arrive(fin_mine, 64);
        }
      }
      // Stage the next segment's Q once the segment's last QK is complete (the other warp may
      // have consumed that S), so its first QKs overlap this epilogue.
      mbar_wait(&s_full[(g - 1) % C::NSB], ((g - 1) / C::NSB) & 1);
      tc_fence_after();
      if (b < S.b_last) load_q(b + 1);
      if (!q_active) continue;
      // ---- epilogue of the segment: unnormalised partial (O, m, l); the two sets' sums meet
      red_l[half][r] = l_w;
      red_m[half][r] = m_w;
      mbar_wait(&pv_done[(g - 1) % C::NSB], ((g - 1) / C::NSB) & 1);
      tc_fence_after();
      named_bar_sync(pair_bar, 64);
      const float m_o = red_m[half ^ 1][r], l_o = red_l[half ^ 1][r];
      const float m_seg = fmaxf(m_w, m_o);              // the last tile's max (maxima only grow)
      const float l = (m_w == -INFINITY ? 0.f : l_w * ex2(m_w - m_seg)) +
                      (m_o == -INFINITY ? 0.f : l_o * ex2(m_o - m_seg));
      const int seg_id = S.seg_base + seg;
      {
        // the partial leaves normalised (O / l, values of the cache's range) in fp16: half the bytes of
        // fp32 at 2^-11 relative rounding (R23)
        uint16_t* op = a.o_part + ((long)seg_id * n_rows + r) * W_LAT;
        const float inv_l = 1.f / l;
#pragma unroll 1
        for (int c0 = half * (C::WL / 2); c0 < (half + 1) * (C::WL / 2); c0 += 32) {
          uint32_t ov[32];
          tmem_ld32(lane_base + C::O_COL + c0, ov);
          tmem_ld_wait();
          if (row_ok) {
#pragma unroll
            for (int j = 0; j < 32; j += 8)
              *reinterpret_cast<uint4*>(op + c0 + j) =
                  make_uint4(pack_f16(__uint_as_float(ov[j]) * inv_l, __uint_as_float(ov[j + 1]) * inv_l),
                             pack_f16(__uint_as_float(ov[j + 2]) * inv_l, __uint_as_float(ov[j + 3]) * inv_l),
                             pack_f16(__uint_as_float(ov[j + 4]) * inv_l, __uint_as_float(ov[j + 5]) * inv_l),
                             pack_f16(__uint_as_float(ov[j + 6]) * inv_l, __uint_as_float(ov[j + 7]) * inv_l));
          }
        }
        if (row_ok && half == 0) {
          a.ml_part[((long)seg_id * n_rows + r) * 2] = m_seg;
          a.ml_part[((long)seg_id * n_rows + r) * 2 + 1] = l;
        }
      }
      if (r == 0 && half == 0 && t0 == cum[b]) a.meta[2 * b] = seg_id;
      if (r == 0 && half == 0 && t1 == cum[b + 1]) a.meta[2 * b + 1] = seg_id;
      named_bar_sync(pair_bar, 64);                     // red_l / red_m free again
      tc_fence_before();
    }
    } else {
    int g = 0, seg = 0;
    int xk = 0;                                          // PAIR: logit exchanges done by this warp
    if (q0_ok) q_store(q0, S.b_first);               // fetched in the prologue
    for (int b = S.b_first; b <= S.b_last; ++b, ++seg) {
      const int t0 = max(S.lo, cum[b]), t1 = min(S.hi, cum[b + 1]);
      const int S_b = slen[b] + len_adj;                 // this row's visible length
      float m_used = -INFINITY;                          // running max, log2 units (same in both halves)
      float l0 = 0.f, l1 = 0.f, l2 = 0.f, l3 = 0.f;      // this half's running sum (4 chains)
      for (int t = t0; t < t1; ++t, ++g) {
        const int sb = g % C::NSB;
        if (warp == 4 && lane == 0) TRACE(18, g);
        mbar_wait(&s_full[sb], (g / C::NSB) & 1);
        if (warp == 4 && lane == 0) TRACE(2, g);
        if (!q_active) {                                 // no head rows here: P stays 0 (S rows are 0)
          if (lane == 0) mbar_arrive(&p_full[sb]);
          continue;
        }
        tc_fence_after();
        constexpr int CH = C::CH;
        uint32_t sv[CH / 32][32];
        if (MODE & 8) {                                 // diagnostic: no TMEM traffic in softmax
#pragma unroll
          for (int q = 0; q < CH / 32; ++q)
#pragma unroll
            for (int j = 0; j < 32; ++j) sv[q][j] = __float_as_uint(float((lane * 7 + j * 3 + g + q) & 15));
        } else {
#pragma unroll
          for (int q = 0; q < CH / 32; ++q) tmem_ld32(lane_base + C::S_COL0 + sb * C::TT + CH * half + 32 * q, sv[q]);
          tmem_ld_wait();
        }
        if constexpr (C::PAIR) {
          // Send this CTA's partial logits (its latent half + half of the RoPE term) into the peer's
          // buffer, receive the peer's into ours, add: both CTAs then hold the exact logits
          // (a + b == b + a in fp32, so the two softmaxes are bit-identical).
          // buffer of this warp: float4 group v of lane l at [v][l] (conflict-free 16-byte accesses)
          const int xw = warp - 4;
          float* xb = s_xch + xw * 32 * CH + lane * 4;
          const uint32_t peer = crank ^ 1u;
          mbar_wait_poll(&x_ok[xw], (xk & 1) ^ 1);       // the peer consumed our previous send
          if (warp == 4 && lane == 0) TRACE(19, g);
          float* xs = xb + 8 * 32 * CH;                    // this warp's send staging buffer
#pragma unroll
          for (int q = 0; q < CH / 32; ++q)
#pragma unroll
            for (int v = 0; v < 8; ++v)
              *reinterpret_cast<uint4*>(xs + (8 * q + v) * 32 * 4) =
                  make_uint4(sv[q][4 * v], sv[q][4 * v + 1], sv[q][4 * v + 2], sv[q][4 * v + 3]);
          fence_proxy_async_smem();                        // generic stores -> visible to the bulk copy
          __syncwarp();
          if (lane == 0) {
            mbar_arrive_expect_tx(&x_full[xw], 32 * CH * 4);
            bulk_copy_to_peer(mapa(smem_addr(s_xch + xw * 32 * CH), peer), s_xch + 8 * 32 * CH + xw * 32 * CH,
                              32 * CH * 4, mapa(smem_addr(&x_full[xw]), peer));
          }
          if (warp == 4 && lane == 0) TRACE(20, g);
          mbar_wait_poll(&x_full[xw], xk & 1);
          if (warp == 4 && lane == 0) TRACE(21, g);
#pragma unroll
          for (int q = 0; q < CH / 32; ++q)
#pragma unroll
            for (int v = 0; v < 8; ++v) {
              const float4 o = *reinterpret_cast<const float4*>(xb + (8 * q + v) * 32 * 4);
              sv[q][4 * v] = __float_as_uint(__uint_as_float(sv[q][4 * v]) + o.x);
              sv[q][4 * v + 1] = __float_as_uint(__uint_as_float(sv[q][4 * v + 1]) + o.y);
              sv[q][4 * v + 2] = __float_as_uint(__uint_as_float(sv[q][4 * v + 2]) + o.z);
              sv[q][4 * v + 3] = __float_as_uint(__uint_as_float(sv[q][4 * v + 3]) + o.w);
            }
          __syncwarp();
          // (relaxed: the buffer's reads above have returned; a release arrive cost ~1500 cycles)
          if (lane == 0) mbar_arrive_remote_relaxed(mapa(smem_addr(&x_ok[xw]), peer));
          ++xk;
        }
        if (warp == 4 && lane == 0) TRACE(15, g);
        float* x = reinterpret_cast<float*>(&sv[0][0]); // raw logits (sm_scale not applied yet)
        const int nvalid = S_b - (t - cum[b]) * C::TT - CH * half;   // (per row when n_q > 1)
        if (nvalid < CH) {                               // ragged last tile of the sequence
#pragma unroll
          for (int j = 0; j < CH; ++j) x[j] = j < nvalid ? x[j] : -INFINITY;
        }
        float m0 = x[0], m1 = x[1], m2 = x[2], m3 = x[3];
#pragma unroll
        for (int j = 4; j < CH; j += 4) {
          m0 = fmaxf(m0, x[j]); m1 = fmaxf(m1, x[j + 1]); m2 = fmaxf(m2, x[j + 2]); m3 = fmaxf(m3, x[j + 3]);
        }
        float mx = fmaxf(fmaxf(m0, m1), fmaxf(m2, m3));
        red_max[sb][half][r] = mx;
        named_bar_sync(pair_bar, 64);
        mx = fmaxf(mx, red_max[sb][half ^ 1][r]) * sc;   // sc > 0: max commutes with scaling
        if (warp == 4 && lane == 0) TRACE(16, g);
        // Raise the running max only when it grew by more than 2^8 (p stays <= 256 in between).
        // The decision is per row (identical in both halves), but TMEM loads/stores are
        // warp-collective (.sync.aligned), so a warp rescales if any of its rows needs it.
        const bool need = mx > m_used + kRescaleThreshold;
        if (__any_sync(0xffffffffu, need)) {
          const float m_new = need ? mx : m_used;
          if (t > t0) {
            // O holds PV(g-1) and earlier: wait for it, then scale this half's O columns
            const float f = need ? ex2(m_used - m_new) : 1.f;
            mbar_wait(&pv_done[(g - 1) % C::NSB], ((g - 1) / C::NSB) & 1);
            tc_fence_after();
#pragma unroll 1
            for (int c0 = half * (C::WL / 2); c0 < (half + 1) * (C::WL / 2); c0 += 32) {
              uint32_t ov[32];
              tmem_ld32(lane_base + C::O_COL + c0, ov);
              tmem_ld_wait();
#pragma unroll
              for (int j = 0; j < 32; ++j) ov[j] = __float_as_uint(__uint_as_float(ov[j]) * f);
              tmem_st32(lane_base + C::O_COL + c0, ov);
            }
            l0 *= f; l1 *= f; l2 *= f; l3 *= f;
          }
          m_used = m_new;
        }
        // Paired fp32 ops (FFMA2 / FADD2: two lanes of work per instruction) for the scale-and-
        // subtract and the row sums; the loop is close to both the MUFU and the issue limit, so
        // only a small share of the exponentials moves to the FMA-pipe polynomial (kPolyEvery).
        // (a row with no visible token yet keeps m = -inf and must give p = 0, not NaN)
        const float neg_m = m_used == -INFINITY ? 0.f : -m_used;
        const uint64_t sc2 = f2_pack(sc, sc), nm2 = f2_pack(neg_m, neg_m);
        uint64_t l01 = f2_pack(l0, l1), l23 = f2_pack(l2, l3);
        uint32_t pw[CH / 2];
#pragma unroll
        for (int j = 0; j < CH / 2; j += 2) {
          float y0, y1, y2, y3;
          f2_unpack(ffma2(f2_pack(x[2 * j], x[2 * j + 1]), sc2, nm2), y0, y1);
          f2_unpack(ffma2(f2_pack(x[2 * j + 2], x[2 * j + 3]), sc2, nm2), y2, y3);
          const float p0 = ex2(y0), p1 = ex2(y1);
          float p2, p3;
          if (kPolyEvery<W_LAT> > 0 && (j / 2) % kPolyEvery<W_LAT> == 0) {
            ex2_poly2(y2, y3, p2, p3);                   // this pair on the FMA pipe (MUFU relief)
          } else {
            p2 = ex2(y2);
            p3 = ex2(y3);
          }
          l01 = fadd2(l01, f2_pack(p0, p1));
          l23 = fadd2(l23, f2_pack(p2, p3));
          pw[j] = pack_bf16x2(p0, p1);
          pw[j + 1] = pack_bf16x2(p2, p3);
        }
        f2_unpack(l01, l0, l1);
        f2_unpack(l23, l2, l3);
        if (warp == 4 && lane == 0) TRACE(17, g);
        // P (bf16 pairs) over columns [CH/2*half, CH/2*(half+1)) of S(g): tokens CH*half .. +CH-1
        const uint32_t p_addr = lane_base + C::S_COL0 + sb * C::TT + (CH / 2) * half;
        if (!(MODE & 8) || pw[0] == 0x7fc00001u) {       // (diagnostic nold: keep the math, skip the store)
          if constexpr (CH == 64) tmem_st32(p_addr, pw);
          else tmem_st16(p_addr, pw);
        }
        tmem_st_wait();
        tc_fence_before();
        if (warp == 4 && lane == 0) TRACE(3, g);
        if (lane == 0) TRACE(6 + warp - 4, g);
        // one arrival per warp: 32 lane arrivals cost ~350 cycles per tile (measured)
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[sb]);
      }
      // The segment's QKs are all complete (its last S was just consumed): stage the next
      // segment's Q now, so its first QKs run on the tensor pipe during this epilogue.  Its
      // first PV still waits for this epilogue: it needs p_full, which these warps signal later.
      if (b < S.b_last) load_q(b + 1);
      if (!q_active) continue;                          // (both warps of the quadrant skip)
      // ---- epilogue of the segment: unnormalised partial (O, m, l)
      float l = (l0 + l1) + (l2 + l3);
      red_l[half][r] = l;
      mbar_wait(&pv_done[(g - 1) % C::NSB], ((g - 1) / C::NSB) & 1);
      tc_fence_after();
      named_bar_sync(pair_bar, 64);
      l += red_l[half ^ 1][r];
      const int seg_id = S.seg_base + seg;
      {
        uint16_t* op = a.o_part + ((long)seg_id * n_rows + r) * W_LAT + crank * C::WL;   // (fp16 O / l)
        const float inv_l = 1.f / l;
#pragma unroll 1
        for (int c0 = half * (C::WL / 2); c0 < (half + 1) * (C::WL / 2); c0 += 32) {
          uint32_t ov[32];
          tmem_ld32(lane_base + C::O_COL + c0, ov);     // whole warp (.sync.aligned)
          tmem_ld_wait();
          if (row_ok) {
#pragma unroll
            for (int j = 0; j < 32; j += 8)
              *reinterpret_cast<uint4*>(op + c0 + j) =
                  make_uint4(pack_f16(__uint_as_float(ov[j]) * inv_l, __uint_as_float(ov[j + 1]) * inv_l),
                             pack_f16(__uint_as_float(ov[j + 2]) * inv_l, __uint_as_float(ov[j + 3]) * inv_l),
                             pack_f16(__uint_as_float(ov[j + 4]) * inv_l, __uint_as_float(ov[j + 5]) * inv_l),
                             pack_f16(__uint_as_float(ov[j + 6]) * inv_l, __uint_as_float(ov[j + 7]) * inv_l));
          }
        }
        if (row_ok && half == 0 && crank == 0) {
          a.ml_part[((long)seg_id * n_rows + r) * 2] = m_used;
          a.ml_part[((long)seg_id * n_rows + r) * 2 + 1] = l;
        }
      }
      // publish the sequence's segment range for K4: the CTA holding its first tile writes the
      // first segment id, the CTA holding its last tile the last one (ids are contiguous)
      if (r == 0 && half == 0 && crank == 0 && t0 == cum[b]) a.meta[2 * b] = seg_id;
      if (r == 0 && half == 0 && crank == 0 && t1 == cum[b + 1]) a.meta[2 * b + 1] = seg_id;
      named_bar_sync(pair_bar, 64);                     // red_l free again
      tc_fence_before();
    }
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if ((MODE & 2) && tid == 0) {
    a.trace[kSlots * kTrace + 2 * c + 1] = globaltimer();
    a.trace[kSlots * kTrace + 2 * kMaxCta + 2 * c + 1] = clock64();
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    long long* ci = a.trace + kSlots * kTrace + 4 * kMaxCta + 16;   // per-CTA (smid, tiles, segments)
    ci[3 * c] = smid;
    ci[3 * c + 1] = S.hi - S.lo;
    ci[3 * c + 2] = S.b_last - S.b_first + 1;
  }
  if (C::PAIR) cluster_sync();   // the peer may still be writing into our smem / arriving on our barriers
  if (warp == 2) tmem_dealloc<C::TMEM_COLS>(tb);
}

// K4 for the persistent kernel: O = Σ_s 2^{m_s - M} l_s Ô_s / Σ_s 2^{m_s - M} l_s over the
// contiguous segment range of sequence b (Ô_s = O_s / l_s, the fp16 partials)
__global__ void combine_seg_kernel(const uint16_t* __restrict__ o_part, const float* __restrict__ ml_part,
                                   const int32_t* __restrict__ meta, int h_loc, int w_lat,
                                   uint16_t* __restrict__ o_bf16, float* __restrict__ o_f32, float* __restrict__ lse) {
  pdl_trigger();
  pdl_wait();
  const int h = blockIdx.x, b = blockIdx.y;
  const int s0 = meta[2 * b], ns = meta[2 * b + 1] - s0 + 1;
  float M = -INFINITY;
  for (int s = 0; s < ns; ++s) M = fmaxf(M, ml_part[((long)(s0 + s) * h_loc + h) * 2]);
  float L = 0.f;
  for (int s = 0; s < ns; ++s) {
    const float* ml = ml_part + ((long)(s0 + s) * h_loc + h) * 2;
    L += exp2f(ml[0] - M) * ml[1];
  }
  const float inv = 1.f / L;
  for (int col = threadIdx.x * 4; col < w_lat; col += blockDim.x * 4) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < ns; ++s) {
      const float* ml = ml_part + ((long)(s0 + s) * h_loc + h) * 2;
      const float w = exp2f(ml[0] - M) * ml[1];
      const uint2 u = *reinterpret_cast<const uint2*>(o_part + ((long)(s0 + s) * h_loc + h) * w_lat + col);
      acc.x += w * f16_lo(u.x); acc.y += w * f16_hi(u.x); acc.z += w * f16_lo(u.y); acc.w += w * f16_hi(u.y);
    }
    acc.x *= inv; acc.y *= inv; acc.z *= inv; acc.w *= inv;
    const long off = ((long)b * h_loc + h) * w_lat + col;
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

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
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

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int W_LAT, int MODE>
cudaError_t launch_tc_mode(const CUtensorMap& map, const TcArgs& a, int n_cta, cudaStream_t s) {
  using C = Cfg<W_LAT>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e =
        cudaFuncSetAttribute(attn_tc_kernel<W_LAT, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  KernelScope ks(MODE == 0 ? "K3_attn_tc" : "K3_stream_only", s);
  // PAIR: n_cta logical CTAs = n_cta clusters of two
  return launch_kc(attn_tc_kernel<W_LAT, MODE>, C::PAIR ? 2 : 1, C::PAIR ? 2 * n_cta : n_cta, kThreads, C::SMEM, s,
                   map, a);
}

template <int W_LAT>
cudaError_t launch_tc(const CUtensorMap& map, const TcArgs& a, int n_cta, cudaStream_t s) {
  static const char* mode = getenv("TPLA_K3_MODE");
  if (mode && strcmp(mode, "stream") == 0) return launch_tc_mode<W_LAT, 1>(map, a, n_cta, s);
  if (mode && strcmp(mode, "nold") == 0) return launch_tc_mode<W_LAT, 8>(map, a, n_cta, s);
  if (mode && strcmp(mode, "notma") == 0) return launch_tc_mode<W_LAT, 4>(map, a, n_cta, s);
  if (mode && strcmp(mode, "nosm") == 0) return launch_tc_mode<W_LAT, 4 | 16>(map, a, n_cta, s);
  if (mode && strcmp(mode, "nomma") == 0) return launch_tc_mode<W_LAT, 4 | 32>(map, a, n_cta, s);
  if (mode && strncmp(mode, "trace", 5) == 0) {   // trace, trace_notma, trace_nold
    static long long* buf = nullptr;
    const int nb = kSlots * kTrace + 2 * n_cta;
    if (!buf) cudaMalloc(&buf, (kSlots * kTrace + 7 * kMaxCta + 16) * sizeof(long long));
    TcArgs b = a;
    b.trace = buf;
    const char* tc = getenv("TPLA_K3_TRACE_CTA");
    b.trace_cta = tc ? atoi(tc) : 0;
    cudaError_t e = strcmp(mode, "trace_notma") == 0   ? launch_tc_mode<W_LAT, 6>(map, b, n_cta, s)
                    : strcmp(mode, "trace_nosm") == 0  ? launch_tc_mode<W_LAT, 2 | 4 | 16>(map, b, n_cta, s)
                    : strcmp(mode, "trace_nold") == 0  ? launch_tc_mode<W_LAT, 10>(map, b, n_cta, s)
                                                        : launch_tc_mode<W_LAT, 2>(map, b, n_cta, s);
    static long long h[kSlots * kTrace + 7 * kMaxCta + 16];
    cudaStreamSynchronize(s);
    cudaMemcpy(h, buf, (kSlots * kTrace + 7 * kMaxCta + 16) * sizeof(long long), cudaMemcpyDeviceToHost);
    (void)nb;
    const long long* cs = h + kSlots * kTrace;
    const long long* cc = cs + 2 * kMaxCta;        // clock64 at the same two points
    long long t0 = cs[0], t1 = 0, s_max = 0;
    for (int c = 0; c < n_cta; ++c) {
      t0 = std::min(t0, cs[2 * c]);
      t1 = std::max(t1, cs[2 * c + 1]);
    }
    for (int c = 0; c < n_cta; ++c) {
      long long st = cs[2 * c] - t0, en = cs[2 * c + 1] - t0;
      s_max = std::max(s_max, st);
      if (c % 8 == 0 || c == b.trace_cta)
        fprintf(stderr, "[k3 cta] %3d start %6lld ns end %6lld ns  %lld cycles (%.0f MHz)\n", c, st, en,
                cc[2 * c + 1] - cc[2 * c], 1e3 * double(cc[2 * c + 1] - cc[2 * c]) / double(en - st));
    }
    fprintf(stderr, "[k3 cta] span %lld ns, latest start %lld ns\n", t1 - t0, s_max);
    fprintf(stderr, "[k3 ends]");                   // every CTA's end (ns), for balance analysis
    for (int c = 0; c < n_cta; ++c) fprintf(stderr, " %lld", cs[2 * c + 1] - t0);
    fprintf(stderr, "\n");
    {
      const long long* ci = h + kSlots * kTrace + 4 * kMaxCta + 16;
      fprintf(stderr, "[k3 ctainfo] cta smid tiles segs start_ns end_ns\n");
      for (int c = 0; c < n_cta; ++c)
        fprintf(stderr, "[k3 ctainfo] %d %lld %lld %lld %lld %lld\n", c, ci[3 * c], ci[3 * c + 1], ci[3 * c + 2],
                cs[2 * c] - t0, cs[2 * c + 1] - t0);
    }
    fprintf(stderr, "[k3 cta] traced CTA: start -> qk_issue[0] %lld cycles, qk_issue[0] -> end %lld cycles\n",
            h[0] - cc[2 * b.trace_cta], cc[2 * b.trace_cta + 1] - h[0]);
    {
      const long long* ev = h + kSlots * kTrace + 4 * kMaxCta;
      fprintf(stderr, "[k3 start] cycles from kernel entry: setup %lld, producer %lld, lookups %lld, tma0 %lld, "
              "q_loaded %lld, mma_q %lld, mma_kv0 %lld, qk0 %lld\n", ev[1] - ev[0], ev[2] - ev[0], ev[3] - ev[0],
              ev[4] - ev[0], ev[5] - ev[0], ev[6] - ev[0], ev[7] - ev[0], h[0] - ev[0]);
      fprintf(stderr, "[k3 start] plan loaded %lld\n", ev[11] - ev[0]);
    }
    fprintf(stderr, "[k3 trace] g qk_issue qk_issued s_ready p_done pv_issue pv_issued (cycles rel. to qk_issue[0])\n");
    for (int g = 0; g < kTrace; ++g)
      fprintf(stderr, "[k3 trace] %3d %8lld %8lld %8lld %8lld %8lld %8lld\n", g, h[g] - h[0], h[4 * kTrace + g] - h[0],
              h[2 * kTrace + g] - h[0], h[3 * kTrace + g] - h[0], h[kTrace + g] - h[0], h[5 * kTrace + g] - h[0]);
    fprintf(stderr, "[k3 tma] g tma_issue landed qk_issue (rel. to qk_issue[0])\n");
    for (int g = 0; g < kTrace; ++g)
      fprintf(stderr, "[k3 tma] %3d %8lld %8lld %8lld\n", g, h[14 * kTrace + g] - h[0], h[22 * kTrace + g] - h[0],
              h[g] - h[0]);
    fprintf(stderr, "[k3 mma] g kv_wait_start kv_wait_done qk_issue pv_wait_start(g) pv_issue(g) (rel. qk_issue[0])\n");
    for (int g = 0; g < kTrace; ++g)
      fprintf(stderr, "[k3 mma] %3d %8lld %8lld %8lld %8lld %8lld\n", g, h[19 * kTrace + g] - h[0],
              h[20 * kTrace + g] - h[0], h[g] - h[0], h[21 * kTrace + g] - h[0], h[kTrace + g] - h[0]);
    fprintf(stderr, "[k3 xchg] g x_ok sent x_full (warp 4, rel. to s_ready)\n");
    for (int g = 0; g < kTrace; ++g)
      fprintf(stderr, "[k3 xchg] %3d %6lld %6lld %6lld\n", g, h[19 * kTrace + g] - h[2 * kTrace + g],
              h[20 * kTrace + g] - h[2 * kTrace + g], h[21 * kTrace + g] - h[2 * kTrace + g]);
    fprintf(stderr, "[k3 phases] g s_ready wait_start ld_done max_done exp_done p_done (warp 4, rel. to s_ready)\n");
    for (int g = 0; g < kTrace; ++g)
      fprintf(stderr, "[k3 phases] %3d %8lld %6lld %6lld %6lld %6lld %6lld\n", g, h[2 * kTrace + g] - h[0],
              h[18 * kTrace + g] - h[2 * kTrace + g],
              h[15 * kTrace + g] - h[2 * kTrace + g], h[16 * kTrace + g] - h[2 * kTrace + g],
              h[17 * kTrace + g] - h[2 * kTrace + g], h[3 * kTrace + g] - h[2 * kTrace + g]);
    fprintf(stderr, "[k3 warps] g p_done of softmax warps 4..11 relative to warp 4\n");
    for (int g = 0; g < kTrace; ++g) {
      fprintf(stderr, "[k3 warps] %3d", g);
      for (int w = 0; w < 8; ++w) fprintf(stderr, " %6lld", h[(6 + w) * kTrace + g] - h[6 * kTrace + g]);
      fprintf(stderr, "\n");
    }
    return e;
  }
  return launch_tc_mode<W_LAT, 0>(map, a, n_cta, s);
}

}  // namespace

bool tc_attention_supported(const Geom& g, int B) {
  return g.d_r == 64 && (g.w_lat == 64 || g.w_lat == 128 || g.w_lat == 256 || g.w_lat == 512) && g.h_loc <= 128 &&
         B <= kMaxB;
}

// At least kMinBoxes 64-token boxes per CTA: with one box each (small batch x short context) a
// CTA's fixed costs dominate — its epilogue writes a 128 x W_lat fp32 partial (3x the bytes of a
// 64-token C1 tile) and the merge then reads one partial per CTA (measured at batch 1, 4K: K3
// 19 us and K45 26 us per rank with 64 one-box CTAs).  8 boxes (512 tokens) per CTA, measured over
// context 4K-64K x batch 1-8 (tools/gpu_minboxes.sh): per rank, K3 + K45 within 1 us of the 4-box floor,
// half the partials; with the two co-located ranks of the bench the K3s then share the SMs (32K
// batch 1: step 101 -> 84 us).  Large batches are unaffected (the grid is the SM count there).
constexpr long kMinBoxes = 8;
int tc_num_ctas(const Geom& g, int B, int max_seq_len) {
  long boxes = (long)B * ((max_seq_len + kSub - 1) / kSub);
  const int slots = g.w_lat == 512 ? num_sms() / 2 : num_sms();   // W_lat = 512: CTA pairs
  static const long min_boxes = getenv("TPLA_K3_MIN_BOXES") ? std::max(1L, atol(getenv("TPLA_K3_MIN_BOXES"))) : kMinBoxes;
  return int(std::max(1L, std::min<long>(std::min(slots, kMaxCta), boxes / min_boxes)));
}

size_t attn_plan_bytes(int n_cta, int B) {
  return size_t(n_cta) * (kPlanStride + 32) * 4 + size_t(2 * B + 1) * 4;
}

template <int W_LAT>
cudaError_t launch_plan_w(const PlanArgs& p, cudaStream_t s) {
  KernelScope ks("K3p_attn_plan", s);
  return launch_k(attn_plan_kernel<W_LAT>, plan_ctas(p.n_cta), kPlanThreads, 0, s, p);
}

template <int W_LAT>
cudaError_t launch_pre_w(const CUtensorMap& wmap, const CUtensorMap& qmap, const PlanArgs& p, const absorb::Args& a,
                         cudaStream_t s) {
  const size_t smem = absorb::smem_bytes(a.w_lat, a.d_h);
  static size_t attr = 0;
  if (smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(pre_attn_kernel<W_LAT>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  const int n_plan = plan_ctas(p.n_cta);
  const int n_items = a.h_loc * ((a.R + absorb::kRows - 1) / absorb::kRows);
  KernelScope ks("K3p_K2_pre_attn", s);
  return launch_k(pre_attn_kernel<W_LAT>, n_plan + n_items, kPlanThreads, smem, s, wmap, qmap, p, a, n_plan);
}

cudaError_t launch_attn_plan(const Geom& g, const tpla_cache& cache, const int32_t* seq_lens, int B, int n_cta,
                             int32_t* plan, cudaStream_t s) {
  if (B > kMaxB || n_cta > kMaxCta) return cudaErrorInvalidValue;
  PlanArgs p{seq_lens, cache.block_table, plan, B, n_cta, cache.max_pages_per_seq * cache.page_size, cache.page_size,
             cache.max_pages_per_seq};
  switch (g.w_lat) {
    case 64: return launch_plan_w<64>(p, s);
    case 128: return launch_plan_w<128>(p, s);
    case 256: return launch_plan_w<256>(p, s);
    case 512: return launch_plan_w<512>(p, s);
  }
  return cudaErrorNotSupported;
}

bool pre_attn_supported(const Geom& g) { return absorb::supported(g.w_lat, g.d_h); }

cudaError_t launch_pre_attn(const Geom& g, const tpla_cache& cache, const int32_t* seq_lens, int B, int n_cta,
                            int32_t* plan, const uint16_t* W_UK, const uint16_t* q_nope, int R, uint16_t* q_lat,
                            cudaStream_t s) {
  if (B > kMaxB || n_cta > kMaxCta || !pre_attn_supported(g)) return cudaErrorInvalidValue;
  EncodeFn enc = get_encode();
  if (!enc) return cudaErrorNotSupported;
  auto map2d = [&](CUtensorMap* m, const void* base, long cols, long rows, int box_c, int box_r) {
    cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
    cuuint64_t strides[1] = {cuuint64_t(cols) * 2};
    cuuint32_t box[2] = {cuuint32_t(box_c), cuuint32_t(box_r)};
    cuuint32_t es[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  };
  CUtensorMap wmap, qmap;
  if (!map2d(&wmap, W_UK, g.d_h, long(g.h_loc) * g.w_lat, 64, std::min(g.w_lat, 256)) ||
      !map2d(&qmap, q_nope, long(g.h_q) * g.d_h, R, 64, absorb::kRows))
    return cudaErrorInvalidValue;
  PlanArgs p{seq_lens, cache.block_table, plan, B, n_cta, cache.max_pages_per_seq * cache.page_size, cache.page_size,
             cache.max_pages_per_seq};
  absorb::Args a{q_lat, R, g.h_loc, g.w_lat, g.d_h, g.head_begin * g.d_h};
  switch (g.w_lat) {
    case 64: return launch_pre_w<64>(wmap, qmap, p, a, s);
    case 128: return launch_pre_w<128>(wmap, qmap, p, a, s);
    case 256: return launch_pre_w<256>(wmap, qmap, p, a, s);
    case 512: return launch_pre_w<512>(wmap, qmap, p, a, s);
  }
  return cudaErrorNotSupported;
}

cudaError_t launch_decode_attn_tc(const Geom& g, const tpla_cache& cache, const uint16_t* q_lat, const uint16_t* q_pe,
                                  const int32_t* seq_lens, int B, int n_q, int n_cta, const int32_t* plan,
                                  uint16_t* o_part, float* ml_part, int32_t* meta, cudaStream_t s) {
  EncodeFn enc = get_encode();
  if (!enc) return cudaErrorNotSupported;
  CUtensorMap map;
  cuuint64_t dims[2] = {cuuint64_t(cache.row_stride), cuuint64_t(cache.num_pages) * cache.page_size};
  cuuint64_t strides[1] = {cuuint64_t(cache.row_stride) * 2};
  cuuint32_t box[2] = {64, kSub};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, cache.base, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  TcArgs a;
  a.q_lat = q_lat; a.q_pe = q_pe; a.block_table = cache.block_table; a.seq_lens = seq_lens;
  a.plan = plan;
  a.o_part = o_part; a.ml_part = ml_part; a.meta = meta;
  a.B = B; a.h_loc = g.h_loc; a.h_q = g.h_q; a.head_begin = g.head_begin; a.page_size = cache.page_size;
  a.max_pages = cache.max_pages_per_seq; a.scale_log2 = g.sm_scale * 1.4426950408889634f;
  a.cap = cache.max_pages_per_seq * cache.page_size;
  a.n_q = n_q;
  a.trace = nullptr;
  a.trace_cta = 0;
  switch (g.w_lat) {
    case 64: return launch_tc<64>(map, a, n_cta, s);
    case 128: return launch_tc<128>(map, a, n_cta, s);
    case 256: return launch_tc<256>(map, a, n_cta, s);
    case 512: return launch_tc<512>(map, a, n_cta, s);
  }
  return cudaErrorNotSupported;
}

cudaError_t launch_combine_seg(const Geom& g, int B, const uint16_t* o_part, const float* ml_part, const int32_t* meta,
                               uint16_t* o_bf16, float* o_f32, float* lse, cudaStream_t s) {
  dim3 grid(g.h_loc, B);
  int threads = std::min(64, std::max(32, g.w_lat / 4));
  KernelScope ks("K4_combine", s);
  return launch_k(combine_seg_kernel, grid, threads, 0, s, o_part, ml_part, meta, g.h_loc, g.w_lat, o_bf16, o_f32,
                  lse);
}

}  // namespace tpla
