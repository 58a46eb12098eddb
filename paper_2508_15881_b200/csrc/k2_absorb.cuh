// K2 — query absorption for one (head, 32-row tile), the device body of the fused pre-attention
// kernel (K3p + K2, k3_attn_tc.cu):
//   Q'_j[m, h, :] = W^UK'_j[h] · q[m, h, :]       (absorption; mu_j folded into W^UK')
// q: [R, h_q * d_h] bf16 rows (all heads; this rank's head h at column (head_begin + h) * d_h);
// W^UK'_j: [H_loc, W_lat, d_h] bf16; Q'_j: [R, H_loc, W_lat] bf16.
// Both operands land in shared memory by TMA on one mbarrier — the head's W_lat x d_h weight slice
// as 128B-swizzled boxes of 64 columns x min(W_lat, 256) rows, the 32 query rows as boxes of
// 64 columns (rows past R zero-filled by the TMA) — then mma.sync m16n8k16 over the d_h contraction:
// ~2 MFLOP per head, so the kernel is bound by the 64 KB slice load, not by the tensor pipe.  The
// result is staged in shared memory and leaves in 16 B row vectors after the PDL wait (the previous
// step's K3 reads Q'_j: write-after-read).
#pragma once

namespace absorb {

constexpr int kRows = 32;                       // query rows per CTA

struct Args {
  uint16_t* q_lat;                              // [R, H_loc, W_lat]
  int R, h_loc, w_lat, d_h;
  int q_col0;                                   // q column of this rank's head 0 (head_begin * d_h)
};

inline size_t smem_bytes(int w_lat, int d_h) {
  return size_t(w_lat) * d_h * 2 + size_t(kRows) * d_h * 2 + size_t(kRows) * (w_lat + 8) * 2 + 1024;
}
inline bool supported(int w_lat, int d_h) {
  return d_h % 64 == 0 && w_lat % 8 == 0 && (w_lat <= 256 || w_lat % 256 == 0) && smem_bytes(w_lat, d_h) <= 200 * 1024;
}

// 128B swizzle of a [rows][64] bf16 box: 16 B chunk ch of row r
__device__ __forceinline__ int swz(int r, int ch) { return r * 64 + ((ch ^ (r & 7)) << 3); }

// item: the (head, row tile) this CTA computes; smem_raw: smem_bytes() of dynamic shared memory
__device__ __forceinline__ void body(const CUtensorMap* wmap, const CUtensorMap* qmap, const Args& a, int item,
                                     uint8_t* smem_raw, uint64_t* bar) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, n_warps = blockDim.x >> 5;
  const int h = item % a.h_loc, m0 = (item / a.h_loc) * kRows;
  const int n_cb = a.d_h / 64, wr = a.w_lat < 256 ? a.w_lat : 256;
  uint16_t* sW = reinterpret_cast<uint16_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint16_t* sQ = sW + a.w_lat * a.d_h;          // [n_cb][kRows][64]   (boxes stay 1024-aligned: 4 KB each)
  uint16_t* sO = sQ + kRows * a.d_h;            // [kRows][W_lat + 8]  (padded rows: conflict-free stores)
  const int OP = a.w_lat + 8;
  if (tid == 0) {
    sm100::mbar_init(bar, 1);
    sm100::fence_barrier_init();
  }
  __syncthreads();
  if (tid == 0) {
    sm100::mbar_arrive_expect_tx(bar, uint32_t(a.w_lat + kRows) * a.d_h * 2);
    for (int rb = 0; rb < a.w_lat / wr; ++rb)
      for (int cb = 0; cb < n_cb; ++cb)
        sm100::tma_load_2d(sW + (rb * n_cb + cb) * wr * 64, wmap, cb * 64, h * a.w_lat + rb * wr, bar,
                           sm100::kEvictNormal);
    for (int cb = 0; cb < n_cb; ++cb)
      sm100::tma_load_2d(sQ + cb * kRows * 64, qmap, a.q_col0 + h * a.d_h + cb * 64, m0, bar, sm100::kEvictFirst);
  }
  sm100::mbar_wait(bar, 0);

  // warp w: the n8 tiles w, w + n_warps, ... (latent columns), both m16 halves, full d_h
  for (int nt = warp; nt < a.w_lat / 8; nt += n_warps) {
    float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    const int n = nt * 8 + (lane & 7), rb = n / wr, rr = n % wr;
    for (int k0 = 0; k0 < a.d_h; k0 += 16) {
      const int cb = k0 >> 6, ch = (k0 & 63) >> 3;
      uint32_t bf[2];
      ldmatrix_x2(bf[0], bf[1], smem_u32(sW + (rb * n_cb + cb) * wr * 64 + swz(rr, ch + ((lane >> 3) & 1))));
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        uint32_t af[4];
        ldmatrix_x4(af[0], af[1], af[2], af[3],
                    smem_u32(sQ + cb * kRows * 64 + swz(mi * 16 + (lane & 15), ch + (lane >> 4))));
        mma_bf16_16816(acc[mi], af, bf);
      }
    }
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh)
        *reinterpret_cast<uint32_t*>(sO + (mi * 16 + (lane >> 2) + hh * 8) * OP + nt * 8 + (lane & 3) * 2) =
            pack_bf16(acc[mi][2 * hh], acc[mi][2 * hh + 1]);
  }
  __syncthreads();
  pdl_wait();                                   // first global store (write-after-read on Q'_j)
  const int vpr = a.w_lat / 8;                  // 16 B vectors per row
  for (int i = tid; i < kRows * vpr; i += blockDim.x) {
    const int r = i / vpr, c = (i % vpr) * 8;
    if (m0 + r < a.R)
      *reinterpret_cast<uint4*>(a.q_lat + ((long)(m0 + r) * a.h_loc + h) * a.w_lat + c) =
          *reinterpret_cast<const uint4*>(sO + r * OP + c);
  }
}

}  // namespace absorb
