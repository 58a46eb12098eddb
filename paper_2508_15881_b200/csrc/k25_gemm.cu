// K2 / K5 — skinny "NT" GEMMs of the decode step on the tensor cores (mma.sync m16n8k16 bf16).
//
//   C[z][m][n] = Σ_k A[z][m][k] · Bw[z][n][k]      (both operands K-major)
//
//   K2  absorb_q   z = head h, m = batch b, n = latent l, k = d_h:   Q'_j[b,h,l] = Σ_d q[b,h,d] W^UK'_j[h,l,d]
//                  (absorption of W^UK into q; mu_j folded)
//   K5a W_UV       z = head h, m = b, n = d_h, k = latent:           v[b,h,e] = Σ_l O_j[b,h,l] W^UV'_j[h,e,l]
//   K5b W_O        z = K-slice, m = b, n = D, k = H_loc·d_h:         Õ_j[b,n] = Σ_k v[b,k] W^O_j[n,k]
//
// The weights (Bw) are read exactly once; M = batch is small, so every kernel here is
// weight-bandwidth bound (DESIGN.md roofline table).  Tiles: BM=32, BN=128, BK=64, 4 warps,
// 4-stage cp.async pipeline into XOR-swizzled shared memory, ldmatrix fragments.
#include "common.cuh"
#include "internal.h"

namespace tpla {
namespace {

constexpr int BM = 32, BN = 128, BK = 64, STAGES = 4, THREADS = 128;
constexpr int A_TILE = BM * BK, B_TILE = BN * BK;  // elements

struct GemmArgs {
  const uint16_t* A; long a_zs, a_ms;
  const uint16_t* Bw; long b_zs, b_ns;
  int M, N, K;
  // output: bf16 (out_bf16 != null) at out + z*o_zs + m*o_ms + n, else fp32 at out_f32 + ...
  uint16_t* out_bf16; float* out_f32; long o_zs, o_ms;
  int inputs_from_host;   // 1: A/Bw are not written by the preceding kernel (PDL wait before the stores)
  int b_blocked;          // 1: Bw is W^O's blocked layout [ceil(N/128)][k_total/64][128][64] (tpla_convert_weights)
  int b_ktiles;           // k_total / 64 of the blocked layout (z-slices start at z * K / 64)
};

__device__ __forceinline__ void nt_gemm_body(const GemmArgs& g);

// swizzled element offset of (row, chunk-of-8) in a [rows][64] bf16 tile
__device__ __forceinline__ int swz(int row, int chunk) { return row * BK + ((chunk ^ (row & 7)) << 3); }

__global__ void __launch_bounds__(THREADS) nt_gemm_kernel(GemmArgs g) {
  pdl_trigger();
  if (!g.inputs_from_host) pdl_wait();
  nt_gemm_body(g);   // (inputs_from_host: waits inside, after the math, before the first store)
}

__device__ __forceinline__ void nt_gemm_body(const GemmArgs& g) {
  extern __shared__ __align__(128) uint16_t smem[];
  uint16_t* sA = smem;
  uint16_t* sB = smem + STAGES * A_TILE;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n0 = blockIdx.x * BN, m0 = blockIdx.y * BM, z = blockIdx.z;
  const uint16_t* A = g.A + z * g.a_zs;
  const uint16_t* Bw = g.Bw + z * g.b_zs;
  const int ktiles = (g.K + BK - 1) / BK;

  auto load_stage = [&](int kt, int st) {
    const int k0 = kt * BK;
    // A: 32 rows x 8 chunks = 256 chunks, 2 per thread
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      int c = tid + i * THREADS, r = c >> 3, ch = c & 7;
      int m = m0 + r, k = k0 + ch * 8;
      bool ok = m < g.M && k < g.K;
      const uint16_t* src = ok ? A + (long)m * g.a_ms + k : A;
      cp_async16(sA + st * A_TILE + swz(r, ch), src, ok);
    }
    // B: 128 rows x 8 chunks = 1024 chunks, 8 per thread.  Blocked W^O: the [128 x 64] tile
    // (row tile blockIdx.x, k tile z*K/64 + kt) is one contiguous 16 KB block
    const uint16_t* bblk = g.b_blocked
        ? g.Bw + ((long)blockIdx.x * g.b_ktiles + (long)z * (g.K / BK) + kt) * (BN * BK) : nullptr;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      int c = tid + i * THREADS, r = c >> 3, ch = c & 7;
      int n = n0 + r, k = k0 + ch * 8;
      bool ok = n < g.N && k < g.K;
      const uint16_t* src = !ok ? g.Bw : g.b_blocked ? bblk + r * BK + ch * 8 : Bw + (long)n * g.b_ns + k;
      cp_async16(sB + st * B_TILE + swz(r, ch), src, ok);
    }
  };

  float acc[2][4][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[i][j][q] = 0.f;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) load_stage(s, s);
    cp_async_commit();
  }
  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      int nk = kt + STAGES - 1;
      if (nk < ktiles) load_stage(nk, nk % STAGES);
      cp_async_commit();
    }
    const uint16_t* a_st = sA + (kt % STAGES) * A_TILE;
    const uint16_t* b_st = sB + (kt % STAGES) * B_TILE;
#pragma unroll
    for (int kk = 0; kk < BK / 16; ++kk) {
      uint32_t af[2][4];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        int r = mi * 16 + (lane & 15), ch = kk * 2 + (lane >> 4);
        ldmatrix_x4(af[mi][0], af[mi][1], af[mi][2], af[mi][3], smem_u32(a_st + swz(r, ch)));
      }
      uint32_t bf[4][2];
#pragma unroll
      for (int nj = 0; nj < 2; ++nj) {
        int r = warp * 32 + nj * 16 + (lane & 7) + ((lane >> 4) << 3);
        int ch = kk * 2 + ((lane >> 3) & 1);
        ldmatrix_x4(bf[2 * nj][0], bf[2 * nj][1], bf[2 * nj + 1][0], bf[2 * nj + 1][1], smem_u32(b_st + swz(r, ch)));
      }
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) mma_bf16_16816(acc[mi][ni], af[mi], bf[ni]);
    }
  }
  cp_async_wait<0>();
  if (g.inputs_from_host) pdl_wait();   // the first global store of a host-input GEMM (K2)

  // epilogue
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        int m = m0 + mi * 16 + (lane >> 2) + hh * 8;
        int n = n0 + warp * 32 + ni * 8 + (lane & 3) * 2;
        if (m >= g.M || n >= g.N) continue;
        float v0 = acc[mi][ni][2 * hh], v1 = acc[mi][ni][2 * hh + 1];
        long off = z * g.o_zs + (long)m * g.o_ms + n;
        if (g.out_bf16) {
          if (n + 1 < g.N) *reinterpret_cast<uint32_t*>(g.out_bf16 + off) = pack_bf16(v0, v1);
          else g.out_bf16[off] = f2bf(v0);
        } else {
          if (n + 1 < g.N) *reinterpret_cast<float2*>(g.out_f32 + off) = make_float2(v0, v1);
          else g.out_f32[off] = v0;
        }
      }
}

cudaError_t launch_nt(const GemmArgs& a, int Z, const char* name, cudaStream_t s) {
  static bool attr = false;
  const int smem = STAGES * (A_TILE + B_TILE) * 2;
  if (!attr) {
    cudaFuncSetAttribute(nt_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  dim3 grid((a.N + BN - 1) / BN, (a.M + BM - 1) / BM, Z);
  KernelScope ks(name, s);
  return launch_k(nt_gemm_kernel, grid, THREADS, smem, s, a);
}

__global__ void reduce_slices_kernel(const float* __restrict__ y_part, int kslices, long n, float* __restrict__ y,
                                     int accumulate) {
  pdl_trigger();
  pdl_wait();
  long i = (blockIdx.x * (long)blockDim.x + threadIdx.x) * 4;
  if (i >= n) return;
  float4 acc = accumulate ? *reinterpret_cast<const float4*>(y + i) : make_float4(0.f, 0.f, 0.f, 0.f);
  for (int s = 0; s < kslices; ++s) {      // fixed slice order: deterministic
    float4 v = *reinterpret_cast<const float4*>(y_part + s * n + i);
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
  }
  *reinterpret_cast<float4*>(y + i) = acc;
}

__global__ void cast_kernel(const float* __restrict__ y, long n, uint16_t* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  long i = (blockIdx.x * (long)blockDim.x + threadIdx.x) * 4;
  if (i >= n) return;
  float4 v = *reinterpret_cast<const float4*>(y + i);
  uint2 o;
  o.x = pack_bf16(v.x, v.y);
  o.y = pack_bf16(v.z, v.w);
  *reinterpret_cast<uint2*>(out + i) = o;
}

struct SumSrc {
  const float* p[kMaxSumSrc];
};

__global__ void sum_cast_kernel(SumSrc src, int n_src, long n, uint16_t* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  long i = (blockIdx.x * (long)blockDim.x + threadIdx.x) * 4;
  if (i >= n) return;
  float4 v = *reinterpret_cast<const float4*>(src.p[0] + i);
  for (int k = 1; k < n_src; ++k) {          // fixed order: deterministic
    const float4 u = *reinterpret_cast<const float4*>(src.p[k] + i);
    v.x += u.x; v.y += u.y; v.z += u.z; v.w += u.w;
  }
  uint2 o;
  o.x = pack_bf16(v.x, v.y);
  o.y = pack_bf16(v.z, v.w);
  *reinterpret_cast<uint2*>(out + i) = o;
}

}  // namespace

cudaError_t launch_sum_cast_bf16(const float* const* src, int n_src, long n, uint16_t* out, cudaStream_t s,
                                 const char* name) {
  if (n_src < 1 || n_src > kMaxSumSrc) return cudaErrorInvalidValue;
  SumSrc a{};
  for (int k = 0; k < n_src; ++k) a.p[k] = src[k];
  int blocks = (int)((n / 4 + 255) / 256);
  KernelScope ks(name, s);
  return launch_k(sum_cast_kernel, blocks, 256, 0, s, a, n_src, n, out);
}

cudaError_t launch_head_gemv(const char* name, const uint16_t* W, const uint16_t* x, long x_batch_stride, int H,
                             int R, int C, int B, uint16_t* out_bf16, bool inputs_from_host, cudaStream_t s) {
  GemmArgs a{};
  a.inputs_from_host = inputs_from_host ? 1 : 0;
  a.A = x; a.a_zs = C; a.a_ms = x_batch_stride;
  a.Bw = W; a.b_zs = (long)R * C; a.b_ns = C;
  a.M = B; a.N = R; a.K = C;
  a.out_bf16 = out_bf16; a.out_f32 = nullptr; a.o_zs = R; a.o_ms = (long)H * R;
  return launch_nt(a, H, name, s);
}

cudaError_t launch_skinny_gemm(const uint16_t* Wt, const uint16_t* v, int N, int K, int B, int kslices, float* y_part,
                               cudaStream_t s) {
  GemmArgs a{};
  const int Kc = K / kslices;
  if (wo_blocked(K)) {                  // (the K-slices are 64-multiples: ws_layout)
    if (Kc % BK) return cudaErrorInvalidValue;
    a.b_blocked = 1;
    a.b_ktiles = K / BK;
  }
  a.A = v; a.a_zs = Kc; a.a_ms = K;
  a.Bw = Wt; a.b_zs = Kc; a.b_ns = K;
  a.M = B; a.N = N; a.K = Kc;
  a.out_bf16 = nullptr; a.out_f32 = y_part; a.o_zs = (long)B * N; a.o_ms = N;
  return launch_nt(a, kslices, "K5_W_O", s);
}

cudaError_t launch_reduce_slices(const float* y_part, int kslices, int B, int N, float* y, bool accumulate,
                                 cudaStream_t s) {
  long n = (long)B * N;  // N % 8 == 0 (validated) so n % 4 == 0
  int blocks = (int)((n / 4 + 255) / 256);
  KernelScope ks("K5_reduce", s);
  return launch_k(reduce_slices_kernel, blocks, 256, 0, s, y_part, kslices, n, y, accumulate ? 1 : 0);
}

cudaError_t launch_cast_bf16(const float* y, long n, uint16_t* out, cudaStream_t s, const char* name) {
  int blocks = (int)((n / 4 + 255) / 256);
  KernelScope ks(name, s);
  return launch_k(cast_kernel, blocks, 256, 0, s, y, n, out);
}

}  // namespace tpla
