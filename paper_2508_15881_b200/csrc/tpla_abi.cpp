// C-ABI entry points of libtpla.so (include/tpla.h): validation, host-side conversion,
// workspace carving, kernel sequencing and the NCCL communicator.
//
// Citations "P:n" refer to lines of the paper text.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <string>
#include <thread>
#include <vector>

#include "internal.h"
#include "nccl.h"
#include "nccl_device.h"

namespace tpla {
std::atomic<int64_t> g_launches{0};
}

using namespace tpla;

namespace {

thread_local std::string t_err;

tpla_status fail(tpla_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  t_err = buf;
  return st;
}

tpla_status ok() {
  t_err.clear();
  return TPLA_OK;
}

tpla_status cuda_fail(cudaError_t e, const char* where) {
  return fail(TPLA_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

#define TPLA_CUDA(call, where)                    \
  do {                                            \
    cudaError_t e_ = (call);                      \
    if (e_ != cudaSuccess) return cuda_fail(e_, where); \
  } while (0)

bool is_pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Validate cfg and resolve this device's geometry.
tpla_status make_geom(const tpla_config* c, Geom* g) {
  if (!c || !g) return fail(TPLA_ERR_INVALID_ARG, "NULL config");
  if (c->h_q < 1 || c->d_c < 1 || c->d_r < 0 || c->d_h < 1 || c->D < 1 || c->k < 1 || c->g < 1)
    return fail(TPLA_ERR_SHAPE, "non-positive dimension");
  if (c->k % c->g) return fail(TPLA_ERR_DIVISIBILITY, "g=%d must divide k=%d", c->g, c->k);
  if (c->d_c % c->g) return fail(TPLA_ERR_DIVISIBILITY, "g=%d must divide d_c=%d", c->g, c->d_c);
  int per_group = c->k / c->g;
  if (c->h_q % per_group) return fail(TPLA_ERR_DIVISIBILITY, "k/g=%d must divide h_q=%d", per_group, c->h_q);
  if (c->rank < 0 || c->rank >= c->k) return fail(TPLA_ERR_INVALID_ARG, "rank %d outside [0,%d)", c->rank, c->k);
  if (c->d_r % 2) return fail(TPLA_ERR_SHAPE, "d_r must be even");
  if (!(c->eps >= 0.f) || !(c->sm_scale > 0.f)) return fail(TPLA_ERR_INVALID_ARG, "eps/sm_scale out of range");
  g->h_q = c->h_q; g->d_c = c->d_c; g->d_r = c->d_r; g->d_h = c->d_h; g->D = c->D;
  g->k = c->k; g->g = c->g; g->rank = c->rank;
  int j = c->rank / per_group, i = c->rank % per_group;
  g->h_loc = c->h_q / per_group;
  g->w_lat = c->d_c / c->g;
  g->W = g->w_lat + c->d_r;
  g->head_begin = i * g->h_loc;
  g->lat_begin = j * g->w_lat;
  g->eps = c->eps;
  g->sm_scale = c->sm_scale;
  return TPLA_OK;
}

// Kernel-side limits of this build (checked before any launch).
tpla_status check_kernel_shapes(const Geom& g) {
  if (!is_pow2(g.d_c) || g.d_c < 32 || g.d_c > 1024)
    return fail(TPLA_ERR_SHAPE, "d_c=%d: kernels need a power of two in [32, 1024]", g.d_c);
  // W_lat = 512 (g = 1, plain MLA) runs on the tcgen05 kernel's CTA-pair path only (d_r = 64)
  if (g.w_lat % 32 || (g.w_lat > 256 && !(g.w_lat == 512 && g.d_r == 64)))
    return fail(TPLA_ERR_UNSUPPORTED, "W_lat=%d: decode kernels support multiples of 32 up to 256, and 512 with d_r=64",
                g.w_lat);
  if (!(g.d_r == 16 || g.d_r == 64)) return fail(TPLA_ERR_UNSUPPORTED, "d_r=%d: decode kernels support 16 or 64", g.d_r);
  if (g.h_loc > 128) return fail(TPLA_ERR_UNSUPPORTED, "H_loc=%d > 128", g.h_loc);
  if (g.d_h % 16 || g.d_h > 256) return fail(TPLA_ERR_UNSUPPORTED, "d_h=%d: multiple of 16 up to 256", g.d_h);
  if ((g.h_loc * g.d_h) % 8) return fail(TPLA_ERR_UNSUPPORTED, "H_loc*d_h must be a multiple of 8");
  if (g.D % 8) return fail(TPLA_ERR_UNSUPPORTED, "D must be a multiple of 8");
  return TPLA_OK;
}

tpla_status check_cache(const Geom& g, const tpla_cache* c) {
  if (!c || !c->base || !c->block_table) return fail(TPLA_ERR_INVALID_ARG, "NULL cache");
  if (!aligned16(c->base)) return fail(TPLA_ERR_INVALID_ARG, "cache base not 16-byte aligned");
  if (c->page_size < 64 || c->page_size % 64) return fail(TPLA_ERR_SHAPE, "page_size must be a positive multiple of 64");
  if (c->row_stride < g.W || c->row_stride % 64) return fail(TPLA_ERR_SHAPE, "row_stride=%d must be a multiple of 64 >= W=%d", c->row_stride, g.W);
  if (c->num_pages < 1 || c->max_pages_per_seq < 1 || c->batch < 1) return fail(TPLA_ERR_SHAPE, "empty cache");
  return TPLA_OK;
}

uint64_t splitmix64_next(uint64_t& state) {
  state += 0x9E3779B97F4A7C15ull;
  uint64_t z = state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

double bf16_to_double(uint16_t b) {
  uint32_t u = static_cast<uint32_t>(b) << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

uint16_t double_to_bf16(double x) {
  // nearest bf16 (8 significant bits), ties to even, taken directly on the fp64 value
  if (x == 0.0) return signbit(x) ? 0x8000u : 0u;
  int e;
  double m = frexp(x, &e);                 // x = m 2^e, 0.5 <= |m| < 1
  double r = nearbyint(m * 256.0);         // FE_TONEAREST: ties to even
  float f = static_cast<float>(ldexp(r / 256.0, e));
  uint32_t u;
  memcpy(&u, &f, 4);
  return static_cast<uint16_t>(u >> 16);
}

template <class F>
void parallel_for(int n, F f) {
  int nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  nt = std::min(nt, n);
  if (nt <= 1) { for (int i = 0; i < n; ++i) f(i); return; }
  std::vector<std::thread> th;
  std::atomic<int> next{0};
  for (int t = 0; t < nt; ++t)
    th.emplace_back([&] { for (int i; (i = next.fetch_add(1)) < n;) f(i); });
  for (auto& x : th) x.join();
}

// ---- NCCL, loaded at run time (the library must load without it) ----
struct NcclApi {
  bool tried = false, ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  // device API (NCCL >= 2.28; optional: the fused all-reduce of SURVEY f2(i))
  ncclResult_t (*GetVersion)(int*) = nullptr;
  ncclResult_t (*MemAlloc)(void**, size_t) = nullptr;
  ncclResult_t (*MemFree)(void*) = nullptr;
  ncclResult_t (*WinRegister)(ncclComm_t, void*, size_t, ncclWindow_t*, int) = nullptr;
  ncclResult_t (*WinDeregister)(ncclComm_t, ncclWindow_t) = nullptr;
  ncclResult_t (*DevCommCreate)(ncclComm_t, ncclDevCommRequirements_t const*, ncclDevComm_t*) = nullptr;
  ncclResult_t (*DevCommDestroy)(ncclComm_t, ncclDevComm_t const*) = nullptr;
  bool device_api = false;
};
NcclApi g_nccl;

bool load_nccl() {
  if (g_nccl.tried) return g_nccl.ok;
  g_nccl.tried = true;
  const char* env = getenv("TPLA_NCCL_LIB");
  const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
  void* h = nullptr;
  for (const char* n : names) {
    if (!n) continue;
    h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
    if (h) break;
  }
  if (!h) return false;
  g_nccl.GetUniqueId = (decltype(g_nccl.GetUniqueId))dlsym(h, "ncclGetUniqueId");
  g_nccl.CommInitRank = (decltype(g_nccl.CommInitRank))dlsym(h, "ncclCommInitRank");
  g_nccl.AllReduce = (decltype(g_nccl.AllReduce))dlsym(h, "ncclAllReduce");
  g_nccl.ReduceScatter = (decltype(g_nccl.ReduceScatter))dlsym(h, "ncclReduceScatter");
  g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))dlsym(h, "ncclCommDestroy");
  g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))dlsym(h, "ncclGetErrorString");
  g_nccl.GetVersion = (decltype(g_nccl.GetVersion))dlsym(h, "ncclGetVersion");
  g_nccl.MemAlloc = (decltype(g_nccl.MemAlloc))dlsym(h, "ncclMemAlloc");
  g_nccl.MemFree = (decltype(g_nccl.MemFree))dlsym(h, "ncclMemFree");
  g_nccl.WinRegister = (decltype(g_nccl.WinRegister))dlsym(h, "ncclCommWindowRegister");
  g_nccl.WinDeregister = (decltype(g_nccl.WinDeregister))dlsym(h, "ncclCommWindowDeregister");
  g_nccl.DevCommCreate = (decltype(g_nccl.DevCommCreate))dlsym(h, "ncclDevCommCreate");
  g_nccl.DevCommDestroy = (decltype(g_nccl.DevCommDestroy))dlsym(h, "ncclDevCommDestroy");
  int ver = 0;
  // the device communicator's layout is the one of the headers this library was compiled with
  g_nccl.device_api = g_nccl.GetVersion && g_nccl.GetVersion(&ver) == ncclSuccess && ver >= 22800 &&
                      ver / 100 == NCCL_VERSION_CODE / 100 && g_nccl.MemAlloc && g_nccl.MemFree &&
                      g_nccl.WinRegister && g_nccl.WinDeregister && g_nccl.DevCommCreate && g_nccl.DevCommDestroy;
  g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.AllReduce && g_nccl.ReduceScatter &&
             g_nccl.CommDestroy && g_nccl.GetErrorString;
  return g_nccl.ok;
}

}  // namespace

struct tpla_comm {
  ncclComm_t comm;
  int world, rank;
  // fused W^O epilogue + one-shot all-reduce (tpla_comm_enable_fused_allreduce)
  void* sym = nullptr;                 // ncclMemAlloc'd symmetric buffer (2 halves)
  ncclWindow_t win = nullptr;
  ncclDevComm dev{};
  bool dev_ok = false;
  tpla::FusedAr ar{};
};

namespace {
// the fused path for a call of R rows of D outputs (or null: the plain ncclAllReduce follows)
const tpla::FusedAr* fused_ar(const tpla_comm* c, long R, int D) {
  if (!c || !c->ar.window) return nullptr;
  static const char* env = getenv("TPLA_FUSED_AR");
  if (env && env[0] == '0') return nullptr;
  return size_t(R) * D <= c->ar.half_elems ? &c->ar : nullptr;
}
}  // namespace

namespace tpla {

SplitPlan choose_split(int B, int max_seq_len) {
  // Fixed split of every sequence into n_split chunks of 64-token multiples, sized from the
  // capacity bound (not the live lengths) so the launch shape is graph-capturable:
  // B * n_split ≈ 2 waves of 148 SMs.
  const int kSMs = 148;
  int tiles = (max_seq_len + 63) / 64;
  int want = std::max(1, (2 * kSMs + B - 1) / B);
  int n_split = std::max(1, std::min(tiles, want));
  int chunk = ((tiles + n_split - 1) / n_split) * 64;
  n_split = (max_seq_len + chunk - 1) / chunk;
  return SplitPlan{n_split, chunk};
}

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
constexpr size_t kWsHeader = 64 << 10;   // decode workspace: [K3p plan | segment map] header, then Q'_j ...

// The tcgen05 W^O GEMM takes at most kWoRows output rows per launch (the MMA N of its swap-AB
// tile): larger batches run as consecutive row chunks sharing the partial workspace (each
// chunk's GEMM waits for the previous chunk's reduce before writing it: PDL wait at entry).
constexpr int kWoRows = 256;
// K3p (when the persistent K3 follows) and K2 ahead of the attention: one fused launch where the
// shapes allow (TPLA_PRE_SPLIT=1: the two separate kernels, for A/B), else K3p then the mma.sync K2.
static cudaError_t launch_pre(const Geom& g, const tpla_cache& cache, const int32_t* seq_lens, int B, int n_cta,
                              int32_t* plan, bool with_plan, const uint16_t* W_UK, const uint16_t* qn, int R,
                              uint16_t* q_lat, cudaStream_t s) {
  static const bool split = getenv("TPLA_PRE_SPLIT") && atoi(getenv("TPLA_PRE_SPLIT")) != 0;
  if (with_plan && !split && pre_attn_supported(g))
    return launch_pre_attn(g, cache, seq_lens, B, n_cta, plan, W_UK, qn, R, q_lat, s);
  cudaError_t e = cudaSuccess;
  if (with_plan && (e = launch_attn_plan(g, cache, seq_lens, B, n_cta, plan, s)) != cudaSuccess) return e;
  return launch_head_gemv("K2_absorb_q", W_UK, qn + size_t(g.head_begin) * g.d_h, long(g.h_q) * g.d_h, g.h_loc,
                          g.w_lat, g.d_h, R, q_lat, true, s);
}

static cudaError_t run_wo_tc(const uint16_t* Wo, const uint16_t* v, int D, int K, int R, void* part, float* y,
                             bool accumulate, uint16_t* out16, cudaStream_t s, int k_begin = 0, int k_len = 0,
                             const FusedAr* ar = nullptr) {
  const int kl = k_len > 0 ? k_len : K;             // v's row length (the K-slice's columns)
  for (int r0 = 0; r0 < R; r0 += kWoRows) {
    const int n = std::min(kWoRows, R - r0);
    cudaError_t e = launch_wo_tc(Wo, v + size_t(r0) * kl, D, K, n, part, y + size_t(r0) * D, accumulate,
                                 out16 ? out16 + size_t(r0) * D : nullptr, s, k_begin, k_len, 0, ar, r0);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

WsLayout ws_layout(const Geom& g, int B, int n_q, int max_seq_len) {
  WsLayout L{};
  const int R = B * n_q;                                 // output rows (sequence, query token)
  SplitPlan sp = choose_split(B, max_seq_len);
  int K = g.h_loc * g.d_h;
  // split K = H_loc*d_h of the W^O GEMM into equal 64-multiples (at most 16) to fill the SMs
  L.kslices = std::max(1, std::min(K / 64, 16));
  while (L.kslices > 1 && (K / 64) % L.kslices) --L.kslices;
  if (K % (64 * L.kslices)) L.kslices = 1;
  // partial (O, m, l) slots: B*n_split for the fixed split (mma.sync K3), n_cta + B segments
  // for the persistent tcgen05 K3 (each CTA range touches at most one more sequence than it starts in)
  L.n_cta = tc_num_ctas(g, B, max_seq_len);
  const size_t parts = std::max(size_t(B) * sp.n_split, size_t(L.n_cta) + B);
  const size_t rows = size_t(n_q) * g.h_loc;            // partial rows per segment / split
  // the K3p plan and the segment map lead the workspace, in the same 2 MB page as Q'_j (the first
  // global loads of every K3 CTA: plan, then Q'; one TLB walk instead of two)
  L.plan = 0;
  L.meta = align256(attn_plan_bytes(L.n_cta, B));
  size_t off = std::max(kWsHeader, L.meta + align256(size_t(B) * 2 * 4));
  L.q_lat = off;   off += align256(size_t(R) * g.h_loc * g.w_lat * 2);
  L.o_part = off;  off += align256(parts * rows * g.w_lat * 4);
  L.ml_part = off; off += align256(parts * rows * 2 * 4);
  L.o_lat = off;   off += align256(size_t(R) * g.h_loc * g.w_lat * 2);
  L.v = off;       off += align256(size_t(R) * K * 2);
  L.y_part = off;  off += align256(size_t(L.kslices) * R * g.D * 4);

  L.wo_part = off; off += align256(wo_tc_supported(g.D, K, std::min(R, kWoRows)) ? wo_tc_part_bytes(g.D, K, std::min(R, kWoRows)) : 0);
  L.total = off;
  return L;
}

// K3 + K4: the tcgen05 kernel where its shapes allow (TPLA_ATTN=mma forces the legacy path)
static bool use_tc_attention(const Geom& g, int B) {
  const char* force = getenv("TPLA_ATTN");
  return tc_attention_supported(g, B) && !(force && strcmp(force, "mma") == 0);
}

static cudaError_t run_attention(const Geom& g, const tpla_cache& cache, const uint16_t* q_lat, const uint16_t* q_pe,
                                 const int32_t* seq_lens, int B, int max_seq_len, const WsLayout& L, char* base,
                                 uint16_t* o_bf16, float* o_f32, float* lse, cudaStream_t s, bool reuse_plan = false) {
  auto* o_part = reinterpret_cast<float*>(base + L.o_part);
  auto* ml_part = reinterpret_cast<float*>(base + L.ml_part);
  cudaError_t e;
  if (use_tc_attention(g, B)) {
    auto* o16 = reinterpret_cast<uint16_t*>(base + L.o_part);       // (fp16 partials)
    auto* meta = reinterpret_cast<int32_t*>(base + L.meta);
    auto* plan = reinterpret_cast<int32_t*>(base + L.plan);
    if (!reuse_plan && (e = launch_attn_plan(g, cache, seq_lens, B, L.n_cta, plan, s)) != cudaSuccess) return e;
    e = launch_decode_attn_tc(g, cache, q_lat, q_pe, seq_lens, B, 1, L.n_cta, plan, o16, ml_part, meta, s);
    if (e != cudaSuccess || (!o_bf16 && !o_f32 && !lse)) return e;   // no output requested: K3 alone
    return launch_combine_seg(g, B, o16, ml_part, meta, o_bf16, o_f32, lse, s);
  }
  SplitPlan sp = choose_split(B, max_seq_len);
  e = launch_decode_attn(g, cache, q_lat, q_pe, seq_lens, B, sp, o_part, ml_part, s);
  if (e != cudaSuccess || (!o_bf16 && !o_f32 && !lse)) return e;   // no output requested: K3 alone
  return launch_combine(g, B, sp, o_part, ml_part, o_bf16, o_f32, lse, s);
}

}  // namespace tpla

// =====================================================================================
extern "C" {

#ifndef TPLA_SRC_HASH
#define TPLA_SRC_HASH "unknown"
#endif
const char* tpla_version(void) { return "tpla-b200 0.2 (sm_100a) src " TPLA_SRC_HASH; }
const char* tpla_last_error(void) { return t_err.c_str(); }
int64_t tpla_launch_count(void) { return g_launches.load(); }

tpla_status tpla_make_plan(const tpla_config* cfg, tpla_device_plan* out) {
  Geom g{};
  tpla_status st = make_geom(cfg, &g);
  if (st) return st;
  if (!out) return fail(TPLA_ERR_INVALID_ARG, "NULL plan");
  out->rank = g.rank;
  out->shard = g.lat_begin / g.w_lat;
  out->head_block = g.head_begin / g.h_loc;
  out->head_begin = g.head_begin;
  out->head_end = g.head_begin + g.h_loc;
  out->lat_begin = g.lat_begin;
  out->lat_end = g.lat_begin + g.w_lat;
  out->row_width = g.W;
  out->h_loc = g.h_loc;
  out->w_lat = g.w_lat;
  return ok();
}

tpla_status tpla_hadamard_signs(uint64_t seed, int32_t d, float* out) {
  if (!out || d < 1) return fail(TPLA_ERR_INVALID_ARG, "bad arguments");
  uint64_t state = seed;
  for (int i = 0; i < d; ++i) out[i] = (splitmix64_next(state) >> 63) ? -1.f : 1.f;
  return ok();
}

tpla_status tpla_pca_alpha(const double* lambda, int32_t d_c, int32_t g, float* alpha_out) {
  if (!lambda || !alpha_out || d_c < 1 || g < 1) return fail(TPLA_ERR_INVALID_ARG, "bad arguments");
  if (d_c % g) return fail(TPLA_ERR_DIVISIBILITY, "g must divide d_c");
  double total = 0;
  for (int i = 0; i < d_c; ++i) total += lambda[i];
  int w = d_c / g;
  for (int j = 0; j < g; ++j) {
    double s = 0;
    for (int i = j * w; i < (j + 1) * w; ++i) s += lambda[i];
    if (!(s > 0)) return fail(TPLA_ERR_INVALID_ARG, "slice %d has no energy", j);
    alpha_out[j] = static_cast<float>(total / s);
  }
  return ok();
}

tpla_status tpla_weights_bytes(const tpla_config* cfg, int32_t xform_kind, size_t* W_UK, size_t* W_UV,
                               size_t* W_O, size_t* xform) {
  Geom g{};
  tpla_status st = make_geom(cfg, &g);
  if (st) return st;
  if (W_UK) *W_UK = size_t(g.h_loc) * g.w_lat * g.d_h * 2;
  if (W_UV) *W_UV = size_t(g.h_loc) * g.d_h * g.w_lat * 2;
  if (W_O) {
    const int K = g.h_loc * g.d_h;
    *W_O = (wo_blocked(K) ? size_t((g.D + 127) / 128) * 128 : size_t(g.D)) * K * 2;
  }
  if (xform) {
    if (xform_kind == TPLA_XFORM_HADAMARD) *xform = size_t(g.d_c) * 4;
    else if (xform_kind == TPLA_XFORM_PCA) *xform = size_t(g.d_c) * g.w_lat * 4;
    else if (xform_kind == TPLA_XFORM_IDENTITY) *xform = 0;
    else return fail(TPLA_ERR_INVALID_ARG, "bad xform_kind");
  }
  return ok();
}

tpla_status tpla_convert_weights(const tpla_config* cfg, int32_t xform_kind, uint64_t sign_seed,
                                 const float* U_pca, const float* alpha, const float* mu,
                                 const uint16_t* W_UK, const uint16_t* W_UV, const uint16_t* gamma,
                                 const uint16_t* W_O, tpla_weights* out, void* stream) {
  Geom g{};
  tpla_status st = make_geom(cfg, &g);
  if (st) return st;
  if (!alpha || !mu || !W_UK || !W_UV || !gamma || !W_O || !out || !out->W_UK || !out->W_UV || !out->W_O)
    return fail(TPLA_ERR_INVALID_ARG, "NULL argument");
  if (xform_kind == TPLA_XFORM_HADAMARD && !is_pow2(g.d_c))
    return fail(TPLA_ERR_DIVISIBILITY, "Hadamard needs d_c a power of two (P:274)");
  if (xform_kind == TPLA_XFORM_PCA && !U_pca) return fail(TPLA_ERR_INVALID_ARG, "PCA needs U_pca");
  if (xform_kind < 0 || xform_kind > 2) return fail(TPLA_ERR_INVALID_ARG, "bad xform_kind");
  if (xform_kind != TPLA_XFORM_IDENTITY && !out->xform) return fail(TPLA_ERR_INVALID_ARG, "NULL xform buffer");
  const int d_c = g.d_c, d_h = g.d_h, hq = g.h_q, H = g.h_loc, WL = g.w_lat, D = g.D;
  const int shard = g.lat_begin / WL;
  const double mu_j = mu[shard];
  cudaStream_t s = static_cast<cudaStream_t>(stream);

  std::vector<double> signs(d_c, 1.0);
  if (xform_kind == TPLA_XFORM_HADAMARD) {
    uint64_t state = sign_seed;
    for (int i = 0; i < d_c; ++i) signs[i] = (splitmix64_next(state) >> 63) ? -1.0 : 1.0;
  }
  // W^UKV_new = U^T W_γ W^UKV, only for the device's latent rows and head columns.
  // U^T (x) for Hadamard: U = D H / sqrt(d) so U^T x = H (D x) / sqrt(d) (H symmetric).
  std::vector<uint16_t> uk(size_t(H) * WL * d_h), uv(size_t(H) * d_h * WL);
  const double inv_sqrt_d = 1.0 / sqrt(double(d_c));
  parallel_for(H * d_h, [&](int col_local) {
    const int h = col_local / d_h, e = col_local % d_h;
    const size_t col = size_t(g.head_begin + h) * d_h + e;
    std::vector<double> a(d_c), b(d_c), ta(WL), tb(WL);
    for (int r = 0; r < d_c; ++r) {
      double gm = bf16_to_double(gamma[r]);
      a[r] = gm * bf16_to_double(W_UK[size_t(r) * hq * d_h + col]);
      b[r] = gm * bf16_to_double(W_UV[size_t(r) * hq * d_h + col]);
    }
    if (xform_kind == TPLA_XFORM_HADAMARD) {
      for (int r = 0; r < d_c; ++r) { a[r] *= signs[r]; b[r] *= signs[r]; }
      for (int len = 1; len < d_c; len <<= 1)
        for (int i = 0; i < d_c; i += 2 * len)
          for (int q = i; q < i + len; ++q) {
            double x = a[q], y = a[q + len];
            a[q] = x + y; a[q + len] = x - y;
            x = b[q]; y = b[q + len];
            b[q] = x + y; b[q + len] = x - y;
          }
      for (int l = 0; l < WL; ++l) { ta[l] = a[g.lat_begin + l] * inv_sqrt_d; tb[l] = b[g.lat_begin + l] * inv_sqrt_d; }
    } else if (xform_kind == TPLA_XFORM_PCA) {
      for (int l = 0; l < WL; ++l) {
        double sa = 0, sb = 0;
        for (int r = 0; r < d_c; ++r) {
          double u = U_pca[size_t(r) * d_c + g.lat_begin + l];   // (U^T)[l][r] = U[r][l]
          sa += u * a[r];
          sb += u * b[r];
        }
        ta[l] = sa; tb[l] = sb;
      }
    } else {
      for (int l = 0; l < WL; ++l) { ta[l] = a[g.lat_begin + l]; tb[l] = b[g.lat_begin + l]; }
    }
    for (int l = 0; l < WL; ++l) {
      uk[(size_t(h) * WL + l) * d_h + e] = double_to_bf16(mu_j * ta[l]);   // mu_j folded
      uv[(size_t(h) * d_h + e) * WL + l] = double_to_bf16(tb[l]);
    }
  });
  // W^O rows of head block i, transposed to K-major for the up-projection GEMM: blocked
  // [ceil(D/128)][K/64][128][64] (each 128-row x 64-k tile one contiguous 16 KB block for the
  // TMA weight stream, rows >= D zero) when 64 | K, else plain [D, K]
  const int K = H * d_h;
  const bool blocked = wo_blocked(K);
  const int n_tiles = (D + 127) / 128, k_steps = K / 64;
  std::vector<uint16_t> wo(blocked ? size_t(n_tiles) * 128 * K : size_t(D) * K, 0);
  parallel_for(K, [&](int kk) {
    const uint16_t* src = W_O + (size_t(g.head_begin) * d_h + kk) * D;
    if (blocked) {
      const int ks = kk / 64, kc = kk % 64;
      for (int n = 0; n < D; ++n)
        wo[((size_t(n / 128) * k_steps + ks) * 128 + n % 128) * 64 + kc] = src[n];
    } else {
      for (int n = 0; n < D; ++n) wo[size_t(n) * K + kk] = src[n];
    }
  });
  std::vector<float> xf;
  if (xform_kind == TPLA_XFORM_HADAMARD) {
    xf.resize(d_c);
    for (int i = 0; i < d_c; ++i) xf[i] = static_cast<float>(signs[i]);
  } else if (xform_kind == TPLA_XFORM_PCA) {
    xf.resize(size_t(d_c) * WL);
    for (int r = 0; r < d_c; ++r)
      for (int l = 0; l < WL; ++l) xf[size_t(r) * WL + l] = U_pca[size_t(r) * d_c + g.lat_begin + l];
  }
  TPLA_CUDA(cudaMemcpyAsync(out->W_UK, uk.data(), uk.size() * 2, cudaMemcpyHostToDevice, s), "copy W_UK");
  TPLA_CUDA(cudaMemcpyAsync(out->W_UV, uv.data(), uv.size() * 2, cudaMemcpyHostToDevice, s), "copy W_UV");
  TPLA_CUDA(cudaMemcpyAsync(out->W_O, wo.data(), wo.size() * 2, cudaMemcpyHostToDevice, s), "copy W_O");
  if (!xf.empty())
    TPLA_CUDA(cudaMemcpyAsync(out->xform, xf.data(), xf.size() * 4, cudaMemcpyHostToDevice, s), "copy xform");
  TPLA_CUDA(cudaStreamSynchronize(s), "convert sync");
  out->xform_kind = xform_kind;
  out->alpha_j = alpha[shard];
  out->mu_j = mu[shard];
  return ok();
}

static tpla_status append_common(const tpla_config* cfg, const tpla_weights* w, const tpla_cache* cache,
                                 const void* c_kv, const void* k_pe, const int32_t* seq_idx, const int32_t* pos,
                                 int32_t n, int32_t rms_mode, int32_t* n_dropped, void* stream, int n_norm = 0,
                                 const float* alpha_s = nullptr) {
  Geom g{};
  tpla_status st = make_geom(cfg, &g);
  if (st) return st;
  if ((st = check_cache(g, cache))) return st;
  if (!is_pow2(g.d_c) || g.d_c < 32 || g.d_c > 1024)
    return fail(TPLA_ERR_SHAPE, "d_c=%d: cache-write kernel needs a power of two in [32, 1024]", g.d_c);
  if (g.d_r % 2) return fail(TPLA_ERR_SHAPE, "d_r must be even");
  if (!w) return fail(TPLA_ERR_INVALID_ARG, "NULL weights");
  if (w->xform_kind < 0 || w->xform_kind > 2) return fail(TPLA_ERR_INVALID_ARG, "bad xform_kind");
  if (w->xform_kind != TPLA_XFORM_IDENTITY && !w->xform) return fail(TPLA_ERR_INVALID_ARG, "NULL xform");
  if (rms_mode < 0 || rms_mode > 2) return fail(TPLA_ERR_INVALID_ARG, "bad rms_mode");
  if (rms_mode == TPLA_RMS_SLICED && !(w->alpha_j > 0.f)) return fail(TPLA_ERR_INVALID_ARG, "alpha_j must be > 0");
  if (n < 0) return fail(TPLA_ERR_INVALID_ARG, "n < 0");
  if (n == 0) return ok();
  if (!c_kv || !k_pe || !seq_idx || !pos) return fail(TPLA_ERR_INVALID_ARG, "NULL input");
  if (!aligned16(c_kv)) return fail(TPLA_ERR_INVALID_ARG, "c_kv not 16-byte aligned");
  // the Hadamard / identity cache write gives each lane d_c/32 consecutive latents: the device's
  // slice must be whole lanes (g <= 32 at d_c = 1024, any g <= d_c/32 in general)
  if (w->xform_kind != TPLA_XFORM_PCA && g.w_lat % (g.d_c / 32))
    return fail(TPLA_ERR_UNSUPPORTED, "W_lat=%d: the cache-write kernel needs W_lat a multiple of d_c/32=%d", g.w_lat,
                g.d_c / 32);
  cudaError_t e = launch_append_kv(g, w->xform_kind, static_cast<const float*>(w->xform), w->alpha_j, *cache,
                                   static_cast<const uint16_t*>(c_kv), static_cast<const uint16_t*>(k_pe), seq_idx,
                                   pos, n, rms_mode, n_dropped, static_cast<cudaStream_t>(stream), n_norm, alpha_s);
  if (e != cudaSuccess) return cuda_fail(e, "append_kv launch");
  return ok();
}

tpla_status tpla_append_kv_norm_only(const tpla_config* cfg, const tpla_weights* w, const tpla_cache* cache,
                                     const void* c_kv, const void* k_pe, const int32_t* seq_idx, const int32_t* pos,
                                     int32_t n, int32_t n_slices, const float* alpha, int32_t* n_dropped,
                                     void* stream) {
  if (!cfg || cfg->g != 1) return fail(TPLA_ERR_INVALID_ARG, "norm-only rows are g = 1 rows (the whole latent)");
  if (n_slices < 1 || n_slices > 8 || (n_slices & (n_slices - 1)) || !alpha)
    return fail(TPLA_ERR_INVALID_ARG, "n_slices=%d: a power of two in [1, 8], with alpha[n_slices]", n_slices);
  for (int q = 0; q < n_slices; ++q)
    if (!(alpha[q] > 0.f)) return fail(TPLA_ERR_INVALID_ARG, "alpha[%d] must be > 0", q);
  if (cfg->d_c % (32 * n_slices) && !(w && w->xform_kind == TPLA_XFORM_PCA))
    return fail(TPLA_ERR_UNSUPPORTED, "d_c=%d: slices must be whole lanes (d_c / 32 per lane)", cfg->d_c);
  return append_common(cfg, w, cache, c_kv, k_pe, seq_idx, pos, n, TPLA_RMS_SLICED, n_dropped, stream, n_slices, alpha);
}

tpla_status tpla_append_kv(const tpla_config* cfg, const tpla_weights* w, const tpla_cache* cache,
                           const void* c_kv, const void* k_pe, const int32_t* seq_idx, const int32_t* pos,
                           int32_t n, int32_t rms_mode, int32_t* n_dropped, void* stream) {
  return append_common(cfg, w, cache, c_kv, k_pe, seq_idx, pos, n, rms_mode, n_dropped, stream);
}

tpla_status tpla_prefill_mla(const tpla_config* cfg, const tpla_weights* w, const tpla_cache* cache,
                             const void* c_kv, const void* k_pe, const int32_t* seq_idx, const int32_t* pos,
                             int32_t n, const void* q, void* stream) {
  if (q) return fail(TPLA_ERR_UNSUPPORTED, "MLA prefill attention is not part of this build (SURVEY f1)");
  return append_common(cfg, w, cache, c_kv, k_pe, seq_idx, pos, n, TPLA_RMS_EXACT, nullptr, stream);
}

tpla_status tpla_decode_workspace_bytes_mtp(const tpla_config* cfg, int32_t B, int32_t n_q, int32_t max_seq_len,
                                            size_t* bytes) {
  Geom g{};
  tpla_status st = make_geom(cfg, &g);
  if (st) return st;
  if (B < 1 || n_q < 1 || max_seq_len < 1 || !bytes) return fail(TPLA_ERR_INVALID_ARG, "bad B/n_q/max_seq_len");
  *bytes = ws_layout(g, B, n_q, max_seq_len).total;
  return ok();
}

tpla_status tpla_decode_workspace_bytes(const tpla_config* cfg, int32_t B, int32_t max_seq_len, size_t* bytes) {
  return tpla_decode_workspace_bytes_mtp(cfg, B, 1, max_seq_len, bytes);
}

static tpla_status check_decode_common(const Geom& g, const tpla_cache* cache, const void* q_pe,
                                       const int32_t* seq_lens, int B, int max_seq_len) {
  tpla_status st;
  if ((st = check_kernel_shapes(g))) return st;
  const char* req = getenv("TPLA_REQUIRE_TC");
  if (req && req[0] == '1' && !use_tc_attention(g, B))
    return fail(TPLA_ERR_UNSUPPORTED, "TPLA_REQUIRE_TC: this shape runs the mma.sync K3 (W_lat=%d, d_r=%d, B=%d)",
                g.w_lat, g.d_r, B);
  if ((st = check_cache(g, cache))) return st;
  if (B < 1 || B > cache->batch) return fail(TPLA_ERR_SHAPE, "B=%d outside [1, cache batch %d]", B, cache->batch);
  if (max_seq_len < 1 || int64_t(max_seq_len) > int64_t(cache->max_pages_per_seq) * cache->page_size)
    return fail(TPLA_ERR_CAPACITY, "max_seq_len=%d exceeds page-table capacity", max_seq_len);
  if (!q_pe || !seq_lens) return fail(TPLA_ERR_INVALID_ARG, "NULL input");
  if (!aligned16(q_pe)) return fail(TPLA_ERR_INVALID_ARG, "q_pe not 16-byte aligned");
  return TPLA_OK;
}

tpla_status tpla_decode(const tpla_config* cfg, const tpla_weights* w, const tpla_cache* cache,
                        const void* q_nope, const void* q_pe, const int32_t* seq_lens, int32_t B,
                        int32_t max_seq_len, void* ws, size_t ws_bytes, float* y, void* out, int32_t flags,
                        tpla_comm* comm, void* stream) {
  return tpla_decode_mtp(cfg, w, cache, q_nope, q_pe, seq_lens, B, 1, max_seq_len, ws, ws_bytes, y, out, flags, comm,
                         stream);
}

tpla_status tpla_decode_mtp(const tpla_config* cfg, const tpla_weights* w, const tpla_cache* cache,
                            const void* q_nope, const void* q_pe, const int32_t* seq_lens, int32_t B, int32_t n_q,
                            int32_t max_seq_len, void* ws, size_t ws_bytes, float* y, void* out, int32_t flags,
                            tpla_comm* comm, void* stream) {
  Geom g{};
  tpla_status st = make_geom(cfg, &g);
  if (st) return st;
  if ((st = check_decode_common(g, cache, q_pe, seq_lens, B, max_seq_len))) return st;
  if (n_q < 1) return fail(TPLA_ERR_INVALID_ARG, "n_q=%d", n_q);
  if (n_q > 1 && !(use_tc_attention(g, B) && combine_wuv_supported(g) && n_q * g.h_loc <= 128))
    return fail(TPLA_ERR_UNSUPPORTED, "multi-token decode needs the tcgen05 path and n_q*H_loc <= 128 (n_q=%d, H_loc=%d)",
                n_q, g.h_loc);
  const int R = B * n_q;                                  // output rows (sequence, token)
  if (!w || !w->W_UK || !w->W_UV || !w->W_O) return fail(TPLA_ERR_INVALID_ARG, "NULL weights");
  if (!q_nope || !y || !ws) return fail(TPLA_ERR_INVALID_ARG, "NULL q_nope/y/ws");
  if (!aligned16(q_nope) || !aligned16(ws) || !aligned16(y)) return fail(TPLA_ERR_INVALID_ARG, "misaligned pointer");
  if (out && !aligned16(out)) return fail(TPLA_ERR_INVALID_ARG, "out misaligned");
  // A process may hold several of the k ranks (they accumulate into y before the all-reduce),
  // so the communicator spans k/m processes for some m >= 1.
  if (comm && (g.k % comm->world))
    return fail(TPLA_ERR_INVALID_ARG, "communicator world %d does not divide k=%d", comm->world, g.k);
  WsLayout L = ws_layout(g, B, n_q, max_seq_len);
  if (ws_bytes < L.total) return fail(TPLA_ERR_CAPACITY, "workspace %zu < %zu bytes", ws_bytes, L.total);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* base = static_cast<char*>(ws);
  auto* q_lat = reinterpret_cast<uint16_t*>(base + L.q_lat);
  auto* o_lat = reinterpret_cast<uint16_t*>(base + L.o_lat);
  auto* v = reinterpret_cast<uint16_t*>(base + L.v);
  auto* y_part = reinterpret_cast<float*>(base + L.y_part);
  const auto* qn = static_cast<const uint16_t*>(q_nope);
  cudaError_t e;
  const bool tc_path = use_tc_attention(g, B) && combine_wuv_supported(g);
  auto* plan = reinterpret_cast<int32_t*>(base + L.plan);
  // K3p (K3's schedule) and K2: Q'_j[b,h,:] = W^UK'_j[h] q[b,h,:]   (mu_j folded)
  e = launch_pre(g, *cache, seq_lens, B, L.n_cta, plan, tc_path, static_cast<const uint16_t*>(w->W_UK), qn, R, q_lat, s);
  if (e != cudaSuccess) return cuda_fail(e, "K3p/K2 pre-attention");
  if (tc_path) {
    // K3: per-shard split-K flash decoding (Eq. tpla_softmax_one_device) -> partials;
    // K4 + K5a fused: merge the partials of each (b, h) into O_j and apply W^UV'_j
    auto* o_part = reinterpret_cast<uint16_t*>(base + L.o_part);   // (fp16 partials)
    auto* ml_part = reinterpret_cast<float*>(base + L.ml_part);
    auto* meta = reinterpret_cast<int32_t*>(base + L.meta);
    e = launch_decode_attn_tc(g, *cache, q_lat, static_cast<const uint16_t*>(q_pe), seq_lens, B, n_q, L.n_cta,
                              plan, o_part, ml_part, meta, s);
    if (e != cudaSuccess) return cuda_fail(e, "K3 decode attention");
    e = launch_combine_wuv(g, B, n_q, o_part, ml_part, meta, static_cast<const uint16_t*>(w->W_UV), v, s);
    if (e != cudaSuccess) return cuda_fail(e, "K4+K5a combine/W_UV");
  } else {
    // K3 + K4: per-shard split-K flash decoding (Eq. tpla_softmax_one_device) -> O_j
    e = run_attention(g, *cache, q_lat, static_cast<const uint16_t*>(q_pe), seq_lens, B, max_seq_len, L, base, o_lat,
                      nullptr, nullptr, s);
    if (e != cudaSuccess) return cuda_fail(e, "K3/K4 decode attention");
    // K5a: v[b,h,:] = W^UV'_j[h]^T-applied O_j  (W^VO factored)
    e = launch_head_gemv("K5_W_UV", static_cast<const uint16_t*>(w->W_UV), o_lat, long(g.h_loc) * g.w_lat, g.h_loc,
                         g.d_h, g.w_lat, B, v, false, s);
    if (e != cudaSuccess) return cuda_fail(e, "K5a W_UV");
  }
  // K5b: Õ_j = v W^O_rows — tcgen05 weight stream where the shapes allow
  const bool accumulate = (flags & TPLA_DECODE_ACCUMULATE) != 0;
  const int Kw = g.h_loc * g.d_h;
  const char* force = getenv("TPLA_WO");
  bool out_done = false, reduced = false;
  if (wo_tc_supported(g.D, Kw, std::min(R, kWoRows)) && !(force && strcmp(force, "mma") == 0)) {
    // without an all-reduce the segment reduce also writes the bf16 output (no cast launch); with the
    // fused one-shot all-reduce (f2(i)) it also sums the ranks
    const FusedAr* ar = fused_ar(comm, R, g.D);
    uint16_t* out16 = (comm && !ar) ? nullptr : static_cast<uint16_t*>(out);
    e = run_wo_tc(static_cast<const uint16_t*>(w->W_O), v, g.D, Kw, R, base + L.wo_part, y, accumulate, out16, s, 0,
                  0, ar);
    if (e != cudaSuccess) return cuda_fail(e, "K5b W_O (tcgen05)");
    out_done = out16 != nullptr;
    reduced = ar != nullptr;
  } else {
    e = launch_skinny_gemm(static_cast<const uint16_t*>(w->W_O), v, g.D, Kw, R, L.kslices, y_part, s);
    if (e != cudaSuccess) return cuda_fail(e, "K5b W_O");
    e = launch_reduce_slices(y_part, L.kslices, R, g.D, y, accumulate, s);
    if (e != cudaSuccess) return cuda_fail(e, "K5b reduce");
  }
  // C1: O = AllReduce(Σ_r Õ_r)
  if (comm && !reduced) {
    ncclResult_t r = g_nccl.AllReduce(y, y, size_t(R) * g.D, ncclFloat32, ncclSum, comm->comm, s);
    if (r != ncclSuccess) return fail(TPLA_ERR_NCCL, "ncclAllReduce: %s", g_nccl.GetErrorString(r));
  }
  if (out && !out_done) {
    e = launch_cast_bf16(y, long(R) * g.D, static_cast<uint16_t*>(out), s);
    if (e != cudaSuccess) return cuda_fail(e, "cast");
  }
  return ok();
}

// ---- prefill attention as multi-token decode over prefixes (k6_prefill.cu) ----
namespace {
struct PrefillPlan {
  int n_q;        // prompt tokens per pseudo-sequence: n_q * H_loc <= 128 MMA rows
  int rows;       // prompt rows per chunk (one decode call; <= 256 keeps the tcgen05 W^O path)
  int n_chunks;
  size_t dec_bytes, tab_bytes, total;
};
PrefillPlan prefill_plan(const Geom& g, int L, int max_pages) {
  PrefillPlan p{};
  p.n_q = std::max(1, 128 / g.h_loc);
  p.rows = std::max(p.n_q, (256 / p.n_q) * p.n_q);
  p.n_chunks = (L + p.rows - 1) / p.rows;
  const int n_seq = p.rows / p.n_q + 1;                     // (+1: the remainder pseudo-sequence)
  // the two decode calls of a chunk: rows / n_q pseudo-sequences of n_q tokens, and one of the
  // remainder (ws_layout is not monotonic in the row count: <= 256 rows add the tcgen05 W^O partials)
  p.dec_bytes = align256(std::max(ws_layout(g, p.rows / p.n_q, p.n_q, L).total,
                                  ws_layout(g, 1, std::max(1, p.n_q - 1), L).total));
  p.tab_bytes = align256(size_t(n_seq) * (max_pages + 1) * 4);
  p.total = p.dec_bytes + size_t(p.n_chunks) * p.tab_bytes;
  return p;
}
}  // namespace

tpla_status tpla_prefill_workspace_bytes(const tpla_config* cfg, int32_t L, int32_t max_pages_per_seq, size_t* bytes) {
  Geom g{};
  tpla_status st = make_geom(cfg, &g);
  if (st) return st;
  if (!bytes || L < 1 || max_pages_per_seq < 1) return fail(TPLA_ERR_INVALID_ARG, "L=%d, max_pages=%d", L, max_pages_per_seq);
  *bytes = prefill_plan(g, L, max_pages_per_seq).total;
  return ok();
}

tpla_status tpla_prefill_attention(const tpla_config* cfg, const tpla_weights* w, const tpla_cache* cache,
                                   const void* q_nope, const void* q_pe, int32_t seq, int32_t L, void* ws,
                                   size_t ws_bytes, float* y, void* out, int32_t flags, tpla_comm* comm,
                                   void* stream) {
  Geom g{};
  tpla_status st = make_geom(cfg, &g);
  if (st) return st;
  if (!cache || !cache->block_table) return fail(TPLA_ERR_INVALID_ARG, "NULL cache");
  if (seq < 0 || seq >= cache->batch) return fail(TPLA_ERR_SHAPE, "seq=%d outside [0, %d)", seq, cache->batch);
  if (L < 1 || int64_t(L) > int64_t(cache->max_pages_per_seq) * cache->page_size)
    return fail(TPLA_ERR_CAPACITY, "L=%d outside the page table", L);
  if (!q_nope || !q_pe || !y || !ws) return fail(TPLA_ERR_INVALID_ARG, "NULL q_nope/q_pe/y/ws");
  const PrefillPlan p = prefill_plan(g, L, cache->max_pages_per_seq);
  if (!(use_tc_attention(g, p.rows / p.n_q + 1) && combine_wuv_supported(g)))
    return fail(TPLA_ERR_UNSUPPORTED, "prefill attention needs the tcgen05 path (W_lat=%d, d_r=%d)", g.w_lat, g.d_r);
  if (ws_bytes < p.total) return fail(TPLA_ERR_CAPACITY, "workspace %zu < %zu bytes", ws_bytes, p.total);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* base = static_cast<char*>(ws);
  const auto* qn = static_cast<const uint16_t*>(q_nope);
  const auto* qp = static_cast<const uint16_t*>(q_pe);
  auto* o16 = static_cast<uint16_t*>(out);
  const int n_seq_max = p.rows / p.n_q + 1;
  for (int c = 0; c < p.n_chunks; ++c) {
    const int r0 = c * p.rows, nr = std::min(p.rows, L - r0);
    const int full = nr / p.n_q, rem = nr % p.n_q;
    // each chunk has its own table region: a later chunk's table kernel may start (PDL) while
    // this chunk's attention still reads its table
    auto* table = reinterpret_cast<int32_t*>(base + p.dec_bytes + size_t(c) * p.tab_bytes);
    int32_t* lens = table + size_t(n_seq_max) * cache->max_pages_per_seq;
    cudaError_t e = launch_prefix_table(cache->block_table, seq, cache->max_pages_per_seq, full, p.n_q, r0, nr, table,
                                        lens, s);
    if (e != cudaSuccess) return cuda_fail(e, "K6 prefix table");
    tpla_cache pc = *cache;
    pc.block_table = table;
    struct Part { int n_seq, n_q, row0; };
    const Part parts[2] = {{full, p.n_q, r0}, {rem ? 1 : 0, rem, r0 + full * p.n_q}};
    for (int k = 0; k < 2; ++k) {
      if (parts[k].n_seq == 0) continue;
      pc.batch = parts[k].n_seq;
      pc.block_table = table + size_t(k ? full : 0) * cache->max_pages_per_seq;
      const size_t r = size_t(parts[k].row0);
      // K3 reads the pseudo-sequence table and lengths before its PDL wait (its schedule runs
      // under the predecessor's tail), so the first launch after K6 (K2) waits for K6 in plain
      // stream order; K3, launched after K2 started, then sees K6's writes.
      g_no_pdl_next = k == 0;
      st = tpla_decode_mtp(cfg, w, &pc, qn + r * g.h_q * g.d_h, qp + r * g.h_q * g.d_r, lens + (k ? full : 0),
                           parts[k].n_seq, parts[k].n_q, L, base, p.dec_bytes, y + r * g.D, o16 ? o16 + r * g.D : nullptr,
                           flags, comm, stream);
      g_no_pdl_next = false;
      if (st) return st;
    }
  }
  return ok();
}

tpla_status tpla_decode_v(const tpla_config* cfg, const tpla_weights* w, const tpla_cache* cache, const void* q_nope,
                          const void* q_pe, const int32_t* seq_lens, int32_t B, int32_t n_q, int32_t max_seq_len,
                          void* ws, size_t ws_bytes, float* v_acc, int32_t n_chunks, int32_t flags, void* stream) {
  Geom g{};
  tpla_status st = make_geom(cfg, &g);
  if (st) return st;
  if ((st = check_decode_common(g, cache, q_pe, seq_lens, B, max_seq_len))) return st;
  if (!w || !w->W_UK || !w->W_UV) return fail(TPLA_ERR_INVALID_ARG, "NULL weights");
  if (!q_nope || !v_acc || !ws) return fail(TPLA_ERR_INVALID_ARG, "NULL q_nope/v_acc/ws");
  if (!aligned16(q_nope) || !aligned16(ws) || !aligned16(v_acc)) return fail(TPLA_ERR_INVALID_ARG, "misaligned pointer");
  if (n_q < 1 || !(use_tc_attention(g, B) && combine_wuv_supported(g) && n_q * g.h_loc <= 128))
    return fail(TPLA_ERR_UNSUPPORTED, "tpla_decode_v needs the tcgen05 path (n_q=%d, H_loc=%d)", n_q, g.h_loc);
  if (n_chunks < 1 || (g.h_loc * g.d_h) % (64 * n_chunks))
    return fail(TPLA_ERR_DIVISIBILITY, "n_chunks=%d: 64*n_chunks must divide H_loc*d_h=%d", n_chunks, g.h_loc * g.d_h);
  WsLayout L = ws_layout(g, B, n_q, max_seq_len);
  if (ws_bytes < L.total) return fail(TPLA_ERR_CAPACITY, "workspace %zu < %zu bytes", ws_bytes, L.total);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* base = static_cast<char*>(ws);
  auto* q_lat = reinterpret_cast<uint16_t*>(base + L.q_lat);
  auto* o_part = reinterpret_cast<uint16_t*>(base + L.o_part);     // (fp16 partials)
  auto* ml_part = reinterpret_cast<float*>(base + L.ml_part);
  auto* meta = reinterpret_cast<int32_t*>(base + L.meta);
  const auto* qn = static_cast<const uint16_t*>(q_nope);
  auto* plan = reinterpret_cast<int32_t*>(base + L.plan);
  const bool pre = !(flags & TPLA_DECODE_STAGE_ATTN), attn = !(flags & TPLA_DECODE_STAGE_PRE);
  if (!pre && !attn) return fail(TPLA_ERR_INVALID_ARG, "STAGE_PRE and STAGE_ATTN together");
  cudaError_t e = cudaSuccess;
  if (pre) {
    e = launch_pre(g, *cache, seq_lens, B, L.n_cta, plan, true, static_cast<const uint16_t*>(w->W_UK), qn, B * n_q,
                   q_lat, s);
    if (e != cudaSuccess) return cuda_fail(e, "K3p/K2 pre-attention");
  }
  if (!attn) return ok();
  e = launch_decode_attn_tc(g, *cache, q_lat, static_cast<const uint16_t*>(q_pe), seq_lens, B, n_q, L.n_cta, plan,
                            o_part, ml_part, meta, s);
  if (e != cudaSuccess) return cuda_fail(e, "K3 decode attention");
  e = launch_combine_wuv(g, B, n_q, o_part, ml_part, meta, static_cast<const uint16_t*>(w->W_UV), nullptr, s, v_acc,
                         (flags & TPLA_DECODE_ACCUMULATE) != 0, n_chunks);
  if (e != cudaSuccess) return cuda_fail(e, "K4+K5a combine/W_UV");
  return ok();
}

static tpla_status project_out_common(const tpla_config* cfg, const tpla_weights* w, float* const* v_list, int32_t n_v,
                                      int32_t R, int32_t n_chunks, int32_t chunk, void* ws, size_t ws_bytes, float* y,
                                      void* out, int32_t flags, tpla_comm* group_comm, tpla_comm* comm, void* stream) {
  Geom g{};
  tpla_status st = make_geom(cfg, &g);
  if (st) return st;
  if (!w || !w->W_O) return fail(TPLA_ERR_INVALID_ARG, "NULL weights");
  if (!v_list || n_v < 1 || n_v > kMaxSumSrc) return fail(TPLA_ERR_INVALID_ARG, "n_v=%d outside [1, %d]", n_v, kMaxSumSrc);
  for (int i = 0; i < n_v; ++i)
    if (!v_list[i] || !aligned16(v_list[i])) return fail(TPLA_ERR_INVALID_ARG, "v_acc %d NULL or misaligned", i);
  if (!ws || !y) return fail(TPLA_ERR_INVALID_ARG, "NULL ws/y");
  if (!aligned16(ws) || !aligned16(y) || (out && !aligned16(out))) return fail(TPLA_ERR_INVALID_ARG, "misaligned pointer");
  const int K = g.h_loc * g.d_h;
  if (R < 1 || n_chunks < 1 || chunk < 0 || chunk >= n_chunks)
    return fail(TPLA_ERR_INVALID_ARG, "R=%d, chunk %d of %d", R, chunk, n_chunks);
  if (K % (64 * n_chunks))
    return fail(TPLA_ERR_DIVISIBILITY, "n_chunks=%d: 64*n_chunks must divide H_loc*d_h=%d", n_chunks, K);
  if (group_comm && n_v != 1) return fail(TPLA_ERR_INVALID_ARG, "a reduce-scattered group takes one accumulator");
  if (group_comm && (group_comm->world != n_chunks || group_comm->rank != chunk))
    return fail(TPLA_ERR_INVALID_ARG, "group communicator (rank %d of %d) must be chunk %d of %d", group_comm->rank,
                group_comm->world, chunk, n_chunks);
  const int kc = K / n_chunks;
  if (!wo_tc_supported(g.D, K, std::min(R, kWoRows)))
    return fail(TPLA_ERR_UNSUPPORTED, "tpla_project_out needs the tcgen05 W^O path (K=%d, R=%d)", K, R);
  if (comm && (g.k % comm->world))
    return fail(TPLA_ERR_INVALID_ARG, "communicator world %d does not divide k=%d", comm->world, g.k);
  if ((group_comm || comm) && !load_nccl()) return fail(TPLA_ERR_NCCL, "NCCL not loadable");
  const size_t v_bytes = align256(size_t(R) * kc * 2);
  const size_t part_bytes = wo_tc_part_bytes(g.D, kc, std::min(R, kWoRows));
  if (ws_bytes < kWsHeader + v_bytes + part_bytes)
    return fail(TPLA_ERR_CAPACITY, "workspace %zu < %zu bytes", ws_bytes, kWsHeader + v_bytes + part_bytes);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const float* v_mine[kMaxSumSrc];
  for (int i = 0; i < n_v; ++i) v_mine[i] = v_list[i] + size_t(chunk) * R * kc;   // chunk c: [R, kc] contiguous
  if (group_comm && n_chunks > 1) {                                // Σ over the group, chunk c to its rank
    ncclResult_t r = g_nccl.ReduceScatter(v_list[0], v_list[0] + size_t(chunk) * R * kc, size_t(R) * kc, ncclFloat32,
                                          ncclSum, group_comm->comm, s);
    if (r != ncclSuccess) return fail(TPLA_ERR_NCCL, "ncclReduceScatter: %s", g_nccl.GetErrorString(r));
  }
  auto* v16 = reinterpret_cast<uint16_t*>(static_cast<char*>(ws) + kWsHeader);   // (past the K3p plan)
  // v = bf16(Σ_j v_j), this slice (one source: the group sum is already in place)
  cudaError_t e = n_v == 1 ? launch_cast_bf16(v_mine[0], long(R) * kc, v16, s, "K5_v_cast")
                           : launch_sum_cast_bf16(v_mine, n_v, long(R) * kc, v16, s);
  if (e != cudaSuccess) return cuda_fail(e, "v cast");
  const FusedAr* ar = fused_ar(comm, R, g.D);                     // f2(i): the all-reduce in the K5 reduce
  uint16_t* out16 = (comm && !ar) ? nullptr : static_cast<uint16_t*>(out);
  e = run_wo_tc(static_cast<const uint16_t*>(w->W_O), v16, g.D, K, R, static_cast<char*>(ws) + kWsHeader + v_bytes, y,
                (flags & TPLA_DECODE_ACCUMULATE) != 0, out16, s, chunk * kc, kc, ar);
  if (e != cudaSuccess) return cuda_fail(e, "K5b W_O (tcgen05)");
  if (comm && !ar) {                                               // C1: O = AllReduce(Σ Õ)
    ncclResult_t r = g_nccl.AllReduce(y, y, size_t(R) * g.D, ncclFloat32, ncclSum, comm->comm, s);
    if (r != ncclSuccess) return fail(TPLA_ERR_NCCL, "ncclAllReduce: %s", g_nccl.GetErrorString(r));
    if (out) {
      e = launch_cast_bf16(y, long(R) * g.D, static_cast<uint16_t*>(out), s);
      if (e != cudaSuccess) return cuda_fail(e, "cast");
    }
  }
  return ok();
}

tpla_status tpla_project_out(const tpla_config* cfg, const tpla_weights* w, float* v_acc, int32_t R, int32_t n_chunks,
                             int32_t chunk, void* ws, size_t ws_bytes, float* y, void* out, int32_t flags,
                             tpla_comm* group_comm, tpla_comm* comm, void* stream) {
  float* const list[1] = {v_acc};
  return project_out_common(cfg, w, list, 1, R, n_chunks, chunk, ws, ws_bytes, y, out, flags, group_comm, comm, stream);
}

tpla_status tpla_project_out_sum(const tpla_config* cfg, const tpla_weights* w, const float* const* v_list, int32_t n_v,
                                 int32_t R, int32_t n_chunks, int32_t chunk, void* ws, size_t ws_bytes, float* y,
                                 void* out, int32_t flags, tpla_comm* comm, void* stream) {
  if (!v_list) return fail(TPLA_ERR_INVALID_ARG, "NULL v_list");
  float* list[kMaxSumSrc];
  if (n_v < 1 || n_v > kMaxSumSrc) return fail(TPLA_ERR_INVALID_ARG, "n_v=%d outside [1, %d]", n_v, kMaxSumSrc);
  for (int i = 0; i < n_v; ++i) list[i] = const_cast<float*>(v_list[i]);
  return project_out_common(cfg, w, list, n_v, R, n_chunks, chunk, ws, ws_bytes, y, out, flags, nullptr, comm, stream);
}

// ---- MLA prefill, non-absorbed: K8 ------------------------------------------------
namespace {
// Blocked K-major layout of a [N, K] bf16 matrix for the tcgen05 weight-stream GEMM: element (n, k)
// at ((n / 128) * (K / 64) + k / 64) * 8192 + (n % 128) * 64 + k % 64; rows >= N zero.
size_t blocked_elems(int N, int K) { return size_t((N + 127) / 128) * 128 * K; }
inline size_t blocked_index(int n, int k, int K) {
  return (size_t(n / 128) * (K / 64) + k / 64) * 8192 + size_t(n % 128) * 64 + k % 64;
}
struct PfGeom {
  int H, h0, Kf;   // heads of this device, first head, H·d_h
};
tpla_status prefill_geom(const tpla_config* cfg, Geom* g, PfGeom* p) {
  tpla_status st = make_geom(cfg, g);
  if (st) return st;
  if (g->g != 1) return fail(TPLA_ERR_UNSUPPORTED, "MLA prefill splits heads only (g = 1, P:421), got g=%d", g->g);
  if (g->d_h != 128 || g->d_r != 64 || g->d_c % 64)
    return fail(TPLA_ERR_UNSUPPORTED, "MLA prefill kernels need d_h=128, d_r=64, 64 | d_c (got %d, %d, %d)", g->d_h,
                g->d_r, g->d_c);
  p->H = g->h_loc;
  p->h0 = g->head_begin;
  p->Kf = g->h_loc * g->d_h;
  if (p->Kf % 64) return fail(TPLA_ERR_UNSUPPORTED, "H*d_h=%d must be a multiple of 64", p->Kf);
  return TPLA_OK;
}
struct PfWs {
  size_t c_hat, K, V, O, total;
};
PfWs pf_ws(const Geom& g, const PfGeom& p, int L) {
  PfWs w{};
  size_t off = 0;
  w.c_hat = off; off += align256(size_t(L) * g.d_c * 2);
  w.K = off;     off += align256(size_t(L) * p.Kf * 2);
  w.V = off;     off += align256(size_t(L) * p.Kf * 2);
  w.O = off;     off += align256(size_t(L) * p.Kf * 2);
  w.total = off;
  return w;
}
}  // namespace

tpla_status tpla_prefill_weights_bytes(const tpla_config* cfg, size_t* W_UK, size_t* W_UV, size_t* W_O) {
  Geom g{};
  PfGeom p{};
  tpla_status st = prefill_geom(cfg, &g, &p);
  if (st) return st;
  if (W_UK) *W_UK = blocked_elems(p.Kf, g.d_c) * 2;
  if (W_UV) *W_UV = blocked_elems(p.Kf, g.d_c) * 2;
  if (W_O) *W_O = blocked_elems(g.D, p.Kf) * 2;
  return ok();
}

tpla_status tpla_convert_prefill_weights(const tpla_config* cfg, const uint16_t* W_UK, const uint16_t* W_UV,
                                         const uint16_t* gamma, const uint16_t* W_O, tpla_prefill_weights* out,
                                         void* stream) {
  Geom g{};
  PfGeom p{};
  tpla_status st = prefill_geom(cfg, &g, &p);
  if (st) return st;
  if (!W_UK || !W_UV || !gamma || !W_O || !out || !out->W_UK || !out->W_UV || !out->W_O)
    return fail(TPLA_ERR_INVALID_ARG, "NULL argument");
  const int d_c = g.d_c, hq_dh = g.h_q * g.d_h, D = g.D;
  std::vector<uint16_t> uk(blocked_elems(p.Kf, d_c), 0), uv(blocked_elems(p.Kf, d_c), 0), wo(blocked_elems(D, p.Kf), 0);
  // k = ĉ W_γ W^UK[:, heads]: row n = local feature (h·d_h + e), column k = latent l (original basis)
  parallel_for(d_c, [&](int l) {
    const double gm = bf16_to_double(gamma[l]);
    for (int n = 0; n < p.Kf; ++n) {
      const size_t src = size_t(l) * hq_dh + size_t(p.h0) * g.d_h + n;
      uk[blocked_index(n, l, d_c)] = double_to_bf16(gm * bf16_to_double(W_UK[src]));
      uv[blocked_index(n, l, d_c)] = double_to_bf16(gm * bf16_to_double(W_UV[src]));
    }
  });
  parallel_for(p.Kf, [&](int kk) {      // y = O W^O[head rows]: row n = output d, column = local feature kk
    const uint16_t* src = W_O + (size_t(p.h0) * g.d_h + kk) * D;
    for (int n = 0; n < D; ++n) wo[blocked_index(n, kk, p.Kf)] = src[n];
  });
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  TPLA_CUDA(cudaMemcpyAsync(out->W_UK, uk.data(), uk.size() * 2, cudaMemcpyHostToDevice, s), "copy W_UK");
  TPLA_CUDA(cudaMemcpyAsync(out->W_UV, uv.data(), uv.size() * 2, cudaMemcpyHostToDevice, s), "copy W_UV");
  TPLA_CUDA(cudaMemcpyAsync(out->W_O, wo.data(), wo.size() * 2, cudaMemcpyHostToDevice, s), "copy W_O");
  TPLA_CUDA(cudaStreamSynchronize(s), "convert sync");
  return ok();
}

tpla_status tpla_prefill_mla_workspace_bytes(const tpla_config* cfg, int32_t L, size_t* bytes) {
  Geom g{};
  PfGeom p{};
  tpla_status st = prefill_geom(cfg, &g, &p);
  if (st) return st;
  if (L < 1 || !bytes) return fail(TPLA_ERR_INVALID_ARG, "L=%d", L);
  *bytes = pf_ws(g, p, L).total;
  return ok();
}

tpla_status tpla_prefill_mla_forward(const tpla_config* cfg, const tpla_prefill_weights* w, const void* c_kv,
                                     const void* k_pe, const void* q_nope, const void* q_pe, int32_t L, void* ws,
                                     size_t ws_bytes, float* y, void* out, int32_t flags, tpla_comm* comm,
                                     void* stream) {
  Geom g{};
  PfGeom p{};
  tpla_status st = prefill_geom(cfg, &g, &p);
  if (st) return st;
  if (!w || !w->W_UK || !w->W_UV || !w->W_O) return fail(TPLA_ERR_INVALID_ARG, "NULL weights");
  if (!c_kv || !k_pe || !q_nope || !q_pe || !ws || !y) return fail(TPLA_ERR_INVALID_ARG, "NULL input");
  if (!aligned16(c_kv) || !aligned16(k_pe) || !aligned16(q_nope) || !aligned16(q_pe) || !aligned16(ws) || !aligned16(y) ||
      (out && !aligned16(out)))
    return fail(TPLA_ERR_INVALID_ARG, "misaligned pointer");
  if (L < 1) return fail(TPLA_ERR_INVALID_ARG, "L=%d", L);
  if (comm && (g.k % comm->world))
    return fail(TPLA_ERR_INVALID_ARG, "communicator world %d does not divide k=%d", comm->world, g.k);
  if (comm && !load_nccl()) return fail(TPLA_ERR_NCCL, "NCCL not loadable");
  const PfWs L_ = pf_ws(g, p, L);
  if (ws_bytes < L_.total) return fail(TPLA_ERR_CAPACITY, "workspace %zu < %zu bytes", ws_bytes, L_.total);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* base = static_cast<char*>(ws);
  auto* c_hat = reinterpret_cast<uint16_t*>(base + L_.c_hat);
  auto* Kb = reinterpret_cast<uint16_t*>(base + L_.K);
  auto* Vb = reinterpret_cast<uint16_t*>(base + L_.V);
  auto* Ob = reinterpret_cast<uint16_t*>(base + L_.O);
  // ĉ = RMSNorm(c) (full RMS)
  cudaError_t e = launch_prefill_rmsnorm(static_cast<const uint16_t*>(c_kv), L, g.d_c, g.eps, c_hat, s);
  if (e != cudaSuccess) return cuda_fail(e, "K8 rmsnorm");
  // k = ĉ W^UK_h, v = ĉ W^UV_h for this device's heads (K9 tcgen05 GEMM, bf16 out)
  e = launch_gemm_tn(static_cast<const uint16_t*>(w->W_UK), c_hat, g.d_c, p.Kf, g.d_c, L, nullptr, false, Kb, s);
  if (e != cudaSuccess) return cuda_fail(e, "K9 k up-projection");
  e = launch_gemm_tn(static_cast<const uint16_t*>(w->W_UV), c_hat, g.d_c, p.Kf, g.d_c, L, nullptr, false, Vb, s);
  if (e != cudaSuccess) return cuda_fail(e, "K9 v up-projection");
  // causal attention per head (Eq. isolate_rope)
  e = launch_attn_fwd_causal(static_cast<const uint16_t*>(q_nope), static_cast<const uint16_t*>(q_pe), g.h_q, p.h0, Kb,
                             Vb, p.H, static_cast<const uint16_t*>(k_pe), g.d_r, L, g.sm_scale, Ob, s);
  if (e != cudaSuccess) return cuda_fail(e, "K8 attention");
  // y = concat_h O_h · W^O[head rows], then the all-reduce over the head-split devices
  const bool accumulate = (flags & TPLA_DECODE_ACCUMULATE) != 0;
  uint16_t* out16 = comm ? nullptr : static_cast<uint16_t*>(out);
  e = launch_gemm_tn(static_cast<const uint16_t*>(w->W_O), Ob, p.Kf, g.D, p.Kf, L, y, accumulate,
                     accumulate ? nullptr : out16, s);
  if (e != cudaSuccess) return cuda_fail(e, "K9 W^O");
  if (accumulate && out16) {                     // (y was reduce-added: its bf16 copy after the sum)
    e = launch_cast_bf16(y, long(L) * g.D, out16, s);
    if (e != cudaSuccess) return cuda_fail(e, "cast");
  }
  if (comm) {
    ncclResult_t r = g_nccl.AllReduce(y, y, size_t(L) * g.D, ncclFloat32, ncclSum, comm->comm, s);
    if (r != ncclSuccess) return fail(TPLA_ERR_NCCL, "ncclAllReduce: %s", g_nccl.GetErrorString(r));
    if (out) {
      e = launch_cast_bf16(y, long(L) * g.D, static_cast<uint16_t*>(out), s);
      if (e != cudaSuccess) return cuda_fail(e, "cast");
    }
  }
  return ok();
}

tpla_status tpla_decode_attention(const tpla_config* cfg, const tpla_cache* cache, const void* q_lat,
                                  const void* q_pe, const int32_t* seq_lens, int32_t B, int32_t max_seq_len,
                                  void* ws, size_t ws_bytes, float* O, float* lse, void* stream) {
  return tpla_decode_attention_ex(cfg, cache, q_lat, q_pe, seq_lens, B, max_seq_len, ws, ws_bytes, O, lse, 0, stream);
}

tpla_status tpla_decode_attention_ex(const tpla_config* cfg, const tpla_cache* cache, const void* q_lat,
                                     const void* q_pe, const int32_t* seq_lens, int32_t B, int32_t max_seq_len,
                                     void* ws, size_t ws_bytes, float* O, float* lse, int32_t flags, void* stream) {
  Geom g{};
  tpla_status st = make_geom(cfg, &g);
  if (st) return st;
  if ((st = check_decode_common(g, cache, q_pe, seq_lens, B, max_seq_len))) return st;
  if (!q_lat || !ws) return fail(TPLA_ERR_INVALID_ARG, "NULL q_lat/ws");
  if (!O && lse) return fail(TPLA_ERR_INVALID_ARG, "lse requires O");
  if (!aligned16(q_lat) || !aligned16(ws)) return fail(TPLA_ERR_INVALID_ARG, "misaligned pointer");
  if (flags & ~int32_t(TPLA_ATTN_REUSE_PLAN)) return fail(TPLA_ERR_INVALID_ARG, "unknown flags 0x%x", flags);
  const bool reuse = (flags & TPLA_ATTN_REUSE_PLAN) != 0;
  if (reuse && !use_tc_attention(g, B))
    return fail(TPLA_ERR_UNSUPPORTED, "TPLA_ATTN_REUSE_PLAN needs the tcgen05 K3 (no schedule otherwise)");
  WsLayout L = ws_layout(g, B, 1, max_seq_len);
  if (ws_bytes < L.total) return fail(TPLA_ERR_CAPACITY, "workspace %zu < %zu bytes", ws_bytes, L.total);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* base = static_cast<char*>(ws);
  cudaError_t e = run_attention(g, *cache, static_cast<const uint16_t*>(q_lat), static_cast<const uint16_t*>(q_pe),
                                seq_lens, B, max_seq_len, L, base, nullptr, O, lse, s, reuse);
  if (e != cudaSuccess) return cuda_fail(e, "K3/K4 decode attention");
  return ok();
}

tpla_status tpla_comm_unique_id(void* out128) {
  if (!out128) return fail(TPLA_ERR_INVALID_ARG, "NULL id buffer");
  if (!load_nccl()) return fail(TPLA_ERR_NCCL, "libnccl.so.2 not loadable (set TPLA_NCCL_LIB)");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  ncclResult_t r = g_nccl.GetUniqueId(&id);
  if (r != ncclSuccess) return fail(TPLA_ERR_NCCL, "ncclGetUniqueId: %s", g_nccl.GetErrorString(r));
  memcpy(out128, &id, 128);
  return ok();
}

tpla_status tpla_comm_init(tpla_comm** out, const void* unique_id128, int32_t world, int32_t rank) {
  if (!out || !unique_id128 || world < 1 || rank < 0 || rank >= world) return fail(TPLA_ERR_INVALID_ARG, "bad arguments");
  if (!load_nccl()) return fail(TPLA_ERR_NCCL, "libnccl.so.2 not loadable (set TPLA_NCCL_LIB)");
  ncclUniqueId id;
  memcpy(&id, unique_id128, 128);
  ncclComm_t c;
  ncclResult_t r = g_nccl.CommInitRank(&c, world, id, rank);
  if (r != ncclSuccess) return fail(TPLA_ERR_NCCL, "ncclCommInitRank: %s", g_nccl.GetErrorString(r));
  *out = new tpla_comm{c, world, rank};
  return ok();
}

int32_t tpla_decode_kernel_path(const tpla_config* cfg, int32_t B) {
  Geom g{};
  tpla_status st = make_geom(cfg, &g);
  if (st) return -st;
  if ((st = check_kernel_shapes(g))) return -st;
  if (B < 1) return -fail(TPLA_ERR_INVALID_ARG, "B=%d", B);
  ok();
  return use_tc_attention(g, B) ? 1 : 0;
}

tpla_status tpla_comm_enable_fused_allreduce(tpla_comm* comm, int64_t max_elems) {
  if (!comm || max_elems < 1) return fail(TPLA_ERR_INVALID_ARG, "bad arguments");
  if (!load_nccl()) return fail(TPLA_ERR_NCCL, "NCCL not loadable");
  if (!g_nccl.device_api)
    return fail(TPLA_ERR_UNSUPPORTED, "the loaded NCCL has no device API matching %d (symmetric windows, LSA barriers)",
                NCCL_VERSION_CODE);
  if (comm->ar.window) return ok();
  const size_t bytes = 2 * size_t(max_elems) * 4;              // two halves (selected by the barrier epoch)
  void* buf = nullptr;
  ncclResult_t r = g_nccl.MemAlloc(&buf, bytes);
  if (r != ncclSuccess) return fail(TPLA_ERR_NCCL, "ncclMemAlloc: %s", g_nccl.GetErrorString(r));
  TPLA_CUDA(cudaMemset(buf, 0, bytes), "zero symmetric buffer");
  ncclWindow_t win = nullptr;
  r = g_nccl.WinRegister(comm->comm, buf, bytes, &win, NCCL_WIN_COLL_SYMMETRIC);   // (collective)
  if (r != ncclSuccess) {
    g_nccl.MemFree(buf);
    return fail(TPLA_ERR_NCCL, "ncclCommWindowRegister: %s", g_nccl.GetErrorString(r));
  }
  // LSA barriers for the reduce CTAs; the NVLS multicast (lsaMultimem) when the system offers it
  const char* env = getenv("TPLA_FUSED_AR");
  bool want_mm = !(env && strcmp(env, "unicast") == 0);
  ncclDevCommRequirements_t req{};
  req.lsaBarrierCount = kArCtas;
  req.lsaMultimem = want_mm;
  r = g_nccl.DevCommCreate(comm->comm, &req, &comm->dev);       // (collective)
  if (r != ncclSuccess && want_mm) {
    want_mm = false;
    req.lsaMultimem = false;
    r = g_nccl.DevCommCreate(comm->comm, &req, &comm->dev);
  }
  if (r != ncclSuccess) {
    g_nccl.WinDeregister(comm->comm, win);
    g_nccl.MemFree(buf);
    return fail(TPLA_ERR_NCCL, "ncclDevCommCreate: %s", g_nccl.GetErrorString(r));
  }
  comm->sym = buf;
  comm->win = win;
  comm->dev_ok = true;
  comm->ar.dev_comm = &comm->dev;
  comm->ar.window = win;
  comm->ar.half_elems = size_t(max_elems);
  comm->ar.multimem = want_mm && comm->world > 1 ? 1 : 0;
  return ok();
}

int32_t tpla_comm_fused_allreduce_mode(const tpla_comm* comm) {
  if (!comm || !comm->ar.window) return 0;
  return comm->ar.multimem ? 2 : 1;
}

tpla_status tpla_comm_destroy(tpla_comm* comm) {
  if (!comm) return ok();
  if (g_nccl.ok && comm->dev_ok) g_nccl.DevCommDestroy(comm->comm, &comm->dev);
  if (g_nccl.ok && comm->win) g_nccl.WinDeregister(comm->comm, comm->win);
  if (g_nccl.ok && comm->sym) g_nccl.MemFree(comm->sym);
  if (g_nccl.ok) g_nccl.CommDestroy(comm->comm);
  delete comm;
  return ok();
}

tpla_status tpla_sync(void* stream) {
  cudaError_t e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "tpla_sync");
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "tpla_sync");
  return ok();
}

}  // extern "C"
