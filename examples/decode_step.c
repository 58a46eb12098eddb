/*
 * decode_step.c — one TPLA decode step through the C ABI alone (no Python, no PyTorch).
 *
 * A DeepSeek-V3-shaped layer cut to 16 query heads (d_c 512, d_r 64, d_h 128, D 1024) on k = 2
 * devices with g = 2 latent groups (§4.4), both ranks held by this process on one
 * GPU (rank 1 accumulates into rank 0's y, as tpla_decode documents).  Per rank:
 *   tpla_convert_weights (host fp64 -> device bf16, Hadamard transform)   §4.3
 *   tpla_append_kv       prompt rows EXACT, the new token SLICED
 *   tpla_decode          K2..K5 on the tcgen05 path
 * Checks: every call returns TPLA_OK; y is finite and replays bit-identically; a bad argument is
 * rejected before any launch (the launch counter does not move).  Prints "decode_step OK".
 *
 * Build (tests/test_abi_host.py does this): gcc -std=c99 -Iinclude examples/decode_step.c
 *   -Lpaper_2508_15881_b200 -ltpla -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,... -lm
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "tpla.h"

#define CK(x)                                                                             \
  do {                                                                                    \
    tpla_status st_ = (x);                                                                \
    if (st_ != TPLA_OK) {                                                                 \
      fprintf(stderr, "%s:%d: %s -> %d (%s)\n", __FILE__, __LINE__, #x, st_, tpla_last_error()); \
      exit(1);                                                                            \
    }                                                                                     \
  } while (0)
#define CU(x)                                                                             \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess) {                                                              \
      fprintf(stderr, "%s:%d: %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                            \
    }                                                                                     \
  } while (0)

static uint64_t rng = 0x9E3779B97F4A7C15ull;
static float urand(void) { /* xorshift64*, uniform in [-1, 1) */
  rng ^= rng >> 12; rng ^= rng << 25; rng ^= rng >> 27;
  return (float)((rng * 0x2545F4914F6CDD1Dull) >> 40) / (float)(1 << 23) - 1.0f;
}
static uint16_t bf16(float x) { /* round to nearest even */
  uint32_t u;
  memcpy(&u, &x, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
static uint16_t* host_bf16(size_t n, float scale) {
  uint16_t* p = (uint16_t*)malloc(n * 2);
  for (size_t i = 0; i < n; ++i) p[i] = bf16(scale * urand());
  return p;
}
static void* dev_copy(const void* h, size_t bytes) {
  void* d = NULL;
  CU(cudaMalloc(&d, bytes));
  CU(cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice));
  return d;
}

int main(void) {
  enum { H = 16, DC = 512, DR = 64, DH = 128, DM = 1024, K = 2, G = 2, B = 4, S = 300, PAGE = 64 };
  const int max_pages = (S + PAGE - 1) / PAGE;
  printf("%s\n", tpla_version());

  /* layer weights (host bf16, synthetic) */
  uint16_t* W_UK = host_bf16((size_t)DC * H * DH, 0.05f);
  uint16_t* W_UV = host_bf16((size_t)DC * H * DH, 0.05f);
  uint16_t* W_O = host_bf16((size_t)H * DH * DM, 0.02f);
  uint16_t* gamma = (uint16_t*)malloc(DC * 2);
  for (int i = 0; i < DC; ++i) gamma[i] = bf16(1.0f + 0.1f * urand());
  const float alpha[G] = {2.0f, 2.0f}, mu[G] = {2.0f, 2.0f}; /* Hadamard: alpha_j = g, mu_j = alpha_j */

  /* per-step inputs: B sequences of S tokens (S - 1 prompt rows + the new token), queries */
  uint16_t* c_kv = host_bf16((size_t)B * S * DC, 1.0f);
  uint16_t* k_pe = host_bf16((size_t)B * S * DR, 1.0f);
  int32_t* seq = (int32_t*)malloc(sizeof(int32_t) * B * S);
  int32_t* pos = (int32_t*)malloc(sizeof(int32_t) * B * S);
  for (int b = 0; b < B; ++b)
    for (int t = 0; t < S; ++t) { seq[b * S + t] = b; pos[b * S + t] = t; }
  uint16_t* q_nope = host_bf16((size_t)B * H * DH, 1.0f);
  uint16_t* q_pe = host_bf16((size_t)B * H * DR, 1.0f);
  int32_t lens[B], table[B * max_pages];
  for (int b = 0; b < B; ++b) lens[b] = S;
  for (int i = 0; i < B * max_pages; ++i) table[i] = i;

  void *d_ckv = dev_copy(c_kv, (size_t)B * S * DC * 2), *d_kpe = dev_copy(k_pe, (size_t)B * S * DR * 2);
  int32_t *d_seq = (int32_t*)dev_copy(seq, sizeof(int32_t) * B * S), *d_pos = (int32_t*)dev_copy(pos, sizeof(int32_t) * B * S);
  void *d_q = dev_copy(q_nope, (size_t)B * H * DH * 2), *d_qpe = dev_copy(q_pe, (size_t)B * H * DR * 2);
  int32_t *d_lens = (int32_t*)dev_copy(lens, sizeof lens), *d_table = (int32_t*)dev_copy(table, sizeof table);
  float* d_y = NULL;
  void* d_out = NULL;
  CU(cudaMalloc((void**)&d_y, sizeof(float) * B * DM));
  CU(cudaMalloc(&d_out, (size_t)B * DM * 2));

  tpla_config cfg[K];
  tpla_weights w[K];
  tpla_cache cache[K];
  void* ws[K];
  size_t ws_bytes[K];
  for (int r = 0; r < K; ++r) {
    tpla_config c = {H, DC, DR, DH, DM, K, G, r, 1e-6f, 1.0f / sqrtf((float)(DH + DR))};
    cfg[r] = c;
    tpla_device_plan p;
    CK(tpla_make_plan(&cfg[r], &p));
    size_t b_uk, b_uv, b_o, b_x;
    CK(tpla_weights_bytes(&cfg[r], TPLA_XFORM_HADAMARD, &b_uk, &b_uv, &b_o, &b_x));
    memset(&w[r], 0, sizeof w[r]);
    CU(cudaMalloc(&w[r].W_UK, b_uk));
    CU(cudaMalloc(&w[r].W_UV, b_uv));
    CU(cudaMalloc(&w[r].W_O, b_o));
    CU(cudaMalloc(&w[r].xform, b_x));
    CK(tpla_convert_weights(&cfg[r], TPLA_XFORM_HADAMARD, 1234, NULL, alpha, mu, W_UK, W_UV, gamma, W_O,
                            &w[r], NULL));
    /* paged cache: row = [ĉ_j (W_lat) ‖ k^PE (d_r)], stride a multiple of 64, zero-filled pages */
    const int row_stride = (p.row_width + 63) / 64 * 64;
    memset(&cache[r], 0, sizeof cache[r]);
    CU(cudaMalloc(&cache[r].base, (size_t)B * max_pages * PAGE * row_stride * 2));
    CU(cudaMemset(cache[r].base, 0, (size_t)B * max_pages * PAGE * row_stride * 2));
    cache[r].block_table = d_table;
    cache[r].num_pages = B * max_pages;
    cache[r].page_size = PAGE;
    cache[r].max_pages_per_seq = max_pages;
    cache[r].row_stride = row_stride;
    cache[r].batch = B;
    /* prompt rows with the full RMS (PD-separated prefill), then each sequence's new token sliced */
    for (int b = 0; b < B; ++b) {
      const size_t o = (size_t)b * S;
      CK(tpla_append_kv(&cfg[r], &w[r], &cache[r], (uint16_t*)d_ckv + o * DC, (uint16_t*)d_kpe + o * DR, d_seq + o,
                        d_pos + o, S - 1, TPLA_RMS_EXACT, NULL, NULL));
      CK(tpla_append_kv(&cfg[r], &w[r], &cache[r], (uint16_t*)d_ckv + (o + S - 1) * DC,
                        (uint16_t*)d_kpe + (o + S - 1) * DR, d_seq + o + S - 1, d_pos + o + S - 1, 1,
                        TPLA_RMS_SLICED, NULL, NULL));
    }
    CK(tpla_decode_workspace_bytes(&cfg[r], B, S, &ws_bytes[r]));
    CU(cudaMalloc(&ws[r], ws_bytes[r]));
  }
  printf("K3 path: %d (1 = tcgen05)\n", tpla_decode_kernel_path(&cfg[0], B));

  /* the step: rank 0 writes y, rank 1 accumulates and writes the bf16 output */
  float* y[2];
  for (int rep = 0; rep < 2; ++rep) {
    for (int r = 0; r < K; ++r)
      CK(tpla_decode(&cfg[r], &w[r], &cache[r], d_q, d_qpe, d_lens, B, S, ws[r], ws_bytes[r], d_y,
                     r == K - 1 ? d_out : NULL, r ? TPLA_DECODE_ACCUMULATE : 0, NULL, NULL));
    CK(tpla_sync(NULL));
    y[rep] = (float*)malloc(sizeof(float) * B * DM);
    CU(cudaMemcpy(y[rep], d_y, sizeof(float) * B * DM, cudaMemcpyDeviceToHost));
  }
  double norm = 0.0;
  for (int i = 0; i < B * DM; ++i) {
    if (!isfinite(y[0][i])) { fprintf(stderr, "non-finite y[%d]\n", i); return 1; }
    norm += (double)y[0][i] * y[0][i];
  }
  if (memcmp(y[0], y[1], sizeof(float) * B * DM) != 0) { fprintf(stderr, "replay differs\n"); return 1; }

  /* validation happens before any launch: a zero batch is rejected and launches nothing */
  const int64_t n0 = tpla_launch_count();
  if (tpla_decode(&cfg[0], &w[0], &cache[0], d_q, d_qpe, d_lens, 0, S, ws[0], ws_bytes[0], d_y, NULL, 0, NULL, NULL) ==
          TPLA_OK ||
      tpla_launch_count() != n0) {
    fprintf(stderr, "B = 0 accepted\n");
    return 1;
  }
  printf("rejected B=0: %s\n", tpla_last_error());
  printf("decode_step OK: |y| = %.6e, %lld launches\n", sqrt(norm), (long long)tpla_launch_count());
  return 0;
}
