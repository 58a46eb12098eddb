// K6 — page tables of the prefill-as-prefixes decomposition (tpla_prefill_attention).
//
// The causal prefill attention of one prompt (in PD separation the prompt is attended
// with MLA, g = 1, and its rows are stored with the full RMS) is the multi-token decode
// (K2..K5) over pseudo-sequences: pseudo-sequence j holds the n_q prompt tokens
// [r0 + j·n_q, r0 + (j+1)·n_q) as its newest tokens and attends causally to the first
// r0 + (j+1)·n_q cached rows — all pseudo-sequences share the prompt's pages.  This kernel writes
// their page-table rows (copies of the prompt's row) and lengths.  The decode launch that follows
// runs without PDL (tpla_prefill_attention): K3 reads the tables before its griddepcontrol.wait.
#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace tpla {
namespace {

__global__ void prefix_table_kernel(const int32_t* __restrict__ block_table, int seq, int max_pages, int n_full,
                                    int n_q, int r0, int n_rows, int32_t* __restrict__ table,
                                    int32_t* __restrict__ lens) {
  pdl_trigger();
  pdl_wait();   // the previous call's K3 may still read this region (write-after-read)
  const int n_seq = n_full + (n_rows > n_full * n_q ? 1 : 0);
  const int32_t* src = block_table + long(seq) * max_pages;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_seq * max_pages; i += gridDim.x * blockDim.x)
    table[i] = src[i % max_pages];
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n_seq; j += gridDim.x * blockDim.x)
    lens[j] = j < n_full ? r0 + (j + 1) * n_q : r0 + n_rows;
}

}  // namespace

cudaError_t launch_prefix_table(const int32_t* block_table, int seq, int max_pages, int n_full, int n_q, int r0,
                                int n_rows, int32_t* table, int32_t* lens, cudaStream_t s) {
  const int n = (n_full + 1) * max_pages;
  const int blocks = std::max(1, std::min(64, (n + 255) / 256));
  KernelScope ks("K6_prefix_table", s);
  return launch_k(prefix_table_kernel, blocks, 256, 0, s, block_table, seq, max_pages, n_full, n_q, r0, n_rows, table,
                  lens);
}

}  // namespace tpla
