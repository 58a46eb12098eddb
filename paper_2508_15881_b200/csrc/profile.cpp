// Launch counting and optional per-kernel device timing (tpla_profile_* in include/tpla.h).
//
// When enabled, every kernel launch of the library is bracketed by two CUDA events recorded
// on the launching stream, so bench.py can attribute device time to each kernel live inside
// its timed region (the events add no device work between the kernels).
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>
#include <string>
#include <vector>

#include "internal.h"

namespace tpla {

std::atomic<int> g_profile_on{0};
thread_local bool g_no_pdl_next = false;

namespace {
struct Pending {
  std::string name;
  cudaEvent_t start, stop;
};
struct Acc {
  std::string name;
  double ms = 0;
  int64_t launches = 0;
};
std::mutex g_mu;
std::vector<Pending> g_pending;
std::vector<cudaEvent_t> g_free;
std::vector<Acc> g_acc;

// Under stream capture the record must be an external event node (so the graph records a
// timestamp); outside capture the flag is not valid and a plain record is used.
void record(cudaEvent_t e, cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &st);
  if (st == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
  else cudaEventRecord(e, s);
}

cudaEvent_t take_event() {
  if (!g_free.empty()) {
    cudaEvent_t e = g_free.back();
    g_free.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("TPLA_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

KernelScope::KernelScope(const char* name, cudaStream_t s) : stream(s), name_(name) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  const int mode = g_profile_on.load(std::memory_order_relaxed);
  if (!mode || (mode == 2 && strncmp(name, "K3", 2) != 0)) return;   // mode 2: the attention kernel only
  std::lock_guard<std::mutex> lk(g_mu);
  Pending p{name, take_event(), take_event()};
  record(p.start, s);
  g_pending.push_back(p);
  slot = static_cast<int>(g_pending.size()) - 1;
}

KernelScope::~KernelScope() {
  static const bool debug_sync = getenv("TPLA_DEBUG_SYNC") != nullptr;
  if (debug_sync) {
    // diagnostic mode: run every launch to completion and name the kernel that faulted
    if (getenv("TPLA_DEBUG_SYNC")[0] == '2') fprintf(stderr, "[tpla] sync after %s\n", name_);
    cudaError_t e = cudaStreamSynchronize(stream);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) fprintf(stderr, "[tpla] kernel %s failed: %s\n", name_, cudaGetErrorString(e));
  }
  if (slot < 0) return;
  std::lock_guard<std::mutex> lk(g_mu);
  if (slot < static_cast<int>(g_pending.size())) record(g_pending[slot].stop, stream);
}

}  // namespace tpla

using namespace tpla;

extern "C" {

tpla_status tpla_profile_enable(int32_t on) {
  g_profile_on.store(on == 2 ? 2 : (on ? 1 : 0));
  return TPLA_OK;
}

tpla_status tpla_profile_collect(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto& p : g_pending) {
    if (cudaEventSynchronize(p.stop) != cudaSuccess) return TPLA_ERR_CUDA;
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, p.start, p.stop) != cudaSuccess) return TPLA_ERR_CUDA;
    Acc* a = nullptr;
    for (auto& x : g_acc)
      if (x.name == p.name) a = &x;
    if (!a) {
      g_acc.push_back(Acc{p.name});
      a = &g_acc.back();
    }
    a->ms += ms;
    a->launches += 1;
    g_free.push_back(p.start);
    g_free.push_back(p.stop);
  }
  g_pending.clear();
  return TPLA_OK;
}

int32_t tpla_profile_count(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  return static_cast<int32_t>(g_acc.size());
}

tpla_status tpla_profile_get(int32_t i, char* name64, double* total_ms, int64_t* launches) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (i < 0 || i >= static_cast<int32_t>(g_acc.size()) || !name64) return TPLA_ERR_INVALID_ARG;
  strncpy(name64, g_acc[i].name.c_str(), 63);
  name64[63] = 0;
  if (total_ms) *total_ms = g_acc[i].ms;
  if (launches) *launches = g_acc[i].launches;
  return TPLA_OK;
}

tpla_status tpla_profile_reset(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto& p : g_pending) {
    cudaEventSynchronize(p.stop);
    g_free.push_back(p.start);
    g_free.push_back(p.stop);
  }
  g_pending.clear();
  g_acc.clear();
  return TPLA_OK;
}

}  // extern "C"
