// profile.cu -- optional per-kernel CUDA-event timing (nw_profile_begin/end) and
// the launch counter; used by bench.py for the roofline's per-kernel durations.
#include <cstring>
#include <mutex>
#include <vector>

#include <cstdio>
#include <cstdlib>

#include "nw_internal.h"

namespace nw {

namespace {
struct Rec {
  const char *kind;
  cudaEvent_t a, b;
};
std::mutex g_mu;
bool g_on = false;
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;

cudaEvent_t get_event() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

LaunchScope::LaunchScope(const char *kind, cudaStream_t s) : kind_(kind), s_(s) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_on) return;
  a_ = get_event();
  b_ = get_event();
  cudaEventRecord(a_, s_);
}

// NW_DEBUG_SYNC=1 (diagnostics only): synchronise after every library launch and name the
// kernel kind on stderr if it faulted.
static bool debug_sync() {
  static const bool on = [] {
    const char *v = getenv("NW_DEBUG_SYNC");
    return v && atoi(v) != 0;
  }();
  return on;
}

LaunchScope::~LaunchScope() {
  if (debug_sync()) {
    const cudaError_t e = cudaStreamSynchronize(s_);
    if (e != cudaSuccess) fprintf(stderr, "[nw] kernel %s: %s\n", kind_, cudaGetErrorString(e));
  }
  if (!a_) return;
  cudaEventRecord(b_, s_);
  std::lock_guard<std::mutex> lk(g_mu);
  g_recs.push_back({kind_, a_, b_});
}

}  // namespace nw

using namespace nw;

extern "C" {

nw_status_t nw_profile_begin(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto &r : g_recs) {
    g_pool.push_back(r.a);
    g_pool.push_back(r.b);
  }
  g_recs.clear();
  g_on = true;
  return NW_OK;
}

nw_status_t nw_profile_end(const char **names, unsigned long long *launches, double *ms, size_t cap, size_t *n) {
  if (!n) return NW_ERR_INVALID;
  std::lock_guard<std::mutex> lk(g_mu);
  g_on = false;
  std::vector<const char *> kinds;
  std::vector<unsigned long long> cnt;
  std::vector<double> tot;
  for (auto &r : g_recs) {
    if (cudaEventSynchronize(r.b) != cudaSuccess) return NW_ERR_CUDA;
    float t = 0.f;
    if (cudaEventElapsedTime(&t, r.a, r.b) != cudaSuccess) return NW_ERR_CUDA;
    size_t k = 0;
    for (; k < kinds.size(); ++k)
      if (std::strcmp(kinds[k], r.kind) == 0) break;
    if (k == kinds.size()) {
      kinds.push_back(r.kind);
      cnt.push_back(0);
      tot.push_back(0.0);
    }
    cnt[k] += 1;
    tot[k] += t;
  }
  *n = kinds.size();
  for (size_t k = 0; k < kinds.size() && k < cap; ++k) {
    if (names) names[k] = kinds[k];
    if (launches) launches[k] = cnt[k];
    if (ms) ms[k] = tot[k];
  }
  return NW_OK;
}

}  // extern "C"
