// prof.cu — opt-in kernel timing.  When enabled (masq_profile_enable), every kernel launch of
// the library is bracketed by a cudaEvent pair recorded on the launching stream; the durations
// are aggregated per kernel name by masq_profile_collect.  This is the only process-global
// state in the library and it is off by default.  Launches inside a CUDA-graph capture record
// their pairs as graph nodes (the pool is pre-filled), so each replay re-times them and a
// collect after replays reports the last replay.
#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "internal.h"

namespace masq {
namespace {
struct Rec {
  const char* name;
  cudaEvent_t a, b;
  int launches;
};
std::mutex g_mu;
bool g_on = false;
std::string g_only;                     // non-empty: record only the scopes of this name
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

namespace {
// inside a stream capture the record must be an external event node to stay timeable at replay
void record(cudaEvent_t e, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(e, st, cudaEventRecordExternal);
  else
    cudaEventRecord(e, st);
}
}  // namespace

ProfScope::ProfScope(const char* name, cudaStream_t st, int launches) : name_(name), st_(st), launches_(launches) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_on || (!g_only.empty() && g_only != name)) return;
  a_ = get_event();
  if (a_) record(static_cast<cudaEvent_t>(a_), st_);
}

ProfScope::~ProfScope() {
  if (!a_) return;
  std::lock_guard<std::mutex> lk(g_mu);
  cudaEvent_t b = get_event();
  if (!b) return;
  record(b, st_);
  g_recs.push_back(Rec{name_, static_cast<cudaEvent_t>(a_), b, launches_});
}

}  // namespace masq

using namespace masq;

extern "C" {

int32_t masq_profile_enable(int32_t on) {
  std::lock_guard<std::mutex> lk(g_mu);
  const int32_t prev = g_on ? 1 : 0;
  g_on = on != 0;
  for (auto& r : g_recs) { g_pool.push_back(r.a); g_pool.push_back(r.b); }
  g_recs.clear();
  // pre-create the events so that launches recorded inside a CUDA-graph capture never need
  // cudaEventCreate (not a capturable call); the records then become graph nodes
  while (g_on && g_pool.size() < 2048) {
    cudaEvent_t e = nullptr;
    if (cudaEventCreate(&e) != cudaSuccess) break;
    g_pool.push_back(e);
  }
  return prev;
}

int32_t masq_profile_only(const char* name) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_only = name ? name : "";
  return 0;
}

int32_t masq_profile_collect(int32_t max_entries, char* names, double* total_ms, int64_t* launches) {
  std::lock_guard<std::mutex> lk(g_mu);
  std::vector<std::string> keys;
  std::vector<double> ms;
  std::vector<int64_t> cnt;
  int failed = 0;
  for (auto& r : g_recs) {
    float t = 0.f;
    if (cudaEventSynchronize(r.b) != cudaSuccess || cudaEventElapsedTime(&t, r.a, r.b) != cudaSuccess) {
      cudaGetLastError();                           // do not leave a sticky error for the caller
      ++failed;
      continue;
    }
    size_t k = 0;
    while (k < keys.size() && keys[k] != r.name) ++k;
    if (k == keys.size()) { keys.emplace_back(r.name); ms.push_back(0.0); cnt.push_back(0); }
    ms[k] += t;
    cnt[k] += r.launches;
    g_pool.push_back(r.a);
    g_pool.push_back(r.b);
  }
  g_recs.clear();
  if (failed && keys.empty()) return -1;
  const int32_t n = (int32_t)std::min<size_t>(keys.size(), (size_t)std::max(max_entries, 0));
  for (int32_t i = 0; i < n; ++i) {
    if (names) {
      std::memset(names + 32 * i, 0, 32);
      std::strncpy(names + 32 * i, keys[i].c_str(), 31);
    }
    if (total_ms) total_ms[i] = ms[i];
    if (launches) launches[i] = cnt[i];
  }
  return n;
}

}  // extern "C"
