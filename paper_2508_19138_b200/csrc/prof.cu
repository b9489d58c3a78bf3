// CUDA-event profiler (see prof.cuh). Each begin/end pair records two events
// on the launching stream, so the measured span is exactly the device time
// of the bracketed kernel(s) in stream order.
#include <atomic>
#include <mutex>
#include <vector>

#include "../../include/negf_b200.h"
#include "prof.cuh"

namespace negf {
namespace {

struct Rec {
  int cls;
  cudaEvent_t a, b;
  double flops, bytes;
  bool closed;
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
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

}  // namespace

namespace {
std::atomic<long long> g_launch_count{0};
}
void count_launch() { g_launch_count.fetch_add(1, std::memory_order_relaxed); }

bool prof_enabled() { return g_on; }

int prof_begin(int cls, cudaStream_t st) {
  if (!g_on) return -1;
  std::lock_guard<std::mutex> lk(g_mu);
  Rec r;
  r.cls = cls;
  r.a = get_event();
  r.b = get_event();
  r.flops = r.bytes = 0.0;
  r.closed = false;
  cudaEventRecord(r.a, st);
  g_recs.push_back(r);
  return (int)g_recs.size() - 1;
}

void prof_end(int token, cudaStream_t st, double flops, double bytes) {
  if (token < 0) return;
  std::lock_guard<std::mutex> lk(g_mu);
  if (token >= (int)g_recs.size()) return;
  Rec& r = g_recs[token];
  cudaEventRecord(r.b, st);
  r.flops = flops;
  r.bytes = bytes;
  r.closed = true;
}

}  // namespace negf

using namespace negf;

extern "C" {

long long negf_launch_count(void) { return g_launch_count.load(std::memory_order_relaxed); }

void negf_prof_enable(int on) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_on = on != 0;
}

void negf_prof_reset(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto& r : g_recs) {
    g_pool.push_back(r.a);
    g_pool.push_back(r.b);
  }
  g_recs.clear();
}

int negf_prof_query(int cls, double* ms, double* flops, double* bytes, long long* launches) {
  std::lock_guard<std::mutex> lk(g_mu);
  double t = 0.0, f = 0.0, by = 0.0;
  long long n = 0;
  for (auto& r : g_recs) {
    if (r.cls != cls || !r.closed) continue;
    cudaError_t e = cudaEventSynchronize(r.b);
    if (e != cudaSuccess) return (int)e;
    float x = 0.f;
    cudaEventElapsedTime(&x, r.a, r.b);
    t += x;
    f += r.flops;
    by += r.bytes;
    ++n;
  }
  if (ms) *ms = t;
  if (flops) *flops = f;
  if (bytes) *bytes = by;
  if (launches) *launches = n;
  return 0;
}

}  // extern "C"
