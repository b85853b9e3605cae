// Library runtime services: launch counter and named CUDA-event spans used by
// bench.py to time individual kernels live, on the stream they run on.
#include <atomic>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace vx {

static std::atomic<long> g_launches{0};
static std::atomic<int> g_timing{0};

struct SpanLog {
  std::string name;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
};
static std::mutex g_tmu;
static std::vector<SpanLog> g_spans;
static std::vector<cudaEvent_t> g_evpool;  // recycled span events (creation is a driver call)

static cudaEvent_t ev_get() {
  {
    std::lock_guard<std::mutex> lock(g_tmu);
    if (!g_evpool.empty()) {
      cudaEvent_t e = g_evpool.back();
      g_evpool.pop_back();
      return e;
    }
  }
  cudaEvent_t e = nullptr;
  if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
  return e;
}

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// names of the spans open on this thread: a span nested inside one of the
// same name (an entry point that times its whole solve phase around helpers
// that time their own) records nothing, so each phase is counted once
static thread_local std::vector<const char*> t_open;

Span::Span(const char* name, cudaStream_t s) : nm(name), st(s), a(nullptr), on(g_timing.load() != 0) {
  if (!on) return;
  for (const char* o : t_open)
    if (std::strcmp(o, name) == 0) { on = false; return; }
  a = ev_get();
  if (!a) { on = false; return; }
  cudaEventRecord(a, st);
  t_open.push_back(nm);
}

Span::~Span() {
  if (!on) return;
  if (!t_open.empty()) t_open.pop_back();
  cudaEvent_t b = ev_get();
  if (!b) return;
  cudaEventRecord(b, st);
  std::lock_guard<std::mutex> lock(g_tmu);
  for (auto& s : g_spans)
    if (s.name == nm) { s.ev.emplace_back(a, b); return; }
  g_spans.push_back(SpanLog{nm, {{a, b}}});
}

}  // namespace vx

extern "C" long vx_launch_count(void) { return vx::g_launches.load(); }

extern "C" int vx_timing_enable(int on) {
  vx::g_timing.store(on ? 1 : 0);
  return VX_OK;
}

extern "C" int vx_timing_read(const char* span, double* total_ms, long* count) {
  std::lock_guard<std::mutex> lock(vx::g_tmu);
  *total_ms = 0.0;
  *count = 0;
  for (auto& s : vx::g_spans) {
    if (s.name != span) continue;
    for (auto& e : s.ev) {
      float ms = 0.f;
      VX_CUDA(cudaEventSynchronize(e.second));
      VX_CUDA(cudaEventElapsedTime(&ms, e.first, e.second));
      *total_ms += ms;
      *count += 1;
      vx::g_evpool.push_back(e.first);
      vx::g_evpool.push_back(e.second);
    }
    s.ev.clear();
  }
  return VX_OK;
}
