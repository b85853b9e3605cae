// Host -> device uploads of pageable host buffers (numpy arrays at the
// reference-facing API: the field vectors and coefficient map a caller of
// apply_n / apply_system / gmres passes, reference operator.py:82-105,
// solver.py:114).  A pageable cudaMemcpy stages through one driver buffer with
// a single host thread (~10 GB/s); here a small persistent pool of host threads
// copies 2 MB chunks into a ring of pinned slots (non-temporal stores) and each
// issues the DMA of its own chunk on the caller's stream, so the host copy runs
// at memory bandwidth and overlaps the PCIe/C2C transfer.  Semantics match cudaMemcpy from
// pageable memory: the call returns once `src` has been consumed; the DMA may
// still be in flight on `stream`.
#include <emmintrin.h>

#include <atomic>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"

namespace vx {
namespace {

constexpr size_t kChunk = size_t(2) << 20;
constexpr int kSlots = 32;

struct Job {
  char* dst;
  const char* src;
  size_t bytes;      // bytes of this round
  long nchunks;
  cudaStream_t stream;
  int device;
  std::atomic<long> next{0};
  std::atomic<int> err{0};
};

struct Pool {
  std::mutex mu;             // serialises callers (one round in flight)
  std::mutex jm;
  std::condition_variable cv, cv_done;
  long gen = 0;
  int inflight = 0;          // workers currently inside a round
  Job* job = nullptr;
  int nthreads = 0;
  char* slot[kSlots] = {};
  cudaEvent_t ev[kSlots] = {};
  bool ready = false;
};

Pool* g_pool = nullptr;
std::once_flag g_once;

// pageable -> pinned slot with non-temporal stores: the slot is read next by
// the DMA engine, not by this core, so the lines need not be fetched for
// ownership nor kept in this core's caches (VX_H2D_NT=0: plain memcpy)
void copy_stream(char* dst, const char* src, size_t n) {
  static const int nt = [] { const char* e = getenv("VX_H2D_NT"); return e ? atoi(e) : 1; }();
  if (!nt || (reinterpret_cast<uintptr_t>(dst) & 15)) { std::memcpy(dst, src, n); return; }
  size_t i = 0;
  for (; i + 64 <= n; i += 64) {
    const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
    const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 16));
    const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 32));
    const __m128i d = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 48));
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), a);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 16), b);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 32), c);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 48), d);
  }
  if (i < n) std::memcpy(dst + i, src + i, n - i);
  _mm_sfence();
}

void run_chunks(Pool* p, Job* j) {
  cudaSetDevice(j->device);
  for (;;) {
    long c = j->next.fetch_add(1);
    if (c >= j->nchunks) break;
    size_t off = size_t(c) * kChunk;
    size_t n = j->bytes - off < kChunk ? j->bytes - off : kChunk;
    // the slot's previous DMA (an earlier round or call) must have drained
    if (cudaEventSynchronize(p->ev[c]) != cudaSuccess) { j->err = 1; continue; }
    copy_stream(p->slot[c], j->src + off, n);
    if (cudaMemcpyAsync(j->dst + off, p->slot[c], n, cudaMemcpyHostToDevice, j->stream) != cudaSuccess ||
        cudaEventRecord(p->ev[c], j->stream) != cudaSuccess)
      j->err = 1;
  }
}

void worker(Pool* p) {
  long seen = 0;
  for (;;) {
    Job* j;
    {
      std::unique_lock<std::mutex> lk(p->jm);
      p->cv.wait(lk, [&] { return p->gen != seen; });
      seen = p->gen;
      j = p->job;            // null once the caller has finished the round
      if (!j) continue;
      ++p->inflight;
    }
    run_chunks(p, j);
    std::lock_guard<std::mutex> lk(p->jm);
    if (--p->inflight == 0) p->cv_done.notify_all();
  }
}

int init_pool() {
  std::call_once(g_once, [] {
    Pool* p = new Pool();  // never destroyed: workers are detached
    unsigned hc = std::thread::hardware_concurrency();
    // a few helpers saturate the copy; more contend with the launching thread
    // (c1 e2e per solve: 3 helpers 32.0 ms, 7: 32.3, 11: 33.6, 15: 34.2)
    int n = hc > 2 ? int(hc) / 2 : 1;
    if (n > 4) n = 4;
    if (const char* e = getenv("VX_H2D_THREADS")) n = atoi(e);
    if (n > 15) n = 15;
    if (n < 0) n = 0;
    p->nthreads = n;
    bool ok = true;
    for (int s = 0; s < kSlots && ok; ++s) {
      ok = cudaHostAlloc(reinterpret_cast<void**>(&p->slot[s]), kChunk, cudaHostAllocPortable) == cudaSuccess &&
           cudaEventCreateWithFlags(&p->ev[s], cudaEventDisableTiming) == cudaSuccess;
    }
    if (!ok) { g_pool = p; return; }
    for (int t = 0; t < n; ++t) std::thread(worker, p).detach();
    p->ready = true;
    g_pool = p;
  });
  return g_pool && g_pool->ready ? VX_OK : VX_ECUDA;
}

}  // namespace
}  // namespace vx

extern "C" int vx_h2d_staged(void* dst, const void* src, size_t bytes, void* stream) {
  using namespace vx;
  if (bytes == 0) return VX_OK;
  if (!dst || !src) { set_error("vx_h2d_staged: null pointer"); return VX_EINVAL; }
  if (init_pool() != VX_OK) { set_error("vx_h2d_staged: pinned staging allocation failed"); return VX_ECUDA; }
  Pool* p = g_pool;
  int dev = 0;
  VX_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> call_lock(p->mu);
  const size_t round_bytes = kChunk * kSlots;
  int err = 0;
  for (size_t off = 0; off < bytes; off += round_bytes) {
    Job j;
    j.dst = static_cast<char*>(dst) + off;
    j.src = static_cast<const char*>(src) + off;
    j.bytes = bytes - off < round_bytes ? bytes - off : round_bytes;
    j.nchunks = long((j.bytes + kChunk - 1) / kChunk);
    j.stream = static_cast<cudaStream_t>(stream);
    j.device = dev;
    // helpers claim chunks dynamically; the caller never waits for a worker
    // to wake up, only for the ones that joined this round to leave it
    bool wake = p->nthreads > 0 && j.nchunks > 1;
    if (wake) {
      std::lock_guard<std::mutex> lk(p->jm);
      p->job = &j;
      ++p->gen;
      p->cv.notify_all();
    }
    run_chunks(p, &j);
    if (wake) {
      std::unique_lock<std::mutex> lk(p->jm);
      p->job = nullptr;
      p->cv_done.wait(lk, [&] { return p->inflight == 0; });
    }
    err |= j.err.load();
  }
  if (err) { set_error("vx_h2d_staged: cudaMemcpyAsync/event failure"); return VX_ECUDA; }
  return VX_OK;
}

extern "C" int vx_h2d_threads(void) {
  using namespace vx;
  return init_pool() == VX_OK ? g_pool->nthreads + 1 : 0;
}

// Pinned host blocks for device -> host results (the Python side pools them
// and hands them out as numpy arrays, so a result copy never page-faults a
// fresh allocation).
extern "C" int vx_host_alloc(size_t bytes, void** out) {
  VX_CUDA(cudaHostAlloc(out, bytes, cudaHostAllocPortable));
  return VX_OK;
}

extern "C" int vx_host_free(void* p) {
  VX_CUDA(cudaFreeHost(p));
  return VX_OK;
}

// Device -> pinned host copy on `stream`, synchronous (returns with the data).
extern "C" int vx_d2h_pinned(void* dst, const void* src, size_t bytes, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  VX_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
  VX_CUDA(cudaStreamSynchronize(s));
  return VX_OK;
}

// the same copy without the final synchronisation: the caller overlaps it with
// work on another stream and synchronises `stream` before reading dst
extern "C" int vx_d2h_pinned_async(void* dst, const void* src, size_t bytes, void* stream) {
  VX_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream)));
  return VX_OK;
}

