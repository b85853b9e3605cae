// Shared helpers for the voxvie_b200 CUDA library (sm_100a).
//
// All device arrays are interleaved complex128 (double2).  Every entry point
// of the C-ABI (include/voxvie_b200.h) returns an int status and records a
// thread-local message retrievable with vx_last_error().
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/voxvie_b200.h"

namespace vx {

// ---------------------------------------------------------------- errors
void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* where);

#define VX_CHECK_LAUNCH(where)                                      \
  do {                                                              \
    ::vx::count_launch();                                           \
    cudaError_t _e = cudaGetLastError();                            \
    if (_e != cudaSuccess) return ::vx::cuda_status(_e, where);     \
  } while (0)

#define VX_CUDA(call)                                               \
  do {                                                              \
    cudaError_t _e = (call);                                        \
    if (_e != cudaSuccess) return ::vx::cuda_status(_e, #call);     \
  } while (0)

#define VX_REQUIRE(cond, ...)                                       \
  do {                                                              \
    if (!(cond)) { ::vx::set_error(__VA_ARGS__); return VX_EINVAL; } \
  } while (0)

// ---------------------------------------------------------------- complex
__host__ __device__ __forceinline__ double2 cmk(double a, double b) { return make_double2(a, b); }
__host__ __device__ __forceinline__ double2 cadd(double2 a, double2 b) { return cmk(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ double2 csub(double2 a, double2 b) { return cmk(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return cmk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a * conj(b)
__host__ __device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
  return cmk(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
// conj(a) * b
__host__ __device__ __forceinline__ double2 cconjmul(double2 a, double2 b) {
  return cmk(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__host__ __device__ __forceinline__ double2 cconj(double2 a) { return cmk(a.x, -a.y); }
__host__ __device__ __forceinline__ double2 cscale(double2 a, double s) { return cmk(a.x * s, a.y * s); }
// acc += a * b (fma form)
__host__ __device__ __forceinline__ void cfma(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
// acc -= a * b
__host__ __device__ __forceinline__ void cfms(double2& acc, double2 a, double2 b) {
  acc.x = fma(-a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(-a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
}
// 1/z computed like numpy's complex division (Smith's algorithm)
__host__ __device__ __forceinline__ double2 cinv(double2 z) {
  if (fabs(z.x) >= fabs(z.y)) {
    double r = z.y / z.x, d = z.x + z.y * r;
    return cmk(1.0 / d, -r / d);
  } else {
    double r = z.x / z.y, d = z.x * r + z.y;
    return cmk(r / d, -1.0 / d);
  }
}
// a / b (Smith)
__host__ __device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  if (fabs(b.x) >= fabs(b.y)) {
    double r = b.y / b.x, d = b.x + b.y * r;
    return cmk((a.x + a.y * r) / d, (a.y - a.x * r) / d);
  } else {
    double r = b.x / b.y, d = b.x * r + b.y;
    return cmk((a.x * r + a.y) / d, (a.y * r - a.x) / d);
  }
}

// streaming (read-once) 16-byte load that does not allocate in L1
__device__ __forceinline__ double2 ld_stream(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
               : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}

inline unsigned div_up(long a, long b) { return (unsigned)((a + b - 1) / b); }

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int device_smem_optin();   // max dynamic shared memory per block (bytes)
int device_sm_count();

// runtime.cu: launch accounting and optional event spans (vx_timing_enable)
void count_launch(int n = 1);
struct Span {
  const char* nm;
  cudaStream_t st;
  cudaEvent_t a;
  bool on;
  Span(const char* name, cudaStream_t s);
  ~Span();
};

}  // namespace vx
