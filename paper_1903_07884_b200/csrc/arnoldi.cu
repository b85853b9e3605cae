// Arnoldi orthogonalisation and vector kernels for the device-resident GMRES
// (reference solver.py:45-111).
//
// The reference uses modified Gram-Schmidt with one DGKS re-orthogonalisation
// pass when ||w1|| < 0.7071 ||w0||.  Here each pass is classical Gram-Schmidt
// (one multi-dot sweep over the basis, one multi-axpy sweep): mathematically
// identical, 2 streaming passes over V instead of j+1 dependent ones.  The
// DGKS decision is taken on the device (flag in `stats`), so the conditional
// second pass costs two early-exit launches and no host round trip.
// All reductions are two-stage with a fixed order (per-CTA partials, then one
// CTA summing them in index order): results are bitwise reproducible.
#include "common.cuh"

#include <cstdlib>

namespace vx {

constexpr int AR_THREADS = 256;

// one resident wave of the dots / update kernels (3 CTAs of 256 per SM)
static int ar_grid(long n) {
  long g = (n + 2047) / 2048;
  const long cap = 3L * device_sm_count();
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

__device__ __forceinline__ double2 warp_sum(double2 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_down_sync(0xffffffffu, v.x, o);
    v.y += __shfl_down_sync(0xffffffffu, v.y, o);
  }
  return v;
}

// CTA-wide sum in fixed order; result valid in thread 0.
__device__ __forceinline__ double2 block_sum(double2 v, double2* sh) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double2 r = cmk(0.0, 0.0);
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = cadd(r, sh[w]);
  return r;
}

__device__ __forceinline__ void chunk(long n, long& beg, long& end) {
  const long per = (n + gridDim.x - 1) / gridDim.x;
  beg = (long)blockIdx.x * per;
  end = beg + per < n ? beg + per : n;
}

// part[i*G + b] = sum_{e in chunk b} conj(V_i[e]) w[e], i < nvec; part[nvec*G+b] = ||w||^2
// Each thread takes two elements per step and a group of AR_DG basis vectors:
// 2 + 2*AR_DG independent 16-byte loads in flight per thread; the grid is one
// resident wave (ar_grid), so there is no tail.  ||w||^2 is accumulated in the
// first group's sweep.
constexpr int AR_DG = 8;
constexpr int AR_UG = 4;  // update: basis vectors per load group (register budget)

__global__ void __launch_bounds__(AR_THREADS, 3) dots_kernel(long n, int nvec, const double2* __restrict__ V,
                                                             long ldv, const double2* __restrict__ w,
                                                             double2* __restrict__ part,
                                                             const double* cond) {
  if (cond && cond[2] == 0.0) return;
  __shared__ double2 sh[AR_THREADS / 32];
  long beg, end;
  chunk(n, beg, end);
  const int G = gridDim.x;
  double nrm = 0.0;
  for (int i0 = 0; i0 < (nvec > 0 ? nvec : 1); i0 += AR_DG) {
    double2 acc[AR_DG];
#pragma unroll
    for (int g = 0; g < AR_DG; ++g) acc[g] = cmk(0.0, 0.0);
    for (long e = beg + threadIdx.x; e < end; e += 2 * AR_THREADS) {
      const long e2 = e + AR_THREADS;
      const bool has2 = e2 < end;
      const double2 x0 = w[e];
      const double2 x1 = has2 ? w[e2] : cmk(0.0, 0.0);
      if (i0 == 0) {
        nrm = fma(x0.x, x0.x, nrm);
        nrm = fma(x0.y, x0.y, nrm);
        nrm = fma(x1.x, x1.x, nrm);
        nrm = fma(x1.y, x1.y, nrm);
      }
      double2 v0[AR_DG], v1[AR_DG];
#pragma unroll
      for (int g = 0; g < AR_DG; ++g) {
        const bool ok = i0 + g < nvec;
        const double2* vp = V + (long)(i0 + g) * ldv;
        v0[g] = ok ? ld_stream(vp + e) : cmk(0.0, 0.0);
        v1[g] = (ok && has2) ? ld_stream(vp + e2) : cmk(0.0, 0.0);
      }
#pragma unroll
      for (int g = 0; g < AR_DG; ++g) {  // conj(v) * x
        acc[g].x = fma(v0[g].x, x0.x, acc[g].x);
        acc[g].x = fma(v0[g].y, x0.y, acc[g].x);
        acc[g].y = fma(v0[g].x, x0.y, acc[g].y);
        acc[g].y = fma(-v0[g].y, x0.x, acc[g].y);
        acc[g].x = fma(v1[g].x, x1.x, acc[g].x);
        acc[g].x = fma(v1[g].y, x1.y, acc[g].x);
        acc[g].y = fma(v1[g].x, x1.y, acc[g].y);
        acc[g].y = fma(-v1[g].y, x1.x, acc[g].y);
      }
    }
#pragma unroll
    for (int g = 0; g < AR_DG; ++g) {
      if (i0 + g < nvec) {
        double2 s = block_sum(acc[g], sh);
        if (threadIdx.x == 0) part[(long)(i0 + g) * G + blockIdx.x] = s;
      }
    }
  }
  double2 r = block_sum(cmk(nrm, 0.0), sh);
  if (threadIdx.x == 0) part[(long)nvec * G + blockIdx.x] = r;
}

// w[e] -= sum_i coef[i] V_i[e]; part[b] = ||w_new||^2 over chunk b
// (two elements per thread and step, AR_DG basis loads in flight per element)
__global__ void __launch_bounds__(AR_THREADS, 3) update_kernel(long n, int nvec, const double2* __restrict__ V,
                                                               long ldv, const double2* __restrict__ coef,
                                                               double2* __restrict__ w,
                                                               double2* __restrict__ part,
                                                               const double* cond) {
  if (cond && cond[2] == 0.0) return;
  __shared__ double2 sh[AR_THREADS / 32];
  __shared__ double2 cf[128];
  long beg, end;
  chunk(n, beg, end);
  double nrm = 0.0;
  for (int i0 = 0; i0 < (nvec > 0 ? nvec : 1); i0 += 128) {
    const int m = nvec - i0 < 128 ? nvec - i0 : 128;
    __syncthreads();
    for (int i = threadIdx.x; i < m; i += AR_THREADS) cf[i] = coef[i0 + i];
    __syncthreads();
    const bool last = (i0 + 128 >= nvec);
    for (long e = beg + threadIdx.x; e < end; e += 2 * AR_THREADS) {
      const long e2 = e + AR_THREADS;
      const bool has2 = e2 < end;
      double2 x0 = w[e];
      double2 x1 = has2 ? w[e2] : cmk(0.0, 0.0);
      for (int i = 0; i < m; i += AR_UG) {
        double2 v0[AR_UG], v1[AR_UG];
#pragma unroll
        for (int g = 0; g < AR_UG; ++g) {
          const bool ok = i + g < m;
          const double2* vp = V + (long)(i0 + i + g) * ldv;
          v0[g] = ok ? ld_stream(vp + e) : cmk(0.0, 0.0);
          v1[g] = (ok && has2) ? ld_stream(vp + e2) : cmk(0.0, 0.0);
        }
#pragma unroll
        for (int g = 0; g < AR_UG; ++g) {
          if (i + g < m) {
            const double2 c = cf[i + g];
            cfms(x0, c, v0[g]);
            cfms(x1, c, v1[g]);
          }
        }
      }
      w[e] = x0;
      if (has2) w[e2] = x1;
      if (last) {
        nrm = fma(x0.x, x0.x, nrm);
        nrm = fma(x0.y, x0.y, nrm);
        nrm = fma(x1.x, x1.x, nrm);
        nrm = fma(x1.y, x1.y, nrm);
      }
    }
  }
  double2 r = block_sum(cmk(nrm, 0.0), sh);
  if (threadIdx.x == 0) part[blockIdx.x] = r;
}

// First-pass update fused with the DGKS second pass's dot products (nvec <=
// NV): w1 = w - V h is formed element by element as in update_kernel, and the
// same thread immediately re-reads the basis values it just streamed (L1 /
// L2 hits) for the partial sums of V^H w1, so the second pass needs no dots
// sweep over V from HBM.  part[i*G + b] = partial (V_i^H w1) (i < nvec),
// part[nvec*G + b] = partial ||w1||^2 (the layout of dots_kernel).
template <int NV>
__global__ void __launch_bounds__(AR_THREADS, 3)
    update_dots_kernel(long n, int nvec, const double2* __restrict__ V, long ldv, const double2* __restrict__ coef,
                       double2* __restrict__ w, double2* __restrict__ part) {
  __shared__ double2 sh[AR_THREADS / 32];
  __shared__ double2 cf[NV];
  long beg, end;
  chunk(n, beg, end);
  const int G = gridDim.x;
  for (int i = threadIdx.x; i < nvec; i += AR_THREADS) cf[i] = coef[i];
  __syncthreads();
  double2 acc[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) acc[i] = cmk(0.0, 0.0);
  double nrm = 0.0;
  for (long e = beg + threadIdx.x; e < end; e += 2 * AR_THREADS) {
    const long e2 = e + AR_THREADS;
    const bool has2 = e2 < end;
    double2 x0 = w[e];
    double2 x1 = has2 ? w[e2] : cmk(0.0, 0.0);
#pragma unroll
    for (int i = 0; i < NV; i += AR_UG) {
      double2 v0[AR_UG], v1[AR_UG];
#pragma unroll
      for (int g = 0; g < AR_UG; ++g) {
        const bool ok = i + g < nvec;
        const double2* vp = V + (long)(i + g) * ldv;
        v0[g] = ok ? __ldg(vp + e) : cmk(0.0, 0.0);
        v1[g] = (ok && has2) ? __ldg(vp + e2) : cmk(0.0, 0.0);
      }
#pragma unroll
      for (int g = 0; g < AR_UG; ++g)
        if (i + g < nvec) {
          cfms(x0, cf[i + g], v0[g]);
          cfms(x1, cf[i + g], v1[g]);
        }
    }
    w[e] = x0;
    if (has2) w[e2] = x1;
    nrm = fma(x0.x, x0.x, nrm);
    nrm = fma(x0.y, x0.y, nrm);
    nrm = fma(x1.x, x1.x, nrm);
    nrm = fma(x1.y, x1.y, nrm);
#pragma unroll
    for (int i = 0; i < NV; ++i)
      if (i < nvec) {
        const double2* vp = V + (long)i * ldv;
        const double2 v0 = __ldg(vp + e);
        const double2 v1 = has2 ? __ldg(vp + e2) : cmk(0.0, 0.0);
        acc[i].x = fma(v0.x, x0.x, acc[i].x);
        acc[i].x = fma(v0.y, x0.y, acc[i].x);
        acc[i].y = fma(v0.x, x0.y, acc[i].y);
        acc[i].y = fma(-v0.y, x0.x, acc[i].y);
        acc[i].x = fma(v1.x, x1.x, acc[i].x);
        acc[i].x = fma(v1.y, x1.y, acc[i].x);
        acc[i].y = fma(v1.x, x1.y, acc[i].y);
        acc[i].y = fma(-v1.y, x1.x, acc[i].y);
      }
  }
#pragma unroll
  for (int i = 0; i < NV; ++i)
    if (i < nvec) {
      const double2 r = block_sum(acc[i], sh);
      if (threadIdx.x == 0) part[(long)i * G + blockIdx.x] = r;
    }
  const double2 r = block_sum(cmk(nrm, 0.0), sh);
  if (threadIdx.x == 0) part[(long)nvec * G + blockIdx.x] = r;
}

// Fixed-order finalisation of the partial sums (single CTA).
//  mode 0: h[i] = sum part_i (i<nvec); stats[0] = sqrt(sum part_nvec)
//  mode 1: stats[1] = sqrt(sum part_0); stats[2] = stats[1] < 0.7071 stats[0]; h[nvec] = stats[1]
//  mode 2 (cond): c[i] = sum part_i; h[i] += c[i]
//  mode 3 (cond): h[nvec] = sqrt(sum part_0)
__global__ void __launch_bounds__(AR_THREADS) finalize_kernel(int nvec, int G, const double2* __restrict__ part,
                                                              double2* __restrict__ h,
                                                              double2* __restrict__ c, double* stats,
                                                              int mode) {
  if ((mode == 2 || mode == 3) && stats[2] == 0.0) return;
  __shared__ double2 sh[AR_THREADS / 32];
  const int rows = (mode == 0) ? nvec + 1 : (mode == 2 ? nvec : 1);
  const int row0 = (mode == 5) ? nvec : 0;  // mode 5: mode 1 on the norm row of update_dots_kernel
  if (mode == 5) mode = 1;
  // one CTA per row (grid-strided): each row is summed in the same fixed order
  for (int i = blockIdx.x; i < rows; i += gridDim.x) {
    double2 v = cmk(0.0, 0.0);
    for (int b = threadIdx.x; b < G; b += AR_THREADS) v = cadd(v, part[(long)(row0 + i) * G + b]);
    v = block_sum(v, sh);
    if (threadIdx.x == 0) {
      if (mode == 0) {
        if (i < nvec) h[i] = v;
        else stats[0] = sqrt(v.x);
      } else if (mode == 1) {
        stats[1] = sqrt(v.x);
        stats[2] = (stats[1] < 0.7071 * stats[0]) ? 1.0 : 0.0;
        h[nvec] = cmk(stats[1], 0.0);
      } else if (mode == 2) {
        c[i] = v;
        h[i] = cadd(h[i], v);
      } else {
        h[nvec] = cmk(sqrt(v.x), 0.0);
      }
    }
  }
}

// out[i] = sum_b part[i*G + b], fixed order (single CTA)
__global__ void __launch_bounds__(AR_THREADS) sum_rows_kernel(int rows, int G, const double2* __restrict__ part,
                                                              double2* __restrict__ out) {
  __shared__ double2 sh[AR_THREADS / 32];
  for (int i = blockIdx.x; i < rows; i += gridDim.x) {
    double2 v = cmk(0.0, 0.0);
    for (int b = threadIdx.x; b < G; b += AR_THREADS) v = cadd(v, part[(long)i * G + b]);
    v = block_sum(v, sh);
    if (threadIdx.x == 0) out[i] = v;
  }
}

// out[i] = sum_b part[i*G + b] if the device flag cond[2] is set, else 0 (the
// conditional DGKS pass of the sharded step: the value is all-reduced either way)
__global__ void __launch_bounds__(AR_THREADS) sum_rows_cond_kernel(int rows, int G,
                                                                   const double2* __restrict__ part,
                                                                   double2* __restrict__ out,
                                                                   const double* __restrict__ cond) {
  __shared__ double2 sh[AR_THREADS / 32];
  const bool on = cond[2] != 0.0;
  for (int i = blockIdx.x; i < rows; i += gridDim.x) {
    double2 v = cmk(0.0, 0.0);
    if (on)
      for (int b = threadIdx.x; b < G; b += AR_THREADS) v = cadd(v, part[(long)i * G + b]);
    v = block_sum(v, sh);
    if (threadIdx.x == 0) out[i] = v;
  }
}

// DGKS decision of the sharded step from the all-reduced squared norms
// (reference solver.py:69-73): ctl = (||w0||, ||w1||, fired, .)
__global__ void dgks_ctl_kernel(const double2* __restrict__ n0sq, const double2* __restrict__ n1sq,
                                double* __restrict__ ctl) {
  const double n0 = sqrt(n0sq->x), n1 = sqrt(n1sq->x);
  ctl[0] = n0;
  ctl[1] = n1;
  ctl[2] = (n1 < 0.7071 * n0) ? 1.0 : 0.0;
}

// Hessenberg column of the sharded step: h = d (+ c when the second pass ran),
// h[nvec] = ctl[3] = the final norm (||w2|| from the all-reduced n2sq if it ran, else ||w1||)
__global__ void dgks_finish_kernel(int nvec, const double2* __restrict__ d, const double2* __restrict__ c,
                                   const double2* __restrict__ n2sq, double* __restrict__ ctl,
                                   double2* __restrict__ hcol) {
  const bool on = ctl[2] != 0.0;
  for (int i = threadIdx.x; i < nvec; i += blockDim.x) hcol[i] = on ? cadd(d[i], c[i]) : d[i];
  if (threadIdx.x == 0) {
    const double nf = on ? sqrt(n2sq->x) : ctl[1];
    ctl[3] = nf;
    hcol[nvec] = cmk(nf, 0.0);
  }
}

__global__ void scale_kernel(long n, const double2* __restrict__ w, double2* __restrict__ out,
                             const double2* __restrict__ hn) {
  const double s = hn->x;
  const double inv = s > 0.0 ? 1.0 / s : 0.0;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < n; e += (long)gridDim.x * blockDim.x) {
    const double2 x = w[e];
    // the reference divides (w / h); division keeps parity with numpy
    out[e] = s > 0.0 ? cmk(x.x / s, x.y / s) : cmk(x.x * inv, x.y * inv);
  }
}

__global__ void combine_kernel(long n, int nvec, const double2* __restrict__ V, long ldv,
                               const double2* __restrict__ y, double2* __restrict__ u) {
  __shared__ double2 ys[128];
  for (long base = (long)blockIdx.x * blockDim.x; base < n; base += (long)gridDim.x * blockDim.x) {
    const long e = base + threadIdx.x;
    double2 acc = cmk(0.0, 0.0);
    for (int i0 = 0; i0 < nvec; i0 += 128) {
      const int m = nvec - i0 < 128 ? nvec - i0 : 128;
      __syncthreads();
      for (int i = threadIdx.x; i < m; i += blockDim.x) ys[i] = y[i0 + i];
      __syncthreads();
      if (e < n)
        for (int i = 0; i < m; ++i) cfma(acc, ys[i], ld_stream(V + (long)(i0 + i) * ldv + e));
    }
    if (e < n) u[e] = acc;
  }
}

// u = sum_i y[i] Z_i with the basis vectors given by a device pointer array
// (the preconditioned vectors z_j = P^-1 v_j kept where the preconditioner
// wrote them, instead of copying each into a basis matrix)
__global__ void combine_ptrs_kernel(long n, int nvec, const double2* const* __restrict__ Z,
                                    const double2* __restrict__ y, double2* __restrict__ u) {
  __shared__ double2 ys[128];
  __shared__ const double2* zp[128];
  for (long base = (long)blockIdx.x * blockDim.x; base < n; base += (long)gridDim.x * blockDim.x) {
    const long e = base + threadIdx.x;
    double2 acc = cmk(0.0, 0.0);
    for (int i0 = 0; i0 < nvec; i0 += 128) {
      const int m = nvec - i0 < 128 ? nvec - i0 : 128;
      __syncthreads();
      for (int i = threadIdx.x; i < m; i += blockDim.x) {
        ys[i] = y[i0 + i];
        zp[i] = Z[i0 + i];
      }
      __syncthreads();
      if (e < n)
        for (int i = 0; i < m; ++i) cfma(acc, ys[i], ld_stream(zp[i] + e));
    }
    if (e < n) u[e] = acc;
  }
}

__global__ void axpby_kernel(long n, double2 a, const double2* __restrict__ x, double2 b,
                             const double2* __restrict__ y, double2* __restrict__ out) {
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < n; e += (long)gridDim.x * blockDim.x) {
    double2 v = cmul(a, x[e]);
    if (y) cfma(v, b, y[e]);
    out[e] = v;
  }
}

__global__ void __launch_bounds__(AR_THREADS) norm_part_kernel(long n, const double2* __restrict__ x,
                                                               double2* __restrict__ part) {
  __shared__ double2 sh[AR_THREADS / 32];
  long beg, end;
  chunk(n, beg, end);
  double2 nrm = cmk(0.0, 0.0);
  for (long e = beg + threadIdx.x; e < end; e += AR_THREADS) {
    const double2 v = x[e];
    nrm.x = fma(v.x, v.x, nrm.x);
    nrm.x = fma(v.y, v.y, nrm.x);
  }
  double2 r = block_sum(nrm, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = r;
}

__global__ void __launch_bounds__(AR_THREADS) norm_final_kernel(int G, const double2* __restrict__ part,
                                                                double* out) {
  __shared__ double2 sh[AR_THREADS / 32];
  double2 v = cmk(0.0, 0.0);
  for (int b = threadIdx.x; b < G; b += AR_THREADS) v = cadd(v, part[b]);
  v = block_sum(v, sh);
  if (threadIdx.x == 0) out[0] = sqrt(v.x);
}

static unsigned stream_grid(long n) {
  long g = (n + 255) / 256;
  const long cap = 16L * device_sm_count();
  return (unsigned)(g < 1 ? 1 : (g > cap ? cap : g));
}

}  // namespace vx

using namespace vx;

extern "C" long vx_arnoldi_part_elems(long n, int nvec) {
  return (long)(nvec + 2) * ar_grid(n) + nvec + 2;
}

extern "C" int vx_arnoldi_step(long n, int nvec, const vx_c128* V, long ldv, vx_c128* w,
                               vx_c128* vnext, vx_c128* hout, double* stats, vx_c128* part,
                               void* stream) {
  VX_REQUIRE(n >= 1 && nvec >= 0 && ldv >= n, "bad Arnoldi arguments");
  cudaStream_t s = as_stream(stream);
  Span span("arnoldi_step", s);
  const int G = ar_grid(n);
  const double2* Vd = reinterpret_cast<const double2*>(V);
  double2* wd = reinterpret_cast<double2*>(w);
  double2* hd = reinterpret_cast<double2*>(hout);
  double2* pd = reinterpret_cast<double2*>(part);
  double2* cd = pd + (long)(nvec + 2) * G;  // second-pass coefficients
  dots_kernel<<<G, AR_THREADS, 0, s>>>(n, nvec, Vd, ldv, wd, pd, nullptr);
  finalize_kernel<<<nvec + 1, AR_THREADS, 0, s>>>(nvec, G, pd, hd, cd, stats, 0);
  static const int fuse = [] { const char* v = getenv("VX_AR_FUSE"); return v ? atoi(v) : 1; }();
  // fused only while the re-read basis values are still in L1 (measured at
  // c1: nvec <= 8 saves the second dots sweep; at 9..16 the re-read goes to
  // L2/HBM and the fused kernel costs as much as the two passes)
  if (fuse && nvec >= 1 && nvec <= 8) {
    // first update + the second pass's dots in one sweep (partials for the
    // conditional DGKS pass are ready whether or not it fires)
    const int Gf = G;
    update_dots_kernel<8><<<Gf, AR_THREADS, 0, s>>>(n, nvec, Vd, ldv, hd, wd, pd);
    finalize_kernel<<<1, AR_THREADS, 0, s>>>(nvec, Gf, pd, hd, cd, stats, 5);
    finalize_kernel<<<nvec, AR_THREADS, 0, s>>>(nvec, Gf, pd, hd, cd, stats, 2);
  } else {
    update_kernel<<<G, AR_THREADS, 0, s>>>(n, nvec, Vd, ldv, hd, wd, pd, nullptr);
    finalize_kernel<<<1, AR_THREADS, 0, s>>>(nvec, G, pd, hd, cd, stats, 1);
    // DGKS second pass, executed only if the device flag stats[2] is set
    dots_kernel<<<G, AR_THREADS, 0, s>>>(n, nvec, Vd, ldv, wd, pd, stats);
    finalize_kernel<<<nvec > 0 ? nvec : 1, AR_THREADS, 0, s>>>(nvec, G, pd, hd, cd, stats, 2);
  }
  update_kernel<<<G, AR_THREADS, 0, s>>>(n, nvec, Vd, ldv, cd, wd, pd, stats);
  finalize_kernel<<<1, AR_THREADS, 0, s>>>(nvec, G, pd, hd, cd, stats, 3);
  if (vnext)
    scale_kernel<<<stream_grid(n), 256, 0, s>>>(n, wd, reinterpret_cast<double2*>(vnext), hd + nvec);
  if (vnext) count_launch();
  count_launch(7);
  VX_CHECK_LAUNCH("arnoldi_step");
  return VX_OK;
}

extern "C" int vx_basis_combine(long n, int nvec, const vx_c128* V, long ldv, const vx_c128* y,
                                vx_c128* u, void* stream) {
  VX_REQUIRE(n >= 1 && nvec >= 0, "bad combine arguments");
  combine_kernel<<<stream_grid(n), 256, 0, as_stream(stream)>>>(
      n, nvec, reinterpret_cast<const double2*>(V), ldv, reinterpret_cast<const double2*>(y),
      reinterpret_cast<double2*>(u));
  VX_CHECK_LAUNCH("combine_kernel");
  return VX_OK;
}

extern "C" int vx_axpby(long n, vx_c128 a, const vx_c128* x, vx_c128 b, const vx_c128* y,
                        vx_c128* out, void* stream) {
  if (n <= 0) return VX_OK;
  axpby_kernel<<<stream_grid(n), 256, 0, as_stream(stream)>>>(
      n, make_double2(a.re, a.im), reinterpret_cast<const double2*>(x), make_double2(b.re, b.im),
      reinterpret_cast<const double2*>(y), reinterpret_cast<double2*>(out));
  VX_CHECK_LAUNCH("axpby_kernel");
  return VX_OK;
}

extern "C" int vx_norm2(long n, const vx_c128* x, double* out, vx_c128* part, void* stream) {
  VX_REQUIRE(n >= 1, "bad norm arguments");
  const int G = ar_grid(n);
  cudaStream_t s = as_stream(stream);
  norm_part_kernel<<<G, AR_THREADS, 0, s>>>(n, reinterpret_cast<const double2*>(x),
                                            reinterpret_cast<double2*>(part));
  norm_final_kernel<<<1, AR_THREADS, 0, s>>>(G, reinterpret_cast<const double2*>(part), out);
  count_launch();
  VX_CHECK_LAUNCH("norm2");
  return VX_OK;
}

extern "C" int vx_cgs_dots(long n, int nvec, const vx_c128* V, long ldv, const vx_c128* w, vx_c128* out,
                           vx_c128* part, void* stream) {
  VX_REQUIRE(n >= 1 && nvec >= 0 && ldv >= n, "bad cgs_dots arguments");
  cudaStream_t s = as_stream(stream);
  const int G = ar_grid(n);
  double2* pd = reinterpret_cast<double2*>(part);
  dots_kernel<<<G, AR_THREADS, 0, s>>>(n, nvec, reinterpret_cast<const double2*>(V), ldv,
                                       reinterpret_cast<const double2*>(w), pd, nullptr);
  sum_rows_kernel<<<nvec + 1, AR_THREADS, 0, s>>>(nvec + 1, G, pd, reinterpret_cast<double2*>(out));
  count_launch();
  VX_CHECK_LAUNCH("cgs_dots");
  return VX_OK;
}

extern "C" int vx_cgs_update(long n, int nvec, const vx_c128* V, long ldv, const vx_c128* coef, vx_c128* w,
                             vx_c128* out_norm2, vx_c128* part, void* stream) {
  VX_REQUIRE(n >= 1 && nvec >= 0 && ldv >= n, "bad cgs_update arguments");
  cudaStream_t s = as_stream(stream);
  const int G = ar_grid(n);
  double2* pd = reinterpret_cast<double2*>(part);
  update_kernel<<<G, AR_THREADS, 0, s>>>(n, nvec, reinterpret_cast<const double2*>(V), ldv,
                                         reinterpret_cast<const double2*>(coef), reinterpret_cast<double2*>(w),
                                         pd, nullptr);
  sum_rows_kernel<<<1, AR_THREADS, 0, s>>>(1, G, pd, reinterpret_cast<double2*>(out_norm2));
  count_launch();
  VX_CHECK_LAUNCH("cgs_update");
  return VX_OK;
}

extern "C" int vx_basis_combine_ptrs(long n, int nvec, const void* zptrs, const vx_c128* y, vx_c128* u,
                                     void* stream) {
  VX_REQUIRE(n >= 1 && nvec >= 0, "bad combine arguments");
  combine_ptrs_kernel<<<stream_grid(n), 256, 0, as_stream(stream)>>>(
      n, nvec, reinterpret_cast<const double2* const*>(zptrs), reinterpret_cast<const double2*>(y),
      reinterpret_cast<double2*>(u));
  VX_CHECK_LAUNCH("combine_ptrs_kernel");
  return VX_OK;
}

// ---- device-driven Arnoldi step of the SHARDED solver (dist.py): the stages of
// vx_arnoldi_step as separate calls so that the caller can all-reduce every
// partial result between them on the same stream, with the DGKS decision taken
// on the device (ctl[2]) -- no host read inside a step.
extern "C" int vx_cgs_dots_cond(long n, int nvec, const vx_c128* V, long ldv, const vx_c128* w, vx_c128* out,
                                vx_c128* part, const double* ctl, void* stream) {
  VX_REQUIRE(n >= 1 && nvec >= 0 && ldv >= n && ctl, "bad cgs_dots_cond arguments");
  cudaStream_t s = as_stream(stream);
  const int G = ar_grid(n);
  double2* pd = reinterpret_cast<double2*>(part);
  dots_kernel<<<G, AR_THREADS, 0, s>>>(n, nvec, reinterpret_cast<const double2*>(V), ldv,
                                       reinterpret_cast<const double2*>(w), pd, ctl);
  sum_rows_cond_kernel<<<nvec + 1, AR_THREADS, 0, s>>>(nvec + 1, G, pd, reinterpret_cast<double2*>(out), ctl);
  count_launch();
  VX_CHECK_LAUNCH("cgs_dots_cond");
  return VX_OK;
}

extern "C" int vx_cgs_update_cond(long n, int nvec, const vx_c128* V, long ldv, const vx_c128* coef, vx_c128* w,
                                  vx_c128* out_norm2, vx_c128* part, const double* ctl, void* stream) {
  VX_REQUIRE(n >= 1 && nvec >= 0 && ldv >= n && ctl, "bad cgs_update_cond arguments");
  cudaStream_t s = as_stream(stream);
  const int G = ar_grid(n);
  double2* pd = reinterpret_cast<double2*>(part);
  update_kernel<<<G, AR_THREADS, 0, s>>>(n, nvec, reinterpret_cast<const double2*>(V), ldv,
                                         reinterpret_cast<const double2*>(coef), reinterpret_cast<double2*>(w),
                                         pd, ctl);
  sum_rows_cond_kernel<<<1, AR_THREADS, 0, s>>>(1, G, pd, reinterpret_cast<double2*>(out_norm2), ctl);
  count_launch();
  VX_CHECK_LAUNCH("cgs_update_cond");
  return VX_OK;
}

extern "C" int vx_dgks_ctl(const vx_c128* n0sq, const vx_c128* n1sq, double* ctl, void* stream) {
  VX_REQUIRE(n0sq && n1sq && ctl, "bad dgks_ctl arguments");
  dgks_ctl_kernel<<<1, 1, 0, as_stream(stream)>>>(reinterpret_cast<const double2*>(n0sq),
                                                  reinterpret_cast<const double2*>(n1sq), ctl);
  VX_CHECK_LAUNCH("dgks_ctl_kernel");
  return VX_OK;
}

extern "C" int vx_dgks_finish(int nvec, const vx_c128* d, const vx_c128* c, const vx_c128* n2sq, double* ctl,
                              vx_c128* hcol, void* stream) {
  VX_REQUIRE(nvec >= 0 && d && c && n2sq && ctl && hcol, "bad dgks_finish arguments");
  dgks_finish_kernel<<<1, 128, 0, as_stream(stream)>>>(nvec, reinterpret_cast<const double2*>(d),
                                                       reinterpret_cast<const double2*>(c),
                                                       reinterpret_cast<const double2*>(n2sq), ctl,
                                                       reinterpret_cast<double2*>(hcol));
  VX_CHECK_LAUNCH("dgks_finish_kernel");
  return VX_OK;
}

extern "C" int vx_scale_dev(long n, const vx_c128* w, vx_c128* out, const vx_c128* hn, void* stream) {
  VX_REQUIRE(n >= 1 && w && out && hn, "bad scale arguments");
  scale_kernel<<<stream_grid(n), 256, 0, as_stream(stream)>>>(n, reinterpret_cast<const double2*>(w),
                                                             reinterpret_cast<double2*>(out),
                                                             reinterpret_cast<const double2*>(hn));
  VX_CHECK_LAUNCH("scale_kernel");
  return VX_OK;
}

