// Register-resident short FFTs for the operator's strided passes.
//
// The y and z transforms of the padded grid are short (c1: 45 and 21, c4 z:
// 16) and strided by the x extent, so one thread owns one whole column: it
// loads the column (consecutive threads = consecutive x, so every load is a
// coalesced row), transforms it in registers with a compile-time mixed-radix
// recursion (all indices and twiddles are constants after unrolling: no
// shared memory, no barriers, no index arithmetic), and stores it back.  The
// shared-memory engine (fft.cuh) stays for long lines and for lengths not in
// REG_LENGTHS.  Output order is natural.
#pragma once

#include "fft.cuh"
#include "fft_reg_tw.cuh"

namespace vx {

// the operator's padded lengths <= 56 (vx_op_padded_length of n = 1..28; 60+
// would spill);
// must match tools/gen_fft_reg_tw.py
#define VX_REG_LENGTHS(X) \
  X(2) X(4) X(6) X(8) X(10) X(12) X(14) X(16) X(18) X(20) X(21) X(24) X(25) X(28) X(30) X(32) X(35) X(36) \
  X(40) X(42) X(45) X(48) X(50) X(54) X(56)

__host__ __device__ constexpr int reg_radix(int n) {
  return (n % 8 == 0 && n > 8 && n != 16) ? 8
       : n % 4 == 0                       ? 4
       : n % 2 == 0                       ? 2
       : n % 3 == 0                       ? 3
       : n % 5 == 0                       ? 5
                                          : 7;
}

// w_N^j for the forward (INV = false: exp(-2 pi i j/N)) or inverse transform
template <int N, bool INV>
__device__ __forceinline__ double2 reg_tw(int j) {
  constexpr int o = reg_tw_off(N);
  static_assert(o >= 0, "length not in the register twiddle table");
  const double re = c_rtw[2 * (o + j)], im = c_rtw[2 * (o + j) + 1];
  return cmk(re, INV ? -im : im);
}

// In-register DFT of v[0..N) (natural order in and out), decimation in time:
// N = R*M, R sub-transforms of the stride-R subsequences, then M radix-R
// butterflies with twiddles w_N^{r k}.
template <int N, bool INV>
__device__ __forceinline__ void reg_fft(double2* v) {
  constexpr double sgn = INV ? 1.0 : -1.0;
  if constexpr (N == 1) {
    return;
  } else if constexpr (N == 2 || N == 3 || N == 4 || N == 5 || N == 7 || N == 8 || N == 11 || N == 13) {
    dft_codelet<N>(v, sgn);
  } else {
    constexpr int R = reg_radix(N), M = N / R;
    double2 sub[R][M];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int m = 0; m < M; ++m) sub[r][m] = v[m * R + r];
#pragma unroll
    for (int r = 0; r < R; ++r) reg_fft<M, INV>(sub[r]);
#pragma unroll
    for (int k = 0; k < M; ++k) {
      double2 t[R];
      t[0] = sub[0][k];
#pragma unroll
      for (int r = 1; r < R; ++r) t[r] = (k == 0) ? sub[r][k] : cmul(sub[r][k], reg_tw<N, INV>((r * k) % N));
      dft_codelet<R>(t, sgn);
#pragma unroll
      for (int q = 0; q < R; ++q) v[k + q * M] = t[q];
    }
  }
}

__host__ inline bool reg_fft_supported(int n) {
#define VX_REG_CASE(L) if (n == L) return true;
  VX_REG_LENGTHS(VX_REG_CASE)
#undef VX_REG_CASE
  return false;
}

// Column transform: ncols columns, column c = (o, i) with o = c / n_inner,
// i = c % n_inner (i fastest across threads); element e of the input at
// in + o*in_os + i + e*in_es (e < n_in, zero padded to L), output element e
// (e < n_out, cropped) at out + o*out_os + i + e*out_es, scaled.
template <int L, bool INV>
__global__ void __launch_bounds__(128)
    reg_cols_kernel(const double2* __restrict__ in, long in_os, long in_es, int n_in, double2* __restrict__ out,
                    long out_os, long out_es, int n_out, long ncols, FastDiv fd_inner, int n_inner, double scale) {
  const long c = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (c >= ncols) return;
  const int o = (int)fd_inner.div((unsigned)c), i = (int)(c - (long)o * n_inner);
  const double2* src = in + (long)o * in_os + i;
  double2 v[L];
#pragma unroll
  for (int e = 0; e < L; ++e) v[e] = (e < n_in) ? __ldg(src + e * in_es) : cmk(0.0, 0.0);
  reg_fft<L, INV>(v);
  double2* dst = out + (long)o * out_os + i;
#pragma unroll
  for (int e = 0; e < L; ++e)
    if (e < n_out) dst[e * out_es] = cscale(v[e], scale);
}

// Two-pass column transform for lengths L = R1 * R2 beyond the one-thread
// register kernel (c3's py = 112, c4's 800): CW adjacent columns per CTA
// (consecutive x: every global access is a coalesced run of CW entries), R2
// threads per column run the R1-point sub-transforms of the stride-R2
// subsequences in registers (zero padding in the load), multiply by the
// twiddles w_L^{b k1} and exchange through shared memory; R1 threads per
// column then run the R2-point transforms and store the (cropped) outputs in
// natural order: X[k1 + R1 k2] = sum_b w_R2^{b k2} w_L^{b k1} DFT_R1(x[R2 a + b])[k1].
template <int R1, int R2>
struct Cols2Cfg {
  static constexpr int L = R1 * R2;
  static constexpr int TP = R1 > R2 ? R1 : R2;
  // columns per CTA: 256 threads, at least 8 columns (128-byte runs), shared memory <= ~100 KB
  static constexpr int CW = (256 / TP) < 8 ? 8 : ((256 / TP) > 16 ? 16 : (256 / TP));
  static constexpr int THREADS = CW * TP;
  static constexpr size_t SMEM = (size_t)CW * L * sizeof(double2);
};

template <int R1, int R2, bool INV>
__global__ void __launch_bounds__(Cols2Cfg<R1, R2>::THREADS)
    cols2_kernel(const double2* __restrict__ in, long in_os, long in_es, int n_in, double2* __restrict__ out,
                 long out_os, long out_es, int n_out, long ncols, FastDiv fd_inner, int n_inner, double scale,
                 const double2* __restrict__ tw) {
  using C = Cols2Cfg<R1, R2>;
  constexpr int L = C::L, CW = C::CW;
  extern __shared__ double2 c2sm[];  // entry (k1, b) of column ci at ((k1 * R2 + b) * CW + ci)
  const int ci = threadIdx.x % CW, t = threadIdx.x / CW;
  const long c = (long)blockIdx.x * CW + ci;
  const bool colok = c < ncols;
  const long cc = colok ? c : 0;
  const int o = (int)fd_inner.div((unsigned)cc), i = (int)(cc - (long)o * n_inner);
  if (t < R2) {
    const double2* src = in + (long)o * in_os + i;
    double2 v[R1];
#pragma unroll
    for (int a = 0; a < R1; ++a) {
      const int e = R2 * a + t;
      v[a] = (colok && e < n_in) ? __ldg(src + (long)e * in_es) : cmk(0.0, 0.0);
    }
    reg_fft<R1, INV>(v);
#pragma unroll
    for (int k1 = 0; k1 < R1; ++k1) {
      double2 x = v[k1];
      if (t != 0 && k1 != 0) {
        double2 w = __ldg(tw + (t * k1) % L);
        if (INV) w.y = -w.y;
        x = cmul(x, w);
      }
      c2sm[(k1 * R2 + t) * CW + ci] = x;
    }
  }
  __syncthreads();
  if (t < R1) {
    double2 u[R2];
#pragma unroll
    for (int b = 0; b < R2; ++b) u[b] = c2sm[(t * R2 + b) * CW + ci];
    reg_fft<R2, INV>(u);
    double2* dst = out + (long)o * out_os + i;
#pragma unroll
    for (int k2 = 0; k2 < R2; ++k2) {
      const int e = t + R1 * k2;
      if (colok && e < n_out) dst[(long)e * out_es] = cscale(u[k2], scale);
    }
  }
}

// (R1, R2) of the supported two-pass lengths
#define VX_COLS2_PAIRS(X) \
  X(8, 8) X(12, 6) X(16, 5) X(16, 6) X(20, 5) X(16, 7) X(24, 5) X(16, 8) X(20, 20) X(32, 25)

__host__ inline bool cols2_supported(int n) {
#define VX_C2_CASE(A, B) if (n == (A) * (B)) return true;
  VX_COLS2_PAIRS(VX_C2_CASE)
#undef VX_C2_CASE
  return false;
}

// launch the two-pass column transform of length f.L (f.tw: the plan's twiddle table)
template <bool INV>
inline int launch_cols2(const FftPlan& f, const double2* in, long in_os, long in_es, int n_in, double2* out,
                        long out_os, long out_es, int n_out, long ncols, int n_inner, double scale,
                        cudaStream_t s) {
  if (ncols <= 0) return VX_OK;
  const FastDiv fd((unsigned)n_inner);
#define VX_C2_LAUNCH(A, B)                                                                                   \
  if (f.L == (A) * (B)) {                                                                                    \
    using C = Cols2Cfg<A, B>;                                                                                \
    auto k = cols2_kernel<A, B, INV>;                                                                        \
    if (C::SMEM > 48 * 1024)                                                                                 \
      VX_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));          \
    k<<<(unsigned)div_up(ncols, C::CW), C::THREADS, C::SMEM, s>>>(in, in_os, in_es, n_in, out, out_os, out_es, \
                                                                  n_out, ncols, fd, n_inner, scale, f.tw);   \
    VX_CHECK_LAUNCH("cols2_kernel");                                                                         \
    return VX_OK;                                                                                            \
  }
  VX_COLS2_PAIRS(VX_C2_LAUNCH)
#undef VX_C2_LAUNCH
  set_error("no two-pass column FFT for length %d", f.L);
  return VX_EINVAL;
}


}  // namespace vx
