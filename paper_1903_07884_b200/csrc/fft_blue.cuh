// Bluestein DFTs of contiguous lines in three register passes (prime and other
// non-smooth lengths n with 2n-1 <= 32^2: the 2-level preconditioner's nx = 367
// at c4).  The length-n DFT is the cyclic convolution of a[j] = x[j] c[j] with
// conj(c) (c[j] = exp(-pi i j^2/n)) over M = R*R points, R a register DFT
// length, and both length-M transforms are split M = R x R:
//   pass 1  task m < R:  a[n1 R + m] straight from global memory (chirp applied
//           at the load, zero beyond n), length-R register DFT over n1, twiddle
//           w_M^(k1 m), to shared memory at (k1, m)
//   pass 2  task k1 < R: the row (k1, .) -> length-R DFT over m gives the
//           spectrum A[k1 + R k2]; times Bhat[k1 + R k2]; inverse length-R DFT
//           over k2; conjugate twiddle; back in place -- the forward transform's
//           last pass and the inverse's first pass never leave the registers
//   pass 3  task m < R:  the column (., m) -> inverse length-R DFT over k1 gives
//           the convolution at n1 R + m; times c, cropped to n, through the
//           storer.
// Two shared-memory round trips and two barriers per line (the stage engine
// runs 8 radix stages plus the pointwise product).  Rows are padded to R+1
// entries: 8 consecutive rows land on 8 distinct 16-byte bank groups.
#pragma once

#include "fft_lines.cuh"
#include "fft_reg.cuh"

namespace vx {

#ifndef VX_BLUE_MINB
#define VX_BLUE_MINB 1
#endif
template <int R, bool INV, class Loader, class Storer>
__global__ void __launch_bounds__(8 * R, VX_BLUE_MINB)
    blue_reg_kernel(Loader ld, Storer st, const double2* __restrict__ chirp, const double2* __restrict__ bhat,
                    const double2* __restrict__ twm, int n, int n_lines, int W, int n_in, int n_out) {
  constexpr int LD = R + 1, LS = R * LD;  // row pitch, line pitch
  extern __shared__ double2 bsm[];
  const int l0 = blockIdx.x * W;
  // pass 1
  for (int i = threadIdx.x; i < W * R; i += blockDim.x) {
    const int w = i / R, m = i - w * R;
    const int l = l0 + w;
    double2 v[R];
    const long b = l < n_lines ? ld.line_base(l) : 0;
#pragma unroll
    for (int n1 = 0; n1 < R; ++n1) {
      const int e = n1 * R + m;
      double2 x = cmk(0.0, 0.0);
      if (l < n_lines && e < n_in) {
        x = ld(b, e);
        if (INV) x = cconj(x);
        x = cmul(x, __ldg(chirp + e));
      }
      v[n1] = x;
    }
    reg_fft<R, false>(v);
    double2* s = bsm + w * LS + m;
    s[0] = v[0];
#pragma unroll
    for (int k1 = 1; k1 < R; ++k1) s[k1 * LD] = m ? cmul(v[k1], __ldg(twm + k1 * m)) : v[k1];
  }
  __syncthreads();
  // pass 2
  for (int i = threadIdx.x; i < W * R; i += blockDim.x) {
    const int w = i / R, k1 = i - w * R;
    double2* s = bsm + w * LS + k1 * LD;
    double2 v[R];
#pragma unroll
    for (int m = 0; m < R; ++m) v[m] = s[m];
    reg_fft<R, false>(v);
#pragma unroll
    for (int k2 = 0; k2 < R; ++k2) v[k2] = cmul(v[k2], __ldg(bhat + k1 + R * k2));
    reg_fft<R, true>(v);
    s[0] = v[0];
#pragma unroll
    for (int m = 1; m < R; ++m) s[m] = k1 ? cmulc(v[m], __ldg(twm + k1 * m)) : v[m];
  }
  __syncthreads();
  // pass 3
  for (int i = threadIdx.x; i < W * R; i += blockDim.x) {
    const int w = i / R, m = i - w * R;
    const int l = l0 + w;
    if (l >= n_lines) continue;
    const double2* s = bsm + w * LS + m;
    double2 v[R];
#pragma unroll
    for (int k1 = 0; k1 < R; ++k1) v[k1] = s[k1 * LD];
    reg_fft<R, true>(v);
    const long b = st.line_base(l);
#pragma unroll
    for (int n1 = 0; n1 < R; ++n1) {
      const int e = n1 * R + m;
      if (e < n_out && e < n) {
        double2 y = cmul(v[n1], __ldg(chirp + e));
        if (INV) y = cconj(y);
        st(b, e, y);
      }
    }
  }
}

inline bool blue_reg_supported(const FftPlan& p) {
  static const int on = env_int("VX_BLUE_REG", 1);
  return on && p.bluestein && p.blue_R > 0;
}

template <int R, class Loader, class Storer>
int launch_blue_reg_t(const FftPlan& p, const Loader& ld, const Storer& st, int n_lines, int n_in, int n_out,
                      bool inv, cudaStream_t s) {
  constexpr int W = 8;
  const size_t smem = (size_t)W * R * (R + 1) * sizeof(double2);
  if (inv) {
    auto k = blue_reg_kernel<R, true, Loader, Storer>;
    if (smem > 48 * 1024) VX_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<div_up(n_lines, W), W * R, smem, s>>>(ld, st, p.chirp, p.blue_bhat, p.blue_tw, p.n, n_lines, W, n_in, n_out);
  } else {
    auto k = blue_reg_kernel<R, false, Loader, Storer>;
    if (smem > 48 * 1024) VX_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<div_up(n_lines, W), W * R, smem, s>>>(ld, st, p.chirp, p.blue_bhat, p.blue_tw, p.n, n_lines, W, n_in, n_out);
  }
  VX_CHECK_LAUNCH("blue_reg_kernel");
  return VX_OK;
}

// Contiguous lines of a Bluestein plan through the register passes.
template <class Loader, class Storer>
int launch_blue_reg(const FftPlan& p, const Loader& ld, const Storer& st, int n_lines, int n_in, int n_out, bool inv,
                    cudaStream_t s) {
  if (n_lines <= 0) return VX_OK;
  switch (p.blue_R) {
    case 16: return launch_blue_reg_t<16>(p, ld, st, n_lines, n_in, n_out, inv, s);
    case 20: return launch_blue_reg_t<20>(p, ld, st, n_lines, n_in, n_out, inv, s);
    case 24: return launch_blue_reg_t<24>(p, ld, st, n_lines, n_in, n_out, inv, s);
    case 28: return launch_blue_reg_t<28>(p, ld, st, n_lines, n_in, n_out, inv, s);
    case 32: return launch_blue_reg_t<32>(p, ld, st, n_lines, n_in, n_out, inv, s);
    default: break;
  }
  set_error("no register Bluestein for length %d", p.n);
  return VX_EINVAL;
}

}  // namespace vx
