// Long-line FFTs (the x-direction transforms: operator padded lengths 400 ...
// 10000, preconditioner DFT lengths 200 ... 5000) as two or three register
// passes instead of 5-6 radix-8 shared-memory stages.
//
// L = R1*R2*R3 (R3 = 1 for two factors), decimation in frequency:
//   pass 1  task m < M1 = L/R1: the R1 inputs x[n1*M1 + m] come straight from
//           global memory (coalesced across m; zero padding by the loader),
//           length-R1 register DFT, twiddle w_L^(k1 m), store to smem
//           position k1*M1 + m.
//   pass 2  task (k1, m2 < M2 = R3): R2 values at stride M2 inside block k1,
//           register DFT, twiddle w_L^(R1 k2 m2), back in place.
//   last    task t = k1 + R1*k2: R3 contiguous values, register DFT, and the
//           outputs X[t + (L/R3)*k3] go straight to global memory through the
//           storer (consecutive t -> consecutive addresses: natural order,
//           coalesced, crop / scale / operator epilogue fused).
// Only two smem round trips and two barriers per line; the last pass reads
// with a lane stride of M1 (odd for every factorisation used -> no bank
// conflicts).  Twiddles: the plan's two-level tables staged in smem, powers
// by products (twiddle_row).
#pragma once

#include "fft_lines.cuh"
#include "fft_reg.cuh"
#include "fft_blue.cuh"

#include <cooperative_groups.h>

namespace vx {

// CTA size cap: register codelets above 32 points (735 = 21 x 35) need more than the 128
// registers a 512-thread CTA leaves per thread (they spill 300 bytes).  The forward
// transform runs them at most 256 threads per CTA with up to 255 registers (c4: 0.083 ->
// 0.068 ms); the inverse with the operator epilogue prefers two spilling CTAs per SM
// (0.136 ms against 0.191 ms with one).
template <int R1, int R2, int R3, bool INV>
constexpr int fft_long_max_threads() {
  return (!INV && (R1 > 32 || R2 > 32 || R3 > 32)) ? 256 : 512;
}

template <int R1, int R2, int R3, bool INV, class Loader, class Storer>
__global__ void __launch_bounds__((fft_long_max_threads<R1, R2, R3, INV>()), 1)
    fft_long_kernel(Loader ld, Storer st, const double2* __restrict__ tw_lo, const double2* __restrict__ tw_hi,
                    int nhi, int n_lines, int W, int n_in, int n_out) {
  constexpr int L = R1 * R2 * R3;
  constexpr int M1 = L / R1;
  constexpr int M2 = R3;
  constexpr int RL = R3 > 1 ? R3 : R2;  // last radix
  constexpr int T = L / RL;             // last-pass tasks per line
  constexpr double sgn = INV ? 1.0 : -1.0;
  extern __shared__ double2 lsm[];
  double2* tw = lsm + (size_t)W * L;
  for (int i = threadIdx.x; i < 64 + nhi; i += blockDim.x)
    tw[i] = i < 64 ? __ldg(tw_lo + i) : __ldg(tw_hi + (i - 64));
  const int l0 = blockIdx.x * W;
  __syncthreads();
  // pass 1: global -> registers -> smem
  for (int i = threadIdx.x; i < W * M1; i += blockDim.x) {
    const int w = i / M1, m = i - w * M1;
    const int l = l0 + w;
    double2 v[R1];
    if (l < n_lines) {
      const long b = ld.line_base(l);
#pragma unroll
      for (int n1 = 0; n1 < R1; ++n1) {
        const int e = n1 * M1 + m;
        v[n1] = e < n_in ? ld(b, e) : cmk(0.0, 0.0);
      }
    } else {
#pragma unroll
      for (int n1 = 0; n1 < R1; ++n1) v[n1] = cmk(0.0, 0.0);
    }
    reg_fft<R1, INV>(v);
    if (m) twiddle_row<R1>(v, tw, m, sgn);
    double2* s = lsm + (size_t)w * L + m;
#pragma unroll
    for (int k1 = 0; k1 < R1; ++k1) s[k1 * M1] = v[k1];
  }
  __syncthreads();
  if constexpr (R3 > 1) {
    for (int i = threadIdx.x; i < W * R1 * M2; i += blockDim.x) {
      const int w = i / (R1 * M2), r = i - w * (R1 * M2);
      const int k1 = r / M2, m2 = r - k1 * M2;
      double2* s = lsm + (size_t)w * L + k1 * M1 + m2;
      double2 v[R2];
#pragma unroll
      for (int n2 = 0; n2 < R2; ++n2) v[n2] = s[n2 * M2];
      reg_fft<R2, INV>(v);
      if (m2) twiddle_row<R2>(v, tw, R1 * m2, sgn);
#pragma unroll
      for (int k2 = 0; k2 < R2; ++k2) s[k2 * M2] = v[k2];
    }
    __syncthreads();
  }
  // last pass: smem -> registers -> global (natural order)
  for (int i = threadIdx.x; i < W * T; i += blockDim.x) {
    const int w = i / T, t = i - w * T;
    const int l = l0 + w;
    if (l >= n_lines) continue;
    int pos;
    if constexpr (R3 > 1) {
      const int k2 = t / R1, k1 = t - k2 * R1;
      pos = k1 * M1 + k2 * M2;
    } else {
      pos = t * M1;
    }
    const double2* s = lsm + (size_t)w * L + pos;
    double2 v[RL];
#pragma unroll
    for (int n = 0; n < RL; ++n) v[n] = s[n];
    reg_fft<RL, INV>(v);
    const long b = st.line_base(l);
#pragma unroll
    for (int k = 0; k < RL; ++k) {
      const int e = t + T * k;
      if (e < n_out) st(b, e, v[k]);
    }
  }
}

// Lines too long for two CTAs per SM (L = 10000: 160 KB) are split over a
// 2-CTA cluster: each CTA holds half of the line's smem (positions
// [rank L/2, (rank+1) L/2)), so two 80 KB CTAs of different lines share an SM
// and overlap their load / compute / store phases.  Pass 1 writes its outputs
// k1 >= R1/2 into the partner's shared memory (DSMEM); after one cluster
// barrier passes 2 and 3 only touch the CTA's own half (blocks k1 of its
// half).  Requires R1 even.
template <int R1, int R2, int R3, bool INV, class Loader, class Storer>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 2)
    fft_long2_kernel(Loader ld, Storer st, const double2* __restrict__ tw_lo, const double2* __restrict__ tw_hi,
                     int nhi, int n_lines, int n_in, int n_out) {
  constexpr int L = R1 * R2 * R3;
  constexpr int M1 = L / R1;
  constexpr int M2 = R3;
  constexpr int H1 = R1 / 2;  // k1 blocks per CTA
  constexpr int HALF = H1 * M1;
  constexpr double sgn = INV ? 1.0 : -1.0;
  static_assert(R1 % 2 == 0 && R3 > 1, "cluster split needs an even first radix and three factors");
  extern __shared__ double2 lsm[];
  double2* tw = lsm + HALF;
  namespace cgx = cooperative_groups;
  cgx::cluster_group cl = cgx::this_cluster();
  const int rank = (int)cl.block_rank();
  const int l = blockIdx.x >> 1;
  for (int i = threadIdx.x; i < 64 + nhi; i += blockDim.x)
    tw[i] = i < 64 ? __ldg(tw_lo + i) : __ldg(tw_hi + (i - 64));
  double2* half0 = cl.map_shared_rank(lsm, 0);
  double2* half1 = cl.map_shared_rank(lsm, 1);
  __syncthreads();
  // pass 1: this CTA's share of the M1 tasks; outputs to both halves
  const int m0 = rank * ((M1 + 1) / 2), m1 = rank ? M1 : (M1 + 1) / 2;
  if (l < n_lines) {
    const long b = ld.line_base(l);
    for (int m = m0 + threadIdx.x; m < m1; m += blockDim.x) {
      double2 v[R1];
#pragma unroll
      for (int n1 = 0; n1 < R1; ++n1) {
        const int e = n1 * M1 + m;
        v[n1] = e < n_in ? ld(b, e) : cmk(0.0, 0.0);
      }
      reg_fft<R1, INV>(v);
      if (m) twiddle_row<R1>(v, tw, m, sgn);
#pragma unroll
      for (int k1 = 0; k1 < H1; ++k1) half0[k1 * M1 + m] = v[k1];
#pragma unroll
      for (int k1 = 0; k1 < H1; ++k1) half1[k1 * M1 + m] = v[H1 + k1];
    }
  }
  cl.sync();
  if (l >= n_lines) return;
  // pass 2: blocks k1 = rank H1 + k1l, local
  for (int i = threadIdx.x; i < H1 * M2; i += blockDim.x) {
    const int k1l = i / M2, m2 = i - k1l * M2;
    double2* s = lsm + k1l * M1 + m2;
    double2 v[R2];
#pragma unroll
    for (int n2 = 0; n2 < R2; ++n2) v[n2] = s[n2 * M2];
    reg_fft<R2, INV>(v);
    if (m2) twiddle_row<R2>(v, tw, R1 * m2, sgn);
#pragma unroll
    for (int k2 = 0; k2 < R2; ++k2) s[k2 * M2] = v[k2];
  }
  __syncthreads();
  // last pass: tasks t = k1 + R1 k2 with k1 in this CTA's half
  constexpr int T = L / R3;
  const long bo = st.line_base(l);
  for (int i = threadIdx.x; i < H1 * R2; i += blockDim.x) {
    const int k1l = i % H1, k2 = i / H1;
    const int t = rank * H1 + k1l + R1 * k2;
    const double2* s = lsm + k1l * M1 + k2 * M2;
    double2 v[R3];
#pragma unroll
    for (int n = 0; n < R3; ++n) v[n] = s[n];
    reg_fft<R3, INV>(v);
#pragma unroll
    for (int k = 0; k < R3; ++k) {
      const int e = t + T * k;
      if (e < n_out) st(bo, e, v[k]);
    }
  }
}

template <int R1, int R2, int R3, bool INV, class Loader, class Storer>
int launch_fft_long2_t(const FftPlan& p, const Loader& ld, const Storer& st, int n_lines, int n_in, int n_out,
                       cudaStream_t s) {
  constexpr int L = R1 * R2 * R3;
  const size_t smem = ((size_t)L / 2 + 64 + p.nhi) * sizeof(double2);
  auto kern = fft_long2_kernel<R1, R2, R3, INV, Loader, Storer>;
  VX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  static const int thr_env = env_int("VX_FFT_LONG2_THREADS", 256);
  kern<<<2 * n_lines, thr_env, smem, s>>>(ld, st, p.tw_lo, p.tw_hi, p.nhi, n_lines, n_in, n_out);
  VX_CHECK_LAUNCH("fft_long2_kernel");
  return VX_OK;
}

// Factorisations with a register kernel (M1 = L/R1 odd for the conflict-free
// last pass).  X(L, R1, R2, R3)
#define VX_LONG_FACTORS(X)                                                                    \
  X(10000, 16, 25, 25) X(5000, 8, 25, 25) X(2500, 4, 25, 25) X(3000, 8, 15, 25)              \
  X(1500, 4, 15, 25) X(400, 16, 25, 1) X(200, 8, 25, 1) X(735, 21, 35, 1)

inline bool fft_long_supported(int L) {
#define VX_LONG_CASE(N, A, B, C) if (L == N) return true;
  VX_LONG_FACTORS(VX_LONG_CASE)
#undef VX_LONG_CASE
  return false;
}

template <int R1, int R2, int R3, bool INV, class Loader, class Storer>
int launch_fft_long_t(const FftPlan& p, const Loader& ld, const Storer& st, int n_lines, int n_in, int n_out,
                      cudaStream_t s) {
  constexpr int L = R1 * R2 * R3;
  constexpr int RL = R3 > 1 ? R3 : R2;
  static const int target = env_int("VX_FFT_LONG_ELEMS", 5000);
  int W = target / L;
  if (W < 1) W = 1;
  if (W > n_lines) W = n_lines;
  const int tasks = W * (L / R1 > L / RL ? L / R1 : L / RL);
  // lines that fill the SM alone get up to 640 threads; shorter lines run
  // 2+ CTAs per SM with fewer threads each
  const size_t smem = ((size_t)W * L + 64 + p.nhi) * sizeof(double2);
  const int cap = smem > 100 * 1024 ? fft_long_max_threads<R1, R2, R3, INV>() : 256;
  int thr = ((tasks < cap ? tasks : cap) + 31) / 32 * 32;
  auto kern = fft_long_kernel<R1, R2, R3, INV, Loader, Storer>;
  if (smem > 48 * 1024)
    VX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<div_up(n_lines, W), thr, smem, s>>>(ld, st, p.tw_lo, p.tw_hi, p.nhi, n_lines, W, n_in, n_out);
  VX_CHECK_LAUNCH("fft_long_kernel");
  return VX_OK;
}

// Contiguous lines of length p.n (direct plan) through the register passes.
template <class Loader, class Storer>
int launch_fft_long(const FftPlan& p, const Loader& ld, const Storer& st, int n_lines, int n_in, int n_out,
                    bool inv, cudaStream_t s) {
  if (n_lines <= 0) return VX_OK;
  static const int split = env_int("VX_FFT_LONG2", 1);
  if (split && p.n == 10000)
    return inv ? launch_fft_long2_t<16, 25, 25, true>(p, ld, st, n_lines, n_in, n_out, s)
               : launch_fft_long2_t<16, 25, 25, false>(p, ld, st, n_lines, n_in, n_out, s);
  switch (p.n) {
#define VX_LONG_LAUNCH(N, A, B, C)                                                              \
  case N:                                                                                       \
    return inv ? launch_fft_long_t<A, B, C, true>(p, ld, st, n_lines, n_in, n_out, s)           \
               : launch_fft_long_t<A, B, C, false>(p, ld, st, n_lines, n_in, n_out, s);
    VX_LONG_FACTORS(VX_LONG_LAUNCH)
#undef VX_LONG_LAUNCH
    default:
      break;
  }
  set_error("no long-line register FFT for length %d", p.n);
  return VX_EINVAL;
}

inline bool fft_long_enabled() {
  static const int on = env_int("VX_FFT_LONG", 1);
  return on != 0;
}

// Contiguous line FFT: register passes when the length has a kernel, else the
// shared-memory stage engine.
template <class Loader, class Storer>
int launch_fft_contig(const FftPlan& p, const Loader& ld, const Storer& st, int n_lines, int n_in, int n_out,
                      bool inv, cudaStream_t s) {
  if (fft_long_enabled() && !p.bluestein && fft_long_supported(p.n))
    return launch_fft_long(p, ld, st, n_lines, n_in, n_out, inv, s);
  if (blue_reg_supported(p)) return launch_blue_reg(p, ld, st, n_lines, n_in, n_out, inv, s);
  return launch_fft_lines(p, ld, st, n_lines, n_in, n_out, inv, true, s);
}

}  // namespace vx

namespace vx {
// drop-in for launch_fft_lines: contiguous lines take the register passes
template <class Loader, class Storer>
int launch_fft_auto(const FftPlan& p, const Loader& ld, const Storer& st, int n_lines, int n_in, int n_out,
                    bool inv, bool contig, cudaStream_t s) {
  if (contig) return launch_fft_contig(p, ld, st, n_lines, n_in, n_out, inv, s);
  return launch_fft_lines(p, ld, st, n_lines, n_in, n_out, inv, false, s);
}
}  // namespace vx
