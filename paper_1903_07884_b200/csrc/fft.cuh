// Shared-memory mixed-radix FFT engine (sm_100a, complex128).
//
// A CTA loads W lines of one batched 1-D DFT into shared memory, runs
// in-place mixed-radix stages (decimation in frequency; its transpose, the
// decimation-in-time pass, for inverse transforms that consume digit-reversed
// spectra), and writes the lines back through a user "storer" that reads the
// digit-reversed positions.  Radices 2,4,8 (special) and 3,5,7,11,13
// (symmetric odd-prime codelet); any other length goes through Bluestein
// (chirp-z) on a smooth length M >= 2n-1, still entirely in shared memory.
//
// Convention is scipy's (reference operator.py:89,97 / circulant.py:182,187):
// forward X_k = sum_j x_j e^{-2 pi i jk/n}, inverse unnormalised here (the
// caller folds 1/n into its storer).
#pragma once

#include "common.cuh"

namespace vx {

constexpr int FFT_MAX_STAGES = 24;

// Division by a runtime-invariant divisor with one multiply-high (the stage
// loops would otherwise spend most of their issue slots in integer division).
// Valid for numerators < 2^31.
struct FastDiv {
  unsigned d, mul, shr;
  __host__ __device__ FastDiv() : d(1), mul(0), shr(0) {}
  __host__ explicit FastDiv(unsigned dv) : d(dv) {
    unsigned l = 0;
    while ((1ull << l) < dv) ++l;
    shr = l;
    mul = (unsigned)(((1ull << 32) * ((1ull << l) - dv)) / dv + 1);
  }
  __device__ __forceinline__ unsigned div(unsigned n) const {
    const unsigned long long t = (unsigned long long)__umulhi(n, mul) + n;
    return (unsigned)(t >> shr);
  }
};

struct FftPlan {
  int n;          // DFT length
  int L;          // executed length: n (direct) or M (Bluestein)
  int bluestein;  // 0/1
  int nst;        // number of radix stages of the length-L transform
  int radix[FFT_MAX_STAGES];
  const double2* tw;        // [L]  exp(-2 pi i m / L)
  const int* pos_of;        // [L]  smem position of frequency k after the DIF
  const int* k_of;          // [L]  frequency held at smem position pos after the DIF
  const double2* chirp;     // [n]  exp(-pi i j^2 / n)                 (Bluestein)
  const double2* bhat_rev;  // [L]  FFT_L(conj chirp, wrapped)/L at DIF positions
  const double2* tw_hi;     // [nhi] exp(-2 pi i 64 a / L)   (two-level twiddles:
  const double2* tw_lo;     // [64]  exp(-2 pi i b / L)       w^t = hi[t>>6] * lo[t&63])
  int nhi;
  // register Bluestein (fft_blue.cuh): convolution length R*R >= 2n-1 with R a register DFT length
  int blue_R;                // 0: none
  const double2* blue_bhat;  // [R*R] FFT_{R^2}(conj chirp, wrapped) / R^2, natural order
  const double2* blue_tw;    // [R*R] exp(-2 pi i j / R^2)
  FastDiv fd_m[FFT_MAX_STAGES];   // butterfly span m of stage st (DIF order)
  FastDiv fd_nb[FFT_MAX_STAGES];  // butterflies per line L / R_st
};

// Host: cached plan for length n on the current device (thread-safe).
int fft_get_plan(int n, FftPlan* out);
// Host: a 13-smooth length >= n (used for the operator padding).
int fft_good_length(int n);
bool fft_is_smooth(int n);

// Smem element (w, e) lives at s[w*ldw + e*lde].
struct SmemLay {
  int lde, ldw;
};

// ------------------------------------------------------------------ codelets
// cos/sin(2 pi m / R) for the odd-prime codelets, in constant memory
// (indices are compile-time after unrolling -> constant-bank operands).
__constant__ double c_rt3[2][3] = {{1.0, -0.5, -0.5}, {0.0, 0.86602540378443864676, -0.86602540378443864676}};
__constant__ double c_rt5[2][5] = {
    {1.0, 0.30901699437494742410, -0.80901699437494742410, -0.80901699437494742410, 0.30901699437494742410},
    {0.0, 0.95105651629515357212, 0.58778525229247312917, -0.58778525229247312917, -0.95105651629515357212}};
__constant__ double c_rt7[2][7] = {
    {1.0, 0.62348980185873353053, -0.22252093395631440429, -0.90096886790241912624,
     -0.90096886790241912624, -0.22252093395631440429, 0.62348980185873353053},
    {0.0, 0.78183148246802980871, 0.97492791218182360702, 0.43388373911755812048,
     -0.43388373911755812048, -0.97492791218182360702, -0.78183148246802980871}};
__constant__ double c_rt11[2][11] = {
    {1.0, 0.84125353283118116886, 0.41541501300188642553, -0.14231483827328514044,
     -0.65486073394528506406, -0.95949297361449738989, -0.95949297361449738989,
     -0.65486073394528506406, -0.14231483827328514044, 0.41541501300188642553,
     0.84125353283118116886},
    {0.0, 0.54064081745559758210, 0.90963199535451837141, 0.98982144188093273238,
     0.75574957435425828377, 0.28173255684142969771, -0.28173255684142969771,
     -0.75574957435425828377, -0.98982144188093273238, -0.90963199535451837141,
     -0.54064081745559758210}};
__constant__ double c_rt13[2][13] = {
    {1.0, 0.88545602565320989590, 0.56806474673115580251, 0.12053668025532305335,
     -0.35460488704253562597, -0.74851074817110109863, -0.97094181742605202716,
     -0.97094181742605202716, -0.74851074817110109863, -0.35460488704253562597,
     0.12053668025532305335, 0.56806474673115580251, 0.88545602565320989590},
    {0.0, 0.46472317204376854566, 0.82298386589365639458, 0.99270887409805399280,
     0.93501624268541482344, 0.66312265824079520238, 0.23931566428755776715,
     -0.23931566428755776715, -0.66312265824079520238, -0.93501624268541482344,
     -0.99270887409805399280, -0.82298386589365639458, -0.46472317204376854566}};

template <int R>
__device__ __forceinline__ double root_c(int m) {
  if constexpr (R == 3) return c_rt3[0][m];
  else if constexpr (R == 5) return c_rt5[0][m];
  else if constexpr (R == 7) return c_rt7[0][m];
  else if constexpr (R == 11) return c_rt11[0][m];
  else return c_rt13[0][m];
}
template <int R>
__device__ __forceinline__ double root_s(int m) {
  if constexpr (R == 3) return c_rt3[1][m];
  else if constexpr (R == 5) return c_rt5[1][m];
  else if constexpr (R == 7) return c_rt7[1][m];
  else if constexpr (R == 11) return c_rt11[1][m];
  else return c_rt13[1][m];
}

// i*z with sign: sg=+1 -> i z, sg=-1 -> -i z
__device__ __forceinline__ double2 mul_i(double2 z, double sg) { return cmk(-sg * z.y, sg * z.x); }

// sgn = -1 forward, +1 inverse
template <int R>
__device__ __forceinline__ void dft_codelet(double2* v, double sgn) {
  if constexpr (R == 2) {
    double2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  } else if constexpr (R == 4) {
    double2 s02 = cadd(v[0], v[2]), d02 = csub(v[0], v[2]);
    double2 s13 = cadd(v[1], v[3]), d13 = csub(v[1], v[3]);
    double2 t = mul_i(d13, sgn);  // forward: -i d13
    v[0] = cadd(s02, s13);
    v[2] = csub(s02, s13);
    v[1] = cadd(d02, t);
    v[3] = csub(d02, t);
  } else if constexpr (R == 8) {
    const double h = 0.70710678118654752440;
    double2 a[4] = {v[0], v[2], v[4], v[6]};
    double2 b[4] = {v[1], v[3], v[5], v[7]};
    dft_codelet<4>(a, sgn);
    dft_codelet<4>(b, sgn);
    // twiddles w8^k, forward w8 = e^{-i pi/4}
    double2 b1 = cmk(h * (b[1].x - sgn * b[1].y), h * (b[1].y + sgn * b[1].x));
    double2 b2 = mul_i(b[2], sgn);
    double2 b3 = cmk(h * (-b[3].x - sgn * b[3].y), h * (-b[3].y + sgn * b[3].x));
    v[0] = cadd(a[0], b[0]);
    v[4] = csub(a[0], b[0]);
    v[1] = cadd(a[1], b1);
    v[5] = csub(a[1], b1);
    v[2] = cadd(a[2], b2);
    v[6] = csub(a[2], b2);
    v[3] = cadd(a[3], b3);
    v[7] = csub(a[3], b3);
  } else {
    // odd prime: X_k = x0 + sum_{j=1}^{(R-1)/2} (x_j + x_{R-j}) c_{jk} + sgn*i (x_j - x_{R-j}) s_{jk}
    constexpr int H = (R - 1) / 2;
    double2 sp[H], dm[H];
    double2 x0 = v[0];
    double2 tot = x0;
#pragma unroll
    for (int j = 1; j <= H; ++j) {
      sp[j - 1] = cadd(v[j], v[R - j]);
      dm[j - 1] = csub(v[j], v[R - j]);
      tot = cadd(tot, sp[j - 1]);
    }
    v[0] = tot;
#pragma unroll
    for (int k = 1; k <= H; ++k) {
      double2 re = x0, im = cmk(0.0, 0.0);
#pragma unroll
      for (int j = 1; j <= H; ++j) {
        const int m = (j * k) % R;
        const double c = root_c<R>(m), s = root_s<R>(m);
        re.x = fma(c, sp[j - 1].x, re.x);
        re.y = fma(c, sp[j - 1].y, re.y);
        im.x = fma(s, dm[j - 1].x, im.x);
        im.y = fma(s, dm[j - 1].y, im.y);
      }
      double2 t = mul_i(im, sgn);
      v[k] = cadd(re, t);
      v[R - k] = csub(re, t);
    }
  }
}

// In-place mixed-radix stages.  Every butterfly reads and writes the same R
// smem slots, so a thread needs only R values in registers and no barrier
// separates the read and write of a stage (one barrier per stage).
//
// DIF (Gentleman-Sande): natural order in -> digit-reversed order out
//   (position pos holds X[k_of[pos]]).
// DIT: digit-reversed in -> natural out (exact transpose of the DIF, so the
//   pair DIF -> pointwise -> DIT needs no permutation at all).
// Butterfly enumeration: line fastest for interleaved smem (lde != 1), butterfly
// fastest for line-contiguous smem.
// twiddle w_L^t from the two-level tables staged in shared memory
__device__ __forceinline__ double2 tw_get(const double2* twsm, int t) {
  return cmul(twsm[64 + (t >> 6)], twsm[t & 63]);
}

// v[r] *= w^(t0*r), r = 1..R-1 (w = e^{sgn 2 pi i / L}): two table lookups
// (w^t0 and w^(2 t0)), the rest by products of those -- the stage loops are
// shared-memory-bound and every lookup is two scattered smem loads.
// VX_TW_EXACT keeps one lookup per twiddle.
template <int R>
__device__ __forceinline__ void twiddle_row(double2* v, const double2* twsm, int t0, double sgn) {
#ifdef VX_TW_EXACT
#pragma unroll
  for (int r = 1; r < R; ++r) {
    double2 t = tw_get(twsm, t0 * r);
    t.y *= -sgn;
    v[r] = cmul(v[r], t);
  }
#else
  double2 w1 = tw_get(twsm, t0);
  w1.y *= -sgn;
  v[1] = cmul(v[1], w1);
  if constexpr (R > 2) {
    double2 w2 = tw_get(twsm, 2 * t0);
    w2.y *= -sgn;
    v[2] = cmul(v[2], w2);
    double2 wo = w1;  // odd powers w^(2k+1) = w^(2k-1) w^2, even ones w^(2k) = w^(2k-2) w^2
    double2 we = w2;
#pragma unroll
    for (int r = 3; r < R; ++r) {
      if (r & 1) { wo = cmul(wo, w2); v[r] = cmul(v[r], wo); }
      else       { we = cmul(we, w2); v[r] = cmul(v[r], we); }
    }
  }
#endif
}

template <int R, bool DIT>
__device__ __forceinline__ void fft_stage(double2* s, SmemLay lay, int W, const FastDiv& fdW, int n, int m,
                                          const FastDiv& fdm, const FastDiv& fdnb,
                                          const double2* __restrict__ tw, double sgn) {
  const int nb = n / R;
  const int total = nb * W;
  const int blockL = m * R;
  const int tws = n / blockL;  // twiddle table stride for w_{blockL}
  const bool bfast = (lay.lde == 1);
  const int st = m * lay.lde;
  for (int b = threadIdx.x; b < total; b += blockDim.x) {
    int w, f;
    if (bfast) { w = (int)fdnb.div(b); f = b - w * nb; }
    else       { f = (int)fdW.div(b);  w = b - f * W; }
    const int blk = (int)fdm.div(f), j = f - blk * m;
    double2* q = s + w * lay.ldw + (blk * blockL + j) * lay.lde;
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = q[r * st];
    if (DIT && j) twiddle_row<R>(v, tw, j * tws, sgn);
    dft_codelet<R>(v, sgn);
    if (!DIT && j) twiddle_row<R>(v, tw, j * tws, sgn);
#pragma unroll
    for (int r = 0; r < R; ++r) q[r * st] = v[r];
  }
  __syncthreads();
}

template <bool DIT, int RMAX>
__device__ __forceinline__ void fft_one_stage(int st, const FftPlan& p, const double2* twsm, double2* s,
                                              SmemLay lay, int W, const FastDiv& fdW, int m, double sgn) {
  const int n = p.L;
  const FastDiv& fm = p.fd_m[st];
  const FastDiv& fnb = p.fd_nb[st];
  switch (p.radix[st]) {
    case 2: fft_stage<2, DIT>(s, lay, W, fdW, n, m, fm, fnb, twsm, sgn); break;
    case 4: fft_stage<4, DIT>(s, lay, W, fdW, n, m, fm, fnb, twsm, sgn); break;
    case 8: fft_stage<8, DIT>(s, lay, W, fdW, n, m, fm, fnb, twsm, sgn); break;
    case 3: fft_stage<3, DIT>(s, lay, W, fdW, n, m, fm, fnb, twsm, sgn); break;
    case 5: fft_stage<5, DIT>(s, lay, W, fdW, n, m, fm, fnb, twsm, sgn); break;
    case 7: fft_stage<7, DIT>(s, lay, W, fdW, n, m, fm, fnb, twsm, sgn); break;
    default:
      if constexpr (RMAX >= 11) {
        if (p.radix[st] == 11) fft_stage<11, DIT>(s, lay, W, fdW, n, m, fm, fnb, twsm, sgn);
        else if (p.radix[st] == 13) fft_stage<13, DIT>(s, lay, W, fdW, n, m, fm, fnb, twsm, sgn);
      }
      break;
  }
}

// natural -> digit-reversed
// Stage the two-level twiddle tables of a plan into shared memory (64 + nhi
// entries); must be followed by a barrier before the transform.
__device__ __forceinline__ void fft_load_twiddles(const FftPlan& p, double2* twsm) {
  for (int i = threadIdx.x; i < 64 + p.nhi; i += blockDim.x)
    twsm[i] = i < 64 ? __ldg(p.tw_lo + i) : __ldg(p.tw_hi + (i - 64));
}

template <int RMAX = 13>
__device__ __forceinline__ void fft_dif(double2* s, SmemLay lay, int W, const FastDiv& fdW, const FftPlan& p,
                                        const double2* twsm, double sgn) {
  int m = p.L;
  for (int st = 0; st < p.nst; ++st) {
    m /= p.radix[st];
    fft_one_stage<false, RMAX>(st, p, twsm, s, lay, W, fdW, m, sgn);
  }
}

// digit-reversed -> natural
template <int RMAX = 13>
__device__ __forceinline__ void fft_dit(double2* s, SmemLay lay, int W, const FastDiv& fdW, const FftPlan& p,
                                        const double2* twsm, double sgn) {
  int m = 1;
  for (int st = p.nst - 1; st >= 0; --st) {
    fft_one_stage<true, RMAX>(st, p, twsm, s, lay, W, fdW, m, sgn);
    m *= p.radix[st];
  }
}

// Pre/post hooks: identity for direct plans; chirp multiply for Bluestein.
// inverse Bluestein uses conj(F(conj x)).
__device__ __forceinline__ double2 fft_pre(const FftPlan& p, int e, double2 v, bool inv) {
  if (!p.bluestein) return v;
  if (inv) v = cconj(v);
  return cmul(v, __ldg(p.chirp + e));
}
__device__ __forceinline__ double2 fft_post(const FftPlan& p, int e, double2 v, bool inv) {
  if (!p.bluestein) return v;
  v = cmul(v, __ldg(p.chirp + e));
  return inv ? cconj(v) : v;
}

// Full transform of W lines loaded in natural order (through fft_pre, zero
// padded to L).  Afterwards output element e of a line sits at smem position
// fft_out_pos(p, e) (digit-reversed for direct plans, natural for Bluestein).
template <int RMAX = 13>
__device__ __forceinline__ void fft_exec(double2* s, SmemLay lay, int W, const FastDiv& fdW, const FftPlan& p,
                                         const double2* twsm, bool inv) {
  if (!p.bluestein) {
    fft_dif<RMAX>(s, lay, W, fdW, p, twsm, inv ? 1.0 : -1.0);
    return;
  }
  fft_dif<RMAX>(s, lay, W, fdW, p, twsm, -1.0);
  const int total = W * p.L;
  for (int i = threadIdx.x; i < total; i += blockDim.x) {
    int w, e;
    if (lay.lde == 1) { w = i / p.L; e = i - w * p.L; }
    else              { e = i / W;   w = i - e * W; }
    double2* q = s + w * lay.ldw + e * lay.lde;
    *q = cmul(*q, __ldg(p.bhat_rev + e));
  }
  __syncthreads();
  fft_dit<RMAX>(s, lay, W, fdW, p, twsm, 1.0);
}

// largest radix of a plan (host and device)
__host__ __device__ inline int fft_max_radix(const FftPlan& p) {
  int r = 1;
  for (int i = 0; i < p.nst; ++i) r = p.radix[i] > r ? p.radix[i] : r;
  return r;
}

__device__ __forceinline__ int fft_out_pos(const FftPlan& p, int e) {
  return p.bluestein ? e : __ldg(p.pos_of + e);
}

// Host helper: a reasonable CTA size for W lines of executed length L.
int fft_threads_for(const FftPlan& p, int W);

}  // namespace vx
