// Generic batched line-FFT kernel: W lines per CTA, shared-memory transform,
// templated loader (zero-pad / Chan / embed hooks) and storer (crop / scale /
// operator epilogue hooks) so pads, crops and elementwise epilogues never
// cost an extra HBM round trip.
#pragma once

#include "fft.cuh"

namespace vx {

// Line l = (o, i) with o = l / n_inner, i = l % n_inner; element e at
// base + o*os + i*is + e*es.
struct LineAddr {
  long os, is, es;
  int n_inner;
  __device__ __forceinline__ long base(int l) const {
    const int o = l / n_inner;
    return (long)o * os + (long)(l - o * n_inner) * is;
  }
};

struct LoadStrided {
  const double2* __restrict__ p;
  LineAddr a;
  __device__ __forceinline__ long line_base(int l) const { return a.base(l); }
  __device__ __forceinline__ double2 operator()(long b, int e) const { return __ldg(p + b + e * a.es); }
};

// T. Chan optimal circulant generator from a (2n-1)-long offset line
// (reference circulant.py:61-73): c_0 = t_0, c_s = ((n-s) t_s + s t_{s-n}) / n.
struct LoadChan {
  const double2* __restrict__ p;
  LineAddr a;
  int n;
  __device__ __forceinline__ long line_base(int l) const { return a.base(l); }
  __device__ __forceinline__ double2 operator()(long b, int s) const {
    const double2 tp = __ldg(p + b + (long)(n - 1 + s) * a.es);
    if (s == 0) return tp;
    const double2 tn = __ldg(p + b + (long)(s - 1) * a.es);
    const double fn = (double)n, ws = (double)(n - s), wt = (double)s;
    return cmk((ws * tp.x + wt * tn.x) / fn, (ws * tp.y + wt * tn.y) / fn);
  }
};

struct StoreStrided {
  double2* __restrict__ p;
  LineAddr a;
  double scale;
  __device__ __forceinline__ long line_base(int l) const { return a.base(l); }
  __device__ __forceinline__ void operator()(long b, int e, double2 v) const {
    p[b + e * a.es] = cscale(v, scale);
  }
};

// Contiguous-line storer with the operator epilogue
// y = x - m .* (scale*v)   (reference operator.py:101-105), or y = scale*v.
struct StoreSystem {
  double2* __restrict__ y;
  const double2* __restrict__ x;
  const double2* __restrict__ m;  // may be null -> apply_n
  long pitch;                     // = nx
  long nvox;                      // = N (m is broadcast over the 3 components)
  double scale;
  long moff = 0;                  // global index of this slice's first element (sharded runs)
  __device__ __forceinline__ long line_base(int l) const { return (long)l * pitch; }
  __device__ __forceinline__ void operator()(long b, int e, double2 v) const {
    const long i = b + e;
    v = cscale(v, scale);
    if (m) {
      // a line never straddles a component (nvox is a multiple of pitch) and the global index is
      // below 3 nvox (three field components): the voxel index without a 64-bit modulo per element
      long gi = moff + b;
      if (gi >= 2 * nvox) gi -= 2 * nvox;
      else if (gi >= nvox) gi -= nvox;
      const double2 mv = __ldg(m + gi + e);
      const double2 xv = __ldg(x + i);
      v = csub(xv, cmul(mv, v));
    }
    y[i] = v;
  }
};

// RMAX = largest radix compiled in: 8 (radices 2..8, 3, 5, 7 -> ~64 registers,
// two 512-thread CTAs per SM) or 13 (adds the 11/13 codelets).
template <class Loader, class Storer, int RMAX>
__global__ void __launch_bounds__(RMAX <= 8 ? 1024 : 512, 1)
    fft_lines_kernel(FftPlan p, Loader ld, Storer st, int n_lines, int W, FastDiv fdW, int n_in, int n_out,
                     int inv, int contig) {
  extern __shared__ double2 smem[];
  double2* twsm = smem + (size_t)W * p.L;
  long* lbase_in = reinterpret_cast<long*>(twsm + 64 + p.nhi);
  long* lbase_out = lbase_in + W;
  fft_load_twiddles(p, twsm);
  const int l0 = blockIdx.x * W;
  const int L = p.L;
  SmemLay lay = contig ? SmemLay{1, L} : SmemLay{W, 1};
  for (int w = threadIdx.x; w < W; w += blockDim.x) {
    const int l = l0 + w;
    lbase_in[w] = (l < n_lines) ? ld.line_base(l) : 0;
    lbase_out[w] = (l < n_lines) ? st.line_base(l) : 0;
  }
  __syncthreads();
  const int total = W * L;
  // 4 independent global loads in flight per thread before their smem stores
  constexpr int U = 4;
  for (int i0 = threadIdx.x; i0 < total; i0 += U * blockDim.x) {
    double2 v[U];
    int pos[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * blockDim.x;
      pos[u] = -1;
      v[u] = cmk(0.0, 0.0);
      if (i < total) {
        int w, e;
        if (contig) { w = i / L; e = i - w * L; }
        else        { e = i / W; w = i - e * W; }
        pos[u] = w * lay.ldw + e * lay.lde;
        if (e < n_in && l0 + w < n_lines) v[u] = fft_pre(p, e, ld(lbase_in[w], e), inv);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (pos[u] >= 0) smem[pos[u]] = v[u];
  }
  __syncthreads();
  fft_exec<RMAX>(smem, lay, W, fdW, p, twsm, inv);
  const int tot_out = W * n_out;
  for (int i = threadIdx.x; i < tot_out; i += blockDim.x) {
    int w, e;
    if (contig) { w = i / n_out; e = i - w * n_out; }
    else        { e = i / W;     w = i - e * W; }
    if (l0 + w < n_lines)
      st(lbase_out[w], e, fft_post(p, e, smem[w * lay.ldw + fft_out_pos(p, e) * lay.lde], inv));
  }
}

// Choose lines-per-CTA and threads for a line FFT of executed length L.
struct LineLaunch {
  int W, threads;
  size_t smem;
};

inline int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

inline int pick_line_launch(const FftPlan& p, bool contig, int n_lines, LineLaunch* out) {
  const int budget = device_smem_optin() - 1024;
  static const int contig_elems = env_int("VX_FFT_CONTIG_ELEMS", 4096);
  static const int strided_w = env_int("VX_FFT_STRIDED_W", 16);
  static const int strided_kb = env_int("VX_FFT_STRIDED_KB", 96);
  int W;
  if (contig) {
    W = (int)(contig_elems / p.L);  // ~64 KB of data per CTA
    if (W < 1) W = 1;
  } else {
    W = strided_w;
    while (W > 1 && (size_t)W * p.L * sizeof(double2) > (size_t)strided_kb * 1024) W /= 2;
  }
  if (W > n_lines) W = n_lines > 0 ? n_lines : 1;
  // a CTA that fills the SM's shared memory alone gets up to 1024 threads
  // (radix <= 8 kernels fit 64 registers): the stages are smem-latency bound
  static const int max_thr = env_int("VX_FFT_MAXTHR", 1024);
  for (;;) {
    size_t smem = ((size_t)W * p.L + 64 + p.nhi) * sizeof(double2) + 2 * W * sizeof(long);
    int thr = fft_threads_for(p, W);
    if (fft_max_radix(p) <= 8 && smem > (size_t)budget / 2 && max_thr > 512) {
      long t2 = ((long)W * p.L / 4 + 31) / 32 * 32;
      thr = (int)(t2 < max_thr ? (t2 > thr ? t2 : thr) : max_thr);
    }
    if (smem <= (size_t)budget) {
      out->W = W;
      out->threads = thr;
      out->smem = smem;
      return VX_OK;
    }
    if (W == 1) break;
    W = W / 2;
  }
  set_error("FFT length %d (executed %d) does not fit one CTA's shared memory", p.n, p.L);
  return VX_EINVAL;
}

template <class Loader, class Storer>
int launch_fft_lines(const FftPlan& p, const Loader& ld, const Storer& st, int n_lines, int n_in,
                     int n_out, bool inv, bool contig, cudaStream_t stream) {
  if (n_lines <= 0) return VX_OK;
  LineLaunch ll;
  int s = pick_line_launch(p, contig, n_lines, &ll);
  if (s) return s;
  auto kern = fft_max_radix(p) <= 8 ? fft_lines_kernel<Loader, Storer, 8>
                                    : fft_lines_kernel<Loader, Storer, 13>;
  if (ll.smem > 48 * 1024)
    VX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ll.smem));
  kern<<<div_up(n_lines, ll.W), ll.threads, ll.smem, stream>>>(p, ld, st, n_lines, ll.W, FastDiv(ll.W),
                                                                n_in, n_out, inv ? 1 : 0, contig ? 1 : 0);
  VX_CHECK_LAUNCH("fft_lines_kernel");
  return VX_OK;
}

}  // namespace vx
