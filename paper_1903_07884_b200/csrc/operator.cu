// Three-level Toeplitz operator N on the padded grid (reference operator.py).
//
// apply = 5 launches over the pruned padded FFT:
//   K1  x-forward   lines (c,z,y) of x, zero-pad nx -> px            -> A (3,nz,ny,px)
//   K2  y-forward   strided lines, pad ny -> py, only z < nz          -> B (3,nz,py,px)
//   K3  z-forward + 9-term spectral multiply (6 unique spectra) + z-inverse,
//       crop z < nz, 1/(px py pz) folded in                           -> B (in place)
//   K4  y-inverse   crop y < ny                                       -> A
//   K5  x-inverse   crop x < nx, epilogue y = x - m .* (N x)          -> y
// Zero padding and cropping happen in the loaders/storers, so the padded
// volume is only touched where it carries data.
#include "fft_lines.cuh"

namespace vx {

// Loader for the plan: line l = (p, iz, iy) of the padded grid, generator
// embedded in its circulant extension (reference operator.py:21-41).
struct LoadEmbed {
  const double2* __restrict__ g;
  long sp, sz, sy, sx;
  int nx, ny, nz, px, py, pz;
  __device__ __forceinline__ static int off(int i, int n, int P) {
    if (i < n) return i;
    if (i > P - n) return i - P;
    return INT32_MIN;
  }
  __device__ __forceinline__ long line_base(int l) const {
    const int p = l / (pz * py);
    const int r = l - p * pz * py;
    const int iz = r / py, iy = r - (r / py) * py;
    const int dz = off(iz, nz, pz), dy = off(iy, ny, py);
    if (dz == INT32_MIN || dy == INT32_MIN) return -1;
    return p * sp + (long)(dz + nz - 1) * sz + (long)(dy + ny - 1) * sy;
  }
  __device__ __forceinline__ double2 operator()(long b, int e) const {
    if (b < 0) return cmk(0.0, 0.0);
    const int dx = off(e, nx, px);
    if (dx == INT32_MIN) return cmk(0.0, 0.0);
    return __ldg(g + b + (long)(dx + nx - 1) * sx);
  }
};

__constant__ int c_pair_of[9] = {0, 1, 2, 1, 3, 4, 2, 4, 5};

// K3: per column (ky,kx) of the padded spectrum: forward z-DFT of the three
// components, y_a = sum_b S[PAIR_OF[a,b]] x_b, inverse z-DFT, crop.
template <int RMAX>
__global__ void __launch_bounds__(512, (RMAX <= 8 ? 2 : 1))
    op_zmul_kernel(FftPlan pzp, double2* __restrict__ B, const double2* __restrict__ S, int nz, long cols,
                   int W, FastDiv fdW3, double scale) {
  extern __shared__ double2 smem[];
  const int Pz = pzp.L;
  const int W3 = 3 * W;
  const long col0 = (long)blockIdx.x * W;
  SmemLay lay{W3, 1};
  double2* twsm = smem + (size_t)Pz * W3;
  fft_load_twiddles(pzp, twsm);
  for (int i = threadIdx.x; i < Pz * W3; i += blockDim.x) {
    const int e = i / W3, lw = i - e * W3;
    const int c = lw / W, w = lw - c * W;
    const long col = col0 + w;
    double2 v = cmk(0.0, 0.0);
    if (e < nz && col < cols) v = __ldg(B + ((long)c * nz + e) * cols + col);
    smem[lw + e * W3] = v;
  }
  __syncthreads();
  fft_dif<RMAX>(smem, lay, W3, fdW3, pzp, twsm, -1.0);  // natural -> digit-reversed positions
  for (int i = threadIdx.x; i < Pz * W; i += blockDim.x) {
    const int e = i / W, w = i - e * W;  // e = smem position
    const long col = col0 + w;
    if (col >= cols) continue;
    double2* q = smem + e * W3 + w;
    const double2 x0 = q[0], x1 = q[W], x2 = q[2 * W];
    const int kz = __ldg(pzp.k_of + e);
    const long so = (long)kz * cols + col, sstr = (long)Pz * cols;
    double2 s[6];
#pragma unroll
    for (int p = 0; p < 6; ++p) s[p] = ld_stream(S + p * sstr + so);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      double2 acc = cmul(s[c_pair_of[3 * a + 0]], x0);
      cfma(acc, s[c_pair_of[3 * a + 1]], x1);
      cfma(acc, s[c_pair_of[3 * a + 2]], x2);
      q[a * W] = cscale(acc, scale);
    }
  }
  __syncthreads();
  fft_dit<RMAX>(smem, lay, W3, fdW3, pzp, twsm, 1.0);  // digit-reversed -> natural
  for (int i = threadIdx.x; i < nz * W3; i += blockDim.x) {
    const int e = i / W3, lw = i - e * W3;
    const int c = lw / W, w = lw - c * W;
    const long col = col0 + w;
    if (col < cols) B[((long)c * nz + e) * cols + col] = smem[lw + e * W3];
  }
}

static int check_dims(int nx, int ny, int nz, int px, int py, int pz) {
  VX_REQUIRE(nx >= 1 && ny >= 1 && nz >= 1, "grid dims must be >= 1");
  VX_REQUIRE(px >= 2 * nx - 1 && py >= 2 * ny - 1 && pz >= 2 * nz - 1,
             "padded dims (%d,%d,%d) must be >= 2n-1 for grid (%d,%d,%d)", px, py, pz, nx, ny, nz);
  VX_REQUIRE(fft_is_smooth(px) && fft_is_smooth(py) && fft_is_smooth(pz),
             "padded dims (%d,%d,%d) must be 13-smooth", px, py, pz);
  return VX_OK;
}

}  // namespace vx

using namespace vx;

extern "C" int vx_fft_lines(int n, int n_lines, int n_inner, const vx_c128* in, long in_os,
                            long in_is, long in_es, int n_in, vx_c128* out, long out_os,
                            long out_is, long out_es, int n_out, int inverse, double scale,
                            void* stream) {
  VX_REQUIRE(n >= 1 && n_lines >= 0 && n_inner >= 1, "bad fft_lines geometry");
  VX_REQUIRE(n_in >= 0 && n_in <= n && n_out >= 0 && n_out <= n, "n_in/n_out must be in [0, n]");
  FftPlan p;
  int st = fft_get_plan(n, &p);
  if (st) return st;
  LoadStrided ld{reinterpret_cast<const double2*>(in), {in_os, in_is, in_es, n_inner}};
  StoreStrided sv{reinterpret_cast<double2*>(out), {out_os, out_is, out_es, n_inner}, scale};
  const bool contig = (in_es == 1 && out_es == 1);
  return launch_fft_lines(p, ld, sv, n_lines, n_in, n_out, inverse != 0, contig, as_stream(stream));
}

extern "C" int vx_op_plan(int nx, int ny, int nz, int px, int py, int pz, const vx_c128* gen,
                          long g_sp, long g_sz, long g_sy, long g_sx, vx_c128* spectra,
                          void* stream) {
  int st = check_dims(nx, ny, nz, px, py, pz);
  if (st) return st;
  cudaStream_t s = as_stream(stream);
  FftPlan fx, fy, fz;
  if ((st = fft_get_plan(px, &fx)) || (st = fft_get_plan(py, &fy)) || (st = fft_get_plan(pz, &fz)))
    return st;
  double2* S = reinterpret_cast<double2*>(spectra);
  const long cols = (long)py * px;
  // x pass over every padded (p, z, y) line, generator embedded on load
  LoadEmbed le{reinterpret_cast<const double2*>(gen), g_sp, g_sz, g_sy, g_sx, nx, ny, nz, px, py, pz};
  StoreStrided sx{S, {px, 0, 1, 1}, 1.0};
  if ((st = launch_fft_lines(fx, le, sx, 6 * pz * py, px, px, false, true, s))) return st;
  // y pass (in place), lines (p,z) x kx
  LoadStrided ly{S, {cols, 1, px, px}};
  StoreStrided sy{S, {cols, 1, px, px}, 1.0};
  if ((st = launch_fft_lines(fy, ly, sy, 6 * pz * px, py, py, false, false, s))) return st;
  // z pass (in place), lines p x (ky,kx)
  LoadStrided lz{S, {(long)pz * cols, 1, cols, (int)cols}};
  StoreStrided sz{S, {(long)pz * cols, 1, cols, (int)cols}, 1.0};
  return launch_fft_lines(fz, lz, sz, (int)(6 * cols), pz, pz, false, false, s);
}

extern "C" int vx_op_padded_length(int n) {
  // 2n when it is 7-smooth (the reference grid), else the smallest 7-smooth
  // length >= 2n-1: every such length gives the same linear convolution, and
  // radices <= 8 keep the transforms in the low-register kernel variants.
  auto smooth7 = [](int m) {
    for (int p : {2, 3, 5, 7})
      while (m % p == 0) m /= p;
    return m == 1;
  };
  if (smooth7(2 * n)) return 2 * n;
  int m = 2 * n - 1;
  while (!smooth7(m)) ++m;
  return m;
}

extern "C" long vx_op_work_elems(int nx, int ny, int nz, int px, int py, int pz) {
  (void)pz;
  return 3L * nz * px * ((long)ny + py);
}

namespace vx {

// K1: forward x-DFT of nlines contiguous x-lines, zero-padded nx -> px.
static int op_x_forward(const FftPlan& fx, int nx, int px, int nlines, const double2* X, double2* A,
                        cudaStream_t s) {
  LoadStrided ld{X, {nx, 0, 1, 1}};
  StoreStrided sv{A, {px, 0, 1, 1}, 1.0};
  return launch_fft_lines(fx, ld, sv, nlines, nx, px, false, true, s);
}

// K2-K4 on nkx x-frequency columns held as A (3, nz, ny, nkx): y-DFT (pad ny ->
// py), z-DFT + spectral multiply + inverse z-DFT (crop nz), inverse y-DFT
// (crop ny), result back in A.  Spectra for these columns: (6, pz, py, nkx).
// `scale` = 1/(px py pz) of the full transform.
static int op_yz(const FftPlan& fy, const FftPlan& fz, int ny, int nz, int nkx, int py, int pz,
                 const double2* spectra, double2* A, double2* B, double scale, cudaStream_t s) {
  int st;
  const long cols = (long)py * nkx;
  {
    LoadStrided ld{A, {(long)ny * nkx, 1, nkx, nkx}};
    StoreStrided sv{B, {cols, 1, nkx, nkx}, 1.0};
    if ((st = launch_fft_lines(fy, ld, sv, 3 * nz * nkx, ny, py, false, false, s))) return st;
  }
  {
    static const int zw = env_int("VX_ZMUL_W", 64);
    int W = zw;
    while (W > 1 && (long)W > cols) W /= 2;
    const size_t smem = ((size_t)3 * W * fz.L + 64 + fz.nhi) * sizeof(double2);
    int thr = fft_threads_for(fz, 3 * W);
    auto kern = fft_max_radix(fz) <= 8 ? op_zmul_kernel<8> : op_zmul_kernel<13>;
    if (smem > 48 * 1024)
      VX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<div_up(cols, W), thr, smem, s>>>(fz, B, spectra, nz, cols, W, FastDiv(3 * W), scale);
    VX_CHECK_LAUNCH("op_zmul_kernel");
  }
  {
    LoadStrided ld{B, {cols, 1, nkx, nkx}};
    StoreStrided sv{A, {(long)ny * nkx, 1, nkx, nkx}, 1.0};
    if ((st = launch_fft_lines(fy, ld, sv, 3 * nz * nkx, py, ny, true, false, s))) return st;
  }
  return VX_OK;
}

// K5: inverse x-DFT of nlines lines (global line index line0 + l), crop to nx,
// epilogue y = x - m .* v (m indexed by the global voxel) or y = v.
static int op_x_inverse(const FftPlan& fx, int nx, int px, int nlines, long line0, long nvox,
                        const double2* A, const double2* X, const double2* m, double2* Y, cudaStream_t s) {
  LoadStrided ld{A, {px, 0, 1, 1}};
  StoreSystem sv{Y, X, m, nx, nvox, 1.0, line0 * nx};
  return launch_fft_lines(fx, ld, sv, nlines, px, nx, true, true, s);
}

}  // namespace vx

extern "C" int vx_op_apply(int nx, int ny, int nz, int px, int py, int pz, const vx_c128* spectra,
                           const vx_c128* m, const vx_c128* x, vx_c128* y, vx_c128* work,
                           void* stream) {
  int st = check_dims(nx, ny, nz, px, py, pz);
  if (st) return st;
  cudaStream_t s = as_stream(stream);
  Span span("op_apply", s);
  FftPlan fx, fy, fz;
  if ((st = fft_get_plan(px, &fx)) || (st = fft_get_plan(py, &fy)) || (st = fft_get_plan(pz, &fz)))
    return st;
  const double2* X = reinterpret_cast<const double2*>(x);
  double2* A = reinterpret_cast<double2*>(work);
  double2* B = A + 3L * nz * ny * px;
  const int lines_xyz = 3 * nz * ny;
  if ((st = op_x_forward(fx, nx, px, lines_xyz, X, A, s))) return st;
  if ((st = op_yz(fy, fz, ny, nz, px, py, pz, reinterpret_cast<const double2*>(spectra), A, B,
                  1.0 / ((double)px * py * pz), s)))
    return st;
  return op_x_inverse(fx, nx, px, lines_xyz, 0, (long)nx * ny * nz, A, X,
                      reinterpret_cast<const double2*>(m), reinterpret_cast<double2*>(y), s);
}

extern "C" int vx_op_x_forward(int nx, int px, int nlines, const vx_c128* x, vx_c128* A, void* stream) {
  VX_REQUIRE(nx >= 1 && px >= nx && nlines >= 0, "bad x-forward arguments");
  FftPlan fx;
  int st = fft_get_plan(px, &fx);
  if (st) return st;
  return op_x_forward(fx, nx, px, nlines, reinterpret_cast<const double2*>(x),
                      reinterpret_cast<double2*>(A), as_stream(stream));
}

extern "C" long vx_op_yz_work_elems(int ny, int nz, int nkx, int py) {
  (void)ny;
  return 3L * nz * py * nkx;
}

extern "C" int vx_op_yz(int ny, int nz, int nkx, int px, int py, int pz, const vx_c128* spectra_local,
                        vx_c128* A, vx_c128* work, void* stream) {
  VX_REQUIRE(ny >= 1 && nz >= 1 && nkx >= 0, "bad yz arguments");
  VX_REQUIRE(fft_is_smooth(py) && fft_is_smooth(pz), "padded dims must be 13-smooth");
  if (nkx == 0) return VX_OK;
  FftPlan fy, fz;
  int st;
  if ((st = fft_get_plan(py, &fy)) || (st = fft_get_plan(pz, &fz))) return st;
  return op_yz(fy, fz, ny, nz, nkx, py, pz, reinterpret_cast<const double2*>(spectra_local),
               reinterpret_cast<double2*>(A), reinterpret_cast<double2*>(work),
               1.0 / ((double)px * py * pz), as_stream(stream));
}

extern "C" int vx_op_x_inverse(int nx, int ny, int nz, int px, int nlines, long line0,
                               const vx_c128* A, const vx_c128* m, const vx_c128* x_local,
                               vx_c128* y_local, void* stream) {
  VX_REQUIRE(nx >= 1 && px >= nx && nlines >= 0 && line0 >= 0, "bad x-inverse arguments");
  FftPlan fx;
  int st = fft_get_plan(px, &fx);
  if (st) return st;
  return op_x_inverse(fx, nx, px, nlines, line0, (long)nx * ny * nz, reinterpret_cast<const double2*>(A),
                      reinterpret_cast<const double2*>(x_local), reinterpret_cast<const double2*>(m),
                      reinterpret_cast<double2*>(y_local), as_stream(stream));
}
