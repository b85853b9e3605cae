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
#include "fft_long.cuh"
#include "fft_reg.cuh"

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

// PAIR_OF[a][b] (reference accel.py:41) as a constexpr so the spectral MAC
// indexes registers, not local memory
__host__ __device__ constexpr int pair_of(int a, int b) {
  return a == b ? (a == 0 ? 0 : (a == 1 ? 3 : 5)) : (a + b == 1 ? 1 : (a + b == 2 ? 2 : 4));
}
// parity of component p (xx,xy,xz,yy,yz,zz) under a sign flip of x / y / z
__host__ __device__ constexpr bool odd_x(int p) { return p == 1 || p == 2; }
__host__ __device__ constexpr bool odd_y(int p) { return p == 1 || p == 4; }
__host__ __device__ constexpr bool odd_z(int p) { return p == 2 || p == 4; }

// Compact (symmetry-reduced) spectra: for a parity-symmetric kernel
// S_p(-k) = +-S_p(k) on every axis, so only k <= P/2 is stored per axis,
// (Hz, Hy, Hx, 6) with H = P/2 + 1 -- 1/8 of the full spectra's bytes; the six
// components of one frequency are adjacent (96 bytes), so the three lanes of a
// column that each need three of them share the same L1 lines.
struct SpecView {
  const double2* S;
  int compact;
  int Pz, Py, Px, Hz, Hy, Hx;
  int Mx;  // x-mirror period (Px); huge for spectra compacted in y and z only (a rank's kx columns)
  FastDiv fdPx;
};

// K3: per column (ky,kx) of the padded spectrum: forward z-DFT of the three
// components, y_a = sum_b S[PAIR_OF[a,b]] x_b, inverse z-DFT, crop.
template <int RMAX>
__global__ void __launch_bounds__(512, (RMAX <= 8 ? 2 : 1))
    op_zmul_kernel(FftPlan pzp, double2* __restrict__ B, SpecView sv, int nz, long cols, int W, FastDiv fdW3,
                   double scale) {
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
    double2 sp[6];
    if (!sv.compact) {
      const long so = (long)kz * cols + col, sstr = (long)Pz * cols;
#pragma unroll
      for (int p = 0; p < 6; ++p) sp[p] = ld_stream(sv.S + p * sstr + so);
    } else {
      const int ky = (int)sv.fdPx.div((unsigned)col), kx = (int)(col - (long)ky * sv.Px);
      const bool mz = 2 * kz > sv.Pz, my = 2 * ky > sv.Py, mx = 2 * kx > sv.Mx;
      const int kzs = mz ? sv.Pz - kz : kz, kys = my ? sv.Py - ky : ky, kxs = mx ? sv.Px - kx : kx;
      const long so = (((long)kzs * sv.Hy + kys) * sv.Hx + kxs) * 6;
      const long sstr = 1;
#pragma unroll
      for (int p = 0; p < 6; ++p) {
        double2 v = ld_stream(sv.S + p * sstr + so);
        const bool neg = (mx && odd_x(p)) ^ (my && odd_y(p)) ^ (mz && odd_z(p));
        sp[p] = neg ? cmk(-v.x, -v.y) : v;
      }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      double2 acc = cmul(sp[pair_of(a, 0)], x0);
      cfma(acc, sp[pair_of(a, 1)], x1);
      cfma(acc, sp[pair_of(a, 2)], x2);
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
  // columns (consecutive lines are adjacent in memory) of a two-pass length: register transforms
  static const int use_cols2 = env_int("VX_COLS2", 1);
  if (use_cols2 && !contig && in_is == 1 && out_is == 1 && !p.bluestein && p.L == n && cols2_supported(n)) {
    const double2* ip = reinterpret_cast<const double2*>(in);
    double2* op = reinterpret_cast<double2*>(out);
    return inverse ? launch_cols2<true>(p, ip, in_os, in_es, n_in, op, out_os, out_es, n_out, n_lines, n_inner,
                                        scale, as_stream(stream))
                   : launch_cols2<false>(p, ip, in_os, in_es, n_in, op, out_os, out_es, n_out, n_lines, n_inner,
                                         scale, as_stream(stream));
  }
  return launch_fft_auto(p, ld, sv, n_lines, n_in, n_out, inverse != 0, contig, as_stream(stream));
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
  if ((st = launch_fft_auto(fx, le, sx, 6 * pz * py, px, px, false, true, s))) return st;
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

// z padding: the reference's 2 nz whenever the pair kernel covers nz
extern "C" int vx_op_padded_length_z(int nz) {
  if (env_int("VX_ZPAIR", 0) && nz >= 1 && nz <= 16) return 2 * nz;
  return vx_op_padded_length(nz);
}

extern "C" long vx_op_work_elems(int nx, int ny, int nz, int px, int py, int pz) {
  (void)pz;
  return 3L * nz * px * ((long)ny + py);

}

namespace vx {

// K3 with register z-transforms: one thread per column (ky,kx), 64 columns
// per CTA.  Each component's z-line is transformed in registers one at a time
// (holding all three would spill) and parked in the thread's private slice of
// shared memory ([c][kz][thread]: conflict-free, no barriers), then the
// spectral multiply runs kz by kz, then the inverse transforms.
constexpr int ZR_T = 64;

template <int PZ>
__global__ void __launch_bounds__(ZR_T)
    op_zmul_reg_kernel(double2* __restrict__ B, SpecView sv, int nz, long cols, double scale) {
  extern __shared__ double2 zr_sm[];
  const int tid = threadIdx.x;
  long col = blockIdx.x * (long)ZR_T + tid;
  if (col >= cols) return;
  if (sv.compact) {
    // launch rows ky = 0, 1, Py-1, 2, Py-2, ...: a row and its mirror (same
    // compact spectra) run back to back, so the second read hits L2
    const int lr = (int)sv.fdPx.div((unsigned)col);
    const int ky = (lr == 0) ? 0 : ((lr & 1) ? (lr + 1) / 2 : sv.Py - lr / 2);
    col += (long)(ky - lr) * sv.Px;
  }
#pragma unroll 1
  for (int c = 0; c < 3; ++c) {
    double2 v[PZ];
#pragma unroll
    for (int e = 0; e < PZ; ++e) v[e] = (e < nz) ? __ldg(B + ((long)c * nz + e) * cols + col) : cmk(0.0, 0.0);
    reg_fft<PZ, false>(v);
#pragma unroll
    for (int e = 0; e < PZ; ++e) zr_sm[(c * PZ + e) * ZR_T + tid] = v[e];
  }
  long so0 = col, sstr = (long)PZ * cols, kstr = cols;
  bool my = false, mx = false;
  if (sv.compact) {
    const int ky = (int)sv.fdPx.div((unsigned)col), kx = (int)(col - (long)ky * sv.Px);
    my = 2 * ky > sv.Py;
    mx = 2 * kx > sv.Mx;
    so0 = ((long)(my ? sv.Py - ky : ky) * sv.Hx + (mx ? sv.Px - kx : kx)) * 6;
    sstr = 1;
    kstr = (long)sv.Hy * sv.Hx * 6;
  }
#pragma unroll 7
  for (int kz = 0; kz < PZ; ++kz) {
    double2 sp[6];
    if (!sv.compact) {
#pragma unroll
      for (int p = 0; p < 6; ++p) sp[p] = ld_stream(sv.S + p * sstr + (long)kz * kstr + so0);
    } else {
      const bool mz = 2 * kz > PZ;
      const long so = (long)(mz ? PZ - kz : kz) * kstr + so0;
#pragma unroll
      for (int p = 0; p < 6; ++p) {
        const double2 v = ld_stream(sv.S + p * sstr + so);
        const bool neg = (mx && odd_x(p)) ^ (my && odd_y(p)) ^ (mz && odd_z(p));
        sp[p] = neg ? cmk(-v.x, -v.y) : v;
      }
    }
    double2* q = zr_sm + kz * ZR_T + tid;
    const double2 x0 = q[0], x1 = q[PZ * ZR_T], x2 = q[2 * PZ * ZR_T];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      double2 acc = cmul(sp[pair_of(a, 0)], x0);
      cfma(acc, sp[pair_of(a, 1)], x1);
      cfma(acc, sp[pair_of(a, 2)], x2);
      q[a * PZ * ZR_T] = cscale(acc, scale);
    }
  }
#pragma unroll 1
  for (int c = 0; c < 3; ++c) {
    double2 v[PZ];
#pragma unroll
    for (int e = 0; e < PZ; ++e) v[e] = zr_sm[(c * PZ + e) * ZR_T + tid];
    reg_fft<PZ, true>(v);
#pragma unroll
    for (int e = 0; e < PZ; ++e)
      if (e < nz) B[((long)c * nz + e) * cols + col] = v[e];
  }
}

// K3 without shared memory: three lanes per column (ky,kx), one per field
// component.  Lane (c, j) of a warp (c = lane / 10, j = lane % 10; lanes 30, 31
// idle) holds component c's z-line of column j in registers, transforms it,
// and at each kz pulls the other two components' values with warp shuffles
// for y_c = sum_b S[PAIR_OF[c,b]] x_b.  No smem and ~1/3 of the registers of
// the one-thread-per-column kernel -> full occupancy; loads of the 3 spectra a
// lane needs hit L1 for the entries its column partners also use.
constexpr int ZS_COLS = 10;
#ifndef ZMUL_MINB_BIG
#define ZMUL_MINB_BIG 2
#endif
#ifndef ZMUL_MINB_SMALL
#define ZMUL_MINB_SMALL 2
#endif

// v or -v: XOR of the sign bits (m = 0 or 0x80000000)
__device__ __forceinline__ double2 sign_flip(double2 v, unsigned m) {
  return cmk(__hiloint2double(__double2hiint(v.x) ^ (int)m, __double2loint(v.x)),
             __hiloint2double(__double2hiint(v.y) ^ (int)m, __double2loint(v.y)));
}

__device__ __forceinline__ double2 shfl_c(double2 v, int src) {
  return cmk(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

template <int PZ, bool COMPACT>
__global__ void __launch_bounds__(256, (PZ <= 8 ? 3 : (PZ <= 16 ? ZMUL_MINB_SMALL : ZMUL_MINB_BIG)))
    op_zmul_shfl_kernel(double2* __restrict__ B, SpecView sv, int nz, long cols, double scale) {
  const int lane = threadIdx.x & 31;
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const int c = lane < 3 * ZS_COLS ? lane / ZS_COLS : 2;
  const int j = lane < 3 * ZS_COLS ? lane - c * ZS_COLS : 0;
  long col = warp * ZS_COLS + j;
  const bool active = lane < 3 * ZS_COLS && col < cols;
  if (!active) col = 0;
  if constexpr (COMPACT) {
    // rows ky = 0, 1, Py-1, 2, Py-2, ...: a row and its mirror (same compact
    // spectra) run back to back, so the second read hits L2
    const int lr = (int)sv.fdPx.div((unsigned)col);
    const int ky = (lr == 0) ? 0 : ((lr & 1) ? (lr + 1) / 2 : sv.Py - lr / 2);
    col += (long)(ky - lr) * sv.Px;
  }
  double2 v[PZ];
  const double2* src = B + (long)c * nz * cols + col;
#pragma unroll
  for (int e = 0; e < PZ; ++e) v[e] = (active && e < nz) ? __ldg(src + (long)e * cols) : cmk(0.0, 0.0);
  reg_fft<PZ, false>(v);
  // spectra this lane needs, in the order own component c, then c+1, c+2 (mod 3):
  // PAIR_OF[c][c], PAIR_OF[c][c+1], PAIR_OF[c][c+2] -- the lane's own z-line needs no
  // shuffle, the partners' values come with two rotating shuffles instead of three broadcasts
  const int p0 = pair_of(c, c);
  const int p1 = pair_of(c, (c + 1) % 3);
  const int p2 = pair_of(c, (c + 2) % 3);
  const int la = ((c + 1) % 3) * ZS_COLS + j, lb = ((c + 2) % 3) * ZS_COLS + j;
  long so0 = col, sstr = (long)PZ * cols, kstr = cols;
  bool my = false, mx = false;
  if constexpr (COMPACT) {
    const int ky = (int)sv.fdPx.div((unsigned)col), kx = (int)(col - (long)ky * sv.Px);
    my = 2 * ky > sv.Py;
    mx = 2 * kx > sv.Mx;
    so0 = ((long)(my ? sv.Py - ky : ky) * sv.Hx + (mx ? sv.Px - kx : kx)) * 6;
    sstr = 1;
    kstr = (long)sv.Hy * sv.Hx * 6;
  }
  // sign of S_p at a mirrored (x, y) index; z mirror added per kz
  const bool n0 = (mx && odd_x(p0)) ^ (my && odd_y(p0));
  const bool n1 = (mx && odd_x(p1)) ^ (my && odd_y(p1));
  const bool n2 = (mx && odd_x(p2)) ^ (my && odd_y(p2));
  const double2* S0 = sv.S + p0 * sstr + so0;
  const double2* S1 = sv.S + p1 * sstr + so0;
  const double2* S2 = sv.S + p2 * sstr + so0;
  if constexpr (COMPACT) {
    // compact spectra: S(PZ - kz) = +-S(kz) (sign by the z parity of the
    // component), so kz and its mirror share ONE load of the three spectra --
    // the loads, not the arithmetic, fill the L1 data pipe of this kernel
    // signs as XOR masks on the high words (integer pipe) instead of FP64 negations / selects
    const unsigned m0 = n0 ? 0x80000000u : 0u, m1 = n1 ? 0x80000000u : 0u, m2 = n2 ? 0x80000000u : 0u;
    const unsigned zm0 = odd_z(p0) ? 0x80000000u : 0u, zm1 = odd_z(p1) ? 0x80000000u : 0u,
                   zm2 = odd_z(p2) ? 0x80000000u : 0u;
#pragma unroll
    for (int kz = 0; kz <= PZ / 2; ++kz) {
      const long ko = (long)kz * kstr;
      double2 s0 = __ldg(S0 + ko), s1 = __ldg(S1 + ko), s2 = __ldg(S2 + ko);
      s0 = sign_flip(s0, m0), s1 = sign_flip(s1, m1), s2 = sign_flip(s2, m2);
      {
        const double2 x0 = v[kz], x1 = shfl_c(v[kz], la), x2 = shfl_c(v[kz], lb);
        double2 acc = cmul(s0, x0);
        cfma(acc, s1, x1);
        cfma(acc, s2, x2);
        v[kz] = cscale(acc, scale);
      }
      const int km = PZ - kz;
      if (kz > 0 && km > kz && km < PZ) {
        s0 = sign_flip(s0, zm0), s1 = sign_flip(s1, zm1), s2 = sign_flip(s2, zm2);
        const double2 x0 = v[km], x1 = shfl_c(v[km], la), x2 = shfl_c(v[km], lb);
        double2 acc = cmul(s0, x0);
        cfma(acc, s1, x1);
        cfma(acc, s2, x2);
        v[km] = cscale(acc, scale);
      }
    }
  } else {
#pragma unroll
    for (int kz = 0; kz < PZ; ++kz) {
      const long ko = (long)kz * kstr;
      const double2 s0 = __ldg(S0 + ko), s1 = __ldg(S1 + ko), s2 = __ldg(S2 + ko);
      const double2 x0 = v[kz], x1 = shfl_c(v[kz], la), x2 = shfl_c(v[kz], lb);
      double2 acc = cmul(s0, x0);
      cfma(acc, s1, x1);
      cfma(acc, s2, x2);
      v[kz] = cscale(acc, scale);
    }
  }
  reg_fft<PZ, true>(v);
  if (active) {
    double2* dst = B + (long)c * nz * cols + col;
#pragma unroll
    for (int e = 0; e < PZ; ++e)
      if (e < nz) dst[(long)e * cols] = v[e];
  }
}

// K3 for the reference's own z padding pz = 2 nz: six lanes per column
// (component c, frequency parity par) -- lane = 10 c + 5 par + j, five
// columns per warp.  Because the z-line is zero beyond nz, the even and odd
// halves of the length-2nz spectrum are two independent length-nz DFTs,
//   X[2k] = DFT_nz(x)[k],  X[2k+1] = DFT_nz(w^z x)[k]   (w = e^{-2 pi i / 2nz}),
// and the cropped inverse is y[z] = IDFT_nz(Y_even)[z] + w^{-z} IDFT_nz(Y_odd)[z]
// (z < nz), one shuffle-add between the lane pair.  A lane holds nz values
// (11 at c1/c2 instead of 21): few registers, full occupancy, and fewer FP64
// instructions than one length-21 transform per component.
template <int NZ>
__global__ void __launch_bounds__(256)
    op_zpair_kernel(double2* __restrict__ B, SpecView sv, long cols, long nkx, double scale) {
  constexpr int PZ = 2 * NZ;
  __shared__ double2 twz[PZ];  // w^t, forward sign
  for (int t = threadIdx.x; t < PZ; t += blockDim.x) {
    double sn, cs;
    sincospi((double)t / NZ, &sn, &cs);
    twz[t] = cmk(cs, -sn);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const int lc = lane < 30 ? lane : 29;
  const int c = lc / 10, par = (lc / 5) & 1, j = lc % 5;
  long col = warp * 5 + j;
  const bool active = lane < 30 && col < cols;
  if (!active) col = 0;
  if (sv.compact) {
    const int lr = (int)sv.fdPx.div((unsigned)col);
    const int ky = (lr == 0) ? 0 : ((lr & 1) ? (lr + 1) / 2 : sv.Py - lr / 2);
    col += (long)(ky - lr) * sv.Px;
  }
  double2 v[NZ];
  const double2* src = B + (long)c * NZ * cols + col;
#pragma unroll
  for (int z = 0; z < NZ; ++z) v[z] = active ? __ldg(src + (long)z * cols) : cmk(0.0, 0.0);
  if (par) {
#pragma unroll
    for (int z = 1; z < NZ; ++z) v[z] = cmul(v[z], twz[z]);
  }
  reg_fft<NZ, false>(v);  // v[k] = X[2k + par]
  const int p0 = c == 0 ? 0 : (c == 1 ? 1 : 2);
  const int p1 = c == 0 ? 1 : (c == 1 ? 3 : 4);
  const int p2 = c == 0 ? 2 : (c == 1 ? 4 : 5);
  long so0, sstr, kstr;
  bool my = false, mx = false;
  if (sv.compact) {
    const int ky = (int)sv.fdPx.div((unsigned)col), kx = (int)(col - (long)ky * sv.Px);
    my = 2 * ky > sv.Py;
    mx = 2 * kx > sv.Mx;
    so0 = ((long)(my ? sv.Py - ky : ky) * sv.Hx + (mx ? sv.Px - kx : kx)) * 6;
    sstr = 1;
    kstr = (long)sv.Hy * sv.Hx * 6;
  } else {
    so0 = col;
    kstr = cols;
    sstr = (long)PZ * cols;
  }
  const bool n0 = (mx && odd_x(p0)) ^ (my && odd_y(p0));
  const bool n1 = (mx && odd_x(p1)) ^ (my && odd_y(p1));
  const bool n2 = (mx && odd_x(p2)) ^ (my && odd_y(p2));
  const double2* S0 = sv.S + p0 * sstr + so0;
  const double2* S1 = sv.S + p1 * sstr + so0;
  const double2* S2 = sv.S + p2 * sstr + so0;
  const int base = par * 5 + j;
#pragma unroll
  for (int k = 0; k < NZ; ++k) {
    const int kz = 2 * k + par;
    const bool mz = sv.compact && kz > NZ;
    const long ko = (long)(mz ? PZ - kz : kz) * kstr;
    double2 s0 = __ldg(S0 + ko), s1 = __ldg(S1 + ko), s2 = __ldg(S2 + ko);
    if (n0 ^ (mz && odd_z(p0))) s0 = cmk(-s0.x, -s0.y);
    if (n1 ^ (mz && odd_z(p1))) s1 = cmk(-s1.x, -s1.y);
    if (n2 ^ (mz && odd_z(p2))) s2 = cmk(-s2.x, -s2.y);
    const double2 x0 = shfl_c(v[k], base), x1 = shfl_c(v[k], 10 + base), x2 = shfl_c(v[k], 20 + base);
    double2 acc = cmul(s0, x0);
    cfma(acc, s1, x1);
    cfma(acc, s2, x2);
    v[k] = cscale(acc, scale);
  }
  reg_fft<NZ, true>(v);
  if (par) {
#pragma unroll
    for (int z = 1; z < NZ; ++z) v[z] = cmulc(v[z], twz[z]);
  }
  // pair sum: lanes 5 apart hold the even / odd halves of the same column
  constexpr int H = (NZ + 1) / 2;
  double2* dst = B + (long)c * NZ * cols + col;
#pragma unroll
  for (int z = 0; z < NZ; ++z) {
    const double2 o = shfl_c(v[z], par ? lane - 5 : lane + 5);
    if (active && ((z < H) == (par == 0))) dst[(long)z * cols] = cadd(v[z], o);
  }
  (void)nkx;
}

#define VX_ZPAIR_NZ(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16)

// opt-in (VX_ZPAIR=1): measured 0.37 ms vs 0.26 ms for op_zmul_shfl_kernel at c1
// (more load/shuffle instructions per column; the same FP64 work)
static bool zpair_supported(int nz, int pz) {
  static const int on = env_int("VX_ZPAIR", 0);
  return on && pz == 2 * nz && nz >= 1 && nz <= 16;
}

static int launch_zpair(int nz, double2* B, const SpecView& sv, long cols, long nkx, double scale, cudaStream_t s) {
  const long warps = (cols + 4) / 5;
  const unsigned g = div_up(warps, 8);
  switch (nz) {
#define VX_ZP_CASE(N) \
  case N:             \
    op_zpair_kernel<N><<<g, 256, 0, s>>>(B, sv, cols, nkx, scale); \
    break;
    VX_ZPAIR_NZ(VX_ZP_CASE)
#undef VX_ZP_CASE
    default:
      set_error("no z-pair kernel for nz = %d", nz);
      return VX_EINVAL;
  }
  VX_CHECK_LAUNCH("op_zpair_kernel");
  return VX_OK;
}

constexpr int REG_ZMUL_MAX = 32;  // longer z-lines spill; they keep the smem kernel

static int g_reg_fft = -1;  // -1: from VX_REG_FFT (default on); vx_op_reg_fft() overrides
static bool reg_fft_enabled() {
  if (g_reg_fft < 0) g_reg_fft = env_int("VX_REG_FFT", 1) != 0;
  return g_reg_fft != 0;
}

template <bool INV>
static int launch_reg_cols(int L, const double2* in, long in_os, long in_es, int n_in, double2* out, long out_os,
                           long out_es, int n_out, long ncols, int n_inner, double scale, cudaStream_t s) {
  if (ncols <= 0) return VX_OK;
  const unsigned grid = (unsigned)div_up(ncols, 128);
  const FastDiv fd((unsigned)n_inner);
  switch (L) {
#define VX_REG_LAUNCH(N)                                                                              \
  case N:                                                                                             \
    reg_cols_kernel<N, INV><<<grid, 128, 0, s>>>(in, in_os, in_es, n_in, out, out_os, out_es, n_out, \
                                                 ncols, fd, n_inner, scale);                          \
    break;
    VX_REG_LENGTHS(VX_REG_LAUNCH)
#undef VX_REG_LAUNCH
    default:
      set_error("no register FFT for length %d", L);
      return VX_EINVAL;
  }
  VX_CHECK_LAUNCH("reg_cols_kernel");
  return VX_OK;
}

static int launch_zmul_reg(int PZ, double2* B, const SpecView& sv, int nz, long cols, double scale,
                           cudaStream_t s) {
  static const int shfl = env_int("VX_ZMUL_SHFL", 1);
  if (shfl) {
    const long warps = (cols + ZS_COLS - 1) / ZS_COLS;
    const unsigned g = div_up(warps, 8);
    switch (PZ) {
#define VX_ZSH_LAUNCH(N)                                                           \
  case N:                                                                          \
    if constexpr (N <= REG_ZMUL_MAX) {                                                                  \
      if (sv.compact) op_zmul_shfl_kernel<N, true><<<g, 256, 0, s>>>(B, sv, nz, cols, scale);           \
      else op_zmul_shfl_kernel<N, false><<<g, 256, 0, s>>>(B, sv, nz, cols, scale);                     \
    }                                                                                                   \
    break;
      VX_REG_LENGTHS(VX_ZSH_LAUNCH)
#undef VX_ZSH_LAUNCH
      default:
        set_error("no register z-multiply for length %d", PZ);
        return VX_EINVAL;
    }
    VX_CHECK_LAUNCH("op_zmul_shfl_kernel");
    return VX_OK;
  }
  const unsigned grid = (unsigned)div_up(cols, ZR_T);
  const size_t smem = (size_t)3 * PZ * ZR_T * sizeof(double2);
  switch (PZ) {
#define VX_ZREG_LAUNCH(N)                                                                            \
  case N:                                                                                            \
    if constexpr (N <= REG_ZMUL_MAX) {                                                               \
      if (smem > 48 * 1024)                                                                          \
        VX_CUDA(cudaFuncSetAttribute(op_zmul_reg_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                     (int)smem));                                                    \
      op_zmul_reg_kernel<N><<<grid, ZR_T, smem, s>>>(B, sv, nz, cols, scale);                        \
    }                                                                                                \
    break;
    VX_REG_LENGTHS(VX_ZREG_LAUNCH)
#undef VX_ZREG_LAUNCH
    default:
      set_error("no register z-multiply for length %d", PZ);
      return VX_EINVAL;
  }
  VX_CHECK_LAUNCH("op_zmul_reg_kernel");
  return VX_OK;
}


// K1: forward x-DFT of nlines contiguous x-lines, zero-padded nx -> px.
static int op_x_forward(const FftPlan& fx, int nx, int px, int nlines, const double2* X, double2* A,
                        cudaStream_t s) {
  LoadStrided ld{X, {nx, 0, 1, 1}};
  StoreStrided sv{A, {px, 0, 1, 1}, 1.0};
  return launch_fft_auto(fx, ld, sv, nlines, nx, px, false, true, s);
}

// ------------------------------------------- fused y/z pass, register FFTs
// One CTA per G consecutive x-frequencies kx (all c, z, y of them): the y/z
// padded slab never reaches HBM -- per apply the pass reads A once, the
// spectra once and writes A once (c1: 353 MB instead of 1.28 GB for the
// separate y / z+multiply / y passes).
//   A  y-forward: task (c, z, g): ny values of A -> register DFT (pad to PY)
//      -> smem S[(c,z)][ky][g]   (only the nz nonzero z-rows are kept)
//   B  z + multiply: 3 lanes per column (ky, g) (lane = c*10 + j, as in
//      op_zmul_shfl_kernel): nz values from S -> register DFT (pad to PZ),
//      y_c = sum_b S[PAIR_OF[c,b]] x_b with the partners' values by shuffle,
//      inverse DFT, crop z < nz -> back to S
//   C  y-inverse: task (c, z, g): PY values from S -> register DFT, crop
//      y < ny -> A (in place: the CTA owns its kx columns)
// Launch order interleaves kx groups with their mirrors (blockIdx 2i -> group
// i, 2i+1 -> the last-but-i group) so the compact spectra of kx and px-kx are
// read from DRAM once.  Row stride of S padded for conflict-free phases A/C.
template <int G>
__host__ __device__ constexpr int yzf_row(int py) {
  // quarter-warp of phase A/C = (G g-values) x (8/G rows): rows must land on
  // distinct 16-byte bank slots
  return G == 4 ? (((py * 4) & 7) == 4 ? py * 4 : py * 4 + 4)
       : G == 2 ? (((py * 2) & 7) == 2 || ((py * 2) & 7) == 6 ? py * 2 : py * 2 + 2)
                : py + ((py & 1) ? 0 : 1);
}

// y transforms in two register passes through the slab (PY = R1 * M1, task
// registers <= max(R1, M1) values): forward n = n1*M1 + m, k = k1 + R1*k2
// (slab position k1*M1 + k2); inverse = the transpose.
__host__ __device__ constexpr int yzf_r1(int py) {
  return py % 5 == 0 ? 5 : py % 4 == 0 ? 4 : py % 3 == 0 ? 3 : py % 2 == 0 ? 2 : 1;
}

template <int PY, int PZ, int G>
__global__ void __launch_bounds__(256, 2)
    op_yz_reg_kernel(double2* __restrict__ A, SpecView sv, int ny, int nz, int nkx, int ngroups, double scale) {
  extern __shared__ __align__(16) double2 ysm[];
  constexpr int ROW = yzf_row<G>(PY);
  constexpr int R1 = yzf_r1(PY), M1 = PY / R1;
  static_assert(R1 > 1 && M1 > 1, "PY must split into two register lengths");
  __shared__ double2 twy[PY];  // w_PY^j (forward sign)
  for (int i = threadIdx.x; i < PY; i += blockDim.x) {
    constexpr int o = reg_tw_off(PY);
    twy[i] = cmk(c_rtw[2 * (o + i)], c_rtw[2 * (o + i) + 1]);
  }
  const int b = blockIdx.x;
  const int grp = (b & 1) ? ngroups - 1 - (b >> 1) : (b >> 1);
  const int kx0 = grp * G;
  const long cols = nkx;  // A is (3, nz, ny, nkx)
  const int nlines = 3 * nz;
  __syncthreads();
  // ---- A1: y-forward, first factor (global -> slab)
  for (int i = threadIdx.x; i < nlines * M1 * G; i += blockDim.x) {
    const int g = i % G, r = i / G;
    const int m = r % M1, cz = r / M1;
    const int kx = kx0 + g;
    double2 v[R1];
    const double2* src = A + (long)cz * ny * cols + kx;
#pragma unroll
    for (int n1 = 0; n1 < R1; ++n1) {
      const int y = n1 * M1 + m;
      v[n1] = (y < ny && kx < nkx) ? __ldg(src + (long)y * cols) : cmk(0.0, 0.0);
    }
    reg_fft<R1, false>(v);
    double2* s = ysm + cz * ROW + m * G + g;
    s[0] = v[0];
#pragma unroll
    for (int k1 = 1; k1 < R1; ++k1) s[k1 * M1 * G] = cmul(v[k1], twy[(k1 * m) % PY]);
  }
  __syncthreads();
  // ---- A2: second factor in place (position k1*M1 + k2 = frequency k1 + R1*k2)
  for (int i = threadIdx.x; i < nlines * R1 * G; i += blockDim.x) {
    const int g = i % G, r = i / G;
    const int k1 = r % R1, cz = r / R1;
    double2* s = ysm + cz * ROW + k1 * M1 * G + g;
    double2 v[M1];
#pragma unroll
    for (int n2 = 0; n2 < M1; ++n2) v[n2] = s[n2 * G];
    reg_fft<M1, false>(v);
#pragma unroll
    for (int k2 = 0; k2 < M1; ++k2) s[k2 * G] = v[k2];
  }
  __syncthreads();
  // ---- B: z-forward, spectral multiply, z-inverse (3 lanes per column)
  {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int c = lane < 3 * ZS_COLS ? lane / ZS_COLS : 2;
    const int j = lane < 3 * ZS_COLS ? lane - c * ZS_COLS : 0;
    const int p0 = c == 0 ? 0 : (c == 1 ? 1 : 2);
    const int p1 = c == 0 ? 1 : (c == 1 ? 3 : 4);
    const int p2 = c == 0 ? 2 : (c == 1 ? 4 : 5);
    constexpr int ncol = PY * G;
    for (int col0 = wid * ZS_COLS; col0 < ncol; col0 += nw * ZS_COLS) {
      const int col = col0 + j;
      const bool act = lane < 3 * ZS_COLS && col < ncol;
      const int pos = act ? col / G : 0, g = act ? col - (col / G) * G : 0;
      const int k1 = pos / M1, k2 = pos - (pos / M1) * M1;
      const int ky = k1 + R1 * k2;
      const int kx = kx0 + g;
      const bool live = act && kx < nkx;
      double2* s = ysm + c * nz * ROW + pos * G + g;
      double2 v[PZ];
#pragma unroll
      for (int z = 0; z < PZ; ++z) v[z] = (live && z < nz) ? s[z * ROW] : cmk(0.0, 0.0);
      reg_fft<PZ, false>(v);
      long so0, sstr, kstr;
      bool my = false, mx = false;
      if (sv.compact) {
        my = 2 * ky > sv.Py;
        mx = 2 * kx > sv.Mx;
        so0 = ((long)(my ? sv.Py - ky : ky) * sv.Hx + (mx ? sv.Px - kx : kx)) * 6;
        sstr = 1;
        kstr = (long)sv.Hy * sv.Hx * 6;
      } else {
        so0 = (long)ky * nkx + kx;
        kstr = (long)PY * nkx;
        sstr = (long)PZ * kstr;
      }
      if (!live) so0 = 0;
      const bool n0 = (mx && odd_x(p0)) ^ (my && odd_y(p0));
      const bool n1 = (mx && odd_x(p1)) ^ (my && odd_y(p1));
      const bool n2 = (mx && odd_x(p2)) ^ (my && odd_y(p2));
      const double2* S0 = sv.S + p0 * sstr + so0;
      const double2* S1 = sv.S + p1 * sstr + so0;
      const double2* S2 = sv.S + p2 * sstr + so0;
#pragma unroll
      for (int kz = 0; kz < PZ; ++kz) {
        const bool mz = sv.compact && 2 * kz > PZ;
        const long ko = (long)(mz ? PZ - kz : kz) * kstr;
        double2 s0 = __ldg(S0 + ko), s1 = __ldg(S1 + ko), s2 = __ldg(S2 + ko);
        if (n0 ^ (mz && odd_z(p0))) s0 = cmk(-s0.x, -s0.y);
        if (n1 ^ (mz && odd_z(p1))) s1 = cmk(-s1.x, -s1.y);
        if (n2 ^ (mz && odd_z(p2))) s2 = cmk(-s2.x, -s2.y);
        const double2 x0 = shfl_c(v[kz], j), x1 = shfl_c(v[kz], ZS_COLS + j),
                      x2 = shfl_c(v[kz], 2 * ZS_COLS + j);
        double2 acc = cmul(s0, x0);
        cfma(acc, s1, x1);
        cfma(acc, s2, x2);
        v[kz] = cscale(acc, scale);
      }
      reg_fft<PZ, true>(v);
      if (live) {
#pragma unroll
        for (int z = 0; z < PZ; ++z)
          if (z < nz) s[z * ROW] = v[z];
      }
    }
  }
  __syncthreads();
  // ---- C1: y-inverse over k2 (-> m), conjugate twiddle, in place
  for (int i = threadIdx.x; i < nlines * R1 * G; i += blockDim.x) {
    const int g = i % G, r = i / G;
    const int k1 = r % R1, cz = r / R1;
    double2* s = ysm + cz * ROW + k1 * M1 * G + g;
    double2 v[M1];
#pragma unroll
    for (int k2 = 0; k2 < M1; ++k2) v[k2] = s[k2 * G];
    reg_fft<M1, true>(v);
    s[0] = v[0];
#pragma unroll
    for (int m = 1; m < M1; ++m) s[m * G] = cmulc(v[m], twy[(k1 * m) % PY]);
  }
  __syncthreads();
  // ---- C2: y-inverse over k1 (-> n1), crop y < ny, back to A
  for (int i = threadIdx.x; i < nlines * M1 * G; i += blockDim.x) {
    const int g = i % G, r = i / G;
    const int m = r % M1, cz = r / M1;
    const int kx = kx0 + g;
    if (kx >= nkx) continue;
    const double2* s = ysm + cz * ROW + m * G + g;
    double2 v[R1];
#pragma unroll
    for (int k1 = 0; k1 < R1; ++k1) v[k1] = s[k1 * M1 * G];
    reg_fft<R1, true>(v);
    double2* dst = A + (long)cz * ny * cols + kx;
#pragma unroll
    for (int n1 = 0; n1 < R1; ++n1) {
      const int y = n1 * M1 + m;
      if (y < ny) dst[(long)y * cols] = v[n1];
    }
  }
}

// (PY, PZ) pairs with a fused kernel: the BASELINE grids (c0 20x10, c1 45x21,
// c2 50x21) and the test grids
#define VX_YZF_PAIRS(X) X(20, 10) X(45, 21) X(50, 21) X(12, 6) X(16, 8) X(24, 10) X(14, 6)

static int g_yz_fused = -1;  // -1: from VX_YZ_FUSED
static size_t yzf_smem(int py, int nz, int G) {
  const int row = G == 4 ? yzf_row<4>(py) : G == 2 ? yzf_row<2>(py) : yzf_row<1>(py);
  return (size_t)3 * nz * row * sizeof(double2);
}

// Fused y/z pass when (py, pz) has an instantiation; returns 1 if it ran.
static int op_yz_fused_reg(int ny, int nz, int nkx, int py, int pz, const SpecView& sv, double2* A, double scale,
                           cudaStream_t s, int* ran) {
  *ran = 0;
  if (g_yz_fused < 0) g_yz_fused = env_int("VX_YZ_FUSED", 0) != 0;  // opt-in: latency-bound (0.51 vs 0.40 ms at c1)
  if (!g_yz_fused || nkx <= 0) return VX_OK;
  static const int genv = env_int("VX_YZF_G", 4);
  const size_t budget = (size_t)device_smem_optin() / 2 - 2048;  // two CTAs per SM
  int G = genv;
  while (G > 1 && yzf_smem(py, nz, G) > budget) G /= 2;
  if (yzf_smem(py, nz, G) > (size_t)device_smem_optin()) return VX_OK;
  const int ngroups = (nkx + G - 1) / G;
  const size_t smem = yzf_smem(py, nz, G);
#define VX_YZF_G(PY_, PZ_, G_)                                                                  \
  {                                                                                             \
    auto k = op_yz_reg_kernel<PY_, PZ_, G_>;                                                    \
    if (smem > 48 * 1024) VX_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    k<<<ngroups, 256, smem, s>>>(A, sv, ny, nz, nkx, ngroups, scale);                           \
  }
#define VX_YZF_CASE(PY_, PZ_)                                                                   \
  if (py == PY_ && pz == PZ_) {                                                                 \
    if (G == 4) VX_YZF_G(PY_, PZ_, 4) else if (G == 2) VX_YZF_G(PY_, PZ_, 2) else VX_YZF_G(PY_, PZ_, 1) \
    VX_CHECK_LAUNCH("op_yz_reg_kernel");                                                        \
    *ran = 1;                                                                                   \
    return VX_OK;                                                                               \
  }
  VX_YZF_PAIRS(VX_YZF_CASE)
#undef VX_YZF_CASE
#undef VX_YZF_G
  return VX_OK;
}

// K2-K4 on nkx x-frequency columns held as A (3, nz, ny, nkx): y-DFT (pad ny ->
// py), z-DFT + spectral multiply + inverse z-DFT (crop nz), inverse y-DFT
// (crop ny), result back in A.  Spectra for these columns: (6, pz, py, nkx).
// `scale` = 1/(px py pz) of the full transform.
static int op_yz(const FftPlan& fy, const FftPlan& fz, int ny, int nz, int nkx, int py, int pz,
                 const SpecView& spectra, double2* A, double2* B, double scale, cudaStream_t s) {
  int st, ran;
  if ((st = op_yz_fused_reg(ny, nz, nkx, py, pz, spectra, A, scale, s, &ran))) return st;
  if (ran) return VX_OK;
  const long cols = (long)py * nkx;
  const bool reg_y = reg_fft_enabled() && reg_fft_supported(py);
  const bool reg_z = reg_fft_enabled() && reg_fft_supported(pz) && pz <= REG_ZMUL_MAX;
  static const int use_cols2 = env_int("VX_COLS2", 1);
  const bool two_y = !reg_y && use_cols2 && reg_fft_enabled() && !fy.bluestein && fy.L == py && cols2_supported(py);
  if (reg_y) {
    if ((st = launch_reg_cols<false>(py, A, (long)ny * nkx, nkx, ny, B, cols, nkx, py, 3L * nz * nkx, nkx, 1.0, s)))
      return st;
  } else if (two_y) {
    if ((st = launch_cols2<false>(fy, A, (long)ny * nkx, nkx, ny, B, cols, nkx, py, 3L * nz * nkx, nkx, 1.0, s)))
      return st;
  } else {
    LoadStrided ld{A, {(long)ny * nkx, 1, nkx, nkx}};
    StoreStrided sv{B, {cols, 1, nkx, nkx}, 1.0};
    if ((st = launch_fft_lines(fy, ld, sv, 3 * nz * nkx, ny, py, false, false, s))) return st;
  }
  if (zpair_supported(nz, pz)) {
    if ((st = launch_zpair(nz, B, spectra, cols, nkx, scale, s))) return st;
  } else if (reg_z) {
    if ((st = launch_zmul_reg(pz, B, spectra, nz, cols, scale, s))) return st;
  } else {
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
  if (reg_y) {
    if ((st = launch_reg_cols<true>(py, B, cols, nkx, py, A, (long)ny * nkx, nkx, ny, 3L * nz * nkx, nkx, 1.0, s)))
      return st;
  } else if (two_y) {
    if ((st = launch_cols2<true>(fy, B, cols, nkx, py, A, (long)ny * nkx, nkx, ny, 3L * nz * nkx, nkx, 1.0, s)))
      return st;
  } else {
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
  return launch_fft_auto(fx, ld, sv, nlines, px, nx, true, true, s);
}

// ------------------------------------------------ fused y/z pass (default)
// Layout "kx-pair-major" A2: x-frequency kx and its mirror px-kx share pair
// p = min(kx, px-kx) (slot 0: kx <= px/2, slot 1: the mirror); entry
// (p, line l = (c, z, y), slot) at (p*nl + l)*2 + slot.  K1 writes it, K5
// reads it, and the fused kernel below reads and writes one contiguous
// 2*nl-entry block per pair -- the y/z-padded slab never reaches HBM, and
// the two columns of a pair read the same compact spectra (mirror in x).
struct StoreKxPair {
  double2* __restrict__ p;
  int nl, px;
  __device__ __forceinline__ long line_base(int l) const { return 2L * l; }
  __device__ __forceinline__ void operator()(long b, int kx, double2 v) const {
    const int m = px - kx;
    const int pr = kx <= m ? kx : m, slot = kx <= m ? 0 : 1;
    p[(long)pr * 2 * nl + b + slot] = v;
  }
};
struct LoadKxPair {
  const double2* __restrict__ p;
  int nl, px;
  __device__ __forceinline__ long line_base(int l) const { return 2L * l; }
  __device__ __forceinline__ double2 operator()(long b, int kx) const {
    const int m = px - kx;
    const int pr = kx <= m ? kx : m, slot = kx <= m ? 0 : 1;
    return __ldg(p + (long)pr * 2 * nl + b + slot);
  }
};

// One CTA per kx pair: slab S[z][w*3 + c][y] (pz x 6 x py) in shared memory;
// y-DIF on the nz nonzero z-rows, z-DIF on every (w, c, ky) line, the 9-term
// spectral multiply at digit-reversed positions, z-DIT, y-DIT on the kept
// z-rows, crop y < ny, z < nz.  scale = 1/(px py pz).
template <int RMAX>
__global__ void __launch_bounds__(512, 2) op_yz_fused_kernel(FftPlan fy, FftPlan fz, double2* __restrict__ A2, SpecView sv,
                                                          int ny, int nz, double scale, FastDiv fdWy, FastDiv fdWz) {
  extern __shared__ __align__(16) double2 fsm[];
  const int py = fy.L, pz = fz.L;
  const int nl = 3 * nz * ny;
  const int row6 = 6 * py;            // one z-row of the slab
  double2* S = fsm;                   // [pz][6][py]
  double2* twy = S + (long)pz * row6;
  double2* twz = twy + 64 + fy.nhi;
  const int pr = blockIdx.x;
  const int px = sv.Px;
  const bool two = (pr != 0) && (2 * pr != px);  // slot 1 holds a distinct column
  fft_load_twiddles(fy, twy);
  fft_load_twiddles(fz, twz);
  for (int i = threadIdx.x; i < pz * row6; i += blockDim.x) S[i] = cmk(0.0, 0.0);
  __syncthreads();
  const double2* src = A2 + (long)pr * 2 * nl;
  for (int i = threadIdx.x; i < 2 * nl; i += blockDim.x) {
    const int slot = i & 1, l = i >> 1;
    if (slot && !two) continue;
    const int c = l / (nz * ny), r = l - c * nz * ny;
    const int z = r / ny, y = r - z * ny;
    S[(z * 6 + slot * 3 + c) * py + y] = __ldg(src + i);
  }
  __syncthreads();
  const int nw = two ? 2 : 1;
  {
    const SmemLay ly{1, py};
    const int W = 6 * nz;
    fft_dif<RMAX>(S, ly, W, fdWy, fy, twy, -1.0);
  }
  {
    const SmemLay lz{row6, 1};
    fft_dif<RMAX>(S, lz, row6, fdWz, fz, twz, -1.0);
  }
  // spectral multiply (positions are digit-reversed in y and z)
  for (int i = threadIdx.x; i < pz * nw * py; i += blockDim.x) {
    const int zp = i / (nw * py), r = i - zp * nw * py;
    const int w = r / py, yp = r - w * py;
    const int kz = __ldg(fz.k_of + zp), ky = __ldg(fy.k_of + yp);
    const int kx = w ? px - pr : pr;
    double2 sp[6];
    if (!sv.compact) {
      const long so = ((long)kz * sv.Py + ky) * px + kx, sstr = (long)sv.Pz * sv.Py * px;
#pragma unroll
      for (int q = 0; q < 6; ++q) sp[q] = ld_stream(sv.S + q * sstr + so);
    } else {
      const bool mz = 2 * kz > sv.Pz, my = 2 * ky > sv.Py, mx = 2 * kx > sv.Mx;
      const int kzs = mz ? sv.Pz - kz : kz, kys = my ? sv.Py - ky : ky, kxs = mx ? sv.Px - kx : kx;
      const long so = (((long)kzs * sv.Hy + kys) * sv.Hx + kxs) * 6;
      const long sstr = 1;
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        const double2 v = __ldg(sv.S + q * sstr + so);
        const bool neg = (mx && odd_x(q)) ^ (my && odd_y(q)) ^ (mz && odd_z(q));
        sp[q] = neg ? cmk(-v.x, -v.y) : v;
      }
    }
    double2* qv = S + (zp * 6 + w * 3) * py + yp;
    const double2 x0 = qv[0], x1 = qv[py], x2 = qv[2 * py];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      double2 acc = cmul(sp[pair_of(a, 0)], x0);
      cfma(acc, sp[pair_of(a, 1)], x1);
      cfma(acc, sp[pair_of(a, 2)], x2);
      qv[a * py] = cscale(acc, scale);
    }
  }
  __syncthreads();
  {
    const SmemLay lz{row6, 1};
    fft_dit<RMAX>(S, lz, row6, fdWz, fz, twz, 1.0);
  }
  {
    const SmemLay ly{1, py};
    const int W = 6 * nz;
    fft_dit<RMAX>(S, ly, W, fdWy, fy, twy, 1.0);
  }
  double2* dst = A2 + (long)pr * 2 * nl;
  for (int i = threadIdx.x; i < 2 * nl; i += blockDim.x) {
    const int slot = i & 1, l = i >> 1;
    if (slot && !two) continue;
    const int c = l / (nz * ny), r = l - c * nz * ny;
    const int z = r / ny, y = r - z * ny;
    dst[i] = S[(z * 6 + slot * 3 + c) * py + y];
  }
}

static size_t yz_fused_smem(const FftPlan& fy, const FftPlan& fz) {
  return ((size_t)fz.L * 6 * fy.L + 128 + fy.nhi + fz.nhi) * sizeof(double2);
}

static int op_apply_fused(const FftPlan& fx, const FftPlan& fy, const FftPlan& fz, int nx, int ny, int nz,
                          const SpecView& sv, const double2* m, const double2* X, double2* Y, double2* A2,
                          double scale, cudaStream_t s) {
  int st;
  const int px = fx.n;
  const int nl = 3 * nz * ny;
  {
    LoadStrided ld{X, {nx, 0, 1, 1}};
    StoreKxPair sv2{A2, nl, px};
    if ((st = launch_fft_lines(fx, ld, sv2, nl, nx, px, false, true, s))) return st;
  }
  {
    const size_t smem = yz_fused_smem(fy, fz);
    const bool hi = fft_max_radix(fy) > 8 || fft_max_radix(fz) > 8;
    auto kern = hi ? op_yz_fused_kernel<13> : op_yz_fused_kernel<8>;
    if (smem > 48 * 1024)
      VX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<px / 2 + 1, 512, smem, s>>>(fy, fz, A2, sv, ny, nz, scale, FastDiv((unsigned)(6 * nz)),
                                       FastDiv((unsigned)(6 * fy.L)));
    VX_CHECK_LAUNCH("op_yz_fused_kernel");
  }
  LoadKxPair ld{A2, nl, px};
  StoreSystem sv3{Y, X, m, nx, (long)nx * ny * nz, 1.0, 0};
  return launch_fft_lines(fx, ld, sv3, nl, px, nx, true, true, s);
}

}  // namespace vx

static SpecView spec_view(const vx_c128* spectra, int compact, int px, int py, int pz) {
  SpecView v;
  v.S = reinterpret_cast<const double2*>(spectra);
  v.compact = compact;
  v.Pz = pz; v.Py = py; v.Px = px;
  v.Hz = pz / 2 + 1; v.Hy = py / 2 + 1; v.Hx = px / 2 + 1;
  v.Mx = px;
  if (compact == 2) {  // compacted in y and z only: every local kx column is stored
    v.compact = 1;
    v.Hx = px;
    v.Mx = 1 << 30;
  }
  v.fdPx = FastDiv((unsigned)px);
  return v;
}

extern "C" int vx_op_apply(int nx, int ny, int nz, int px, int py, int pz, const vx_c128* spectra,
                           int compact, const vx_c128* m, const vx_c128* x, vx_c128* y, vx_c128* work,
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
  // fused y/z pass (VX_OP_FUSED=1) when the padded (6 x pz x py) slab of a kx
  // pair fits two CTAs per SM (c0-c2); default: the 5-launch path
  static const int fused_env = env_int("VX_OP_FUSED", 0);  // opt-in: smem-stage bound (0.59 vs 0.52 ms at c1)
  if (fused_env && !fy.bluestein && !fz.bluestein &&
      2 * (yz_fused_smem(fy, fz) + 1024) <= (size_t)device_smem_optin() + 1024)
    return op_apply_fused(fx, fy, fz, nx, ny, nz, spec_view(spectra, compact, px, py, pz),
                          reinterpret_cast<const double2*>(m), X, reinterpret_cast<double2*>(y), A,
                          1.0 / ((double)px * py * pz), s);
  if ((st = op_x_forward(fx, nx, px, lines_xyz, X, A, s))) return st;
  if ((st = op_yz(fy, fz, ny, nz, px, py, pz, spec_view(spectra, compact, px, py, pz), A, B,
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
  return op_yz(fy, fz, ny, nz, nkx, py, pz, spec_view(spectra_local, 0, nkx, py, pz),
               reinterpret_cast<double2*>(A), reinterpret_cast<double2*>(work),
               1.0 / ((double)px * py * pz), as_stream(stream));
}

// vx_op_yz on spectra compacted in y and z (vx_spec_compact_yz): a rank's kx columns of the
// parity-symmetric kernel's spectra at a quarter of the bytes (and one load per kz mirror pair)
extern "C" int vx_op_yz_compact(int ny, int nz, int nkx, int px, int py, int pz, const vx_c128* spectra_cyz,
                                vx_c128* A, vx_c128* work, void* stream) {
  VX_REQUIRE(ny >= 1 && nz >= 1 && nkx >= 0, "bad yz arguments");
  VX_REQUIRE(fft_is_smooth(py) && fft_is_smooth(pz), "padded dims must be 13-smooth");
  if (nkx == 0) return VX_OK;
  FftPlan fy, fz;
  int st;
  if ((st = fft_get_plan(py, &fy)) || (st = fft_get_plan(pz, &fz))) return st;
  return op_yz(fy, fz, ny, nz, nkx, py, pz, spec_view(spectra_cyz, 2, nkx, py, pz),
               reinterpret_cast<double2*>(A), reinterpret_cast<double2*>(work),
               1.0 / ((double)px * py * pz), as_stream(stream));
}

extern "C" long vx_spec_compact_yz_elems(int nkx, int py, int pz) {
  return 6L * (pz / 2 + 1) * (py / 2 + 1) * nkx;
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

namespace vx {
// gather the k <= P/2 half-octant of full spectra (6, pz, py, px)
__global__ void spec_compact_kernel(const double2* __restrict__ full, double2* __restrict__ out, int px, int py,
                                    int pz, int hx) {
  const int hy = py / 2 + 1, hz = pz / 2 + 1;
  const long total = 6L * hz * hy * hx;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    long r = i;
    const int kx = (int)(r % hx); r /= hx;
    const int ky = (int)(r % hy); r /= hy;
    const int kz = (int)(r % hz);
    const int p = (int)(r / hz);
    out[(((long)kz * hy + ky) * hx + kx) * 6 + p] = full[(((long)p * pz + kz) * py + ky) * px + kx];
  }
}

// per-CTA max |t_p(d) - s_p t_p(d')| for d' = d mirrored in x, in y and in z
// separately (s_p = the component's parity on that axis), and max |t_p(d)|
__global__ void gen_asym_kernel(const double2* __restrict__ g, long sp, long sz, long sy, long sx, int nx, int ny,
                                int nz, double* __restrict__ out) {
  __shared__ double sa[4][256];
  const int X = 2 * nx - 1, Y = 2 * ny - 1, Z = 2 * nz - 1;
  const long total = 6L * Z * Y * X;
  double ax = 0.0, ay = 0.0, az = 0.0, tmax = 0.0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    long r = i;
    const int ix = (int)(r % X); r /= X;
    const int iy = (int)(r % Y); r /= Y;
    const int iz = (int)(r % Z);
    const int p = (int)(r / Z);
    const double2* gp = g + p * sp;
    const double2 a = gp[iz * sz + iy * sy + ix * sx];
    const double2 bx = gp[iz * sz + iy * sy + (X - 1 - ix) * sx];
    const double2 by = gp[iz * sz + (Y - 1 - iy) * sy + ix * sx];
    const double2 bz = gp[(Z - 1 - iz) * sz + iy * sy + ix * sx];
    const double fx = odd_x(p) ? -1.0 : 1.0, fy = odd_y(p) ? -1.0 : 1.0, fz = odd_z(p) ? -1.0 : 1.0;
    ax = fmax(ax, fmax(fabs(a.x - fx * bx.x), fabs(a.y - fx * bx.y)));
    ay = fmax(ay, fmax(fabs(a.x - fy * by.x), fabs(a.y - fy * by.y)));
    az = fmax(az, fmax(fabs(a.x - fz * bz.x), fabs(a.y - fz * bz.y)));
    tmax = fmax(tmax, fmax(fabs(a.x), fabs(a.y)));
  }
  sa[0][threadIdx.x] = ax;
  sa[1][threadIdx.x] = ay;
  sa[2][threadIdx.x] = az;
  sa[3][threadIdx.x] = tmax;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o)
      for (int c = 0; c < 4; ++c) sa[c][threadIdx.x] = fmax(sa[c][threadIdx.x], sa[c][threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x < 4) out[4 * blockIdx.x + threadIdx.x] = sa[threadIdx.x][0];
}
}  // namespace vx

extern "C" long vx_op_compact_elems(int px, int py, int pz) {
  return 6L * (pz / 2 + 1) * (py / 2 + 1) * (px / 2 + 1);
}

extern "C" int vx_op_compact(int px, int py, int pz, const vx_c128* full, vx_c128* compact, void* stream) {
  const long total = vx_op_compact_elems(px, py, pz);
  const unsigned g = div_up(total, 256) < 8192 ? div_up(total, 256) : 8192;
  spec_compact_kernel<<<g, 256, 0, as_stream(stream)>>>(reinterpret_cast<const double2*>(full),
                                                        reinterpret_cast<double2*>(compact), px, py, pz, px / 2 + 1);
  VX_CHECK_LAUNCH("spec_compact_kernel");
  return VX_OK;
}

// the k <= P/2 halves in y and z of a rank's kx columns (full: (6, pz, py, nkx)), all nkx kept
extern "C" int vx_spec_compact_yz(int nkx, int py, int pz, const vx_c128* full, vx_c128* compact, void* stream) {
  VX_REQUIRE(nkx >= 0 && py >= 1 && pz >= 1, "bad compaction arguments");
  const long total = vx_spec_compact_yz_elems(nkx, py, pz);
  if (total == 0) return VX_OK;
  const unsigned g = div_up(total, 256) < 8192 ? div_up(total, 256) : 8192;
  spec_compact_kernel<<<g, 256, 0, as_stream(stream)>>>(reinterpret_cast<const double2*>(full),
                                                        reinterpret_cast<double2*>(compact), nkx, py, pz, nkx);
  VX_CHECK_LAUNCH("spec_compact_kernel");
  return VX_OK;
}

extern "C" int vx_gen_asymmetry(int nx, int ny, int nz, const vx_c128* gen, long g_sp, long g_sz, long g_sy,
                                long g_sx, double* out, void* stream) {
  gen_asym_kernel<<<256, 256, 0, as_stream(stream)>>>(reinterpret_cast<const double2*>(gen), g_sp, g_sz, g_sy,
                                                      g_sx, nx, ny, nz, out);
  VX_CHECK_LAUNCH("gen_asym_kernel");
  return VX_OK;
}

extern "C" int vx_op_reg_fft(int on) {
  vx::g_reg_fft = on ? 1 : 0;
  return VX_OK;
}
