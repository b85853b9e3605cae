// Generating tensors of N assembled on the device (reference kernel.py:119-198,
// accel.py:131-155): the six dyadic Green components
// V * (k0^2 I + grad grad) g at every signed voxel offset, written straight
// into the (6, 2nz-1, 2ny-1, 2nx-1) layout the operator plan and the Chan
// spectra read, so the ~0.9 GB (c1) generator array is never formed on the
// host or copied over the link.
//
// One thread per offset evaluates the non-negative-octant point (|dx|, |dy|,
// |dz|) delta with the reference's operation order (no FMA contraction: every
// product and sum is rounded as numpy rounds it) and applies each component's
// parity sign for the negative coordinates -- the host mirrors the octant with
// the same exact sign flips (kernel.py:37-51).  The zero offset takes the
// self term (computed on the host by the Duffy quadrature, kernel.py:59-116).
// HBM-bound: 6 x 16 bytes written per offset.
#include <math_constants.h>

#include "common.cuh"

namespace vx {
namespace {

struct Cx {
  double re, im;
};
__device__ __forceinline__ Cx cx_mul(Cx a, Cx b) {  // numpy: (ac - bd) + i(ad + bc)
  return {__dsub_rn(__dmul_rn(a.re, b.re), __dmul_rn(a.im, b.im)),
          __dadd_rn(__dmul_rn(a.re, b.im), __dmul_rn(a.im, b.re))};
}
__device__ __forceinline__ Cx cx_scale(Cx a, double s) { return {__dmul_rn(a.re, s), __dmul_rn(a.im, s)}; }
// complex / real as numpy evaluates it (complex division by (s, 0): a * (1/s))
__device__ __forceinline__ Cx cx_div(Cx a, double s) { return cx_scale(a, __drcp_rn(s)); }

// parity of (xx, xy, xz, yy, yz, zz) under x, y, z sign flips (+1 even, -1 odd)
__constant__ int kParX[6] = {1, -1, -1, 1, 1, 1};
__constant__ int kParY[6] = {1, -1, 1, 1, -1, 1};
__constant__ int kParZ[6] = {1, 1, -1, 1, -1, 1};

__global__ void __launch_bounds__(256) assemble_green_kernel(int nx, int ny, int nz, double delta, double k0,
                                                             double vol, double2 self_val,
                                                             double2* __restrict__ out) {
  const long Lx = 2L * nx - 1, Ly = 2L * ny - 1, Lz = 2L * nz - 1;
  const long plane = Lx * Ly * Lz;
  for (long o = blockIdx.x * (long)blockDim.x + threadIdx.x; o < plane; o += (long)gridDim.x * blockDim.x) {
    const long ix = o % Lx, t = o / Lx;
    const long iy = t % Ly, iz = t / Ly;
    const int dx = (int)(ix - (nx - 1)), dy = (int)(iy - (ny - 1)), dz = (int)(iz - (nz - 1));
    const int ax = dx < 0 ? -dx : dx, ay = dy < 0 ? -dy : dy, az = dz < 0 ? -dz : dz;
    Cx c[6];
    if (ax == 0 && ay == 0 && az == 0) {
      const Cx s = {self_val.x, self_val.y};
      const Cx zero = {0.0, 0.0};
      c[0] = s; c[1] = zero; c[2] = zero; c[3] = s; c[4] = zero; c[5] = s;  // xx, yy, zz
    } else {
      const double X = __dmul_rn(delta, (double)ax), Y = __dmul_rn(delta, (double)ay),
                   Z = __dmul_rn(delta, (double)az);
      const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(X, X), __dmul_rn(Y, Y)), __dmul_rn(Z, Z));
      const double r = __dsqrt_rn(r2);
      const double kr = __dmul_rn(k0, r);
      double sn, cs;
      sincos(kr, &sn, &cs);
      const double fpr = __dmul_rn(4.0 * CUDART_PI, r);
      const Cx g = cx_div(Cx{cs, -sn}, fpr);  // exp(-i k0 r) / (4 pi r)
      const double k2 = __dmul_rn(k0, k0);
      const double ir2 = __drcp_rn(r2);
      // d = g * (k2 - (1 + i k0 r) / r2)
      const Cx dterm = {__dsub_rn(k2, ir2), -__dmul_rn(kr, ir2)};
      const Cx d = cx_mul(g, dterm);
      // rad = g * (3 / r2 + 3 i k0 / r - k2) / r2
      const Cx rterm = {__dsub_rn(__ddiv_rn(3.0, r2), k2), __dmul_rn(__dmul_rn(3.0, k0), __drcp_rn(r))};
      const Cx rad = cx_div(cx_mul(g, rterm), r2);
      const Cx rX = cx_scale(rad, X), rY = cx_scale(rad, Y);
      const Cx xx = cx_scale(rX, X), yy = cx_scale(rY, Y), zz = cx_scale(cx_scale(rad, Z), Z);
      c[0] = {__dadd_rn(d.re, xx.re), __dadd_rn(d.im, xx.im)};
      c[1] = cx_scale(rX, Y);
      c[2] = cx_scale(rX, Z);
      c[3] = {__dadd_rn(d.re, yy.re), __dadd_rn(d.im, yy.im)};
      c[4] = cx_scale(rY, Z);
      c[5] = {__dadd_rn(d.re, zz.re), __dadd_rn(d.im, zz.im)};
#pragma unroll
      for (int p = 0; p < 6; ++p) c[p] = cx_scale(c[p], vol);
    }
#pragma unroll
    for (int p = 0; p < 6; ++p) {
      const int sg = (dx < 0 ? kParX[p] : 1) * (dy < 0 ? kParY[p] : 1) * (dz < 0 ? kParZ[p] : 1);
      const double2 v = sg > 0 ? make_double2(c[p].re, c[p].im) : make_double2(-c[p].re, -c[p].im);
      __stcs(out + (long)p * plane + o, v);
    }
  }
}

}  // namespace
}  // namespace vx

extern "C" int vx_assemble_green(int nx, int ny, int nz, double delta, double k0, double vol, vx_c128 self_val,
                                 vx_c128* out, void* stream) {
  using namespace vx;
  VX_REQUIRE(nx >= 1 && ny >= 1 && nz >= 1 && delta > 0.0 && out, "bad assemble arguments");
  const long plane = (2L * nx - 1) * (2L * ny - 1) * (2L * nz - 1);
  long g = (plane + 255) / 256;
  const long cap = 16L * device_sm_count();
  if (g > cap) g = cap;
  assemble_green_kernel<<<(int)g, 256, 0, as_stream(stream)>>>(nx, ny, nz, delta, k0, vol,
                                                               make_double2(self_val.re, self_val.im),
                                                               reinterpret_cast<double2*>(out));
  VX_CHECK_LAUNCH("assemble_green_kernel");
  return VX_OK;
}
