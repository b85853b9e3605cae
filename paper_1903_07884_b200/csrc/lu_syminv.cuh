// Symmetric INVERSE storage of the 1-level sector blocks and its one-pass
// apply -- included by circulant.cu after lu_sym.cuh (same geometry: SymGeom,
// sym_band, trap_off, sym_swz; the mbarrier / bulk-copy helpers).
//
// Why: the two triangular passes of lu_sym.cuh read every factor byte twice
// (the second time from L2) and are a chain of dependent tile rows; measured
// on c1 the pair of passes cannot go below ~0.65 ms even with the arithmetic
// removed (forward alone: 0.44 ms = the HBM peak; profiles/r02_sym_phases.txt).
// With B = W A^ (A^ complex symmetric, W = S M on the sector rows) the inverse
// is B^-1 = G W^-1 with G = A^^-1 complex SYMMETRIC, and from the unpivoted
// factors B = L U, U = diag(u) W L^T W^-1:
//     G = (L^-1 W)^T diag(h) (L^-1 W),      h = 1 / (u W).
// Storing the lower triangle of G costs the bytes of L, and x = G (b / W) is a
// symmetric matrix-vector product: ONE streaming pass over the stored bytes,
// every tile used for both its product and its transposed product while it
// sits in shared memory, no dependencies between tiles.  The reference's
// zgetrs (circulant.py:183-186) becomes a bandwidth-bound SYMV.
// The blocks here are well conditioned (cond <= 1.6e2 on the BASELINE
// workloads), the caller verifies G against the triangular solves on a random
// vector (relative 1e-13 over the whole vector, observed ~1e-15) and keeps the factors otherwise.
//
// Layout of G: the lu_sym.cuh layout (tile rows of row-major swizzled t_i x 32
// tiles, then the diagonal trapezoid); the diagonal 8 x 8 blocks of the
// trapezoid hold both triangles of the symmetric block.
//
// Included INSIDE namespace vx.

// ------------------------------------------------------------------ build
// One CTA per slot.  N = L^-1 by tile columns (N_ij = -sum_{j<=k<i} L'_ik N_kj,
// N_jj = inv(L_jj), with the premultiplied tiles L' of the symmetric layout),
// written to the scratch buffer in the same layout; then
// G_ij = W_i [sum_{k>=i} N_ki^T diag(h_k) N_kj] W_j for i >= j.
__device__ __forceinline__ void syminv_load_tile(double2 (*dst)[33], const double2* blk, int nb, int i, int j,
                                                 const double2* rowscale, int tid) {
  // dst[r][c] = entry (r, c) of tile (i, j) (j == i: the trapezoid; zeros outside), rows scaled
  const int ti = min(32, nb - 32 * i);
  const double2* base = blk + sym_band(i) + 32L * ti * j;
  for (int e = tid; e < 1024; e += 256) {
    const int r = e >> 5, c = e & 31;
    double2 v = cmk(0.0, 0.0);
    if (r < ti) {
      if (i != j) v = base[r * 32 + sym_swz(r, c)];
      else if (c < 8 * (r >> 3) + 8) v = base[trap_off(r) + sym_swz(r, c)];
      if (rowscale) v = cmul(v, rowscale[32 * i + r]);
    }
    dst[r][c] = v;
  }
}

__global__ void __launch_bounds__(256) lu_sym_invert_kernel(SymGeom sg, const double2* __restrict__ Lp,
                                                            double2* __restrict__ Nq, double2* __restrict__ Gq) {
  __shared__ double2 As[32][33];
  __shared__ double2 Bs[32][33];
  const int slot = blockIdx.x;
  int nb, sec;
  const double2* Lb = sym_block(sg, Lp, slot, nb, sec);
  double2* Nb = const_cast<double2*>(sym_block(sg, Nq, slot, nb, sec));
  double2* Gb = const_cast<double2*>(sym_block(sg, Gq, slot, nb, sec));
  const double2* W = sg.w + (long)sec * sg.dmax;
  const double2* H = sg.h + (long)slot * sg.dmax;
  const int tid = threadIdx.x;
  const int nt = (nb + 31) / 32;
  const int r0 = tid >> 5, c = tid & 31;  // outputs (r0 + 8 m, c), m = 0..3
  // ---- N = L^-1
  for (int j = 0; j < nt; ++j) {
    {  // N_jj = inv(L_jj): the trapezoid as stored
      const int tj = min(32, nb - 32 * j);
      const long o = sym_band(j) + 32L * tj * j;
      for (int e = tid; e < trap_size(tj); e += 256) Nb[o + e] = Lb[o + e];
    }
    for (int i = j + 1; i < nt; ++i) {
      const int ti = min(32, nb - 32 * i);
      double2 acc[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) acc[m] = cmk(0.0, 0.0);
      for (int k = j; k < i; ++k) {
        __syncthreads();  // previous product done with As / Bs; N_kj of this block written
        syminv_load_tile(As, Lb, nb, i, k, nullptr, tid);
        syminv_load_tile(Bs, Nb, nb, k, j, nullptr, tid);
        __syncthreads();
#pragma unroll 8
        for (int mm = 0; mm < 32; ++mm) {
          const double2 b = Bs[mm][c];
#pragma unroll
          for (int m = 0; m < 4; ++m) cfma(acc[m], As[r0 + 8 * m][mm], b);
        }
      }
      double2* dst = Nb + sym_band(i) + 32L * ti * j;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const int r = r0 + 8 * m;
        if (r < ti) dst[r * 32 + sym_swz(r, c)] = cmk(-acc[m].x, -acc[m].y);
      }
    }
  }
  // ---- G_ij = W_i sum_k N_ki^T diag(h_k) N_kj W_j (rows a of tile row i, columns b of tile row j)
  for (int i = 0; i < nt; ++i) {
    const int ti = min(32, nb - 32 * i);
    for (int j = 0; j <= i; ++j) {
      double2 acc[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) acc[m] = cmk(0.0, 0.0);
      for (int k = i; k < nt; ++k) {
        __syncthreads();
        syminv_load_tile(As, Nb, nb, k, i, H, tid);  // As[m][a] = h_k[m] N_ki[m][a]
        syminv_load_tile(Bs, Nb, nb, k, j, nullptr, tid);
        __syncthreads();
#pragma unroll 8
        for (int mm = 0; mm < 32; ++mm) {
          const double2 b = Bs[mm][c];
#pragma unroll
          for (int m = 0; m < 4; ++m) cfma(acc[m], As[mm][r0 + 8 * m], b);
        }
      }
      double2* dst = Gb + sym_band(i) + 32L * ti * j;
      const double2 wj = W[32 * j + c < nb ? 32 * j + c : 0];
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const int a = r0 + 8 * m;
        if (a < ti) {
          const double2 v = cmul(cmul(acc[m], W[32 * i + a]), wj);
          if (i != j) dst[a * 32 + sym_swz(a, c)] = v;
          else if (c < 8 * (a >> 3) + 8) dst[trap_off(a) + sym_swz(a, c)] = v;
        }
      }
    }
  }
}

// ------------------------------------------------------------------ apply
// x = G (b / W): one CTA per work item (a stored sector block and its one or
// two right-hand sides: the x-mirror pair), 4 tensor-core warps + a producer
// warp.  The producer streams the block's storage in order, one 16 KB tile per
// slot of an in-order mbarrier ring (plus an L2 prefetch window ahead of it);
// every tile is consumed by all four warps on the FP64 tensor cores (fragment
// scheme of lu_sym.cuh: A = stored entries, B = (Re, Im) columns of the two
// right-hand sides).  Warp w OWNS entries 8w .. 8w+7 of every tile row of the
// result: it computes rows 8w.. of (tile x c_j) and columns 8w.. of
// (tile^T x c_i).  The result vector therefore exists once in shared memory
// (no per-warp partial vectors, no reduction, no atomics: bitwise
// reproducible), and the c_i fragments of the transposed products stay in
// registers for a whole tile row.
// (A first version gave each warp its own 8 KB units and partial vector: same
// speed on c1, but its ring needed a slot-per-warp protocol and its shared
// memory grew with 4 x the block size; profiles/r02_symv_v1_ncu.txt, v2.)
constexpr int SYMV_WARPS = 4;

// Per-lane fragment offsets (doubles), fixed for the whole kernel, so that every
// fragment load of the unrolled unit bodies is [register + immediate]:
//   nb[kl]  product A fragment: row g of a row block, unit (kc & 3) == kl; + 512 rb + 16 (kc >> 2)
//   tb[par] transposed A fragment: rows 2 kc + (t >> 1), kc & 1 == par; + 128 kc + 16 cb
//   cb      operand fragment in the signed right-hand-side array c3; + 192 panel + 12 kc
struct SymvLane {
  int nb[4];
  int tb[2];
  int cb;
  int g, t;
};

// c3: per (entry, right-hand side) three doubles (y_i, y_r, -y_i): the B
// fragment column "Re" reads (y_r, -y_i) at +1, the column "Im" reads (y_i, y_r)
// at +0 -- no sign arithmetic in the loops.  Lanes g >= 4 mirror lanes g - 4:
// their C columns are never stored.
__device__ __forceinline__ SymvLane symv_lane(int lane) {
  SymvLane L;
  L.g = lane >> 2;
  L.t = lane & 3;
  const int g = L.g, t = L.t;
  const int fsw = ((g & 1) << 1) | ((g >> 1) & 1);
#pragma unroll
  for (int kl = 0; kl < 4; ++kl) L.nb[kl] = g * 64 + ((kl ^ fsw) << 2) + t;
  const int bcol = ((g & 1) << 1) + (t & 1);
#pragma unroll
  for (int par = 0; par < 2; ++par) L.tb[par] = (t >> 1) * 64 + ((((g >> 1) ^ (((t >> 1) << 1) | par)) << 2)) + bcol;
  const int rr = (g >> 1) & 1, im = g & 1;
  L.cb = (t >> 1) * 6 + rr * 3 + (1 - im) + (t & 1);
  return L;
}

struct Symv2Stage {
  double an[2], bn[2], at[2];
};

template <int R, int MINB>
__global__ void __launch_bounds__((SYMV_WARPS + 1) * 32, MINB)
    symv2_inv_kernel(SymGeom sg, const double2* __restrict__ G, const int* __restrict__ items, int nwork,
                     const int* __restrict__ klist, double2* Y, long s_row, long s_k, int S, int q, int pfwin) {
  extern __shared__ __align__(128) unsigned char smraw[];
  constexpr int NC = SYMV_WARPS * 32;
  constexpr int T2 = 1024;  // entries per ring slot (16 KB)
  const int npad = (sg.dmax + 31) / 32 * 32;
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw);
  uint64_t* empty = full + S;
  double2* slots = reinterpret_cast<double2*>(smraw + (2 * S * 8 + 127) / 128 * 128);
  double2* out = slots + (long)S * T2;                       // [npad][2]: the result
  double* c3 = reinterpret_cast<double*>(out + 2L * npad);   // [npad][2][3]: c = b / W, signed
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, SYMV_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == SYMV_WARPS) {
    if (lane == 0) {
      uint32_t n = 0;  // tiles emitted (all work items)
      for (int w = blockIdx.x; w < nwork; w += gridDim.x) {
        const int slot = items[3 * w], cnt = items[3 * w + 2];
        int nb, sec;
        const double2* Gb = sym_block(sg, G, slot, nb, sec);
        const int nt = (nb + 31) / 32;
        const long total = sym_size(nb);
        for (int ch = 0; ch < (cnt + R - 1) / R; ++ch) {
          long pf = 0;
          auto prefetch_to = [&](long upto) {
            upto = upto < total ? upto : total;
            while (pf < upto) {
              const long m = upto - pf < 1024 ? upto - pf : 1024;
              bulk_prefetch_l2(Gb + pf, (uint32_t)(m * sizeof(double2)));
              pf += m;
            }
          };
          for (int i = 0; i < nt; ++i) {
            const int ti = min(32, nb - 32 * i);
            const double2* band = Gb + sym_band(i);
            for (int j = 0; j <= i; ++j, ++n) {
              const double2* src = band + 32L * ti * j;
              const uint32_t elems = (uint32_t)(j < i ? ti * 32 : trap_size(ti));
              if (pfwin > 0) prefetch_to((src - Gb) + elems + pfwin);
              const int s = n % S;
              const uint32_t use = n / S;
              if (use > 0) mbar_wait_hint(empty + s, (use - 1) & 1u);
              mbar_expect_tx(full + s, elems * (uint32_t)sizeof(double2));
              bulk_g2s(slots + s * T2, src, elems * (uint32_t)sizeof(double2), full + s);
            }
          }
        }
      }
    }
    return;
  }

  const SymvLane L = symv_lane(lane);
  const int g = L.g, t = L.t;
  // this warp's fragment bases inside a tile: product rows 8w + g; transposed columns 8w + g
  const int nbw[4] = {L.nb[0] + 512 * warp, L.nb[1] + 512 * warp, L.nb[2] + 512 * warp, L.nb[3] + 512 * warp};
  const int tbw[2] = {L.tb[0] + 16 * warp, L.tb[1] + 16 * warp};
  // C fragment owner: lanes t < 2 hold (entry 8w + g, right-hand side t)
  auto add_out = [&](int panel, double c0, double c1) {
    if (t < 2) {
      double2* p = out + (((panel * 32 + 8 * warp + g) << 1) + t);
      const double2 o = *p;
      *p = cmk(o.x + c0, o.y + c1);
    }
  };
  uint32_t n = 0;
  for (int w = blockIdx.x; w < nwork; w += gridDim.x) {
    const int slot = items[3 * w], beg = items[3 * w + 1], cnt = items[3 * w + 2];
    int nb, sec;
    (void)sym_block(sg, G, slot, nb, sec);
    const int nt = (nb + 31) / 32;
    const double2* wrow = sg.w + (long)sec * sg.dmax;
    for (int ch = 0; ch < (cnt + R - 1) / R; ++ch) {
      const int rho0 = ch * R;
      const int nr = min(R, cnt - rho0);
      long rb0 = 0, rb1 = 0;
      {
        const int k0 = klist ? klist[beg + rho0] : beg + rho0;
        rb0 = rhs_base(k0, rho0, 1, s_k);
        if (nr > 1) {
          const int k1 = klist ? klist[beg + rho0 + 1] : beg + rho0 + 1;
          rb1 = rhs_base(k1, rho0 + 1, 1, s_k);
        }
      }
      consumers_sync(NC);  // the previous item's result has been written out
      for (int idx = tid; idx < npad * 2; idx += NC) {
        const int row = idx >> 1, rr = idx & 1;
        double2 v = cmk(0.0, 0.0);
        if (row < nb && rr < nr) {
          const long rb = rr ? rb1 : rb0;
          v = cdiv(cflip(Y[(long)row * s_row + (rb & ROFF)], flip_row((int)(rb >> 56), row, q)), wrow[row]);
        }
        double* o = c3 + 3 * idx;
        o[0] = v.y;
        o[1] = v.x;
        o[2] = -v.y;
        out[idx] = cmk(0.0, 0.0);
      }
      consumers_sync(NC);
      for (int i = 0; i < nt; ++i) {
        const int ti = min(32, nb - 32 * i);
        const double* ci = c3 + 192 * i + L.cb;
        double bi[16];  // c_i fragments: operands of every transposed product of this tile row
#pragma unroll
        for (int k = 0; k < 16; ++k) bi[k] = ci[12 * k];
        double aN[4][2];
#pragma unroll
        for (int b = 0; b < 4; ++b) aN[b][0] = aN[b][1] = 0.0;
        for (int j = 0; j < i; ++j, ++n) {
          const int s = n % S;
          mbar_wait_hint(full + s, (n / S) & 1u);
          const double* A = reinterpret_cast<const double*>(slots + s * T2);
          const double* cj = c3 + 192 * j + L.cb;
          double aT[4][2];
#pragma unroll
          for (int b = 0; b < 4; ++b) aT[b][0] = aT[b][1] = 0.0;
          if (ti == 32) {
            // 8 stages of (2 product + 2 transposed) tensor-core products, fragment loads one stage ahead
            Symv2Stage f0, f1;
            auto load = [&](Symv2Stage& f, int st) {
#pragma unroll
              for (int u = 0; u < 2; ++u) {
                const int kc = 2 * st + u;
                f.bn[u] = cj[12 * kc];
                f.an[u] = A[nbw[kc & 3] + 16 * (kc >> 2)];
                f.at[u] = A[tbw[kc & 1] + 128 * kc];
              }
            };
            load(f0, 0);
#pragma unroll
            for (int st = 0; st < 8; st += 2) {
              load(f1, st + 1);
              dmma_884(aN[0][0], aN[0][1], f0.an[0], f0.bn[0]);
              dmma_884(aT[0][0], aT[0][1], f0.at[0], bi[2 * st]);
              dmma_884(aN[1][0], aN[1][1], f0.an[1], f0.bn[1]);
              dmma_884(aT[1][0], aT[1][1], f0.at[1], bi[2 * st + 1]);
              if (st + 2 < 8) load(f0, st + 2);
              dmma_884(aN[2][0], aN[2][1], f1.an[0], f1.bn[0]);
              dmma_884(aT[2][0], aT[2][1], f1.at[0], bi[2 * st + 2]);
              dmma_884(aN[3][0], aN[3][1], f1.an[1], f1.bn[1]);
              dmma_884(aT[3][0], aT[3][1], f1.at[1], bi[2 * st + 3]);
            }
          } else {
            // last tile row of the block: ti < 32 rows
            if (8 * warp < ti) {
#pragma unroll 4
              for (int kc = 0; kc < 16; ++kc)
                dmma_884(aN[kc & 3][0], aN[kc & 3][1], A[nbw[kc & 3] + 16 * (kc >> 2)], cj[12 * kc]);
            }
#pragma unroll
            for (int kc = 0; kc < 16; ++kc)
              if (2 * kc < ti) {
                const bool ok = 2 * kc + (t >> 1) < ti;
                const double a = ok ? A[tbw[kc & 1] + 128 * kc] : 0.0;
                dmma_884(aT[kc & 3][0], aT[kc & 3][1], a, bi[kc]);
              }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(empty + s);
          add_out(j, (aT[0][0] + aT[1][0]) + (aT[2][0] + aT[3][0]), (aT[0][1] + aT[1][1]) + (aT[2][1] + aT[3][1]));
        }
        {
          // diagonal trapezoid: row block w times c_i (columns < 8w + 8) and column block w of
          // the row blocks below it, transposed, times c_i -- both land on entries 8w + g of tile row i
          const int s = n % S;
          mbar_wait_hint(full + s, (n / S) & 1u);
          const double* A = reinterpret_cast<const double*>(slots + s * T2);
          if (8 * warp < ti) {
            const double* Arow = A + 2 * (32 * warp * (warp + 1) + g * (8 * warp + 8)) - g * 64;
#pragma unroll
            for (int kc = 0; kc < 16; ++kc)
              if (kc < 4 * warp + 4) dmma_884(aN[kc & 3][0], aN[kc & 3][1], Arow[L.nb[kc & 3] + 16 * (kc >> 2)], bi[kc]);
#pragma unroll
            for (int rb = 1; rb < 4; ++rb)
              if (rb > warp && 8 * rb < ti) {
                const double* Ab = A + 2 * (32 * rb * (rb + 1)) - (t >> 1) * 64;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                  const int r = 2 * k + (t >> 1);
                  const bool ok = 8 * rb + r < ti;
                  const double a = ok ? Ab[2 * r * (8 * rb + 8) + tbw[k & 1]] : 0.0;
                  dmma_884(aN[k][0], aN[k][1], a, bi[4 * rb + k]);
                }
              }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(empty + s);
          ++n;
        }
        add_out(i, (aN[0][0] + aN[1][0]) + (aN[2][0] + aN[3][0]), (aN[0][1] + aN[1][1]) + (aN[2][1] + aN[3][1]));
      }
      consumers_sync(NC);
      for (int idx = tid; idx < nb * 2; idx += NC) {
        const int row = idx >> 1, rr = idx & 1;
        if (rr < nr) {
          const long rb = rr ? rb1 : rb0;
          Y[(long)row * s_row + (rb & ROFF)] = cflip(out[idx], flip_row((int)(rb >> 56), row, q));
        }
      }
    }
  }
}

template <int R>
static int launch_symv2_inv_t(const SymGeom& sg, const double2* G, const int* items, int nblocks, const int* klist,
                              double2* Y, long s_row, long s_k, int q, cudaStream_t s) {
  // measured (c1 / c2 / c3 applies, ms): 96 registers + a 2-slot ring (4 CTAs per SM at c1)
  // 0.667 / 0.760 / 1.239; 128 registers + 3 slots 0.681 / 0.801 / 1.260 -- the extra resident
  // CTA covers the other CTAs' right-hand-side gathers, a third slot does not pay
  static const int slots_env = env_int("VX_SYMV2_SLOTS", 2);
  // resident CTAs per SM the kernel is compiled for (4: 96 registers, 3: 128).  Measured
  // (apply kernel, ms): c1 (187-row sectors) 0.539 with 4 / 0.554 with 3; c3 (231 rows)
  // 0.513 / 0.486; c2 (413 rows, three CTAs fit in shared memory either way) 0.670 / 0.616
  static const int minb_env = env_int("VX_SYMV_MINB", 0);
  const int minb = minb_env ? minb_env : (sg.dmax <= 208 ? 4 : 3);
  static const int pfwin = env_int("VX_SYMV_PF", 24) * 64;  // L2 prefetch window, entries
  const int S = slots_env < 2 ? 2 : (slots_env > 12 ? 12 : slots_env);
  const int npad = (sg.dmax + 31) / 32 * 32;
  const size_t smem = ((size_t)2 * S * 8 + 127) / 128 * 128 + (size_t)S * 1024 * sizeof(double2) +
                      (size_t)npad * 2 * sizeof(double2) + (size_t)npad * 6 * sizeof(double);
  auto kern = minb == 2 ? symv2_inv_kernel<R, 2> : minb == 4 ? symv2_inv_kernel<R, 4> : symv2_inv_kernel<R, 3>;
  VX_REQUIRE((int)smem + 1024 <= device_smem_optin(), "symmetric inverse apply smem %zu too large", smem);
  static size_t smem_set[3] = {0, 0, 0};  // per kernel variant: raise the limit once per size, not per launch
  size_t& have = smem_set[minb == 2 ? 0 : minb == 4 ? 2 : 1];
  if (have < smem) {
    VX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    have = smem;
  }
  kern<<<nblocks, (SYMV_WARPS + 1) * 32, smem, s>>>(sg, G, items, nblocks, klist, Y, s_row, s_k, S, q, pfwin);
  VX_CHECK_LAUNCH("symv2_inv_kernel");
  return VX_OK;
}

static int launch_symv_inv(const SymGeom& sg, const double2* G, const int* items, int nblocks, int direct_r,
                           const int* klist, double2* Y, long s_row, long s_k, int q, cudaStream_t s) {
  if (nblocks <= 0) return VX_OK;
  VX_REQUIRE(direct_r == 1 || direct_r == 2, "symmetric inverse apply: direct_r must be 1 or 2");
  return direct_r == 2 ? launch_symv2_inv_t<2>(sg, G, items, nblocks, klist, Y, s_row, s_k, q, s)
                       : launch_symv2_inv_t<1>(sg, G, items, nblocks, klist, Y, s_row, s_k, q, s);
}
