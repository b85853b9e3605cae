// Symmetric ("W-symmetric") factor storage and its block solve -- included by
// circulant.cu after the ragged LU solve (uses LuGeom, dl_n, dl_off, du_off,
// the mbarrier / bulk-copy helpers and the flip conventions defined there).
//
// Why: D_k = I - M N_k with M = diag(m~) (reference accel.py:71-91).  The
// Galerkin Green's tensor is even under d -> -d, so N_k^T = S N_k S with S =
// -1 on the x-component rows (the x-mirror used for factor sharing), hence
// A_k = S M^-1 D_k = S M^-1 - S N_k is complex SYMMETRIC whenever m~ has no
// zero entry.  The orbit (sector) transform is real orthogonal and commutes
// with S M, so every sector block B = W (V^T A V) keeps the property with the
// diagonal W = S M restricted to the sector rows.  Factorised WITHOUT row
// interchanges, B = L U with U = diag(u) W L^T W^-1, so L (unit lower) and the
// pivots u determine U:
//     forward   L y = b
//     scale     c = y / (u W)          (h = 1 / (u W) per row)
//     backward  L^T z = c,  x = W z
// Only the lower triangle is stored: HALF the factor bytes of the LU layout.
// The build factorises without pivoting (panel kernel nopiv flag) and the
// pack kernel CHECKS, per block, that the computed U equals the symmetric
// reconstruction (relative deviation <= SYM_TOL) and that no pivot is tiny;
// otherwise the caller falls back to the pivoted LU layout.
//
// Stored form (tiles of 32, t_i = rows of tile row i): the off-diagonal tiles
// are PRE-MULTIPLIED by the inverse diagonal tile of their row,
//     L'_ij = inv(L_ii) L_ij   (i > j),
// which removes the diagonal solve from both recurrences:
//     forward   y_i = inv(L_ii) b_i - sum_{j<i} L'_ij y_j
//     backward  t_i = c_i - sum_{j>i} L'_ji^T t_j      (t_i = L_ii^T z_i)
//               z_i = inv(L_ii)^T t_i                  (off the critical path:
//                                                       evaluated one step late)
// so a tile row costs ONE reduction + publication instead of two.
//
// Layout of one block of dimension d (nt = ceil(d/32)): tile row i ("band") at
// sym_band(i); inside it the off-diagonal tiles (i, j < i), t_i x 32, ROW-major
// (row r at 32 r), then the diagonal "trapezoid": row r of inv(L_ii) with
// 8 (r / 8) + 8 entries (the lower triangle by 8-row blocks: explicit unit
// diagonal and zeros above it inside the diagonal 8 x 8 blocks), row r at
// trap_off(r).  Inside every row the 32-byte units (two entries) are
// XOR-swizzled by sw(r) = the two low bits of r exchanged: entry [r][c] at unit
// ((c >> 1) ^ sw(r)), so the FP64 tensor-core fragment loads of both passes
// (per half warp: 4 rows x 32 bytes forward, 2 rows x 64 bytes backward) are
// shared-memory bank-conflict free.
// Per frequency slot the nsec sector blocks follow each other (soff/kstride);
// h: [slot][dmax] (1 / (u W)), w: [sector][dmax] (W; shared by all k).
//
// Included INSIDE namespace vx.

__host__ __device__ __forceinline__ long sym_band(int i) { return 512L * i * (i - 1) + 640L * i; }
// offset of trapezoid row r (entries), rows of 8 (r / 8) + 8
__host__ __device__ __forceinline__ int trap_off(int r) {
  const int rb = r >> 3;
  return 32 * rb * (rb + 1) + (r & 7) * (8 * rb + 8);
}
__host__ __device__ __forceinline__ int trap_size(int t) { return trap_off(t); }  // rows 0..t-1
__host__ __device__ __forceinline__ long sym_size(int d) {
  const int nt = (d + 31) / 32, tl = d - 32 * (nt - 1);
  return sym_band(nt - 1) + 32L * tl * (nt - 1) + trap_size(tl);
}
// position of column c inside (swizzled) row r
__host__ __device__ __forceinline__ int sym_rsw(int r) { return ((r & 1) << 1) | ((r >> 1) & 1); }
__host__ __device__ __forceinline__ int sym_swz(int r, int c) { return ((((c >> 1) ^ sym_rsw(r)) << 1) | (c & 1)); }

struct SymGeom {
  int nsec, dmax;
  int dims[4];
  long soff[4];
  long kstride;
  const double2* h;  // [slot][dmax]
  const double2* w;  // [sector][dmax]
  int inverse;       // 0: factors (lu_solve_sym_kernel); 1: symmetric inverse G (lu_syminv.cuh)
};

constexpr int SYM_MAX_DIM = 1024;

static int make_sym(int nsec, const int* dims, int dmax, const void* h, const void* w, SymGeom* sg) {
  VX_REQUIRE(nsec >= 1 && nsec <= 4 && dims, "symmetric geometry needs 1..4 sector dims");
  VX_REQUIRE(dmax > 32 && dmax <= SYM_MAX_DIM, "symmetric storage is for multi-tile blocks (32 < dmax <= %d)",
             SYM_MAX_DIM);
  sg->nsec = nsec;
  sg->dmax = dmax;
  sg->inverse = 0;
  long off = 0;
  for (int s = 0; s < 4; ++s) {
    sg->dims[s] = s < nsec ? dims[s] : 0;
    sg->soff[s] = off;
    if (s < nsec) {
      VX_REQUIRE(dims[s] >= 1 && dims[s] <= dmax, "sector dim %d out of range (dmax %d)", dims[s], dmax);
      off += sym_size(dims[s]);
    }
  }
  sg->kstride = off;
  sg->h = reinterpret_cast<const double2*>(h);
  sg->w = reinterpret_cast<const double2*>(w);
  return VX_OK;
}

__device__ __forceinline__ const double2* sym_block(const SymGeom& sg, const double2* F, int slot, int& nb,
                                                    int& sec) {
  sec = slot % sg.nsec;
  nb = sec == 0 ? sg.dims[0] : sec == 1 ? sg.dims[1] : sec == 2 ? sg.dims[2] : sg.dims[3];
  const long so = sec == 0 ? sg.soff[0] : sec == 1 ? sg.soff[1] : sec == 2 ? sg.soff[2] : sg.soff[3];
  return F + (long)(slot / sg.nsec) * sg.kstride + so;
}

// ------------------------------------------------------------------ pack
// padded (dmax geometry, split diagonal tiles) -> symmetric layout + h, and
// the per-block check: dev[2 slot] = max |U - diag(u) W L^T W^-1| / max|U|
// over the off-diagonal tiles and the inverse diagonal tiles, dev[2 slot + 1]
// = min |u| / max |u|.  One CTA per slot.
__global__ void __launch_bounds__(256) lu_sym_pack_kernel(LuGeom g, SymGeom sg, const double2* __restrict__ P,
                                                          double2* __restrict__ Q, double2* __restrict__ H,
                                                          double* __restrict__ dev) {
  __shared__ double2 Di[32][33];  // inv(L_ii), full (unit diagonal, zeros above)
  __shared__ double2 Ls[32][33];  // L_ij
  __shared__ double rs[6][8];
  const int slot = blockIdx.x;
  int nb, sec;
  double2* dst = const_cast<double2*>(sym_block(sg, Q, slot, nb, sec));
  const double2* src = P + (long)slot * g.blk;
  const double2* W = sg.w + (long)sec * sg.dmax;
  const int T = g.T, T2 = T * T, nt = g.nt;
  const int tid = threadIdx.x;
  auto uinv = [&](int row) {  // 1 / u_row from the inverse diagonal tile
    const int i = row / T, r = row - i * T;
    return src[(long)(i * nt + i) * T2 + dl_n(T) + du_off(T, r, r)];
  };
  // NaN never compares: map it to a huge deviation so fmax keeps it
  auto mag = [](double2 v) { const double a = hypot(v.x, v.y); return a == a ? a : 1e300; };
  double d_off = 0.0, m_off = 0.0, d_dia = 0.0, m_dia = 0.0;
  double umin = 1e300, umax = 0.0;
  // ---- the symmetry check on the unpivoted factors, and h
  const long tot = (long)nb * nb;
  for (long e = tid; e < tot; e += blockDim.x) {
    const int R = (int)(e / nb), C = (int)(e - (long)R * nb);
    const int i = R / T, j = C / T, r = R - i * T, c = C - j * T;
    if (i > j) {
      const double2 v = src[(long)(i * nt + j) * T2 + c * T + r];
      // partner: U[C][R] (C < R) = u_C W_C L[R][C] / W_R
      const double2 uv = src[(long)(j * nt + i) * T2 + r * T + c];
      const double2 rec = cdiv(cmul(v, W[C]), cmul(uinv(C), W[R]));
      const double2 df = csub(uv, rec);
      d_off = fmax(d_off, mag(df));
      m_off = fmax(m_off, mag(uv));
    } else if (i == j && r > c) {
      const double2 v = src[(long)(i * nt + i) * T2 + dl_off(T, r, c)];
      // partner: inv(U_ii)[c][r] = W_c invL[r][c] / (W_r u_r)
      const double2 iu = src[(long)(i * nt + i) * T2 + dl_n(T) + du_off(T, c, r)];
      const double2 rec = cdiv(cmul(cmul(W[C], v), uinv(R)), W[R]);
      const double2 df = csub(iu, rec);
      d_dia = fmax(d_dia, mag(df));
      m_dia = fmax(m_dia, mag(iu));
    } else if (R == C) {
      const double2 ui = uinv(R);  // 1/u
      const double a = mag(ui);
      m_dia = fmax(m_dia, a);
      umin = fmin(umin, 1.0 / a);
      umax = fmax(umax, 1.0 / a);
      // h = 1 / (u W) = (1/u) / W
      H[(long)slot * sg.dmax + R] = cdiv(ui, W[R]);
    }
  }
  // ---- the stored tiles: trapezoid inv(L_ii), L'_ij = inv(L_ii) L_ij
  const int ntb = (nb + 31) / 32;
  for (int i = 0; i < ntb; ++i) {
    const int ti = min(32, nb - 32 * i);
    const double2* dsrc = src + (long)(i * nt + i) * T2;
    __syncthreads();
    for (int e = tid; e < 1024; e += blockDim.x) {
      const int r = e >> 5, c = e & 31;
      Di[r][c] = r > c ? dsrc[dl_off(T, r, c)] : cmk(r == c ? 1.0 : 0.0, 0.0);
    }
    __syncthreads();
    double2* band = dst + sym_band(i);
    double2* trap = band + 32L * ti * i;
    for (int e = tid; e < 1024; e += blockDim.x) {
      const int r = e >> 5, c = e & 31;
      if (r < ti && c < 8 * (r >> 3) + 8) trap[trap_off(r) + sym_swz(r, c)] = Di[r][c];
    }
    for (int j = 0; j < i; ++j) {
      const double2* tsrc = src + (long)(i * nt + j) * T2;
      __syncthreads();
      for (int e = tid; e < 1024; e += blockDim.x) {
        const int c = e >> 5, r = e & 31;  // source tile is column-major
        Ls[r][c] = tsrc[e];
      }
      __syncthreads();
      double2* tile = band + 32L * ti * j;
      for (int e = tid; e < 1024; e += blockDim.x) {
        const int r = e >> 5, c = e & 31;
        if (r < ti) {
          double2 a = Ls[r][c];  // unit diagonal term
          for (int k = 0; k < r; ++k) cfma(a, Di[r][k], Ls[k][c]);
          tile[r * 32 + sym_swz(r, c)] = a;
        }
      }
    }
  }
  // block reductions (max of d_off, m_off, d_dia, m_dia, umax; min of umin)
  double v6[6] = {d_off, m_off, d_dia, m_dia, umax, -umin};
  const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int qq = 0; qq < 6; ++qq) {
    double v = v6[qq];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) rs[qq][warp] = v;
  }
  __syncthreads();
  if (tid == 0) {
    double o6[6];
    for (int qq = 0; qq < 6; ++qq) {
      o6[qq] = rs[qq][0];
      for (int w = 1; w < (int)(blockDim.x / 32); ++w) o6[qq] = fmax(o6[qq], rs[qq][w]);
    }
    const double r1 = o6[1] > 0 ? o6[0] / o6[1] : 0.0, r2 = o6[3] > 0 ? o6[2] / o6[3] : 0.0;
    double devv = fmax(r1, r2);
    if (!(devv == devv)) devv = 1e300;  // NaN
    dev[2L * slot] = devv;
    const double mn = -o6[5], mx = o6[4];
    dev[2L * slot + 1] = (mx > 0 && mn == mn) ? mn / mx : 0.0;
  }
}

// symmetric layout -> padded LU layout (dmax geometry, split diagonal tiles,
// identity padding): the views and multi-RHS applies read that layout.
// One CTA per slot: L_ij = L_ii L'_ij with L_ii = inv(inv(L_ii)) rebuilt per
// tile row by one warp (column-wise forward substitution).
__global__ void __launch_bounds__(256) lu_sym_unpack_kernel(LuGeom g, SymGeom sg, const double2* __restrict__ Q,
                                                            double2* __restrict__ P) {
  __shared__ double2 Di[32][33];  // inv(L_ii) full, then (same storage) the tiles L'_ij
  __shared__ double2 Li[32][33];  // L_ii full
  double2 (*Xs)[33] = Di;
  const int slot = blockIdx.x;
  int nb, sec;
  const double2* src = sym_block(sg, Q, slot, nb, sec);
  const double2* W = sg.w + (long)sec * sg.dmax;
  const double2* Hs = sg.h + (long)slot * sg.dmax;
  double2* dst = P + (long)slot * g.blk;
  const int T = g.T, T2 = T * T, np = g.npad, nt = g.nt;
  const int tid = threadIdx.x;
  auto invL = [&](int R, int C) {  // inv(L_ii)[r][c] of the diagonal tile holding (R, C), R > C
    const int i = R / T, r = R - i * T, c = C - i * T;
    const int ti = min(T, nb - T * i);
    return src[sym_band(i) + 32L * ti * i + trap_off(r) + sym_swz(r, c)];
  };
  // ---- padding and diagonal tiles (element-wise)
  const long tot = (long)np * np;
  for (long e = tid; e < tot; e += blockDim.x) {
    const int C = (int)(e / np), R = (int)(e - (long)C * np);
    const int i = R / T, j = C / T, r = R - i * T, c = C - j * T;
    long po;
    if (i != j) po = (long)(i * nt + j) * T2 + (long)c * T + r;
    else if (r > c) po = (long)(i * nt + i) * T2 + dl_off(T, r, c);
    else po = (long)(i * nt + i) * T2 + dl_n(T) + du_off(T, r, c);
    if (R >= nb || C >= nb) {
      dst[po] = cmk(R == C ? 1.0 : 0.0, 0.0);
    } else if (i == j) {
      double2 v;
      if (r > c) v = invL(R, C);
      else if (r == c) v = cmul(Hs[R], W[R]);  // 1/u
      else v = cmul(cmul(W[R], invL(C, R)), Hs[C]);  // inv(U_ii)[r][c] = W_r invL[c][r] h_c
      dst[po] = v;
    }
  }
  // ---- off-diagonal tiles: L_ij = L_ii L'_ij and U_ji[R][C] = L[C][R] / (h_R W_C)
  const int ntb = (nb + 31) / 32;
  for (int i = 1; i < ntb; ++i) {
    const int ti = min(32, nb - 32 * i);
    const double2* band = src + sym_band(i);
    const double2* trap = band + 32L * ti * i;
    __syncthreads();
    for (int e = tid; e < 1024; e += blockDim.x) {
      const int r = e >> 5, c = e & 31;
      double2 v = cmk(r == c ? 1.0 : 0.0, 0.0);
      if (r < ti && c < r) v = trap[trap_off(r) + sym_swz(r, c)];
      Di[r][c] = v;
      Li[r][c] = cmk(r == c ? 1.0 : 0.0, 0.0);
    }
    __syncthreads();
    if (tid < 32) {  // column c of L_ii: Di x = e_c
      const int c = tid;
      for (int r = c + 1; r < 32; ++r) {
        double2 a = cmk(0.0, 0.0);
        for (int k = c; k < r; ++k) cfms(a, Di[r][k], Li[k][c]);
        Li[r][c] = a;
      }
    }
    for (int j = 0; j < i; ++j) {
      const double2* tile = band + 32L * ti * j;
      __syncthreads();
      for (int e = tid; e < 1024; e += blockDim.x) {
        const int r = e >> 5, c = e & 31;
        Xs[r][c] = r < ti ? tile[r * 32 + sym_swz(r, c)] : cmk(0.0, 0.0);
      }
      __syncthreads();
      for (int e = tid; e < 1024; e += blockDim.x) {
        const int r = e >> 5, c = e & 31;
        if (r < ti) {
          double2 a = Xs[r][c];
          for (int k = 0; k < r; ++k) cfma(a, Li[r][k], Xs[k][c]);
          const int R = 32 * i + r, C = 32 * j + c;
          dst[(long)(i * nt + j) * T2 + (long)c * T + r] = a;
          dst[(long)(j * nt + i) * T2 + (long)r * T + c] = cdiv(a, cmul(Hs[C], W[R]));
        }
      }
    }
  }
}

// ------------------------------------------------------------------ solve
// One CTA per work item (a stored sector block and its one or two right-hand
// sides: the x-mirror pair).  A producer warp streams the tiles with
// cp.async.bulk into an S-slot mbarrier ring; 8 consumer warps run every tile
// product on the FP64 TENSOR CORES (mma.sync.m8n8k4):
//   A fragment = 8 x 4 doubles of the stored tile = 8 rows x 2 complex entries
//                (re, im interleaved), straight from the ring slot;
//   B fragment = 4 x 8: column "Re(rhs)" = (y_r, -y_i) per entry, column
//                "Im(rhs)" = (y_i, y_r): the two right-hand sides fill 4 of
//                the 8 columns;
//   C          = 8 rows x (Re1, Im1, Re2, Im2): lanes t < 2 hold the complex sums.
// Warp w owns the entries 4w..4w+3 of the CONTRACTED index of every tile
// (columns forward, rows backward: the transposed product only changes the
// fragment addresses), so one B fragment serves the four 8-row blocks of a
// tile, there are no shuffle reductions, and a warp only ever reads ITS OWN
// slice of the solution vector.  The eight warps' partial sums meet in shared
// memory once per tile row (fixed order: bitwise reproducible) through a pair
// of mbarriers (written / read) instead of CTA barriers, and the tiles of a
// row that do not depend on the previous row's result run before the wait.
// Shared-memory wavefronts per tile byte drop ~3x against the scalar
// row-owner kernel this replaces (its L1/shared data pipe ran 89 % busy at
// 41 % of the HBM peak, profiles/r02_sym_v1_ncu.txt).
// The backward pass re-reads the triangle the forward pass just streamed, last
// band first (evict_last / evict_first L2 hints): with 3 CTAs per SM the
// in-flight triangles (148 x 3 x 290 KB at c1) stay in L2 and HBM delivers
// each factor byte once.
constexpr int SYM_WARPS = 8;

// (volatile: the warp-collective must stay where it is written -- without it the
// compiler sinks the products into the divergent "lanes t < 2 store" branches)
__device__ __forceinline__ void dmma_884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// bulk copy with an L2 eviction-priority hint (evict_last: the forward pass's
// tiles, which the backward pass re-reads; evict_first: the re-read itself)
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              bool keep) {
  uint64_t pol;
  if (keep) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  else asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// L2 prefetch of a span of the factor stream (no shared-memory destination):
// the forward pass's tiles are requested from HBM a window ahead of the ring,
// so the ring's own loads see L2 latency
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// wait with a suspend-time hint: the polling warp sleeps in hardware instead
// of spinning through the issue slots of the warps that have work
__device__ __forceinline__ void mbar_wait_hint(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      " @!p bra W%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity), "r"(20000u)
      : "memory");
}

template <int R, int MINB>
__global__ void __launch_bounds__((SYM_WARPS + 1) * 32, MINB)
    lu_solve_sym_kernel(SymGeom sg, const double2* __restrict__ F, const int* __restrict__ items, int nwork,
                        const int* __restrict__ klist, double2* Y, long s_row, long s_k, int S, int q, int l2hint,
                        int pfwin) {
  extern __shared__ __align__(128) unsigned char smraw[];
  constexpr int T2 = 1024;
  const int npad = (sg.dmax + 31) / 32 * 32;
  const int ystr = npad + 4;  // right-hand side 1 starts 64 bytes off a 512-byte multiple (B-fragment banks)
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw);
  uint64_t* empty = full + S;
  uint64_t* pbar = empty + S;   // all warps' partial sums of a step are written
  uint64_t* rdone = pbar + 1;   // all warps have read them
  double2* slots = reinterpret_cast<double2*>(smraw + ((2 * S + 2) * 8 + 127) / 128 * 128);
  double2* y = slots + (long)S * T2;           // [2][ystr]; warp w owns rows 4w..4w+3 of every tile row
  double2* pt = y + 2L * ystr;                 // [SYM_WARPS][32][2]: partial sums of the recurrence
  double2* pz = pt + SYM_WARPS * 64;           // [SYM_WARPS][32][2]: partial sums of the late z_i
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, SYM_WARPS);
    }
    mbar_init(pbar, SYM_WARPS);
    mbar_init(rdone, SYM_WARPS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == SYM_WARPS) {
    if (lane == 0) {
      int s = 0;
      uint32_t use = 0;  // completed passes over the ring
      bool fwd = true;
      auto emit = [&](const double2* src, uint32_t elems) {
        if (use > 0) mbar_wait_hint(empty + s, (use - 1) & 1u);
        const uint32_t bytes = elems * (uint32_t)sizeof(double2);
        mbar_expect_tx(full + s, bytes);
        if (l2hint) bulk_g2s_hint(slots + s * T2, src, bytes, full + s, fwd);
        else bulk_g2s(slots + s * T2, src, bytes, full + s);
        if (++s == S) {
          s = 0;
          ++use;
        }
      };
      for (int w = blockIdx.x; w < nwork; w += gridDim.x) {
        const int slot = items[3 * w], cnt = items[3 * w + 2];
        int nb, sec;
        const double2* Fb = sym_block(sg, F, slot, nb, sec);
        const int nt = (nb + 31) / 32;
        const long total = sym_size(nb);
        long pf = 0;  // entries of this block already requested into L2
        auto prefetch_to = [&](long upto) {
          upto = upto < total ? upto : total;
          while (pf < upto) {
            const long n = upto - pf < 1024 ? upto - pf : 1024;
            bulk_prefetch_l2(Fb + pf, (uint32_t)(n * sizeof(double2)));
            pf += n;
          }
        };
        auto tile = [&](int i, int j) {  // j == i: the trapezoid
          const int ti = min(32, nb - 32 * i);
          const long off = sym_band(i) + 32L * ti * j;
          const uint32_t n = (uint32_t)(i == j ? trap_size(ti) : ti * 32);
          if (fwd && pfwin > 0) prefetch_to(off + n + pfwin);
          emit(Fb + off, n);
        };
        for (int ch = 0; ch < (cnt + R - 1) / R; ++ch) {
          fwd = true;
          pf = 0;
          for (int i = 0; i < nt; ++i) {
            for (int j = 0; j < i; ++j) tile(i, j);
            tile(i, i);
          }
          fwd = false;
          for (int i = nt - 1; i >= 0; --i) {
            for (int j = nt - 1; j > i; --j) tile(j, i);
            if (i + 1 < nt) tile(i + 1, i + 1);
          }
          tile(0, 0);
        }
      }
    }
    return;
  }

  int cs = 0;
  uint32_t cph = 0;
  auto wait_tile = [&]() -> const double* {
    mbar_wait_hint(full + cs, cph);
    return reinterpret_cast<const double*>(slots + cs * T2);
  };
  auto release_tile = [&]() {
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + cs);
    if (++cs == S) {
      cs = 0;
      cph ^= 1u;
    }
  };
  // fragment coordinates
  const int g = lane >> 2, t = lane & 3;
  // B fragment: column g < 4 is (Re, Im)[g & 1] of right-hand side g >> 1; row t
  // is part t & 1 of contracted entry t >> 1
  const int bim = g & 1;
  const double bsg = g < 4 ? ((!bim && (t & 1)) ? -1.0 : 1.0) : 0.0;
  double* yd = reinterpret_cast<double*>(y);
  const int boff = ((((g >> 1) & 1) * ystr + (t >> 1)) << 1) + ((t & 1) ^ bim) + 8 * warp;
  const int kc0 = 2 * warp;                               // this warp's two 32-byte units of the contracted index
  const int fsw = ((g & 1) << 1) | ((g >> 1) & 1);        // forward: row = 8 rb + g
  const int r0 = 4 * warp + (t >> 1);                     // backward: contracted rows r0 (kk = 0), r0 + 2 (kk = 1)
  const int bsw = (t >> 1) << 1;                          // backward: swizzle of row r0 + 2 kk is bsw | kk
  const int bcol = ((g & 1) << 1) + (t & 1);
  double acc[4][2], acz[4][2];
  auto zero = [&](double (&a)[4][2]) {
#pragma unroll
    for (int b = 0; b < 4; ++b) a[b][0] = a[b][1] = 0.0;
  };
  // forward product of a full-width tile: rows 8 rb + g (rb < nrb), entries 4w..4w+3
  auto fwd_tile = [&](const double* A, int nrb, int opbase) {
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      const double b = -bsg * yd[boff + 2 * opbase + 4 * kk];
      const int ko = ((kc0 + kk) ^ fsw) << 2;
#pragma unroll
      for (int rb = 0; rb < 4; ++rb)
        if (rb < nrb) dmma_884(acc[rb][0], acc[rb][1], A[(8 * rb + g) * 64 + ko + t], b);
    }
  };
  // forward product of the trapezoid: row block rb holds 8 rb + 8 entries per row
  auto fwd_trap = [&](const double* A, int nrb, int opbase) {
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      const double b = bsg * yd[boff + 2 * opbase + 4 * kk];
      const int ko = ((kc0 + kk) ^ fsw) << 2;
#pragma unroll
      for (int rb = 0; rb < 4; ++rb)
        if (rb < nrb && rb >= (warp >> 1))
          dmma_884(acc[rb][0], acc[rb][1], A[2 * (32 * rb * (rb + 1) + g * (8 * rb + 8)) + ko + t], b);
    }
  };
  // transposed product of a tile with tj rows: contracted rows 4w..4w+3, outputs 8 cb + g
  auto bwd_tile = [&](const double* A, int tj, int opbase) {
    if (4 * warp >= tj) return;
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      const int r = r0 + 2 * kk;
      const bool ok = r < tj;
      const double b = -bsg * yd[boff + 2 * opbase + 4 * kk];
      const double* Ar = A + r * 64 + bcol;
#pragma unroll
      for (int cb = 0; cb < 4; ++cb) {
        const double a = ok ? Ar[((4 * cb + (g >> 1)) ^ (bsw | kk)) << 2] : 0.0;
        dmma_884(acc[cb][0], acc[cb][1], a, b);
      }
    }
  };
  // transposed product of the trapezoid (tp rows) with t_p: z_p = inv(L_pp)^T t_p
  auto bwd_trap = [&](const double* A, int tp, int opbase) {
    if (4 * warp >= tp) return;
    const int rbk = warp >> 1;
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      const int r = r0 + 2 * kk;
      const bool ok = r < tp;
      const double b = bsg * yd[boff + 2 * opbase + 4 * kk];
      const double* Ar = A + 2 * (32 * rbk * (rbk + 1) + (r & 7) * (8 * rbk + 8)) + bcol;
#pragma unroll
      for (int cb = 0; cb < 4; ++cb)
        if (cb <= rbk) {
          const double a = ok ? Ar[((4 * cb + (g >> 1)) ^ (bsw | kk)) << 2] : 0.0;
          dmma_884(acz[cb][0], acz[cb][1], a, b);
        }
    }
  };
  // ---- cross-warp exchange of the partial sums: pbar completes once per step
  // when every warp has stored its partials, rdone once every warp has read them
  uint32_t nput = 0, nget = 0;
  auto put_partials = [&](bool with_z) {
    if (nput > 0) mbar_wait_hint(rdone, (nput - 1) & 1u);
    if (t < 2) {
#pragma unroll
      for (int b = 0; b < 4; ++b) pt[((warp * 32 + 8 * b + g) << 1) + t] = cmk(acc[b][0], acc[b][1]);
      if (with_z) {
#pragma unroll
        for (int b = 0; b < 4; ++b) pz[((warp * 32 + 8 * b + g) << 1) + t] = cmk(acz[b][0], acz[b][1]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(pbar);
    ++nput;
  };
  auto wait_partials = [&]() {
    mbar_wait_hint(pbar, nget & 1u);
    ++nget;
  };
  auto done_partials = [&]() {
    __syncwarp();
    if (lane == 0) mbar_arrive(rdone);
  };
  // this lane's entry of the warp's slice (lanes 0..7: row 4w + (lane >> 1), right-hand side lane & 1)
  const int sl_row = 4 * warp + ((lane >> 1) & 3), sl_rr = lane & 1;
  auto sum8 = [&](const double2* p) {
    const int e = (sl_row << 1) + sl_rr;
    double2 s = p[e];
#pragma unroll
    for (int w = 1; w < SYM_WARPS; ++w) s = cadd(s, p[w * 64 + e]);
    return s;
  };

  for (int w = blockIdx.x; w < nwork; w += gridDim.x) {
    const int slot = items[3 * w], beg = items[3 * w + 1], cnt = items[3 * w + 2];
    int nb, sec;
    (void)sym_block(sg, F, slot, nb, sec);
    const int nt = (nb + 31) / 32;
    const double2* hrow = sg.h + (long)slot * sg.dmax;
    const double2* wrow = sg.w + (long)sec * sg.dmax;
    for (int ch = 0; ch < (cnt + R - 1) / R; ++ch) {
      const int rho0 = ch * R;
      const int nr = min(R, cnt - rho0);
      long rb_own = 0;  // global offset / flips of this lane's right-hand side (sl_rr)
      if (sl_rr < nr) {
        const int kraw = klist ? klist[beg + rho0 + sl_rr] : beg + rho0 + sl_rr;
        rb_own = rhs_base(kraw, rho0 + sl_rr, 1, s_k);
      }
      const bool rhs_on = sl_rr < nr;
      // the warp's slices of b (rows 4w..4w+3 of every tile row, both right-hand sides)
      const long rb_0 = __shfl_sync(0xffffffffu, rb_own, 0), rb_1 = __shfl_sync(0xffffffffu, rb_own, 1);
      for (int e = lane; e < 8 * (npad / 32); e += 32) {
        const int row = 32 * (e >> 3) + 4 * warp + ((e >> 1) & 3), rr = e & 1;
        const long rb = rr ? rb_1 : rb_0;
        double2 v = cmk(0.0, 0.0);
        if (row < nb && rr < nr) v = cflip(Y[(long)row * s_row + (rb & ROFF)], flip_row((int)(rb >> 56), row, q));
        y[rr * ystr + row] = v;
      }
      __syncwarp();
      // ---------------- forward: y_i = inv(L_ii) b_i - sum_{j<i} L'_ij y_j
      // the tiles that do not need y_{i-1} run before the wait for it
      auto finish_fwd = [&](int i) {  // y_i slice <- sum of the partials
        const int ti = min(32, nb - 32 * i);
        wait_partials();
        if (lane < 8) {
          const double2 s = sum8(pt);
          y[sl_rr * ystr + 32 * i + sl_row] = sl_row < ti ? s : cmk(0.0, 0.0);
        }
        done_partials();
      };
      for (int i = 0; i < nt; ++i) {
        const int ti = min(32, nb - 32 * i), nrb = (ti + 7) >> 3;
        zero(acc);
        for (int j = 0; j + 1 < i; ++j) {
          fwd_tile(wait_tile(), nrb, 32 * j);
          release_tile();
        }
        if (i > 0) {
          finish_fwd(i - 1);
          fwd_tile(wait_tile(), nrb, 32 * (i - 1));
          release_tile();
        }
        fwd_trap(wait_tile(), nrb, 32 * i);
        release_tile();
        put_partials(false);
      }
      finish_fwd(nt - 1);
      // ---------------- backward: t_i = c_i - sum_{j>i} L'_ji^T t_j with c = y / (u W);
      // z_{i+1} = inv(L_{i+1})^T t_{i+1} rides one step behind
      auto finish_bwd = [&](int p, double2 hv) {  // t_p slice <- c_p + partials; z_{p+1} -> global
        wait_partials();
        if (lane < 8) {
          const double2 s = sum8(pt);
          const int o = sl_rr * ystr + 32 * p + sl_row;
          y[o] = cadd(cmul(y[o], hv), s);
        } else if (lane < 16 && p + 1 < nt) {
          const double2 z = sum8(pz);
          const int row = 32 * (p + 1) + sl_row;
          if (row < nb && rhs_on)
            Y[(long)row * s_row + (rb_own & ROFF)] = cflip(cmul(z, wrow[row]), flip_row((int)(rb_own >> 56), row, q));
        }
        done_partials();
      };
      auto hval = [&](int p) {  // h of this lane's slice row in tile row p (issued early: used at finish_bwd)
        const int row = 32 * p + sl_row;
        return (lane < 8 && row < nb) ? hrow[row] : cmk(0.0, 0.0);
      };
      for (int i = nt - 1; i >= 0; --i) {
        zero(acc);
        zero(acz);
        const bool dep = i + 1 < nt;
        double2 hv = cmk(0.0, 0.0);
        if (dep) hv = hval(i + 1);
        for (int j = nt - 1; j > i + 1; --j) {
          bwd_tile(wait_tile(), min(32, nb - 32 * j), 32 * j);
          release_tile();
        }
        if (dep) {
          const int tp = min(32, nb - 32 * (i + 1));
          finish_bwd(i + 1, hv);
          bwd_tile(wait_tile(), tp, 32 * (i + 1));
          release_tile();
          bwd_trap(wait_tile(), tp, 32 * (i + 1));
          release_tile();
        }
        put_partials(dep);
      }
      {
        const double2 hv = hval(0);
        finish_bwd(0, hv);
        zero(acz);
        bwd_trap(wait_tile(), min(32, nb), 0);
        release_tile();
        put_partials(true);
        wait_partials();
        if (lane >= 8 && lane < 16) {
          const double2 z = sum8(pz);
          if (sl_row < nb && rhs_on)
            Y[(long)sl_row * s_row + (rb_own & ROFF)] =
                cflip(cmul(z, wrow[sl_row]), flip_row((int)(rb_own >> 56), sl_row, q));
        }
        done_partials();
      }
    }
  }
}

template <int R>
static int launch_solve_sym_t(const SymGeom& sg, const double2* F, const int* items, int nblocks,
                              const int* klist, double2* Y, long s_row, long s_k, int q, cudaStream_t s) {
  static const int slots_env = env_int("VX_SYM_SLOTS", 3);
  // 3 CTAs per SM: the in-flight triangles fit L2, so DRAM traffic ~= the stored bytes
  static const int minb = env_int("VX_SYM_MINB", 3);
  static const int l2hint = env_int("VX_SYM_L2HINT", 1);
  // forward tiles can be requested into L2 this many KB ahead of the ring (measured: no
  // effect on this kernel -- it is bound by its two dependent passes, not by HBM latency)
  static const int pfwin = env_int("VX_SYM_PF", 0) * 64;  // entries (16 bytes)
  const int S = slots_env < 2 ? 2 : (slots_env > 12 ? 12 : slots_env);
  const int npad = (sg.dmax + 31) / 32 * 32;
  const size_t smem = (((size_t)2 * S + 2) * 8 + 127) / 128 * 128 + (size_t)S * 1024 * sizeof(double2) +
                      ((size_t)(npad + 4) * 2 + 2 * SYM_WARPS * 64) * sizeof(double2);
  auto kern = minb == 2 ? lu_solve_sym_kernel<R, 2> : minb == 4 ? lu_solve_sym_kernel<R, 4> : lu_solve_sym_kernel<R, 3>;
  VX_REQUIRE((int)smem + 1024 <= device_smem_optin(), "symmetric solve smem %zu too large", smem);
  VX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<nblocks, (SYM_WARPS + 1) * 32, smem, s>>>(sg, F, items, nblocks, klist, Y, s_row, s_k, S, q, l2hint,
                                                   pfwin);
  VX_CHECK_LAUNCH("lu_solve_sym_kernel");
  return VX_OK;
}

static int launch_solve_sym(const SymGeom& sg, const double2* F, const int* items, int nblocks, int direct_r,
                            const int* klist, double2* Y, long s_row, long s_k, int q, cudaStream_t s) {
  if (nblocks <= 0) return VX_OK;
  VX_REQUIRE(direct_r == 1 || direct_r == 2, "symmetric solve: direct_r must be 1 or 2");
  return direct_r == 2 ? launch_solve_sym_t<2>(sg, F, items, nblocks, klist, Y, s_row, s_k, q, s)
                       : launch_solve_sym_t<1>(sg, F, items, nblocks, klist, Y, s_row, s_k, q, s);
}
