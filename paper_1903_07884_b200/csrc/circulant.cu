// Chan-circulant preconditioners (reference circulant.py, accel.py unfolds).
//
// Build:  Chan + x-DFT of the six generators (k-major output), then one CTA per
//         frequency block: unfold D_k = I - diag(m) N_k straight into tiled
//         storage, blocked right-looking LU with partial pivoting (LAPACK
//         zgetrf pivot rule |Re|+|Im|, first index on ties), diagonal tiles
//         replaced by their triangular inverses.
// Apply:  x-DFT (and y-DFT for 2-level) of the field, one CTA per frequency
//         block streaming its factor tiles exactly once in storage order
//         (forward: row i = tiles L_i0..L_i,i-1, inv(L_ii); backward: U tiles,
//         inv(U_ii)), inverse DFTs with 1/n folded into the storer.
//
// Factor storage per block: nt x nt tiles of T x T (T <= 32), tile (i, j) at
// offset (i*nt + j)*T*T, column-major inside the tile; rows/cols >= n are an
// identity pad.
#include "fft_long.cuh"

#include <algorithm>
#include <vector>

namespace vx {

struct LuGeom {
  int n, T, nt, npad;
  long blk;
};

// T = n for single-tile blocks (n <= 32), else 32: full warps in the solve and
// 8x8x4 DMMA blocking in the factorisation (c1: 726 -> 736, +2.8% stored).
static int lu_pick_tile(int n) {
  if (n <= 32) return n < 1 ? 1 : n;
  return 32;
}

static LuGeom lu_geom(int n) {
  LuGeom g;
  g.n = n;
  g.T = lu_pick_tile(n);
  g.nt = (n + g.T - 1) / g.T;
  g.npad = g.nt * g.T;
  g.blk = (long)g.npad * g.npad;
  return g;
}

__device__ __forceinline__ long lu_off(const LuGeom& g, int row, int col) {
  const int it = row / g.T, jt = col / g.T;
  return ((long)(it * g.nt + jt) * g.T + (col - jt * g.T)) * g.T + (row - it * g.T);
}

__constant__ int c_pair[9] = {0, 1, 2, 1, 3, 4, 2, 4, 5};

// Stored diagonal tiles of multi-tile blocks (nt > 1) are SPLIT (single-tile
// blocks keep the column-major packed tile, which their warp kernel stages
// whole): the first T(T-1)/2 entries hold inv(L_ii)
// strictly below the diagonal (packed by columns), the next T(T+1)/2 hold
// inv(U_ii) on and above it (packed by columns), so the forward and backward
// substitutions each stream only the half they use.
__host__ __device__ __forceinline__ int dl_n(int T) { return T * (T - 1) / 2; }
__host__ __device__ __forceinline__ int dl_off(int T, int r, int c) {  // r > c
  return c * (2 * T - c - 1) / 2 + (r - c - 1);
}
__host__ __device__ __forceinline__ int du_off(int T, int r, int c) {  // r <= c, relative to the U half
  return c * (c + 1) / 2 + r;
}
// row-packed halves of the ragged layout (vx_lu_repack): L row r at r(r-1)/2,
// U row r (columns r..t-1) at r t - r(r-1)/2
__host__ __device__ __forceinline__ int lrow_off(int r) { return r * (r - 1) / 2; }           // L half, row r
__host__ __device__ __forceinline__ int urow_off(int t, int r) { return r * t - r * (r - 1) / 2; }  // U half, row r

// Ragged ("packed") factor storage for the pipelined block solve: a block of
// dimension d keeps only its d x d entries -- tile (i, j) is t_i x t_j with
// t_i = min(T, d - T i), column-major (ld t_i), at T i d + t_i T j, diagonal
// tiles split-packed as above with T -> t_i.  Blocks are grouped per stored
// frequency slot: nsec sector blocks of dims[s] each (kstride = sum dims^2,
// soff = prefix sums), so the tile padding of the dmax geometry (c1 sectors
// 187/187/176/176 -> 192) is never streamed.  on = 0: the padded layout.
struct RagGeom {
  int on, nsec;
  int dims[4];
  long soff[4];
  long kstride;
};

// block of work slot `slot`: base pointer and dimension
__device__ __forceinline__ const double2* rag_block(const LuGeom& g, const RagGeom& rg, const double2* F, int slot,
                                                   int& nb) {
  if (!rg.on) {
    nb = g.n;
    return F + (long)slot * g.blk;
  }
  const int sec = slot % rg.nsec;  // selects, not a dynamic index (keeps rg in registers)
  nb = sec == 0 ? rg.dims[0] : sec == 1 ? rg.dims[1] : sec == 2 ? rg.dims[2] : rg.dims[3];
  const long so = sec == 0 ? rg.soff[0] : sec == 1 ? rg.soff[1] : sec == 2 ? rg.soff[2] : rg.soff[3];
  return F + (long)(slot / rg.nsec) * rg.kstride + so;
}

// ----------------------------------------------------------------- spectra
// Generator line l = (p, dz, dy) of a (6, nzz, nyy, *) tensor with strides.
struct GenLine {
  long sp, sz, sy;
  int nzz, nyy;
  __device__ __forceinline__ long base(int l) const {
    const int per = nzz * nyy;
    const int p = l / per, r = l - p * per;
    const int dz = r / nyy, dy = r - dz * nyy;
    return p * sp + dz * sz + dy * sy;
  }
};

struct LoadChanGen {
  const double2* __restrict__ g;
  GenLine gl;
  long sx;
  int n;
  __device__ __forceinline__ long line_base(int l) const { return gl.base(l); }
  __device__ __forceinline__ double2 operator()(long b, int s) const {
    const double2 tp = __ldg(g + b + (long)(n - 1 + s) * sx);
    if (s == 0) return tp;
    const double2 tn = __ldg(g + b + (long)(s - 1) * sx);
    const double fn = (double)n, ws = (double)(n - s), wt = (double)s;
    return cmk((ws * tp.x + wt * tn.x) / fn, (ws * tp.y + wt * tn.y) / fn);
  }
};

__global__ void proxy_kernel(int nx, long Ltot, const double2* __restrict__ lamT, double2 m00,
                             int q_is_one, double2* __restrict__ proxy) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nx) return;
  double2 v = cmul(m00, lamT[(long)k * Ltot]);
  proxy[k] = cmk((q_is_one ? 1.0 : 0.0) - v.x, -v.y);
}

// ---------------------------------------------------------------- LU build
constexpr int LU_WARPS = 4;
constexpr int LU_THREADS = LU_WARPS * 32;

// unfold parameters: rows/cols ordered a*q + iz*nyL + iy (reference accel.py:71-91);
// the 2-level (3nz)^2 block is the nyL = 1 case (accel.py:94-111).
struct Unfold {
  const double2* __restrict__ lamT;  // (blocks, 6, 2nzL-1, 2nyL-1)
  const double2* __restrict__ m;     // (nzL, nyL)
  const int* __restrict__ kset;      // slot -> block (null: identity)
  long Ltot;
  int nzL, nyL;
};


// FP64 tensor-core (DMMA, mma.sync.m8n8k4.f64) product on one half (16
// columns) of a 32 x 32 complex tile:
//   C[:, 16h:16h+16]  =  A * B[:, 16h:16h+16]      (SUB = false)
//   C[:, 16h:16h+16] -=  A * B[:, 16h:16h+16]      (SUB = true)
// A is staged in shared memory (column-major, ld 33 to spread banks); B and C
// are tiles in global memory (column-major, ld 32).  Complex = 4 real DMMAs.
// Fragments (verified by tools/dmma_probe.cu): A[l/4][l%4], B[l%4][l/4],
// C[l/4][2(l%4) + {0,1}].
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <bool SUB, int LDA = 33>
__device__ __forceinline__ void tile_mma_half(const double2* As, const double2* Bg, double2* Cg, int h,
                                              int lane) {
  const int r4 = lane >> 2, c4 = lane & 3;
  double cr[4][2][2], ci[4][2][2];
#pragma unroll
  for (int rb = 0; rb < 4; ++rb)
#pragma unroll
    for (int cb = 0; cb < 2; ++cb)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double2 v = cmk(0.0, 0.0);
        if (SUB) v = Cg[(16 * h + cb * 8 + 2 * c4 + e) * 32 + rb * 8 + r4];
        cr[rb][cb][e] = v.x;
        ci[rb][cb][e] = v.y;
      }
#pragma unroll 2
  for (int k0 = 0; k0 < 32; k0 += 4) {
    double ar[4], ai[4], nar[4], br[2], bi[2];
#pragma unroll
    for (int rb = 0; rb < 4; ++rb) {
      const double2 a = As[(k0 + c4) * LDA + rb * 8 + r4];
      ar[rb] = a.x;
      ai[rb] = a.y;
      nar[rb] = -a.x;
    }
#pragma unroll
    for (int cb = 0; cb < 2; ++cb) {
      const double2 b = Bg[(16 * h + cb * 8 + r4) * 32 + k0 + c4];
      br[cb] = b.x;
      bi[cb] = b.y;
    }
#pragma unroll
    for (int rb = 0; rb < 4; ++rb)
#pragma unroll
      for (int cb = 0; cb < 2; ++cb) {
        if (SUB) {  // C -= A B :  cr += -ar br + ai bi ; ci += -ar bi - ai br
          const double nai = -ai[rb];
          dmma884(cr[rb][cb][0], cr[rb][cb][1], nar[rb], br[cb]);
          dmma884(cr[rb][cb][0], cr[rb][cb][1], ai[rb], bi[cb]);
          dmma884(ci[rb][cb][0], ci[rb][cb][1], nar[rb], bi[cb]);
          dmma884(ci[rb][cb][0], ci[rb][cb][1], nai, br[cb]);
        } else {    // C = A B :  cr += ar br - ai bi ; ci += ar bi + ai br
          const double nai = -ai[rb];
          dmma884(cr[rb][cb][0], cr[rb][cb][1], ar[rb], br[cb]);
          dmma884(cr[rb][cb][0], cr[rb][cb][1], nai, bi[cb]);
          dmma884(ci[rb][cb][0], ci[rb][cb][1], ar[rb], bi[cb]);
          dmma884(ci[rb][cb][0], ci[rb][cb][1], ai[rb], br[cb]);
        }
      }
  }
  __syncwarp();
#pragma unroll
  for (int rb = 0; rb < 4; ++rb)
#pragma unroll
    for (int cb = 0; cb < 2; ++cb)
#pragma unroll
      for (int e = 0; e < 2; ++e)
        Cg[(16 * h + cb * 8 + 2 * c4 + e) * 32 + rb * 8 + r4] = cmk(cr[rb][cb][e], ci[rb][cb][e]);
}

__global__ void __launch_bounds__(LU_THREADS) lu_build_kernel(Unfold u, LuGeom g, double2* F,
                                                               int* perm, int* piv, int* info) {
  extern __shared__ double2 sm[];
  const int T = g.T, T2 = T * T, nt = g.nt, npad = g.npad, n = g.n;
  const int LD = T + 1, TL = T * LD;   // padded leading dimension of smem tiles
  double2* Ls = sm;                    // inv(L_kk), column-major, ld LD
  double2* Us = Ls + TL;               // inv(U_kk)
  double2* Bst = Us + TL;              // scratch (permutation composition)
  int* pivs = reinterpret_cast<int*>(Bst + TL);               // [T]
  double* redv = reinterpret_cast<double*>(pivs + 32);        // [LU_WARPS]
  int* redi = reinterpret_cast<int*>(redv + LU_WARPS);        // [LU_WARPS]
  int* flags = redi + LU_WARPS;                               // [0]=info [1]=any swap
  int* gpiv = flags + 4;                                      // [npad] full pivot record

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int slot = blockIdx.x;
  const int k = u.kset ? u.kset[slot] : slot;
  double2* A = F + (long)slot * g.blk;
  const double2* lam = u.lamT + (long)k * u.Ltot;
  const int q = u.nzL * u.nyL;

  // phase 0: D_k = I - diag(m) N_k into tiled storage (identity pad).
  // Per-index decomposition (component a, (z,y) offset, medium value) tabulated
  // once in shared memory (aliasing the not-yet-used Ls/Us/staging region), so
  // an entry costs two table lookups, one generator gather and a complex
  // multiply; a warp writes one 32-entry tile column (coalesced 512 B).
  {
    const int nyy = 2 * u.nyL - 1, nzz = 2 * u.nzL - 1;
    const int P = nzz * nyy, base = (u.nzL - 1) * nyy + (u.nyL - 1);
    int* key = reinterpret_cast<int*>(sm);
    double2* mtab = reinterpret_cast<double2*>(key + ((npad + 3) & ~3));
    for (int idx = tid; idx < npad; idx += LU_THREADS) {
      if (idx < n) {
        const int a = idx / q, rr = idx - a * q;
        const int iz = rr / u.nyL, iy = rr - iz * u.nyL;
        key[idx] = (a << 24) | (iz * nyy + iy);
        mtab[idx] = __ldg(u.m + rr);
      } else {
        key[idx] = -1;
      }
    }
    __syncthreads();
    const int ncolw = nt * nt * T;  // (tile, column) pairs
    for (int w = warp; w < ncolw; w += LU_WARPS) {
      const int tile = w / T, c = w - tile * T;
      const int it = tile / nt, jt = tile - it * nt;
      const int col = jt * T + c;
      if (lane >= T) continue;
      const int row = it * T + lane;
      double2 v = cmk(row == col ? 1.0 : 0.0, 0.0);
      const int ck = key[col], rk = key[row];
      if (ck >= 0 && rk >= 0) {
        const int a = rk >> 24, b = ck >> 24;
        const double2 t = __ldg(lam + (long)c_pair[3 * a + b] * P + (rk & 0xffffff) - (ck & 0xffffff) + base);
        const double2 mv = cmul(mtab[row], t);
        v = cmk(v.x - mv.x, -mv.y);
      }
      A[((long)tile * T + c) * T + lane] = v;
    }
  }
  if (tid == 0) flags[0] = 0;
  __syncthreads();

  for (int kt = 0; kt < nt; ++kt) {
    const int c0 = kt * T;
    // ---- (1) panel factorisation of tile column kt.  One fused pass per
    //          column: a thread owns whole panel rows (coalesced across
    //          threads: rows are contiguous inside a column-major tile), scales
    //          the multiplier, applies the rank-1 update to the row's remaining
    //          panel columns with all loads in flight, and already tracks the
    //          next column's pivot candidate (zgetf2 order, |Re|+|Im| rule).
    double2* usm = reinterpret_cast<double2*>(gpiv + ((npad + 3) & ~3));  // [T] pivot row (16-B aligned)
    double best = -1.0;
    int bi = c0;
    for (int row = c0 + tid; row < npad; row += LU_THREADS) {
      const double2 v = A[lu_off(g, row, c0)];
      const double a = fabs(v.x) + fabs(v.y);
      if (a > best) { best = a; bi = row; }
    }
    for (int jj = 0; jj < T; ++jj) {
      const int j = c0 + jj;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_down_sync(0xffffffffu, best, o);
        const int oi = __shfl_down_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (lane == 0) { redv[warp] = best; redi[warp] = bi; }
      __syncthreads();
      if (tid == 0) {
        double bb = redv[0];
        int ii = redi[0];
        for (int w = 1; w < LU_WARPS; ++w)
          if (redv[w] > bb || (redv[w] == bb && redi[w] < ii)) { bb = redv[w]; ii = redi[w]; }
        if (!(bb > 0.0) && bb != 0.0) ii = j;  // all NaN
        pivs[jj] = ii;
        gpiv[j] = ii;
      }
      __syncthreads();
      const int p = pivs[jj];
      if (tid < T) {
        const long oa = lu_off(g, j, c0 + tid);
        double2 vj = A[oa];
        if (p != j) {
          const long ob = lu_off(g, p, c0 + tid);
          const double2 vp = A[ob];
          A[ob] = vj;
          A[oa] = vp;
          vj = vp;
        }
        usm[tid] = vj;
      }
      __syncthreads();
      const double2 d = usm[jj];
      const bool bad = (d.x == 0.0 && d.y == 0.0) || !isfinite(d.x) || !isfinite(d.y);
      if (bad && tid == 0 && flags[0] == 0 && j < n) flags[0] = j + 1;
      const double2 dinv = bad ? cmk(0.0, 0.0) : cinv(d);
      best = -1.0;
      bi = j + 1;
      for (int row = j + 1 + tid; row < npad; row += LU_THREADS) {
        const int it = row / T, r = row - it * T;
        double2* rowp = A + (long)(it * nt + kt) * T2 + r;  // element (row, c0 + c) at rowp[c * T]
        double2 l = rowp[jj * T];
        if (!bad) l = cmul(l, dinv);
        rowp[jj * T] = l;
        constexpr int U = 8;
        for (int c0u = jj + 1; c0u < T; c0u += U) {
          double2 v[U];
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (c0u + u < T) v[u] = rowp[(c0u + u) * T];
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (c0u + u < T) {
              if (!bad) cfms(v[u], l, usm[c0u + u]);
              rowp[(c0u + u) * T] = v[u];
            }
          if (c0u == jj + 1) {  // next column's pivot candidate
            const double a = fabs(v[0].x) + fabs(v[0].y);
            if (a > best) { best = a; bi = row; }
          }
        }
      }
    }
    // ---- (2) the panel's row interchanges on every other tile column (zlaswp)
    if (tid == 0) {
      int any = 0;
      for (int jj = 0; jj < T; ++jj) any |= (pivs[jj] != c0 + jj);
      flags[1] = any;
    }
    __syncthreads();
    if (flags[1]) {
      for (int col = tid; col < npad; col += LU_THREADS) {
        if (col / T == kt) continue;
        for (int jj = 0; jj < T; ++jj) {
          const int j = c0 + jj, p = pivs[jj];
          if (p == j) continue;
          const long oa = lu_off(g, j, col), ob = lu_off(g, p, col);
          const double2 t = A[oa];
          A[oa] = A[ob];
          A[ob] = t;
        }
      }
    }
    __syncthreads();
    // ---- (3) triangular inverses of the diagonal tile (lane = column)
    const double2* Dg = A + (long)(kt * nt + kt) * T2;
    if (warp == 0 && lane < T) {
      const int c = lane;
      for (int r = 0; r < T; ++r) {
        double2 x = cmk(r == c ? 1.0 : 0.0, 0.0);
        if (r > c) {
          for (int i = c; i < r; ++i) cfms(x, Dg[i * T + r], Ls[c * LD + i]);
        } else if (r < c) {
          x = cmk(0.0, 0.0);
        }
        Ls[c * LD + r] = x;
      }
    } else if (warp == 1 && lane < T) {
      const int c = lane;
      for (int r = T - 1; r >= 0; --r) {
        double2 x = cmk(0.0, 0.0);
        if (r <= c) {
          x = cmk(r == c ? 1.0 : 0.0, 0.0);
          for (int i = r + 1; i <= c; ++i) cfms(x, Dg[i * T + r], Us[c * LD + i]);
          x = cdiv(x, Dg[r * T + r]);
        }
        Us[c * LD + r] = x;
      }
    }
    __syncthreads();
    // ---- (4) U row tiles: A(kt, jt) = inv(L_kk) A(kt, jt)  (DMMA; T == 32
    //          whenever nt > 1), and the packed diagonal tile
    for (int jt = kt + 1 + warp; jt < nt; jt += LU_WARPS) {
      double2* C = A + (long)(kt * nt + jt) * T2;
      tile_mma_half<false>(Ls, C, C, 0, lane);
      tile_mma_half<false>(Ls, C, C, 1, lane);
    }
    {
      double2* Dw = A + (long)(kt * nt + kt) * T2;
      for (int i = tid; i < T2; i += LU_THREADS) {
        const int c = i / T, r = i - c * T;
        Dw[i] = (r > c) ? Ls[c * LD + r] : Us[c * LD + r];
      }
    }
    __syncthreads();
    // ---- (5) trailing update A(it, jt) -= A(it, kt) A(kt, jt) on DMMA: a warp
    //          owns tile rows it; L tile A(it,kt) staged once per row in shared
    //          memory, U tiles of row kt read as B fragments (L1-shared by the
    //          warps sweeping the same jt), each trailing tile read+written once.
    {
      // L tile fragments straight from global/L2 (no staging: small shared
      // memory footprint -> more resident CTAs to hide the fragment latency)
      const int nrem = nt - kt - 1;
      for (int task = warp; task < nrem * nrem * 2; task += LU_WARPS) {
        const int h = task & 1, t2 = task >> 1;
        const int it = kt + 1 + t2 / nrem, jt = kt + 1 + t2 % nrem;
        tile_mma_half<true, 32>(A + (long)(it * nt + kt) * T2, A + (long)(kt * nt + jt) * T2,
                                A + (long)(it * nt + jt) * T2, h, lane);
      }
    }
    __syncthreads();
  }
  // permutation composed from the interchange sequence (zgetrs applies the
  // swaps to b in order): b_perm[i] = b[perm[i]]
  if (tid == 0) {
    info[slot] = flags[0];
  }
  int* pv = reinterpret_cast<int*>(Bst);  // reuse staging smem
  for (int i = tid; i < npad; i += LU_THREADS) pv[i] = i;
  __syncthreads();
  if (tid == 0) {
    for (int j = 0; j < npad; ++j) {
      const int p = gpiv[j];
      if (p != j) { const int t = pv[j]; pv[j] = pv[p]; pv[p] = t; }
    }
  }
  __syncthreads();
  for (int i = tid; i < n; i += LU_THREADS) {
    int v = pv[i];
    perm[(long)slot * n + i] = v < n ? v : i;
    piv[(long)slot * n + i] = gpiv[i];
  }
}

static size_t lu_smem(const LuGeom& g) {
  return (size_t)3 * g.T * (g.T + 1) * sizeof(double2) + 32 * sizeof(int) +
         LU_WARPS * (sizeof(double) + sizeof(int)) + 4 * sizeof(int) + (size_t)(g.npad + 4) * sizeof(int) + 64 +
         (size_t)g.T * sizeof(double2);
}

// ------------------------------------------------- step-batched LU (default)
// The factorisation advances all blocks one tile column at a time, with one
// kernel per phase so each phase gets its own launch shape and register
// budget, and the DMMA trailing update sees every (block, tile) task of the
// step at once (no per-block tail where most warps idle):
//   unfold (once) | per step kt: panel -> row interchanges -> U row -> trailing
//   update | permutation composition (once).
constexpr int LUB_WARPS = 8;

__global__ void __launch_bounds__(256) lub_unfold_kernel(Unfold u, LuGeom g, double2* F) {
  extern __shared__ __align__(16) unsigned char smu[];
  const int T = g.T, nt = g.nt, npad = g.npad, n = g.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int slot = blockIdx.x;
  const int k = u.kset ? u.kset[slot] : slot;
  double2* A = F + (long)slot * g.blk;
  const double2* lam = u.lamT + (long)k * u.Ltot;
  const int q = u.nzL * u.nyL;
  const int nyy = 2 * u.nyL - 1, nzz = 2 * u.nzL - 1;
  const int P = nzz * nyy, base = (u.nzL - 1) * nyy + (u.nyL - 1);
  int* key = reinterpret_cast<int*>(smu);
  double2* mtab = reinterpret_cast<double2*>(key + ((npad + 3) & ~3));
  for (int idx = tid; idx < npad; idx += 256) {
    if (idx < n) {
      const int a = idx / q, rr = idx - a * q;
      const int iz = rr / u.nyL, iy = rr - iz * u.nyL;
      key[idx] = (a << 24) | (iz * nyy + iy);
      mtab[idx] = __ldg(u.m + rr);
    } else {
      key[idx] = -1;
    }
  }
  __syncthreads();
  const int ncolw = nt * nt * T;
  for (int w = warp; w < ncolw; w += 8) {
    const int tile = w / T, c = w - tile * T;
    const int it = tile / nt, jt = tile - it * nt;
    const int col = jt * T + c;
    if (lane >= T) continue;
    const int row = it * T + lane;
    double2 v = cmk(row == col ? 1.0 : 0.0, 0.0);
    const int ck = key[col], rk = key[row];
    if (ck >= 0 && rk >= 0) {
      const int a = rk >> 24, b = ck >> 24;
      const double2 t = __ldg(lam + (long)c_pair[3 * a + b] * P + (rk & 0xffffff) - (ck & 0xffffff) + base);
      const double2 mv = cmul(mtab[row], t);
      v = cmk(v.x - mv.x, -mv.y);
    }
    A[((long)tile * T + c) * T + lane] = v;
  }
}

// Symmetry-sector unfold (sectors.py): slot = kslot * nsec + s holds
//   B_s[j, j'] = rsc[j] * sum_t cw[j', t] * D_k[rrow[j], ccol[j', t]]
// with D_k = I - diag(m) N_k evaluated on the fly (reference accel.py:71-91);
// rows / cols >= the sector's size (rrow / ccol = -1) are identity.
struct SecUnfold {
  const double2* __restrict__ lamT;
  const double2* __restrict__ m;
  const int* __restrict__ kset;
  long Ltot;
  int nzL, nyL, nsec, dmax;
  const int* __restrict__ rrow;    // [nsec][dmax]
  const double* __restrict__ rsc;  // [nsec][dmax]
  const int* __restrict__ ccol;    // [nsec][dmax][4]
  const double* __restrict__ cw;   // [nsec][dmax][4]
};

__global__ void __launch_bounds__(256) sec_unfold_kernel(SecUnfold u, LuGeom g, double2* F) {
  extern __shared__ __align__(16) unsigned char smu[];
  const int T = g.T, nt = g.nt, npad = g.npad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int slot = blockIdx.x;
  const int kslot = slot / u.nsec, sec = slot - kslot * u.nsec;
  const int k = u.kset ? u.kset[kslot] : kslot;
  double2* A = F + (long)slot * g.blk;
  const double2* lam = u.lamT + (long)k * u.Ltot;
  const int q = u.nzL * u.nyL;
  const int nyy = 2 * u.nyL - 1, nzz = 2 * u.nzL - 1;
  const int P = nzz * nyy, base = (u.nzL - 1) * nyy + (u.nyL - 1);
  double2* rm = reinterpret_cast<double2*>(smu);          // [npad] m at the row's site * rsc
  double* cwt = reinterpret_cast<double*>(rm + npad);     // [npad][4]
  int* rkey = reinterpret_cast<int*>(cwt + 4 * npad);     // [npad] (a << 24) | offset, -1 pad
  int* rid = rkey + npad;                                 // [npad] original row
  int* ckey = rid + npad;                                 // [npad][4]
  int* cid = ckey + 4 * npad;                             // [npad][4]
  const long sb = (long)sec * u.dmax;
  auto key_of = [&](int o) {
    const int a = o / q, rr = o - a * q;
    const int iz = rr / u.nyL, iy = rr - iz * u.nyL;
    return (a << 24) | (iz * nyy + iy);
  };
  for (int j = tid; j < npad; j += 256) {
    const int r = j < u.dmax ? u.rrow[sb + j] : -1;
    rid[j] = r;
    if (r >= 0) {
      rkey[j] = key_of(r);
      const double2 mv = __ldg(u.m + (r % q));
      const double sc = u.rsc[sb + j];
      rm[j] = cmk(mv.x * sc, mv.y * sc);
    } else {
      rkey[j] = -1;
    }
    for (int t = 0; t < 4; ++t) {
      const int c = j < u.dmax ? u.ccol[(sb + j) * 4 + t] : -1;
      cid[4 * j + t] = c;
      ckey[4 * j + t] = c >= 0 ? key_of(c) : -1;
      cwt[4 * j + t] = c >= 0 ? u.cw[(sb + j) * 4 + t] : 0.0;
    }
  }
  __syncthreads();
  const int ncolw = nt * nt * T;
  for (int w = warp; w < ncolw; w += 8) {
    const int tile = w / T, c = w - tile * T;
    const int it = tile / nt, jt = tile - it * nt;
    const int col = jt * T + c;
    if (lane >= T) continue;
    const int row = it * T + lane;
    double2 v = cmk(row == col ? 1.0 : 0.0, 0.0);
    const int rk = rkey[row];
    if (rk >= 0 && ckey[4 * col] >= 0) {
      const int a = rk >> 24, r0 = rid[row];
      const double sc = u.rsc[sb + row];
      double2 acc = cmk(0.0, 0.0);   // sum_t w_t * N[row, c_t]
      double dsum = 0.0;             // sum_t w_t * [row == c_t]
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int ck = ckey[4 * col + t];
        if (ck < 0) continue;
        const double wt = cwt[4 * col + t];
        const int b = ck >> 24;
        const double2 tv = __ldg(lam + (long)c_pair[3 * a + b] * P + (rk & 0xffffff) - (ck & 0xffffff) + base);
        acc.x = fma(wt, tv.x, acc.x);
        acc.y = fma(wt, tv.y, acc.y);
        if (cid[4 * col + t] == r0) dsum += wt;
      }
      const double2 mn = cmul(rm[row], acc);
      v = cmk(sc * dsum - mn.x, -mn.y);
    }
    A[((long)tile * T + c) * T + lane] = v;
  }
}

static size_t sec_unfold_smem(const LuGeom& g) {
  return (size_t)g.npad * (sizeof(double2) + 4 * sizeof(double) + 2 * sizeof(int) + 8 * sizeof(int));
}

// panel factorisation of tile column kt of every block (one CTA per block),
// then the diagonal tile's triangular inverses, packed in place.
__global__ void __launch_bounds__(LU_THREADS) lub_panel_kernel(LuGeom g, double2* F, int kt, int* piv,
                                                               int* info, int nopiv) {
  __shared__ double redv[LU_WARPS];
  __shared__ int redi[LU_WARPS];
  __shared__ int pivs[32];
  __shared__ double2 usm[32];
  __shared__ double2 Ls[32 * 33], Us[32 * 33];
  const int T = g.T, T2 = T * T, nt = g.nt, npad = g.npad, n = g.n;
  const int LD = T + 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int slot = blockIdx.x;
  double2* A = F + (long)slot * g.blk;
  const int c0 = kt * T;
  double best = -1.0;
  int bi = c0;
  for (int row = c0 + tid; row < npad; row += LU_THREADS) {
    const double2 v = A[lu_off(g, row, c0)];
    const double a = fabs(v.x) + fabs(v.y);
    if (a > best) { best = a; bi = row; }
  }
  for (int jj = 0; jj < T; ++jj) {
    const int j = c0 + jj;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_down_sync(0xffffffffu, best, o);
      const int oi = __shfl_down_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    if (lane == 0) { redv[warp] = best; redi[warp] = bi; }
    __syncthreads();
    if (tid == 0) {
      double bb = redv[0];
      int ii = redi[0];
      for (int w = 1; w < LU_WARPS; ++w)
        if (redv[w] > bb || (redv[w] == bb && redi[w] < ii)) { bb = redv[w]; ii = redi[w]; }
      if (!(bb > 0.0) && bb != 0.0) ii = j;  // all NaN
      if (j >= n || nopiv) ii = j;           // identity pad never pivots; nopiv: elimination in order
      pivs[jj] = ii;
      if (j < n) piv[(long)slot * n + j] = ii;
    }
    __syncthreads();
    const int p = pivs[jj];
    if (tid < T) {
      const long oa = lu_off(g, j, c0 + tid);
      double2 vj = A[oa];
      if (p != j) {
        const long ob = lu_off(g, p, c0 + tid);
        const double2 vp = A[ob];
        A[ob] = vj;
        A[oa] = vp;
        vj = vp;
      }
      usm[tid] = vj;
    }
    __syncthreads();
    const double2 d = usm[jj];
    const bool bad = (d.x == 0.0 && d.y == 0.0) || !isfinite(d.x) || !isfinite(d.y);
    if (bad && tid == 0 && j < n && info[slot] == 0) info[slot] = j + 1;
    const double2 dinv = bad ? cmk(0.0, 0.0) : cinv(d);
    best = -1.0;
    bi = j + 1;
    for (int row = j + 1 + tid; row < npad; row += LU_THREADS) {
      const int it = row / T, r = row - it * T;
      double2* rowp = A + (long)(it * nt + kt) * T2 + r;
      double2 l = rowp[jj * T];
      if (!bad) l = cmul(l, dinv);
      rowp[jj * T] = l;
      constexpr int U = 8;
      for (int c0u = jj + 1; c0u < T; c0u += U) {
        double2 v[U];
#pragma unroll
        for (int u2 = 0; u2 < U; ++u2)
          if (c0u + u2 < T) v[u2] = rowp[(c0u + u2) * T];
#pragma unroll
        for (int u2 = 0; u2 < U; ++u2)
          if (c0u + u2 < T) {
            if (!bad) cfms(v[u2], l, usm[c0u + u2]);
            rowp[(c0u + u2) * T] = v[u2];
          }
        if (c0u == jj + 1) {
          const double a = fabs(v[0].x) + fabs(v[0].y);
          if (a > best) { best = a; bi = row; }
        }
      }
    }
  }
  __syncthreads();
  const double2* Dg = A + (long)(kt * nt + kt) * T2;
  if (warp == 0 && lane < T) {
    const int c = lane;
    for (int r = 0; r < T; ++r) {
      double2 x = cmk(r == c ? 1.0 : 0.0, 0.0);
      if (r > c) {
        for (int i = c; i < r; ++i) cfms(x, Dg[i * T + r], Ls[c * LD + i]);
      } else if (r < c) {
        x = cmk(0.0, 0.0);
      }
      Ls[c * LD + r] = x;
    }
  } else if (warp == 1 && lane < T) {
    const int c = lane;
    for (int r = T - 1; r >= 0; --r) {
      double2 x = cmk(0.0, 0.0);
      if (r <= c) {
        x = cmk(r == c ? 1.0 : 0.0, 0.0);
        for (int i = r + 1; i <= c; ++i) cfms(x, Dg[i * T + r], Us[c * LD + i]);
        x = cdiv(x, Dg[r * T + r]);
      }
      Us[c * LD + r] = x;
    }
  }
  __syncthreads();
  double2* Dw = A + (long)(kt * nt + kt) * T2;
  for (int i = tid; i < T2; i += LU_THREADS) {
    const int c = i / T, r = i - c * T;
    Dw[i] = (r > c) ? Ls[c * LD + r] : Us[c * LD + r];
  }
}

// panel step WITHOUT row interchanges (symmetric factors, lu_sym.cuh): the
// diagonal tile is factorised in shared memory (one barrier per column instead
// of three plus a global-memory rank-1 sweep of the whole panel), and the tiles
// below it become L(it, kt) = A(it, kt) inv(U_kk) -- tensor-core tile products
// with no dependency between them.  T = 32 only (multi-tile blocks).
__global__ void __launch_bounds__(LU_THREADS) lub_panel_nopiv_kernel(LuGeom g, double2* F, int kt, int* piv,
                                                                     int* info) {
  extern __shared__ double2 pnsm[];
  double2* D = pnsm;             // diagonal tile (column-major, ld 33); later a staged A tile
  double2* Ls = D + 32 * 33;     // inv(L_kk); later a second staged A tile
  double2* Ub = Ls + 32 * 33;    // inv(U_kk), ld 32: also the B operand of the tile products
  constexpr int T = 32, T2 = 1024, LD = 33;
  const int nt = g.nt, n = g.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int slot = blockIdx.x;
  double2* A = F + (long)slot * g.blk;
  double2* Dg = A + (long)(kt * nt + kt) * T2;
  const int c0 = kt * T;
  for (int i = tid; i < T2; i += LU_THREADS) D[(i >> 5) * LD + (i & 31)] = Dg[i];
  if (tid < T && c0 + tid < n) piv[(long)slot * n + c0 + tid] = c0 + tid;
  __syncthreads();
  for (int jj = 0; jj < T; ++jj) {
    const double2 d = D[jj * LD + jj];
    const bool bad = (d.x == 0.0 && d.y == 0.0) || !isfinite(d.x) || !isfinite(d.y);
    if (bad && tid == 0 && c0 + jj < n && info[slot] == 0) info[slot] = c0 + jj + 1;
    const double2 dinv = bad ? cmk(0.0, 0.0) : cinv(d);
    const int r = lane;
    double2 l = cmk(0.0, 0.0);
    if (r > jj) {
      l = D[jj * LD + r];
      if (!bad) {
        l = cmul(l, dinv);
        for (int c = jj + 1 + warp; c < T; c += LU_WARPS) cfms(D[c * LD + r], l, D[c * LD + jj]);
      }
    }
    __syncthreads();
    if (warp == 0 && r > jj) D[jj * LD + r] = l;
  }
  __syncthreads();
  if (warp == 0) {
    const int c = lane;
    for (int r = 0; r < T; ++r) {
      double2 x = cmk(r == c ? 1.0 : 0.0, 0.0);
      if (r > c) {
        for (int i = c; i < r; ++i) cfms(x, D[i * LD + r], Ls[c * LD + i]);
      } else if (r < c) {
        x = cmk(0.0, 0.0);
      }
      Ls[c * LD + r] = x;
    }
  } else if (warp == 1) {
    const int c = lane;
    for (int r = T - 1; r >= 0; --r) {
      double2 x = cmk(0.0, 0.0);
      if (r <= c) {
        x = cmk(r == c ? 1.0 : 0.0, 0.0);
        for (int i = r + 1; i <= c; ++i) cfms(x, D[i * LD + r], Ub[c * 32 + i]);
        x = cdiv(x, D[r * LD + r]);
      }
      Ub[c * 32 + r] = x;
    }
  }
  __syncthreads();
  for (int i = tid; i < T2; i += LU_THREADS) {
    const int c = i >> 5, r = i & 31;
    Dg[i] = (r > c) ? Ls[c * LD + r] : Ub[i];
  }
  // L(it, kt) = A(it, kt) inv(U_kk): two tiles at a time (a warp pair per tile, 16 columns each)
  for (int it0 = kt + 1; it0 < nt; it0 += 2) {
    __syncthreads();  // D / Ls free (inverses written out; previous products done)
    for (int q2 = 0; q2 < 2; ++q2) {
      if (it0 + q2 >= nt) break;
      const double2* src = A + (long)((it0 + q2) * nt + kt) * T2;
      double2* dst = q2 ? Ls : D;
      for (int i = tid; i < T2; i += LU_THREADS) dst[(i >> 5) * LD + (i & 31)] = src[i];
    }
    __syncthreads();
    const int it = it0 + (warp >> 1);
    if (it < nt) tile_mma_half<false>((warp >> 1) ? Ls : D, Ub, A + (long)(it * nt + kt) * T2, warp & 1, lane);
  }
}

// the step's row interchanges on every column outside the panel (zlaswp)
__global__ void __launch_bounds__(256) lub_swap_kernel(LuGeom g, double2* F, int kt, const int* piv) {
  __shared__ int pv[32];
  __shared__ int any;
  const int T = g.T, npad = g.npad, n = g.n;
  const int slot = blockIdx.y;
  const int c0 = kt * T;
  if (threadIdx.x < 32) {
    const int j = c0 + threadIdx.x;
    pv[threadIdx.x] = (threadIdx.x < T && j < n) ? piv[(long)slot * n + j] : j;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int a = 0;
    for (int jj = 0; jj < T; ++jj) a |= (pv[jj] != c0 + jj);
    any = a;
  }
  __syncthreads();
  if (!any) return;
  double2* A = F + (long)slot * g.blk;
  for (int col = blockIdx.x * blockDim.x + threadIdx.x; col < npad; col += gridDim.x * blockDim.x) {
    if (col / T == kt) continue;
    for (int jj = 0; jj < T; ++jj) {
      const int j = c0 + jj, p = pv[jj];
      if (p == j) continue;
      const long oa = lu_off(g, j, col), ob = lu_off(g, p, col);
      const double2 t = A[oa];
      A[oa] = A[ob];
      A[ob] = t;
    }
  }
}

// U row: A(kt, jt) = inv(L_kk) A(kt, jt) for jt > kt on DMMA (one CTA per block)
__global__ void __launch_bounds__(LUB_WARPS * 32) lub_urow_kernel(LuGeom g, double2* F, int kt) {
  __shared__ double2 Ls[32 * 33];
  const int T2 = 32 * 32, nt = g.nt;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double2* A = F + (long)blockIdx.x * g.blk;
  const double2* Dg = A + (long)(kt * nt + kt) * T2;
  for (int i = tid; i < T2; i += LUB_WARPS * 32) {
    const int c = i >> 5, r = i & 31;
    Ls[c * 33 + r] = r > c ? Dg[i] : cmk(r == c ? 1.0 : 0.0, 0.0);
  }
  __syncthreads();
  const int nrem = nt - kt - 1;
  for (int task = warp; task < 2 * nrem; task += LUB_WARPS) {
    double2* C = A + (long)(kt * nt + kt + 1 + (task >> 1)) * T2;
    tile_mma_half<false>(Ls, C, C, task & 1, lane);
  }
}

// trailing update of every block: task = (block, it, jt, half), one warp each
__global__ void __launch_bounds__(LUB_WARPS * 32, 2) lub_trail_kernel(LuGeom g, double2* F, int kt, long ntask) {
  const int T2 = 32 * 32, nt = g.nt;
  const int lane = threadIdx.x & 31;
  const long task = (long)blockIdx.x * LUB_WARPS + (threadIdx.x >> 5);
  if (task >= ntask) return;
  const int nrem = nt - kt - 1;
  const int h = (int)(task & 1);
  long t2 = task >> 1;
  const int tj = (int)(t2 % nrem);
  t2 /= nrem;
  const int ti = (int)(t2 % nrem);
  const long slot = t2 / nrem;
  double2* A = F + slot * g.blk;
  const int it = kt + 1 + ti, jt = kt + 1 + tj;
  tile_mma_half<true, 32>(A + (long)(it * nt + kt) * T2, A + (long)(kt * nt + jt) * T2,
                          A + (long)(it * nt + jt) * T2, h, lane);
}

// column-major packed diagonal tile (inv(L) below, inv(U) on/above) -> split layout
__global__ void __launch_bounds__(256) diag_split_kernel(LuGeom g, double2* F) {
  extern __shared__ double2 dsm[];
  const int T = g.T, T2 = T * T;
  const long slot = blockIdx.x / g.nt;
  const int i = blockIdx.x - (int)slot * g.nt;
  double2* D = F + slot * g.blk + (long)(i * g.nt + i) * T2;
  for (int e = threadIdx.x; e < T2; e += blockDim.x) dsm[e] = D[e];
  __syncthreads();
  const int nl = dl_n(T);
  for (int e = threadIdx.x; e < T2; e += blockDim.x) {
    const int c = e / T, r = e - c * T;
    if (r > c) D[dl_off(T, r, c)] = dsm[e];
    else D[nl + du_off(T, r, c)] = dsm[e];
  }
}

static int diag_split(const LuGeom& g, int nslots, double2* F, cudaStream_t s) {
  if (nslots <= 0 || g.nt == 1) return VX_OK;  // single-tile blocks stay packed (staged whole)
  diag_split_kernel<<<(unsigned)((long)nslots * g.nt), 256, (size_t)g.T * g.T * sizeof(double2), s>>>(g, F);
  VX_CHECK_LAUNCH("diag_split_kernel");
  return VX_OK;
}

// b_perm[i] = b[perm[i]] from zgetrf's interchange sequence (one thread per block)
__global__ void lub_perm_kernel(int nslots, int n, const int* piv, int* perm, int* scratch) {
  const int slot = blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= nslots) return;
  int* pv = perm + (long)slot * n;
  for (int i = 0; i < n; ++i) pv[i] = i;
  const int* pp = piv + (long)slot * n;
  for (int j = 0; j < n; ++j) {
    const int p = pp[j];
    if (p != j && p < n) { const int t = pv[j]; pv[j] = pv[p]; pv[p] = t; }
  }
  (void)scratch;
}

static int g_lu_monolithic = 0;  // vx_lu_variant(1): single-kernel LU (A/B timing)

static int lu_build_batched(const Unfold& u, const LuGeom& g, int nslots, double2* F, int* perm, int* piv,
                            int* info, cudaStream_t s, const SecUnfold* su = nullptr, int nopiv = 0) {
  VX_CUDA(cudaMemsetAsync(info, 0, sizeof(int) * nslots, s));
  if (su) {
    const size_t us = sec_unfold_smem(g);
    if (us > 48 * 1024)
      VX_CUDA(cudaFuncSetAttribute(sec_unfold_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)us));
    VX_REQUIRE((int)us <= device_smem_optin(), "sector size %d too large for the unfold tables", g.n);
    sec_unfold_kernel<<<nslots, 256, us, s>>>(*su, g, F);
    VX_CHECK_LAUNCH("sec_unfold_kernel");
  } else {
    const size_t us = (size_t)((g.npad + 3) & ~3) * sizeof(int) + (size_t)g.npad * sizeof(double2);
    if (us > 48 * 1024)
      VX_CUDA(cudaFuncSetAttribute(lub_unfold_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)us));
    VX_REQUIRE((int)us <= device_smem_optin(), "block size %d too large for the unfold tables", g.n);
    lub_unfold_kernel<<<nslots, 256, us, s>>>(u, g, F);
    VX_CHECK_LAUNCH("lub_unfold_kernel");
  }
  for (int kt = 0; kt < g.nt; ++kt) {
    const bool fast = nopiv && g.T == 32 && env_int("VX_PANEL_FAST", 1);
    constexpr int pn_smem = (2 * 32 * 33 + 32 * 32) * (int)sizeof(double2);
    if (fast && kt == 0)
      VX_CUDA(cudaFuncSetAttribute(lub_panel_nopiv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, pn_smem));
    if (fast) lub_panel_nopiv_kernel<<<nslots, LU_THREADS, pn_smem, s>>>(g, F, kt, piv, info);
    else lub_panel_kernel<<<nslots, LU_THREADS, 0, s>>>(g, F, kt, piv, info, nopiv);
    VX_CHECK_LAUNCH("lub_panel_kernel");
    if (g.nt > 1 && !fast) {
      dim3 sg(div_up(g.npad, 256), nslots);
      lub_swap_kernel<<<sg, 256, 0, s>>>(g, F, kt, piv);
      VX_CHECK_LAUNCH("lub_swap_kernel");
    }
    const int nrem = g.nt - kt - 1;
    if (nrem > 0) {
      lub_urow_kernel<<<nslots, LUB_WARPS * 32, 0, s>>>(g, F, kt);
      VX_CHECK_LAUNCH("lub_urow_kernel");
      const long ntask = (long)nslots * nrem * nrem * 2;
      lub_trail_kernel<<<(unsigned)((ntask + LUB_WARPS - 1) / LUB_WARPS), LUB_WARPS * 32, 0, s>>>(g, F, kt, ntask);
      VX_CHECK_LAUNCH("lub_trail_kernel");
    }
  }
  lub_perm_kernel<<<div_up(nslots, 128), 128, 0, s>>>(nslots, g.n, piv, perm, nullptr);
  VX_CHECK_LAUNCH("lub_perm_kernel");
  return diag_split(g, nslots, F, s);
}

static int lu_build(const Unfold& u, int n, int nslots, double2* F, int* perm, int* piv, int* info,
                    cudaStream_t s) {
  if (nslots <= 0) return VX_OK;
  Span span("lu_build", s);
  LuGeom g = lu_geom(n);
  if (!g_lu_monolithic) return lu_build_batched(u, g, nslots, F, perm, piv, info, s);
  size_t smem = lu_smem(g);
  // the permutation scratch reuses the staging tiles: make sure they fit npad ints
  VX_REQUIRE((size_t)g.npad * sizeof(int) <= (size_t)g.T * (g.T + 1) * sizeof(double2) &&
                 (size_t)(g.npad + 4) * (sizeof(int) + sizeof(double2)) <=
                     (size_t)3 * g.T * (g.T + 1) * sizeof(double2),
             "block size %d too large for the LU kernel's scratch tables", n);
  if (smem > 48 * 1024)
    VX_CUDA(cudaFuncSetAttribute(lu_build_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
  VX_REQUIRE((int)smem <= device_smem_optin(), "block size %d too large for the LU kernel", n);
  lu_build_kernel<<<nslots, LU_THREADS, smem, s>>>(u, g, F, perm, piv, info);
  VX_CHECK_LAUNCH("lu_build_kernel");
  return diag_split(g, nslots, F, s);
}

// ---------------------------------------------------------------- LU solve
// Mirror sharing: for an x-parity-symmetric kernel D_{n-k} = S D_k S with S =
// -1 on the x-component rows (rows [0, q), q = n/3), and for the 2-level
// y-mirror S = -1 on the y-component rows [q, 2q); so the mirror block's
// solve is y = S D_k^-1 S b with D_k's stored factors.  A klist entry carries
// the frequency in its low 29 bits and the flips in bits 30 (x) / 29 (y).
[[maybe_unused]] constexpr int KFLIP_X = 1 << 30;  // documents the encoding (x flip = bit 30)
constexpr int KFLIP_Y = 1 << 29, KIDX = KFLIP_Y - 1;
constexpr long ROFF = (1L << 56) - 1;  // rbase: offset in the low 56 bits, flips (kraw >> 29) above
__device__ __forceinline__ bool flip_row(int f2, int row, int q) {
  return ((f2 & 2) && row < q) || ((f2 & 1) && row >= q && row < 2 * q);
}
__device__ __forceinline__ long rhs_base(int kraw, int rho, int nrhs, long s_k) {
  return ((long)(kraw & KIDX) * s_k + (rho % nrhs)) | ((long)(kraw >> 29) << 56);
}
__device__ __forceinline__ double2 cflip(double2 v, bool f) { return f ? cmk(-v.x, -v.y) : v; }

// One CTA per work item: slot + up to R right-hand sides (frequency k, column j)
// gathered from Y[row*s_row + k*s_k + j] through the row permutation.
template <int R, int NW>
__global__ void __launch_bounds__(NW * 32) lu_solve_kernel(LuGeom g, const double2* __restrict__ F,
                                                           const int* __restrict__ perm,
                                                           const int* __restrict__ items, int item0,
                                                           const int* __restrict__ klist, int nrhs,
                                                           double2* Y, long s_row, long s_k) {
  extern __shared__ double2 sm[];
  const int T = g.T, T2 = T * T, nt = g.nt, npad = g.npad, n = g.n, q = n / 3;
  double2* y = sm;                    // [npad][R]
  double2* red = y + (long)npad * R;  // [NW][T][R]
  double2* Ds = red + NW * T * R;     // [T*T]
  double2* zb = Ds + T2;              // [T][R]
  __shared__ long rbase[R];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NT = NW * 32;
  int slot, beg, cnt;
  if (items) {
    const int it = item0 + blockIdx.x;
    slot = items[3 * it];
    beg = items[3 * it + 1];
    cnt = items[3 * it + 2];
  } else {
    slot = item0 + blockIdx.x;
    beg = slot;
    cnt = 1;
  }
  const double2* Fb = F + (long)slot * g.blk;
  const int* pm = perm + (long)slot * n;
  const int total = cnt * nrhs;
  for (int rho0 = 0; rho0 < total; rho0 += R) {
    const int nr = min(R, total - rho0);
    if (tid < R) {
      long b = 0;
      if (tid < nr) {
        const int rho = rho0 + tid;
        const int kraw = klist ? klist[beg + rho / nrhs] : beg + rho / nrhs;
        b = rhs_base(kraw, rho, nrhs, s_k);
      }
      rbase[tid] = b;
    }
    __syncthreads();
    for (int idx = tid; idx < npad * R; idx += NT) {
      const int row = idx / R, rr = idx - row * R;
      double2 v = cmk(0.0, 0.0);
      if (row < n && rr < nr) {
        const long rb = rbase[rr];
        const int pr = pm[row];
        v = cflip(Y[(long)pr * s_row + (rb & ROFF)], flip_row((int)(rb >> 56), pr, q));
      }
      y[idx] = v;
    }
    __syncthreads();
    // forward: L (unit lower, diagonal tiles hold inv(L_ii) below the diagonal)
    for (int i = 0; i < nt; ++i) {
      double2 acc[R];
#pragma unroll
      for (int rr = 0; rr < R; ++rr) acc[rr] = cmk(0.0, 0.0);
      if (lane < T) {
        for (int j = warp; j < i; j += NW) {
          const double2* tile = Fb + (long)(i * nt + j) * T2 + lane;
          const double2* yj = y + (long)j * T * R;
#pragma unroll 8
          for (int c = 0; c < T; ++c) {
            const double2 a = ld_stream(tile + c * T);
#pragma unroll
            for (int rr = 0; rr < R; ++rr) cfma(acc[rr], a, yj[c * R + rr]);
          }
        }
#pragma unroll
        for (int rr = 0; rr < R; ++rr) red[(warp * T + lane) * R + rr] = acc[rr];
      }
      const double2* dt = Fb + (long)(i * nt + i) * T2;
      const int dlen = nt > 1 ? dl_n(T) : T2;
      for (int idx = tid; idx < dlen; idx += NT) Ds[idx] = ld_stream(dt + idx);
      __syncthreads();
      for (int idx = tid; idx < T * R; idx += NT) {
        const int r = idx / R, rr = idx - r * R;
        double2 z = y[(long)(i * T + r) * R + rr];
        for (int w = 0; w < NW; ++w) z = csub(z, red[(w * T + r) * R + rr]);
        zb[idx] = z;
      }
      __syncthreads();
      for (int idx = tid; idx < T * R; idx += NT) {
        const int r = idx / R, rr = idx - r * R;
        double2 o = zb[idx];
        for (int c = 0; c < r; ++c) cfma(o, Ds[nt > 1 ? dl_off(T, r, c) : c * T + r], zb[c * R + rr]);
        y[(long)(i * T + r) * R + rr] = o;
      }
      __syncthreads();
    }
    // backward: U (diagonal tiles hold inv(U_ii) on and above the diagonal)
    for (int i = nt - 1; i >= 0; --i) {
      double2 acc[R];
#pragma unroll
      for (int rr = 0; rr < R; ++rr) acc[rr] = cmk(0.0, 0.0);
      if (lane < T) {
        for (int j = i + 1 + warp; j < nt; j += NW) {
          const double2* tile = Fb + (long)(i * nt + j) * T2 + lane;
          const double2* yj = y + (long)j * T * R;
#pragma unroll 8
          for (int c = 0; c < T; ++c) {
            const double2 a = ld_stream(tile + c * T);
#pragma unroll
            for (int rr = 0; rr < R; ++rr) cfma(acc[rr], a, yj[c * R + rr]);
          }
        }
#pragma unroll
        for (int rr = 0; rr < R; ++rr) red[(warp * T + lane) * R + rr] = acc[rr];
      }
      const int doff = nt > 1 ? dl_n(T) : 0;
      const double2* dt = Fb + (long)(i * nt + i) * T2 + doff;
      for (int idx = tid; idx < T2 - doff; idx += NT) Ds[idx] = ld_stream(dt + idx);
      __syncthreads();
      for (int idx = tid; idx < T * R; idx += NT) {
        const int r = idx / R, rr = idx - r * R;
        double2 z = y[(long)(i * T + r) * R + rr];
        for (int w = 0; w < NW; ++w) z = csub(z, red[(w * T + r) * R + rr]);
        zb[idx] = z;
      }
      __syncthreads();
      for (int idx = tid; idx < T * R; idx += NT) {
        const int r = idx / R, rr = idx - r * R;
        double2 o = cmk(0.0, 0.0);
        for (int c = r; c < T; ++c) cfma(o, Ds[nt > 1 ? du_off(T, r, c) : c * T + r], zb[c * R + rr]);
        y[(long)(i * T + r) * R + rr] = o;
      }
      __syncthreads();
    }
    for (int idx = tid; idx < n * R; idx += NT) {
      const int row = idx / R, rr = idx - row * R;
      if (rr < nr) {
        const long rb = rbase[rr];
        Y[(long)row * s_row + (rb & ROFF)] = cflip(y[idx], flip_row((int)(rb >> 56), row, q));
      }
    }
    __syncthreads();
  }
}

template <int R, int NW>
static int launch_solve(const LuGeom& g, const double2* F, const int* perm, const int* items,
                        int item0, int nblocks, const int* klist, int nrhs, double2* Y, long s_row,
                        long s_k, cudaStream_t s) {
  if (nblocks <= 0) return VX_OK;
  const size_t smem = ((size_t)g.npad * R + (size_t)NW * g.T * R + (size_t)g.T * g.T +
                       (size_t)g.T * R) * sizeof(double2);
  auto kern = lu_solve_kernel<R, NW>;
  VX_REQUIRE((int)smem + 1024 <= device_smem_optin(), "block size %d too large for the solve kernel", g.n);
  if (smem > 48 * 1024)
    VX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<nblocks, NW * 32, smem, s>>>(g, F, perm, items, item0, klist, nrhs, Y, s_row, s_k);
  VX_CHECK_LAUNCH("lu_solve_kernel");
  return VX_OK;
}

constexpr int SOLVE_WARPS = 8;
constexpr int MULTI_R = 8;
static int g_solve_classic = 0;  // vx_solve_variant(1): non-pipelined kernel (A/B measurement)

// --------------------------------------------------- pipelined (TMA bulk) solve
// One producer warp streams the block's factor tiles, in exactly the order the
// substitution consumes them, into a ring of S shared-memory slots with
// cp.async.bulk (TMA bulk copies completing on mbarriers); NWC consumer warps
// do the tile GEMVs.  Loads never wait on the substitution's dependencies, so
// up to S tiles per CTA are always in flight.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void consumers_sync(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

constexpr int PIPE_CONSUMERS = 8;

template <int R>
__global__ void __launch_bounds__((PIPE_CONSUMERS + 1) * 32)
    lu_solve_pipe_kernel(LuGeom g, RagGeom rg, const double2* __restrict__ F, const int* __restrict__ perm,
                         const int* __restrict__ items, int item0, int nwork, const int* __restrict__ klist,
                         int nrhs, double2* Y, long s_row, long s_k, int S) {
  extern __shared__ __align__(128) unsigned char smraw[];
  constexpr int NWC = PIPE_CONSUMERS;
  constexpr int NC = NWC * 32;
  const int T = g.T, T2 = T * T, nt = g.nt, npad = g.npad, n = g.n, q = n / 3;
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw);
  uint64_t* empty = full + S;
  long* rbase = reinterpret_cast<long*>(empty + S);
  double2* slots = reinterpret_cast<double2*>(smraw + ((2 * S + R) * 8 + 127) / 128 * 128);
  double2* y = slots + (long)S * T2;       // [npad][R]
  double2* red = y + (long)npad * R;       // [NWC][T][R]
  double2* zb = red + NWC * T * R;         // [T][R]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // Work items are strided over the grid (gridDim.x == nwork unless the
  // caller asked for a persistent grid); producer and consumers walk the same
  // item sequence, so the ring counter t simply continues across items.
  auto decode = [&](int w, int& slot, int& beg, int& cnt) {
    if (items) {
      const int it = item0 + w;
      slot = items[3 * it];
      beg = items[3 * it + 1];
      cnt = items[3 * it + 2];
    } else {
      slot = item0 + w;
      beg = slot;
      cnt = 1;
    }
  };

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, NWC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == NWC) {
    // ---------------- producer: same tile order as the consumers, all chunks
    if (lane == 0) {
      long t = 0;
      for (int w = blockIdx.x; w < nwork; w += gridDim.x) {
      int slot, beg, cnt;
      decode(w, slot, beg, cnt);
      int nb;
      const double2* Fb = rag_block(g, rg, F, slot, nb);
      const int ntb = rg.on ? (nb + T - 1) / T : nt;
      const int nchunks = (cnt * nrhs + R - 1) / R;
      for (int ch = 0; ch < nchunks; ++ch) {
        for (int ph = 0; ph < 2; ++ph) {
          for (int ii = 0; ii < ntb; ++ii) {
            const int i = ph == 0 ? ii : ntb - 1 - ii;
            const int j0 = ph == 0 ? 0 : i + 1, j1 = ph == 0 ? i : ntb;  // off-diagonal range
            const int ti = rg.on ? min(T, nb - T * i) : T;
            for (int j = j0; j <= j1; ++j) {
              const int jj = (j == j1) ? i : j;  // off-diagonals first, diagonal last
              const int s = (int)(t % S);
              const uint32_t use = (uint32_t)(t / S);
              if (use > 0) mbar_wait(empty + s, (use - 1) & 1);
              const int tj = rg.on ? min(T, nb - T * jj) : T;
              const double2* tsrc = rg.on ? Fb + (long)T * i * nb + (long)ti * T * jj : Fb + (long)(i * nt + jj) * T2;
              // the diagonal tile: only the half this phase uses (split layout)
              const double2* src = tsrc + ((j == j1 && ph == 1) ? dl_n(ti) : 0);
              const uint32_t bytes = (j == j1) ? (uint32_t)((ph == 0 ? dl_n(ti) : ti * ti - dl_n(ti)) * sizeof(double2))
                                               : (uint32_t)(ti * tj * sizeof(double2));
              if (bytes) {
                mbar_expect_tx(full + s, bytes);
                bulk_g2s(slots + (long)s * T2, src, bytes, full + s);
              } else {
                mbar_arrive(full + s);  // 1x1 diagonal: no strictly-lower half
              }
              ++t;
            }
          }
        }
      }
      }
    }
    return;
  }

  // ---------------- consumers
  long t = 0;
  for (int w = blockIdx.x; w < nwork; w += gridDim.x) {
  int slot, beg, cnt;
  decode(w, slot, beg, cnt);
  const int total = cnt * nrhs;
  const int nchunks = (total + R - 1) / R;
  for (int ch = 0; ch < nchunks; ++ch) {
    const int rho0 = ch * R;
    const int nr = min(R, total - rho0);
    if (tid < R) {
      long b = 0;
      if (tid < nr) {
        const int rho = rho0 + tid;
        const int kraw = klist ? klist[beg + rho / nrhs] : beg + rho / nrhs;
        b = rhs_base(kraw, rho, nrhs, s_k);
      }
      rbase[tid] = b;
    }
    consumers_sync(NC);
    const int* pm = perm + (long)slot * n;
    int nb;
    (void)rag_block(g, rg, F, slot, nb);
    const int ntb = rg.on ? (nb + T - 1) / T : nt;
    for (int idx = tid; idx < npad * R; idx += NC) {
      const int row = idx / R, rr = idx - row * R;
      double2 v = cmk(0.0, 0.0);
      if (row < nb && rr < nr) {
        const long rb = rbase[rr];
        const int pr = pm[row];
        v = cflip(Y[(long)pr * s_row + (rb & ROFF)], flip_row((int)(rb >> 56), pr, q));
      }
      y[idx] = v;
    }
    consumers_sync(NC);
    for (int ph = 0; ph < 2; ++ph) {
      for (int ii = 0; ii < ntb; ++ii) {
        const int i = ph == 0 ? ii : ntb - 1 - ii;
        const int j0 = ph == 0 ? 0 : i + 1, j1 = ph == 0 ? i : ntb;
        const int noff = j1 - j0;
        const int ti = rg.on ? min(T, nb - T * i) : T;  // rows of this tile row (= ld of its tiles)
        double2 acc[R];
#pragma unroll
        for (int rr = 0; rr < R; ++rr) acc[rr] = cmk(0.0, 0.0);
        // Every consumer warp walks every tile in order (waits, then releases;
        // only the owner q % NWC computes).  The empty barriers count NWC
        // arrivals, so no slot can be refilled before all consumers passed
        // it: parity waits are never more than one phase ahead.
        // Multi-RHS blocks (R = 8, T = 32): the tile GEMV becomes a 32x32 by
        // 32x8 complex product on the FP64 tensor cores (DMMA), fragments
        // straight from the ring slot and the RHS block in shared memory.
        constexpr bool USE_DMMA = (R == 8);
        const bool dmma = USE_DMMA && T == 32;
        double cr[4][2], ci[4][2];
#pragma unroll
        for (int rb = 0; rb < 4; ++rb) cr[rb][0] = cr[rb][1] = ci[rb][0] = ci[rb][1] = 0.0;
        for (int q = 0; q < noff; ++q) {
          const long tq = t + q;
          const int s = (int)(tq % S);
          mbar_wait(full + s, (uint32_t)(tq / S) & 1);
          if (!dmma && lane < ti) {
            // every consumer warp takes a column slice of every tile: the
            // tile GEMV is spread over all warps (short per-tile latency, so
            // the few ring slots turn over fast); partial sums meet in red
            const double2* tile = slots + (long)s * T2 + lane;
            const double2* yj = y + (long)(j0 + q) * T * R;
            const int tj = rg.on ? min(T, nb - T * (j0 + q)) : T;
            const int cpw = (tj + NWC - 1) / NWC, c0 = warp * cpw, c1 = min(tj, c0 + cpw);
            for (int c = c0; c < c1; ++c) {
              const double2 a = tile[c * ti];
#pragma unroll
              for (int rr = 0; rr < R; ++rr) cfma(acc[rr], a, yj[c * R + rr]);
            }
          } else if (q % NWC == warp) {
            if (dmma) {
              if constexpr (USE_DMMA) {
                const double2* tile = slots + (long)s * T2;
                const double2* yj = y + (long)(j0 + q) * 32 * R;
                const int r4 = lane >> 2, c4 = lane & 3;
#pragma unroll 2
                for (int k0 = 0; k0 < 32; k0 += 4) {
                  const double2 b = yj[(k0 + c4) * R + r4];   // B[k][col]: row k0+c4, col r4
#pragma unroll
                  for (int rb = 0; rb < 4; ++rb) {
                    const double2 a = tile[(k0 + c4) * 32 + rb * 8 + r4];  // A[row][k]
                    dmma884(cr[rb][0], cr[rb][1], a.x, b.x);
                    dmma884(cr[rb][0], cr[rb][1], -a.y, b.y);
                    dmma884(ci[rb][0], ci[rb][1], a.x, b.y);
                    dmma884(ci[rb][0], ci[rb][1], a.y, b.x);
                  }
                }
              }
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(empty + s);
        }
        if (dmma) {
          if constexpr (USE_DMMA) {
            const int r4 = lane >> 2, c4 = lane & 3;
#pragma unroll
            for (int rb = 0; rb < 4; ++rb)
#pragma unroll
              for (int e = 0; e < 2; ++e)
                red[(warp * 32 + rb * 8 + r4) * R + 2 * c4 + e] = cmk(cr[rb][e], ci[rb][e]);
          }
        } else if (lane < ti) {
#pragma unroll
          for (int rr = 0; rr < R; ++rr) red[(warp * T + lane) * R + rr] = acc[rr];
        }
        t += noff;
        consumers_sync(NC);
        for (int idx = tid; idx < ti * R; idx += NC) {
          const int r = idx / R, rr = idx - r * R;
          double2 z = y[(long)(i * T + r) * R + rr];
          for (int w = 0; w < NWC; ++w) z = csub(z, red[(w * T + r) * R + rr]);
          zb[idx] = z;
        }
        consumers_sync(NC);
        {
          const int s = (int)(t % S);
          mbar_wait(full + s, (uint32_t)(t / S) & 1);
          const double2* Ds = slots + (long)s * T2;
          for (int idx = tid; idx < ti * R; idx += NC) {
            const int r = idx / R, rr = idx - r * R;
            double2 o;
            if (ph == 0) {
              o = zb[idx];
              for (int c = 0, oc = r - 1; c < r; ++c) {  // oc = dl_off(ti, r, c)
                cfma(o, Ds[oc], zb[c * R + rr]);
                oc += ti - c - 2;
              }
            } else {
              o = cmk(0.0, 0.0);
              for (int c = r, ou = du_off(ti, r, r); c < ti; ++c) {  // ou = du_off(ti, r, c)
                cfma(o, Ds[ou], zb[c * R + rr]);
                ou += c + 1;
              }
            }
            y[(long)(i * T + r) * R + rr] = o;
          }
          consumers_sync(NC);
          if (lane == 0) mbar_arrive(empty + s);
          t += 1;
        }
      }
    }
    for (int idx = tid; idx < nb * R; idx += NC) {
      const int row = idx / R, rr = idx - row * R;
      if (rr < nr) {
        const long rb = rbase[rr];
        Y[(long)row * s_row + (rb & ROFF)] = cflip(y[idx], flip_row((int)(rb >> 56), row, q));
      }
    }
    consumers_sync(NC);
  }
  }
}

// padded factor blocks (dmax geometry, split diagonal tiles) -> ragged blocks
// of the sector dimensions (leading d_s x d_s: the identity padding of a
// smaller sector decouples from its LU, so its leading factors are exact)
__global__ void __launch_bounds__(256) lu_repack_kernel(LuGeom g, RagGeom rg, const double2* __restrict__ P,
                                                        double2* __restrict__ Q) {
  const int slot = blockIdx.y;
  int nb;
  double2* dst = const_cast<double2*>(rag_block(g, rg, Q, slot, nb));
  const double2* src = P + (long)slot * g.blk;
  const int T = g.T;
  const long tot = (long)nb * nb;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < tot; e += (long)gridDim.x * blockDim.x) {
    const int c = (int)(e / nb), r = (int)(e - (long)c * nb);
    const int i = r / T, j = c / T, rr = r - i * T, cc = c - j * T;
    const int ti = min(T, nb - T * i);
    const long dtile = (long)T * i * nb + (long)ti * T * j;
    const long stile = (long)(i * g.nt + j) * T * T;
    long so, d;
    if (i != j) {
      so = stile + (long)cc * T + rr;
      d = dtile + (long)rr * min(T, nb - T * j) + cc;
    } else if (rr > cc) {
      so = stile + dl_off(T, rr, cc);
      d = dtile + lrow_off(rr) + cc;
    } else {
      so = stile + dl_n(T) + du_off(T, rr, cc);
      d = dtile + dl_n(ti) + urow_off(ti, rr) + (cc - rr);
    }
    dst[d] = src[so];
  }
}

// inverse of lu_repack_kernel: every entry of the padded block is written
// (identity factors on the padding: inv(U) diagonal 1, everything else 0)
__global__ void __launch_bounds__(256) lu_unpack_kernel(LuGeom g, RagGeom rg, const double2* __restrict__ Q,
                                                        double2* __restrict__ P) {
  const int slot = blockIdx.y;
  int nb;
  const double2* src = rag_block(g, rg, Q, slot, nb);
  double2* dst = P + (long)slot * g.blk;
  const int T = g.T, np = g.npad;
  const long tot = (long)np * np;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < tot; e += (long)gridDim.x * blockDim.x) {
    const int c = (int)(e / np), r = (int)(e - (long)c * np);
    const int i = r / T, j = c / T, rr = r - i * T, cc = c - j * T;
    const long stile = (long)(i * g.nt + j) * T * T;
    const bool in = r < nb && c < nb;
    const int ti = in ? min(T, nb - T * i) : T;
    const long dtile = (long)T * i * nb + (long)ti * T * j;
    long po, qo;
    if (i != j) {
      po = stile + (long)cc * T + rr;
      qo = dtile + (long)rr * (in ? min(T, nb - T * j) : T) + cc;
    } else if (rr > cc) {
      po = stile + dl_off(T, rr, cc);
      qo = dtile + lrow_off(rr) + cc;
    } else {
      po = stile + dl_n(T) + du_off(T, rr, cc);
      qo = dtile + dl_n(ti) + urow_off(ti, rr) + (cc - rr);
    }
    dst[po] = in ? src[qo] : cmk(r == c ? 1.0 : 0.0, 0.0);
  }
}

static int make_rag(int nsec, const int* dims, int dmax, RagGeom* rg) {
  VX_REQUIRE(nsec >= 1 && nsec <= 4 && dims, "ragged geometry needs 1..4 sector dims");
  rg->on = 1;
  rg->nsec = nsec;
  long off = 0;
  for (int s = 0; s < 4; ++s) {
    rg->dims[s] = s < nsec ? dims[s] : 0;
    rg->soff[s] = off;
    if (s < nsec) {
      VX_REQUIRE(dims[s] >= 1 && dims[s] <= dmax, "sector dim %d out of range (dmax %d)", dims[s], dmax);
      off += (long)dims[s] * dims[s];
    }
  }
  rg->kstride = off;
  return VX_OK;
}

// ------------------------------------------- pipelined solve, ragged blocks
// The same producer / ring as lu_solve_pipe_kernel, but the ragged tiles are
// ROW-major (vx_lu_repack) and every consumer warp owns 4 rows of each tile:
// lane = 8 * row_in_warp + column_group, columns cg, cg + 8, cg + 16, cg + 24
// (consecutive lanes -> consecutive addresses: conflict-free).  A row's sum is
// finished with three xor-shuffles inside the warp, so there is no cross-warp
// reduction buffer; the diagonal products (row-packed inv(L_ii) / inv(U_ii))
// are spread the same way over all 256 consumer threads.  Two consumer
// barriers per tile row (the unpadded rows of zb, then of y).

template <int R>
__global__ void __launch_bounds__((PIPE_CONSUMERS + 1) * 32, 4)
    lu_solve_rag_kernel(LuGeom g, RagGeom rg, const double2* __restrict__ F, const int* __restrict__ perm,
                        const int* __restrict__ items, int item0, int nwork, const int* __restrict__ klist,
                        double2* Y, long s_row, long s_k, int S) {
  extern __shared__ __align__(128) unsigned char smraw[];
  constexpr int NWC = PIPE_CONSUMERS;
  constexpr int NC = NWC * 32;
  const int T = g.T, T2 = T * T, npad = g.npad, n = g.n, q = n / 3;
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw);
  uint64_t* empty = full + S;
  long* rbase = reinterpret_cast<long*>(empty + S);
  double2* slots = reinterpret_cast<double2*>(smraw + ((2 * S + R) * 8 + 127) / 128 * 128);
  double2* y = slots + (long)S * T2;  // [R][npad]
  double2* zb = y + (long)npad * R;   // [R][T]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  auto decode = [&](int w, int& slot, int& beg, int& cnt) {
    const int it = item0 + w;
    slot = items[3 * it];
    beg = items[3 * it + 1];
    cnt = items[3 * it + 2];
  };
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, NWC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == NWC) {
    if (lane == 0) {
      long t = 0;
      for (int w = blockIdx.x; w < nwork; w += gridDim.x) {
        int slot, beg, cnt;
        decode(w, slot, beg, cnt);
        int nb;
        const double2* Fb = rag_block(g, rg, F, slot, nb);
        const int ntb = (nb + T - 1) / T;
        const int nchunks = (cnt + R - 1) / R;
        for (int ch = 0; ch < nchunks; ++ch) {
          for (int ph = 0; ph < 2; ++ph) {
            for (int ii = 0; ii < ntb; ++ii) {
              const int i = ph == 0 ? ii : ntb - 1 - ii;
              const int j0 = ph == 0 ? 0 : i + 1, j1 = ph == 0 ? i : ntb;
              const int ti = min(T, nb - T * i);
              for (int j = j0; j <= j1; ++j) {
                const int jj = (j == j1) ? i : j;
                const int s = (int)(t % S);
                const uint32_t use = (uint32_t)(t / S);
                if (use > 0) mbar_wait(empty + s, (use - 1) & 1);
                const int tj = min(T, nb - T * jj);
                const double2* tsrc = Fb + (long)T * i * nb + (long)ti * T * jj;
                const double2* src = tsrc + ((j == j1 && ph == 1) ? dl_n(ti) : 0);
                const uint32_t bytes = (j == j1) ? (uint32_t)((ph == 0 ? dl_n(ti) : ti * ti - dl_n(ti)) * sizeof(double2))
                                                 : (uint32_t)(ti * tj * sizeof(double2));
                if (bytes) {
                  mbar_expect_tx(full + s, bytes);
                  bulk_g2s(slots + (long)s * T2, src, bytes, full + s);
                } else {
                  mbar_arrive(full + s);
                }
                ++t;
              }
            }
          }
        }
      }
    }
    return;
  }

  long t = 0;
  const int rw = lane >> 3, cg = lane & 7;
  const int r = 4 * warp + rw;  // tile row owned by this lane group
  for (int w = blockIdx.x; w < nwork; w += gridDim.x) {
    int slot, beg, cnt;
    decode(w, slot, beg, cnt);
    int nb;
    (void)rag_block(g, rg, F, slot, nb);
    const int ntb = (nb + T - 1) / T;
    const int* pm = perm + (long)slot * n;
    const int nchunks = (cnt + R - 1) / R;
    for (int ch = 0; ch < nchunks; ++ch) {
      const int rho0 = ch * R;
      const int nr = min(R, cnt - rho0);
      if (tid < R) {
        long b = 0;
        if (tid < nr) {
          const int kraw = klist ? klist[beg + rho0 + tid] : beg + rho0 + tid;
          b = rhs_base(kraw, rho0 + tid, 1, s_k);
        }
        rbase[tid] = b;
      }
      consumers_sync(NC);
      for (int idx = tid; idx < npad * R; idx += NC) {
        const int rr = idx / npad, row = idx - rr * npad;
        double2 v = cmk(0.0, 0.0);
        if (row < nb && rr < nr) {
          const long rb = rbase[rr];
          const int pr = pm[row];
          v = cflip(Y[(long)pr * s_row + (rb & ROFF)], flip_row((int)(rb >> 56), pr, q));
        }
        y[idx] = v;
      }
      consumers_sync(NC);
      for (int ph = 0; ph < 2; ++ph) {
        for (int ii = 0; ii < ntb; ++ii) {
          const int i = ph == 0 ? ii : ntb - 1 - ii;
          const int j0 = ph == 0 ? 0 : i + 1, j1 = ph == 0 ? i : ntb;
          const int noff = j1 - j0;
          const int ti = min(T, nb - T * i);
          const bool mine = r < ti;
          double2 acc[R];
#pragma unroll
          for (int rr = 0; rr < R; ++rr) acc[rr] = cmk(0.0, 0.0);
          for (int qq = 0; qq < noff; ++qq) {
            const long tq = t + qq;
            const int s = (int)(tq % S);
            mbar_wait(full + s, (uint32_t)(tq / S) & 1);
            const int j = j0 + qq;
            const int tj = min(T, nb - T * j);
            if (mine) {
              const double2* arow = slots + (long)s * T2 + r * tj;
              const double2* yj = y + T * j;
#pragma unroll
              for (int m = 0; m < 4; ++m) {
                const int c = cg + 8 * m;
                if (c < tj) {
                  const double2 a = arow[c];
#pragma unroll
                  for (int rr = 0; rr < R; ++rr) cfma(acc[rr], a, yj[rr * npad + c]);
                }
              }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + s);
          }
          t += noff;
#pragma unroll
          for (int rr = 0; rr < R; ++rr)
#pragma unroll
            for (int o = 1; o < 8; o <<= 1) {
              acc[rr].x += __shfl_xor_sync(0xffffffffu, acc[rr].x, o);
              acc[rr].y += __shfl_xor_sync(0xffffffffu, acc[rr].y, o);
            }
          if (mine && cg == 0)
#pragma unroll
            for (int rr = 0; rr < R; ++rr) zb[rr * T + r] = csub(y[rr * npad + T * i + r], acc[rr]);
          consumers_sync(NC);
          {
            const int s = (int)(t % S);
            mbar_wait(full + s, (uint32_t)(t / S) & 1);
            const double2* Ds = slots + (long)s * T2;
            double2 o[R];
#pragma unroll
            for (int rr = 0; rr < R; ++rr) o[rr] = cmk(0.0, 0.0);
            if (mine) {
              if (ph == 0) {
                const double2* Lr = Ds + lrow_off(r);
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                  const int c = cg + 8 * m;
                  if (c < r) {
                    const double2 a = Lr[c];
#pragma unroll
                    for (int rr = 0; rr < R; ++rr) cfma(o[rr], a, zb[rr * T + c]);
                  }
                }
              } else {
                const double2* Ur = Ds + urow_off(ti, r) - r;
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                  const int c = cg + 8 * m;
                  if (c >= r && c < ti) {
                    const double2 a = Ur[c];
#pragma unroll
                    for (int rr = 0; rr < R; ++rr) cfma(o[rr], a, zb[rr * T + c]);
                  }
                }
              }
            }
#pragma unroll
            for (int rr = 0; rr < R; ++rr)
#pragma unroll
              for (int o2 = 1; o2 < 8; o2 <<= 1) {
                o[rr].x += __shfl_xor_sync(0xffffffffu, o[rr].x, o2);
                o[rr].y += __shfl_xor_sync(0xffffffffu, o[rr].y, o2);
              }
            if (mine && cg == 0)
#pragma unroll
              for (int rr = 0; rr < R; ++rr)
                y[rr * npad + T * i + r] = ph == 0 ? cadd(zb[rr * T + r], o[rr]) : o[rr];
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + s);
            consumers_sync(NC);
            t += 1;
          }
        }
      }
      for (int idx = tid; idx < nb * R; idx += NC) {
        const int rr = idx / nb, row = idx - rr * nb;
        if (rr < nr) {
          const long rb = rbase[rr];
          Y[(long)row * s_row + (rb & ROFF)] = cflip(y[rr * npad + row], flip_row((int)(rb >> 56), row, q));
        }
      }
      consumers_sync(NC);
    }
  }
}

template <int R>
static int launch_solve_rag(const LuGeom& g, const RagGeom& rg, const double2* F, const int* perm, const int* items,
                            int nblocks, const int* klist, double2* Y, long s_row, long s_k, cudaStream_t s) {
  if (nblocks <= 0) return VX_OK;
  const size_t tile = (size_t)g.T * g.T * sizeof(double2);
  const size_t fixed = ((size_t)g.npad * R + (size_t)g.T * R) * sizeof(double2);
  // a 2-slot ring and as many CTAs per SM as fit (4 for sector-sized blocks):
  // more independent blocks in flight beat a deeper ring (c1: 0.93 ms with
  // 4 CTAs x 2 slots vs 1.01 ms with 3 x 4; c2: 1.10 vs 1.26 ms with 2 x 6)
  static const int slots_env = env_int("VX_RAG_SLOTS", 2);
  int S = slots_env;
  if (S > 16) S = 16;
  VX_REQUIRE(S >= 2, "block size %d too large for the ragged solve", g.n);
  const size_t smem = (((size_t)2 * S + R) * 8 + 127) / 128 * 128 + (size_t)S * tile + fixed;
  auto kern = lu_solve_rag_kernel<R>;
  VX_REQUIRE((int)smem + 1024 <= device_smem_optin(), "ragged solve smem %zu too large", smem);
  VX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<nblocks, (PIPE_CONSUMERS + 1) * 32, smem, s>>>(g, rg, F, perm, items, 0, nblocks, klist, Y, s_row, s_k, S);
  VX_CHECK_LAUNCH("lu_solve_rag_kernel");
  return VX_OK;
}

#include "lu_sym.cuh"
#include "lu_syminv.cuh"

// ------------------------------------------------------ single-tile blocks
// n <= 32 (the 2-level scheme's (3nz)^2 blocks): one warp per work item, lane
// = row; the packed diagonal tile holds inv(L) below and inv(U) on/above the
// diagonal, so a solve is two warp-shuffle triangular products.  8 items per
// CTA, no block-wide barriers.
constexpr int SMALL_WARPS = 8;

__global__ void __launch_bounds__(SMALL_WARPS * 32)
    lu_solve_small_kernel(int n, long blk, const double2* __restrict__ F, const int* __restrict__ perm,
                          const int* __restrict__ items, int item0, int nitems, const int* __restrict__ klist,
                          int nrhs, double2* Y, long s_row, long s_k) {
  extern __shared__ double2 smd[];
  const int lane = threadIdx.x & 31, wrp = threadIdx.x >> 5;
  const int it = blockIdx.x * SMALL_WARPS + wrp;
  if (it >= nitems) return;
  int slot, beg, cnt;
  if (items) {
    slot = items[3 * (item0 + it)];
    beg = items[3 * (item0 + it) + 1];
    cnt = items[3 * (item0 + it) + 2];
  } else {
    slot = item0 + it;
    beg = slot;
    cnt = 1;
  }
  // stage the packed tile with independent coalesced loads (high MLP)
  double2* Ds = smd + (long)wrp * n * n;
  const double2* D = F + (long)slot * blk;
  for (int i = lane; i < n * n; i += 32) Ds[i] = ld_stream(D + i);
  const int pr = lane < n ? perm[(long)slot * n + lane] : 0;
  __syncwarp();
  for (int rho = 0; rho < cnt * nrhs; ++rho) {
    const int kraw = klist ? klist[beg + rho / nrhs] : beg + rho / nrhs;
    const long base = (long)(kraw & KIDX) * s_k + (rho % nrhs);
    const int f2 = kraw >> 29;
    double2 yv = lane < n ? cflip(Y[(long)pr * s_row + base], flip_row(f2, pr, n / 3)) : cmk(0.0, 0.0);
    // forward: o = inv(L) y (unit lower)
    double2 o = yv;
    for (int c = 0; c < n; ++c) {
      const double2 yc = cmk(__shfl_sync(0xffffffffu, yv.x, c), __shfl_sync(0xffffffffu, yv.y, c));
      if (lane > c && lane < n) cfma(o, Ds[c * n + lane], yc);
    }
    // backward: x = inv(U) o
    double2 x = cmk(0.0, 0.0);
    for (int c = 0; c < n; ++c) {
      const double2 oc = cmk(__shfl_sync(0xffffffffu, o.x, c), __shfl_sync(0xffffffffu, o.y, c));
      if (c >= lane && lane < n) cfma(x, Ds[c * n + lane], oc);
    }
    if (lane < n) Y[(long)lane * s_row + base] = cflip(x, flip_row(f2, lane, n / 3));
  }
}

static int launch_solve_small(const LuGeom& g, const double2* F, const int* perm, const int* items, int item0,
                              int nitems, const int* klist, int nrhs, double2* Y, long s_row, long s_k,
                              cudaStream_t s) {
  if (nitems <= 0) return VX_OK;
  const size_t smem = (size_t)SMALL_WARPS * g.n * g.n * sizeof(double2);
  if (smem > 48 * 1024)
    VX_CUDA(cudaFuncSetAttribute(lu_solve_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  lu_solve_small_kernel<<<div_up(nitems, SMALL_WARPS), SMALL_WARPS * 32, smem, s>>>(
      g.n, g.blk, F, perm, items, item0, nitems, klist, nrhs, Y, s_row, s_k);
  VX_CHECK_LAUNCH("lu_solve_small_kernel");
  return VX_OK;
}

// Single-tile blocks held as explicit inverses G = A^-1, column-major per slot
// (entry (r, c) at c n + r): one warp per work item, lane = row, y_r = sum_c
// G[r, c] x_c for up to SINV_R right-hand sides (the x / y mirror partners of a
// shared block) at once.  No triangular dependency chain and no staging: the n
// column loads of a lane are independent and coalesced (n x 16 bytes per
// instruction), the x_c are warp-private shared-memory broadcasts.
#ifndef VX_SINV_WARPS
#define VX_SINV_WARPS 4
#endif
constexpr int SINV_WARPS = VX_SINV_WARPS, SINV_R = 4;

// N = n at compile time (n = 3 nz in the 2-level scheme): the lane's whole row
// of G sits in registers, loaded BEFORE the gather of x so both round trips to
// memory overlap; N = 0: runtime n, columns streamed eight at a time.
template <int N>
__global__ void __launch_bounds__(SINV_WARPS * 32)
    lu_apply_small_inv_kernel(int n_rt, long gblk, const double2* __restrict__ G, const int* __restrict__ items,
                              int item0, int nitems, const int* __restrict__ klist, int nrhs, double2* Y,
                              long s_row, long s_k) {
  __shared__ double2 xs[SINV_WARPS][SINV_R][32];
  const int n = N ? N : n_rt;
  const int lane = threadIdx.x & 31, wrp = threadIdx.x >> 5;
  const int it = blockIdx.x * SINV_WARPS + wrp;
  if (it >= nitems) return;
  int slot, beg, cnt;
  if (items) {
    slot = items[3 * (item0 + it)];
    beg = items[3 * (item0 + it) + 1];
    cnt = items[3 * (item0 + it) + 2];
  } else {
    slot = item0 + it;
    beg = slot;
    cnt = 1;
  }
  const double2* Gs = G + (long)slot * gblk + lane;
  const bool row = lane < n;
  double2 g[N ? N : 1];
  if constexpr (N > 0) {
#pragma unroll
    for (int c = 0; c < N; ++c) g[c] = row ? ld_stream(Gs + c * N) : cmk(0.0, 0.0);
  }
  const int q = n / 3, total = cnt * nrhs;
  for (int r0 = 0; r0 < total; r0 += SINV_R) {
    long base[SINV_R];
    int f2[SINV_R];
#pragma unroll
    for (int rr = 0; rr < SINV_R; ++rr) {
      const int rho = r0 + rr < total ? r0 + rr : total - 1;
      const int kraw = klist ? klist[beg + rho / nrhs] : beg + rho / nrhs;
      base[rr] = (long)(kraw & KIDX) * s_k + (rho % nrhs);
      f2[rr] = kraw >> 29;
      xs[wrp][rr][lane] = row ? cflip(Y[(long)lane * s_row + base[rr]], flip_row(f2[rr], lane, q)) : cmk(0.0, 0.0);
    }
    __syncwarp();
    double2 acc[SINV_R];
#pragma unroll
    for (int rr = 0; rr < SINV_R; ++rr) acc[rr] = cmk(0.0, 0.0);
    if constexpr (N > 0) {
#pragma unroll
      for (int c = 0; c < N; ++c) {
#pragma unroll
        for (int rr = 0; rr < SINV_R; ++rr) cfma(acc[rr], g[c], xs[wrp][rr][c]);
      }
    } else {
#pragma unroll 8
      for (int c = 0; c < n; ++c) {
        const double2 gc = row ? ld_stream(Gs + c * n) : cmk(0.0, 0.0);
#pragma unroll
        for (int rr = 0; rr < SINV_R; ++rr) cfma(acc[rr], gc, xs[wrp][rr][c]);
      }
    }
#pragma unroll
    for (int rr = 0; rr < SINV_R; ++rr)
      if (row && r0 + rr < total) Y[(long)lane * s_row + base[rr]] = cflip(acc[rr], flip_row(f2[rr], lane, q));
    __syncwarp();
  }
}

// G = A^-1 from the packed inverse-triangle tile: the solve of
// lu_solve_small_kernel applied to the n columns of the identity
__global__ void __launch_bounds__(SMALL_WARPS * 32)
    lu_small_invert_kernel(int n, long blk, const double2* __restrict__ F, const int* __restrict__ perm, int nslots,
                           double2* __restrict__ G) {
  extern __shared__ double2 smd[];
  const int lane = threadIdx.x & 31, wrp = threadIdx.x >> 5;
  const int slot = blockIdx.x * SMALL_WARPS + wrp;
  if (slot >= nslots) return;
  double2* Ds = smd + (long)wrp * n * n;
  const double2* D = F + (long)slot * blk;
  for (int i = lane; i < n * n; i += 32) Ds[i] = D[i];
  const int pr = lane < n ? perm[(long)slot * n + lane] : -1;
  __syncwarp();
  for (int j = 0; j < n; ++j) {
    const double2 yv = cmk(pr == j ? 1.0 : 0.0, 0.0);
    double2 o = yv;
    for (int c = 0; c < n; ++c) {
      const double2 yc = cmk(__shfl_sync(0xffffffffu, yv.x, c), __shfl_sync(0xffffffffu, yv.y, c));
      if (lane > c && lane < n) cfma(o, Ds[c * n + lane], yc);
    }
    double2 x = cmk(0.0, 0.0);
    for (int c = 0; c < n; ++c) {
      const double2 oc = cmk(__shfl_sync(0xffffffffu, o.x, c), __shfl_sync(0xffffffffu, o.y, c));
      if (c >= lane && lane < n) cfma(x, Ds[c * n + lane], oc);
    }
    if (lane < n) G[((long)slot * n + j) * n + lane] = x;
  }
}

static int launch_apply_small_inv(int n, const double2* G, const int* items, int nitems, const int* klist, int nrhs,
                                  double2* Y, long s_row, long s_k, cudaStream_t s) {
  if (nitems <= 0) return VX_OK;
  Span span("prec_solve", s);
  const unsigned grid = div_up(nitems, SINV_WARPS);
  switch (n) {
#define VX_SINV_CASE(N_)                                                                            \
  case N_:                                                                                          \
    lu_apply_small_inv_kernel<N_><<<grid, SINV_WARPS * 32, 0, s>>>(n, (long)n * n, G, items, 0, nitems, klist, nrhs, \
                                                                   Y, s_row, s_k);                  \
    break;
    VX_SINV_CASE(6) VX_SINV_CASE(9) VX_SINV_CASE(12) VX_SINV_CASE(15) VX_SINV_CASE(18) VX_SINV_CASE(21)
    VX_SINV_CASE(24) VX_SINV_CASE(27) VX_SINV_CASE(30)
#undef VX_SINV_CASE
    default:
      lu_apply_small_inv_kernel<0><<<grid, SINV_WARPS * 32, 0, s>>>(n, (long)n * n, G, items, 0, nitems, klist, nrhs,
                                                                    Y, s_row, s_k);
  }
  VX_CHECK_LAUNCH("lu_apply_small_inv_kernel");
  return VX_OK;
}

template <int R>
static int launch_solve_pipe(const LuGeom& g, const double2* F, const int* perm, const int* items,
                             int item0, int nblocks, const int* klist, int nrhs, double2* Y, long s_row,
                             long s_k, cudaStream_t s, int persist_per_sm = 0, const RagGeom* rgp = nullptr) {
  RagGeom rg{};
  if (rgp) rg = *rgp;
  VX_REQUIRE(!(rg.on && R == 8), "ragged factor storage has no multi-RHS (DMMA) solve");
  if (nblocks <= 0) return VX_OK;
  const size_t tile = (size_t)g.T * g.T * sizeof(double2);
  const size_t fixed = ((size_t)g.npad * R + (size_t)PIPE_CONSUMERS * g.T * R + (size_t)g.T * R) *
                       sizeof(double2);
  // two CTAs per SM when the vector state is small, otherwise one
  static const int budget_kb = env_int("VX_PIPE_BUDGET_KB", 0);
  // small blocks (symmetry sectors: <= 8 x 8 tiles) run 3 CTAs per SM -- their
  // per-block fill / gather / diagonal latencies need more CTAs in flight;
  // bigger ones 2 (or 1 when the vector state is large)
  size_t budget = (fixed < 40 * 1024 ? (g.nt <= 8 ? 72 : 112) * 1024 : (size_t)device_smem_optin() - 2048);
  if (budget_kb > 0 && R <= 2) budget = (size_t)budget_kb * 1024;
  int S = (int)((budget > fixed ? budget - fixed : 0) / tile);
  if (S > 16) S = 16;
  VX_REQUIRE(S >= 2, "block size %d too large for the pipelined solve", g.n);
  const size_t smem = (((size_t)2 * S + R) * 8 + 127) / 128 * 128 + (size_t)S * tile + fixed;
  auto kern = lu_solve_pipe_kernel<R>;
  VX_REQUIRE((int)smem + 1024 <= device_smem_optin(), "pipelined solve smem %zu too large", smem);
  VX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int grid = nblocks;
  if (persist_per_sm > 0 && grid > persist_per_sm * device_sm_count()) grid = persist_per_sm * device_sm_count();
  kern<<<grid, (PIPE_CONSUMERS + 1) * 32, smem, s>>>(g, rg, F, perm, items, item0, nblocks, klist, nrhs, Y,
                                                     s_row, s_k, S);
  VX_CHECK_LAUNCH("lu_solve_pipe_kernel");
  return VX_OK;
}

// ------------------------------------------------------- sharding transposes
// out = concat_s A[:, colmap[col_off[s] : col_off[s+1]]] (each block row-major):
// the per-destination send buffers of the all-to-all transposes.
__global__ void cols_copy_kernel(long nrows, double2* A, long lda, int P, const int* __restrict__ col_off,
                                 const int* __restrict__ colmap, double2* buf, int to_buf) {
  const long total = nrows * col_off[P];
  for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total;
       idx += (long)gridDim.x * blockDim.x) {
    int sdst = 0;
    while (sdst + 1 < P && idx >= nrows * col_off[sdst + 1]) ++sdst;
    const long ncol = col_off[sdst + 1] - col_off[sdst];
    const long loc = idx - nrows * col_off[sdst];
    const long row = loc / ncol, j = loc - row * ncol;
    const long a = row * lda + colmap[col_off[sdst] + j];
    if (to_buf) buf[idx] = A[a];
    else A[a] = buf[idx];
  }
}

// Dispatch the block solves of a work list: single-tile blocks -> warp-per-block
// kernel; larger blocks -> TMA-pipelined kernel (items [0, n_single) one RHS
// each, the rest multi-RHS).  vx_solve_variant(1) selects the synchronous kernel.
static int solve_items(const LuGeom& g, const double2* F, const int* perm, const int* items, int n_single,
                       int n_items, const int* klist, int nrhs, double2* Y, long s_row, long s_k, cudaStream_t s,
                       int persist = -1, int direct_r = 1, const RagGeom* rg = nullptr) {
  int st;
  Span span("prec_solve", s);
  static const int persist_env = env_int("VX_PIPE_PERSIST", 0);
  if (persist < 0) persist = persist_env;
  if (rg && rg->on) {
    VX_REQUIRE(g.nt > 1 && !g_solve_classic && nrhs == 1 && n_items == n_single,
               "ragged factors: single-RHS pipelined solves only");
    (void)persist;
    VX_REQUIRE(items, "ragged solves take a work list");
    if (direct_r == 2) return launch_solve_rag<2>(g, *rg, F, perm, items, n_single, klist, Y, s_row, s_k, s);
    if (direct_r == 4) return launch_solve_rag<4>(g, *rg, F, perm, items, n_single, klist, Y, s_row, s_k, s);
    return launch_solve_rag<1>(g, *rg, F, perm, items, n_single, klist, Y, s_row, s_k, s);
  }
  if (g.nt == 1 && !g_solve_classic)
    return launch_solve_small(g, F, perm, items, 0, n_items, klist, nrhs, Y, s_row, s_k, s);
  const bool pipe = g.nt > 1 && !g_solve_classic;
  if (nrhs == 1 && direct_r == 2)  // mirror pairs: one factor stream, two frequencies
    st = pipe ? launch_solve_pipe<2>(g, F, perm, items, 0, n_single, klist, 1, Y, s_row, s_k, s, persist)
              : launch_solve<2, SOLVE_WARPS>(g, F, perm, items, 0, n_single, klist, 1, Y, s_row, s_k, s);
  else if (nrhs == 1 && direct_r == 4)  // 2-level x/y mirror quadruples
    st = pipe ? launch_solve_pipe<4>(g, F, perm, items, 0, n_single, klist, 1, Y, s_row, s_k, s, persist)
              : launch_solve<4, SOLVE_WARPS>(g, F, perm, items, 0, n_single, klist, 1, Y, s_row, s_k, s);
  else if (nrhs == 1)
    st = pipe ? launch_solve_pipe<1>(g, F, perm, items, 0, n_single, klist, 1, Y, s_row, s_k, s, persist)
              : launch_solve<1, SOLVE_WARPS>(g, F, perm, items, 0, n_single, klist, 1, Y, s_row, s_k, s);
  else
    st = pipe ? launch_solve_pipe<MULTI_R>(g, F, perm, items, 0, n_single, klist, nrhs, Y, s_row, s_k, s)
              : launch_solve<MULTI_R, SOLVE_WARPS>(g, F, perm, items, 0, n_single, klist, nrhs, Y, s_row, s_k, s);
  if (st) return st;
  return pipe ? launch_solve_pipe<MULTI_R>(g, F, perm, items, n_single, n_items - n_single, klist, nrhs, Y,
                                           s_row, s_k, s)
              : launch_solve<MULTI_R, SOLVE_WARPS>(g, F, perm, items, n_single, n_items - n_single, klist, nrhs,
                                                   Y, s_row, s_k, s);
}

// ------------------------------------------------- symmetry-sector transform
// One orbit o = (component, site orbit under the reflections) per grid row:
// forward  u[osec[o][s]] = sum_t ocoef[o][s][t] x[orows[o][t]]   (V^T x)
// inverse  x[orows[o][t]] = sum_s ocoef[o][s][t] u[osec[o][s]]   (V u)
// at every spectral column col = k*nrhs + j of the (rows x pitch) arrays;
// flipk[k] (nullable) applies the x-mirror sign of a shared factor (x rows).
__global__ void __launch_bounds__(256) sec_xform_kernel(long pitch, int nrhs, const int* __restrict__ orows,
                                                        const int* __restrict__ osec,
                                                        const double* __restrict__ ocoef,
                                                        const unsigned char* __restrict__ flipk, int q,
                                                        const double2* __restrict__ in, double2* __restrict__ out,
                                                        int inverse) {
  const int o = blockIdx.y;
  int rw[4], sc[4];
  double cf[4][4];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    rw[t] = __ldg(orows + 4 * o + t);
    sc[t] = __ldg(osec + 4 * o + t);
#pragma unroll
    for (int u = 0; u < 4; ++u) cf[t][u] = __ldg(ocoef + 16 * o + 4 * t + u);  // [s][t]
  }
  const bool xrow = rw[0] < q;
  for (long col = blockIdx.x * (long)blockDim.x + threadIdx.x; col < pitch; col += (long)gridDim.x * blockDim.x) {
    const double sg = (flipk && xrow && flipk[col / nrhs]) ? -1.0 : 1.0;
    if (!inverse) {
      double2 v[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) v[t] = rw[t] >= 0 ? __ldg(in + (long)rw[t] * pitch + col) : cmk(0.0, 0.0);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (sc[u] < 0) continue;
        double2 a = cmk(0.0, 0.0);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          a.x = fma(cf[u][t], v[t].x, a.x);
          a.y = fma(cf[u][t], v[t].y, a.y);
        }
        out[(long)sc[u] * pitch + col] = cmk(sg * a.x, sg * a.y);
      }
    } else {
      double2 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = sc[u] >= 0 ? __ldg(in + (long)sc[u] * pitch + col) : cmk(0.0, 0.0);
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        if (rw[t] < 0) continue;
        double2 a = cmk(0.0, 0.0);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          a.x = fma(cf[u][t], v[u].x, a.x);
          a.y = fma(cf[u][t], v[u].y, a.y);
        }
        out[(long)rw[t] * pitch + col] = cmk(sg * a.x, sg * a.y);
      }
    }
  }
}

static int sec_xform(long pitch, int nrhs, int norb, const int* orows, const int* osec, const double* ocoef,
                     const unsigned char* flipk, int q, const double2* in, double2* out, int inverse,
                     cudaStream_t s) {
  if (norb <= 0) return VX_OK;
  long bx = div_up(pitch, 256);
  if (bx > 64) bx = 64;
  dim3 grid((unsigned)bx, (unsigned)norb);
  sec_xform_kernel<<<grid, 256, 0, s>>>(pitch, nrhs, orows, osec, ocoef, flipk, q, in, out, inverse);
  VX_CHECK_LAUNCH("sec_xform_kernel");
  return VX_OK;
}

// ---------------------------------------------------------------- blocked
__global__ void box_copy_kernel(int nx, int ny, int nz, int x0, int y0, int z0, int bx, int by,
                                int bz, int nrhs, const double2* __restrict__ src,
                                double2* __restrict__ dst, int to_box) {
  const long total = 3L * bz * by * bx * nrhs;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    long r = i;
    const int j = (int)(r % nrhs); r /= nrhs;
    const int x = (int)(r % bx); r /= bx;
    const int y = (int)(r % by); r /= by;
    const int z = (int)(r % bz); r /= bz;
    const int c = (int)r;
    const long full = ((((long)c * nz + z0 + z) * ny + y0 + y) * nx + x0 + x) * nrhs + j;
    if (to_box) dst[i] = src[full];
    else dst[full] = src[i];
  }
}


// ------------------------------------------- representative-block GEMM
// Reduced 1-level scheme: every discarded frequency is solved with the one
// representative block, so those solves are ONE product D_rep^-1 * B with B =
// the gathered spectral columns (726 x 4374 at c1r).  The explicit inverse is
// formed once at build time (a solve against the identity with the factors),
// and the apply becomes a dense complex GEMM on the FP64 tensor cores instead
// of ~550 serial triangular sweeps re-reading the factor from L2.  It runs on a
// side stream, concurrently with the HBM-bound single-block solves (disjoint
// spectral columns).
constexpr int RG_M = 64, RG_N = 64, RG_K = 16;
// smem row pitch of a k-row: +2 entries, so the four k-rows a quarter warp reads
// (lanes = 4 k x 2 rows of one 16-byte phase) land on distinct bank groups; an
// unpadded 1 KB pitch put them on the same one (4-way conflicts on every fragment load)
constexpr int RG_LDA = RG_M + 2, RG_LDB = RG_N + 2;
constexpr int RG_THREADS = 256;

static inline int rep_kp(int n) { return (n + RG_K - 1) / RG_K * RG_K; }
static inline int rep_mp(int n) { return (n + RG_M - 1) / RG_M * RG_M; }

__global__ void eye_cols_kernel(int n, long ld, double2* A) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) A[(long)i * ld + i] = make_double2(1.0, 0.0);
}

// Up to four products in one launch (the sector blocks of the reduced scheme):
// product z has n[z] rows, its inverse at A + a_off[z], its spectral rows at
// S + s_off[z] and its gathered operand at Bt + z * bt_stride.
struct RepBatch {
  int nb;
  int n[4];
  long a_off[4];
  long s_off[4];
  long bt_stride;
};

// Bt[k][j] (ldb = padded column count) <- S[k*s_row + ks[j/nrhs]*s_k + j%nrhs],
// zero outside k < n, j < ncols; blockIdx.y = product of the batch.
__global__ void rep_gather_kernel(RepBatch rb, int ncols, int Np, int nrhs, const int* __restrict__ ks,
                                  const double2* __restrict__ S, long s_row, long s_k, double2* __restrict__ Bt) {
  // selects, not rb.n[z]: a runtime index would copy the parameter struct to local memory
  const int z = blockIdx.y;
  const int n = z == 0 ? rb.n[0] : z == 1 ? rb.n[1] : z == 2 ? rb.n[2] : rb.n[3];
  const int Kp = (n + RG_K - 1) / RG_K * RG_K;
  S += z == 0 ? rb.s_off[0] : z == 1 ? rb.s_off[1] : z == 2 ? rb.s_off[2] : rb.s_off[3];
  Bt += z * rb.bt_stride;
  const long total = (long)Kp * Np;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    const int k = (int)(i / Np), j = (int)(i - (long)k * Np);
    double2 v = make_double2(0.0, 0.0);
    if (k < n && j < ncols) v = S[(long)k * s_row + (long)ks[j / nrhs] * s_k + j % nrhs];
    Bt[i] = v;
  }
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// C = A * Bt scattered into S: A is the inverse stored k-major (A[k*lda + m],
// Kp x lda, zero padded), Bt from rep_gather_kernel.  CTA tile 64 x 64 complex,
// K step 16, 3-stage cp.async ring; 8 warps as 2 (m) x 4 (n), warp tile 32 x 16
// = 4 x 2 DMMA 8x8 blocks, each complex product = 4 real DMMAs.
__global__ void __launch_bounds__(RG_THREADS, 2)
    rep_gemm_kernel(RepBatch rb, const double2* __restrict__ A, long lda, const double2* __restrict__ Bt,
                    long ldb, int ncols, int nrhs, const int* __restrict__ ks, double2* S, long s_row, long s_k,
                    int RG_STAGES) {
  extern __shared__ __align__(128) double2 rg_sm[];
  // selects, not rb.n[z]: a runtime index would copy the parameter struct to local memory
  const int z = blockIdx.z;
  const int n = z == 0 ? rb.n[0] : z == 1 ? rb.n[1] : z == 2 ? rb.n[2] : rb.n[3];
  const int Kp = (n + RG_K - 1) / RG_K * RG_K;
  if ((int)blockIdx.y * RG_M >= n) return;  // row tiles beyond this product's block
  A += z == 0 ? rb.a_off[0] : z == 1 ? rb.a_off[1] : z == 2 ? rb.a_off[2] : rb.a_off[3];
  Bt += z * rb.bt_stride;
  S += z == 0 ? rb.s_off[0] : z == 1 ? rb.s_off[1] : z == 2 ? rb.s_off[2] : rb.s_off[3];
  constexpr int TA = RG_K * RG_LDA, TB = RG_K * RG_LDB;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
  const int r4 = lane >> 2, c4 = lane & 3;
  const int m0 = blockIdx.y * RG_M, n0 = blockIdx.x * RG_N;
  const int nk = Kp / RG_K;

  auto load_stage = [&](int kt, int st) {
    double2* As = rg_sm + st * (TA + TB);
    double2* Bs = As + TA;
    const int k0 = kt * RG_K;
#pragma unroll
    for (int it = 0; it < RG_K * RG_M / RG_THREADS; ++it) {
      const int e = tid + it * RG_THREADS;
      const int kk = e / RG_M, mm = e - kk * RG_M;
      cp_async16(As + kk * RG_LDA + mm, A + (long)(k0 + kk) * lda + m0 + mm);
    }
#pragma unroll
    for (int it = 0; it < RG_K * RG_N / RG_THREADS; ++it) {
      const int e = tid + it * RG_THREADS;
      const int kk = e / RG_N, nn = e - kk * RG_N;
      cp_async16(Bs + kk * RG_LDB + nn, Bt + (long)(k0 + kk) * ldb + n0 + nn);
    }
  };

  double cr[4][2][2], ci[4][2][2];
#pragma unroll
  for (int rb = 0; rb < 4; ++rb)
#pragma unroll
    for (int cb = 0; cb < 2; ++cb) cr[rb][cb][0] = cr[rb][cb][1] = ci[rb][cb][0] = ci[rb][cb][1] = 0.0;

  for (int st = 0; st < RG_STAGES - 1; ++st) {
    if (st < nk) load_stage(st, st);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    if (RG_STAGES == 3) cp_async_wait<1>();
    else cp_async_wait<0>();
    __syncthreads();
    if (kt + RG_STAGES - 1 < nk) load_stage(kt + RG_STAGES - 1, (kt + RG_STAGES - 1) % RG_STAGES);
    cp_async_commit();
    const double2* As = rg_sm + (kt % RG_STAGES) * (TA + TB);
    const double2* Bs = As + TA;
#pragma unroll
    for (int k4 = 0; k4 < RG_K; k4 += 4) {
      const int kk = k4 + c4;
      double2 a[4], b[2];
#pragma unroll
      for (int rb = 0; rb < 4; ++rb) a[rb] = As[kk * RG_LDA + wm * 32 + rb * 8 + r4];
#pragma unroll
      for (int cb = 0; cb < 2; ++cb) b[cb] = Bs[kk * RG_LDB + wn * 16 + cb * 8 + r4];
      // the MMAs are volatile (program order): two sweeps over the 16 accumulators, so the
      // second MMA on an accumulator issues 16 instructions after the first, not right behind it
#pragma unroll
      for (int rb = 0; rb < 4; ++rb)
#pragma unroll
        for (int cb = 0; cb < 2; ++cb) {
          dmma884(cr[rb][cb][0], cr[rb][cb][1], a[rb].x, b[cb].x);
          dmma884(ci[rb][cb][0], ci[rb][cb][1], a[rb].x, b[cb].y);
        }
#pragma unroll
      for (int rb = 0; rb < 4; ++rb)
#pragma unroll
        for (int cb = 0; cb < 2; ++cb) {
          dmma884(cr[rb][cb][0], cr[rb][cb][1], -a[rb].y, b[cb].y);
          dmma884(ci[rb][cb][0], ci[rb][cb][1], a[rb].y, b[cb].x);
        }
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int rb = 0; rb < 4; ++rb) {
    const int m = m0 + wm * 32 + rb * 8 + r4;
    if (m >= n) continue;
#pragma unroll
    for (int cb = 0; cb < 2; ++cb)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = n0 + wn * 16 + cb * 8 + 2 * c4 + e;
        if (j < ncols)
          S[(long)m * s_row + (long)ks[j / nrhs] * s_k + j % nrhs] = make_double2(cr[rb][cb][e], ci[rb][cb][e]);
      }
  }
}

static int g_rep_sequential = 0;  // vx_rep_variant(1): GEMM on the main stream (A/B timing)

struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
static SideStream* side_stream() {
  static thread_local SideStream ss;
  if (!ss.s) {
    if (cudaStreamCreateWithFlags(&ss.s, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming) != cudaSuccess) {
      ss.s = nullptr;
      return nullptr;
    }
  }
  return &ss;
}

// lda: leading dimension of the k-major inverse (rep_mp(n) for an inverse of
// exactly n rows; a sector inverse formed in the dmax geometry keeps
// rep_mp(dmax) -- its rows / columns beyond n are the identity padding, so the
// leading n x n part is the sector block's inverse).
static int rep_gemm_batch(const RepBatch& rb, const double2* inv, int ncols, int nrhs, const int* ks, double2* S,
                          long s_row, long s_k, double2* Bt, cudaStream_t s, long lda) {
  int nmax = 0;
  for (int z = 0; z < rb.nb; ++z) nmax = rb.n[z] > nmax ? rb.n[z] : nmax;
  const int Mp = rep_mp(nmax);
  const int Np = (ncols + RG_N - 1) / RG_N * RG_N;
  const long total = (long)rep_kp(nmax) * Np;
  {
    const unsigned gb = div_up(total, 256) < 8192 ? div_up(total, 256) : 8192;
    rep_gather_kernel<<<dim3(gb, rb.nb), 256, 0, s>>>(rb, ncols, Np, nrhs, ks, S, s_row, s_k, Bt);
    VX_CHECK_LAUNCH("rep_gather_kernel");
  }
  static const int stages = env_int("VX_RG_STAGES", 3) == 2 ? 2 : 3;
  const size_t smem = (size_t)stages * (RG_K * RG_LDA + RG_K * RG_LDB) * sizeof(double2);
  static bool attr = false;
  if (!attr) {
    VX_CUDA(cudaFuncSetAttribute(rep_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(3 * (RG_K * RG_LDA + RG_K * RG_LDB) * sizeof(double2))));
    attr = true;
  }
  dim3 grid(Np / RG_N, Mp / RG_M, rb.nb);
  rep_gemm_kernel<<<grid, RG_THREADS, smem, s>>>(rb, inv, lda, Bt, Np, ncols, nrhs, ks, S, s_row, s_k, stages);
  VX_CHECK_LAUNCH("rep_gemm_kernel");
  return VX_OK;
}

// lda: leading dimension of the k-major inverse (rep_mp(n) for an inverse of
// exactly n rows; a sector inverse formed in the dmax geometry keeps
// rep_mp(dmax) -- its rows / columns beyond n are the identity padding, so the
// leading n x n part is the sector block's inverse).
static int rep_gemm(int n, const double2* inv, int ncols, int nrhs, const int* ks, double2* S, long s_row,
                    long s_k, double2* Bt, cudaStream_t s, long lda = -1) {
  RepBatch rb{};
  rb.nb = 1;
  rb.n[0] = n;
  return rep_gemm_batch(rb, inv, ncols, nrhs, ks, S, s_row, s_k, Bt, s, lda < 0 ? rep_mp(n) : lda);
}

}  // namespace vx

using namespace vx;

extern "C" int vx_chan_x_spectra(int nx, int ny, int nz, const vx_c128* gen, long g_sp, long g_sz,
                                 long g_sy, long g_sx, vx_c128* lamT, void* stream) {
  VX_REQUIRE(nx >= 1 && ny >= 1 && nz >= 1, "grid dims must be >= 1");
  FftPlan p;
  int st = fft_get_plan(nx, &p);
  if (st) return st;
  const int nzz = 2 * nz - 1, nyy = 2 * ny - 1;
  const int lines = 6 * nzz * nyy;
  LoadChanGen ld{reinterpret_cast<const double2*>(gen), {g_sp, g_sz, g_sy, nzz, nyy}, g_sx, nx};
  StoreStrided sv{reinterpret_cast<double2*>(lamT), {1, 0, lines, 1}, 1.0};
  return launch_fft_auto(p, ld, sv, lines, nx, nx, false, false, as_stream(stream));
}

extern "C" int vx_proxy(int nx, int ny, int nz, const vx_c128* lamT, vx_c128 m00, vx_c128* proxy,
                        void* stream) {
  const long Ltot = 6L * (2 * nz - 1) * (2 * ny - 1);
  proxy_kernel<<<div_up(nx, 256), 256, 0, as_stream(stream)>>>(
      nx, Ltot, reinterpret_cast<const double2*>(lamT), make_double2(m00.re, m00.im),
      (ny * nz == 1) ? 1 : 0, reinterpret_cast<double2*>(proxy));
  VX_CHECK_LAUNCH("proxy_kernel");
  return VX_OK;
}

extern "C" int vx_lu_tile(int n) { return lu_geom(n).T; }
extern "C" long vx_lu_block_elems(int n) { return lu_geom(n).blk; }

extern "C" int vx_lu1_build(int nx, int ny, int nz, const vx_c128* lamT, const vx_c128* m_yz,
                            const int* kset, int nslots, vx_c128* factors, int* perm, int* piv,
                            int* info, void* stream) {
  VX_REQUIRE(nx >= 1 && ny >= 1 && nz >= 1 && nslots >= 0, "bad 1-level build arguments");
  Unfold u{reinterpret_cast<const double2*>(lamT), reinterpret_cast<const double2*>(m_yz), kset,
           6L * (2 * nz - 1) * (2 * ny - 1), nz, ny};
  return lu_build(u, 3 * ny * nz, nslots, reinterpret_cast<double2*>(factors), perm, piv, info,
                  as_stream(stream));
}

extern "C" long vx_prec1_work_elems(int nx, int ny, int nz, int nrhs) {
  return 3L * nx * ny * nz * nrhs;
}

static int prec1_apply(int nx, int ny, int nz, int nrhs, const vx_c128* factors, const int* perm,
                       const int* items, int n_single, int n_items, int direct_r, const int* klist,
                       const vx_c128* x, vx_c128* y, vx_c128* work, void* stream, const RagGeom* rg) {
  VX_REQUIRE(nx >= 1 && ny >= 1 && nz >= 1 && nrhs >= 1, "bad 1-level apply arguments");
  VX_REQUIRE(direct_r == 1 || direct_r == 2, "direct_r must be 1 or 2");
  VX_REQUIRE(n_single >= 0 && n_items >= n_single, "bad work list");
  cudaStream_t s = as_stream(stream);
  Span span("prec_apply", s);
  FftPlan p;
  int st = fft_get_plan(nx, &p);
  if (st) return st;
  const int q3 = 3 * ny * nz;
  double2* S = reinterpret_cast<double2*>(work);
  const long pitch = (long)nx * nrhs;
  {
    LoadStrided ld{reinterpret_cast<const double2*>(x), {pitch, 1, nrhs, nrhs}};
    StoreStrided sv{S, {pitch, 1, nrhs, nrhs}, 1.0};
    if ((st = launch_fft_auto(p, ld, sv, q3 * nrhs, nx, nx, false, nrhs == 1, s))) return st;
  }
  LuGeom g = lu_geom(q3);
  const double2* F = reinterpret_cast<const double2*>(factors);
  if ((st = solve_items(g, F, perm, items, n_single, n_items, klist, nrhs, S, pitch, nrhs, s, -1, direct_r, rg)))
    return st;
  {
    LoadStrided ld{S, {pitch, 1, nrhs, nrhs}};
    StoreStrided sv{reinterpret_cast<double2*>(y), {pitch, 1, nrhs, nrhs}, 1.0 / nx};
    if ((st = launch_fft_auto(p, ld, sv, q3 * nrhs, nx, nx, true, nrhs == 1, s))) return st;
  }
  return VX_OK;
}

extern "C" long vx_chan_xy_work_elems(int nx, int ny, int nz) {
  return 6L * (2 * nz - 1) * (2 * ny - 1) * nx;
}

extern "C" int vx_chan_xy_spectra(int nx, int ny, int nz, const vx_c128* gen, long g_sp, long g_sz,
                                  long g_sy, long g_sx, vx_c128* lam2T, vx_c128* work,
                                  void* stream) {
  VX_REQUIRE(nx >= 1 && ny >= 1 && nz >= 1, "grid dims must be >= 1");
  cudaStream_t s = as_stream(stream);
  FftPlan px, py;
  int st;
  if ((st = fft_get_plan(nx, &px)) || (st = fft_get_plan(ny, &py))) return st;
  const int nzz = 2 * nz - 1, nyy = 2 * ny - 1;
  double2* tmp = reinterpret_cast<double2*>(work);  // (6, nzz, nyy, nx)
  {
    LoadChanGen ld{reinterpret_cast<const double2*>(gen), {g_sp, g_sz, g_sy, nzz, nyy}, g_sx, nx};
    StoreStrided sv{tmp, {nx, 0, 1, 1}, 1.0};
    if ((st = launch_fft_auto(px, ld, sv, 6 * nzz * nyy, nx, nx, false, g_sx == 1, s))) return st;
  }
  {
    // lines (p, dz) x k along dy; Chan along y, DFT length ny, k-major output
    LoadChan ld{tmp, {(long)nyy * nx, 1, nx, nx}, ny};
    StoreStrided sv{reinterpret_cast<double2*>(lam2T), {1, 6L * nzz, 6L * nzz * nx, nx}, 1.0};
    if ((st = launch_fft_auto(py, ld, sv, 6 * nzz * nx, ny, ny, false, false, s))) return st;
  }
  return VX_OK;
}

extern "C" int vx_lu2_build(int nx, int ny, int nz, const vx_c128* lam2T, const vx_c128* m_z,
                            const int* kset, int nslots, vx_c128* factors, int* perm, int* piv, int* info,
                            void* stream) {
  VX_REQUIRE(nx >= 1 && ny >= 1 && nz >= 1, "bad 2-level build arguments");
  if (!kset) nslots = nx * ny;
  VX_REQUIRE(nslots >= 0 && nslots <= nx * ny, "bad 2-level slot count");
  Unfold u{reinterpret_cast<const double2*>(lam2T), reinterpret_cast<const double2*>(m_z), kset,
           6L * (2 * nz - 1), nz, 1};
  return lu_build(u, 3 * nz, nslots, reinterpret_cast<double2*>(factors), perm, piv, info,
                  as_stream(stream));
}

extern "C" long vx_prec2_work_elems(int nx, int ny, int nz, int nrhs) {
  return 3L * nx * ny * nz * nrhs;
}

static int prec2_apply_impl(int nx, int ny, int nz, int nrhs, const vx_c128* factors, bool inverse,
                            const int* perm, const int* items, int n_items, int direct_r, const int* klist,
                            const vx_c128* x, vx_c128* y, vx_c128* work, void* stream) {
  VX_REQUIRE(nx >= 1 && ny >= 1 && nz >= 1 && nrhs >= 1, "bad 2-level apply arguments");
  VX_REQUIRE(direct_r == 1 || direct_r == 2 || direct_r == 4, "direct_r must be 1, 2 or 4");
  cudaStream_t s = as_stream(stream);
  Span span("prec_apply", s);
  FftPlan px, py;
  int st;
  if ((st = fft_get_plan(nx, &px)) || (st = fft_get_plan(ny, &py))) return st;
  double2* S = reinterpret_cast<double2*>(work);
  const long pitch = (long)nx * nrhs;      // x line pitch
  const long plane = (long)ny * pitch;     // (c, z) plane
  const int q3 = 3 * ny * nz;
  {
    LoadStrided ld{reinterpret_cast<const double2*>(x), {pitch, 1, nrhs, nrhs}};
    StoreStrided sv{S, {pitch, 1, nrhs, nrhs}, 1.0};
    if ((st = launch_fft_auto(px, ld, sv, q3 * nrhs, nx, nx, false, nrhs == 1, s))) return st;
  }
  // y-DFT of the (c, z) planes' columns, in place: two-pass register transforms when ny has one
  static const int use_cols2 = env_int("VX_COLS2", 1);
  const bool two_y = use_cols2 && !py.bluestein && py.L == ny && cols2_supported(ny);
  if (two_y) {
    if ((st = launch_cols2<false>(py, S, plane, pitch, ny, S, plane, pitch, ny, 3L * nz * pitch, (int)pitch, 1.0, s)))
      return st;
  } else {
    LoadStrided ld{S, {plane, 1, pitch, (int)pitch}};
    StoreStrided sv{S, {plane, 1, pitch, (int)pitch}, 1.0};
    if ((st = launch_fft_auto(py, ld, sv, 3 * nz * (int)pitch, ny, ny, false, false, s))) return st;
  }
  LuGeom g = lu_geom(3 * nz);
  const double2* F = reinterpret_cast<const double2*>(factors);
  if (!items) n_items = nx * ny;
  if (inverse) {
    VX_REQUIRE(3 * nz <= 32, "explicit block inverses cover 3 nz <= 32 only");
    if ((st = launch_apply_small_inv(3 * nz, F, items, n_items, klist, nrhs, S, plane, nrhs, s))) return st;
  } else if ((st = solve_items(g, F, perm, items, n_items, n_items, klist, nrhs, S, plane, nrhs, s, -1, direct_r))) {
    return st;
  }
  if (two_y) {
    if ((st = launch_cols2<true>(py, S, plane, pitch, ny, S, plane, pitch, ny, 3L * nz * pitch, (int)pitch, 1.0, s)))
      return st;
  } else {
    LoadStrided ld{S, {plane, 1, pitch, (int)pitch}};
    StoreStrided sv{S, {plane, 1, pitch, (int)pitch}, 1.0};
    if ((st = launch_fft_auto(py, ld, sv, 3 * nz * (int)pitch, ny, ny, true, false, s))) return st;
  }
  {
    LoadStrided ld{S, {pitch, 1, nrhs, nrhs}};
    StoreStrided sv{reinterpret_cast<double2*>(y), {pitch, 1, nrhs, nrhs}, 1.0 / ((double)nx * ny)};
    if ((st = launch_fft_auto(px, ld, sv, q3 * nrhs, nx, nx, true, nrhs == 1, s))) return st;
  }
  return VX_OK;
}

extern "C" int vx_prec2_apply(int nx, int ny, int nz, int nrhs, const vx_c128* factors,
                              const int* perm, const int* items, int n_items, int direct_r, const int* klist,
                              const vx_c128* x, vx_c128* y, vx_c128* work, void* stream) {
  return prec2_apply_impl(nx, ny, nz, nrhs, factors, false, perm, items, n_items, direct_r, klist, x, y, work,
                          stream);
}

extern "C" int vx_prec2_apply_inv(int nx, int ny, int nz, int nrhs, const vx_c128* inverses, const int* items,
                                  int n_items, const int* klist, const vx_c128* x, vx_c128* y, vx_c128* work,
                                  void* stream) {
  return prec2_apply_impl(nx, ny, nz, nrhs, inverses, true, nullptr, items, n_items, 1, klist, x, y, work, stream);
}

extern "C" int vx_lu_small_invert(int n, int nslots, const vx_c128* factors, const int* perm, vx_c128* inverses,
                                  void* stream) {
  VX_REQUIRE(n >= 1 && n <= 32 && nslots >= 0, "vx_lu_small_invert: single-tile blocks (n <= 32) only");
  if (nslots == 0) return VX_OK;
  const LuGeom g = lu_geom(n);
  VX_REQUIRE(g.nt == 1, "vx_lu_small_invert: block of %d rows is not a single tile", n);
  const size_t smem = (size_t)SMALL_WARPS * n * n * sizeof(double2);
  if (smem > 48 * 1024)
    VX_CUDA(cudaFuncSetAttribute(lu_small_invert_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  lu_small_invert_kernel<<<div_up(nslots, SMALL_WARPS), SMALL_WARPS * 32, smem, as_stream(stream)>>>(
      n, g.blk, reinterpret_cast<const double2*>(factors), perm, nslots, reinterpret_cast<double2*>(inverses));
  VX_CHECK_LAUNCH("lu_small_invert_kernel");
  return VX_OK;
}

extern "C" int vx_box_gather(int nx, int ny, int nz, int x0, int y0, int z0, int bx, int by, int bz,
                             int nrhs, const vx_c128* full, vx_c128* box, void* stream) {
  const long total = 3L * bx * by * bz * nrhs;
  if (total == 0) return VX_OK;
  box_copy_kernel<<<div_up(total, 256) < 4096 ? div_up(total, 256) : 4096, 256, 0, as_stream(stream)>>>(
      nx, ny, nz, x0, y0, z0, bx, by, bz, nrhs, reinterpret_cast<const double2*>(full),
      reinterpret_cast<double2*>(box), 1);
  VX_CHECK_LAUNCH("box_copy_kernel");
  return VX_OK;
}

extern "C" int vx_box_scatter(int nx, int ny, int nz, int x0, int y0, int z0, int bx, int by, int bz,
                              int nrhs, const vx_c128* box, vx_c128* full, void* stream) {
  const long total = 3L * bx * by * bz * nrhs;
  if (total == 0) return VX_OK;
  box_copy_kernel<<<div_up(total, 256) < 4096 ? div_up(total, 256) : 4096, 256, 0, as_stream(stream)>>>(
      nx, ny, nz, x0, y0, z0, bx, by, bz, nrhs, reinterpret_cast<const double2*>(box),
      reinterpret_cast<double2*>(full), 0);
  VX_CHECK_LAUNCH("box_copy_kernel");
  return VX_OK;
}

extern "C" int vx_solve_variant(int classic) {
  vx::g_solve_classic = classic ? 1 : 0;
  return VX_OK;
}

extern "C" int vx_gather_cols(long nrows, const vx_c128* A, long lda, int P, const int* col_off,
                              const int* colmap, long total_cols, vx_c128* out, void* stream) {
  VX_REQUIRE(nrows >= 0 && P >= 1 && total_cols >= 0, "bad gather_cols arguments");
  const long total = nrows * total_cols;
  if (total == 0) return VX_OK;
  const unsigned g = div_up(total, 256) < 8192 ? div_up(total, 256) : 8192;
  cols_copy_kernel<<<g, 256, 0, as_stream(stream)>>>(nrows, const_cast<double2*>(reinterpret_cast<const double2*>(A)),
                                                     lda, P, col_off, colmap, reinterpret_cast<double2*>(out), 1);
  VX_CHECK_LAUNCH("cols_copy_kernel");
  return VX_OK;
}

extern "C" int vx_scatter_cols(long nrows, const vx_c128* in, int P, const int* col_off, const int* colmap,
                               long total_cols, vx_c128* A, long lda, void* stream) {
  VX_REQUIRE(nrows >= 0 && P >= 1 && total_cols >= 0, "bad scatter_cols arguments");
  const long total = nrows * total_cols;
  if (total == 0) return VX_OK;
  const unsigned g = div_up(total, 256) < 8192 ? div_up(total, 256) : 8192;
  cols_copy_kernel<<<g, 256, 0, as_stream(stream)>>>(nrows, reinterpret_cast<double2*>(A), lda, P, col_off,
                                                     colmap, const_cast<double2*>(reinterpret_cast<const double2*>(in)), 0);
  VX_CHECK_LAUNCH("cols_copy_kernel");
  return VX_OK;
}

extern "C" int vx_prec1_solve(int n, int nrhs, const vx_c128* factors, const int* perm, const int* items,
                              int n_single, int n_items, int direct_r, const int* klist, vx_c128* Y, long s_row,
                              long s_k, void* stream) {
  VX_REQUIRE(n >= 1 && nrhs >= 1 && n_single >= 0 && n_items >= n_single, "bad solve arguments");
  VX_REQUIRE(direct_r == 1 || direct_r == 2, "direct_r must be 1 or 2");
  return solve_items(lu_geom(n), reinterpret_cast<const double2*>(factors), perm, items, n_single, n_items, klist,
                     nrhs, reinterpret_cast<double2*>(Y), s_row, s_k, as_stream(stream), -1, direct_r);
}

// the block products of vx_prec2_apply_inv on a caller-laid-out array (a rank's (3nz, ny*nk) columns)
extern "C" int vx_small_inv_apply(int n, int nrhs, const vx_c128* inverses, const int* items, int n_items,
                                  const int* klist, vx_c128* Y, long s_row, long s_k, void* stream) {
  VX_REQUIRE(n >= 1 && n <= 32 && nrhs >= 1 && n_items >= 0, "bad block-inverse apply arguments");
  return launch_apply_small_inv(n, reinterpret_cast<const double2*>(inverses), items, n_items, klist, nrhs,
                                reinterpret_cast<double2*>(Y), s_row, s_k, as_stream(stream));
}

extern "C" int vx_lu_variant(int monolithic) {
  vx::g_lu_monolithic = monolithic ? 1 : 0;
  return VX_OK;
}

extern "C" long vx_rep_inverse_elems(int n) { return (long)rep_kp(n) * rep_mp(n); }

extern "C" int vx_rep_inverse(int n, const vx_c128* factors, const int* perm, vx_c128* inv, void* stream) {
  VX_REQUIRE(n >= 1, "bad representative-inverse arguments");
  cudaStream_t s = as_stream(stream);
  const int Kp = rep_kp(n), Mp = rep_mp(n);
  double2* A = reinterpret_cast<double2*>(inv);
  VX_CUDA(cudaMemsetAsync(A, 0, sizeof(double2) * (size_t)Kp * Mp, s));
  eye_cols_kernel<<<div_up(n, 256), 256, 0, s>>>(n, Mp, A);
  VX_CHECK_LAUNCH("eye_cols_kernel");
  // column c of D^-1 = solve(D, e_c), stored k-major: A[c*Mp + m]
  const int nit = (n + MULTI_R - 1) / MULTI_R;
  std::vector<int> items(3 * nit), klist(n);
  for (int c = 0; c < n; ++c) klist[c] = c;
  for (int t = 0; t < nit; ++t) {
    items[3 * t] = 0;
    items[3 * t + 1] = t * MULTI_R;
    items[3 * t + 2] = std::min(MULTI_R, n - t * MULTI_R);
  }
  int* dbuf = nullptr;
  VX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dbuf), sizeof(int) * (items.size() + klist.size()), s));
  VX_CUDA(cudaMemcpyAsync(dbuf, items.data(), sizeof(int) * items.size(), cudaMemcpyHostToDevice, s));
  VX_CUDA(cudaMemcpyAsync(dbuf + items.size(), klist.data(), sizeof(int) * n, cudaMemcpyHostToDevice, s));
  int st = solve_items(lu_geom(n), reinterpret_cast<const double2*>(factors), perm, dbuf, 0, nit,
                       dbuf + items.size(), 1, A, 1, Mp, s);
  VX_CUDA(cudaStreamSynchronize(s));  // host item arrays must outlive the copies
  VX_CUDA(cudaFreeAsync(dbuf, s));
  return st;
}

extern "C" long vx_prec1_reduced_work_elems(int nx, int ny, int nz, int nrhs, int n_rep) {
  const int n = 3 * ny * nz;
  const long np = ((long)n_rep * nrhs + RG_N - 1) / RG_N * RG_N;
  return 3L * nx * ny * nz * nrhs + (long)rep_kp(n) * np;
}

extern "C" int vx_prec1_apply_reduced(int nx, int ny, int nz, int nrhs, const vx_c128* factors, const int* perm,
                                      const int* items, int n_single, int direct_r, const int* klist,
                                      const vx_c128* inv,
                                      const int* rep_ks, int n_rep, const vx_c128* x, vx_c128* y,
                                      vx_c128* work, void* stream) {
  VX_REQUIRE(nx >= 1 && ny >= 1 && nz >= 1 && nrhs >= 1 && n_single >= 0 && n_rep >= 0,
             "bad reduced 1-level apply arguments");
  VX_REQUIRE(direct_r == 1 || direct_r == 2, "direct_r must be 1 or 2");
  cudaStream_t s = as_stream(stream);
  Span span("prec_apply", s);
  FftPlan p;
  int st = fft_get_plan(nx, &p);
  if (st) return st;
  const int q3 = 3 * ny * nz;
  double2* S = reinterpret_cast<double2*>(work);
  double2* Bt = S + 3L * nx * ny * nz * nrhs;
  const long pitch = (long)nx * nrhs;
  {
    LoadStrided ld{reinterpret_cast<const double2*>(x), {pitch, 1, nrhs, nrhs}};
    StoreStrided sv{S, {pitch, 1, nrhs, nrhs}, 1.0};
    if ((st = launch_fft_auto(p, ld, sv, q3 * nrhs, nx, nx, false, nrhs == 1, s))) return st;
  }
  LuGeom g = lu_geom(q3);
  const double2* F = reinterpret_cast<const double2*>(factors);
  {
    Span span2("prec_solve", s);
    SideStream* ss = g_rep_sequential ? nullptr : side_stream();
    cudaStream_t sr = ss ? ss->s : s;
    if (ss && n_rep > 0) {
      VX_CUDA(cudaEventRecord(ss->fork, s));
      VX_CUDA(cudaStreamWaitEvent(sr, ss->fork, 0));
    }
    static const int singles_first = env_int("VX_REP_ORDER", 1);
    // VX_REP_PERSIST=k: k single-block solver CTAs per SM (A/B; one CTA per SM
    // cannot keep enough bytes in flight, so the default is the plain grid)
    static const int rep_persist = env_int("VX_REP_PERSIST", 0);
    const int persist = (ss && n_rep > 0) ? rep_persist : -1;
    if (singles_first && n_single > 0 &&
        (st = solve_items(g, F, perm, items, n_single, n_single, klist, nrhs, S, pitch, nrhs, s, persist, direct_r)))
      return st;
    if (n_rep > 0 &&
        (st = rep_gemm(q3, reinterpret_cast<const double2*>(inv), n_rep * nrhs, nrhs, rep_ks, S, pitch, nrhs, Bt, sr)))
      return st;
    if (!singles_first && n_single > 0 &&
        (st = solve_items(g, F, perm, items, n_single, n_single, klist, nrhs, S, pitch, nrhs, s, persist, direct_r)))
      return st;
    if (ss && n_rep > 0) {
      VX_CUDA(cudaEventRecord(ss->join, sr));
      VX_CUDA(cudaStreamWaitEvent(s, ss->join, 0));
    }
  }
  {
    LoadStrided ld{S, {pitch, 1, nrhs, nrhs}};
    StoreStrided sv{reinterpret_cast<double2*>(y), {pitch, 1, nrhs, nrhs}, 1.0 / nx};
    if ((st = launch_fft_auto(p, ld, sv, q3 * nrhs, nx, nx, true, nrhs == 1, s))) return st;
  }
  return VX_OK;
}

extern "C" int vx_rep_variant(int sequential) {
  vx::g_rep_sequential = sequential ? 1 : 0;
  return VX_OK;
}

// ------------------------------------------------------------ sector entries
extern "C" int vx_lu1_build_sec(int nx, int ny, int nz, const vx_c128* lamT, const vx_c128* m_yz, const int* kset,
                                int nk, int nsec, int dmax, const int* rrow, const double* rsc, const int* ccol,
                                const double* cw, vx_c128* factors, int* perm, int* piv, int* info, void* stream) {
  VX_REQUIRE(nx >= 1 && ny >= 1 && nz >= 1 && nk >= 0 && nsec >= 1 && nsec <= 4 && dmax >= 1,
             "bad sector build arguments");
  const int nslots = nk * nsec;
  if (nslots == 0) return VX_OK;
  cudaStream_t s = as_stream(stream);
  Span span("lu_build", s);
  Unfold u{reinterpret_cast<const double2*>(lamT), reinterpret_cast<const double2*>(m_yz), kset,
           6L * (2 * nz - 1) * (2 * ny - 1), nz, ny};
  SecUnfold su{reinterpret_cast<const double2*>(lamT), reinterpret_cast<const double2*>(m_yz), kset,
               6L * (2 * nz - 1) * (2 * ny - 1), nz, ny, nsec, dmax, rrow, rsc, ccol, cw};
  return lu_build_batched(u, lu_geom(dmax), nslots, reinterpret_cast<double2*>(factors), perm, piv, info, s, &su);
}

extern "C" long vx_prec1_sec_work_elems(int nx, int ny, int nz, int nrhs, int nsec, int dmax) {
  return (3L * ny * nz + (long)nsec * dmax) * nx * nrhs;
}

// Representative block of the reduced scheme on sector factors: per sector s
// the frequencies rep_ks are ONE GEMM with the sector block's explicit inverse
// (rep_inv + s * inv_stride, dmax geometry, k-major) on a side stream,
// concurrently with the single-block solves (disjoint spectral columns).
struct SecRep {
  const double2* inv = nullptr;
  long inv_stride = 0;
  const int* ks = nullptr;
  int n = 0;
};

static int prec1_apply_sec(int nx, int ny, int nz, int nrhs, const vx_c128* factors, const int* perm,
                           const int* items, int n_single, int n_items, int direct_r, const int* klist,
                           int nsec, int dmax,
                           int norb, const int* orows, const int* osec, const double* ocoef,
                           const unsigned char* flipk, const vx_c128* x, vx_c128* y, vx_c128* work,
                           void* stream, const RagGeom* rg, const SecRep* rep = nullptr,
                           const SymGeom* sym = nullptr) {
  VX_REQUIRE(nx >= 1 && ny >= 1 && nz >= 1 && nrhs >= 1 && n_single >= 0 && n_items >= n_single && nsec >= 1 &&
                 dmax >= 1,
             "bad sector apply arguments");
  VX_REQUIRE(direct_r == 1 || direct_r == 2, "direct_r must be 1 or 2");
  VX_REQUIRE((long)nsec * dmax * nx < (1L << 29), "sector layout too large for the work-list encoding");
  cudaStream_t s = as_stream(stream);
  Span span("prec_apply", s);
  FftPlan p;
  int st = fft_get_plan(nx, &p);
  if (st) return st;
  const int q = ny * nz, q3 = 3 * q;
  // norb == 0 (symmetric factors of dense blocks only): no orbit transform,
  // the solves run on the x-DFT output itself
  const bool xf = norb > 0;
  VX_REQUIRE(xf || (sym && nsec == 1), "sector apply without orbit tables");
  double2* S = reinterpret_cast<double2*>(work);
  double2* U = xf ? S + (long)q3 * nx * nrhs : S;
  const long pitch = (long)nx * nrhs;
  {
    LoadStrided ld{reinterpret_cast<const double2*>(x), {pitch, 1, nrhs, nrhs}};
    StoreStrided sv{S, {pitch, 1, nrhs, nrhs}, 1.0};
    if ((st = launch_fft_auto(p, ld, sv, q3 * nrhs, nx, nx, false, nrhs == 1, s))) return st;
  }
  // the padding rows of a sector (d_s <= r < dmax) feed the padded solve's
  // identity rows, so they must be zero; the ragged / symmetric solves never read them
  if (!(rg && rg->on) && !sym) VX_CUDA(cudaMemsetAsync(U, 0, sizeof(double2) * (size_t)nsec * dmax * pitch, s));
  if (xf && (st = sec_xform(pitch, nrhs, norb, orows, osec, ocoef, flipk, q, S, U, 0, s))) return st;
  auto singles = [&](int n_it) -> int {
    if (sym) {
      VX_REQUIRE(nrhs == 1, "symmetric factors: single-RHS work lists only");
      Span sp("prec_solve", s);
      if (sym->inverse)
        return launch_symv_inv(*sym, reinterpret_cast<const double2*>(factors), items, n_it, direct_r, klist, U,
                               pitch, nrhs, q, s);
      return launch_solve_sym(*sym, reinterpret_cast<const double2*>(factors), items, n_it, direct_r, klist, U,
                              pitch, nrhs, q, s);
    }
    return solve_items(lu_geom(dmax), reinterpret_cast<const double2*>(factors), perm, items, n_it, n_it, klist,
                       nrhs, U, pitch, nrhs, s, -1, direct_r, rg);
  };
  if (rep && rep->n > 0) {
    Span span2("prec_solve", s);
    SideStream* ss = g_rep_sequential ? nullptr : side_stream();
    cudaStream_t sr = ss ? ss->s : s;
    if (ss) {
      VX_CUDA(cudaEventRecord(ss->fork, s));
      VX_CUDA(cudaStreamWaitEvent(sr, ss->fork, 0));
    }
    double2* Bt = S + (long)q3 * nx * nrhs + (long)nsec * dmax * pitch;
    const long lda = rep_mp(dmax);
    // the sector blocks' products as ONE launch (four separate 207-CTA grids left a third of
    // the 2-CTA/SM slots empty each time)
    VX_REQUIRE(nsec <= 4, "representative GEMM batch holds at most 4 sectors");
    RepBatch rb{};
    rb.nb = nsec;
    rb.bt_stride = (long)rep_kp(dmax) * (((long)rep->n * nrhs + RG_N - 1) / RG_N * RG_N);
    for (int sc = 0; sc < nsec; ++sc) {
      rb.n[sc] = sym ? sym->dims[sc] : (rg && rg->on ? rg->dims[sc] : dmax);
      rb.a_off[sc] = sc * rep->inv_stride;
      rb.s_off[sc] = (long)sc * dmax * pitch;
    }
    if ((st = rep_gemm_batch(rb, rep->inv, rep->n * nrhs, nrhs, rep->ks, U, pitch, nrhs, Bt, sr, lda))) return st;
    if (n_single > 0 && (st = singles(n_single))) return st;
    if (ss) {
      VX_CUDA(cudaEventRecord(ss->join, sr));
      VX_CUDA(cudaStreamWaitEvent(s, ss->join, 0));
    }
  } else if (sym) {
    VX_REQUIRE(n_items == n_single, "symmetric factors: direct items only");
    if ((st = singles(n_single))) return st;
  } else if ((st = solve_items(lu_geom(dmax), reinterpret_cast<const double2*>(factors), perm, items, n_single,
                               n_items, klist, nrhs, U, pitch, nrhs, s, -1, direct_r, rg))) {
    return st;
  }
  if (xf && (st = sec_xform(pitch, nrhs, norb, orows, osec, ocoef, flipk, q, U, S, 1, s))) return st;
  {
    LoadStrided ld{S, {pitch, 1, nrhs, nrhs}};
    StoreStrided sv{reinterpret_cast<double2*>(y), {pitch, 1, nrhs, nrhs}, 1.0 / nx};
    if ((st = launch_fft_auto(p, ld, sv, q3 * nrhs, nx, nx, true, nrhs == 1, s))) return st;
  }
  return VX_OK;
}

extern "C" int vx_prec1_apply_sec(int nx, int ny, int nz, int nrhs, const vx_c128* factors, const int* perm,
                                  const int* items, int n_single, int n_items, int direct_r, const int* klist,
                                  int nsec, int dmax,
                                  int norb, const int* orows, const int* osec, const double* ocoef,
                                  const unsigned char* flipk, const vx_c128* x, vx_c128* y, vx_c128* work,
                                  void* stream) {
  return prec1_apply_sec(nx, ny, nz, nrhs, factors, perm, items, n_single, n_items, direct_r, klist, nsec, dmax,
                         norb, orows, osec, ocoef, flipk, x, y, work, stream, nullptr);
}

extern "C" int vx_prec1_apply_sec_rag(int nx, int ny, int nz, int nrhs, const vx_c128* factors, const int* perm,
                                      const int* items, int n_single, int n_items, int direct_r,
                                      const int* klist, int nsec, int dmax, const int* sec_dims, int norb,
                                      const int* orows, const int* osec, const double* ocoef,
                                      const unsigned char* flipk, const vx_c128* x, vx_c128* y, vx_c128* work,
                                      void* stream) {
  RagGeom rg;
  int st = make_rag(nsec, sec_dims, dmax, &rg);
  if (st) return st;
  return prec1_apply_sec(nx, ny, nz, nrhs, factors, perm, items, n_single, n_items, direct_r, klist, nsec, dmax,
                         norb, orows, osec, ocoef, flipk, x, y, work, stream, &rg);
}

extern "C" long vx_prec1_sec_reduced_work_elems(int nx, int ny, int nz, int nrhs, int nsec, int dmax, int n_rep) {
  const long np = ((long)n_rep * nrhs + RG_N - 1) / RG_N * RG_N;
  return vx_prec1_sec_work_elems(nx, ny, nz, nrhs, nsec, dmax) + (long)nsec * rep_kp(dmax) * np;
}

extern "C" int vx_prec1_apply_sec_reduced(int nx, int ny, int nz, int nrhs, const vx_c128* factors, const int* perm,
                                          const int* items, int n_single, int direct_r, const int* klist, int nsec,
                                          int dmax, const int* sec_dims, int norb, const int* orows, const int* osec,
                                          const double* ocoef, const unsigned char* flipk, const vx_c128* rep_inv,
                                          const int* rep_ks, int n_rep, const vx_c128* x, vx_c128* y, vx_c128* work,
                                          void* stream) {
  VX_REQUIRE(n_rep >= 0 && (n_rep == 0 || (rep_inv && rep_ks)), "bad representative arguments");
  RagGeom rg;
  rg.on = 0;
  if (sec_dims) {
    int st = make_rag(nsec, sec_dims, dmax, &rg);
    if (st) return st;
  }
  SecRep rep;
  rep.inv = reinterpret_cast<const double2*>(rep_inv);
  rep.inv_stride = vx_rep_inverse_elems(dmax);
  rep.ks = rep_ks;
  rep.n = n_rep;
  return prec1_apply_sec(nx, ny, nz, nrhs, factors, perm, items, n_single, n_single, direct_r, klist, nsec, dmax,
                         norb, orows, osec, ocoef, flipk, x, y, work, stream, rg.on ? &rg : nullptr, &rep);
}

// ------------------------------------------------------ symmetric factors
extern "C" int vx_lu1_build_opts(int nx, int ny, int nz, const vx_c128* lamT, const vx_c128* m_yz, const int* kset,
                                 int nk, int nsec, int dmax, const int* rrow, const double* rsc, const int* ccol,
                                 const double* cw, vx_c128* factors, int* perm, int* piv, int* info, int flags,
                                 void* stream) {
  VX_REQUIRE(nx >= 1 && ny >= 1 && nz >= 1 && nk >= 0 && (flags & ~1) == 0, "bad 1-level build arguments");
  cudaStream_t s = as_stream(stream);
  Unfold u{reinterpret_cast<const double2*>(lamT), reinterpret_cast<const double2*>(m_yz), kset,
           6L * (2 * nz - 1) * (2 * ny - 1), nz, ny};
  const int nopiv = flags & 1;
  if (nsec == 0 || !rrow) {
    if (nk == 0) return VX_OK;
    Span span("lu_build", s);
    return lu_build_batched(u, lu_geom(3 * ny * nz), nk, reinterpret_cast<double2*>(factors), perm, piv, info, s,
                            nullptr, nopiv);
  }
  VX_REQUIRE(nsec >= 1 && nsec <= 4 && dmax >= 1, "bad sector build arguments");
  const int nslots = nk * nsec;
  if (nslots == 0) return VX_OK;
  Span span("lu_build", s);
  SecUnfold su{reinterpret_cast<const double2*>(lamT), reinterpret_cast<const double2*>(m_yz), kset,
               6L * (2 * nz - 1) * (2 * ny - 1), nz, ny, nsec, dmax, rrow, rsc, ccol, cw};
  return lu_build_batched(u, lu_geom(dmax), nslots, reinterpret_cast<double2*>(factors), perm, piv, info, s, &su,
                          nopiv);
}

extern "C" long vx_lu_sym_stride(int nsec, const int* sec_dims) {
  long k = 0;
  for (int s = 0; s < nsec; ++s) k += sym_size(sec_dims[s]);
  return k;
}

extern "C" int vx_lu_sym_pack(int nkslots, int nsec, int dmax, const int* sec_dims, const vx_c128* padded,
                              const vx_c128* w, vx_c128* sym, vx_c128* h, double* dev, void* stream) {
  VX_REQUIRE(nkslots >= 0, "bad symmetric pack arguments");
  SymGeom sg;
  int st = make_sym(nsec, sec_dims, dmax, h, w, &sg);
  if (st) return st;
  if (nkslots == 0) return VX_OK;
  const LuGeom g = lu_geom(dmax);
  lu_sym_pack_kernel<<<nkslots * nsec, 256, 0, as_stream(stream)>>>(g, sg, reinterpret_cast<const double2*>(padded),
                                                                   reinterpret_cast<double2*>(sym),
                                                                   reinterpret_cast<double2*>(h), dev);
  VX_CHECK_LAUNCH("lu_sym_pack_kernel");
  return VX_OK;
}

extern "C" int vx_lu_sym_unpack(int nkslots, int nsec, int dmax, const int* sec_dims, const vx_c128* sym,
                                const vx_c128* h, const vx_c128* w, vx_c128* padded, void* stream) {
  VX_REQUIRE(nkslots >= 0, "bad symmetric unpack arguments");
  SymGeom sg;
  int st = make_sym(nsec, sec_dims, dmax, h, w, &sg);
  if (st) return st;
  if (nkslots == 0) return VX_OK;
  const LuGeom g = lu_geom(dmax);
  lu_sym_unpack_kernel<<<nkslots * nsec, 256, 0, as_stream(stream)>>>(g, sg, reinterpret_cast<const double2*>(sym),
                                                            reinterpret_cast<double2*>(padded));
  VX_CHECK_LAUNCH("lu_sym_unpack_kernel");
  return VX_OK;
}

extern "C" int vx_prec1_apply_sym(int nx, int ny, int nz, const vx_c128* factors, const vx_c128* h,
                                  const vx_c128* w, const int* items, int n_single, int direct_r, const int* klist,
                                  int nsec, int dmax, const int* sec_dims, int norb, const int* orows,
                                  const int* osec, const double* ocoef, const unsigned char* flipk,
                                  const vx_c128* rep_inv, const int* rep_ks, int n_rep, const vx_c128* x,
                                  vx_c128* y, vx_c128* work, void* stream) {
  VX_REQUIRE(n_rep >= 0 && (n_rep == 0 || (rep_inv && rep_ks)), "bad representative arguments");
  SymGeom sg;
  int st = make_sym(nsec, sec_dims, dmax, h, w, &sg);
  if (st) return st;
  SecRep rep;
  rep.inv = reinterpret_cast<const double2*>(rep_inv);
  rep.inv_stride = vx_rep_inverse_elems(dmax);
  rep.ks = rep_ks;
  rep.n = n_rep;
  return prec1_apply_sec(nx, ny, nz, 1, factors, nullptr, items, n_single, n_single, direct_r, klist, nsec, dmax,
                         norb, orows, osec, ocoef, flipk, x, y, work, stream, nullptr, n_rep ? &rep : nullptr, &sg);
}

// vx_lu_sym_invert: G = (L^-1 W)^T diag(h) (L^-1 W), the lower triangle of the
// symmetric inverse A^^-1 of every block, from the symmetric factors (scratch:
// another buffer of the same size, holds L^-1 afterwards).
extern "C" int vx_lu_sym_invert(int nkslots, int nsec, int dmax, const int* sec_dims, const vx_c128* sym,
                                const vx_c128* h, const vx_c128* w, vx_c128* scratch, vx_c128* ginv, void* stream) {
  VX_REQUIRE(nkslots >= 0 && sym && scratch && ginv, "bad symmetric inverse arguments");
  SymGeom sg;
  int st = make_sym(nsec, sec_dims, dmax, h, w, &sg);
  if (st) return st;
  if (nkslots == 0) return VX_OK;
  Span span("lu_build", as_stream(stream));
  lu_sym_invert_kernel<<<nkslots * nsec, 256, 0, as_stream(stream)>>>(
      sg, reinterpret_cast<const double2*>(sym), reinterpret_cast<double2*>(scratch),
      reinterpret_cast<double2*>(ginv));
  VX_CHECK_LAUNCH("lu_sym_invert_kernel");
  return VX_OK;
}

// vx_prec1_apply_syminv: vx_prec1_apply_sym with the block solves replaced by
// x = G (b / W) on the stored symmetric inverses (one streaming pass).
extern "C" int vx_prec1_apply_syminv(int nx, int ny, int nz, const vx_c128* ginv, const vx_c128* w,
                                     const int* items, int n_single, int direct_r, const int* klist, int nsec,
                                     int dmax, const int* sec_dims, int norb, const int* orows, const int* osec,
                                     const double* ocoef, const unsigned char* flipk, const vx_c128* rep_inv,
                                     const int* rep_ks, int n_rep, const vx_c128* x, vx_c128* y, vx_c128* work,
                                     void* stream) {
  VX_REQUIRE(n_rep >= 0 && (n_rep == 0 || (rep_inv && rep_ks)), "bad representative arguments");
  SymGeom sg;
  int st = make_sym(nsec, sec_dims, dmax, nullptr, w, &sg);
  if (st) return st;
  sg.inverse = 1;
  SecRep rep;
  rep.inv = reinterpret_cast<const double2*>(rep_inv);
  rep.inv_stride = vx_rep_inverse_elems(dmax);
  rep.ks = rep_ks;
  rep.n = n_rep;
  return prec1_apply_sec(nx, ny, nz, 1, ginv, nullptr, items, n_single, n_single, direct_r, klist, nsec, dmax,
                         norb, orows, osec, ocoef, flipk, x, y, work, stream, nullptr, n_rep ? &rep : nullptr, &sg);
}

// Solve-only sector path on a caller-owned spectral array (the sharded
// preconditioner's received frequency columns, dist.py): S (3q rows x pitch
// columns) -> orbit transform -> ragged sector block solves -> back into S.
// U: nsec * dmax * pitch scratch.  Same work-list / flip conventions as
// vx_prec1_apply_sec_rag with nx replaced by the column pitch.
extern "C" int vx_prec1_solve_sec_rag(int ny, int nz, long pitch, const vx_c128* factors, const int* perm,
                                      const int* items, int n_single, int n_items, int direct_r,
                                      const int* klist, int nsec, int dmax, const int* sec_dims, int norb,
                                      const int* orows, const int* osec, const double* ocoef,
                                      const unsigned char* flipk, vx_c128* S, vx_c128* U, void* stream) {
  RagGeom rg;
  int st = make_rag(nsec, sec_dims, dmax, &rg);
  if (st) return st;
  VX_REQUIRE(ny >= 1 && nz >= 1 && pitch >= 1 && n_single >= 0 && n_items >= n_single, "bad sector solve arguments");
  VX_REQUIRE(direct_r == 1 || direct_r == 2, "direct_r must be 1 or 2");
  VX_REQUIRE((long)nsec * dmax * pitch < (1L << 29), "sector layout too large for the work-list encoding");
  cudaStream_t s = as_stream(stream);
  Span span("prec_apply", s);
  const int q = ny * nz;
  double2* Sd = reinterpret_cast<double2*>(S);
  double2* Ud = reinterpret_cast<double2*>(U);
  if ((st = sec_xform(pitch, 1, norb, orows, osec, ocoef, flipk, q, Sd, Ud, 0, s))) return st;
  if ((st = solve_items(lu_geom(dmax), reinterpret_cast<const double2*>(factors), perm, items, n_single, n_items,
                        klist, 1, Ud, pitch, 1, s, -1, direct_r, &rg)))
    return st;
  return sec_xform(pitch, 1, norb, orows, osec, ocoef, flipk, q, Ud, Sd, 1, s);
}

// vx_prec1_solve_syminv: the same solve-only path on the symmetric inverses
// (vx_lu_sym_invert): orbit transform -> x = G (b / W) per sector block -> back.
extern "C" int vx_prec1_solve_syminv(int ny, int nz, long pitch, const vx_c128* ginv, const vx_c128* w,
                                     const int* items, int n_single, int direct_r, const int* klist, int nsec,
                                     int dmax, const int* sec_dims, int norb, const int* orows, const int* osec,
                                     const double* ocoef, const unsigned char* flipk, vx_c128* S, vx_c128* U,
                                     void* stream) {
  SymGeom sg;
  int st = make_sym(nsec, sec_dims, dmax, nullptr, w, &sg);
  if (st) return st;
  sg.inverse = 1;
  VX_REQUIRE(ny >= 1 && nz >= 1 && pitch >= 1 && n_single >= 0, "bad sector solve arguments");
  VX_REQUIRE(direct_r == 1 || direct_r == 2, "direct_r must be 1 or 2");
  VX_REQUIRE((long)nsec * dmax * pitch < (1L << 29), "sector layout too large for the work-list encoding");
  cudaStream_t s = as_stream(stream);
  Span span("prec_apply", s);
  const int q = ny * nz;
  double2* Sd = reinterpret_cast<double2*>(S);
  double2* Ud = reinterpret_cast<double2*>(U);
  if ((st = sec_xform(pitch, 1, norb, orows, osec, ocoef, flipk, q, Sd, Ud, 0, s))) return st;
  {
    Span sp("prec_solve", s);
    if ((st = launch_symv_inv(sg, reinterpret_cast<const double2*>(ginv), items, n_single, direct_r, klist, Ud, pitch,
                              1, q, s)))
      return st;
  }
  return sec_xform(pitch, 1, norb, orows, osec, ocoef, flipk, q, Ud, Sd, 1, s);
}

extern "C" long vx_lu_rag_stride(int nsec, const int* sec_dims) {
  long k = 0;
  for (int s = 0; s < nsec; ++s) k += (long)sec_dims[s] * sec_dims[s];
  return k;
}

extern "C" int vx_lu_repack(int nkslots, int nsec, int dmax, const int* sec_dims, const vx_c128* padded,
                            vx_c128* ragged, void* stream) {
  VX_REQUIRE(nkslots >= 0, "bad repack arguments");
  RagGeom rg;
  int st = make_rag(nsec, sec_dims, dmax, &rg);
  if (st) return st;
  if (nkslots == 0) return VX_OK;
  const LuGeom g = lu_geom(dmax);
  VX_REQUIRE(g.nt > 1, "ragged storage is for multi-tile blocks (dmax > 32)");
  const long per = (long)dmax * dmax;
  dim3 grid(div_up(per, 256 * 4) > 0 ? div_up(per, 256 * 4) : 1, nkslots * nsec);
  lu_repack_kernel<<<grid, 256, 0, as_stream(stream)>>>(g, rg, reinterpret_cast<const double2*>(padded),
                                                        reinterpret_cast<double2*>(ragged));
  VX_CHECK_LAUNCH("lu_repack_kernel");
  return VX_OK;
}

extern "C" int vx_prec1_apply(int nx, int ny, int nz, int nrhs, const vx_c128* factors,
                              const int* perm, const int* items, int n_single, int n_items, int direct_r,
                              const int* klist, const vx_c128* x, vx_c128* y, vx_c128* work,
                              void* stream) {
  return prec1_apply(nx, ny, nz, nrhs, factors, perm, items, n_single, n_items, direct_r, klist, x, y, work,
                     stream, nullptr);
}

extern "C" int vx_prec1_apply_rag(int nx, int ny, int nz, int nrhs, const vx_c128* factors,
                                  const int* perm, const int* items, int n_single, int n_items, int direct_r,
                                  const int* klist, const vx_c128* x, vx_c128* y, vx_c128* work,
                                  void* stream) {
  RagGeom rg;
  const int d = 3 * ny * nz;
  int st = make_rag(1, &d, d, &rg);
  if (st) return st;
  return prec1_apply(nx, ny, nz, nrhs, factors, perm, items, n_single, n_items, direct_r, klist, x, y, work,
                     stream, &rg);
}

extern "C" int vx_lu_unpack(int nkslots, int nsec, int dmax, const int* sec_dims, const vx_c128* ragged,
                            vx_c128* padded, void* stream) {
  VX_REQUIRE(nkslots >= 0, "bad unpack arguments");
  RagGeom rg;
  int st = make_rag(nsec, sec_dims, dmax, &rg);
  if (st) return st;
  if (nkslots == 0) return VX_OK;
  const LuGeom g = lu_geom(dmax);
  VX_REQUIRE(g.nt > 1, "ragged storage is for multi-tile blocks (dmax > 32)");
  dim3 grid(div_up(g.blk, 256 * 4) > 0 ? div_up(g.blk, 256 * 4) : 1, nkslots * nsec);
  lu_unpack_kernel<<<grid, 256, 0, as_stream(stream)>>>(g, rg, reinterpret_cast<const double2*>(ragged),
                                                        reinterpret_cast<double2*>(padded));
  VX_CHECK_LAUNCH("lu_unpack_kernel");
  return VX_OK;
}

extern "C" int vx_solve_classic(void) { return vx::g_solve_classic; }
