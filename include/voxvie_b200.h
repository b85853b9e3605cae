/*
 * voxvie_b200 -- C-ABI of the B200-native hot path of the circulant-
 * preconditioned voxel VIE (arXiv 1903.07884; reference package `voxvie`).
 *
 * Every array argument is a DEVICE pointer to interleaved complex128
 * (vx_c128, 16 bytes) or int32, owned by the caller; every call is
 * asynchronous on the given CUDA stream (`stream` = cudaStream_t, NULL =
 * legacy default).  Calls return a status:
 *
 *   VX_OK 0  |  VX_EINVAL 1 -> ValueError  |  VX_ESINGULAR 2 -> PreconditionerBuildError
 *   VX_ECAP 3 -> PreconditionerBuildError  |  VX_ECUDA 4  |  VX_ENCCL 5
 *
 * and vx_last_error() returns a thread-local message for the last failure.
 *
 * Layouts (reference grid.py:1-9): fields are (3, nz, ny, nx) C-order, x
 * fastest; the generating tensors are (6, 2nz-1, 2ny-1, 2nx-1) ordered
 * xx,xy,xz,yy,yz,zz (reference kernel.py:119-141, accel.py:38-41).
 *
 * Each entry point names the reference interface it replaces.
 */
#ifndef VOXVIE_B200_H
#define VOXVIE_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VX_ABI_VERSION 1

#define VX_OK 0
#define VX_EINVAL 1
#define VX_ESINGULAR 2
#define VX_ECAP 3
#define VX_ECUDA 4
#define VX_ENCCL 5

typedef struct vx_c128 { double re, im; } vx_c128;

const char* vx_last_error(void);
int vx_version(void);

/* ------------------------------------------------------------------ FFT */
/* 13-smooth length >= n (operator padding), and smoothness test. */
int vx_fft_good_length(int n);
int vx_fft_is_smooth(int n);

/* Batched strided 1-D DFT, scipy convention (forward unnormalised, inverse
 * scaled by `scale`): line l = (o, i), o = l / n_inner, i = l % n_inner,
 * element e at base + o*os + i*is + e*es.  Input read for e < n_in (zero
 * padded to n), output written for e < n_out.  Used by every transform below;
 * exported for the FFT parity tests (scipy.fft.fft on strided axes). */
int vx_fft_lines(int n, int n_lines, int n_inner, const vx_c128* in, long in_os, long in_is,
                 long in_es, int n_in, vx_c128* out, long out_os, long out_is, long out_es,
                 int n_out, int inverse, double scale, void* stream);

/* ------------------------------------------------------------- operator */
/* Replaces operator.plan_operator (operator.py:61-70): spectra (6, pz, py, px)
 * of the generators embedded in their (pz, py, px) circulant extension
 * (operator.py:21-41; any p >= 2n-1 gives the same matvec).  gen strides are
 * in elements for axes (component, z, y, x). */
int vx_op_plan(int nx, int ny, int nz, int px, int py, int pz, const vx_c128* gen, long g_sp,
               long g_sz, long g_sy, long g_sx, vx_c128* spectra, void* stream);

/* Padded FFT length used per axis by the operator plan: 2n when 2n is 7-smooth,
 * else the smallest 7-smooth length >= 2n-1. */
int vx_op_padded_length(int n);

/* Padded z length: vx_op_padded_length(nz), or with VX_ZPAIR=1 (opt-in
 * paired-parity z kernel, nz <= 16) the reference's own 2 nz
 * (operator.py:21-41 embeds on 2n). */
int vx_op_padded_length_z(int nz);

/* Scratch (in vx_c128 elements) needed by vx_op_apply. */
long vx_op_work_elems(int nx, int ny, int nz, int px, int py, int pz);

/* Replaces operator.apply_n / apply_system (operator.py:82-105):
 * y = N x (m == NULL) or y = x - m .* (N x), m of shape (nz, ny, nx).
 * compact = 1: spectra in the symmetry-reduced layout of vx_op_compact. */
int vx_op_apply(int nx, int ny, int nz, int px, int py, int pz, const vx_c128* spectra, int compact,
                const vx_c128* m, const vx_c128* x, vx_c128* y, vx_c128* work, void* stream);

/* Parity-symmetric kernels (every Green component even/odd in each offset
 * coordinate, reference kernel.py:37-51) have spectra with S_p(-k) = +-S_p(k):
 * vx_gen_asymmetry writes per-CTA quadruples (max |t(d) - s_x t(d mirrored in x)|,
 * the same for y and for z, max |t|) (256 CTAs -> 1024 doubles); the x (and y)
 * parity also lets the preconditioners share one factor between the frequency
 * blocks k and n-k (vx_prec1_apply's KFLIP flags); vx_op_compact keeps the k <= P/2 half-octant
 * (6, pz/2+1, py/2+1, px/2+1) of full spectra. */
int vx_gen_asymmetry(int nx, int ny, int nz, const vx_c128* gen, long g_sp, long g_sz, long g_sy, long g_sx,
                     double* out, void* stream);
long vx_op_compact_elems(int px, int py, int pz);
int vx_op_compact(int px, int py, int pz, const vx_c128* full, vx_c128* compact, void* stream);

/* --------------------------------------------------- 1-level preconditioner */
/* Replaces circulant._chan_x_spectra (circulant.py:129-136): lamT (nx, 6, 2nz-1, 2ny-1),
 * k-major, = fft_x(chan_x(gen)) transposed so block k's generators are contiguous. */
int vx_chan_x_spectra(int nx, int ny, int nz, const vx_c128* gen, long g_sp, long g_sz, long g_sy,
                      long g_sx, vx_c128* lamT, void* stream);

/* Proxies (circulant.py:99-110, 328-332): proxy[k] = (ny*nz==1) - m00 * lamT[k,0,0,0]. */
int vx_proxy(int nx, int ny, int nz, const vx_c128* lamT, vx_c128 m00, vx_c128* proxy, void* stream);

/* Tile geometry used for the stored factors of an n x n block. */
int vx_lu_tile(int n);
long vx_lu_block_elems(int n);   /* complex entries per stored block (padded tiles) */

/* Replaces the unfold + lu_factor loop of build_one_level / build_reduced_one_level
 * (circulant.py:216-224, 341-343; accel.py:157-179): for slot s, block k = kset[s]:
 * D = I - diag(m_yz) N_k assembled straight into tiled storage and factorised with
 * partial pivoting (zgetrf semantics, pivot = argmax |Re|+|Im|).  Writes factors,
 * row permutation perm (n per slot, composed from the LAPACK pivots), piv
 * (LAPACK ipiv, 0-based) and info[s] (0 ok, j+1 = first zero pivot column). */
int vx_lu1_build(int nx, int ny, int nz, const vx_c128* lamT, const vx_c128* m_yz, const int* kset,
                 int nslots, vx_c128* factors, int* perm, int* piv, int* info, void* stream);

/* Replaces OneLevelPrec.apply / ReducedOneLevelPrec.apply (circulant.py:162-188,
 * 264-269): y = F_x^-1 blockdiag(D_k^-1) F_x x for x of shape (3N, nrhs).
 * Work list: item t solves slot items[3t] for the frequencies
 * klist[items[3t+1] .. items[3t+1]+items[3t+2]); items [0, n_single) are
 * direct items with up to direct_r (1 or 2) frequencies each, items
 * [n_single, n_items) up to 16 (representative block).  A klist entry is the
 * frequency k in bits 0-28, plus VX_KFLIP_X (bit 30) when block k is the
 * x-mirror of the stored one (x-parity-symmetric kernels: D_{nx-k} = S D_k S,
 * S = -1 on the x-component rows) and VX_KFLIP_Y (bit 29, 2-level) for the
 * y-mirror; the solve is then y = S D^-1 S b with the stored factors. */
#define VX_KFLIP_X (1 << 30)
#define VX_KFLIP_Y (1 << 29)
long vx_prec1_work_elems(int nx, int ny, int nz, int nrhs);
int vx_prec1_apply(int nx, int ny, int nz, int nrhs, const vx_c128* factors, const int* perm,
                   const int* items, int n_single, int n_items, int direct_r, const int* klist,
                   const vx_c128* x, vx_c128* y, vx_c128* work, void* stream);

/* Reduced scheme, representative block (ReducedOneLevelPrec.apply,
 * circulant.py:264-269, which calls lu_solve with the representative factor
 * for every discarded frequency): vx_rep_inverse forms the explicit inverse of
 * the representative block from its factors, k-major and zero padded
 * (vx_rep_inverse_elems entries); vx_prec1_apply_reduced then solves items
 * [0, n_single) (one frequency each) with the factors and the n_rep
 * frequencies rep_ks with one FP64 tensor-core GEMM against that inverse, on
 * a side stream concurrently with the single-block solves.  work holds
 * vx_prec1_reduced_work_elems entries.  vx_rep_variant(1) runs the GEMM on
 * the caller's stream (A/B timing). */
long vx_rep_inverse_elems(int n);
int vx_rep_inverse(int n, const vx_c128* factors, const int* perm, vx_c128* inv, void* stream);
long vx_prec1_reduced_work_elems(int nx, int ny, int nz, int nrhs, int n_rep);
int vx_prec1_apply_reduced(int nx, int ny, int nz, int nrhs, const vx_c128* factors, const int* perm,
                           const int* items, int n_single, int direct_r, const int* klist, const vx_c128* inv,
                           const int* rep_ks, int n_rep, const vx_c128* x, vx_c128* y, vx_c128* work,
                           void* stream);
int vx_rep_variant(int sequential);

/* Symmetry sectors (paper_1903_07884_b200/sectors.py): when the kernel has y
 * (z) parity and m_yz is mirror-symmetric in y (z), every D_k commutes with
 * the reflections and is block-diagonal in their joint eigenbasis (2 or 4
 * sectors of <= dmax rows).  vx_lu1_build_sec factorises slot kslot*nsec + s =
 * sector s of block kset[kslot] (unfold tables rrow/rsc (nsec, dmax) and
 * ccol/cw (nsec, dmax, 4), see sectors.py).  vx_prec1_apply_sec = x-DFT,
 * orbit transform to sector coordinates U (nsec*dmax rows; orbit tables
 * orows/osec (norb, 4), ocoef (norb, 4, 4); flipk[k] != 0 applies the x-mirror
 * sign of a shared factor), the block solves (klist entries s*dmax*nx + k, no
 * flags), the inverse transform and the inverse x-DFT.  Same result as
 * vx_prec1_apply on the unreduced blocks up to rounding. */
int vx_lu1_build_sec(int nx, int ny, int nz, const vx_c128* lamT, const vx_c128* m_yz, const int* kset, int nk,
                     int nsec, int dmax, const int* rrow, const double* rsc, const int* ccol, const double* cw,
                     vx_c128* factors, int* perm, int* piv, int* info, void* stream);
long vx_prec1_sec_work_elems(int nx, int ny, int nz, int nrhs, int nsec, int dmax);
int vx_prec1_apply_sec(int nx, int ny, int nz, int nrhs, const vx_c128* factors, const int* perm,
                       const int* items, int n_single, int n_items, int direct_r, const int* klist,
                       int nsec, int dmax,
                       int norb, const int* orows, const int* osec, const double* ocoef,
                       const unsigned char* flipk, const vx_c128* x, vx_c128* y, vx_c128* work, void* stream);

/* Operator y / z passes: 1 (default) = register-resident column FFTs for the
 * padded lengths that have them (fft_reg.cuh), 0 = shared-memory line engine
 * only (A/B timing and cross-checks). */
int vx_op_reg_fft(int on);

/* Select the factorisation: 0 (default) = step-batched kernels (unfold, then per
 * tile column: panel / interchanges / U row / DMMA trailing update over all
 * blocks), 1 = one CTA per block for the whole LU (A/B timing). */
int vx_lu_variant(int monolithic);

/* Select the block-solve kernel: 0 (default) = TMA-bulk pipelined producer/
 * consumer kernel, 1 = the classic synchronous kernel (kept for A/B timing). */
int vx_solve_variant(int classic);

/* --------------------------------------------------- 2-level preconditioner */
/* circulant.py:434-435: lam2T (ny*nx, 6, 2nz-1) = fftn_{y,x}(chan_y(chan_x(gen))). */
long vx_chan_xy_work_elems(int nx, int ny, int nz);
int vx_chan_xy_spectra(int nx, int ny, int nz, const vx_c128* gen, long g_sp, long g_sz, long g_sy,
                       long g_sx, vx_c128* lam2T, vx_c128* work, void* stream);
/* circulant.py:436-446 + accel.py:181-197: (3nz)^2 blocks; slot s factors block
 * kset[s] = l*nx + k (kset NULL: all nx*ny blocks in order). */
int vx_lu2_build(int nx, int ny, int nz, const vx_c128* lam2T, const vx_c128* m_z, const int* kset,
                 int nslots, vx_c128* factors, int* perm, int* piv, int* info, void* stream);
/* TwoLevelPrec.apply (circulant.py:379-394).  items/klist as vx_prec1_apply
 * (frequency = l*nx + k; direct_r 1, 2 or 4 for the x/y mirror orbits);
 * items NULL: slot b solves block b. */
long vx_prec2_work_elems(int nx, int ny, int nz, int nrhs);
int vx_prec2_apply(int nx, int ny, int nz, int nrhs, const vx_c128* factors, const int* perm,
                   const int* items, int n_items, int direct_r, const int* klist,
                   const vx_c128* x, vx_c128* y, vx_c128* work, void* stream);
/* The same apply on explicit block inverses (3 nz <= 32): vx_lu_small_invert
 * turns the packed factors of vx_lu2_build into G = A^-1, column-major
 * (n, n) per slot, and vx_prec2_apply_inv replaces the two triangular
 * products of TwoLevelPrec.apply's lu_solve (circulant.py:388-390) by one
 * streaming product per block. */
int vx_lu_small_invert(int n, int nslots, const vx_c128* factors, const int* perm, vx_c128* inverses,
                       void* stream);
int vx_prec2_apply_inv(int nx, int ny, int nz, int nrhs, const vx_c128* inverses, const int* items,
                       int n_items, const int* klist, const vx_c128* x, vx_c128* y, vx_c128* work,
                       void* stream);

/* ------------------------------------------------------ sharded (multi-GPU) */
/* Pieces of vx_op_apply for the x-slab/line-sharded matvec:
 * forward x-DFT of local lines, the y/z work on the locally owned x-frequency
 * columns (A is (3, nz, ny, nkx), spectra (6, pz, py, nkx)), inverse x-DFT +
 * epilogue of local lines (global line offset line0 for the medium map). */
int vx_op_x_forward(int nx, int px, int nlines, const vx_c128* x, vx_c128* A, void* stream);
long vx_op_yz_work_elems(int ny, int nz, int nkx, int py);
int vx_op_yz(int ny, int nz, int nkx, int px, int py, int pz, const vx_c128* spectra_local, vx_c128* A,
             vx_c128* work, void* stream);
/* vx_op_yz on a rank's spectra compacted in y and z (vx_spec_compact_yz: the
 * k <= P/2 halves of a parity-symmetric kernel's spectra, every local kx kept:
 * (pz/2+1, py/2+1, nkx, 6), vx_spec_compact_yz_elems entries) -- a quarter of
 * the bytes of the slice vx_op_yz reads (operator.py:87-97 on a rank's columns). */
int vx_op_yz_compact(int ny, int nz, int nkx, int px, int py, int pz, const vx_c128* spectra_cyz, vx_c128* A,
                     vx_c128* work, void* stream);
long vx_spec_compact_yz_elems(int nkx, int py, int pz);
int vx_spec_compact_yz(int nkx, int py, int pz, const vx_c128* full, vx_c128* compact, void* stream);
int vx_op_x_inverse(int nx, int ny, int nz, int px, int nlines, long line0, const vx_c128* A,
                    const vx_c128* m, const vx_c128* x_local, vx_c128* y_local, void* stream);
/* All-to-all pack/unpack: out = concat_s A[:, colmap[col_off[s]:col_off[s+1]]]. */
int vx_gather_cols(long nrows, const vx_c128* A, long lda, int P, const int* col_off, const int* colmap,
                   long total_cols, vx_c128* out, void* stream);
int vx_scatter_cols(long nrows, const vx_c128* in, int P, const int* col_off, const int* colmap,
                    long total_cols, vx_c128* A, long lda, void* stream);
/* Block solves only (no DFTs): RHS element (row, k, j) at Y[row*s_row + k*s_k + j]. */
int vx_prec1_solve(int n, int nrhs, const vx_c128* factors, const int* perm, const int* items,
                   int n_single, int n_items, int direct_r, const int* klist, vx_c128* Y, long s_row,
                   long s_k, void* stream);
/* The same call on explicit single-tile inverses (vx_lu_small_invert), n <= 32:
 * a rank's share of TwoLevelPrec.apply's block solves (circulant.py:388-390). */
int vx_small_inv_apply(int n, int nrhs, const vx_c128* inverses, const int* items, int n_items,
                       const int* klist, vx_c128* Y, long s_row, long s_k, void* stream);
/* Local halves of one classical Gram-Schmidt pass (the all-reduce goes in
 * between): out[0..nvec) = V^H w, out[nvec] = ||w||^2; then w -= V coef and
 * out_norm2 = ||w||^2. */
int vx_cgs_dots(long n, int nvec, const vx_c128* V, long ldv, const vx_c128* w, vx_c128* out,
                vx_c128* part, void* stream);
int vx_cgs_update(long n, int nvec, const vx_c128* V, long ldv, const vx_c128* coef, vx_c128* w,
                  vx_c128* out_norm2, vx_c128* part, void* stream);
/* The same stages with the DGKS decision on the device (the sharded solver's
 * device-driven step, dist.py): vx_dgks_ctl turns the all-reduced ||w0||^2,
 * ||w1||^2 into ctl = (||w0||, ||w1||, fired, .) (reference solver.py:69-73);
 * vx_cgs_dots_cond / vx_cgs_update_cond run (and return zeros otherwise) only
 * when ctl[2] is set; vx_dgks_finish forms the Hessenberg column h = d (+ c),
 * h[nvec] = ctl[3] = the final norm; vx_scale_dev is v = w / hn.re with the
 * scalar on the device (reference solver.py:77). */
int vx_cgs_dots_cond(long n, int nvec, const vx_c128* V, long ldv, const vx_c128* w, vx_c128* out, vx_c128* part,
                     const double* ctl, void* stream);
int vx_cgs_update_cond(long n, int nvec, const vx_c128* V, long ldv, const vx_c128* coef, vx_c128* w,
                       vx_c128* out_norm2, vx_c128* part, const double* ctl, void* stream);
int vx_dgks_ctl(const vx_c128* n0sq, const vx_c128* n1sq, double* ctl, void* stream);
int vx_dgks_finish(int nvec, const vx_c128* d, const vx_c128* c, const vx_c128* n2sq, double* ctl, vx_c128* hcol,
                   void* stream);
int vx_scale_dev(long n, const vx_c128* w, vx_c128* out, const vx_c128* hn, void* stream);

/* --------------------------------------------------------------- blocked */
/* BlockedPrec.apply gather/scatter (circulant.py:558-563, 603-607): box
 * (x0,y0,z0) of size (bx,by,bz) inside the (nx,ny,nz) grid, nrhs columns. */
int vx_box_gather(int nx, int ny, int nz, int x0, int y0, int z0, int bx, int by, int bz, int nrhs,
                  const vx_c128* full, vx_c128* box, void* stream);
int vx_box_scatter(int nx, int ny, int nz, int x0, int y0, int z0, int bx, int by, int bz, int nrhs,
                   const vx_c128* box, vx_c128* full, void* stream);

/* ---------------------------------------------------------------- GMRES */
/* Arnoldi orthogonalisation of solver._gmres_cycle (solver.py:62-77) as
 * classical Gram-Schmidt with the reference's DGKS criterion
 * (||w1|| < 0.7071 ||w0|| -> second pass).  Deterministic fixed-order
 * reductions.  V holds nvec = j+1 basis vectors of length n at stride ldv;
 * w is orthogonalised in place and written (normalised) to V[j+1] when
 * `vnext` is non-null.  hout receives j+2 complex: h_0..h_j, h_{j+1} = ||w||;
 * stats receives (||w0||, ||w1||, reorth flag).  part: scratch of
 * vx_arnoldi_part_elems(n, nvec) entries. */
long vx_arnoldi_part_elems(long n, int nvec);
int vx_arnoldi_step(long n, int nvec, const vx_c128* V, long ldv, vx_c128* w, vx_c128* vnext,
                    vx_c128* hout, double* stats, vx_c128* part, void* stream);
/* solver.py:110 -- u = sum_i y_i V_i. */
int vx_basis_combine(long n, int nvec, const vx_c128* V, long ldv, const vx_c128* y, vx_c128* u,
                     void* stream);
/* The same with the basis vectors given by a device array of nvec pointers
 * (each a (n,) complex128 vector): GMRES keeps z_j = P^-1 v_j where the
 * preconditioner wrote it (reference solver.py:106-110, 160-161). */
int vx_basis_combine_ptrs(long n, int nvec, const void* zptrs, const vx_c128* y, vx_c128* u, void* stream);
/* Vector helpers: out = a*x + b*y ; norm2 -> dots[0].re (deterministic). */
int vx_axpby(long n, vx_c128 a, const vx_c128* x, vx_c128 b, const vx_c128* y, vx_c128* out,
             void* stream);
int vx_norm2(long n, const vx_c128* x, double* out, vx_c128* part, void* stream);

/* -------------------------------------------------------------- runtime */
/* Number of kernels this library has launched since it was loaded. */
long vx_launch_count(void);
/* Named CUDA-event spans recorded on the launching stream while enabled:
 * "op_apply", "prec_apply", "prec_solve" (the factor-streaming solve kernel),
 * "arnoldi_step", "lu_build".  vx_timing_read synchronises on the recorded
 * events, returns their summed duration and count, and clears them. */
int vx_timing_enable(int on);
int vx_timing_read(const char* span, double* total_ms, long* count);

/* Generating tensors assembled on the device (replaces the host assembly of
 * reference kernel.py:152-198 / accel.py:131-155): out = (6, 2nz-1, 2ny-1,
 * 2nx-1) complex128, component order xx, xy, xz, yy, yz, zz, entry at offset d
 * = vol * G(delta d) (centroid rule), the zero offset = self_val on xx/yy/zz
 * and 0 elsewhere (self term from the host quadrature, kernel.py:101-116). */
int vx_assemble_green(int nx, int ny, int nz, double delta, double k0, double vol, vx_c128 self_val,
                      vx_c128* out, void* stream);

/* Host -> device upload of a PAGEABLE host buffer (the numpy field vectors /
 * coefficient maps callers pass to apply_n, apply_system and gmres:
 * reference operator.py:82-105, solver.py:114-174).  A persistent pool of
 * host threads copies 2 MB chunks into a ring of pinned slots and each issues
 * its chunk's DMA on `stream`.  Returns once `src` has been consumed (same
 * contract as cudaMemcpy from pageable memory); the DMA is ordered on
 * `stream`.  vx_h2d_threads() = host threads used (pool + caller). */
int vx_h2d_staged(void* dst, const void* src, size_t bytes, void* stream);
int vx_h2d_threads(void);
/* Pinned host blocks for results (pooled by the host side) and a synchronous
 * device -> pinned-host copy ordered on `stream`. */
int vx_host_alloc(size_t bytes, void** out);
int vx_host_free(void* p);
int vx_d2h_pinned(void* dst, const void* src, size_t bytes, void* stream);
/* vx_d2h_pinned without the final stream synchronisation (the caller overlaps
 * the copy with work on another stream, e.g. gmres's true-residual matvec). */
int vx_d2h_pinned_async(void* dst, const void* src, size_t bytes, void* stream);

/* ---- ragged ("packed") factor storage for the 1-level block solves.
 * The build writes every block in the padded tile geometry of dmax (tiles of
 * 32, reference zgetrf blocks circulant.py:113-118 re-tiled); the repack keeps
 * only the leading d_s x d_s entries of each sector block (tile (i,j) is
 * t_i x t_j, t_i = min(32, d_s - 32 i)), so the per-iteration solve streams
 * sum_s d_s^2 entries per stored frequency instead of nsec * npad^2.
 * sec_dims: host array of nsec (<= 4) dims, each <= dmax; dense blocks use
 * nsec = 1, dims = {3 ny nz}.  Ragged storage per frequency slot:
 * vx_lu_rag_stride(nsec, sec_dims) entries. */
long vx_lu_rag_stride(int nsec, const int* sec_dims);
/* Solve-only sector path (sharded preconditioner, dist.py): on S (3 ny nz rows
 * x pitch frequency columns): orbit transform, ragged sector block solves
 * (work list as vx_prec1_apply_sec_rag with nx -> pitch), inverse transform,
 * in place.  U: nsec*dmax*pitch scratch. */
int vx_prec1_solve_sec_rag(int ny, int nz, long pitch, const vx_c128* factors, const int* perm, const int* items,
                           int n_single, int n_items, int direct_r, const int* klist, int nsec, int dmax,
                           const int* sec_dims, int norb, const int* orows, const int* osec, const double* ocoef,
                           const unsigned char* flipk, vx_c128* S, vx_c128* U, void* stream);

/* 1 while vx_solve_variant(1) selects the synchronous (padded-only) solve. */
int vx_solve_classic(void);
int vx_lu_repack(int nkslots, int nsec, int dmax, const int* sec_dims, const vx_c128* padded,
                 vx_c128* ragged, void* stream);
int vx_lu_unpack(int nkslots, int nsec, int dmax, const int* sec_dims, const vx_c128* ragged,
                 vx_c128* padded, void* stream);
/* vx_prec1_apply / vx_prec1_apply_sec (reference OneLevelPrec.apply,
 * circulant.py:162-188) on ragged factors (single-RHS work lists only). */
int vx_prec1_apply_rag(int nx, int ny, int nz, int nrhs, const vx_c128* factors, const int* perm,
                       const int* items, int n_single, int n_items, int direct_r, const int* klist,
                       const vx_c128* x, vx_c128* y, vx_c128* work, void* stream);
int vx_prec1_apply_sec_rag(int nx, int ny, int nz, int nrhs, const vx_c128* factors, const int* perm,
                           const int* items, int n_single, int n_items, int direct_r, const int* klist,
                           int nsec, int dmax, const int* sec_dims, int norb, const int* orows,
                           const int* osec, const double* ocoef, const unsigned char* flipk,
                           const vx_c128* x, vx_c128* y, vx_c128* work, void* stream);

/* Reduced scheme on sector factors (ReducedOneLevelPrec.apply,
 * circulant.py:264-269, with the symmetry sectors above): items [0, n_single)
 * are the kept blocks' sector solves (ragged factors when sec_dims is given,
 * else the padded dmax geometry); the n_rep discarded frequencies rep_ks are,
 * per sector s, one FP64 tensor-core GEMM with the representative sector
 * block's explicit inverse rep_inv + s * vx_rep_inverse_elems(dmax) (formed
 * by vx_rep_inverse on the padded sector factor), on a side stream
 * concurrently with the single-block solves.  work holds
 * vx_prec1_sec_reduced_work_elems entries. */
long vx_prec1_sec_reduced_work_elems(int nx, int ny, int nz, int nrhs, int nsec, int dmax, int n_rep);
int vx_prec1_apply_sec_reduced(int nx, int ny, int nz, int nrhs, const vx_c128* factors, const int* perm,
                               const int* items, int n_single, int direct_r, const int* klist, int nsec, int dmax,
                               const int* sec_dims, int norb, const int* orows, const int* osec, const double* ocoef,
                               const unsigned char* flipk, const vx_c128* rep_inv, const int* rep_ks, int n_rep,
                               const vx_c128* x, vx_c128* y, vx_c128* work, void* stream);

/* ---- symmetric factors (csrc/lu_sym.cuh).  S M^-1 D_k is complex symmetric
 * (the Green's tensor is even under d -> -d; S = -1 on the x-component rows,
 * M = diag(m~)), so when m~ has no zero entry an UNPIVOTED factorisation
 * D_k = L U has U = diag(u) W L^T W^-1 with W = S M on the (sector) rows and
 * only L is stored: half the factor bytes of the LU layout (reference
 * circulant.py:113-118 stores the full zgetrf LU).
 * vx_lu1_build_opts: vx_lu1_build (nsec == 0 or rrow == NULL) or
 *   vx_lu1_build_sec with flags bit 0 = eliminate without row interchanges.
 * vx_lu_sym_pack: padded unpivoted sector factors -> symmetric layout
 *   (vx_lu_sym_stride entries per frequency slot), h = 1/(u W) per row
 *   ([slot][dmax]) and per slot dev[2 slot] = max |U - diag(u) W L^T W^-1| /
 *   max |U|, dev[2 slot + 1] = min |u| / max |u| (the caller keeps the
 *   symmetric layout only when every block passes).  w: [sector][dmax] W.
 * vx_lu_sym_unpack: back to the padded LU layout (multi-RHS applies, views).
 * vx_prec1_apply_sym: vx_prec1_apply_sec_reduced on symmetric factors
 *   (single RHS; n_rep = 0 for the full 1-level scheme); sector dims up to 256. */
int vx_lu1_build_opts(int nx, int ny, int nz, const vx_c128* lamT, const vx_c128* m_yz, const int* kset, int nk,
                      int nsec, int dmax, const int* rrow, const double* rsc, const int* ccol, const double* cw,
                      vx_c128* factors, int* perm, int* piv, int* info, int flags, void* stream);
long vx_lu_sym_stride(int nsec, const int* sec_dims);
int vx_lu_sym_pack(int nkslots, int nsec, int dmax, const int* sec_dims, const vx_c128* padded, const vx_c128* w,
                   vx_c128* sym, vx_c128* h, double* dev, void* stream);
int vx_lu_sym_unpack(int nkslots, int nsec, int dmax, const int* sec_dims, const vx_c128* sym, const vx_c128* h,
                     const vx_c128* w, vx_c128* padded, void* stream);
int vx_prec1_apply_sym(int nx, int ny, int nz, const vx_c128* factors, const vx_c128* h, const vx_c128* w,
                       const int* items, int n_single, int direct_r, const int* klist, int nsec, int dmax,
                       const int* sec_dims, int norb, const int* orows, const int* osec, const double* ocoef,
                       const unsigned char* flipk, const vx_c128* rep_inv, const int* rep_ks, int n_rep,
                       const vx_c128* x, vx_c128* y, vx_c128* work, void* stream);

/* ---- symmetric inverse (csrc/lu_syminv.cuh).  With B = W A^ (A^ complex
 * symmetric) the block inverse is B^-1 = G W^-1, G = A^^-1 = (L^-1 W)^T diag(h)
 * (L^-1 W) complex symmetric: its lower triangle costs the bytes of L and
 * x = G (b / W) is ONE streaming pass (a symmetric matrix-vector product on
 * the FP64 tensor cores) instead of zgetrs's two dependent triangular sweeps
 * (reference circulant.py:183-186).
 * vx_lu_sym_invert: G of every block from the symmetric factors (layout and
 *   stride of vx_lu_sym_pack; scratch: same size, receives L^-1).
 * vx_prec1_apply_syminv: vx_prec1_apply_sym on G.
 * vx_prec1_solve_syminv: vx_prec1_solve_sec_rag on G (the sharded
 *   preconditioner's received frequency columns, dist.py). */
int vx_prec1_solve_syminv(int ny, int nz, long pitch, const vx_c128* ginv, const vx_c128* w, const int* items,
                          int n_single, int direct_r, const int* klist, int nsec, int dmax, const int* sec_dims,
                          int norb, const int* orows, const int* osec, const double* ocoef,
                          const unsigned char* flipk, vx_c128* S, vx_c128* U, void* stream);
int vx_lu_sym_invert(int nkslots, int nsec, int dmax, const int* sec_dims, const vx_c128* sym, const vx_c128* h,
                     const vx_c128* w, vx_c128* scratch, vx_c128* ginv, void* stream);
int vx_prec1_apply_syminv(int nx, int ny, int nz, const vx_c128* ginv, const vx_c128* w, const int* items,
                          int n_single, int direct_r, const int* klist, int nsec, int dmax, const int* sec_dims,
                          int norb, const int* orows, const int* osec, const double* ocoef,
                          const unsigned char* flipk, const vx_c128* rep_inv, const int* rep_ks, int n_rep,
                          const vx_c128* x, vx_c128* y, vx_c128* work, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* VOXVIE_B200_H */
