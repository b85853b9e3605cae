"""Sharded (multi-GPU) preconditioned GMRES -- SURVEY section 8(e).

One process per GPU, ``torch.distributed`` (NCCL) for the exchanges.  Every
field vector is distributed by *lines*: the 3*ny*nz lines (c, z, y) of length nx
(reference grid.py:1-9 layout) are split into P contiguous ranges, so a rank's
part of a vector is one contiguous slice and every x-direction transform is
local.  Then:

* operator ``A = I - M N`` (reference operator.py:82-105): local forward
  x-DFT of the owned lines, one all-to-all to x-frequency-column ownership
  (contiguous kx blocks; the rank holds only its columns of the six spectra),
  y/z transforms + spectral multiply on owned columns, all-to-all back,
  local inverse x-DFT with the ``x - m(Nx)`` epilogue;
* 1-level / reduced preconditioner (reference circulant.py:174-188, 264-269):
  local x-DFT, one all-to-all to frequency ownership -- frequencies dealt
  **cyclically** (k = s mod P) so the reduced scheme's kept modes, clustered
  at both spectral ends, spread evenly -- local block solves against the
  rank's factors only (1/P of the memory; the representative block replicated),
  all-to-all back, local inverse DFT;
* Arnoldi: classical Gram-Schmidt with partial dot products all-reduced
  (one all-reduce for the j+2 projections + norm, one for the updated norm,
  two more only when the reference's DGKS test fires).

The GMRES control flow and Givens arithmetic are the single-GPU ones
(``solver.GivensQR``), replicated on every rank on identical all-reduced
scalars.  Local compute goes through a *backend*: ``CudaBackend`` calls the
C-ABI kernels; the CPU multi-process tests (gloo) plug in a numpy backend
from ``tests/`` to check the data movement against the oracle.
"""

from __future__ import annotations

import os
import time

import numpy as np

from . import _native as nv
from .circulant import SMALLINV_TOL, _check_cap, _coerce_mtilde, _coerce_mz, _select_kept
from .errors import BreakdownError, PreconditionerBuildError
from .solver import GivensQR, SolveReport, _speculate


def split_even(n: int, P: int) -> list:
    return [(n * r) // P for r in range(P + 1)]


class Layout:
    """Ownership maps of the sharded solve (host logic, identical on every rank)."""

    def __init__(self, dims, P: int, rank: int, px: int):
        nx, ny, nz = dims
        self.dims, self.P, self.rank, self.px = tuple(dims), P, rank, px
        self.nlines = 3 * ny * nz
        self.lb = split_even(self.nlines, P)
        self.line0, self.line1 = self.lb[rank], self.lb[rank + 1]
        self.nl = self.line1 - self.line0
        self.nloc = self.nl * nx
        self.kxb = split_even(px, P)
        self.nkx = self.kxb[rank + 1] - self.kxb[rank]
        self.kown = [np.arange(s, nx, P) for s in range(P)]
        self.nk = self.kown[rank].size

    def lines_of(self, r):
        return self.lb[r + 1] - self.lb[r]

    def op_cols(self):
        """(col_off, colmap) packing contiguous kx blocks per destination."""
        return np.asarray(self.kxb, np.int32), np.arange(self.px, dtype=np.int32)

    def prec_cols(self):
        off = np.cumsum([0] + [k.size for k in self.kown]).astype(np.int32)
        return off, np.concatenate(self.kown).astype(np.int32)

    def local_slice(self, full):
        nx = self.dims[0]
        return full[self.line0 * nx:self.line1 * nx]


class _Comm:
    def __init__(self, group=None):
        import torch.distributed as dist

        self.d = dist
        self.group = group

    @staticmethod
    def _real(t):
        import torch

        return torch.view_as_real(t).reshape(-1) if t.is_complex() else t

    def all_to_all(self, out, inp, out_splits, in_splits):
        # complex128 travels as pairs of float64 (backend-agnostic)
        f = 2 if out.is_complex() else 1
        self.d.all_to_all_single(self._real(out), self._real(inp), [f * int(v) for v in out_splits],
                                 [f * int(v) for v in in_splits], group=self.group)

    def all_reduce(self, t):
        self.d.all_reduce(self._real(t), group=self.group)
        return t


# ---------------------------------------------------------------- backends
class CudaBackend:
    """Local compute on the C-ABI kernels (product path)."""

    sectors = True   # symmetry-reduced (mirror + sector, ragged) 1-level factors

    def __init__(self):
        self.t = nv.require_cuda()

    def empty(self, shape):
        return nv.empty_c128(shape)

    def ints(self, a):
        return self.t.from_numpy(np.ascontiguousarray(a, np.int32)).cuda()

    def to_dev(self, a):
        return nv.device_c128(a)

    def spectra(self, kernel):
        from .operator import plan_operator

        return plan_operator(kernel, compact=False).spectra_device

    def symmetric(self, kernel) -> bool:
        """Parity-symmetric generators (what plan_operator's compact spectra need)."""
        from .operator import SYMMETRY_RTOL, kernel_asymmetry

        return os.environ.get("VX_SHARD_COMPACT", "1") != "0" and kernel_asymmetry(kernel) <= SYMMETRY_RTOL

    def compact_yz(self, spec_loc):
        """A rank's kx columns (6, pz, py, nkx) -> the y / z half-octant (pz/2+1, py/2+1, nkx, 6)."""
        pz, py, nkx = (int(v) for v in spec_loc.shape[1:])
        out = self.empty(max(1, int(nv.query("vx_spec_compact_yz_elems", nkx, py, pz))))
        nv.call("vx_spec_compact_yz", nkx, py, pz, spec_loc.data_ptr(), out.data_ptr(), nv.stream_ptr())
        return out

    def x_forward(self, x_loc, nl, nx, px):
        A = self.empty((nl, px))
        nv.call("vx_op_x_forward", nx, px, nl, x_loc.data_ptr(), A.data_ptr(), nv.stream_ptr())
        return A

    def op_yz(self, A, spectra_loc, dims, nkx, px, py, pz, compact=False):
        nx, ny, nz = dims
        work = self.empty(int(nv.query("vx_op_yz_work_elems", ny, nz, nkx, py)))
        nv.call("vx_op_yz_compact" if compact else "vx_op_yz", ny, nz, nkx, px, py, pz, spectra_loc.data_ptr(),
                A.data_ptr(), work.data_ptr(), nv.stream_ptr())

    def x_inverse(self, A, dims, px, nl, line0, m_full, x_loc):
        nx, ny, nz = dims
        y = self.empty(nl * nx)
        nv.call("vx_op_x_inverse", nx, ny, nz, px, nl, line0, A.data_ptr(), nv.ptr(m_full), x_loc.data_ptr(),
                y.data_ptr(), nv.stream_ptr())
        return y

    def dft_lines(self, x, nl, n, inverse):
        y = self.empty((nl, n))
        nv.call("vx_fft_lines", n, nl, 1, x.data_ptr(), n, 0, 1, n, y.data_ptr(), n, 0, 1, n,
                1 if inverse else 0, (1.0 / n) if inverse else 1.0, nv.stream_ptr())
        return y

    def gather_cols(self, A, nrows, lda, col_off, colmap, total):
        out = self.empty(max(1, nrows * total))
        nv.call("vx_gather_cols", nrows, A.data_ptr(), lda, col_off.numel() - 1, col_off.data_ptr(),
                colmap.data_ptr(), total, out.data_ptr(), nv.stream_ptr())
        return out

    def scatter_cols(self, buf, A, nrows, lda, col_off, colmap, total):
        nv.call("vx_scatter_cols", nrows, buf.data_ptr(), col_off.numel() - 1, col_off.data_ptr(),
                colmap.data_ptr(), total, A.data_ptr(), lda, nv.stream_ptr())

    def chan_x(self, kernel):
        from .circulant import _lamhat_x
        from .operator import upload_tensors

        nx, ny, nz = kernel.grid.dims
        return _lamhat_x(upload_tensors(kernel), nx, ny, nz)

    def proxies(self, lam, dims, m00):
        from .circulant import _proxies

        nx, ny, nz = dims
        return _proxies(lam, nx, ny, nz, m00).cpu().numpy()

    def build_factors(self, lam, dims, m_yz, kset):
        from .circulant import _first_bad, _lu1

        nx, ny, nz = dims
        fac, perm, piv, info = _lu1(lam, nv.device_c128(m_yz), self.ints(kset), len(kset), nx, ny, nz)
        bad = _first_bad(info)
        if bad >= 0:
            raise PreconditionerBuildError(f"1-level build failed: singular frequency block k={int(kset[bad])}")
        return fac, perm

    def chan_xy(self, kernel):
        from .circulant import _gen_strides
        from .operator import upload_tensors

        nx, ny, nz = kernel.grid.dims
        gen = upload_tensors(kernel)
        work = self.empty(int(nv.query("vx_chan_xy_work_elems", nx, ny, nz)))
        lam2 = self.empty((nx * ny, 6 * (2 * nz - 1)))
        nv.call("vx_chan_xy_spectra", nx, ny, nz, gen.data_ptr(), *_gen_strides(gen), lam2.data_ptr(),
                work.data_ptr(), nv.stream_ptr())
        return lam2

    def build_factors2(self, lam2, dims, m_z, kset):
        from .circulant import _first_bad

        nx, ny, nz = dims
        n, nb = 3 * nz, len(kset)
        fac = self.t.empty((max(1, nb), int(nv.query("vx_lu_block_elems", n))), dtype=self.t.complex128,
                           device="cuda")
        perm = self.t.empty((max(1, nb), n), dtype=self.t.int32, device="cuda")
        piv = self.t.empty((max(1, nb), n), dtype=self.t.int32, device="cuda")
        info = self.t.zeros((max(1, nb),), dtype=self.t.int32, device="cuda")
        if nb:
            # keep the argument tensors referenced until the launch is ordered
            m_dev, k_dev = nv.device_c128(np.ascontiguousarray(m_z)), self.ints(kset)
            nv.call("vx_lu2_build", nx, ny, nz, lam2.data_ptr(), m_dev.data_ptr(), k_dev.data_ptr(), nb,
                    fac.data_ptr(), perm.data_ptr(), piv.data_ptr(), info.data_ptr(), nv.stream_ptr())
        bad = _first_bad(info[:nb]) if nb else -1
        if bad >= 0:
            l, k = divmod(int(kset[bad]), nx)
            raise PreconditionerBuildError(f"2-level build failed: singular block (k={k}, l={l})")
        return fac, perm

    def dft_y(self, Y, nplanes, ny, nk, inverse):
        """In-place DFT along y of Y laid out (plane, y, kx_local)."""
        if nplanes * nk == 0:
            return
        nv.call("vx_fft_lines", ny, nplanes * nk, nk, Y.data_ptr(), ny * nk, 1, nk, ny, Y.data_ptr(), ny * nk, 1,
                nk, ny, 1 if inverse else 0, (1.0 / ny) if inverse else 1.0, nv.stream_ptr())

    def solve(self, Y, n, factors, perm, items, n_single, n_items, klist, s_row):
        nv.call("vx_prec1_solve", n, 1, factors.data_ptr(), perm.data_ptr(), items.data_ptr(), n_single, n_items,
                1, klist.data_ptr(), Y.data_ptr(), s_row, 1, nv.stream_ptr())

    def invert_small(self, n, factors, perm):
        """Explicit inverses of single-tile blocks (n <= 32), column-major per slot."""
        g = self.empty(max(1, int(factors.shape[0]) * n * n))
        nv.call("vx_lu_small_invert", n, int(factors.shape[0]), factors.data_ptr(), perm.data_ptr(), g.data_ptr(),
                nv.stream_ptr())
        return g

    def solve_inv(self, Y, n, ginv, items, n_items, klist, s_row):
        nv.call("vx_small_inv_apply", n, 1, ginv.data_ptr(), items.data_ptr(), n_items, klist.data_ptr(),
                Y.data_ptr(), s_row, 1, nv.stream_ptr())

    def cgs_dots(self, V, nvec, w, part):
        out = self.empty(nvec + 1)
        nv.call("vx_cgs_dots", w.numel(), nvec, V.data_ptr(), V.shape[1], w.data_ptr(), out.data_ptr(),
                part.data_ptr(), nv.stream_ptr())
        return out

    def cgs_update(self, V, nvec, coef, w, part):
        out = self.empty(1)
        nv.call("vx_cgs_update", w.numel(), nvec, V.data_ptr(), V.shape[1], coef.data_ptr(), w.data_ptr(),
                out.data_ptr(), part.data_ptr(), nv.stream_ptr())
        return out

    def part(self, n, nvec):
        return self.empty(int(nv.query("vx_arnoldi_part_elems", n, nvec + 2)))

    # ---- device-driven Arnoldi step: no host read between the operator and the next operator
    device_driven = True

    def step_workspace(self, mmax):
        """Pinned result buffers (two, alternating by step parity) and events of a solve."""
        t = self.t
        return {"h": [t.empty(mmax + 2, dtype=t.complex128).pin_memory() for _ in range(2)],
                "ctl": [t.empty(4, dtype=t.float64).pin_memory() for _ in range(2)],
                "ev": [t.cuda.Event() for _ in range(2)]}

    def arnoldi_step(self, C, V, j, w, part, ws):
        """Classical Gram-Schmidt of w against V[0..j] with the reference's DGKS second pass
        (solver.py:62-77) on line-sharded vectors: local partial sums, all-reduced on the stream,
        the decision taken on the device; V[j+1] = w / ||w|| is formed on the device.  Returns a
        handle whose result() waits for this step only and gives (h[0..j+1], ||w0||, fired)."""
        t = self.t
        n, nvec, ldv = w.numel(), j + 1, V.shape[1]
        st = nv.stream_ptr()
        d = self.empty(nvec + 1)
        nv.call("vx_cgs_dots", n, nvec, V.data_ptr(), ldv, w.data_ptr(), d.data_ptr(), part.data_ptr(), st)
        C.all_reduce(d)
        n1 = self.empty(1)
        nv.call("vx_cgs_update", n, nvec, V.data_ptr(), ldv, d.data_ptr(), w.data_ptr(), n1.data_ptr(),
                part.data_ptr(), st)
        C.all_reduce(n1)
        ctl = t.empty(4, dtype=t.float64, device="cuda")
        nv.call("vx_dgks_ctl", d[nvec:].data_ptr(), n1.data_ptr(), ctl.data_ptr(), st)
        c = self.empty(nvec + 1)
        nv.call("vx_cgs_dots_cond", n, nvec, V.data_ptr(), ldv, w.data_ptr(), c.data_ptr(), part.data_ptr(),
                ctl.data_ptr(), st)
        C.all_reduce(c)
        n2 = self.empty(1)
        nv.call("vx_cgs_update_cond", n, nvec, V.data_ptr(), ldv, c.data_ptr(), w.data_ptr(), n2.data_ptr(),
                part.data_ptr(), ctl.data_ptr(), st)
        C.all_reduce(n2)
        hcol = self.empty(nvec + 1)
        nv.call("vx_dgks_finish", nvec, d.data_ptr(), c.data_ptr(), n2.data_ptr(), ctl.data_ptr(),
                hcol.data_ptr(), st)
        nv.call("vx_scale_dev", n, w.data_ptr(), V[j + 1].data_ptr(), hcol[nvec:].data_ptr(), st)
        b = j % 2
        ws["h"][b][: nvec + 1].copy_(hcol, non_blocking=True)
        ws["ctl"][b].copy_(ctl, non_blocking=True)
        ws["ev"][b].record()
        return _DevStep(ws, b, nvec, (d, n1, c, n2, ctl, hcol, w))

    def axpby(self, a, x, b, y, out=None):
        out = self.empty(x.numel()) if out is None else out
        nv.call("vx_axpby", x.numel(), nv.cval(a), x.data_ptr(), nv.cval(b), nv.ptr(y), out.data_ptr(),
                nv.stream_ptr())
        return out

    def combine(self, V, nvec, y):
        u = self.empty(V.shape[1])
        yd = nv.device_c128(y)
        nv.call("vx_basis_combine", V.shape[1], nvec, V.data_ptr(), V.shape[1], yd.data_ptr(), u.data_ptr(),
                nv.stream_ptr())
        return u

    def combine_list(self, zs, y):
        """u = sum_i y_i z_i over separately stored vectors (the kept z_j = P^-1 v_j)."""
        t = self.t
        n = zs[0].numel()
        u = self.empty(n)
        yd = nv.device_c128(np.asarray(y, np.complex128))
        ptrs = t.tensor([z.data_ptr() for z in zs], dtype=t.int64).cuda()
        nv.call("vx_basis_combine_ptrs", n, len(zs), ptrs.data_ptr(), yd.data_ptr(), u.data_ptr(), nv.stream_ptr())
        return u

    def to_host(self, t):
        return t.cpu().numpy()


# ------------------------------------------------------------------ operator
class DistOperator:
    """Line-sharded ``A = I - M N`` (or ``N`` with m None)."""

    def __init__(self, kernel, layout: Layout, backend, comm: _Comm):
        self.L, self.B, self.C = layout, backend, comm
        spec = backend.spectra(kernel)
        self.pz, self.py, self.px = (int(v) for v in spec.shape[1:])
        assert self.px == layout.px, "layout built for a different x padding"
        k0, k1 = layout.kxb[layout.rank], layout.kxb[layout.rank + 1]
        self.spec_loc = spec[..., k0:k1].contiguous()
        del spec
        # parity-symmetric kernels: keep only the y / z half-octant of the rank's columns (a quarter
        # of the bytes; the z-multiply then shares one spectra load between kz and its mirror)
        self.compact = bool(getattr(backend, "symmetric", lambda k: False)(kernel)) and k1 > k0
        if self.compact:
            self.spec_loc = backend.compact_yz(self.spec_loc)
        off, cmap = layout.op_cols()
        self.col_off, self.colmap = backend.ints(off), backend.ints(cmap)

    def apply(self, m_full, x_loc):
        L, B, C = self.L, self.B, self.C
        nx, ny, nz = L.dims
        px, nkx = self.px, L.nkx
        A = B.x_forward(x_loc, L.nl, nx, px)
        send = B.gather_cols(A, L.nl, px, self.col_off, self.colmap, px)
        recv = B.empty(L.nlines * nkx)
        C.all_to_all(recv, send[:L.nl * px],
                     [L.lines_of(r) * nkx for r in range(L.P)],
                     [L.nl * (L.kxb[s + 1] - L.kxb[s]) for s in range(L.P)])
        if self.compact:
            B.op_yz(recv, self.spec_loc, L.dims, nkx, px, self.py, self.pz, compact=True)
        else:
            B.op_yz(recv, self.spec_loc, L.dims, nkx, px, self.py, self.pz)
        back = B.empty(L.nl * px)
        C.all_to_all(back, recv,
                     [L.nl * (L.kxb[s + 1] - L.kxb[s]) for s in range(L.P)],
                     [L.lines_of(r) * nkx for r in range(L.P)])
        B.scatter_cols(back, A, L.nl, px, self.col_off, self.colmap, px)
        return B.x_inverse(A, L.dims, px, L.nl, L.line0, m_full, x_loc)


# ------------------------------------------------------------ preconditioner
class DistOneLevelPrec:
    """Frequency-sharded 1-level (``tol=None``) or reduced 1-level preconditioner."""

    def __init__(self, kernel, mtilde, layout: Layout, backend, comm: _Comm, tol=None, cap_bytes=2 ** 62):
        self.L, self.B, self.C = layout, backend, comm
        grid = kernel.grid
        nx, ny, nz = grid.dims
        m_yz = _coerce_mtilde(grid, mtilde)
        q3 = 3 * ny * nz
        self.n = q3
        self.kown = layout.kown
        self.sec = None
        if tol is None and getattr(backend, "sectors", False) and self._init_sectors(kernel, m_yz):
            return
        lam = backend.chan_x(kernel)
        owned = layout.kown[layout.rank]
        col_of = {int(k): i for i, k in enumerate(owned)}
        if tol is None:
            kset = owned
            items = [(i, i, 1) for i in range(owned.size)]
            klist = list(range(owned.size))
            n_single = len(items)
            self.n_stored_global = nx
        else:
            proxy = backend.proxies(lam, grid.dims, m_yz[0, 0])
            kept, slot_of, rep, _ = _select_kept(proxy, nx, tol)
            self.n_stored_global = int(kept.size)
            keptset = set(int(k) for k in kept)
            own_kept = [int(k) for k in owned if int(k) in keptset and int(k) != rep]
            kset = np.asarray(own_kept + [rep], dtype=np.int64)
            rep_local = len(own_kept)
            items, klist = [], []
            for s, k in enumerate(own_kept):
                items.append((s, len(klist), 1))
                klist.append(col_of[k])
            n_single = len(items)
            rep_ks = [int(k) for k in owned if int(k) not in keptset or int(k) == rep]
            for c0 in range(0, len(rep_ks), 8):
                chunk = rep_ks[c0:c0 + 8]
                items.append((rep_local, len(klist), len(chunk)))
                klist.extend(col_of[k] for k in chunk)
        self.bytes_local = len(kset) * q3 * q3 * 16
        self.factors, self.perm = backend.build_factors(lam, grid.dims, m_yz, np.asarray(kset))
        del lam
        self.items = backend.ints(np.asarray(items, np.int32).reshape(-1) if items else np.zeros(3, np.int32))
        self.klist = backend.ints(np.asarray(klist if klist else [0], np.int32))
        self.n_single, self.n_items = n_single, len(items)
        off, cmap = layout.prec_cols()
        self.col_off, self.colmap = backend.ints(off), backend.ints(cmap)

    def _init_sectors(self, kernel, m_yz) -> bool:
        """Symmetry-reduced factors (the single-GPU layout, circulant.py /
        sectors.py): mirror orbits {k, nx-k} are dealt to ranks whole, each rank
        factorises the sector blocks of its canonical frequencies only and
        stores them ragged, and the apply runs the orbit transform + ragged
        sector solves on the received columns (vx_prec1_solve_sec_rag).  False
        when the kernel / m~ lack the symmetries (dense path)."""
        from .circulant import (SYMINV_TOL, _SectorDev, _first_bad, _lamhat_x, _lu1_sec_auto, _mirror_store,
                                mirror_axes, sector_axes)
        from .operator import upload_tensors
        from .sectors import sector_plan

        L = self.L
        grid = kernel.grid
        nx, ny, nz = grid.dims
        gen = upload_tensors(kernel)
        share = mirror_axes(gen, grid.dims)[0]
        sy, sz = sector_axes(gen, grid.dims, m_yz)
        if not (share and (sy or sz)):
            return False
        plan = sector_plan(ny, nz, sy, sz)
        if plan.dmax <= 32:
            return False
        kc = np.arange(nx // 2 + 1)
        owner = kc % L.P
        self.kown = [np.unique(np.concatenate([kc[owner == r], (nx - kc[owner == r]) % nx])) for r in range(L.P)]
        owned = self.kown[L.rank]
        nk = owned.size
        kset, store, flip = _mirror_store(owned, nx, True)
        sec = _SectorDev(plan)
        t = self.B.t
        kdev = t.from_numpy(kset.astype(np.int32)).cuda()
        m_dev = nv.device_c128(m_yz)
        lam = _lamhat_x(gen, nx, ny, nz)
        # unpivoted + symmetric when eligible (circulant._lu1_sec_auto), else zgetrf's pivoting
        fac, perm, piv, info, sym = _lu1_sec_auto(lam, m_dev, kdev, int(kset.size), nx, ny, nz, sec, m_yz)
        del lam, piv
        bad = _first_bad(info)
        if bad >= 0:
            raise PreconditionerBuildError(
                f"1-level build failed: singular frequency block k={int(kset[bad // plan.nsec])}")
        dims_a = np.ascontiguousarray(plan.dims, np.int32)
        stride = int(nv.query("vx_lu_rag_stride", plan.nsec, dims_a.ctypes.data))
        rag = nv.empty_c128((max(1, int(kset.size)), stride))
        if kset.size:
            nv.call("vx_lu_repack", int(kset.size), plan.nsec, plan.dmax, dims_a.ctypes.data, fac.data_ptr(),
                    rag.data_ptr(), nv.stream_ptr())
        del fac
        ns, dm = plan.nsec, plan.dmax
        st = (store[None, :] * ns + np.arange(ns)[:, None]).reshape(-1)
        ent = (np.arange(ns)[:, None] * dm * nk + np.arange(nk)[None, :]).reshape(-1)
        order = np.argsort(st, kind="stable")
        slots, starts, counts = np.unique(st[order], return_index=True, return_counts=True)
        flipk = np.zeros(max(1, nk), np.uint8)
        flipk[:nk][flip] = 1
        self.sec, self.sec_dims, self.factors, self.perm = sec, dims_a, rag, perm
        self.items = t.from_numpy(np.stack([slots, starts, counts], 1).astype(np.int32).reshape(-1).copy()).cuda()
        self.klist = t.from_numpy(ent[order].astype(np.int32) if ent.size else np.zeros(1, np.int32)).cuda()
        self.flipk = t.from_numpy(flipk).cuda()
        self.n_single = self.n_items = int(slots.size)
        self.direct_r = int(counts.max()) if counts.size else 1
        self.n_stored_global = nx // 2 + 1
        self.bytes_local = int(kset.size) * stride * 16
        self.stored_local = [(int(d), int(kset.size)) for d in plan.dims]
        self.stored_global = [(int(d), nx // 2 + 1) for d in plan.dims]
        off = np.cumsum([0] + [k.size for k in self.kown]).astype(np.int32)
        self.col_off = self.B.ints(off)
        self.colmap = self.B.ints(np.concatenate(self.kown).astype(np.int32))
        # symmetric inverses of this rank's blocks (csrc/lu_syminv.cuh): kept when one solve on
        # seeded random columns agrees with the ragged factors; then they are what the applies stream
        self.sym = self.ginv = None
        if sym is not None and self.n_items:
            ginv = sym.build_inverse()
            if ginv is not None:
                gen_ = t.Generator(device="cuda")
                gen_.manual_seed(20240811 + L.rank)
                S0 = t.view_as_complex(t.randn(3 * ny * nz * nk, 2, dtype=t.float64, device="cuda", generator=gen_))
                ref = S0.clone()
                self._solve_sectors(ref, nk)
                self.sym, self.ginv = sym, ginv
                got = S0.clone()
                self._solve_sectors(got, nk)
                err = float(t.linalg.vector_norm(got - ref) / t.linalg.vector_norm(ref))
                self.syminv_err = err
                if err <= SYMINV_TOL:
                    self.factors = None          # the ragged factors are not needed any more
                    self.bytes_local = int(ginv.numel()) * 16
                else:
                    self.sym = self.ginv = None
        return True

    def _solve_sectors(self, recv, nk):
        """Sector block solves on the received frequency columns (in place)."""
        L, B = self.L, self.B
        sd, sp = self.sec, self.sec.plan
        U = B.empty(max(1, sp.nsec * sp.dmax * nk))
        if self.ginv is not None:
            nv.call("vx_prec1_solve_syminv", L.dims[1], L.dims[2], nk, self.ginv.data_ptr(), self.sym.w.data_ptr(),
                    self.items.data_ptr(), self.n_single, self.direct_r, self.klist.data_ptr(), sp.nsec, sp.dmax,
                    self.sec_dims.ctypes.data, sd.norb, sd.orows.data_ptr(), sd.osec.data_ptr(),
                    sd.ocoef.data_ptr(), self.flipk.data_ptr(), recv.data_ptr(), U.data_ptr(), nv.stream_ptr())
            return
        nv.call("vx_prec1_solve_sec_rag", L.dims[1], L.dims[2], nk, self.factors.data_ptr(),
                self.perm.data_ptr(), self.items.data_ptr(), self.n_single, self.n_items, self.direct_r,
                self.klist.data_ptr(), sp.nsec, sp.dmax, self.sec_dims.ctypes.data, sd.norb,
                sd.orows.data_ptr(), sd.osec.data_ptr(), sd.ocoef.data_ptr(), self.flipk.data_ptr(),
                recv.data_ptr(), U.data_ptr(), nv.stream_ptr())

    def apply(self, x_loc):
        L, B, C = self.L, self.B, self.C
        nx = L.dims[0]
        kown = self.kown
        S = B.dft_lines(x_loc, L.nl, nx, False)
        send = B.gather_cols(S, L.nl, nx, self.col_off, self.colmap, nx)
        nk = kown[L.rank].size
        recv = B.empty(max(1, L.nlines * nk))
        C.all_to_all(recv[:L.nlines * nk], send[:L.nl * nx],
                     [L.lines_of(r) * nk for r in range(L.P)],
                     [L.nl * kown[s].size for s in range(L.P)])
        if self.sec is not None:
            if self.n_items:
                self._solve_sectors(recv, nk)
        elif self.n_items:
            B.solve(recv, self.n, self.factors, self.perm, self.items, self.n_single, self.n_items, self.klist, nk)
        back = B.empty(max(1, L.nl * nx))
        C.all_to_all(back[:L.nl * nx], recv[:L.nlines * nk],
                     [L.nl * kown[s].size for s in range(L.P)],
                     [L.lines_of(r) * nk for r in range(L.P)])
        B.scatter_cols(back, S, L.nl, nx, self.col_off, self.colmap, nx)
        return B.dft_lines(S, L.nl, nx, True).reshape(-1)


class DistTwoLevelPrec:
    """Frequency-sharded 2-level preconditioner (reference circulant.py:362-447,
    SURVEY 8(e) "2-level"): local x-DFT of the owned lines, one all-to-all to
    kx ownership (kx dealt cyclically, as for the 1-level scheme), the y-DFT
    and the (3nz)^2 block solves of every (ky, owned kx) locally -- the rank
    stores only the factors of its kx columns (1/P of them) -- then the
    inverse path.  Two all-to-alls of one vector per apply."""

    def __init__(self, kernel, mtilde, layout: Layout, backend, comm: _Comm, cap_bytes=2 ** 62):
        self.L, self.B, self.C = layout, backend, comm
        grid = kernel.grid
        nx, ny, nz = grid.dims
        m_z = _coerce_mz(grid, mtilde)
        self.n = 3 * nz
        _check_cap(nx * ny * self.n ** 2 * 16, cap_bytes, "reduce the box size or cross-section")
        lam2 = backend.chan_xy(kernel)
        owned = layout.kown[layout.rank]
        nk = owned.size
        # slot l*nk + kl factors block (l, owned[kl]); its right-hand side is
        # column l*nk + kl of the (3nz, ny*nk) received array
        kset = (np.arange(ny)[:, None] * nx + owned[None, :]).reshape(-1).astype(np.int64)
        self.n_slots = int(kset.size)
        self.n_stored_global = nx * ny
        self.bytes_local = self.n_slots * self.n ** 2 * 16
        self.factors, self.perm = backend.build_factors2(lam2, grid.dims, m_z, kset)
        del lam2
        items = np.stack([np.arange(self.n_slots)] * 2 + [np.ones(self.n_slots, np.int64)], 1)
        self.items = backend.ints(items.reshape(-1) if self.n_slots else np.zeros(3, np.int32))
        self.klist = backend.ints(np.arange(max(1, self.n_slots)))
        off, cmap = layout.prec_cols()
        self.col_off, self.colmap = backend.ints(off), backend.ints(cmap)
        self.ginv = None
        self.ginv_err = None
        self._init_inverse(ny * nk)

    def _init_inverse(self, s_row):
        """Single-tile blocks as explicit inverses where the backend has them (the
        GPU one), kept only if they reproduce the factor solve on a seeded
        random array (the single-GPU TwoLevelPrec's rule); VX_SMALLINV=0: factors."""
        B = self.B
        if (self.n > 32 or not self.n_slots or not hasattr(B, "invert_small")
                or os.environ.get("VX_SMALLINV", "1") == "0"):
            return
        g = B.invert_small(self.n, self.factors, self.perm)
        rng = np.random.default_rng(20190307)
        probe = rng.normal(size=self.n * s_row) + 1j * rng.normal(size=self.n * s_row)
        y0, y1 = B.to_dev(probe), B.to_dev(probe)
        B.solve(y0, self.n, self.factors, self.perm, self.items, self.n_slots, self.n_slots, self.klist, s_row)
        B.solve_inv(y1, self.n, g, self.items, self.n_slots, self.klist, s_row)
        a, b = np.asarray(B.to_host(y0)), np.asarray(B.to_host(y1))
        self.ginv_err = float(np.abs(a - b).max() / np.abs(a).max())
        if self.ginv_err <= SMALLINV_TOL:
            self.ginv = g

    def apply(self, x_loc):
        L, B, C = self.L, self.B, self.C
        nx, ny, nz = L.dims
        S = B.dft_lines(x_loc, L.nl, nx, False)
        send = B.gather_cols(S, L.nl, nx, self.col_off, self.colmap, nx)
        nk = L.nk
        recv = B.empty(max(1, L.nlines * nk))
        C.all_to_all(recv[:L.nlines * nk], send[:L.nl * nx],
                     [L.lines_of(r) * nk for r in range(L.P)],
                     [L.nl * L.kown[s].size for s in range(L.P)])
        if self.n_slots:
            B.dft_y(recv, 3 * nz, ny, nk, False)
            if self.ginv is not None:
                B.solve_inv(recv, self.n, self.ginv, self.items, self.n_slots, self.klist, ny * nk)
            else:
                B.solve(recv, self.n, self.factors, self.perm, self.items, self.n_slots, self.n_slots, self.klist,
                        ny * nk)
            B.dft_y(recv, 3 * nz, ny, nk, True)
        back = B.empty(max(1, L.nl * nx))
        C.all_to_all(back[:L.nl * nx], recv[:L.nlines * nk],
                     [L.nl * L.kown[s].size for s in range(L.P)],
                     [L.lines_of(r) * nk for r in range(L.P)])
        B.scatter_cols(back, S, L.nl, nx, self.col_off, self.colmap, nx)
        return B.dft_lines(S, L.nl, nx, True).reshape(-1)


class DistBlockedPrec:
    """Sharded blocked preconditioner (reference circulant.py:540-651; SURVEY
    8(e) "Blocked": each box's frequency blocks spread over all ranks).  Per
    box: the box's lines (c, z in box, y in box; x range [x0, x1)) move from
    the global line ownership to the box's own line Layout (one all-to-all),
    the box's sharded 1-level / reduced / 2-level preconditioner runs on them
    (built on the box's generators and homogenised map, as build_blocked
    does), and the result moves back (second all-to-all) into the box's x
    range; identity outside the boxes."""

    def __init__(self, kernel, pmap, partition, levels: dict, layout: Layout, backend, comm: _Comm, *,
                 homog: dict | None = None, reduce_tol: float = 1e-3, cap_bytes=2 ** 62):
        from .circulant import _DEFAULT_HOMOG, _slice_kernel, _sub_grid
        from .grid import PermittivityMap, homogenize

        self.L, self.B, self.C = layout, backend, comm
        homog = homog or {}
        grid = kernel.grid
        nx, ny, nz = grid.dims
        P, rank = layout.P, layout.rank
        self.boxes, self.box_precs = [], []
        self.bytes_local = 0
        for box in partition.boxes:
            choice = levels[box.label]
            sgrid = _sub_grid(grid, box)
            smap = PermittivityMap(sgrid, pmap.eps_r[box.z0:box.z1, box.y0:box.y1, box.x0:box.x1])
            mt = homogenize(smap, homog.get(box.label, _DEFAULT_HOMOG.get(choice, "real_mean_x")))
            skern = _slice_kernel(kernel, box)
            bx, by, bz = box.dims
            bL = Layout(sgrid.dims, P, rank, 2 * bx)
            if choice == "one-level":
                prec = DistOneLevelPrec(skern, mt, bL, backend, comm, cap_bytes=cap_bytes)
            elif choice == "reduced-one-level":
                if not 0.0 <= reduce_tol <= 1.0:
                    raise ValueError(f"reduction tolerance must lie in [0, 1], got {reduce_tol}")
                prec = DistOneLevelPrec(skern, mt, bL, backend, comm, tol=reduce_tol, cap_bytes=cap_bytes)
            elif choice == "two-level":
                prec = DistTwoLevelPrec(skern, mt, bL, backend, comm, cap_bytes=cap_bytes)
            else:
                raise ValueError(f"unknown per-box level {choice!r} for {box.label!r}")
            self.bytes_local += prec.bytes_local
            # global line and box line of every box line, in box-line order
            c, z, y = np.meshgrid(np.arange(3), np.arange(box.z0, box.z1), np.arange(box.y0, box.y1),
                                  indexing="ij")
            gline = ((c * nz + z) * ny + y).reshape(-1)
            bline = np.arange(gline.size)
            og = np.searchsorted(layout.lb, gline, side="right") - 1
            ob = np.searchsorted(bL.lb, bline, side="right") - 1
            xr = np.arange(box.x0, box.x1)
            send_idx, send_splits = [], []
            for d in range(P):   # my global lines, grouped by their box owner
                sel = gline[(og == rank) & (ob == d)]
                send_idx.append(((sel - layout.line0)[:, None] * nx + xr[None, :]).reshape(-1))
                send_splits.append(sel.size * bx)
            recv_pos, recv_splits = [], []
            for src in range(P):  # my box lines, grouped by their global owner
                sel = bline[(ob == rank) & (og == src)]
                recv_pos.append(((sel - bL.line0)[:, None] * bx + np.arange(bx)[None, :]).reshape(-1))
                recv_splits.append(sel.size * bx)
            self.box_precs.append(prec)
            self.boxes.append(dict(prec=prec, n_loc=bL.nloc,
                                   send_idx=np.concatenate(send_idx).astype(np.int64),
                                   recv_pos=np.concatenate(recv_pos).astype(np.int64),
                                   send_splits=send_splits, recv_splits=recv_splits, idx_dev={}))

    @staticmethod
    def _idx(bx_, key, dev):
        import torch

        t = bx_["idx_dev"].get((key, str(dev)))
        if t is None:
            t = torch.as_tensor(bx_[key], dtype=torch.long, device=dev)
            bx_["idx_dev"][(key, str(dev))] = t
        return t

    def apply(self, x_loc):
        B, C = self.B, self.C
        y = x_loc.clone()
        for bx_ in self.boxes:
            si, rp = self._idx(bx_, "send_idx", x_loc.device), self._idx(bx_, "recv_pos", x_loc.device)
            sendbuf = x_loc.reshape(-1)[si]
            recv = B.empty(max(1, int(sum(bx_["recv_splits"]))))
            C.all_to_all(recv[:rp.numel()], sendbuf, bx_["recv_splits"], bx_["send_splits"])
            xb = B.empty(max(1, bx_["n_loc"]))
            xb[rp] = recv[:rp.numel()]
            yb = bx_["prec"].apply(xb[:bx_["n_loc"]])
            back = B.empty(max(1, si.numel()))
            C.all_to_all(back[:si.numel()], yb.reshape(-1)[rp], bx_["send_splits"], bx_["recv_splits"])
            y.reshape(-1)[si] = back[:si.numel()]
        return y


# ------------------------------------------------------------------- GMRES
def _norm(B, C, x, part):
    d = B.cgs_dots(x.reshape(1, -1), 0, x, part)
    C.all_reduce(d)
    return float(np.sqrt(B.to_host(d)[0].real))


class _DevStep:
    """A device-driven Arnoldi step in flight (CudaBackend.arnoldi_step)."""

    def __init__(self, ws, b, nvec, keep):
        self.ws, self.b, self.nvec = ws, b, nvec
        self.keep = keep   # the step's device buffers stay alive until it has been read

    def result(self):
        ws, b = self.ws, self.b
        ws["ev"][b].synchronize()
        h = ws["h"][b][: self.nvec + 1].numpy().copy()
        cv = ws["ctl"][b].numpy()
        self.keep = None
        return h, float(cv[0]), bool(cv[2] != 0.0)


class _HostStep:
    """Host-driven Arnoldi step (backends without a device-side DGKS decision: the CPU test
    backend): CGS against V[0..j], the reference's DGKS second pass, v_{j+1} = w / ||w||; every
    partial result is all-reduced and read on the host before the next stage."""

    def __init__(self, B, C, V, j, w, part):
        d = C.all_reduce(B.cgs_dots(V, j + 1, w, part))
        dh = B.to_host(d)
        h = np.empty(j + 2, np.complex128)
        h[: j + 1] = dh[: j + 1]
        n0 = float(np.sqrt(dh[j + 1].real))
        n1 = float(np.sqrt(B.to_host(C.all_reduce(B.cgs_update(V, j + 1, d, w, part)))[0].real))
        fired = n1 < 0.7071 * n0   # DGKS second pass (reference solver.py:69-73)
        if fired:
            c = C.all_reduce(B.cgs_dots(V, j + 1, w, part))
            h[: j + 1] += B.to_host(c)[: j + 1]
            n1 = float(np.sqrt(B.to_host(C.all_reduce(B.cgs_update(V, j + 1, c, w, part)))[0].real))
        h[j + 1] = n1
        B.axpby(1.0 / n1 if n1 > 0 else 0.0, w, 0.0, None, out=V[j + 1])
        self._res = (h, n0, bool(fired))

    def result(self):
        return self._res


class _Basis:
    """Krylov basis rows on the backend, grown geometrically (as the
    single-GPU solver._Krylov): a solve that converges in a few iterations
    never allocates the (mmax + 1) x n basis of the worst case."""

    def __init__(self, B, n, maxrows):
        self.B, self.n, self.maxrows = B, n, maxrows
        self.V, self.cap = None, 0
        self.ensure(min(maxrows, 32))

    def ensure(self, rows):
        if rows <= self.cap:
            return self.V
        rows = min(max(rows, 2 * self.cap), max(self.maxrows, rows))
        V = self.B.empty((rows, self.n))
        if self.V is not None:
            V[: self.cap].copy_(self.V[: self.cap])
        self.V, self.cap = V, rows
        return V


def gmres_sharded(apply_a, b_loc, backend, comm: _Comm, *, apply_pinv=None, tol=1e-4, maxit=2000,
                  restart=None):
    """Right-preconditioned restarted GMRES on line-sharded vectors (reference
    solver.py:114-174 control flow; see module docstring for the exchanges).
    The garbage collector is paused during the solve (solver.gc_paused)."""
    from .solver import gc_paused

    with gc_paused():
        return _gmres_sharded(apply_a, b_loc, backend, comm, apply_pinv=apply_pinv, tol=tol, maxit=maxit,
                              restart=restart)


def _gmres_sharded(apply_a, b_loc, backend, comm: _Comm, *, apply_pinv=None, tol=1e-4, maxit=2000,
                   restart=None):
    if not tol > 0:
        raise ValueError("tol must be positive")
    if maxit < 1:
        raise ValueError("maxit must be >= 1")
    B, C = backend, comm
    t0 = time.perf_counter()
    n = b_loc.numel()
    mmax = maxit if restart is None else min(restart, maxit)
    part = B.part(max(n, 1), mmax + 1)
    bnorm = _norm(B, C, b_loc, part)
    if bnorm == 0.0:
        return B.axpby(0.0, b_loc, 0.0, None), SolveReport(iterations=1, residuals=[1.0, 0.0], converged=True,
                                                           solve_seconds=time.perf_counter() - t0,
                                                           true_residual=0.0)
    op = apply_a if apply_pinv is None else (lambda v: apply_a(apply_pinv(v)))
    x = B.axpby(0.0, b_loc, 0.0, None)
    basis = _Basis(B, n, mmax + 1)
    residuals = [1.0]
    total = 0
    converged = False
    reorth = 0
    keep_z = apply_pinv is not None and hasattr(B, "combine_list") and os.environ.get("VX_KEEP_Z", "1") != "0"
    ws = B.step_workspace(mmax) if getattr(B, "device_driven", False) and \
        os.environ.get("VX_SHARD_DEVICE_STEP", "1") != "0" else None
    while total < maxit and not converged:
        r0 = B.axpby(1.0, b_loc, -1.0, apply_a(x)) if total else B.axpby(1.0, b_loc, 0.0, None)
        beta = _norm(B, C, r0, part)
        if beta / bnorm <= tol:
            converged = True
            break
        m = maxit - total if restart is None else min(restart, maxit - total)
        V = basis.V
        B.axpby(1.0 / beta, r0, 0.0, None, out=V[0])
        qr = GivensQR(beta)
        j = 0
        lucky = False
        pending = {}
        zl = []

        def launch(jj):
            # step jj: operator, orthogonalisation and v_{jj+1}, all enqueued (device-driven
            # backends) or computed (host-driven ones) without looking at earlier results
            Vc = basis.ensure(jj + 2)
            if keep_z:
                # z_j = P^-1 v_j is needed for the operator anyway: kept, so the cycle's
                # correction is u = Z y with no extra preconditioner apply (as solver._gmres_cycle)
                z = apply_pinv(Vc[jj])
                if any(z.data_ptr() == q.data_ptr() for q in zl[:jj]):
                    z = z.clone()   # the callable reuses its output buffer
                del zl[jj:]
                zl.append(z)
                w = apply_a(z)
            else:
                w = op(Vc[jj])
            if ws is not None:
                pending[jj] = B.arnoldi_step(C, Vc, jj, w, part, ws)
            else:
                pending[jj] = _HostStep(B, C, Vc, jj, B.axpby(1.0, w, 0.0, None), part)

        launched = 0
        while j < m:
            if launched <= j:
                launch(j)
                launched = j + 1
            # one step of lookahead (as solver._gmres_cycle): the next step is enqueued before this
            # one's Hessenberg column is read, unless the residual trend says this one converges
            if ws is not None and launched == j + 1 and j + 1 < m and _speculate(residuals, tol):
                launch(j + 1)
                launched = j + 2
            h, n0, fired = pending.pop(j).result()
            reorth += int(fired)
            lucky = h[j + 1].real <= 1e-14 * max(n0, 1e-300)
            V = basis.V
            qr.add_column(h, j, residuals, tol)
            j += 1
            est = abs(qr.g[j]) / bnorm
            residuals.append(float(est))
            if est <= tol or lucky:
                converged = est <= tol
                if lucky and not converged:
                    raise BreakdownError(f"Arnoldi breakdown at iteration {len(residuals) - 1}")
                break
        total += j
        if keep_z:
            x = B.axpby(1.0, x, 1.0, B.combine_list(zl[:j], qr.solve(j)))
        else:
            u = B.combine(V, j, qr.solve(j))
            x = B.axpby(1.0, x, 1.0, u if apply_pinv is None else apply_pinv(u))
    true_res = _norm(B, C, B.axpby(1.0, b_loc, -1.0, apply_a(x)), part) / bnorm
    report = SolveReport(iterations=int(total), residuals=residuals, converged=bool(converged),
                         solve_seconds=time.perf_counter() - t0, true_residual=float(true_res))
    report.reorth_passes = int(reorth)
    return x, report
