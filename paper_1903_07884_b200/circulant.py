"""Drop-in ``voxvie.circulant`` on the GPU (reference: pkg/src/voxvie/circulant.py).

Builds and applies the Chan-circulant preconditioners through the C-ABI:
``vx_chan_x_spectra`` / ``vx_chan_xy_spectra`` (Chan + DFT of the generators),
``vx_lu1_build`` / ``vx_lu2_build`` (unfold + batched pivoted LU, one CTA per
frequency block) and ``vx_prec1_apply`` / ``vx_prec2_apply`` (DFT -> streaming
block solves -> inverse DFT).  Factors live on the device in tiled storage;
``.lu`` / ``.piv`` are reconstructed host views in LAPACK layout for
inspection (small problems).

Host-side pieces are the reference's host logic only: argument validation,
the memory cap, the kept-set selection from the (device-computed) proxies,
and the geometry partition.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import os

import numpy as np
from scipy.linalg import circulant as _dense_circulant

from . import _native as nv
from .errors import PartitionError, PreconditionerBuildError
from .grid import PermittivityMap, VoxelGrid, homogenize
from .kernel import ToeplitzKernel
from .operator import SYMMETRY_RTOL, generator_axis_asymmetry, upload_tensors

BYTES_PER_ENTRY = 16
KFLIP_X = 1 << 30   # klist flag: block is the x-mirror of the stored one (include/voxvie_b200.h)
KFLIP_Y = 1 << 29   # klist flag: y-mirror (2-level)


# ---------------------------------------------------------------------------
# Chan circulant (host utilities; reference circulant.py:32-73)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class ChanCirculant:
    n: int
    c: np.ndarray

    def to_dense(self) -> np.ndarray:
        return _dense_circulant(self.c)


def chan_circulant(first_col, first_row=None) -> ChanCirculant:
    """Frobenius-closest circulant of a Toeplitz matrix (reference circulant.py:43-58)."""
    col = np.asarray(first_col, dtype=np.complex128).reshape(-1)
    row = col if first_row is None else np.asarray(first_row, np.complex128).reshape(-1)
    n = col.size
    if n < 1 or row.size != n:
        raise ValueError("first column and first row must share a length >= 1")
    i = np.arange(1, n)
    c = np.empty(n, np.complex128)
    c[0] = col[0]
    c[1:] = ((n - i) * col[1:] + i * row[n - i]) / n
    return ChanCirculant(n=n, c=c)


def chan_along_axis(gen: np.ndarray, axis: int) -> np.ndarray:
    """Chan formula along one offset axis (reference circulant.py:61-73)."""
    g = np.moveaxis(np.asarray(gen, np.complex128), axis, -1)
    n = (g.shape[-1] + 1) // 2
    s = np.arange(1, n)
    out = np.empty(g.shape[:-1] + (n,), np.complex128)
    out[..., 0] = g[..., n - 1]
    out[..., 1:] = ((n - s) * g[..., n - 1 + s] + s * g[..., s - 1]) / n
    return np.moveaxis(out, -1, axis)


# ---------------------------------------------------------------------------
# host-side validation (reference circulant.py:81-126)
# ---------------------------------------------------------------------------

def _constant_along(m: np.ndarray, axis: int, what: str) -> None:
    lead = np.take(m, [0], axis=axis)
    # exactly constant (what homogenize() returns): one comparison pass, no temporaries of m's size
    if np.array_equal(m, np.broadcast_to(lead, m.shape)):
        return
    # == np.allclose(m, lead, rtol=0, atol) (a NaN fails both), one pass cheaper
    if not np.abs(m - lead).max() <= 1e-12 * max(1.0, np.abs(m).max()):
        raise ValueError(f"homogenized coefficient must be constant along {what}")


def _coerce_mtilde(grid: VoxelGrid, mtilde) -> np.ndarray:
    m = np.asarray(mtilde, dtype=np.complex128)
    if m.shape == grid.shape:
        _constant_along(m, 2, "x")
        return np.ascontiguousarray(m[:, :, 0])
    if m.shape == (grid.nz, grid.ny):
        return np.ascontiguousarray(m)
    raise ValueError(f"mtilde shape {m.shape} not compatible with grid {grid.shape}")


def _proxy_column(ny: int, nz: int) -> int:
    """Proxy = unfactorised entry (row 1, col ny*nz) 1-based (reference circulant.py:99-110)."""
    return ny * nz - 1


def _check_cap(bytes_needed: int, cap_bytes: int, hint: str):
    if bytes_needed > cap_bytes:
        raise PreconditionerBuildError(
            f"preconditioner needs {bytes_needed} bytes, above the cap {cap_bytes}; {hint}")


def _select_kept(proxy: np.ndarray, nx: int, tol: float):
    """reference circulant.py:283-294."""
    if not 0.0 <= tol <= 1.0:
        raise ValueError(f"reduction tolerance must lie in [0, 1], got {tol}")
    mag = np.abs(proxy)
    vmax = mag.max()
    v_hat = mag / vmax if vmax > 0 else np.zeros(proxy.shape)
    rep = int(np.ceil(nx / 2)) - 1
    mask = v_hat > tol
    mask[rep] = True
    kept = np.flatnonzero(mask)
    slot_of = np.full(nx, int(np.searchsorted(kept, rep)), dtype=np.int64)
    slot_of[kept] = np.arange(kept.size)
    return kept, slot_of, rep, v_hat


# ---------------------------------------------------------------------------
# device helpers
# ---------------------------------------------------------------------------

def _torch():
    return nv.require_cuda()


def _gen_strides(g):
    s = g.stride()
    return s[0], s[1], s[2], s[3]


def _lamhat_x(gen, nx, ny, nz):
    """lamT (nx, 6*(2nz-1)*(2ny-1)) on device (reference circulant.py:129-136)."""
    lam = nv.empty_c128((nx, 6 * (2 * nz - 1) * (2 * ny - 1)))
    nv.call("vx_chan_x_spectra", nx, ny, nz, gen.data_ptr(), *_gen_strides(gen), lam.data_ptr(),
            nv.stream_ptr())
    return lam


def _proxies(lam, nx, ny, nz, m00):
    proxy = nv.empty_c128(nx)
    nv.call("vx_proxy", nx, ny, nz, lam.data_ptr(), nv.cval(m00), proxy.data_ptr(), nv.stream_ptr())
    return proxy


def _lu1(lam, m_yz_dev, kset_dev, nslots, nx, ny, nz):
    t = _torch()
    n = 3 * ny * nz
    blk = int(nv.query("vx_lu_block_elems", n))
    fac = t.empty((nslots, blk), dtype=t.complex128, device="cuda")
    perm = t.empty((nslots, n), dtype=t.int32, device="cuda")
    piv = t.empty((nslots, n), dtype=t.int32, device="cuda")
    info = t.empty((nslots,), dtype=t.int32, device="cuda")
    nv.call("vx_lu1_build", nx, ny, nz, lam.data_ptr(), m_yz_dev.data_ptr(), nv.ptr(kset_dev), nslots,
            fac.data_ptr(), perm.data_ptr(), piv.data_ptr(), info.data_ptr(), nv.stream_ptr())
    return fac, perm, piv, info


def _lu1_sec(lam, m_yz_dev, kset_dev, nk, nx, ny, nz, sec, nopiv=False):
    """Sector factorisation (vx_lu1_build_opts): nk * nsec blocks of dmax rows
    (nopiv: elimination without row interchanges, for the symmetric layout)."""
    t = _torch()
    sp = sec.plan
    nslots = nk * sp.nsec
    blk = int(nv.query("vx_lu_block_elems", sp.dmax))
    fac = t.empty((nslots, blk), dtype=t.complex128, device="cuda")
    perm = t.empty((nslots, sp.dmax), dtype=t.int32, device="cuda")
    piv = t.empty((nslots, sp.dmax), dtype=t.int32, device="cuda")
    info = t.empty((nslots,), dtype=t.int32, device="cuda")
    nv.call("vx_lu1_build_opts", nx, ny, nz, lam.data_ptr(), m_yz_dev.data_ptr(), kset_dev.data_ptr(), nk,
            sp.nsec, sp.dmax, sec.rrow.data_ptr(), sec.rsc.data_ptr(), sec.ccol.data_ptr(), sec.cw.data_ptr(),
            fac.data_ptr(), perm.data_ptr(), piv.data_ptr(), info.data_ptr(), 1 if nopiv else 0, nv.stream_ptr())
    return fac, perm, piv, info


# ---------------------------------------------------------------------------
# symmetric factors (csrc/lu_sym.cuh): S M^-1 D_k is complex symmetric (the
# Green's tensor is even under d -> -d), so an unpivoted factorisation D = L U
# has U = diag(u) W L^T W^-1 with W = S M restricted to the (sector) rows, and
# only L is stored -- half the bytes every apply streams.  Used when m~ has no
# zero entry (sector blocks of up to SYM_MAX_DIM rows); the pack kernel verifies
# the relation per block, else the pivoted LU is kept.
SYM_TOL = 1e-11        # max |U - diag(u) W L^T W^-1| / max |U| per block
SYM_MIN_PIVOT = 1e-8   # min |u| / max |u| per block
SYM_MAX_DIM = int(os.environ.get("VX_SYM_MAX_DIM", "1024"))   # csrc/lu_sym.cuh SYM_MAX_DIM


def _sym_eligible(m_yz: np.ndarray, dmax: int) -> bool:
    if os.environ.get("VX_SYM", "1") == "0":
        return False
    a = np.abs(np.asarray(m_yz))
    return 32 < dmax <= SYM_MAX_DIM and bool(np.all(np.isfinite(a))) and bool(a.min() > 0.0)


def _sym_weights(plan, m_yz: np.ndarray) -> np.ndarray:
    """W (nsec, dmax): S M on the sector rows -- -m~ on x-component rows, +m~
    on the others, at the orbit's representative site (m~ is equal on every
    site of an orbit when the sectors exist)."""
    q = m_yz.size
    mf = np.asarray(m_yz, np.complex128).reshape(-1)
    W = np.ones((plan.nsec, plan.dmax), np.complex128)
    rr = plan.rrow
    ok = rr >= 0
    a, site = rr // q, rr % q
    W[ok] = np.where(a[ok] == 0, -1.0, 1.0) * mf[site[ok]]
    return W


# inverse apply vs triangular solves on a seeded random vector (relative L2 over the whole
# vector: one block among 10^4 with a relative error e contributes e / 100, so 1e-13 bounds every
# block's error by 1e-11; observed 5e-16 .. 1.4e-15 on c0-c3)
SYMINV_TOL = 1e-13
SMALLINV_TOL = 1e-13   # explicit inverses of the 2-level blocks vs their factor solves


class _SymFactors:
    """Device symmetric factors: packed lower triangles, h = 1/(u W) per row, W;
    inv: the lower triangles of the symmetric inverses G = A^^-1 (csrc/lu_syminv.cuh)
    once build_inverse() has produced and verified them."""

    def __init__(self, fac, h, w, dims, nsec, dmax):
        self.fac, self.h, self.w, self.dims = fac, h, w, dims
        self.nsec, self.dmax = int(nsec), int(dmax)
        self.inv = None

    def build_inverse(self):
        """G = (L^-1 W)^T diag(h) (L^-1 W) per block (vx_lu_sym_invert)."""
        if os.environ.get("VX_SYMINV", "1") == "0":
            return None
        nk = int(self.fac.shape[0])
        scratch = nv.empty_c128(tuple(self.fac.shape))
        ginv = nv.empty_c128(tuple(self.fac.shape))
        nv.call("vx_lu_sym_invert", nk, self.nsec, self.dmax, self.dims.ctypes.data, self.fac.data_ptr(),
                self.h.data_ptr(), self.w.data_ptr(), scratch.data_ptr(), ginv.data_ptr(), nv.stream_ptr())
        return ginv


def _sym_pack(fac, sec, m_yz, nk):
    """Pack unpivoted sector factors into the symmetric layout; None when a
    block fails the symmetric-reconstruction or pivot-size check."""
    sp = sec.plan
    dims_a = np.ascontiguousarray(sp.dims, np.int32)
    w = nv.device_c128(_sym_weights(sp, m_yz))
    stride = int(nv.query("vx_lu_sym_stride", sp.nsec, dims_a.ctypes.data))
    t = _torch()
    sym = nv.empty_c128((max(1, nk), stride))
    h = nv.empty_c128((max(1, nk * sp.nsec), sp.dmax))
    dev = t.zeros((max(1, nk * sp.nsec), 2), dtype=t.float64, device="cuda")
    nv.call("vx_lu_sym_pack", nk, sp.nsec, sp.dmax, dims_a.ctypes.data, fac.data_ptr(), w.data_ptr(),
            sym.data_ptr(), h.data_ptr(), dev.data_ptr(), nv.stream_ptr())
    d = dev[: nk * sp.nsec].cpu().numpy()
    if d.size and not (d[:, 0].max() <= SYM_TOL and d[:, 1].min() >= SYM_MIN_PIVOT):
        return None
    return _SymFactors(sym, h, w, dims_a, sp.nsec, sp.dmax)


def _lu1_sec_auto(lam, m_dev, kdev, nk, nx, ny, nz, sec, m_yz):
    """Sector factorisation: symmetric (unpivoted, verified) when eligible,
    else zgetrf's partial pivoting -> (fac, perm, piv, info, sym or None)."""
    if _sym_eligible(m_yz, sec.plan.dmax):
        fac, perm, piv, info = _lu1_sec(lam, m_dev, kdev, nk, nx, ny, nz, sec, nopiv=True)
        if _first_bad(info) < 0:
            sym = _sym_pack(fac, sec, m_yz, nk)
            if sym is not None:
                return fac, perm, piv, info, sym
        del fac, perm, piv, info
    return _lu1_sec(lam, m_dev, kdev, nk, nx, ny, nz, sec) + (None,)


def _first_bad(info) -> int:
    bad = (info != 0).nonzero()
    return -1 if bad.numel() == 0 else int(bad[0, 0])


# ---------------------------------------------------------------------------
# mirror sharing of factors (x / y parity of the kernel)
# ---------------------------------------------------------------------------
# For a kernel whose Green components are even/odd under x -> -x (reference
# kernel.py:37-51: the off-diagonal (a, b) entry is odd under a sign flip of
# either coordinate), the Chan x-spectra satisfy lam_p(nx-k) = s_p lam_p(k)
# (s = -1 for xy, xz), so D_{nx-k} = S D_k S with S = -1 on the x-component
# rows.  zgetrf picks the same pivots on S D S (|Re|+|Im| is sign-blind), so
# the factors of D_{nx-k} are sign flips of D_k's: one stored factor serves
# both blocks and one streamed read of it solves both right-hand sides.  The
# 2-level blocks get the same from the y parity (S = -1 on the y rows).

def mirror_axes(gen, dims) -> tuple:
    """(x_ok, y_ok): the generators are parity-symmetric on x / y to SYMMETRY_RTOL
    (VX_MIRROR=0 disables the factor sharing)."""
    if os.environ.get("VX_MIRROR", "1") == "0":
        return False, False
    ax, ay, _ = generator_axis_asymmetry(gen, dims)
    return ax <= SYMMETRY_RTOL, ay <= SYMMETRY_RTOL


def sector_axes(gen, dims, m_yz) -> tuple:
    """(y, z): reflections that commute with every 1-level block -- kernel
    parity on that axis and m~ mirror-symmetric (sectors.py; VX_SECTORS=0
    disables the sector factorisation)."""
    if os.environ.get("VX_SECTORS", "1") == "0":
        return False, False
    from .sectors import m_symmetric

    _, ay, az = generator_axis_asymmetry(gen, dims)
    return (ay <= SYMMETRY_RTOL and m_symmetric(m_yz, "y"),
            az <= SYMMETRY_RTOL and m_symmetric(m_yz, "z"))


class _SectorDev:
    """Device copies of a SectorPlan's tables."""

    def __init__(self, plan):
        t = _torch()
        self.plan = plan
        dev = lambda a: t.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
        self.rrow, self.rsc, self.ccol, self.cw = dev(plan.rrow), dev(plan.rsc), dev(plan.ccol), dev(plan.cw)
        self.orows, self.osec, self.ocoef = dev(plan.orows), dev(plan.osec), dev(plan.ocoef)
        self.norb = int(plan.orows.shape[0])


def _flip_signs(n: int, fx: bool, fy: bool) -> np.ndarray:
    """Diagonal of S for an (n, n) block with rows ordered a*q + ... (q = n/3)."""
    q = n // 3
    s = np.ones(n)
    if fx:
        s[:q] = -1.0
    if fy:
        s[q:2 * q] = -1.0
    return s


def _lu_mirror(lu: np.ndarray, piv: np.ndarray, s: np.ndarray) -> np.ndarray:
    """LAPACK LU of S D S from the LU of D (same pivots): L' = S_p L S_p,
    U' = S_p U S with S_p = P S P^T."""
    n = lu.shape[0]
    perm = np.arange(n)
    for i, p in enumerate(piv):
        perm[i], perm[p] = perm[p], perm[i]
    sp = s[perm]
    out = lu * sp[:, None]
    lower = np.tril(np.ones((n, n), bool), -1)
    return np.where(lower, out * sp[None, :], out * s[None, :])


def _items_groups(groups):
    """groups: list of (slot, [klist entries]) -> (items int32 (3t,), klist int32, max group size)."""
    t = _torch()
    items, klist = [], []
    for slot, ks in groups:
        items.append((slot, len(klist), len(ks)))
        klist.extend(ks)
    r = max((len(ks) for _, ks in groups), default=1)
    return (t.from_numpy(np.asarray(items, np.int32).reshape(-1).copy()).cuda(),
            t.from_numpy(np.asarray(klist if klist else [0], np.int32)).cuda(), r)


def _items_by_slot(store: np.ndarray, entries: np.ndarray):
    """Vectorised _items_groups: one item per distinct storage slot, its klist
    entries in logical-block order -> (items, klist, max group size, n_items)."""
    t = _torch()
    order = np.argsort(store, kind="stable")
    slots, starts, counts = np.unique(store[order], return_index=True, return_counts=True)
    items = np.stack([slots, starts, counts], 1).astype(np.int32)
    return (t.from_numpy(items.reshape(-1).copy()).cuda(),
            t.from_numpy(entries[order].astype(np.int32)).cuda(), int(counts.max()), int(slots.size))


def _untile(fac_row: np.ndarray, n: int) -> np.ndarray:
    """Tiled factor storage -> LAPACK combined LU (n, n) (host, for inspection)."""
    from scipy.linalg import solve_triangular

    nv.load()
    T = int(nv.query("vx_lu_tile", n))
    nt = -(-n // T)
    npad = nt * T
    tiles = fac_row.reshape(nt, nt, T, T)            # (it, jt, col, row)
    full = tiles.transpose(0, 3, 1, 2).reshape(npad, npad).copy()
    eye = np.eye(T)
    # diagonal tiles are stored split (csrc/circulant.cu dl_off/du_off):
    # inv(L) strictly lower packed by columns, then inv(U) upper packed by columns
    lo_r, lo_c = np.tril_indices(T, -1)
    up_r, up_c = np.triu_indices(T)
    lo_order = np.lexsort((lo_r, lo_c))   # column-major order of the packing
    up_order = np.lexsort((up_r, up_c))
    nl = T * (T - 1) // 2
    for i in range(nt if nt > 1 else 0):   # single-tile blocks keep the packed tile
        flat = fac_row[(i * nt + i) * T * T:(i * nt + i + 1) * T * T]
        d = np.zeros((T, T), fac_row.dtype)
        d[lo_r[lo_order], lo_c[lo_order]] = flat[:nl]
        d[up_r[up_order], up_c[up_order]] = flat[nl:]
        full[i * T:(i + 1) * T, i * T:(i + 1) * T] = d
    for i in range(nt):
        d = full[i * T:(i + 1) * T, i * T:(i + 1) * T]
        linv = np.tril(d, -1) + eye
        uinv = np.triu(d)
        L = solve_triangular(linv, eye, lower=True, unit_diagonal=True)
        U = solve_triangular(uinv, eye, lower=False)
        full[i * T:(i + 1) * T, i * T:(i + 1) * T] = np.tril(L, -1) + np.triu(U)
    return full[:n, :n]


def _as_rhs(x, nunk):
    """-> (device tensor (nunk, r) contiguous, r, flat_in, was_tensor, orig_shape)."""
    is_t = nv.is_tensor(x)
    if is_t:
        xd = nv.device_c128(x)
        shape = tuple(x.shape)
    else:
        a = np.asarray(x, dtype=np.complex128)
        shape = a.shape
        xd = nv.device_c128(a)
    # reference circulant.py:176-188: any array whose size is a multiple of
    # the unknown count is read as x.reshape(n_unknowns, -1) (C order) and the
    # result returned in the input's shape (flat for 1-D input)
    flat = len(shape) == 1
    if xd.numel() % nunk != 0:
        raise ValueError(f"cannot reshape array of size {xd.numel()} into shape ({nunk},newaxis)")
    r = xd.numel() // nunk
    return xd.reshape(nunk, r).contiguous(), r, flat, is_t, shape


def _ret(yd, flat, is_t, shape):
    out = yd.reshape(shape)
    return out if is_t else nv.to_host(out)


# ---------------------------------------------------------------------------
# 1-level (reference circulant.py:144-225)
# ---------------------------------------------------------------------------

class _OneLevelBase:
    grid: VoxelGrid
    _sec = None            # _SectorDev when the blocks are stored as symmetry sectors
    _full_builder = None   # builds the plain dense-block preconditioner (for .lu / .piv)
    _full = None
    _sym = None            # _SymFactors when the sector factors are stored symmetric

    @property
    def sectors(self) -> int:
        """Symmetry sectors per frequency block (1: the plain dense factorisation)."""
        return 1 if self._sec is None else self._sec.plan.nsec

    def _dense(self):
        """The plain (unsectored) preconditioner, built on demand for .lu/.piv."""
        if self._full is None:
            self._full = self._full_builder()
        return self._full

    def _sector_items(self, store, ks, flip, rep=None):
        """Work list over sector slots: direct items (store[i]*nsec + s, frequencies
        ks[i] with equal store) and, for the reduced scheme, chunks of 8 of the
        representative's frequencies rep = (slot, ks) per sector."""
        t = _torch()
        nx = self.grid.nx
        ns, dm = self._sec.plan.nsec, self._sec.plan.dmax
        st = (np.asarray(store)[None, :] * ns + np.arange(ns)[:, None]).reshape(-1)
        ent = (np.arange(ns)[:, None] * dm * nx + np.asarray(ks)[None, :]).reshape(-1)
        order = np.argsort(st, kind="stable")
        slots, starts, counts = np.unique(st[order], return_index=True, return_counts=True)
        items = [np.stack([slots, starts, counts], 1)]
        klist = [ent[order]]
        n_single = int(slots.size)
        direct_r = int(counts.max()) if counts.size else 1
        if rep is not None:
            rslot, rks = rep
            off = int(klist[0].size)
            for s in range(ns):
                for c0 in range(0, len(rks), 8):
                    chunk = np.asarray(rks[c0:c0 + 8])
                    items.append(np.array([[rslot * ns + s, off, chunk.size]]))
                    klist.append(s * dm * nx + chunk)
                    off += chunk.size
        items = np.concatenate(items).astype(np.int32)
        klist = np.concatenate(klist).astype(np.int32)
        flipk = np.zeros(nx, np.uint8)
        flipk[np.asarray(ks)[np.asarray(flip, bool)]] = 1
        self._items = t.from_numpy(items.reshape(-1).copy()).cuda()
        self._klist = t.from_numpy(klist if klist.size else np.zeros(1, np.int32)).cuda()
        self._flipk = t.from_numpy(flipk).cuda()
        self._n_single, self._n_items, self._direct_r = n_single, int(items.shape[0]), direct_r

    def _apply_sym(self, xd, rep_inv=None, rep_ks=None, force_factors=False):
        """Single-RHS apply on symmetric sector factors -- or, once built and
        verified, on the symmetric inverses (one streaming pass) -- optionally
        with the reduced scheme's representative GEMM."""
        nx, ny, nz = self.grid.dims
        sp, sd, sy = self._sec.plan, self._sec, self._sym
        n_rep = 0 if rep_ks is None else int(rep_ks.numel())
        y = nv.empty_c128((self.grid.n_unknowns, 1))
        work = nv.empty_c128(int(nv.query("vx_prec1_sec_reduced_work_elems", nx, ny, nz, 1, sp.nsec, sp.dmax, n_rep)))
        if sy.inv is not None and not force_factors:
            nv.call("vx_prec1_apply_syminv", nx, ny, nz, sy.inv.data_ptr(), sy.w.data_ptr(),
                    self._items.data_ptr(), self._n_single, self._direct_r, self._klist.data_ptr(), sp.nsec,
                    sp.dmax, sy.dims.ctypes.data, sd.norb, sd.orows.data_ptr(), sd.osec.data_ptr(),
                    sd.ocoef.data_ptr(), self._flipk.data_ptr(), nv.ptr(rep_inv), nv.ptr(rep_ks), n_rep,
                    xd.data_ptr(), y.data_ptr(), work.data_ptr(), nv.stream_ptr())
            return y
        nv.call("vx_prec1_apply_sym", nx, ny, nz, sy.fac.data_ptr(), sy.h.data_ptr(), sy.w.data_ptr(),
                self._items.data_ptr(), self._n_single, self._direct_r, self._klist.data_ptr(), sp.nsec, sp.dmax,
                sy.dims.ctypes.data, sd.norb, sd.orows.data_ptr(), sd.osec.data_ptr(), sd.ocoef.data_ptr(),
                self._flipk.data_ptr(), nv.ptr(rep_inv), nv.ptr(rep_ks), n_rep, xd.data_ptr(), y.data_ptr(),
                work.data_ptr(), nv.stream_ptr())
        return y

    def _apply_dev(self, xd, r):
        nx, ny, nz = self.grid.dims
        if self._sym is not None and r == 1 and not nv.query("vx_solve_classic"):
            return self._apply_sym(xd)
        rag = getattr(self, "_rag_dims", None) is not None and r == 1 and not nv.query("vx_solve_classic")
        if rag:
            self._padded_fac = None
        fac = (self._fac if (rag or getattr(self, "_rag_dims", None) is None) and self._sym is None
               else self._padded())
        if self._sec is not None:
            sp, sd = self._sec.plan, self._sec
            y = nv.empty_c128((self.grid.n_unknowns, r))
            work = nv.empty_c128(int(nv.query("vx_prec1_sec_work_elems", nx, ny, nz, r, sp.nsec, sp.dmax)))
            if rag:
                nv.call("vx_prec1_apply_sec_rag", nx, ny, nz, r, fac.data_ptr(), self._perm.data_ptr(),
                        self._items.data_ptr(), self._n_single, self._n_items, self._direct_r,
                        self._klist.data_ptr(), sp.nsec, sp.dmax, self._rag_dims.ctypes.data, sd.norb,
                        sd.orows.data_ptr(), sd.osec.data_ptr(), sd.ocoef.data_ptr(), self._flipk.data_ptr(),
                        xd.data_ptr(), y.data_ptr(), work.data_ptr(), nv.stream_ptr())
            else:
                nv.call("vx_prec1_apply_sec", nx, ny, nz, r, fac.data_ptr(), self._perm.data_ptr(),
                        self._items.data_ptr(), self._n_single, self._n_items, self._direct_r,
                        self._klist.data_ptr(), sp.nsec, sp.dmax, sd.norb, sd.orows.data_ptr(),
                        sd.osec.data_ptr(), sd.ocoef.data_ptr(), self._flipk.data_ptr(), xd.data_ptr(),
                        y.data_ptr(), work.data_ptr(), nv.stream_ptr())
            return y
        y = nv.empty_c128((self.grid.n_unknowns, r))
        work = nv.empty_c128(int(nv.query("vx_prec1_work_elems", nx, ny, nz, r)))
        nv.call("vx_prec1_apply_rag" if rag else "vx_prec1_apply", nx, ny, nz, r, fac.data_ptr(),
                self._perm.data_ptr(), self._items.data_ptr(), self._n_single, self._n_items, self._direct_r,
                self._klist.data_ptr(), xd.data_ptr(), y.data_ptr(), work.data_ptr(), nv.stream_ptr())
        return y

    # ---- ragged factor storage (vx_lu_repack): the per-iteration solve streams
    # only the d x d entries of every (sector) block, not the 32-padded tiles
    _rag_dims = None
    _padded_fac = None

    def _rag_geometry(self):
        if self._sec is not None:
            return self._sec.plan.nsec, self._sec.plan.dmax, tuple(self._sec.plan.dims)
        n = self.block_size
        return 1, n, (n,)

    def _make_ragged(self):
        """Repack the padded factors into ragged storage (frees the padded copy);
        symmetric factors replace them by the packed lower triangles."""
        if self._sym is not None:
            self._nslots = int(self._fac.shape[0])
            self._fac = self._sym.fac
            self._make_inverse()
            return
        nsec, dmax, dims = self._rag_geometry()
        if dmax <= 32 or os.environ.get("VX_RAGGED", "1") == "0":
            return
        dims_a = np.ascontiguousarray(dims, np.int32)
        nslots = int(self._fac.shape[0])
        nk = nslots // nsec
        stride = int(nv.query("vx_lu_rag_stride", nsec, dims_a.ctypes.data))
        rag = nv.empty_c128((nk, stride))
        nv.call("vx_lu_repack", nk, nsec, dmax, dims_a.ctypes.data, self._fac.data_ptr(), rag.data_ptr(),
                nv.stream_ptr())
        self._fac = rag
        self._rag_dims = dims_a
        self._nslots = nslots

    def _make_inverse(self):
        """Symmetric inverses of the stored blocks, kept only when one apply on a
        random vector agrees with the triangular solves to SYMINV_TOL."""
        sy = self._sym
        if sy is None or sy.inv is not None or self._sec is None:
            return
        ginv = sy.build_inverse()
        if ginv is None:
            return
        t = _torch()
        gen = t.Generator(device="cuda")
        gen.manual_seed(20240811)
        n = self.grid.n_unknowns
        x = t.randn(n, 2, dtype=t.float64, device="cuda", generator=gen)
        xd = t.view_as_complex(x).reshape(n, 1)
        rep = (getattr(self, "_inv", None), getattr(self, "_rep_ks", None)) if getattr(self, "_inv", None) is not None \
            else (None, None)
        ref = self._apply_sym(xd, rep[0], rep[1], force_factors=True)
        sy.inv = ginv
        got = self._apply_sym(xd, rep[0], rep[1])
        err = float(t.linalg.vector_norm(got - ref) / t.linalg.vector_norm(ref))
        if not err <= SYMINV_TOL:
            sy.inv = None
        self._syminv_err = err

    def _padded(self):
        """Padded-tile factors (nslots, npad^2): the layout the reduced scheme,
        multi-RHS applies and the LAPACK views read (unpacked on demand)."""
        if self._sym is not None:
            if self._padded_fac is None:
                nsec, dmax, _ = self._rag_geometry()
                blk = int(nv.query("vx_lu_block_elems", dmax))
                pad = nv.empty_c128((self._nslots, blk))
                sy = self._sym
                nv.call("vx_lu_sym_unpack", self._nslots // nsec, nsec, dmax, sy.dims.ctypes.data, sy.fac.data_ptr(),
                        sy.h.data_ptr(), sy.w.data_ptr(), pad.data_ptr(), nv.stream_ptr())
                self._padded_fac = pad
            return self._padded_fac
        if self._rag_dims is None:
            return self._fac
        if self._padded_fac is None:
            nsec, dmax, _ = self._rag_geometry()
            blk = int(nv.query("vx_lu_block_elems", dmax))
            pad = nv.empty_c128((self._nslots, blk))
            nv.call("vx_lu_unpack", self._nslots // nsec, nsec, dmax, self._rag_dims.ctypes.data,
                    self._fac.data_ptr(), pad.data_ptr(), nv.stream_ptr())
            self._padded_fac = pad
        return self._padded_fac

    @nv.fresh_output
    def apply(self, x):
        xd, r, flat, is_t, shape = _as_rhs(x, self.grid.n_unknowns)
        if r == 0:
            return _ret(xd.clone(), flat, is_t, shape)
        return _ret(self._apply_dev(xd, r), flat, is_t, shape)

    @property
    def block_size(self) -> int:
        return 3 * self.grid.ny * self.grid.nz

    @property
    def stored_blocks(self) -> list:
        """[(dim, count)] of the factors actually stored (and streamed once per
        apply): mirror sharing halves the count, sectors split each block."""
        sec = getattr(self, "_sec", None)
        nslots = getattr(self, "_nslots", None) or int(self._fac.shape[0])
        if sec is None:
            return [(self.block_size, nslots)]
        nk = nslots // sec.plan.nsec
        return [(d, nk) for d in sec.plan.dims]

    @property
    def storage_bytes(self) -> int:
        """Bytes actually resident on the device for the factors (symmetric,
        ragged, or padded tiles)."""
        extra = self._sym.inv.numel() if self._sym is not None and self._sym.inv is not None else 0
        return int(self._fac.numel() + extra) * 16

    @property
    def factor_bytes_per_apply(self) -> int:
        """Compulsory factor bytes of one single-RHS apply: every stored factor
        entry read once (symmetric layout: the lower triangles only)."""
        if self._sym is not None:
            return int(self._sym.fac.numel()) * 16   # inverse layout: same size as the factor layout
        return 16 * sum(d * d * c for d, c in self.stored_blocks)

    @property
    def factor_layout(self) -> str:
        if self._sym is not None:
            return "symmetric-inverse" if self._sym.inv is not None else "symmetric"
        return "ragged" if getattr(self, "_rag_dims", None) is not None else "padded"

    @property
    def stored_slots(self) -> int:
        """Stored factor blocks (sector blocks count separately)."""
        return getattr(self, "_nslots", None) or int(self._fac.shape[0])

    # per logical block (frequency k for the full scheme, kept index for the
    # reduced one): storage slot and whether it is the x-mirror of that slot
    _store: np.ndarray
    _flip: np.ndarray

    @property
    def mirror_shared(self) -> bool:
        """True when mirror blocks share stored factors (x-parity-symmetric kernel)."""
        return bool(np.any(self._flip))

    @property
    def lu(self) -> np.ndarray:
        if self._sec is not None:
            return self._dense().lu
        f = self._padded().cpu().numpy()
        pv = self._piv.cpu().numpy()
        n = self.block_size
        base = [_untile(f[s], n) for s in range(f.shape[0])]
        sx = _flip_signs(n, True, False)
        return np.stack([_lu_mirror(base[s], pv[s], sx) if fl else base[s]
                         for s, fl in zip(self._store, self._flip)])

    @property
    def piv(self) -> np.ndarray:
        if self._sec is not None:
            return self._dense().piv
        return self._piv.cpu().numpy()[self._store]


def _mirror_store(ks: np.ndarray, nx: int, share: bool):
    """Storage plan for the logical blocks ks (sorted frequencies): the blocks
    to factorise (kset), and per block its storage slot and x-flip."""
    ks = np.asarray(ks, np.int64)
    km = (nx - ks) % nx
    # position of each block's mirror frequency in ks (ks is sorted), if present
    pos = np.searchsorted(ks, km)
    pos_c = np.minimum(pos, ks.size - 1)
    flip = (km < ks) & (ks[pos_c] == km) if share else np.zeros(ks.size, bool)
    own = ~flip
    store = np.empty(ks.size, np.int64)
    store[own] = np.arange(int(own.sum()))
    store[flip] = store[pos_c[flip]]      # the mirror has the smaller frequency: it owns its factor
    return ks[own].copy(), store, flip


class OneLevelPrec(_OneLevelBase):
    """Per-x-frequency LU blocks on the device (reference circulant.py:144-171)."""

    level = "one-level"

    def __init__(self, grid, fac, perm, piv, proxy, store=None, flip=None, sec=None, full_builder=None, sym=None):
        self.grid = grid
        self._fac, self._perm, self._piv, self._proxy = fac, perm, piv, proxy
        self._sym = sym
        nx = grid.nx
        self._store = np.arange(nx) if store is None else np.asarray(store)
        self._flip = np.zeros(nx, bool) if flip is None else np.asarray(flip, bool)
        self._sec = sec
        self._full_builder = full_builder
        if sec is None:
            entries = np.arange(nx) | np.where(self._flip, KFLIP_X, 0)
            self._items, self._klist, self._direct_r, self._n_items = _items_by_slot(self._store, entries)
            self._n_single = self._n_items
        else:
            self._sector_items(self._store, np.arange(nx), self._flip)
        self._make_ragged()

    @property
    def proxy(self) -> np.ndarray:
        return self._proxy.cpu().numpy()

    @property
    def bytes(self) -> int:
        return self.grid.nx * self.block_size ** 2 * BYTES_PER_ENTRY

    def summary(self) -> dict:
        return {"level": self.level, "blocks": int(self.grid.nx),
                "block_size": int(self.block_size), "bytes": int(self.bytes)}


def _build_one_level_dev(grid, gen, m_yz, cap_bytes, tol=None, sectors=True):
    """Shared device build for full (tol None) and reduced 1-level."""
    t = _torch()
    nx, ny, nz = grid.dims
    q = ny * nz
    if tol is None:
        _check_cap(nx * (3 * q) ** 2 * BYTES_PER_ENTRY, cap_bytes, "consider the 2-level preconditioner")
    share = mirror_axes(gen, grid.dims)[0]
    lam = _lamhat_x(gen, nx, ny, nz)
    proxy = _proxies(lam, nx, ny, nz, m_yz[0, 0])
    m_dev = nv.device_c128(m_yz)
    if tol is None:
        kset, store, flip = _mirror_store(np.arange(nx), nx, share)
        kdev = t.from_numpy(kset.astype(np.int32)).cuda()
        sy, sz = sector_axes(gen, grid.dims, m_yz) if sectors else (False, False)
        if sy or sz:
            from .sectors import sector_plan

            sec = _SectorDev(sector_plan(ny, nz, sy, sz))
            fac, perm, piv, info, sym = _lu1_sec_auto(lam, m_dev, kdev, int(kset.size), nx, ny, nz, sec, m_yz)
            bad = _first_bad(info)
            if bad >= 0:
                raise PreconditionerBuildError(
                    f"1-level build failed: singular frequency block k={int(kset[bad // sec.plan.nsec])}")
            return OneLevelPrec(grid, fac, perm, piv, proxy, store, flip, sec=sec,
                                full_builder=lambda: _build_one_level_dev(grid, gen, m_yz, cap_bytes,
                                                                          sectors=False), sym=sym)
        fac, perm, piv, info = _lu1(lam, m_dev, kdev, int(kset.size), nx, ny, nz)
        bad = _first_bad(info)
        if bad >= 0:
            raise PreconditionerBuildError(f"1-level build failed: singular frequency block k={int(kset[bad])}")
        return OneLevelPrec(grid, fac, perm, piv, proxy, store, flip)
    ph = proxy.cpu().numpy()
    kept, slot_of, rep, v_hat = _select_kept(ph, nx, tol)
    _check_cap(kept.size * (3 * q) ** 2 * BYTES_PER_ENTRY, cap_bytes, "consider the 2-level preconditioner")
    kset, store, flip = _mirror_store(kept, nx, share)
    kdev = t.from_numpy(kset.astype(np.int32)).cuda()
    sy, sz = sector_axes(gen, grid.dims, m_yz) if sectors else (False, False)
    if sy or sz:
        from .sectors import sector_plan

        sec = _SectorDev(sector_plan(ny, nz, sy, sz))
        fac, perm, piv, info, sym = _lu1_sec_auto(lam, m_dev, kdev, int(kset.size), nx, ny, nz, sec, m_yz)
        bad = _first_bad(info)
        if bad >= 0:
            raise PreconditionerBuildError(f"singular frequency block k={int(kset[bad // sec.plan.nsec])}")
        return ReducedOneLevelPrec(grid, kept, slot_of, rep, fac, perm, piv, ph, v_hat, float(tol), store, flip,
                                   sec=sec, full_builder=lambda: _build_one_level_dev(grid, gen, m_yz, cap_bytes,
                                                                                      tol=tol, sectors=False),
                                   sym=sym)
    fac, perm, piv, info = _lu1(lam, m_dev, kdev, int(kset.size), nx, ny, nz)
    bad = _first_bad(info)
    if bad >= 0:
        raise PreconditionerBuildError(f"singular frequency block k={int(kset[bad])}")
    return ReducedOneLevelPrec(grid, kept, slot_of, rep, fac, perm, piv, ph, v_hat, float(tol), store, flip)


def build_one_level(kernel: ToeplitzKernel, mtilde, *, cap_bytes: int = 2 ** 31) -> OneLevelPrec:
    """reference circulant.py:191-225."""
    grid = kernel.grid
    m_yz = _coerce_mtilde(grid, mtilde)
    nx, ny, nz = grid.dims
    _check_cap(nx * (3 * ny * nz) ** 2 * BYTES_PER_ENTRY, cap_bytes, "consider the 2-level preconditioner")
    return _build_one_level_dev(grid, upload_tensors(kernel), m_yz, cap_bytes)


# ---------------------------------------------------------------------------
# reduced 1-level (reference circulant.py:233-354)
# ---------------------------------------------------------------------------

class ReducedOneLevelPrec(_OneLevelBase):
    """Kept blocks only; discarded frequencies solved with the representative block."""

    level = "reduced-one-level"

    def __init__(self, grid, kept, slot_of, representative, fac, perm, piv, proxy, v_hat, tol,
                 store=None, flip=None, sec=None, full_builder=None, sym=None):
        self.grid = grid
        self._sym = sym
        self.kept = np.asarray(kept)
        self.slot_of = np.asarray(slot_of)
        self.representative = int(representative)
        self._fac, self._perm, self._piv = fac, perm, piv
        self._store = np.arange(self.kept.size) if store is None else np.asarray(store)
        self._flip = np.zeros(self.kept.size, bool) if flip is None else np.asarray(flip, bool)
        self.proxy = np.asarray(proxy)
        self.proxy_normalized = np.asarray(v_hat)
        self.tol = float(tol)
        self._sec, self._full_builder = sec, full_builder
        self._make_worklist()

    def _make_worklist(self):
        t = _torch()
        rep_idx = int(self.slot_of[self.representative])   # kept index of the representative
        rep_slot = int(self._store[rep_idx])                 # its storage slot (never flipped)
        self._inv = None
        if self._sec is not None:
            keep = np.arange(self.kept.size) != rep_idx
            rep_ks = np.flatnonzero(self.slot_of == rep_idx)
            ns, dm = self._sec.plan.nsec, self._sec.plan.dmax
            if dm > 32 and rep_ks.size >= 8 and os.environ.get("VX_REP_GEMM", "1") != "0":
                # the discarded frequencies: per sector ONE GEMM with the
                # representative sector block's explicit inverse (side stream);
                # the kept blocks' sector solves stream ragged factors
                self._sector_items(self._store[keep], self.kept[keep], self._flip[keep])
                per = int(nv.query("vx_rep_inverse_elems", dm))
                inv = nv.empty_c128(ns * per)
                for sc in range(ns):
                    sl = rep_slot * ns + sc
                    nv.call("vx_rep_inverse", dm, self._fac[sl].data_ptr(), self._perm[sl].data_ptr(),
                            inv[sc * per:].data_ptr(), nv.stream_ptr())
                self._inv = inv
                self._rep_ks = t.from_numpy(rep_ks.astype(np.int32)).cuda()
                self._make_ragged()
                return
            self._sym = None   # representative chunks are multi-RHS items: padded pivot-free LU factors
            self._sector_items(self._store[keep], self.kept[keep], self._flip[keep], rep=(rep_slot, rep_ks))
            return
        groups = {}
        for i, k in enumerate(self.kept):
            if i != rep_idx:
                groups.setdefault(int(self._store[i]), []).append(int(k) | (KFLIP_X if self._flip[i] else 0))
        groups = sorted(groups.items())
        n_single = len(groups)
        rep_ks = np.flatnonzero(self.slot_of == rep_idx)
        for c0 in range(0, rep_ks.size, 8):
            groups.append((rep_slot, [int(k) for k in rep_ks[c0:c0 + 8]]))
        self._items, self._klist, _ = _items_groups(groups)
        self._direct_r = max((len(ks) for _, ks in groups[:n_single]), default=1)
        self._n_single, self._n_items = n_single, len(groups)
        # Multi-tile blocks: the representative's frequencies go through one
        # dense GEMM with its explicit inverse (vx_rep_inverse), concurrently
        # with the single-block solves; VX_REP_GEMM=0 keeps the chunked solves.
        self._inv = None
        n = self.block_size
        if n > 32 and rep_ks.size >= 8 and os.environ.get("VX_REP_GEMM", "1") != "0":
            inv = nv.empty_c128(int(nv.query("vx_rep_inverse_elems", n)))
            nv.call("vx_rep_inverse", n, self._fac[rep_slot].data_ptr(), self._perm[rep_slot].data_ptr(),
                    inv.data_ptr(), nv.stream_ptr())
            self._inv = inv
            self._rep_ks = t.from_numpy(rep_ks.astype(np.int32)).cuda()

    def _apply_dev(self, xd, r):
        if self._inv is not None and self._sec is not None:
            return self._apply_sec_rep(xd, r)
        if self._inv is None or self._sec is not None:
            return super()._apply_dev(xd, r)
        nx, ny, nz = self.grid.dims
        n_rep = int(self._rep_ks.numel())
        y = nv.empty_c128((self.grid.n_unknowns, r))
        work = nv.empty_c128(int(nv.query("vx_prec1_reduced_work_elems", nx, ny, nz, r, n_rep)))
        nv.call("vx_prec1_apply_reduced", nx, ny, nz, r, self._fac.data_ptr(), self._perm.data_ptr(),
                self._items.data_ptr(), self._n_single, self._direct_r, self._klist.data_ptr(), self._inv.data_ptr(),
                self._rep_ks.data_ptr(), n_rep, xd.data_ptr(), y.data_ptr(), work.data_ptr(), nv.stream_ptr())
        return y

    def _apply_sec_rep(self, xd, r):
        if self._sym is not None and r == 1 and not nv.query("vx_solve_classic"):
            return self._apply_sym(xd, self._inv, self._rep_ks)
        nx, ny, nz = self.grid.dims
        sp, sd = self._sec.plan, self._sec
        rag = self._rag_dims is not None and r == 1 and not nv.query("vx_solve_classic")
        fac = self._fac if (rag or self._rag_dims is None) and self._sym is None else self._padded()
        n_rep = int(self._rep_ks.numel())
        y = nv.empty_c128((self.grid.n_unknowns, r))
        work = nv.empty_c128(int(nv.query("vx_prec1_sec_reduced_work_elems", nx, ny, nz, r, sp.nsec, sp.dmax, n_rep)))
        nv.call("vx_prec1_apply_sec_reduced", nx, ny, nz, r, fac.data_ptr(), self._perm.data_ptr(),
                self._items.data_ptr(), self._n_single, self._direct_r, self._klist.data_ptr(), sp.nsec, sp.dmax,
                self._rag_dims.ctypes.data if rag else None, sd.norb, sd.orows.data_ptr(), sd.osec.data_ptr(),
                sd.ocoef.data_ptr(), self._flipk.data_ptr(), self._inv.data_ptr(), self._rep_ks.data_ptr(), n_rep,
                xd.data_ptr(), y.data_ptr(), work.data_ptr(), nv.stream_ptr())
        return y

    @property
    def n_kept(self) -> int:
        return int(self.kept.size)

    @property
    def bytes(self) -> int:
        return self.n_kept * self.block_size ** 2 * BYTES_PER_ENTRY

    def summary(self) -> dict:
        return {"level": self.level, "blocks": int(self.grid.nx), "kept": int(self.n_kept),
                "discarded": int(self.grid.nx - self.n_kept), "block_size": int(self.block_size),
                "tol": self.tol, "bytes": int(self.bytes)}


def reduce_one_level(prec: OneLevelPrec, tol: float = 1e-3) -> ReducedOneLevelPrec:
    """Keep only significant-proxy factors of a built 1-level (reference circulant.py:297-311)."""
    t = _torch()
    nx = prec.grid.nx
    proxy = prec.proxy
    kept, slot_of, rep, v_hat = _select_kept(proxy, nx, tol)
    slots = prec._store[kept]
    uniq, store = np.unique(slots, return_inverse=True)
    flip = prec._flip[kept].copy()
    # a kept block whose stored partner was discarded keeps that partner's
    # factor (stored under the kept block's index, flipped)
    ns = prec.sectors
    rows = (uniq[:, None] * ns + np.arange(ns)[None, :]).reshape(-1)
    idx = t.from_numpy(rows.astype(np.int64)).cuda()
    fb = None
    if prec._sec is not None:
        fb = lambda: reduce_one_level(prec._dense(), tol)  # noqa: E731
    return ReducedOneLevelPrec(prec.grid, kept, slot_of, rep, prec._padded().index_select(0, idx),
                               prec._perm.index_select(0, idx), prec._piv.index_select(0, idx),
                               proxy.copy(), v_hat, float(tol), store, flip, sec=prec._sec, full_builder=fb)


def build_reduced_one_level(kernel: ToeplitzKernel, mtilde, tol: float = 1e-3, *,
                            cap_bytes: int = 2 ** 31) -> ReducedOneLevelPrec:
    """Proxies first, LU only for kept blocks (reference circulant.py:314-354)."""
    grid = kernel.grid
    m_yz = _coerce_mtilde(grid, mtilde)
    if not 0.0 <= tol <= 1.0:
        raise ValueError(f"reduction tolerance must lie in [0, 1], got {tol}")
    return _build_one_level_dev(grid, upload_tensors(kernel), m_yz, cap_bytes, tol=tol)


# ---------------------------------------------------------------------------
# 2-level (reference circulant.py:362-447)
# ---------------------------------------------------------------------------

class TwoLevelPrec:
    """(3nz)^2 LU blocks per (x, y) frequency pair, on the device."""

    level = "two-level"

    def __init__(self, grid, fac, perm, piv, store=None, flips=None):
        self.grid = grid
        self._fac, self._perm, self._piv = fac, perm, piv
        nb = grid.nx * grid.ny
        # per block b = l*nx + k: storage slot and (x, y) mirror flips
        self._store = np.arange(nb) if store is None else np.asarray(store)
        self._flips = np.zeros((nb, 2), bool) if flips is None else np.asarray(flips, bool)
        if store is None:
            self._items, self._klist, self._direct_r, self._n_items = None, None, 1, nb
        else:
            entries = (np.arange(nb) | np.where(self._flips[:, 0], KFLIP_X, 0)
                       | np.where(self._flips[:, 1], KFLIP_Y, 0))
            self._items, self._klist, r, self._n_items = _items_by_slot(self._store, entries)
            self._direct_r = 1 if r == 1 else (2 if r == 2 else 4)

    @property
    def mirror_shared(self) -> bool:
        return bool(np.any(self._flips))

    @property
    def stored_blocks(self) -> list:
        return [(self.block_size, int(self._fac.shape[0]))]

    @property
    def block_size(self) -> int:
        return 3 * self.grid.nz

    @property
    def bytes(self) -> int:
        return self.grid.nx * self.grid.ny * self.block_size ** 2 * BYTES_PER_ENTRY

    @property
    def lu(self) -> np.ndarray:
        f = self._fac.cpu().numpy()
        pv = self._piv.cpu().numpy()
        n = self.block_size
        base = [_untile(f[s], n) for s in range(f.shape[0])]
        out = np.stack([_lu_mirror(base[s], pv[s], _flip_signs(n, fx, fy)) if (fx or fy) else base[s]
                        for s, (fx, fy) in zip(self._store, self._flips)])
        return out.reshape(self.grid.ny, self.grid.nx, n, n)

    @property
    def piv(self) -> np.ndarray:
        return self._piv.cpu().numpy()[self._store].reshape(self.grid.ny, self.grid.nx, -1)

    _ginv = None
    _inv_err = None

    @property
    def factor_layout(self) -> str:
        return "inverse" if self._ginv is not None else "factors"

    def _make_inverse(self):
        """Explicit inverses of the single-tile blocks (3 nz <= 32), kept only if
        they reproduce the factor solve on a seeded random vector to
        SMALLINV_TOL (relative, max norm); VX_SMALLINV=0 keeps the factors."""
        n = self.block_size
        if n > 32 or os.environ.get("VX_SMALLINV", "1") == "0":
            return
        t = _torch()
        nslots = int(self._fac.shape[0])
        g = t.empty((nslots, n * n), dtype=t.complex128, device="cuda")
        nv.call("vx_lu_small_invert", n, nslots, self._fac.data_ptr(), self._perm.data_ptr(), g.data_ptr(),
                nv.stream_ptr())
        gen = t.Generator(device="cuda").manual_seed(20190307)
        probe = t.randn((self.grid.n_unknowns, 1, 2), dtype=t.float64, device="cuda", generator=gen)
        probe = t.view_as_complex(probe).contiguous()
        want = self._apply_dev(probe, 1)
        self._ginv = g
        got = self._apply_dev(probe, 1)
        err = float((got - want).abs().max() / want.abs().max())
        self._inv_err = err
        if not err <= SMALLINV_TOL:
            self._ginv = None

    def _apply_dev(self, xd, r):
        nx, ny, nz = self.grid.dims
        y = nv.empty_c128((self.grid.n_unknowns, r))
        work = nv.empty_c128(int(nv.query("vx_prec2_work_elems", nx, ny, nz, r)))
        if self._ginv is not None:
            nv.call("vx_prec2_apply_inv", nx, ny, nz, r, self._ginv.data_ptr(), nv.ptr(self._items), self._n_items,
                    nv.ptr(self._klist), xd.data_ptr(), y.data_ptr(), work.data_ptr(), nv.stream_ptr())
            return y
        nv.call("vx_prec2_apply", nx, ny, nz, r, self._fac.data_ptr(), self._perm.data_ptr(),
                nv.ptr(self._items), self._n_items, self._direct_r, nv.ptr(self._klist),
                xd.data_ptr(), y.data_ptr(), work.data_ptr(), nv.stream_ptr())
        return y

    @nv.fresh_output
    def apply(self, x):
        xd, r, flat, is_t, shape = _as_rhs(x, self.grid.n_unknowns)
        if r == 0:
            return _ret(xd.clone(), flat, is_t, shape)
        return _ret(self._apply_dev(xd, r), flat, is_t, shape)

    def summary(self) -> dict:
        return {"level": self.level, "blocks": int(self.grid.nx * self.grid.ny),
                "block_size": int(self.block_size), "bytes": int(self.bytes)}


def _coerce_mz(grid, mtilde) -> np.ndarray:
    """m~ for the 2-level scheme: (nz, ny, nx) constant in x and y, (nz,), or a
    scalar (reference circulant.py:405-433) -> (nz,)."""
    nz = grid.nz
    m = np.asarray(mtilde, dtype=np.complex128)
    if m.shape == grid.shape:
        _constant_along(m, 2, "x")
        _constant_along(m, 1, "y")
        return m[:, 0, 0]
    if m.shape == (nz,):
        return m
    if m.ndim == 0:
        return np.full(nz, m, dtype=np.complex128)
    raise ValueError(f"mtilde shape {m.shape} not usable for a 2-level build")


def _build_two_level_dev(grid, gen, mtilde, cap_bytes):
    t = _torch()
    nx, ny, nz = grid.dims
    m_z = _coerce_mz(grid, mtilde)
    _check_cap(nx * ny * (3 * nz) ** 2 * BYTES_PER_ENTRY, cap_bytes, "reduce the box size or cross-section")
    share_x, share_y = mirror_axes(gen, grid.dims)
    work = nv.empty_c128(int(nv.query("vx_chan_xy_work_elems", nx, ny, nz)))
    lam2 = nv.empty_c128((nx * ny, 6 * (2 * nz - 1)))
    nv.call("vx_chan_xy_spectra", nx, ny, nz, gen.data_ptr(), *_gen_strides(gen), lam2.data_ptr(),
            work.data_ptr(), nv.stream_ptr())
    del work
    n = 3 * nz
    # canonical representative of each (l, k) mirror orbit
    ks, ls = np.arange(nx), np.arange(ny)
    kc = np.minimum(ks, (nx - ks) % nx) if share_x else ks
    lc = np.minimum(ls, (ny - ls) % ny) if share_y else ls
    canon = (lc[:, None] * nx + kc[None, :]).reshape(-1)
    kset, store = np.unique(canon, return_inverse=True)
    flips = np.stack([np.broadcast_to((kc != ks)[None, :], (ny, nx)).reshape(-1),
                      np.broadcast_to((lc != ls)[:, None], (ny, nx)).reshape(-1)], 1)
    nb = int(kset.size)
    blk = int(nv.query("vx_lu_block_elems", n))
    fac = t.empty((nb, blk), dtype=t.complex128, device="cuda")
    perm = t.empty((nb, n), dtype=t.int32, device="cuda")
    piv = t.empty((nb, n), dtype=t.int32, device="cuda")
    info = t.empty((nb,), dtype=t.int32, device="cuda")
    m_dev = nv.device_c128(np.ascontiguousarray(m_z))
    kdev = t.from_numpy(kset.astype(np.int32)).cuda()
    nv.call("vx_lu2_build", nx, ny, nz, lam2.data_ptr(), m_dev.data_ptr(), kdev.data_ptr(), nb, fac.data_ptr(),
            perm.data_ptr(), piv.data_ptr(), info.data_ptr(), nv.stream_ptr())
    bad = _first_bad(info)
    if bad >= 0:
        l, k = divmod(int(kset[bad]), nx)
        raise PreconditionerBuildError(f"2-level build failed: singular block (k={k}, l={l})")
    prec = TwoLevelPrec(grid, fac, perm, piv) if nb == nx * ny else TwoLevelPrec(grid, fac, perm, piv, store, flips)
    prec._make_inverse()
    return prec


def build_two_level(kernel: ToeplitzKernel, mtilde, *, cap_bytes: int = 2 ** 31) -> TwoLevelPrec:
    """reference circulant.py:405-447."""
    return _build_two_level_dev(kernel.grid, upload_tensors(kernel), mtilde, cap_bytes)


def apply_one_level(prec, x):
    return prec.apply(x)


def apply_two_level(prec: TwoLevelPrec, x):
    return prec.apply(x)


# ---------------------------------------------------------------------------
# partition + blocked (reference circulant.py:464-651)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Box:
    """Half-open voxel box [x0,x1) x [y0,y1) x [z0,z1)."""

    label: str
    x0: int
    x1: int
    y0: int
    y1: int
    z0: int
    z1: int

    @property
    def dims(self):
        return (self.x1 - self.x0, self.y1 - self.y0, self.z1 - self.z0)

    def n_voxels(self) -> int:
        bx, by, bz = self.dims
        return bx * by * bz

    def overlaps(self, other: "Box") -> bool:
        return all(a0 < b1 and b0 < a1 for a0, a1, b0, b1 in (
            (self.x0, self.x1, other.x0, other.x1),
            (self.y0, self.y1, other.y0, other.y1),
            (self.z0, self.z1, other.z0, other.z1)))


@dataclass(frozen=True)
class Partition:
    grid: VoxelGrid
    boxes: tuple

    @property
    def covered_voxels(self) -> int:
        return sum(b.n_voxels() for b in self.boxes)

    @property
    def identity_voxels(self) -> int:
        return self.grid.n_voxels - self.covered_voxels


def partition_boxes(grid: VoxelGrid, boxes) -> Partition:
    """Validate boxes: inside the grid, pairwise disjoint (reference circulant.py:509-530)."""
    boxes = tuple(boxes)
    outside = [b.label for b in boxes if not (0 <= b.x0 < b.x1 <= grid.nx and 0 <= b.y0 < b.y1 <= grid.ny
                                              and 0 <= b.z0 < b.z1 <= grid.nz)]
    if outside:
        raise PartitionError(f"boxes out of grid bounds: {outside}")
    clash = [(a.label, b.label) for i, a in enumerate(boxes) for b in boxes[i + 1:] if a.overlaps(b)]
    if clash:
        raise PartitionError(f"overlapping boxes: {clash}")
    return Partition(grid=grid, boxes=boxes)


_DEFAULT_HOMOG = {"one-level": "real_mean_x", "reduced-one-level": "real_mean_x", "two-level": "mode"}


def _sub_grid(grid: VoxelGrid, box: Box) -> VoxelGrid:
    bx, by, bz = box.dims
    ox, oy, oz = grid.origin
    d = grid.delta
    return VoxelGrid(bx, by, bz, d, origin=(ox + d * box.x0, oy + d * box.y0, oz + d * box.z0))


def _slice_kernel(kernel: ToeplitzKernel, box: Box) -> ToeplitzKernel:
    """Host copy of the box's offset range (reference circulant.py:577-600)."""
    nz, ny, nx = kernel.grid.shape
    bx, by, bz = box.dims
    cz, cy, cx = nz - 1, ny - 1, nx - 1
    sub = kernel.tensors[:, cz - (bz - 1):cz + bz, cy - (by - 1):cy + by, cx - (bx - 1):cx + bx]
    return ToeplitzKernel(grid=_sub_grid(kernel.grid, box), k0=kernel.k0, tensors=np.ascontiguousarray(sub))


def _slice_device(gen, grid: VoxelGrid, box: Box):
    """Strided device view of the box's generators (no copy)."""
    nz, ny, nx = grid.shape
    bx, by, bz = box.dims
    cz, cy, cx = nz - 1, ny - 1, nx - 1
    return gen[:, cz - (bz - 1):cz + bz, cy - (by - 1):cy + by, cx - (bx - 1):cx + bx]


def _box_dof_indices(grid: VoxelGrid, box: Box) -> np.ndarray:
    idx = np.arange(grid.n_unknowns).reshape((3,) + grid.shape)
    return np.ascontiguousarray(idx[:, box.z0:box.z1, box.y0:box.y1, box.x0:box.x1]).reshape(-1)


class BlockedPrec:
    """Block-diagonal circulant preconditioner over a partition; identity outside."""

    level = "blocked"

    def __init__(self, grid, partition, box_precs):
        self.grid = grid
        self.partition = partition
        self.box_precs = list(box_precs)

    @property
    def box_dofs(self):
        return [_box_dof_indices(self.grid, b) for b in self.partition.boxes]

    @property
    def bytes(self) -> int:
        return sum(p.bytes for p in self.box_precs)

    def _apply_dev(self, xd, r):
        nx, ny, nz = self.grid.dims
        y = nv.empty_c128(tuple(xd.shape))  # identity outside every box
        nv.call("vx_axpby", xd.numel(), nv.cval(1.0), xd.data_ptr(), nv.cval(0.0), None, y.data_ptr(),
                nv.stream_ptr())
        for box, prec in zip(self.partition.boxes, self.box_precs):
            bx, by, bz = box.dims
            sub = nv.empty_c128((3 * bx * by * bz, r))
            nv.call("vx_box_gather", nx, ny, nz, box.x0, box.y0, box.z0, bx, by, bz, r,
                    xd.data_ptr(), sub.data_ptr(), nv.stream_ptr())
            ys = prec._apply_dev(sub, r)
            nv.call("vx_box_scatter", nx, ny, nz, box.x0, box.y0, box.z0, bx, by, bz, r,
                    ys.data_ptr(), y.data_ptr(), nv.stream_ptr())
        return y

    @nv.fresh_output
    def apply(self, x):
        xd, r, flat, is_t, shape = _as_rhs(x, self.grid.n_unknowns)
        if r == 0:
            return _ret(xd.clone(), flat, is_t, shape)
        return _ret(self._apply_dev(xd, r), flat, is_t, shape)

    def summary(self) -> dict:
        return {"level": self.level,
                "boxes": [dict(label=b.label, **p.summary())
                          for b, p in zip(self.partition.boxes, self.box_precs)],
                "identity_voxels": int(self.partition.identity_voxels),
                "bytes": int(self.bytes)}


def build_blocked(kernel: ToeplitzKernel, pmap: PermittivityMap, partition: Partition, levels: dict,
                  *, homog: dict | None = None, reduce_tol: float = 1e-3,
                  cap_bytes: int = 2 ** 31) -> BlockedPrec:
    """Per-box circulant preconditioners (reference circulant.py:610-651)."""
    homog = homog or {}
    gen = upload_tensors(kernel)
    precs = []
    for box in partition.boxes:
        choice = levels[box.label]
        sgrid = _sub_grid(kernel.grid, box)
        smap = PermittivityMap(sgrid, pmap.eps_r[box.z0:box.z1, box.y0:box.y1, box.x0:box.x1])
        mt = homogenize(smap, homog.get(box.label, _DEFAULT_HOMOG.get(choice, "real_mean_x")))
        sgen = _slice_device(gen, kernel.grid, box)
        if choice == "one-level":
            m_yz = _coerce_mtilde(sgrid, mt)
            bx, by, bz = box.dims
            _check_cap(bx * (3 * by * bz) ** 2 * BYTES_PER_ENTRY, cap_bytes,
                       "consider the 2-level preconditioner")
            p = _build_one_level_dev(sgrid, sgen, m_yz, cap_bytes)
        elif choice == "reduced-one-level":
            if not 0.0 <= reduce_tol <= 1.0:
                raise ValueError(f"reduction tolerance must lie in [0, 1], got {reduce_tol}")
            p = _build_one_level_dev(sgrid, sgen, _coerce_mtilde(sgrid, mt), cap_bytes, tol=reduce_tol)
        elif choice == "two-level":
            p = _build_two_level_dev(sgrid, sgen, mt, cap_bytes)
        else:
            raise ValueError(f"unknown per-box level {choice!r} for {box.label!r}")
        precs.append(p)
    return BlockedPrec(kernel.grid, partition, precs)


# ---------------------------------------------------------------------------
# test helpers: artificially circulant kernels (reference circulant.py:659-677)
# ---------------------------------------------------------------------------

def wrap_circulant_x(kernel: ToeplitzKernel) -> ToeplitzKernel:
    nx = kernel.grid.nx
    t = np.array(kernel.tensors, copy=True)
    t[..., :nx - 1] = t[..., nx:2 * nx - 1]
    return ToeplitzKernel(grid=kernel.grid, k0=kernel.k0, tensors=t)


def wrap_circulant_xy(kernel: ToeplitzKernel) -> ToeplitzKernel:
    ny = kernel.grid.ny
    t = np.array(wrap_circulant_x(kernel).tensors, copy=True)
    t[:, :, :ny - 1, :] = t[:, :, ny:2 * ny - 1, :]
    return ToeplitzKernel(grid=kernel.grid, k0=kernel.k0, tensors=t)
