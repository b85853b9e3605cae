"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

A numpy/scipy restatement of the reference hot path (arXiv 1903.07884,
package ``voxvie`` under /root/reference/pkg/src/voxvie).  It is the checker
for the CUDA path: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.
The product package ``paper_1903_07884_b200`` never imports this module and
has no CPU fallback.

Parity pinning: ``tests/golden/make_golden.py`` runs the *unmodified*
reference (importable in the build container) on seeded inputs and commits
its outputs under ``tests/golden/``; ``tests/test_oracle_golden.py`` checks
every function here against those vectors (and against the reference's own
committed artefact ``pkg/frontend/tests/fixtures/sweep.csv`` for GMRES
iteration counts).

Third-party arithmetic the reference delegates to (not under /root/reference):
scipy.fft (pocketfft/ducc) and LAPACK zgetrf/zgetrs via scipy.linalg
(scipy 1.18.1 in this image); numpy vdot/norm.  The oracle calls the same
routines, as the reference does.

Every function cites the reference file:line it restates.
"""

from __future__ import annotations

import numpy as np
import scipy.fft
from scipy.linalg import lu_factor, lu_solve

PAIR_OF = np.array([[0, 1, 2], [1, 3, 4], [2, 4, 5]], dtype=np.int64)  # accel.py:41
DENSE_GUARD = 6000  # kernel.py:26


# ----------------------------------------------------------------------------
# operator (reference operator.py)
# ----------------------------------------------------------------------------

def embed_circulant(gen, dims):
    """operator.py:21-41 -- generator (2nz-1,2ny-1,2nx-1) -> (2nz,2ny,2nx)."""
    nx, ny, nz = dims
    out = np.zeros((2 * nz, 2 * ny, 2 * nx), dtype=np.complex128)

    def halves(n):
        # (src slice, dst slice): offsets 0..n-1 -> 0..n-1 ; -(n-1)..-1 -> n+1..2n-1
        return [(slice(n - 1, 2 * n - 1), slice(0, n)), (slice(0, n - 1), slice(n + 1, 2 * n))]

    for sz, dz in halves(nz):
        for sy, dy in halves(ny):
            for sx, dx in halves(nx):
                out[dz, dy, dx] = gen[sz, sy, sx]
    return out


def plan_spectra(tensors, dims, workers=1):
    """operator.py:61-70 -- six padded spectra (6, 2nz, 2ny, 2nx)."""
    nx, ny, nz = dims
    spec = np.empty((6, 2 * nz, 2 * ny, 2 * nx), dtype=np.complex128)
    for p in range(6):
        spec[p] = scipy.fft.fftn(embed_circulant(tensors[p], dims), workers=workers)
    return spec


def apply_n(spectra, dims, x, workers=1):
    """operator.py:82-98 -- y = N x by zero-padded FFT convolution."""
    nx, ny, nz = dims
    xf = np.asarray(x, dtype=np.complex128).reshape(3, nz, ny, nx)
    shape = spectra.shape[1:]
    xh = np.stack([scipy.fft.fftn(xf[c], shape, workers=workers) for c in range(3)])
    out = np.empty_like(xf)
    for a in range(3):
        acc = spectra[PAIR_OF[a, 0]] * xh[0]
        acc += spectra[PAIR_OF[a, 1]] * xh[1]
        acc += spectra[PAIR_OF[a, 2]] * xh[2]
        out[a] = scipy.fft.ifftn(acc, workers=workers)[:nz, :ny, :nx]
    return out.reshape(-1)


def apply_system(spectra, dims, m, x, workers=1):
    """operator.py:101-105 -- y = x - m * (N x)."""
    nx, ny, nz = dims
    m = np.asarray(m, dtype=np.complex128).reshape(nz, ny, nx)
    nxx = apply_n(spectra, dims, x, workers).reshape(3, nz, ny, nx)
    return (np.asarray(x, np.complex128).reshape(3, nz, ny, nx) - m[None] * nxx).reshape(-1)


def rhs_from_incident(m, e_inc, omega, eps0):
    """operator.py:108-112."""
    m = np.asarray(m, dtype=np.complex128)
    return (1j * omega * eps0 * m[None] * np.asarray(e_inc, np.complex128).reshape((3,) + m.shape)).reshape(-1)


def field_from_currents(spectra, dims, w, e_inc, omega, eps0):
    """operator.py:115-121."""
    w = np.asarray(w, np.complex128).reshape(-1)
    return np.asarray(e_inc, np.complex128).reshape(-1) + (apply_n(spectra, dims, w) - w) / (1j * omega * eps0)


def dense_n(tensors, dims):
    """kernel.py:208-230 -- explicit 3N x 3N matrix (small grids only)."""
    nx, ny, nz = dims
    n = nx * ny * nz
    if 3 * n > DENSE_GUARD:
        raise ValueError("dense oracle refused")
    iz, iy, ix = np.unravel_index(np.arange(n), (nz, ny, nx))
    off = ((iz[:, None] - iz[None, :] + nz - 1) * (2 * ny - 1)
           + (iy[:, None] - iy[None, :] + ny - 1)) * (2 * nx - 1) + (ix[:, None] - ix[None, :] + nx - 1)
    flat = tensors.reshape(6, -1)
    out = np.empty((3 * n, 3 * n), dtype=np.complex128)
    for a in range(3):
        for b in range(3):
            out[a * n:(a + 1) * n, b * n:(b + 1) * n] = flat[PAIR_OF[a, b]][off]
    return out


def dense_operator(tensors, dims, m):
    """kernel.py:233-242 -- A = I - M N."""
    mf = np.tile(np.asarray(m, np.complex128).reshape(-1), 3)
    a = -mf[:, None] * dense_n(tensors, dims)
    a[np.diag_indices_from(a)] += 1.0
    return a


# ----------------------------------------------------------------------------
# circulant preconditioners (reference circulant.py, accel.py)
# ----------------------------------------------------------------------------

def chan_circulant(col, row=None):
    """circulant.py:43-58 -- c_i = ((n-i) t_i + i t_{-(n-i)})/n."""
    col = np.asarray(col, np.complex128).reshape(-1)
    row = col if row is None else np.asarray(row, np.complex128).reshape(-1)
    n = col.size
    c = np.empty(n, np.complex128)
    c[0] = col[0]
    for i in range(1, n):
        c[i] = ((n - i) * col[i] + i * row[n - i]) / n
    return c


def chan_along_axis(gen, axis):
    """circulant.py:61-73 -- odd axis of offsets -(n-1)..n-1 -> n generators."""
    g = np.moveaxis(gen, axis, -1)
    n = (g.shape[-1] + 1) // 2
    s = np.arange(1, n)
    out = np.empty(g.shape[:-1] + (n,), np.complex128)
    out[..., 0] = g[..., n - 1]
    out[..., 1:] = ((n - s) * g[..., n - 1 + s] + s * g[..., s - 1]) / n
    return np.moveaxis(out, -1, axis)


def chan_x_spectra(tensors):
    """circulant.py:129-136 -- lamhat (6, 2nz-1, 2ny-1, nx)."""
    return scipy.fft.fft(chan_along_axis(tensors, axis=3), axis=3)


def unfold_block_yz(lam, m_yz):
    """accel.py:71-91 -- D = I - diag(m) N_k, rows/cols a*q + iz*ny + iy."""
    nz, ny = (lam.shape[1] + 1) // 2, (lam.shape[2] + 1) // 2
    q = ny * nz
    zi, yi = [a.reshape(-1) for a in np.meshgrid(np.arange(nz), np.arange(ny), indexing="ij")]
    idx = (zi[:, None] - zi[None, :] + nz - 1) * (2 * ny - 1) + (yi[:, None] - yi[None, :] + ny - 1)
    blk = lam.reshape(6, -1)[:, idx]
    nm = np.empty((3 * q, 3 * q), np.complex128)
    for a in range(3):
        for b in range(3):
            nm[a * q:(a + 1) * q, b * q:(b + 1) * q] = blk[PAIR_OF[a, b]]
    out = -np.tile(m_yz.reshape(-1), 3)[:, None] * nm
    out[np.diag_indices_from(out)] += 1.0
    return out


def unfold_block_z(lam, m_z):
    """accel.py:94-111 -- (3nz)^2 block for the 2-level scheme."""
    nz = (lam.shape[1] + 1) // 2
    iz = np.arange(nz)
    blk = lam[:, iz[:, None] - iz[None, :] + nz - 1]
    nm = np.empty((3 * nz, 3 * nz), np.complex128)
    for a in range(3):
        for b in range(3):
            nm[a * nz:(a + 1) * nz, b * nz:(b + 1) * nz] = blk[PAIR_OF[a, b]]
    out = -np.tile(np.asarray(m_z).reshape(-1), 3)[:, None] * nm
    out[np.diag_indices_from(out)] += 1.0
    return out


def coerce_mtilde(dims, mtilde):
    """circulant.py:81-96 -- x-constant map -> (nz, ny)."""
    nx, ny, nz = dims
    m = np.asarray(mtilde, np.complex128)
    if m.shape == (nz, ny, nx):
        lead = m[:, :, :1]
        if not np.allclose(m, lead, rtol=0.0, atol=1e-12 * max(1.0, np.abs(m).max())):
            raise ValueError("homogenized coefficient must be constant along x")
        return m[:, :, 0]
    if m.shape == (nz, ny):
        return m
    raise ValueError("mtilde shape not compatible")


def lu_checked(block):
    """circulant.py:113-118."""
    lu, piv = lu_factor(block, check_finite=False)
    d = np.abs(np.diag(lu))
    if not np.all(np.isfinite(d)) or np.any(d == 0.0):
        raise ZeroDivisionError("singular block")
    return lu, piv


def build_one_level(tensors, dims, mtilde):
    """circulant.py:191-225 -> dict(lu, piv, proxy)."""
    nx, ny, nz = dims
    m_yz = coerce_mtilde(dims, mtilde)
    q = ny * nz
    lam = chan_x_spectra(tensors)
    c0 = ny * nz - 1  # circulant.py:99-110
    lu = np.empty((nx, 3 * q, 3 * q), np.complex128)
    piv = np.empty((nx, 3 * q), np.int32)
    proxy = np.empty(nx, np.complex128)
    for k in range(nx):
        blk = unfold_block_yz(lam[:, :, :, k], m_yz)
        proxy[k] = blk[0, c0]
        lu[k], piv[k] = lu_checked(blk)
    return dict(kind="one-level", dims=dims, lu=lu, piv=piv, proxy=proxy)


def select_kept(proxy, nx, tol):
    """circulant.py:283-294."""
    if not 0.0 <= tol <= 1.0:
        raise ValueError("reduction tolerance must lie in [0, 1]")
    vmax = np.abs(proxy).max()
    vhat = np.abs(proxy) / vmax if vmax > 0 else np.zeros(proxy.shape)
    rep = int(np.ceil(nx / 2)) - 1
    mask = vhat > tol
    mask[rep] = True
    kept = np.flatnonzero(mask)
    slot_of = np.full(nx, int(np.searchsorted(kept, rep)), dtype=np.int64)
    slot_of[kept] = np.arange(kept.size)
    return kept, slot_of, rep, vhat


def reduce_one_level(prec, tol):
    """circulant.py:297-311."""
    nx = prec["dims"][0]
    kept, slot_of, rep, vhat = select_kept(prec["proxy"], nx, tol)
    return dict(kind="reduced-one-level", dims=prec["dims"], kept=kept, slot_of=slot_of,
                representative=rep, lu=prec["lu"][kept].copy(), piv=prec["piv"][kept].copy(),
                proxy=prec["proxy"].copy(), proxy_normalized=vhat)


def build_reduced_one_level(tensors, dims, mtilde, tol):
    """circulant.py:314-354 (analytic proxy, LU only for kept blocks)."""
    nx, ny, nz = dims
    m_yz = coerce_mtilde(dims, mtilde)
    q = ny * nz
    lam = chan_x_spectra(tensors)
    c0 = ny * nz - 1
    jz, jy = divmod(c0, ny)
    proxy = (1.0 if c0 == 0 else 0.0) + -m_yz[0, 0] * lam[0, nz - 1 - jz, ny - 1 - jy, :]
    kept, slot_of, rep, vhat = select_kept(proxy, nx, tol)
    lu = np.empty((kept.size, 3 * q, 3 * q), np.complex128)
    piv = np.empty((kept.size, 3 * q), np.int32)
    for s, k in enumerate(kept):
        lu[s], piv[s] = lu_checked(unfold_block_yz(lam[:, :, :, k], m_yz))
    return dict(kind="reduced-one-level", dims=dims, kept=kept, slot_of=slot_of,
                representative=rep, lu=lu, piv=piv, proxy=proxy, proxy_normalized=vhat)


def _solve_blocks_x(dims, x, factor_of):
    """circulant.py:174-188 -- DFT_x, per-frequency lu_solve, inverse DFT."""
    nx, ny, nz = dims
    x = np.asarray(x, np.complex128)
    flat = x.ndim == 1
    x2 = x.reshape(3 * nx * ny * nz, -1)
    r = x2.shape[1]
    spec = scipy.fft.fft(x2.reshape(3, nz, ny, nx, r), axis=3)
    for k in range(nx):
        rhs = np.ascontiguousarray(spec[:, :, :, k, :]).reshape(-1, r)
        spec[:, :, :, k, :] = lu_solve(factor_of(k), rhs, check_finite=False).reshape(3, nz, ny, r)
    out = scipy.fft.ifft(spec, axis=3).reshape(x2.shape)
    return out.reshape(-1) if flat else out.reshape(x.shape)


def build_two_level(tensors, dims, mtilde):
    """circulant.py:405-447 -> dict(lu (ny,nx,3nz,3nz), piv)."""
    nx, ny, nz = dims
    m = np.asarray(mtilde, np.complex128)
    if m.shape == (nz, ny, nx):
        m_z = m[:, 0, 0]
    elif m.shape == (nz,):
        m_z = m
    elif m.ndim == 0:
        m_z = np.full(nz, m, np.complex128)
    else:
        raise ValueError("mtilde shape not usable for a 2-level build")
    lam = scipy.fft.fftn(chan_along_axis(chan_along_axis(tensors, 3), 2), axes=(2, 3))
    lu = np.empty((ny, nx, 3 * nz, 3 * nz), np.complex128)
    piv = np.empty((ny, nx, 3 * nz), np.int32)
    for l in range(ny):
        for k in range(nx):
            lu[l, k], piv[l, k] = lu_checked(unfold_block_z(lam[:, :, l, k], m_z))
    return dict(kind="two-level", dims=dims, lu=lu, piv=piv)


def apply_two_level(prec, x):
    """circulant.py:379-394."""
    nx, ny, nz = prec["dims"]
    x = np.asarray(x, np.complex128)
    flat = x.ndim == 1
    x2 = x.reshape(3 * nx * ny * nz, -1)
    r = x2.shape[1]
    spec = scipy.fft.fftn(x2.reshape(3, nz, ny, nx, r), axes=(2, 3))
    for l in range(ny):
        for k in range(nx):
            rhs = np.ascontiguousarray(spec[:, :, l, k, :]).reshape(-1, r)
            spec[:, :, l, k, :] = lu_solve((prec["lu"][l, k], prec["piv"][l, k]), rhs,
                                           check_finite=False).reshape(3, nz, r)
    out = scipy.fft.ifftn(spec, axes=(2, 3)).reshape(x2.shape)
    return out.reshape(-1) if flat else out.reshape(x.shape)


def apply_prec(prec, x):
    """Dispatch: OneLevelPrec.apply (circulant.py:162-163), Reduced (264-269),
    TwoLevel (379-394), Blocked (558-563)."""
    kind = prec["kind"]
    if kind == "one-level":
        return _solve_blocks_x(prec["dims"], x, lambda k: (prec["lu"][k], prec["piv"][k]))
    if kind == "reduced-one-level":
        so = prec["slot_of"]
        return _solve_blocks_x(prec["dims"], x, lambda k: (prec["lu"][so[k]], prec["piv"][so[k]]))
    if kind == "two-level":
        return apply_two_level(prec, x)
    if kind == "blocked":
        x = np.asarray(x, np.complex128)
        y = x.copy()
        for p, dofs in zip(prec["box_precs"], prec["box_dofs"]):
            y[dofs] = apply_prec(p, x[dofs])
        return y
    raise ValueError(kind)


def slice_kernel(tensors, dims, box):
    """circulant.py:577-600 -- box = (x0,x1,y0,y1,z0,z1)."""
    nx, ny, nz = dims
    x0, x1, y0, y1, z0, z1 = box
    bx, by, bz = x1 - x0, y1 - y0, z1 - z0
    cz, cy, cx = nz - 1, ny - 1, nx - 1
    sub = tensors[:, cz - (bz - 1):cz + bz, cy - (by - 1):cy + by, cx - (bx - 1):cx + bx]
    return np.ascontiguousarray(sub), (bx, by, bz)


def box_dof_indices(dims, box):
    """circulant.py:603-607."""
    nx, ny, nz = dims
    x0, x1, y0, y1, z0, z1 = box
    idx = np.arange(3 * nx * ny * nz).reshape(3, nz, ny, nx)
    return np.ascontiguousarray(idx[:, z0:z1, y0:y1, x0:x1]).reshape(-1)


def build_blocked(tensors, dims, boxes, levels, mtildes, reduce_tol=1e-3):
    """circulant.py:610-651 with the per-box homogenised maps supplied."""
    precs, dofs = [], []
    for box, lvl, mt in zip(boxes, levels, mtildes):
        sub, sdims = slice_kernel(tensors, dims, box)
        if lvl == "one-level":
            p = build_one_level(sub, sdims, mt)
        elif lvl == "reduced-one-level":
            p = build_reduced_one_level(sub, sdims, mt, reduce_tol)
        elif lvl == "two-level":
            p = build_two_level(sub, sdims, mt)
        else:
            raise ValueError(lvl)
        precs.append(p)
        dofs.append(box_dof_indices(dims, box))
    return dict(kind="blocked", dims=dims, box_precs=precs, box_dofs=dofs)


def wrap_circulant_x(tensors, nx):
    """circulant.py:659-669."""
    t = tensors.copy()
    t[..., :nx - 1] = t[..., nx:2 * nx - 1]
    return t


def wrap_circulant_xy(tensors, nx, ny):
    """circulant.py:672-677."""
    t = wrap_circulant_x(tensors, nx)
    t[:, :, :ny - 1, :] = t[:, :, ny:2 * ny - 1, :]
    return t


def dense_chan_circulant_x(tensors, dims, mtilde):
    """test_circulant.py:107-116 -- dense system of the x-Chan-circulant kernel."""
    nx = dims[0]
    chan = chan_along_axis(tensors, 3)
    g = np.empty_like(tensors)
    g[..., nx - 1:] = chan
    g[..., :nx - 1] = chan[..., 1:]
    return dense_operator(g, dims, mtilde)


def dense_chan_circulant_xy(tensors, dims, mtilde):
    """test_circulant.py:119-128."""
    nx, ny = dims[0], dims[1]
    chan = chan_along_axis(chan_along_axis(tensors, 3), 2)
    g = np.empty_like(tensors)
    g[..., ny - 1:, nx - 1:] = chan
    g[..., :ny - 1, nx - 1:] = chan[..., 1:, :]
    g[..., ny - 1:, :nx - 1] = chan[..., :, 1:]
    g[..., :ny - 1, :nx - 1] = chan[..., 1:, 1:]
    return dense_operator(g, dims, mtilde)


# ----------------------------------------------------------------------------
# GMRES (reference solver.py:45-174)
# ----------------------------------------------------------------------------

class Breakdown(Exception):
    pass


def _cycle(op, r0, beta, bnorm, tol, m, hist):
    """solver.py:45-111 -- MGS + one DGKS pass, complex Givens."""
    V = [r0 / beta]
    rcols, cs, sn = [], [], []
    g = [beta + 0.0j]
    conv = lucky = False
    j = 0
    while j < m:
        w = np.array(op(V[j]), dtype=np.complex128)
        n0 = np.linalg.norm(w)
        h = np.empty(j + 2, np.complex128)
        for i in range(j + 1):
            h[i] = np.vdot(V[i], w)
            w -= h[i] * V[i]
        if np.linalg.norm(w) < 0.7071 * n0:
            for i in range(j + 1):
                c = np.vdot(V[i], w)
                h[i] += c
                w -= c * V[i]
        h[j + 1] = np.linalg.norm(w)
        lucky = h[j + 1].real <= 1e-14 * max(n0.real, 1e-300)
        if not lucky:
            V.append(w / h[j + 1])
        for i in range(j):
            hi = h[i]
            h[i] = np.conj(cs[i]) * hi + np.conj(sn[i]) * h[i + 1]
            h[i + 1] = -sn[i] * hi + cs[i] * h[i + 1]
        den = np.hypot(abs(h[j]), abs(h[j + 1]))
        if den == 0.0:
            raise Breakdown("zero Hessenberg column")
        c, s = h[j] / den, h[j + 1] / den
        cs.append(c)
        sn.append(s)
        h[j] = np.conj(c) * h[j] + np.conj(s) * h[j + 1]
        rcols.append(h[:j + 1].copy())
        g.append(-s * g[j])
        g[j] = np.conj(c) * g[j]
        j += 1
        est = abs(g[j]) / bnorm
        hist.append(float(est))
        if est <= tol or lucky:
            conv = est <= tol
            if lucky and not conv:
                raise Breakdown("Arnoldi breakdown")
            break
    R = np.zeros((j, j), np.complex128)
    for col, v in enumerate(rcols):
        R[:col + 1, col] = v
    y = np.linalg.solve(R, np.asarray(g[:j]))
    return np.stack(V[:j], axis=1) @ y, j, conv


def gmres(apply_a, b, apply_pinv=None, tol=1e-4, maxit=2000, restart=None):
    """solver.py:114-174 -> (x, dict(iterations, residuals, converged, true_residual))."""
    b = np.asarray(b, np.complex128).reshape(-1)
    bnorm = np.linalg.norm(b)
    if bnorm == 0.0:
        return np.zeros_like(b), dict(iterations=1, residuals=[1.0, 0.0], converged=True,
                                      true_residual=0.0)
    op = apply_a if apply_pinv is None else (lambda v: apply_a(apply_pinv(v)))
    x = np.zeros_like(b)
    hist = [1.0]
    total = 0
    conv = False
    while total < maxit and not conv:
        r0 = b - apply_a(x) if total else b.copy()
        beta = np.linalg.norm(r0)
        if beta / bnorm <= tol:
            conv = True
            break
        m = maxit - total if restart is None else min(restart, maxit - total)
        u, used, conv = _cycle(op, r0, beta, bnorm, tol, m, hist)
        total += used
        x = x + (u if apply_pinv is None else apply_pinv(u))
    tr = float(np.linalg.norm(b - apply_a(x)) / bnorm)
    return x, dict(iterations=int(total), residuals=hist, converged=bool(conv), true_residual=tr)
