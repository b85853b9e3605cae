"""Symmetry-sector factorisation of the 1-level blocks (sectors.py): the
sector path equals the dense-block path (VX_SECTORS=0) and the CPU oracle,
with and without mirror sharing, for 1 and several right-hand sides."""

import numpy as np
import pytest

import voxvie_oracle as O
from conftest import random_field, relerr

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def C():
    from paper_1903_07884_b200 import circulant

    return circulant


def _wl(dims, delta=0.02e-6):
    from paper_1903_07884_b200 import workloads

    return workloads.small(*dims, delta=delta)


def _sym_m(rng, nz, ny, nx, sy, sz):
    m = 0.6 + 0.3 * rng.random((nz, ny)) - 0.02j * rng.random((nz, ny))
    if sy:
        m = 0.5 * (m + m[:, ::-1])
    if sz:
        m = 0.5 * (m + m[::-1, :])
    return np.repeat(m[:, :, None], nx, axis=2)


@pytest.mark.parametrize("dims,sy,sz,nsec", [((8, 3, 2), True, True, 4), ((12, 4, 3), True, True, 4),
                                             ((9, 6, 5), True, False, 2), ((10, 5, 4), False, True, 2),
                                             ((50, 22, 11), True, True, 4), ((7, 9, 3), False, False, 1)])
def test_sectors_equal_dense_blocks(rng, C, monkeypatch, dims, sy, sz, nsec):
    nx, ny, nz = dims
    W = _wl(dims)
    kern = W.kernel()
    m = _sym_m(rng, nz, ny, nx, sy, sz)
    if not sy and ny > 1:
        m[:, 0, :] += 0.05
    if not sz and nz > 1:
        m[0, :, :] += 0.07
    p = C.build_one_level(kern, m)
    assert p.sectors == nsec
    monkeypatch.setenv("VX_SECTORS", "0")
    q = C.build_one_level(kern, m)
    monkeypatch.delenv("VX_SECTORS")
    assert q.sectors == 1
    n = W.grid.n_unknowns
    for r in (None, 3):
        x = random_field(rng, n, r)
        assert relerr(p.apply(x), q.apply(x)) < 1e-12
    if n <= 3 * 12 * 4 * 3:
        ref = O.build_one_level(kern.tensors, W.grid.dims, m)
        x = random_field(rng, n)
        assert relerr(p.apply(x), O.apply_prec(ref, x)) < 1e-10
        assert np.array_equal(p.piv, q.piv) and relerr(p.lu, q.lu) < 1e-13
    if nsec > 1:
        sb = p.stored_blocks
        assert sum(d for d, _ in sb) == p.block_size
        assert sum(d * d * c for d, c in sb) < 0.6 * p.block_size ** 2 * q.stored_slots


def test_sectors_without_mirror(rng, C, monkeypatch):
    W = _wl((10, 6, 3))
    kern, mt = W.kernel(), W.mtilde()
    p = C.build_one_level(kern, mt)
    monkeypatch.setenv("VX_MIRROR", "0")
    q = C.build_one_level(kern, mt)
    monkeypatch.setenv("VX_SECTORS", "0")
    d = C.build_one_level(kern, mt)
    assert p.sectors == 4 and q.sectors == 4 and d.sectors == 1
    assert p.mirror_shared and not q.mirror_shared
    x = random_field(rng, W.grid.n_unknowns)
    assert relerr(p.apply(x), d.apply(x)) < 1e-12
    assert relerr(q.apply(x), d.apply(x)) < 1e-12


def test_sector_reduce_and_classic_solve(rng, C, monkeypatch):
    from paper_1903_07884_b200 import _native as nv

    W = _wl((40, 12, 4))
    kern, mt = W.kernel(), W.mtilde()
    p = C.build_one_level(kern, mt)
    assert p.sectors == 4
    ref = O.build_one_level(kern.tensors, W.grid.dims, mt)
    x = random_field(rng, W.grid.n_unknowns)
    red = C.reduce_one_level(p, 1e-3)
    rref = O.reduce_one_level(ref, 1e-3)
    assert red.sectors == 4
    assert relerr(red.apply(x), O.apply_prec(rref, x)) < 1e-10
    red2 = C.build_reduced_one_level(kern, mt, 1e-3)
    assert red2.sectors == 4 and np.array_equal(red2.kept, rref["kept"])
    for r in (None, 2):
        xr = random_field(rng, W.grid.n_unknowns, r)
        assert relerr(red2.apply(xr), O.apply_prec(rref, xr)) < 1e-10
    assert np.array_equal(red2.piv, red.piv)
    nv.call("vx_solve_variant", 1)
    try:
        assert relerr(p.apply(x), O.apply_prec(ref, x)) < 1e-10
    finally:
        nv.call("vx_solve_variant", 0)


def test_sector_singular_block_raises(C):
    """D_k = (1 - m s) I: singular for m = 1/s in every sector; the message names k."""
    from paper_1903_07884_b200.errors import PreconditionerBuildError
    from paper_1903_07884_b200.grid import VoxelGrid
    from paper_1903_07884_b200.kernel import ToeplitzKernel

    dims = (4, 3, 2)
    t = np.zeros((6, 3, 5, 7), dtype=complex)
    t[[0, 3, 5], 1, 2, 3] = 2.0
    kern = ToeplitzKernel(VoxelGrid(*dims, 0.05), 2 * np.pi, t)
    with pytest.raises(PreconditionerBuildError, match="k=0"):
        C.build_one_level(kern, np.full((2, 3, 4), 0.5))
    ok = C.build_one_level(kern, np.full((2, 3, 4), 0.25))
    assert ok.sectors == 4
    x = np.arange(72, dtype=complex)
    assert relerr(ok.apply(x), 2 * x) < 1e-14


@pytest.mark.parametrize("tol", [1e-3, 0.3])
def test_sector_reduced_representative_gemm(rng, C, monkeypatch, tol):
    """Reduced scheme on sector factors: the discarded frequencies go through
    one GEMM per sector with the representative sector block's explicit
    inverse (side stream), the kept ones through the ragged sector solves;
    equal to the chunked representative solves (VX_REP_GEMM=0) and the oracle."""
    W = _wl((64, 10, 6))          # 3q = 180: sectors of 45 rows (> one tile)
    kern, mt = W.kernel(), W.mtilde()
    red = C.build_reduced_one_level(kern, mt, tol)
    assert red.sectors == 4 and red._inv is not None and red.factor_layout in ("ragged", "symmetric", "symmetric-inverse")
    assert int(red._rep_ks.numel()) >= 8
    monkeypatch.setenv("VX_REP_GEMM", "0")
    chunked = C.build_reduced_one_level(kern, mt, tol)
    monkeypatch.delenv("VX_REP_GEMM")
    assert chunked._inv is None
    ref = O.build_reduced_one_level(kern.tensors, W.grid.dims, mt, tol)
    assert np.array_equal(red.kept, ref["kept"])
    for r in (None, 3):
        x = random_field(rng, W.grid.n_unknowns, r)
        y = red.apply(x)
        assert relerr(y, O.apply_prec(ref, x)) < 1e-10
        assert relerr(y, chunked.apply(x)) < 1e-12


@pytest.mark.parametrize("dims", [(50, 22, 11), (40, 12, 4), (64, 10, 6), (30, 16, 9)])
def test_symmetric_factors_equal_pivoted(rng, C, monkeypatch, dims):
    """Symmetric sector factors (unpivoted L, U = diag(u) W L^T W^-1; half the
    stored bytes) give the same P^-1 x as the pivoted LU factors (VX_SYM=0),
    for one right-hand side (symmetric solve kernel) and several (unpacked
    padded layout); the LAPACK views are the pivoted dense ones."""
    W = _wl(dims)
    kern, mt = W.kernel(), W.mtilde()
    p = C.build_one_level(kern, mt)
    monkeypatch.setenv("VX_SYM", "0")
    q = C.build_one_level(kern, mt)
    monkeypatch.delenv("VX_SYM")
    assert p.factor_layout.startswith("symmetric") and q.factor_layout == "ragged"
    # lower triangle + the 8-row-block trapezoid of the diagonal tiles: ~0.53 of the LU bytes
    # for c1-size sectors, more for blocks of only two tiles
    assert p.factor_bytes_per_apply < (0.56 if p.block_size > 500 else 0.66) * q.storage_bytes
    # resident: the factors (views, multi-RHS applies) and, when verified, the inverses the applies stream
    assert p.storage_bytes == p.factor_bytes_per_apply * (2 if p.factor_layout == "symmetric-inverse" else 1)
    n = W.grid.n_unknowns
    for r in (None, 2):
        x = random_field(rng, n, r)
        assert relerr(p.apply(x), q.apply(x)) < 1e-12
    if n <= 3 * 40 * 12 * 4:
        ref = O.build_one_level(kern.tensors, W.grid.dims, mt)
        x = random_field(rng, n)
        assert relerr(p.apply(x), O.apply_prec(ref, x)) < 1e-10
        assert np.array_equal(p.piv, q.piv)


def test_symmetric_factors_not_used_with_zero_coefficients(rng, C):
    """m~ with a zero row (cladding with eps = 1 in interpretation B) breaks
    S M^-1 D symmetry: the pivoted ragged layout is kept."""
    W = _wl((40, 12, 4))
    m = np.repeat(W.mtilde()[:, :, :1], 40, axis=2).copy()
    m[:, 0, :] = 0.0
    m[:, -1, :] = 0.0
    p = C.build_one_level(W.kernel(), m)
    assert p.sectors > 1 and p.factor_layout == "ragged"
    ref = O.build_one_level(W.kernel().tensors, W.grid.dims, m)
    x = random_field(rng, W.grid.n_unknowns)
    assert relerr(p.apply(x), O.apply_prec(ref, x)) < 1e-10


def test_symmetric_reduced_and_solve(rng, C, monkeypatch):
    """Reduced scheme with symmetric kept factors + representative GEMM, and a
    full GMRES solve on symmetric factors vs the pivoted layout."""
    from paper_1903_07884_b200.operator import apply_system, plan_operator
    from paper_1903_07884_b200.solver import gmres

    W = _wl((64, 10, 6))
    kern, mt = W.kernel(), W.mtilde()
    red = C.build_reduced_one_level(kern, mt, 0.3)
    assert red.factor_layout.startswith("symmetric") and red._inv is not None
    ref = O.build_reduced_one_level(kern.tensors, W.grid.dims, mt, 0.3)
    x = random_field(rng, W.grid.n_unknowns)
    assert relerr(red.apply(x), O.apply_prec(ref, x)) < 1e-10
    plan = plan_operator(kern)
    p = C.build_one_level(kern, mt)
    monkeypatch.setenv("VX_SYM", "0")
    q = C.build_one_level(kern, mt)
    monkeypatch.delenv("VX_SYM")
    A = lambda v: apply_system(plan, W.m, v)  # noqa: E731
    x1, r1 = gmres(A, W.b, apply_pinv=p.apply, tol=1e-10, maxit=300)
    x2, r2 = gmres(A, W.b, apply_pinv=q.apply, tol=1e-10, maxit=300)
    assert r1.iterations == r2.iterations and relerr(x1, x2) < 1e-9


@pytest.mark.parametrize("dims", [(50, 22, 11), (40, 12, 4), (30, 16, 9), (33, 14, 12)])
def test_symmetric_inverse_equals_factors(rng, C, monkeypatch, dims):
    """The one-pass symmetric-inverse apply (G = A^^-1, x = G (b / W), csrc/lu_syminv.cuh)
    equals the two triangular sweeps on the symmetric factors (VX_SYMINV=0) and the
    pivoted LU (VX_SYM=0); it is bitwise reproducible; several right-hand sides still
    go through the factors; block sizes with full and ragged last tile rows
    (sector dims 176..187, 36, 108, 126)."""
    W = _wl(dims)
    kern, mt = W.kernel(), W.mtilde()
    p = C.build_one_level(kern, mt)
    monkeypatch.setenv("VX_SYMINV", "0")
    f = C.build_one_level(kern, mt)
    monkeypatch.delenv("VX_SYMINV")
    monkeypatch.setenv("VX_SYM", "0")
    q = C.build_one_level(kern, mt)
    monkeypatch.delenv("VX_SYM")
    assert (p.factor_layout, f.factor_layout, q.factor_layout) == ("symmetric-inverse", "symmetric", "ragged")
    assert p._syminv_err < 1e-12
    n = W.grid.n_unknowns
    x = random_field(rng, n)
    y = p.apply(x)
    assert np.array_equal(y, p.apply(x))
    assert relerr(y, f.apply(x)) < 1e-12
    assert relerr(y, q.apply(x)) < 1e-12
    x3 = random_field(rng, n, 3)
    assert relerr(p.apply(x3), q.apply(x3)) < 1e-12
    if n <= 3 * 40 * 12 * 4:
        ref = O.build_one_level(kern.tensors, W.grid.dims, mt)
        assert relerr(y, O.apply_prec(ref, x)) < 1e-10


def test_symmetric_inverse_rejected_when_inaccurate(rng, C, monkeypatch):
    """The inverses are kept only if one apply agrees with the triangular solves:
    with an impossible tolerance the factors stay in use."""
    W = _wl((40, 12, 4))
    monkeypatch.setattr(C, "SYMINV_TOL", 0.0)
    p = C.build_one_level(W.kernel(), W.mtilde())
    assert p.factor_layout == "symmetric" and p._sym.inv is None
    ref = O.build_one_level(W.kernel().tensors, W.grid.dims, W.mtilde())
    x = random_field(rng, W.grid.n_unknowns)
    assert relerr(p.apply(x), O.apply_prec(ref, x)) < 1e-10


@pytest.mark.parametrize("scale", [1.0, 4.0, 12.0, 40.0])
def test_symmetric_paths_stay_accurate_for_strong_contrast(rng, C, scale):
    """Stronger contrast (|m~| up to 40 x the waveguide's) makes the blocks D_k = I - M N_k far from
    diagonally dominant and worse conditioned: whichever layout the build keeps (symmetric inverse,
    symmetric factors after a rejected inverse, or the pivoted LU after a rejected unpivoted
    factorisation), P^-1 x agrees with the oracle's zgetrs to 1e-10 x max(1, cond / 100)."""
    W = _wl((24, 12, 4))
    kern = W.kernel()
    nx, ny, nz = W.grid.dims
    m = _sym_m(rng, nz, ny, nx, True, True) * scale
    p = C.build_one_level(kern, m)
    ref = O.build_one_level(kern.tensors, W.grid.dims, m)
    lam = O.chan_x_spectra(kern.tensors)
    cond = max(np.linalg.cond(O.unfold_block_yz(lam[:, :, :, k], m[:, :, 0])) for k in (0, 1, nx // 2))
    x = random_field(rng, W.grid.n_unknowns)
    err = relerr(p.apply(x), O.apply_prec(ref, x))
    assert err < 1e-10 * max(1.0, cond / 100.0), (p.factor_layout, cond, err)
