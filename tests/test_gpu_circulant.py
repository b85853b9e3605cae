"""GPU parity for the circulant preconditioners: golden vectors produced by the
reference, the reference test-suite's own properties (test_circulant.py), and
the CPU oracle."""

import numpy as np
import pytest
import scipy.fft

import voxvie_oracle as O
from conftest import random_field, relerr

pytestmark = pytest.mark.gpu

PC_TAGS = ["wg", "pr", "py", "sq"]


def _kern(tensors, dims, delta=0.05):
    from paper_1903_07884_b200.grid import VoxelGrid
    from paper_1903_07884_b200.kernel import ToeplitzKernel

    return ToeplitzKernel(VoxelGrid(*dims, delta), 2 * np.pi, tensors)


@pytest.fixture(scope="module")
def C():
    from paper_1903_07884_b200 import circulant

    return circulant


@pytest.fixture(scope="module")
def wg(C):
    from paper_1903_07884_b200.grid import PermittivityMap, VoxelGrid, homogenize
    from paper_1903_07884_b200.kernel import assemble_kernel

    grid = VoxelGrid(8, 3, 2, 0.05)
    kern = assemble_kernel(grid, 2 * np.pi)
    mt = homogenize(PermittivityMap(grid, np.full(grid.shape, 5.8, dtype=complex)), "real_mean_x")
    return kern, mt


# ------------------------------------------------------------------ golden
@pytest.mark.parametrize("tag", PC_TAGS)
def test_one_level_golden(golden_small, C, tag):
    g = golden_small
    dims = tuple(int(v) for v in g[f"pc_{tag}_dims"])
    kern = _kern(g[f"pc_{tag}_tensors"], dims)
    p1 = C.build_one_level(kern, g[f"pc_{tag}_mtilde"])
    assert relerr(p1.proxy, g[f"pc_{tag}_one_proxy"]) < 1e-13
    assert relerr(p1.apply(g[f"pc_{tag}_x"]), g[f"pc_{tag}_one_y"]) < 1e-10
    assert relerr(p1.apply(g[f"pc_{tag}_xr"]), g[f"pc_{tag}_one_yr"]) < 1e-10
    red = C.reduce_one_level(p1, 0.3)
    assert np.array_equal(red.kept, g[f"pc_{tag}_red_kept"])
    assert np.array_equal(red.slot_of, g[f"pc_{tag}_red_slot"])
    assert relerr(red.apply(g[f"pc_{tag}_x"]), g[f"pc_{tag}_red_y"]) < 1e-10
    red2 = C.build_reduced_one_level(kern, g[f"pc_{tag}_mtilde"], 0.3)
    assert np.array_equal(red2.kept, g[f"pc_{tag}_red2_kept"])
    assert relerr(red2.proxy, g[f"pc_{tag}_red2_proxy"]) < 1e-13
    assert relerr(red2.apply(g[f"pc_{tag}_x"]), g[f"pc_{tag}_red2_y"]) < 1e-10


@pytest.mark.parametrize("tag", PC_TAGS)
def test_two_level_golden(golden_small, C, tag):
    g = golden_small
    dims = tuple(int(v) for v in g[f"pc_{tag}_dims"])
    p2 = C.build_two_level(_kern(g[f"pc_{tag}_tensors"], dims), g[f"pc_{tag}_m2"])
    assert relerr(p2.apply(g[f"pc_{tag}_x"]), g[f"pc_{tag}_two_y"]) < 1e-10
    assert relerr(p2.apply(g[f"pc_{tag}_xr"]), g[f"pc_{tag}_two_yr"]) < 1e-10


def test_blocked_golden(golden_small, C):
    from paper_1903_07884_b200.grid import PermittivityMap, VoxelGrid

    g = golden_small
    grid = VoxelGrid(8, 6, 2, 0.05)
    kern = _kern(g["blk_tensors"], (8, 6, 2))
    pmap = PermittivityMap(grid, g["blk_eps"])
    part = C.partition_boxes(grid, [C.Box("lo", 0, 8, 0, 3, 0, 2), C.Box("hi", 0, 8, 3, 6, 0, 2)])
    bp = C.build_blocked(kern, pmap, part, {"lo": "one-level", "hi": "two-level"})
    assert relerr(bp.apply(g["blk_x"]), g["blk_y"]) < 1e-10
    part2 = C.partition_boxes(grid, [C.Box("a", 1, 7, 1, 5, 0, 2)])
    bp2 = C.build_blocked(kern, pmap, part2, {"a": "reduced-one-level"}, reduce_tol=0.2)
    assert relerr(bp2.apply(g["blk_x"]), g["blk2_y"]) < 1e-10


# --------------------------------------------- reference test-suite mirrors
def test_one_level_air_identity(C, wg, rng):
    kern, _ = wg
    prec = C.build_one_level(kern, np.zeros(kern.grid.shape))
    x = random_field(rng, kern.grid.n_unknowns)
    assert np.abs(prec.apply(x) - x).max() < 1e-12 * np.abs(x).max()


def test_one_level_inverts_dense_chan_circulant(C, wg, rng):
    kern, mt = wg
    prec = C.build_one_level(kern, mt)
    c = O.dense_chan_circulant_x(kern.tensors, kern.grid.dims, mt)
    x = random_field(rng, kern.grid.n_unknowns)
    assert np.abs(c @ prec.apply(x) - x).max() / np.abs(x).max() < 1e-12


def test_one_level_linearity(C, wg, rng):
    kern, mt = wg
    prec = C.build_one_level(kern, mt)
    x1, x2 = random_field(rng, kern.grid.n_unknowns), random_field(rng, kern.grid.n_unknowns)
    lhs = prec.apply(2.0 * x1 + 1j * x2)
    rhs = 2.0 * prec.apply(x1) + 1j * prec.apply(x2)
    assert np.abs(lhs - rhs).max() / np.abs(lhs).max() < 1e-12


def test_one_level_exact_inverse_on_wrapped_kernel(C, wg, rng):
    from paper_1903_07884_b200.solver import gmres

    kern, _ = wg
    wrapped = C.wrap_circulant_x(kern)
    m = np.full(kern.grid.shape, 0.7 + 0.05j)
    a = O.dense_operator(wrapped.tensors, kern.grid.dims, m)
    prec = C.build_one_level(wrapped, m)
    b = random_field(rng, kern.grid.n_unknowns)
    x, rep = gmres(lambda v: a @ v, b, apply_pinv=prec.apply, tol=1e-10, maxit=10)
    assert rep.converged and rep.iterations <= 2


def test_one_level_guards(C, wg, rng):
    from paper_1903_07884_b200.errors import PreconditionerBuildError

    kern, mt = wg
    with pytest.raises(ValueError, match="constant along x"):
        C.build_one_level(kern, rng.normal(size=kern.grid.shape))
    with pytest.raises(PreconditionerBuildError, match="2-level"):
        C.build_one_level(kern, mt, cap_bytes=1024)
    prec = C.build_one_level(kern, mt)
    nx, ny, nz = kern.grid.dims
    assert prec.bytes == nx * (3 * ny * nz) ** 2 * 16
    assert prec.summary()["bytes"] == prec.bytes


def test_one_level_proxy_characterisation_against_dense(C, wg):
    kern, mt = wg
    prec = C.build_one_level(kern, mt)
    nz, ny, nx = kern.grid.shape
    q = ny * nz
    c8 = O.dense_chan_circulant_x(kern.tensors, kern.grid.dims, mt).reshape(3, nz, ny, nx, 3, nz, ny, nx)
    bs = np.stack([c8[:, :, :, s, :, :, :, 0].reshape(3 * q, 3 * q) for s in range(nx)])
    proxy = prec.proxy
    for k in range(nx):
        dk = np.tensordot(np.exp(-2j * np.pi * k * np.arange(nx) / nx), bs, axes=1)
        assert proxy[k] == pytest.approx(dk[0, q - 1], rel=1e-10)


def test_lu_and_piv_reconstruct_blocks(C, wg):
    """.lu/.piv (LAPACK layout) reproduce P D_k = L U for every frequency block."""
    kern, mt = wg
    prec = C.build_one_level(kern, mt)
    lam = O.chan_x_spectra(kern.tensors)
    m_yz = mt[:, :, 0]
    lu, piv = prec.lu, prec.piv
    for k in range(kern.grid.nx):
        d = O.unfold_block_yz(lam[:, :, :, k], m_yz)
        L = np.tril(lu[k], -1) + np.eye(d.shape[0])
        U = np.triu(lu[k])
        pd = d.copy()
        for i, p in enumerate(piv[k]):
            pd[[i, p]] = pd[[p, i]]
        assert np.abs(L @ U - pd).max() < 1e-12 * np.abs(d).max()


def test_reduced_boundaries(C, wg, rng):
    kern, mt = wg
    full = C.build_one_level(kern, mt)
    red = C.reduce_one_level(full, 0.0)
    assert red.n_kept == kern.grid.nx
    x = random_field(rng, kern.grid.n_unknowns)
    assert np.array_equal(red.apply(x), full.apply(x))
    red1 = C.reduce_one_level(full, 1.0)
    rep = int(np.ceil(kern.grid.nx / 2)) - 1
    assert red1.n_kept == 1 and red1.kept.tolist() == [rep] and red1.representative == rep
    with pytest.raises(ValueError):
        C.reduce_one_level(full, 1.5)


def test_reduced_agrees_with_full_on_kept(C, wg, rng):
    kern, mt = wg
    full = C.build_one_level(kern, mt)
    red = C.reduce_one_level(full, 0.3)
    assert 1 <= red.n_kept < kern.grid.nx
    nz, ny, nx = kern.grid.shape
    spec = np.zeros((3, nz, ny, nx), dtype=complex)
    for k in red.kept:
        spec[:, :, :, k] = rng.normal(size=(3, nz, ny))
    x = scipy.fft.ifft(spec, axis=3).reshape(-1)
    a, b = red.apply(x), full.apply(x)
    assert np.abs(a - b).max() < 1e-13 * np.abs(b).max()


def test_reduced_direct_matches_reduction(C, wg, rng):
    kern, mt = wg
    full = C.build_one_level(kern, mt)
    red1 = C.reduce_one_level(full, 0.3)
    red2 = C.build_reduced_one_level(kern, mt, 0.3)
    assert np.array_equal(red1.kept, red2.kept)
    assert np.abs(red1.proxy - red2.proxy).max() < 1e-15
    x = random_field(rng, kern.grid.n_unknowns)
    assert np.abs(red1.apply(x) - red2.apply(x)).max() < 1e-14 * np.abs(x).max()
    red = C.build_reduced_one_level(kern, mt, 0.5)
    assert np.all(red.proxy_normalized >= 0.0) and red.proxy_normalized.max() == 1.0
    r3 = C.reduce_one_level(full, 0.3)
    assert r3.bytes == r3.n_kept * full.block_size ** 2 * 16 and r3.bytes < full.bytes


def test_two_level_properties(C, wg, rng):
    from paper_1903_07884_b200.solver import gmres

    kern, _ = wg
    x = random_field(rng, kern.grid.n_unknowns)
    p0 = C.build_two_level(kern, np.zeros(kern.grid.shape))
    assert np.abs(p0.apply(x) - x).max() < 1e-12 * np.abs(x).max()
    m = np.full(kern.grid.shape, 0.55 + 0.02j)
    p2 = C.build_two_level(kern, m)
    c = O.dense_chan_circulant_xy(kern.tensors, kern.grid.dims, m)
    assert np.abs(c @ p2.apply(x) - x).max() / np.abs(x).max() < 1e-12
    wrapped = C.wrap_circulant_xy(kern)
    mw = np.full(kern.grid.shape, 0.6 + 0.1j)
    a = O.dense_operator(wrapped.tensors, kern.grid.dims, mw)
    pw = C.build_two_level(wrapped, mw)
    _, rep = gmres(lambda v: a @ v, x, apply_pinv=pw.apply, tol=1e-10, maxit=10)
    assert rep.converged and rep.iterations <= 2
    mh = np.full(kern.grid.shape, 0.5)
    p1, p2h = C.build_one_level(kern, mh), C.build_two_level(kern, mh)
    nx, ny, nz = kern.grid.dims
    assert p2h.bytes == nx * ny * (3 * nz) ** 2 * 16 and p1.bytes == p2h.bytes * ny


@pytest.fixture(scope="module")
def coupler_like():
    from paper_1903_07884_b200.grid import PermittivityMap, VoxelGrid
    from paper_1903_07884_b200.kernel import assemble_kernel

    grid = VoxelGrid(8, 6, 2, 0.05)
    kern = assemble_kernel(grid, 2 * np.pi)
    eps = np.ones(grid.shape, dtype=complex)
    eps[:, 1:3, :] = 5.8
    eps[:, 3:5, :] = 5.8
    return kern, PermittivityMap(grid, eps)


def test_blocked_properties(C, coupler_like, rng):
    from paper_1903_07884_b200.grid import PermittivityMap, homogenize
    from paper_1903_07884_b200.kernel import assemble_kernel

    kern, pmap = coupler_like
    grid = kern.grid
    x = random_field(rng, grid.n_unknowns)
    air = PermittivityMap(grid, np.ones(grid.shape))
    pa = C.build_blocked(kern, air, C.partition_boxes(grid, [C.Box("a", 0, 2, 0, 3, 0, 2)]), {"a": "one-level"})
    assert np.abs(pa.apply(x) - x).max() < 1e-12 * np.abs(x).max()
    part = C.partition_boxes(grid, [C.Box("all", 0, grid.nx, 0, grid.ny, 0, grid.nz)])
    blocked = C.build_blocked(kern, pmap, part, {"all": "one-level"}, homog={"all": "real_mean_x"})
    plain = C.build_one_level(kern, homogenize(pmap, "real_mean_x"))
    assert np.abs(blocked.apply(x) - plain.apply(x)).max() < 1e-13 * np.abs(x).max()
    box = C.Box("lo", 0, grid.nx, 0, 3, 0, grid.nz)
    bl = C.build_blocked(kern, pmap, C.partition_boxes(grid, [box]), {"lo": "one-level"},
                         homog={"lo": "real_mean_x"})
    y = bl.apply(x)
    outside = np.arange(grid.n_unknowns).reshape((3,) + grid.shape)[:, :, 3:, :].reshape(-1)
    assert np.array_equal(y[outside], x[outside])
    sub = C._slice_kernel(kern, box)
    standalone = C.build_one_level(sub, homogenize(PermittivityMap(sub.grid, pmap.eps_r[:, 0:3, :]),
                                                   "real_mean_x"))
    dofs = C._box_dof_indices(grid, box)
    xb = np.zeros(grid.n_unknowns, dtype=complex)
    xb[dofs] = random_field(rng, sub.grid.n_unknowns)
    yb = bl.apply(xb)
    assert np.abs(yb[dofs] - standalone.apply(xb[dofs])).max() < 1e-13
    fresh = assemble_kernel(C._slice_kernel(kern, C.Box("b", 2, 7, 1, 5, 0, 2)).grid, kern.k0)
    assert np.allclose(C._slice_kernel(kern, C.Box("b", 2, 7, 1, 5, 0, 2)).tensors, fresh.tensors, rtol=1e-13)
    two = C.build_blocked(kern, pmap, C.partition_boxes(grid, [C.Box("lo", 0, 8, 0, 3, 0, 2),
                                                               C.Box("hi", 0, 8, 3, 6, 0, 2)]),
                          {"lo": "one-level", "hi": "two-level"})
    assert two.bytes == sum(p.bytes for p in two.box_precs)
    assert [b["label"] for b in two.summary()["boxes"]] == ["lo", "hi"]


def test_singular_blocks_raise(C):
    """D_k = (1 - m s) I with s the only generator entry: singular for m = 1/s."""
    from paper_1903_07884_b200.errors import PreconditionerBuildError

    dims = (4, 3, 2)
    t = np.zeros((6, 3, 5, 7), dtype=complex)
    t[[0, 3, 5], 1, 2, 3] = 2.0
    kern = _kern(t, dims)
    with pytest.raises(PreconditionerBuildError, match="k=0"):
        C.build_one_level(kern, np.full((2, 3, 4), 0.5))
    with pytest.raises(PreconditionerBuildError, match=r"k=0, l=0"):
        C.build_two_level(kern, np.full((2, 3, 4), 0.5))
    ok = C.build_one_level(kern, np.full((2, 3, 4), 0.25))   # D = 0.5 I
    x = np.arange(72, dtype=complex)
    assert relerr(ok.apply(x), 2 * x) < 1e-14


@pytest.mark.parametrize("dims", [(200, 10, 5), (50, 22, 11), (37, 7, 3), (30, 12, 4)])
def test_one_level_vs_oracle_waveguide(rng, C, dims):
    """Block sizes 150, 726 (c1), 63, 144 (padded tiles), non-smooth nx = 37 (Bluestein)."""
    from paper_1903_07884_b200 import workloads

    W = workloads.small(*dims, delta=0.02e-6)
    kern = W.kernel()
    mt = W.mtilde()
    p = C.build_one_level(kern, mt)
    ref = O.build_one_level(kern.tensors, W.grid.dims, mt)
    x = random_field(rng, W.grid.n_unknowns)
    assert relerr(p.apply(x), O.apply_prec(ref, x)) < 1e-10
    r = C.reduce_one_level(p, 1e-3)
    rr = O.reduce_one_level(ref, 1e-3)
    assert np.array_equal(r.kept, rr["kept"])
    assert relerr(r.apply(x), O.apply_prec(rr, x)) < 1e-10


def test_two_level_vs_oracle_disk_like(rng, C):
    """nx = 37 (Bluestein DFT), ny = 40, nz = 8 (24 x 24 blocks, as c4)."""
    from paper_1903_07884_b200 import workloads

    W = workloads.small(37, 40, 8, delta=0.03e-6)
    kern = W.kernel()
    m = np.full(W.grid.shape, 0.75 - 0.01j)
    p = C.build_two_level(kern, m)
    ref = O.build_two_level(kern.tensors, W.grid.dims, m)
    x = random_field(rng, W.grid.n_unknowns)
    assert relerr(p.apply(x), O.apply_prec(ref, x)) < 1e-10


@pytest.mark.parametrize("dims", [(37, 40, 8), (12, 9, 10), (16, 10, 3), (9, 8, 11)])
def test_two_level_block_inverses_equal_factor_solves(rng, C, monkeypatch, dims):
    """3 nz <= 32: the blocks are applied as explicit inverses (one product per
    block); the result equals the two triangular solves on the factors
    (VX_SMALLINV=0) and the oracle, single and multiple right-hand sides.
    3 nz = 33 stays on the factors."""
    from paper_1903_07884_b200 import workloads

    W = workloads.small(*dims, delta=0.03e-6)
    kern = W.kernel()
    m = np.full(W.grid.shape, 0.75 - 0.01j)
    p = C.build_two_level(kern, m)
    small = 3 * dims[2] <= 32
    assert p.factor_layout == ("inverse" if small else "factors")
    if small:
        assert p._inv_err <= C.SMALLINV_TOL
    monkeypatch.setenv("VX_SMALLINV", "0")
    pf = C.build_two_level(kern, m)
    assert pf.factor_layout == "factors"
    ref = O.build_two_level(kern.tensors, W.grid.dims, m)
    x = random_field(rng, W.grid.n_unknowns)
    y = p.apply(x)
    assert relerr(y, pf.apply(x)) < 1e-12
    assert relerr(y, O.apply_prec(ref, x)) < 1e-10
    xs = np.stack([random_field(rng, W.grid.n_unknowns) for _ in range(3)], axis=1)
    assert relerr(p.apply(xs), pf.apply(xs)) < 1e-12
    np.testing.assert_allclose(p.lu, pf.lu, rtol=0, atol=0)


@pytest.mark.parametrize("dims,tol", [((60, 7, 3), 0.05), ((40, 12, 4), 1e-3), ((24, 22, 11), 1e-3)])
def test_reduced_representative_gemm_path(rng, C, monkeypatch, dims, tol):
    """The representative block's frequencies through the explicit-inverse GEMM
    equal the chunked triangular solves and the oracle (1 and 3 RHS; block
    sizes 63, 144, 726 exercise the K/M padding)."""
    from paper_1903_07884_b200 import workloads

    monkeypatch.setenv("VX_SECTORS", "0")  # the GEMM path serves dense (unsectored) blocks
    W = workloads.small(*dims, delta=0.02e-6)
    kern = W.kernel()
    full = C.build_one_level(kern, W.mtilde())
    red = C.reduce_one_level(full, tol)
    assert red._inv is not None and red._rep_ks.numel() >= 8
    monkeypatch.setenv("VX_REP_GEMM", "0")
    red0 = C.reduce_one_level(full, tol)
    assert red0._inv is None
    ref = O.reduce_one_level(O.build_one_level(kern.tensors, W.grid.dims, W.mtilde()), tol)
    n = W.grid.n_unknowns
    for r in (1, 3):
        x = random_field(rng, n * r).reshape(n, r) if r > 1 else random_field(rng, n)
        a, b = red.apply(x), red0.apply(x)
        assert relerr(a, b) < 1e-12
        assert relerr(a, O.apply_prec(ref, x)) < 1e-10
    from paper_1903_07884_b200 import _native as nv

    nv.call("vx_rep_variant", 1)
    try:
        x = random_field(rng, n)
        assert relerr(red.apply(x), red0.apply(x)) < 1e-12
    finally:
        nv.call("vx_rep_variant", 0)
