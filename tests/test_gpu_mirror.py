"""Mirror sharing of preconditioner factors (x / y parity of the kernel).

For a parity-symmetric kernel the blocks D_{n-k} = S D_k S share D_k's stored
factors (circulant.py "mirror sharing").  These tests pin the shared path to
the unshared one (VX_MIRROR=0, every block factorised) and to the CPU oracle,
on both solve kernels (warp-per-block for single-tile blocks, the TMA
pipeline with 2 / 4 right-hand sides per factor stream for multi-tile ones).
"""

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


def _pair(C, monkeypatch, build):
    p = build()
    monkeypatch.setenv("VX_MIRROR", "0")
    q = build()
    monkeypatch.delenv("VX_MIRROR")
    return p, q


@pytest.mark.parametrize("dims", [(8, 3, 2), (7, 3, 2), (12, 4, 3), (9, 5, 3), (2, 3, 2), (1, 3, 2)])
def test_one_level_mirror_equals_unshared(rng, C, monkeypatch, dims):
    """Even / odd nx, single-tile (18) and multi-tile (36, 45) blocks, nx = 1, 2."""
    W = _wl(dims)
    kern, mt = W.kernel(), W.mtilde()
    p, q = _pair(C, monkeypatch, lambda: C.build_one_level(kern, mt))
    nx = dims[0]
    assert p.mirror_shared == (nx > 2)
    assert not q.mirror_shared
    assert p.stored_slots == (nx // 2 + 1) * p.sectors and q.stored_slots == nx * q.sectors
    assert p.bytes == q.bytes  # the reference's accounting is unchanged
    n = W.grid.n_unknowns
    for r in (None, 3):
        x = random_field(rng, n, r)
        assert relerr(p.apply(x), q.apply(x)) < 1e-12
    ref = O.build_one_level(kern.tensors, W.grid.dims, mt)
    x = random_field(rng, n)
    assert relerr(p.apply(x), O.apply_prec(ref, x)) < 1e-10
    # LAPACK-layout views of the mirrored blocks equal the directly factorised ones
    assert np.array_equal(p.piv, q.piv)
    assert relerr(p.lu, q.lu) < 1e-12


@pytest.mark.parametrize("dims", [(8, 3, 2), (12, 4, 3)])
def test_one_level_mirror_classic_kernel(rng, C, monkeypatch, dims):
    from paper_1903_07884_b200 import _native as nv

    W = _wl(dims)
    kern, mt = W.kernel(), W.mtilde()
    p, q = _pair(C, monkeypatch, lambda: C.build_one_level(kern, mt))
    x = random_field(rng, W.grid.n_unknowns)
    nv.call("vx_solve_variant", 1)
    try:
        assert relerr(p.apply(x), q.apply(x)) < 1e-12
    finally:
        nv.call("vx_solve_variant", 0)


@pytest.mark.parametrize("dims,tol", [((60, 7, 3), 0.05), ((40, 12, 4), 1e-3), ((41, 4, 3), 0.2)])
def test_reduced_mirror_equals_unshared(rng, C, monkeypatch, dims, tol):
    W = _wl(dims)
    kern, mt = W.kernel(), W.mtilde()
    p, q = _pair(C, monkeypatch, lambda: C.build_reduced_one_level(kern, mt, tol))
    assert np.array_equal(p.kept, q.kept) and np.array_equal(p.slot_of, q.slot_of)
    assert p._fac.shape[0] < q._fac.shape[0]
    n = W.grid.n_unknowns
    for r in (None, 2):
        x = random_field(rng, n, r)
        assert relerr(p.apply(x), q.apply(x)) < 1e-12
    # reduction of a shared full build
    full = C.build_one_level(kern, mt)
    red = C.reduce_one_level(full, tol)
    x = random_field(rng, n)
    assert relerr(red.apply(x), q.apply(x)) < 1e-12
    rr = O.reduce_one_level(O.build_one_level(kern.tensors, W.grid.dims, mt), tol)
    assert relerr(red.apply(x), O.apply_prec(rr, x)) < 1e-10


@pytest.mark.parametrize("dims", [(9, 8, 2), (8, 7, 3), (37, 40, 8), (6, 5, 11)])
def test_two_level_mirror_equals_unshared(rng, C, monkeypatch, dims):
    """Orbits of 1, 2 and 4 blocks; nz = 11 gives 33 x 33 blocks (pipelined
    solve with 4 right-hand sides per factor stream)."""
    W = _wl(dims, delta=0.03e-6)
    kern = W.kernel()
    m = np.full(W.grid.shape, 0.75 - 0.01j)
    p, q = _pair(C, monkeypatch, lambda: C.build_two_level(kern, m))
    nx, ny, _ = dims
    assert p.mirror_shared and not q.mirror_shared
    assert p._fac.shape[0] == (nx // 2 + 1) * (ny // 2 + 1)
    n = W.grid.n_unknowns
    for r in (None, 2):
        x = random_field(rng, n, r)
        assert relerr(p.apply(x), q.apply(x)) < 1e-12
    ref = O.build_two_level(kern.tensors, W.grid.dims, m)
    x = random_field(rng, n)
    assert relerr(p.apply(x), O.apply_prec(ref, x)) < 1e-10
    if n <= 3 * 9 * 8 * 2:
        assert np.array_equal(p.piv, q.piv)
        assert relerr(p.lu, q.lu) < 1e-12


def test_asymmetric_kernel_is_not_shared(rng, C):
    """A kernel without x parity factorises every block."""
    from paper_1903_07884_b200.grid import VoxelGrid
    from paper_1903_07884_b200.kernel import ToeplitzKernel

    dims = (6, 3, 2)
    t = rng.normal(size=(6, 3, 5, 11)) + 1j * rng.normal(size=(6, 3, 5, 11))
    t *= 0.05
    kern = ToeplitzKernel(VoxelGrid(*dims, 0.05), 2 * np.pi, t)
    m = np.full((2, 3, 6), 0.5 + 0.1j)
    p = C.build_one_level(kern, m)
    assert not p.mirror_shared and p.stored_slots == 6
    ref = O.build_one_level(t, dims, m)
    x = random_field(rng, 3 * 36)
    assert relerr(p.apply(x), O.apply_prec(ref, x)) < 1e-10
    p2 = C.build_two_level(kern, m)
    assert not p2.mirror_shared
    assert relerr(p2.apply(x), O.apply_prec(O.build_two_level(t, dims, m), x)) < 1e-10
