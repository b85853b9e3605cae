"""GPU parity for the (3N, r) preconditioner applies and the dense spectrum
probes built on them (reference circulant.py:175-188, solver.py:177-193,
harness.py:309-331): `dense_pinv_matrix` is the preconditioner applied to the
identity, `spectrum` the eigenvalues of A P^-1."""

import numpy as np
import pytest

import voxvie_oracle as O
from conftest import random_field

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def wg():
    from paper_1903_07884_b200.grid import PermittivityMap, VoxelGrid, homogenize
    from paper_1903_07884_b200.kernel import assemble_kernel

    grid = VoxelGrid(8, 3, 2, 0.05)
    kern = assemble_kernel(grid, 2 * np.pi)
    eps = PermittivityMap(grid, np.full(grid.shape, 5.8, dtype=complex))
    mt = homogenize(eps, "real_mean_x")  # a uniform slab: constant along x and y (1- and 2-level builds)
    return kern, mt, mt


def _builds(kern, mt_x, mt_xy):
    from paper_1903_07884_b200 import circulant as C

    dims = kern.grid.dims
    return [
        ("one_level", C.build_one_level(kern, mt_x), O.build_one_level(kern.tensors, dims, mt_x)),
        ("reduced", C.build_reduced_one_level(kern, mt_x, 1e-3),
         O.build_reduced_one_level(kern.tensors, dims, mt_x, 1e-3)),
        ("two_level", C.build_two_level(kern, mt_xy), O.build_two_level(kern.tensors, dims, mt_xy)),
    ]


def test_multi_rhs_apply_equals_columnwise(wg, rng):
    kern, mt_x, mt_xy = wg
    n = kern.grid.n_unknowns
    for name, prec, _ in _builds(kern, mt_x, mt_xy):
        for r in (1, 2, 5):
            x = np.stack([random_field(rng, n) for _ in range(r)], axis=1)
            y = prec.apply(x)
            assert y.shape == (n, r), name
            for c in range(r):
                yc = prec.apply(np.ascontiguousarray(x[:, c]))
                assert np.abs(y[:, c] - yc).max() <= 1e-13 * np.abs(yc).max(), (name, r, c)


def test_dense_pinv_matrix_matches_oracle(wg):
    from paper_1903_07884_b200.solver import dense_pinv_matrix

    kern, mt_x, mt_xy = wg
    n = kern.grid.n_unknowns
    eye = np.eye(n, dtype=np.complex128)
    for name, prec, oprec in _builds(kern, mt_x, mt_xy):
        got = dense_pinv_matrix(prec, n)
        want = np.stack([O.apply_prec(oprec, eye[:, c]) for c in range(n)], axis=1)
        assert got.shape == (n, n)
        assert np.abs(got - want).max() <= 1e-10 * np.abs(want).max(), name


def test_dense_pinv_inverts_the_chan_circulant(wg):
    from paper_1903_07884_b200 import circulant as C
    from paper_1903_07884_b200.solver import dense_pinv_matrix

    kern, mt_x, mt_xy = wg
    n = kern.grid.n_unknowns
    p1 = dense_pinv_matrix(C.build_one_level(kern, mt_x), n)
    c1 = O.dense_chan_circulant_x(kern.tensors, kern.grid.dims, mt_x)
    assert np.abs(c1 @ p1 - np.eye(n)).max() < 1e-11
    p2 = dense_pinv_matrix(C.build_two_level(kern, mt_xy), n)
    c2 = O.dense_chan_circulant_xy(kern.tensors, kern.grid.dims, mt_xy)
    assert np.abs(c2 @ p2 - np.eye(n)).max() < 1e-11


def test_spectrum_of_preconditioned_operator(wg):
    """The eigenvalues of A P^-1 equal the oracle's and cluster at 1 more
    tightly than those of A (the property harness.py:309-331 plots)."""
    from paper_1903_07884_b200 import circulant as C
    from paper_1903_07884_b200.solver import dense_pinv_matrix, spectrum

    kern, mt_x, _ = wg
    n = kern.grid.n_unknowns
    a = O.dense_operator(kern.tensors, kern.grid.dims, mt_x)
    pinv = dense_pinv_matrix(C.build_one_level(kern, mt_x), n)
    oprec = O.build_one_level(kern.tensors, kern.grid.dims, mt_x)
    eye = np.eye(n, dtype=np.complex128)
    opinv = np.stack([O.apply_prec(oprec, eye[:, c]) for c in range(n)], axis=1)
    ev, oev = spectrum(a, pinv), np.linalg.eigvals(a @ opinv)
    # same multiset: every eigenvalue has a partner within 1e-8
    d = np.abs(ev[:, None] - oev[None, :])
    assert d.min(axis=1).max() < 1e-8 and d.min(axis=0).max() < 1e-8
    assert np.abs(ev - 1).max() < np.abs(spectrum(a) - 1).max()


def test_spectrum_guards():
    from paper_1903_07884_b200.errors import SizeLimitError
    from paper_1903_07884_b200.solver import SPECTRUM_GUARD, dense_pinv_matrix, spectrum

    with pytest.raises(SizeLimitError):
        dense_pinv_matrix(None, SPECTRUM_GUARD + 1)
    with pytest.raises(SizeLimitError):
        spectrum(np.broadcast_to(np.zeros(1), (SPECTRUM_GUARD + 1, SPECTRUM_GUARD + 1)))
