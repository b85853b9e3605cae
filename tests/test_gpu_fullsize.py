"""Parity at the BASELINE sizes through size-independent properties:

* c1 matvec against the oracle's scipy FFT convolution on the full grid;
* c1 1-level preconditioner applied to a vector whose x-spectrum lives on a
  few frequencies: the result must live on the same frequencies and equal the
  oracle's dense zgetrs solves of exactly those blocks (P^-1 is block diagonal
  in k), at 1e-10;
* converged GPU solutions of c1 / c2 / c3 checked with the oracle's own matvec:
  true relative residual <= tol (1e-5).
"""

import numpy as np
import pytest
import scipy.fft
from scipy.linalg import lu_factor, lu_solve

import voxvie_oracle as O
from conftest import relerr

pytestmark = pytest.mark.gpu

CORES = 8


@pytest.fixture(scope="module")
def c1():
    from paper_1903_07884_b200 import workloads

    W = workloads.make("c1")
    W.kernel()
    return W


@pytest.fixture(scope="module")
def c1_spectra(c1):
    return O.plan_spectra(c1.kernel().tensors, c1.grid.dims, workers=CORES)


def test_c1_matvec_fullsize(c1, c1_spectra, rng):
    from paper_1903_07884_b200.operator import apply_system, plan_operator

    plan = plan_operator(c1.kernel())
    n = c1.grid.n_unknowns
    x = rng.normal(size=n) + 1j * rng.normal(size=n)
    got = apply_system(plan, c1.m, x)
    ref = O.apply_system(c1_spectra, c1.grid.dims, c1.m, x, workers=CORES)
    assert relerr(got, ref) < 1e-10


def test_c1_prec_on_sampled_frequencies(c1, rng):
    from paper_1903_07884_b200.circulant import build_one_level

    nx, ny, nz = c1.grid.dims
    prec = build_one_level(c1.kernel(), c1.mtilde(), cap_bytes=2 ** 62)
    ks = [0, 1, 17, 2499, 2500, 4321, 4999]
    spec = np.zeros((3, nz, ny, nx), complex)
    for k in ks:
        spec[..., k] = rng.normal(size=(3, nz, ny)) + 1j * rng.normal(size=(3, nz, ny))
    x = scipy.fft.ifft(spec, axis=3).reshape(-1)
    y = prec.apply(x)
    yh = scipy.fft.fft(y.reshape(3, nz, ny, nx), axis=3)
    lam = O.chan_x_spectra(c1.kernel().tensors)
    m_yz = c1.mtilde()[:, :, 0]
    mask = np.zeros(nx, bool)
    mask[ks] = True
    assert np.abs(yh[..., ~mask]).max() < 1e-9 * np.abs(yh).max()
    for k in ks:
        d = O.unfold_block_yz(lam[:, :, :, k], m_yz)
        ref = lu_solve(lu_factor(d), spec[..., k].reshape(-1))
        assert relerr(yh[..., k].reshape(-1), ref) < 1e-10, k


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_converged_solution_true_residual_by_oracle(name):
    from paper_1903_07884_b200 import workloads
    from paper_1903_07884_b200.operator import apply_system, plan_operator
    from paper_1903_07884_b200.solver import gmres

    import bench

    W = workloads.make(name)
    kern = W.kernel()
    plan = plan_operator(kern)
    prec = bench.build_prec(W, kern)
    m = W.m
    x, rep = gmres(lambda v: apply_system(plan, m, v), W.b, apply_pinv=prec.apply, tol=W.tol,
                   maxit=W.maxit, restart=W.restart)
    assert rep.converged
    spec = O.plan_spectra(kern.tensors, W.grid.dims, workers=CORES)
    r = W.b - O.apply_system(spec, W.grid.dims, m, x, workers=CORES)
    true_res = np.linalg.norm(r) / np.linalg.norm(W.b)
    assert true_res <= 1.0001 * W.tol
    assert abs(true_res - rep.true_residual) < 1e-8
