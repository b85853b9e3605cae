"""GPU GMRES: the reference solver test-suite (test_solver.py) on the device
Krylov basis, golden solves produced by the reference, iteration counts of the
reference's own sweep.csv artefact, and BASELINE config c0."""

import json

import numpy as np
import pytest

import voxvie_oracle as O
from conftest import relerr

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gmres():
    from paper_1903_07884_b200.solver import gmres

    return gmres


def random_system(rng, n, diag_boost=3.0):
    a = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
    a += diag_boost * np.sqrt(n) * np.eye(n)
    b = rng.normal(size=n) + 1j * rng.normal(size=n)
    return a, b


def test_identity_and_zero_rhs(gmres, rng):
    b = rng.normal(size=20) + 0j
    x, rep = gmres(lambda v: v, b, tol=1e-10)
    assert rep.iterations == 1 and rep.converged and np.allclose(x, b)
    x, rep = gmres(lambda v: v, np.zeros(5, dtype=complex), tol=1e-6)
    assert rep.converged and rep.iterations == 1 and np.all(x == 0)
    assert rep.residuals[0] == 1.0 and rep.residuals[-1] == 0.0


def test_matches_direct_solve(gmres, rng):
    a, b = random_system(rng, 50)
    x, rep = gmres(lambda v: a @ v, b, tol=1e-9, maxit=100)
    assert rep.converged
    assert relerr(x, np.linalg.solve(a, b)) < 1e-8


def test_exact_inverse_preconditioner(gmres, rng):
    a, b = random_system(rng, 40)
    ai = np.linalg.inv(a)
    x, rep = gmres(lambda v: a @ v, b, apply_pinv=lambda v: ai @ v, tol=1e-10, maxit=10)
    assert rep.converged and rep.iterations <= 2


def test_residual_history_and_true_residual(gmres, rng):
    a, b = random_system(rng, 60, diag_boost=1.0)
    x, rep = gmres(lambda v: a @ v, b, tol=1e-8, maxit=200)
    hist = np.asarray(rep.residuals)
    assert hist[0] == 1.0 and len(hist) == rep.iterations + 1
    assert np.all(np.diff(hist) <= 1e-14)
    a, b = random_system(rng, 50)
    x, rep = gmres(lambda v: a @ v, b, tol=1e-8, maxit=100)
    explicit = np.linalg.norm(b - a @ x) / np.linalg.norm(b)
    assert rep.true_residual == pytest.approx(explicit, rel=1e-10)
    assert abs(rep.true_residual - rep.residuals[-1]) < 1e-10


def test_preconditioned_and_invariance(gmres, rng):
    a, b = random_system(rng, 40)
    p = np.diag(1.0 / np.diag(a))
    x, rep = gmres(lambda v: a @ v, b, apply_pinv=lambda v: p @ v, tol=1e-9, maxit=100)
    assert abs(rep.residuals[-1] - np.linalg.norm(b - a @ x) / np.linalg.norm(b)) < 1e-9
    a, b = random_system(rng, 50)
    x1, r1 = gmres(lambda v: a @ v, b, tol=1e-7, maxit=200)
    pi = np.linalg.inv(a + 0.1 * np.eye(50))
    x2, r2 = gmres(lambda v: a @ v, b, apply_pinv=lambda v: pi @ v, tol=1e-7, maxit=200)
    assert r1.converged and r2.converged and relerr(x2, x1) < 1e-6


def test_deterministic_maxit_restart_errors(gmres, rng):
    a, b = random_system(rng, 45, diag_boost=1.5)
    _, r1 = gmres(lambda v: a @ v, b, tol=1e-7, maxit=120)
    _, r2 = gmres(lambda v: a @ v, b, tol=1e-7, maxit=120)
    assert r1.iterations == r2.iterations and r1.residuals == r2.residuals
    a, b = random_system(rng, 50, diag_boost=0.0)
    _, rep = gmres(lambda v: a @ v, b, tol=1e-14, maxit=5)
    assert not rep.converged and rep.iterations == 5
    a, b = random_system(rng, 50)
    x, rep = gmres(lambda v: a @ v, b, tol=1e-8, maxit=400, restart=10)
    assert rep.converged and relerr(x, np.linalg.solve(a, b)) < 1e-6
    with pytest.raises(ValueError):
        gmres(lambda v: v, np.ones(3), tol=0.0)
    with pytest.raises(ValueError):
        gmres(lambda v: v, np.ones(3), maxit=0)
    _, rep = gmres(lambda v: a @ v, b, tol=1e-6, maxit=50)
    json.dumps(rep.to_dict())


@pytest.mark.parametrize("tag,restart,prec", [("none", None, False), ("one", None, True),
                                              ("rst", 4, True), ("nrs", 7, False)])
def test_gmres_golden_vie(golden_small, gmres, tag, restart, prec):
    from paper_1903_07884_b200.circulant import build_one_level
    from paper_1903_07884_b200.grid import PermittivityMap, VoxelGrid, homogenize, medium_coefficient
    from paper_1903_07884_b200.kernel import ToeplitzKernel
    from paper_1903_07884_b200.operator import apply_system, plan_operator

    g = golden_small
    grid = VoxelGrid(16, 4, 3, 0.05)
    kern = ToeplitzKernel(grid, 2 * np.pi, g["gm_tensors"])
    plan = plan_operator(kern)
    pmap = PermittivityMap(grid, g["gm_eps"])
    m = medium_coefficient(pmap)
    pinv = build_one_level(kern, homogenize(pmap, "real_mean_x")).apply if prec else None
    x, rep = gmres(lambda v: apply_system(plan, m, v), g["gm_b"], apply_pinv=pinv, tol=1e-8,
                   maxit=200, restart=restart)
    assert abs(rep.iterations - int(g[f"gm_{tag}_its"])) <= 2
    assert relerr(x, g[f"gm_{tag}_x"]) < 1e-6
    n = min(len(rep.residuals), len(g[f"gm_{tag}_res"]))
    assert np.allclose(rep.residuals[:n], g[f"gm_{tag}_res"][:n], rtol=1e-4, atol=1e-12)


@pytest.mark.parametrize("L", [32, 64, 128])
def test_sweep_iteration_counts(golden_sweep, gmres, L):
    """Iteration counts of the reference's committed sweep.csv (waveguide-length preset)."""
    from paper_1903_07884_b200.circulant import build_one_level, build_reduced_one_level
    from paper_1903_07884_b200.grid import PermittivityMap, VoxelGrid, homogenize, medium_coefficient
    from paper_1903_07884_b200.kernel import ToeplitzKernel
    from paper_1903_07884_b200.operator import apply_system, plan_operator

    g = golden_sweep
    tag = f"L{L}"
    dims = tuple(int(v) for v in g[f"{tag}_dims"])
    grid = VoxelGrid(*dims, float(g[f"{tag}_delta"]))
    kern = ToeplitzKernel(grid, float(g[f"{tag}_k0"]), g[f"{tag}_tensors"])
    plan = plan_operator(kern)
    pmap = PermittivityMap(grid, g[f"{tag}_eps"])
    m = medium_coefficient(pmap)
    b = g[f"{tag}_b"]
    tol, maxit = float(g[f"{tag}_tol"]), int(g[f"{tag}_maxit"])
    A = lambda v: apply_system(plan, m, v)  # noqa: E731
    mt = homogenize(pmap, "real_mean_x")
    _, r1 = gmres(A, b, apply_pinv=build_one_level(kern, mt).apply, tol=tol, maxit=maxit)
    assert abs(r1.iterations - int(g[f"{tag}_its_one_level_real_mean_x"])) <= 2
    red = build_reduced_one_level(kern, mt, 1e-3)
    assert red.bytes == int(g[f"{tag}_bytes_reduced"])
    _, r2 = gmres(A, b, apply_pinv=red.apply, tol=tol, maxit=maxit)
    assert abs(r2.iterations - int(g[f"{tag}_its_reduced_one_level_real_mean_x"])) <= 2
    _, r0 = gmres(A, b, tol=tol, maxit=maxit)
    assert abs(r0.iterations - int(g[f"{tag}_its_none"])) <= 2


def test_c0_against_reference_solution(golden_c0, gmres):
    """BASELINE config c0: iterations within +-2 and field within 1e-4 of the
    reference's own solve (tests/golden/make_golden.py)."""
    from paper_1903_07884_b200 import workloads
    from paper_1903_07884_b200.circulant import build_one_level
    from paper_1903_07884_b200.operator import apply_system, plan_operator

    W = workloads.make("c0")
    kern = W.kernel()
    plan = plan_operator(kern)
    prec = build_one_level(kern, W.mtilde())
    m = W.m
    x, rep = gmres(lambda v: apply_system(plan, m, v), W.b, apply_pinv=prec.apply, tol=W.tol,
                   maxit=W.maxit, restart=W.restart)
    assert abs(rep.iterations - int(golden_c0["c0_its"])) <= 2
    assert relerr(x, golden_c0["c0_x"]) < 1e-4
    assert rep.true_residual < 2 * W.tol


def test_device_mode_tensor_in_tensor_out(gmres):
    import torch

    from paper_1903_07884_b200 import workloads
    from paper_1903_07884_b200.circulant import build_one_level
    from paper_1903_07884_b200.operator import apply_system, plan_operator

    W = workloads.small(64, 6, 3)
    kern = W.kernel()
    plan = plan_operator(kern)
    prec = build_one_level(kern, W.mtilde())
    m = torch.from_numpy(W.m.reshape(-1)).cuda()
    b = torch.from_numpy(W.b).cuda()
    x, rep = gmres(lambda v: apply_system(plan, m, v), b, apply_pinv=prec.apply, tol=1e-8, maxit=200)
    assert isinstance(x, torch.Tensor) and x.is_cuda
    spec = O.plan_spectra(kern.tensors, W.grid.dims)
    pr = O.build_one_level(kern.tensors, W.grid.dims, W.mtilde())
    xo, ro = O.gmres(lambda v: O.apply_system(spec, W.grid.dims, W.m, v), W.b,
                     apply_pinv=lambda v: O.apply_prec(pr, v), tol=1e-8, maxit=200)
    assert abs(rep.iterations - ro["iterations"]) <= 2
    assert relerr(x.cpu().numpy(), xo) < 1e-6
