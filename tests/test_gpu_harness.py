"""Harness integration on the GPU path: the reference's `waveguide-length`
sweep problems (golden_sweep.npz, built by the reference) through
build_preconditioner / solve_problem / run_problem, checked against the
reference's own sweep.csv artefact and the reference byte formulas."""

import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _problem(g, L):
    from paper_1903_07884_b200.grid import PermittivityMap, Physics, VoxelGrid, medium_coefficient
    from paper_1903_07884_b200.harness import Problem
    from paper_1903_07884_b200.kernel import ToeplitzKernel
    from paper_1903_07884_b200.operator import plan_operator

    tag = f"L{L}"
    dims = tuple(int(v) for v in g[f"{tag}_dims"])
    grid = VoxelGrid(*dims, float(g[f"{tag}_delta"]))
    kern = ToeplitzKernel(grid, float(g[f"{tag}_k0"]), g[f"{tag}_tensors"])
    pmap = PermittivityMap(grid, g[f"{tag}_eps"])
    phys = Physics.from_wavelength(2 * np.pi / float(g[f"{tag}_k0"]))
    cfg = {"solver": {"tol": float(g[f"{tag}_tol"]), "maxit": int(g[f"{tag}_maxit"]), "restart": None}}
    b = g[f"{tag}_b"]
    m = medium_coefficient(pmap)
    return Problem(config=cfg, physics=phys, pmap=pmap, hint=None, kernel=kern, plan=plan_operator(kern),
                   m=m, e_inc=np.zeros_like(b), b=b)


@pytest.mark.parametrize("L", [32, 64])
def test_sweep_point_through_harness(golden_sweep, L):
    from paper_1903_07884_b200.harness import solve_problem

    g = golden_sweep
    prob = _problem(g, L)
    for kind, key in [("none", "none"), ("one-level", "one_level_real_mean_x"),
                      ("reduced-one-level", "reduced_one_level_real_mean_x")]:
        cfg = {"kind": kind, "homogenization": "real-mean-x", "cap_mb": 2048, "reduce_tol": 1e-3}
        x, rep, summary = solve_problem(prob, cfg)
        assert abs(rep.iterations - int(g[f"L{L}_its_{key}"])) <= 2, (kind, rep.iterations)
        assert rep.converged
        mem = rep.memory
        assert mem["krylov_basis_bytes"] == rep.iterations * prob.b.size * 16
        assert mem["kernel_bytes"] == prob.kernel.storage_bytes()
        if kind == "reduced-one-level" and L == 128:
            assert summary["bytes"] == int(g["L128_bytes_reduced"])


def test_run_problem_writes_reference_formats(golden_sweep, tmp_path):
    from paper_1903_07884_b200.harness import read_field, read_residuals, run_problem

    prob = _problem(golden_sweep, 32)
    out = run_problem(prob, {"kind": "one-level", "homogenization": "real-mean-x"}, tmp_path / "run")
    rep = json.loads((out / "report.json").read_text())
    assert rep["solve"]["iterations"] == int(golden_sweep["L32_its_one_level_real_mean_x"])
    assert rep["preconditioner"]["level"] == "one-level"
    field, side = read_field(out / "field.bin")
    assert field.size == prob.pmap.grid.n_unknowns and side["dtype"] == "complex128-le"
    res = read_residuals(out / "residuals.csv")
    assert res[0] == 1.0 and len(res) == rep["solve"]["iterations"] + 1
