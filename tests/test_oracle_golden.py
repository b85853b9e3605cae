"""Pin the CPU oracle against vectors produced by the unmodified reference
(tests/golden/make_golden.py) and the reference's own committed artefact
(pkg/frontend/tests/fixtures/sweep.csv -> golden_sweep.npz)."""

import numpy as np
import pytest

import voxvie_oracle as O
from conftest import relerr
from paper_1903_07884_b200.grid import PermittivityMap, VoxelGrid, homogenize, medium_coefficient
from paper_1903_07884_b200.kernel import assemble_kernel

OP_TAGS = ["small", "cube", "one", "odd", "prime", "long"]
PC_TAGS = ["wg", "pr", "py", "sq"]


@pytest.mark.parametrize("tag", OP_TAGS)
def test_operator_matches_reference(golden_small, tag):
    g = golden_small
    dims = tuple(int(v) for v in g[f"op_{tag}_dims"])
    spec = O.plan_spectra(g[f"op_{tag}_tensors"], dims)
    assert relerr(O.apply_n(spec, dims, g[f"op_{tag}_x"]), g[f"op_{tag}_n"]) < 1e-14
    assert relerr(O.apply_system(spec, dims, g[f"op_{tag}_m"], g[f"op_{tag}_x"]), g[f"op_{tag}_a"]) < 1e-14


@pytest.mark.parametrize("tag", ["small", "cube", "odd"])
def test_operator_matches_dense(golden_small, tag):
    g = golden_small
    dims = tuple(int(v) for v in g[f"op_{tag}_dims"])
    a = O.dense_operator(g[f"op_{tag}_tensors"], dims, g[f"op_{tag}_m"])
    assert relerr(a @ g[f"op_{tag}_x"], g[f"op_{tag}_a"]) < 1e-12


@pytest.mark.parametrize("tag", PC_TAGS)
def test_preconditioners_match_reference(golden_small, tag):
    g = golden_small
    dims = tuple(int(v) for v in g[f"pc_{tag}_dims"])
    t = g[f"pc_{tag}_tensors"]
    x, xr = g[f"pc_{tag}_x"], g[f"pc_{tag}_xr"]
    p1 = O.build_one_level(t, dims, g[f"pc_{tag}_mtilde"])
    assert relerr(p1["proxy"], g[f"pc_{tag}_one_proxy"]) < 1e-14
    assert relerr(O.apply_prec(p1, x), g[f"pc_{tag}_one_y"]) < 1e-13
    assert relerr(O.apply_prec(p1, xr), g[f"pc_{tag}_one_yr"]) < 1e-13
    red = O.reduce_one_level(p1, 0.3)
    assert np.array_equal(red["kept"], g[f"pc_{tag}_red_kept"])
    assert np.array_equal(red["slot_of"], g[f"pc_{tag}_red_slot"])
    assert relerr(O.apply_prec(red, x), g[f"pc_{tag}_red_y"]) < 1e-13
    red2 = O.build_reduced_one_level(t, dims, g[f"pc_{tag}_mtilde"], 0.3)
    assert np.array_equal(red2["kept"], g[f"pc_{tag}_red2_kept"])
    assert relerr(O.apply_prec(red2, x), g[f"pc_{tag}_red2_y"]) < 1e-13
    p2 = O.build_two_level(t, dims, g[f"pc_{tag}_m2"])
    assert relerr(O.apply_prec(p2, x), g[f"pc_{tag}_two_y"]) < 1e-13
    assert relerr(O.apply_prec(p2, xr), g[f"pc_{tag}_two_yr"]) < 1e-13


def test_blocked_matches_reference(golden_small):
    g = golden_small
    dims = (8, 6, 2)
    grid = VoxelGrid(*dims, 0.05)
    pmap = PermittivityMap(grid, g["blk_eps"])

    def mt(box, strat):
        x0, x1, y0, y1, z0, z1 = box
        sub = VoxelGrid(x1 - x0, y1 - y0, z1 - z0, 0.05)
        return homogenize(PermittivityMap(sub, pmap.eps_r[z0:z1, y0:y1, x0:x1]), strat)

    boxes = [(0, 8, 0, 3, 0, 2), (0, 8, 3, 6, 0, 2)]
    bp = O.build_blocked(g["blk_tensors"], dims, boxes, ["one-level", "two-level"],
                         [mt(boxes[0], "real_mean_x"), mt(boxes[1], "mode")])
    assert relerr(O.apply_prec(bp, g["blk_x"]), g["blk_y"]) < 1e-13
    box = (1, 7, 1, 5, 0, 2)
    bp2 = O.build_blocked(g["blk_tensors"], dims, [box], ["reduced-one-level"],
                          [mt(box, "real_mean_x")], reduce_tol=0.2)
    assert relerr(O.apply_prec(bp2, g["blk_x"]), g["blk2_y"]) < 1e-13


@pytest.mark.parametrize("tag,restart,prec", [("none", None, False), ("one", None, True),
                                              ("rst", 4, True), ("nrs", 7, False)])
def test_gmres_matches_reference(golden_small, tag, restart, prec):
    g = golden_small
    dims = (16, 4, 3)
    t = g["gm_tensors"]
    spec = O.plan_spectra(t, dims)
    m = medium_coefficient(PermittivityMap(VoxelGrid(*dims, 0.05), g["gm_eps"]))
    pinv = None
    if prec:
        mt = homogenize(PermittivityMap(VoxelGrid(*dims, 0.05), g["gm_eps"]), "real_mean_x")
        p1 = O.build_one_level(t, dims, mt)
        pinv = lambda v: O.apply_prec(p1, v)  # noqa: E731
    x, rep = O.gmres(lambda v: O.apply_system(spec, dims, m, v), g["gm_b"], apply_pinv=pinv,
                     tol=1e-8, maxit=200, restart=restart)
    assert rep["iterations"] == int(g[f"gm_{tag}_its"])
    assert np.allclose(rep["residuals"], g[f"gm_{tag}_res"], rtol=1e-6, atol=1e-14)
    assert relerr(x, g[f"gm_{tag}_x"]) < 1e-10


@pytest.mark.parametrize("L", [32, 64, 128])
def test_sweep_iteration_counts_match_reference_artefact(golden_sweep, L):
    """Iteration counts of sweep.csv (reference-produced) reproduced by the oracle."""
    g = golden_sweep
    tag = f"L{L}"
    dims = tuple(int(v) for v in g[f"{tag}_dims"])
    t = g[f"{tag}_tensors"]
    grid = VoxelGrid(*dims, float(g[f"{tag}_delta"]))
    pmap = PermittivityMap(grid, g[f"{tag}_eps"])
    m = medium_coefficient(pmap)
    spec = O.plan_spectra(t, dims)
    tol, maxit = float(g[f"{tag}_tol"]), int(g[f"{tag}_maxit"])
    A = lambda v: O.apply_system(spec, dims, m, v)  # noqa: E731
    mt = homogenize(pmap, "real_mean_x")
    p1 = O.build_one_level(t, dims, mt)
    _, r1 = O.gmres(A, g[f"{tag}_b"], apply_pinv=lambda v: O.apply_prec(p1, v), tol=tol, maxit=maxit)
    assert r1["iterations"] == int(g[f"{tag}_its_one_level_real_mean_x"])
    red = O.build_reduced_one_level(t, dims, mt, 1e-3)
    assert red["lu"].shape[0] * red["lu"].shape[1] ** 2 * 16 == int(g[f"{tag}_bytes_reduced"])
    _, r2 = O.gmres(A, g[f"{tag}_b"], apply_pinv=lambda v: O.apply_prec(red, v), tol=tol, maxit=maxit)
    assert r2["iterations"] == int(g[f"{tag}_its_reduced_one_level_real_mean_x"])
    if L <= 64:
        _, r0 = O.gmres(A, g[f"{tag}_b"], tol=tol, maxit=maxit)
        assert r0["iterations"] == int(g[f"{tag}_its_none"])


def test_c0_reference_solution(golden_c0):
    """The oracle on c0 (my workload arrays, my kernel assembly) vs the reference
    solve recorded with the reference's own assembly."""
    from paper_1903_07884_b200 import workloads

    W = workloads.make("c0")
    t = W.kernel().tensors
    dims = W.grid.dims
    spec = O.plan_spectra(t, dims)
    m = W.m
    p1 = O.build_one_level(t, dims, W.mtilde())
    x, rep = O.gmres(lambda v: O.apply_system(spec, dims, m, v), W.b,
                     apply_pinv=lambda v: O.apply_prec(p1, v), tol=W.tol, maxit=W.maxit,
                     restart=W.restart)
    assert abs(rep["iterations"] - int(golden_c0["c0_its"])) <= 0
    assert relerr(x, golden_c0["c0_x"]) < 1e-8


def test_own_kernel_assembly_matches_reference_tensors(golden_small):
    for tag in ["small", "cube", "one", "odd", "prime", "long"]:
        dims = tuple(int(v) for v in golden_small[f"op_{tag}_dims"])
        t = assemble_kernel(VoxelGrid(*dims, 0.05), 2 * np.pi, near_gauss=(tag == "odd")).tensors
        assert relerr(t, golden_small[f"op_{tag}_tensors"]) < 1e-14
