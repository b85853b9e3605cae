"""Generate the golden fixtures by running the UNMODIFIED reference package.

Run in the build container (the reference exists only there):

    NUMBA_CACHE_DIR=/tmp/numba PYTHONPATH=/root/reference/pkg/src:/root/repo \
        python tests/golden/make_golden.py

Writes, next to this script:
  golden_small.npz  -- operator / preconditioner / GMRES input+output vectors on
                       the reference test-suite grids (conftest.py:18-34,
                       test_circulant.py:116-121,317-324) and odd/prime sizes.
  golden_sweep.npz  -- the ``waveguide-length`` preset problems (presets.py:14-31)
                       as built by harness.build_problem, plus the iteration
                       counts of the reference's own committed artefact
                       pkg/frontend/tests/fixtures/sweep.csv.
  golden_c0.npz     -- BASELINE config c0 (workloads.make("c0")) solved by the
                       reference: iteration count, residual history, solution.
The GPU box never reads /root/reference; tests only read these files.
"""

from __future__ import annotations

import copy
import csv
import os
import sys
from pathlib import Path

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba")
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))

from voxvie import circulant as C  # noqa: E402
from voxvie import operator as O  # noqa: E402
from voxvie import solver as S  # noqa: E402
from voxvie.config import normalize  # noqa: E402
from voxvie.grid import PermittivityMap, VoxelGrid, homogenize, medium_coefficient  # noqa: E402
from voxvie.harness import build_problem  # noqa: E402
from voxvie.kernel import assemble_kernel  # noqa: E402
from voxvie.presets import preset  # noqa: E402

HERE = Path(__file__).resolve().parent
SEED = 20240811  # conftest.py:8-10


def rfield(rng, n, r=None):
    shape = (n,) if r is None else (n, r)
    return rng.normal(size=shape) + 1j * rng.normal(size=shape)


def small_cases(out):
    rng = np.random.default_rng(SEED)
    k0 = 2 * np.pi
    # --- operator cases: (nx, ny, nz) incl. odd / prime / non-smooth 2n
    for tag, dims, ng in [("small", (4, 3, 2), False), ("cube", (3, 3, 3), False),
                          ("one", (1, 1, 1), False), ("odd", (7, 5, 3), True),
                          ("prime", (17, 3, 2), False), ("long", (37, 2, 1), False)]:
        grid = VoxelGrid(*dims, 0.05)
        kern = assemble_kernel(grid, k0, near_gauss=ng)
        plan = O.plan_operator(kern)
        eps = rng.uniform(1.2, 3.5, grid.shape) - 1j * rng.uniform(0, 0.4, grid.shape)
        m = medium_coefficient(PermittivityMap(grid, eps))
        x = rfield(rng, grid.n_unknowns)
        out[f"op_{tag}_dims"] = np.array(dims)
        out[f"op_{tag}_tensors"] = kern.tensors
        out[f"op_{tag}_m"] = m
        out[f"op_{tag}_x"] = x
        out[f"op_{tag}_n"] = O.apply_n(plan, x)
        out[f"op_{tag}_a"] = O.apply_system(plan, m, x)

    # --- preconditioner cases on test_circulant.py's wg grid + prime sizes
    for tag, dims in [("wg", (8, 3, 2)), ("pr", (17, 3, 2)), ("py", (6, 19, 2)),
                      ("sq", (12, 5, 3))]:
        grid = VoxelGrid(*dims, 0.05)
        kern = assemble_kernel(grid, k0)
        mt = homogenize(PermittivityMap(grid, np.full(grid.shape, 5.8, complex)), "real_mean_x")
        x = rfield(rng, grid.n_unknowns)
        xr = rfield(rng, grid.n_unknowns, 3)
        p1 = C.build_one_level(kern, mt)
        red = C.reduce_one_level(p1, 0.3)
        red2 = C.build_reduced_one_level(kern, mt, 0.3)
        m2 = np.full(grid.shape, 0.55 + 0.02j)
        p2 = C.build_two_level(kern, m2)
        out[f"pc_{tag}_dims"] = np.array(dims)
        out[f"pc_{tag}_tensors"] = kern.tensors
        out[f"pc_{tag}_mtilde"] = mt
        out[f"pc_{tag}_x"] = x
        out[f"pc_{tag}_xr"] = xr
        out[f"pc_{tag}_one_proxy"] = p1.proxy
        out[f"pc_{tag}_one_y"] = p1.apply(x)
        out[f"pc_{tag}_one_yr"] = p1.apply(xr)
        out[f"pc_{tag}_red_kept"] = red.kept
        out[f"pc_{tag}_red_slot"] = red.slot_of
        out[f"pc_{tag}_red_y"] = red.apply(x)
        out[f"pc_{tag}_red2_kept"] = red2.kept
        out[f"pc_{tag}_red2_proxy"] = red2.proxy
        out[f"pc_{tag}_red2_y"] = red2.apply(x)
        out[f"pc_{tag}_m2"] = m2
        out[f"pc_{tag}_two_y"] = p2.apply(x)
        out[f"pc_{tag}_two_yr"] = p2.apply(xr)

    # --- blocked (test_circulant.py:317-324 coupler_like)
    grid = VoxelGrid(8, 6, 2, 0.05)
    kern = assemble_kernel(grid, k0)
    eps = np.ones(grid.shape, complex)
    eps[:, 1:3, :] = 5.8
    eps[:, 3:5, :] = 5.8
    pmap = PermittivityMap(grid, eps)
    part = C.partition_boxes(grid, [C.Box("lo", 0, 8, 0, 3, 0, 2), C.Box("hi", 0, 8, 3, 6, 0, 2)])
    bp = C.build_blocked(kern, pmap, part, {"lo": "one-level", "hi": "two-level"})
    x = rfield(rng, grid.n_unknowns)
    out["blk_tensors"] = kern.tensors
    out["blk_eps"] = eps
    out["blk_x"] = x
    out["blk_y"] = bp.apply(x)
    part2 = C.partition_boxes(grid, [C.Box("a", 1, 7, 1, 5, 0, 2)])
    bp2 = C.build_blocked(kern, pmap, part2, {"a": "reduced-one-level"}, reduce_tol=0.2)
    out["blk2_y"] = bp2.apply(x)

    # --- GMRES on a small preconditioned VIE problem
    grid = VoxelGrid(16, 4, 3, 0.05)
    kern = assemble_kernel(grid, k0)
    plan = O.plan_operator(kern)
    eps = np.full(grid.shape, 5.8 + 0j)
    eps[:, :, 12:] -= 0.3j
    pmap = PermittivityMap(grid, eps)
    m = medium_coefficient(pmap)
    b = rfield(rng, grid.n_unknowns) * np.tile(m.reshape(-1), 3)
    p1 = C.build_one_level(kern, homogenize(pmap, "real_mean_x"))
    for tag, pinv, restart in [("none", None, None), ("one", p1.apply, None),
                               ("rst", p1.apply, 4), ("nrs", None, 7)]:
        xs, rep = S.gmres(lambda v: O.apply_system(plan, m, v), b, apply_pinv=pinv,
                          tol=1e-8, maxit=200, restart=restart)
        out[f"gm_{tag}_x"] = xs
        out[f"gm_{tag}_res"] = np.array(rep.residuals)
        out[f"gm_{tag}_its"] = np.array(rep.iterations)
        out[f"gm_{tag}_true"] = np.array(rep.true_residual)
    out["gm_tensors"] = kern.tensors
    out["gm_eps"] = eps
    out["gm_b"] = b


def sweep_cases(out):
    cfg = normalize(preset("waveguide-length"))
    rows = list(csv.DictReader(open("/root/reference/pkg/frontend/tests/fixtures/sweep.csv")))
    for row in rows:
        L = int(row["length_vox"])
        c = copy.deepcopy(cfg)
        c["device"]["geometry"]["length_vox"] = L
        prob = build_problem(c)
        tag = f"L{L}"
        out[f"{tag}_dims"] = np.array(prob.pmap.grid.dims)
        out[f"{tag}_delta"] = np.array(prob.pmap.grid.delta)
        out[f"{tag}_k0"] = np.array(prob.kernel.k0)
        out[f"{tag}_tensors"] = prob.kernel.tensors
        out[f"{tag}_eps"] = prob.pmap.eps_r
        out[f"{tag}_b"] = prob.b
        out[f"{tag}_tol"] = np.array(c["solver"]["tol"])
        out[f"{tag}_maxit"] = np.array(c["solver"]["maxit"])
        for key in ("none", "one_level_real_mean_x", "reduced_one_level_real_mean_x"):
            out[f"{tag}_its_{key}"] = np.array(int(row[f"iterations_{key}"]))
        out[f"{tag}_bytes_reduced"] = np.array(int(row["prec_bytes_reduced_one_level_real_mean_x"]))


def c0_case(out):
    from paper_1903_07884_b200 import workloads

    W = workloads.make("c0")
    grid = VoxelGrid(*W.grid.dims, W.grid.delta)
    kern = assemble_kernel(grid, W.physics.k0)
    plan = O.plan_operator(kern)
    pmap = PermittivityMap(grid, W.pmap.eps_r)
    m = medium_coefficient(pmap)
    b = W.b
    p1 = C.build_one_level(kern, homogenize(pmap, "real_mean_x"))
    xs, rep = S.gmres(lambda v: O.apply_system(plan, m, v), b, apply_pinv=p1.apply,
                      tol=W.tol, maxit=W.maxit, restart=W.restart)
    out["c0_b"] = b
    out["c0_x"] = xs
    out["c0_res"] = np.array(rep.residuals)
    out["c0_its"] = np.array(rep.iterations)
    out["c0_true"] = np.array(rep.true_residual)
    print("c0 iterations", rep.iterations, "true residual", rep.true_residual)


if __name__ == "__main__":
    for name, fn in [("golden_small.npz", small_cases), ("golden_sweep.npz", sweep_cases),
                     ("golden_c0.npz", c0_case)]:
        data = {}
        fn(data)
        np.savez_compressed(HERE / name, **data)
        print(name, sum(v.nbytes for v in data.values()) / 1e6, "MB raw")
