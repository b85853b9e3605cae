"""Harness integration of the GPU hot path.

The reference's orchestration layer (pkg/src/voxvie/harness.py:103-236) builds a
``Problem`` and calls ``build_preconditioner`` / ``solve_problem`` / ``run``.
This module provides the same three entry points on top of the GPU operator,
preconditioners and GMRES, with the same configuration keys, summaries, byte
accounting and output files (reference io.py:23-119), so a caller can swap
``voxvie.harness.solve_problem`` for this one.  Problem *construction*
(geometry builders, dipole source, YAML config) stays in the reference and is
out of scope here: any object with the reference ``Problem``'s attributes is
accepted (``problem_from`` builds one from host arrays).
"""

from __future__ import annotations

import csv
import json
import time
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .circulant import (Box, build_blocked, build_one_level, build_reduced_one_level, build_two_level,
                        partition_boxes)
from .errors import ConfigError
from .grid import PermittivityMap, Physics, dielectric_ratio, homogenize, medium_coefficient
from .operator import OperatorPlan, field_from_currents, plan_operator, rhs_from_incident
from .operator import apply_system
from .solver import gmres

HOMOG_NAMES = ("mode", "mean-x", "real-mean-x", "mean_x", "real_mean_x")


def homog_internal(name: str) -> str:
    """reference config.py:75-78."""
    if name not in HOMOG_NAMES:
        raise ConfigError(f"unknown homogenization {name!r}; expected one of {HOMOG_NAMES}")
    return name.replace("-", "_")


@dataclass
class Problem:
    """Everything one solve needs (reference harness.py:59-71)."""

    config: dict
    physics: Physics
    pmap: PermittivityMap
    hint: object
    kernel: object
    plan: object
    m: np.ndarray
    e_inc: np.ndarray
    b: np.ndarray
    extra: dict = field(default_factory=dict)


def problem_from(kernel, pmap: PermittivityMap, e_inc, physics: Physics, *, hint=None, config=None) -> Problem:
    """Problem from host inputs: GPU operator plan, medium map and RHS."""
    m = medium_coefficient(pmap)
    return Problem(config=config or {}, physics=physics, pmap=pmap, hint=hint, kernel=kernel,
                   plan=plan_operator(kernel), m=m, e_inc=np.asarray(e_inc, np.complex128).reshape(-1),
                   b=rhs_from_incident(m, e_inc, physics))


def _gpu_plan(problem) -> OperatorPlan:
    """Our plan for the problem (a reference Problem carries a numpy plan)."""
    if isinstance(problem.plan, OperatorPlan):
        return problem.plan
    cached = getattr(problem, "_vx_plan", None)
    if cached is None:
        cached = plan_operator(problem.kernel)
        try:
            object.__setattr__(problem, "_vx_plan", cached)
        except Exception:  # pragma: no cover
            pass
    return cached


def build_preconditioner(problem, prec_cfg: dict):
    """Returns (apply or None, summary dict, build seconds) (reference harness.py:145-188)."""
    kind = prec_cfg["kind"]
    if kind == "none":
        return None, {"level": "none", "bytes": 0}, 0.0
    cap = int(prec_cfg.get("cap_mb", 2048) * 2 ** 20)
    strategy = homog_internal(prec_cfg.get("homogenization", "real-mean-x"))
    reduce_tol = prec_cfg.get("reduce_tol", 1e-3)
    t0 = time.perf_counter()
    if kind == "blocked":
        partition = partition_boxes(problem.pmap.grid, problem.hint.boxes)
        levels = dict(problem.hint.levels)
        if prec_cfg.get("box_levels"):
            levels.update(prec_cfg["box_levels"])
        homog_map = {label: homog_internal(name)
                     for label, name in (prec_cfg.get("box_homogenization") or {}).items()}
        prec = build_blocked(problem.kernel, problem.pmap, partition, levels, homog=homog_map,
                             reduce_tol=reduce_tol, cap_bytes=cap)
    else:
        mtilde = homogenize(problem.pmap, strategy)
        if kind == "one-level":
            prec = build_one_level(problem.kernel, mtilde, cap_bytes=cap)
        elif kind == "reduced-one-level":
            prec = build_reduced_one_level(problem.kernel, mtilde, reduce_tol, cap_bytes=cap)
        elif kind == "two-level":
            mode_const = homogenize(problem.pmap, "mode") if strategy != "mode" else mtilde
            prec = build_two_level(problem.kernel, mode_const, cap_bytes=cap)
        else:
            raise ConfigError(f"unknown preconditioner kind {kind!r}")
    import torch

    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    summary = prec.summary()
    summary["build_seconds"] = build_s
    summary["homogenization"] = prec_cfg.get("homogenization", "real-mean-x")
    return prec.apply, summary, build_s


def solve_problem(problem, prec_cfg: dict):
    """One preconditioned solve -> (currents, report, prec summary) (reference harness.py:191-211)."""
    apply_pinv, summary, build_s = build_preconditioner(problem, prec_cfg)
    scfg = problem.config.get("solver", {})
    plan = _gpu_plan(problem)
    m = problem.m
    x, report = gmres(lambda v: apply_system(plan, m, v), problem.b, apply_pinv=apply_pinv,
                      tol=scfg.get("tol", 1e-4), maxit=scfg.get("maxit", 2000), restart=scfg.get("restart"))
    report.build_seconds = build_s
    report.memory = {
        "kernel_bytes": problem.kernel.storage_bytes(),
        "operator_plan_bytes": plan.storage_bytes(),
        "preconditioner_bytes": int(summary.get("bytes", 0)),
        "krylov_basis_bytes": report.iterations * problem.b.size * 16,
    }
    return x, report, summary


# ---------------------------------------------------------------- file formats
def write_field(path, grid, field_vals, *, wavelength=None):
    """field.bin (little-endian interleaved complex128, canonical ordering) + JSON
    sidecar (reference io.py:23-40)."""
    path = Path(path)
    data = np.ascontiguousarray(field_vals, dtype="<c16").reshape(-1)
    if data.size != grid.n_unknowns:
        raise ValueError(f"field has {data.size} entries, expected {grid.n_unknowns}")
    data.tofile(path)
    side = {"dims": [grid.nx, grid.ny, grid.nz], "delta": grid.delta, "origin": list(grid.origin),
            "component_order": "x,y,z", "layout": "component-major, x fastest", "dtype": "complex128-le",
            "wavelength": wavelength}
    path.with_suffix(".json").write_text(json.dumps(side, indent=2) + "\n")


def read_field(path):
    path = Path(path)
    side = json.loads(path.with_suffix(".json").read_text())
    nx, ny, nz = side["dims"]
    data = np.fromfile(path, dtype="<c16")
    if data.size != 3 * nx * ny * nz:
        raise ValueError(f"{path} holds {data.size} entries, sidecar promises {3 * nx * ny * nz}")
    return data.astype(np.complex128), side


def write_residuals(path, residuals, seconds_per_iter=None):
    """residuals.csv (reference io.py:81-91)."""
    with Path(path).open("w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["iter", "relative_residual", "cumulative_seconds"])
        cum = 0.0
        for i, res in enumerate(residuals):
            if seconds_per_iter is not None and i > 0:
                cum += seconds_per_iter
            w.writerow([i, f"{res:.16e}", f"{cum:.6f}"])


def read_residuals(path):
    with Path(path).open(newline="") as fh:
        return [float(r["relative_residual"]) for r in csv.DictReader(fh)]


def write_report(path, report: dict):
    Path(path).write_text(json.dumps(report, indent=2, sort_keys=True) + "\n")


def run_problem(problem, prec_cfg: dict, outdir) -> Path:
    """Solve and write field.bin/.json, residuals.csv, report.json (the output
    half of reference harness.py:214-236)."""
    outdir = Path(outdir)
    outdir.mkdir(parents=True, exist_ok=True)
    w, report, summary = solve_problem(problem, prec_cfg)
    e_total = field_from_currents(_gpu_plan(problem), w, problem.e_inc, problem.physics)
    grid = problem.pmap.grid
    write_field(outdir / "field.bin", grid, e_total, wavelength=problem.physics.lambda0)
    spi = report.solve_seconds / report.iterations if report.iterations else None
    write_residuals(outdir / "residuals.csv", report.residuals, spi)
    write_report(outdir / "report.json", {
        "solve": report.to_dict(), "preconditioner": summary,
        "grid": {"dims": list(grid.dims), "delta": grid.delta, "voxels": grid.n_voxels},
        "dielectric_ratio": dielectric_ratio(problem.pmap)})
    return outdir


__all__ = ["Box", "Problem", "build_preconditioner", "homog_internal", "problem_from", "read_field",
           "read_residuals", "run_problem", "solve_problem", "write_field", "write_report", "write_residuals"]
