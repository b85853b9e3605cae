"""One-off full-size check of BASELINE c4 (2-level, restart 100): the GPU
residual history of the first restart cycle against the CPU oracle's on the
same arrays (~8 min of CPU).  usage: python tests/manual_check_c4.py [maxit]"""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import voxvie_oracle as O  # noqa: E402
from paper_1903_07884_b200 import workloads  # noqa: E402
from paper_1903_07884_b200.circulant import build_two_level  # noqa: E402
from paper_1903_07884_b200.operator import apply_system, plan_operator  # noqa: E402
from paper_1903_07884_b200.solver import gmres  # noqa: E402

maxit = int(sys.argv[1]) if len(sys.argv) > 1 else 100
W = workloads.make("c4")
kern = W.kernel()
m = W.m
plan = plan_operator(kern)
prec = build_two_level(kern, W.mtilde(), cap_bytes=2 ** 62)
t0 = time.time()
x, rep = gmres(lambda v: apply_system(plan, m, v), W.b, apply_pinv=prec.apply, tol=W.tol, maxit=maxit,
               restart=W.restart)
print("gpu", rep.iterations, rep.converged, rep.residuals[-1], time.time() - t0, flush=True)
dims = W.grid.dims
t0 = time.time()
spec = O.plan_spectra(kern.tensors, dims, workers=16)
p2 = O.build_two_level(kern.tensors, dims, W.mtilde())
print("oracle setup", time.time() - t0, flush=True)
rng = np.random.default_rng(1)
v = rng.normal(size=W.grid.n_unknowns) + 1j * rng.normal(size=W.grid.n_unknowns)
e_op = np.linalg.norm(apply_system(plan, m, v) - O.apply_system(spec, dims, m, v, workers=16)) / np.linalg.norm(v)
pv = O.apply_prec(p2, v)
e_pc = np.linalg.norm(prec.apply(v) - pv) / np.linalg.norm(pv)
print(f"full-size parity: matvec {e_op:.2e}  2-level apply {e_pc:.2e}", flush=True)
t0 = time.time()
xo, ro = O.gmres(lambda u: O.apply_system(spec, dims, m, u, workers=16), W.b,
                 apply_pinv=lambda u: O.apply_prec(p2, u), tol=W.tol, maxit=maxit, restart=W.restart)
print("oracle", ro["iterations"], ro["converged"], ro["residuals"][-1], time.time() - t0, flush=True)
r_g = np.array(rep.residuals)
r_o = np.array(ro["residuals"])
n = min(len(r_g), len(r_o))
print("max rel diff of residual histories:", np.max(np.abs(r_g[:n] - r_o[:n]) / r_o[:n]))
print("field rel diff:", np.linalg.norm(x - xo) / np.linalg.norm(xo))
for i in (1, 10, 25, 50, 75, n - 1):
    if i < n:
        print(i, r_g[i], r_o[i])
