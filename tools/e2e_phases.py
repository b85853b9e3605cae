"""Host-side phases of one end-to-end solve (numpy b and m in, numpy x out):
solver.TRACE marks + wall time, next to the device-resident solve.

usage: python tools/e2e_phases.py [c1] [--reps 5]
"""
import argparse
import gc
import sys
import time
from pathlib import Path

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="c1")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()

import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1903_07884_b200 import solver, workloads  # noqa: E402
from paper_1903_07884_b200.operator import apply_system, plan_operator  # noqa: E402

W = workloads.make(a.config)
kern = W.kernel()
plan = plan_operator(kern)
prec = bench.build_prec(W, kern)
m_host = np.ascontiguousarray(W.m)
b_host = np.ascontiguousarray(W.b)
m_dev = torch.from_numpy(m_host.reshape(-1)).cuda()
b_dev = torch.from_numpy(b_host).cuda()


def run(host):
    if host:
        return solver.gmres(lambda v: apply_system(plan, m_host, v), b_host, apply_pinv=prec.apply, tol=W.tol,
                            maxit=W.maxit, restart=W.restart)
    return solver.gmres(lambda v: apply_system(plan, m_dev, v), b_dev, apply_pinv=prec.apply, tol=W.tol,
                        maxit=W.maxit, restart=W.restart)


for host in (False, True):
    keep = None
    for _ in range(3):
        keep = run(host)
    torch.cuda.synchronize()
    gc.collect()
    solver.TRACE = []
    walls = []
    for _ in range(a.reps):
        t0 = time.perf_counter()
        keep = run(host)
        torch.cuda.synchronize()
        walls.append((time.perf_counter() - t0) * 1e3)
    print("host buffers" if host else "device buffers", "wall ms:", [round(w, 2) for w in walls])
    for ent in [e for e in solver.TRACE if e[0] == "phases"][-3:]:
        print("   ", ent[1])
    solver.TRACE = None
