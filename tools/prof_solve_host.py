"""Host-side cost of a device-resident GMRES solve (cProfile, tottime) and the
host time per iteration spent outside the event waits.  usage: prof_solve_host.py [c1]"""
import cProfile
import pstats
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1903_07884_b200 import workloads  # noqa: E402
from paper_1903_07884_b200.operator import apply_system, plan_operator  # noqa: E402
from paper_1903_07884_b200.solver import gmres  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
W = workloads.make(name)
kern = W.kernel()
plan = plan_operator(kern)
prec = bench.build_prec(W, kern)
m_dev = torch.from_numpy(W.m.reshape(-1).copy()).cuda()
b_dev = torch.from_numpy(W.b.copy()).cuda()


def solve():
    return gmres(lambda v: apply_system(plan, m_dev, v), b_dev, apply_pinv=prec.apply, tol=W.tol,
                 maxit=W.maxit, restart=W.restart)


for _ in range(3):
    solve()
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
x, rep = solve()
torch.cuda.synchronize()
pr.disable()
dt = time.perf_counter() - t0
print(f"{name}: {rep.iterations} its, {dt * 1e3:.2f} ms ({dt / rep.iterations * 1e3:.3f} ms/it)")
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
