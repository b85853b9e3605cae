"""Kernel-level timeline of one full preconditioned GMRES solve (torch.profiler
/ CUPTI): per-kernel totals, GPU-busy time vs the solve's wall time (= host
bubbles), number of launches.  usage: python tools/solve_timeline.py [c1]"""
import os
import sys
import time
from pathlib import Path

import numpy as np
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
                 maxit=min(W.maxit, int(os.environ.get("MAXIT", W.maxit))), restart=W.restart)


for _ in range(2):
    solve()
torch.cuda.synchronize()
t0 = time.perf_counter()
x, rep = solve()
torch.cuda.synchronize()
wall = time.perf_counter() - t0
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    x, rep = solve()
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
busy = sum(e.device_time_total for e in evs) / 1e3 if evs else 0.0
its = rep.iterations
print(f"{name}: {its} iterations, wall {wall * 1e3:.2f} ms ({wall * 1e3 / its:.3f} ms/it), "
      f"GPU busy {busy:.2f} ms ({busy / its:.3f} ms/it), launches {len(evs)} ({len(evs) / its:.1f}/it)")
rows = {}
for e in evs:
    k = e.name[:100]
    c, t = rows.get(k, (0, 0.0))
    rows[k] = (c + 1, t + e.device_time_total / 1e3)
for k, (c, t) in sorted(rows.items(), key=lambda kv: -kv[1][1]):
    print(f"{t:9.3f} ms {t / its:7.4f} ms/it {c:6d}  {k}")
