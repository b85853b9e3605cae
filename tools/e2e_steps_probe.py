"""Per-step wall times of the bench's e2e loop (numpy b, alternating numpy m,
numpy x out) with phase split: which step stalls and where."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1903_07884_b200 import workloads  # noqa: E402
from paper_1903_07884_b200.kernel import assemble_kernel_device  # noqa: E402
from paper_1903_07884_b200.operator import apply_system, plan_operator  # noqa: E402
from paper_1903_07884_b200.solver import gmres  # noqa: E402

W = workloads.make(sys.argv[1] if len(sys.argv) > 1 else "c1")
kern = assemble_kernel_device(W.grid, W.physics.k0)
plan = plan_operator(kern)
prec = bench.build_prec(W, kern)
mc = [np.array(W.m, copy=True), np.array(W.m, copy=True)]
b_host = W.b
cnt = [0]


def step():
    ms = mc[cnt[0] % 2]
    cnt[0] += 1
    return gmres(lambda v: apply_system(plan, ms, v), b_host, apply_pinv=prec.apply, tol=W.tol, maxit=W.maxit,
                 restart=W.restart)


x = None
for _ in range(3):
    x, _ = step()
torch.cuda.synchronize()
for i in range(10):
    t0 = time.perf_counter()
    x, rep = step()
    t1 = time.perf_counter()
    print(f"step {i}: {(t1 - t0) * 1e3:.2f} ms  (solve_seconds {rep.solve_seconds * 1e3:.2f})", flush=True)
bd, md = torch.from_numpy(b_host.copy()).cuda(), torch.from_numpy(W.m.reshape(-1).copy()).cuda()
for i in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    xd, rep = gmres(lambda v: apply_system(plan, md, v), bd, apply_pinv=prec.apply, tol=W.tol, maxit=W.maxit,
                    restart=W.restart)
    torch.cuda.synchronize()
    print(f"device-resident solve {i}: {(time.perf_counter() - t0) * 1e3:.2f} ms, its {rep.iterations}", flush=True)
