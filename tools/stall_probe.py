"""Where do the sporadic stalls come from?  (1) 400 operator + preconditioner applies
enqueued without any host synchronisation, one CUDA event per apply: gaps between
events show GPU-side stalls; (2) the same with a host synchronisation after every
apply: gaps show host-side stalls (the GMRES loop synchronises every iteration)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1903_07884_b200 import workloads  # noqa: E402
from paper_1903_07884_b200.operator import apply_device, plan_operator  # noqa: E402

W = workloads.make(sys.argv[1] if len(sys.argv) > 1 else "c1")
kern = W.kernel()
plan = plan_operator(kern)
prec = bench.build_prec(W, kern)
m = torch.from_numpy(W.m.reshape(-1).copy()).cuda()
x = torch.from_numpy(W.b.copy()).cuda()
N = 400


def run(sync):
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(N + 1)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    evs[0].record()
    for i in range(N):
        y = apply_device(plan, m, prec._apply_dev(x.reshape(-1, 1), 1).reshape(-1))
        evs[i + 1].record()
        if sync:
            evs[i + 1].synchronize()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    dt = np.array([evs[i].elapsed_time(evs[i + 1]) for i in range(N)])
    print(f"sync={sync}: wall {wall * 1e3:.1f} ms, per apply median {np.median(dt):.3f} ms, max {dt.max():.3f} ms, "
          f"n > 1.5 x median: {(dt > 1.5 * np.median(dt)).sum()}, sum of excess {np.clip(dt - np.median(dt), 0, None).sum():.1f} ms")


for rep in range(3):
    run(False)
    run(True)

# (3) full GMRES solves with the per-step host trace: which host phase stalls
from paper_1903_07884_b200 import solver  # noqa: E402
from paper_1903_07884_b200.operator import apply_system  # noqa: E402

b = torch.from_numpy(W.b.copy()).cuda()
A = lambda v: apply_system(plan, m, v)  # noqa: E731
for _ in range(3):
    solver.gmres(A, b, apply_pinv=prec.apply, tol=W.tol, maxit=W.maxit, restart=W.restart)
import gc  # noqa: E402

if "--freeze" in sys.argv:
    gc.collect()
    gc.freeze()
solver.TRACE = []
walls = []
for i in range(40):
    n0 = len(solver.TRACE)
    t0 = time.perf_counter()
    xs, rep = solver.gmres(A, b, apply_pinv=prec.apply, tol=W.tol, maxit=W.maxit, restart=W.restart)
    torch.cuda.synchronize()
    wl = (time.perf_counter() - t0) * 1e3
    walls.append(wl)
    if wl > 1.3 * min(walls):
        tr = [e for e in solver.TRACE[n0:] if e[0] != "phases"]
        print("   phases", [e[1] for e in solver.TRACE[n0:] if e[0] == "phases"])
        inloop = sum(a + c for _, a, c in tr) * 1e3
        worst = max(tr, key=lambda e: e[1] + e[2])
        print(f"solve {i}: {wl:.1f} ms (best {min(walls):.1f}); Arnoldi loop {inloop:.1f} ms; worst step j={worst[0]} "
              f"launch {worst[1] * 1e3:.2f} ms wait {worst[2] * 1e3:.2f} ms; launch total {sum(a for _, a, _ in tr) * 1e3:.1f}")
print("solve walls: median %.2f max %.2f" % (np.median(walls), max(walls)))
