"""Replicates bench.py's e2e loop (numpy b and alternating numpy m in, numpy x
out) with a per-phase wall breakdown.  usage: e2e_loop_probe.py [c1]"""
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1903_07884_b200 import _native as nv  # noqa: E402
from paper_1903_07884_b200 import workloads  # noqa: E402
import bench  # noqa: E402
from paper_1903_07884_b200.operator import apply_system, plan_operator  # noqa: E402
from paper_1903_07884_b200.solver import gmres  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
W = workloads.make(name)
kern = W.kernel()
plan = plan_operator(kern)
prec = bench.build_prec(W, kern)
m_host, b_host = W.m, W.b
m_copies = [np.array(m_host, copy=True), np.array(m_host, copy=True)]
print("staged min", nv.H2D_STAGED_MIN, "threads env", os.environ.get("VX_H2D_THREADS"), flush=True)
cnt = [0]


def step():
    ms = m_copies[cnt[0] % 2]
    cnt[0] += 1
    return gmres(lambda v: apply_system(plan, ms, v), b_host, apply_pinv=prec.apply,
                 tol=W.tol, maxit=W.maxit, restart=W.restart)


m_dev = torch.from_numpy(m_host.reshape(-1).copy()).cuda()
b_dev = torch.from_numpy(b_host.copy()).cuda()


def variant(b, m_alt):
    def f():
        ms = m_copies[cnt[0] % 2] if m_alt else m_dev
        cnt[0] += 1
        return gmres(lambda v: apply_system(plan, ms, v), b, apply_pinv=prec.apply,
                     tol=W.tol, maxit=W.maxit, restart=W.restart)
    return f


for lab, fn in [("A dev b, dev m", variant(b_dev, False)), ("B host b, dev m", variant(b_host, False)),
                ("C dev b, host m alt", variant(b_dev, True)), ("D host b, host m alt (e2e)", variant(b_host, True)),
                ("A dev b, dev m", variant(b_dev, False))]:
    for _ in range(3):
        keep = fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(6):
        keep = fn()
    torch.cuda.synchronize()
    print(f"{lab:28s} {(time.perf_counter() - t0) / 6 * 1e3:.2f} ms/solve  its {keep[1].iterations}", flush=True)
xd = nv.device_c128(b_host)
for lab, fn in [("upload b", lambda: nv.device_c128(b_host)), ("upload m", lambda: nv.device_c128(m_copies[0])),
                ("to_host x", lambda: nv.to_host(xd))]:
    for _ in range(3):
        keep = fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(6):
        keep = fn()
    torch.cuda.synchronize()
    print(f"{lab:28s} {(time.perf_counter() - t0) / 6 * 1e3:.2f} ms", flush=True)
