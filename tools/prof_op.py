"""Profiling driver: build a workload's operator (and 1-level preconditioner)
and run N applies, so ncu can capture exactly the hot kernels.

usage: python tools/prof_op.py [c1] [--apply op|prec|both] [--reps 3]
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1903_07884_b200 import workloads  # noqa: E402
from paper_1903_07884_b200.circulant import build_one_level  # noqa: E402
from paper_1903_07884_b200.operator import apply_device, plan_operator  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="c1")
ap.add_argument("--apply", default="op")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
W = workloads.make(a.config)
kern = W.kernel()
plan = plan_operator(kern)
m = torch.from_numpy(W.m.reshape(-1).copy()).cuda()
x = torch.from_numpy(W.b.copy()).cuda()
prec = build_one_level(kern, W.mtilde(), cap_bytes=2 ** 62) if a.apply in ("prec", "both") else None
torch.cuda.synchronize()
for _ in range(2):
    y = apply_device(plan, m, x)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    if a.apply in ("op", "both"):
        y = apply_device(plan, m, x)
    if prec is not None:
        y = prec._apply_dev(x.reshape(-1, 1), 1)
e1.record()
torch.cuda.synchronize()
print(f"{a.config} {a.apply}: {e0.elapsed_time(e1) / a.reps:.3f} ms per apply")
