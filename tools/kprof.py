"""Per-kernel device times of the hot path via torch.profiler (CUPTI), no ncu
replay: builds a workload's operator + preconditioner, warms up, then profiles
`reps` operator applies, preconditioner applies and Arnoldi steps.

usage: python tools/kprof.py [c1] [--reps 5] [--env K=V ...]
"""
import argparse
import os
import sys
from pathlib import Path

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="c1")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--env", nargs="*", default=[])
ap.add_argument("--what", default="op,prec,arnoldi")
ap.add_argument("--nvec", type=int, default=20)
ap.add_argument("--seq", action="store_true", help="also list the launches of one step in order")
a = ap.parse_args()
for kv in a.env:
    k, v = kv.split("=", 1)
    os.environ[k] = v

import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1903_07884_b200 import _native as nv  # noqa: E402
from paper_1903_07884_b200 import workloads  # noqa: E402
from paper_1903_07884_b200.operator import apply_device, plan_operator  # noqa: E402

W = workloads.make(a.config)
kern = W.kernel()
what = a.what.split(",")
plan = plan_operator(kern)
m = torch.from_numpy(W.m.reshape(-1).copy()).cuda()
rng = np.random.default_rng(0)
n = W.grid.n_unknowns
x = torch.from_numpy(rng.normal(size=n) + 1j * rng.normal(size=n)).cuda()
prec = bench.build_prec(W, kern) if "prec" in what else None
nvec = a.nvec
V = torch.from_numpy(rng.normal(size=(nvec + 1, n)) + 0j).cuda()
h = torch.zeros(nvec + 2, dtype=torch.complex128, device="cuda")
stats = torch.zeros(4, dtype=torch.float64, device="cuda")
part = torch.zeros(int(nv.query("vx_arnoldi_part_elems", n, nvec + 2)), dtype=torch.complex128, device="cuda")


def step():
    if "op" in what:
        apply_device(plan, m, x)
    if prec is not None:
        prec._apply_dev(x.reshape(-1, 1), 1)
    if "arnoldi" in what:
        w = x.clone()
        nv.call("vx_arnoldi_step", n, nvec, V.data_ptr(), n, w.data_ptr(), V[nvec].data_ptr(), h.data_ptr(),
                stats.data_ptr(), part.data_ptr(), nv.stream_ptr())


for _ in range(2):
    step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    step()
e1.record()
torch.cuda.synchronize()
print(f"{a.config} [{a.what}] {e0.elapsed_time(e1) / a.reps:.3f} ms per step (events, no profiler)")
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(a.reps):
        step()
    torch.cuda.synchronize()
rows = []
for ev in prof.key_averages():
    t = getattr(ev, "device_time_total", None) or getattr(ev, "cuda_time_total", 0)
    if t > 0:
        rows.append((t / a.reps / 1e3, ev.count / a.reps, ev.key[:110]))
rows.sort(reverse=True)
tot = sum(r[0] for r in rows)
print(f"{'ms/step':>9} {'n/step':>6}  kernel   (total {tot:.3f} ms)")
for t, c, k in rows:
    print(f"{t:9.4f} {c:6.1f}  {k}")

if a.seq:
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof2:
        step()
        torch.cuda.synchronize()
    evs = [e for e in prof2.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    print("-- one step in launch order")
    for e in sorted(evs, key=lambda e: e.time_range.start):
        print(f"{e.device_time_total / 1e3:9.4f}  {e.name[:110]}")
