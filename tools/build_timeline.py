"""Kernel timeline of one warm preconditioner build (torch.profiler / CUPTI):
per-kernel totals, GPU busy vs wall.  usage: python tools/build_timeline.py [c1]"""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1903_07884_b200 import workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
W = workloads.make(name)
kern = W.kernel()
p = bench.build_prec(W, kern)
torch.cuda.synchronize()
del p
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA, torch.profiler.ProfilerActivity.CPU]) as prof:
    t0 = time.perf_counter()
    p = bench.build_prec(W, kern)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
busy = sum(e.device_time_total for e in evs) / 1e3
t_first = min(e.time_range.start for e in evs)
t_last = max(e.time_range.end for e in evs)
print(f"{name}: warm build wall {wall * 1e3:.2f} ms, GPU busy {busy:.2f} ms, first..last kernel {(t_last - t_first) / 1e3:.2f} ms")
rows = {}
for e in evs:
    r = rows.setdefault(e.name[:90], [0, 0.0])
    r[0] += 1
    r[1] += e.device_time_total / 1e3
for k, (n, t) in sorted(rows.items(), key=lambda kv: -kv[1][1]):
    print(f"{t:9.3f} ms {n:5d}  {k}")
print("-- launch order (start offset ms, duration ms)")
for e in sorted(evs, key=lambda e: e.time_range.start):
    print(f"{(e.time_range.start - t_first) / 1e3:9.3f} {e.device_time_total / 1e3:8.3f}  {e.name[:80]}")
