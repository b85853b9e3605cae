"""Kernel timeline of one SHARDED solve on a 1-rank NCCL group (the code path `bench.py --gpus N`
runs on every rank): per-kernel totals per iteration.  usage: python tools/shard_timeline.py [c1]"""
import os
import socket
import sys
import time
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1903_07884_b200 import workloads  # noqa: E402
from paper_1903_07884_b200.dist import (CudaBackend, DistOneLevelPrec, DistOperator, Layout, _Comm,  # noqa: E402
                                        gmres_sharded)
from paper_1903_07884_b200.operator import padded_length  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
sk = socket.socket()
sk.bind(("127.0.0.1", 0))
os.environ.setdefault("MASTER_PORT", str(sk.getsockname()[1]))
sk.close()
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
W = workloads.make(name)
kern = W.kernel()
B, C = CudaBackend(), _Comm()
L = Layout(W.grid.dims, 1, 0, padded_length(W.grid.nx))
op = DistOperator(kern, L, B, C)
prec = DistOneLevelPrec(kern, W.mtilde(), L, B, C, cap_bytes=2 ** 62)
m = torch.from_numpy(W.m.reshape(-1).copy()).cuda()
b = torch.from_numpy(np.ascontiguousarray(L.local_slice(W.b))).cuda()


def solve():
    return gmres_sharded(lambda v: op.apply(m, v), b, B, C, apply_pinv=prec.apply, tol=W.tol, maxit=W.maxit,
                         restart=W.restart)


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
busy = sum(e.device_time_total for e in evs) / 1e3
its = rep.iterations
print(f"{name} sharded P=1: {its} iterations, wall {wall * 1e3:.2f} ms ({wall * 1e3 / its:.3f} ms/it), "
      f"GPU busy {busy:.2f} ms ({busy / its:.3f} ms/it), launches {len(evs)} ({len(evs) / its:.1f}/it)")
rows = {}
for e in evs:
    c, t = rows.get(e.name[:100], (0, 0.0))
    rows[e.name[:100]] = (c + 1, t + e.device_time_total / 1e3)
for k, (c, t) in sorted(rows.items(), key=lambda kv: -kv[1][1])[:28]:
    print(f"{t / its:8.4f} ms/it {c / its:6.1f}/it  {k}")
dist.destroy_process_group()
