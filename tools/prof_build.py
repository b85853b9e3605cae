"""Profiling driver: one 1-level preconditioner build of a workload (one
lu_build_kernel launch over all frequency blocks).  usage: prof_build.py [c1]"""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1903_07884_b200 import workloads  # noqa: E402
from paper_1903_07884_b200.circulant import build_one_level  # noqa: E402

from paper_1903_07884_b200 import _native as nv  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
nv.load()
nv.query("vx_lu_variant", 1 if "--mono" in sys.argv else 0)
W = workloads.make(name)
kern = W.kernel()
torch.cuda.synchronize()
t0 = time.perf_counter()
prec = build_one_level(kern, W.mtilde(), cap_bytes=2 ** 62)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
torch.cuda.synchronize()
t0 = time.perf_counter()
prec = build_one_level(kern, W.mtilde(), cap_bytes=2 ** 62)
torch.cuda.synchronize()
print(f"{name} build {dt:.3f} s (first), {time.perf_counter() - t0:.3f} s (second), "
      f"{prec.grid.nx} blocks of {prec.block_size}^2, {'monolithic' if '--mono' in sys.argv else 'step-batched'}")
