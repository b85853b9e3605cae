"""Profiling driver: build a workload's preconditioner (bench.build_prec) and
time N applies with CUDA events.  usage: prof_prec.py [c1r] [napply]"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1903_07884_b200 import workloads  # noqa: E402

from paper_1903_07884_b200 import _native as nv  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
name = args[0] if args else "c1r"
napply = int(args[1]) if len(args) > 1 else 5
if "--seq" in sys.argv:
    nv.load()
    nv.call("vx_rep_variant", 1)
W = workloads.make(name)
kern = W.kernel()
prec = bench.build_prec(W, kern)
rng = np.random.default_rng(0)
n = W.grid.n_unknowns
x = torch.from_numpy(rng.normal(size=n) + 1j * rng.normal(size=n)).cuda()
y = prec.apply(x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(napply):
    y = prec.apply(x)
e1.record()
torch.cuda.synchronize()
print(f"{name}: {e0.elapsed_time(e1) / napply:.3f} ms/apply, prec bytes {prec.bytes / 1e9:.3f} GB")
print("layout", getattr(prec, "factor_layout", None), "syminv_err", getattr(prec, "_syminv_err", None))
