"""Time (and profile) the c1 preconditioner apply in isolation: builds the
c1 1-level preconditioner and applies it K times to a random vector.
Usage: python tools/solve_probe.py [config] [K]"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1903_07884_b200 import _native as nv, workloads  # noqa: E402
from paper_1903_07884_b200.kernel import assemble_kernel_device  # noqa: E402
import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 10
W = workloads.make(cfg)
kern = assemble_kernel_device(W.grid, W.physics.k0)
W._kernel = kern
prec = bench.build_prec(W, kern)
x = torch.randn(W.grid.n_unknowns, dtype=torch.complex128, device="cuda")
for _ in range(3):
    y = prec.apply(x)
torch.cuda.synchronize()
nv.timing_enable(True)
nv.timing_read("prec_solve")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(K):
    y = prec.apply(x)
e1.record()
torch.cuda.synchronize()
ms, n = nv.timing_read("prec_solve")
print(f"{cfg}: layout {getattr(prec, 'factor_layout', '?')} apply {e0.elapsed_time(e1) / K:.3f} ms, "
      f"solve {ms / max(n, 1):.3f} ms x {n}, factor bytes {getattr(prec, 'factor_bytes_per_apply', 0) / 1e9:.3f} GB")
