"""Profiling driver for the device generator assembly: python tools/prof_assemble.py [c1]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1903_07884_b200 import workloads  # noqa: E402
from paper_1903_07884_b200.kernel import assemble_kernel_device  # noqa: E402

W = workloads.make(sys.argv[1] if len(sys.argv) > 1 else "c1")
for _ in range(2):
    k = assemble_kernel_device(W.grid, W.physics.k0)
    del k
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
k = assemble_kernel_device(W.grid, W.physics.k0)
e1.record()
torch.cuda.synchronize()
print(f"assembly {W.grid.dims}: {e0.elapsed_time(e1):.3f} ms, {k.storage_bytes() / 1e9:.3f} GB written")
