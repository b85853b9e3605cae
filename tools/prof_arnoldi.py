"""Profiling driver: vx_arnoldi_step on a random orthonormal-ish basis.
usage: prof_arnoldi.py [n=3524000] [nvec=50] [reps=10]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1903_07884_b200 import _native as nv  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3524000
nvec = int(sys.argv[2]) if len(sys.argv) > 2 else 50
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
nv.load()
g = torch.Generator(device="cuda").manual_seed(0)
V = torch.randn(nvec + 1, n, dtype=torch.complex128, device="cuda", generator=g) / n ** 0.5
w0 = torch.randn(n, dtype=torch.complex128, device="cuda", generator=g)
h = nv.empty_c128(nvec + 2)
stats = torch.zeros(4, dtype=torch.float64, device="cuda")
part = nv.empty_c128(int(nv.query("vx_arnoldi_part_elems", n, nvec + 2)))
vn = nv.empty_c128(n)
w = w0.clone()


def step():
    w.copy_(w0)
    nv.call("vx_arnoldi_step", n, nvec, V.data_ptr(), n, w.data_ptr(), vn.data_ptr(), h.data_ptr(),
            stats.data_ptr(), part.data_ptr(), nv.stream_ptr())


step()
torch.cuda.synchronize()
e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
e0.record()
for _ in range(reps):
    w.copy_(w0)
e1.record()
for _ in range(reps):
    step()
e2.record()
torch.cuda.synchronize()
ms = (e1.elapsed_time(e2) - e0.elapsed_time(e1)) / reps
gb = (2 * nvec + 5) * n * 16 / 1e9
print(f"arnoldi n={n} nvec={nvec}: {ms:.3f} ms/step, {gb / ms:.0f} GB/s algorithmic (2(j+1)+5 vectors)")
