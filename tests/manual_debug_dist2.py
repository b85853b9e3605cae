"""Debug: stages of DistTwoLevelPrec (P=1) against numpy."""
import sys
from pathlib import Path

import numpy as np
import scipy.fft
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
import voxvie_oracle as O  # noqa: E402
from paper_1903_07884_b200 import workloads  # noqa: E402
from paper_1903_07884_b200.dist import CudaBackend, DistTwoLevelPrec, Layout  # noqa: E402
from paper_1903_07884_b200.operator import padded_length  # noqa: E402


class C1:
    def all_to_all(self, out, inp, os_, is_):
        out.copy_(inp[:out.numel()])

    def all_reduce(self, t):
        return t


W = workloads.small(37, 10, 4, delta=0.03e-6)
kern = W.kernel()
nx, ny, nz = W.grid.dims
mt = complex(np.mean(W.m))
print("mt", mt)
B = CudaBackend()
L = Layout(W.grid.dims, 1, 0, padded_length(nx))
p = DistTwoLevelPrec(kern, mt, L, B, C1())
rng = np.random.default_rng(0)
Y = rng.normal(size=3 * nz * ny * nx) + 1j * rng.normal(size=3 * nz * ny * nx)
Yd = torch.from_numpy(Y.copy()).cuda()
B.dft_y(Yd, 3 * nz, ny, nx, False)
ref = scipy.fft.fft(Y.reshape(3 * nz, ny, nx), axis=1).reshape(-1)
print("dft_y err", np.abs(Yd.cpu().numpy() - ref).max() / np.abs(ref).max())
Z = Yd.clone()
B.solve(Z, p.n, p.factors, p.perm, p.items, p.n_slots, p.n_slots, p.klist, ny * nx)
print("solve changed", np.abs(Z.cpu().numpy() - Yd.cpu().numpy()).max())
op = O.build_two_level(kern.tensors, W.grid.dims, mt)
from scipy.linalg import lu_solve  # noqa: E402
zz = ref.reshape(3 * nz, ny, nx).copy()
for l in range(ny):
    for k in range(nx):
        zz[:, l, k] = lu_solve((op["lu"][l, k], op["piv"][l, k]), zz[:, l, k])
print("solve err", np.abs(Z.cpu().numpy() - zz.reshape(-1)).max() / np.abs(zz).max())
print("items", p.items[:9].cpu().numpy(), p.items.dtype, "klist", p.klist[:5].cpu().numpy(), p.klist.dtype,
      "n_slots", p.n_slots, "fac", tuple(p.factors.shape), "perm", tuple(p.perm.shape))
