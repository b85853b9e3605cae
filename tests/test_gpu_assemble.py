"""Device kernel assembly (vx_assemble_green) against the
host restatement of the reference assembly (kernel.py:152-198) that the golden
vectors pin (tests/test_oracle_golden.py), and the operator / preconditioner
built from the device generators against the host-generator path."""

import numpy as np
import pytest

from paper_1903_07884_b200.grid import VoxelGrid
from paper_1903_07884_b200.kernel import assemble_kernel

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dims,delta,k0,near", [((7, 5, 3), 0.05, 2 * np.pi, False),
                                                ((6, 4, 5), 0.05, 2 * np.pi, True),
                                                ((200, 10, 5), 0.045, 2 * np.pi / 1.55, False),
                                                ((1, 1, 1), 0.1, 3.0, False),
                                                ((40, 1, 3), 0.02, 4.05, True)])
def test_device_generators_match_host(dims, delta, k0, near):
    from paper_1903_07884_b200.kernel import assemble_kernel_device

    g = VoxelGrid(*dims, delta)
    host = assemble_kernel(g, k0, near_gauss=near).tensors
    dev = assemble_kernel_device(g, k0, near_gauss=near)
    d = dev._vx_device_tensors.cpu().numpy()
    assert d.shape == host.shape
    scale = np.abs(host).max()
    assert np.max(np.abs(d - host)) <= 1e-14 * scale
    # exact structure: zeros where the host has zeros, the parity signs
    assert np.array_equal(host == 0, d == 0)
    assert np.array_equal(np.sign(host.real[np.abs(host.real) > 1e-12 * scale]),
                          np.sign(d.real[np.abs(host.real) > 1e-12 * scale]))
    assert np.array_equal(dev.tensors, d)          # lazy host view
    assert dev.storage_bytes() == host.nbytes


def test_device_kernel_drives_operator_and_preconditioner():
    import torch

    from paper_1903_07884_b200 import workloads
    from paper_1903_07884_b200.circulant import build_one_level
    from paper_1903_07884_b200.kernel import assemble_kernel_device
    from paper_1903_07884_b200.operator import apply_system, plan_operator

    W = workloads.make("c0")
    kh = W.kernel()
    kd = assemble_kernel_device(W.grid, W.physics.k0)
    x = np.random.default_rng(3).normal(size=W.grid.n_unknowns) + 0.25j
    yh = apply_system(plan_operator(kh), W.m, x)
    yd = apply_system(plan_operator(kd), W.m, x)
    assert np.linalg.norm(yd - yh) <= 1e-12 * np.linalg.norm(yh)
    ph = build_one_level(kh, W.mtilde())
    pd = build_one_level(kd, W.mtilde())
    xd = torch.from_numpy(x).cuda()
    zh, zd = ph.apply(xd).cpu().numpy(), pd.apply(xd).cpu().numpy()
    assert np.linalg.norm(zd - zh) <= 1e-11 * np.linalg.norm(zh)


def test_device_generators_match_reference_golden(golden_small):
    """Pinned against tensors produced by the unmodified reference (make_golden.py)."""
    from conftest import relerr

    from paper_1903_07884_b200.kernel import assemble_kernel_device

    for tag in ["small", "cube", "one", "odd", "prime", "long"]:
        dims = tuple(int(v) for v in golden_small[f"op_{tag}_dims"])
        k = assemble_kernel_device(VoxelGrid(*dims, 0.05), 2 * np.pi, near_gauss=(tag == "odd"))
        assert relerr(k._vx_device_tensors.cpu().numpy(), golden_small[f"op_{tag}_tensors"]) < 1e-14
