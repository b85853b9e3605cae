"""Host-buffer boundary: pageable numpy uploads through the library's threaded
pinned ring (vx_h2d_staged) are bitwise the host data, for sizes around the
chunk (2 MB) and round (64 MB) boundaries, on a side stream, and through the
public API (apply_system with numpy in/out equals the device-tensor call)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [1, 131071, 131072, 131073, 4 << 20, (4 << 20) + 7, 9_000_001])
def test_staged_upload_bitwise(n):
    import torch

    from paper_1903_07884_b200 import _native as nv

    rng = np.random.default_rng(n)
    a = rng.normal(size=n) + 1j * rng.normal(size=n)
    out = torch.empty(n, dtype=torch.complex128, device="cuda")
    nv.call("vx_h2d_staged", out.data_ptr(), a.ctypes.data, a.nbytes, nv.stream_ptr())
    back = out.cpu().numpy()
    assert np.array_equal(back.view(np.float64), a.view(np.float64))


def test_staged_upload_side_stream_and_reuse():
    import torch

    from paper_1903_07884_b200 import _native as nv

    rng = np.random.default_rng(5)
    s = torch.cuda.Stream()
    outs, srcs = [], []
    with torch.cuda.stream(s):
        for k in range(4):  # consecutive calls recycle the same pinned slots
            a = rng.normal(size=3_000_000) + 1j * k
            srcs.append(a)
            outs.append(nv.device_c128(a))
    s.synchronize()
    for a, o in zip(srcs, outs):
        assert np.array_equal(o.cpu().numpy(), a)
    assert nv.query("vx_h2d_threads") >= 1


def test_numpy_boundary_equals_device_call(monkeypatch):
    import torch

    from paper_1903_07884_b200 import _native as nv
    from paper_1903_07884_b200 import workloads

    monkeypatch.setattr(nv, "H2D_STAGED_MIN", 0)  # c0 vectors are below the staging threshold
    from paper_1903_07884_b200.operator import apply_system, plan_operator

    W = workloads.make("c0")
    plan = plan_operator(W.kernel())
    x = np.random.default_rng(1).normal(size=W.grid.n_unknowns) + 0.5j
    y_host = apply_system(plan, W.m, x)
    y_dev = apply_system(plan, torch.from_numpy(W.m.reshape(-1).copy()).cuda(), torch.from_numpy(x).cuda())
    assert isinstance(y_host, np.ndarray)
    assert np.array_equal(y_host, y_dev.cpu().numpy())


def test_to_host_pinned_pool_lifetime():
    import torch

    from paper_1903_07884_b200 import _native as nv

    d = torch.arange(300_000, dtype=torch.float64, device="cuda").to(torch.complex128) * (1 + 2j)
    a = nv.to_host(d)
    b = nv.to_host(d * 2)          # a still alive: a second block
    assert a.ctypes.data != b.ctypes.data
    assert np.array_equal(a, d.cpu().numpy()) and np.array_equal(b, (d * 2).cpu().numpy())
    pa = a.ctypes.data
    del a
    c = nv.to_host(d * 3)          # a's block is recycled, b untouched
    assert c.ctypes.data == pa
    assert np.array_equal(b, (d * 2).cpu().numpy()) and np.array_equal(c, (d * 3).cpu().numpy())
    v = nv.to_host(d.reshape(600, 500).real.contiguous())
    assert v.shape == (600, 500) and v.dtype == np.float64
