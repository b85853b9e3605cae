"""GPU parity: FFT engine vs scipy, operator vs the oracle / dense matrix / golden."""

import numpy as np
import pytest
import scipy.fft

import voxvie_oracle as O
from conftest import random_field, relerr

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch

    assert torch.cuda.is_available()
    return torch


def _fft_lines(torch, a, axis, inverse, n_out=None, n=None):
    """Run vx_fft_lines over one axis of a C-contiguous complex array."""
    from paper_1903_07884_b200 import _native as nv

    a = np.ascontiguousarray(a, np.complex128)
    n = a.shape[axis] if n is None else n
    n_out = n if n_out is None else n_out
    shp_out = list(a.shape)
    shp_out[axis] = n_out
    outer = int(np.prod(a.shape[:axis]))
    inner = int(np.prod(a.shape[axis + 1:]))
    x = nv.device_c128(a)
    y = nv.empty_c128(tuple(shp_out))
    nin = a.shape[axis]
    nv.call("vx_fft_lines", n, outer * inner, inner, x.data_ptr(), nin * inner, 1, inner, nin,
            y.data_ptr(), n_out * inner, 1, inner, n_out, int(inverse),
            (1.0 / n) if inverse else 1.0, nv.stream_ptr())
    return y.cpu().numpy()


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 7, 8, 11, 13, 16, 17, 24, 31, 45, 64, 97, 200, 367,
                               400, 734, 735, 1500, 2500, 3000, 5000, 10000])
def test_fft_contiguous_lengths(torch, rng, n):
    lines = max(1, min(64, 20000 // n))
    a = random_field(rng, lines * n).reshape(lines, n)
    assert relerr(_fft_lines(torch, a, 1, False), scipy.fft.fft(a, axis=1)) < 1e-13
    assert relerr(_fft_lines(torch, a, 1, True), scipy.fft.ifft(a, axis=1)) < 1e-13


@pytest.mark.parametrize("n", [127, 131, 199, 211, 283, 293, 367, 389, 397, 509, 521, 2 * 211])
def test_fft_register_bluestein_lengths(torch, rng, n):
    """Non-smooth lengths on contiguous lines: the three-pass register Bluestein
    (convolution length R^2 >= 2n-1, R = 16 / 20 / 24 / 28 / 32 -- both edges of
    every bucket) and, above 2n-1 = 1024, the shared-memory stage engine; with
    zero padding in and a cropped output."""
    lines = 37
    a = random_field(rng, lines * n).reshape(lines, n)
    assert relerr(_fft_lines(torch, a, 1, False), scipy.fft.fft(a, axis=1)) < 1e-13
    assert relerr(_fft_lines(torch, a, 1, True), scipy.fft.ifft(a, axis=1)) < 1e-13
    short = a[:, : n // 2 + 1]
    assert relerr(_fft_lines(torch, short, 1, False, n=n), scipy.fft.fft(short, n, axis=1)) < 1e-13
    assert relerr(_fft_lines(torch, a, 1, True, n=n, n_out=n // 3), scipy.fft.ifft(a, axis=1)[:, : n // 3]) < 1e-13


@pytest.mark.parametrize("shape,axis", [((3, 10, 7), 1), ((2, 44, 33), 1), ((5, 19, 16), 1),
                                        ((6, 16, 9), 0), ((4, 800, 3), 1), ((3, 11, 2, 5), 1)])
def test_fft_strided(torch, rng, shape, axis):
    a = random_field(rng, int(np.prod(shape))).reshape(shape)
    assert relerr(_fft_lines(torch, a, axis, False), scipy.fft.fft(a, axis=axis)) < 1e-13
    assert relerr(_fft_lines(torch, a, axis, True), scipy.fft.ifft(a, axis=axis)) < 1e-13


def test_fft_zero_pad_and_crop(torch, rng):
    a = random_field(rng, 6 * 7).reshape(6, 7)
    got = _fft_lines(torch, a, 1, False, n=16)
    assert relerr(got, scipy.fft.fft(a, 16, axis=1)) < 1e-14
    got = _fft_lines(torch, a, 1, True, n=7, n_out=3)
    assert relerr(got, scipy.fft.ifft(a, axis=1)[:, :3]) < 1e-14


@pytest.mark.parametrize("n_in,n,n_out", [(5000, 10000, 10000), (200, 400, 400), (1500, 3000, 3000),
                                          (367, 735, 735)])
def test_fft_long_pad_and_crop(torch, rng, n_in, n, n_out):
    # the operator's x passes: zero-pad n_in -> n forward, crop n -> n_in inverse
    a = random_field(rng, 7 * n_in).reshape(7, n_in)
    fw = _fft_lines(torch, a, 1, False, n=n)
    assert relerr(fw, scipy.fft.fft(a, n, axis=1)) < 1e-13
    got = _fft_lines(torch, fw, 1, True, n=n, n_out=n_in)
    assert relerr(got, scipy.fft.ifft(fw, axis=1)[:, :n_in]) < 1e-13
    assert relerr(got, a) < 1e-13


OP_TAGS = ["small", "cube", "one", "odd", "prime", "long"]


@pytest.mark.parametrize("tag", OP_TAGS)
def test_operator_matches_golden(golden_small, tag):
    from paper_1903_07884_b200.grid import VoxelGrid
    from paper_1903_07884_b200.kernel import ToeplitzKernel
    from paper_1903_07884_b200.operator import apply_n, apply_system, plan_operator

    g = golden_small
    dims = tuple(int(v) for v in g[f"op_{tag}_dims"])
    kern = ToeplitzKernel(VoxelGrid(*dims, 0.05), 2 * np.pi, g[f"op_{tag}_tensors"])
    plan = plan_operator(kern)
    x = g[f"op_{tag}_x"]
    assert relerr(apply_n(plan, x), g[f"op_{tag}_n"]) < 1e-12
    assert relerr(apply_system(plan, g[f"op_{tag}_m"], x), g[f"op_{tag}_a"]) < 1e-12


def test_operator_columns_vs_dense(golden_small):
    """test_operator.py:48-59 -- every column of A against the dense oracle."""
    from paper_1903_07884_b200.grid import VoxelGrid
    from paper_1903_07884_b200.kernel import ToeplitzKernel
    from paper_1903_07884_b200.operator import apply_system, plan_operator

    g = golden_small
    dims = (4, 3, 2)
    t = g["op_small_tensors"]
    m = g["op_small_m"]
    plan = plan_operator(ToeplitzKernel(VoxelGrid(*dims, 0.05), 2 * np.pi, t))
    a = O.dense_operator(t, dims, m)
    scale = np.abs(a).max()
    for col in range(a.shape[0]):
        e = np.zeros(a.shape[0], complex)
        e[col] = 1.0
        assert np.abs(apply_system(plan, m, e) - a[:, col]).max() / scale < 1e-12


def test_operator_padded_shape_and_plan(golden_small):
    from paper_1903_07884_b200.grid import VoxelGrid
    from paper_1903_07884_b200.kernel import ToeplitzKernel
    from paper_1903_07884_b200.operator import plan_operator

    g = golden_small
    kern = ToeplitzKernel(VoxelGrid(4, 3, 2, 0.05), 2 * np.pi, g["op_small_tensors"])
    p1, p2 = plan_operator(kern), plan_operator(kern)
    assert p1.padded_shape == (4, 6, 8)
    assert np.array_equal(p1.spectra, p2.spectra)
    ref = O.plan_spectra(g["op_small_tensors"], (4, 3, 2))
    assert relerr(p1.spectra, ref) < 1e-13


def test_operator_torch_in_torch_out(torch, rng):
    from paper_1903_07884_b200 import workloads
    from paper_1903_07884_b200.operator import apply_system, plan_operator

    W = workloads.small(40, 6, 3)
    plan = plan_operator(W.kernel())
    x = random_field(rng, W.grid.n_unknowns)
    xd = torch.from_numpy(x).cuda()
    y = apply_system(plan, W.m, xd)
    assert isinstance(y, torch.Tensor) and y.is_cuda
    spec = O.plan_spectra(W.kernel().tensors, W.grid.dims)
    assert relerr(y.cpu().numpy(), O.apply_system(spec, W.grid.dims, W.m, x)) < 1e-12
    assert np.array_equal(xd.cpu().numpy(), x)  # input untouched


@pytest.mark.parametrize("dims", [(200, 10, 5), (367, 40, 8), (64, 22, 11)])
def test_operator_vs_oracle_waveguides(rng, dims):
    from paper_1903_07884_b200 import workloads
    from paper_1903_07884_b200.operator import apply_system, plan_operator

    W = workloads.small(*dims, delta=0.03e-6)
    plan = plan_operator(W.kernel())
    x = random_field(rng, W.grid.n_unknowns)
    spec = O.plan_spectra(W.kernel().tensors, W.grid.dims)
    assert relerr(apply_system(plan, W.m, x), O.apply_system(spec, W.grid.dims, W.m, x)) < 1e-12


def test_operator_linearity_and_shape_error(rng, golden_small):
    from paper_1903_07884_b200.grid import VoxelGrid
    from paper_1903_07884_b200.kernel import ToeplitzKernel
    from paper_1903_07884_b200.operator import apply_n, plan_operator

    g = golden_small
    plan = plan_operator(ToeplitzKernel(VoxelGrid(4, 3, 2, 0.05), 2 * np.pi, g["op_small_tensors"]))
    x1, x2 = random_field(rng, 72), random_field(rng, 72)
    a, b = 1.3 - 0.4j, -0.7 + 2.1j
    lhs = apply_n(plan, a * x1 + b * x2)
    rhs = a * apply_n(plan, x1) + b * apply_n(plan, x2)
    assert np.abs(lhs - rhs).max() / np.abs(lhs).max() < 1e-13
    assert np.all(apply_n(plan, np.zeros(72, complex)) == 0)
    with pytest.raises(ValueError):
        apply_n(plan, np.zeros(7, complex))


def test_operator_air_identity_and_concurrency(rng, golden_small):
    from concurrent.futures import ThreadPoolExecutor

    from paper_1903_07884_b200.grid import VoxelGrid
    from paper_1903_07884_b200.kernel import ToeplitzKernel
    from paper_1903_07884_b200.operator import apply_system, plan_operator

    g = golden_small
    plan = plan_operator(ToeplitzKernel(VoxelGrid(4, 3, 2, 0.05), 2 * np.pi, g["op_small_tensors"]))
    x = random_field(rng, 72)
    assert np.array_equal(apply_system(plan, np.zeros((2, 3, 4)), x), x)
    m = g["op_small_m"]
    serial = apply_system(plan, m, x)
    with ThreadPoolExecutor(max_workers=4) as pool:
        res = list(pool.map(lambda _: apply_system(plan, m, x), range(8)))
    for r in res:
        assert np.array_equal(r, serial)


def test_compact_spectra_symmetric_kernel(rng, golden_small):
    """Parity-symmetric kernels use the half-octant spectra; the result must not
    change; asymmetric kernels (wrapped, reference circulant.py:659-669) keep
    the full spectra."""
    from paper_1903_07884_b200 import workloads
    from paper_1903_07884_b200.circulant import wrap_circulant_x
    from paper_1903_07884_b200.operator import apply_system, plan_operator

    W = workloads.small(37, 7, 4, delta=0.03e-6)
    kern = W.kernel()
    pc = plan_operator(kern)
    pf = plan_operator(kern, compact=False)
    assert pc.compact and not pf.compact
    assert pc.storage_bytes() < pf.storage_bytes() / 4
    assert pc.padded_shape == pf.padded_shape
    assert relerr(pc.spectra, pf.spectra) < 1e-13
    x = random_field(rng, W.grid.n_unknowns)
    assert relerr(apply_system(pc, W.m, x), apply_system(pf, W.m, x)) < 1e-13
    spec = O.plan_spectra(kern.tensors, W.grid.dims)
    assert relerr(apply_system(pc, W.m, x), O.apply_system(spec, W.grid.dims, W.m, x)) < 1e-12
    wrapped = wrap_circulant_x(kern)
    assert not plan_operator(wrapped).compact


@pytest.mark.parametrize("ny", list(range(1, 30)))
def test_operator_register_fft_lengths(rng, ny):
    """Every register-FFT length (padded y = 2..56, and pz <= 8 for the
    register z-multiply) against the oracle and against the shared-memory
    engine (vx_op_reg_fft(0))."""
    from paper_1903_07884_b200 import _native as nv
    from paper_1903_07884_b200 import workloads
    from paper_1903_07884_b200.operator import apply_system, plan_operator

    nz = 1 + ny % 4
    W = workloads.small(6, ny, nz, delta=0.03e-6)
    plan = plan_operator(W.kernel())
    x = random_field(rng, W.grid.n_unknowns)
    spec = O.plan_spectra(W.kernel().tensors, W.grid.dims)
    ref = O.apply_system(spec, W.grid.dims, W.m, x)
    y_reg = apply_system(plan, W.m, x)
    nv.call("vx_op_reg_fft", 0)
    try:
        y_smem = apply_system(plan, W.m, x)
    finally:
        nv.call("vx_op_reg_fft", 1)
    assert relerr(y_reg, ref) < 1e-12
    assert relerr(y_reg, y_smem) < 1e-13


@pytest.mark.parametrize("ny,py", [(32, 64), (36, 72), (40, 80), (48, 96), (50, 100), (56, 112), (60, 120), (64, 128),
                                   (400, 800)])
def test_operator_two_pass_column_lengths(rng, monkeypatch, ny, py):
    """The two-pass register column transforms (cols2_kernel: padded y of 64 .. 128 and c4's 800)
    against the oracle and against the generic shared-memory engine (VX_COLS2=0 is read once per
    process, so the comparison run uses vx_op_reg_fft(0), which disables both register paths)."""
    from paper_1903_07884_b200 import _native as nv
    from paper_1903_07884_b200 import workloads
    from paper_1903_07884_b200.operator import apply_system, plan_operator

    W = workloads.small(5, ny, 2, delta=0.03e-6)
    plan = plan_operator(W.kernel())
    assert plan.padded_shape[1] == py
    x = random_field(rng, W.grid.n_unknowns)
    spec = O.plan_spectra(W.kernel().tensors, W.grid.dims)
    ref = O.apply_system(spec, W.grid.dims, W.m, x)
    y2 = apply_system(plan, W.m, x)
    nv.call("vx_op_reg_fft", 0)
    try:
        y_smem = apply_system(plan, W.m, x)
    finally:
        nv.call("vx_op_reg_fft", 1)
    assert relerr(y2, ref) < 1e-12
    assert relerr(y2, y_smem) < 1e-13
