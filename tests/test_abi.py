"""CPU-side checks of the C-ABI boundary: the in-tree library loads and exports
every function include/voxvie_b200.h declares; status codes map to the
reference's exception types.  No compute call is made (no GPU needed)."""

import ctypes

import pytest

from paper_1903_07884_b200 import _native as nv
from paper_1903_07884_b200.errors import NativeError, PreconditionerBuildError


def test_header_declares_the_hot_path():
    syms = nv.header_symbols()
    for s in ["vx_op_plan", "vx_op_apply", "vx_chan_x_spectra", "vx_lu1_build", "vx_prec1_apply",
              "vx_chan_xy_spectra", "vx_lu2_build", "vx_prec2_apply", "vx_arnoldi_step",
              "vx_basis_combine", "vx_box_gather", "vx_box_scatter", "vx_fft_lines"]:
        assert s in syms


def test_library_exports_every_header_symbol():
    if not nv.LIB_PATH.exists():
        pytest.skip("library not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(str(nv.LIB_PATH))
    missing = [s for s in nv.header_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(nv._SIGS) >= set(nv.header_symbols())


def test_host_only_queries():
    if not nv.LIB_PATH.exists():
        pytest.skip("library not built")
    assert nv.query("vx_version") >= 1
    assert nv.query("vx_fft_is_smooth", 10000) == 1
    assert nv.query("vx_fft_is_smooth", 734) == 0
    assert nv.query("vx_fft_good_length", 733) == 735
    for n, T in [(24, 24), (18, 18), (150, 32), (726, 32), (825, 32), (924, 32)]:
        assert nv.query("vx_lu_tile", n) == T
        assert nv.query("vx_lu_block_elems", n) == (-(-n // T) * T) ** 2


def test_status_mapping():
    if not nv.LIB_PATH.exists():
        pytest.skip("library not built")
    nv.check(nv.VX_OK)
    with pytest.raises(ValueError):
        nv.check(nv.VX_EINVAL)
    with pytest.raises(PreconditionerBuildError):
        nv.check(nv.VX_ESINGULAR)
    with pytest.raises(NativeError):
        nv.check(nv.VX_ECUDA)


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1903_07884_b200 import VoxelGrid, assemble_kernel, plan_operator

    with pytest.raises(NativeError):
        plan_operator(assemble_kernel(VoxelGrid(4, 3, 2, 0.05), 6.28))


def test_symmetric_layout_stride_formula():
    """vx_lu_sym_stride (host function, no GPU): per block of dimension d the symmetric layouts
    (factors and inverses, csrc/lu_sym.cuh) hold, per tile row i of t_i rows, i off-diagonal
    t_i x 32 tiles and the diagonal trapezoid of 8-row blocks (row r: 8 (r // 8) + 8 entries)."""
    import numpy as np

    from paper_1903_07884_b200 import _native as nv

    def trap(t):
        return sum(8 * (r // 8) + 8 for r in range(t))

    def size(d):
        nt = (d + 31) // 32
        tot = 0
        for i in range(nt):
            ti = min(32, d - 32 * i)
            tot += 32 * ti * i + trap(ti)
        return tot

    nv.load()
    for dims in ([33], [36, 36, 36, 36], [187, 187, 176, 176], [413, 412], [462, 462], [1024]):
        a = np.ascontiguousarray(dims, np.int32)
        assert int(nv.query("vx_lu_sym_stride", len(dims), a.ctypes.data)) == sum(size(d) for d in dims)
    # the lower triangle plus the trapezoid padding: ~0.52 of the LU bytes at c1's sector sizes
    assert size(187) / 187 ** 2 < 0.53
