"""ctypes binding of the C-ABI library ``libvoxvie_b200.so`` (include/voxvie_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).
There is no CPU fallback: if the library or a CUDA device is missing, every
hot-path call raises ``NativeError``.  PyTorch is used only for device memory
and the current CUDA stream.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

from .errors import NativeError, PreconditionerBuildError

LIB_PATH = Path(__file__).resolve().parent / "libvoxvie_b200.so"
HEADER = Path(__file__).resolve().parents[1] / "include" / "voxvie_b200.h"

VX_OK, VX_EINVAL, VX_ESINGULAR, VX_ECAP, VX_ECUDA, VX_ENCCL = range(6)

_lib = None
_lock = threading.Lock()

c_int, c_long, c_double, c_void_p = C.c_int, C.c_long, C.c_double, C.c_void_p
c_size_t = C.c_size_t


class c128(C.Structure):
    _fields_ = [("re", C.c_double), ("im", C.c_double)]


def cval(z) -> c128:
    z = complex(z)
    return c128(z.real, z.imag)


P = c_void_p  # every device pointer crosses the ABI as void*
_SIGS = {
    "vx_last_error": (C.c_char_p, []),
    "vx_version": (c_int, []),
    "vx_fft_good_length": (c_int, [c_int]),
    "vx_fft_is_smooth": (c_int, [c_int]),
    "vx_fft_lines": (c_int, [c_int, c_int, c_int, P, c_long, c_long, c_long, c_int,
                             P, c_long, c_long, c_long, c_int, c_int, c_double, P]),
    "vx_op_plan": (c_int, [c_int] * 6 + [P, c_long, c_long, c_long, c_long, P, P]),
    "vx_op_work_elems": (c_long, [c_int] * 6),
    "vx_op_padded_length": (c_int, [c_int]),
    "vx_op_padded_length_z": (c_int, [c_int]),
    "vx_op_apply": (c_int, [c_int] * 6 + [P, c_int, P, P, P, P, P]),
    "vx_gen_asymmetry": (c_int, [c_int] * 3 + [P, c_long, c_long, c_long, c_long, P, P]),
    "vx_op_compact_elems": (c_long, [c_int] * 3),
    "vx_op_compact": (c_int, [c_int] * 3 + [P, P, P]),
    "vx_chan_x_spectra": (c_int, [c_int] * 3 + [P, c_long, c_long, c_long, c_long, P, P]),
    "vx_proxy": (c_int, [c_int] * 3 + [P, c128, P, P]),
    "vx_lu_tile": (c_int, [c_int]),
    "vx_lu_block_elems": (c_long, [c_int]),
    "vx_lu1_build": (c_int, [c_int] * 3 + [P, P, P, c_int, P, P, P, P, P]),
    "vx_prec1_work_elems": (c_long, [c_int] * 4),
    "vx_prec1_apply": (c_int, [c_int] * 4 + [P, P, P, c_int, c_int, c_int, P, P, P, P, P]),
    "vx_chan_xy_work_elems": (c_long, [c_int] * 3),
    "vx_chan_xy_spectra": (c_int, [c_int] * 3 + [P, c_long, c_long, c_long, c_long, P, P, P]),
    "vx_lu2_build": (c_int, [c_int] * 3 + [P, P, P, c_int, P, P, P, P, P]),
    "vx_prec2_work_elems": (c_long, [c_int] * 4),
    "vx_prec2_apply": (c_int, [c_int] * 4 + [P, P, P, c_int, c_int, P, P, P, P, P]),
    "vx_box_gather": (c_int, [c_int] * 10 + [P, P, P]),
    "vx_box_scatter": (c_int, [c_int] * 10 + [P, P, P]),
    "vx_arnoldi_part_elems": (c_long, [c_long, c_int]),
    "vx_arnoldi_step": (c_int, [c_long, c_int, P, c_long, P, P, P, P, P, P]),
    "vx_basis_combine_ptrs": (c_int, [c_long, c_int, P, P, P, P]),
    "vx_basis_combine": (c_int, [c_long, c_int, P, c_long, P, P, P]),
    "vx_axpby": (c_int, [c_long, c128, P, c128, P, P, P]),
    "vx_norm2": (c_int, [c_long, P, P, P, P]),
    "vx_op_x_forward": (c_int, [c_int, c_int, c_int, P, P, P]),
    "vx_op_yz_work_elems": (c_long, [c_int] * 4),
    "vx_op_yz": (c_int, [c_int] * 6 + [P, P, P, P]),
    "vx_op_x_inverse": (c_int, [c_int] * 5 + [c_long, P, P, P, P, P]),
    "vx_gather_cols": (c_int, [c_long, P, c_long, c_int, P, P, c_long, P, P]),
    "vx_scatter_cols": (c_int, [c_long, P, c_int, P, P, c_long, P, c_long, P]),
    "vx_rep_inverse_elems": (c_long, [c_int]),
    "vx_rep_inverse": (c_int, [c_int, P, P, P, P]),
    "vx_prec1_reduced_work_elems": (c_long, [c_int] * 5),
    "vx_prec1_apply_reduced": (c_int, [c_int] * 4 + [P, P, P, c_int, c_int, P, P, P, c_int, P, P, P, P]),
    "vx_lu1_build_sec": (c_int, [c_int] * 3 + [P, P, P, c_int, c_int, c_int, P, P, P, P, P, P, P, P, P]),
    "vx_prec1_sec_work_elems": (c_long, [c_int] * 6),
    "vx_prec1_apply_sec": (c_int, [c_int] * 4 + [P, P, P, c_int, c_int, c_int, P, c_int, c_int, c_int, P, P, P, P,
                                                  P, P, P, P]),
    "vx_prec1_apply_sec_rag": (c_int, [c_int] * 4 + [P, P, P, c_int, c_int, c_int, P, c_int, c_int, P, c_int,
                                                      P, P, P, P, P, P, P, P]),
    "vx_prec1_apply_rag": (c_int, [c_int] * 4 + [P, P, P, c_int, c_int, c_int, P, P, P, P, P]),
    "vx_lu_rag_stride": (c_long, [c_int, P]),
    "vx_solve_classic": (c_int, []),
    "vx_lu_repack": (c_int, [c_int, c_int, c_int, P, P, P, P]),
    "vx_lu_unpack": (c_int, [c_int, c_int, c_int, P, P, P, P]),
    "vx_rep_variant": (c_int, [c_int]),
    "vx_op_reg_fft": (c_int, [c_int]),
    "vx_prec1_solve": (c_int, [c_int, c_int, P, P, P, c_int, c_int, c_int, P, P, c_long, c_long, P]),
    "vx_cgs_dots": (c_int, [c_long, c_int, P, c_long, P, P, P, P]),
    "vx_cgs_update": (c_int, [c_long, c_int, P, c_long, P, P, P, P, P]),
    "vx_launch_count": (c_long, []),
    "vx_solve_variant": (c_int, [c_int]),
    "vx_lu_variant": (c_int, [c_int]),
    "vx_timing_enable": (c_int, [c_int]),
    "vx_timing_read": (c_int, [C.c_char_p, C.POINTER(C.c_double), C.POINTER(C.c_long)]),
}


def header_symbols() -> list[str]:
    """Function names declared in include/voxvie_b200.h."""
    import re

    txt = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\*?\s+\*?(vx_[a-z_0-9]+)\s*\(", txt, re.M)))


def load(path: Path | None = None):
    """Load (once) and return the ctypes library; raises NativeError if absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = Path(path or os.environ.get("VOXVIE_B200_LIB", LIB_PATH))
        if not p.exists():
            raise NativeError(
                f"CUDA library {p} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = C.CDLL(str(p))
        for name, (res, args) in _SIGS.items():
            f = getattr(lib, name, None)
            if f is None:
                continue  # reported by call(); tests check every header symbol is exported
            f.restype = res
            f.argtypes = args
        _lib = lib
        return lib


def check(status: int, what: str = ""):
    if status == VX_OK:
        return
    msg = load().vx_last_error().decode(errors="replace")
    if status == VX_EINVAL:
        raise ValueError(msg or what)
    if status in (VX_ESINGULAR, VX_ECAP):
        raise PreconditionerBuildError(msg or what)
    raise NativeError(f"{what}: {msg}")


def _fn(name: str):
    f = getattr(load(), name, None)
    if f is None:
        raise NativeError(f"{LIB_PATH.name} does not export {name}")
    return f


def call(name: str, *args):
    """Invoke a status-returning C-ABI function and map failures to exceptions."""
    check(_fn(name)(*args), name)


def query(name: str, *args):
    return _fn(name)(*args)


# --------------------------------------------------------------- torch glue
def torch():
    import torch as _t

    return _t


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise NativeError("no CUDA device: the voxvie_b200 hot path has no CPU fallback")
    load()
    return t


def stream_ptr():
    t = torch()
    return t.cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def device_c128(a, device=None):
    """Host array-like / tensor -> contiguous complex128 CUDA tensor."""
    t = require_cuda()
    if isinstance(a, t.Tensor):
        if not a.is_cuda:
            a = a.to("cuda" if device is None else device, non_blocking=False)
        return a.to(t.complex128).contiguous()
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.complex128))
    if not arr.flags.writeable:
        arr = arr.copy()
    host = t.from_numpy(arr)
    return host.to("cuda" if device is None else device)


def empty_c128(n, device=None):
    t = require_cuda()
    shape = (n,) if isinstance(n, int) else tuple(n)
    return t.empty(shape, dtype=t.complex128, device="cuda" if device is None else device)


def is_tensor(a) -> bool:
    try:
        import torch as _t
    except ImportError:  # pragma: no cover
        return False
    return isinstance(a, _t.Tensor)


def timing_enable(on: bool):
    query("vx_timing_enable", 1 if on else 0)


def timing_read(span: str):
    """(total_ms, count) of the named event span since the last read."""
    ms, cnt = C.c_double(0.0), C.c_long(0)
    call("vx_timing_read", span.encode(), C.byref(ms), C.byref(cnt))
    return ms.value, cnt.value


def launch_count() -> int:
    return int(query("vx_launch_count"))


def to_host(t):
    """Device tensor -> numpy through pinned memory (pageable D2H of large
    vectors runs at ~2 GB/s; pinned at link speed)."""
    if t.numel() * t.element_size() < (1 << 20) or not t.is_cuda:
        return t.cpu().numpy()
    tt = torch()
    h = tt.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t, non_blocking=True)
    tt.cuda.current_stream().synchronize()
    return h.numpy()
