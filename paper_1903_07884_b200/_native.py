"""ctypes binding of the C-ABI library ``libvoxvie_b200.so`` (include/voxvie_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).
There is no CPU fallback: if the library or a CUDA device is missing, every
hot-path call raises ``NativeError``.  PyTorch is used only for device memory
and the current CUDA stream.
"""

from __future__ import annotations

import contextlib
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
    "vx_lu_small_invert": (c_int, [c_int, c_int, P, P, P, P]),
    "vx_prec2_apply_inv": (c_int, [c_int] * 4 + [P, P, c_int, P, P, P, P, P]),
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
    "vx_op_yz_compact": (c_int, [c_int] * 6 + [P, P, P, P]),
    "vx_spec_compact_yz_elems": (c_long, [c_int, c_int, c_int]),
    "vx_spec_compact_yz": (c_int, [c_int, c_int, c_int, P, P, P]),
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
    "vx_prec1_solve_sec_rag": (c_int, [c_int, c_int, c_long, P, P, P, c_int, c_int, c_int, P, c_int, c_int, P,
                                       c_int, P, P, P, P, P, P, P]),
    "vx_prec1_sec_reduced_work_elems": (c_long, [c_int] * 7),
    "vx_prec1_apply_sec_reduced": (c_int, [c_int] * 4 + [P, P, P, c_int, c_int, P, c_int, c_int, P, c_int, P, P, P,
                                                      P, P, P, c_int, P, P, P, P]),
    "vx_lu1_build_opts": (c_int, [c_int] * 3 + [P, P, P, c_int, c_int, c_int, P, P, P, P, P, P, P, P, c_int, P]),
    "vx_lu_sym_stride": (c_long, [c_int, P]),
    "vx_lu_sym_pack": (c_int, [c_int, c_int, c_int, P, P, P, P, P, P, P]),
    "vx_lu_sym_unpack": (c_int, [c_int, c_int, c_int, P, P, P, P, P, P]),
    "vx_prec1_apply_sym": (c_int, [c_int] * 3 + [P, P, P, P, c_int, c_int, P, c_int, c_int, P, c_int, P, P, P, P,
                                                  P, P, c_int, P, P, P, P]),
    "vx_lu_sym_invert": (c_int, [c_int, c_int, c_int, P, P, P, P, P, P, P]),
    "vx_prec1_apply_syminv": (c_int, [c_int] * 3 + [P, P, P, c_int, c_int, P, c_int, c_int, P, c_int, P, P, P, P,
                                                     P, P, c_int, P, P, P, P]),
    "vx_prec1_solve_syminv": (c_int, [c_int, c_int, c_long, P, P, P, c_int, c_int, P, c_int, c_int, P, c_int, P, P,
                                       P, P, P, P, P]),
    "vx_solve_classic": (c_int, []),
    "vx_lu_repack": (c_int, [c_int, c_int, c_int, P, P, P, P]),
    "vx_lu_unpack": (c_int, [c_int, c_int, c_int, P, P, P, P]),
    "vx_rep_variant": (c_int, [c_int]),
    "vx_op_reg_fft": (c_int, [c_int]),
    "vx_prec1_solve": (c_int, [c_int, c_int, P, P, P, c_int, c_int, c_int, P, P, c_long, c_long, P]),
    "vx_small_inv_apply": (c_int, [c_int, c_int, P, P, c_int, P, P, c_long, c_long, P]),
    "vx_cgs_dots": (c_int, [c_long, c_int, P, c_long, P, P, P, P]),
    "vx_cgs_update": (c_int, [c_long, c_int, P, c_long, P, P, P, P, P]),
    "vx_cgs_dots_cond": (c_int, [c_long, c_int, P, c_long, P, P, P, P, P]),
    "vx_cgs_update_cond": (c_int, [c_long, c_int, P, c_long, P, P, P, P, P, P]),
    "vx_dgks_ctl": (c_int, [P, P, P, P]),
    "vx_dgks_finish": (c_int, [c_int, P, P, P, P, P, P]),
    "vx_scale_dev": (c_int, [c_long, P, P, P, P]),
    "vx_launch_count": (c_long, []),
    "vx_h2d_staged": (c_int, [P, P, c_size_t, P]),
    "vx_assemble_green": (c_int, [c_int] * 3 + [c_double] * 3 + [c128, P, P]),
    "vx_h2d_threads": (c_int, []),
    "vx_host_alloc": (c_int, [c_size_t, C.POINTER(C.c_void_p)]),
    "vx_host_free": (c_int, [P]),
    "vx_d2h_pinned": (c_int, [P, P, c_size_t, P]),
    "vx_d2h_pinned_async": (c_int, [P, P, c_size_t, P]),
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


H2D_STAGED_MIN = int(os.environ.get("VX_H2D_STAGED_MIN", 4 << 20))


_side_streams = {}


def _upload_stream(t):
    dev = t.cuda.current_device()
    s = _side_streams.get(dev)
    if s is None:
        s = _side_streams[dev] = t.cuda.Stream(device=dev)
    return s


def device_c128(a, device=None, side=False):
    """Host array-like / tensor -> contiguous complex128 CUDA tensor.

    ``side``: a large host array is copied on the library's upload stream, so
    the DMA overlaps work already queued on the current stream (an input that
    is first read LATER on the current stream, e.g. the medium map uploaded
    while the first preconditioner apply runs).  The tensor is allocated from
    the upload stream's pool and handed to the current stream with an event
    wait + ``record_stream`` (the caching allocator's cross-stream protocol)."""
    t = require_cuda()
    if isinstance(a, t.Tensor):
        if not a.is_cuda:
            a = a.to("cuda" if device is None else device, non_blocking=False)
        return a.to(t.complex128).contiguous()
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.complex128))
    if arr.nbytes >= H2D_STAGED_MIN and device is None:
        # large pageable upload: threaded copy through the library's pinned ring
        if side and os.environ.get("VX_H2D_SIDE", "1") != "0":
            up, cur = _upload_stream(t), t.cuda.current_stream()
            with t.cuda.stream(up):
                out = t.empty(arr.shape, dtype=t.complex128, device="cuda")
                call("vx_h2d_staged", out.data_ptr(), arr.ctypes.data, arr.nbytes, up.cuda_stream)
            cur.wait_stream(up)
            out.record_stream(cur)
            return out
        out = t.empty(arr.shape, dtype=t.complex128, device="cuda")
        call("vx_h2d_staged", out.data_ptr(), arr.ctypes.data, arr.nbytes, stream_ptr())
        return out
    if not arr.flags.writeable:
        arr = arr.copy()
    host = t.from_numpy(arr)
    return host.to("cuda" if device is None else device)


def empty_c128(n, device=None):
    t = require_cuda()
    shape = (n,) if isinstance(n, int) else tuple(n)
    return t.empty(shape, dtype=t.complex128, device="cuda" if device is None else device)


_scope = threading.local()


@contextlib.contextmanager
def solve_scope():
    """A solve in progress on this thread: host inputs that the caller passes
    unchanged to every operator call of the solve (the medium map m) may be
    uploaded once per scope instead of once per call.  Nested scopes share the
    outermost token."""
    outer = getattr(_scope, "token", None)
    if outer is None:
        _scope.token = object()
    try:
        yield
    finally:
        if outer is None:
            _scope.token = None


def scope_token():
    """The active solve scope's token on this thread (None outside a solve)."""
    return getattr(_scope, "token", None)


def fresh_output(f):
    """Mark a callable whose every result is a newly allocated buffer (the
    GMRES Z basis may then keep the result itself instead of a copy)."""
    f._vx_fresh_output = True
    return f


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


class _PinnedBlock:
    """One pooled pinned host block, exposed to numpy through the array
    interface; when the last numpy view dies the block returns to the pool."""

    __slots__ = ("ptr", "nbytes", "__weakref__")

    def __init__(self, ptr: int, nbytes: int):
        self.ptr = ptr
        self.nbytes = nbytes

    @property
    def __array_interface__(self):
        return {"shape": (self.nbytes,), "typestr": "|u1", "data": (self.ptr, False), "version": 3}

    def __del__(self):
        try:
            _pinned_release(self.ptr, self.nbytes)
        except Exception:  # pragma: no cover - interpreter shutdown
            pass


_pin_lock = threading.Lock()
_pin_free: dict[int, list[int]] = {}
_PIN_KEEP = 4            # free blocks kept per size


def _pinned_acquire(nbytes: int) -> _PinnedBlock:
    with _pin_lock:
        lst = _pin_free.get(nbytes)
        if lst:
            return _PinnedBlock(lst.pop(), nbytes)
    out = C.c_void_p()
    call("vx_host_alloc", nbytes, C.byref(out))
    return _PinnedBlock(out.value, nbytes)


def _pinned_release(ptr: int, nbytes: int):
    with _pin_lock:
        lst = _pin_free.setdefault(nbytes, [])
        if len(lst) < _PIN_KEEP:
            lst.append(ptr)
            return
    query("vx_host_free", ptr)


_copy_stream = None


class HostCopy:
    """A device -> host copy of a large result in flight on a side stream
    (to_host_begin); result() waits for it and returns the numpy array."""

    def __init__(self, t):
        global _copy_stream
        th = torch()
        self._arr = None
        self._t = None
        np_dtype = {th.complex128: np.complex128, th.float64: np.float64}.get(t.dtype)
        if t.numel() * t.element_size() < (1 << 20) or not t.is_cuda or np_dtype is None:
            self._t = t
            return
        t = t.contiguous()
        nbytes = t.numel() * t.element_size()
        if _copy_stream is None:
            _copy_stream = th.cuda.Stream()
        self._stream = _copy_stream
        self._stream.wait_stream(th.cuda.current_stream())   # t is final on the caller's stream
        self._keep = t
        blk = _pinned_acquire(nbytes)
        call("vx_d2h_pinned_async", blk.ptr, t.data_ptr(), nbytes, self._stream.cuda_stream)
        self._arr = np.asarray(blk).view(np_dtype).reshape(tuple(t.shape))

    def result(self):
        if self._arr is None:
            return to_host(self._t)
        self._stream.synchronize()
        self._keep = None
        return self._arr


def to_host_begin(t) -> HostCopy:
    """Start copying a device tensor to the host without waiting for it."""
    return HostCopy(t)


def to_host(t):
    """Device tensor -> numpy.  Large results land in a pooled pinned block
    (DMA at link speed, no page faults on a fresh allocation); the returned
    array owns its block until it is garbage collected."""
    if t.numel() * t.element_size() < (1 << 20) or not t.is_cuda:
        return t.cpu().numpy()
    t = t.contiguous()
    nbytes = t.numel() * t.element_size()
    blk = _pinned_acquire(nbytes)
    call("vx_d2h_pinned", blk.ptr, t.data_ptr(), nbytes, stream_ptr())
    raw = np.asarray(blk)
    np_dtype = {torch().complex128: np.complex128, torch().float64: np.float64,
                torch().complex64: np.complex64, torch().float32: np.float32}.get(t.dtype)
    if np_dtype is None:
        return t.cpu().numpy()
    return raw.view(np_dtype).reshape(tuple(t.shape))
