"""Drop-in ``voxvie.solver.gmres`` with a device-resident Krylov basis
(reference: pkg/src/voxvie/solver.py:21-174).

Right-preconditioned restarted GMRES with the reference's exact control flow:
x0 = 0, restart residual b - A x (extra matvec per restart), x += P^-1 u per
cycle, true residual after the solve, ``iterations`` = total Arnoldi steps,
residual history with ``iterations + 1`` entries starting at 1.0.

Per Arnoldi step the basis never leaves HBM: the orthogonalisation is one
C-ABI call (``vx_arnoldi_step``: classical Gram-Schmidt + the reference's DGKS
criterion decided on the device) and only the j+2 Hessenberg entries and
the norm come back to the host, where the complex Givens rotations run
exactly as in the reference (solver.py:78-105).

Callables: our GPU operators/preconditioners take and return CUDA tensors and
run device-resident.  Plain numpy callables (as in the reference tests) are
detected on first use and fed host copies -- a boundary adapter, the Arnoldi
work itself still runs on the GPU.  ``b`` as numpy -> ``x`` as numpy; ``b`` as
a CUDA tensor -> ``x`` as a CUDA tensor.
"""

from __future__ import annotations

import contextlib
import gc
import os
import threading
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as nv
from .errors import BreakdownError, SizeLimitError

SPECTRUM_GUARD = 3000


@dataclass
class SolveReport:
    """reference solver.py:21-42."""

    iterations: int
    residuals: list
    converged: bool
    solve_seconds: float = 0.0
    build_seconds: float = 0.0
    true_residual: float = float("nan")
    memory: dict = field(default_factory=dict)

    def to_dict(self) -> dict:
        return {
            "iterations": self.iterations,
            "converged": self.converged,
            "relative_residuals": list(self.residuals),
            "solve_seconds": self.solve_seconds,
            "build_seconds": self.build_seconds,
            "true_residual": self.true_residual,
            "memory": dict(self.memory),
        }


class _Callable:
    """Dual-mode adapter: CUDA tensor in/out when the callable supports it,
    host numpy copies otherwise (decided once, on the first call)."""

    def __init__(self, f, n):
        self.f = f
        self.n = n
        self.mode = None
        # our preconditioners / operators allocate a new output every call
        # (marked by _native.fresh_output); anything else may hand back a
        # buffer it reuses on the next call
        self.declared_fresh = bool(getattr(f, "_vx_fresh_output", False))

    @property
    def fresh(self) -> bool:
        """True when every result is a new buffer (host-mode copies always are)."""
        return self.mode == "host" or self.declared_fresh

    def __call__(self, v):
        if self.mode != "host":
            try:
                out = self.f(v)
            except Exception:
                if self.mode == "dev":
                    raise
                self.mode = "host"
            else:
                if nv.is_tensor(out) and out.is_cuda:
                    self.mode = "dev"
                    out = out.reshape(-1)
                    if out.dtype != v.dtype:
                        out = out.to(v.dtype)
                    return out
                if self.mode == "dev":
                    raise TypeError("callable returned a non-CUDA result after returning CUDA tensors")
                self.mode = "host"
                return nv.device_c128(np.asarray(out, dtype=np.complex128).reshape(-1))
        out = self.f(v.cpu().numpy())
        return nv.device_c128(np.asarray(out, dtype=np.complex128).reshape(-1))


class _Krylov:
    """Device workspace: basis V (grown on demand), Arnoldi scratch, pinned mirrors."""

    def __init__(self, n, m, keep_z=False):
        self.t = nv.require_cuda()
        self.n = n
        self.cap = 0
        self.maxrows = m + 1
        self.V = None
        self.Z = None      # copies of z_j for callables that may reuse their output buffer
        self.zcap = 0
        self.keep_z = keep_z
        self._grow(min(m + 1, 32))
        self.h = nv.empty_c128(m + 2)
        self.stats = self.t.zeros(4, dtype=self.t.float64, device="cuda")
        self.part = nv.empty_c128(int(nv.query("vx_arnoldi_part_elems", n, m + 2)))
        # double-buffered pinned mirrors of (h column, stats): iteration j
        # lands in slot j % 2, so the host can read step j while step j+1
        # (launched speculatively) writes the other slot
        self.h_host = [self.t.empty(m + 2, dtype=self.t.complex128, pin_memory=True) for _ in range(2)]
        self.s_host = [self.t.empty(4, dtype=self.t.float64, pin_memory=True) for _ in range(2)]
        self.ev = [self.t.cuda.Event() for _ in range(2)]
        self.nrm = self.t.zeros(1, dtype=self.t.float64, device="cuda")
        self.nrm_host = self.t.empty(1, dtype=self.t.float64, pin_memory=True)

    def _grow(self, rows):
        if rows <= self.cap:
            return
        V = nv.empty_c128((rows, self.n))
        if self.V is not None:
            V[: self.cap].copy_(self.V)
        self.V, self.cap = V, rows

    def row(self, i):
        """Make basis row i available (growing V geometrically up to m+1 rows)."""
        if i >= self.cap:
            self._grow(min(max(i + 1, 2 * self.cap), max(self.maxrows, i + 1)))
        return self.V[i]

    def zrow(self, i):
        """Row i of the Z basis (grown geometrically like V, allocated only
        when the preconditioner may reuse its output buffer)."""
        if i >= self.zcap:
            rows = min(max(i + 1, 2 * self.zcap, min(self.maxrows, 32)), max(self.maxrows, i + 1))
            Z = nv.empty_c128((rows, self.n))
            if self.Z is not None:
                Z[: self.zcap].copy_(self.Z)
            self.Z, self.zcap = Z, rows
        return self.Z[i]

    def norm(self, x) -> float:
        nv.call("vx_norm2", self.n, x.data_ptr(), self.nrm.data_ptr(), self.part.data_ptr(),
                nv.stream_ptr())
        self.nrm_host.copy_(self.nrm, non_blocking=True)
        self.t.cuda.current_stream().synchronize()
        return float(self.nrm_host[0])

    def axpby(self, a, x, b, y, out=None):
        out = nv.empty_c128(self.n) if out is None else out
        nv.call("vx_axpby", self.n, nv.cval(a), x.data_ptr(), nv.cval(b), nv.ptr(y), out.data_ptr(),
                nv.stream_ptr())
        return out


_WS_LOCK = threading.Lock()
_WS_CACHE: dict = {}


_KEEP_Z_CACHE: dict = {}


def _keep_z_fits(t, n, mmax) -> bool:
    """Whether a second basis Z = P^-1 V fits comfortably (a quarter of the free
    device memory).  Asked ONCE per (device, n, mmax): cudaMemGetInfo takes
    2-60 ms on a busy driver (tools/stall_probe.py traced every slow solve of
    the bench to this call), and the answer only changes with the shape."""
    key = (t.cuda.current_device(), n, mmax)
    fits = _KEEP_Z_CACHE.get(key)
    if fits is None:
        free, _ = t.cuda.mem_get_info()
        with _WS_LOCK:
            have = any(k[:3] == key and k[3] for k in _WS_CACHE)   # a cached workspace already holds Z
        fits = have or (mmax + 1) * n * 16 <= free // 4
        _KEEP_Z_CACHE[key] = fits
    return fits


def _workspace(n, m, keep_z):
    """A reusable Krylov workspace (bases of up to m+1 rows); one per shape,
    handed to one solve at a time, so repeated solves do not re-allocate
    gigabytes of basis every call."""
    key = (nv.require_cuda().cuda.current_device(), n, m, keep_z)
    with _WS_LOCK:
        K = _WS_CACHE.pop(key, None)
    return K if K is not None else _Krylov(n, m, keep_z=keep_z)


def _release(K):
    key = (K.t.cuda.current_device(), K.n, K.maxrows - 1, K.keep_z)
    with _WS_LOCK:
        _WS_CACHE.clear()  # keep at most one cached workspace
        _WS_CACHE[key] = K


def clear_workspace() -> None:
    """Drop the cached Krylov workspace (its device memory returns to torch)."""
    with _WS_LOCK:
        _WS_CACHE.clear()
    _KEEP_Z_CACHE.clear()


def _aliases(a, b) -> bool:
    sa, sb = a.data_ptr(), b.data_ptr()
    return sb <= sa < sb + b.numel() * b.element_size()


class GivensQR:
    """Host-side complex Givens QR of the Arnoldi Hessenberg matrix, exactly
    the reference's arithmetic (solver.py:78-110); shared by the single-GPU and
    the sharded GMRES."""

    def __init__(self, beta: float):
        self.g = [np.complex128(beta + 0.0j)]
        self.cs, self.sn, self.r_cols = [], [], []

    def add_column(self, h: np.ndarray, j: int, residuals: list, tol: float) -> None:
        cs, sn = self.cs, self.sn
        for i in range(j):
            hi = h[i]
            h[i] = np.conj(cs[i]) * hi + np.conj(sn[i]) * h[i + 1]
            h[i + 1] = -sn[i] * hi + cs[i] * h[i + 1]
        denom = np.hypot(abs(h[j]), abs(h[j + 1]))
        if denom == 0.0:
            raise BreakdownError(
                f"GMRES stalled at iteration {len(residuals)}: zero Hessenberg "
                f"column with relative residual {residuals[-1]:.3e} above tol {tol:.3e}")
        c, s = h[j] / denom, h[j + 1] / denom
        cs.append(c)
        sn.append(s)
        h[j] = np.conj(c) * h[j] + np.conj(s) * h[j + 1]
        self.r_cols.append(h[: j + 1].copy())
        self.g.append(-s * self.g[j])
        self.g[j] = np.conj(c) * self.g[j]

    def solve(self, j: int) -> np.ndarray:
        r_mat = np.zeros((j, j), dtype=np.complex128)
        for col, vals in enumerate(self.r_cols[:j]):
            r_mat[: col + 1, col] = vals
        return np.linalg.solve(r_mat, np.asarray(self.g[:j], dtype=np.complex128))


# debugging aid (tools/stall_probe.py): a list that receives, per Arnoldi step,
# (j, host seconds spent launching, host seconds waiting for the step's event)
TRACE = None


def _speculate(residuals, tol) -> bool:
    """Launch step j+1 before step j's residual is known, unless the
    geometric trend of the estimates says step j is likely to converge (the
    speculative step would then be wasted work)."""
    if os.environ.get("VX_SPECULATE", "1") == "0":
        return False
    if len(residuals) < 3:
        return True
    r1, r2 = residuals[-1], residuals[-2]
    rho = r1 / r2 if r2 > 0 else 1.0
    return r1 * min(rho, 1.0) > 2.0 * tol


def _gmres_cycle(K: _Krylov, op, r0, beta, bnorm, tol, m, residuals, P=None, A=None):
    """One Arnoldi/Givens cycle (reference solver.py:45-111).

    With ``K.keep_z`` the preconditioned vectors z_j = P^-1 v_j that the
    operator needs anyway are kept, and the cycle returns u = Z y = P^-1 V y
    (the reference's correction, solver.py:106-110 then 160-161) without the
    extra preconditioner apply per cycle.

    Steps are pipelined: step j+1 (operator, preconditioner, orthogonalisation
    -- all device-resident, v_{j+1} = w / h_{j+1,j} is formed on the device)
    is enqueued before the host reads step j's Hessenberg column, so the GPU
    never idles while the host runs the reference's Givens arithmetic.  If
    step j ends the cycle (convergence / breakdown), the speculative step's
    output is simply never used; _speculate() avoids it near convergence."""
    t = K.t
    zl = []  # z_j = P^-1 v_j, kept where the preconditioner wrote them (no copy)
    if K.keep_z:
        def op(v, j):
            z = P(v)
            if not z.is_contiguous() or z.numel() != K.n:
                z = z.reshape(-1).contiguous()
            if not P.fresh or _aliases(z, K.V):
                # the callable may hand the same buffer back next call (or
                # returned a view of its argument): keep a private copy, or
                # z_j would be overwritten before u = Z y is formed
                zr = K.zrow(j)
                zr.copy_(z)
                z = zr
            if len(zl) > j:
                zl[j] = z
            else:
                zl.append(z)
            return A(z)
    else:
        op_base = op

        def op(v, j):
            return op_base(v)
    K.row(0)
    K.axpby(1.0 / beta, r0, 0.0, None, out=K.V[0])

    def launch(j):
        w = op(K.V[j], j)
        K.row(j + 1)
        if _aliases(w, K.V) or not w.is_contiguous():
            w = K.axpby(1.0, w, 0.0, None)  # the op returned (a view of) its argument: copy
        nv.call("vx_arnoldi_step", K.n, j + 1, K.V.data_ptr(), K.n, w.data_ptr(), K.V[j + 1].data_ptr(),
                K.h.data_ptr(), K.stats.data_ptr(), K.part.data_ptr(), nv.stream_ptr())
        b = j % 2
        K.h_host[b][: j + 2].copy_(K.h[: j + 2], non_blocking=True)
        K.s_host[b].copy_(K.stats, non_blocking=True)
        K.ev[b].record()

    qr = GivensQR(beta)
    converged = lucky = False
    j = 0
    launched = 0
    trace = TRACE
    while j < m:
        if trace is not None:
            tr0 = time.perf_counter()
        if launched <= j:
            launch(j)
            launched = j + 1
        if launched == j + 1 and j + 1 < m and _speculate(residuals, tol):
            launch(j + 1)
            launched = j + 2
        b = j % 2
        if trace is not None:
            tr1 = time.perf_counter()
        K.ev[b].synchronize()
        if trace is not None:
            trace.append((j, tr1 - tr0, time.perf_counter() - tr1))
        h = K.h_host[b][: j + 2].numpy().copy()
        norm_before = float(K.s_host[b][0])
        K.reorth_passes += int(K.s_host[b][2] != 0.0)   # the DGKS second pass ran in this step
        lucky = h[j + 1].real <= 1e-14 * max(norm_before, 1e-300)
        qr.add_column(h, j, residuals, tol)
        j += 1
        est = abs(qr.g[j]) / bnorm
        residuals.append(float(est))
        if est <= tol or lucky:
            converged = est <= tol
            if lucky and not converged:
                raise BreakdownError(
                    f"Arnoldi breakdown at iteration {len(residuals) - 1} with "
                    f"relative residual {est:.3e} above tol {tol:.3e}")
            break
    y = qr.solve(j)
    yd = nv.device_c128(y)
    u = nv.empty_c128(K.n)
    if K.keep_z:
        ptrs = t.tensor([z.data_ptr() for z in zl[:j]] or [0], dtype=t.int64).to("cuda", non_blocking=True)
        nv.call("vx_basis_combine_ptrs", K.n, j, ptrs.data_ptr(), yd.data_ptr(), u.data_ptr(), nv.stream_ptr())
    else:
        nv.call("vx_basis_combine", K.n, j, K.V.data_ptr(), K.n, yd.data_ptr(), u.data_ptr(), nv.stream_ptr())
    return u, j, converged


def gmres(apply_a, b, *, apply_pinv=None, tol: float = 1e-4, maxit: int = 2000,
          restart: int | None = None):
    """Right-preconditioned (restarted) GMRES from x0 = 0 (reference solver.py:114-174).

    Python's cyclic garbage collector is paused for the duration of the solve
    (and restored afterwards): a full collection with torch loaded walks ~10^6
    objects (tens of ms), long enough to drain the one-iteration-deep device
    queue of the pipelined Arnoldi loop; the solve itself creates no cycles."""
    with gc_paused(), nv.solve_scope():
        return _gmres(apply_a, b, apply_pinv=apply_pinv, tol=tol, maxit=maxit, restart=restart)


@contextlib.contextmanager
def gc_paused():
    """Pause the cyclic garbage collector inside a solve, restoring its state."""
    gc_on = gc.isenabled()
    gc.disable()
    try:
        yield
    finally:
        if gc_on:
            gc.enable()


def _gmres(apply_a, b, *, apply_pinv=None, tol: float = 1e-4, maxit: int = 2000,
           restart: int | None = None):
    if not tol > 0:
        raise ValueError("tol must be positive")
    if maxit < 1:
        raise ValueError("maxit must be >= 1")
    t = nv.require_cuda()
    on_device = nv.is_tensor(b)
    t0 = time.perf_counter()
    bd = nv.device_c128(b.reshape(-1) if on_device else np.asarray(b, np.complex128).reshape(-1))
    n = bd.numel()
    mmax = maxit if restart is None else min(restart, maxit)
    # keep Z = P^-1 V when a preconditioner is given and a second basis fits
    # comfortably (a quarter of the free device memory)
    keep_z = False
    marks = [("start", t0)] if TRACE is not None else None
    if apply_pinv is not None and os.environ.get("VX_KEEP_Z", "1") != "0":
        keep_z = _keep_z_fits(t, n, mmax)
    if marks is not None:
        marks.append(("mem_get_info", time.perf_counter()))
    K = _workspace(n, mmax, keep_z)
    K.reorth_passes = 0
    bnorm = K.norm(bd)
    if marks is not None:
        marks.append(("workspace+norm", time.perf_counter()))

    def _out(xd):
        return xd if on_device else nv.to_host(xd)

    if bnorm == 0.0:
        x = t.zeros(n, dtype=t.complex128, device="cuda")
        t.cuda.current_stream().synchronize()
        _release(K)
        return _out(x), SolveReport(iterations=1, residuals=[1.0, 0.0], converged=True,
                                    solve_seconds=time.perf_counter() - t0, true_residual=0.0)
    A = _Callable(apply_a, n)
    P = _Callable(apply_pinv, n) if apply_pinv is not None else None
    op = A if P is None else (lambda v: A(P(v)))
    x = t.zeros(n, dtype=t.complex128, device="cuda")
    residuals = [1.0]
    total = 0
    converged = False
    while total < maxit and not converged:
        if total:
            r0 = K.axpby(1.0, bd, -1.0, A(x))
            beta = K.norm(r0)
        else:
            r0, beta = bd, bnorm   # x0 = 0: the first residual is b itself (read only by the cycle)
        if beta / bnorm <= tol:
            converged = True
            break
        m = maxit - total if restart is None else min(restart, maxit - total)
        if marks is not None:
            marks.append(("r0", time.perf_counter()))
        u, used, converged = _gmres_cycle(K, op, r0, beta, bnorm, tol, m, residuals, P=P, A=A)
        total += used
        if marks is not None:
            marks.append(("cycle", time.perf_counter()))
        x = K.axpby(1.0, x, 1.0, u if (P is None or K.keep_z) else P(u))
    # host callers: the copy of x to the host runs on a side stream while the
    # true-residual matvec (reference solver.py:166) runs on this one
    pending = None if on_device else nv.to_host_begin(x)
    true_res = K.norm(K.axpby(1.0, bd, -1.0, A(x))) / bnorm
    _release(K)
    x_out = x if on_device else pending.result()
    if marks is not None:
        marks.append(("true_residual+out", time.perf_counter()))
        TRACE.append(("phases", [(nm, round((tt - marks[i][1]) * 1e3, 2)) for i, (nm, tt) in enumerate(marks[1:])]))
    report = SolveReport(iterations=int(total), residuals=residuals, converged=bool(converged),
                         solve_seconds=time.perf_counter() - t0, true_residual=float(true_res))
    report.reorth_passes = int(K.reorth_passes)   # steps whose DGKS re-orthogonalisation fired (not in to_dict)
    return x_out, report


def spectrum(dense_a, dense_pinv=None) -> np.ndarray:
    """Dense eigenvalue probe (reference solver.py:177-186; host, small n only)."""
    a = np.asarray(dense_a)
    if a.shape[0] > SPECTRUM_GUARD:
        raise SizeLimitError(f"spectrum refused: size {a.shape[0]} exceeds guard {SPECTRUM_GUARD}")
    if dense_pinv is not None:
        a = a @ np.asarray(dense_pinv)
    return np.linalg.eigvals(a)


def dense_pinv_matrix(prec, n: int) -> np.ndarray:
    """Dense P^-1 by applying the preconditioner to the identity (reference solver.py:189-193)."""
    if n > SPECTRUM_GUARD:
        raise SizeLimitError(f"dense inverse refused: {n} exceeds {SPECTRUM_GUARD}")
    return prec.apply(np.eye(n, dtype=np.complex128))
