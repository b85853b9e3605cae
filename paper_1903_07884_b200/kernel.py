"""Generating tensors of the discretised operator N (host setup input).

The six unique dyadic components (order ``xx, xy, xz, yy, yz, zz``) are held as
``(6, 2nz-1, 2ny-1, 2nx-1)`` complex128 arrays indexed by signed voxel offset
``(dz+nz-1, dy+ny-1, dx+nx-1)`` (reference: pkg/src/voxvie/kernel.py:119-141).
Assembly runs once per problem and is *not* on the GMRES hot path; it is
restated here so the GPU box can build the BASELINE workloads without the
reference package (reference kernel.py:101-198, accel.py:44-68).

Off-self entries are ``V * G(delta*d)`` (centroid rule); the d = 0 entry is the
Duffy-quadrature self term.  Because every component is even or odd in each
offset coordinate and the offset grid is symmetric, only the non-negative
octant is evaluated and the rest is mirrored with exact sign flips -- the
mirrored values are bitwise what a direct evaluation gives.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from .errors import QuadratureError, SizeLimitError
from .grid import VoxelGrid

FOUR_PI = 4.0 * np.pi
DENSE_GUARD = 6000

PAIRS = ("xx", "xy", "xz", "yy", "yz", "zz")
#: PAIR_OF[a, b] -> index into PAIRS (reference accel.py:38-41)
PAIR_OF = np.array([[0, 1, 2], [1, 3, 4], [2, 4, 5]], dtype=np.int64)
#: parity of each component under (x, y, z) sign flips: +1 even, -1 odd
_PARITY = {
    "xx": (1, 1, 1), "xy": (-1, -1, 1), "xz": (-1, 1, -1),
    "yy": (1, 1, 1), "yz": (1, -1, -1), "zz": (1, 1, 1),
}


@dataclass(frozen=True)
class ToeplitzKernel:
    """Six generating tensors of N on a grid (reference kernel.py:119-141)."""

    grid: VoxelGrid
    k0: float
    tensors: np.ndarray

    def storage_entries(self) -> int:
        nx, ny, nz = self.grid.dims
        return 6 * (2 * nx - 1) * (2 * ny - 1) * (2 * nz - 1)

    def storage_bytes(self) -> int:
        return 16 * self.storage_entries()

    def component(self, name: str) -> np.ndarray:
        return self.tensors[PAIRS.index(name)]


def scalar_green(r, k0: float):
    r = np.asarray(r, dtype=float)
    if np.any(r <= 0):
        raise ValueError("scalar_green requires r > 0")
    return np.exp(-1j * k0 * r) / (FOUR_PI * r)


def dyadic_green(rvec, k0: float) -> np.ndarray:
    """(k0^2 I + grad grad) g at a non-zero offset (reference kernel.py:37-51)."""
    rv = np.asarray(rvec, dtype=float)
    r2 = float(rv @ rv)
    if r2 == 0.0:
        raise ValueError("dyadic_green is singular at zero offset")
    r = np.sqrt(r2)
    g = np.exp(-1j * k0 * r) / (FOUR_PI * r)
    d = g * (k0 * k0 - (1.0 + 1j * k0 * r) / r2)
    rad = g * (3.0 / r2 + 3j * k0 / r - k0 * k0) / r2
    return d * np.eye(3) + rad * np.outer(rv, rv)


def _green_octant(z, y, x, k0):
    """Six components on the non-negative offset octant (z, y, x >= 0)."""
    Z, Y, X = np.meshgrid(z, y, x, indexing="ij")
    r2 = X * X + Y * Y + Z * Z
    at0 = r2 == 0.0
    r2s = np.where(at0, 1.0, r2)
    r = np.sqrt(r2s)
    g = np.exp(-1j * k0 * r) / (FOUR_PI * r)
    k2 = k0 * k0
    d = g * (k2 - (1.0 + 1j * k0 * r) / r2s)
    rad = g * (3.0 / r2s + 3j * k0 / r - k2) / r2s
    comps = {
        "xx": d + rad * X * X, "xy": rad * X * Y, "xz": rad * X * Z,
        "yy": d + rad * Y * Y, "yz": rad * Y * Z, "zz": d + rad * Z * Z,
    }
    out = np.stack([comps[p] for p in PAIRS])
    out[:, at0] = 0.0
    return out


def green_tensors(nx, ny, nz, delta, k0) -> np.ndarray:
    """Full offset grid (6, 2nz-1, 2ny-1, 2nx-1), mirrored from one octant."""
    oct_ = _green_octant(delta * np.arange(nz), delta * np.arange(ny),
                         delta * np.arange(nx), k0)
    out = np.empty((6, 2 * nz - 1, 2 * ny - 1, 2 * nx - 1), dtype=np.complex128)
    for p, name in enumerate(PAIRS):
        sx, sy, sz = _PARITY[name]
        o = oct_[p]
        # positive offsets
        out[p, nz - 1:, ny - 1:, nx - 1:] = o
        # mirror x
        out[p, nz - 1:, ny - 1:, :nx - 1] = sx * o[:, :, :0:-1]
        # mirror y (both x halves)
        out[p, nz - 1:, :ny - 1, :] = sy * out[p, nz - 1:, 2 * ny - 2:ny - 1:-1, :]
        # mirror z
        out[p, :nz - 1, :, :] = sz * out[p, 2 * nz - 2:nz - 1:-1, :, :]
    return out


def _gauss01(order: int):
    x, w = np.polynomial.legendre.leggauss(order)
    return 0.5 * (x + 1.0), 0.5 * w


def _coincident_cube_integral(delta: float, k0: float, order: int) -> complex:
    """Double voxel integral of the scalar kernel (Duffy pyramid, reference
    kernel.py:59-84)."""
    t, w = _gauss01(order)
    A, B = np.meshgrid(t, t, indexing="ij")
    wab = np.outer(w, w)
    u = np.sqrt(1.0 + A * A + B * B)
    acc = 0.0 + 0.0j
    for ti, wi in zip(t, w):
        p = delta * ti
        f = (delta - p) * (delta - p * A) * (delta - p * B) * p * np.exp(-1j * k0 * p * u) / u
        acc += delta * wi * np.sum(wab * f)
    return 24.0 * acc / FOUR_PI


@lru_cache(maxsize=64)
def _cube_integral_converged(delta: float, k0: float, rtol: float) -> complex:
    prev = _coincident_cube_integral(delta, k0, 8)
    achieved = np.inf
    for order in (12, 18, 27, 40):
        cur = _coincident_cube_integral(delta, k0, order)
        achieved = abs(cur - prev) / max(abs(cur), 1e-300)
        if achieved <= rtol:
            return cur
        prev = cur
    raise QuadratureError("self-term quadrature did not converge", achieved)


def self_term(delta: float, k0: float, rtol: float = 1e-12) -> np.ndarray:
    """S = (2/3)(1 + k0^2 I_g / V) I (reference kernel.py:101-116)."""
    if not delta > 0:
        raise ValueError("delta must be positive")
    ig = _cube_integral_converged(float(delta), float(k0), float(rtol))
    return (2.0 / 3.0) * (1.0 + k0 * k0 * ig / delta ** 3) * np.eye(3, dtype=np.complex128)


def _gauss_cube(delta: float, n: int):
    t, w = _gauss01(n)
    pts = delta * (t - 0.5)
    P = np.stack(np.meshgrid(pts, pts, pts, indexing="ij"), axis=-1).reshape(-1, 3)
    W = np.einsum("i,j,k->ijk", w, w, w).reshape(-1) * delta ** 3
    return P, W


def assemble_kernel(grid: VoxelGrid, k0: float, *, near_gauss: bool = False) -> ToeplitzKernel:
    """Populate the generating tensors (reference kernel.py:152-198)."""
    if not k0 * grid.delta < 2.0:
        raise ValueError(f"k0*delta = {k0 * grid.delta:.3f} too coarse; need k0*delta < 2")
    nx, ny, nz = grid.dims
    d = grid.delta
    t = green_tensors(nx, ny, nz, d, k0)
    t *= grid.voxel_volume
    c = (nz - 1, ny - 1, nx - 1)
    s = self_term(d, k0)[0, 0]
    for p, name in enumerate(PAIRS):
        t[(p,) + c] = s if name in ("xx", "yy", "zz") else 0.0
    if near_gauss:
        for loc, vals in _near_gauss_entries(grid, k0):
            for p in range(6):
                t[(p,) + loc] = vals[p]
    t.setflags(write=False)
    return ToeplitzKernel(grid=grid, k0=float(k0), tensors=t)


def _near_gauss_entries(grid: VoxelGrid, k0: float):
    """3x3x3-point Gauss cube integrals for the 26 face/edge/corner neighbours
    (reference kernel.py:180-196): [(index (z, y, x) into the generator, six values)]."""
    nx, ny, nz = grid.dims
    d = grid.delta
    c = (nz - 1, ny - 1, nx - 1)
    pts, wts = _gauss_cube(d, 3)
    out = []
    for ddz in (-1, 0, 1):
        for ddy in (-1, 0, 1):
            for ddx in (-1, 0, 1):
                if (ddx, ddy, ddz) == (0, 0, 0):
                    continue
                if abs(ddx) >= nx or abs(ddy) >= ny or abs(ddz) >= nz:
                    continue
                rc = d * np.array([ddx, ddy, ddz], dtype=float)
                acc = np.zeros((3, 3), dtype=np.complex128)
                for ps, ws in zip(rc - pts, wts):
                    acc += ws * dyadic_green(ps, k0)
                loc = (c[0] + ddz, c[1] + ddy, c[2] + ddx)
                out.append((loc, [acc["xyz".index(nm[0]), "xyz".index(nm[1])] for nm in PAIRS]))
    return out


class DeviceToeplitzKernel:
    """ToeplitzKernel whose generators live in HBM (assembled by
    ``assemble_kernel_device``).  Same attributes as ToeplitzKernel; ``tensors``
    is a lazily downloaded read-only host copy (only host-side helpers such as
    the blocked preconditioner's box slicing read it)."""

    def __init__(self, grid: VoxelGrid, k0: float, device_tensors):
        self.grid = grid
        self.k0 = float(k0)
        self._vx_device_tensors = device_tensors
        self._host = None

    @property
    def tensors(self) -> np.ndarray:
        if self._host is None:
            from . import _native as nv

            h = np.array(nv.to_host(self._vx_device_tensors), copy=True)
            h.setflags(write=False)
            self._host = h
        return self._host

    def storage_entries(self) -> int:
        nx, ny, nz = self.grid.dims
        return 6 * (2 * nx - 1) * (2 * ny - 1) * (2 * nz - 1)

    def storage_bytes(self) -> int:
        return 16 * self.storage_entries()

    def component(self, name: str) -> np.ndarray:
        return self.tensors[PAIRS.index(name)]


def assemble_kernel_device(grid: VoxelGrid, k0: float, *, near_gauss: bool = False) -> DeviceToeplitzKernel:
    """assemble_kernel (reference kernel.py:152-198) evaluated on the GPU
    (vx_assemble_green): the generators are written straight into HBM; the
    self term (and the optional 26 near-neighbour Gauss integrals) come from
    the host quadrature as in the reference."""
    from . import _native as nv

    if not k0 * grid.delta < 2.0:
        raise ValueError(f"k0*delta = {k0 * grid.delta:.3f} too coarse; need k0*delta < 2")
    t = nv.require_cuda()
    nx, ny, nz = grid.dims
    s = complex(self_term(grid.delta, k0)[0, 0])
    out = t.empty((6, 2 * nz - 1, 2 * ny - 1, 2 * nx - 1), dtype=t.complex128, device="cuda")
    nv.call("vx_assemble_green", nx, ny, nz, float(grid.delta), float(k0), float(grid.voxel_volume),
            nv.c128(s.real, s.imag), out.data_ptr(), nv.stream_ptr())
    if near_gauss:
        ent = _near_gauss_entries(grid, k0)
        if ent:
            idx = t.tensor([loc for loc, _ in ent], dtype=t.long)
            vals = t.tensor(np.array([v for _, v in ent], dtype=np.complex128).T.copy()).cuda()  # (6, m)
            out[:, idx[:, 0], idx[:, 1], idx[:, 2]] = vals
    return DeviceToeplitzKernel(grid, k0, out)


def check_dense_guard(n_unknowns: int, guard: int = DENSE_GUARD):
    if n_unknowns > guard:
        raise SizeLimitError(f"dense oracle refused: {n_unknowns} unknowns exceeds guard {guard}")
