"""Synthetic BASELINE workloads c0..c4.

Deterministic host-side construction of the five configurations named in
BASELINE.json; no dataset is involved.  Interpretation B (homogeneous
background VIE) is canonical: ``k = 2*pi*n_b/lambda0`` and
``eps_rel = (n_voxel/n_b)^2`` with ``n_voxel = n_r - j*kappa``.

Each workload returns a ``Workload`` with the grid, the permittivity map, the
medium coefficient ``m``, the incident field, the right-hand side ``b`` and
the preconditioner recipe; the generating tensors are assembled on demand
(``Workload.kernel()``), since at c1 they are ~0.9 GB.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .grid import PermittivityMap, Physics, VoxelGrid, homogenize, medium_coefficient
from .kernel import assemble_kernel

LAMBDA0 = 1.55e-6
N_BG = 1.45
N_CORE = 3.48


@dataclass
class Workload:
    name: str
    grid: VoxelGrid
    physics: Physics
    pmap: PermittivityMap
    e_inc: np.ndarray
    prec: dict            # {"kind": ..., "homogenization": ..., boxes...}
    restart: int
    tol: float = 1e-5
    maxit: int = 2000
    interpretation: str = "B"
    notes: dict = field(default_factory=dict)
    _kernel: object = None

    @property
    def m(self) -> np.ndarray:
        return medium_coefficient(self.pmap)

    @property
    def b(self) -> np.ndarray:
        m = self.m
        e = self.e_inc.reshape((3,) + m.shape)
        return (1j * self.physics.omega * self.physics.eps0 * m[None] * e).reshape(-1)

    def kernel(self):
        if self._kernel is None:
            self._kernel = assemble_kernel(self.grid, self.physics.k0)
        return self._kernel

    def mtilde(self, box=None):
        """Homogenised map for the whole grid or a box (x0,x1,y0,y1,z0,z1)."""
        strat = self.prec["homogenization"]
        if box is None:
            # memoised: a pure function of the workload's inputs
            if getattr(self, "_mtilde", None) is None:
                object.__setattr__(self, "_mtilde", homogenize(self.pmap, strat))
            return self._mtilde
        x0, x1, y0, y1, z0, z1 = box
        sub = VoxelGrid(x1 - x0, y1 - y0, z1 - z0, self.grid.delta)
        return homogenize(PermittivityMap(sub, self.pmap.eps_r[z0:z1, y0:y1, x0:x1]), strat)


def _eps(n_r: np.ndarray, kappa: np.ndarray, interp: str) -> np.ndarray:
    n = n_r - 1j * kappa
    return (n / N_BG) ** 2 if interp == "B" else n ** 2


def _physics(interp: str) -> Physics:
    return Physics.from_wavelength(LAMBDA0 / N_BG if interp == "B" else LAMBDA0)


def _absorber_kappa(nx: int, n_abs: int) -> np.ndarray:
    ix = np.arange(nx)
    start = nx - n_abs
    return np.where(ix < start, 0.0, 0.05 * (ix - start + 0.5) / max(n_abs, 1))


def _incident(grid: VoxelGrid, mask_yz=None, mask_3d=None) -> np.ndarray:
    nz, ny, nx = grid.shape
    xc = (np.arange(nx) + 0.5) * grid.delta
    wave = np.exp(1j * (2 * np.pi / LAMBDA0) * N_BG * xc)
    e = np.zeros((3, nz, ny, nx), np.complex128)
    e[1] = wave[None, None, :]
    if mask_yz is not None:
        e[1] *= mask_yz[:, :, None]
    if mask_3d is not None:
        e[1] *= mask_3d
    return e.reshape(-1)


def make(name: str, interp: str = "B") -> Workload:
    phys = _physics(interp)
    if name == "c0":
        grid = VoxelGrid(200, 10, 5, 0.045e-6)
        core = np.ones(grid.shape, bool)
        kap = np.broadcast_to(_absorber_kappa(200, 40), grid.shape)
        prec, restart = {"kind": "one-level", "homogenization": "real_mean_x"}, 50
        e = _incident(grid)
    elif name in ("c1", "c1r"):
        grid = VoxelGrid(5000, 22, 11, 0.02e-6)
        core = np.ones(grid.shape, bool)
        kap = np.broadcast_to(_absorber_kappa(5000, 1000), grid.shape)
        if name == "c1":
            prec = {"kind": "one-level", "homogenization": "real_mean_x"}
        else:
            prec = {"kind": "reduced-one-level", "homogenization": "real_mean_x", "tol": 1e-3}
        restart = 50
        e = _incident(grid)
    elif name == "c2":
        grid = VoxelGrid(2500, 25, 11, 0.02e-6)
        ix = np.arange(2500)
        iy = np.arange(25)
        wide = (ix % 16) < 8
        narrow_y = (iy >= 2) & (iy < 22)
        col = wide[None, :] | narrow_y[:, None]          # (ny, nx)
        core = np.broadcast_to(col[None], grid.shape)
        kap = np.broadcast_to(_absorber_kappa(2500, 500), grid.shape)
        prec, restart = {"kind": "one-level", "homogenization": "mean_x"}, 50
        e = _incident(grid)
    elif name == "c3":
        grid = VoxelGrid(1500, 56, 11, 0.02e-6)
        iy = np.arange(56)
        g1 = (iy >= 1) & (iy < 23)
        g2 = (iy >= 33) & (iy < 55)
        core = np.broadcast_to((g1 | g2)[None, :, None], grid.shape)
        kap = np.broadcast_to(_absorber_kappa(1500, 300), grid.shape)
        prec = {"kind": "blocked", "homogenization": "real_mean_x",
                "boxes": [(0, 1500, 0, 28, 0, 11), (0, 1500, 28, 56, 0, 11)],
                "levels": ["one-level", "one-level"], "labels": ["guide1", "guide2"]}
        restart = 50
        e = _incident(grid, mask_yz=np.broadcast_to(g1[None, :], (11, 56)).astype(float))
    elif name in ("c4", "c4b"):
        grid = VoxelGrid(367, 400, 8, 0.03e-6)
        ix = np.arange(367) + 0.5
        iy = np.arange(400) + 0.5
        bus = (iy >= 22) & (iy < 37)
        disk = (ix[None, :] - 183.5) ** 2 + (iy[:, None] - 211.0) ** 2 <= 167.0 ** 2
        cols = bus[:, None] | disk                        # (ny, nx)
        zcore = np.arange(8) < 7
        core = zcore[:, None, None] & cols[None]
        bus3 = zcore[:, None, None] & np.broadcast_to(bus[:, None], (400, 367))[None]
        kap = np.where(bus3, _absorber_kappa(367, 73)[None, None, :], 0.0)
        if name == "c4":
            prec = {"kind": "two-level", "homogenization": "mode"}
        else:
            # the paper's disk-resonator preconditioner (reference
            # photonics.py:249-255 hint): reduced 1-level on the bus box, 2-level
            # on the disk box, identity elsewhere
            prec = {"kind": "blocked", "homogenization": None,
                    "boxes": [(0, 367, 22, 37, 0, 8), (16, 351, 44, 378, 0, 8)],
                    "levels": ["reduced-one-level", "two-level"], "labels": ["bus", "disk"]}
        restart = 100
        e = _incident(grid, mask_3d=bus3.astype(float))
    else:
        raise ValueError(f"unknown workload {name!r}")
    n_r = np.where(core, N_CORE, N_BG)
    kappa = np.where(core | (name not in ("c4", "c4b")), kap, 0.0)
    eps = _eps(n_r, kappa, interp)
    # cladding voxels outside any absorber are exactly background: eps = 1
    eps = np.where((n_r == N_BG) & (kappa == 0.0), 1.0 + 0j, eps)
    pmap = PermittivityMap(grid, eps)
    return Workload(name=name, grid=grid, physics=phys, pmap=pmap, e_inc=e, prec=prec,
                    restart=restart, interpretation=interp)


def small(nx=200, ny=10, nz=5, delta=0.045e-6, interp="B") -> Workload:
    """c0-like straight waveguide with arbitrary dims (tests, smoke)."""
    phys = _physics(interp)
    grid = VoxelGrid(nx, ny, nz, delta)
    kap = np.broadcast_to(_absorber_kappa(nx, round(0.2 * nx)), grid.shape)
    eps = _eps(np.full(grid.shape, N_CORE), kap, interp)
    return Workload(name=f"wg{nx}x{ny}x{nz}", grid=grid, physics=phys,
                    pmap=PermittivityMap(grid, eps), e_inc=_incident(grid),
                    prec={"kind": "one-level", "homogenization": "real_mean_x"}, restart=50)
