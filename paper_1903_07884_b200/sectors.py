"""Symmetry sectors of the 1-level frequency blocks (host tables for the device).

For every x-frequency k the reference factorises the dense block
``D_k = I - diag(m~) N_k`` (reference circulant.py:216-224, unfold
accel.py:71-91) with rows/columns ``a*q + iz*ny + iy``.  When the kernel has
y (z) parity -- every Green component even or odd in dy (dz), reference
kernel.py:37-51 -- and the homogenised coefficient m~ is mirror-symmetric in
y (z), the reflection ``P_y = S_y R_y`` (R_y: iy -> ny-1-iy on the sites,
S_y: -1 on the y-component rows) commutes with D_k, and likewise P_z.  The
block is then block-diagonal in the joint eigenbasis of (P_y, P_z): 2 or 4
independent sectors of about n/2 or n/4 rows.  Factorising the sectors
instead of D_k stores 1/2 or 1/4 of the bytes (the per-iteration block
solve streams them) and takes 1/4 or 1/16 of the LU flops; D_k^-1 b is
unchanged up to rounding.

Basis (orthonormal V_s per sector s = character chi of the group G):
    v_j = (1/c_j) sum_{g in G} chi(g) S_g(a) e_(a, g.i)
for a component a and an orbit representative site i (sites whose sum
vanishes are not in the sector), c_j the norm.  Then (V_s^T D V_s)[j, j'] =
(|G| / (c_j c_j')) sum_h chi(h) S_h(b) D[(a, i), (b, h.i')], which the
device unfold evaluates from four entries of D.

Tables (all int32 / float64, padded to dmax = the largest sector):
    tidx/tco  (nsec, dmax, 4): sector row -> original rows and coefficients
              (forward transform u = V^T x; unused slots -1 / 0)
    iidx/ico  (3q, 4):         original row -> flat sector rows s*dmax + r
              and coefficients (inverse transform x = sum_s V_s u_s)
    rrow/rsc  (nsec, dmax):    representative original row, |G|/c_j (-1: pad)
    ccol/cw   (nsec, dmax, 4): original columns (b, h.i') and chi(h)S_h(b)/c_j'
    orows/osec/ocoef:          the same transform per orbit (component, site
              orbit), so the device reads and writes every row exactly once
"""

from __future__ import annotations

import functools
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class SectorPlan:
    ny: int
    nz: int
    sym_y: bool
    sym_z: bool
    nsec: int
    dims: tuple          # rows per sector
    dmax: int
    tidx: np.ndarray
    tco: np.ndarray
    iidx: np.ndarray
    ico: np.ndarray
    rrow: np.ndarray
    rsc: np.ndarray
    ccol: np.ndarray
    cw: np.ndarray
    orows: np.ndarray    # (norb, 4) original rows of the orbit (-1 unused)
    osec: np.ndarray     # (norb, 4) flat sector row s*dmax + r per sector s (-1: not in s)
    ocoef: np.ndarray    # (norb, 4, 4) [s][t] coefficient of orows[t] in sector s's row

    def basis(self) -> list:
        """Dense V_s (3q, d_s) per sector (host, tests)."""
        q = self.ny * self.nz
        out = []
        for s, d in enumerate(self.dims):
            v = np.zeros((3 * q, d))
            for r in range(d):
                for t in range(4):
                    i = self.tidx[s, r, t]
                    if i >= 0:
                        v[i, r] += self.tco[s, r, t]
            out.append(v)
        return out


def m_symmetric(m_yz: np.ndarray, axis: str, rtol: float = 1e-13) -> bool:
    """m~ (nz, ny) mirror-symmetric in y (axis 'y') or z ('z')."""
    m = np.asarray(m_yz)
    f = m[:, ::-1] if axis == "y" else m[::-1, :]
    scale = max(np.abs(m).max(), 1e-300)
    return bool(np.abs(m - f).max() <= rtol * scale)


@functools.lru_cache(maxsize=16)
def sector_plan(ny: int, nz: int, sym_y: bool, sym_z: bool) -> SectorPlan | None:
    """Sector tables for the enabled reflections (None if neither)."""
    if not (sym_y or sym_z):
        return None
    q = ny * nz
    # group elements as (fy, fz) flags
    G = [(0, 0)]
    if sym_y:
        G.append((1, 0))
    if sym_z:
        G.append((0, 1))
    if sym_y and sym_z:
        G.append((1, 1))
    chars = [(ey, ez) for ey in ((1, -1) if sym_y else (1,)) for ez in ((1, -1) if sym_z else (1,))]

    def act(g, site):
        iz, iy = divmod(site, ny)
        if g[0]:
            iy = ny - 1 - iy
        if g[1]:
            iz = nz - 1 - iz
        return iz * ny + iy

    def sgn(g, a):  # S_g(a)
        return (-1.0 if (g[0] and a == 1) else 1.0) * (-1.0 if (g[1] and a == 2) else 1.0)

    def chi(c, g):
        return (c[0] if g[0] else 1) * (c[1] if g[1] else 1)

    reps = sorted({min(act(g, i) for g in G) for i in range(q)})
    rows = []  # per sector: list of (a, rep, {site: coef}, c)
    for c in chars:
        lst = []
        for a in range(3):
            for i in reps:
                coef = {}
                for g in G:
                    j = act(g, i)
                    coef[j] = coef.get(j, 0.0) + chi(c, g) * sgn(g, a)
                coef = {j: v for j, v in coef.items() if v != 0.0}
                if not coef:
                    continue
                norm = float(np.sqrt(sum(v * v for v in coef.values())))
                lst.append((a, i, coef, norm))
        rows.append(lst)
    nsec = len(chars)
    dims = tuple(len(r) for r in rows)
    dmax = max(dims)
    nG = len(G)
    tidx = np.full((nsec, dmax, 4), -1, np.int32)
    tco = np.zeros((nsec, dmax, 4))
    rrow = np.full((nsec, dmax), -1, np.int32)
    rsc = np.zeros((nsec, dmax))
    ccol = np.full((nsec, dmax, 4), -1, np.int32)
    cw = np.zeros((nsec, dmax, 4))
    iidx = np.full((3 * q, 4), -1, np.int32)
    ico = np.zeros((3 * q, 4))
    fill = np.zeros(3 * q, np.int32)
    for s, (c, lst) in enumerate(zip(chars, rows)):
        for r, (a, i, coef, norm) in enumerate(lst):
            for t, (j, v) in enumerate(sorted(coef.items())):
                tidx[s, r, t] = a * q + j
                tco[s, r, t] = v / norm
                o = a * q + j
                iidx[o, fill[o]] = s * dmax + r
                ico[o, fill[o]] = v / norm
                fill[o] += 1
            rrow[s, r] = a * q + i
            rsc[s, r] = nG / norm
            for t, g in enumerate(G):
                ccol[s, r, t] = a * q + act(g, i)
                cw[s, r, t] = chi(c, g) * sgn(g, a) / norm
    orb = {}
    for s, lst in enumerate(rows):
        for r, (a, i, coef, norm) in enumerate(lst):
            ent = orb.setdefault((a, i), {"sites": sorted({act(g, i) for g in G}), "sec": {}})
            ent["sec"][s] = (r, {j: v / norm for j, v in coef.items()})
    keys = sorted(orb)
    norb = len(keys)
    orows = np.full((norb, 4), -1, np.int32)
    osec = np.full((norb, 4), -1, np.int32)
    ocoef = np.zeros((norb, 4, 4))
    for o, (a, i) in enumerate(keys):
        ent = orb[(a, i)]
        for t, j in enumerate(ent["sites"]):
            orows[o, t] = a * q + j
        for s2, (r, cf) in ent["sec"].items():
            osec[o, s2] = s2 * dmax + r
            for t, j in enumerate(ent["sites"]):
                ocoef[o, s2, t] = cf.get(j, 0.0)
    return SectorPlan(ny, nz, bool(sym_y), bool(sym_z), nsec, dims, dmax, tidx, tco, iidx, ico, rrow, rsc,
                      ccol, cw, orows, osec, ocoef)


def sector_blocks_host(plan: SectorPlan, D: np.ndarray) -> list:
    """Sector blocks from a dense D by the unfold formula (host reference of
    the device unfold; tests compare it with V_s^T D V_s)."""
    out = []
    for s, d in enumerate(plan.dims):
        B = np.zeros((d, d), D.dtype)
        for j in range(d):
            row = plan.rrow[s, j]
            for jp in range(d):
                acc = 0.0
                for t in range(4):
                    col = plan.ccol[s, jp, t]
                    if col >= 0:
                        acc = acc + plan.cw[s, jp, t] * D[row, col]
                B[j, jp] = plan.rsc[s, j] * acc
        out.append(B)
    return out
