"""Host logic of the symmetry sectors (paper_1903_07884_b200/sectors.py) on
the oracle's dense frequency blocks: V orthogonal, V^T D_k V block-diagonal,
and the device unfold formula equal to V_s^T D_k V_s."""

import numpy as np
import pytest

import voxvie_oracle as O


def _kernel(dims):
    from paper_1903_07884_b200.grid import VoxelGrid
    from paper_1903_07884_b200.kernel import assemble_kernel

    return assemble_kernel(VoxelGrid(*dims, 0.05), 2 * np.pi)


@pytest.mark.parametrize("dims,sy,sz", [((6, 4, 3), True, True), ((5, 3, 4), True, True), ((6, 4, 3), True, False),
                                        ((6, 5, 3), False, True), ((4, 1, 3), True, True), ((4, 3, 1), True, True)])
def test_sector_blocks(dims, sy, sz):
    from paper_1903_07884_b200.sectors import m_symmetric, sector_blocks_host, sector_plan

    nx, ny, nz = dims
    kern = _kernel(dims)
    rng = np.random.default_rng(1)
    m = rng.normal(size=(nz, ny)) + 1j * rng.normal(size=(nz, ny))
    if sy:
        m = m + m[:, ::-1]
    if sz:
        m = m + m[::-1, :]
    assert m_symmetric(m, "y") or not sy
    lam = O.chan_x_spectra(kern.tensors)
    plan = sector_plan(ny, nz, sy, sz)
    V = plan.basis()
    Vall = np.concatenate(V, axis=1)
    q = ny * nz
    assert Vall.shape == (3 * q, 3 * q)
    assert np.abs(Vall.T @ Vall - np.eye(3 * q)).max() < 1e-14
    for k in range(nx):
        D = O.unfold_block_yz(lam[:, :, :, k], m)
        T = Vall.T @ D @ Vall
        off = T.copy()
        o = 0
        for d in plan.dims:
            off[o:o + d, o:o + d] = 0
            o += d
        assert np.abs(off).max() < 1e-12 * np.abs(D).max()
        for Vs, Bs in zip(V, sector_blocks_host(plan, D)):
            assert np.abs(Vs.T @ D @ Vs - Bs).max() < 1e-12 * np.abs(D).max()
    # inverse-transform tables reproduce V
    x = rng.normal(size=3 * q)
    u = np.zeros(plan.nsec * plan.dmax)
    for s, Vs in enumerate(V):
        u[s * plan.dmax:s * plan.dmax + Vs.shape[1]] = Vs.T @ x
    back = np.array([sum(plan.ico[i, t] * u[plan.iidx[i, t]] for t in range(4) if plan.iidx[i, t] >= 0)
                     for i in range(3 * q)])
    assert np.abs(back - x).max() < 1e-13
    fwd = np.array([[sum(plan.tco[s, r, t] * x[plan.tidx[s, r, t]] for t in range(4) if plan.tidx[s, r, t] >= 0)
                     for r in range(plan.dmax)] for s in range(plan.nsec)])
    for s, Vs in enumerate(V):
        assert np.abs(fwd[s, :Vs.shape[1]] - Vs.T @ x).max() < 1e-13
    # orbit tables: the same transform, each row read / written once
    uo = np.zeros(plan.nsec * plan.dmax)
    xo = np.zeros(3 * q)
    seen = np.zeros(3 * q, int)
    for o in range(plan.orows.shape[0]):
        rows = [r for r in plan.orows[o] if r >= 0]
        seen[rows] += 1
        for s in range(4):
            if plan.osec[o, s] >= 0:
                uo[plan.osec[o, s]] = sum(plan.ocoef[o, s, t] * x[r] for t, r in enumerate(rows))
    assert (seen == 1).all()
    assert np.abs(uo - u).max() < 1e-13
    for o in range(plan.orows.shape[0]):
        for t, r in enumerate(plan.orows[o]):
            if r >= 0:
                xo[r] = sum(plan.ocoef[o, s, t] * uo[plan.osec[o, s]] for s in range(4) if plan.osec[o, s] >= 0)
    assert np.abs(xo - x).max() < 1e-13


def test_sector_dims_c1():
    from paper_1903_07884_b200.sectors import sector_plan

    p = sector_plan(22, 11, True, True)
    assert sorted(p.dims) == [176, 176, 187, 187] and p.dmax == 187
    p = sector_plan(25, 11, False, True)
    assert sum(p.dims) == 3 * 25 * 11 and p.nsec == 2


def test_mirror_store_plan_matches_the_sequential_rule():
    """_mirror_store (vectorised) == the one-block-at-a-time rule: block k shares the factor
    of nx - k when that frequency is present and smaller, else owns a new slot."""
    from paper_1903_07884_b200.circulant import _mirror_store

    def rule(ks, nx, share):
        pos = {int(k): i for i, k in enumerate(ks)}
        store, flip, kset = np.empty(ks.size, np.int64), np.zeros(ks.size, bool), []
        for i, k in enumerate(ks):
            km = (nx - int(k)) % nx
            if share and km < k and km in pos:
                store[i], flip[i] = store[pos[km]], True
            else:
                store[i] = len(kset)
                kset.append(int(k))
        return np.asarray(kset, np.int64), store, flip

    rng = np.random.default_rng(3)
    for nx in (1, 2, 5, 8, 200, 367, 5000):
        for share in (True, False):
            for trial in range(4):
                ks = np.arange(nx) if trial == 0 else np.sort(rng.choice(nx, size=max(1, nx // 3), replace=False))
                for got, want in zip(_mirror_store(ks, nx, share), rule(ks, nx, share)):
                    assert np.array_equal(got, want), (nx, share, trial)


def test_constant_along_x_check():
    """reference circulant.py:81-96: exactly constant maps pass on the fast path, a deviation
    above 1e-12 max|m| raises, NaN raises."""
    from paper_1903_07884_b200.circulant import _constant_along

    m = np.repeat((0.5 + 0.1j * np.arange(12.0)).reshape(3, 4, 1), 50, axis=2)
    _constant_along(m, 2, "x")
    m2 = m.copy()
    m2[1, 2, 7] += 1e-14
    _constant_along(m2, 2, "x")           # within tolerance: slow path
    m2[1, 2, 7] += 1e-9
    with pytest.raises(ValueError):
        _constant_along(m2, 2, "x")
    m3 = m.copy()
    m3[0, 0, 3] = np.nan
    with pytest.raises(ValueError):
        _constant_along(m3, 2, "x")
