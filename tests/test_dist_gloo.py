"""Sharded solve on CPU with world_size 2 (gloo) and the numpy test backend:
layouts, all-to-all transposes, all-reduced Arnoldi and the replicated GMRES
control must reproduce the single-process oracle."""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, tol, out_dir):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "oracle"))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    from dist_numpy_backend import NumpyBackend
    from paper_1903_07884_b200 import workloads
    from paper_1903_07884_b200.dist import DistOneLevelPrec, DistOperator, Layout, _Comm, gmres_sharded

    W = workloads.small(20, 4, 3, delta=0.045e-6)
    kern = W.kernel()
    B, C = NumpyBackend(), _Comm()
    L = Layout(W.grid.dims, world, rank, 2 * W.grid.nx)
    op = DistOperator(kern, L, B, C)
    m_full = torch.from_numpy(W.m.reshape(-1).copy())
    rng = np.random.default_rng(7)
    x = rng.normal(size=W.grid.n_unknowns) + 1j * rng.normal(size=W.grid.n_unknowns)
    y_op = op.apply(m_full, torch.from_numpy(L.local_slice(x).copy())).numpy()
    results = {"op": y_op, "line0": L.line0, "line1": L.line1}
    prec = DistOneLevelPrec(kern, W.mtilde(), L, B, C, tol=tol)
    results["prec"] = prec.apply(torch.from_numpy(L.local_slice(x).copy())).numpy()
    b_loc = torch.from_numpy(L.local_slice(W.b).copy())
    xs, rep = gmres_sharded(lambda v: op.apply(m_full, v), b_loc, B, C, apply_pinv=prec.apply, tol=1e-8,
                            maxit=200, restart=7)
    results["x"] = xs.numpy()
    results["its"] = rep.iterations
    results["res"] = np.array(rep.residuals)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), **results)
    dist.destroy_process_group()


@pytest.mark.parametrize("tol", [None, 0.3])
def test_sharded_solve_world2_matches_oracle(tmp_path, tol):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), tol, str(tmp_path)), nprocs=world, join=True)
    sys.path.insert(0, str(ROOT / "oracle"))
    import voxvie_oracle as O
    from paper_1903_07884_b200 import workloads

    W = workloads.small(20, 4, 3, delta=0.045e-6)
    dims = W.grid.dims
    t = W.kernel().tensors
    spec = O.plan_spectra(t, dims)
    p = O.build_one_level(t, dims, W.mtilde())
    if tol is not None:
        p = O.reduce_one_level(p, tol)
    rng = np.random.default_rng(7)
    x = rng.normal(size=W.grid.n_unknowns) + 1j * rng.normal(size=W.grid.n_unknowns)
    parts = [dict(np.load(tmp_path / f"r{r}.npz")) for r in range(world)]
    nx = dims[0]
    op = np.concatenate([q["op"] for q in parts])
    pr = np.concatenate([q["prec"] for q in parts])
    ref_op = O.apply_system(spec, dims, W.m, x)
    ref_pr = O.apply_prec(p, x)
    assert np.linalg.norm(op - ref_op) / np.linalg.norm(ref_op) < 1e-12
    assert np.linalg.norm(pr - ref_pr) / np.linalg.norm(ref_pr) < 1e-12
    assert [int(q["line1"]) - int(q["line0"]) for q in parts] == [18, 18]
    xo, ro = O.gmres(lambda v: O.apply_system(spec, dims, W.m, v), W.b,
                     apply_pinv=lambda v: O.apply_prec(p, v), tol=1e-8, maxit=200, restart=7)
    xs = np.concatenate([q["x"] for q in parts])
    assert int(parts[0]["its"]) == int(parts[1]["its"])
    assert abs(int(parts[0]["its"]) - ro["iterations"]) <= 2
    assert np.linalg.norm(xs - xo) / np.linalg.norm(xo) < 1e-7
    assert nx * 36 == xs.size


def _worker2(rank, world, port, out_dir):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "oracle"))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    from dist_numpy_backend import NumpyBackend
    from paper_1903_07884_b200 import workloads
    from paper_1903_07884_b200.dist import DistOperator, DistTwoLevelPrec, Layout, _Comm, gmres_sharded

    W = workloads.small(12, 6, 3, delta=0.045e-6)
    kern = W.kernel()
    B, C = NumpyBackend(), _Comm()
    L = Layout(W.grid.dims, world, rank, 2 * W.grid.nx)
    op = DistOperator(kern, L, B, C)
    m_full = torch.from_numpy(W.m.reshape(-1).copy())
    mt = complex(np.mean(W.m))
    prec = DistTwoLevelPrec(kern, mt, L, B, C)
    rng = np.random.default_rng(11)
    x = rng.normal(size=W.grid.n_unknowns) + 1j * rng.normal(size=W.grid.n_unknowns)
    results = {"prec": prec.apply(torch.from_numpy(L.local_slice(x).copy())).numpy(), "nk": L.nk}
    b_loc = torch.from_numpy(L.local_slice(W.b).copy())
    xs, rep = gmres_sharded(lambda v: op.apply(m_full, v), b_loc, B, C, apply_pinv=prec.apply, tol=1e-8,
                            maxit=200, restart=9)
    results["x"] = xs.numpy()
    results["its"] = rep.iterations
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), **results)
    dist.destroy_process_group()


def test_sharded_two_level_world2_matches_oracle(tmp_path):
    """kx-sharded factors, y-DFT + (3nz)^2 solves per rank."""
    world = 2
    mp.spawn(_worker2, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    sys.path.insert(0, str(ROOT / "oracle"))
    import voxvie_oracle as O
    from paper_1903_07884_b200 import workloads

    W = workloads.small(12, 6, 3, delta=0.045e-6)
    dims = W.grid.dims
    t = W.kernel().tensors
    spec = O.plan_spectra(t, dims)
    p = O.build_two_level(t, dims, complex(np.mean(W.m)))
    rng = np.random.default_rng(11)
    x = rng.normal(size=W.grid.n_unknowns) + 1j * rng.normal(size=W.grid.n_unknowns)
    parts = [dict(np.load(tmp_path / f"r{r}.npz")) for r in range(world)]
    assert [int(q["nk"]) for q in parts] == [6, 6]
    pr = np.concatenate([q["prec"] for q in parts])
    ref = O.apply_prec(p, x)
    assert np.linalg.norm(pr - ref) / np.linalg.norm(ref) < 1e-12
    xo, ro = O.gmres(lambda v: O.apply_system(spec, dims, W.m, v), W.b,
                     apply_pinv=lambda v: O.apply_prec(p, v), tol=1e-8, maxit=200, restart=9)
    xs = np.concatenate([q["x"] for q in parts])
    assert int(parts[0]["its"]) == int(parts[1]["its"])
    assert abs(int(parts[0]["its"]) - ro["iterations"]) <= 2
    assert np.linalg.norm(xs - xo) / np.linalg.norm(xo) < 1e-7


_BOXES = [("a", (0, 14, 0, 4, 0, 3), "one-level"), ("b", (2, 12, 4, 8, 0, 2), "reduced-one-level"),
          ("c", (0, 9, 4, 8, 2, 3), "two-level")]


def _worker3(rank, world, port, out_dir):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "oracle"))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    from dist_numpy_backend import NumpyBackend
    from paper_1903_07884_b200 import workloads
    from paper_1903_07884_b200.circulant import Box, partition_boxes
    from paper_1903_07884_b200.dist import DistBlockedPrec, Layout, _Comm

    W = workloads.small(14, 8, 3, delta=0.045e-6)
    kern = W.kernel()
    B, C = NumpyBackend(), _Comm()
    L = Layout(W.grid.dims, world, rank, 2 * W.grid.nx)
    part = partition_boxes(W.grid, [Box(lbl, *b) for lbl, b, _ in _BOXES])
    prec = DistBlockedPrec(kern, W.pmap, part, {lbl: lv for lbl, _, lv in _BOXES}, L, B, C, reduce_tol=0.3)
    rng = np.random.default_rng(13)
    x = rng.normal(size=W.grid.n_unknowns) + 1j * rng.normal(size=W.grid.n_unknowns)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"),
             prec=prec.apply(torch.from_numpy(L.local_slice(x).copy())).numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_blocked_matches_oracle(tmp_path, world):
    """SURVEY 8(e) blocked: per-box line redistribution + sharded box preconditioners."""
    mp.spawn(_worker3, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    sys.path.insert(0, str(ROOT / "oracle"))
    import voxvie_oracle as O
    from paper_1903_07884_b200 import workloads
    from paper_1903_07884_b200.circulant import _DEFAULT_HOMOG, Box, _sub_grid
    from paper_1903_07884_b200.grid import PermittivityMap, homogenize

    W = workloads.small(14, 8, 3, delta=0.045e-6)
    dims = W.grid.dims
    mts = []
    for lbl, b, lv in _BOXES:
        bb = Box(lbl, *b)
        smap = PermittivityMap(_sub_grid(W.grid, bb), W.pmap.eps_r[bb.z0:bb.z1, bb.y0:bb.y1, bb.x0:bb.x1])
        mts.append(homogenize(smap, _DEFAULT_HOMOG[lv]))
    p = O.build_blocked(W.kernel().tensors, dims, [b for _, b, _ in _BOXES], [lv for _, _, lv in _BOXES], mts,
                        reduce_tol=0.3)
    rng = np.random.default_rng(13)
    x = rng.normal(size=W.grid.n_unknowns) + 1j * rng.normal(size=W.grid.n_unknowns)
    pr = np.concatenate([dict(np.load(tmp_path / f"r{r}.npz"))["prec"] for r in range(world)])
    ref = O.apply_prec(p, x)
    assert np.linalg.norm(pr - ref) / np.linalg.norm(ref) < 1e-12
