"""GPU: the sharded-solve CUDA backend on a single-rank NCCL group (the
multi-rank data movement is covered on CPU by test_dist_gloo.py), and the
all-to-all pack/unpack kernels with P > 1 maps against numpy."""

import os
import socket

import numpy as np
import pytest

import voxvie_oracle as O
from conftest import random_field, relerr

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def group():
    import torch
    import torch.distributed as dist

    if not dist.is_initialized():
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield None
    if dist.is_initialized():
        dist.destroy_process_group()


def test_gather_scatter_cols_p3(rng):
    import torch

    from paper_1903_07884_b200 import _native as nv

    nrows, lda = 7, 23
    a = random_field(rng, nrows * lda).reshape(nrows, lda)
    kown = [np.arange(s, lda, 3) for s in range(3)]
    off = np.cumsum([0] + [k.size for k in kown]).astype(np.int32)
    cmap = np.concatenate(kown).astype(np.int32)
    A = torch.from_numpy(a.copy()).cuda()
    out = nv.empty_c128(nrows * lda)
    d_off, d_map = torch.from_numpy(off).cuda(), torch.from_numpy(cmap).cuda()
    nv.call("vx_gather_cols", nrows, A.data_ptr(), lda, 3, d_off.data_ptr(), d_map.data_ptr(), lda,
            out.data_ptr(), nv.stream_ptr())
    ref = np.concatenate([a[:, k].reshape(-1) for k in kown])
    assert np.array_equal(out.cpu().numpy(), ref)
    B = torch.zeros_like(A)
    nv.call("vx_scatter_cols", nrows, out.data_ptr(), 3, d_off.data_ptr(), d_map.data_ptr(), lda,
            B.data_ptr(), lda, nv.stream_ptr())
    assert np.array_equal(B.cpu().numpy(), a)


@pytest.mark.parametrize("tol", [None, 1e-3])
def test_sharded_path_single_rank_matches(group, tol):
    import torch

    from paper_1903_07884_b200 import workloads
    from paper_1903_07884_b200.dist import CudaBackend, DistOneLevelPrec, DistOperator, Layout, _Comm, gmres_sharded
    from paper_1903_07884_b200.operator import padded_length

    W = workloads.small(60, 8, 5, delta=0.03e-6)
    kern = W.kernel()
    dims = W.grid.dims
    B, C = CudaBackend(), _Comm()
    L = Layout(dims, 1, 0, padded_length(dims[0]))
    op = DistOperator(kern, L, B, C)
    prec = DistOneLevelPrec(kern, W.mtilde(), L, B, C, tol=tol)
    m = torch.from_numpy(W.m.reshape(-1).copy()).cuda()
    rng = np.random.default_rng(3)
    x = random_field(rng, W.grid.n_unknowns)
    xd = torch.from_numpy(x).cuda()
    spec = O.plan_spectra(kern.tensors, dims)
    p = O.build_one_level(kern.tensors, dims, W.mtilde())
    if tol is not None:
        p = O.reduce_one_level(p, tol)
    assert relerr(op.apply(m, xd).cpu().numpy(), O.apply_system(spec, dims, W.m, x)) < 1e-12
    assert relerr(prec.apply(xd).cpu().numpy(), O.apply_prec(p, x)) < 1e-10
    b = torch.from_numpy(W.b.copy()).cuda()
    xs, rep = gmres_sharded(lambda v: op.apply(m, v), b, B, C, apply_pinv=prec.apply, tol=1e-8, maxit=300,
                            restart=20)
    xo, ro = O.gmres(lambda v: O.apply_system(spec, dims, W.m, v), W.b,
                     apply_pinv=lambda v: O.apply_prec(p, v), tol=1e-8, maxit=300, restart=20)
    assert abs(rep.iterations - ro["iterations"]) <= 2
    assert relerr(xs.cpu().numpy(), xo) < 1e-6


class LoopbackComm:
    """TEST INFRASTRUCTURE: P simulated ranks as threads of one process on one
    GPU.  Collectives synchronise the device, exchange through host-side slots
    behind a threading barrier, and copy back -- no kernel ever waits on another
    rank's kernel, so this is safe on a single GPU."""

    def __init__(self, P):
        import threading

        self.P = P
        self.bar = threading.Barrier(P)
        self.slots = [None] * P

    def view(self, rank):
        comm = self

        class _R:
            def all_to_all(self, out, inp, out_splits, in_splits):
                import torch

                torch.cuda.synchronize()
                chunks, o = [], 0
                for n in in_splits:
                    chunks.append(inp[o:o + int(n)].clone())
                    o += int(n)
                comm.slots[rank] = chunks
                comm.bar.wait()
                parts = [comm.slots[r][rank] for r in range(comm.P)]
                assert [p.numel() for p in parts] == [int(v) for v in out_splits]
                out.copy_(torch.cat(parts))
                torch.cuda.synchronize()
                comm.bar.wait()

            def all_reduce(self, t):
                import torch

                torch.cuda.synchronize()
                comm.slots[rank] = t.clone()
                comm.bar.wait()
                tot = comm.slots[0].clone()
                for r in range(1, comm.P):
                    tot += comm.slots[r]
                comm.bar.wait()
                t.copy_(tot)
                torch.cuda.synchronize()
                return t

        return _R()


@pytest.mark.parametrize("P,tol", [(2, None), (3, None), (4, 1e-3)])
def test_sharded_cuda_backend_multi_rank_loopback(P, tol):
    """The sharded solve with P simulated ranks (threads) on one GPU reproduces
    the single-GPU operator, preconditioner and GMRES."""
    import threading

    import torch

    from paper_1903_07884_b200 import workloads
    from paper_1903_07884_b200.circulant import build_one_level, reduce_one_level
    from paper_1903_07884_b200.dist import CudaBackend, DistOneLevelPrec, DistOperator, Layout, gmres_sharded
    from paper_1903_07884_b200.operator import apply_system, padded_length, plan_operator
    from paper_1903_07884_b200.solver import gmres

    W = workloads.small(48, 6, 4, delta=0.03e-6)
    kern = W.kernel()
    dims = W.grid.dims
    comm = LoopbackComm(P)
    rng = np.random.default_rng(11)
    x = random_field(rng, W.grid.n_unknowns)
    results = [None] * P
    errors = []

    def run(rank):
        try:
            torch.cuda.set_device(0)
            B, C = CudaBackend(), comm.view(rank)
            L = Layout(dims, P, rank, padded_length(dims[0]))
            op = DistOperator(kern, L, B, C)
            prec = DistOneLevelPrec(kern, W.mtilde(), L, B, C, tol=tol)
            m = torch.from_numpy(W.m.reshape(-1).copy()).cuda()
            xl = torch.from_numpy(L.local_slice(x).copy()).cuda()
            y_op = op.apply(m, xl).cpu().numpy()
            y_pc = prec.apply(xl).cpu().numpy()
            bl = torch.from_numpy(L.local_slice(W.b).copy()).cuda()
            xs, rep = gmres_sharded(lambda v: op.apply(m, v), bl, B, C, apply_pinv=prec.apply, tol=1e-8,
                                    maxit=300, restart=15)
            results[rank] = (y_op, y_pc, xs.cpu().numpy(), rep.iterations)
        except Exception as e:  # surface worker failures in the main thread
            errors.append(e)
            comm.bar.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    plan = plan_operator(kern)
    p1 = build_one_level(kern, W.mtilde())
    p = p1 if tol is None else reduce_one_level(p1, tol)
    y_op = np.concatenate([r[0] for r in results])
    y_pc = np.concatenate([r[1] for r in results])
    assert relerr(y_op, apply_system(plan, W.m, x)) < 1e-12
    assert relerr(y_pc, p.apply(x)) < 1e-11
    xs = np.concatenate([r[2] for r in results])
    x1, rep1 = gmres(lambda v: apply_system(plan, W.m, v), W.b, apply_pinv=p.apply, tol=1e-8, maxit=300,
                     restart=15)
    assert len({r[3] for r in results}) == 1
    assert abs(results[0][3] - rep1.iterations) <= 2
    assert relerr(xs, x1) < 1e-6


@pytest.mark.parametrize("P", [1, 2, 3])
def test_sharded_two_level_loopback(P):
    """kx-sharded (3nz)^2 factors on the CUDA backend with
    P simulated ranks reproduce the single-GPU TwoLevelPrec and its GMRES."""
    import threading

    import torch

    from paper_1903_07884_b200 import workloads
    from paper_1903_07884_b200.circulant import build_two_level
    from paper_1903_07884_b200.dist import CudaBackend, DistOperator, DistTwoLevelPrec, Layout, gmres_sharded
    from paper_1903_07884_b200.operator import apply_system, padded_length, plan_operator
    from paper_1903_07884_b200.solver import gmres

    W = workloads.small(37, 10, 4, delta=0.03e-6)
    kern = W.kernel()
    dims = W.grid.dims
    mt = complex(np.mean(W.m))
    comm = LoopbackComm(P)
    rng = np.random.default_rng(5)
    x = random_field(rng, W.grid.n_unknowns)
    results = [None] * P
    errors = []

    def run(rank):
        try:
            torch.cuda.set_device(0)
            B, C = CudaBackend(), comm.view(rank)
            L = Layout(dims, P, rank, padded_length(dims[0]))
            op = DistOperator(kern, L, B, C)
            prec = DistTwoLevelPrec(kern, mt, L, B, C)
            m = torch.from_numpy(W.m.reshape(-1).copy()).cuda()
            xl = torch.from_numpy(L.local_slice(x).copy()).cuda()
            y_pc = prec.apply(xl).cpu().numpy()
            # 12 x 12 blocks: applied as explicit inverses, equal to the rank's factor solves
            assert prec.ginv is not None and prec.ginv_err <= 1e-13
            ginv, prec.ginv = prec.ginv, None
            y_fac = prec.apply(xl).cpu().numpy()
            prec.ginv = ginv
            assert relerr(y_pc, y_fac) < 1e-12
            bl = torch.from_numpy(L.local_slice(W.b).copy()).cuda()
            xs, rep = gmres_sharded(lambda v: op.apply(m, v), bl, B, C, apply_pinv=prec.apply, tol=1e-8,
                                    maxit=300, restart=15)
            results[rank] = (y_pc, xs.cpu().numpy(), rep.iterations)
        except Exception as e:  # surface worker failures in the main thread
            errors.append(e)
            comm.bar.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    plan = plan_operator(kern)
    p = build_two_level(kern, mt)
    y_pc = np.concatenate([r[0] for r in results])
    assert relerr(y_pc, p.apply(x)) < 1e-11
    assert relerr(y_pc, O.apply_prec(O.build_two_level(kern.tensors, dims, mt), x)) < 1e-10
    x1, rep1 = gmres(lambda v: apply_system(plan, W.m, v), W.b, apply_pinv=p.apply, tol=1e-8, maxit=300,
                     restart=15)
    xs = np.concatenate([r[1] for r in results])
    assert all(r[2] == results[0][2] for r in results)
    assert abs(results[0][2] - rep1.iterations) <= 2
    assert relerr(xs, x1) < 1e-6


@pytest.mark.parametrize("P", [1, 2, 3])
def test_sharded_blocked_loopback(P):
    """SURVEY 8(e) blocked: per-box line redistribution and sharded box
    preconditioners (1-level, reduced, 2-level boxes) on the CUDA backend
    reproduce the single-GPU BlockedPrec (identity outside the boxes)."""
    import threading

    import torch

    from paper_1903_07884_b200 import workloads
    from paper_1903_07884_b200.circulant import Box, build_blocked, partition_boxes
    from paper_1903_07884_b200.dist import CudaBackend, DistBlockedPrec, Layout
    from paper_1903_07884_b200.operator import padded_length

    W = workloads.small(30, 9, 4, delta=0.03e-6)
    kern = W.kernel()
    dims = W.grid.dims
    spec = [("a", (0, 30, 0, 4, 0, 4), "one-level"), ("b", (3, 25, 4, 9, 0, 2), "reduced-one-level"),
            ("c", (0, 17, 5, 9, 2, 4), "two-level")]
    part = partition_boxes(W.grid, [Box(lbl, *b) for lbl, b, _ in spec])
    levels = {lbl: lv for lbl, _, lv in spec}
    comm = LoopbackComm(P)
    rng = np.random.default_rng(17)
    x = random_field(rng, W.grid.n_unknowns)
    results = [None] * P
    errors = []

    def run(rank):
        try:
            torch.cuda.set_device(0)
            B, C = CudaBackend(), comm.view(rank)
            L = Layout(dims, P, rank, padded_length(dims[0]))
            prec = DistBlockedPrec(kern, W.pmap, part, levels, L, B, C, reduce_tol=0.3)
            xl = torch.from_numpy(L.local_slice(x).copy()).cuda()
            results[rank] = prec.apply(xl).cpu().numpy()
        except Exception as e:  # surface worker failures in the main thread
            errors.append(e)
            comm.bar.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    p = build_blocked(kern, W.pmap, part, levels, reduce_tol=0.3, cap_bytes=2 ** 40)
    assert relerr(np.concatenate(results), p.apply(x)) < 1e-11


@pytest.mark.parametrize("P", [2, 3])
def test_sharded_sector_factors_loopback(P):
    """The default CudaBackend path for symmetric kernels with P > 1 ranks:
    mirror orbits {k, nx-k} dealt whole to ranks, per-rank ragged sector
    factors, orbit transform + vx_prec1_solve_sec_rag on the received columns.
    Sharded P^-1 x and GMRES reproduce the single-GPU OneLevelPrec."""
    import threading

    import torch

    from paper_1903_07884_b200 import workloads
    from paper_1903_07884_b200.circulant import build_one_level
    from paper_1903_07884_b200.dist import CudaBackend, DistOneLevelPrec, DistOperator, Layout, gmres_sharded
    from paper_1903_07884_b200.operator import apply_system, padded_length, plan_operator
    from paper_1903_07884_b200.solver import gmres

    W = workloads.small(40, 10, 6, delta=0.03e-6)   # 3q = 180: 4 sectors of 45 rows (> one 32-row tile)
    kern = W.kernel()
    dims = W.grid.dims
    comm = LoopbackComm(P)
    rng = np.random.default_rng(23)
    x = random_field(rng, W.grid.n_unknowns)
    results = [None] * P
    errors = []

    def run(rank):
        try:
            torch.cuda.set_device(0)
            B, C = CudaBackend(), comm.view(rank)
            L = Layout(dims, P, rank, padded_length(dims[0]))
            op = DistOperator(kern, L, B, C)
            prec = DistOneLevelPrec(kern, W.mtilde(), L, B, C)
            assert prec.sec is not None, "sector path not taken"
            m = torch.from_numpy(W.m.reshape(-1).copy()).cuda()
            xl = torch.from_numpy(L.local_slice(x).copy()).cuda()
            y_pc = prec.apply(xl).cpu().numpy()
            bl = torch.from_numpy(L.local_slice(W.b).copy()).cuda()
            xs, rep = gmres_sharded(lambda v: op.apply(m, v), bl, B, C, apply_pinv=prec.apply, tol=1e-8,
                                    maxit=300, restart=15)
            results[rank] = (y_pc, xs.cpu().numpy(), rep.iterations, prec.bytes_local, prec.ginv is not None)
        except Exception as e:  # surface worker failures in the main thread
            errors.append(e)
            comm.bar.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    plan = plan_operator(kern)
    p = build_one_level(kern, W.mtilde())
    assert p._sec is not None
    y_pc = np.concatenate([r[0] for r in results])
    assert relerr(y_pc, p.apply(x)) < 1e-11
    x1, rep1 = gmres(lambda v: apply_system(plan, W.m, v), W.b, apply_pinv=p.apply, tol=1e-8, maxit=300,
                     restart=15)
    xs = np.concatenate([r[1] for r in results])
    assert len({r[2] for r in results}) == 1
    assert abs(results[0][2] - rep1.iterations) <= 2
    assert relerr(xs, x1) < 1e-6
    # every rank holds a share of the symmetry-reduced factors
    assert all(r[3] > 0 for r in results)
    # (symmetric inverses per rank when the blocks are eligible, else ragged LU sector factors)
    assert sum(r[3] for r in results) <= 1.5 * 16 * sum(d * d * c for d, c in p.stored_blocks)
    if p.factor_layout == "symmetric-inverse":
        assert all(r[4] for r in results), "ranks did not keep the symmetric inverses"
        assert sum(r[3] for r in results) <= 1.5 * p.factor_bytes_per_apply


def test_device_driven_step_equals_host_driven(group, monkeypatch):
    """The sharded solver's device-driven Arnoldi step (all-reduces on the stream, DGKS decision on
    the device, one Hessenberg read per step with lookahead, Z kept) reproduces the host-driven
    loop: same iteration count and DGKS pattern, residual history and solution to rounding."""
    import torch

    from paper_1903_07884_b200 import workloads
    from paper_1903_07884_b200.dist import CudaBackend, DistOneLevelPrec, DistOperator, Layout, _Comm, gmres_sharded
    from paper_1903_07884_b200.operator import padded_length

    W = workloads.small(60, 10, 6, delta=0.03e-6)
    kern = W.kernel()
    B, C = CudaBackend(), _Comm()
    L = Layout(W.grid.dims, 1, 0, padded_length(W.grid.dims[0]))
    op = DistOperator(kern, L, B, C)
    prec = DistOneLevelPrec(kern, W.mtilde(), L, B, C)
    m = torch.from_numpy(W.m.reshape(-1).copy()).cuda()
    b = torch.from_numpy(W.b.copy()).cuda()

    def solve():
        return gmres_sharded(lambda v: op.apply(m, v), b, B, C, apply_pinv=prec.apply, tol=1e-9, maxit=200,
                             restart=12)

    x1, r1 = solve()
    monkeypatch.setenv("VX_SHARD_DEVICE_STEP", "0")
    monkeypatch.setenv("VX_KEEP_Z", "0")
    x0, r0 = solve()
    assert r1.converged and r0.converged
    assert r1.iterations == r0.iterations and r1.iterations > 12          # at least one restart
    assert r1.reorth_passes == r0.reorth_passes
    assert np.allclose(r1.residuals, r0.residuals, rtol=1e-6, atol=1e-14)
    assert relerr(x1.cpu().numpy(), x0.cpu().numpy()) < 1e-9
