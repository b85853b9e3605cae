#!/usr/bin/env python
"""Benchmark: preconditioned-GMRES iterations/s and time-to-solution (complex128).

One *step* = one complete right-preconditioned GMRES solve (x0 = 0, tol 1e-5,
restart 50 (c0-c3) / 100 (c4), maxit 2000) of a BASELINE workload with the
operator plan and the preconditioner factors resident in HBM.  ``value`` =
total Arnoldi iterations / device-timed seconds over the K timed steps.

Default workload: BASELINE config c1 (5000 x 22 x 11 straight Si waveguide,
3.63 M unknowns, 1-level Chan circulant along x: 5000 LU blocks of 726^2,
42.17 GB of factors) -- configs[1], the configuration the metric is quoted on.
``--config`` selects c0/c1/c1r(reduced)/c2/c3/c4.

Extra keys: ``roofline`` for the dominant kernel (the factor-streaming block
solve, timed live with CUDA events on its launch stream), ``iteration_roofline``
for the whole iteration (SURVEY section 8(d) B_it), ``cpu_baseline`` (the CPU
oracle port timed on this host on a bounded sample), ``e2e`` (same metric
through the public API with host numpy buffers, copies inside the timed
region), ``clocks`` sampled by nvidia-smi during the timed region.

``--impl reference`` times the CPU reference path (oracle port of the
reference algorithm, scipy/LAPACK; the Python reference cannot travel to the
GPU box) on the same config and prints the same JSON line with impl=reference.
Under torchrun (N > 1) every rank solves its own replica (weak scaling); the
reference arm runs on rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

METRIC = "precond. GMRES iterations/s and time-to-solution (complex128) vs HBM roofline"
FALLBACK_HBM = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c1", choices=["c0", "c1", "c1r", "c2", "c3", "c4", "c4b"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--shard", action="store_true",
                    help="run the sharded (multi-GPU) code path even at N=1 (1-rank NCCL group)")
    ap.add_argument("--host-kernel", action="store_true",
                    help="assemble the generators on the host (numpy) instead of vx_assemble_green")
    ap.add_argument("--cpu-sample-blocks", type=int, default=24)
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent replicas instead of the sharded solve")
    ap.add_argument("--solve-classic", action="store_true",
                    help="use the non-pipelined block-solve kernel (A/B measurement)")
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", FALLBACK_HBM)), "measured"
    return FALLBACK_HBM, "fallback"


# ------------------------------------------------------------------ clocks
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index=0):
        self.idx = device_index
        self.proc = None
        self.f = None

    def start(self):
        if os.environ.get("VX_BENCH_CLOCKS", "1") == "0":   # A/B: host-jitter experiments only
            return
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
            # nvidia-smi's start-up (NVML init) can stall CUDA calls for tens of
            # ms: wait for its first sample so that happens before the timed region
            t0 = time.perf_counter()
            while time.perf_counter() - t0 < 3.0 and self.proc.poll() is None:
                if os.path.getsize(self.f.name) > 0:
                    break
                time.sleep(0.02)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable or disabled"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.flush()
        rows = [r.split(",") for r in Path(self.f.name).read_text().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            r = [c.strip() for c in r]
            if len(r) < 9:
                continue
            try:
                sm.append(float(r[1]))
                smax = float(r[2])
            except ValueError:
                continue
            for nm, v in zip(names, r[5:9]):
                if v.lower() in ("active", "1"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ dist helpers
def dist_setup(torch, force=False):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world == 1 and force:
        # --shard on one GPU: a 1-rank NCCL group drives the sharded code path
        import socket

        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if "MASTER_PORT" not in os.environ:
            sk = socket.socket()
            sk.bind(("127.0.0.1", 0))
            os.environ["MASTER_PORT"] = str(sk.getsockname()[1])
            sk.close()
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    elif world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank, local


def barrier(torch, world):
    if world > 1:
        torch.distributed.barrier()


def reduce_max(torch, world, v):
    if world == 1:
        return v
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(torch, world, v):
    if world == 1:
        return v
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.SUM)
    return float(t.item())


# --------------------------------------------------------- byte accounting
def block_sizes(W):
    """(list of stored block dims, number of stored blocks) per SURVEY 8(d)."""
    nx, ny, nz = W.grid.dims
    k = W.prec["kind"]
    if k == "one-level":
        return [(3 * ny * nz, nx)]
    if k == "two-level":
        return [(3 * nz, nx * ny)]
    if k == "blocked":
        out = []
        for (x0, x1, y0, y1, z0, z1), lvl in zip(W.prec["boxes"], W.prec["levels"]):
            if lvl == "two-level":
                out.append((3 * (z1 - z0), (x1 - x0) * (y1 - y0)))
            else:
                out.append((3 * (y1 - y0) * (z1 - z0), x1 - x0))
        return out
    raise ValueError(k)


def iteration_bytes(W, stored_blocks, restart_eff):
    """B_it = B_mv + B_pc + B_ar."""
    N = W.grid.n_voxels
    vec = 48 * N
    b_mv = 2 * vec + 16 * N + 6 * 16 * 8 * N
    b_pc = 2 * vec + 16 * sum(n * n * cnt for n, cnt in stored_blocks)
    b_ar = vec * (restart_eff + 5)
    return b_mv + b_pc + b_ar, b_mv, b_pc, b_ar


# ------------------------------------------------------------ CPU baseline
def cpu_iteration_sample(W, kern, m, sample_blocks, mean_j, spectra=None):
    """Seconds of one preconditioned GMRES iteration of the CPU oracle port on a
    bounded sample: full matvec, prec apply with `sample_blocks` LU solves scaled
    to all blocks, MGS over mean_j basis vectors.  Returns (sec, cores, desc)."""
    import scipy.fft
    from scipy.linalg import lu_factor, lu_solve

    import voxvie_oracle as O

    cores = len(os.sched_getaffinity(0))
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    dims = W.grid.dims
    nx, ny, nz = dims
    rng = np.random.default_rng(20240811)
    n = W.grid.n_unknowns
    x = rng.normal(size=n) + 1j * rng.normal(size=n)
    if spectra is None:
        spectra = O.plan_spectra(kern.tensors, dims, workers=cores)
    t0 = time.perf_counter()
    O.apply_system(spectra, dims, m, x, workers=cores)
    t_mv = time.perf_counter() - t0
    kind = W.prec["kind"]
    from paper_1903_07884_b200.grid import PermittivityMap, VoxelGrid, homogenize

    def box_mtilde(box, level):
        strat = W.prec.get("homogenization") or ("mode" if level == "two-level" else "real_mean_x")
        if box is None:
            return homogenize(W.pmap, strat)
        x0, x1, y0, y1, z0, z1 = box
        sub = VoxelGrid(x1 - x0, y1 - y0, z1 - z0, W.grid.delta)
        return homogenize(PermittivityMap(sub, W.pmap.eps_r[z0:z1, y0:y1, x0:x1]), strat)

    def one_level_box(sub, sdims, mt):
        m_yz = O.coerce_mtilde(sdims, mt)
        bx, by, bz = sdims
        lam = O.chan_x_spectra(sub)
        ks = np.linspace(0, bx - 1, min(sample_blocks, bx)).astype(int)
        facs = [lu_factor(O.unfold_block_yz(lam[:, :, :, k], m_yz), check_finite=False) for k in ks]
        xf = rng.normal(size=(3, bz, by, bx)) + 0j
        t0 = time.perf_counter()
        spec = scipy.fft.fft(xf, axis=3)
        scipy.fft.ifft(spec, axis=3)
        t_fft = time.perf_counter() - t0
        t0 = time.perf_counter()
        for k, f in zip(ks, facs):
            lu_solve(f, np.ascontiguousarray(spec[:, :, :, k]).reshape(-1, 1), check_finite=False)
        return t_fft + (time.perf_counter() - t0) * bx / len(ks), len(ks), bx

    def two_level_box(sub, sdims, mt):
        bx, by, bz = sdims
        lam2 = scipy.fft.fftn(O.chan_along_axis(O.chan_along_axis(sub, 3), 2), axes=(2, 3))
        m_z = np.asarray(mt)[:, 0, 0]
        xf = rng.normal(size=(3, bz, by, bx)) + 0j
        t0 = time.perf_counter()
        spec = scipy.fft.fftn(xf, axes=(2, 3))
        scipy.fft.ifftn(spec, axes=(2, 3))
        t_fft = time.perf_counter() - t0
        S = min(sample_blocks * 40, bx * by)
        idx = np.linspace(0, bx * by - 1, S).astype(int)
        facs = [lu_factor(O.unfold_block_z(lam2[:, :, i // bx, i % bx], m_z), check_finite=False) for i in idx]
        t0 = time.perf_counter()
        for i, f in zip(idx, facs):
            lu_solve(f, np.ascontiguousarray(spec[:, :, i // bx, i % bx]).reshape(-1, 1), check_finite=False)
        return t_fft + (time.perf_counter() - t0) * bx * by / S, S, bx * by

    if kind == "blocked":
        boxes, levels = W.prec["boxes"], W.prec["levels"]
    else:
        boxes, levels = [None], [kind]
    t_pc = 0.0
    parts_desc = []
    for box, lvl in zip(boxes, levels):
        sub, sdims = O.slice_kernel(kern.tensors, dims, box or (0, nx, 0, ny, 0, nz))
        mt = box_mtilde(box, lvl)
        t, ns, ntot = (two_level_box if lvl == "two-level" else one_level_box)(sub, sdims, mt)
        t_pc += t
        parts_desc.append(f"{ns} of {ntot} {lvl} lu_solve calls")
    desc = (f"oracle port (scipy.fft + LAPACK zgetrs as the reference) on {W.name}: full matvec "
            f"(fftn workers={cores}), preconditioner DFTs of the full field, "
            + "; ".join(parts_desc) + f" timed and scaled to all blocks, MGS over {mean_j} vectors")
    V = [rng.normal(size=n) + 1j * rng.normal(size=n) for _ in range(max(1, mean_j))]
    w = x.copy()
    t0 = time.perf_counter()
    for v in V:
        h = np.vdot(v, w)
        w -= h * v
    np.linalg.norm(w)
    t_ar = time.perf_counter() - t0
    return t_mv + t_pc + t_ar, cores, desc, dict(matvec_s=t_mv, prec_s=t_pc, arnoldi_s=t_ar)


def bench_config(name, W, mode):
    """The `config` object of the JSON line: identical on both arms (the driver
    compares them), so it only names the workload and the step definition."""
    return {"workload": f"{name}: {W.grid.nx}x{W.grid.ny}x{W.grid.nz} {W.prec['kind']}",
            "unknowns": W.grid.n_unknowns, "restart": W.restart, "tol": W.tol,
            "step": "one full preconditioned GMRES solve (x0=0); value = Arnoldi iterations / second",
            "l2": "inputs larger than L2 (the preconditioner factor stream of every iteration is GBs >> 126 MB)",
            "parallelism": mode}


# -------------------------------------------------------------- our arm
def build_prec(W, kern):
    from paper_1903_07884_b200 import circulant as C

    kind = W.prec["kind"]
    big = 2 ** 62
    if kind == "one-level":
        return C.build_one_level(kern, W.mtilde(), cap_bytes=big)
    if kind == "reduced-one-level":
        return C.build_reduced_one_level(kern, W.mtilde(), W.prec.get("tol", 1e-3), cap_bytes=big)
    if kind == "two-level":
        return C.build_two_level(kern, W.mtilde(), cap_bytes=big)
    if kind == "blocked":
        boxes = [C.Box(lbl, *b) for lbl, b in zip(W.prec["labels"], W.prec["boxes"])]
        part = C.partition_boxes(W.grid, boxes)
        levels = dict(zip(W.prec["labels"], W.prec["levels"]))
        homog = ({lbl: W.prec["homogenization"] for lbl in W.prec["labels"]}
                 if W.prec.get("homogenization") else None)   # None: per-level defaults
        return C.build_blocked(kern, W.pmap, part, levels, homog=homog, cap_bytes=big)
    raise ValueError(kind)


def solve_kernel_traffic(name, W, world, layout=None):
    """(kernel name, DRAM bytes per launch) of the dominant block-solve kernel:
    the name from the factor layout in use, the traffic from the committed ncu
    capture (dram__bytes_read.sum + dram__bytes_write.sum of one launch,
    profiles/r01_solve_traffic.json) when it was taken on this workload."""
    import os
    ragged = os.environ.get("VX_RAGGED", "1") != "0" and W.prec["kind"] in ("one-level", "blocked")
    kname = "lu_solve_rag_kernel<2>" if ragged else "lu_solve_pipe_kernel<2>"
    if W.prec["kind"] == "two-level":
        kname = ("lu_apply_small_inv_kernel<%d>" % (3 * W.grid.nz)) if layout == "inverse" else "lu_solve_small_kernel"
    elif W.prec["kind"] == "reduced-one-level":
        kname = "lu_solve_rag_kernel<2> + rep_gemm_kernel"
    if layout == "symmetric-inverse":
        kname = "symv2_inv_kernel<2>" + (" + rep_gemm_kernel" if W.prec["kind"] == "reduced-one-level" else "")
        return kname, _committed_traffic(name, kname, world)
    if layout == "symmetric":
        kname = "lu_solve_sym_kernel<2>" + (" + rep_gemm_kernel" if W.prec["kind"] == "reduced-one-level" else "")
    return kname, _committed_traffic(name, kname, world)


def _committed_traffic(name, kname, world):
    if world != 1:
        return None
    for fn in ("r02_solve_traffic.json", "r01_solve_traffic.json"):
        f = ROOT / "profiles" / fn
        if f.exists():
            ent = json.loads(f.read_text()).get(name)
            if ent and ent.get("kernel") == kname:
                return int(ent["dram_bytes_per_launch"])
    return None


def stored_blocks_of(W, prec):
    """(block dim, factors actually stored and streamed once per apply): with
    mirror sharing (parity-symmetric kernels) one stored factor serves the
    blocks k and n-k, so this is about half the reference's block count."""
    precs = prec.box_precs if W.prec["kind"] == "blocked" else [prec]
    return [blk for p in precs for blk in p.stored_blocks]


def run_ours(args):
    import torch

    from paper_1903_07884_b200 import _native as nv
    from paper_1903_07884_b200 import workloads
    from paper_1903_07884_b200.operator import apply_system, plan_operator
    from paper_1903_07884_b200.solver import gmres

    world, rank, local = dist_setup(torch, force=args.shard)
    nv.load()
    nv.query("vx_solve_variant", 1 if args.solve_classic else 0)
    name = args.config
    W = workloads.make(name)
    assembly_s = None
    if args.host_kernel:
        kern = W.kernel()
    else:
        # generators assembled on the device (vx_assemble_green): warm call,
        # then one timed with CUDA events
        from paper_1903_07884_b200.kernel import assemble_kernel_device

        kern = assemble_kernel_device(W.grid, W.physics.k0)
        del kern
        torch.cuda.synchronize()
        ev_k0, ev_k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tk = time.perf_counter()
        ev_k0.record()
        kern = assemble_kernel_device(W.grid, W.physics.k0)
        ev_k1.record()
        torch.cuda.synchronize()
        assembly_s = {"device_s": ev_k0.elapsed_time(ev_k1) / 1e3, "wall_s": time.perf_counter() - tk}
        W._kernel = kern
    m_host = W.m
    b_host = W.b
    torch.cuda.synchronize()
    # N > 1: every config runs ONE sharded solve across all ranks (strong
    # scaling: line-sharded vectors, k-sharded factors, NCCL all-to-all; the
    # blocked config redistributes each box's lines to the box's own layout);
    # --replicas runs one independent solve per rank instead (weak scaling).
    sharded = (world > 1 or args.shard) and not args.replicas
    mode = "sharded" if sharded else ("replicas" if world > 1 else "single-gpu")

    # ---- setup (time-to-solution part 1): plan + preconditioner build
    m_dev = torch.from_numpy(np.ascontiguousarray(m_host).reshape(-1)).cuda()
    t0 = time.perf_counter()
    ev_a, ev_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if sharded:
        from paper_1903_07884_b200.dist import (CudaBackend, DistOneLevelPrec, DistOperator, DistTwoLevelPrec,
                                                Layout, _Comm, gmres_sharded)
        from paper_1903_07884_b200.operator import padded_length

        Bk, Cm = CudaBackend(), _Comm()
        L = Layout(W.grid.dims, world, rank, padded_length(W.grid.nx))
        dop = DistOperator(kern, L, Bk, Cm)
        torch.cuda.synchronize()
        plan_s = time.perf_counter() - t0
        ptol = W.prec.get("tol") if W.prec["kind"] == "reduced-one-level" else None

        def dist_prec():
            if W.prec["kind"] == "two-level":
                return DistTwoLevelPrec(kern, W.mtilde(), L, Bk, Cm)
            if W.prec["kind"] == "blocked":
                from paper_1903_07884_b200 import circulant as CC
                from paper_1903_07884_b200.dist import DistBlockedPrec

                boxes = [CC.Box(lbl, *b) for lbl, b in zip(W.prec["labels"], W.prec["boxes"])]
                homog = ({lbl: W.prec["homogenization"] for lbl in W.prec["labels"]}
                         if W.prec.get("homogenization") else None)
                return DistBlockedPrec(kern, W.pmap, CC.partition_boxes(W.grid, boxes),
                                       dict(zip(W.prec["labels"], W.prec["levels"])), L, Bk, Cm, homog=homog)
            return DistOneLevelPrec(kern, W.mtilde(), L, Bk, Cm, tol=ptol)

        prec = dist_prec()   # warm build
        del prec
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        ev_a.record()
        prec = dist_prec()
        ev_b.record()
        torch.cuda.synchronize()
        build_s = ev_a.elapsed_time(ev_b) / 1e3
        build_cached_s = None
        b_dev = torch.from_numpy(np.ascontiguousarray(L.local_slice(b_host))).cuda()
        A = lambda v: dop.apply(m_dev, v)  # noqa: E731

        def solve(b):
            return gmres_sharded(A, b, Bk, Cm, apply_pinv=prec.apply, tol=W.tol, maxit=W.maxit,
                                 restart=W.restart)
    else:
        plan = plan_operator(kern)
        torch.cuda.synchronize()
        plan_s = time.perf_counter() - t0
        # warm build first (module load, FFT tables, kernel attributes), then the
        # timed build of the factors that the solves use
        prec = build_prec(W, kern)
        del prec
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        ev_a.record()
        prec = build_prec(W, kern)
        ev_b.record()
        torch.cuda.synchronize()
        build_s = ev_a.elapsed_time(ev_b) / 1e3
        # the same build with the allocator's blocks still cached (a process that rebuilds for a new
        # medium): build_s above pays a cudaMalloc for every buffer after empty_cache()
        del prec
        torch.cuda.synchronize()
        ev_a.record()
        prec = build_prec(W, kern)
        ev_b.record()
        torch.cuda.synchronize()
        build_cached_s = ev_a.elapsed_time(ev_b) / 1e3
        b_dev = torch.from_numpy(b_host.copy()).cuda()
        A = lambda v: apply_system(plan, m_dev, v)  # noqa: E731

        def solve(b):
            return gmres(A, b, apply_pinv=prec.apply, tol=W.tol, maxit=W.maxit, restart=W.restart)

    # setup objects (torch / numpy / scipy modules, the workload) move to the
    # GC's permanent generation, so a collection triggered between solves
    # scans only what the solves allocate (a full collection otherwise walks
    # ~10^6 objects: 50-100 ms stalls in the timed loops)
    import gc

    gc.collect()
    gc.freeze()
    # clock sampler runs from before the warm-up until after the timed region
    clocks = Clocks(local)
    clocks.start()
    for _ in range(args.warmup):
        _, rep = solve(b_dev)
    torch.cuda.synchronize()
    # the warm-up imports and allocates lazily (torch / numpy submodules, workspaces): move those
    # objects to the permanent generation too, or the first full collection after a solve walks
    # them (8-60 ms stalls between timed solves, tools/stall_probe.py)
    gc.collect()
    gc.freeze()

    # ---- timed region (device resident)
    barrier(torch, world)
    torch.cuda.synchronize()
    nv.timing_enable(True)
    for sp in ("prec_solve", "op_apply", "prec_apply", "arnoldi_step"):
        nv.timing_read(sp)
    l0 = nv.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev_steps = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    trace = os.environ.get("VX_BENCH_TRACE", "0") != "0"   # stderr: where a slow solve spent its host time
    if trace:
        from paper_1903_07884_b200 import solver as _solver
        _solver.TRACE = []
    e0.record()
    its = 0
    reports = []
    for k in range(args.steps):
        if trace:
            n0, tw = len(_solver.TRACE), time.perf_counter()
        x, rep = solve(b_dev)
        its += rep.iterations
        reports.append(rep)
        ev_steps[k].record()
        if trace:
            ph = [e[1] for e in _solver.TRACE[n0:] if e[0] == "phases"]
            tr = [e for e in _solver.TRACE[n0:] if e[0] != "phases"]
            print(f"[trace] phases {ph}", file=sys.stderr)
            print(f"[trace] solve {k}: wall {(time.perf_counter() - tw) * 1e3:.1f} ms, in Arnoldi loop "
                  f"{sum(a + c for _, a, c in tr) * 1e3:.1f} ms (launching {sum(a for _, a, _ in tr) * 1e3:.1f}, "
                  f"max wait {max(c for _, _, c in tr) * 1e3:.2f}, max launch {max(a for _, a, _ in tr) * 1e3:.2f}), "
                  f"gc {gc.get_count()}", file=sys.stderr)
    e1.record()
    torch.cuda.synchronize()
    if trace:
        _solver.TRACE = None
    step_ms = [round(e0.elapsed_time(ev_steps[0]), 2)] + [round(ev_steps[k - 1].elapsed_time(ev_steps[k]), 2)
                                                           for k in range(1, args.steps)]
    launches = nv.launch_count() - l0
    clk = clocks.stop()
    barrier(torch, world)
    t_local = e0.elapsed_time(e1) / 1e3
    spans = {sp: nv.timing_read(sp) for sp in ("prec_solve", "op_apply", "prec_apply", "arnoldi_step")}
    nv.timing_enable(False)
    t_max = reduce_max(torch, world, t_local)
    its_all = its if sharded else reduce_sum(torch, world, its)
    value = its_all / t_max
    ms_per_step = t_max / args.steps * 1e3
    solve_s = t_local / args.steps

    # ---- roofline of the dominant kernel (factor-streaming block solve)
    peak, peak_kind = peaks()
    if sharded:
        pl = prec.box_precs if W.prec["kind"] == "blocked" else [prec]
        stored_global = [b for q in pl for b in (getattr(q, "stored_global", None) or [(q.n, q.n_stored_global)])]
        stored = (getattr(pl[0], "stored_local", None)       # per launch: first box / whole prec
                  or [(pl[0].n, pl[0].bytes_local // (16 * pl[0].n ** 2))])
        nvec = prec.boxes[0]["n_loc"] if W.prec["kind"] == "blocked" else W.grid.n_unknowns // world
    else:
        stored = stored_global = stored_blocks_of(W, prec)
        nvec = W.grid.n_unknowns
        if W.prec["kind"] == "blocked":   # one solve launch per box: per-launch bytes of one box
            x0, x1, y0, y1, z0, z1 = W.prec["boxes"][0]
            stored = list(prec.box_precs[0].stored_blocks)   # every (sector) block of box 0
            nvec = 3 * (x1 - x0) * (y1 - y0) * (z1 - z0)
    sol_ms, sol_n = spans["prec_solve"]
    solve_bytes = 16 * sum(n * n * c for n, c in stored) + 2 * 16 * nvec
    # compulsory factor bytes: per launch (one box of the blocked scheme) and per iteration (all boxes)
    fb = fb_launch = None
    layout = getattr(prec, "factor_layout", None)
    if not sharded:
        if W.prec["kind"] == "blocked":
            per_box = [getattr(q, "factor_bytes_per_apply", None) for q in prec.box_precs]
            if all(v is not None for v in per_box):
                fb, fb_launch = sum(per_box), per_box[0]
            layout = getattr(prec.box_precs[0], "factor_layout", None)
        else:
            fb = fb_launch = getattr(prec, "factor_bytes_per_apply", None)
    elif getattr(pl[0], "ginv", None) is not None:
        # sharded symmetric inverses: this rank's stored triangles per launch; every rank's per iteration
        layout = "inverse" if W.prec["kind"] == "two-level" else "symmetric-inverse"
        fb_launch = int(pl[0].bytes_local)
        loc = sum(int(q.bytes_local) for q in pl)
        fb = int(reduce_sum(torch, world, loc)) if world > 1 else loc
    if fb_launch is not None:   # symmetric layouts: the stored lower triangles, read once per apply
        solve_bytes = fb_launch + 2 * 16 * nvec
    roof = None
    if sol_n:
        avg = sol_ms / sol_n / 1e3
        ach = solve_bytes / avg / 1e9
        kname, traffic = solve_kernel_traffic(name, W, world, layout)
        if sharded:
            traffic = None   # the committed ncu captures are of the single-GPU launches
        roof = {"kernel": kname + " (prec_solve span)", "bound": "hbm", "achieved": ach,
                "peak": peak, "unit": "GB/s", "frac": ach / peak, "peak_source": peak_kind,
                "traffic": traffic, "bytes_per_launch": solve_bytes, "avg_launch_ms": avg * 1e3,
                "launches": sol_n}
    its_per_solve = its / args.steps
    restart_eff = min(W.restart, its_per_solve)
    b_it, b_mv, b_pc, b_ar = iteration_bytes(W, stored_global, restart_eff)
    b_pc = 2 * 48 * W.grid.n_voxels + (fb if fb is not None else 16 * sum(n * n * c for n, c in stored_global))
    # the reference's DGKS re-orthogonalisation (solver.py:69-73) is a second sweep over the basis in
    # the steps where its criterion fires: count it for those steps (SURVEY's B_ar is the first sweep)
    reorth = sum(getattr(r, "reorth_passes", 0) for r in reports)
    f_reorth = reorth / max(1, its)
    b_ar_first = b_ar
    b_ar = b_ar + f_reorth * 48 * W.grid.n_voxels * (restart_eff + 3)
    b_it = b_mv + b_pc + b_ar
    it_roof = {"bytes_per_iteration": b_it, "B_mv": b_mv, "B_pc": b_pc, "B_ar": b_ar,
               "B_ar_first_sweep": b_ar_first, "reorth_fraction": f_reorth,
               "achieved": b_it * its_all / t_max / 1e9, "peak": peak * (world if sharded else 1),
               "unit": "GB/s", "frac": b_it * its_all / t_max / 1e9 / (peak * (world if sharded else 1))}
    breakdown = {sp: {"ms_total": v[0], "launches": v[1]} for sp, v in spans.items()}

    # ---- e2e through the public API with host numpy buffers
    e2e = None
    if not args.no_e2e:
        # m is a writeable host array: the API uploads it once per solve (its
        # device copy lives only for the solve's scope, operator._medium_in)
        m_step = m_host

        def e2e_step():
            if sharded:
                # host buffers through the sharded API: local slice of b in, local x out
                m_d = torch.from_numpy(m_step.reshape(-1)).cuda()
                b_d = torch.from_numpy(np.ascontiguousarray(L.local_slice(b_host))).cuda()
                xs, rep = gmres_sharded(lambda v: dop.apply(m_d, v), b_d, Bk, Cm, apply_pinv=prec.apply,
                                        tol=W.tol, maxit=W.maxit, restart=W.restart)
                x_h = nv.to_host(xs)
            else:
                x_h, rep = gmres(lambda v: apply_system(plan, m_step, v), b_host,
                                 apply_pinv=prec.apply, tol=W.tol, maxit=W.maxit, restart=W.restart)
            return x_h, rep

        # untimed e2e warm-up in the timed loop's own pattern (the previous
        # result stays alive while the next is produced): the library's pooled
        # pinned result blocks and upload ring are allocated here, then recycled
        x_h = None
        for _ in range(max(2, min(3, args.warmup))):
            x_h, _rep = e2e_step()
        torch.cuda.synchronize()
        gc.collect()
        gc.freeze()
        barrier(torch, world)
        t0 = time.perf_counter()
        its_e = 0
        step_wall = []
        e2e_steps = max(args.steps, 6)   # a few more solves: one host stall weighs less
        for _ in range(e2e_steps):
            ts = time.perf_counter()
            x_h, rep = e2e_step()
            its_e += rep.iterations
            step_wall.append((time.perf_counter() - ts) * 1e3)
        torch.cuda.synchronize()
        te = reduce_max(torch, world, time.perf_counter() - t0)
        its_e_all = its_e if sharded else reduce_sum(torch, world, its_e)
        nb_loc = b_host.nbytes // world if sharded else b_host.nbytes
        e2e = {"value": its_e_all / te, "unit": "it/s", "h2d_bytes_per_step": int(nb_loc + m_host.nbytes),
               "d2h_bytes_per_step": int(nb_loc), "ms_per_step": te / e2e_steps * 1e3, "steps": e2e_steps,
               "step_wall_ms": [round(v, 2) for v in step_wall],
               "tts_s": build_s + te / e2e_steps,
               "note": "numpy b and m in (threaded pinned-ring upload, vx_h2d_staged), numpy x out (pooled pinned block); plan+factors resident (setup)"}

    # ---- CPU baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        mean_j = int(max(1, min(W.restart, its_per_solve) // 2))
        sec, cores, desc, parts = cpu_iteration_sample(W, kern, m_host, args.cpu_sample_blocks, mean_j,
                                                       spectra=plan.spectra if (not sharded and plan.padded_shape
                                                                                == tuple(2 * d for d in W.grid.shape))
                                                       else None)
        cpu = {"value": 1.0 / sec, "unit": "it/s", "cores": cores, "kind": "port", "sample": desc,
               "seconds_per_iteration": sec, **parts,
               "tts_s_estimate": None}

    line = {
        "metric": METRIC,
        "value": value,
        "unit": "it/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": "strong" if sharded else "weak",
        "vs_baseline": None,
        "dtype": "c128",
        "data": "synthetic (BASELINE workload, interpretation B, deterministic)",
        "config": bench_config(name, W, mode),
        "factor_stream_gb": solve_bytes / 1e9,
        "iterations_per_solve": its_per_solve,
        "step_ms": step_ms,
        "build_s": build_s,
        "build_cached_s": build_cached_s,
        "build_note": "warm build (second in process): Chan + x-DFT spectra, proxies, unfold + LU of all blocks",
        "plan_s": plan_s,
        "assembly": assembly_s,
        "solve_s": solve_s,
        "tts_s": build_s + solve_s,
        "tts_cold_s": ((assembly_s["wall_s"] if assembly_s else 0.0) + plan_s + build_s + solve_s),
        "tts_cold_note": "generator assembly (device) + operator plan (first, cold) + factor build + solve",
        "true_residual": reports[-1].true_residual,
        "roofline": roof,
        "iteration_roofline": it_roof,
        "breakdown": breakdown,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk,
        "cpu_baseline": cpu,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1 or args.shard:
        torch.distributed.destroy_process_group()


# --------------------------------------------------------- reference arm
def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_1903_07884_b200 import workloads

    import voxvie_oracle as O

    W = workloads.make(args.config)
    kern = W.kernel()
    m = W.m
    cores = len(os.sched_getaffinity(0))
    spectra = O.plan_spectra(kern.tensors, W.grid.dims, workers=cores)
    mean_j = 10
    for _ in range(args.warmup):
        cpu_iteration_sample(W, kern, m, 4, 2, spectra=spectra)
    tot = 0.0
    desc = ""
    t_wall = time.perf_counter()
    for _ in range(args.steps):
        sec, cores, desc, _ = cpu_iteration_sample(W, kern, m, args.cpu_sample_blocks, mean_j, spectra=spectra)
        tot += sec
    t_wall = time.perf_counter() - t_wall
    value = args.steps / tot
    sharded = (world > 1 or args.shard) and not args.replicas   # as run_ours names its mode
    mode = "sharded" if sharded else ("replicas" if world > 1 else "single-gpu")
    line = {
        "metric": METRIC, "impl": "reference", "value": value, "unit": "it/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        # wall time of one timed step (a bounded sample of one CPU iteration); the
        # sampled block solves are scaled to all blocks in `value`
        "ms_per_step": t_wall / args.steps * 1e3,
        "seconds_per_iteration": tot / args.steps,
        "higher_is_better": True, "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic (BASELINE workload, interpretation B, deterministic)",
        "config": bench_config(args.config, W, mode),
        "reference_step": "each timed step samples ONE preconditioned GMRES iteration of the CPU path "
                          "(value = 1 / its extrapolated seconds); a full solve is iterations_per_solve of them",
        "cpu_baseline": {"value": value, "unit": "it/s", "cores": cores, "kind": "port", "sample": desc},
        "e2e": {"value": value, "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
