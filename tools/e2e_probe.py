"""Where does the host-buffer (e2e) solve spend its time?  usage: e2e_probe.py [c1]"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1903_07884_b200 import workloads  # noqa: E402
from paper_1903_07884_b200.circulant import build_one_level  # noqa: E402
from paper_1903_07884_b200.operator import apply_system, plan_operator  # noqa: E402
from paper_1903_07884_b200.solver import gmres  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
W = workloads.make(name)
kern = W.kernel()
plan = plan_operator(kern)
prec = build_one_level(kern, W.mtilde(), cap_bytes=2 ** 62)
m_host, b_host = W.m, W.b
m_dev = torch.from_numpy(m_host.reshape(-1).copy()).cuda()
b_dev = torch.from_numpy(b_host.copy()).cuda()


def timed(label, fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    print(f"{label:40s} {(time.perf_counter() - t0) / reps * 1e3:8.2f} ms", flush=True)


timed("device solve", lambda: gmres(lambda v: apply_system(plan, m_dev, v), b_dev, apply_pinv=prec.apply,
                                    tol=W.tol, maxit=W.maxit, restart=W.restart))
timed("host b + host m solve", lambda: gmres(lambda v: apply_system(plan, m_host, v), b_host, apply_pinv=prec.apply,
                                             tol=W.tol, maxit=W.maxit, restart=W.restart))
timed("H2D b (pageable)", lambda: torch.from_numpy(b_host).cuda())
pin = torch.from_numpy(b_host.copy()).pin_memory()
timed("H2D b (pinned)", lambda: pin.cuda(non_blocking=True))
timed("D2H x", lambda: b_dev.cpu().numpy())
timed("apply_system host m", lambda: apply_system(plan, m_host, b_dev))
timed("apply_system dev m", lambda: apply_system(plan, m_dev, b_dev))
timed("prec.apply dev", lambda: prec.apply(b_dev))
from paper_1903_07884_b200 import _native as nv  # noqa: E402

print("h2d threads", nv.query("vx_h2d_threads"))
timed("H2D b (staged ring)", lambda: nv.device_c128(b_host))
timed("H2D m (staged ring)", lambda: nv.device_c128(m_host))
timed("H2D m (pageable)", lambda: torch.from_numpy(m_host).cuda())
timed("D2H x (to_host pinned)", lambda: nv.to_host(b_dev))
