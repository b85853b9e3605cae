import os, sys, time
import numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_1903_07884_b200 import _native as nv
n = 3630000
src = (np.random.default_rng(0).normal(size=n) + 0j)
pin = torch.empty(n, dtype=torch.complex128).pin_memory()
dst = torch.empty(n, dtype=torch.complex128, device="cuda")
print("cores", os.cpu_count(), "h2d threads", nv.query("vx_h2d_threads") if hasattr(nv, "query") else "?")
def tm(f, reps=10):
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append((time.perf_counter() - t0) * 1e3)
    return min(ts), sorted(ts)[len(ts)//2]
print("pinned->dev 58MB ms (min, med):", tm(lambda: dst.copy_(pin, non_blocking=True)))
print("dev->pinned 58MB ms:", tm(lambda: pin.copy_(dst, non_blocking=True)))
pn = pin.numpy()
print("host memcpy np.copyto pageable->pinned ms:", tm(lambda: np.copyto(pn, src)))
print("staged upload ms:", tm(lambda: nv.call("vx_h2d_staged", dst.data_ptr(), src.ctypes.data, src.nbytes, nv.stream_ptr())))
print("torch pageable .cuda() ms:", tm(lambda: dst.copy_(torch.from_numpy(src))))
