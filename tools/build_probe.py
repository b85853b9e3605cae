import sys, time
sys.path.insert(0, "/root/repo")
import torch
import bench
from paper_1903_07884_b200 import workloads, solver
name = sys.argv[1] if len(sys.argv) > 1 else "c1r"
W = workloads.make(name)
kern = W.kernel()
for i in range(4):
    p = bench.build_prec(W, kern)
    del p
    torch.cuda.synchronize()
    if i % 2 == 1:
        torch.cuda.empty_cache()
    t0 = time.perf_counter()
    p = bench.build_prec(W, kern)
    torch.cuda.synchronize()
    print(name, "empty_cache" if i % 2 == 1 else "cached", round((time.perf_counter() - t0) * 1e3, 2), "ms")
    del p
