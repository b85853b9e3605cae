"""Host-side profile of a warm 1-level build: wall time per phase (cProfile,
cumulative), usage: python tools/prof_build_host.py [c1]"""
import cProfile
import pstats
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1903_07884_b200 import workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
W = workloads.make(name)
kern = W.kernel()
p = bench.build_prec(W, kern)
torch.cuda.synchronize()
del p
t0 = time.perf_counter()
pr = cProfile.Profile()
pr.enable()
p = bench.build_prec(W, kern)
torch.cuda.synchronize()
pr.disable()
print(f"warm build {time.perf_counter() - t0:.4f} s")
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
