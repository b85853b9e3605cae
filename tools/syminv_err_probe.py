import sys
sys.path.insert(0, '/root/repo')
import bench
from paper_1903_07884_b200 import workloads
for name in sys.argv[1:]:
    W = workloads.make(name)
    kern = W.kernel()
    p = bench.build_prec(W, kern)
    ps = p.box_precs if hasattr(p, "box_precs") else [p]
    print(name, [(q.factor_layout, getattr(q, "_syminv_err", None)) for q in ps])
