"""Graph-mode solve time of config 2 (200 iterations) for library variants."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_26659_b200 import _lib, workloads as W
_lib.LIB_PATH = sys.argv[1]
import paper_2605_26659_b200 as fb
x, y, u, v, eps = W.config2()
bs = fb.BatchSolver1D([x], [y], [u], [v], [eps])
for _ in range(2):
    bs.solve(200, 0.0, True, 200.0)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    bs.solve(200, 0.0, True, 200.0)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
print(os.path.basename(sys.argv[1]), "solve %.2f ms  (%.1f us/iteration, %.3e pts*it/s)" % (ms, ms * 5, x.size * 200 / ms * 1e3))
