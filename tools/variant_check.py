"""Correctness of a library variant: config 1 (500 it, stabilized) vs the C oracle,
then the config-2 solve time."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2605_26659_b200 import _lib, workloads as W
_lib.LIB_PATH = sys.argv[1]
import paper_2605_26659_b200 as fb
from oracle import oracle as O
x, y, u, v, eps = W.config1()
sol = fb.sinkhorn_1d(fb.Mesh1D(x), fb.Mesh1D(y), fb.Measure(u), fb.Measure(v),
                     fb.SolverConfig(epsilon=eps, itr_max=500, tol=0.0, stabilize=True))
ref = O.sinkhorn_1d(x, y, u, v, eps, 500, 0.0, True)
rel = lambda a, b: float(np.max(np.abs(a - b)) / np.max(np.abs(b)))
print("config1 phi rel %.2e psi rel %.2e absorbs %s/%s" % (rel(sol.phi, ref["phi"]), rel(sol.psi, ref["psi"]),
      list(sol.absorb_iterations), list(ref["absorb_its"])))
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
