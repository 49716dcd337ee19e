"""Bitwise run-to-run reproducibility of the device loop (config 2, 1D batch, 2D)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2605_26659_b200 as fb
from paper_2605_26659_b200 import workloads as W
x, y, u, v, eps = W.config2()
bs = fb.BatchSolver1D([x], [y], [u], [v], [eps])
outs = []
for r in range(3):
    bs.solve(200, 0.0, True, 200.0)
    torch.cuda.synchronize()
    outs.append((bs.phi.cpu().numpy().copy(), bs.psi.cpu().numpy().copy(), bs.hist.cpu().numpy().copy()))
same = all(np.array_equal(outs[0][k], o[k]) for o in outs[1:] for k in range(3))
print("config2 bitwise reproducible over 3 solves:", same)
x1, y1, x2, y2, U, V, e2 = W.config3()
g = lambda a, b: fb.Grid2D(fb.Mesh1D(a), fb.Mesh1D(b))
cfg = fb.SolverConfig(epsilon=e2, itr_max=300, tol=0.0, stabilize=True)
s = [fb.sinkhorn_2d(g(x1, y1), g(x2, y2), fb.Measure2D(U), fb.Measure2D(V), cfg) for _ in range(3)]
same2 = all(np.array_equal(s[0].phi, t.phi) and np.array_equal(s[0].psi, t.psi) and s[0].cost == t.cost for t in s[1:])
print("config3 bitwise reproducible over 3 solves:", same2)
