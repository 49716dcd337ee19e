"""Per-iteration time of the dense GPU baseline (cuBLAS DGEMV, dense.py) vs the
O(N) path on config-1-style 1D problems (fixed iterations, no stabilization)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2605_26659_b200 as fb
from paper_2605_26659_b200 import dense as D, workloads as W
for n in (4096, 16384, 32768):
    x, y, u, v, eps = W.config1(n=n)
    X, Y, U, V = fb.Mesh1D(x), fb.Mesh1D(y), fb.Measure(u), fb.Measure(v)
    its = 100
    cfg = fb.SolverConfig(epsilon=eps, itr_max=its, tol=0.0, stabilize=False, plan_cap=10**10)
    D.dense_sinkhorn(fb.Problem(X, Y, U, V), fb.SolverConfig(epsilon=eps, itr_max=3, tol=0.0, plan_cap=10**10))
    dn = D.dense_sinkhorn(fb.Problem(X, Y, U, V), cfg)
    bs = fb.BatchSolver1D([x], [y], [u], [v], [eps])
    bs.solve(its, 0.0, False, 200.0); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); bs.solve(its, 0.0, False, 200.0); e1.record(); torch.cuda.synchronize()
    fast_it = e0.elapsed_time(e1) / its * 1e3
    dense_it = (dn.wall_time - dn.setup_time) / its * 1e6
    print("n=%6d  dense %8.1f us/it   O(N) %6.1f us/it   speed-up %6.1fx" % (n, dense_it, fast_it, dense_it / fast_it))
