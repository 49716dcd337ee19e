"""Break down one public-API sinkhorn_1d call on config 2 (host buffers in/out)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2605_26659_b200 as fb
from paper_2605_26659_b200 import workloads as W
x, y, u, v, eps = W.config2()
X, Y, U, V = fb.Mesh1D(x), fb.Mesh1D(y), fb.Measure(u), fb.Measure(v)
cfg = fb.SolverConfig(epsilon=eps, itr_max=200, tol=0.0, stabilize=True)
for r in range(3):
    t0 = time.perf_counter()
    sol = fb.sinkhorn_1d(X, Y, U, V, cfg)
    t1 = time.perf_counter()
    print("total %.1f ms  setup %.1f ms  setup+loop %.1f ms  -> other %.1f ms" % (
        1e3 * (t1 - t0), 1e3 * sol.setup_time, 1e3 * sol.wall_time, 1e3 * (t1 - t0 - sol.wall_time)))
t0 = time.perf_counter(); fb.Mesh1D(x); print("Mesh1D %.1f ms" % (1e3 * (time.perf_counter() - t0)))
