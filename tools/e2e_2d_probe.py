"""Break down one public-API sinkhorn_2d call (config 4 by default, ITERS iterations)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2605_26659_b200 as fb
from paper_2605_26659_b200 import workloads as W
its = int(os.environ.get("ITERS", "100"))
x1, y1, x2, y2, U, V, eps = W.config4() if os.environ.get("CFG", "4") == "4" else W.config3()
t0 = time.perf_counter()
src, tgt = fb.Grid2D(fb.Mesh1D(x1), fb.Mesh1D(y1)), fb.Grid2D(fb.Mesh1D(x2), fb.Mesh1D(y2))
mu, mv = fb.Measure2D(U), fb.Measure2D(V)
print("grids+measures %.1f ms" % (1e3 * (time.perf_counter() - t0)))
c = fb.SolverConfig(epsilon=eps, itr_max=its, tol=0.0, stabilize=True)
for r in range(2):
    t0 = time.perf_counter()
    sol = fb.sinkhorn_2d(src, tgt, mu, mv, c)
    t1 = time.perf_counter()
    print("total %.1f ms  setup %.1f  loop %.1f  -> other %.1f ms" % (
        1e3 * (t1 - t0), 1e3 * sol.setup_time, 1e3 * (sol.wall_time - sol.setup_time),
        1e3 * (t1 - t0 - sol.wall_time)))
t0 = time.perf_counter(); fb.kernel2d.build_operator_2d(src, tgt, eps); print("build_operator_2d %.1f ms" % (1e3 * (time.perf_counter() - t0)))
t0 = time.perf_counter(); U2 = np.ascontiguousarray(mu.weights.ravel(order="F")); print("ravel F %.1f ms" % (1e3 * (time.perf_counter() - t0)))
