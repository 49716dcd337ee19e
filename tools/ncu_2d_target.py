"""Small 2D target for ncu launch lists: config 3 (1024^2) or config 4 at n (env N4), ITERS iterations."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_26659_b200 as fb
from paper_2605_26659_b200 import workloads as W
cfg = int(os.environ.get("CFG", "3"))
its = int(os.environ.get("ITERS", "3"))
if cfg == 3:
    x1, y1, x2, y2, U, V, eps = W.config3()
else:
    x1, y1, x2, y2, U, V, eps = W.config4(n=int(os.environ.get("N4", "8192")))
src, tgt = fb.Grid2D(fb.Mesh1D(x1), fb.Mesh1D(y1)), fb.Grid2D(fb.Mesh1D(x2), fb.Mesh1D(y2))
sol = fb.sinkhorn_2d(src, tgt, fb.Measure2D(U), fb.Measure2D(V),
                     fb.SolverConfig(epsilon=eps, itr_max=its, tol=0.0, stabilize=True))
print("its", sol.iterations_run, "loop s", sol.wall_time - sol.setup_time)
