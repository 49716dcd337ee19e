"""A/B of two library builds on config 4 (loop time of sinkhorn_2d, 100 it)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_26659_b200 import _lib
_lib.LIB_PATH = sys.argv[1]
import paper_2605_26659_b200 as fb
from paper_2605_26659_b200 import workloads as W
x1, y1, x2, y2, U, V, eps = W.config4() if os.environ.get("CFG", "4") == "4" else W.config3()
its = 100 if os.environ.get("CFG", "4") == "4" else 300
src, tgt = fb.Grid2D(fb.Mesh1D(x1), fb.Mesh1D(y1)), fb.Grid2D(fb.Mesh1D(x2), fb.Mesh1D(y2))
mu, mv = fb.Measure2D(U), fb.Measure2D(V)
c = fb.SolverConfig(epsilon=eps, itr_max=its, tol=0.0, stabilize=True)
loops = []
for r in range(3):
    sol = fb.sinkhorn_2d(src, tgt, mu, mv, c)
    loops.append(sol.wall_time - sol.setup_time)
print(os.path.basename(sys.argv[1]), "loops ms", ["%.1f" % (1e3 * l) for l in loops], "%.3e" % (x1.size * y1.size * its / min(loops[1:])))
