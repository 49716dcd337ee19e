"""Loop time of the 2D solve (config 3, and config 4 with ITERS4 iterations) for library variants."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_26659_b200 import _lib, workloads as W
_lib.LIB_PATH = sys.argv[1]
import paper_2605_26659_b200 as fb
for cfg, its in ((3, 300), (4, int(os.environ.get("ITERS4", "20")))):
    if cfg == 3:
        x1, y1, x2, y2, U, V, eps = W.config3()
    else:
        x1, y1, x2, y2, U, V, eps = W.config4()
    src, tgt = fb.Grid2D(fb.Mesh1D(x1), fb.Mesh1D(y1)), fb.Grid2D(fb.Mesh1D(x2), fb.Mesh1D(y2))
    c = fb.SolverConfig(epsilon=eps, itr_max=its, tol=0.0, stabilize=True)
    loops = []
    for r in range(3):
        sol = fb.sinkhorn_2d(src, tgt, fb.Measure2D(U), fb.Measure2D(V), c)
        loops.append(sol.wall_time - sol.setup_time)
    lp = min(loops[1:])
    print(os.path.basename(sys.argv[1]), "config%d %d it: loop %.1f ms (%.3e pts*it/s)" % (
        cfg, its, 1e3 * lp, x1.size * y1.size * its / lp))
