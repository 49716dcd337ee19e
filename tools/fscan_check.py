"""Bitwise check of a 2D solve under two environment settings (e.g. FB_SQ_FSCAN=0 / 1):
usage: fscan_check.py VAR  (config 3 full size and a 40x40 grid with ragged tiles)."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 2:  # child: solve, save
    sys.path.insert(0, ROOT)
    import paper_2605_26659_b200 as fb
    from paper_2605_26659_b200 import workloads as W
    n = int(sys.argv[2])
    x1, y1, x2, y2, U, V, eps = W.config3(n=n)
    g = lambda x, y: fb.Grid2D(fb.Mesh1D(x), fb.Mesh1D(y))
    cfg = fb.SolverConfig(epsilon=eps, itr_max=300 if n > 100 else 80, tol=0.0, stabilize=True,
                          absorb_threshold=200.0 if n > 100 else 30.0)
    s = fb.sinkhorn_2d(g(x1, y1), g(x2, y2), fb.Measure2D(U), fb.Measure2D(V), cfg)
    np.savez(sys.argv[1], phi=s.phi, psi=s.psi, a=s.a, b=s.b, cost=s.cost,
             hist=np.array([e for _, e in s.marginal_error_history]),
             absorbs=np.array(s.absorb_iterations))
    sys.exit(0)
var = sys.argv[1]
for n in (1024, 40):
    outs = []
    for val in ("0", "1"):
        f = "/tmp/fscan_%s_%d.npz" % (val, n)
        subprocess.check_call([sys.executable, __file__, f, str(n)], env=dict(os.environ, **{var: val}))
        outs.append(np.load(f))
    same = all(np.array_equal(outs[0][k], outs[1][k]) for k in outs[0].files)
    print("n=%d %s=0 vs 1: bitwise %s; absorbs %s; cost %.17g" % (
        n, var, same, list(outs[1]["absorbs"]), float(outs[1]["cost"])), flush=True)
