"""Run every golden solver case through sinkhorn_1d and report failures (debug aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2605_26659_b200 as fb
from conftest import load_golden
g = load_golden("solver_cases.npz")
for k in range(int(g["ncases"])):
    s = lambda key: g["s%d_%s" % (k, key)]
    eps, itr, tol, stab, thr, ce = s("cfg")
    cfg = fb.SolverConfig(epsilon=eps, itr_max=int(itr), tol=tol, stabilize=bool(stab),
                          absorb_threshold=thr, check_every=int(ce))
    try:
        sol = fb.sinkhorn_1d(fb.Mesh1D(s("x")), fb.Mesh1D(s("y")), fb.Measure(s("u")), fb.Measure(s("v")), cfg)
        err = np.max(np.abs(sol.phi - s("phi")) / np.max(np.abs(s("phi"))))
        print(k, "ok", len(s("x")), len(s("y")), "eps", eps, "stab", stab, "its", sol.iterations_run, int(s("iterations")), "phi err %.2e" % err)
    except Exception as e:
        print(k, "EXC", type(e).__name__, len(s("x")), len(s("y")), "eps", eps, "stab", stab, "itr", itr, "absorbs ref", s("absorb_its"))
