"""The single-pass square sweeps -- k_sq_chain ("chain": FB_SQ_CHAIN=1) and the
cluster line sweep k_sq_line ("44" / "24" / "42": FB_SQ_LINE) -- against the
three-kernel square sweeps (FB_SQ_CHAIN=0 FB_SQ_LINE=0) on config-4-style grids whose lines
have 5..32 tiles (ragged last tiles, cluster sizes 2..16), with absorptions:
max relative deviation of phi / psi / a / b / cost / history, and the oracle's
on the small case.  usage: line_check.py [variants...]"""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = [(1300, 40, 30.0), (2048, 30, 30.0), (2300, 24, 50.0), (4100, 16, 50.0)]
if len(sys.argv) > 2 and sys.argv[1] == "--child":
    sys.path.insert(0, ROOT)
    import paper_2605_26659_b200 as fb
    from paper_2605_26659_b200 import workloads as W
    out = {}
    for n, its, thr in CASES:
        x1, y1, x2, y2, U, V, eps = W.config4(n=n)
        g = lambda x, y: fb.Grid2D(fb.Mesh1D(x), fb.Mesh1D(y))
        cfg = fb.SolverConfig(epsilon=eps, itr_max=its, tol=0.0, stabilize=True, absorb_threshold=thr)
        s = fb.sinkhorn_2d(g(x1, y1), g(x2, y2), fb.Measure2D(U), fb.Measure2D(V), cfg)
        for k, v in dict(phi=s.phi, psi=s.psi, a=s.a, b=s.b, cost=np.array([s.cost]),
                         hist=np.array([e for _, e in s.marginal_error_history]),
                         absorbs=np.array(s.absorb_iterations, dtype=np.int64)).items():
            out["%s_%d" % (k, n)] = v
    np.savez(sys.argv[2], **out)
    sys.exit(0)
variants = sys.argv[1:] or ["chain", "44"]
res = {}
for v in ["0"] + variants:
    f = "/tmp/line_%s.npz" % v
    env = {"FB_SQ_CHAIN": "1" if v == "chain" else "0", "FB_SQ_LINE": v if v.isdigit() else "0"}
    subprocess.check_call([sys.executable, __file__, "--child", f], env=dict(os.environ, **env), timeout=600)
    res[v] = np.load(f)
rel = lambda a, b: float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)) if a.size else 0.0
bad = False
for v in variants:
    for n, its, thr in CASES:
        d = {k: rel(res[v]["%s_%d" % (k, n)], res["0"]["%s_%d" % (k, n)])
             for k in ("phi", "psi", "a", "b", "cost", "hist")}
        same_abs = np.array_equal(res[v]["absorbs_%d" % n], res["0"]["absorbs_%d" % n])
        print("variant %s n=%d: %s absorbs %s (same %s)" % (
            v, n, " ".join("%s %.2e" % kv for kv in d.items()), list(res[v]["absorbs_%d" % n]), same_abs),
            flush=True)
        bad |= (not same_abs) or max(d[k] for k in ("phi", "psi", "a", "b", "cost")) > 1e-11
print("LINE CHECK", "FAILED" if bad else "ok")
sys.exit(1 if bad else 0)
