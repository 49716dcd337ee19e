"""Measured parity of the CUDA path against the reference's own outputs
(tests/golden), per config: rel-inf of phi / psi / a / b, cost, and the
marginal-error history -- the largest PURE relative deviation (no floor),
the largest over entries above the 1e-12 floor the tests use, and how many
entries sit below that floor.  Writes JSON to argv[1] (default stdout)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                "tests"))
import paper_2605_26659_b200 as fb  # noqa: E402
from paper_2605_26659_b200 import workloads as W  # noqa: E402
from conftest import load_golden, rel_inf  # noqa: E402

from parity_numbers_stats import FLOOR, hist_stats  # noqa: E402,F401


def vec_stats(sol, g, stride=None, pre=""):
    s = slice(None, None, stride)
    out = {}
    for k in ("phi", "psi", "a", "b"):
        ref = g[pre + k + ("_s" if stride else "")]
        out[k] = rel_inf(getattr(sol, k)[s], ref)
    out["cost"] = abs(sol.cost - float(g[pre + "cost"])) / abs(float(g[pre + "cost"]))
    return out


def run1d(x, y, u, v, eps, itr):
    cfg = fb.SolverConfig(epsilon=eps, itr_max=itr, tol=0.0, stabilize=True)
    return fb.sinkhorn_1d(fb.Mesh1D(x), fb.Mesh1D(y), fb.Measure(u), fb.Measure(v), cfg)


def run2d(x1, y1, x2, y2, U, V, eps, itr):
    cfg = fb.SolverConfig(epsilon=eps, itr_max=itr, tol=0.0, stabilize=True)
    return fb.sinkhorn_2d(fb.Grid2D(fb.Mesh1D(x1), fb.Mesh1D(y1)),
                          fb.Grid2D(fb.Mesh1D(x2), fb.Mesh1D(y2)), fb.Measure2D(U),
                          fb.Measure2D(V), cfg)


def main():
    res = {}
    g = load_golden("config1.npz")
    sol = run1d(*W.config1(), 500)
    res["config1"] = dict(vec_stats(sol, g), **hist_stats([e for _, e in sol.marginal_error_history],
                                                          g["hist_err"]))
    g = load_golden("config2_n65536.npz")
    sol = run1d(*W.config2(n=1 << 16), 200)
    res["config2_n65536"] = dict(vec_stats(sol, g),
                                 **hist_stats([e for _, e in sol.marginal_error_history],
                                              g["hist_err"]))
    g = load_golden("config2_full_pins.npz")
    sol = run1d(*W.config2(), 200)
    res["config2_full"] = dict(vec_stats(sol, g, int(g["stride"])),
                               **hist_stats([e for _, e in sol.marginal_error_history],
                                            g["hist_err"]))
    g = load_golden("config3_full_pins.npz")
    sol = run2d(*W.config3(), 300)
    res["config3_full"] = dict(vec_stats(sol, g, int(g["stride"])),
                               **hist_stats([e for _, e in sol.marginal_error_history],
                                            g["hist_err"]))
    g = load_golden("config4_full_pins.npz")
    sol = run2d(*W.config4(), 100)
    res["config4_full"] = dict(vec_stats(sol, g, int(g["stride"])),
                               **hist_stats([e for _, e in sol.marginal_error_history],
                                            g["hist_err"]))
    g = load_golden("config5_p0-3.npz")
    probs = W.config5(problems=[0, 1, 2, 3])
    cfg = fb.SolverConfig(epsilon=1.0, itr_max=200, tol=0.0, stabilize=True)
    for mode in ("0", "1"):  # tile-parallel loop, group solve
        os.environ["FB_GROUP"] = mode
        sols = fb.sinkhorn_1d_batched([fb.Mesh1D(p[0]) for p in probs],
                                      [fb.Mesh1D(p[1]) for p in probs],
                                      [fb.Measure(p[2]) for p in probs],
                                      [fb.Measure(p[3]) for p in probs], cfg,
                                      epsilons=[p[4] for p in probs])
        for k, sol in enumerate(sols):
            res["config5_p%d_%s" % (k, "group" if mode == "1" else "tiles")] = dict(
                vec_stats(sol, g, None, "p%d_" % k),
                **hist_stats([e for _, e in sol.marginal_error_history], g["p%d_hist_err" % k]))
    os.environ.pop("FB_GROUP")
    worst = {}
    for r in res.values():
        for k, v in r.items():
            if isinstance(v, float) and k not in ("hist_abs_max_below_floor",):
                worst[k] = max(worst.get(k, 0.0), v)
    res["worst"] = worst
    out = json.dumps(res, indent=1)
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            f.write(out)
    print(out)


if __name__ == "__main__":
    main()
