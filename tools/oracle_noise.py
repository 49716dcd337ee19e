"""The reference's own sensitivity: the C oracle (the same algorithm and
operation order; libm exp instead of numpy's SIMD exp for the tables, <= 1
ulp apart on a few % of arguments) against the reference's fixtures -- the
deviation any faithful restatement shows, the yardstick for the CUDA path's
history deviation (tools/parity_numbers.py).  CPU only."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle import oracle as O  # noqa: E402
from paper_2605_26659_b200 import workloads as W  # noqa: E402
from conftest import load_golden, rel_inf  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from parity_numbers_stats import hist_stats  # noqa: E402

res = {}
g = load_golden("config2_full_pins.npz")
x, y, u, v, eps = W.config2()
r = O.sinkhorn_1d(x, y, u, v, eps, 200, 0.0, True)
st = int(g["stride"])
res["config2_full"] = dict(phi=rel_inf(r["phi"][::st], g["phi_s"]),
                           psi=rel_inf(r["psi"][::st], g["psi_s"]), **hist_stats(r["hist"], g["hist_err"]))
g = load_golden("config5_p0-3.npz")
for k, p in enumerate(W.config5(problems=[0, 1, 2, 3])):
    r = O.sinkhorn_1d(p[0], p[1], p[2], p[3], p[4], 200, 0.0, True)
    res["config5_p%d" % k] = dict(phi=rel_inf(r["phi"], g["p%d_phi" % k]),
                                  **hist_stats(r["hist"], g["p%d_hist_err" % k]))
print(json.dumps(res, indent=1))
