"""Small ncu target: one config-2 solve of ITERS iterations (default 6)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_26659_b200 as fb  # noqa: E402
from paper_2605_26659_b200 import workloads as W  # noqa: E402

cfg = int(os.environ.get("CFG", "2"))
iters = int(os.environ.get("ITERS", "6"))
if cfg == 2:
    x, y, u, v, eps = W.config2()
else:
    x, y, u, v, eps = W.config1()
bs = fb.BatchSolver1D([x], [y], [u], [v], [eps])
st = bs.solve(iters, 0.0, True, 200.0)
torch.cuda.synchronize()
print("status", st, "iterations", int(bs.info[0].item()))
