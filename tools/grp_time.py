"""Phase timeline of one steady-state iteration of the group solve (FB_DBG_GRP
build: FINOM_LIB=libfinom_dbg_grp.so): warp 0 of problem 0, iteration 20.
usage: grp_time.py config1|config5"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_26659_b200 import _lib  # noqa: E402
import paper_2605_26659_b200 as fb  # noqa: E402
from paper_2605_26659_b200 import workloads as W  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "config1"
if which == "config1":
    x, y, u, v, eps = W.config1()
    bs = fb.BatchSolver1D([x], [y], [u], [v], [eps])
else:
    probs = W.config5(batch=int(os.environ.get("B", "8192")))
    bs = fb.BatchSolver1D(*[[p[k] for p in probs] for k in range(5)])
lib = bs.plan.lib
lib.finom_grp_read.argtypes = [ctypes.c_void_p]
for rep in range(2):
    bs.solve(200)
    torch.cuda.synchronize()
out = np.zeros(16)
lib.finom_grp_read(_lib.ptr(out))
its = out[15]
names = ["A carries", "A tiles", "A partials", "sync", "B carries", "B tiles", "B partials"]
print(which, "group", lib.finom_solve1d_group(bs.plan.handle), "iterations timed", int(its))
tot = 0.0
for k, nm in enumerate(names):
    v = out[k] / its / 1e3
    tot += v
    print("  %-12s %8.2f us (mean over groups and iterations)" % (nm, v))
print("  sum         %8.2f us" % tot)
