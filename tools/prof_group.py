"""Batched 1D solve of config-5 problems for timing / ncu (group solve vs the
tile-parallel loop: FB_GROUP=0/1).  usage: prof_group.py BATCH ITERS [REPS]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_26659_b200 import _lib  # noqa: E402
if os.environ.get("FINOM_LIB"):  # (timing a library variant)
    _lib.LIB_PATH = os.path.abspath(os.environ["FINOM_LIB"])
import paper_2605_26659_b200 as fb  # noqa: E402
from paper_2605_26659_b200 import workloads as W  # noqa: E402

B, its = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
n = int(os.environ.get("FINOM_N", "16384"))
probs = W.config5(batch=B, n=n)
bs = fb.BatchSolver1D([p[0] for p in probs], [p[1] for p in probs], [p[2] for p in probs],
                      [p[3] for p in probs], [p[4] for p in probs])
bs.solve(its)
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    bs.solve(its)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = float(np.median(ts))
info = bs.info.view(bs.P, 5).cpu().numpy()
print("%s B %d n %d its %d: %.3f ms/solve  %.3e pts*it/s  absorbs %d  group=%s" % (
    os.path.basename(_lib.LIB_PATH), B, n, its, ms, B * n * its / (ms * 1e-3), int(info[:, 3].sum()), os.environ.get("FB_GROUP", "auto")))
