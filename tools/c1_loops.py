"""Config 1 per-iteration time through the available loop forms
(FB_CLUSTER=1: the cluster group solve; 0: the tile-parallel graph loop)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_26659_b200 as fb  # noqa: E402
from paper_2605_26659_b200 import workloads as W  # noqa: E402

x, y, u, v, eps = W.config1()
for form in sys.argv[1:] or ["0", "1"]:
    os.environ["FB_CLUSTER"] = form
    bs = fb.BatchSolver1D([x], [y], [u], [v], [eps])
    bs.solve(500)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        bs.solve(500)
    e1.record()
    torch.cuda.synchronize()
    print("config1 FB_CLUSTER=%s: %.2f us/iteration (group %d)" % (
        form, e0.elapsed_time(e1) / 5 / 500 * 1e3, fb._lib.load().finom_solve1d_group(bs.plan.handle)),
        flush=True)
    del bs
