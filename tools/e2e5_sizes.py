"""sinkhorn_1d_batched on config 5 with explicit pipeline stage sizes
(FINOM_PIPE_SIZES), the default stages ("default") or one stage ("single"): wall
clock of the call.  usage: [FINOM_BATCH=B] e2e5_sizes.py default single "592,2368,..." ..."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_26659_b200 as fb  # noqa: E402
from paper_2605_26659_b200 import workloads as W  # noqa: E402

B = int(os.environ.get("FINOM_BATCH", "8192"))
probs = W.config5(batch=B, problems=range(B))
xs = [fb.Mesh1D(p[0]) for p in probs]
ys = [fb.Mesh1D(p[1]) for p in probs]
us = [fb.Measure(p[2]) for p in probs]
vs = [fb.Measure(p[3]) for p in probs]
eps = [p[4] for p in probs]
cfg = fb.SolverConfig(epsilon=1.0, itr_max=200, tol=0.0, stabilize=True)
for st in sys.argv[1:]:
    os.environ.pop("FINOM_PIPE_SIZES", None)
    os.environ.pop("FINOM_PIPE_STAGES", None)
    if st == "single":
        os.environ["FINOM_PIPE_STAGES"] = "1"
    elif st != "default":
        os.environ["FINOM_PIPE_SIZES"] = st
    ts = []
    for r in range(4):
        if r == 3:
            os.environ["FB_VERBOSE"] = "1"
        torch.cuda.synchronize()
        t = time.perf_counter()
        sols = fb.sinkhorn_1d_batched(xs, ys, us, vs, cfg, epsilons=eps)
        ts.append(time.perf_counter() - t)
        del sols
        os.environ.pop("FB_VERBOSE", None)
    print("sizes %s: %s s  e2e %.3e pts*it/s (best of warm), median %.3f s" % (
        st, ["%.3f" % x for x in ts], B * 16384 * 200 / min(ts[1:]), sorted(ts[1:])[1]), flush=True)
