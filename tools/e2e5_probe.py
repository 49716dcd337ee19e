"""Break down sinkhorn_1d_batched on config 5 (host arrays in, Solutions out)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_26659_b200 as fb  # noqa: E402
from paper_2605_26659_b200 import _lib, workloads as W  # noqa: E402

B = int(os.environ.get("FINOM_BATCH", "8192"))
probs = W.config5(batch=B, problems=range(B))
xs = [fb.Mesh1D(p[0]) for p in probs]
ys = [fb.Mesh1D(p[1]) for p in probs]
us = [fb.Measure(p[2]) for p in probs]
vs = [fb.Measure(p[3]) for p in probs]
eps = [p[4] for p in probs]
cfg = fb.SolverConfig(epsilon=1.0, itr_max=200, tol=0.0, stabilize=True)
fb.sinkhorn_1d_batched(xs[:64], ys[:64], us[:64], vs[:64], cfg, epsilons=eps[:64])
T = {}
t = time.perf_counter()
cx = np.concatenate([x.nodes for x in xs]); cy = np.concatenate([y.nodes for y in ys])
T["concat x,y"] = time.perf_counter() - t
t = time.perf_counter()
plan = _lib.Plan1D([x.nodes for x in xs], [y.nodes for y in ys], eps)
torch.cuda.synchronize()
T["Plan1D"] = time.perf_counter() - t
del plan
from paper_2605_26659_b200 import solver as S  # noqa: E402
bs = S.BatchSolver1D(xs, ys, us, vs, eps)
for k in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); bs.solve(200); torch.cuda.synchronize()
    T["solve %d" % k] = time.perf_counter() - t
for k in range(2):
    t = time.perf_counter(); bs.compute_cost(); torch.cuda.synchronize()
    T["cost %d" % k] = time.perf_counter() - t
del bs
t = time.perf_counter()
sols = fb.sinkhorn_1d_batched(xs, ys, us, vs, cfg, epsilons=eps)
T["whole call"] = time.perf_counter() - t
t = time.perf_counter()
_ = [s.phi.sum() for s in sols]
T["touch solutions"] = time.perf_counter() - t
for k, v in T.items():
    print("%-20s %8.1f ms" % (k, 1e3 * v))
print("e2e pts*it/s %.3e" % (B * 16384 * 200 / T["whole call"]))
