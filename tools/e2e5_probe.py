"""Break down sinkhorn_1d_batched on config 5 (host arrays in, Solutions out)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2605_26659_b200 as fb
from paper_2605_26659_b200 import workloads as W, solver as S
B = int(os.environ.get("FINOM_BATCH", "8192"))
probs = W.config5(batch=B, problems=range(B))
xs = [fb.Mesh1D(p[0]) for p in probs]; ys = [fb.Mesh1D(p[1]) for p in probs]
us = [fb.Measure(p[2]) for p in probs]; vs = [fb.Measure(p[3]) for p in probs]
eps = [p[4] for p in probs]
cfg = fb.SolverConfig(epsilon=1.0, itr_max=200, tol=0.0, stabilize=True)
fb.sinkhorn_1d_batched(xs[:64], ys[:64], us[:64], vs[:64], cfg, epsilons=eps[:64])
T = {}
t = time.perf_counter()
bs = S.BatchSolver1D(xs, ys, us, vs, eps); torch.cuda.synchronize(); T["init (plan + H2D)"] = time.perf_counter() - t
t = time.perf_counter(); bs.solve(200, 0.0, True, 200.0); info = bs.info.view(bs.P, 5).cpu().numpy(); T["solve"] = time.perf_counter() - t
t = time.perf_counter(); bs.compute_cost(); torch.cuda.synchronize(); T["cost"] = time.perf_counter() - t
t = time.perf_counter()
hist = bs.hist.view(bs.P, -1).cpu().numpy(); abs_its = bs.abs_its.view(bs.P, -1).cpu().numpy()
phi, psi = bs.phi.cpu().numpy(), bs.psi.cpu().numpy(); a, b = bs.a.cpu().numpy(), bs.b.cpu().numpy()
T["d2h"] = time.perf_counter() - t
t = time.perf_counter(); t0 = time.perf_counter()
sols = fb.sinkhorn_1d_batched(xs, ys, us, vs, cfg, epsilons=eps)
T["whole call"] = time.perf_counter() - t0
for k, v in T.items():
    print("%-20s %8.1f ms" % (k, 1e3 * v))
