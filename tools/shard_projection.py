"""Per-shard work of the row-sharded 2D solve (config 4 shape), measured on ONE
GPU by timing each shard's kernels (events around xpre + finish per shard):
the compute a rank would do at R GPUs, without the collectives.  A projection,
not a multi-GPU measurement."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2605_26659_b200 as fb
from paper_2605_26659_b200 import sharding as S, workloads as W
n = int(os.environ.get("N4", "8192"))
x1, y1, x2, y2, U, V, eps = W.config4(n=n)
Uf, Vf = U.ravel(order="F"), V.ravel(order="F")
its = 10
for R in (1, 2, 4, 8):
    ranges = S.grid_row_ranges(n, R)
    shards = [S.RowShard2D(x1, y1, y2, Uf, Vf, eps, k0, k1) for k0, k1 in ranges]
    times = []
    for k, s in enumerate(shards):
        for half in (0, 1):  # warm
            seg0 = s.xpre(half, False).clone()
            seg = torch.cat([seg0] * R)
            s.finish(half, False, seg, R, k)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(its):
            for half in (0, 1):
                seg0 = s.xpre(half, False).clone()
                seg = torch.cat([seg0] * R)
                s.finish(half, False, seg, R, k)
        e1.record(); torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / its)
    t = max(times)
    print("R=%d  per-shard iteration %.2f ms (max over shards, unabsorbed kernel form, no collectives)"
          "  -> projected %.3e pts*it/s" % (R, t, n * n / (t * 1e-3)))
    for s in shards:
        s.close()
    del shards
    torch.cuda.empty_cache()
