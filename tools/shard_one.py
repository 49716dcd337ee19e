"""One rank's half-steps at R shards (config 4 shape), for ncu launch lists."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_26659_b200 import sharding as S, workloads as W
n, R = 8192, int(os.environ.get("R", "8"))
x1, y1, x2, y2, U, V, eps = W.config4(n=n)
Uf, Vf = U.ravel(order="F"), V.ravel(order="F")
k0, k1 = S.grid_row_ranges(n, R)[0]
s = S.RowShard2D(x1, y1, y2, Uf, Vf, eps, k0, k1)
for _ in range(3):
    for half in (0, 1):
        seg0 = s.xpre(half, False).clone()
        seg = torch.cat([seg0] * R)
        s.finish(half, False, seg, R, 0)
torch.cuda.synchronize()
print("done")
