# compute-sanitizer over small solves: 1D (graph + WHILE loop, absorptions), 2D square + general sweeps
cat > /tmp/san_target.py <<'PY'
import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import numpy as np
import paper_2605_26659_b200 as fb
from paper_2605_26659_b200 import workloads as W
x, y, u, v, eps = W.config1(n=3000)
cfg = fb.SolverConfig(epsilon=eps, itr_max=20, tol=0.0, stabilize=True, absorb_threshold=5.0)
s = fb.sinkhorn_1d(fb.Mesh1D(x), fb.Mesh1D(y), fb.Measure(u), fb.Measure(v), cfg)
print("1d", s.iterations_run, s.absorb_iterations, s.cost)
x1, y1, x2, y2, U, V, e2 = W.config3(n=300)
c2 = fb.SolverConfig(epsilon=e2, itr_max=15, tol=0.0, stabilize=True, absorb_threshold=6.0)
g = lambda a, b: fb.Grid2D(fb.Mesh1D(a), fb.Mesh1D(b))
s2 = fb.sinkhorn_2d(g(x1, y1), g(x2, y2), fb.Measure2D(U), fb.Measure2D(V), c2)
print("2d", s2.iterations_run, s2.absorb_iterations, s2.cost)
PY
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python /tmp/san_target.py > gpurun_out/san_$tool.log 2>&1; echo "$tool rc=$?"
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|^1d|^2d|Error|error" gpurun_out/san_$tool.log | head -8
done
