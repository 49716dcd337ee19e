# Round-2 profiles of the headline (config 5, group solve) and config 1 / 2 timings.
set -x
mkdir -p gpurun_out
# config 1 through both loops (per-iteration latency)
for g in 0 1; do FB_GROUP=$g python - <<'PY'
import os, time, torch, numpy as np, sys
sys.path.insert(0, ".")
import paper_2605_26659_b200 as fb
from paper_2605_26659_b200 import workloads as W
x, y, u, v, eps = W.config1()
bs = fb.BatchSolver1D([x], [y], [u], [v], [eps])
bs.solve(500); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): bs.solve(500)
e1.record(); torch.cuda.synchronize()
print("config1 group=%s: %.2f us/iteration" % (os.environ["FB_GROUP"], e0.elapsed_time(e1) / 5 / 500 * 1e3))
PY
done > gpurun_out/c1_loops.txt 2>&1
# launch list of the default bench command (cold, serialised: shares only)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_c5.log 2>&1
# full capture of the dominant kernel: one whole 200-iteration config-5 solve
ncu --set full --import-source on --clock-control none -k regex:k_solve_group -c 1 -o gpurun_out/prof_group_c5 -f python tools/prof_group.py 8192 200 1 > gpurun_out/ncu_group_c5.log 2>&1
