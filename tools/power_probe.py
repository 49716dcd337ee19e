"""Config 5 solve time right after idle vs back to back (power cap): solves
separated by GAP seconds of idle, then REPS back-to-back solves, with the
SM clock sampled by nvidia-smi."""
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_26659_b200 as fb  # noqa: E402
from paper_2605_26659_b200 import workloads as W  # noqa: E402

probs = W.config5()
bs = fb.BatchSolver1D(*[[p[k] for p in probs] for k in range(5)])
bs.solve(200)
torch.cuda.synchronize()


def timed():
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    bs.solve(200)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def clocks():
    out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,temperature.gpu",
                          "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
    return out


for gap in (5.0, 5.0):
    time.sleep(gap)
    print("after %.0f s idle: %.1f ms  (%s before)" % (gap, timed(), clocks()), flush=True)
ts = [timed() for _ in range(8)]
print("back to back:", ["%.1f" % t for t in ts], clocks(), flush=True)
