#!/bin/bash
# Per-launch list of config 4 (10 iterations, absorbed from iteration 7) with dram bytes.
mkdir -p gpurun_out
CFG=4 ITERS=10 FB_GRAPH2D=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launch4.csv python tools/ncu_2d_target.py > gpurun_out/launch4.log 2>&1; echo rc4=$?
