#!/bin/bash
# Per-launch list of config 4 (10 iterations, absorbed from iteration 7) on the single-pass chain sweep
mkdir -p gpurun_out
CFG=4 ITERS=10 FB_GRAPH2D=0 FB_SQ_CHAIN=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launch4_chain.csv python tools/ncu_2d_target.py > gpurun_out/launch4_chain.log 2>&1; echo rc4=$?
python tools/launch_summary.py gpurun_out/launch4_chain.csv 2>&1 | head -8
