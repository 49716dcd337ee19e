#!/bin/bash
# Per-launch list of config 4 (10 iterations, absorbed from iteration 7) on the cluster line sweep
mkdir -p gpurun_out
for v in ${VARIANTS:-44 24}; do
CFG=4 ITERS=10 FB_GRAPH2D=0 FB_SQ_LINE=$v timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launch4_line$v.csv python tools/ncu_2d_target.py > gpurun_out/launch4_line$v.log 2>&1; echo rc4=$?
python tools/launch_summary.py gpurun_out/launch4_line$v.csv 2>&1 | head -12
grep k_sq_line gpurun_out/launch4_line$v.csv | tail -24 | cut -d, -f5,12-15 | head -40
done
