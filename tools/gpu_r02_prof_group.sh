#!/bin/bash
# ncu --set full of the group solve on a reduced batch (B = 1184 problems,
# 40 iterations: the full batch's buffers make ncu's kernel replay too slow)
mkdir -p gpurun_out
timeout 300 python tools/prof_group.py 1184 40 3 > gpurun_out/group_plain.txt 2>&1; cat gpurun_out/group_plain.txt
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_solve_group -c 1 -o gpurun_out/prof_group -f python tools/prof_group.py 1184 40 1 > gpurun_out/ncu_group.log 2>&1; echo "ncu group rc=$?"
tail -3 gpurun_out/ncu_group.log
