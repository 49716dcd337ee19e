# ncu --set full of the cluster line sweep at config 4: an absorbed x sweep (split records) and y sweep (per-line records, fused update)
CFG=4 ITERS=10 FB_GRAPH2D=0 FB_SQ_LINE=${V:-44} timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sq_line -s 32 -c 2 -o gpurun_out/prof_line -f python tools/ncu_2d_target.py > gpurun_out/ncu_line.log 2>&1; echo rc=$?
tail -2 gpurun_out/ncu_line.log
