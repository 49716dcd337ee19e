CFG=4 ITERS=2 FB_GRAPH2D=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sq_apply|k_sq_pre" -s 4 -c 4 -o gpurun_out/prof_sq python tools/ncu_2d_target.py > gpurun_out/ncu_sq.log 2>&1; echo rc=$?
tail -2 gpurun_out/ncu_sq.log
