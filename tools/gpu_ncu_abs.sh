export ITERS=1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_absorb -c 1 -o gpurun_out/prof_abs python tools/ncu_target.py > gpurun_out/ncu_abs.log 2>&1; echo rc=$?
tail -2 gpurun_out/ncu_abs.log
