export ITERS=3
python tools/ncu_target.py > gpurun_out/plain.log 2>&1 || { echo plain failed; cat gpurun_out/plain.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_resolve|k_absorb" -s 2 -c 4 -o gpurun_out/prof_res python tools/ncu_target.py > gpurun_out/ncu3.log 2>&1; echo "ncu rc=$?"
tail -2 gpurun_out/ncu3.log
