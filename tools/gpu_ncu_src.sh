# ncu --set full with source of k_step on config 2 (one k_step<0> and one k_step<1>)
export ITERS=3
python tools/ncu_target.py > gpurun_out/plain.log 2>&1 || { echo plain failed; cat gpurun_out/plain.log; exit 1; }
FB_WHILE1D=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step -s 2 -c 2 -o gpurun_out/prof_kstep python tools/ncu_target.py > gpurun_out/ncu2.log 2>&1; echo "ncu rc=$?"
tail -2 gpurun_out/ncu2.log
