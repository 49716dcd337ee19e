# ncu capture of the half-step kernels on config 2 (ITERS iterations; K = kernel regex)
ITERS=${ITERS:-3}
K=${K:-k_step}
export ITERS
python tools/ncu_target.py > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 2 -o gpurun_out/prof_kstep python tools/ncu_target.py > gpurun_out/ncu2.log 2>&1; echo "ncu rc=$?"
tail -2 gpurun_out/ncu2.log
