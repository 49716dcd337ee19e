#!/bin/bash
# Round-2 measurement: GPU tests, smoke, default bench (config 5), reference arm,
# bench lines of configs 1-4, launch list of the default bench, ncu --set full
# of the group solve (config 5) and of k_step (config 2).
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -1 gpurun_out/bench.json | cut -c1-400
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1; tail -1 gpurun_out/bench_ref.json | cut -c1-200
for c in 1 2 3 4; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 2>gpurun_out/bench_c$c.err | tail -1 > gpurun_out/bench_c$c.json; cut -c1-200 gpurun_out/bench_c$c.json; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_c5.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_solve_group -c 1 -o gpurun_out/prof_group_c5 -f python tools/prof_group.py 8192 200 1 > gpurun_out/ncu_group_c5.log 2>&1; echo "ncu group rc=$?"
export ITERS=24
FB_WHILE1D=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step -s 42 -c 2 -o gpurun_out/prof_kstep -f python tools/ncu_target.py > gpurun_out/ncu2.log 2>&1; echo "ncu kstep rc=$?"
