#!/bin/bash
# Final round-2 measurement: GPU tests, smoke, default bench (config 5) in the driver's form,
# reference arm, bench lines of configs 1-4, ncu launch list of the default bench command.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
timeout 900 python bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err; tail -1 gpurun_out/bench_ref.json | cut -c1-200
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -1 gpurun_out/bench.json | cut -c1-300
for c in 1 2 3 4; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 2>gpurun_out/bench_c$c.err | tail -1 > gpurun_out/bench_c$c.json; cut -c1-200 gpurun_out/bench_c$c.json; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_c5.log 2>&1; echo "launch list rc=$?"
