#!/bin/bash
# Re-entry check: GPU tests, smoke, bench lines of every config.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -1 gpurun_out/bench.json | cut -c1-600
for c in 1 2 3 4; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 2>gpurun_out/bench_c$c.err | tail -1 > gpurun_out/bench_c$c.json; cut -c1-300 gpurun_out/bench_c$c.json; done
