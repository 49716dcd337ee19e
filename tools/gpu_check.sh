# quick state check: gpu tests, bench config 2, configs 3/4 short
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -5
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -1 gpurun_out/bench.json
for c in 3 4; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_c$c.json; cat gpurun_out/bench_c$c.json; done
