#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/e2e5_stages.py 4 6 8 12 > gpurun_out/e2e5_stages.txt 2>&1; tail -5 gpurun_out/e2e5_stages.txt
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c5b.json 2>&1; tail -1 gpurun_out/bench_c5b.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'])"
