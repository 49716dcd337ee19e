# fused line scan for short lines: bitwise check, config 3 A/B, 2D GPU tests
timeout 600 python tools/fscan_check.py FB_SQ_FSCAN 2>&1 | tail -3
for r in 1 2; do for o in 0 1; do
  FB_SQ_FSCAN=$o timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/fs_c3_$o.json
  python -c "import json; d=json.load(open('gpurun_out/fs_c3_$o.json')); print('c3 fscan=$o', '%.4e'%d['value'], d['ms_per_step'], d['gpu_launches'])"
done; done
timeout 900 python -m pytest -q -x -m gpu tests/test_parity_2d_gpu.py tests/test_determinism_gpu.py 2>&1 | tail -2
