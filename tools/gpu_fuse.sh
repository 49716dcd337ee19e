# fused short-line sweep (k_sq_fused): bitwise check vs the three kernels, config 3 A/B, 2D tests
timeout 600 python tools/fscan_check.py FB_SQ_FUSE 2>&1 | tail -3
for r in 1 2; do for o in 0 1; do
  FB_SQ_FUSE=$o timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/fu_c3_$o.json
  python -c "import json; d=json.load(open('gpurun_out/fu_c3_$o.json')); print('c3 fuse=$o', '%.4e'%d['value'], d['ms_per_step'], d['gpu_launches'])"
done; done
timeout 900 python -m pytest -q -x -m gpu tests/test_parity_2d_gpu.py tests/test_determinism_gpu.py 2>&1 | tail -2
