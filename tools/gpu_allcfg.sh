for c in 1 2 3 4; do timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-600; done
FINOM_BATCH=1024 timeout 900 python bench.py --config 5 --steps 2 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-600
timeout 900 python -m pytest tests/test_parity_2d_gpu.py -q -m gpu -s -k config3 2>&1 | grep -E "parity|passed|failed"
