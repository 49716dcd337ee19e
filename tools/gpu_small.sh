timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
FB_SMALL=0 timeout 900 python -m pytest tests/test_parity_gpu.py -q -m gpu -x 2>&1 | tail -2
for c in 1; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-200; done
FB_SMALL=0 timeout 900 python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-200
