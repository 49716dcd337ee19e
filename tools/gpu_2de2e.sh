timeout 900 python -m pytest tests/test_parity_2d_gpu.py tests/test_dense_gpu.py -q -m gpu -x 2>&1 | tail -2
FB_VERBOSE=1 timeout 600 python tools/e2e_2d_probe.py 2>&1 | grep -E "e2e|total" | tail -3
timeout 900 python bench.py --config 4 --steps 3 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4e'%d['value'], 'e2e %.3e'%d['e2e']['value'])"
