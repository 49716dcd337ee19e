timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
FB_VERBOSE=1 timeout 300 python tools/e2e_probe.py 2>&1 | grep -E "e2e|total" | tail -2
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4e'%d['value'], 'e2e %.4e'%d['e2e']['value'])"
