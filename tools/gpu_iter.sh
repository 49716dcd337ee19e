# quick loop: smoke + parity tests + bench (no cpu baseline)
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity_2d_gpu.py -q -m gpu -s -x 2>&1 | grep -E "passed|failed|Error|error|parity|^E " | head -20
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -2 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l); continue
    r=d['roofline']; print('value %.3e ms/step %.2f frac %.3f halfA %.3f halfB %.3f absorb %.3f e2e %.3e' % (d['value'], d['ms_per_step'], r['frac'], r['ms_half_a'], r['ms_half_b'], r['ms_absorb'], d['e2e']['value']))"
