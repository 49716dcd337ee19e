timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
FB_WHILE1D=0 timeout 900 python -m pytest tests/test_parity_gpu.py -q -m gpu -x 2>&1 | tail -2
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>gpurun_out/bench.err | tail -1 > gpurun_out/bench_q.json
python -c "
import json; d=json.load(open('gpurun_out/bench_q.json')); r=d['roofline']; print('%.4e' % d['value'], d['ms_per_step'], 'frac %.3f' % r['frac'], 'e2e %.3e' % d['e2e']['value'], d['gpu_launches'])"
FB_WHILE1D=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-120
timeout 600 python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-120
