timeout 900 python -m pytest tests/test_parity_2d_gpu.py -q -m gpu -x 2>&1 | tail -5
for c in 3 4; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_c$c.json; python -c "
import json; d=json.load(open('gpurun_out/bench_c$c.json')); print($c, '%.4e' % d['value'], d['ms_per_step'], d.get('e2e',{}) and '%.3e' % d['e2e']['value'])"; done
