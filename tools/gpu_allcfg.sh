for c in 1 3 4; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_c$c.json; python -c "
import json; d=json.load(open('gpurun_out/bench_c$c.json')); print($c, '%.3e' % d['value'], d['ms_per_step'], d.get('e2e',{}) and '%.3e' % d['e2e']['value'])"; done
FINOM_BATCH=8192 timeout 1200 python bench.py --config 5 --steps 2 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_c5.json; python -c "
import json; d=json.load(open('gpurun_out/bench_c5.json')); print(5, '%.3e' % d['value'], d['ms_per_step'], d['roofline']['frac'])"
