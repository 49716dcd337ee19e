timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
FB_GRAPH2D=0 timeout 900 python -m pytest tests/test_parity_2d_gpu.py -q -m gpu -x 2>&1 | tail -2
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>gpurun_out/bench.err | tail -1 > gpurun_out/bench_q.json
python -c "
import json; d=json.load(open('gpurun_out/bench_q.json')); r=d['roofline']; print('%.4e' % d['value'], d['ms_per_step'], 'frac %.3f' % r['frac'], 'A %.1f B %.1f res %.1f abs %.1f us' % (1e3*r['ms_half_a'], 1e3*r['ms_half_b'], 1e3*r['ms_resolve'], 1e3*r['ms_absorb']))"
[ -f paper_2605_26659_b200/libfinom_dbg_res.so ] && timeout 300 python tools/res_time.py paper_2605_26659_b200/libfinom_dbg_res.so 2>&1 | tail -9
