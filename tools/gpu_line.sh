# cluster line sweep: parity vs the three-kernel path, config 4 A/B per variant
timeout 900 python tools/line_check.py 44 24 42 2>&1 | tail -14
for v in 0 44 24 42; do
  FB_SQ_LINE=$v timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline 2>gpurun_out/line_c4_$v.err | tail -1 > gpurun_out/line_c4_$v.json
  python -c "import json; d=json.load(open('gpurun_out/line_c4_$v.json')); print('c4 line=$v', '%.4e'%d['value'], d['ms_per_step'], '%.4e'%d['e2e']['value'], d['roofline']['frac'], d['gpu_launches'])" || tail -5 gpurun_out/line_c4_$v.err
done
