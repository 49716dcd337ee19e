# cluster line sweep: L2 prefetch distance A/B at config 4
for spec in "0 0" "44 0" "44 16" "44 32" "24 32" "42 32"; do
  set -- $spec
  FB_SQ_LINE=$1 FB_SQ_PF=$2 timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline 2>gpurun_out/line_c4.err | tail -1 > gpurun_out/line_c4_$1_$2.json
  python -c "import json; d=json.load(open('gpurun_out/line_c4_$1_$2.json')); print('c4 line=$1 pf=$2', '%.4e'%d['value'], d['ms_per_step'], '%.4e'%d['e2e']['value'], d['roofline']['frac'], d['gpu_launches'])" || tail -5 gpurun_out/line_c4.err
done
