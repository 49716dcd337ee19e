timeout 1200 python tools/line_check.py chain 2>&1 | tail -5
for spec in ${SPECS:-"0 0" "1 0" "1 6" "1 12" "1 24"}; do
  set -- $spec
  FB_SQ_CHAIN=$1 FB_SQ_CHK=$2 timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline 2>gpurun_out/chain_c4.err | tail -1 > gpurun_out/chain_c4_$1_$2.json
  python -c "import json; d=json.load(open('gpurun_out/chain_c4_$1_$2.json')); print('c4 chain=$1 K=$2', '%.4e'%d['value'], d['ms_per_step'], '%.4e'%d['e2e']['value'], d['roofline']['frac'], d['gpu_launches'])" || tail -5 gpurun_out/chain_c4.err
done
