# 2D on-the-fly factors: GPU tests, then config 4 / config 3 A/B (FB_SQ_OTF=0 vs 1)
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -5 > gpurun_out/otf_pytest.txt
for r in 1 2; do
for o in 0 1; do
  FB_SQ_OTF=$o timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/otf_c4_$o.json
  python -c "import json; d=json.load(open('gpurun_out/otf_c4_$o.json')); print('c4 otf=$o', '%.4e'%d['value'], d['ms_per_step'], d['e2e']['value'])"
  FB_SQ_OTF=$o timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/otf_c3_$o.json
  python -c "import json; d=json.load(open('gpurun_out/otf_c3_$o.json')); print('c3 otf=$o', '%.4e'%d['value'], d['ms_per_step'])"
done
done
cat gpurun_out/otf_pytest.txt
