# Round measurement: GPU tests, smoke, bench lines (configs 1-5), reference arm,
# launch list of config 2, ncu --set full of k_step (config 2), launch lists of configs 3/4.
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -1 gpurun_out/bench.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1; tail -1 gpurun_out/bench_ref.json | cut -c1-200
for c in 1 3 4; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench_c$c.json; cut -c1-160 gpurun_out/bench_c$c.json; done
FINOM_BATCH=8192 timeout 1500 python bench.py --config 5 --steps 2 --warmup 3 2>/dev/null | tail -1 > gpurun_out/bench_c5.json; cut -c1-160 gpurun_out/bench_c5.json
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ncu_plain.json 2>&1 && \
  FB_WHILE1D=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
python tools/launch_summary.py gpurun_out/launches.csv | head -12
export ITERS=3
timeout 600 python tools/ncu_target.py > gpurun_out/plain.log 2>&1 && \
  FB_WHILE1D=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step -s 2 -c 2 -o gpurun_out/prof_kstep python tools/ncu_target.py > gpurun_out/ncu2.log 2>&1; echo "ncu rc=$?"
CFG=3 ITERS=6 FB_GRAPH2D=0 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launch3.csv python tools/ncu_2d_target.py > /dev/null 2>&1; echo rc3=$?
CFG=4 ITERS=10 FB_GRAPH2D=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launch4.csv python tools/ncu_2d_target.py > /dev/null 2>&1; echo rc4=$?
timeout 600 python tools/dense_vs_fast.py > gpurun_out/dense_vs_fast.txt 2>&1; cat gpurun_out/dense_vs_fast.txt | tail -4
FB_VERBOSE=1 timeout 300 python tools/e2e_probe.py > gpurun_out/e2e_probe.txt 2>&1; tail -4 gpurun_out/e2e_probe.txt
