set -x
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -3 gpurun_out/bench.err
cat gpurun_out/bench.json
python bench.py --config 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1.json 2>&1; tail -2 gpurun_out/bench_c1.json
python tools/ncu_target.py > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/ncu_target.py > gpurun_out/ncu1.log 2>&1; echo "ncu1 rc=$?"
python tools/ncu_target.py > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_half -s 2 -c 2 -o gpurun_out/prof_khalf python tools/ncu_target.py > gpurun_out/ncu2.log 2>&1; echo "ncu2 rc=$?"
tail -3 gpurun_out/ncu2.log
