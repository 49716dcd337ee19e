bash tools/gpu_ncu_src.sh
# (ncu cannot profile kernel nodes of graphs with conditional nodes: FB_WHILE1D=0 selects the chunk graph)
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ncu_plain.json 2>&1 && \
  FB_WHILE1D=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
