for v in 1; do FB_TAB2D=$v timeout 600 python bench.py --config 4 --steps 2 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-150; done
CFG=3 ITERS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch2d.csv python tools/ncu_2d_target.py > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/launch2d.csv | head -14
