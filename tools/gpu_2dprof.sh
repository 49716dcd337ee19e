# launch lists of configs 3 and 4 (3 iterations), plus an ncu --set full of the square sweep apply on config 4
CFG=3 ITERS=6 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launch3.csv python tools/ncu_2d_target.py > /dev/null 2>&1; echo rc3=$?
python tools/launch_summary.py gpurun_out/launch3.csv | head -20
CFG=4 ITERS=3 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launch4.csv python tools/ncu_2d_target.py > /dev/null 2>&1; echo rc4=$?
python tools/launch_summary.py gpurun_out/launch4.csv | head -20
