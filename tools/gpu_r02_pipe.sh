#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_pipeline_gpu.py tests/test_group_gpu.py tests/test_parity_gpu.py -q -x > gpurun_out/pytest_pipe.txt 2>&1; tail -3 gpurun_out/pytest_pipe.txt
FB_VERBOSE=1 timeout 900 python tools/e2e5_stages.py 1 4 8 16 > gpurun_out/e2e5_stages.txt 2>&1; grep -v finom gpurun_out/e2e5_stages.txt | tail -12
