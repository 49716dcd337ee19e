FB_PERSIST=1 timeout 600 python -m pytest tests/test_parity_gpu.py -q -m gpu -x 2>&1 | tail -2
for v in 0 1; do FB_PERSIST=$v timeout 100 python tools/variant_time.py paper_2605_26659_b200/libfinom_b200.so 2>&1 | tail -1; FB_PERSIST=$v timeout 100 python tools/variant_solve.py paper_2605_26659_b200/libfinom_b200.so 2>&1 | tail -1; done
