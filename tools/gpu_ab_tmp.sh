timeout 900 python -m pytest tests/test_seg1d.py tests/test_decide2d_gpu.py tests/test_parity_2d_gpu.py -q -x 2>&1 | grep -E "Error|error|assert|FAIL|^E " | head -30
