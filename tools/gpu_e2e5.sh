timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
FB_VERBOSE=1 timeout 1200 python tools/e2e5_probe.py 2>&1 | grep -v "solve loop\|k_step" | tail -8
