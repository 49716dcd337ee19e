timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
FB_VERBOSE=1 timeout 300 python tools/e2e_probe.py 2>&1 | tail -4
nproc
