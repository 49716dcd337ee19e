timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2; echo "smoke rc=$?"
timeout 300 python -m pytest tests/test_parity_gpu.py -q -m gpu -x 2>&1 | tail -2
for s in 0 1; do FB_STEP=$s timeout 120 python tools/variant_time.py paper_2605_26659_b200/libfinom_b200.so 2>&1 | tail -1; done
