timeout 1200 python -m pytest tests -q -m gpu -k "full or variants or dense" -s 2>&1 | grep -E "parity|passed|failed|Error" | head -20
timeout 600 python tools/dense_vs_fast.py 2>&1 | tail -4
