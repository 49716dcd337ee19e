set -x
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -20
python -m pytest tests/test_parity_gpu.py -q -m gpu -s 2>&1 | tail -30
