timeout 90 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
timeout 120 python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-160
FB_SMALL=0 timeout 120 python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-160
