# session-3 state check: GPU tests, smoke, default bench line (config 5), config 4 line
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -5 > gpurun_out/c_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c_smoke.txt 2>&1; echo smoke $? >> gpurun_out/c_smoke.txt
timeout 600 python bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/c_bench5.json 2>gpurun_out/c_bench5.err
timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c_bench4.json 2>gpurun_out/c_bench4.err
tail -3 gpurun_out/c_pytest.txt; tail -2 gpurun_out/c_smoke.txt; cat gpurun_out/c_bench5.json gpurun_out/c_bench4.json
