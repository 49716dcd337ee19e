bash tools/gpu_iter.sh
python tools/phase_time.py paper_2605_26659_b200/libfinom_dbg_PHASE.so 2>&1 | tail -14
