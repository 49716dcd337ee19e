for f in paper_2605_26659_b200/libfinom_b200.so paper_2605_26659_b200/libfinom_dbg_*.so; do python tools/variant_time.py $f 2>&1 | tail -1; done
