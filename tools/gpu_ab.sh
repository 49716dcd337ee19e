for r in 1 2; do for v in head new; do timeout 300 python tools/variant_check.py paper_2605_26659_b200/libfinom_dbg_$v.so 2>&1 | tail -1; done; done
