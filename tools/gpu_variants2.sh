for v in e8 e4m4 e4m5 e4m6 e4m8; do timeout 300 python tools/variant_check.py paper_2605_26659_b200/libfinom_dbg_$v.so 2>&1 | tail -2; done
