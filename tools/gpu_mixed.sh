cat > /tmp/mixed.py << 'PY'
import sys
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
from paper_2605_26659_b200 import _lib
_lib.LIB_PATH = sys.argv[1]
import test_parity_gpu as T
try:
    T.test_batched_mixed_sizes_vs_oracle()
    print(sys.argv[1], "mixed OK")
except Exception as e:
    print(sys.argv[1], "mixed FAIL", str(e)[:200])
PY
for f in paper_2605_26659_b200/libfinom_dbg_head.so paper_2605_26659_b200/libfinom_b200.so; do timeout 120 python /tmp/mixed.py $f 2>&1 | tail -1; done
