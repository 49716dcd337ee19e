cat > /tmp/dbgv.py << 'PY'
import sys, runpy, os
sys.path.insert(0, os.getcwd())
sys.argv = ['x']
from paper_2605_26659_b200 import _lib
_lib.LIB_PATH = 'paper_2605_26659_b200/libfinom_dbg_nopre.so'
runpy.run_path('tools/dbg_solver_cases.py', run_name='__main__')
PY
timeout 300 python /tmp/dbgv.py 2>&1 | tail -11
