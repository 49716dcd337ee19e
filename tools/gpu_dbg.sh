timeout 300 python -m pytest tests/test_parity_gpu.py -q -m gpu -x -k "apply_multitile or kernel_cases" 2>&1 | grep -E "^E|assert|rel_inf|Error" | head -20
python - << 'PY'
import sys, numpy as np
sys.path.insert(0, '.')
import paper_2605_26659_b200 as fb
from paper_2605_26659_b200 import kernel1d as k1
from oracle import oracle as O
rng = np.random.default_rng(3)
for n, m, eps in [(5000, 3000, 0.01), (20000, 20000, 1e-3), (777, 4096, 0.05), (1, 9000, 0.1), (9000, 1, 0.1), (30, 20, 0.1)]:
    x = np.sort(rng.uniform(0, 1, n)); y = np.sort(rng.uniform(0, 1, m))
    psi, phi = rng.random(m), rng.random(n)
    op = k1.build_operator(fb.Mesh1D(x), fb.Mesh1D(y), eps)
    a = op.apply(psi); r = O.apply_1d(x, y, eps, psi, 0)
    at = op.apply_transpose(phi); rt = O.apply_1d(x, y, eps, phi, 1)
    p, q = k1.apply_blocks(op, psi); rp, rq = O.apply_1d(x, y, eps, psi, 2)
    e = lambda u, v: np.max(np.abs(u - v)) / np.max(np.abs(v))
    bad = np.argmax(np.abs(a - r))
    print(n, m, "apply %.2e T %.2e p %.2e q %.2e" % (e(a, r), e(at, rt), e(p, rp), e(q, rq)), "worst idx", bad, a[bad], r[bad])
PY
