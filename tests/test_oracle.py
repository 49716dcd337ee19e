"""The C oracle (oracle/finom_oracle.c) against the reference's own outputs.

CPU only.  The golden fixtures were produced by importing the reference
package (tests/golden/make_golden.py).  The oracle restates the reference
in C with libm exp; the reference builds its tables with numpy's SIMD exp,
which differs from libm in the last ulp on a few percent of arguments, so
agreement is ~1e-14 relative rather than bitwise ("Oracle").
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden, rel_inf
from oracle import oracle as O

GX = np.array([1.0, 3.0, 7.0, 9.0, 12.0])
GY = np.array([2.0, 5.0, 6.0, 9.0, 10.0])


def test_dividing_index_golden():
    """kernel1d.py:55-62 on the paper's worked example (test_kernel1d.py:12-15)."""
    import ctypes
    z = np.zeros(5, dtype=np.int64)
    O.load().orc_dividing_index(GX.ctypes.data, 5, GY.ctypes.data, 5, z.ctypes.data)
    assert z.tolist() == [0, 1, 3, 4, 5]


def test_worked_example_matvec_vs_dense():
    """K psi on the 5x5 example equals the dense kernel (test_kernel1d.py:160-165)."""
    K = np.exp(-np.abs(np.subtract.outer(GX, GY)))
    psi = np.full(5, 0.2)
    assert rel_inf(O.apply_1d(GX, GY, 1.0, psi, 0), K @ psi) < 1e-15
    assert rel_inf(O.apply_1d(GX, GY, 1.0, psi, 1), K.T @ psi) < 1e-15


def test_kernel_cases_vs_reference():
    g = load_golden("kernel1d_cases.npz")
    for k in range(int(g["ncases"])):
        c = lambda key: g["c%d_%s" % (k, key)]
        eps = float(c("eps"))
        a, b = c("a"), c("b")
        assert rel_inf(O.apply_1d(c("x"), c("y"), eps, c("psi"), 0, a, b), c("Kpsi")) < 1e-13
        assert rel_inf(O.apply_1d(c("x"), c("y"), eps, c("phi"), 1, a, b), c("KTphi")) < 1e-13
        p, q = O.apply_1d(c("x"), c("y"), eps, c("psi"), 2, a, b)
        assert rel_inf(p, c("p")) < 1e-13 and rel_inf(q, c("q")) < 1e-13


def _same_run(r, ref, tol):
    assert r["iterations"] == int(ref["iterations"])
    assert r["converged"] == bool(ref["converged"])
    assert list(r["absorb_its"]) == [int(t) for t in np.atleast_1d(ref["absorb_its"])]
    assert rel_inf(r["phi"], ref["phi"]) < tol and rel_inf(r["psi"], ref["psi"]) < tol
    assert rel_inf(r["a"], ref["a"]) < tol and rel_inf(r["b"], ref["b"]) < tol
    its = [int(t) for t in np.atleast_1d(ref["hist_it"])]
    errs = r["hist"][np.array(its) - 1]
    assert np.all(np.abs(errs - ref["hist_err"]) <= tol * np.abs(ref["hist_err"]) + 1e-14)
    assert abs(r["cost"] - float(ref["cost"])) <= tol * abs(float(ref["cost"]))


def test_solver_cases_vs_reference():
    g = load_golden("solver_cases.npz")
    for k in range(int(g["ncases"])):
        s = lambda key: g["s%d_%s" % (k, key)]
        eps, itr, tol, stab, thr, ce = s("cfg")
        r = O.sinkhorn_1d(s("x"), s("y"), s("u"), s("v"), eps, int(itr), tol, bool(stab), thr,
                          int(ce))
        _same_run(r, {key: s(key) for key in ("phi", "psi", "a", "b", "hist_it", "hist_err",
                                              "iterations", "converged", "absorb_its",
                                              "cost")}, 1e-10)


def test_failure_cases_vs_reference():
    with open(os.path.join(GOLDEN, "failure_cases.json")) as f:
        cases = json.load(f)
    code = {"ZeroDenominator": 1, "NonFiniteIterate": 2}
    for name, c in cases.items():
        r = O.sinkhorn_1d(c["x"], c["y"], c["u"], c["v"], c["eps"], 10)
        assert r["status"] == code[c["raised"]], name


def test_config1_vs_reference():
    from paper_2605_26659_b200 import workloads as W
    x, y, u, v, eps = W.config1()
    _same_run(O.sinkhorn_1d(x, y, u, v, eps, 500, 0.0, True), load_golden("config1.npz"), 1e-10)


def test_config2_n65536_vs_reference():
    from paper_2605_26659_b200 import workloads as W
    x, y, u, v, eps = W.config2(n=1 << 16)
    _same_run(O.sinkhorn_1d(x, y, u, v, eps, 200, 0.0, True), load_golden("config2_n65536.npz"),
              1e-9)


def test_config5_problem0_vs_reference():
    from paper_2605_26659_b200 import workloads as W
    g = load_golden("config5_p0-3.npz")
    x, y, u, v, eps = W.config5_problem(0)
    assert eps == float(g["p0_eps"])
    _same_run(O.sinkhorn_1d(x, y, u, v, eps, 200, 0.0, True),
              {k[3:]: g[k] for k in g if k.startswith("p0_")}, 1e-9)


def test_grid_cases_vs_reference():
    g = load_golden("grid_cases.npz")
    for k in range(int(g["ncases"])):
        c = lambda key: g["g%d_%s" % (k, key)]
        eps, itr, tol, stab, thr, ce = c("cfg")
        r = O.sinkhorn_2d(c("x1"), c("y1"), c("x2"), c("y2"), c("U"), c("V"), eps, int(itr), tol,
                          bool(stab), thr, int(ce))
        _same_run(r, {key: c(key) for key in ("phi", "psi", "a", "b", "hist_it", "hist_err",
                                              "iterations", "converged", "absorb_its",
                                              "cost")}, 1e-9)


def test_config2_full_pins_header():
    """The full-size config-2 pins exist and are self-consistent (3 absorptions)."""
    g = load_golden("config2_full_pins.npz")
    assert int(g["iterations"]) == 200 and g["hist_err"].size == 200
    assert g["absorb_its"].size >= 1 and np.isfinite(g["cost"])
