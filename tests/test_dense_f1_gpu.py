"""SURVEY 8(f) row f1 on the device: dense_realization (1D / 2D), plan_dense
and marginal_error against the reference's own values
(tests/golden/dense_cases.npz, make_golden.py dense_cases)."""

import numpy as np
import pytest

import paper_2605_26659_b200 as fb
from paper_2605_26659_b200 import kernel1d as k1
from paper_2605_26659_b200 import kernel2d as k2

from conftest import load_golden, rel_elem, rel_inf

pytestmark = pytest.mark.gpu
TOL = 1e-9


def test_dense_realization_1d_vs_reference():
    g = load_golden("dense_cases.npz")
    op = k1.build_operator(fb.Mesh1D(g["r1_x"]), fb.Mesh1D(g["r1_y"]), float(g["r1_eps"]))
    op = op.absorb(g["r1_a"], g["r1_b"])
    d = op.dense_realization()
    assert d.shape == g["r1_dense"].shape
    # the same exponent, evaluated in the same order; exp within an ulp or two
    assert rel_elem(d, g["r1_dense"]) < 1e-14


def test_plan_dense_and_marginal_error_vs_reference():
    g = load_golden("dense_cases.npz")
    x, y, u, v, eps = g["s1_x"], g["s1_y"], g["s1_u"], g["s1_v"], float(g["s1_eps"])
    cfg = fb.SolverConfig(epsilon=eps, itr_max=40, tol=0.0, stabilize=True, absorb_threshold=6.0)
    sol = fb.sinkhorn_1d(fb.Mesh1D(x), fb.Mesh1D(y), fb.Measure(u), fb.Measure(v), cfg)
    assert rel_inf(sol.a, g["s1_a"]) < TOL or np.max(np.abs(sol.a - g["s1_a"])) < 1e-12
    # our solve's plan and residual vs the reference's (solver tolerance)
    plan = fb.plan_dense(sol)
    assert rel_inf(plan, g["s1_plan"]) < TOL
    me = fb.marginal_error(sol, sol.kernel, fb.Measure(v))
    assert abs(me - float(g["s1_marg"])) <= TOL * abs(float(g["s1_marg"])) + 1e-15
    # the reference's own state through our device operators: tighter
    op = k1.KernelOperator1D(fb.Mesh1D(x), fb.Mesh1D(y), eps, g["s1_a"], g["s1_b"],
                             k1._PlanCache(fb.Mesh1D(x), fb.Mesh1D(y), eps))
    st = fb.Solution(phi=g["s1_phi"], psi=g["s1_psi"], a=g["s1_a"], b=g["s1_b"], kernel=op,
                     iterations_run=40, converged=False, marginal_error_history=[],
                     wall_time=0.0, setup_time=0.0, cost=0.0, config=cfg)
    assert rel_elem(fb.plan_dense(st), g["s1_plan"], 1e-300) < 1e-13
    assert rel_elem(op.dense_realization(), g["s1_dense"], 1e-300) < 1e-14
    me2 = fb.marginal_error(st, op, fb.Measure(v))
    assert abs(me2 - float(g["s1_marg"])) <= 1e-12 * abs(float(g["s1_marg"])) + 1e-16


def test_plan_dense_cap():
    x = np.linspace(0, 1, 50)
    u = np.full(50, 1 / 50)
    cfg = fb.SolverConfig(epsilon=0.1, itr_max=5, tol=0.0, plan_cap=100)
    sol = fb.sinkhorn_1d(fb.Mesh1D(x), fb.Mesh1D(x), fb.Measure(u), fb.Measure(u), cfg)
    with pytest.raises(fb.SizeCapExceeded):
        fb.plan_dense(sol)


def test_dense_realization_2d_vs_reference():
    g = load_golden("dense_cases.npz")
    src = fb.Grid2D(fb.Mesh1D(g["g_x1"]), fb.Mesh1D(g["g_y1"]))
    tgt = fb.Grid2D(fb.Mesh1D(g["g_x2"]), fb.Mesh1D(g["g_y2"]))
    op = k2.build_operator_2d(src, tgt, float(g["g_eps"]))
    assert rel_elem(op.dense_realization(), g["g_dense"]) < 1e-14
    opa = op.absorb(g["g_A"], g["g_B"])
    assert rel_elem(opa.dense_realization(), g["g_dense_abs"]) < 1e-14
