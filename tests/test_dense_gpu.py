"""Dense GPU Sinkhorn baseline (reference dense.py:161-193)
against the O(N) path and the C oracle on small problems (1e-9 relative)."""

import numpy as np
import pytest

import paper_2605_26659_b200 as fb
from paper_2605_26659_b200 import dense as D
from paper_2605_26659_b200 import workloads as W

from conftest import rel_inf

pytestmark = pytest.mark.gpu
TOL = 1e-9


@pytest.mark.parametrize("stabilize,thr", [(False, 200.0), (True, 5.0)])
def test_dense_sinkhorn_1d_vs_fast_and_oracle(stabilize, thr):
    from oracle import oracle as O
    x, y, u, v, eps = W.config1(n=700)
    cfg = fb.SolverConfig(epsilon=eps, itr_max=80, tol=0.0, stabilize=stabilize,
                          absorb_threshold=thr)
    X, Y, U, V = fb.Mesh1D(x), fb.Mesh1D(y), fb.Measure(u), fb.Measure(v)
    dn = D.dense_sinkhorn(fb.Problem(X, Y, U, V), cfg)
    fast = fb.sinkhorn_1d(X, Y, U, V, cfg)
    ref = O.sinkhorn_1d(x, y, u, v, eps, 80, 0.0, stabilize, thr)
    assert dn.iterations_run == fast.iterations_run == 80
    assert list(dn.absorb_iterations) == list(fast.absorb_iterations) == list(ref["absorb_its"])
    for got in (dn.phi, fast.phi):
        assert rel_inf(got, ref["phi"]) < TOL
    assert rel_inf(dn.psi, ref["psi"]) < TOL
    assert abs(dn.cost - ref["cost"]) <= TOL * abs(ref["cost"])
    errs = np.array([e for _, e in dn.marginal_error_history])
    errs_f = np.array([e for _, e in fast.marginal_error_history])
    assert np.max(np.abs(errs - errs_f) / (TOL * np.abs(errs_f) + 1e-12)) <= 1.0
    # the materialized plan of the dense run against the O(N) run's
    plan_d = dn.phi[:, None] * dn.kernel.dense_realization() * dn.psi[None, :]
    plan_f = fb.plan_dense(fast)
    assert D.frobenius_diff(plan_d, plan_f) <= TOL * np.linalg.norm(plan_f)


def test_dense_sinkhorn_2d_vs_fast():
    x1, y1, x2, y2, U, V, eps = W.config3(n=24)
    cfg = fb.SolverConfig(epsilon=eps, itr_max=40, tol=0.0, stabilize=True, absorb_threshold=8.0)
    src = fb.Grid2D(fb.Mesh1D(x1), fb.Mesh1D(y1))
    tgt = fb.Grid2D(fb.Mesh1D(x2), fb.Mesh1D(y2))
    mu, mv = fb.Measure2D(U), fb.Measure2D(V)
    dn = D.dense_sinkhorn(fb.Problem(src, tgt, mu, mv), cfg)
    fast = fb.sinkhorn_2d(src, tgt, mu, mv, cfg)
    assert dn.iterations_run == fast.iterations_run
    assert rel_inf(dn.phi, np.ravel(fast.phi, order="F") if np.ndim(fast.phi) == 2 else fast.phi) < TOL
    assert abs(dn.cost - fast.cost) <= TOL * abs(fast.cost)


def test_dense_errors():
    x = fb.Mesh1D(np.linspace(0.0, 1.0, 40))
    with pytest.raises(fb.SizeCapExceeded):
        D.dense_kernel(x, x, 0.1, size_cap=100)
    with pytest.raises(fb.InvalidEpsilon):
        D.dense_kernel(x, x, -1.0)
    with pytest.raises(fb.DimensionMismatch):
        D.frobenius_diff(np.zeros((2, 3)), np.zeros((3, 2)))
