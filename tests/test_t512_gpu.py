"""The 512-element-tile build (libfinom_b200_t512.so, _lib.lib_for: a few
large problems) against the same reference fixtures and oracle checks as the
default build -- forced here (FINOM_TILE=512) on the small cases; the
full-size config 2 test of test_parity_gpu.py selects it by itself."""

import pytest

import test_parity_gpu as T

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def t512(monkeypatch):
    monkeypatch.setenv("FINOM_TILE", "512")
    from paper_2605_26659_b200 import _lib
    assert _lib.use_t512(1, 10)


def test_t512_kernel_cases_vs_reference():
    T.test_kernel_cases_vs_reference()


def test_t512_apply_multitile_vs_oracle():
    T.test_apply_multitile_vs_oracle()


def test_t512_ties_every_node():
    T.test_ties_every_node()


def test_t512_solver_cases_vs_reference():
    T.test_solver_cases_vs_reference()


def test_t512_failure_diagnostics():
    T.test_failure_diagnostics()


def test_t512_config1_vs_reference():
    T.test_config1_vs_reference()


def test_t512_config2_n65536_vs_reference():
    T.test_config2_n65536_vs_reference()


def test_t512_adapter_protocol_under_driver():
    T.test_adapter_protocol_under_driver()


def test_t512_selected_for_config2():
    import numpy as np
    import paper_2605_26659_b200 as fb
    from paper_2605_26659_b200 import workloads as W
    x, y, u, v, eps = W.config2(n=1 << 20)
    bs = fb.BatchSolver1D([x], [y], [u], [v], [eps])
    assert "TILE=512" in bs.plan.lib.finom_build_info().decode()
    assert bs.plan.info()["tile"] == 512
    st = bs.solve(3)
    assert st == 0 and np.all(np.isfinite(bs.phi.cpu().numpy()))
