"""The batched API's pipeline (sinkhorn_1d_batched in stages: plan + staging of
stage k + 1 and results of stage k - 1 around stage k's device loop) gives
exactly the single-stage results, problem by problem, and the oracle's."""

import numpy as np
import pytest

import paper_2605_26659_b200 as fb
from paper_2605_26659_b200 import errors as E
from paper_2605_26659_b200 import solver as S
from paper_2605_26659_b200 import workloads as W
from oracle import oracle as O

def _batch(B, n):
    probs = W.config5(batch=B, problems=range(B), n=n)
    return ([fb.Mesh1D(p[0]) for p in probs], [fb.Mesh1D(p[1]) for p in probs],
            [fb.Measure(p[2]) for p in probs], [fb.Measure(p[3]) for p in probs],
            [p[4] for p in probs], probs)


def test_stage_ranges():
    sizes = np.full(8192, 16384)
    r = S._pipeline_ranges(sizes)
    # short first / last stages (two rounds of resident problems) around equal middle stages
    assert r == [(0, 592), (592, 1776), (1776, 4688), (4688, 7600), (7600, 8192)]
    r = S._pipeline_ranges(np.full(2048, 16384))  # (a rank of a 4-way split)
    assert r == [(0, 296), (296, 888), (888, 1752), (1752, 2048)]
    assert S._pipeline_ranges(np.full(1024, 16384)) == [(0, 296), (296, 728), (728, 1024)]
    for P in (1024, 1500, 4096, 5000, 8192, 20000):  # contiguous, complete, non-empty
        r = S._pipeline_ranges(np.full(P, 16384))
        assert r[0][0] == 0 and r[-1][1] == P and all(lo < hi for lo, hi in r)
        assert all(a[1] == b[0] for a, b in zip(r[:-1], r[1:]))
    assert S._pipeline_ranges(np.full(1000, 16384)) == [(0, 1000)]
    assert S._pipeline_ranges(np.full(2048, 1000)) == [(0, 2048)]  # (few points: one stage)
    r = S._pipeline_ranges(np.full(100000, 200))  # (many small problems: equal stages)
    assert len(r) == 4 and r[0] == (0, 25000) and r[-1] == (75000, 100000)
    assert S._pipeline_ranges(np.full(40, 1000)) == [(0, 40)]


def test_stage_ranges_overrides(monkeypatch):
    sizes = np.full(8192, 16384)
    monkeypatch.setenv("FINOM_PIPE_STAGES", "4")
    r = S._pipeline_ranges(sizes)
    assert len(r) == 4 and r[0] == (0, 2048) and r[-1] == (6144, 8192)
    monkeypatch.setenv("FINOM_PIPE_FIRST", "256")
    r = S._pipeline_ranges(sizes)
    assert len(r) == 5 and r[0] == (0, 256) and r[-1][1] == 8192
    monkeypatch.setenv("FINOM_PIPE_SIZES", "100,200,300")
    assert S._pipeline_ranges(sizes) == [(0, 100), (100, 300), (300, 8192)]


@pytest.mark.gpu
@pytest.mark.parametrize("stages", ["3", "5", "sizes:2,4,19,9,3"])
def test_pipeline_matches_single_stage(monkeypatch, stages):
    xs, ys, us, vs, eps, probs = _batch(37, 1500)
    cfg = fb.SolverConfig(epsilon=1.0, itr_max=60, tol=0.0, stabilize=True, absorb_threshold=30.0)
    monkeypatch.setenv("FINOM_PIPE_STAGES", "1")
    one = fb.sinkhorn_1d_batched(xs, ys, us, vs, cfg, epsilons=eps)
    if stages.startswith("sizes:"):  # short first / last stages (the default shape of large batches)
        monkeypatch.delenv("FINOM_PIPE_STAGES")
        monkeypatch.setenv("FINOM_PIPE_SIZES", stages[6:])
        assert S._pipeline_ranges(np.full(37, 1500)) == [(0, 2), (2, 6), (6, 25), (25, 34), (34, 37)]
    else:
        monkeypatch.setenv("FINOM_PIPE_STAGES", stages)
    many = fb.sinkhorn_1d_batched(xs, ys, us, vs, cfg, epsilons=eps)
    assert np.array_equal(one.phi, many.phi) and np.array_equal(one.psi, many.psi)
    assert np.array_equal(one.a, many.a) and np.array_equal(one.b, many.b)
    for p in range(len(xs)):
        s1, s2 = one[p], many[p]
        assert s1.iterations_run == s2.iterations_run == 60
        assert list(s1.absorb_iterations) == list(s2.absorb_iterations)
        assert s1.cost == s2.cost
        assert list(s1.marginal_error_history) == list(s2.marginal_error_history)
    # and against the oracle for a few problems (different stages)
    for p in (0, 18, 36):
        x, y, u, v, e = probs[p]
        r = O.sinkhorn_1d(x, y, u, v, e, 60, 0.0, True, 30.0)
        s = many[p]
        assert list(s.absorb_iterations) == list(r["absorb_its"])
        assert np.max(np.abs(s.phi - r["phi"])) <= 1e-9 * np.max(np.abs(r["phi"]))
        assert abs(s.cost - r["cost"]) <= 1e-9 * abs(r["cost"])


@pytest.mark.gpu
def test_pipeline_failure_raises(monkeypatch):
    """A failing problem in a later stage raises the reference's exception."""
    xs, ys, us, vs, eps, _ = _batch(9, 800)
    cfg = fb.SolverConfig(epsilon=1.0, itr_max=30, tol=0.0, stabilize=False)
    eps = list(eps)
    eps[7] = 1e-9  # every kernel entry underflows: K v = 0 at positive mass
    monkeypatch.setenv("FINOM_PIPE_STAGES", "3")
    with pytest.raises((E.ZeroDenominator, E.NonFiniteIterate)):
        fb.sinkhorn_1d_batched(xs, ys, us, vs, cfg, epsilons=eps)
