"""CUDA path vs the reference (golden fixtures) and the C oracle.

Tolerances: north star = relative 1e-9 on W1, scaling vectors and
marginal residuals (BASELINE.json); gate on rel-inf as the reference's
tests do (test_solver.py:35-37) and also check elementwise where the
values are not underflow-dominated.
"""

import json
import os

import numpy as np
import pytest

import paper_2605_26659_b200 as fb
from paper_2605_26659_b200 import kernel1d as k1
from paper_2605_26659_b200 import workloads as W

from conftest import GOLDEN, load_golden, rel_elem, rel_inf

pytestmark = pytest.mark.gpu
TOL = 1e-9
# Marginal errors are L1 norms of a unit-mass defect: below ~1e-14 they are
# rounding noise (absolute floor for converged residuals).
ERR_FLOOR = 1e-12


def hist_ok(errs, ref):
    """1e-9 relative on every history entry above the rounding floor.

    Below ~1e-12 an L1 marginal error is dominated by cancellation noise
    (sum_j |psi_j t_j - v_j| with every term at the ulp level); the
    reference's own 1-ulp exponent perturbation moves it by 1.5e-12 at
    config 2, so that is the absolute floor."""
    errs, ref = np.asarray(errs), np.asarray(ref)
    return float(np.max(np.abs(errs - ref) / (TOL * np.abs(ref) + ERR_FLOOR)))


def _oracle():
    from oracle import oracle as O
    return O


def _op(x, y, eps, a=None, b=None):
    op = k1.build_operator(fb.Mesh1D(x), fb.Mesh1D(y), eps)
    if a is not None and (np.any(a != 0) or np.any(b != 0)):
        op = op.absorb(a, b)
    return op


def test_kernel_cases_vs_reference():
    g = load_golden("kernel1d_cases.npz")
    for k in range(int(g["ncases"])):
        c = lambda key: g["c%d_%s" % (k, key)]
        op = _op(c("x"), c("y"), float(c("eps")), c("a"), c("b"))
        assert rel_inf(op.apply(c("psi")), c("Kpsi")) < 1e-12, k
        assert rel_inf(op.apply_transpose(c("phi")), c("KTphi")) < 1e-12, k
        p, q = k1.apply_blocks(op, c("psi"))
        assert rel_inf(p, c("p")) < 1e-12 and rel_inf(q, c("q")) < 1e-12, k


def test_apply_multitile_vs_oracle():
    O = _oracle()
    rng = np.random.default_rng(3)
    for n, m, eps in [(5000, 3000, 0.01), (20000, 20000, 1e-3), (777, 4096, 0.05),
                      (1, 9000, 0.1), (9000, 1, 0.1)]:
        x = np.sort(rng.uniform(0, 1, n))
        y = np.sort(rng.uniform(0, 1, m))
        psi, phi = rng.random(m), rng.random(n)
        a = rng.normal(0, 1, n) * eps
        b = rng.normal(0, 1, m) * eps
        for aa, bb in [(None, None), (a, b)]:
            op = _op(x, y, eps, aa, bb)
            assert rel_inf(op.apply(psi), O.apply_1d(x, y, eps, psi, 0, aa, bb)) < 1e-12
            assert rel_inf(op.apply_transpose(phi), O.apply_1d(x, y, eps, phi, 1, aa, bb)) < 1e-12


def test_ties_every_node():
    O = _oracle()
    x = np.sort(np.random.default_rng(1).uniform(0, 1, 6000))
    op = _op(x, x.copy(), 0.02)
    psi = np.random.default_rng(2).random(6000)
    assert rel_inf(op.apply(psi), O.apply_1d(x, x, 0.02, psi, 0)) < 1e-12


def _check_solution(sol, r, tol=TOL):
    m = dict(
        iterations=(sol.iterations_run, int(r["iterations"])),
        converged=(bool(sol.converged), bool(r["converged"])),
        absorbs=(list(sol.absorb_iterations), [int(t) for t in np.atleast_1d(r["absorb_its"])]),
        hist_its=([h[0] for h in sol.marginal_error_history],
                  [int(t) for t in np.atleast_1d(r["hist_it"])]),
    )
    q = dict(
        phi=rel_inf(sol.phi, r["phi"]), psi=rel_inf(sol.psi, r["psi"]),
        a=rel_inf(sol.a, r["a"]), b=rel_inf(sol.b, r["b"]),
        cost=abs(sol.cost - float(r["cost"])) / abs(float(r["cost"])),
        hist=hist_ok([h[1] for h in sol.marginal_error_history], r["hist_err"]),
    )
    bad = {k: v for k, v in m.items() if v[0] != v[1]}
    bad.update({k: v for k, v in q.items() if not v < (1.0 if k == "hist" else tol)})
    assert not bad, (bad, q)
    return q


def test_solver_cases_vs_reference():
    g = load_golden("solver_cases.npz")
    for k in range(int(g["ncases"])):
        s = lambda key: g["s%d_%s" % (k, key)]
        eps, itr, tol, stab, thr, ce = s("cfg")
        cfg = fb.SolverConfig(epsilon=eps, itr_max=int(itr), tol=tol, stabilize=bool(stab),
                              absorb_threshold=thr, check_every=int(ce))
        sol = fb.sinkhorn_1d(fb.Mesh1D(s("x")), fb.Mesh1D(s("y")), fb.Measure(s("u")),
                             fb.Measure(s("v")), cfg)
        r = {key: s(key) for key in ("phi", "psi", "a", "b", "hist_it", "hist_err", "iterations",
                                     "converged", "absorb_its", "cost")}
        _check_solution(sol, r)


def test_failure_diagnostics():
    with open(os.path.join(GOLDEN, "failure_cases.json")) as f:
        cases = json.load(f)
    for name, c in cases.items():
        exc = getattr(fb.errors, c["raised"])
        with pytest.raises(exc) as info:
            fb.sinkhorn_1d(fb.Mesh1D(c["x"]), fb.Mesh1D(c["y"]), fb.Measure(c["u"]),
                           fb.Measure(c["v"]), fb.SolverConfig(epsilon=c["eps"], itr_max=10,
                                                               tol=0.0))
        assert str(info.value) == c["message"]


def _run_cfg(x, y, u, v, eps, itr):
    cfg = fb.SolverConfig(epsilon=eps, itr_max=itr, tol=0.0, stabilize=True)
    return fb.sinkhorn_1d(fb.Mesh1D(x), fb.Mesh1D(y), fb.Measure(u), fb.Measure(v), cfg)


def test_config1_vs_reference():
    x, y, u, v, eps = W.config1()
    _check_solution(_run_cfg(x, y, u, v, eps, 500), load_golden("config1.npz"))


def test_config2_n65536_vs_reference():
    x, y, u, v, eps = W.config2(n=1 << 16)
    _check_solution(_run_cfg(x, y, u, v, eps, 200), load_golden("config2_n65536.npz"))


def test_config2_full_vs_reference_pins():
    g = load_golden("config2_full_pins.npz")
    x, y, u, v, eps = W.config2()
    sol = _run_cfg(x, y, u, v, eps, 200)
    st = int(g["stride"])
    assert list(sol.absorb_iterations) == [int(t) for t in g["absorb_its"]]
    assert abs(sol.cost - float(g["cost"])) <= TOL * abs(float(g["cost"]))
    pot = lambda s, a: eps * np.log(s) + a
    q = dict(
        hist=hist_ok([h[1] for h in sol.marginal_error_history], g["hist_err"]),
        phi=rel_inf(sol.phi[::st], g["phi_s"]), psi=rel_inf(sol.psi[::st], g["psi_s"]),
        phi_elem=rel_elem(sol.phi[::st], g["phi_s"]), psi_elem=rel_elem(sol.psi[::st], g["psi_s"]),
        # gauge-invariant potentials eps*log(phi) + a (absolute, cost units)
        pot=float(np.max(np.abs(pot(sol.phi[::st], sol.a[::st]) - pot(g["phi_s"], g["a_s"])))),
        cost=abs(sol.cost - float(g["cost"])) / abs(float(g["cost"])))
    print("config2 full parity", q)
    assert q["hist"] < 1 and q["phi"] < TOL and q["psi"] < TOL and q["pot"] < 1e-9, q


def test_config5_subset_batched_vs_reference():
    g = load_golden("config5_p0-3.npz")
    probs = W.config5(problems=[0, 1, 2, 3])
    cfg = fb.SolverConfig(epsilon=1.0, itr_max=200, tol=0.0, stabilize=True)
    sols = fb.sinkhorn_1d_batched([fb.Mesh1D(p[0]) for p in probs],
                                  [fb.Mesh1D(p[1]) for p in probs],
                                  [fb.Measure(p[2]) for p in probs],
                                  [fb.Measure(p[3]) for p in probs], cfg,
                                  epsilons=[p[4] for p in probs])
    for k, sol in enumerate(sols):
        r = {key: g["p%d_%s" % (k, key)] for key in (
            "phi", "psi", "a", "b", "hist_it", "hist_err", "iterations", "converged",
            "absorb_its", "cost")}
        _check_solution(sol, r)


def test_batched_mixed_sizes_vs_oracle():
    O = _oracle()
    rng = np.random.default_rng(11)
    xs, ys, us, vs, es = [], [], [], [], []
    for p in range(7):
        n, m = int(rng.integers(1, 3000)), int(rng.integers(1, 3000))
        xs.append(np.sort(rng.uniform(0, 1, n)))
        ys.append(np.sort(rng.uniform(0, 1, m)))
        uu, vv = rng.random(n) + 1e-3, rng.random(m) + 1e-3
        us.append(uu / uu.sum())
        vs.append(vv / vv.sum())
        es.append(float(10 ** rng.uniform(-2.5, -1)))
    cfg = fb.SolverConfig(epsilon=1.0, itr_max=120, tol=0.0, stabilize=True,
                          absorb_threshold=20.0)
    sols = fb.sinkhorn_1d_batched([fb.Mesh1D(z) for z in xs], [fb.Mesh1D(z) for z in ys],
                                  [fb.Measure(z) for z in us], [fb.Measure(z) for z in vs], cfg,
                                  epsilons=es)
    for p, sol in enumerate(sols):
        r = O.sinkhorn_1d(xs[p], ys[p], us[p], vs[p], es[p], 120, 0.0, True, 20.0)
        assert list(sol.absorb_iterations) == list(r["absorb_its"])
        assert rel_inf(sol.phi, r["phi"]) < TOL and rel_inf(sol.psi, r["psi"]) < TOL
        assert abs(sol.cost - r["cost"]) <= TOL * abs(r["cost"])


@pytest.mark.parametrize("while_loop", ["1", "0"])
def test_batched_tol_stops_per_problem(monkeypatch, while_loop):
    """tol > 0 on a batch whose problems converge at different iterations (and
    one that never does): every problem keeps its own iteration count,
    convergence flag and history while the device loop runs until the last
    one finishes (WHILE-node graph, and the host-replayed chunk graph)."""
    monkeypatch.setenv("FB_WHILE1D", while_loop)
    O = _oracle()
    rng = np.random.default_rng(23)
    xs, ys, us, vs = [], [], [], []
    for p in range(5):
        n = int(rng.integers(300, 1500))
        xs.append(np.sort(rng.uniform(0, 1, n)))
        ys.append(np.sort(rng.uniform(0, 1, n + 17)))
        uu, vv = rng.random(n) + 0.05, rng.random(n + 17) + 0.05
        us.append(uu / uu.sum())
        vs.append(vv / vv.sum())
    es = [0.5, 0.3, 0.2, 0.15, 0.004]  # converge at 12, 19, 34, 54 and never (oracle)
    cfg = fb.SolverConfig(epsilon=1.0, itr_max=90, tol=1e-10, stabilize=True,
                          absorb_threshold=30.0)
    sols = fb.sinkhorn_1d_batched([fb.Mesh1D(z) for z in xs], [fb.Mesh1D(z) for z in ys],
                                  [fb.Measure(z) for z in us], [fb.Measure(z) for z in vs], cfg,
                                  epsilons=es)
    its = []
    for p, sol in enumerate(sols):
        r = O.sinkhorn_1d(xs[p], ys[p], us[p], vs[p], es[p], 90, 1e-10, True, 30.0)
        assert sol.iterations_run == r["iterations"] and sol.converged == r["converged"], p
        assert list(sol.absorb_iterations) == list(r["absorb_its"])
        assert rel_inf(sol.phi, r["phi"]) < TOL and rel_inf(sol.psi, r["psi"]) < TOL
        errs = [e for _, e in sol.marginal_error_history]
        assert hist_ok(errs, r["hist"]) <= 1.0
        its.append(sol.iterations_run)
    assert len(set(its)) > 2 and max(its) == 90 and min(its) < 90, its


def test_batched_many_problems_vs_oracle():
    """A batch large enough for the host-threaded per-problem tiling (>= 64
    problems): every problem matches its own oracle run."""
    O = _oracle()
    rng = np.random.default_rng(31)
    xs, ys, us, vs, es = [], [], [], [], []
    for p in range(70):
        n, m = int(rng.integers(20, 400)), int(rng.integers(20, 400))
        xs.append(np.sort(rng.uniform(0, 1, n)))
        ys.append(np.sort(rng.uniform(0, 1, m)))
        uu, vv = rng.random(n) + 1e-3, rng.random(m) + 1e-3
        us.append(uu / uu.sum())
        vs.append(vv / vv.sum())
        es.append(float(10 ** rng.uniform(-2.5, -1)))
    cfg = fb.SolverConfig(epsilon=1.0, itr_max=60, tol=0.0, stabilize=True, absorb_threshold=20.0)
    sols = fb.sinkhorn_1d_batched([fb.Mesh1D(z) for z in xs], [fb.Mesh1D(z) for z in ys],
                                  [fb.Measure(z) for z in us], [fb.Measure(z) for z in vs], cfg,
                                  epsilons=es)
    for p, sol in enumerate(sols):
        r = O.sinkhorn_1d(xs[p], ys[p], us[p], vs[p], es[p], 60, 0.0, True, 20.0)
        assert list(sol.absorb_iterations) == list(r["absorb_its"]), p
        assert rel_inf(sol.phi, r["phi"]) < TOL and rel_inf(sol.psi, r["psi"]) < TOL, p
        assert abs(sol.cost - r["cost"]) <= TOL * abs(r["cost"]), p


def test_adapter_protocol_under_driver():
    """GpuAdapter1D driven by the reference-semantics host loop (solver.py:156-199)."""
    O = _oracle()
    x, y, u, v, eps = W.config1(n=2000)
    cfg = fb.SolverConfig(epsilon=eps, itr_max=40, tol=0.0, stabilize=True, absorb_threshold=8.0)
    ad = fb.GpuAdapter1D(fb.Mesh1D(x), fb.Mesh1D(y), eps)
    phi, psi, it, conv, hist, _ = fb.run_driver(ad, u, v, cfg)
    r = O.sinkhorn_1d(x, y, u, v, eps, 40, 0.0, True, 8.0)
    assert it == 40 and rel_inf(phi, r["phi"]) < TOL and rel_inf(psi, r["psi"]) < TOL
    assert rel_inf([h[1] for h in hist], r["hist"]) < TOL


def test_row_marginal_exact_full_size():
    """Size-independent property at config-2 size: after the phi half,
    phi * (K' psi) == u up to rounding (the update's defining identity)."""
    x, y, u, v, eps = W.config2()
    sol = _run_cfg(x, y, u, v, eps, 20)
    s = sol.kernel.apply(sol.psi)
    assert rel_elem(sol.phi * s, u, 1e-300) < 1e-12
