"""2D grid path (kernel2d) vs the reference (golden fixtures) and the C oracle.

The reference ships no kernel2d tests; tests/golden/
make_golden.py records the reference's own sinkhorn_2d / operator outputs.
"""

import os

import numpy as np
import pytest

import paper_2605_26659_b200 as fb
from paper_2605_26659_b200 import kernel2d as k2
from paper_2605_26659_b200 import workloads as W

from conftest import GOLDEN, load_golden, rel_inf
from test_parity_gpu import TOL, _check_solution

pytestmark = pytest.mark.gpu


def _grid(x, y):
    return fb.Grid2D(fb.Mesh1D(x), fb.Mesh1D(y))


def test_grid_cases_vs_reference():
    g = load_golden("grid_cases.npz")
    for k in range(int(g["ncases"])):
        c = lambda key: g["g%d_%s" % (k, key)]
        eps, itr, tol, stab, thr, ce = c("cfg")
        cfg = fb.SolverConfig(epsilon=eps, itr_max=int(itr), tol=tol, stabilize=bool(stab),
                              absorb_threshold=thr, check_every=int(ce))
        src, tgt = _grid(c("x1"), c("y1")), _grid(c("x2"), c("y2"))
        sol = fb.sinkhorn_2d(src, tgt, fb.Measure2D(c("U")), fb.Measure2D(c("V")), cfg)
        r = {key: c(key) for key in ("phi", "psi", "a", "b", "hist_it", "hist_err",
                                     "iterations", "converged", "absorb_its", "cost")}
        _check_solution(sol, r)
        op = k2.build_operator_2d(src, tgt, eps)
        assert rel_inf(op.apply(c("vin")), c("Kv")) < 1e-12, k
        assert rel_inf(op.apply_transpose(c("win")), c("KTw")) < 1e-12, k
        if "g%d_Kv_abs" % k in g:
            A = c("a").reshape((len(c("x1")), len(c("y1"))), order="F")
            B = c("b").reshape((len(c("x2")), len(c("y2"))), order="F")
            opa = op.absorb(A, B)
            assert rel_inf(opa.apply(c("vin")), c("Kv_abs")) < 1e-12, k
            assert rel_inf(opa.apply_transpose(c("win")), c("KTw_abs")) < 1e-12, k


def test_cost_2d_state_vs_oracle():
    from oracle import oracle as O
    x1, y1, x2, y2, U, V, eps = W.config3(n=48)
    r = O.sinkhorn_2d(x1, y1, x2, y2, U, V, eps, 80, 0.0, True, 30.0)
    src, tgt = _grid(x1, y1), _grid(x2, y2)
    sol = fb.sinkhorn_2d(src, tgt, fb.Measure2D(U), fb.Measure2D(V),
                         fb.SolverConfig(epsilon=eps, itr_max=80, tol=0.0, stabilize=True,
                                         absorb_threshold=30.0))
    assert list(sol.absorb_iterations) == list(r["absorb_its"])
    assert rel_inf(sol.phi, r["phi"]) < TOL and rel_inf(sol.psi, r["psi"]) < TOL
    assert abs(sol.cost - r["cost"]) <= TOL * abs(r["cost"])
    # the standalone cost entry on the same state
    c = k2.transport_cost_fast_2d(sol)
    assert abs(c - r["cost"]) <= TOL * abs(r["cost"])


@pytest.mark.skipif(not os.path.exists(os.path.join(GOLDEN, "config3_full_pins.npz")),
                    reason="config-3 pins not generated")
def test_config3_full_vs_reference_pins():
    g = load_golden("config3_full_pins.npz")
    x1, y1, x2, y2, U, V, eps = W.config3()
    sol = fb.sinkhorn_2d(_grid(x1, y1), _grid(x2, y2), fb.Measure2D(U), fb.Measure2D(V),
                         fb.SolverConfig(epsilon=eps, itr_max=300, tol=0.0, stabilize=True))
    st = int(g["stride"])
    from test_parity_gpu import hist_ok
    q = dict(hist=hist_ok([h[1] for h in sol.marginal_error_history], g["hist_err"]),
             phi=rel_inf(sol.phi[::st], g["phi_s"]), psi=rel_inf(sol.psi[::st], g["psi_s"]),
             a=rel_inf(sol.a[::st], g["a_s"]), b=rel_inf(sol.b[::st], g["b_s"]),
             cost=abs(sol.cost - float(g["cost"])) / abs(float(g["cost"])))
    print("config3 full parity", q)
    assert list(sol.absorb_iterations) == [int(t) for t in g["absorb_its"]]
    assert q["hist"] < 1 and q["phi"] < TOL and q["psi"] < TOL and q["cost"] < TOL, q
    assert q["a"] < TOL and q["b"] < TOL, q


@pytest.mark.skipif(not os.path.exists(os.path.join(GOLDEN, "config4_full_pins.npz")),
                    reason="config-4 pins not generated")
def test_config4_full_vs_reference_pins():
    """Full-size config 4 (8192^2, 100 it, 3 absorptions) against the
    reference's own run (tests/golden/make_golden.py config4_full)."""
    g = load_golden("config4_full_pins.npz")
    x1, y1, x2, y2, U, V, eps = W.config4()
    sol = fb.sinkhorn_2d(_grid(x1, y1), _grid(x2, y2), fb.Measure2D(U), fb.Measure2D(V),
                         fb.SolverConfig(epsilon=eps, itr_max=100, tol=0.0, stabilize=True))
    st = int(g["stride"])
    from test_parity_gpu import hist_ok
    q = dict(hist=hist_ok([h[1] for h in sol.marginal_error_history], g["hist_err"]),
             phi=rel_inf(sol.phi[::st], g["phi_s"]), psi=rel_inf(sol.psi[::st], g["psi_s"]),
             a=rel_inf(sol.a[::st], g["a_s"]), b=rel_inf(sol.b[::st], g["b_s"]),
             cost=abs(sol.cost - float(g["cost"])) / abs(float(g["cost"])))
    print("config4 full parity", q)
    assert list(sol.absorb_iterations) == [int(t) for t in g["absorb_its"]]
    assert q["hist"] < 1 and q["phi"] < TOL and q["psi"] < TOL and q["cost"] < TOL, q
    assert q["a"] < TOL and q["b"] < TOL, q


def _sharded_case(n, m1, m2, eps, itr, seed, zero_rows=False, thr=200.0, square_y=False):
    rng = np.random.default_rng(seed)
    x = W.gap_mesh(rng, n, 0.1, 1.9)
    y1 = W.gap_mesh(rng, m1, 0.1, 1.9)
    y2 = y1.copy() if square_y else W.gap_mesh(rng, m2, 0.1, 1.9)
    U = W.blobs(x, y1, rng, 8)
    V = W.blobs(x, y2, rng, 8)
    if zero_rows:  # zero-mass stretches across the shard boundaries (np.interp fill)
        U[n // 2 - 3:n // 2 + 4, :] = 0.0
        V[n // 4 - 2:n // 4 + 3, : m2 // 2] = 0.0
    U /= U.sum()
    V /= V.sum()
    cfg = fb.SolverConfig(epsilon=eps, itr_max=itr, tol=0.0, stabilize=True,
                          absorb_threshold=thr)
    return x, y1, y2, U, V, cfg


@pytest.mark.parametrize("R,zero,thr,m2,sq", [(2, False, 200.0, 40, False),
                                              (3, True, 30.0, 40, False),
                                              (4, False, 30.0, 52, False),
                                              (2, False, 30.0, 300, True),
                                              (3, True, 30.0, 300, True)])
def test_row_sharded_2d_vs_oracle(R, zero, thr, m2, sq):
    """SURVEY 8(e) config-4 decomposition: R row shards with carry exchange
    (run one after another on one GPU, collectives as concatenation) against
    the oracle of the unsharded reference algorithm.  sq: source y == target
    y (config 4's shape), so the shard-local y sweeps take the square path."""
    from oracle import oracle as O
    from paper_2605_26659_b200 import sharding as S
    m1 = m2 if sq else 40
    x, y1, y2, U, V, cfg = _sharded_case(96, m1, m2, 2e-3, 50, 11 + R, zero, thr, square_y=sq)
    src, tgt = _grid(x, y1), _grid(x.copy(), y2)
    sol = S.sinkhorn_2d_row_sharded_sim(src, tgt, fb.Measure2D(U), fb.Measure2D(V), cfg, R)
    r = O.sinkhorn_2d(x, y1, x, y2, U, V, cfg.epsilon, cfg.itr_max, 0.0, True, thr)
    assert r["status"] == 0
    assert sol.iterations_run == r["iterations"]
    assert list(sol.absorb_iterations) == list(r["absorb_its"])
    assert len(r["absorb_its"]) > 0  # the absorbed (dyn) path is exercised
    for key in ("phi", "psi", "a", "b"):
        assert rel_inf(getattr(sol, key), r[key]) < TOL, key
    assert abs(sol.cost - r["cost"]) <= TOL * abs(r["cost"])
    hist = np.array([h[1] for h in sol.marginal_error_history])
    assert np.allclose(hist, r["hist"], rtol=TOL, atol=1e-12)


def test_row_sharded_2d_matches_single_gpu():
    from paper_2605_26659_b200 import sharding as S
    x, y1, y2, U, V, cfg = _sharded_case(64, 48, 48, 5e-3, 30, 7)
    src, tgt = _grid(x, y1), _grid(x.copy(), y2)
    a = S.sinkhorn_2d_row_sharded_sim(src, tgt, fb.Measure2D(U), fb.Measure2D(V), cfg, 4)
    b = fb.sinkhorn_2d(src, tgt, fb.Measure2D(U), fb.Measure2D(V), cfg)
    for key in ("phi", "psi", "a", "b"):
        assert rel_inf(getattr(a, key), getattr(b, key)) < 1e-11, key


def test_row_sharded_2d_nccl_world1():
    """The torch.distributed driver itself (NCCL collectives, one rank)."""
    import socket
    import torch
    import torch.distributed as dist
    from paper_2605_26659_b200 import sharding as S
    x, y1, y2, U, V, cfg = _sharded_case(64, 40, 40, 2e-3, 25, 5, thr=30.0)
    src, tgt = _grid(x, y1), _grid(x.copy(), y2)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    own = not dist.is_initialized()
    if own:
        dist.init_process_group("nccl", init_method="tcp://127.0.0.1:%d" % port, rank=0,
                                world_size=1, device_id=torch.device("cuda", 0))
    try:
        a = S.sinkhorn_2d_row_sharded(src, tgt, fb.Measure2D(U), fb.Measure2D(V), cfg)
        # the iteration (kernels + NCCL all-gathers) replayed from CUDA graphs,
        # one per kernel form (before / after the first absorption)
        assert S.LAST_LOOP["captured"] and S.LAST_LOOP["graphs"] == 2, S.LAST_LOOP
    finally:
        if own:
            dist.destroy_process_group()
    b = fb.sinkhorn_2d(src, tgt, fb.Measure2D(U), fb.Measure2D(V), cfg)
    assert a.absorb_iterations == b.absorb_iterations
    for key in ("phi", "psi", "a", "b"):
        assert rel_inf(getattr(a, key), getattr(b, key)) < 1e-11, key
    assert abs(a.cost - b.cost) <= 1e-11 * abs(b.cost)


@pytest.mark.parametrize("env,n", [({"FB_GRAPH2D": "0"}, 96), ({"FB_SQ_SPLIT": "0"}, 96),
                                   ({"FB_SQ": "0"}, 96), ({"FB_SQ_FUSE": "0"}, 96),
                                   ({"FB_SQ_FUSE": "0"}, 700), ({"FB_SQ_FUSE": "2"}, 96),
                                   ({"FB_SQ_FUSE": "2"}, 700), ({"FB_SQ_FUSE": "2"}, 1024)])
def test_2d_loop_variants_agree(monkeypatch, env, n):
    """The device-looped graph vs the host-stepped loop (bitwise: the same
    operations); the one-scan fused short-line sweep (default) vs the three
    kernels and vs the two-scan fused sweep, split vs full square-sweep
    records and square vs general sweeps (1e-12): absorbed config-3-style grid
    with a zero-mass stretch and a tol stop (n = 700: three ragged tiles per
    line; 1024: four full tiles)."""
    x1, y1, x2, y2, U, V, eps = W.config3(n=n)
    U = U.copy()
    U[10:30, 40:50] = 0.0
    U /= U.sum()
    cfg = fb.SolverConfig(epsilon=eps, itr_max=60, tol=1e-7, stabilize=True, absorb_threshold=6.0)
    args = (_grid(x1, y1), _grid(x2, y2), fb.Measure2D(U), fb.Measure2D(V), cfg)
    base = fb.sinkhorn_2d(*args)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    alt = fb.sinkhorn_2d(*args)
    assert base.iterations_run == alt.iterations_run and base.converged == alt.converged
    assert list(base.absorb_iterations) == list(alt.absorb_iterations)
    assert len(base.absorb_iterations) >= 1
    tol = 0.0 if "FB_GRAPH2D" in env else 1e-12
    assert rel_inf(alt.phi, base.phi) <= tol and rel_inf(alt.psi, base.psi) <= tol
    assert abs(alt.cost - base.cost) <= max(tol, 1e-15) * abs(base.cost)


@pytest.mark.parametrize("n", [96, 700])
def test_two_scan_fused_sweep_is_the_three_kernels(monkeypatch, n):
    """k_sq_fused (FB_SQ_FUSE=2) runs the three kernels' operations in their
    order: bitwise equal results."""
    x1, y1, x2, y2, U, V, eps = W.config3(n=n)
    cfg = fb.SolverConfig(epsilon=eps, itr_max=40, tol=0.0, stabilize=True, absorb_threshold=6.0)
    args = (_grid(x1, y1), _grid(x2, y2), fb.Measure2D(U), fb.Measure2D(V), cfg)
    monkeypatch.setenv("FB_SQ_FUSE", "2")
    two = fb.sinkhorn_2d(*args)
    monkeypatch.setenv("FB_SQ_FUSE", "0")
    three = fb.sinkhorn_2d(*args)
    assert list(two.absorb_iterations) == list(three.absorb_iterations)
    assert np.array_equal(two.phi, three.phi) and np.array_equal(two.psi, three.psi)
    assert two.cost == three.cost


@pytest.mark.parametrize("graph", ["1", "0"])
def test_2d_failure_diagnostics_vs_oracle(monkeypatch, graph):
    """ZERO_DENOM / NONFINITE in the 2D loop raise the reference's exceptions
    with its messages, at the oracle's iteration (device-looped graph and the
    host-stepped loop)."""
    monkeypatch.setenv("FB_GRAPH2D", graph)
    from oracle import oracle as O
    cases = [  # (source x, y, target x, y, eps, exception, oracle status)
        ([0.0, 0.5], [0.0, 0.5], [0.0, 50.0], [0.0, 50.0], 0.01, fb.ZeroDenominator, 1),
        ([0.0], [0.0], [713.0], [0.0], 1.0, fb.NonFiniteIterate, 2),
    ]
    for x1, y1, x2, y2, eps, exc, st in cases:
        x1, y1, x2, y2 = (np.array(z, dtype=float) for z in (x1, y1, x2, y2))
        U = np.full((x1.size, y1.size), 1.0 / (x1.size * y1.size))
        V = np.full((x2.size, y2.size), 1.0 / (x2.size * y2.size))
        r = O.sinkhorn_2d(x1, y1, x2, y2, U, V, eps, 10, 0.0, False)
        assert r["status"] == st
        cfg = fb.SolverConfig(epsilon=eps, itr_max=10, tol=0.0)
        with pytest.raises(exc) as info:
            fb.sinkhorn_2d(_grid(x1, y1), _grid(x2, y2), fb.Measure2D(U), fb.Measure2D(V), cfg)
        assert "enable stabilization or increase epsilon" in str(info.value)
