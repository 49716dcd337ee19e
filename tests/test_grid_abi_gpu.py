"""The 2D device-pointer ABI (finom_grid_* / finom_solve2d / finom_cost2d /
finom_iterate2d) and the GPU grid adapter under the reference driver,
against the reference's own 2D runs (tests/golden/grid_cases.npz) and the
host-buffer sinkhorn_2d."""

import numpy as np
import pytest

import paper_2605_26659_b200 as fb
from paper_2605_26659_b200 import workloads as W

from conftest import load_golden, rel_inf
from test_parity_gpu import TOL, _check_solution, hist_ok

pytestmark = pytest.mark.gpu


def _grid(x, y):
    return fb.Grid2D(fb.Mesh1D(x), fb.Mesh1D(y))


def _cases():
    g = load_golden("grid_cases.npz")
    for k in range(int(g["ncases"])):
        yield k, (lambda key, k=k: g["g%d_%s" % (k, key)])


def test_grid_adapter_under_run_driver_vs_reference():
    """GpuGridAdapter (the _GridAdapter protocol, kernel2d.py:293-360) driven by
    the reference-semantics host loop reproduces the reference's own runs:
    same iteration counts, absorptions (the driver calls absorb), history."""
    for k, c in _cases():
        eps, itr, tol, stab, thr, ce = c("cfg")
        cfg = fb.SolverConfig(epsilon=eps, itr_max=int(itr), tol=tol, stabilize=bool(stab),
                              absorb_threshold=thr, check_every=int(ce))
        src, tgt = _grid(c("x1"), c("y1")), _grid(c("x2"), c("y2"))
        ad = fb.GpuGridAdapter(src, tgt, eps)
        u = np.ascontiguousarray(c("U").ravel(order="F"))
        v = np.ascontiguousarray(c("V").ravel(order="F"))
        phi, psi, it, conv, hist, _ = fb.run_driver(ad, u, v, cfg)
        assert it == int(c("iterations")) and conv == bool(c("converged")), k
        assert rel_inf(phi, c("phi")) < TOL and rel_inf(psi, c("psi")) < TOL, k
        assert rel_inf(ad.a, c("a")) < TOL or np.max(np.abs(ad.a - c("a"))) < 1e-12, k
        assert [h[0] for h in hist] == [int(t) for t in c("hist_it")], k
        assert hist_ok([h[1] for h in hist], c("hist_err")) <= 1.0, k


def test_grid_solver_device_buffers_vs_reference():
    """GridSolver2D: weights and iterates as torch device tensors, the solve and
    the W1 cost through finom_solve2d / finom_cost2d (no host arrays)."""
    import torch
    for k, c in _cases():
        eps, itr, tol, stab, thr, ce = c("cfg")
        src, tgt = _grid(c("x1"), c("y1")), _grid(c("x2"), c("y2"))
        gs = fb.GridSolver2D(src, tgt, eps)
        gs.set_weights(torch.from_numpy(np.ascontiguousarray(c("U").ravel(order="F"))).cuda(),
                       torch.from_numpy(np.ascontiguousarray(c("V").ravel(order="F"))).cuda())
        st = gs.solve(int(itr), tol, bool(stab), thr)
        assert st == 0
        info = gs.info.cpu().numpy()
        assert int(info[0]) == int(c("iterations")) and bool(info[1]) == bool(c("converged")), k
        assert list(gs.absorb_its.cpu().numpy()[:int(info[3])]) == [int(t) for t in
                                                                       c("absorb_its")], k
        assert rel_inf(gs.phi.cpu().numpy(), c("phi")) < TOL, k
        assert rel_inf(gs.psi.cpu().numpy(), c("psi")) < TOL, k
        cost = float(gs.compute_cost(absorbed=int(info[3]) > 0).item())
        assert abs(cost - float(c("cost"))) <= TOL * abs(float(c("cost"))), k
        # a second solve on the same plan (tables of the plain kernel rebuilt)
        gs.solve(int(itr), tol, bool(stab), thr)
        assert rel_inf(gs.phi.cpu().numpy(), c("phi")) < TOL, k


def test_grid_solver_matches_host_api_bitwise():
    x1, y1, x2, y2, U, V, eps = W.config3(n=96)
    cfg = fb.SolverConfig(epsilon=eps, itr_max=60, tol=0.0, stabilize=True, absorb_threshold=20.0)
    src, tgt = _grid(x1, y1), _grid(x2, y2)
    sol = fb.sinkhorn_2d(src, tgt, fb.Measure2D(U), fb.Measure2D(V), cfg)
    gs = fb.GridSolver2D(src, tgt, eps, fb.Measure2D(U), fb.Measure2D(V))
    assert gs.solve(60, 0.0, True, 20.0) == 0
    assert np.array_equal(gs.phi.cpu().numpy(), sol.phi)
    assert np.array_equal(gs.psi.cpu().numpy(), sol.psi)
    assert np.array_equal(gs.a.cpu().numpy(), sol.a)
    hist = gs.hist.cpu().numpy()
    assert all(hist[it - 1] == e for it, e in sol.marginal_error_history)
    assert float(gs.compute_cost().item()) == sol.cost
