"""Bit-reproducibility run to run (fixed tile order, fixed
reduction trees, no float atomics): repeated device solves give identical bits."""

import numpy as np
import pytest
import torch

import paper_2605_26659_b200 as fb
from paper_2605_26659_b200 import workloads as W

pytestmark = pytest.mark.gpu


def test_1d_solve_bitwise_reproducible():
    x, y, u, v, eps = W.config2(n=1 << 18)
    bs = fb.BatchSolver1D([x], [y], [u], [v], [eps])
    outs = []
    for _ in range(3):
        bs.solve(120, 0.0, True, 200.0)
        torch.cuda.synchronize()
        outs.append([t.cpu().numpy().copy() for t in (bs.phi, bs.psi, bs.a, bs.b, bs.hist)])
    for o in outs[1:]:
        for k in range(5):
            assert np.array_equal(outs[0][k], o[k]), k


def test_2d_solve_bitwise_reproducible():
    x1, y1, x2, y2, U, V, eps = W.config3(n=160)
    g = lambda a, b: fb.Grid2D(fb.Mesh1D(a), fb.Mesh1D(b))
    cfg = fb.SolverConfig(epsilon=eps, itr_max=80, tol=0.0, stabilize=True, absorb_threshold=20.0)
    sols = [fb.sinkhorn_2d(g(x1, y1), g(x2, y2), fb.Measure2D(U), fb.Measure2D(V), cfg)
            for _ in range(3)]
    assert len(sols[0].absorb_iterations) >= 1
    for s in sols[1:]:
        assert np.array_equal(s.phi, sols[0].phi) and np.array_equal(s.psi, sols[0].psi)
        assert s.cost == sols[0].cost
        assert s.marginal_error_history == sols[0].marginal_error_history
