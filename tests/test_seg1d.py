"""Distributed 1D scan (finom_seg1d_*, sharding.sinkhorn_1d_segmented): one
1D problem split into R segments of the merged order.  GPU: the R-segment
decomposition run in one process (collectives = concatenation) against the
oracle and the single-GPU solver, and the NCCL driver at world size 1.  CPU:
the split, the rank-order combine, and the gloo world-2 exchange."""

import os
import socket
import sys

import numpy as np
import pytest

import paper_2605_26659_b200 as fb
from paper_2605_26659_b200 import sharding as S
from paper_2605_26659_b200 import workloads as W

from conftest import ROOT, rel_inf


def _case(n, m, eps, seed, zero=False, ties=False):
    rng = np.random.default_rng(seed)
    x = W.gap_mesh(rng, n, 0.2, 1.8)
    y = W.gap_mesh(rng, m, 0.2, 1.8)
    if ties:  # shared nodes: a tie x_i == y_j is never split between segments
        y = np.unique(np.concatenate([y[:: 2], x[1::3]]))
    u = W.mixture(x, (0.3, 0.7), (0.05, 0.1), (0.5, 0.5), 1e-12)
    v = W.mixture(y, (0.35, 0.6), (0.08, 0.1), (0.4, 0.6), 1e-12)
    if zero:  # zero-mass stretches crossing segment boundaries (np.interp fill)
        u[n // 2 - 40:n // 2 + 40] = 0.0
        v[len(y) // 3 - 25:len(y) // 3 + 25] = 0.0
        u, v = u / u.sum(), v / v.sum()
    return x, y, u, v, eps


def test_seg_split_properties():
    for n, m, R, ties in [(1000, 1000, 4, False), (777, 3001, 5, False), (500, 300, 8, True),
                          (50, 9, 3, False)]:
        x, y, _, _, _ = _case(n, m, 1e-2, 7, ties=ties)
        b = S.seg_split(x, y, R)
        assert b[0] == (0, 0) and b[-1] == (len(x), len(y))
        assert all(b[k][0] <= b[k + 1][0] and b[k][1] <= b[k + 1][1] for k in range(R))
        tot = len(x) + len(y)
        for k in range(1, R):
            i, j = b[k]
            assert abs((i + j) - tot * k // R) <= 1  # the diagonal (a tie may move it by one)
            assert not (i > 0 and j < len(y) and x[i - 1] == y[j])  # ties not split
            assert not (j > 0 and i < len(x) and y[j - 1] == x[i])


def test_combine_parts_1d():
    parts = [[0.5, 2.0, 0.1, -1.0], [0.25, 3.0, 0.2, 1.0], [0.125, 1.0, 0.05, 2.0]]
    err, mx, mn, fail = S.combine_parts_1d(parts)
    assert err == 0.875 and mx == 3.0 and mn == 0.05 and fail == 2.0  # the last failing segment
    assert S.combine_parts_1d([[1.0, 1.0, 1.0, -1.0]])[3] == -1.0


def _gloo_worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    from paper_2605_26659_b200 import sharding as S2
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # the exchange of sinkhorn_1d_segmented with host tensors: totals and
    # partials all-gathered in rank order, combined identically on every rank
    tot = torch.full((10,), float(rank + 1), dtype=torch.float64)
    tot_all = torch.empty(10 * world, dtype=torch.float64)
    dist.all_gather_into_tensor(tot_all, tot)
    part = torch.tensor([0.5 * (rank + 1), float(rank), 1.0 - rank, -1.0 if rank == 0 else 1.0],
                        dtype=torch.float64)
    parts = torch.empty(4 * world, dtype=torch.float64)
    dist.all_gather_into_tensor(parts, part)
    comb = S2.combine_parts_1d(parts.numpy())
    wins = [None] * world
    dist.all_gather_object(wins, (0, 5, 0, 3) if rank == 0 else (5, 9, 3, 7))
    vec = torch.full((9,), float(rank), dtype=torch.float64)
    g = torch.empty(9 * world, dtype=torch.float64)
    dist.all_gather_into_tensor(g, vec)
    whole = S2._assemble_1d(np.split(g.numpy(), world), wins, 0)
    q.put((rank, tot_all.numpy().tolist(), comb, whole.tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_seg1d_exchange_gloo_world2():
    import multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for rank, tot_all, comb, whole in res:
        assert tot_all == [1.0] * 10 + [2.0] * 10
        assert comb == (1.5, 1.0, 0.0, 1.0)
        assert whole == [0.0] * 5 + [1.0] * 4


@pytest.mark.gpu
@pytest.mark.parametrize("R,n,m,zero,ties,thr", [(2, 3000, 3000, False, False, 8.0),
                                                 (3, 2000, 3500, True, False, 8.0),
                                                 (5, 4000, 1500, False, True, 6.0),
                                                 (4, 6000, 6000, True, False, 200.0)])
def test_seg1d_sim_vs_oracle_and_single_gpu(R, n, m, zero, ties, thr):
    from oracle import oracle as O
    x, y, u, v, eps = _case(n, m, 2e-3, 3 + R, zero=zero, ties=ties)
    cfg = fb.SolverConfig(epsilon=eps, itr_max=60, tol=0.0, stabilize=True, absorb_threshold=thr)
    a = S.sinkhorn_1d_segmented_sim(x, y, u, v, cfg, R)
    r = O.sinkhorn_1d(x, y, u, v, eps, 60, 0.0, True, thr)
    assert list(a.absorb_iterations) == list(r["absorb_its"])
    assert rel_inf(a.phi, r["phi"]) < 1e-9 and rel_inf(a.psi, r["psi"]) < 1e-9
    assert abs(a.cost - r["cost"]) <= 1e-9 * abs(r["cost"])
    errs = [e for _, e in a.marginal_error_history]
    assert np.max(np.abs(np.array(errs) - r["hist"]) / (1e-9 * np.abs(r["hist"]) + 1e-12)) <= 1
    b = fb.sinkhorn_1d(fb.Mesh1D(x), fb.Mesh1D(y), fb.Measure(u), fb.Measure(v), cfg)
    for key in ("phi", "psi", "a", "b"):
        assert rel_inf(getattr(a, key), getattr(b, key)) < 1e-10, key


@pytest.mark.gpu
def test_seg1d_nccl_world1():
    import torch
    import torch.distributed as dist
    x, y, u, v, eps = _case(2500, 2700, 2e-3, 9, zero=True)
    cfg = fb.SolverConfig(epsilon=eps, itr_max=40, tol=0.0, stabilize=True, absorb_threshold=8.0)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    own = not dist.is_initialized()
    if own:
        dist.init_process_group("nccl", init_method="tcp://127.0.0.1:%d" % port, rank=0,
                                world_size=1, device_id=torch.device("cuda", 0))
    try:
        a = S.sinkhorn_1d_segmented(x, y, u, v, cfg)
        # the iteration (kernels, NCCL all-gathers, device decisions) replayed
        # from CUDA graphs, one per kernel form met after the first iteration
        # (this case absorbs at iteration 1: the shifted form only)
        assert S.LAST_LOOP["captured"] and S.LAST_LOOP["graphs"] >= 1, S.LAST_LOOP
    finally:
        if own:
            dist.destroy_process_group()
    b = fb.sinkhorn_1d(fb.Mesh1D(x), fb.Mesh1D(y), fb.Measure(u), fb.Measure(v), cfg)
    assert a.absorb_iterations == b.absorb_iterations
    for key in ("phi", "psi", "a", "b"):
        assert rel_inf(getattr(a, key), getattr(b, key)) < 1e-10, key
