"""World-size-2 gloo test of the problem-sharded batch path.

The solve function is the C oracle here (no GPU in this container); the
partition / all-gather / max-over-ranks logic is the one bench.py and the
B200 path use."""

import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_solve(problems, config):
    sys.path.insert(0, ROOT)
    from oracle import oracle as O
    out = []
    for x, y, u, v, eps in problems:
        r = O.sinkhorn_1d(x, y, u, v, eps, config.itr_max, config.tol, config.stabilize,
                          config.absorb_threshold)
        out.append(dict(phi=r["phi"], psi=r["psi"], cost=r["cost"], absorb_its=list(r["absorb_its"])))
    return out


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2605_26659_b200 as fb
    from paper_2605_26659_b200 import sharding, workloads as W
    probs = W.config5(batch=5, n=300)
    cfg = fb.SolverConfig(epsilon=1.0, itr_max=40, tol=0.0, stabilize=True, absorb_threshold=20.0)
    res = sharding.solve_batch_sharded(probs, cfg, solve_fn=_oracle_solve)
    t = sharding.max_over_ranks(0.5 + rank)
    if rank == 0:
        q.put(([r["cost"] for r in res], [r["phi"] for r in res], t))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_ranges_cover_batch():
    from paper_2605_26659_b200.sharding import shard_range
    for P in (1, 7, 8192):
        for world in (1, 2, 4, 8):
            rngs = [shard_range(P, r, world) for r in range(world)]
            assert rngs[0][0] == 0 and rngs[-1][1] == P
            assert all(rngs[k][1] == rngs[k + 1][0] for k in range(world - 1))


def test_sharded_batch_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    costs, phis, t = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sys.path.insert(0, ROOT)
    import paper_2605_26659_b200 as fb
    from paper_2605_26659_b200 import workloads as W
    probs = W.config5(batch=5, n=300)
    cfg = fb.SolverConfig(epsilon=1.0, itr_max=40, tol=0.0, stabilize=True, absorb_threshold=20.0)
    ref = _oracle_solve(probs, cfg)
    assert len(costs) == 5
    assert costs == [r["cost"] for r in ref]
    assert all(np.array_equal(a, r["phi"]) for a, r in zip(phis, ref))
    assert t == 1.5
