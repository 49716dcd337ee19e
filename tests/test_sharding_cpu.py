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


def test_row_shard_layout_roundtrip():
    from paper_2605_26659_b200 import sharding as S
    n, m = 12, 5
    g = np.arange(n * m, dtype=np.float64)
    for R in (1, 2, 3, 4):
        ranges = S.grid_row_ranges(n, R)
        parts = [S.to_shard(g, n, m, k0, k1) for k0, k1 in ranges]
        assert np.array_equal(S.from_shards(parts, n, m, ranges), g)
        # local element (kl, l) is global (k0 + kl, l)
        k0, k1 = ranges[-1]
        assert parts[-1][1 + (k1 - k0) * 2] == g[k0 + 1 + n * 2]
    with pytest.raises(ValueError):
        S.grid_row_ranges(10, 3)


def test_combine_parts_and_driver_logic():
    from paper_2605_26659_b200 import sharding as S
    from paper_2605_26659_b200 import SolverConfig
    p = S.combine_parts([[1.0, 2.0, 0.5, -1.0], [2.0, 3.0, 0.25, 9.0], [0.5, 1.0, 0.75, 5.0]])
    assert p == (3.5, 3.0, 0.25, 5.0)
    assert S.combine_parts([[1.0, 2.0, 0.5, -1.0]])[3] == -1.0
    # scripted phases: absorb trigger at iteration 2, failure (code 4 * 7 + 2) at 4
    script = {(1, 0): (1.0, 1.0, 1.0, -1.0), (1, 1): (0.0, 1.0, 1.0, -1.0),
              (2, 0): (0.5, 1e90, 1.0, -1.0), (2, 1): (0.0, 1.0, 1.0, -1.0),
              (3, 0): (0.25, 1.0, 1.0, -1.0), (3, 1): (0.0, 1.0, 1.0, -1.0),
              (4, 0): (0.1, 1.0, 1.0, 30.0), (4, 1): (0.0, 1.0, 1.0, -1.0)}
    state = {"it": 1, "absorbs": 0}

    def phase(half, dyn):
        out = script[(state["it"], half)]
        if half == 1:
            state["it"] += 1
        return out

    def absorb():
        state["absorbs"] += 1

    cfg = SolverConfig(epsilon=1e-2, itr_max=10, stabilize=True, absorb_threshold=200.0)
    it, conv, status, hist, abs_its = S.run_driver_2d(phase, absorb, cfg)
    assert (it, conv, status) == (4, False, 2)
    assert abs_its == [2] and state["absorbs"] == 1
    assert hist == [1.0, 0.5, 0.25, 0.1]


def _gather_shards_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_2605_26659_b200 import sharding as S
    dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % port, rank=rank,
                            world_size=world)
    n, m = 8, 3
    g = np.arange(n * m, dtype=np.float64) * 0.5
    ranges = S.grid_row_ranges(n, world)
    mine = torch.from_numpy(S.to_shard(g, n, m, *ranges[rank]))
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine)
    full = S.from_shards([p.numpy() for p in parts], n, m, ranges)
    # the partial reduction of the sharded epilogue
    part = torch.tensor([float(rank + 1), float(rank), 1.0 / (rank + 1), -1.0 if rank else 6.0],
                        dtype=torch.float64)
    allp = [torch.empty_like(part) for _ in range(world)]
    dist.all_gather(allp, part)
    q.put((rank, bool(np.array_equal(full, g)), S.combine_parts([p.numpy() for p in allp])))
    dist.destroy_process_group()


def test_row_shard_gather_gloo_world2():
    import multiprocessing as mp
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_gather_shards_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for rank, ok, comb in res:
        assert ok
        assert comb == (3.0, 1.0, 0.5, 6.0)


@pytest.mark.parametrize("R", [2, 4])
def test_neighbour_index_of_row_shards(R):
    """The neighbour-only absorption exchange: every zero-mass point's previous /
    next positive-mass point of the whole grid (flat column-major order) is
    either in its own shard or the last / first positive point of another
    shard's segment of a column -- the only values the shards exchange."""
    from paper_2605_26659_b200 import sharding as S
    rng = np.random.default_rng(7)
    n, m = 12, 9
    w = rng.uniform(0.1, 1.0, n * m)
    w[rng.random(n * m) < 0.55] = 0.0  # long zero-mass runs crossing shard segments
    w[:5] = 0.0
    w[-4:] = 0.0
    prv, nxt = S._pos_index(w)
    ranges = S.grid_row_ranges(n, R)
    nbs = [S._nb_index(w, n, m, k0, k1) for k0, k1 in ranges]
    nl = n // R

    def flat_of(q, local):
        return (local // nl) * n + ranges[q][0] + local % nl

    for r, (k0, k1) in enumerate(ranges):
        nb = nbs[r]
        for k in range(nl * m):
            kg = (k // nl) * n + k0 + k % nl
            for src, g, want, key in ((nb["prv_src"][k], nb["prv_g"][k], prv[kg], "lastpos"),
                                      (nb["nxt_src"][k], nb["nxt_g"][k], nxt[kg], "firstpos")):
                if want < 0 or want >= n * m:
                    assert src == -1
                    continue
                assert g == want
                if src >= 0:
                    assert flat_of(r, src) == want
                else:
                    seg = -2 - src
                    q, col = seg // m, seg % m
                    assert flat_of(q, nbs[q][key][col]) == want
