"""Multi-GPU partitioning of the hot path.

One process per GPU (torchrun), torch.distributed for the plumbing.  A
batch of independent 1D problems (BASELINE config 5) shards by problem:
contiguous ranges, no data-path collective; only the results (and the
timing, max over ranks) are gathered.  Configs 1-3 run as independent
replicas.  The solve function is injectable so the partition / gather
logic is testable on CPU with the gloo backend (tests/test_sharding_cpu.py).
"""

import numpy as np


def shard_range(P, rank, world):
    """Contiguous problem range [lo, hi) of `rank` among `world` ranks."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return (rank * P) // world, ((rank + 1) * P) // world


def _default_solve(problems, config):
    from .mesh import Measure, Mesh1D
    from .solver import sinkhorn_1d_batched
    if not problems:
        return []
    sols = sinkhorn_1d_batched([Mesh1D(p[0]) for p in problems], [Mesh1D(p[1]) for p in problems],
                               [Measure(p[2]) for p in problems],
                               [Measure(p[3]) for p in problems], config,
                               epsilons=[p[4] for p in problems])
    return [dict(phi=s.phi, psi=s.psi, a=s.a, b=s.b, cost=s.cost,
                 iterations=s.iterations_run, converged=s.converged,
                 hist=[h[1] for h in s.marginal_error_history],
                 absorb_its=list(s.absorb_iterations)) for s in sols]


def solve_batch_sharded(problems, config, solve_fn=None, gather_to_all=True):
    """Solve `problems` [(x, y, u, v, eps), ...] sharded over the process group.

    Every rank passes the same problem list (or at least the same length);
    rank r solves its contiguous range with `solve_fn` (default: the B200
    batched solver) and the per-problem results are all-gathered in problem
    order.  Returns the full result list (every rank, or rank 0 only)."""
    import torch.distributed as dist
    solve_fn = solve_fn or _default_solve
    if not (dist.is_available() and dist.is_initialized()):
        return solve_fn(list(problems), config)
    rank, world = dist.get_rank(), dist.get_world_size()
    lo, hi = shard_range(len(problems), rank, world)
    local = solve_fn(list(problems[lo:hi]), config)
    parts = [None] * world
    if gather_to_all:
        dist.all_gather_object(parts, local)
    else:
        dist.gather_object(local, parts if rank == 0 else None, dst=0)
        if rank != 0:
            return None
    out = []
    for part in parts:
        out.extend(part)
    return out


def max_over_ranks(seconds):
    """Device-timed seconds -> max over ranks (the job's time)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(seconds)
    t = torch.tensor([float(seconds)], dtype=torch.float64)
    if dist.get_backend() == "nccl":
        t = t.cuda()
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
