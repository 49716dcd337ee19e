"""Multi-GPU partitioning of the hot path.

One process per GPU (torchrun), torch.distributed for the plumbing.  A
batch of independent 1D problems (BASELINE config 5) shards by problem:
contiguous ranges, no data-path collective; only the results (and the
timing, max over ranks) are gathered.  Configs 1-3 run as independent
replicas.  The solve function is injectable so the partition / gather
logic is testable on CPU with the gloo backend (tests/test_sharding_cpu.py).
"""

import os

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


# ---------------------------------------------------------------------------
# Row-sharded 2D grids (BASELINE config 4).
#
# Rank r holds grid rows [k0, k1) (x index) of source == target grids.  The
# y sweeps are local; the x sweep of every half needs the other shards'
# carries: each shard resolves its segment of every column line on the
# device, the segment totals (10 doubles per line) are all-gathered, and the
# shard composes the totals of the shards before / after it into each line's
# incoming state (finom_grid2d_xpre / finom_grid2d_finish).  The reductions
# of the epilogue (marginal error, extremes, failure) are all-gathered and
# run_driver's decisions (solver.py:173-198) are taken on the device, in rank
# order, identically on every rank (finom_grid2d_decide); the host reads one
# 8-word control block per iteration.  An absorption exchanges only each
# column segment's scalings at its last / first positive-mass points (the only
# values solver._shift's np.interp can reach in another shard):
# finom_grid2d_edges / finom_grid2d_absorb_nb.


def grid_row_ranges(n, world):
    """Row shards [k0, k1) of an n-row grid (equal sizes: n % world == 0)."""
    if n % world:
        raise ValueError("row-sharded grids need n divisible by the world size")
    nl = n // world
    return [(r * nl, (r + 1) * nl) for r in range(world)]


def to_shard(flat, n, m, k0, k1):
    """Rows [k0, k1) of a column-major n x m grid, column-major (k1-k0) x m."""
    return np.ascontiguousarray(np.asarray(flat).reshape(m, n)[:, k0:k1]).ravel()


def from_shards(parts, n, m, ranges):
    """Reassemble column-major shards into the flat column-major n x m grid."""
    g = np.empty((m, n))
    for part, (k0, k1) in zip(parts, ranges):
        g[:, k0:k1] = np.asarray(part).reshape(m, k1 - k0)
    return g.ravel()


def _nb_index(w, n, m, k0, k1):
    """Neighbour references of one row shard for the neighbour-only absorption
    exchange (finom_grid2d_absorb_nb): per local point the previous / next
    positive-mass point of the whole grid in flat (column-major) order, as a
    local index, or as segment q * m + col of the gathered edges (-2 - seg),
    or -1; their flat indices; and per column the local indices of the
    segment's last / first positive points.  Uses the weights of the whole
    grid once (host, at setup); the device keeps O(N / R) per rank."""
    w = np.asarray(w, dtype=np.float64)
    N, nl = w.size, k1 - k0
    prv, nxt = _pos_index(w)
    cols = np.arange(m, dtype=np.int64)
    kg = (cols[:, None] * n + k0 + np.arange(nl, dtype=np.int64)[None, :]).ravel()
    pg, ng_ = prv[kg].astype(np.int64), nxt[kg].astype(np.int64)

    def src(gi, none):
        gi = np.where(none, 0, gi)
        row, col = gi % n, gi // n
        inside = (row >= k0) & (row < k1)
        ref = np.where(inside, col * nl + (row - k0), -2 - ((row // nl) * m + col))
        return np.where(none, -1, ref).astype(np.int32)

    wl = w.reshape(m, n)[:, k0:k1] > 0
    has = wl.any(axis=1)
    last = np.where(has, cols * nl + (nl - 1 - np.argmax(wl[:, ::-1], axis=1)), -1)
    first = np.where(has, cols * nl + np.argmax(wl, axis=1), -1)
    return dict(prv_src=src(pg, pg < 0), nxt_src=src(ng_, ng_ >= N),
                prv_g=np.where(pg < 0, 0, pg).astype(np.int32),
                nxt_g=np.where(ng_ >= N, 0, ng_).astype(np.int32),
                lastpos=last.astype(np.int32), firstpos=first.astype(np.int32))


def _pos_index(w):
    """Previous / next positive-mass flat index (solver._shift's np.interp support)."""
    idx = np.arange(w.size)
    pos = w > 0
    prv = np.maximum.accumulate(np.where(pos, idx, -1))
    nxt = np.minimum.accumulate(np.where(pos, idx, w.size)[::-1])[::-1]
    return prv.astype(np.int32), nxt.astype(np.int32)


class RowShard2D:
    """One rank's state of a row-sharded 2D solve (device buffers + C handle)."""

    def __init__(self, x, y1, y2, U, V, eps, k0, k1):
        import ctypes
        import torch
        from . import _lib
        self.lib = _lib.load()
        self._lib = _lib
        n, m1, m2 = len(x), len(y1), len(y2)
        self.n, self.m1, self.m2, self.k0, self.k1, self.eps = n, m1, m2, k0, k1, eps
        h = ctypes.c_void_p()
        _lib.check(self.lib.finom_grid2d_create(n, _lib.ptr(x), m1, _lib.ptr(y1), m2,
                                                _lib.ptr(y2), float(eps), k0, k1,
                                                ctypes.byref(h)), "finom_grid2d_create")
        self.h = h
        dev = torch.device("cuda")
        f64 = dict(dtype=torch.float64, device=dev)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)
        self.U = t(to_shard(U, n, m1, k0, k1))
        self.V = t(to_shard(V, n, m2, k0, k1))
        self.PHI = torch.full(((k1 - k0) * m1,), 1.0 / (n * m1), **f64)
        self.PSI = torch.full(((k1 - k0) * m2,), 1.0 / (n * m1), **f64)
        self.A = torch.zeros((k1 - k0) * m1, **f64)
        self.B = torch.zeros((k1 - k0) * m2, **f64)
        self.seg = torch.empty(10 * max(m1, m2), **f64)
        self.part = torch.empty(4, **f64)
        self.edges = torch.empty(2 * max(m1, m2), **f64)
        ti = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        # neighbour references of this shard only (O(N / R) on the device)
        self.nb = [{k: ti(a) for k, a in _nb_index(W, n, mm, k0, k1).items()}
                   for W, mm in ((U, m1), (V, m2))]

    def close(self):
        if self.h:
            self.lib.finom_grid2d_destroy(self.h)
            self.h = None

    def lines(self, half):
        return self.m1 if half == 0 else self.m2

    def xpre(self, half, dyn):
        L, P = self._lib, self._lib.ptr
        inp, sh = (self.PHI, self.A) if half == 0 else (self.PSI, self.B)
        L.check(self.lib.finom_grid2d_xpre(self.h, half, P(inp), P(sh), int(dyn), P(self.seg),
                                           L.stream_ptr()), "finom_grid2d_xpre")
        return self.seg[:10 * self.lines(half)]

    def finish(self, half, dyn, seg_all, R, r):
        L, P = self._lib, self._lib.ptr
        inp, W, SC = (self.PHI, self.V, self.PSI) if half == 0 else (self.PSI, self.U, self.PHI)
        L.check(self.lib.finom_grid2d_finish(self.h, half, P(inp), P(self.A), P(self.B), int(dyn),
                                             P(seg_all), R, r, P(W), P(SC), P(self.part),
                                             L.stream_ptr()), "finom_grid2d_finish")
        return self.part

    def edges_out(self, side):
        """This shard's per-column scalings at its segments' last / first
        positive points (2 m doubles) for the neighbour exchange."""
        L, P = self._lib, self._lib.ptr
        sc, nb, m = (self.PHI, self.nb[0], self.m1) if side == 0 else (self.PSI, self.nb[1], self.m2)
        L.check(self.lib.finom_grid2d_edges(self.h, P(sc), P(nb["lastpos"]), P(nb["firstpos"]), m,
                                            P(self.edges), L.stream_ptr()), "finom_grid2d_edges")
        return self.edges[:2 * m]

    def absorb(self, side, edges_all):
        """shift += _shift(W, SC) with the gathered edges ([R][m][2])."""
        L, P = self._lib, self._lib.ptr
        sh, W, sc = (self.A, self.U, self.PHI) if side == 0 else (self.B, self.V, self.PSI)
        nb = self.nb[side]
        L.check(self.lib.finom_grid2d_absorb_nb(
            self.h, side, P(sh), P(W), P(sc), P(nb["prv_src"]), P(nb["nxt_src"]), P(nb["prv_g"]),
            P(nb["nxt_g"]), P(edges_all), L.stream_ptr()), "finom_grid2d_absorb_nb")

    def decide(self, parts_a, parts_b, R, ctl, hist, abs_its, config):
        """run_driver's decisions of the iteration on the device (finom_grid2d_decide)."""
        L, P = self._lib, self._lib.ptr
        L.check(self.lib.finom_grid2d_decide(
            P(parts_a), P(parts_b), R, P(ctl), P(hist), P(abs_its), int(config.itr_max),
            float(config.tol), int(bool(config.stabilize)), float(config.absorb_threshold),
            L.stream_ptr()), "finom_grid2d_decide")

    def refresh_shifts(self):
        L, P = self._lib, self._lib.ptr
        L.check(self.lib.finom_grid2d_set_shifts(self.h, P(self.A), P(self.B), L.stream_ptr()),
                "finom_grid2d_set_shifts")


def combine_parts(parts):
    """All-reduce of per-shard epilogue partials (err, max, min, failure code)."""
    parts = np.asarray(parts, dtype=np.float64).reshape(-1, 4)
    fails = parts[:, 3][parts[:, 3] >= 0]
    return (float(np.sum(parts[:, 0])), float(np.max(parts[:, 1])), float(np.min(parts[:, 2])),
            float(np.min(fails)) if fails.size else -1.0)


def run_driver_2d(phase, absorb, config):
    """run_driver (solver.py:156-199) over a sharded 2D iteration: phase(half,
    dyn) returns the combined partials, absorb() performs _shift + absorb on
    every shard.  Returns (iterations, converged, status, hist, absorb_its)."""
    import math
    hi, lo = math.exp(config.absorb_threshold), math.exp(-config.absorb_threshold)
    it, dyn, status, converged = 0, False, 0, False
    hist, abs_its = [], []
    while it < config.itr_max:
        pa = phase(0, dyn)
        pb = phase(1, dyn)
        it += 1
        hist.append(pa[0])
        if pa[3] >= 0 or pb[3] >= 0:
            f = pa[3] if pa[3] >= 0 else pb[3]
            status = int(f) & 3
            break
        if config.tol > 0 and pa[0] <= config.tol:
            converged = True
            break
        if config.stabilize and (pb[1] > hi or pa[1] > hi or pb[2] < lo or pa[2] < lo):
            absorb()
            abs_its.append(it)
            dyn = True
    return it, converged, status, hist, abs_its


def _solution_2d(source, target, config, phi, psi, A, B, it, conv, status, hist, abs_its,
                 wall):
    import dataclasses
    from .kernel2d import KernelOperator2D, build_operator_2d, transport_cost_fast_2d
    from .solver import Solution, history_from, raise_status
    raise_status(status)
    (n1, m1), (n2, m2) = source.shape, target.shape
    op = build_operator_2d(source, target, config.epsilon)
    op = KernelOperator2D(op.kx, op.ky, op.epsilon, A.reshape((n1, m1), order="F"),
                          B.reshape((n2, m2), order="F"))
    h = np.zeros(config.itr_max)
    h[:len(hist)] = hist
    sol = Solution(phi=phi, psi=psi, a=A, b=B, kernel=op, iterations_run=it, converged=conv,
                   marginal_error_history=history_from(h, it, conv, config), wall_time=wall,
                   setup_time=0.0, cost=float("nan"), config=config,
                   absorb_iterations=list(abs_its))
    return dataclasses.replace(sol, cost=float(transport_cost_fast_2d(sol)))


def _check_grids(source, target):
    from .errors import ConfigError
    x1, x2 = source.x_nodes.nodes, target.x_nodes.nodes
    if len(x1) != len(x2) or not np.array_equal(x1, x2):
        raise ConfigError("row sharding needs source and target grids with the same x nodes")


LAST_LOOP = {}  # (the last _device_loop: iterations replayed from captured graphs, for tests)


def _device_loop(config, dev, iterate, absorb, capture=False):
    """run_driver over a sharded 2D iteration with the decisions on the device:
    iterate(dyn, ctl, hist, abs_its) queues both halves, the partials'
    exchange and finom_grid2d_decide; the host reads the 8-word control block
    once per iteration (absorb when flagged, stop when done).  capture: after
    one eager iteration (NCCL communicators up, buffers allocated) the
    iteration -- its kernels and its NCCL all-gathers -- is captured once per
    kernel form (before / after the first absorption) into a CUDA graph and
    replayed (FINOM_GRAPH_SHARD=0: eager).  Returns (it, converged, status,
    hist, absorb_its)."""
    import torch
    itr = int(config.itr_max)
    ctl = torch.zeros(8, dtype=torch.int64, device=dev)
    hist = torch.zeros(itr, dtype=torch.float64, device=dev)
    abs_its = torch.zeros(itr, dtype=torch.int64, device=dev)
    ctl_h = torch.zeros(8, dtype=torch.int64).pin_memory()
    dyn = False
    capture = capture and os.environ.get("FINOM_GRAPH_SHARD", "1") != "0"
    graphs = {}
    first = True
    while True:
        g = graphs.get(dyn) if capture and not first else None
        if capture and not first and g is None:
            try:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    iterate(dyn, ctl, hist, abs_its)
                graphs[dyn] = g
            except Exception:  # noqa: BLE001  (capture unsupported: stay eager)
                capture, g = False, None
                torch.cuda.synchronize()
        if g is not None:
            g.replay()
        else:
            iterate(dyn, ctl, hist, abs_its)
        first = False
        ctl_h.copy_(ctl, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        c = ctl_h.numpy()
        if c[3]:
            absorb()
            dyn = True
        if c[4]:
            break
    it, status, conv, nab = int(c[0]), int(c[1]), bool(c[2]), int(c[5])
    LAST_LOOP.clear()
    LAST_LOOP.update(graphs=len(graphs), captured=capture)
    return it, conv, status, hist[:it].cpu().numpy().tolist(), abs_its[:nab].cpu().tolist()


def sinkhorn_2d_row_sharded(source, target, u, v, config, group=None):
    """sinkhorn_2d with the grid rows sharded over the process group (one GPU
    per rank, NCCL).  Every rank passes the whole problem; returns the
    Solution (gathered) on every rank.  Per iteration: 4 all-gathers (segment
    totals and partials of each half) and one 64-byte control-block read;
    decisions on the device; absorptions exchange 2 doubles per column
    segment."""
    import time
    import torch
    import torch.distributed as dist
    _check_grids(source, target)
    R, r = dist.get_world_size(group), dist.get_rank(group)
    n, m1, m2 = source.shape[0], source.shape[1], target.shape[1]
    ranges = grid_row_ranges(n, R)
    k0, k1 = ranges[r]
    U = u.weights.ravel(order="F")
    V = v.weights.ravel(order="F")
    sh = RowShard2D(source.x_nodes.nodes, source.y_nodes.nodes, target.y_nodes.nodes, U, V,
                    config.epsilon, k0, k1)
    dev = sh.PHI.device
    seg_all = {h: torch.empty(R * 10 * sh.lines(h), dtype=torch.float64, device=dev)
               for h in (0, 1)}
    parts = {h: torch.empty(4 * R, dtype=torch.float64, device=dev) for h in (0, 1)}
    edges_all = {h: torch.empty(R * 2 * sh.lines(h), dtype=torch.float64, device=dev)
                 for h in (0, 1)}

    def iterate(dyn, ctl, hist, abs_its):
        for half in (0, 1):
            seg = sh.xpre(half, dyn)
            dist.all_gather_into_tensor(seg_all[half], seg.contiguous(), group=group)
            part = sh.finish(half, dyn, seg_all[half], R, r)
            dist.all_gather_into_tensor(parts[half], part, group=group)
        sh.decide(parts[0], parts[1], R, ctl, hist, abs_its, config)

    def absorb():
        for side in (0, 1):
            dist.all_gather_into_tensor(edges_all[side], sh.edges_out(side).contiguous(),
                                        group=group)
            sh.absorb(side, edges_all[side])
        sh.PHI.fill_(1.0)
        sh.PSI.fill_(1.0)
        sh.refresh_shifts()

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    it, conv, status, hist, abs_its = _device_loop(config, dev, iterate, absorb, capture=True)
    torch.cuda.synchronize()
    wall = max_over_ranks(time.perf_counter() - t0)
    out = {}
    for name, t in (("phi", sh.PHI), ("psi", sh.PSI), ("A", sh.A), ("B", sh.B)):
        g = torch.empty(R * t.numel(), dtype=torch.float64, device=dev)
        dist.all_gather_into_tensor(g, t, group=group)
        m = m1 if name in ("phi", "A") else m2
        out[name] = from_shards(np.split(g.cpu().numpy(), R), n, m, ranges)
    sh.close()
    return _solution_2d(source, target, config, out["phi"], out["psi"], out["A"], out["B"], it,
                        conv, status, hist, abs_its, wall)


def sinkhorn_2d_row_sharded_sim(source, target, u, v, config, R):
    """The row-sharded algorithm with R shards in ONE process on one GPU: the
    shards' phases run one after another and the collectives are plain
    concatenations (a correctness check of the decomposition, including the
    device decisions and the neighbour-only absorption exchange; never a
    timing)."""
    import torch
    _check_grids(source, target)
    n, m1, m2 = source.shape[0], source.shape[1], target.shape[1]
    ranges = grid_row_ranges(n, R)
    U = u.weights.ravel(order="F")
    V = v.weights.ravel(order="F")
    shards = [RowShard2D(source.x_nodes.nodes, source.y_nodes.nodes, target.y_nodes.nodes, U, V,
                         config.epsilon, k0, k1) for k0, k1 in ranges]

    def iterate(dyn, ctl, hist, abs_its):
        parts = []
        for half in (0, 1):
            seg_all = torch.cat([s.xpre(half, dyn).clone() for s in shards])
            parts.append(torch.cat([s.finish(half, dyn, seg_all, R, k).clone()
                                    for k, s in enumerate(shards)]))
        shards[0].decide(parts[0], parts[1], R, ctl, hist, abs_its, config)

    def absorb():
        for side in (0, 1):
            edges_all = torch.cat([s.edges_out(side).clone() for s in shards])
            for s in shards:
                s.absorb(side, edges_all)
        for s in shards:
            s.PHI.fill_(1.0)
            s.PSI.fill_(1.0)
            s.refresh_shifts()

    it, conv, status, hist, abs_its = _device_loop(config, shards[0].PHI.device, iterate, absorb)
    torch.cuda.synchronize()
    out = {name: from_shards([getattr(s, name).cpu().numpy() for s in shards], n,
                             m1 if name in ("PHI", "A") else m2, ranges)
           for name in ("PHI", "PSI", "A", "B")}
    for s in shards:
        s.close()
    return _solution_2d(source, target, config, out["PHI"], out["PSI"], out["A"], out["B"], it,
                        conv, status, hist, abs_its, 0.0)



# ---------------------------------------------------------------------------
# Distributed 1D scan (BASELINE north star: "very long 1D meshes use a
# distributed scan, where each GPU scans its segment and per-segment carries
# are exchanged with a small NCCL all-gather over NVLink before a fix-up
# pass").  Rank r owns segment r of the merged order x U y (merge-path
# splits, finom_seg1d_*): per half its tile maps and resolve tree give the
# segment's totals of both recurrences (_kernels.py:53-88), the totals are
# all-gathered (10 doubles per rank), each rank composes those of the
# segments before / after it into its incoming states and computes its rows
# and their scaling update; the partials are all-gathered and combined in
# rank order, so run_driver's decisions are identical on every rank.  An
# absorption all-gathers the scalings (np.interp over the whole vector).

def seg_split(x, y, R):
    """Merge-path split points [(i_k, j_k)] k = 0..R of a 1D problem."""
    from . import _lib
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    b = np.zeros(2 * (R + 1), dtype=np.int64)
    _lib.check(_lib.load(False).finom_seg1d_split(x.size, _lib.ptr(x), y.size, _lib.ptr(y), R,
                                                  _lib.ptr(b)), "finom_seg1d_split")
    return [(int(b[2 * k]), int(b[2 * k + 1])) for k in range(R + 1)]


def combine_parts_1d(parts):
    """Rank-order combine of per-segment partials (err, max, min, status or -1):
    errors summed in rank order, extremes, and the failure of the LAST failing
    segment (the reference's loops run downward, _kernels.py:293-314)."""
    parts = np.asarray(parts, dtype=np.float64).reshape(-1, 4)
    err = 0.0
    for e in parts[:, 0]:
        err += float(e)
    fails = [f for f in parts[:, 3] if f >= 0]
    return err, float(np.max(parts[:, 1])), float(np.min(parts[:, 2])), (
        float(fails[-1]) if fails else -1.0)


class Segment1D:
    """Device state of one segment (whole-length vectors, this rank's rows)."""

    def __init__(self, x, y, u, v, eps, R, r):
        import ctypes
        import torch
        from . import _lib
        self._lib = _lib
        self.lib = _lib.load()
        x, y = (np.ascontiguousarray(z, dtype=np.float64) for z in (x, y))
        h = ctypes.c_void_p()
        _lib.check(self.lib.finom_seg1d_create(x.size, _lib.ptr(x), y.size, _lib.ptr(y), eps, R, r,
                                               _lib.stream_ptr(), ctypes.byref(h)),
                   "finom_seg1d_create")
        self.h = h
        w = np.zeros(4, dtype=np.int64)
        self.lib.finom_seg1d_window(h, _lib.ptr(w))
        self.window = tuple(int(k) for k in w)
        dev = torch.device("cuda")
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)
        n, m = x.size, y.size
        self.U, self.V = t(u), t(v)
        self.PHI = torch.full((n,), 1.0 / n, dtype=torch.float64, device=dev)  # solver.py:165-166
        self.PSI = torch.full((m,), 1.0 / n, dtype=torch.float64, device=dev)
        self.A = torch.zeros(n, dtype=torch.float64, device=dev)
        self.B = torch.zeros(m, dtype=torch.float64, device=dev)
        self.tot = torch.zeros(10, dtype=torch.float64, device=dev)
        self.part = torch.zeros(4, dtype=torch.float64, device=dev)
        pu, nu = _pos_index(np.asarray(u))
        pv, nv = _pos_index(np.asarray(v))
        it = lambda a: torch.from_numpy(a).to(dev)
        self.prvU, self.nxtU, self.prvV, self.nxtV = it(pu), it(nu), it(pv), it(nv)
        self.shifted = False

    def _sh(self):
        return (self.A, self.B) if self.shifted else (None, None)

    def pre(self, half):
        L, P = self._lib, self._lib.ptr
        a, b = self._sh()
        L.check(self.lib.finom_seg1d_pre(self.h, half, P(self.PHI if half == 0 else self.PSI),
                                         P(a), P(b), P(self.tot), L.stream_ptr()),
                "finom_seg1d_pre")
        return self.tot

    def finish(self, half, tot_all):
        L, P = self._lib, self._lib.ptr
        a, b = self._sh()
        inp, W, SC = (self.PHI, self.V, self.PSI) if half == 0 else (self.PSI, self.U, self.PHI)
        L.check(self.lib.finom_seg1d_finish(self.h, half, P(inp), P(a), P(b), P(tot_all), P(W),
                                            P(SC), P(self.part), L.stream_ptr()),
                "finom_seg1d_finish")
        return self.part

    def decide(self, parts_a, parts_b, R, ctl, hist, abs_its, config):
        """run_driver's decisions of the iteration on the device (finom_seg1d_decide)."""
        L, P = self._lib, self._lib.ptr
        L.check(self.lib.finom_seg1d_decide(
            P(parts_a), P(parts_b), R, P(ctl), P(hist), P(abs_its), int(config.itr_max),
            float(config.tol), int(bool(config.stabilize)), float(config.absorb_threshold),
            L.stream_ptr()), "finom_seg1d_decide")

    def absorb(self, side, sc_whole):
        L, P = self._lib, self._lib.ptr
        sh, W = (self.A, self.U) if side == 0 else (self.B, self.V)
        prv, nxt = (self.prvU, self.nxtU) if side == 0 else (self.prvV, self.nxtV)
        L.check(self.lib.finom_seg1d_absorb(self.h, side, P(sh), P(W), P(sc_whole), P(prv),
                                            P(nxt), L.stream_ptr()), "finom_seg1d_absorb")

    def close(self):
        if getattr(self, "h", None):
            self.lib.finom_seg1d_destroy(self.h)
            self.h = None


def _assemble_1d(vectors, windows, side):
    """Whole vector from per-segment copies: segment k's window of `side` (0: x, 1: y)."""
    out = np.array(vectors[0], dtype=np.float64)
    for vec, w in zip(vectors, windows):
        lo, hi = (w[0], w[1]) if side == 0 else (w[2], w[3])
        out[lo:hi] = np.asarray(vec)[lo:hi]
    return out


def _solution_1d(x, y, config, phi, psi, a, b, it, conv, status, hist, abs_its, wall):
    import dataclasses
    from . import kernel1d
    from .mesh import Mesh1D
    from .solver import Solution, history_from, raise_status, transport_cost_fast
    raise_status(status)
    X, Y = Mesh1D(x), Mesh1D(y)
    op = kernel1d.KernelOperator1D(X, Y, config.epsilon, a, b,
                                   kernel1d._PlanCache(X, Y, config.epsilon))
    h = np.zeros(config.itr_max)
    h[:len(hist)] = hist
    sol = Solution(phi=phi, psi=psi, a=a, b=b, kernel=op, iterations_run=it, converged=conv,
                   marginal_error_history=history_from(h, it, conv, config), wall_time=wall,
                   setup_time=0.0, cost=float("nan"), config=config,
                   absorb_iterations=list(abs_its))
    return dataclasses.replace(sol, cost=float(transport_cost_fast(sol)))


def sinkhorn_1d_segmented(x, y, u, v, config, group=None):
    """sinkhorn_1d of ONE problem as a distributed scan over the process group
    (one GPU per rank, NCCL).  Every rank passes the whole problem; returns
    the Solution on every rank."""
    import time
    import torch
    import torch.distributed as dist
    X = np.asarray(getattr(x, "nodes", x), dtype=np.float64)
    Y = np.asarray(getattr(y, "nodes", y), dtype=np.float64)
    Uw = np.asarray(getattr(u, "weights", u), dtype=np.float64)
    Vw = np.asarray(getattr(v, "weights", v), dtype=np.float64)
    R, r = dist.get_world_size(group), dist.get_rank(group)
    sg = Segment1D(X, Y, Uw, Vw, config.epsilon, R, r)
    dev = sg.PHI.device
    tot_all = torch.empty(10 * R, dtype=torch.float64, device=dev)
    parts = {h: torch.empty(4 * R, dtype=torch.float64, device=dev) for h in (0, 1)}

    def iterate(dyn, ctl, hist, abs_its):  # (device-resident: decisions in finom_seg1d_decide)
        for half in (0, 1):
            dist.all_gather_into_tensor(tot_all, sg.pre(half).contiguous(), group=group)
            dist.all_gather_into_tensor(parts[half], sg.finish(half, tot_all).contiguous(),
                                        group=group)
        sg.decide(parts[0], parts[1], R, ctl, hist, abs_its, config)

    wins = [None] * R
    dist.all_gather_object(wins, sg.window, group=group)

    def gather_whole(t, side):
        g = torch.empty(R * t.numel(), dtype=torch.float64, device=dev)
        dist.all_gather_into_tensor(g, t.contiguous(), group=group)
        return _assemble_1d(np.split(g.cpu().numpy(), R), wins, side)

    def absorb():
        for side, sc in ((0, sg.PHI), (1, sg.PSI)):
            whole = torch.from_numpy(gather_whole(sc, side)).to(dev)
            sg.absorb(side, whole)
        sg.PHI.fill_(1.0)
        sg.PSI.fill_(1.0)
        sg.shifted = True

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    it, conv, status, hist, abs_its = _device_loop(config, dev, iterate, absorb, capture=True)
    torch.cuda.synchronize()
    wall = max_over_ranks(time.perf_counter() - t0)
    phi, psi = gather_whole(sg.PHI, 0), gather_whole(sg.PSI, 1)
    a, b = sg.A.cpu().numpy(), sg.B.cpu().numpy()
    sg.close()
    return _solution_1d(X, Y, config, phi, psi, a, b, it, conv, status, hist, abs_its, wall)


def sinkhorn_1d_segmented_sim(x, y, u, v, config, R):
    """The distributed scan with R segments in ONE process on one GPU: the
    segments' phases run one after another and the collectives are plain
    concatenations (a correctness check of the decomposition; never a
    timing)."""
    import torch
    X = np.asarray(getattr(x, "nodes", x), dtype=np.float64)
    Y = np.asarray(getattr(y, "nodes", y), dtype=np.float64)
    Uw = np.asarray(getattr(u, "weights", u), dtype=np.float64)
    Vw = np.asarray(getattr(v, "weights", v), dtype=np.float64)
    segs = [Segment1D(X, Y, Uw, Vw, config.epsilon, R, k) for k in range(R)]
    wins = [s.window for s in segs]

    def iterate(dyn, ctl, hist, abs_its):
        parts = []
        for half in (0, 1):
            tot_all = torch.cat([s.pre(half).clone() for s in segs])
            parts.append(torch.cat([s.finish(half, tot_all).clone() for s in segs]))
        segs[0].decide(parts[0], parts[1], R, ctl, hist, abs_its, config)

    def absorb():
        for side in (0, 1):
            vecs = [(s.PHI if side == 0 else s.PSI).cpu().numpy() for s in segs]
            whole = torch.from_numpy(_assemble_1d(vecs, wins, side)).cuda()
            for s in segs:
                s.absorb(side, whole)
        for s in segs:
            s.PHI.fill_(1.0)
            s.PSI.fill_(1.0)
            s.shifted = True

    it, conv, status, hist, abs_its = _device_loop(config, segs[0].PHI.device, iterate, absorb)
    torch.cuda.synchronize()
    phi = _assemble_1d([s.PHI.cpu().numpy() for s in segs], wins, 0)
    psi = _assemble_1d([s.PSI.cpu().numpy() for s in segs], wins, 1)
    a, b = segs[0].A.cpu().numpy(), segs[0].B.cpu().numpy()
    for s in segs:
        s.close()
    return _solution_1d(X, Y, config, phi, psi, a, b, it, conv, status, hist, abs_its, 0.0)
