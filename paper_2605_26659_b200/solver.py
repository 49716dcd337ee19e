"""Scaling-iteration driver and the B200 1D solver (drop-in for finom.solver).

Same names, fields, defaults, validation and exceptions as the reference
(pkg/src/finom/solver.py).  The difference is where the loop runs:
``sinkhorn_1d`` hands the whole ``run_driver`` loop (solver.py:156-199) to
the device (finom_solve1d: one CUDA graph per chunk of iterations, with
history, stopping rule and absorption decided on device), so there is no
per-iteration host round trip.  ``run_driver`` itself is kept for the
adapter protocol (solver.py:1-16) and accepts the GPU adapter
``GpuAdapter1D`` as well as any reference adapter.
"""

import ctypes
import os
from collections.abc import Sequence
from dataclasses import dataclass, replace
from time import perf_counter
from typing import Optional

import numpy as np

from . import _lib, kernel1d
from .errors import (
    ConfigError,
    DimensionMismatch,
    InvalidEpsilon,
    NonFiniteIterate,
    SizeCapExceeded,
    ZeroDenominator,
)

OK, ZERO_DENOM, NONFINITE = 0, 1, 2  # _kernels.py:47-50

_MSG_ZD = ("a matvec underflowed to zero on an entry with positive "
           "target mass; enable stabilization or increase epsilon")
_MSG_NF = ("scaling update produced a non-finite value; enable "
           "stabilization or increase epsilon")


@dataclass(frozen=True)
class SolverConfig:
    """solver.py:36-61, same defaults and validation."""

    epsilon: float
    itr_max: int = 1000
    tol: float = 1e-9
    stabilize: bool = False
    absorb_threshold: float = 200.0
    check_every: int = 1
    plan_cap: int = 10**8

    def __post_init__(self):
        eps = float(self.epsilon)
        if not np.isfinite(eps) or eps <= 0:
            raise InvalidEpsilon("epsilon must be a positive finite real")
        object.__setattr__(self, "epsilon", eps)
        if self.itr_max < 1:
            raise ConfigError("itr_max must be at least 1")
        if not np.isfinite(self.tol) or self.tol < 0:
            raise ConfigError("tol must be a nonnegative finite real")
        if not np.isfinite(self.absorb_threshold) or self.absorb_threshold <= 1:
            raise ConfigError("absorb_threshold must exceed 1")
        if self.check_every < 1:
            raise ConfigError("check_every must be at least 1")
        if self.plan_cap < 1:
            raise ConfigError("plan_cap must be positive")


@dataclass
class SolverState:
    """solver.py:64-73."""

    phi: np.ndarray
    psi: np.ndarray
    a: Optional[np.ndarray] = None
    b: Optional[np.ndarray] = None
    iteration: int = 0
    last_marginal_error: float = np.inf


@dataclass
class Solution:
    """solver.py:76-89.  ``kernel`` is a device-backed operator handle."""

    phi: np.ndarray
    psi: np.ndarray
    a: np.ndarray
    b: np.ndarray
    kernel: object
    iterations_run: int
    converged: bool
    marginal_error_history: list
    wall_time: float
    setup_time: float
    cost: float
    config: SolverConfig
    absorb_iterations: Optional[list] = None


def raise_status(status):
    """Status code -> the reference's exception (solver.py:177-184)."""
    if status == ZERO_DENOM:
        raise ZeroDenominator(_MSG_ZD)
    if status == NONFINITE:
        raise NonFiniteIterate(_MSG_NF)


def history_from(errs, iterations, converged, config):
    """Apply the reference's recording cadence (solver.py:185-192) to per-iteration errors."""
    its = np.arange(1, iterations + 1)
    keep = (its % config.check_every == 0) | (its == config.itr_max)
    vals = np.asarray(errs[:iterations], dtype=np.float64)
    hist = list(zip(its[keep].tolist(), vals[keep].tolist()))
    if converged and (not hist or hist[-1][0] != iterations):
        hist.append((iterations, float(vals[iterations - 1])))
    return hist


def _shift(weights, scaling, epsilon):
    """solver.py:135-153 (host copy, used by run_driver with reference adapters)."""
    pos = weights > 0
    vals = epsilon * np.log(scaling[pos])
    if pos.all():
        return vals
    out = np.empty(weights.shape[0])
    idx = np.arange(weights.shape[0], dtype=float)
    out[pos] = vals
    out[~pos] = np.interp(idx[~pos], idx[pos], vals)
    return out


def run_driver(adapter, u, v, config):
    """The reference's scaling loop over any adapter (solver.py:156-199)."""
    n = u.shape[0]
    phi = np.full(n, 1.0 / n)
    psi = np.full(v.shape[0], 1.0 / n)
    hi_cut = np.exp(config.absorb_threshold)
    lo_cut = np.exp(-config.absorb_threshold)
    history = []
    converged = False
    it = 0
    t0 = perf_counter()
    while it < config.itr_max:
        err, status, psmax, psmin, phmax, phmin = adapter.iterate(u, v, phi, psi)
        it += 1
        raise_status(status)
        recorded = it % config.check_every == 0 or it == config.itr_max
        if recorded:
            history.append((it, float(err)))
        if config.tol > 0 and err <= config.tol:
            if not recorded:
                history.append((it, float(err)))
            converged = True
            break
        if config.stabilize and (phmax > hi_cut or psmax > hi_cut
                                 or phmin < lo_cut or psmin < lo_cut):
            adapter.absorb(_shift(u, phi, config.epsilon), _shift(v, psi, config.epsilon))
            phi[:] = 1.0
            psi[:] = 1.0
    return phi, psi, it, converged, history, perf_counter() - t0


class GpuAdapter1D:
    """Adapter-protocol backend on the B200 kernels (solver.py:1-16, :92-132).

    ``iterate`` runs one fused iteration on device (finom_iterate1d) and
    updates phi/psi in place, so the reference's own run_driver can drive it.
    """

    def __init__(self, x, y, epsilon):
        self.op = kernel1d.build_operator(x, y, epsilon)

    @property
    def kernel(self):
        return self.op

    @property
    def a(self):
        return self.op.absorption_left

    @property
    def b(self):
        return self.op.absorption_right

    def iterate(self, u, v, phi, psi):
        import torch
        dev = torch.device("cuda")
        plan = self.op.plan()
        tu = torch.from_numpy(np.ascontiguousarray(u, dtype=np.float64)).to(dev)
        tv = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)).to(dev)
        tphi = torch.from_numpy(np.ascontiguousarray(phi)).to(dev)
        tpsi = torch.from_numpy(np.ascontiguousarray(psi)).to(dev)
        ta = tb = None
        if self.op.absorbed:
            ta = torch.from_numpy(np.ascontiguousarray(self.a)).to(dev)
            tb = torch.from_numpy(np.ascontiguousarray(self.b)).to(dev)
        res = torch.zeros(6, dtype=torch.float64, device=dev)
        lib = plan.lib
        _lib.check(lib.finom_iterate1d(plan.handle, _lib.ptr(tu), _lib.ptr(tv), _lib.ptr(tphi),
                                       _lib.ptr(tpsi), _lib.ptr(ta), _lib.ptr(tb), _lib.ptr(res),
                                       _lib.stream_ptr()), "finom_iterate1d", lib)
        r = res.cpu().numpy()
        phi[:] = tphi.cpu().numpy()
        psi[:] = tpsi.cpu().numpy()
        return float(r[0]), int(r[1]), float(r[2]), float(r[3]), float(r[4]), float(r[5])

    def absorb(self, delta_a, delta_b):
        self.op = kernel1d.absorb(self.op, delta_a, delta_b)


def sinkhorn_1d(x, y, u, v, config):
    """Entropic scaling on 1D meshes, whole loop on the B200 (solver.py:202-230)."""
    if len(u.weights) != len(x):
        raise DimensionMismatch("u must have one weight per source node")
    if len(v.weights) != len(y):
        raise DimensionMismatch("v must have one weight per target node")
    n, m, itr = len(x), len(y), int(config.itr_max)
    lib = _lib.lib_for(1, n + m)
    phi, a = np.empty(n), np.empty(n)
    psi, b = np.empty(m), np.empty(m)
    hist = np.zeros(itr)
    info = np.zeros(5, dtype=np.int64)
    abs_its = np.zeros(itr, dtype=np.int64)
    cost = np.zeros(1)
    timing = np.zeros(3)
    status = _lib.check(lib.finom_sinkhorn1d_host(
        n, _lib.ptr(x.nodes), m, _lib.ptr(y.nodes), _lib.ptr(u.weights), _lib.ptr(v.weights),
        config.epsilon, itr, float(config.tol), int(bool(config.stabilize)),
        float(config.absorb_threshold), _lib.ptr(phi), _lib.ptr(psi), _lib.ptr(a), _lib.ptr(b),
        _lib.ptr(hist), _lib.ptr(info), _lib.ptr(abs_its), _lib.ptr(cost), _lib.ptr(timing)),
        "finom_sinkhorn1d_host", lib)
    raise_status(status)
    its, conv = int(info[0]), bool(info[1])
    op = kernel1d.build_operator(x, y, config.epsilon)
    op = kernel1d.KernelOperator1D(x, y, op.epsilon, a, b, op._plans)
    return Solution(
        phi=phi, psi=psi, a=a, b=b, kernel=op, iterations_run=its, converged=conv,
        marginal_error_history=history_from(hist, its, conv, config),
        wall_time=float(timing[0] + timing[1]), setup_time=float(timing[0]),
        cost=float(cost[0]), config=config,
        absorb_iterations=[int(k) for k in abs_its[:int(info[3])]])


class BatchSolver1D:
    """Device-resident batch of independent 1D problems (no reference equivalent;
    per-problem semantics == sinkhorn_1d).  Inputs stay in HBM between solves."""

    def __init__(self, xs, ys, us, vs, epsilons):
        import torch
        if not (len(xs) == len(ys) == len(us) == len(vs)):
            raise DimensionMismatch("xs, ys, us, vs must have one entry per problem")
        for k, (x, y, u, v) in enumerate(zip(xs, ys, us, vs)):
            if len(u) != len(x) or len(v) != len(y):
                raise DimensionMismatch("problem %d: weight/mesh length mismatch" % k)
        eps = np.broadcast_to(np.asarray(epsilons, dtype=np.float64), (len(xs),))
        for e in eps:
            if not np.isfinite(e) or e <= 0:
                raise InvalidEpsilon("epsilon must be a positive finite real")
        node = lambda z: z.nodes if hasattr(z, "nodes") else np.asarray(z, dtype=np.float64)
        wts = lambda z: z.weights if hasattr(z, "weights") else np.asarray(z, dtype=np.float64)
        self.plan = _lib.Plan1D([node(x) for x in xs], [node(y) for y in ys], eps)
        dev = torch.device("cuda")
        self.P = self.plan.P
        self.eps = np.array(eps)
        f64 = dict(dtype=torch.float64, device=dev)
        hu = [np.ascontiguousarray(wts(u), dtype=np.float64) for u in us]
        hv = [np.ascontiguousarray(wts(v), dtype=np.float64) for v in vs]
        self.u = torch.empty(int(self.plan.xoff[-1]), dtype=torch.float64, device=dev)
        self.v = torch.empty(int(self.plan.yoff[-1]), dtype=torch.float64, device=dev)
        _lib.stage_pieces(0, hu, self.u)  # (straight from the problems' arrays)
        _lib.stage_pieces(0, hv, self.v)
        NX, NY = self.u.numel(), self.v.numel()
        self.phi = torch.empty(NX, **f64)
        self.psi = torch.empty(NY, **f64)
        self.a = torch.empty(NX, **f64)
        self.b = torch.empty(NY, **f64)
        self.cost = torch.empty(self.P, **f64)
        self._itr = None

    def _bufs(self, itr):
        import torch
        if self._itr != itr:
            dev = self.phi.device
            self.hist = torch.zeros(self.P * itr, dtype=torch.float64, device=dev)
            self.info = torch.zeros(self.P * 5, dtype=torch.int64, device=dev)
            self.abs_its = torch.zeros(self.P * itr, dtype=torch.int64, device=dev)
            self._itr = itr

    def solve(self, itr_max, tol=0.0, stabilize=True, absorb_threshold=200.0, sync=True):
        """Run the device loop on the current stream; returns the worst status
        (0/1/2) -- or, with sync=False, 0 as soon as the loop is queued (the
        per-problem status is then info[5 p + 2] once the stream has run)."""
        self._bufs(int(itr_max))
        lib = self.plan.lib
        fn = lib.finom_solve1d if sync else lib.finom_solve1d_async
        return _lib.check(fn(
            self.plan.handle, _lib.ptr(self.u), _lib.ptr(self.v), _lib.ptr(self.phi),
            _lib.ptr(self.psi), _lib.ptr(self.a), _lib.ptr(self.b), int(itr_max), float(tol),
            int(bool(stabilize)), float(absorb_threshold), _lib.ptr(self.hist),
            _lib.ptr(self.info), _lib.ptr(self.abs_its), _lib.stream_ptr()), "finom_solve1d", lib)

    def compute_cost(self):
        lib = self.plan.lib
        _lib.check(lib.finom_cost1d(self.plan.handle, _lib.ptr(self.a), _lib.ptr(self.b),
                                    _lib.ptr(self.phi), _lib.ptr(self.psi),
                                    _lib.ptr(self.cost), _lib.stream_ptr()), "finom_cost1d", lib)
        return self.cost


_STAGE_STREAMS = {}


def _stage_stream(k):
    """The copy stream of pipeline stage k: two per device, created once.
    torch's caching allocator keeps blocks per stream, so stage buffers
    allocated on fresh streams every call find no cached blocks and fall back
    to cudaMalloc -- and, with the cache full, to a cudaFree that waits for the
    running loop (host hiccups of 0.2-0.7 s measured on config 5)."""
    import torch
    dev = torch.cuda.current_device()
    if dev not in _STAGE_STREAMS:
        _STAGE_STREAMS[dev] = (torch.cuda.Stream(), torch.cuda.Stream())
    return _STAGE_STREAMS[dev][k % 2]


def _pipeline_ranges(sizes):
    """Problem ranges of the batched API's pipeline stages.

    Batches of >= 1024 problems and >= 2^24 points run as a short first and
    last stage around equal middle stages of ~2368 problems: the first
    stage's preparation (plan + host -> device) and the last stage's fetch are
    the only transfers the device loops do not hide, so those two stages are
    small -- 4 x 148 problems (two rounds of the 296 problems a B200 holds at
    8 warps per problem) from 4096 problems on, 2 x 148 below -- and a second
    stage of twice the first follows when the batch allows, so that every
    stage's preparation hides behind the loop before it.  Smaller batches
    take one stage; batches of many small problems (< 4096 points each on
    average) equal stages of >= 2048 problems and >= 2^22 points.  FINOM_PIPE_SIZES = "n0,n1,..." sets the stages'
    problem counts; FINOM_PIPE_STAGES = k asks for k equal stages
    (FINOM_PIPE_FIRST: a small first stage of that many problems before them).
    Config 5 (8192 x 16384, warm calls): 1 stage 1.53 s; 8 stages of 1024
    1.23-1.81 s (each stage's loop takes 144 ms against 131 for 1/8 of the
    batch, and the host's preparation of a stage sometimes outlasts it); 4
    stages of 2048 1.07-1.08 s; 592 + 3 x 2336 + 592 1.02-1.03 s; 592 + 1184 +
    2 x 2912 + 592 1.01 s for 0.97 s of device loops.  A rank's share of the
    batch at 2 / 4 / 8 GPUs (4096 / 2048 / 1024 problems): 0.521 / 0.267 /
    0.151 s against 0.588 / 0.355 / 0.197 s unstaged or in stages of 2048."""
    P, pts = len(sizes), int(np.sum(sizes))
    explicit = os.environ.get("FINOM_PIPE_SIZES")
    if explicit:
        cuts = np.minimum(np.cumsum([0] + [int(t) for t in explicit.split(",")]), P)
        cuts[-1] = P
        return [(int(lo), int(hi)) for lo, hi in zip(cuts[:-1], cuts[1:]) if hi > lo]
    env = os.environ.get("FINOM_PIPE_STAGES")
    if env:
        k = max(1, min(int(env), P))
        f = int(os.environ.get("FINOM_PIPE_FIRST", "0")) if k > 1 else 0
        f = max(0, min(f, P - k))
        return ([(0, f)] if f else []) + [(f + (P - f) * i // k, f + (P - f) * (i + 1) // k)
                                          for i in range(k)]
    if P < 1024 or pts < (1 << 24):
        return [(0, P)]
    if pts < 4096 * P:
        # many small problems: equal stages of >= 2048 problems and >= 2^22
        # points (the short stages above would be all overhead)
        k = max(1, min(8, P // 2048, pts >> 22))
        return [(P * i // k, P * (i + 1) // k) for i in range(k)]
    edge = 4 * 148 if P >= 4096 else 2 * 148
    # a second stage of twice the first when the batch allows: its preparation
    # hides behind the first stage's loop, the big stages' behind its own
    head = [edge, 2 * edge] if P - 4 * edge >= 2 * edge else [edge]
    lo = sum(head)
    mid = P - lo - edge
    k = max(1, int(round(mid / 2368.0)))
    cuts = [0] + list(np.cumsum(head)) + [lo + mid * (i + 1) // k for i in range(k)] + [P]
    return [(int(a), int(b)) for a, b in zip(cuts[:-1], cuts[1:])]


def sinkhorn_1d_batched(xs, ys, us, vs, config, epsilons=None):
    """Batch of independent sinkhorn_1d problems in one device loop.

    ``config`` supplies itr_max / tol / stabilize / threshold / cadence for all
    problems; ``epsilons`` (optional) overrides config.epsilon per problem.
    Raises the reference's exception if any problem fails.

    Large batches run as a pipeline of stages (problem ranges): stage k + 1's
    plan and host -> device staging (a copy stream) and stage k - 1's results
    device -> host run while stage k's loop runs on the compute stream, so the
    transfers and host-side tiling hide behind the device loop.  Every problem
    is solved exactly as in a single-stage call (problems are independent).
    """
    import torch
    if not (len(xs) == len(ys) == len(us) == len(vs)):
        raise DimensionMismatch("xs, ys, us, vs must have one entry per problem")
    P = len(xs)
    eps = np.broadcast_to(np.asarray(config.epsilon if epsilons is None else epsilons,
                                     dtype=np.float64), (P,))
    verbose = os.environ.get("FB_VERBOSE")
    node = lambda z: z.nodes if hasattr(z, "nodes") else np.asarray(z, dtype=np.float64)
    nx = np.array([len(node(x)) for x in xs], dtype=np.int64)
    ny = np.array([len(node(y)) for y in ys], dtype=np.int64)
    xoff = np.zeros(P + 1, dtype=np.int64)
    yoff = np.zeros(P + 1, dtype=np.int64)
    xoff[1:] = np.cumsum(nx)
    yoff[1:] = np.cumsum(ny)
    itr = int(config.itr_max)
    # the batch's results, filled stage by stage (device -> host through the pinned staging)
    phi = np.empty(int(xoff[-1]))
    psi = np.empty(int(yoff[-1]))
    a = np.empty(int(xoff[-1]))
    b = np.empty(int(yoff[-1]))
    hist = np.empty((P, itr))
    abs_its = np.empty((P, itr), dtype=np.int64)
    info = np.empty((P, 5), dtype=np.int64)
    cost = np.empty(P)
    comp = torch.cuda.current_stream()
    t0 = perf_counter()
    setup = [0.0]
    ranges = _pipeline_ranges(nx)
    # First-touch page faults of the fresh result arrays cost about as much as
    # the device -> host copies into them: host threads touch each stage's
    # slices while the device loops run (ctypes.memset releases the GIL), and
    # a stage's results are fetched once its slices are touched.
    import ctypes
    import threading

    def touch(lo, hi):
        x0, x1, y0, y1 = xoff[lo], xoff[hi], yoff[lo], yoff[hi]
        for arr, s0, s1 in ((phi, x0, x1), (psi, y0, y1), (a, x0, x1), (b, y0, y1),
                            (hist, lo, hi), (abs_its, lo, hi)):
            v = arr[s0:s1]
            if v.nbytes:
                ctypes.memset(v.ctypes.data, 0, v.nbytes)

    touched = {k: threading.Event() for k in range(len(ranges))}
    if len(ranges) > 1 and os.environ.get("FINOM_PIPE_TOUCH", "1") != "0":
        def toucher():
            for k, (lo, hi) in enumerate(ranges):
                touch(lo, hi)
                touched[k].set()
        tt = threading.Thread(target=toucher, daemon=True)
    else:
        tt = None

    def fetch(stage):
        lo, hi, bs, done, k = stage
        if tt is not None:
            touched[k].wait()
        done.synchronize()
        x0, x1, y0, y1 = xoff[lo], xoff[hi], yoff[lo], yoff[hi]
        for h, d in ((phi[x0:x1], bs.phi), (psi[y0:y1], bs.psi), (a[x0:x1], bs.a),
                     (b[y0:y1], bs.b), (hist[lo:hi].reshape(-1), bs.hist),
                     (abs_its[lo:hi].reshape(-1), bs.abs_its), (info[lo:hi].reshape(-1), bs.info),
                     (cost[lo:hi], bs.cost)):
            _lib.stage_copy(1, h, d)

    pending = None
    marks = []
    stages = []  # (kept to the end: destroying a plan waits for every stream it ran on)
    for si, (lo, hi) in enumerate(ranges):
        ts = perf_counter()
        # plan (host tiling + H2D) and weights on a stream of the stage's own:
        # nothing queued on it can make its pageable copies wait for the
        # stages before (whose kernels wait for the SMs the running loop holds)
        copy = _stage_stream(si) if os.environ.get("FINOM_PIPE_FIXED", "1") != "0" \
            else torch.cuda.Stream()
        with torch.cuda.stream(copy):
            bs = BatchSolver1D(xs[lo:hi], ys[lo:hi], us[lo:hi], vs[lo:hi], eps[lo:hi])
            bs._bufs(itr)
            ready = torch.cuda.Event()
            ready.record(copy)
        tp = perf_counter()
        setup[0] += tp - ts
        comp.wait_event(ready)
        for t in (bs.u, bs.v, bs.phi, bs.psi, bs.a, bs.b, bs.cost, bs.hist, bs.info, bs.abs_its):
            t.record_stream(comp)
        start = torch.cuda.Event(enable_timing=True)
        start.record(comp)
        bs.solve(itr, config.tol, config.stabilize, config.absorb_threshold, sync=False)
        bs.compute_cost()
        done = torch.cuda.Event(enable_timing=True)
        done.record(comp)
        if si == 0 and tt is not None:
            tt.start()  # (after the first stage's loop is queued: the host is idle meanwhile)
        if verbose:
            marks.append((start, done))
        tq = perf_counter()
        if pending is not None:
            fetch(pending)
        if verbose:
            print("  stage %d-%d: prep %.1f ms, queue %.1f ms, fetch (previous) %.1f ms" % (
                lo, hi, 1e3 * (tp - ts), 1e3 * (tq - tp), 1e3 * (perf_counter() - tq)), flush=True)
        pending = (lo, hi, bs, done, si)
        stages.append(bs)
    fetch(pending)
    wall = perf_counter() - t0
    del stages, bs, pending
    raise_status(int(info[:, 2].max()) if P else 0)
    sols = BatchSolutions(xs, ys, xoff, yoff, np.array(eps), config, info, cost,
                          phi, psi, a, b, hist, abs_its, wall, setup[0])
    if verbose:
        print("sinkhorn_1d_batched: %d stage(s), setup %.1f ms, call %.1f ms; device loop "
              "+ cost per stage %s ms, gaps %s ms" % (
                  len(ranges), 1e3 * setup[0], 1e3 * wall,
                  ["%.1f" % a.elapsed_time(b) for a, b in marks],
                  ["%.1f" % marks[k][1].elapsed_time(marks[k + 1][0])
                   for k in range(len(marks) - 1)]), flush=True)
    return sols


class BatchSolutions(Sequence):
    """The per-problem Solutions of a batched solve, as a sequence.

    Every result is already on the host in the batch's arrays when the call
    returns (phi / psi / a / b, histories, infos, costs); element p is a
    Solution whose vectors are disjoint views of those arrays (no copies),
    built when first accessed -- a list of 8192 dataclass objects and
    operator handles costs ~0.3 s of Python that a caller iterating over a
    few problems never needs."""

    def __init__(self, xs, ys, xoff, yoff, eps, config, info, cost, phi, psi, a, b, hist,
                 abs_its, wall, setup):
        self._xs, self._ys, self._xo, self._yo = xs, ys, xoff, yoff
        self._eps, self._config = eps, config
        self._info, self._cost = info, cost
        self.phi, self.psi, self.a, self.b = phi, psi, a, b
        self._hist, self._abs_its = hist, abs_its
        self._wall, self._setup = wall, setup
        self._cache = {}

    def __len__(self):
        return len(self._xs)

    def _make(self, p):
        config = self._config
        x = self._xs[p] if hasattr(self._xs[p], "nodes") else None
        y = self._ys[p] if hasattr(self._ys[p], "nodes") else None
        sl = slice(self._xo[p], self._xo[p + 1])
        tl = slice(self._yo[p], self._yo[p + 1])
        e = float(self._eps[p])
        cfg = config if e == config.epsilon else replace(config, epsilon=e)
        ap, bp = self.a[sl], self.b[tl]
        op = None
        if x is not None and y is not None:
            op = kernel1d.KernelOperator1D(x, y, e, ap, bp, kernel1d._PlanCache(x, y, e))
        its, conv, _, nab, _ = (int(v) for v in self._info[p])
        return Solution(
            phi=self.phi[sl], psi=self.psi[tl], a=ap, b=bp, kernel=op,
            iterations_run=its, converged=bool(conv),
            marginal_error_history=history_from(self._hist[p], its, bool(conv), cfg),
            wall_time=self._wall, setup_time=self._setup, cost=float(self._cost[p]),
            config=cfg, absorb_iterations=self._abs_its[p, :nab].tolist())

    def __getitem__(self, k):
        if isinstance(k, slice):
            return [self[i] for i in range(*k.indices(len(self)))]
        if k < 0:
            k += len(self)
        if not 0 <= k < len(self):
            raise IndexError(k)
        if k not in self._cache:
            self._cache[k] = self._make(k)
        return self._cache[k]


def marginal_error(state, kernel, v):
    """L1 distance of diag(psi) K^T phi from the target weights (solver.py:233-237)."""
    w = v.weights if hasattr(v, "weights") else np.asarray(v, dtype=float)
    t = kernel.apply_transpose(state.phi)
    return float(np.sum(np.abs(state.psi * t - w)))


def plan_dense(solution):
    """diag(phi) K diag(psi) (solver.py:240-249), materialized on the device
    in one pass: (phi_i * K'_ij) * psi_j (finom_dense1d / finom_dense2d)."""
    kern = solution.kernel
    n, m = kern.shape
    if n * m > solution.config.plan_cap:
        raise SizeCapExceeded("plan has %d entries, cap is %d" % (n * m, solution.config.plan_cap))
    if isinstance(kern, kernel1d.KernelOperator1D):
        return _lib.dense1d(kern.x_mesh.nodes, kern.y_mesh.nodes, kern.absorption_left,
                            kern.absorption_right, kern.epsilon, solution.phi, solution.psi)
    from .kernel2d import KernelOperator2D, dense_realization_2d
    if isinstance(kern, KernelOperator2D):
        return dense_realization_2d(kern, solution.phi, solution.psi)
    dense = kern.dense_realization()  # (the dense baseline's kernel)
    return solution.phi[:, None] * dense * solution.psi[None, :]


def transport_cost_fast(solution):
    """<C, plan> in linear time on the device (solver.py:252-271)."""
    import torch
    op = solution.kernel
    if not isinstance(op, kernel1d.KernelOperator1D):
        from .kernel2d import transport_cost_fast_2d
        return transport_cost_fast_2d(solution)
    dev = torch.device("cuda")
    plan = op.plan()
    t = lambda arr: torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64)).to(dev)
    tphi, tpsi = t(solution.phi), t(solution.psi)
    ta = t(op.absorption_left) if op.absorbed else None
    tb = t(op.absorption_right) if op.absorbed else None
    out = torch.zeros(1, dtype=torch.float64, device=dev)
    lib = plan.lib
    _lib.check(lib.finom_cost1d(plan.handle, _lib.ptr(ta), _lib.ptr(tb), _lib.ptr(tphi),
                                _lib.ptr(tpsi), _lib.ptr(out), _lib.stream_ptr()), "finom_cost1d",
               lib)
    return float(out.item())
