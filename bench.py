"""Benchmark of the FINOM Sinkhorn hot path on B200 (driver contract).

Default workload: BASELINE.json config 5 at every GPU count (the metric is
quoted on 1/2/4/8 B200; config 5 is the configuration that shards): a batch
of 8192 1D W1 Sinkhorn problems, fp64, N = M = 16384 each, eps per problem
10^U[-3,-1], 200 fixed iterations, log-domain stabilization on
(absorptions happen inside the timed loop), the batch split by problem
across the ranks ("scaling": "strong", no data-path collective).  One step
= one full 200-iteration solve of the rank's problems through the device
loop.  --config 2 is the single-GPU 1D problem (N = M = 2^22), --config
1/3/4 the other BASELINE configs (4 row-sharded under torchrun).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--config 1..5]

--gpus N without torchrun re-executes itself under torch.distributed.run
with N ranks (127.0.0.1); under torchrun WORLD_SIZE must equal N.

value: mesh-points x iterations / s over the device loop, inputs resident
in HBM (CUDA events on the launching stream, barrier + sync both sides, max
over ranks).  e2e: the same metric through the public API with host
buffers (solver.sinkhorn_1d), every copy inside the timed region.
--impl reference: the reference algorithm on the host CPU (the C oracle
port, oracle/finom_oracle.c), a bounded sample of the same workload.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Sinkhorn mesh-points x iterations/s (fp64)"
UNIT = "pts*it/s"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:  # noqa: BLE001
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json copy test)"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(name, cfg):
    """dram bytes per launch of the dominant kernel (per iteration for a
    whole-solve kernel) from the committed ncu summary of this config."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        e = d.get("config%d" % cfg, {}).get(name) or (d.get(name) if cfg == 2 else None)
        return None if e is None else e.get("dram_bytes_per_iteration",
                                             e.get("dram_bytes_per_launch"))
    except Exception:  # noqa: BLE001
        return None


def workload(cfg, rank=0, world=1):
    from paper_2605_26659_b200 import workloads as W
    if cfg == 1:
        x, y, u, v, eps = W.config1()
        return dict(xs=[x], ys=[y], us=[u], vs=[v], eps=[eps], itr=500, name="config1")
    if cfg == 2:
        x, y, u, v, eps = W.config2()
        return dict(xs=[x], ys=[y], us=[u], vs=[v], eps=[eps], itr=200, name="config2")
    if cfg == 5:
        B = int(os.environ.get("FINOM_BATCH", "8192"))
        lo, hi = rank * B // world, (rank + 1) * B // world
        probs = W.config5(batch=B, problems=range(lo, hi))
        return dict(xs=[p[0] for p in probs], ys=[p[1] for p in probs],
                    us=[p[2] for p in probs], vs=[p[3] for p in probs],
                    eps=[p[4] for p in probs], itr=200, name="config5", batch=B)
    if cfg in (3, 4):
        x1, y1, x2, y2, U, V, eps = W.config3() if cfg == 3 else W.config4()
        return dict(grid=(x1, y1, x2, y2, U, V), eps=[eps], itr=300 if cfg == 3 else 100,
                    name="config%d" % cfg)
    raise SystemExit("unknown config %r" % cfg)


def run_2d(args, cfg, wl, world=1, rank=0):
    """2D configs (3: 1024^2, 4: 8192^2).  One GPU: sinkhorn_2d (value from its
    loop window).  Under torchrun (world > 1): the row-sharded solve
    (sharding.sinkhorn_2d_row_sharded, NCCL carry exchange), time = max over
    ranks, total work fixed ("scaling": "strong")."""
    import paper_2605_26659_b200 as fb
    x1, y1, x2, y2, U, V = wl["grid"]
    src = fb.Grid2D(fb.Mesh1D(x1), fb.Mesh1D(y1))
    tgt = fb.Grid2D(fb.Mesh1D(x2), fb.Mesh1D(y2))
    scfg = fb.SolverConfig(epsilon=wl["eps"][0], itr_max=wl["itr"], tol=0.0, stabilize=True)
    mu, mv = fb.Measure2D(U), fb.Measure2D(V)
    pts = x1.size * y1.size
    if world > 1:
        from paper_2605_26659_b200 import sharding as S
        run = lambda: S.sinkhorn_2d_row_sharded(src, tgt, mu, mv, scfg)
    else:
        run = lambda: fb.sinkhorn_2d(src, tgt, mu, mv, scfg)
    launches = None
    if world > 1:
        for _ in range(max(1, min(args.warmup, 2))):
            run()
        loops, walls = [], []
        clocks = Clocks(int(os.environ.get("LOCAL_RANK", "0")))
        clocks.start()
        for _ in range(args.steps):
            t0 = time.perf_counter()
            sol = run()
            walls.append(time.perf_counter() - t0)
            loops.append(sol.wall_time - sol.setup_time)
        ck = clocks.stop()
        loop = statistics.median(loops)
    else:
        # device-resident solve (GridSolver2D: weights and iterates in HBM,
        # finom_solve2d), CUDA events on its stream around the K timed solves
        import torch
        gs = fb.GridSolver2D(src, tgt, wl["eps"][0], mu, mv)
        for _ in range(max(args.warmup, 3)):
            gs.solve(wl["itr"], 0.0, True, 200.0)
        torch.cuda.synchronize()
        clocks = Clocks(int(os.environ.get("LOCAL_RANK", "0")))
        clocks.start()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            gs.solve(wl["itr"], 0.0, True, 200.0)
        e1.record()
        torch.cuda.synchronize()
        ck = clocks.stop()
        loop = e0.elapsed_time(e1) * 1e-3 / args.steps
        loops = [loop]
        launches = gs.grid.info()["launches"] * args.steps
        del gs
        # end to end: the public host-array API (plan, copies, loop, cost, results out)
        run()
        walls = []
        for _ in range(max(1, min(args.steps, 3))):
            t0 = time.perf_counter()
            sol = run()
            walls.append(time.perf_counter() - t0)
    if rank != 0:
        return
    # roofline of the whole iteration: 88 B/pt before the first
    # absorption, 120 B/pt after (the two-sweep algorithm with a materialised
    # intermediate), weighted by the iterations spent in either state
    cpu = None
    if not args.no_cpu_baseline:
        # the C port (oracle/) of the reference's 2D loop on one host core: a
        # bounded number of iterations of the full-size grid, wall clock of the
        # call (its setup is O(n + m) table builds, negligible at these sizes)
        from oracle import oracle as O
        its = 60 if cfg == 3 else 3
        t0 = time.perf_counter()
        O.sinkhorn_2d(x1, y1, x2, y2, U, V, wl["eps"][0], its, 0.0, True)
        dt = time.perf_counter() - t0
        cpu = {"value": pts * its / dt, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": "config%d full-size grid, first %d of %d iterations (stabilize=True), "
                         "wall clock of the call" % (cfg, its, wl["itr"])}
    a0 = sol.absorb_iterations[0] if len(sol.absorb_iterations) else sol.iterations_run
    abytes = pts * (88.0 * a0 + 120.0 * (sol.iterations_run - a0))
    peak, psrc = peaks()
    achieved = abytes / loop / 1e9
    line = {
        "metric": METRIC, "value": pts * wl["itr"] / loop, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * loop,
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generators, BASELINE.json shapes; see DESIGN.md)",
        "config": {"workload": "config%d: 2D %dx%d eps=%g %d it (stabilize=True)" % (
            cfg, x1.size, y1.size, wl["eps"][0], wl["itr"]), "itr_max": wl["itr"],
            "parallelism": "row shards x%d (carry exchange)" % world if world > 1 else "1 GPU",
            "timing": ("loop window (max over ranks); host-driven loop, one sync per "
                       "iteration") if world > 1 else (
                "CUDA events around K device-resident solves (GridSolver2D / finom_solve2d: "
                "device-looped CUDA graph, host sync only at absorptions)")},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": ncu_traffic("iteration", cfg),
                     "traffic_unit": "DRAM bytes per iteration (ncu launch list)",
                     "peak_source": psrc,
                     "kernel": "whole iteration: 4 line sweeps (k_sq_pre/k_sq_scan/k_sq_apply) "
                               "+ fused scaling updates",
                     "algorithmic_bytes_per_solve": abytes,
                     "bytes_rule": "88 B/pt unabsorbed, 120 B/pt absorbed (SURVEY 8d)"},
        "e2e": {"value": pts * wl["itr"] / statistics.median(walls), "unit": UNIT,
                "h2d_bytes_per_step": 8 * (2 * pts + 2 * x1.size + 2 * y1.size),
                "d2h_bytes_per_step": 8 * 4 * pts},
        "cpu_baseline": cpu,
        "gpu_launches": launches,
        "iterations_run": sol.iterations_run, "absorbs": sol.absorb_iterations,
        "cost": sol.cost, "clocks": ck, "loops_ms": [round(1e3 * x, 2) for x in loops],
    }
    print(json.dumps(line), flush=True)


def config_json(cfg, wl, world):
    base = {"l2": "inputs larger than L2 (working set > 126 MB per iteration)",
            "tol": 0.0, "stabilize": True, "absorb_threshold": 200.0}
    if cfg == 1:
        base.update(workload="config1: 1D N=M=1e4 random gaps U[0.2,1.8], eps=1e-2, 500 it",
                    n=10_000, m=10_000, itr_max=500,
                    l2="working set 0.9 MB is L2/SM-resident (latency-bound config)")
    elif cfg == 2:
        base.update(workload="config2: 1D N=M=2^22 graded meshes x=(i/N)^2, y=1-(1-j/N)^2, "
                             "3-component mixtures, eps=1e-3, 200 it", n=1 << 22, m=1 << 22,
                    itr_max=200)
    else:
        base.update(workload="config5: batch of %d 1D problems, N=M=16384, eps=10^U[-3,-1], "
                             "200 it, sharded by problem" % wl["batch"], n=16_384, m=16_384,
                    batch=wl["batch"], itr_max=200)
    base["parallelism"] = ("replicas" if cfg != 5 else "problem-sharded") + " x%d" % world
    return base


def cpu_batch(probs, its):
    """Config 5 on the host: the C port over independent problems on every
    core (ctypes releases the GIL; SPEC.md:389 allows concurrent instances).
    Returns (pts*it/s, wall seconds, threads)."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle import oracle as O
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=cores) as ex:
        list(ex.map(lambda p: O.sinkhorn_1d(p[0], p[1], p[2], p[3], p[4], its, 0.0, True), probs))
    wall = time.perf_counter() - t0
    return sum(p[0].size for p in probs) * its / wall, wall, cores


def run_reference(args):
    """Reference arm: the reference algorithm (C port of pkg/src/finom) on host CPU."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O
    cfg = args.config
    wl = workload(cfg) if cfg != 5 else None
    cores = 1
    if cfg == 5:
        from paper_2605_26659_b200 import workloads as W
        nprob = 4 * (os.cpu_count() or 1)
        probs = W.config5(problems=range(nprob))
        sample_its = 200
    else:
        sample_its = {1: 500, 2: 20}[cfg]
    vals, loops = [], []
    for s in range(args.warmup + args.steps):
        if cfg == 5:
            v5, t, cores = cpu_batch(probs, sample_its)
            pts = sum(p[0].size for p in probs)
        else:
            r = O.sinkhorn_1d(wl["xs"][0], wl["ys"][0], wl["us"][0], wl["vs"][0], wl["eps"][0],
                              sample_its, 0.0, True)
            t = r["loop_s"]
            pts = wl["xs"][0].size
        if s >= args.warmup:
            vals.append(pts * sample_its / t)
            loops.append(t)
    value = float(statistics.median(vals))
    sample = ("%s, %d iterations of the full-size problem (stabilize=True), loop window "
              "(wall_time - setup_time) per step" % ({1: "config1", 2: "config2"}.get(cfg, ""),
                                                     sample_its)) if cfg != 5 else (
        "config5 problems 0-%d (of 8192), 200 iterations each, one C-port instance per "
        "host thread" % (len(probs) - 1))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(loops),
        "higher_is_better": True, "scaling": "strong" if cfg in (4, 5) else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE.json shapes)",
        "config": config_json(cfg, {"batch": 8192}, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def relaunch_distributed(args):
    """--gpus N > 1 outside torchrun: run this script under torch.distributed.run
    with N ranks on this node (the driver's own launch form)."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           "--nproc-per-node", str(args.gpus), "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=5, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        relaunch_distributed(args)
    if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) != args.gpus:
        raise SystemExit("bench.py: WORLD_SIZE=%s but --gpus %d" % (os.environ["WORLD_SIZE"],
                                                                  args.gpus))
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2605_26659_b200 as fb
    from paper_2605_26659_b200 import _lib

    cfg = args.config
    wl = workload(cfg, rank, world)
    if cfg in (3, 4):
        if cfg == 4 or world == 1:
            run_2d(args, cfg, wl, world, rank)
        elif rank == 0:
            run_2d(args, cfg, wl)
        if world > 1:
            torch.distributed.destroy_process_group()
        return
    itr = wl["itr"]
    bs = fb.BatchSolver1D(wl["xs"], wl["ys"], wl["us"], wl["vs"], wl["eps"])
    pts = int(sum(x.size for x in wl["xs"]))
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    for _ in range(max(args.warmup, 3) if args.warmup >= 3 else 3):
        st = bs.solve(itr, 0.0, True, 200.0)
    torch.cuda.synchronize()
    if st != 0:
        raise SystemExit("solve failed with status %d" % st)

    clocks = Clocks(local)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        bs.solve(itr, 0.0, True, 200.0)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1)
    ck = clocks.stop()
    info = bs.info.view(bs.P, 5).cpu().numpy()
    ms_t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        torch.distributed.all_reduce(ms_t, op=torch.distributed.ReduceOp.MAX)
        tot = torch.tensor([pts], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(tot)
        pts_all = int(tot.item())
    else:
        pts_all = pts
    ms_max = float(ms_t.item())
    value = pts_all * itr * args.steps / (ms_max * 1e-3)

    lib = bs.plan.lib  # (the 512-element-tile build for config 2, lib_for)
    group = int(lib.finom_solve1d_group(bs.plan.handle))
    NX, NY = bs.u.numel(), bs.v.numel()
    # algorithmic bytes: per iteration 40n + 48m unabsorbed,
    # 56n + 64m once the problem has absorbed (shift reads), weighted by the
    # iterations each problem spends in either state in this solve
    ns = np.array([x.size for x in wl["xs"]], dtype=np.float64)
    ms_ = np.array([y.size for y in wl["ys"]], dtype=np.float64)
    abs_its = bs.abs_its.view(bs.P, itr).cpu().numpy()
    first = np.where(info[:, 3] > 0, abs_its[:, 0], itr).astype(np.float64)
    alg_bytes_it = float(np.sum((40 * ns + 48 * ms_) * first
                                + (56 * ns + 64 * ms_) * (itr - first))) / itr
    peak, peak_src = peaks()
    launches = int(lib.finom_solve1d_launches(bs.plan.handle, itr, 1)) * args.steps
    prof = np.zeros(6)
    if group:
        # the group solve is ONE kernel (k_solve_group) for the whole loop: its
        # duration is the timed step (CUDA events on its stream, this rank)
        t_it = ms / args.steps / itr * 1e-3
        kernel = ("k_solve_group (whole %d-iteration solve in one launch, %d warp(s) per "
                  "problem)" % (itr, group))
        traffic_key = "k_solve_group"
    else:
        # per-kernel timing (events around each launch) of the tile-parallel loop
        hist_dev = torch.zeros(bs.P * itr, dtype=torch.float64, device="cuda")
        _lib.check(lib.finom_profile1d(bs.plan.handle, _lib.ptr(bs.u), _lib.ptr(bs.v),
                                       _lib.ptr(bs.phi), _lib.ptr(bs.psi), _lib.ptr(bs.a),
                                       _lib.ptr(bs.b), itr, 1, 200.0, _lib.ptr(hist_dev),
                                       _lib.ptr(prof), _lib.stream_ptr()), "finom_profile1d", lib)
        t_it = (prof[0] + prof[1]) * 1e-3
        kernel = "k_step<A>+k_resolve<A>+k_step<B>+k_resolve<B>"
        traffic_key = "k_step"
    achieved = alg_bytes_it / t_it / 1e9

    e2e = None
    if rank == 0 and cfg != 5:
        # public API with host buffers: plan + H2D + loop + cost + D2H every step
        X, Y, U, V = (fb.Mesh1D(wl["xs"][0]), fb.Mesh1D(wl["ys"][0]), fb.Measure(wl["us"][0]),
                      fb.Measure(wl["vs"][0]))
        scfg = fb.SolverConfig(epsilon=wl["eps"][0], itr_max=itr, tol=0.0, stabilize=True)
        fb.sinkhorn_1d(X, Y, U, V, scfg)
        t0 = time.perf_counter()
        n_e2e = max(1, min(args.steps, 3))
        for _ in range(n_e2e):
            sol = fb.sinkhorn_1d(X, Y, U, V, scfg)
        dt = (time.perf_counter() - t0) / n_e2e
        e2e = {"value": pts * itr / dt, "unit": UNIT,
               "h2d_bytes_per_step": 8 * 2 * (NX + NY), "d2h_bytes_per_step":
               8 * (2 * NX + 2 * NY + itr + 5 + 1), "cost": sol.cost,
               "path": "paper_2605_26659_b200.sinkhorn_1d (host numpy in/out, incl. W1 cost)"}
    elif cfg == 5 and os.environ.get("FINOM_E2E5", "1") != "0":
        # this rank's share of the batch through the public batched API: plan,
        # H2D of every problem's arrays, loop, W1 costs, D2H into per-problem Solutions
        ms = [fb.Mesh1D(z) for z in wl["xs"]]
        mt = [fb.Mesh1D(z) for z in wl["ys"]]
        mu = [fb.Measure(z) for z in wl["us"]]
        mv = [fb.Measure(z) for z in wl["vs"]]
        scfg = fb.SolverConfig(epsilon=1.0, itr_max=itr, tol=0.0, stabilize=True)
        fb.sinkhorn_1d_batched(ms, mt, mu, mv, scfg, epsilons=wl["eps"])  # (warm-up call)
        walls = []
        for _ in range(max(1, min(args.steps, 3))):
            torch.cuda.synchronize()
            barrier()
            t0 = time.perf_counter()
            sols = fb.sinkhorn_1d_batched(ms, mt, mu, mv, scfg, epsilons=wl["eps"])
            walls.append(time.perf_counter() - t0)
            del sols
        dt = statistics.median(walls)
        tdt = torch.tensor([dt], dtype=torch.float64, device="cuda")
        if world > 1:
            torch.distributed.all_reduce(tdt, op=torch.distributed.ReduceOp.MAX)
        e2e = {"value": pts_all * itr / float(tdt.item()), "unit": UNIT,
               "h2d_bytes_per_step": 8 * 2 * (NX + NY),
               "d2h_bytes_per_step": 8 * (2 * NX + 2 * NY) + 8 * len(wl["xs"]) * (2 * itr + 6),
               "path": "paper_2605_26659_b200.sinkhorn_1d_batched (host numpy in, per-problem "
                       "Solutions out, incl. W1 costs; a warm-up call, then the median of %d "
                       "calls, max over ranks; pipelined in stages)" % len(walls)}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        from oracle import oracle as O
        if cfg == 5:
            nprob = min(len(wl["xs"]), 4 * (os.cpu_count() or 1))
            probs = [(wl["xs"][k], wl["ys"][k], wl["us"][k], wl["vs"][k], wl["eps"][k])
                     for k in range(nprob)]
            v5, wall, cores = cpu_batch(probs, 200)
            cpu = {"value": v5, "unit": UNIT, "cores": cores, "kind": "port",
                   "sample": "config5 problems 0-%d, 200 iterations each, one C-port instance "
                             "per host thread (wall clock)" % (nprob - 1)}
        else:
            its = {1: 500, 2: 60}[cfg]
            r = O.sinkhorn_1d(wl["xs"][0], wl["ys"][0], wl["us"][0], wl["vs"][0], wl["eps"][0],
                              its, 0.0, True)
            cpu = {"value": pts * its / r["loop_s"], "unit": UNIT, "cores": 1, "kind": "port",
                   "sample": "%s full size, first %d of %d iterations (stabilize=True), loop "
                             "window" % (wl["name"], its, itr)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong" if cfg == 5 else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators, BASELINE.json shapes; see DESIGN.md)",
            "config": config_json(cfg, wl, world),
            "roofline": dict({"bound": "hbm", "achieved": achieved, "peak": peak,
                              "unit": "GB/s", "frac": achieved / peak,
                              "traffic": ncu_traffic(traffic_key, cfg),
                              "peak_source": peak_src, "kernel": kernel,
                              "algorithmic_bytes_per_iteration": alg_bytes_it,
                              "bytes_rule": "88 B/pt unabsorbed, 120 B/pt absorbed (SURVEY 8d)",
                              "ms_iteration": t_it * 1e3},
                             **({} if group else {
                                 "ms_half_a": prof[0], "ms_half_b": prof[1],
                                 "ms_resolve": prof[2], "ms_absorb": prof[3],
                                 "ms_iteration_ungraphed": prof[4]})),
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gpu_launches": launches,
            "clocks": ck,
            "iterations_run": int(info[0, 0]), "absorbs": int(info[0, 3]),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
