"""Command-line harness (SPEC.md cli: gen / solve / compare / bench) on the
B200 path.

    python -m paper_2605_26659_b200.cli gen --dim 1 --nodes chebyshev --n 100 --seed 5 -o p.json
    python -m paper_2605_26659_b200.cli solve --input p.json --eps 0.01 --iters 1000 [--tol 1e-9]
    python -m paper_2605_26659_b200.cli solve --dim 1 --nodes random --n 500 --eps 0.01 --iters 1000
    python -m paper_2605_26659_b200.cli compare --dim 1 --n 500 --eps 0.01 --iters 1000 --trials 3
    python -m paper_2605_26659_b200.cli bench --solver finom --sizes 1000,2000,4000,8000 --iters 1000
    python -m paper_2605_26659_b200.cli bench --time-to-error --n 2000 --eps-list 0.1,0.01

Reports are one JSON object per invocation (schema_version 1) on stdout or
--output; bench also writes CSV rows with --csv.  Timing: wall clock around
the iteration loop (Solution.wall_time - setup_time), mean over --trials.
finom runs the O(N) solver (sinkhorn_1d / sinkhorn_2d), dense the GPU
dense baseline (dense.dense_sinkhorn, cuBLAS matvecs).  Exit status 0 on
success, 2 on usage errors, 1 on solver / parse errors (diagnostic on
stderr).
"""

import argparse
import csv
import json
import sys

import numpy as np

from . import dense as D
from . import problem_io as io
from .errors import FinomError
from .solver import SolverConfig, marginal_error, plan_dense

REPORT_SCHEMA = 1


def _floats(s):
    return [float(t) for t in str(s).split(",") if t.strip()]


def _ints(s):
    return [int(float(t)) for t in str(s).split(",") if t.strip()]


def _problem(a):
    if getattr(a, "input", None):
        return io.load_problem(a.input)
    if a.n is None:
        raise FinomError("an --input file or a generator spec (--dim, --nodes, --n) is required")
    return io.generate(a.dim, a.nodes, a.n, a.m, a.seed)


def _config(a, tol=None):
    return SolverConfig(epsilon=a.eps, itr_max=a.iters, tol=a.tol if tol is None else tol,
                        stabilize=a.stabilize == "on", check_every=1,
                        plan_cap=getattr(a, "plan_cap", 10 ** 8))


def _solve(problem, cfg, solver):
    if solver == "dense":
        return D.dense_sinkhorn(problem, cfg)
    from .kernel2d import sinkhorn_2d
    from .solver import sinkhorn_1d
    run = sinkhorn_1d if problem.dim == 1 else sinkhorn_2d
    return run(problem.source, problem.target, problem.u, problem.v, cfg)


def _final_marginal(problem, sol):
    """||diag(psi) K^T phi - v||_1 of the final iterate (solver.py:233-237)."""
    if problem.dim == 1:
        return marginal_error(sol, sol.kernel, problem.v)
    v = problem.v.weights.ravel(order="F")
    return marginal_error(sol, sol.kernel, v)


def _problem_desc(problem, a):
    d = {"dim": problem.dim}
    if problem.dim == 1:
        d.update(n=len(problem.source), m=len(problem.target))
    else:
        d.update(source_shape=list(problem.source.shape), target_shape=list(problem.target.shape))
    if getattr(a, "input", None):
        d["input"] = a.input
    else:
        d.update(generator=a.nodes, seed=a.seed)
    return d


def _record(problem, sol, solver, cfg):
    return {"solver": solver, "iterations": sol.iterations_run, "converged": sol.converged,
            "cost": sol.cost, "final_marginal_error": _final_marginal(problem, sol),
            "last_history_error": sol.marginal_error_history[-1][1]
            if sol.marginal_error_history else None,
            "wall_time": sol.wall_time, "setup_time": sol.setup_time,
            "loop_time": sol.wall_time - sol.setup_time, "epsilon": cfg.epsilon}


def _emit(report, a):
    report = dict({"schema_version": REPORT_SCHEMA}, **report)
    text = json.dumps(report, indent=1, default=float)
    if getattr(a, "output", None):
        with open(a.output, "w") as fh:
            fh.write(text + "\n")
    else:
        print(text)


def cmd_gen(a):
    problem = io.generate(a.dim, a.nodes, a.n, a.m, a.seed)
    if a.csv:
        io.save_problem_csv(problem, a.output)
    else:
        io.save_problem(problem, a.output)
    return 0


def cmd_solve(a):
    problem = _problem(a)
    cfg = _config(a)
    sol = _solve(problem, cfg, a.solver)
    rep = {"command": "solve", "problem": _problem_desc(problem, a),
           "config": {"epsilon": cfg.epsilon, "itr_max": cfg.itr_max, "tol": cfg.tol,
                      "stabilize": cfg.stabilize},
           "result": _record(problem, sol, a.solver, cfg),
           "absorb_iterations": list(getattr(sol, "absorb_iterations", None) or [])}
    if a.plan_dump:
        np.save(a.plan_dump, plan_dense(sol))
        rep["plan_dump"] = a.plan_dump
    _emit(rep, a)
    return 0


def cmd_compare(a):
    """finom vs dense with identical config and inputs (SPEC cmd_compare):
    mean loop times over --trials, speed-up, ||dGamma||_F of the two plans
    (same iteration counts), max relative divergence of the scalings."""
    problem = _problem(a)
    cfg = _config(a)
    times = {"finom": [], "dense": []}
    sols = {}
    for _ in range(a.trials):
        for s in ("finom", "dense"):
            sols[s] = _solve(problem, cfg, s)
            times[s].append(sols[s].wall_time - sols[s].setup_time)
    fa, de = sols["finom"], sols["dense"]
    if fa.iterations_run != de.iterations_run:
        raise FinomError("the two solvers stopped at different iterations (%d vs %d)" % (
            fa.iterations_run, de.iterations_run))
    dgam = D.frobenius_diff(plan_dense(fa), plan_dense(de))
    rel = lambda x, y: float(np.max(np.abs(x - y)) / max(np.max(np.abs(y)), 1e-300))
    pot = lambda s, a_: cfg.epsilon * np.log(np.maximum(s, 1e-300)) + a_
    mf, md = float(np.mean(times["finom"])), float(np.mean(times["dense"]))
    _emit({"command": "compare", "problem": _problem_desc(problem, a),
           "config": {"epsilon": cfg.epsilon, "itr_max": cfg.itr_max, "tol": cfg.tol,
                      "stabilize": cfg.stabilize, "trials": a.trials},
           "finom": _record(problem, fa, "finom", cfg), "dense": _record(problem, de, "dense", cfg),
           "mean_time": {"finom": mf, "dense": md}, "speedup": md / mf,
           "frobenius_plan_diff": dgam,
           "max_rel_divergence": {"phi": rel(fa.phi, de.phi), "psi": rel(fa.psi, de.psi)},
           "max_potential_divergence": float(np.max(np.abs(pot(fa.phi, fa.a) -
                                                           pot(de.phi, de.a))))}, a)
    return 0


def _fit(sizes, times):
    """Least-squares slope of log(time) against log(size), with the residual."""
    if len(sizes) < 4:
        raise FinomError("the scaling fit needs at least 4 sizes (got %d)" % len(sizes))
    X = np.log(np.asarray(sizes, dtype=float))
    Y = np.log(np.asarray(times, dtype=float))
    A = np.vstack([X, np.ones_like(X)]).T
    coef, res, _, _ = np.linalg.lstsq(A, Y, rcond=None)
    resid = float(res[0]) if res.size else float(np.sum((A @ coef - Y) ** 2))
    return {"exponent": float(coef[0]), "intercept": float(coef[1]), "residual": resid}


def cmd_bench(a):
    if a.time_to_error:
        return _time_to_error(a)
    solvers = ["finom", "dense"] if a.solver == "both" else [a.solver]
    sizes = _ints(a.sizes)
    if len(sizes) < 4:
        raise FinomError("the scaling fit needs at least 4 sizes (got %d)" % len(sizes))
    rows, fits = [], {}
    for s in solvers:
        means = []
        for n in sizes:
            m = n if a.dim == 1 else (a.m or n)
            problem = io.generate(a.dim, a.nodes, n, m, a.seed)
            cfg = _config(a)
            _solve(problem, cfg, s)  # warm-up (plans, graphs)
            ts = []
            for _ in range(a.trials):
                sol = _solve(problem, cfg, s)
                ts.append(sol.wall_time - sol.setup_time)
            mt = float(np.mean(ts))
            pts = n if a.dim == 1 else n * m
            means.append(mt)
            rows.append({"solver": s, "size": pts, "mean_time": mt, "iterations": sol.iterations_run,
                         "cost": sol.cost})
        fits[s] = _fit([r["size"] for r in rows if r["solver"] == s], means)
    if a.csv:
        with open(a.csv, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["solver", "size", "mean_time"])
            w.writerows([r["solver"], r["size"], repr(r["mean_time"])] for r in rows)
    rep = {"command": "bench", "dim": a.dim, "nodes": a.nodes, "iters": a.iters,
           "trials": a.trials, "rows": rows, "fits": fits}
    if len(solvers) == 2:
        rep["speedup"] = [d["mean_time"] / f["mean_time"]
                          for f, d in zip(rows[:len(sizes)], rows[len(sizes):])]
    _emit(rep, a)
    return 0


def _time_to_error(a):
    """Figures' right panels: the loop time at which the marginal error first
    drops to each threshold, per epsilon (the device loop stops at tol)."""
    problem = _problem(a)
    rows = []
    for eps in _floats(a.eps_list):
        for thr in sorted(_floats(a.thresholds), reverse=True):
            cfg = SolverConfig(epsilon=eps, itr_max=a.iters, tol=thr, stabilize=a.stabilize == "on")
            _solve(problem, cfg, a.solver if a.solver != "both" else "finom")
            sol = _solve(problem, cfg, a.solver if a.solver != "both" else "finom")
            rows.append({"epsilon": eps, "threshold": thr, "reached": sol.converged,
                         "iterations": sol.iterations_run,
                         "loop_time": sol.wall_time - sol.setup_time})
    _emit({"command": "bench", "mode": "time_to_error", "problem": _problem_desc(problem, a),
           "rows": rows}, a)
    return 0


def parser():
    p = argparse.ArgumentParser(prog="python -m paper_2605_26659_b200.cli",
                                description="FINOM harness on the B200 path (SPEC.md cli)")
    sub = p.add_subparsers(dest="cmd", required=True)

    def gen_args(q, n_required=False):
        q.add_argument("--dim", type=int, choices=[1, 2], default=1)
        q.add_argument("--nodes", choices=["chebyshev", "random"], default="random")
        q.add_argument("--n", type=int, required=n_required)
        q.add_argument("--m", type=int)
        q.add_argument("--seed", type=int, default=0)

    def cfg_args(q):
        q.add_argument("--eps", type=float, default=0.01)
        q.add_argument("--iters", type=int, default=1000)
        q.add_argument("--tol", type=float, default=0.0)
        q.add_argument("--stabilize", choices=["on", "off"], default="on")
        q.add_argument("--output", "-o")

    g = sub.add_parser("gen", help="write a problem file (JSON schema v1, or CSV with --csv)")
    gen_args(g, n_required=True)
    g.add_argument("--output", "-o", required=True)
    g.add_argument("--csv", action="store_true")
    s = sub.add_parser("solve", help="solve one problem, report cost / iterations / residual")
    gen_args(s)
    cfg_args(s)
    s.add_argument("--input")
    s.add_argument("--solver", choices=["finom", "dense"], default="finom")
    s.add_argument("--plan-dump", dest="plan_dump")
    s.add_argument("--plan-cap", dest="plan_cap", type=int, default=10 ** 8)
    c = sub.add_parser("compare", help="finom vs dense: times, speed-up, ||dGamma||_F")
    gen_args(c)
    cfg_args(c)
    c.add_argument("--input")
    c.add_argument("--trials", type=int, default=3)
    c.add_argument("--plan-cap", dest="plan_cap", type=int, default=10 ** 8)
    b = sub.add_parser("bench", help="size sweep with log-log fit, or time-to-error")
    gen_args(b)
    cfg_args(b)
    b.add_argument("--input")
    b.add_argument("--solver", choices=["finom", "dense", "both"], default="finom")
    b.add_argument("--sizes", default="1000,2000,4000,8000")
    b.add_argument("--trials", type=int, default=3)
    b.add_argument("--csv")
    b.add_argument("--time-to-error", dest="time_to_error", action="store_true")
    b.add_argument("--thresholds", default="1e-2,1e-4,1e-6")
    b.add_argument("--eps-list", dest="eps_list", default="0.1,0.01,0.001")
    return p


def main(argv=None):
    a = parser().parse_args(argv)
    try:
        return {"gen": cmd_gen, "solve": cmd_solve, "compare": cmd_compare,
                "bench": cmd_bench}[a.cmd](a)
    except (FinomError, OSError) as exc:
        print("error: %s" % exc, file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
