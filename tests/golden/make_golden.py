"""Generate the golden fixtures in tests/golden from the REFERENCE package.

Run in the build container (the reference is not available on the GPU box):
    python tests/golden/make_golden.py
It imports /root/reference/pkg/src/finom (read-only; numba cache redirected)
and records the reference's own outputs on seeded inputs.  The fixtures pin
both the C oracle (tests/test_oracle.py, CPU) and the CUDA path
(tests/test_parity_gpu.py).
"""

import json
import os
import sys
import time

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_finom_golden")
REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import numpy as np  # noqa: E402
from finom import kernel1d as rk  # noqa: E402
from finom import mesh as rm  # noqa: E402
from finom import solver as rs  # noqa: E402
from finom import kernel2d as r2  # noqa: E402

from paper_2605_26659_b200 import workloads as W  # noqa: E402


class CountingAdapter(rs._FastAdapter1D):
    """The reference adapter, recording the iterations at which it absorbs."""

    def __init__(self, *a):
        super().__init__(*a)
        self.calls = 0
        self.absorbs = []

    def iterate(self, *a):
        self.calls += 1
        return super().iterate(*a)

    def absorb(self, da, db):
        self.absorbs.append(self.calls)
        super().absorb(da, db)


def ref_solve(x, y, u, v, cfg):
    """sinkhorn_1d (solver.py:202-230) with absorb iterations recorded."""
    X, Y, Um, Vm = rm.Mesh1D(x), rm.Mesh1D(y), rm.Measure(u), rm.Measure(v)
    ad = CountingAdapter(X, Y, cfg.epsilon)
    phi, psi, it, conv, hist, loop = rs.run_driver(ad, Um.weights, Vm.weights, cfg)
    sol = rs.Solution(phi=phi, psi=psi, a=ad.a, b=ad.b, kernel=ad.kernel, iterations_run=it,
                      converged=conv, marginal_error_history=hist, wall_time=loop,
                      setup_time=0.0, cost=np.nan, config=cfg)
    sol.cost = rs.transport_cost_fast(sol)
    return dict(phi=phi, psi=psi, a=np.asarray(ad.a), b=np.asarray(ad.b),
                hist_it=np.array([h[0] for h in hist], dtype=np.int64),
                hist_err=np.array([h[1] for h in hist]), iterations=it, converged=conv,
                absorb_its=np.array(ad.absorbs, dtype=np.int64), cost=sol.cost, loop_s=loop)


def save(name, **arrs):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrs)
    print("wrote", path, os.path.getsize(path), "bytes")


def kernel_cases():
    """Matvec instances mirroring test_kernel1d.py:261-390 (random, rectangular, shifted)."""
    rng = np.random.default_rng(5)
    out = {}
    GX = np.array([1.0, 3.0, 7.0, 9.0, 12.0])
    GY = np.array([2.0, 5.0, 6.0, 9.0, 10.0])
    cases = [(GX, GY, 1.0, None, None)]
    for k in range(40):
        n = int(rng.integers(1, 40)) if k % 7 else 1
        m = int(rng.integers(1, 40)) if k % 5 else 1
        x = rm.random_sorted_nodes(n, seed=int(rng.integers(2**31))).nodes
        y = rm.random_sorted_nodes(m, seed=int(rng.integers(2**31))).nodes
        if k % 9 == 3:  # shared nodes: every node a tie
            y = x.copy()
        eps = float(rng.choice([0.01, 0.1, 1.0]))
        a = b = None
        if k % 3 == 1:
            a = rng.normal(0.0, 0.5, n) * eps * 10
            b = rng.normal(0.0, 0.5, m) * eps * 10
        cases.append((x, y, eps, a, b))
    # large-shift rebuild case (test_kernel1d.py:379-390)
    cases.append((GX, GY, 0.01, np.full(5, 8.0), np.full(5, -8.0)))
    for k, (x, y, eps, a, b) in enumerate(cases):
        op = rk.build_operator(rm.Mesh1D(x), rm.Mesh1D(y), eps)
        if a is not None:
            op = op.absorb(a, b)
        psi = rng.random(len(y))
        phi = rng.random(len(x))
        p, q = rk.apply_blocks(op, psi)
        out["c%d_x" % k] = x
        out["c%d_y" % k] = y
        out["c%d_eps" % k] = np.array(eps)
        out["c%d_a" % k] = np.asarray(op.absorption_left)
        out["c%d_b" % k] = np.asarray(op.absorption_right)
        out["c%d_psi" % k] = psi
        out["c%d_phi" % k] = phi
        out["c%d_Kpsi" % k] = op.apply(psi)
        out["c%d_KTphi" % k] = op.apply_transpose(phi)
        out["c%d_p" % k] = p
        out["c%d_q" % k] = q
    out["ncases"] = np.array(len(cases))
    save("kernel1d_cases.npz", **out)


def solver_cases():
    """Small scaling runs mirroring test_solver.py (plain, stabilized, zero mass, rect)."""
    out = {}
    cases = []
    def rp(n, m, seed):
        return (rm.random_sorted_nodes(n, seed).nodes, rm.random_sorted_nodes(m, seed + 1000).nodes,
                rm.random_measure(n, seed + 2000).weights, rm.random_measure(m, seed + 3000).weights)
    cases.append(rp(40, 55, 3) + (rs.SolverConfig(epsilon=0.05, itr_max=800, tol=0.0),))
    cases.append(rp(40, 55, 3) + (rs.SolverConfig(epsilon=0.05, itr_max=800, tol=0.0, stabilize=True,
                                                  absorb_threshold=1.5),))
    cases.append(rp(40, 55, 3) + (rs.SolverConfig(epsilon=0.05, itr_max=20000, tol=1e-11,
                                                  stabilize=True, absorb_threshold=1.5),))
    cases.append(rp(30, 30, 4) + (rs.SolverConfig(epsilon=0.01, itr_max=20, tol=0.0, check_every=7),))
    cases.append(rp(64, 64, 14) + (rs.SolverConfig(epsilon=0.1, itr_max=20000, tol=1e-10),))
    cases.append(rp(35, 70, 15) + (rs.SolverConfig(epsilon=0.02, itr_max=20000, tol=1e-10,
                                                   check_every=10),))
    # zero-mass stretch with absorption (test_solver.py:339-361)
    x = rm.random_sorted_nodes(80, seed=21).nodes
    y = rm.random_sorted_nodes(90, seed=22).nodes
    uw = np.abs(np.random.default_rng(5).normal(size=80))
    uw[30:45] = 0.0
    uw[:3] = 0.0
    cases.append((x, y, uw / uw.sum(), rm.random_measure(90, seed=23).weights,
                  rs.SolverConfig(epsilon=0.02, itr_max=4000, tol=1e-11, stabilize=True,
                                  absorb_threshold=1.2)))
    # eps = 1e-3 rescue (test_solver.py:321-337)
    x = rm.random_sorted_nodes(300, seed=7).nodes
    y = rm.random_sorted_nodes(300, seed=8).nodes
    gm = lambda z, c, w2: np.exp(-(z - c) ** 2 / w2) / np.exp(-(z - c) ** 2 / w2).sum()
    cases.append((x, y, gm(x, 0.3, 0.001), gm(y, 0.7, 0.001),
                  rs.SolverConfig(epsilon=0.001, itr_max=2000, tol=0.0, stabilize=True)))
    # self transport on shared nodes (every node a tie)
    x = rm.chebyshev_nodes(60).nodes
    u = rm.random_measure(60, seed=1).weights
    cases.append((x, x.copy(), u, u.copy(), rs.SolverConfig(epsilon=0.05, itr_max=3000, tol=1e-10)))
    # single points and degenerate sizes
    cases.append((np.array([0.2]), np.array([0.9]), np.array([1.0]), np.array([1.0]),
                  rs.SolverConfig(epsilon=0.7, itr_max=5, tol=0.0)))
    cases.append((np.array([0.1, 0.4]), np.array([0.25]), np.array([0.3, 0.7]), np.array([1.0]),
                  rs.SolverConfig(epsilon=0.5, itr_max=50, tol=0.0, stabilize=True,
                                  absorb_threshold=1.1)))
    for k, (x, y, u, v, cfg) in enumerate(cases):
        r = ref_solve(x, y, u, v, cfg)
        for key in ("x", "y", "u", "v"):
            out["s%d_%s" % (k, key)] = locals()[key]
        out["s%d_cfg" % k] = np.array([cfg.epsilon, cfg.itr_max, cfg.tol, float(cfg.stabilize),
                                       cfg.absorb_threshold, cfg.check_every])
        for key, val in r.items():
            out["s%d_%s" % (k, key)] = np.asarray(val)
    out["ncases"] = np.array(len(cases))
    save("solver_cases.npz", **out)


def failure_cases():
    """ZeroDenominator / NonFiniteIterate instances (test_solver.py:475-497)."""
    res = {}
    for name, (x, y, u, v, eps) in {
        "zero_denom": ([0.0, 0.5], [0.0, 50.0], [0.5, 0.5], [0.5, 0.5], 0.01),
        "nonfinite": ([0.0], [713.0], [1.0], [1.0], 1.0),
    }.items():
        try:
            rs.sinkhorn_1d(rm.Mesh1D(x), rm.Mesh1D(y), rm.Measure(u), rm.Measure(v),
                           rs.SolverConfig(epsilon=eps, itr_max=10, tol=0.0))
            res[name] = dict(raised=None)
        except Exception as e:  # noqa: BLE001
            res[name] = dict(raised=type(e).__name__, message=str(e), x=x, y=y, u=u, v=v, eps=eps)
    with open(os.path.join(HERE, "failure_cases.json"), "w") as f:
        json.dump(res, f, indent=1)


def config_runs():
    x, y, u, v, eps = W.config1()
    r = ref_solve(x, y, u, v, rs.SolverConfig(epsilon=eps, itr_max=500, tol=0.0, stabilize=True))
    save("config1.npz", **{k: np.asarray(val) for k, val in r.items()})
    x, y, u, v, eps = W.config2(n=1 << 16)
    r = ref_solve(x, y, u, v, rs.SolverConfig(epsilon=eps, itr_max=200, tol=0.0, stabilize=True))
    save("config2_n65536.npz", **{k: np.asarray(val) for k, val in r.items()})
    probs = {}
    for p in (0, 1, 2, 3):
        x, y, u, v, eps = W.config5_problem(p)
        r = ref_solve(x, y, u, v, rs.SolverConfig(epsilon=eps, itr_max=200, tol=0.0,
                                                  stabilize=True))
        for key, val in r.items():
            probs["p%d_%s" % (p, key)] = np.asarray(val)
        probs["p%d_eps" % p] = np.array(eps)
    save("config5_p0-3.npz", **probs)


def config2_full():
    """Full-size config 2 pins: scalars, history and a strided sample of the vectors."""
    x, y, u, v, eps = W.config2()
    t = time.time()
    r = ref_solve(x, y, u, v, rs.SolverConfig(epsilon=eps, itr_max=200, tol=0.0, stabilize=True))
    dt = time.time() - t
    stride = 4096
    save("config2_full_pins.npz", cost=np.array(r["cost"]), hist_err=r["hist_err"],
         absorb_its=r["absorb_its"], iterations=np.array(r["iterations"]), stride=np.array(stride),
         phi_s=r["phi"][::stride], psi_s=r["psi"][::stride], a_s=r["a"][::stride],
         b_s=r["b"][::stride], loop_s=np.array(r["loop_s"]), ref_wall_s=np.array(dt))


if __name__ == "__main__":
    which = sys.argv[1:] or ["kernel", "solver", "failure", "configs", "config2_full"]
    if "kernel" in which:
        kernel_cases()
    if "solver" in which:
        solver_cases()
    if "failure" in which:
        failure_cases()
    if "configs" in which:
        config_runs()
    if "config2_full" in which:
        config2_full()


def ref_solve_2d(x1, y1, x2, y2, U, V, cfg):
    """kernel2d.sinkhorn_2d (kernel2d.py:363-391) with absorb iterations recorded."""
    src = rm.Grid2D(rm.Mesh1D(x1), rm.Mesh1D(y1))
    tgt = rm.Grid2D(rm.Mesh1D(x2), rm.Mesh1D(y2))
    ad = r2._GridAdapter(src, tgt, cfg.epsilon)
    calls, absorbs = [0], []
    it0, ab0 = ad.iterate, ad.absorb
    def it(*a):
        calls[0] += 1
        return it0(*a)
    def ab(da, db):
        absorbs.append(calls[0])
        ab0(da, db)
    ad.iterate, ad.absorb = it, ab
    uw = np.ascontiguousarray(U.ravel(order="F"))
    vw = np.ascontiguousarray(V.ravel(order="F"))
    phi, psi, its, conv, hist, loop = rs.run_driver(ad, uw, vw, cfg)
    sol = rs.Solution(phi=phi, psi=psi, a=ad.a, b=ad.b, kernel=ad.kernel, iterations_run=its,
                      converged=conv, marginal_error_history=hist, wall_time=loop,
                      setup_time=0.0, cost=np.nan, config=cfg)
    sol.cost = r2.transport_cost_fast_2d(sol)
    return dict(phi=phi, psi=psi, a=np.asarray(ad.a), b=np.asarray(ad.b),
                hist_it=np.array([h[0] for h in hist], dtype=np.int64),
                hist_err=np.array([h[1] for h in hist]), iterations=its, converged=conv,
                absorb_its=np.array(absorbs, dtype=np.int64), cost=sol.cost, loop_s=loop)


def grid_cases():
    """2D runs (no kernel2d test exists in the reference: SURVEY.md 8(c))."""
    out = {}
    rng = np.random.default_rng(77)
    cases = []
    def rnd(n):
        return rm.random_sorted_nodes(n, int(rng.integers(2**31))).nodes
    for (n1, m1, n2, m2, eps, stab, thr, itr) in [
        (6, 5, 4, 7, 0.1, False, 200.0, 60), (6, 5, 4, 7, 0.05, True, 2.0, 80),
        (12, 9, 10, 11, 0.05, False, 200.0, 100), (12, 9, 10, 11, 0.02, True, 3.0, 150),
        (40, 33, 37, 41, 0.01, True, 20.0, 120)]:
        x1, y1, x2, y2 = rnd(n1), rnd(m1), rnd(n2), rnd(m2)
        U = rng.random((n1, m1)) + 0.05
        V = rng.random((n2, m2)) + 0.05
        U /= U.sum()
        V /= V.sum()
        cases.append((x1, y1, x2, y2, U, V, rs.SolverConfig(epsilon=eps, itr_max=itr, tol=0.0,
                                                            stabilize=stab, absorb_threshold=thr)))
    x1, y1, x2, y2, U, V, eps = W.config3(n=64)
    cases.append((x1, y1, x2, y2, U, V, rs.SolverConfig(epsilon=eps, itr_max=300, tol=0.0,
                                                        stabilize=True)))
    x1, y1, x2, y2, U, V, eps = W.config4(n=96)
    cases.append((x1, y1, x2, y2, U, V, rs.SolverConfig(epsilon=eps, itr_max=100, tol=0.0,
                                                        stabilize=True)))
    for k, (x1, y1, x2, y2, U, V, cfg) in enumerate(cases):
        r = ref_solve_2d(x1, y1, x2, y2, U, V, cfg)
        for key, val in dict(x1=x1, y1=y1, x2=x2, y2=y2, U=U, V=V).items():
            out["g%d_%s" % (k, key)] = val
        out["g%d_cfg" % k] = np.array([cfg.epsilon, cfg.itr_max, cfg.tol, float(cfg.stabilize),
                                       cfg.absorb_threshold, cfg.check_every])
        for key, val in r.items():
            out["g%d_%s" % (k, key)] = np.asarray(val)
        # operator applies on the final (absorbed) kernel
        op = r2.build_operator_2d(rm.Grid2D(rm.Mesh1D(x1), rm.Mesh1D(y1)),
                                  rm.Grid2D(rm.Mesh1D(x2), rm.Mesh1D(y2)), cfg.epsilon)
        vin = rng.random(len(x2) * len(y2))
        win = rng.random(len(x1) * len(y1))
        out["g%d_vin" % k] = vin
        out["g%d_win" % k] = win
        out["g%d_Kv" % k] = op.apply(vin)
        out["g%d_KTw" % k] = op.apply_transpose(win)
        A = r["a"].reshape((len(x1), len(y1)), order="F")
        B = r["b"].reshape((len(x2), len(y2)), order="F")
        if np.any(A != 0) or np.any(B != 0):
            opa = op.absorb(A, B)
            out["g%d_Kv_abs" % k] = opa.apply(vin)
            out["g%d_KTw_abs" % k] = opa.apply_transpose(win)
    out["ncases"] = np.array(len(cases))
    save("grid_cases.npz", **out)


def config3_full():
    x1, y1, x2, y2, U, V, eps = W.config3()
    t = time.time()
    r = ref_solve_2d(x1, y1, x2, y2, U, V, rs.SolverConfig(epsilon=eps, itr_max=300, tol=0.0,
                                                           stabilize=True))
    dt = time.time() - t
    stride = 997
    save("config3_full_pins.npz", cost=np.array(r["cost"]), hist_err=r["hist_err"],
         absorb_its=r["absorb_its"], iterations=np.array(r["iterations"]), stride=np.array(stride),
         phi_s=r["phi"][::stride], psi_s=r["psi"][::stride], a_s=r["a"][::stride],
         b_s=r["b"][::stride], loop_s=np.array(r["loop_s"]), ref_wall_s=np.array(dt))


if __name__ == "__main__" and len(sys.argv) > 1:
    if "grid" in sys.argv[1:]:
        grid_cases()
    if "config3_full" in sys.argv[1:]:
        config3_full()


def config4_full():
    """Full-size config-4 pins (the reference takes ~20 min on one core)."""
    x1, y1, x2, y2, U, V, eps = W.config4()
    t = time.time()
    r = ref_solve_2d(x1, y1, x2, y2, U, V, rs.SolverConfig(epsilon=eps, itr_max=100, tol=0.0,
                                                           stabilize=True))
    dt = time.time() - t
    stride = 65521
    save("config4_full_pins.npz", cost=np.array(r["cost"]), hist_err=r["hist_err"],
         absorb_its=r["absorb_its"], iterations=np.array(r["iterations"]), stride=np.array(stride),
         phi_s=r["phi"][::stride], psi_s=r["psi"][::stride], a_s=r["a"][::stride],
         b_s=r["b"][::stride], loop_s=np.array(r["loop_s"]), ref_wall_s=np.array(dt))


if __name__ == "__main__" and "config4_full" in sys.argv[1:]:
    config4_full()


def dense_cases():
    """SURVEY 8(f) f1 pins: the reference's dense_realization (1D, 2D; plain and
    shifted), plan_dense and marginal_error of solved states."""
    out = {}
    rng = np.random.default_rng(91)
    # 1D: a solved, absorbed problem (the Solution's kernel carries shifts)
    x, y, u, v, eps = W.config1(n=300)
    cfg = rs.SolverConfig(epsilon=eps, itr_max=40, tol=0.0, stabilize=True, absorb_threshold=6.0)
    X, Y, Um, Vm = rm.Mesh1D(x), rm.Mesh1D(y), rm.Measure(u), rm.Measure(v)
    sol = rs.sinkhorn_1d(X, Y, Um, Vm, cfg)
    out.update(s1_x=x, s1_y=y, s1_u=u, s1_v=v, s1_eps=np.array(eps),
               s1_phi=sol.phi, s1_psi=sol.psi, s1_a=np.asarray(sol.a), s1_b=np.asarray(sol.b),
               s1_dense=rk.dense_realization(sol.kernel), s1_plan=rs.plan_dense(sol),
               s1_marg=np.array(rs.marginal_error(sol, sol.kernel, Vm)))
    # 1D: random operator with shifts, arbitrary state
    n, m = 37, 53
    x2 = np.sort(rng.uniform(0, 1, n)); y2 = np.sort(rng.uniform(0, 1, m))
    a2 = rng.normal(0, 0.02, n); b2 = rng.normal(0, 0.02, m)
    op = rk.absorb(rk.build_operator(rm.Mesh1D(x2), rm.Mesh1D(y2), 0.05), a2, b2)
    out.update(r1_x=x2, r1_y=y2, r1_a=a2, r1_b=b2, r1_eps=np.array(0.05),
               r1_dense=rk.dense_realization(op))
    # 2D: grid operator, plain and absorbed
    x1, y1, xg, yg = (np.sort(rng.uniform(0, 1, k)) for k in (6, 5, 4, 7))
    src = rm.Grid2D(rm.Mesh1D(x1), rm.Mesh1D(y1))
    tgt = rm.Grid2D(rm.Mesh1D(xg), rm.Mesh1D(yg))
    op2 = r2.build_operator_2d(src, tgt, 0.1)
    A = rng.normal(0, 0.05, (6, 5)); B = rng.normal(0, 0.05, (4, 7))
    op2a = r2.absorb_2d(op2, A, B)
    out.update(g_x1=x1, g_y1=y1, g_x2=xg, g_y2=yg, g_A=A, g_B=B, g_eps=np.array(0.1),
               g_dense=r2.dense_realization_2d(op2), g_dense_abs=r2.dense_realization_2d(op2a))
    save("dense_cases.npz", **out)


if __name__ == "__main__" and "dense" in sys.argv[1:]:
    dense_cases()
