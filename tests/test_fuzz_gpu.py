"""Seeded random problems against the C oracle: ragged sizes (1 .. ~900 points,
n != m), x / y ties, repeated near-coincident nodes, zero-mass stretches, eps
over two decades, absorption thresholds from "every few iterations" to
"never", stabilize on / off -- the 1D loop (single problem and batched, i.e.
the tile-parallel graph loop and the group solve) and small rectangular /
square 2D grids (general and square sweeps).  A failing run (ZERO_DENOM /
NONFINITE) must fail the same way at the same iteration."""

import numpy as np
import pytest

import paper_2605_26659_b200 as fb
from paper_2605_26659_b200 import errors as E

from conftest import rel_inf

pytestmark = pytest.mark.gpu
TOL = 1e-9


def _oracle():
    from oracle import oracle as O
    return O


def _mesh(rng, n, other=None):
    z = np.sort(rng.uniform(0.0, 1.0, n))
    if n > 3 and rng.random() < 0.5:  # clusters of nearly coincident nodes
        k = int(rng.integers(0, n - 2))
        z[k + 1] = z[k] + 1e-13 * (1 + rng.random())
        z = np.sort(z)
    if other is not None and n > 2 and rng.random() < 0.7:  # ties with the other mesh
        take = rng.choice(other, size=min(len(other), max(1, n // 4)), replace=False)
        z[rng.choice(n, size=len(take), replace=False)] = take
        z = np.sort(z)
    z = np.unique(z)  # (meshes are strictly increasing)
    return z


def _mass(rng, n):
    w = rng.random(n) + 1e-3
    if n > 4 and rng.random() < 0.6:  # zero-mass stretches (np.interp fill on absorption)
        for _ in range(int(rng.integers(1, 4))):
            lo = int(rng.integers(0, n - 1))
            w[lo:lo + int(rng.integers(1, max(2, n // 5)))] = 0.0
        if w.sum() == 0.0:
            w[int(rng.integers(0, n))] = 1.0
    return w / w.sum()


def _problem(rng, nmax=900):
    n, m = int(rng.integers(1, nmax)), int(rng.integers(1, nmax))
    x = _mesh(rng, n)
    y = _mesh(rng, m, x)
    u, v = _mass(rng, x.size), _mass(rng, y.size)
    eps = float(10 ** rng.uniform(-2.3, -0.3))
    return x, y, u, v, eps


def _check(sol, r, what):
    assert sol.iterations_run == r["iterations"], what
    assert list(sol.absorb_iterations) == list(r["absorb_its"]), what
    assert rel_inf(sol.phi, r["phi"]) < TOL and rel_inf(sol.psi, r["psi"]) < TOL, what
    sa, sb = np.asarray(sol.a).ravel(order="F"), np.asarray(sol.b).ravel(order="F")
    if r["n_absorb"]:
        assert rel_inf(sa, r["a"]) < TOL and rel_inf(sb, r["b"]) < TOL, what
    else:
        assert not sa.any() and not sb.any(), what
    assert abs(sol.cost - r["cost"]) <= TOL * max(abs(r["cost"]), 1e-300), what
    errs = np.array([e for _, e in sol.marginal_error_history])
    assert errs.size == r["hist"].size, what
    assert np.all(np.abs(errs - r["hist"]) <= TOL * np.abs(r["hist"]) + 1e-12), what


EXC = {1: E.ZeroDenominator, 2: E.NonFiniteIterate}


@pytest.mark.parametrize("seed", range(24))
def test_fuzz_1d_vs_oracle(seed):
    O = _oracle()
    rng = np.random.default_rng([7001, seed])
    x, y, u, v, eps = _problem(rng)
    stab = bool(rng.random() < 0.8)
    thr = float(rng.choice([2.0, 5.0, 20.0, 200.0]))
    itr = int(rng.integers(5, 80))
    if not stab and rng.random() < 0.5:  # (underflowing kernels: the failure rules)
        eps = float(10 ** rng.uniform(-4.5, -3.3))
    r = O.sinkhorn_1d(x, y, u, v, eps, itr, 0.0, stab, thr)
    cfg = fb.SolverConfig(epsilon=eps, itr_max=itr, tol=0.0, stabilize=stab, absorb_threshold=thr)
    args = (fb.Mesh1D(x), fb.Mesh1D(y), fb.Measure(u), fb.Measure(v), cfg)
    what = "seed %d n %d m %d eps %.3g thr %g stab %s" % (seed, x.size, y.size, eps, thr, stab)
    if r["status"] in EXC:
        with pytest.raises(EXC[r["status"]]):
            fb.sinkhorn_1d(*args)
        return
    _check(fb.sinkhorn_1d(*args), r, what)


@pytest.mark.parametrize("seed", range(4))
def test_fuzz_batched_vs_oracle(seed):
    O = _oracle()
    rng = np.random.default_rng([7002, seed])
    probs = [_problem(rng, nmax=1500) for _ in range(int(rng.integers(3, 40)))]
    thr = float(rng.choice([3.0, 10.0, 200.0]))
    itr = int(rng.integers(10, 70))
    refs = [O.sinkhorn_1d(x, y, u, v, e, itr, 0.0, True, thr) for x, y, u, v, e in probs]
    if any(r["status"] for r in refs):  # (failures are test_fuzz_1d's and the diagnostics tests')
        probs = [p for p, r in zip(probs, refs) if not r["status"]]
        refs = [r for r in refs if not r["status"]]
    cfg = fb.SolverConfig(epsilon=1.0, itr_max=itr, tol=0.0, stabilize=True, absorb_threshold=thr)
    sols = fb.sinkhorn_1d_batched([fb.Mesh1D(p[0]) for p in probs], [fb.Mesh1D(p[1]) for p in probs],
                                  [fb.Measure(p[2]) for p in probs], [fb.Measure(p[3]) for p in probs],
                                  cfg, epsilons=[p[4] for p in probs])
    for k, (sol, r) in enumerate(zip(sols, refs)):
        _check(sol, r, "seed %d problem %d n %d m %d" % (seed, k, probs[k][0].size, probs[k][1].size))


@pytest.mark.parametrize("seed", range(8))
def test_fuzz_2d_vs_oracle(seed):
    O = _oracle()
    rng = np.random.default_rng([7003, seed])
    square = seed % 2 == 0  # source grid == target grid: the square sweeps
    n1, m1 = int(rng.integers(1, 300)), int(rng.integers(1, 40))
    x1, y1 = _mesh(rng, n1), _mesh(rng, m1)
    if square:
        x2, y2 = x1, y1
    else:
        x2, y2 = _mesh(rng, int(rng.integers(1, 300)), x1), _mesh(rng, int(rng.integers(1, 40)), y1)
    U = _mass(rng, x1.size * y1.size).reshape(x1.size, y1.size)
    V = _mass(rng, x2.size * y2.size).reshape(x2.size, y2.size)
    eps = float(10 ** rng.uniform(-2.0, -0.5))
    thr = float(rng.choice([1.5, 4.0, 20.0]))
    itr = int(rng.integers(5, 40))
    r = O.sinkhorn_2d(x1, y1, x2, y2, U, V, eps, itr, 0.0, True, thr)
    cfg = fb.SolverConfig(epsilon=eps, itr_max=itr, tol=0.0, stabilize=True, absorb_threshold=thr)
    g = lambda x, y: fb.Grid2D(fb.Mesh1D(x), fb.Mesh1D(y))
    args = (g(x1, y1), g(x2, y2), fb.Measure2D(U), fb.Measure2D(V), cfg)
    what = "seed %d grid %dx%d -> %dx%d eps %.3g thr %g" % (seed, x1.size, y1.size, x2.size,
                                                           y2.size, eps, thr)
    if r["status"] in EXC:
        with pytest.raises(EXC[r["status"]]):
            fb.sinkhorn_2d(*args)
        return
    _check(fb.sinkhorn_2d(*args), r, what)
