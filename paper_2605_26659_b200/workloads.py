"""Seeded synthetic inputs for the five BASELINE.json configurations.

Harness code (bench.py, tests), not the hot path.  The reference names no
dataset; the paper's experiments are synthetic too, so
these generators are the stand-in, with the ambiguities of BASELINE.json
resolved as documented in DESIGN.md section "Workloads".  numpy
default_rng (PCG64) like the reference's generators (mesh.py:7-9).
"""

import numpy as np

CONFIGS = {
    1: dict(name="1d_n1e4_eps1e-2", n=10_000, eps=1e-2, itr=500),
    2: dict(name="1d_n2^22_eps1e-3", n=1 << 22, eps=1e-3, itr=200),
    3: dict(name="2d_1024x1024_eps5e-3", n=1024, eps=5e-3, itr=300),
    4: dict(name="2d_8192x8192_eps1e-3", n=8192, eps=1e-3, itr=100),
    5: dict(name="batch8192_n16384_eps_logU", n=16_384, batch=8192, itr=200),
}


def cell_widths(x):
    """w_i = (x_{i+1} - x_{i-1})/2 with half-gaps at the two ends."""
    n = x.size
    if n == 1:
        return np.ones(1)
    w = np.empty(n)
    w[1:-1] = 0.5 * (x[2:] - x[:-2])
    w[0] = 0.5 * (x[1] - x[0])
    w[-1] = 0.5 * (x[-1] - x[-2])
    return w


def gap_mesh(rng, n, lo, hi):
    """n nodes from 0 to 1: cumulative sums of n-1 Uniform[lo, hi] gaps, rescaled."""
    if n == 1:
        return np.array([0.5])
    g = rng.uniform(lo, hi, n - 1)
    x = np.concatenate(([0.0], np.cumsum(g)))
    x /= x[-1]
    return x


def gauss(x, mu, sd):
    return np.exp(-0.5 * ((x - mu) / sd) ** 2) / (sd * np.sqrt(2.0 * np.pi))


def mixture(x, means, sds, weights, floor=0.0):
    d = np.zeros_like(x)
    for mu, sd, wt in zip(means, sds, weights):
        d += wt * gauss(x, mu, sd)
    w = d * cell_widths(x) + floor
    return w / w.sum()


def config1(n=10_000, seed=101):
    """1D, random-gap meshes U[0.2,1.8], 2-blob mixtures (0.3/0.05, 0.7/0.1) + 1e-12."""
    rng = np.random.default_rng(seed)
    x = gap_mesh(rng, n, 0.2, 1.8)
    y = gap_mesh(rng, n, 0.2, 1.8)
    u = mixture(x, (0.3, 0.7), (0.05, 0.1), (0.5, 0.5), 1e-12)
    v = mixture(y, (0.3, 0.7), (0.05, 0.1), (0.5, 0.5), 1e-12)
    return x, y, u, v, 1e-2


def config2(n=1 << 22, seed=202):
    """1D graded meshes x_i=(i/N)^2, y_j=1-(1-j/N)^2, seeded 3-component mixtures."""
    rng = np.random.default_rng(seed)
    i = np.arange(n, dtype=np.float64)
    x = (i / n) ** 2
    y = 1.0 - (1.0 - i / n) ** 2
    def dens(z):
        mu = rng.uniform(0.15, 0.85, 3)
        sd = rng.uniform(0.03, 0.12, 3)
        wt = rng.dirichlet(np.ones(3))
        return mixture(z, mu, sd, wt)
    u = dens(x)
    v = dens(y)
    return x, y, u, v, 1e-3


def config5_problem(p, n=16_384, seed=505):
    """Problem p of the batch: own gap meshes, 2-component mixtures, eps=10^U[-3,-1]."""
    rng = np.random.default_rng([seed, p])
    x = gap_mesh(rng, n, 0.2, 1.8)
    y = gap_mesh(rng, n, 0.2, 1.8)
    def dens(z):
        mu = rng.uniform(0.15, 0.85, 2)
        sd = rng.uniform(0.03, 0.12, 2)
        wt = rng.dirichlet(np.ones(2))
        return mixture(z, mu, sd, wt, 1e-12)
    u = dens(x)
    v = dens(y)
    eps = 10.0 ** rng.uniform(-3.0, -1.0)
    return x, y, u, v, eps


def config5(batch=8192, n=16_384, seed=505, problems=None):
    idx = range(batch) if problems is None else problems
    return [config5_problem(p, n, seed) for p in idx]


def tanh_nodes(n):
    """x_k = 0.5 + 0.5 tanh(3(2k/n - 1)) / tanh(3), k = 0..n-1 (clustered at the edges)."""
    k = np.arange(n, dtype=np.float64)
    return 0.5 + 0.5 * np.tanh(3.0 * (2.0 * k / n - 1.0)) / np.tanh(3.0)


def blobs(x, y, rng, nblob):
    """Seeded anisotropic, rotated Gaussian blobs on the grid x (rows) by y (cols)."""
    X, Y = np.meshgrid(x, y, indexing="ij")
    dens = np.zeros_like(X)
    wts = rng.dirichlet(np.ones(nblob))
    for b in range(nblob):
        cx, cy = rng.uniform(0.2, 0.8, 2)
        sx, sy = rng.uniform(0.05, 0.15, 2)
        th = rng.uniform(0.0, np.pi)
        c, s = np.cos(th), np.sin(th)
        dx, dy = X - cx, Y - cy
        u = (c * dx + s * dy) / sx
        v = (-s * dx + c * dy) / sy
        dens += wts[b] * np.exp(-0.5 * (u * u + v * v))
    w = dens * np.outer(cell_widths(x), cell_widths(y))
    return w / w.sum()


def config3(n=1024, seed=303):
    """2D, tanh-stretched tensor grid (source == target), 2 / 3 blobs, eps = 5e-3."""
    rng = np.random.default_rng(seed)
    x = tanh_nodes(n)
    y = tanh_nodes(n)
    U = blobs(x, y, rng, 2)
    V = blobs(x, y, rng, 3)
    return x, y, x.copy(), y.copy(), U, V, 5e-3


def config4(n=8192, seed=404):
    """2D, random-gap grid U[0.1,1.9] per axis (source == target), 8 blobs each, eps = 1e-3."""
    rng = np.random.default_rng(seed)
    x = gap_mesh(rng, n, 0.1, 1.9)
    y = gap_mesh(rng, n, 0.1, 1.9)
    U = blobs(x, y, rng, 8)
    V = blobs(x, y, rng, 8)
    return x, y, x.copy(), y.copy(), U, V, 1e-3
