"""Problem files (JSON schema v1) and the node / measure generators of the
experiment harness (SPEC.md cli: gen; mesh.py:164-322 of the reference).

Schema v1 (mesh.py:291-322): ``{"schema_version": 1, "dim": 1 | 2,
"x1", "x2" (+ "y1", "y2" for dim 2): node lists, "u", "v": weights (flat
for dim 1, nested rows n x m for dim 2)}``.  Floats are written in
shortest round-trip form (json), so a save / load round trip reproduces
every value; weights that do not sum to 1 within MASS_TOL are
normalized by their exact sum on load (mesh.py:226-256).  Generators use
numpy's PCG64 default_rng, reproducible byte for byte from the seed.
"""

import csv
import json

import numpy as np

from .errors import ConfigError, DimensionMismatch, ParseError, ValidationError
from .mesh import MASS_TOL, Grid2D, Measure, Measure2D, Mesh1D, Problem

SCHEMA_VERSION = 1


# ---- generators (mesh.py:164-223) -----------------------------------------
def _count(n, what="node count"):
    n = int(n)
    if n < 1:
        raise ConfigError("%s must be >= 1" % what)
    return n


def chebyshev_nodes(n):
    """The n Chebyshev points 1/2 + cos((2k-1) pi / (2n)) / 2, k = 1..n, ascending."""
    n = _count(n)
    k = np.arange(n, 0, -1)  # descending k: ascending nodes
    return Mesh1D(0.5 + 0.5 * np.cos((2 * k - 1) * np.pi / (2 * n)))


def random_sorted_nodes(n, seed):
    """n sorted Uniform[0, 1] draws (exact ties redrawn until strictly ascending)."""
    n = _count(n)
    rng = np.random.default_rng(seed)
    z = np.sort(rng.uniform(0.0, 1.0, n))
    while n > 1:
        tie = np.flatnonzero(np.diff(z) == 0)
        if not tie.size:
            break
        z[tie] = rng.uniform(0.0, 1.0, tie.size)
        z = np.sort(z)
    return Mesh1D(z)


def random_measure(n, seed):
    """n Uniform[0, 1] weights normalized to unit mass."""
    n = _count(n, "weight count")
    w = np.random.default_rng(seed).uniform(0.0, 1.0, n)
    s = w.sum()
    if s <= 0:
        raise ValidationError("weights sum to zero; cannot normalize")
    return Measure(w / s)


def random_measure_2d(n, m, seed):
    """n x m Uniform[0, 1] grid weights normalized to unit mass."""
    n, m = int(n), int(m)
    if n < 1 or m < 1:
        raise ConfigError("grid measure shape must be at least 1x1")
    w = np.random.default_rng(seed).uniform(0.0, 1.0, (n, m))
    s = w.sum()
    if s <= 0:
        raise ValidationError("weights sum to zero; cannot normalize")
    return Measure2D(w / s)


def generate(dim, nodes, n, m=None, seed=0):
    """A problem instance of the paper's experiment setups (SPEC cmd_gen):
    dim 1 -> two meshes of n nodes; dim 2 -> two n x m grids.  nodes is
    "chebyshev" or "random"; seeds of the four node lists / two measures are
    derived from seed."""
    n = _count(n)
    m = _count(m if m is not None else n)
    if nodes not in ("chebyshev", "random"):
        raise ConfigError("nodes must be chebyshev or random")
    mk = (lambda k, s: chebyshev_nodes(k)) if nodes == "chebyshev" else random_sorted_nodes
    if dim == 1:
        return Problem(mk(n, [seed, 1]), mk(n, [seed, 2]), random_measure(n, [seed, 3]),
                       random_measure(n, [seed, 4]))
    if dim == 2:
        src = Grid2D(mk(n, [seed, 1]), mk(m, [seed, 2]))
        tgt = Grid2D(mk(n, [seed, 3]), mk(m, [seed, 4]))
        return Problem(src, tgt, random_measure_2d(n, m, [seed, 5]),
                       random_measure_2d(n, m, [seed, 6]))
    raise ConfigError("dim must be 1 or 2")


# ---- JSON v1 (mesh.py:258-322) -------------------------------------------
def _weights(raw, shape, what):
    w = np.asarray(raw, dtype=np.float64)
    if w.ndim != len(shape):
        raise ParseError("%s must be a %s" % (
            what, "flat list of weights" if len(shape) == 1 else "nested list of weight rows"))
    if w.shape != tuple(shape):
        raise DimensionMismatch("%s has shape %s for %s" % (what, w.shape, tuple(shape)))
    s = w.sum()
    if not np.isfinite(s) or s <= 0:
        raise ValidationError("%s has non-positive or non-finite mass" % what)
    if abs(s - 1.0) > MASS_TOL:  # kept bit for bit when already normalized
        w = w / s
    return Measure(w) if w.ndim == 1 else Measure2D(w)


def load_problem(path):
    """Read a schema-v1 problem file (ParseError on malformed input)."""
    try:
        with open(path) as fh:
            doc = json.load(fh)
    except (OSError, json.JSONDecodeError) as exc:
        raise ParseError("cannot read problem file %s: %s" % (path, exc)) from exc
    if not isinstance(doc, dict):
        raise ParseError("problem file must hold a JSON object")
    dim = doc.get("dim")
    try:
        if dim == 1:
            src, tgt = Mesh1D(doc["x1"]), Mesh1D(doc["x2"])
            return Problem(src, tgt, _weights(doc["u"], (len(src),), "u"),
                           _weights(doc["v"], (len(tgt),), "v"))
        if dim == 2:
            src = Grid2D(Mesh1D(doc["x1"]), Mesh1D(doc["y1"]))
            tgt = Grid2D(Mesh1D(doc["x2"]), Mesh1D(doc["y2"]))
            return Problem(src, tgt, _weights(doc["u"], src.shape, "u"),
                           _weights(doc["v"], tgt.shape, "v"))
    except KeyError as exc:
        raise ParseError("problem file is missing field %s" % exc) from exc
    raise ParseError("problem file must declare dim 1 or 2")


def problem_doc(problem):
    """The schema-v1 document of a problem."""
    doc = {"schema_version": SCHEMA_VERSION, "dim": problem.dim}
    if problem.dim == 1:
        doc.update(x1=problem.source.nodes.tolist(), x2=problem.target.nodes.tolist())
    else:
        doc.update(x1=problem.source.x_nodes.nodes.tolist(),
                   y1=problem.source.y_nodes.nodes.tolist(),
                   x2=problem.target.x_nodes.nodes.tolist(),
                   y2=problem.target.y_nodes.nodes.tolist())
    doc.update(u=problem.u.weights.tolist(), v=problem.v.weights.tolist())
    return doc


def save_problem(problem, path):
    """Write a problem as schema-v1 JSON (exact round trip through load_problem)."""
    with open(path, "w") as fh:
        json.dump(problem_doc(problem), fh)
        fh.write("\n")


def save_problem_csv(problem, path):
    """One-way CSV export: 1D rows (role, index, node, weight), 2D rows
    (role, i, j, x, y, weight) over every grid point (mesh.py:325-353)."""
    with open(path, "w", newline="") as fh:
        out = csv.writer(fh)
        sides = (("source", problem.source, problem.u), ("target", problem.target, problem.v))
        if problem.dim == 1:
            out.writerow(["role", "index", "node", "weight"])
            for role, mesh, meas in sides:
                out.writerows([role, i, repr(float(z)), repr(float(w))]
                              for i, (z, w) in enumerate(zip(mesh.nodes, meas.weights)))
        else:
            out.writerow(["role", "i", "j", "x", "y", "weight"])
            for role, grid, meas in sides:
                xs, ys, w = grid.x_nodes.nodes, grid.y_nodes.nodes, meas.weights
                out.writerows([role, i, j, repr(float(xs[i])), repr(float(ys[j])),
                               repr(float(w[i, j]))]
                              for i in range(xs.size) for j in range(ys.size))
