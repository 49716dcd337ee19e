"""Input types of the drop-in boundary: meshes, grids and measures.

Invariants follow the reference's ``finom.mesh`` (pkg/src/finom/mesh.py):
strictly ascending finite nodes (:37-57), nonnegative weights summing to
one within MASS_TOL (:28, :60-82), column-major grid vectorization
(:85-107) and 2D measures (:110-133).  Generators and file I/O are out of
scope for the hot path and live in the reference.
"""

from dataclasses import dataclass, field

import numpy as np

from .errors import (
    DuplicateNode,
    NonFiniteCoordinate,
    UnsortedInput,
    ValidationError,
)

MASS_TOL = 1e-12


def _freeze(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    a.flags.writeable = False
    return a


@dataclass(frozen=True)
class Mesh1D:
    """Strictly ascending finite coordinates; immutable (mesh.py:37-57)."""

    nodes: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "nodes", _freeze(self.nodes))
        nodes = self.nodes
        if nodes.ndim != 1 or nodes.size < 1:
            raise ValidationError("mesh needs a nonempty 1D coordinate list")
        if not np.all(np.isfinite(nodes)):
            raise NonFiniteCoordinate("mesh coordinates must be finite")
        diffs = np.diff(nodes)
        if np.any(diffs < 0):
            raise UnsortedInput("mesh coordinates must be ascending")
        if np.any(diffs == 0):
            raise DuplicateNode("mesh coordinates must be strictly ascending")

    def __len__(self):
        return self.nodes.size


def _check_weights(w, ndim, what):
    if w.ndim != ndim or w.size < 1:
        raise ValidationError("%s needs a nonempty %dD weight array" % (what, ndim))
    if not np.all(np.isfinite(w)):
        raise ValidationError("%s weights must be finite" % what)
    if np.any(w < 0):
        raise ValidationError("%s weights must be nonnegative" % what)
    if abs(w.sum() - 1.0) > MASS_TOL:
        raise ValidationError(
            "%s weights must sum to 1 within %g (got %.17g)" % (what, MASS_TOL, w.sum()))


@dataclass(frozen=True)
class Measure:
    """Nonnegative weights summing to 1 (within MASS_TOL); immutable."""

    weights: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "weights", _freeze(self.weights))
        _check_weights(self.weights, 1, "measure")

    def __len__(self):
        return self.weights.size


@dataclass(frozen=True)
class Grid2D:
    """Tensor-product grid; point (k, i) has linear index i*N + k."""

    x_nodes: Mesh1D
    y_nodes: Mesh1D
    ordering: str = field(default="column-major")

    def __post_init__(self):
        if self.ordering != "column-major":
            raise ValidationError("only column-major grid ordering is defined")

    @property
    def shape(self):
        return (len(self.x_nodes), len(self.y_nodes))

    def __len__(self):
        return len(self.x_nodes) * len(self.y_nodes)


@dataclass(frozen=True)
class Measure2D:
    """Nonnegative N-by-M weight array with total mass 1; immutable."""

    weights: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "weights", _freeze(self.weights))
        _check_weights(self.weights, 2, "grid measure")

    @property
    def shape(self):
        return self.weights.shape


@dataclass(frozen=True)
class Problem:
    """Source/target discretizations with their measures (mesh.py:136-151)."""

    source: object
    target: object
    u: object
    v: object

    @property
    def dim(self):
        return 2 if isinstance(self.source, Grid2D) else 1
