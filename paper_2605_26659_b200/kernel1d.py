"""Device-backed 1D kernel operator (drop-in for finom.kernel1d).

The reference builds four table-backed block representations per
operator (kernel1d.py:194-255) and walks them on one core.  Here an
operator is only (x, y, eps, a, b): its apply / apply_transpose /
apply_blocks kernels (csrc/finom_1d.cu k_pre / k_apply) evaluate every ratio
and edge factor on the fly from exactly the same exponent expressions, so
an operator stores no tables and absorb only records the shifts.  (The
solve loop is different: it keeps per-tile tables for the current
absorption epoch and rebuilds them at every absorption, see DESIGN.md
section 4.)  Same public surface: ``dividing_index``,
``build_operator``, ``apply``, ``apply_transpose``, ``apply_blocks``,
``absorb``, ``dense_realization`` (kernel1d.py:55-338).
"""

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from .errors import DimensionMismatch, InvalidEpsilon, NonFiniteInput
from .mesh import Mesh1D

LOWER = "lower"
UPPER = "upper"


@dataclass(frozen=True)
class DividingIndex:
    """Per-row count of columns at or left of the staircase (kernel1d.py:39-52)."""

    zeta: np.ndarray
    n_cols: int

    def __post_init__(self):
        z = np.ascontiguousarray(np.asarray(self.zeta, dtype=np.int64))
        z.flags.writeable = False
        object.__setattr__(self, "zeta", z)

    def __len__(self):
        return self.zeta.size


def dividing_index(x, y):
    """zeta[i] = #{j : y_j <= x_i}; ties land in the lower block (kernel1d.py:55-62)."""
    z = np.searchsorted(y.nodes, x.nodes, side="right").astype(np.int64)
    return DividingIndex(z, len(y))


def _check_eps(epsilon):
    epsilon = float(epsilon)
    if not np.isfinite(epsilon) or epsilon <= 0:
        raise InvalidEpsilon("epsilon must be a positive finite real")
    return epsilon


def _check_vec(vec, length, what):
    vec = np.ascontiguousarray(np.asarray(vec, dtype=np.float64))
    if vec.ndim != 1 or vec.size != length:
        raise DimensionMismatch("%s must be a vector of length %d" % (what, length))
    if not np.all(np.isfinite(vec)):
        raise NonFiniteInput("%s must be finite" % what)
    return vec


class _PlanCache:
    """Lazily created device plan shared by operators on the same meshes."""

    def __init__(self, x, y, eps):
        self.x, self.y, self.eps = x, y, eps
        self._plan = None

    def get(self):
        if self._plan is None:
            self._plan = _lib.Plan1D([self.x.nodes], [self.y.nodes], self.eps)
        return self._plan


@dataclass(frozen=True)
class KernelOperator1D:
    """K'_ij = exp((-|x_i - y_j| + a_i + b_j) / eps), never materialized.

    ``absorption_left`` (a) and ``absorption_right`` (b) are the
    accumulated log-domain shifts (kernel1d.py:194-215).  Logically
    immutable: absorb() returns a new operator.
    """

    x_mesh: Mesh1D
    y_mesh: Mesh1D
    epsilon: float
    absorption_left: np.ndarray
    absorption_right: np.ndarray
    _plans: Optional[_PlanCache] = field(default=None, repr=False, compare=False)

    @property
    def shape(self):
        return (len(self.x_mesh), len(self.y_mesh))

    @property
    def absorbed(self):
        return bool(np.any(self.absorption_left != 0) or np.any(self.absorption_right != 0))

    def plan(self):
        return self._plans.get()

    def apply(self, psi):
        return apply(self, psi)

    def apply_transpose(self, phi):
        return apply_transpose(self, phi)

    def absorb(self, delta_a, delta_b):
        return absorb(self, delta_a, delta_b)

    def dense_realization(self):
        return dense_realization(self)


def build_operator(x, y, epsilon):
    """Operator for meshes x (rows) and y (columns), zero shifts (kernel1d.py:234-238)."""
    epsilon = _check_eps(epsilon)
    return KernelOperator1D(x, y, epsilon, np.zeros(len(x)), np.zeros(len(y)),
                            _PlanCache(x, y, epsilon))


def _run(op, vec, mode):
    import torch
    plan = op.plan()
    n, m = op.shape
    dev = torch.device("cuda")
    tin = torch.from_numpy(vec).to(dev)
    out = torch.empty(m if mode == 1 else n, dtype=torch.float64, device=dev)
    out2 = torch.empty(n, dtype=torch.float64, device=dev) if mode == 2 else None
    a = b = None
    if op.absorbed:
        a = torch.from_numpy(np.ascontiguousarray(op.absorption_left)).to(dev)
        b = torch.from_numpy(np.ascontiguousarray(op.absorption_right)).to(dev)
    lib = plan.lib
    _lib.check(lib.finom_apply1d(plan.handle, _lib.ptr(a), _lib.ptr(b), _lib.ptr(tin), mode,
                                 _lib.ptr(out), _lib.ptr(out2), _lib.stream_ptr()),
               "finom_apply1d", lib)
    if mode == 2:
        return out.cpu().numpy(), out2.cpu().numpy()
    return out.cpu().numpy()


def apply(op, psi):
    """K' psi (kernel1d.py:284-288)."""
    psi = _check_vec(psi, len(op.y_mesh), "psi")
    return _run(op, psi, 0)


def apply_transpose(op, phi):
    """K'^T phi (kernel1d.py:291-295)."""
    phi = _check_vec(phi, len(op.x_mesh), "phi")
    return _run(op, phi, 1)


def apply_blocks(op, psi):
    """(K'_lower psi, K'_upper psi) separately (kernel1d.py:298-310)."""
    psi = _check_vec(psi, len(op.y_mesh), "psi")
    return _run(op, psi, 2)


def absorb(op, delta_a, delta_b):
    """New operator with shifts a + delta_a, b + delta_b (kernel1d.py:313-325).

    Nothing is rebuilt: the kernels fold the accumulated shifts into each
    exponent, so successive absorbs equal one absorb of the summed deltas.
    """
    delta_a = _check_vec(delta_a, len(op.x_mesh), "delta_a")
    delta_b = _check_vec(delta_b, len(op.y_mesh), "delta_b")
    return KernelOperator1D(op.x_mesh, op.y_mesh, op.epsilon,
                            op.absorption_left + delta_a, op.absorption_right + delta_b,
                            op._plans)


def dense_realization(op):
    """Dense matrix, entry by entry on the device (tests / small-scale debugging;
    kernel1d.py:328-338: exp(((-|x_i - y_j| + a_i) + b_j) / eps), finom_dense1d)."""
    return _lib.dense1d(op.x_mesh.nodes, op.y_mesh.nodes, op.absorption_left,
                        op.absorption_right, op.epsilon)
