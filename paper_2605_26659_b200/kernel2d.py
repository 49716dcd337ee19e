"""Separable 2D kernel and the grid solver on the B200 (drop-in for finom.kernel2d).

K = Ky (x) Kx on tensor-product grids, vectors flattened column-major
(x fastest, mesh.py:85-107, kernel2d.py:1-19).  The device path
(csrc/finom_2d.inc) runs every column sweep and row sweep as a batch of
1D line scans sharing one mesh, with a tiled transpose in between, and
switches to the dynamic-shift exponent form after the first absorption
exactly as _GridAdapter does (kernel2d.py:293-360).
"""

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib, kernel1d
from .errors import DimensionMismatch, NonFiniteInput
from .solver import Solution, history_from, raise_status


def _check_flat(vec, length, what):
    vec = np.ascontiguousarray(np.asarray(vec, dtype=np.float64))
    if vec.ndim != 1 or vec.size != length:
        raise DimensionMismatch("%s must be a vector of length %d" % (what, length))
    if not np.all(np.isfinite(vec)):
        raise NonFiniteInput("%s must be finite" % what)
    return vec


def _check_grid(arr, shape, what):
    arr = np.asfortranarray(np.asarray(arr, dtype=np.float64))
    if arr.shape != shape:
        raise DimensionMismatch("%s must have grid shape %r" % (what, shape))
    if not np.all(np.isfinite(arr)):
        raise NonFiniteInput("%s must be finite" % what)
    return arr


@dataclass(frozen=True)
class KernelOperator2D:
    """Kernel of a grid pair: two shift-free 1D factors plus shift grids (kernel2d.py:34-96)."""

    kx: kernel1d.KernelOperator1D
    ky: kernel1d.KernelOperator1D
    epsilon: float
    absorption_left: np.ndarray
    absorption_right: np.ndarray

    @property
    def source_shape(self):
        return (len(self.kx.x_mesh), len(self.ky.x_mesh))

    @property
    def target_shape(self):
        return (len(self.kx.y_mesh), len(self.ky.y_mesh))

    @property
    def shape(self):
        n1, m1 = self.source_shape
        n2, m2 = self.target_shape
        return (n1 * m1, n2 * m2)

    @property
    def absorbed(self):
        return bool(np.any(self.absorption_left != 0) or np.any(self.absorption_right != 0))

    def _meshes(self):
        return (self.kx.x_mesh.nodes, self.ky.x_mesh.nodes, self.kx.y_mesh.nodes,
                self.ky.y_mesh.nodes)

    def _apply(self, vec, transpose):
        x1, y1, x2, y2 = self._meshes()
        n1, m1 = self.source_shape
        n2, m2 = self.target_shape
        out = np.empty(n2 * m2 if transpose else n1 * m1)
        A = B = None
        if self.absorbed:
            A = np.ascontiguousarray(self.absorption_left.ravel(order="F"))
            B = np.ascontiguousarray(self.absorption_right.ravel(order="F"))
        lib = _lib.load()
        _lib.check(lib.finom_apply2d_host(n1, _lib.ptr(x1), m1, _lib.ptr(y1), n2, _lib.ptr(x2),
                                          m2, _lib.ptr(y2), self.epsilon, _lib.ptr(A),
                                          _lib.ptr(B), _lib.ptr(vec), int(transpose),
                                          _lib.ptr(out)), "finom_apply2d_host")
        return out

    def apply(self, psi):
        """K psi on the flat column-major vector, shifts included (kernel2d.py:70-79)."""
        return self._apply(_check_flat(psi, self.shape[1], "psi"), False)

    def apply_transpose(self, phi):
        """K^T phi (kernel2d.py:81-90)."""
        return self._apply(_check_flat(phi, self.shape[0], "phi"), True)

    def absorb(self, delta_a, delta_b):
        return absorb_2d(self, delta_a, delta_b)

    def dense_realization(self):
        return dense_realization_2d(self)


def build_operator_2d(source, target, epsilon):
    """Operator for source/target grids; one 1D factor per axis (kernel2d.py:99-109)."""
    epsilon = kernel1d._check_eps(epsilon)
    kx = kernel1d.build_operator(source.x_nodes, target.x_nodes, epsilon)
    ky = kernel1d.build_operator(source.y_nodes, target.y_nodes, epsilon)
    return KernelOperator2D(kx, ky, epsilon, np.zeros(source.shape), np.zeros(target.shape))


def absorb_2d(op, delta_a, delta_b):
    """Shift grids advanced by the deltas (kernel2d.py:261-275)."""
    delta_a = _check_grid(delta_a, op.source_shape, "delta_a")
    delta_b = _check_grid(delta_b, op.target_shape, "delta_b")
    return KernelOperator2D(op.kx, op.ky, op.epsilon, op.absorption_left + delta_a,
                            op.absorption_right + delta_b)


def dense_realization_2d(op):
    """Vectorized dense matrix, for tests and small instances (kernel2d.py:278-290)."""
    full = np.kron(op.ky.dense_realization(), op.kx.dense_realization())
    if op.absorbed:
        av = op.absorption_left.ravel(order="F")
        bv = op.absorption_right.ravel(order="F")
        full = full * np.exp((av[:, None] + bv[None, :]) / op.epsilon)
    return full


def sinkhorn_2d(source, target, u, v, config):
    """Entropic scaling between grid measures on the B200 (kernel2d.py:363-391)."""
    if u.shape != source.shape:
        raise DimensionMismatch("u must have one weight per source point")
    if v.shape != target.shape:
        raise DimensionMismatch("v must have one weight per target point")
    (n1, m1), (n2, m2) = source.shape, target.shape
    x1, y1 = source.x_nodes.nodes, source.y_nodes.nodes
    x2, y2 = target.x_nodes.nodes, target.y_nodes.nodes
    # a C-ordered grid goes as is (the library transposes it on the device;
    # numpy's strided F-order ravel of a 512 MB grid costs over a second)
    def weights_arg(w):
        if w.flags.f_contiguous:
            return np.asarray(w, dtype=np.float64).ravel(order="F"), 0
        return np.ascontiguousarray(w, dtype=np.float64), 1
    U, u_rm = weights_arg(u.weights)
    V, v_rm = weights_arg(v.weights)
    if u_rm != v_rm:  # mixed layouts: both flat column-major
        U, u_rm = np.ascontiguousarray(u.weights.ravel(order="F")), 0
        V = np.ascontiguousarray(v.weights.ravel(order="F"))
    itr = int(config.itr_max)
    phi, A = np.empty(n1 * m1), np.empty(n1 * m1)
    psi, B = np.empty(n2 * m2), np.empty(n2 * m2)
    hist = np.zeros(itr)
    info = np.zeros(5, dtype=np.int64)
    abs_its = np.zeros(itr, dtype=np.int64)
    cost = np.zeros(1)
    timing = np.zeros(3)
    lib = _lib.load()
    status = _lib.check(lib.finom_sinkhorn2d_host(
        n1, _lib.ptr(x1), m1, _lib.ptr(y1), n2, _lib.ptr(x2), m2, _lib.ptr(y2), _lib.ptr(U),
        _lib.ptr(V), config.epsilon, itr, float(config.tol), int(bool(config.stabilize)),
        float(config.absorb_threshold), _lib.ptr(phi), _lib.ptr(psi), _lib.ptr(A), _lib.ptr(B),
        _lib.ptr(hist), _lib.ptr(info), _lib.ptr(abs_its), _lib.ptr(cost), _lib.ptr(timing),
        u_rm), "finom_sinkhorn2d_host")
    raise_status(status)
    its, conv = int(info[0]), bool(info[1])
    op = build_operator_2d(source, target, config.epsilon)
    op = KernelOperator2D(op.kx, op.ky, op.epsilon, A.reshape((n1, m1), order="F"),
                          B.reshape((n2, m2), order="F"))
    return Solution(
        phi=phi, psi=psi, a=A, b=B, kernel=op, iterations_run=its, converged=conv,
        marginal_error_history=history_from(hist, its, conv, config),
        wall_time=float(timing[0] + timing[1]), setup_time=float(timing[0]),
        cost=float(cost[0]), config=config,
        absorb_iterations=[int(k) for k in abs_its[:int(info[3])]])


def transport_cost_fast_2d(solution):
    """<C, plan> via the per-axis split of the separable cost (kernel2d.py:394-465)."""
    op = solution.kernel
    x1, y1, x2, y2 = op._meshes()
    (n1, m1), (n2, m2) = op.source_shape, op.target_shape
    A = np.ascontiguousarray(op.absorption_left.ravel(order="F"))
    B = np.ascontiguousarray(op.absorption_right.ravel(order="F"))
    phi = np.ascontiguousarray(solution.phi, dtype=np.float64)
    psi = np.ascontiguousarray(solution.psi, dtype=np.float64)
    out = np.zeros(1)
    lib = _lib.load()
    _lib.check(lib.finom_cost2d_host(n1, _lib.ptr(x1), m1, _lib.ptr(y1), n2, _lib.ptr(x2), m2,
                                     _lib.ptr(y2), op.epsilon, _lib.ptr(A), _lib.ptr(B),
                                     _lib.ptr(phi), _lib.ptr(psi), _lib.ptr(out)),
               "finom_cost2d_host")
    return float(out[0])
