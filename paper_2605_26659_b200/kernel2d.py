"""Separable 2D kernel and the grid solver on the B200 (drop-in for finom.kernel2d).

K = Ky (x) Kx on tensor-product grids, vectors flattened column-major
(x fastest, mesh.py:85-107, kernel2d.py:1-19).  The device path
(csrc/finom_2d.inc) runs every column sweep and row sweep as a batch of
1D line scans sharing one mesh, with a tiled transpose in between, and
switches to the dynamic-shift exponent form after the first absorption
exactly as _GridAdapter does (kernel2d.py:293-360).
"""

from dataclasses import dataclass

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


def dense_realization_2d(op, phi=None, psi=None):
    """Vectorized dense matrix on the device, for tests and small instances
    (kernel2d.py:278-290: kron(Ky, Kx) [* exp((A_I + B_J) / eps)],
    finom_dense2d); with phi / psi the plan diag(phi) K diag(psi)."""
    x1, y1, x2, y2 = op._meshes()
    A = B = None
    if op.absorbed:
        A = op.absorption_left.ravel(order="F")
        B = op.absorption_right.ravel(order="F")
    return _lib.dense2d(x1, y1, x2, y2, A, B, op.epsilon, phi, psi)


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


class GridSolver2D:
    """Device-resident 2D problem (no reference equivalent; semantics ==
    sinkhorn_2d): one grid plan (finom_grid_create), weights and iterates in
    HBM as torch tensors, solve / cost through finom_solve2d / finom_cost2d
    on the current stream -- the device-pointer form of sinkhorn_2d for
    callers whose grids already live on the GPU."""

    def __init__(self, source, target, epsilon, u=None, v=None):
        import torch
        epsilon = kernel1d._check_eps(epsilon)
        self.grid = _lib.Grid(source.x_nodes.nodes, source.y_nodes.nodes,
                              target.x_nodes.nodes, target.y_nodes.nodes, epsilon)
        (n1, m1), (n2, m2) = self.grid.shape_u, self.grid.shape_v
        self.N1, self.N2 = n1 * m1, n2 * m2
        f64 = dict(dtype=torch.float64, device="cuda")
        self.u = torch.zeros(self.N1, **f64)
        self.v = torch.zeros(self.N2, **f64)
        self.phi = torch.empty(self.N1, **f64)
        self.psi = torch.empty(self.N2, **f64)
        self.a = torch.empty(self.N1, **f64)
        self.b = torch.empty(self.N2, **f64)
        self.cost_dev = torch.zeros(1, **f64)
        self.info = torch.zeros(5, dtype=torch.int64, device="cuda")
        self._itr = None
        if u is not None:
            self.set_weights(u, v)

    def set_weights(self, u, v):
        """Weights as flat column-major vectors (numpy or torch)."""
        import torch
        for dst, w in ((self.u, u), (self.v, v)):
            w = getattr(w, "weights", w)
            if isinstance(w, np.ndarray) and w.ndim == 2:
                w = w.ravel(order="F")
            dst.copy_(torch.as_tensor(np.asarray(w) if not torch.is_tensor(w) else w,
                                      dtype=torch.float64).reshape(-1))

    def solve(self, itr_max, tol=0.0, stabilize=True, absorb_threshold=200.0):
        """Run sinkhorn_2d's loop on the device buffers; returns the status (0/1/2)."""
        import torch
        if self._itr != int(itr_max):
            self.hist = torch.zeros(int(itr_max), dtype=torch.float64, device="cuda")
            self.absorb_its = torch.zeros(int(itr_max), dtype=torch.int64, device="cuda")
            self._itr = int(itr_max)
        lib = _lib.load()
        return _lib.check(lib.finom_solve2d(
            self.grid.handle, _lib.ptr(self.u), _lib.ptr(self.v), _lib.ptr(self.phi),
            _lib.ptr(self.psi), _lib.ptr(self.a), _lib.ptr(self.b), int(itr_max), float(tol),
            int(bool(stabilize)), float(absorb_threshold), _lib.ptr(self.hist),
            _lib.ptr(self.info), _lib.ptr(self.absorb_its), _lib.stream_ptr()), "finom_solve2d")

    def compute_cost(self, absorbed=True):
        """transport_cost_fast_2d of the current state into cost_dev (device)."""
        lib = _lib.load()
        a, b = (self.a, self.b) if absorbed else (None, None)
        _lib.check(lib.finom_cost2d(self.grid.handle, _lib.ptr(self.phi), _lib.ptr(self.psi),
                                    _lib.ptr(a), _lib.ptr(b), _lib.ptr(self.cost_dev),
                                    _lib.stream_ptr()), "finom_cost2d")
        return self.cost_dev


class GpuGridAdapter:
    """The adapter protocol (solver.py:1-16) on the device grid path: the B200
    counterpart of _GridAdapter (kernel2d.py:293-360), so run_driver can drive
    the 2D solve (and A/B-test it against the reference loop).  iterate()
    runs one finom_iterate2d on the flat vectors in place; absorb() advances
    the shift grids and rebuilds the sweep tables (finom_grid_set_shifts)."""

    def __init__(self, source, target, epsilon):
        import torch
        self.op = build_operator_2d(source, target, epsilon)
        self.grid = _lib.Grid(source.x_nodes.nodes, source.y_nodes.nodes,
                              target.x_nodes.nodes, target.y_nodes.nodes, self.op.epsilon)
        f64 = dict(dtype=torch.float64, device="cuda")
        (n1, m1), (n2, m2) = source.shape, target.shape
        self._shape_u, self._shape_v = (n1, m1), (n2, m2)
        self._U = torch.empty(n1 * m1, **f64)
        self._V = torch.empty(n2 * m2, **f64)
        self._PHI = torch.empty(n1 * m1, **f64)
        self._PSI = torch.empty(n2 * m2, **f64)
        self._A = None
        self._B = None
        self._res = torch.zeros(6, **f64)

    @property
    def kernel(self):
        return self.op

    @property
    def a(self):
        return self.op.absorption_left.ravel(order="F")

    @property
    def b(self):
        return self.op.absorption_right.ravel(order="F")

    def iterate(self, u, v, phi, psi):
        import torch
        self._U.copy_(torch.from_numpy(np.ascontiguousarray(u, dtype=np.float64)))
        self._V.copy_(torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)))
        self._PHI.copy_(torch.from_numpy(np.ascontiguousarray(phi, dtype=np.float64)))
        self._PSI.copy_(torch.from_numpy(np.ascontiguousarray(psi, dtype=np.float64)))
        lib = _lib.load()
        _lib.check(lib.finom_iterate2d(self.grid.handle, _lib.ptr(self._U), _lib.ptr(self._V),
                                       _lib.ptr(self._PHI), _lib.ptr(self._PSI),
                                       _lib.ptr(self._res), _lib.stream_ptr()), "finom_iterate2d")
        phi[:] = self._PHI.cpu().numpy()
        psi[:] = self._PSI.cpu().numpy()
        r = self._res.cpu().numpy()
        return float(r[0]), int(r[1]), float(r[2]), float(r[3]), float(r[4]), float(r[5])

    def absorb(self, delta_a, delta_b):
        import torch
        dA = np.asarray(delta_a).reshape(self._shape_u, order="F")
        dB = np.asarray(delta_b).reshape(self._shape_v, order="F")
        self.op = absorb_2d(self.op, dA, dB)
        self._A = torch.from_numpy(np.ascontiguousarray(self.a)).cuda()
        self._B = torch.from_numpy(np.ascontiguousarray(self.b)).cuda()
        lib = _lib.load()
        _lib.check(lib.finom_grid_set_shifts(self.grid.handle, _lib.ptr(self._A),
                                             _lib.ptr(self._B), _lib.stream_ptr()),
                   "finom_grid_set_shifts")
