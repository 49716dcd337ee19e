"""Dense (materialized-kernel) Sinkhorn on the B200: the comparison baseline.

The reference's ``finom.dense`` (pkg/src/finom/dense.py:1-215) stores the
full kernel and runs the scaling loop with plain BLAS products; the paper's
speed-up tables are measured against it.
Here the kernel lives in HBM (fp64) and each half is one cuBLAS DGEMV
(``phi @ K`` / ``K @ psi``) plus the same scaling-update rules; the
run_driver decisions (solver.py:156-199) read one small vector back per
iteration.  It exists to be correct and to be beaten: the O(N) path of this
package (csrc/) is the product, this module is the yardstick.  Like every
entry point here it needs a CUDA device (no CPU fallback).
"""

from dataclasses import dataclass
from time import perf_counter

import numpy as np

from . import _lib
from .errors import DimensionMismatch, InvalidEpsilon, SizeCapExceeded
from .solver import Solution, raise_status

SIZE_CAP = 10**8  # dense.py:22
_OK, _ZERO_DENOM, _NONFINITE = 0, 1, 2


def _torch():
    import torch
    _lib.load()  # raises DeviceError without a CUDA device
    return torch


def _check_eps(epsilon):
    """dense.py:69-73."""
    epsilon = float(epsilon)
    if not np.isfinite(epsilon) or epsilon <= 0:
        raise InvalidEpsilon("epsilon must be a positive finite real")
    return epsilon


def _check_cap(n, m, size_cap):
    """dense.py:76-80."""
    if n * m > size_cap:
        raise SizeCapExceeded("dense kernel would hold %d entries, cap is %d" % (n * m, size_cap))


@dataclass(frozen=True)
class DenseKernel:
    """Full kernel in HBM: entries[i, j] = exp((-cost[i, j] + a[i] + b[j]) / eps)
    (dense.py:26-66).  Tensors are fp64 on the CUDA device."""

    entries: object
    cost: object
    epsilon: float
    a: object
    b: object

    @property
    def shape(self):
        return tuple(self.entries.shape)

    def apply(self, psi):
        """K psi (one DGEMV)."""
        torch = _torch()
        v = torch.as_tensor(np.asarray(psi, dtype=np.float64), device=self.entries.device)
        return torch.mv(self.entries, v).cpu().numpy()

    def apply_transpose(self, phi):
        """phi K (one DGEMV with the transposed operand, K^T never formed)."""
        torch = _torch()
        v = torch.as_tensor(np.asarray(phi, dtype=np.float64), device=self.entries.device)
        return torch.mv(self.entries.t(), v).cpu().numpy()

    def absorb(self, delta_a, delta_b):
        """New kernel from the summed exponent, never by rescaling (dense.py:51-62)."""
        torch = _torch()
        dev = self.entries.device
        a = self.a + torch.as_tensor(np.asarray(delta_a, dtype=np.float64), device=dev)
        b = self.b + torch.as_tensor(np.asarray(delta_b, dtype=np.float64), device=dev)
        entries = torch.exp((-self.cost + a[:, None] + b[None, :]) / self.epsilon)
        return DenseKernel(entries=entries, cost=self.cost, epsilon=self.epsilon, a=a, b=b)

    def dense_realization(self):
        return self.entries.cpu().numpy()


def _kernel_from_cost(cost, epsilon):
    torch = _torch()
    n, m = cost.shape
    f64 = dict(dtype=torch.float64, device=cost.device)
    return DenseKernel(entries=torch.exp(-cost / epsilon), cost=cost, epsilon=epsilon,
                       a=torch.zeros(n, **f64), b=torch.zeros(m, **f64))


def dense_kernel(x, y, epsilon, size_cap=SIZE_CAP):
    """Cost and kernel of meshes x (rows) and y (columns) (dense.py:83-90)."""
    torch = _torch()
    epsilon = _check_eps(epsilon)
    _check_cap(len(x), len(y), size_cap)
    dev = torch.device("cuda")
    tx = torch.tensor(np.asarray(x.nodes, dtype=np.float64), device=dev)
    ty = torch.tensor(np.asarray(y.nodes, dtype=np.float64), device=dev)
    return _kernel_from_cost(torch.abs(tx[:, None] - ty[None, :]), epsilon)


def dense_kernel_2d(source, target, epsilon, size_cap=SIZE_CAP):
    """Kronecker kernel of a grid pair, points x-fastest (dense.py:93-111)."""
    torch = _torch()
    epsilon = _check_eps(epsilon)
    n, m = len(source), len(target)
    _check_cap(n, m, size_cap)
    dev = torch.device("cuda")
    t = lambda z: torch.tensor(np.asarray(z.nodes, dtype=np.float64), device=dev)
    cx = torch.abs(t(source.x_nodes)[:, None] - t(target.x_nodes)[None, :])
    cy = torch.abs(t(source.y_nodes)[:, None] - t(target.y_nodes)[None, :])
    cost = torch.kron(cy, torch.ones_like(cx)) + torch.kron(torch.ones_like(cy), cx)
    return _kernel_from_cost(cost, epsilon)


def _half(torch, prod, target, out):
    """scaling_out <- target / prod with the compressed kernels' rules
    (dense.py:132-143): ZERO_DENOM if some prod == 0 carries mass, NONFINITE
    if a quotient overflows; extremes over the positive-mass entries.
    Returns device scalars (status, max, min) -- no host sync here."""
    zero = prod == 0.0
    zd = torch.any(zero & (target > 0.0))
    w = torch.where(zero, torch.zeros_like(prod), target / torch.where(zero, torch.ones_like(prod), prod))
    nf = ~torch.all(torch.isfinite(w))
    pos = target > 0.0
    wmax = torch.max(torch.where(pos, w, torch.full_like(w, -np.inf)))
    wmin = torch.min(torch.where(pos, w, torch.full_like(w, np.inf)))
    status = torch.where(zd, torch.tensor(_ZERO_DENOM, device=prod.device),
                         torch.where(nf, torch.tensor(_NONFINITE, device=prod.device),
                                     torch.tensor(_OK, device=prod.device)))
    ok = status == _OK
    out.copy_(torch.where(ok, w, out))
    return status, wmax, wmin


def _shift(torch, weights, scaling, epsilon):
    """solver._shift (solver.py:135-153) on the host copy: np.interp fill."""
    w = weights.cpu().numpy()
    sc = scaling.cpu().numpy()
    pos = w > 0
    vals = epsilon * np.log(sc[pos])
    if pos.all():
        out = vals
    else:
        out = np.empty(w.shape[0])
        idx = np.arange(w.shape[0], dtype=float)
        out[pos] = vals
        out[~pos] = np.interp(idx[~pos], idx[pos], vals)
    return out


def dense_sinkhorn(problem, config):
    """The scaling loop with dense matvecs (dense.py:161-193): run_driver's
    semantics (solver.py:156-199) with both halves on the device."""
    torch = _torch()
    t0 = perf_counter()
    dev = torch.device("cuda")
    if problem.dim == 1:
        kern = dense_kernel(problem.source, problem.target, config.epsilon, size_cap=config.plan_cap)
        u = np.asarray(problem.u.weights, dtype=np.float64)
        v = np.asarray(problem.v.weights, dtype=np.float64)
    else:
        kern = dense_kernel_2d(problem.source, problem.target, config.epsilon,
                               size_cap=config.plan_cap)
        u = np.ascontiguousarray(problem.u.weights.ravel(order="F"))
        v = np.ascontiguousarray(problem.v.weights.ravel(order="F"))
    n, m = kern.shape
    if u.shape[0] != n or v.shape[0] != m:
        raise DimensionMismatch("weights do not match the kernel's shape")
    tu = torch.tensor(u, device=dev)
    tv = torch.tensor(v, device=dev)
    phi = torch.full((n,), 1.0 / n, dtype=torch.float64, device=dev)  # solver.py:165-166
    psi = torch.full((m,), 1.0 / n, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    setup = perf_counter() - t0
    hi_cut, lo_cut = np.exp(config.absorb_threshold), np.exp(-config.absorb_threshold)
    history, converged, it, absorbs = [], False, 0, []
    t1 = perf_counter()
    while it < config.itr_max:
        t = torch.mv(kern.entries.t(), phi)
        err = torch.sum(torch.abs(psi * t - tv))
        st_a, psmax, psmin = _half(torch, t, tv, psi)
        s = torch.mv(kern.entries, psi)
        st_b, phmax, phmin = _half(torch, s, tu, phi)
        vals = torch.stack([err, st_a.double(), st_b.double(), psmax, psmin, phmax, phmin]).tolist()
        err_h, sa, sb, psmax_h, psmin_h, phmax_h, phmin_h = vals
        it += 1
        raise_status(int(sa) if sa else int(sb))
        recorded = it % config.check_every == 0 or it == config.itr_max
        if recorded:
            history.append((it, float(err_h)))
        if config.tol > 0 and err_h <= config.tol:
            if not recorded:
                history.append((it, float(err_h)))
            converged = True
            break
        if config.stabilize and (phmax_h > hi_cut or psmax_h > hi_cut or phmin_h < lo_cut
                                 or psmin_h < lo_cut):
            kern = kern.absorb(_shift(torch, tu, phi, config.epsilon),
                               _shift(torch, tv, psi, config.epsilon))
            phi.fill_(1.0)
            psi.fill_(1.0)
            absorbs.append(it)
    torch.cuda.synchronize()
    loop = perf_counter() - t1
    plan = phi[:, None] * kern.entries * psi[None, :]
    cost = float(torch.sum(plan * kern.cost).item())
    return Solution(phi=phi.cpu().numpy(), psi=psi.cpu().numpy(), a=kern.a.cpu().numpy(),
                    b=kern.b.cpu().numpy(), kernel=kern, iterations_run=it, converged=converged,
                    marginal_error_history=history, wall_time=setup + loop, setup_time=setup,
                    cost=cost, config=config, absorb_iterations=absorbs)


def frobenius_diff(plan_a, plan_b):
    """Frobenius norm of the difference of two plans (dense.py:196-203)."""
    a = np.asarray(plan_a, dtype=float)
    b = np.asarray(plan_b, dtype=float)
    if a.shape != b.shape:
        raise DimensionMismatch("plans differ in shape: %s vs %s" % (a.shape, b.shape))
    return float(np.linalg.norm(a - b))


def transport_cost_dense(plan, cost):
    """<C, plan> summed entrywise (dense.py:206-215)."""
    p = np.asarray(plan, dtype=float)
    c = np.asarray(cost, dtype=float)
    if p.shape != c.shape:
        raise DimensionMismatch("plan and cost differ in shape: %s vs %s" % (p.shape, c.shape))
    return float(np.sum(p * c))
