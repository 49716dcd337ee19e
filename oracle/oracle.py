"""ctypes wrapper of the C oracle (oracle/finom_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product package
never imports this module.
"""

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libfinom_oracle.so")

_lib = None
_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_d = ctypes.c_double
_i = ctypes.c_int


def build():
    subprocess.check_call(["make", "-s", "-C", HERE])


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        lib = ctypes.CDLL(LIB)
        lib.orc_sinkhorn_1d.restype = _i
        lib.orc_sinkhorn_1d.argtypes = [_i64, _vp, _i64, _vp, _vp, _vp, _d, _i64, _d, _i, _d,
                                        _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
        lib.orc_sinkhorn_1d_timed.restype = _i
        lib.orc_sinkhorn_1d_timed.argtypes = lib.orc_sinkhorn_1d.argtypes + [_vp]
        lib.orc_apply_1d.restype = _i
        lib.orc_apply_1d.argtypes = [_i64, _vp, _i64, _vp, _d, _vp, _vp, _vp, _i, _vp, _vp]
        lib.orc_cost_1d.restype = _i
        lib.orc_cost_1d.argtypes = [_i64, _vp, _i64, _vp, _d, _vp, _vp, _vp, _vp, _vp]
        lib.orc_sinkhorn_1d_batch.restype = _i
        lib.orc_sinkhorn_1d_batch.argtypes = [_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _d,
                                              _i, _d, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
        lib.orc_sinkhorn_2d.restype = _i
        lib.orc_sinkhorn_2d.argtypes = [_i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _vp, _vp, _d,
                                        _i64, _d, _i, _d, _i64, _vp, _vp, _vp, _vp, _vp, _vp,
                                        _vp, _vp]
        lib.orc_cost_2d.restype = _i
        lib.orc_cost_2d.argtypes = [_i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _d, _vp, _vp,
                                    _vp, _vp, _vp]
        lib.orc_dividing_index.restype = None
        lib.orc_dividing_index.argtypes = [_vp, _i64, _vp, _i64, _vp]
        _lib = lib
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def _f(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def sinkhorn_1d(x, y, u, v, eps, itr_max, tol=0.0, stabilize=False, thr=200.0, check_every=1):
    """solver.sinkhorn_1d restated in C.  Returns a dict of outputs."""
    x, y, u, v = _f(x), _f(y), _f(u), _f(v)
    n, m = x.size, y.size
    phi, psi, a, b = np.empty(n), np.empty(m), np.empty(n), np.empty(m)
    hist = np.zeros(itr_max)
    info = np.zeros(5, dtype=np.int64)
    abs_its = np.zeros(itr_max, dtype=np.int64)
    cost = np.zeros(1)
    timing = np.zeros(3)
    st = load().orc_sinkhorn_1d_timed(n, _p(x), m, _p(y), _p(u), _p(v), eps, itr_max, tol,
                                      int(stabilize), thr, check_every, _p(phi), _p(psi), _p(a),
                                      _p(b), _p(hist), _p(info), _p(abs_its), _p(cost),
                                      _p(timing))
    return dict(status=st, phi=phi, psi=psi, a=a, b=b, hist=hist[:info[0]],
                iterations=int(info[0]), converged=bool(info[1]), n_absorb=int(info[3]),
                absorb_its=abs_its[:info[3]].copy(), cost=float(cost[0]),
                setup_s=float(timing[0]), loop_s=float(timing[1]), cost_s=float(timing[2]))


def apply_1d(x, y, eps, vin, mode, a=None, b=None):
    x, y, vin = _f(x), _f(y), _f(vin)
    n, m = x.size, y.size
    a = None if a is None else _f(a)
    b = None if b is None else _f(b)
    out = np.empty(m if mode == 1 else n)
    out2 = np.empty(n) if mode == 2 else None
    load().orc_apply_1d(n, _p(x), m, _p(y), eps, _p(a), _p(b), _p(vin), mode, _p(out), _p(out2))
    return (out, out2) if mode == 2 else out


def cost_1d(x, y, eps, a, b, phi, psi):
    x, y, a, b, phi, psi = (_f(z) for z in (x, y, a, b, phi, psi))
    c = np.zeros(1)
    load().orc_cost_1d(x.size, _p(x), y.size, _p(y), eps, _p(a), _p(b), _p(phi), _p(psi), _p(c))
    return float(c[0])


def sinkhorn_2d(x1, y1, x2, y2, U, V, eps, itr_max, tol=0.0, stabilize=False, thr=200.0,
                check_every=1):
    x1, y1, x2, y2 = _f(x1), _f(y1), _f(x2), _f(y2)
    n1, m1, n2, m2 = x1.size, y1.size, x2.size, y2.size
    uf = np.ascontiguousarray(np.asarray(U, dtype=np.float64).ravel(order="F"))
    vf = np.ascontiguousarray(np.asarray(V, dtype=np.float64).ravel(order="F"))
    phi, psi = np.empty(n1 * m1), np.empty(n2 * m2)
    A, B = np.empty(n1 * m1), np.empty(n2 * m2)
    hist = np.zeros(itr_max)
    info = np.zeros(5, dtype=np.int64)
    abs_its = np.zeros(itr_max, dtype=np.int64)
    cost = np.zeros(1)
    st = load().orc_sinkhorn_2d(n1, _p(x1), m1, _p(y1), n2, _p(x2), m2, _p(y2), _p(uf), _p(vf),
                                eps, itr_max, tol, int(stabilize), thr, check_every, _p(phi),
                                _p(psi), _p(A), _p(B), _p(hist), _p(info), _p(abs_its), _p(cost))
    return dict(status=st, phi=phi, psi=psi, a=A, b=B, hist=hist[:info[0]],
                iterations=int(info[0]), converged=bool(info[1]), n_absorb=int(info[3]),
                absorb_its=abs_its[:info[3]].copy(), cost=float(cost[0]))
