"""Time k_half of config 2 for library variants (timing experiments)."""
import os, sys, ctypes, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_26659_b200 import _lib, workloads as W
lib_path = sys.argv[1]
_lib.LIB_PATH = lib_path
import paper_2605_26659_b200 as fb
x, y, u, v, eps = W.config2()
bs = fb.BatchSolver1D([x], [y], [u], [v], [eps])
lib = _lib.load()
prof = np.zeros(6)
hist = torch.zeros(20, dtype=torch.float64, device="cuda")
for rep in range(2):
    _lib.check(lib.finom_profile1d(bs.plan.handle, _lib.ptr(bs.u), _lib.ptr(bs.v), _lib.ptr(bs.phi), _lib.ptr(bs.psi), _lib.ptr(bs.a), _lib.ptr(bs.b), 10, 1, 200.0, _lib.ptr(hist), _lib.ptr(prof), _lib.stream_ptr()), "prof")
print(os.path.basename(lib_path), "halfA %.3f halfB %.3f (resolve %.3f) absorb %.3f ms" % (prof[0], prof[1], prof[2], prof[3]))
