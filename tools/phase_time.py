"""Per-phase cycle counts of k_step (FB_DBG_PHASE build) on config 2."""
import os, sys, ctypes, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_26659_b200 import _lib, workloads as W
_lib.LIB_PATH = sys.argv[1]
import paper_2605_26659_b200 as fb
x, y, u, v, eps = W.config2()
bs = fb.BatchSolver1D([x], [y], [u], [v], [eps])
lib = _lib.load()
lib.finom_phase_read.argtypes = [ctypes.c_void_p]
prof = np.zeros(6); ph = np.zeros(16)
hist = torch.zeros(20, dtype=torch.float64, device="cuda")
lib.finom_phase_read(_lib.ptr(ph))
iters = 10
_lib.check(lib.finom_profile1d(bs.plan.handle, _lib.ptr(bs.u), _lib.ptr(bs.v), _lib.ptr(bs.phi), _lib.ptr(bs.psi), _lib.ptr(bs.a), _lib.ptr(bs.b), iters, 1, 200.0, _lib.ptr(hist), _lib.ptr(prof), _lib.stream_ptr()), "prof")
lib.finom_phase_read(_lib.ptr(ph))
T = bs.plan.info()["tiles"]
names = ["wait full", "mask", "col operands", "maps+carry+states", "apply", "epilogue", "reduce+node", "-", "P: desc batch", "P: wait empty", "P: issue"]
tot = ph[:8].sum()
for k, n in enumerate(names):
    print("%-14s %8.0f cycles/tile  %5.1f%%" % (n, ph[k] / (T * iters * 2), 100 * ph[k] / tot))
print("halfA %.3f halfB %.3f ms" % (prof[0], prof[1]))
