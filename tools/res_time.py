"""Resolve-chain timeline of iteration 4 (FB_DBG_RES build) on config 2."""
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
ph = np.zeros(16)
for graph in (0, 1):
    lib.finom_phase_read(_lib.ptr(ph))
    if graph:
        bs.solve(8, 0.0, True, 200.0)
    else:
        prof = np.zeros(6); hist = torch.zeros(20, dtype=torch.float64, device="cuda")
        _lib.check(lib.finom_profile1d(bs.plan.handle, _lib.ptr(bs.u), _lib.ptr(bs.v), _lib.ptr(bs.phi), _lib.ptr(bs.psi), _lib.ptr(bs.a), _lib.ptr(bs.b), 8, 1, 200.0, _lib.ptr(hist), _lib.ptr(prof), _lib.stream_ptr()), "prof")
    torch.cuda.synchronize()
    lib.finom_phase_read(_lib.ptr(ph))
    u64 = ph.astype(np.float64)
    raw = [int(v) for v in ph]
    t = {}
    t["k_step0 end"] = raw[8]
    t["resolve0 first start"] = (~raw[9]) & ((1 << 64) - 1) if raw[9] else 0
    t["group loads done (max)"] = raw[10]
    t["group stored (max)"] = raw[11]
    t["L1 last arriver"] = raw[12]
    t["L2 last arriver"] = raw[13]
    t["driver step"] = raw[14]
    t["k_step1 first start"] = (~raw[15]) & ((1 << 64) - 1) if raw[15] else 0
    base = t["k_step0 end"]
    print("graph" if graph else "ungraphed")
    for k, v in t.items():
        print("  %-24s %+9.2f us" % (k, (v - base) / 1e3 if v else float("nan")))
