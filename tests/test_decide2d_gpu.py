"""The device decisions of the row-sharded 2D driver (finom_grid2d_decide)
against the host restatement of run_driver (sharding.run_driver_2d over
sharding.combine_parts, solver.py:156-199), on scripted shard partials."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _device_run(script, R, cfg, fn="finom_grid2d_decide"):
    import torch
    from paper_2605_26659_b200 import _lib
    lib = _lib.load()
    dev = torch.device("cuda")
    ctl = torch.zeros(8, dtype=torch.int64, device=dev)
    hist = torch.zeros(cfg.itr_max, dtype=torch.float64, device=dev)
    abs_its = torch.zeros(cfg.itr_max, dtype=torch.int64, device=dev)
    it = 1
    while True:
        pa = torch.tensor(script[(it, 0)], dtype=torch.float64, device=dev)
        pb = torch.tensor(script[(it, 1)], dtype=torch.float64, device=dev)
        _lib.check(getattr(lib, fn)(_lib.ptr(pa), _lib.ptr(pb), R, _lib.ptr(ctl),
                                           _lib.ptr(hist), _lib.ptr(abs_its), cfg.itr_max,
                                           cfg.tol, int(cfg.stabilize), cfg.absorb_threshold,
                                           _lib.stream_ptr()), "decide")
        c = ctl.cpu().numpy()
        if c[4]:
            break
        it += 1
    n = int(c[0])
    return (n, bool(c[2]), int(c[1]), hist[:n].cpu().tolist(),
            abs_its[:int(c[5])].cpu().tolist())


def _host_run(script, cfg, combine="combine_parts"):
    from paper_2605_26659_b200 import sharding as S
    state = {"it": 1}

    def phase(half, dyn):
        out = getattr(S, combine)(np.asarray(script[(state["it"], half)]).reshape(-1, 4))
        if half == 1:
            state["it"] += 1
        return out

    return S.run_driver_2d(phase, lambda: None, cfg)


@pytest.mark.parametrize("case", ["absorb_then_fail", "tol", "itr_max_absorb_last"])
def test_device_decisions_match_run_driver(case):
    from paper_2605_26659_b200 import SolverConfig
    R = 3
    rng = np.random.default_rng(3)
    script = {}
    for it in range(1, 13):
        for half in (0, 1):
            p = np.zeros((R, 4))
            p[:, 0] = rng.uniform(0.01, 0.1, R) / it
            p[:, 1] = rng.uniform(1.0, 2.0, R)
            p[:, 2] = rng.uniform(0.5, 1.0, R)
            p[:, 3] = -1.0
            script[(it, half)] = p.ravel().tolist()
    if case == "absorb_then_fail":
        script[(3, 0)][1 * 4 + 1] = 1e90           # rank 1 out of range -> absorb at it 3
        script[(5, 1)][2 * 4 + 2] = 1e-90          # rank 2 below range (half B) -> absorb at 5
        script[(7, 0)][0 * 4 + 3] = 4.0 * 77 + 2   # failures on two ranks: the min code wins
        script[(7, 0)][2 * 4 + 3] = 4.0 * 12 + 1
        cfg = SolverConfig(epsilon=1e-2, itr_max=12, tol=0.0, stabilize=True,
                           absorb_threshold=200.0)
    elif case == "tol":
        cfg = SolverConfig(epsilon=1e-2, itr_max=12, tol=0.02, stabilize=True,
                           absorb_threshold=200.0)
    else:
        script[(12, 1)][0 * 4 + 1] = 1e95          # absorption on the last iteration
        cfg = SolverConfig(epsilon=1e-2, itr_max=12, tol=0.0, stabilize=True,
                           absorb_threshold=200.0)
    dev = _device_run(script, R, cfg)
    host = _host_run(script, cfg)
    assert dev[:3] == host[:3]
    assert dev[3] == host[3]  # (rank-order sums: bitwise)
    assert dev[4] == host[4]


def test_seg1d_device_decisions_last_failing_segment():
    """finom_seg1d_decide: partials carry a status, the LAST failing segment's
    is reported (combine_parts_1d)."""
    from paper_2605_26659_b200 import SolverConfig
    R = 4
    script = {}
    for it in range(1, 9):
        for half in (0, 1):
            p = np.zeros((R, 4))
            p[:, 0] = 0.01 * (R - np.arange(R)) / it
            p[:, 1] = 1.5
            p[:, 2] = 0.75
            p[:, 3] = -1.0
            script[(it, half)] = p.ravel().tolist()
    script[(2, 1)][2 * 4 + 1] = 1e90       # absorption at iteration 2
    script[(6, 0)][1 * 4 + 3] = 2.0        # NONFINITE on segment 1 ...
    script[(6, 0)][3 * 4 + 3] = 1.0        # ... and ZERO_DENOM on segment 3: the last one wins
    cfg = SolverConfig(epsilon=1e-2, itr_max=8, tol=0.0, stabilize=True, absorb_threshold=200.0)
    dev = _device_run(script, R, cfg, fn="finom_seg1d_decide")
    host = _host_run(script, cfg, combine="combine_parts_1d")
    assert dev[:3] == host[:3] == (6, False, 1)
    assert dev[3] == host[3] and dev[4] == host[4] == [2]
