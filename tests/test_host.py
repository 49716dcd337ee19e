"""Host-side mirror of the reference interface: config, types, errors, cadence."""

import dataclasses

import numpy as np
import pytest

import paper_2605_26659_b200 as fb
from paper_2605_26659_b200 import errors, kernel1d, solver


class TestConfig:  # mirrors test_solver.py:54-111
    def test_defaults(self):
        cfg = fb.SolverConfig(epsilon=0.5)
        assert (cfg.itr_max, cfg.tol, cfg.stabilize, cfg.absorb_threshold, cfg.check_every,
                cfg.plan_cap) == (1000, 1e-9, False, 200.0, 1, 10**8)

    @pytest.mark.parametrize("eps", [0.0, -1.0, np.nan, np.inf])
    def test_bad_epsilon(self, eps):
        with pytest.raises(errors.InvalidEpsilon):
            fb.SolverConfig(epsilon=eps)

    @pytest.mark.parametrize("kw", [dict(itr_max=0), dict(tol=-1e-9), dict(tol=np.nan),
                                    dict(absorb_threshold=1.0), dict(absorb_threshold=np.inf),
                                    dict(check_every=0), dict(plan_cap=0)])
    def test_bad_values(self, kw):
        with pytest.raises(errors.ConfigError):
            fb.SolverConfig(epsilon=1.0, **kw)

    def test_frozen(self):
        cfg = fb.SolverConfig(epsilon=1.0)
        with pytest.raises(dataclasses.FrozenInstanceError):
            cfg.tol = 0.5


class TestTypes:
    def test_mesh_validation(self):
        with pytest.raises(errors.UnsortedInput):
            fb.Mesh1D([1.0, 0.5])
        with pytest.raises(errors.DuplicateNode):
            fb.Mesh1D([1.0, 1.0, 2.0])
        with pytest.raises(errors.NonFiniteCoordinate):
            fb.Mesh1D([0.0, np.nan])
        with pytest.raises(errors.ValidationError):
            fb.Mesh1D([])

    def test_measure_validation(self):
        with pytest.raises(errors.ValidationError):
            fb.Measure([0.5, 0.6])
        with pytest.raises(errors.ValidationError):
            fb.Measure([1.5, -0.5])
        assert len(fb.Measure([0.25, 0.75])) == 2

    def test_grid(self):
        g = fb.Grid2D(fb.Mesh1D([0, 1, 2]), fb.Mesh1D([0, 1]))
        assert g.shape == (3, 2) and len(g) == 6

    def test_error_hierarchy(self):
        assert issubclass(errors.DuplicateNode, errors.MeshError)
        assert issubclass(errors.DimensionMismatch, errors.ValidationError)
        assert issubclass(errors.ZeroDenominator, errors.FinomError)
        assert issubclass(errors.DeviceError, errors.FinomError)


class TestCadence:  # solver.py:185-192 / test_solver.py:150-170
    def test_check_every(self):
        cfg = fb.SolverConfig(epsilon=0.1, itr_max=20, tol=0.0, check_every=7)
        h = solver.history_from(np.arange(1, 21) * 1.0, 20, False, cfg)
        assert [it for it, _ in h] == [7, 14, 20]

    def test_converged_off_cadence(self):
        cfg = fb.SolverConfig(epsilon=0.1, itr_max=100, tol=1e-3, check_every=10)
        h = solver.history_from(np.arange(1, 101) * 1.0, 23, True, cfg)
        assert [it for it, _ in h] == [10, 20, 23]


def test_dividing_index_matches_brute_force():
    rng = np.random.default_rng(0)
    for _ in range(30):
        x = fb.Mesh1D(np.sort(rng.uniform(0, 1, int(rng.integers(1, 40)))))
        y = fb.Mesh1D(np.sort(rng.uniform(0, 1, int(rng.integers(1, 40)))))
        z = kernel1d.dividing_index(x, y).zeta
        assert z.tolist() == [int(np.sum(y.nodes <= xi)) for xi in x.nodes]


def test_shift_interp_matches_numpy():
    """Host _shift == reference semantics (solver.py:135-153)."""
    w = np.array([0.0, 0.2, 0.0, 0.0, 0.5, 0.3, 0.0])
    s = np.array([9.0, 2.0, 9.0, 9.0, 4.0, 0.5, 9.0])
    eps = 0.1
    out = solver._shift(w, s, eps)
    pos = w > 0
    vals = eps * np.log(s[pos])
    idx = np.arange(7.0)
    want = np.empty(7)
    want[pos] = vals
    want[~pos] = np.interp(idx[~pos], idx[pos], vals)
    assert np.array_equal(out, want)
