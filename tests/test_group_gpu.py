"""The group solve (k_solve_group: one persistent kernel, a group of warps per
problem) against the reference fixtures and the oracle, at every group
width.  The default dispatch picks it for large batches (config 5); these
tests force it (FB_GROUP=1, FB_GROUP_W=g) on the small cases the
tile-parallel loop is checked on."""

import numpy as np
import pytest

import paper_2605_26659_b200 as fb
from paper_2605_26659_b200 import workloads as W

import test_parity_gpu as T
from conftest import rel_inf

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["1", "2", "4", "16"])
def group(monkeypatch, request):
    monkeypatch.setenv("FB_GROUP", "1")
    monkeypatch.setenv("FB_GROUP_W", request.param)
    return int(request.param)


def test_group_solver_cases_vs_reference(group):
    T.test_solver_cases_vs_reference()


def test_group_failure_diagnostics(group):
    T.test_failure_diagnostics()


def test_group_config5_subset_vs_reference(group):
    T.test_config5_subset_batched_vs_reference()


def test_group_mixed_sizes_vs_oracle(group):
    T.test_batched_mixed_sizes_vs_oracle()


def test_group_many_problems_vs_oracle(group):
    T.test_batched_many_problems_vs_oracle()


@pytest.mark.parametrize("g", ["1", "4"])
def test_group_tol_stops_per_problem(monkeypatch, g):
    monkeypatch.setenv("FB_GROUP", "1")
    monkeypatch.setenv("FB_GROUP_W", g)
    T.test_batched_tol_stops_per_problem(monkeypatch, "1")


def test_group_config1_vs_reference(group):
    T.test_config1_vs_reference()


def test_group_matches_tile_parallel_loop(monkeypatch):
    """Same batch through both loops: identical iteration counts and absorb
    iterations, results within the parity tolerance, and the group solve
    bitwise reproducible run to run."""
    probs = W.config5(problems=range(6), n=4096)
    cfg = fb.SolverConfig(epsilon=1.0, itr_max=80, tol=0.0, stabilize=True)
    args = ([fb.Mesh1D(p[0]) for p in probs], [fb.Mesh1D(p[1]) for p in probs],
            [fb.Measure(p[2]) for p in probs], [fb.Measure(p[3]) for p in probs], cfg)
    eps = [p[4] for p in probs]
    monkeypatch.setenv("FB_GROUP", "0")
    ref = fb.sinkhorn_1d_batched(*args, epsilons=eps)
    monkeypatch.setenv("FB_GROUP", "1")
    for g in ("1", "2"):
        monkeypatch.setenv("FB_GROUP_W", g)
        a = fb.sinkhorn_1d_batched(*args, epsilons=eps)
        b = fb.sinkhorn_1d_batched(*args, epsilons=eps)
        for sa, sb, sr in zip(a, b, ref):
            assert np.array_equal(sa.phi, sb.phi) and np.array_equal(sa.psi, sb.psi)
            assert sa.iterations_run == sr.iterations_run
            assert list(sa.absorb_iterations) == list(sr.absorb_iterations)
            assert rel_inf(sa.phi, sr.phi) < 1e-10 and rel_inf(sa.psi, sr.psi) < 1e-10
            assert abs(sa.cost - sr.cost) <= 1e-10 * abs(sr.cost)


@pytest.fixture
def cluster(monkeypatch):
    """The cluster form (a thread-block cluster per problem) on small problems."""
    monkeypatch.setenv("FB_GROUP", "0")
    monkeypatch.setenv("FB_CLUSTER", "1")


def test_cluster_solver_cases_vs_reference(cluster):
    T.test_solver_cases_vs_reference()


def test_cluster_failure_diagnostics(cluster):
    T.test_failure_diagnostics()


def test_cluster_config1_vs_reference(cluster):
    T.test_config1_vs_reference()


def test_cluster_mixed_sizes_vs_oracle(cluster):
    T.test_batched_mixed_sizes_vs_oracle()


def test_cluster_tol_stops_per_problem(monkeypatch):
    monkeypatch.setenv("FB_GROUP", "0")
    monkeypatch.setenv("FB_CLUSTER", "1")
    T.test_batched_tol_stops_per_problem(monkeypatch, "1")
