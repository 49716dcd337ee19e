"""CLI harness and JSON v1 problem files (SPEC.md cli; mesh.py:164-353).
CPU: generators, file round trips, usage errors.  GPU: solve / compare /
bench through the B200 path."""

import json
import subprocess
import sys

import numpy as np
import pytest

from paper_2605_26659_b200 import cli
from paper_2605_26659_b200 import problem_io as io
from paper_2605_26659_b200.errors import ConfigError, DimensionMismatch, ParseError

from conftest import ROOT


def test_chebyshev_nodes():
    m = io.chebyshev_nodes(7)
    z = m.nodes
    assert np.all(np.diff(z) > 0) and 0 < z[0] and z[-1] < 1
    assert np.allclose(z + z[::-1], 1.0)  # symmetric about 1/2
    k = np.arange(1, 8)
    assert np.array_equal(z, (0.5 + 0.5 * np.cos((2 * k - 1) * np.pi / 14))[::-1])


def test_generators_reproducible():
    a, b = io.generate(1, "random", 50, seed=3), io.generate(1, "random", 50, seed=3)
    assert np.array_equal(a.source.nodes, b.source.nodes)
    assert np.array_equal(a.u.weights, b.u.weights)
    assert abs(a.u.weights.sum() - 1) < 1e-12
    g = io.generate(2, "chebyshev", 6, 5, seed=1)
    assert g.dim == 2 and g.source.shape == (6, 5) and g.u.weights.shape == (6, 5)
    with pytest.raises(ConfigError):
        io.generate(1, "random", 0)


@pytest.mark.parametrize("dim", [1, 2])
def test_json_round_trip_exact(tmp_path, dim):
    p = io.generate(dim, "random", 9, 7, seed=11)
    f = tmp_path / "p.json"
    io.save_problem(p, f)
    doc = json.loads(f.read_text())
    assert doc["schema_version"] == 1 and doc["dim"] == dim
    q = io.load_problem(f)
    for attr in ("u", "v"):
        assert np.array_equal(getattr(p, attr).weights, getattr(q, attr).weights)
    if dim == 1:
        assert np.array_equal(p.source.nodes, q.source.nodes)
    else:
        assert np.array_equal(p.target.y_nodes.nodes, q.target.y_nodes.nodes)
    io.save_problem_csv(p, tmp_path / "p.csv")
    rows = (tmp_path / "p.csv").read_text().splitlines()
    assert len(rows) == 1 + (18 if dim == 1 else 2 * 63)


def test_load_errors(tmp_path):
    bad = tmp_path / "bad.json"
    bad.write_text("{not json")
    with pytest.raises(ParseError):
        io.load_problem(bad)
    bad.write_text(json.dumps({"dim": 3}))
    with pytest.raises(ParseError):
        io.load_problem(bad)
    bad.write_text(json.dumps({"dim": 1, "x1": [0, 1], "x2": [0, 1], "u": [0.5, 0.5]}))
    with pytest.raises(ParseError):
        io.load_problem(bad)
    bad.write_text(json.dumps({"dim": 1, "x1": [0, 1], "x2": [0, 1], "u": [1.0], "v": [1, 1]}))
    with pytest.raises(DimensionMismatch):
        io.load_problem(bad)
    # weights off unit mass are normalized by their sum
    ok = tmp_path / "ok.json"
    ok.write_text(json.dumps({"dim": 1, "x1": [0, 1], "x2": [0, 1], "u": [1, 3], "v": [2, 2]}))
    assert np.array_equal(io.load_problem(ok).u.weights, [0.25, 0.75])


def test_cli_usage_errors(tmp_path):
    run = lambda *a: subprocess.run([sys.executable, "-m", "paper_2605_26659_b200.cli", *a],
                                    cwd=ROOT, capture_output=True, text=True)
    assert run("gen", "--dim", "1", "--n", "0", "-o", str(tmp_path / "x.json")).returncode != 0
    assert run("solve").returncode != 0  # no input, no generator spec
    assert run("bogus").returncode != 0
    r = run("gen", "--dim", "1", "--nodes", "chebyshev", "--n", "100", "--seed", "5", "-o",
            str(tmp_path / "p.json"))
    assert r.returncode == 0 and io.load_problem(tmp_path / "p.json").dim == 1
    with pytest.raises(Exception):
        cli._fit([1000], [1.0])


@pytest.mark.gpu
def test_cli_solve_and_compare_1d(tmp_path):
    out = tmp_path / "r.json"
    assert cli.main(["solve", "--dim", "1", "--nodes", "chebyshev", "--n", "500", "--eps",
                     "0.01", "--iters", "1000", "--seed", "1", "-o", str(out)]) == 0
    rep = json.loads(out.read_text())
    assert rep["result"]["iterations"] == 1000 and np.isfinite(rep["result"]["cost"])
    assert cli.main(["compare", "--dim", "1", "--nodes", "random", "--n", "500", "--eps", "0.01",
                     "--iters", "1000", "--trials", "1", "-o", str(out)]) == 0
    rep = json.loads(out.read_text())
    assert rep["frobenius_plan_diff"] <= 1e-12 and rep["speedup"] > 0
    assert rep["finom"]["iterations"] == rep["dense"]["iterations"] == 1000


@pytest.mark.gpu
def test_cli_compare_2d_and_tol(tmp_path):
    out = tmp_path / "r.json"
    assert cli.main(["compare", "--dim", "2", "--n", "20", "--m", "20", "--eps", "0.05",
                     "--iters", "200", "--trials", "1", "-o", str(out)]) == 0
    assert json.loads(out.read_text())["frobenius_plan_diff"] <= 1e-12
    p = tmp_path / "p.json"
    assert cli.main(["gen", "--dim", "1", "--n", "300", "--seed", "2", "-o", str(p)]) == 0
    assert cli.main(["solve", "--input", str(p), "--eps", "0.05", "--iters", "5000", "--tol",
                     "1e-9", "-o", str(out)]) == 0
    rep = json.loads(out.read_text())
    assert rep["result"]["converged"] and rep["result"]["last_history_error"] <= 1e-9


@pytest.mark.gpu
def test_cli_bench_fit_and_time_to_error(tmp_path):
    out = tmp_path / "b.json"
    assert cli.main(["bench", "--solver", "both", "--sizes", "250,500,1000,2000", "--iters",
                     "100", "--trials", "1", "--csv", str(tmp_path / "b.csv"), "-o",
                     str(out)]) == 0
    rep = json.loads(out.read_text())
    assert set(rep["fits"]) == {"finom", "dense"} and len(rep["rows"]) == 8
    assert all(np.isfinite(f["exponent"]) for f in rep["fits"].values())
    assert cli.main(["bench", "--time-to-error", "--n", "400", "--eps-list", "0.1",
                     "--thresholds", "1e-4,1e-6", "--iters", "3000", "-o", str(out)]) == 0
    rows = json.loads(out.read_text())["rows"]
    assert [r["threshold"] for r in rows] == [1e-4, 1e-6] and all(r["reached"] for r in rows)
    assert rows[0]["iterations"] <= rows[1]["iterations"]
