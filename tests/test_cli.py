"""The command-line harness (paraode_b200/cli.py), restating the reference's
CLI tests (proj/tests/test_cli.cpp:40-170): CSV schema, chart, argument
errors and exit codes on CPU; solve / benchmark / compare on the GPU."""
import json
import math

import numpy as np
import pytest

from paraode_b200 import cli


def test_methods_and_unknowns():  # test_cli.cpp:40-45
    assert cli.METHODS == ("paraieks", "paraieks-elements", "ieks", "eks")
    with pytest.raises(cli.UsageError):
        cli._solver("rk45")
    with pytest.raises(cli.UsageError):
        cli._solver("seq")


def test_csv_schema_is_stable():  # test_cli.cpp:47-72
    assert cli.RUN_RECORD_HEADER == ("problem,method,nu,grid_size,rmse,runtime_seconds,iterations,sigma_hat,"
                                     "converged,combine_invocations,sequential_depth")
    rec = dict(problem="logistic", method="paraieks", nu=2, grid_size=32, rmse=0.5, runtime_seconds=0.25,
               iterations=7, sigma_hat=4.0, converged=True, combine_invocations=62, sequential_depth=10)
    assert cli.csv_row(rec) == "logistic,paraieks,2,32,0.5,0.25,7,4,true,62,10"
    rec.update(rmse=None, converged=False)
    assert cli.csv_row(rec) == "logistic,paraieks,2,32,,0.25,7,4,false,62,10"
    assert cli.to_csv([rec]) == cli.RUN_RECORD_HEADER + "\n" + cli.csv_row(rec) + "\n"


def test_chart_tolerates_empty_and_partial_input():  # test_cli.cpp:74-93
    assert cli.to_svg([]).startswith("<svg")
    rec = dict(problem="logistic", method="paraieks", nu=1, grid_size=16, rmse=None, runtime_seconds=0.5)
    assert cli.to_svg([rec]).startswith("<svg")
    rec["rmse"] = 1e-3
    rec2 = dict(rec, grid_size=32, rmse=1e-4, runtime_seconds=1.0)
    svg = cli.to_svg([rec, rec2])
    assert svg.startswith("<svg") and "polyline" in svg and "logistic" in svg


@pytest.mark.parametrize("argv", [["solve", "--problem", "logistic", "--n", "1"], ["solve", "--problem", "nosuch"],
                                  ["solve", "--problem", "logistic", "--nu", "9"], ["--bogus-flag"], [],
                                  ["benchmark", "--repeats", "0"], ["solve", "--method", "rk45"]])
def test_solve_rejects_unusable_arguments(argv):  # test_cli.cpp:128-134
    assert cli.main(argv) == 1


@pytest.mark.gpu
def test_solve_eks_method(tmp_path):  # bench.cpp:139 (Method::kEks): one pass, converged, exit 0
    out = tmp_path / "eks.json"
    assert cli.main(["solve", "--problem", "logistic", "--method", "eks", "--n", "30", "--nu", "2",
                     "--out", str(out)]) == 0
    doc = json.loads(out.read_text())
    assert doc["method"] == "eks" and doc["iterations"] == 1 and doc["converged"] is True
    assert len(doc["objective_trace"]) == 1 and math.isclose(doc["mean"][30][0], 0.9955, rel_tol=1e-2)


@pytest.mark.gpu
def test_ieks_method_matches_paraieks():  # acceptance.cpp:97-123: seq and par agree, equal iterations
    import paraode_b200 as P
    import _oracle as O
    for name, nu, n in (("logistic", 2, 60), ("vanderpol", 2, 200), ("fhn", 2, 300)):
        prob = P.problem_by_name(name)
        prior = P.IwpPrior(nu, prob.dim, 1.0)
        grid = P.uniform_grid(prob.t_end, n)
        seq = cli._solver("ieks")(prob, prior, grid, P.IeksConfig())
        par = cli._solver("paraieks")(prob, prior, grid, P.IeksConfig())
        want = O.ieks(O.problem(name), nu, grid, mode=0)
        assert seq.iterations == par.iterations == want["iterations"]
        assert np.max(np.abs(seq.means - par.means)) <= 1e-8 * max(1.0, np.max(np.abs(par.means)))
        assert np.max(np.abs(seq.means - want["means"])) <= 1e-9 * max(1.0, np.max(np.abs(want["means"])))


@pytest.mark.gpu
def test_solve_writes_a_report(tmp_path):  # test_cli.cpp:95-116
    out = tmp_path / "solve.json"
    assert cli.main(["solve", "--problem", "logistic", "--n", "30", "--nu", "2", "--out", str(out)]) == 0
    doc = json.loads(out.read_text())
    assert doc["problem"] == "logistic" and doc["method"] == "paraieks" and doc["nu"] == 2
    assert doc["grid_size"] == 30 and len(doc["grid"]) == 31 and len(doc["mean"]) == 31 and len(doc["std"]) == 31
    assert doc["converged"] is True and doc["sigma_hat"] > 0.0 and doc["iterations"] >= 2
    assert len(doc["objective_trace"]) == doc["iterations"]
    assert math.isclose(doc["mean"][30][0], 0.9955, rel_tol=1e-2)


@pytest.mark.gpu
def test_solve_identical_across_worker_counts(tmp_path):  # test_cli.cpp:118-126
    a, b = tmp_path / "w1.json", tmp_path / "w4.json"
    assert cli.main(["solve", "--problem", "vanderpol", "--n", "25", "--workers", "1", "--out", str(a)]) == 0
    assert cli.main(["solve", "--problem", "vanderpol", "--n", "25", "--workers", "4", "--out", str(b)]) == 0
    assert a.read_text() == b.read_text()


@pytest.mark.gpu
def test_exhausted_budget_exit_code(tmp_path):  # test_cli.cpp:136-144
    out = tmp_path / "budget.json"
    assert cli.main(["solve", "--problem", "vanderpol", "--n", "40", "--max-iterations", "1", "--out", str(out)]) == 2
    doc = json.loads(out.read_text())
    assert doc["converged"] is False and doc["iterations"] == 1


@pytest.mark.gpu
def test_benchmark_emits_csv_and_chart(tmp_path):  # test_cli.cpp:146-165
    csv, svg = tmp_path / "bench.csv", tmp_path / "bench.svg"
    assert cli.main(["benchmark", "--problems", "logistic", "--methods", "paraieks", "--nu", "1", "--grid-sizes",
                     "16,32", "--repeats", "1", "--out", str(csv), "--svg", str(svg)]) == 0
    lines = [x for x in csv.read_text().split("\n") if x]
    assert lines[0] == cli.RUN_RECORD_HEADER
    assert len(lines) == 3 and all(x.startswith("logistic,paraieks,") for x in lines[1:])
    assert all(x.split(",")[4] != "" for x in lines[1:])  # rmse present
    assert svg.read_text().startswith("<svg")


@pytest.mark.gpu
def test_benchmark_rk4_reference_accuracy(tmp_path):
    """RK4 reference tables (GPU) for the non-closed-form problems: the IEKS
    error shrinks with the grid (accuracy-order sanity)."""
    csv = tmp_path / "b.csv"
    assert cli.main(["benchmark", "--problems", "vanderpol", "--nu", "2", "--grid-sizes", "64,256", "--repeats",
                     "1", "--out", str(csv)]) == 0
    rows = [x.split(",") for x in csv.read_text().split("\n")[1:] if x]
    e64, e256 = float(rows[0][4]), float(rows[1][4])
    assert 0 < e256 < e64 / 4


@pytest.mark.gpu
def test_compare_validates_agreement():  # test_cli.cpp:167-170
    assert cli.main(["compare", "--problems", "logistic"]) == 0
    assert cli.main(["compare", "--problems", "logistic", "--tolerance", "0"]) == 1


def _rk4_numpy(f, y0, t_end, steps):
    """Classical RK4 (an independent host restatement of problems.cpp:11-27)."""
    y = np.array(y0, dtype=np.float64)
    h = t_end / steps
    out = [y.copy()]
    for _ in range(steps):
        k1 = f(y)
        k2 = f(y + 0.5 * h * k1)
        k3 = f(y + 0.5 * h * k2)
        k4 = f(y + h * k3)
        y = y + (h / 6.0) * (((k1 + 2.0 * k2) + 2.0 * k3) + k4)
        out.append(y.copy())
    return np.array(out)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["fhn", "vanderpol", "rigidbody"])
def test_gpu_rk4_table_matches_independent_rk4(name):
    """pode_rk4_table (k_rk4) against an independent numpy RK4 on the same
    steps, and the refined reference of the benchmark harness: at a fine
    grid the RMSE is no longer floored by the 32768-step table."""
    import paraode_b200 as P
    from paraode_b200.accuracy import reference_for, rk4_table
    fields = {
        "fhn": lambda y: np.array([3.0 * ((y[0] - y[0] ** 3 / 3.0) + y[1]), ((y[0] - 0.2) + 0.2 * y[1]) * (-1.0 / 3.0)]),
        "vanderpol": lambda y: np.array([y[1], 1.0 * ((1.0 - y[0] * y[0]) * y[1] - y[0])]),
        "rigidbody": lambda y: np.array([-2.0 * (y[1] * y[2]), 1.25 * (y[0] * y[2]), -0.5 * (y[0] * y[1])]),
    }
    prob = P.problem_by_name(name)
    got = rk4_table(prob, 4096)
    want = _rk4_numpy(fields[name], prob.y0, prob.t_end, 4096)
    assert np.max(np.abs(got - want)) <= 1e-12 * max(1.0, np.abs(want).max())
    n = 2 ** 16  # a grid finer than the reference's fixed 32768-step table
    grid = P.uniform_grid(prob.t_end, n)
    ref = reference_for(name, grid_steps=n)
    table = rk4_table(prob, 2 * n)[::2]  # Rk4Reference keeps the step-halved table
    assert np.array_equal(np.array([ref(float(t)) for t in grid[:: n // 64]]), table[:: n // 64])
