"""The GPU-backed CLI (paper_1907_01729_b200.cli), following the reference's
CLI tests (pkg/tests/test_cli.py): same subcommands, flags, report schema and
exit codes.  Parse and validation failures happen on the host before any GPU
work, so those cases run on CPU; the solves are marked gpu.
"""

from __future__ import annotations

import json
import math

import numpy as np
import pytest

from paper_1907_01729_b200.cli import main


def write(path, text):
    path.write_text(text, encoding="utf-8")
    return str(path)


def run_cli(capsys, *argv):
    code = main(list(argv))
    captured = capsys.readouterr()
    return code, captured.out, captured.err


def read_report(path):
    with open(path, encoding="utf-8") as fh:
        return json.load(fh)


def _pair(tmp_path, mu="0.5,0.5\n", nu="0.5,0.5\n", cost="0.0,1.0\n1.0,0.0\n"):
    return (write(tmp_path / "mu.csv", mu), write(tmp_path / "nu.csv", nu),
            write(tmp_path / "c.csv", cost))


# ---------------------------------------------------------------------------
# host-side failures (CPU)

def test_compute_mismatched_row_counts(tmp_path, capsys):
    mu, nu, cost = _pair(tmp_path, mu="0.5,0.5\n0.5,0.5\n")
    code, _, err = run_cli(capsys, "compute", "--mu", mu, "--nu", nu, "--cost", cost,
                           "--lambda", "1")
    assert code == 1
    assert "2 rows" in err and "1 rows" in err


def test_compute_parse_error_names_file_row_column(tmp_path, capsys):
    mu, nu, cost = _pair(tmp_path, mu="0.5,0.5\n0.4,oops\n", nu="0.5,0.5\n0.5,0.5\n")
    code, _, err = run_cli(capsys, "compute", "--mu", mu, "--nu", nu, "--cost", cost,
                           "--lambda", "1")
    assert code == 1
    assert "mu.csv" in err and "row 1" in err and "column 1" in err


def test_compute_rejects_invalid_histogram_without_renormalising(tmp_path, capsys):
    mu, nu, cost = _pair(tmp_path, mu="0.5,0.4\n")
    code, _, err = run_cli(capsys, "compute", "--mu", mu, "--nu", nu, "--cost", cost,
                           "--lambda", "1")
    assert code == 1
    assert "row 0" in err and "0.9" in err


def test_compute_negative_mass_names_the_column(tmp_path, capsys):
    mu, nu, cost = _pair(tmp_path, mu="1.5,-0.5\n")
    code, _, err = run_cli(capsys, "compute", "--mu", mu, "--nu", nu, "--cost", cost,
                           "--lambda", "1")
    assert code == 1
    assert "row 0, column 1" in err and "negative" in err


def test_compute_requires_exactly_one_cost_source(tmp_path, capsys):
    mu, nu, cost = _pair(tmp_path)
    code, _, err = run_cli(capsys, "compute", "--mu", mu, "--nu", nu, "--lambda", "1")
    assert code == 1 and "cost" in err
    code, _, err = run_cli(capsys, "compute", "--mu", mu, "--nu", nu, "--cost", cost,
                           "--grid-metric", "2", "--lambda", "1")
    assert code == 1 and "exactly one" in err


def test_compute_json_errors_are_located(tmp_path, capsys):
    bundle = write(tmp_path / "b.json", json.dumps({"mu": [[0.5, "x"]], "nu": [[1.0]]}))
    code, _, err = run_cli(capsys, "compute", "--mu", bundle, "--grid-metric", "2",
                           "--lambda", "1")
    assert code == 1 and "b.json" in err and "row 0" in err and "column 1" in err


def test_gradcheck_needs_instance(capsys):
    code, _, err = run_cli(capsys, "gradcheck", "--lambda", "0.5")
    assert code == 1
    assert "--random" in err


# ---------------------------------------------------------------------------
# solves (GPU)

@pytest.mark.gpu
def test_compute_point_mass_pair(tmp_path, capsys):
    mu, nu, cost = _pair(tmp_path, mu="1.0\n", nu="1.0\n", cost="0.0\n")
    out = tmp_path / "report.json"
    code, _, _ = run_cli(capsys, "compute", "--mu", mu, "--nu", nu, "--cost", cost,
                         "--lambda", "1.0", "--out", str(out))
    assert code == 0
    report = read_report(out)
    assert report["schema"] == 1
    assert report["cost_e0"] == [0.0]
    assert report["converged"] == [True]
    assert report["backend"]["path"] == "fp64"


@pytest.mark.gpu
@pytest.mark.parametrize("precision,tol,atol", [("fp64", "1e-12", 1e-9), ("fp32", "0", 1e-6)])
def test_compute_symmetric_closed_form(tmp_path, capsys, precision, tol, atol):
    mu, nu, cost = _pair(tmp_path)
    out = tmp_path / "report.json"
    code, _, _ = run_cli(capsys, "compute", "--mu", mu, "--nu", nu, "--cost", cost,
                         "--lambda", "1", "--max-iters", "2000", "--tol", tol, "--out", str(out),
                         "--precision", precision)
    assert code == 0
    expected = math.exp(-1.0) / (1.0 + math.exp(-1.0))
    assert read_report(out)["cost_e0"][0] == pytest.approx(expected, abs=atol)


@pytest.mark.gpu
def test_compute_json_bundle_input(tmp_path, capsys):
    bundle = write(tmp_path / "instance.json", json.dumps(
        {"mu": [[0.5, 0.5]], "nu": [[0.5, 0.5]], "cost": [[0.0, 1.0], [1.0, 0.0]]}))
    out = tmp_path / "report.json"
    code, _, _ = run_cli(capsys, "compute", "--mu", bundle, "--lambda", "1", "--out", str(out))
    assert code == 0
    expected = math.exp(-1.0) / (1.0 + math.exp(-1.0))
    assert read_report(out)["cost_e0"][0] == pytest.approx(expected, abs=1e-9)


@pytest.mark.gpu
def test_compute_exit_two_on_non_convergence(tmp_path, capsys):
    mu, nu, cost = _pair(tmp_path, mu="0.3,0.7\n", nu="0.6,0.4\n")
    out = tmp_path / "report.json"
    code, _, _ = run_cli(capsys, "compute", "--mu", mu, "--nu", nu, "--cost", cost,
                         "--lambda", "1", "--max-iters", "1", "--tol", "1e-14", "--out", str(out))
    assert code == 2
    assert read_report(out)["converged"] == [False]


@pytest.mark.gpu
def test_compute_emits_requested_artifacts(tmp_path, capsys):
    mu, nu, cost = _pair(tmp_path)
    out = tmp_path / "report.json"
    code, _, _ = run_cli(capsys, "compute", "--mu", mu, "--nu", nu, "--cost", cost,
                         "--lambda", "1", "--out", str(out),
                         "--emit-plan", "--emit-gradients", "--emit-potentials")
    assert code == 0
    report = read_report(out)
    plan = np.asarray(report["plans"][0])
    assert plan.shape == (2, 2)
    assert plan.sum() == pytest.approx(1.0, abs=1e-9)
    assert np.asarray(report["gradients"]["mu"]).shape == (1, 2)
    assert abs(sum(report["gradients"]["mu"][0])) < 1e-12
    assert np.asarray(report["potentials"]["log_u"]).shape == (1, 2)


@pytest.mark.gpu
def test_compute_potentials_encode_neg_inf_as_null(tmp_path, capsys):
    mu, nu, cost = _pair(tmp_path, mu="0.0,1.0\n")
    out = tmp_path / "report.json"
    code, _, _ = run_cli(capsys, "compute", "--mu", mu, "--nu", nu, "--cost", cost,
                         "--lambda", "1", "--out", str(out), "--emit-potentials")
    assert code == 0
    report = read_report(out)
    assert report["potentials"]["log_u"][0][0] is None
    assert isinstance(report["potentials"]["log_u"][0][1], float)


@pytest.mark.gpu
def test_compute_reports_are_deterministic_and_match_the_oracle(tmp_path, capsys):
    from oracle import sinkhorn_oracle as orc

    mu_t, nu_t = "0.25,0.25,0.5\n0.1,0.6,0.3\n", "0.3,0.3,0.4\n0.2,0.2,0.6\n"
    mu = write(tmp_path / "mu.csv", mu_t)
    nu = write(tmp_path / "nu.csv", nu_t)
    out1, out2 = tmp_path / "r1.json", tmp_path / "r2.json"
    argv = ["compute", "--mu", mu, "--nu", nu, "--grid-metric", "2", "--lambda", "0.1",
            "--max-iters", "500", "--tol", "1e-10"]
    assert run_cli(capsys, *argv, "--out", str(out1))[0] == 0
    assert run_cli(capsys, *argv, "--out", str(out2))[0] == 0
    assert out1.read_text() == out2.read_text()
    m = np.array([[0.25, 0.25, 0.5], [0.1, 0.6, 0.3]])
    n = np.array([[0.3, 0.3, 0.4], [0.2, 0.2, 0.6]])
    ref = orc.batch_forward(m, n, orc.index_grid_cost(3), 0.1, max_iters=500, tolerance=1e-10,
                            check_interval=10)
    report = read_report(out1)
    assert report["iterations_run"] == ref.iterations_run
    assert np.abs(np.array(report["cost_e0"]) - ref.cost_e0).max() <= 1e-12


@pytest.mark.gpu
def test_compute_writes_to_stdout_by_default(tmp_path, capsys):
    mu, nu, cost = _pair(tmp_path, mu="1.0\n", nu="1.0\n", cost="0.0\n")
    code, out_text, _ = run_cli(capsys, "compute", "--mu", mu, "--nu", nu, "--cost", cost,
                                "--lambda", "1")
    assert code == 0
    assert json.loads(out_text)["cost_e0"] == [0.0]


@pytest.mark.gpu
def test_gradcheck_reports_errors_and_exits_three(tmp_path, capsys):
    # the multiplier gradient differentiates the regularised objective, the
    # probe the plain transport cost: at this lam the gap exceeds the gate
    out = tmp_path / "report.json"
    code, _, _ = run_cli(capsys, "gradcheck", "--random", "10", "--lambda", "0.05",
                         "--max-iters", "400", "--seed", "7", "--out", str(out))
    report = read_report(out)
    assert code == 3
    assert report["passed"] is False
    assert set(report["max_abs_error"]) == {"mu", "nu"}
    assert report["max_abs_error"]["mu"] > 0


@pytest.mark.gpu
def test_gradcheck_from_files(tmp_path, capsys):
    mu, nu, cost = _pair(tmp_path, mu="0.4,0.6\n")
    out = tmp_path / "report.json"
    code, _, _ = run_cli(capsys, "gradcheck", "--mu", mu, "--nu", nu, "--cost", cost,
                         "--lambda", "0.5", "--max-iters", "500", "--out", str(out))
    assert code in (0, 3)
    assert read_report(out)["d1"] == 2


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_bench_smoke(tmp_path, capsys, precision):
    out = tmp_path / "bench.json"
    code, _, _ = run_cli(capsys, "bench", "--batch", "1", "--random", "2", "--max-iters", "10",
                         "--lambda", "0.5", "--out", str(out), "--precision", precision)
    assert code == 0
    report = read_report(out)
    assert "ratio" in report
    assert report["forward"]["median_s"] > 0
    assert report["worker_determinism_max_dev"] <= 1e-13
    assert report["iterations"] == 10
