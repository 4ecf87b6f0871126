"""The reference's command line on top of the GPU solver (paper_2505_22631_b200/cli.py): report
and CSV schemas, flag plumbing, exit codes 0/1/2/3 -- modelled on the reference's tests/test_cli.py
(schemas :30-36, solve :39-79, exit codes :222-260).  Argument / input errors need no GPU."""
import json

import numpy as np
import pytest

REPORT_KEYS = {"instance", "problem", "n", "edges", "params", "replicas", "workers", "best_objective",
               "satisfied_fraction", "reference", "accuracy_pct", "wall_time_s", "steps", "seed",
               "precision"}          # the reference's keys (cli.py:94-126) + the arithmetic of the run
PARAM_KEYS = {"K", "ks_max", "ks_period", "kn", "h", "t_stop", "n_states", "seed", "batch_size"}


@pytest.fixture()
def files(tmp_path):
    (tmp_path / "tri.gset").write_text("3 3\n1 2 1\n2 3 1\n1 3 1\n")
    (tmp_path / "weighted.gset").write_text("4 4\n1 2 2\n2 3 -1\n3 4 3\n1 4 1\n")
    (tmp_path / "tri.col").write_text("c triangle\np edge 3 3\ne 1 2\ne 2 3\ne 1 3\n")
    (tmp_path / "bad_count.gset").write_text("3 3\n1 2 1\n")
    (tmp_path / "bad_token.gset").write_text("3 1\n1 x 1\n")
    return tmp_path


def run_cli(capsys, *argv):
    from paper_2505_22631_b200.cli import main
    code = main(list(argv))
    cap = capsys.readouterr()
    return code, cap.out, cap.err


# ---- no GPU needed: usage and input errors -------------------------------------------------
def test_usage_errors_exit_1(capsys, files):
    assert run_cli(capsys)[0] == 1                                              # no sub-command
    assert run_cli(capsys, "solve")[0] == 1                                     # missing path
    assert run_cli(capsys, "solve", str(files / "tri.gset"), "--no-such-flag")[0] == 1
    code, _, err = run_cli(capsys, "solve", str(files / "tri.gset"), "--problem", "maxcut", "--colors", "3")
    assert code == 1 and "--colors" in err
    assert run_cli(capsys, "sweep", str(files / "tri.gset"), "--k-range", "1", "--ks-range", "0:1")[0] == 1
    assert run_cli(capsys, "--help")[0] == 0


def test_input_errors_exit_2(capsys, files):
    code, _, err = run_cli(capsys, "solve", str(files / "missing.gset"))
    assert code == 2 and "input error" in err
    assert run_cli(capsys, "solve", str(files / "bad_count.gset"))[0] == 2
    assert run_cli(capsys, "solve", str(files / "bad_token.gset"))[0] == 2
    (files / "m.csv").write_text("path,kind\ntri.gset,maxcut\n")               # manifest without the reference column
    assert run_cli(capsys, "bench", str(files / "m.csv"))[0] == 2


# ---- on the GPU ---------------------------------------------------------------------------
@pytest.mark.gpu
def test_solve_triangle_maxcut_report(capsys, files):
    code, out, _ = run_cli(capsys, "solve", str(files / "tri.gset"), "--problem", "maxcut", "--seed", "7", "--replicas", "4",
                           "--t-stop", "30")
    assert code == 0
    report = json.loads(out)
    assert report["best_objective"] == 2.0 and report["problem"] == "maxcut"
    assert set(report) == REPORT_KEYS and set(report["params"]) == PARAM_KEYS
    assert report["precision"] == "f32"              # the package default, stated in the report
    assert report["steps"] == 3000 and report["replicas"] == 4


@pytest.mark.gpu
def test_solve_flag_overrides_and_reproducibility(capsys, files):
    args = ("solve", str(files / "weighted.gset"), "--K", "0.7", "--ks-max", "3.0", "--ks-period", "2.5", "--kn", "0.05",
            "--h", "0.02", "--t-stop", "12", "--seed", "9", "--batch-size", "32", "--reference", "5")
    code, out, _ = run_cli(capsys, *args)
    assert code == 0
    first = json.loads(out)
    assert first["params"] == {"K": 0.7, "ks_max": 3.0, "ks_period": 2.5, "kn": 0.05, "h": 0.02, "t_stop": 12.0,
                               "n_states": 2, "seed": 9, "batch_size": 32}
    second = json.loads(run_cli(capsys, *args)[1])
    assert first["best_objective"] == second["best_objective"] == 5.0        # the optimum: 2 + 3 with the -1 edge uncut, or 2 - 1 + 3 + 1
    assert first["accuracy_pct"] == 100.0


@pytest.mark.gpu
def test_solve_coloring_and_trace(capsys, files):
    trace = files / "trace.csv"
    code, out, _ = run_cli(capsys, "solve", str(files / "tri.col"), "--problem", "coloring", "--colors", "3", "--seed", "1",
                           "--t-stop", "30", "--trace", str(trace))
    assert code == 0
    report = json.loads(out)
    assert report["problem"] == "coloring" and report["satisfied_fraction"] == 1.0 and report["best_objective"] == 0.0
    rows = trace.read_text().splitlines()
    assert rows[0] == "t,energy,ks,best_objective" and len(rows) >= 3
    t = [float(r.split(",")[0]) for r in rows[1:]]
    assert t[0] == 0.0 and all(b > a for a, b in zip(t, t[1:]))


@pytest.mark.gpu
def test_bench_manifest_table(capsys, files):
    (files / "m.csv").write_text("# two instances\npath,kind,reference,colors,replicas\ntri.gset,maxcut,2,,2\ntri.col,coloring,0,3,2\n"
                                 "missing.gset,maxcut,1,,\n")
    code, out, err = run_cli(capsys, "bench", str(files / "m.csv"), "--t-stop", "20", "--json")
    doc = json.loads(out)
    rows, agg = doc["rows"], doc["aggregate"]
    assert agg["instances"] == 3 and agg["failures"] == 1 and agg["min_accuracy_pct"] == 100.0
    assert [r["instance"] for r in rows] == ["tri.gset", "tri.col", "missing.gset"]
    assert rows[0]["best_objective"] == 2.0 and rows[0]["accuracy_pct"] == 100.0
    assert rows[1]["satisfied_fraction"] == 1.0
    assert rows[2]["error"] and code == 2                                      # a failed row is recorded, the rest still run


@pytest.mark.gpu
def test_sweep_and_scaling_schemas(capsys, files):
    code, out, _ = run_cli(capsys, "sweep", str(files / "tri.gset"), "--k-range", "0.5:1.0", "--ks-range", "1:2", "--grid", "2x2",
                           "--replicas", "4", "--t-stop", "10", "--reference", "2")
    assert code == 0
    rows = out.strip().splitlines()
    assert rows[0] == "K,ks_max,accuracy" and len(rows) == 5
    assert all(0.0 <= float(r.split(",")[2]) <= 100.0 for r in rows[1:])
    code, out, _ = run_cli(capsys, "scaling", "--sizes", "64,128", "--steps", "20")
    assert code == 0
    rows = out.strip().splitlines()
    assert rows[0] == "n,workers,wall_time_s" and [r.split(",")[0] for r in rows[1:]] == ["64", "64", "128", "128"]   # workers = 1 and = --workers, like the reference


@pytest.mark.gpu
def test_numerical_failure_exit_3(capsys, files):
    (files / "huge.gset").write_text("2 1\n1 2 1e200\n")           # the overflow of the reference's own test (test_dynamics.py:186-192)
    code, _, err = run_cli(capsys, "solve", str(files / "huge.gset"), "--K", "1e200", "--ks-max", "0", "--ks-period", "10",
                           "--kn", "0", "--h", "1", "--t-stop", "3", "--precision", "f64")
    assert code == 3 and "oscillator" in err and "step" in err
