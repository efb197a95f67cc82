"""Command-line front end and kernel benchmarks, mirroring
the reference's pkg/tests/test_cli.py and test_bench.py.  Error paths exit
before any device work (CPU); pipeline and benchmark runs need the GPU."""

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2105_12301_b200 as P

ROOT = str(Path(__file__).resolve().parents[1])


def run_cli(*args, env_extra=None):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([ROOT, env.get("PYTHONPATH", "")])
    return subprocess.run([sys.executable, "-m", "paper_2105_12301_b200", *args],
                          capture_output=True, text=True, env={**env, **(env_extra or {})}, timeout=600)


def write_pair_csv(path, length=300, seed=6):
    data = P.coupled_logistic(length, seed=seed, beta=0.3)
    lines = [",".join(data.names)]
    for t in range(data.length):
        lines.append(",".join(repr(float(s.values[t])) for s in data))
    Path(path).write_text("\n".join(lines) + "\n")


# ---------------------------------------------------------------- CPU: argument / input errors
def test_missing_input_file(tmp_path):
    r = run_cli("--input", str(tmp_path / "nope.csv"), "--output", str(tmp_path / "out.csv"))
    assert r.returncode == 2 and r.stderr.startswith("error:")
    assert len(r.stderr.strip().split("\n")) == 1


def test_bad_csv(tmp_path):
    src = tmp_path / "in.csv"
    src.write_text("a,b\n1,2\n3,oops\n")
    r = run_cli("--input", str(src), "--output", str(tmp_path / "out.csv"))
    assert r.returncode == 2 and "column 'b'" in r.stderr


def test_missing_required_flags():
    r = run_cli()
    assert r.returncode == 2 and "--input and --output" in r.stderr


def test_desk_bound_without_override():
    r = run_cli("--bench", "knn", "--length", "20000", "--erange", "1:1")
    assert r.returncode == 2 and "desk-scale" in r.stderr


def test_bad_erange():
    r = run_cli("--bench", "knn", "--length", "300", "--erange", "oops")
    assert r.returncode == 2 and "erange" in r.stderr


def test_resolve_workers_precedence(monkeypatch):
    from paper_2105_12301_b200.cli import resolve_workers
    monkeypatch.setenv("CROSSMAP_WORKERS", "7")
    assert resolve_workers(1) == 1 and resolve_workers() == 7
    monkeypatch.setenv("CROSSMAP_WORKERS", "x")
    with pytest.raises(P.ParameterError):
        resolve_workers()


def test_bench_argument_checks():
    with pytest.raises(P.ParameterError):
        P.run_bench("fft")
    with pytest.raises(P.ParameterError):
        P.run_bench("knn", e_range=(3, 2))
    with pytest.raises(P.ParameterError, match="desk-scale"):
        P.run_bench("lookup", count=20000)


# ---------------------------------------------------------------- GPU: pipeline and benchmarks
@pytest.mark.gpu
def test_end_to_end(tmp_path):
    src, dst = tmp_path / "in.csv", tmp_path / "out.csv"
    write_pair_csv(src)
    r = run_cli("--input", str(src), "--output", str(dst), "--emax", "4")
    assert r.returncode == 0, r.stderr
    m = json.loads(r.stdout)
    assert m["n_series"] == 2 and m["series_length"] == 300 and m["e_max"] == 4
    assert m["tables_built"] == 2 * m["distinct_e"] and m["seconds_optimal_e"] >= 0.0
    matrix = P.read_skill_matrix(dst)
    assert matrix.names == ["driver", "response"] and np.all(np.isfinite(matrix.rho))


@pytest.mark.gpu
def test_emit_predictions_writes_npz(tmp_path):
    src, dst = tmp_path / "in.csv", tmp_path / "out.csv"
    write_pair_csv(src, length=250)
    r = run_cli("--input", str(src), "--output", str(dst), "--emax", "3", "--emit-predictions")
    assert r.returncode == 0, r.stderr
    archive = np.load(dst.with_suffix(".predictions.npz"))
    assert "driver->response" in archive.files and len(archive.files) == 4


@pytest.mark.gpu
def test_workers_flag_env_and_same_bytes(tmp_path):
    src = tmp_path / "in.csv"
    write_pair_csv(src, length=250)
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    r1 = run_cli("--input", str(src), "--output", str(a), "--emax", "3", "--workers", "1",
                 env_extra={"CROSSMAP_WORKERS": "7"})
    r2 = run_cli("--input", str(src), "--output", str(b), "--emax", "3", env_extra={"CROSSMAP_WORKERS": "2"})
    assert r1.returncode == 0 and r2.returncode == 0, r1.stderr + r2.stderr
    assert json.loads(r1.stdout)["workers"] == 1 and json.loads(r2.stdout)["workers"] == 2
    assert a.read_bytes() == b.read_bytes()


@pytest.mark.gpu
def test_knn_bench_rows_and_cli(tmp_path):
    rows = P.run_bench("knn", length=500, e_range=(1, 20), seed=7, workers=1)
    assert len(rows) == 40 and [r.e for r in rows if r.phase == "distance"] == list(range(1, 21))
    assert sum(r.phase == "topk" for r in rows) == 20 and all(r.seconds >= 0.0 for r in rows)
    fused = P.run_bench("knn", length=300, e_range=(2, 3), seed=7, fused=True)
    assert [(r.e, r.phase) for r in fused] == [(2, "distance"), (2, "topk"), (2, "fused"),
                                               (3, "distance"), (3, "topk"), (3, "fused")]
    r = run_cli("--bench", "knn", "--length", "300", "--erange", "1:2", "--seed", "9")
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().split("\n")
    assert lines[0] == "E,phase,seconds" and len(lines) == 5


@pytest.mark.gpu
def test_lookup_bench_rows_and_file(tmp_path):
    rows = P.run_bench("lookup", length=300, count=20, e_range=(1, 3), seed=7, workers=1)
    assert [(r.e, r.phase) for r in rows] == [(1, "lookup"), (2, "lookup"), (3, "lookup")]
    out = tmp_path / "bench.csv"
    r = run_cli("--bench", "lookup", "--length", "300", "--count", "10", "--erange", "2:2",
                "--output", str(out))
    assert r.returncode == 0, r.stderr
    assert out.read_text().startswith("E,phase,seconds")
