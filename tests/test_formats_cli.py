"""File formats, CLI and grid harness vs the reference's own outputs.

Golden values: tests/golden/io_golden.json, produced by the unmodified
reference (`hadamard_ga.io` / `cli` / `bench`) with
tests/golden/make_io_golden.py.  CPU tests cover everything that does not
launch a kernel (text formats, record/trace files, summaries, usage errors,
`verify` with the host Gram, `sylvester`, grid tables); the `gpu` tests run
`search` / `bench grid` with the reference's random streams and must print
the reference's records.
"""

from __future__ import annotations

import contextlib
import io as stdio
import json
import re
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2208_14961_b200 import bench as hbench
from paper_2208_14961_b200 import cli, io
from paper_2208_14961_b200.engine import GAConfig, RunRecord

GOLDEN = json.loads((Path(__file__).parent / "golden" / "io_golden.json").read_text(encoding="utf-8"))
TIME_RE = re.compile(r"in \d+\.\d+s")


def run_cli(argv, stdin_text=None):
    out, err = stdio.StringIO(), stdio.StringIO()
    old = sys.stdin
    if stdin_text is not None:
        sys.stdin = stdio.StringIO(stdin_text)
    try:
        with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
            code = cli.main(argv)
    finally:
        sys.stdin = old
    return code, TIME_RE.sub("in <T>s", out.getvalue()), err.getvalue()


def record_from_golden(r: dict, wall: float = 0.0, complete=None) -> RunRecord:
    cfg = GAConfig(rng="reference", **r["config"])
    return RunRecord(config=cfg, seed=r["seed"], success=r["success"],
                     complete=r["complete"] if complete is None else complete, iterations=r["iterations"],
                     best_fitness=r["best_fitness"], best_matrix=np.array(r["best_matrix"], dtype=np.int8),
                     trace=list(r["trace"]), wall_seconds=wall)


# ------------------------------------------------------------------ matrix text


@pytest.mark.parametrize("case", GOLDEN["matrices"], ids=lambda c: f"m{len(c['matrix'])}")
def test_write_matrix_matches_reference(case):
    q = np.array(case["matrix"], dtype=np.int8)
    assert io.write_matrix(q) == case["text"]
    assert np.array_equal(io.parse_matrix(case["text"]), q)


@pytest.mark.parametrize("case", GOLDEN["parse_cases"], ids=lambda c: repr(c["text"][:24]))
def test_parse_errors_match_reference(case):
    if case["error"] is None:
        assert np.array_equal(io.parse_matrix(case["text"]), np.array(case["matrix"], dtype=np.int8))
        return
    with pytest.raises(io.MatrixFormatError) as ei:
        io.parse_matrix(case["text"])
    assert str(ei.value) == case["error"]
    assert (ei.value.line, ei.value.column) == (case["line"], case["column"])
    assert isinstance(ei.value, ValueError)


def test_matrix_file_roundtrip(tmp_path):
    q = np.where(np.random.default_rng(1).random((36, 36)) < 0.5, 1, -1).astype(np.int8)
    io.save_matrix(q, tmp_path / "q.txt")
    assert np.array_equal(io.load_matrix(tmp_path / "q.txt"), q)
    with pytest.raises(ValueError):
        io.write_matrix(np.zeros((3, 3), dtype=np.int8))


# ------------------------------------------------------------------ records, traces, summaries


@pytest.mark.parametrize("r", GOLDEN["records"], ids=lambda r: f"m{r['config']['order']}")
def test_run_record_document_matches_reference(r, tmp_path):
    rec = record_from_golden(r)
    doc = io.run_record_doc(rec, trace_path="trace.csv")
    assert doc["config"].pop("rng") == "reference"
    assert doc == r["doc"]
    io.write_run_record(rec, tmp_path / "rec.json", trace_path="trace.csv")
    ours = (tmp_path / "rec.json").read_text(encoding="ascii")
    assert "\n".join(ln for ln in ours.splitlines() if '"rng":' not in ln) == r["record_text"].rstrip("\n")
    loaded, q = io.load_run_record(tmp_path / "rec.json")
    assert loaded["iterations"] == r["iterations"] and np.array_equal(q, rec.best_matrix)


@pytest.mark.parametrize("r", GOLDEN["records"], ids=lambda r: f"m{r['config']['order']}")
def test_trace_and_summary_match_reference(r, tmp_path):
    io.write_trace(r["trace"], tmp_path / "t.csv")
    assert (tmp_path / "t.csv").read_bytes().decode("ascii") == r["trace_bytes"]
    assert io.read_trace(tmp_path / "t.csv") == list(enumerate(r["trace"]))
    assert io.format_summary(record_from_golden(r)) == r["summary"]
    assert io.format_summary(record_from_golden(r, wall=12.3456, complete=False)) == r["summary_budget"]


def test_trace_rejects_rise_and_bad_header(tmp_path):
    with pytest.raises(ValueError, match="rises at iteration 2"):
        io.write_trace([5, 3, 4], tmp_path / "t.csv")
    (tmp_path / "bad.csv").write_text("it,fit\n0,1\n")
    with pytest.raises(ValueError, match="unexpected trace header"):
        io.read_trace(tmp_path / "bad.csv")


def test_load_record_rejects_false_success(tmp_path):
    r = GOLDEN["records"][0]
    assert r["success"]
    doc = dict(r["doc"])
    doc["matrix"] = GOLDEN["cli_verify_input"]  # a non-Hadamard order-8 matrix
    (tmp_path / "rec.json").write_text(json.dumps(doc))
    with pytest.raises(ValueError, match="fails verification"):
        io.load_run_record(tmp_path / "rec.json")


# ------------------------------------------------------------------ CLI


def _cli_cases(kind):
    return [c for c in GOLDEN["cli"] if c["argv"][0] == kind]


@pytest.mark.parametrize("case", _cli_cases("sylvester") + _cli_cases("verify"), ids=lambda c: " ".join(c["argv"]))
def test_cli_host_commands_match_reference(case, monkeypatch):
    import torch

    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)  # host Gram only
    stdin = case["stdin"]
    code, out, err = run_cli(case["argv"], stdin)
    assert code == case["code"]
    assert out == case["stdout"]
    assert err == case["stderr"]


@pytest.mark.parametrize("case", [c for c in _cli_cases("search") if c["code"] == 1], ids=lambda c: " ".join(c["argv"]))
def test_cli_usage_errors_match_reference(case):
    code, out, err = run_cli(case["argv"] + ["--rng", "reference"])
    assert code == case["code"] == 1
    assert out == case["stdout"]
    if case["stderr"].startswith("usage:"):
        assert err.startswith("usage: hadamard-ga search")
    else:
        assert err == case["stderr"]


def test_cli_help_and_unknown_command_exit_codes():
    assert run_cli(["--help"])[0] == 0
    assert run_cli(["frobnicate"])[0] == 1
    assert run_cli(["bench", "fitness", "--orders", "6"])[0] == 1


# ------------------------------------------------------------------ grid table


def test_grid_table_and_csv_match_reference():
    gs = GOLDEN["grid"]
    spec = hbench.GridSpec(**{k: tuple(v) if isinstance(v, list) else v for k, v in gs["spec"].items()},
                           rng="reference")
    report = hbench.GridReport(spec=spec, rows=[dict(r) for r in gs["rows"]])
    cells = {}
    for r in report.rows:
        cells.setdefault((r["NC"], r["NR"]), []).append(r)
    report.cells = [hbench._cell_stats(nc, nr, rows) for (nc, nr), rows in cells.items()]
    assert hbench.format_grid_table(report) == gs["table"]
    assert hbench.grid_csv(report) == gs["csv"]


# ------------------------------------------------------------------ on the GPU


@pytest.mark.gpu
@pytest.mark.parametrize("case", [c for c in _cli_cases("search") if c["code"] != 1],
                         ids=lambda c: " ".join(c["argv"]))
def test_cli_search_reference_streams_match_reference(case, cuda_device, tmp_path):
    code, out, err = run_cli(case["argv"] + ["--rng", "reference"])
    assert (code, out, err) == (case["code"], case["stdout"], case["stderr"])


@pytest.mark.gpu
def test_cli_search_writes_reference_files(cuda_device, tmp_path):
    r = GOLDEN["records"][0]
    code, out, _ = run_cli(["search", "--order", "8", "--population", "20", "--max-iter", "200", "--seed", "1",
                            "--rng", "reference", "--out", str(tmp_path / "rec.json"),
                            "--trace", str(tmp_path / "trace.csv")])
    assert code == 0
    assert (tmp_path / "trace.csv").read_bytes().decode("ascii") == r["trace_bytes"]
    doc, q = io.load_run_record(tmp_path / "rec.json")
    assert doc["iterations"] == r["iterations"] and q.tolist() == r["best_matrix"]


@pytest.mark.gpu
def test_cli_search_philox_finds_order_12(cuda_device, tmp_path):
    code, out, _ = run_cli(["search", "--order", "12", "--population", "1000", "--max-iter", "5000", "--seed", "3",
                            "--out", str(tmp_path / "r.json")])
    assert code == 0, out
    doc, q = io.load_run_record(tmp_path / "r.json")  # re-verified on the host
    assert doc["success"] and doc["config"]["rng"] == "philox"
    assert run_cli(["verify", str(tmp_path / "r.json")])[0] == 1  # a record is not a matrix file
    io.save_matrix(q, tmp_path / "q.txt")
    assert run_cli(["verify", str(tmp_path / "q.txt")])[0] == 0


@pytest.mark.gpu
def test_grid_reference_streams_reproduce_reference_rows(cuda_device):
    gs = GOLDEN["grid"]
    spec = hbench.GridSpec(**{k: tuple(v) if isinstance(v, list) else v for k, v in gs["spec"].items()},
                           rng="reference")
    report = hbench.run_grid(spec)
    strip = lambda rows: [{k: v for k, v in r.items() if k != "wall_seconds"} for r in rows]  # noqa: E731
    assert strip(report.rows) == strip(gs["rows"])
    assert hbench.format_grid_table(report) == gs["table"]


@pytest.mark.gpu
def test_bench_fitness_fixed_length_legs(cuda_device):
    t = hbench.bench_fitness([12], population=200, iterations=300)
    assert len(t) == 1 and t[0].seconds_f1 > 0 and t[0].seconds_f2 > 0
    assert "f2/f1" in hbench.format_fitness_table(t)
