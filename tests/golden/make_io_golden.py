"""Golden outputs of the reference's file formats, CLI and grid harness.

Run ONLY in the build container (the reference is not on the GPU box):

    python tests/golden/make_io_golden.py

Everything in tests/golden/io_golden.json is produced by the unmodified
reference package (`hadamard_ga.io`, `hadamard_ga.cli`, `hadamard_ga.bench`,
pkg/src/hadamard_ga/{io,cli,bench}.py) on fixed inputs and seeds.  Wall-clock
fields are zeroed (records) or masked (CLI text) because they are the only
non-deterministic outputs.
"""

from __future__ import annotations

import contextlib
import dataclasses
import io as stdio
import json
import re
import sys
import tempfile
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
REF_FIXTURES = Path("/root/reference/pkg/tests/fixtures")
OUT = Path(__file__).with_name("io_golden.json")
TIME_RE = re.compile(r"in \d+\.\d+s")


def _ref():
    if str(REF_SRC) not in sys.path:
        sys.path.insert(0, str(REF_SRC))
    from hadamard_ga import bench, cli, core, engine, io

    return bench, cli, core, engine, io


def _cli(cli, argv, stdin_text=None):
    out, err = stdio.StringIO(), stdio.StringIO()
    old_stdin = sys.stdin
    if stdin_text is not None:
        sys.stdin = stdio.StringIO(stdin_text)
    try:
        with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
            code = cli.main(argv)
    finally:
        sys.stdin = old_stdin
    return {"argv": argv, "stdin": stdin_text, "code": code, "stdout": TIME_RE.sub("in <T>s", out.getvalue()), "stderr": err.getvalue()}


def main() -> None:
    bench, cli, core, engine, io = _ref()
    g: dict = {}
    tmp = Path(tempfile.mkdtemp())

    # ------------------------------------------------------------- matrix text
    rng = np.random.default_rng(7)
    fx20 = io.load_matrix(REF_FIXTURES / "hadamard_20.txt")
    mats = [core.sylvester(3), fx20.T.copy(), rng.choice(np.array([-1, 1], dtype=np.int8), size=(12, 12)),
            -np.ones((1, 1), dtype=np.int8)]
    g["matrices"] = [{"matrix": q.astype(int).tolist(), "text": io.write_matrix(q)} for q in mats]

    bad = [
        "",
        "hadamard matrix m=4\n++++\n",
        "hadamard-ga matrix m=x\n",
        "hadamard-ga matrix m=0\n",
        "hadamard-ga matrix m=2\n++\n",
        "hadamard-ga matrix m=2\n++\n+-\n--\n",
        "hadamard-ga matrix m=2\n++\n+-\n\n  \n",
        "hadamard-ga matrix m=2\n+++\n+-\n",
        "hadamard-ga matrix m=2\n++\n+x\n",
        "hadamard-ga matrix m=3\n+-+\n+é+\n+++\n",
        "hadamard-ga matrix m=2\n+0\n+\n",
        "hadamard-ga matrix m=2\n++\n+\n",
    ]
    cases = []
    for text in bad:
        try:
            q = io.parse_matrix(text)
            cases.append({"text": text, "error": None, "matrix": q.astype(int).tolist()})
        except ValueError as exc:
            cases.append({"text": text, "error": str(exc), "type": type(exc).__name__,
                          "line": getattr(exc, "line", None), "column": getattr(exc, "column", None)})
    g["parse_cases"] = cases

    # ------------------------------------------------------------- run records, traces, summaries
    runs = [
        dict(order=8, population=20, max_iterations=200, fitness="f2", mutation="multi", seed=1),
        dict(order=12, population=60, max_iterations=80, fitness="f2", mutation="shared", seed=13),
        dict(order=16, population=200, max_iterations=150, fitness="f1", mutation="multi", seed=5,
             mutation_cols=2, mutation_row_pairs=3, stall_window=6),
    ]
    recs = []
    for kw in runs:
        rec = dataclasses.replace(engine.run_search(engine.GAConfig(**kw)), wall_seconds=0.0)
        rec_path, trace_path = tmp / "rec.json", tmp / "trace.csv"
        io.write_run_record(rec, rec_path, trace_path="trace.csv")
        io.write_trace(rec.trace, trace_path)
        recs.append({
            "config": kw,
            "seed": rec.seed,
            "success": rec.success,
            "complete": rec.complete,
            "iterations": rec.iterations,
            "best_fitness": rec.best_fitness,
            "best_matrix": rec.best_matrix.astype(int).tolist(),
            "trace": [int(v) for v in rec.trace],
            "doc": io.run_record_doc(rec, trace_path="trace.csv"),
            "record_text": rec_path.read_text(encoding="ascii"),
            "trace_bytes": trace_path.read_bytes().decode("ascii"),
            "summary": io.format_summary(rec),
            "summary_budget": io.format_summary(dataclasses.replace(rec, complete=False, wall_seconds=12.3456)),
        })
    g["records"] = recs

    # ------------------------------------------------------------- CLI
    fx_path = str(REF_FIXTURES / "hadamard_32.txt")
    notq = core.sylvester(3)
    notq[2, 5] *= -1
    not_path = tmp / "not.txt"
    io.save_matrix(notq, not_path)
    g["cli_verify_input"] = io.write_matrix(notq)
    g["cli"] = [
        _cli(cli, ["sylvester", "--power", "3"]),
        _cli(cli, ["sylvester", "--power", "11"]),
        _cli(cli, ["verify", "-"], stdin_text=(REF_FIXTURES / "hadamard_32.txt").read_text()),
        _cli(cli, ["verify", "-"], stdin_text=io.write_matrix(notq)),
        _cli(cli, ["verify", "-"], stdin_text="hadamard-ga matrix m=2\n+\n"),
        _cli(cli, ["search", "--order", "6", "--seed", "1"]),
        _cli(cli, ["search", "--order", "8", "--population", "0", "--seed", "1"]),
        _cli(cli, ["search", "--seed", "1"]),
        _cli(cli, ["search", "--order", "8", "--seed", "-3"]),
        _cli(cli, ["search", "--order", "8", "--population", "20", "--max-iter", "200", "--seed", "1"]),
        _cli(cli, ["search", "--k", "3", "--population", "60", "--max-iter", "80", "--mutation", "shared",
                   "--seed", "0xd"]),
        _cli(cli, ["search", "--order", "12", "--population", "5", "--max-iter", "3", "--seed", "2"]),
    ]
    del fx_path

    # ------------------------------------------------------------- grid harness
    spec = bench.GridSpec(order=8, population=20, max_iterations=200, nc_values=(1, 2), nr_values=(1, 3), runs=2,
                          seed_base=3)
    report = bench.run_grid(spec)
    for r in report.rows:
        r["wall_seconds"] = 0.0
    for c in report.cells:
        c.mean_wall_seconds = 0.0
    g["grid"] = {
        "spec": dict(order=8, population=20, max_iterations=200, nc_values=[1, 2], nr_values=[1, 3], runs=2,
                     seed_base=3),
        "rows": report.rows,
        "table": bench.format_grid_table(report),
        "csv": bench.grid_csv(report),
    }
    OUT.write_text(json.dumps(g, indent=1, sort_keys=True) + "\n", encoding="utf-8")
    print(f"wrote {OUT} ({OUT.stat().st_size / 1e3:.1f} kB)")


if __name__ == "__main__":
    main()
