"""Experiment harness -- drop-in for hadamard_ga.bench (pkg/src/hadamard_ga/bench.py:1-296).

Two experiments from the paper, on the GPU engine:

* the NC x NR grid (paper Table 1 / Fig. 5; bench.py:33-205): every cell
  runs `runs` seeded searches and reports successes and iteration stats;
  seeds are ``seed_base + cell * runs + run`` in nc-major cell order
  (bench.py:68-70, 96-108), so with ``rng="reference"`` every row's
  iteration count equals the reference's;
* the F1-vs-F2 loop timing (paper Table 2; bench.py:208-296): the same
  fixed-length generation loop under both fitness functions from the same
  seed.  Legs never stop early.  In Philox mode the whole leg is ONE
  persistent kernel launch (`hga_run`, HGA_RUN_FORCE) instead of a host loop
  of `step` calls; the timed region ends with a device synchronize.

Data classes, field names, CSV columns and table layout follow the
reference so existing scripts and plots keep working; `GridSpec` and
`bench_fitness` take the extra `rng` choice.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from itertools import product

import numpy as np
import torch

from . import engine
from .engine import GAConfig

__all__ = [
    "GridSpec",
    "CellStats",
    "GridReport",
    "run_grid",
    "grid_csv",
    "write_grid_csv",
    "format_grid_table",
    "FitnessTiming",
    "bench_fitness",
    "format_fitness_table",
]

GRID_COLUMNS = ("m", "N", "T", "NC", "NR", "run_index", "seed", "success", "iterations", "wall_seconds")


@dataclass(frozen=True)
class GridSpec:
    """An NC x NR sweep; each cell runs `runs` seeded searches (bench.py:33-70)."""

    order: int
    population: int = 1000
    max_iterations: int = 10_000
    nc_values: tuple[int, ...] = (1, 2, 3, 4)
    nr_values: tuple[int, ...] = (1, 2, 3, 4)
    runs: int = 10
    fitness: str = "f2"
    mutation: str = "multi"
    seed_base: int = 0
    rng: str = "philox"

    def __post_init__(self):
        if self.runs < 1:
            raise ValueError("runs must be >= 1")
        for nc, nr in product(self.nc_values, self.nr_values):
            self.config(nc, nr, 0)  # GAConfig validates each cell

    def config(self, nc: int, nr: int, seed: int) -> GAConfig:
        return GAConfig(order=self.order, population=self.population, max_iterations=self.max_iterations,
                        mutation_cols=nc, mutation_row_pairs=nr, fitness=self.fitness, mutation=self.mutation,
                        seed=seed, rng=self.rng)

    def cell_seed(self, cell_index: int, run_index: int) -> int:
        return self.seed_base + cell_index * self.runs + run_index


@dataclass
class CellStats:
    nc: int
    nr: int
    runs: int
    successes: int
    mean_iterations: float | None  # successful runs only; None if none succeeded
    min_iterations: int | None
    max_iterations: int | None
    mean_wall_seconds: float


@dataclass
class GridReport:
    spec: GridSpec
    rows: list[dict] = field(default_factory=list)
    cells: list[CellStats] = field(default_factory=list)

    def cell(self, nc: int, nr: int) -> CellStats:
        hit = [c for c in self.cells if (c.nc, c.nr) == (nc, nr)]
        if not hit:
            raise KeyError(f"no cell NC={nc} NR={nr}")
        return hit[0]


def _cell_stats(nc: int, nr: int, rows: list[dict]) -> CellStats:
    ok = [r["iterations"] for r in rows if r["success"]]
    return CellStats(nc=nc, nr=nr, runs=len(rows), successes=len(ok),
                     mean_iterations=float(np.mean(ok)) if ok else None,
                     min_iterations=min(ok) if ok else None, max_iterations=max(ok) if ok else None,
                     mean_wall_seconds=float(np.mean([r["wall_seconds"] for r in rows])))


def run_grid(spec: GridSpec, workers: int = 1, echo: bool = False) -> GridReport:
    """Run every cell (bench.py:96-145); a failed search is a row, not an error."""
    report = GridReport(spec=spec)
    for cell_index, (nc, nr) in enumerate(product(spec.nc_values, spec.nr_values)):
        rows = []
        for run_index in range(spec.runs):
            seed = spec.cell_seed(cell_index, run_index)
            rec = engine.run_search(spec.config(nc, nr, seed), workers=workers)
            rows.append(dict(zip(GRID_COLUMNS, (spec.order, spec.population, spec.max_iterations, nc, nr, run_index,
                                                seed, rec.success, rec.iterations, rec.wall_seconds))))
        report.rows.extend(rows)
        stats = _cell_stats(nc, nr, rows)
        report.cells.append(stats)
        if echo:
            mean = "-" if stats.mean_iterations is None else f"{stats.mean_iterations:.1f}"
            print(f"NC={nc} NR={nr}: {stats.successes}/{spec.runs} found, mean iterations {mean}", flush=True)
    return report


def grid_csv(report: GridReport) -> str:
    """Per-run rows as CSV text (bench.py:148-173), CRLF like csv.writer."""
    out = [",".join(GRID_COLUMNS)]
    for r in report.rows:
        vals = [r[k] for k in GRID_COLUMNS[:7]] + [int(r["success"]), r["iterations"], f"{r['wall_seconds']:.6f}"]
        out.append(",".join(str(v) for v in vals))
    return "\r\n".join(out) + "\r\n"


def write_grid_csv(report: GridReport, path) -> None:
    with open(path, "w", encoding="ascii", newline="") as fh:
        fh.write(grid_csv(report))


def format_grid_table(report: GridReport) -> str:
    """NR rows x NC columns of mean iterations; '*' some runs failed, '-' none solved (bench.py:181-205)."""
    s, w = report.spec, 10
    text = [
        f"order {s.order}, N={s.population} (population {4 * s.population}), T={s.max_iterations},"
        f" fitness {s.fitness}, {s.runs} runs/cell",
        "mean iterations over successful runs ('*': some runs failed, '-': none succeeded)",
        "",
        "NR \\ NC".ljust(8) + "".join(f"NC={nc}".rjust(w) for nc in s.nc_values),
    ]

    def mean_cell(c: CellStats) -> str:
        if c.mean_iterations is None:
            return "-"
        return f"{c.mean_iterations:.1f}" + ("*" if c.successes < c.runs else "")

    for nr in s.nr_values:
        text.append(f"NR={nr}".ljust(8) + "".join(mean_cell(report.cell(nc, nr)).rjust(w) for nc in s.nc_values))
    text += ["", "successes per cell:"]
    for nr in s.nr_values:
        cells = (report.cell(nc, nr) for nc in s.nc_values)
        text.append(f"NR={nr}".ljust(8) + "".join(f"{c.successes}/{c.runs}".rjust(w) for c in cells))
    return "\n".join(text)


@dataclass
class FitnessTiming:
    order: int
    population: int
    iterations: int
    seconds_f1: float
    seconds_f2: float

    @property
    def ratio(self) -> float:
        """f2 seconds / f1 seconds (< 1: f2 faster)."""
        return self.seconds_f2 / self.seconds_f1


def _timed_loop(config: GAConfig, iterations: int, workers: int = 1) -> float:
    """Seconds for exactly `iterations` generations from a fresh state (bench.py:231-237)."""
    state = engine.initial_state(config, workers=workers)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if config.rng == "reference":
        for _ in range(iterations):
            engine.step(state, workers=workers)
    elif iterations > 0:
        engine._run_device(state, iterations, force=True)
    torch.cuda.synchronize()
    return time.perf_counter() - t0


def bench_fitness(orders, population: int = 1000, iterations: int = 1000, mutation_cols: int = 4,
                  mutation_row_pairs: int = 2, seed: int = 2024, workers: int = 1,
                  rng: str = "philox") -> list[FitnessTiming]:
    """F1 vs F2 loop timing, identical seeds and plans per leg (bench.py:240-284)."""
    out = []
    for order in orders:
        secs = {}
        for fit in ("f1", "f2"):
            cfg = GAConfig(order=order, population=population, max_iterations=max(iterations, 1),
                           mutation_cols=mutation_cols, mutation_row_pairs=mutation_row_pairs, fitness=fit,
                           mutation="multi", seed=seed, rng=rng)
            secs[fit] = _timed_loop(cfg, iterations, workers)
        out.append(FitnessTiming(order, population, iterations, secs["f1"], secs["f2"]))
    return out


def format_fitness_table(timings: list[FitnessTiming]) -> str:
    head = f"{'order':>6} {'matrices':>9} {'iterations':>11} {'f1 (s)':>10} {'f2 (s)':>10} {'f2/f1':>7}"
    body = [f"{t.order:>6} {4 * t.population:>9} {t.iterations:>11} {t.seconds_f1:>10.3f}"
            f" {t.seconds_f2:>10.3f} {t.ratio:>7.3f}" for t in timings]
    return "\n".join([head] + body)
