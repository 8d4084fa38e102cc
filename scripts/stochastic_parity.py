"""Stochastic parity of the Philox production loop against the reference.

SURVEY.md §8(c): the reference (hadamard_ga.run_search, m = 12, N = 1000,
NC = 1, NR = 2, T = 3000, seeds 0-29) solves F1 30/30 (mean 89.9
generations, median 88, range 53-125) and F2 19/30 (mean 116.5, median 106,
range 73-184; failures plateau at 2 and 4).  This script runs the same grid
with rng="philox" (different random numbers, same operators and selection
rule) and with rng="reference" (the reference's own streams, bit-exact), and
prints both distributions.
"""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2208_14961_b200 import engine  # noqa: E402

REFERENCE = {"f1": {"solved": 30, "mean": 89.9, "median": 88, "min": 53, "max": 125},
             "f2": {"solved": 19, "mean": 116.5, "median": 106, "min": 73, "max": 184}}
seeds = range(int(sys.argv[1]) if len(sys.argv) > 1 else 30)
out = {}
for rng in ("philox", "reference"):
    for fit in ("f1", "f2"):
        its, fails = [], []
        for sd in seeds:
            rec = engine.run_search(engine.GAConfig(order=12, population=1000, max_iterations=3000, mutation_cols=1,
                                                    mutation_row_pairs=2, fitness=fit, seed=sd, rng=rng))
            (its if rec.success else fails).append(rec.iterations if rec.success else rec.best_fitness)
        row = {"rng": rng, "fitness": fit, "runs": len(seeds), "solved": len(its),
               "mean": statistics.mean(its) if its else None, "median": statistics.median(its) if its else None,
               "min": min(its) if its else None, "max": max(its) if its else None, "failed_at": sorted(fails),
               "reference_published_in_survey": REFERENCE[fit]}
        print(json.dumps(row), flush=True)
