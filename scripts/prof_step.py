"""Short, deterministic target for ncu: a few generations of the bench
workload (order 20, 40,000 matrices) plus one large fitness batch.

    python scripts/prof_step.py [--gens 6] [--fitness-m 20] [--fitness-n 4000000]
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2208_14961_b200 as hga  # noqa: E402
from paper_2208_14961_b200 import engine  # noqa: E402
from paper_2208_14961_b200._lib import RUN_FORCE, check, lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gens", type=int, default=6)
    ap.add_argument("--fitness-m", type=int, default=20)
    ap.add_argument("--fitness-n", type=int, default=4_000_000)
    ap.add_argument("--ga-m", type=int, default=20)
    ap.add_argument("--ga-n", type=int, default=10_000)
    args = ap.parse_args()
    sp = torch.cuda.current_stream().cuda_stream
    cfg = engine.GAConfig(order=args.ga_m, population=args.ga_n, seed=2024, fitness="f2", mutation_cols=4, mutation_row_pairs=2,
                          max_iterations=engine.MAX_ITERATIONS)
    st = hga.initial_state(cfg)
    res = st._res
    res.ensure_trace(args.gens + 4)
    a = res.run_args()
    a.gens_this_call = 1
    a.flags = RUN_FORCE
    for _ in range(args.gens):
        check(lib.hga_run(a, sp), "hga_run")
    m, n = args.fitness_m, args.fitness_n
    pop = engine.init_population_device(engine.GAConfig(order=m, population=n // 4, seed=7))
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    for _ in range(2):
        check(lib.hga_fitness_i8(pop.data_ptr(), n, m, 2, None, out.data_ptr(), None, None, None, None, 0, sp), "fit")
    packed = engine._pack(pop)
    check(lib.hga_fitness_packed(packed.data_ptr(), n, m, 2, None, out.data_ptr(), None, None, sp), "fitp")
    torch.cuda.synchronize()
    print("ok", st.iteration, int(res.dstate[0].item()))


if __name__ == "__main__":
    main()
