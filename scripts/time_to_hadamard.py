"""Time-to-Hadamard runs (BASELINE metric, configs 2-4 on one GPU).

Each run: paper_2208_14961_b200.run_search with Philox streams, wall clock
from initial_state to the first matrix of fitness 0; the found matrix is
re-verified on the host with the CPU oracle's exact integer Gram (H^T H = mI)
and checked balanced.  One JSON line per run.

    python scripts/time_to_hadamard.py --order 20 --population 1000 --nc 2 --nr 8 --seeds 0 1 2 3 \
        --budget 120 [--fitness f2] [--stall 0]
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402  (verification only)
import paper_2208_14961_b200 as hga  # noqa: E402


def search_with_restarts(cfg, args):
    """Independent attempts within one time budget: attempt a runs the
    production loop from a fresh population (seed mix64(seed, a)) until its
    best fitness has not improved for `restart_stall` generations; the run
    ends at the first fitness-0 matrix or when the budget is spent.  Wall
    time and generations are totals over all attempts."""
    from types import SimpleNamespace

    from paper_2208_14961_b200 import engine
    from paper_2208_14961_b200.rand import mix64

    start = time.perf_counter()
    gens_total, attempt, best_all, best_matrix, per_attempt = 0, 0, None, None, []
    while True:
        seed_a = cfg.seed if attempt == 0 else mix64((cfg.seed * 0x9E3779B97F4A7C15 + attempt) & (2**64 - 1))
        st = engine.initial_state(cfg, seed=seed_a)
        last_improve, best = 0, st.best_fitness
        while st.best_fitness > 0 and time.perf_counter() - start < args.budget:
            engine._run_device(st, args.poll)
            if st.best_fitness < best:
                best, last_improve = st.best_fitness, st.iteration
            if st.iteration - last_improve >= args.restart_stall:
                break
        gens_total += st.iteration
        per_attempt.append(int(st.best_fitness))
        if best_all is None or st.best_fitness < best_all:
            best_all, best_matrix = int(st.best_fitness), st.best_matrix
        attempt += 1
        if st.best_fitness == 0 or time.perf_counter() - start >= args.budget:
            break
    torch.cuda.synchronize()
    return SimpleNamespace(success=best_all == 0, iterations=gens_total, best_fitness=best_all, best_matrix=best_matrix,
                           wall_seconds=time.perf_counter() - start, attempts=attempt, best_per_attempt=per_attempt)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--order", type=int, required=True)
    ap.add_argument("--population", type=int, required=True, help="N (pairs); the engine holds 4N matrices")
    ap.add_argument("--nc", type=int, default=1)
    ap.add_argument("--nr", type=int, default=2)
    ap.add_argument("--fitness", default="f2")
    ap.add_argument("--mutation", default="multi")
    ap.add_argument("--seeds", type=int, nargs="+", default=[0])
    ap.add_argument("--budget", type=float, default=120.0, help="seconds per run")
    ap.add_argument("--stall", type=int, default=0, help="stall window (0 = off)")
    ap.add_argument("--max-iter", type=int, default=hga.engine.MAX_ITERATIONS)
    ap.add_argument("--poll", type=int, default=2048)
    ap.add_argument("--out", default=None)
    ap.add_argument("--restart-stall", type=int, default=0,
                    help="full restart (fresh population, derived seed) when the best fitness has not improved "
                         "for this many generations (0 = one attempt)")
    args = ap.parse_args()
    out = open(args.out, "a") if args.out else None
    for seed in args.seeds:
        cfg = hga.GAConfig(order=args.order, population=args.population, seed=seed, fitness=args.fitness,
                           mutation=args.mutation, mutation_cols=args.nc, mutation_row_pairs=args.nr,
                           max_iterations=args.max_iter, stall_window=args.stall or None,
                           time_budget_secs=args.budget)
        torch.cuda.synchronize()
        if args.restart_stall > 0:
            rec = search_with_restarts(cfg, args)
        else:
            rec = hga.run_search(cfg, poll_interval=args.poll)
        ok = bool(rec.success)
        verified = False
        if ok:
            q = rec.best_matrix
            g = q.astype(np.int64).T @ q.astype(np.int64)
            verified = bool((g == args.order * np.eye(args.order, dtype=np.int64)).all())
            verified &= int(oracle.penalties(q[None])[0, 1]) == 0 and bool(hga.is_balanced(q))
        line = {"order": args.order, "N": args.population, "matrices": 4 * args.population, "seed": seed,
                "fitness": args.fitness, "mutation": args.mutation, "nc": args.nc, "nr": args.nr,
                "stall_window": args.stall,
                "success": ok, "verified_HtH_eq_mI": verified, "generations": rec.iterations,
                "best_fitness": rec.best_fitness, "wall_seconds": rec.wall_seconds,
                "offspring_evals_per_s": 2 * args.population * rec.iterations / max(rec.wall_seconds, 1e-9),
                "budget_s": args.budget, "rng": cfg.rng}
        if hasattr(rec, "attempts"):
            line["attempts"] = rec.attempts
            line["restart_stall"] = args.restart_stall
            line["best_per_attempt"] = rec.best_per_attempt
        if ok:
            line["matrix_rows"] = ["".join("+" if v > 0 else "-" for v in row) for row in rec.best_matrix]
        print(json.dumps(line), flush=True)
        if out:
            out.write(json.dumps(line) + "\n")
            out.flush()


if __name__ == "__main__":
    main()
