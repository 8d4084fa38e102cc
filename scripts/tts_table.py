"""Markdown summary of committed time-to-Hadamard runs (profiles/*tts*.jsonl).

One row per (file, order, population, fitness, NC, NR, stall / restart
protocol, budget): solved / runs, wall-clock and generations to solution
(median and max over the solved seeds), best fitness reached by the unsolved
ones, and the loop's throughput.  Every found matrix in these files was
re-verified on the host (H^T H = mI, balanced) when it was written.

    python scripts/tts_table.py profiles/r01_tts_campaign_d.jsonl profiles/r02_tts28_*.jsonl ...
"""

from __future__ import annotations

import json
import statistics
import sys
from collections import OrderedDict
from pathlib import Path


def main(paths: list[str]) -> None:
    groups: OrderedDict = OrderedDict()
    for p in paths:
        for line in Path(p).read_text().splitlines():
            if not line.strip():
                continue
            r = json.loads(line)
            proto = (f"restart after {r['restart_stall'] // 1000}k stalled gens" if r.get("restart_stall")
                     else (f"stall window {r['stall_window'] // 1000}k" if r.get("stall_window") else "none"))
            key = (Path(p).name, r["order"], r["matrices"], r["fitness"], r["nc"], r["nr"], proto, r["budget_s"])
            groups.setdefault(key, {})[r["seed"]] = r  # a seed re-run at the same key keeps the last record
    print("| file | order | matrices | fitness | NC, NR | restarts | budget (s) | solved | wall s to solution "
          "(median / max) | generations (median) | best F of unsolved | evals/s |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for (name, order, mats, fit, nc, nr, proto, budget), runs in groups.items():
        rs = list(runs.values())
        ok = [r for r in rs if r["success"]]
        assert all(r.get("verified_HtH_eq_mI", True) for r in ok), name
        bad = sorted(r["best_fitness"] for r in rs if not r["success"])
        wall = f"{statistics.median(r['wall_seconds'] for r in ok):.1f} / {max(r['wall_seconds'] for r in ok):.1f}" if ok else "—"
        gens = f"{statistics.median(r['generations'] for r in ok):,.0f}" if ok else "—"
        rate = statistics.median(r["offspring_evals_per_s"] for r in rs) if all("offspring_evals_per_s" in r for r in rs) else None
        print(f"| {name} | {order} | {mats:,} | {fit} | {nc}, {nr} | {proto} | {budget:.0f} | {len(ok)}/{len(rs)} | "
              f"{wall} | {gens} | {', '.join(map(str, bad)) if bad else '—'} | "
              f"{f'{rate:.2e}' if rate else '—'} |")


if __name__ == "__main__":
    main(sys.argv[1:])
