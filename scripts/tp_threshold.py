"""Throughput tiles (default at orders 12..40) vs team tiles (forced) per generation."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2208_14961_b200 import engine  # noqa: E402
from paper_2208_14961_b200._lib import RUN_FORCE, check, lib  # noqa: E402

sp = torch.cuda.current_stream().cuda_stream
for m, N, nc, nr in ((12, 1000, 1, 2), (20, 10000, 4, 2), (20, 10000, 1, 10), (24, 20000, 1, 10), (28, 10000, 1, 10),
                     (28, 31250, 1, 10), (36, 31250, 1, 12), (36, 312500, 1, 12), (40, 50000, 1, 12)):
    row = {"m": m, "N": N, "nc": nc, "nr": nr}
    for name, fl in (("tp", 0), ("team", 1 << 16)):
        engine._RUN_FLAGS = fl
        st = engine.initial_state(engine.GAConfig(order=m, population=N, seed=1, fitness="f2", mutation_cols=nc,
                                                  mutation_row_pairs=nr, max_iterations=engine.MAX_ITERATIONS))
        res = st._res
        res.ensure_trace(100000)
        a = res.run_args()
        a.flags |= RUN_FORCE
        a.gens_this_call = 20
        check(lib.hga_run(a, sp), "run")
        torch.cuda.synchronize()
        a.gens_this_call = 200
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        check(lib.hga_run(a, sp), "run")
        e1.record()
        e1.synchronize()
        row[name + "_us_per_gen"] = round(e0.elapsed_time(e1) / 200 * 1e3, 2)
    print(json.dumps(row), flush=True)
