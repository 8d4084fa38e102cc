"""Single-generation launch time (L2 flushed before each, CUDA events) at the
bench config for internal run-flag variants (A/B of launch-time tricks)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2208_14961_b200 import engine  # noqa: E402
from paper_2208_14961_b200._lib import RUN_FORCE, check, lib  # noqa: E402

VARIANTS = {"none": 0, "fit": 1 << 21, "plain": 1 << 22, "noflush": 0, "plain_noflush": 1 << 22}
cfg = engine.GAConfig(order=20, population=10_000, seed=2024, fitness="f2", mutation_cols=4, mutation_row_pairs=2,
                      max_iterations=engine.MAX_ITERATIONS)
st = engine.initial_state(cfg)
res = st._res
res.ensure_trace(100000)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
sp = torch.cuda.current_stream().cuda_stream
burn = res.run_args()
burn.gens_this_call = 2000
burn.flags = RUN_FORCE
check(lib.hga_run(burn, sp), "hga_run")
torch.cuda.synchronize()
for rep in range(2):
    for name, fl in VARIANTS.items():
        a = res.run_args()
        a.gens_this_call = 1
        a.flags = RUN_FORCE | fl
        ts = []
        for i in range(300):
            if "noflush" not in name:
                flush.fill_(1)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            check(lib.hga_run(a, sp), "hga_run")
            e.record()
            ts.append((s, e))
        torch.cuda.synchronize()
        us = sorted(s.elapsed_time(e) * 1e3 for s, e in ts)
        print(json.dumps({"variant": name, "rep": rep, "median_us": us[len(us) // 2], "mean_us": sum(us) / len(us)}),
              flush=True)
