"""Where a single-generation launch of the bench config spends its time:
event time of the launch vs the kernel's own entry -> exit span
(%globaltimer, HGA_RUN_TIMING), and the bare launch cost of an empty kernel
of the same shape (hga_probe kinds 10 / 11), L2 flushed or not."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2208_14961_b200 import engine  # noqa: E402
from paper_2208_14961_b200._lib import RUN_FORCE, RUN_TIMING, check, lib  # noqa: E402

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
off = int(lib.hga_run_timing_offset(20))


def timed(fn, flushing, reps=200):
    out = []
    for _ in range(reps):
        if flushing:
            flush.fill_(1)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        out.append((s, e))
    torch.cuda.synchronize()
    return float(np.median([s.elapsed_time(e) * 1e3 for s, e in out]))


for flushing in (True, False):
    a = res.run_args()
    a.gens_this_call = 1
    a.flags = RUN_FORCE | RUN_TIMING
    spans, evs = [], []
    for _ in range(200):
        if flushing:
            flush.fill_(1)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        check(lib.hga_run(a, sp), "hga_run")
        e.record()
        torch.cuda.synchronize()
        ts = res.run_ws[off:off + 64 * 20 * 8].view(torch.int64).view(64, 20).cpu().numpy()
        evs.append(s.elapsed_time(e) * 1e3)
        spans.append({"entry_to_loop": (ts[0, 0] - ts[63, 0]) / 1e3, "gen": (ts[0, 4] - ts[0, 0]) / 1e3,
                      "loop_to_exit": (ts[63, 1] - ts[0, 4]) / 1e3, "entry_to_exit": (ts[63, 1] - ts[63, 0]) / 1e3,
                      "B": (ts[0, 1] - ts[0, 0]) / 1e3, "bar1": (ts[0, 2] - ts[0, 1]) / 1e3,
                      "tiles": (ts[0, 8] - ts[0, 7]) / 1e3, "bar2": (ts[0, 4] - ts[0, 9]) / 1e3})
    med = {k: float(np.median([x[k] for x in spans])) for k in spans[0]}
    print(json.dumps({"what": "single-generation launch (RUN_TIMING)", "l2_flushed": flushing,
                      "event_us": float(np.median(evs)), "kernel_us": med}), flush=True)
    for kind, name in ((10, "empty plain"), (11, "empty cooperative")):
        for smem in (0, 200 * 1024):
            us = timed(lambda: check(lib.hga_probe(kind, smem, 148, 640, None, sp), "probe"), flushing)
            print(json.dumps({"what": f"{name} launch 148x640, {smem // 1024} KB smem", "l2_flushed": flushing,
                              "event_us": us}), flush=True)
