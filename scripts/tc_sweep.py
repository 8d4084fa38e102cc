"""int8 fitness sweep at orders 36..64 on one path (for A/B of the fitness kernels).

Usage: python scripts/tc_sweep.py TAG [PATH]
  PATH = tc2 (round-2 tcgen05 kernel, HGA_FITNESS_TC=2) | tc (round-1, HGA_FITNESS_TC=all)
       | popc (XOR+POPC, HGA_FITNESS_TC=0) | default
One JSON line per (m, variant): best of 10 CUDA-event timings after 3 warm-ups.
"""
import json
import os
import sys
from pathlib import Path

tag = sys.argv[1] if len(sys.argv) > 1 else "run"
path = sys.argv[2] if len(sys.argv) > 2 else "tc"
if path != "default":
    os.environ["HGA_FITNESS_TC"] = {"tc": "all", "tc2": "2", "popc": "0"}[path]

import torch  # noqa: E402

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2208_14961_b200 import engine  # noqa: E402
from paper_2208_14961_b200._lib import lib  # noqa: E402

orders = [int(x) for x in os.environ.get("ORDERS", "36,40,44,48,52,56,60,64").split(",")]
n = int(os.environ.get("NMAT", "1000000"))
st = torch.cuda.current_stream().cuda_stream
for m in orders:
    if os.environ.get("HGA_LIB_VARIANT"):  # fitness-only A/B library: random +-1 input from torch
        g = torch.Generator(device="cuda").manual_seed(2024 + m)
        pop = (torch.randint(0, 2, (n, m, m), device="cuda", dtype=torch.int8, generator=g) * 2 - 1).contiguous()
    else:
        pop = engine.init_population_device(engine.GAConfig(order=m, population=n // 4, seed=2024))
    for var, name in [(v, nm) for v, nm in ((2, "f2"), (1, "f1"), (8, "sq"), (15, "all"))
                      if nm in os.environ.get("VARIANTS", "f2,f1,all").split(",")]:
        o = [torch.empty(n, dtype=torch.int64, device="cuda") if var & b else None for b in (1, 2, 4, 8)]
        ptrs = [x.data_ptr() if x is not None else None for x in o]

        def one():
            rc = lib.hga_fitness_i8(pop.data_ptr(), n, m, var, *ptrs, None, None, 0, st)
            assert rc == 0, rc

        for _ in range(3):
            one()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e30
        for _ in range(10):
            s.record()
            one()
            e.record()
            e.synchronize()
            best = min(best, s.elapsed_time(e) / 1e3)
        byts = n * (m * m + 8 * bin(var).count("1"))
        print(json.dumps({"tag": tag, "path": path, "m": m, "n": n, "variant": name, "evals_per_s": n / best,
                          "GBps": byts / best / 1e9, "frac_hbm": byts / best / 6547.5e9, "us": best * 1e6}),
              flush=True)
    del pop
    torch.cuda.empty_cache()
