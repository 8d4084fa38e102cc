"""Where the time of one drop-in host-state step goes (bench e2e leg)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2208_14961_b200 import engine  # noqa: E402

sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from test_gpu_parity import _host_state  # noqa: E402

cfg = engine.GAConfig(order=20, population=10_000, seed=2024, fitness="f2", mutation_cols=4, mutation_row_pairs=2)
dev = engine.initial_state(cfg)
hs = _host_state(cfg, dev.seed, dev.population.copy(), dev.fitness.copy(), dev.best_matrix.copy(), dev.best_fitness)
for _ in range(3):
    engine.step(hs)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(30):
    engine.step(hs)
full = (time.perf_counter() - t0) / 30
br = hs._hga_bridge
pop_t, fit_t = torch.from_numpy(hs.population), torch.from_numpy(hs.fitness)
t0 = time.perf_counter()
for _ in range(30):
    br.pop_i8.copy_(pop_t, non_blocking=True)
    pop_t.copy_(br.pop_i8, non_blocking=True)
    torch.cuda.synchronize()
copies = (time.perf_counter() - t0) / 30
t0 = time.perf_counter()
for _ in range(30):
    engine.step(dev)
res_only = (time.perf_counter() - t0) / 30
print({"full_step_us": full * 1e6, "h2d_plus_d2h_us": copies * 1e6, "resident_step_us": res_only * 1e6,
       "pinned": pop_t.is_pinned()})
