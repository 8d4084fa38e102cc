"""One int8 fitness launch per order on the tensor-core path (for ncu)."""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["HGA_FITNESS_TC"] = os.environ.get("HGA_FITNESS_TC", "all")
from paper_2208_14961_b200 import engine  # noqa: E402
from paper_2208_14961_b200._lib import lib  # noqa: E402

orders = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "20,48").split(",")]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 250_000
st = torch.cuda.current_stream().cuda_stream
for m in orders:
    pop = engine.init_population_device(engine.GAConfig(order=m, population=n // 4, seed=1))
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    for _ in range(3):
        rc = lib.hga_fitness_i8(pop.data_ptr(), n, m, 2, None, out.data_ptr(), None, None, None, None, 0, st)
        assert rc == 0, rc
    torch.cuda.synchronize()
    print(m, int(out[:4].sum()))
