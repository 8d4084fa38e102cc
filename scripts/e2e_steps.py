"""A few drop-in host-state steps at the bench config (for ncu launch lists)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch

import bench
import paper_2208_14961_b200 as hga
from paper_2208_14961_b200 import engine


class A:
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5


cfg = engine.GAConfig(order=20, population=10_000, seed=2024, fitness="f2", mutation_cols=4, mutation_row_pairs=2,
                      max_iterations=engine.MAX_ITERATIONS)
print(bench.run_e2e(A, cfg, hga, engine, torch))
