"""A few reference-stream host-state steps at the bench config (bench.py's
e2e_same_config), for ncu launch lists and host timing."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch

import bench
from paper_2208_14961_b200 import engine


class A:
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5


r = bench.run_e2e_same_config(A, engine, torch)
print({k: r[k] for k in ("ms_per_step", "identical_to_reference_arm_step1")})
