"""A/B of the drop-in host-state step: population as int8 bytes
(hga_step_host) vs as a bit stream (hga_step_host_bits), bench config."""
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import json

import torch

import bench
import paper_2208_14961_b200 as hga
from paper_2208_14961_b200 import engine


class A:
    steps = 30


for mode in ("bits", "bytes", "bits-nograph", "bits-2pieces", "bits-8pieces", "bits"):
    os.environ.pop("HGA_STEP_HOST", None)
    os.environ.pop("HGA_STEP_GRAPH", None)
    engine._BIT_CHUNKS = 4
    if mode == "bytes":
        os.environ["HGA_STEP_HOST"] = "bytes"
    if mode == "bits-nograph":
        os.environ["HGA_STEP_GRAPH"] = "0"
    if mode.endswith("pieces"):
        engine._BIT_CHUNKS = int(mode.split("-")[1][0])
    cfg = engine.GAConfig(order=20, population=10_000, seed=2024, fitness="f2", mutation_cols=4, mutation_row_pairs=2,
                          max_iterations=engine.MAX_ITERATIONS)
    r = bench.run_e2e(A, cfg, hga, engine, torch)
    print(json.dumps({"mode": mode, "ms_per_step": r["ms_per_step"], "evals_per_s": r["value"]}), flush=True)
os.environ.pop("HGA_STEP_HOST", None)
os.environ.pop("HGA_STEP_GRAPH", None)
engine._BIT_CHUNKS = 4
os.environ["HGA_STEP_TIMING"] = "1"
cfg = engine.GAConfig(order=20, population=10_000, seed=2024, fitness="f2", mutation_cols=4, mutation_row_pairs=2,
                      max_iterations=engine.MAX_ITERATIONS)
A.steps = 5
bench.run_e2e(A, cfg, hga, engine, torch)
