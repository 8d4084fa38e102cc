"""Measure pipe rates and first kernel throughputs on the B200 (one JSON line each).

    python scripts/probe.py [--quick]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2208_14961_b200 import engine  # noqa: E402
from paper_2208_14961_b200._lib import lib  # noqa: E402


def timed(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    return best


def probe_pipes():
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    out = torch.zeros(4096, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    iters = 20000
    for kind, name in ((0, "popc"), (1, "alu_lop3_iadd")):
        blocks, threads = sms * 8, 256
        t = timed(lambda: lib.hga_probe(kind, iters, blocks, threads, out.data_ptr(), st), reps=5, warm=2)
        ops = blocks * threads * iters * 8
        clk = torch.cuda.clock_rate() if hasattr(torch.cuda, "clock_rate") else None
        print(json.dumps({"probe": name, "ops_per_s": ops / t, "per_sm_per_clk_at_1965MHz": ops / t / sms / 1.965e9,
                          "sm_clock_mhz_now": clk}), flush=True)
    # dense int8 tcgen05.mma: kind 2 = 128x256x32 (pipe peak), kind 3 = 64x64x32 (the fitness kernels' shape)
    for kind, (M, N), iters, tag in ((2, (128, 256), 20000, "same_tile"), (3, (64, 64), 200000, "same_tile"),
                                     (4, (64, 64), 200000, "rotating_tiles"), (5, (64, 48), 200000, "rotating_tiles"),
                                     (6, (128, 128), 100000, "rotating_tiles"), (7, (128, 96), 100000, "rotating_tiles"),
                                     (8, (128, 64), 100000, "rotating_tiles"), (9, (128, 256), 20000, "rotating_tiles")):
        t = timed(lambda: lib.hga_probe(kind, iters, sms, 128, out.data_ptr(), st), reps=5, warm=2)
        ops = sms * iters * 2 * M * N * 32
        print(json.dumps({"probe": f"tcgen05_mma_i8_{M}x{N}x32_{tag}", "ops_per_s": ops / t, "mma_per_s_per_sm": iters / t,
                          "clk_per_mma_at_1965MHz": 1.965e9 * t / iters}), flush=True)


def probe_fitness(quick):
    st = torch.cuda.current_stream().cuda_stream
    for m in (8, 12, 16, 20, 24, 28, 32, 36, 40, 44, 48, 52, 56, 60, 64, 96, 128):
        n = 2_000_000 if m <= 32 else (1_000_000 if m <= 64 else 200_000)
        if quick:
            n //= 4
        cfg = engine.GAConfig(order=m, population=n // 4, seed=2024)
        pop = engine.init_population_device(cfg)
        outs = torch.empty(n, dtype=torch.int64, device="cuda")
        for var, name in ((2, "f2"), (1, "f1"), (15, "all")):
            o = [outs if var & b else None for b in (1, 2, 4, 8)]
            if var == 15:
                o = [torch.empty(n, dtype=torch.int64, device="cuda") for _ in range(4)]
            ptrs = [x.data_ptr() if x is not None else None for x in o]
            tc = m <= 64
            paths = (("tcgen05_r2", "tcgen05", "popc") if 36 <= m <= 64 else ("tcgen05", "popc")) if tc else ("popc",)
            for path in paths:
                if tc:
                    os.environ["HGA_FITNESS_TC"] = {"popc": "0", "tcgen05": "all", "tcgen05_r2": "2"}[path]
                t = timed(lambda: lib.hga_fitness_i8(pop.data_ptr(), n, m, var, *ptrs, None, None, 0, st))
                os.environ.pop("HGA_FITNESS_TC", None)
                bytes_ = n * (m * m + 8 * bin(var).count("1"))
                print(json.dumps({"kernel": "fitness_i8", "path": path, "m": m, "n": n, "variant": name,
                                  "evals_per_s": n / t, "GBps": bytes_ / t / 1e9, "us": t * 1e6}), flush=True)
        packed = engine._pack(pop)
        t = timed(lambda: lib.hga_fitness_packed(packed.data_ptr(), n, m, 2, None, outs.data_ptr(), None, None, st))
        W = (m + 31) // 32
        print(json.dumps({"kernel": "fitness_packed", "m": m, "n": n, "variant": "f2", "evals_per_s": n / t,
                          "GBps": n * (4 * m * W + 8) / t / 1e9, "us": t * 1e6,
                          "pairs_per_s": n * m * (m - 1) / 2 / t}), flush=True)
        del pop, packed
        torch.cuda.empty_cache()


def probe_ga():
    for m, N in ((20, 10_000), (28, 31_250), (36, 312_500), (12, 1000)):
        for fit in ("f2", "f1"):
            cfg = engine.GAConfig(order=m, population=N, seed=1, fitness=fit, max_iterations=10**6)
            st = engine.initial_state(cfg)
            res = st._res
            a = res.run_args()
            gens = 200
            res.ensure_trace(gens + 10)
            a = res.run_args()
            a.gens_this_call = 20
            lib.hga_run(a, torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            a.gens_this_call = gens
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            rc = lib.hga_run(a, torch.cuda.current_stream().cuda_stream)
            e.record()
            e.synchronize()
            t = s.elapsed_time(e) / 1e3
            dstate = res.dstate.cpu().tolist()
            print(json.dumps({"ga": "philox_run", "m": m, "N": N, "fitness": fit, "rc": rc, "gens_done": dstate[0],
                              "best": dstate[1], "us_per_gen": t / max(1, dstate[0] - 20) * 1e6,
                              "offspring_evals_per_s": 2 * N * max(1, dstate[0] - 20) / t}), flush=True)
            # single generation launches (what bench steps do)
            def one():
                a.gens_this_call = 1
                res.dstate[5] = 0
                lib.hga_run(a, torch.cuda.current_stream().cuda_stream)
            a.max_generation = 10**7
            t1 = timed(one, reps=20, warm=3)
            print(json.dumps({"ga": "philox_one_gen_launch", "m": m, "N": N, "fitness": fit, "us": t1 * 1e6,
                              "offspring_evals_per_s": 2 * N / t1}), flush=True)
            del st, res
            torch.cuda.empty_cache()


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--only", choices=("pipes", "fitness", "ga"), default=None)
    args = ap.parse_args()
    print(json.dumps({"device": torch.cuda.get_device_name(0)}), flush=True)
    if args.only in (None, "pipes"):
        probe_pipes()
    if args.only in (None, "fitness"):
        probe_fitness(args.quick)
    if args.only in (None, "ga"):
        probe_ga()
