"""Per-phase device timing of the persistent generation loop (HGA_RUN_TIMING)."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2208_14961_b200 import engine  # noqa: E402
from paper_2208_14961_b200._lib import RUN_FORCE, RUN_TIMING, RUN_ONE_BARRIER, check, lib  # noqa: E402

# ramp the SM clock first (~0.5 s of integer work; a bf16 GEMM burn drives the
# part into its power cap and leaves the clocks low for the measurement)
_pop = engine.init_population_device(engine.GAConfig(order=20, population=250_000, seed=1))
_t0 = __import__("time").time()
while __import__("time").time() - _t0 < 0.5:
    engine.evaluate(_pop, "f2")
torch.cuda.synchronize()
del _pop

CASES = [(12, 1000, 0), (20, 10_000, 0), (20, 10_000, RUN_ONE_BARRIER), (28, 31_250, 0),
         (28, 31_250, RUN_ONE_BARRIER), (36, 312_500, 0)]
for m, N, xflags in CASES:
    engine._RUN_FLAGS = xflags
    cfg = engine.GAConfig(order=m, population=N, seed=1, fitness="f2", mutation_cols=4, mutation_row_pairs=2,
                          max_iterations=engine.MAX_ITERATIONS)
    st = engine.initial_state(cfg)
    res = st._res
    res.ensure_trace(200)
    a = res.run_args()
    a.flags = RUN_FORCE | RUN_TIMING | xflags
    a.gens_this_call = 40
    sp = torch.cuda.current_stream().cuda_stream
    check(lib.hga_run(a, sp), "run")
    torch.cuda.synchronize()
    off = int(lib.hga_run_timing_offset(m))
    ts = res.run_ws[off:off + 64 * 20 * 8].view(torch.int64).view(64, 20).cpu().numpy().astype(np.float64)[:40]
    med = lambda x: float(np.median(x)) / 1e3
    print(json.dumps({"m": m, "one_barrier": bool(xflags), "detail_us": {"B": med(ts[:, 1] - ts[:, 0]), "bar1": med(ts[:, 2] - ts[:, 1]),
                                             "E_prefix": med(ts[:, 7] - ts[:, 2]), "E_tiles": med(ts[:, 8] - ts[:, 7]),
                                             "E_flush": med(ts[:, 9] - ts[:, 8]), "bar2": med(ts[:, 4] - ts[:, 9]),
                                             "F": med(ts[1:, 0] - ts[:-1, 4])},
                      "sm_mhz": float(np.median((ts[:, 11] - ts[:, 10]) / (ts[:, 4] - ts[:, 0]) * 1e3))}))
    d = lambda a, b: med(ts[:, b] - ts[:, a])  # noqa: E731
    print(json.dumps({"m": m, "fine_us": {
        "B_tau": d(0, 3), "B_scan": d(3, 1), "E_prefix": d(2, 5), "E_init": d(5, 7),
        "t_prepare": d(7, 12), "t_gather": d(12, 13), "t_copy": d(13, 14), "t_xover": d(14, 15),
        "t_mutate": d(15, 16), "t_chain": d(16, 17), "t_fit": d(17, 18), "t_store": d(18, 19),
        "t_rest": d(19, 8)}}))
    gen = np.diff(ts[:, 0])
    print(json.dumps({"m": m, "N": N, "one_barrier": bool(xflags), "us_per_gen": float(np.median(gen)) / 1e3,
                      "offspring_evals_per_s": 2 * N / (float(np.median(gen)) / 1e9)}), flush=True)

# launch overhead: single-generation launches, plain vs CUDA-graph replay
engine._RUN_FLAGS = 0
for m, N in ((20, 10_000),):
    cfg = engine.GAConfig(order=m, population=N, seed=1, fitness="f2", mutation_cols=4, mutation_row_pairs=2,
                          max_iterations=engine.MAX_ITERATIONS)
    st = engine.initial_state(cfg)
    res = st._res
    res.ensure_trace(5000)
    a = res.run_args()
    a.flags = RUN_FORCE
    a.gens_this_call = 1
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        sp = s.cuda_stream
        for _ in range(5):
            check(lib.hga_run(a, sp), "run")
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(50):
            check(lib.hga_run(a, sp), "run")
        e1.record(s)
        e1.synchronize()
        plain = e0.elapsed_time(e1) / 50 * 1e3
        out = {"m": m, "N": N, "single_launch_us": plain}
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                check(lib.hga_run(a, torch.cuda.current_stream().cuda_stream), "run")
            for _ in range(3):
                g.replay()
            s.synchronize()
            e0.record(s)
            for _ in range(50):
                g.replay()
            e1.record(s)
            e1.synchronize()
            out["graph_replay_us"] = e0.elapsed_time(e1) / 50 * 1e3
        except Exception as exc:  # noqa: BLE001
            out["graph_error"] = repr(exc)[:200]
    print(json.dumps(out), flush=True)
