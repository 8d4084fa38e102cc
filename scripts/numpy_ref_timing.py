"""Time the UNMODIFIED NumPy reference (hadamard_ga) on this host.

The reference is installed (not copied into the tree) under baseline/_ref
(`pip install --no-deps --target baseline/_ref <copy of /root/reference/pkg>`;
git-ignored, travels to the GPU box with the gpurun snapshot).  Measures, on
the box's own host cores:
  * engine.evaluate(pop, "f2", workers=W) for W in {1, os.cpu_count()} at
    m = 20 / 36 / 64 (the reference's thread pool, engine.py:216-230), best of 3;
  * bench._timed_loop (bench.py:231-237) at BASELINE configs[1]: order 20,
    N = 10,000 (40,000 matrices), f2, multi NC = 4 NR = 2 -- the bench
    metric's workload -- with workers 1 and os.cpu_count().
OPENBLAS_NUM_THREADS=1 (the survey's setting: the worker pool supplies the
parallelism; default BLAS threading collapses at small matrices).
One JSON line per measurement.

    python scripts/numpy_ref_timing.py [--gens K]
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import time
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gens", type=int, default=5)
    args = ap.parse_args()
    if not (REF / "hadamard_ga").exists():
        print(json.dumps({"numpy_reference": "unavailable", "why": f"{REF} not installed"}))
        return
    sys.path.insert(0, str(REF))
    import numpy as np
    from hadamard_ga import bench as rbench
    from hadamard_ga import engine as reng

    cores = os.cpu_count() or 1
    cpu = platform.processor() or platform.machine()
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                cpu = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    base = {"host_cores": cores, "cpu": cpu, "numpy": np.__version__, "openblas_threads": os.environ["OPENBLAS_NUM_THREADS"],
            "reference": "hadamard_ga (unmodified, baseline/_ref)"}
    for m, n in ((20, 20_000), (36, 20_000), (64, 5_000)):
        pop = reng.init_population(reng.GAConfig(order=m, population=n // 4, seed=2024), seed=2024)
        for w in sorted({1, cores}):
            best = 1e30
            for _ in range(3):
                t0 = time.perf_counter()
                reng.evaluate(pop, "f2", workers=w)
                best = min(best, time.perf_counter() - t0)
            print(json.dumps({**base, "what": "engine.evaluate f2", "m": m, "n": n, "workers": w,
                              "evals_per_s": n / best, "seconds": best}), flush=True)
    cfg = reng.GAConfig(order=20, population=10_000, max_iterations=10**6, mutation_cols=4, mutation_row_pairs=2,
                        fitness="f2", mutation="multi", seed=2024)
    for w in sorted({1, cores}):
        t = rbench._timed_loop(cfg, args.gens, w)
        print(json.dumps({**base, "what": "bench._timed_loop (BASELINE configs[1]: order 20, 40,000 matrices, f2, "
                                          "multi NC=4 NR=2)", "workers": w, "generations": args.gens,
                          "ms_per_generation": t / args.gens * 1e3,
                          "offspring_evals_per_s": 2 * 10_000 * args.gens / t}), flush=True)


if __name__ == "__main__":
    main()
