"""Benchmark of the GA inner loop (BASELINE.json metric: matrix fitness evals/s).

Workload (BASELINE.json configs[1]): order-20 GA, population 40,000 matrices
(N = 10,000 pairs), on one B200 per rank.  One step = one generation:
select over all 4N -> column-block crossover -> +-1 pair-flip mutation ->
fitness of the 2N offspring (engine.py:449-469), i.e. 2N = 20,000 matrix
fitness evaluations per step per GPU.  Fitness F2 (the reference default),
mutation "multi" with NC=4, NR=2 (the reference's own bench setting,
bench.py:264-273 of hadamard_ga); Philox streams.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

`value`  device-timed throughput: per-step CUDA events around the one
         persistent-kernel launch of that generation, L2 flushed (256 MiB
         write) between steps outside the events; max over ranks.
`e2e`    the same metric through the public drop-in API with HOST buffers:
         engine.step() on a reference-style state whose population/fitness
         are numpy arrays -> H2D of the int8 population + fitness, the
         generation, D2H of both, every step (wall clock).
`roofline` the generation kernel (k_run) against the measured HBM peak with
         its algorithmic bytes; `fitness_sweep`
         adds the large-batch fitness kernel (config 5) at m = 20..64.
`cpu_baseline` the C oracle port (oracle/hga_oracle.c) on the host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

ORDER, N_PAIRS, FITNESS, NC, NR = 20, 10_000, "f2", 4, 2
MIGRATE_EVERY, MIGRATION_SIZE = 50, 16  # islands (n_gpus > 1): ring migration of 16 elites every 50 generations
METRIC = "matrix fitness evals/sec (order-20 GA generation, 40,000 matrices, 2N offspring evaluated per generation)"
UNIT = "evals/s"


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


# ---------------------------------------------------------------- clocks


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, ValueError):
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict | None:
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- our arm


def load_peaks() -> dict:
    """HBM from the driver-written MEASURED_PEAKS.json; the pipe ceilings
    (POPC, int8 tcgen05) from the committed probe output profiles/r02_peaks.json
    (scripts/probe.py --only pipes on this pool's B200)."""
    peaks = {}
    mp = ROOT / "MEASURED_PEAKS.json"
    if mp.exists():
        peaks.update({k: v for k, v in json.loads(mp.read_text()).items() if k in ("hbm_gbs", "bf16_tflops")})
        peaks["hbm_source"] = "MEASURED_PEAKS.json hbm_gbs"
    pp = ROOT / "profiles" / "r02_peaks.json"
    if pp.exists():
        d = json.loads(pp.read_text())
        for k in ("popc_per_s", "alu_per_s", "int8_tc_dense_ops_per_s"):
            if k in d:
                peaks[k] = d[k]
        for r in d.get("probes", []):
            if r.get("probe", "").startswith("tcgen05_mma_i8_64x64x32_rotating"):
                peaks["mma_64x64x32_per_s_per_sm"] = r["mma_per_s_per_sm"]
        peaks["pipe_source"] = "profiles/r02_peaks.json (scripts/probe.py --only pipes)"
    if "hbm_gbs" not in peaks:
        peaks["hbm_gbs"], peaks["hbm_source"] = 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"
    return peaks


_NCU_SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1024.0, "MB": 1024.0**2, "GB": 1024.0**3}


def ncu_traffic(path: Path) -> float | None:
    """dram__bytes_read.sum + dram__bytes_write.sum of one launch from a
    committed ncu summary ({"metrics": {name: [unit, value]}})."""
    try:
        m = json.loads(path.read_text()).get("metrics", {})
        tot = 0.0
        for name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            unit, val = m[name]
            tot += float(str(val).replace(",", "")) * _NCU_SCALE[unit]
        return tot
    except (OSError, ValueError, KeyError, TypeError):
        return None


def algorithmic_bytes_per_generation(m: int, n_pairs: int) -> int:
    """Minimum HBM traffic of one generation:
    read 4N fitness (selection), read the 2N selected parents, write the new
    population (2N parent copies + 2N offspring) and its 4N fitness."""
    mat = 4 * m * ((m + 31) // 32)
    total = 4 * n_pairs
    return total * 8 + 2 * n_pairs * mat + total * mat + total * 8


def run_ours(args, rank, world, local_rank):
    if world > 1 and "HGA_HOST_THREADS" not in os.environ:
        # one host thread pool per rank (the host-state step's bit packing): share the cores
        cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
        local = env_int("LOCAL_WORLD_SIZE", world)
        os.environ["HGA_HOST_THREADS"] = str(max(1, cores // max(1, local)))
    import torch

    torch.cuda.set_device(local_rank)
    import paper_2208_14961_b200 as hga
    from paper_2208_14961_b200 import engine
    from paper_2208_14961_b200._lib import RUN_FORCE, lib, check

    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream

    from paper_2208_14961_b200.islands import Exchange, GpuIsland, island_seed, pack_payload, unpack_payload

    cfg = engine.GAConfig(order=ORDER, population=N_PAIRS, seed=2024, fitness=FITNESS, mutation_cols=NC,
                          mutation_row_pairs=NR, max_iterations=engine.MAX_ITERATIONS)
    island = GpuIsland(cfg, island_seed(2024, rank))
    st = island.state
    res = st._res
    ex = Exchange() if world > 1 else None

    def migrate():
        # ring elite migration (islands.py): E best -> next island's offspring slots
        rec, fit = island.elites(MIGRATION_SIZE)
        r2, f2 = unpack_payload(ex.ring_shift(pack_payload(rec, fit)), MIGRATION_SIZE, rec.shape[1])
        island.receive(r2, f2)
    res.ensure_trace(args.warmup + args.steps + 8)
    a = res.run_args()
    a.gens_this_call = 1
    a.flags = RUN_FORCE
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def one_generation():
        check(lib.hga_run(a, sp), "hga_run")

    sampler = ClockSampler(local_rank)
    sampler.start()
    # untimed: ramp the SM clock (~0.4 s of generations), then the W warm-up steps
    burn = res.run_args()
    burn.gens_this_call = 256
    burn.flags = RUN_FORCE
    t_burn = time.perf_counter()
    while time.perf_counter() - t_burn < 0.4:
        check(lib.hga_run(burn, sp), "hga_run")  # trace writes past capacity are skipped
        torch.cuda.synchronize()
    for _ in range(args.warmup):
        flush.fill_(1)
        one_generation()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    wall0 = time.perf_counter()
    for i, (s, e) in enumerate(evs):
        flush.fill_(1)  # write 256 MiB > 126 MB L2 between timed steps
        s.record(stream)
        one_generation()
        if ex is not None and (i + 1) % MIGRATE_EVERY == 0:
            migrate()  # the exchange step of the island model, inside the timed step
        e.record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    clocks = sampler.stop()
    step_s = [s.elapsed_time(e) / 1e3 for s, e in evs]
    t_total = sum(step_s)
    if dist:
        tt = torch.tensor([t_total], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_total = float(tt.item())
    per_step = t_total / args.steps
    evals_per_step = 2 * N_PAIRS
    value = evals_per_step * world / per_step

    # roofline of the dominant (only) kernel of the step: k_run
    alg_bytes = algorithmic_bytes_per_generation(ORDER, N_PAIRS)
    peaks = load_peaks()
    peak = float(peaks["hbm_gbs"])
    achieved = alg_bytes / per_step / 1e9
    pairs = (ORDER - 1) * (ORDER - 2) // 2  # column 0 is all +1 in every GA individual
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": None, "kernel": "k_run_v3 (one generation, persistent cooperative kernel)",
                "algorithmic_bytes_per_launch": alg_bytes, "peak_source": peaks["hbm_source"],
                "popc_frac": 2 * N_PAIRS * pairs / per_step / peaks["popc_per_s"] if "popc_per_s" in peaks else None,
                "note": "latency-bound: a 40,000-matrix generation moves 5.4 MB and does 3.4M POPC "
                        "(< 1 us of either ceiling); DESIGN.md section 3"}
    for prof in (ROOT / "profiles" / "r02_k_run_traffic.json", ROOT / "profiles" / "r01_k_run_traffic.json"):
        if prof.exists():
            roofline["traffic"] = ncu_traffic(prof)
            roofline["traffic_source"] = str(prof.relative_to(ROOT))
            break

    # production mode: K generations back to back in ONE launch (no flush)
    a2 = res.run_args()
    a2.gens_this_call = args.steps
    a2.flags = RUN_FORCE
    res.ensure_trace(st.iteration + 2 * args.steps + 2 * args.warmup + 16)
    a2 = res.run_args()
    a2.gens_this_call = args.steps
    a2.flags = RUN_FORCE
    s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    check(lib.hga_run(a2, sp), "hga_run")
    e0.record(stream)
    torch.cuda.synchronize()
    persistent = evals_per_step * args.steps / (s0.elapsed_time(e0) / 1e3)

    # e2e through the public API with host (numpy) buffers
    e2e = run_e2e(args, cfg, hga, engine, torch)
    # the same public call computing exactly what the reference arm computes:
    # reference streams, the reference arm's seed and initial population
    e2e_same = run_e2e_same_config(args, engine, torch) if (not args.no_cpu and world == 1) else None
    # the same public call on the device-resident SearchState (each step reads
    # back its trace entry / best fitness): what run_search-style users get
    st2 = hga.initial_state(cfg)
    for _ in range(3):
        hga.step(st2)
    torch.cuda.synchronize()
    n_res = max(10, min(args.steps, 200))
    t0 = time.perf_counter()
    for _ in range(n_res):
        hga.step(st2)
    t_res = (time.perf_counter() - t0) / n_res
    e2e_resident = {"value": 2 * N_PAIRS / t_res, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 72,
                    "steps": n_res, "ms_per_step": t_res * 1e3,
                    "api": "paper_2208_14961_b200.step(state) on the device-resident SearchState (trace entry + "
                           "8-word state read back every step)"}

    # fitness-only sweep (config 5) at large n: the kernel's own roofline
    sweep = run_fitness_sweep(args, engine, torch, lib, peaks) if not args.no_sweep else None
    # the config-3 / config-4 island generation loops against their ceilings
    gen_rows = run_generation_rows(args, engine, torch, lib, peaks) if not args.no_sweep else None

    out = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": per_step * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u32 bit-packed +-1 (int64 fitness)",
        "data": "synthetic: Philox-seeded random balanced sign matrices (seed 2024 + rank)",
        "config": {"workload": "BASELINE configs[1]: order-20 GA, population 40,000 matrices (N=10,000 pairs), "
                               "fitness f2, mutation multi NC=4 NR=2, rng philox",
                   "order": ORDER, "matrices": 4 * N_PAIRS, "offspring_evals_per_step": evals_per_step,
                   "parallelism": f"islands x{world} (one 40,000-matrix population per GPU"
                                  + (f"; NCCL ring migration of {MIGRATION_SIZE} elites every {MIGRATE_EVERY} steps)"
                                     if world > 1 else ")"),
                   "l2": "flushed between timed steps (256 MiB write, outside the CUDA events)"},
        "gpu_launches": args.steps + (5 * (args.steps // MIGRATE_EVERY) if world > 1 else 0),
        "roofline": roofline,
        "e2e": e2e,
        "e2e_resident": e2e_resident,
        "e2e_same_config": e2e_same,
        "persistent_run": {"value": persistent * world, "unit": UNIT, "generations_per_launch": args.steps,
                           "note": "production run_search mode: K generations in one launch, L2 warm"},
        "wall_seconds_timed_region": wall,
        "clocks": clocks,
        "clocks_note": "nvidia-smi sampled every 100 ms from the clock ramp through the timed region",
    }
    if sweep:
        out["fitness_sweep"] = sweep
    if gen_rows:
        out["generation_rows"] = gen_rows
    if rank == 0 and world == 1 and not args.no_cpu:
        out["cpu_baseline"] = cpu_baseline(args)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return out


def run_e2e(args, cfg, hga, engine, torch):
    """engine.step() on a host-resident (numpy) reference-style state."""

    @dataclass
    class HostState:  # field-for-field the reference's SearchState (engine.py:376-387)
        config: object
        seed: int
        population: np.ndarray
        fitness: np.ndarray
        iteration: int
        best_matrix: np.ndarray
        best_fitness: int
        trace: list = field(default_factory=list)

    dev_state = hga.initial_state(cfg)
    pop = dev_state.population
    fit = dev_state.fitness
    hs = HostState(cfg, dev_state.seed, pop, fit, 0, dev_state.best_matrix, dev_state.best_fitness,
                   [dev_state.best_fitness])
    del dev_state
    steps = max(3, min(args.steps, 30))
    for _ in range(2):
        engine.step(hs)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        engine.step(hs)
    t = (time.perf_counter() - t0) / steps
    assert hs.population[:, :, 0].min() == 1
    bridge = hs._hga_bridge
    if bridge.bit_buffers() is not None:  # the population crosses PCIe as a bit stream
        stream_bytes = (pop.nbytes + 31) // 32 * 4
        api = ("paper_2208_14961_b200.engine.step(state) with numpy population/fitness (drop-in for hadamard_ga.step; "
               "one hga_step_host_bits call: host AVX2 pack + validation of the int8 population into a bit stream "
               "(8x fewer PCIe bytes) pipelined with its upload and the device stream->column kernels, one CUDA "
               "graph for the generation and the piecewise download, host unpack as the pieces land)")
    else:
        stream_bytes = pop.nbytes
        api = ("paper_2208_14961_b200.engine.step(state) with numpy population/fitness (drop-in for "
               "hadamard_ga.step; one hga_step_host call: H2D, pack, generation, chunked unpack + D2H)")
    return {"value": 2 * N_PAIRS / t, "unit": UNIT, "h2d_bytes_per_step": int(stream_bytes + fit.nbytes + 64),
            "d2h_bytes_per_step": int(stream_bytes + fit.nbytes + 68), "steps": steps, "ms_per_step": t * 1e3,
            "host_population_bytes": int(pop.nbytes), "api": api}


def run_e2e_same_config(args, engine, torch):
    """engine.step() on a host state with rng="reference": the reference's
    splitmix64 streams, seed 2024 and the oracle's initial population, i.e.
    step for step the computation the reference arm (`--impl reference`)
    times; the first step is checked bit for bit against the oracle."""
    import oracle

    @dataclass
    class HostState:
        config: object
        seed: int
        population: np.ndarray
        fitness: np.ndarray
        iteration: int
        best_matrix: np.ndarray
        best_fitness: int
        trace: list = field(default_factory=list)

    cfg = engine.GAConfig(order=ORDER, population=N_PAIRS, seed=2024, fitness=FITNESS, mutation_cols=NC,
                          mutation_row_pairs=NR, max_iterations=engine.MAX_ITERATIONS, rng="reference")
    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    ref = oracle.initial_state(ORDER, N_PAIRS, 2024, FITNESS, NC, NR, "multi", threads=threads)
    hs = HostState(cfg, 2024, ref.population.copy(), ref.fitness.copy(), 0, ref.best_matrix.copy(),
                   ref.best_fitness, [ref.best_fitness])
    engine.step(hs)
    oracle.step(ref, threads)
    identical = bool(np.array_equal(hs.population, ref.population) and np.array_equal(hs.fitness, ref.fitness))
    torch.cuda.synchronize()
    steps = max(3, min(args.steps, 20))
    t0 = time.perf_counter()
    for _ in range(steps):
        engine.step(hs)
    t = (time.perf_counter() - t0) / steps
    bits = hs._hga_bridge.bit_buffers() is not None
    moved = (hs.population.nbytes + 31) // 32 * 4 if bits else hs.population.nbytes
    return {"value": 2 * N_PAIRS / t, "unit": UNIT, "h2d_bytes_per_step": int(moved + hs.fitness.nbytes),
            "d2h_bytes_per_step": int(moved + hs.fitness.nbytes), "steps": steps, "ms_per_step": t * 1e3,
            "rng": "reference", "seed": 2024, "identical_to_reference_arm_step1": identical,
            "api": "engine.step(state) on numpy arrays with GAConfig(rng='reference'): the reference arm's streams, "
                   "seed and initial population (explicit-plan kernels; population moved as a bit stream: "
                   "hga_host_pack_bits -> hga_bits_to_cols ... hga_cols_to_bits -> hga_host_unpack_bits)"}


def run_fitness_sweep(args, engine, torch, lib, peaks):
    """hga_fitness_i8 (the drop-in evaluate) at config-5 sizes, F2, inputs
    larger than L2; each row against its binding ceiling (committed peaks)."""
    sp = torch.cuda.current_stream().cuda_stream
    peak = float(peaks["hbm_gbs"])
    rows = []
    for m in (20, 28, 36, 44, 48, 52, 56, 60, 64):
        n = 4_000_000 if m <= 28 else (2_000_000 if m <= 36 else 1_000_000)
        cfg = engine.GAConfig(order=m, population=n // 4, seed=7)
        pop = engine.init_population_device(cfg)
        out = torch.empty(n, dtype=torch.int64, device=pop.device)
        fn = lambda: lib.hga_fitness_i8(pop.data_ptr(), n, m, 2, None, out.data_ptr(), None, None, None, None, 0, sp)
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn()
            e.record()
            e.synchronize()
            ts.append(s.elapsed_time(e) / 1e3)
        t = statistics.median(ts)
        bytes_ = n * (m * m + 8)
        hbm_ceiling = peak * 1e9 / (m * m + 8)
        ev = n / t
        # orders >= 44 run the Gram on tcgen05 (kind::i8, csrc/fitness_tc2.cu): HBM is that
        # path's roofline; the XOR+POPC kernels are bound by min(HBM, POPC)
        tc = 44 <= m <= 64
        row = {"m": m, "n": n, "path": "tcgen05 kind::i8" if tc else "XOR+POPC", "evals_per_s": ev,
               "GBps": bytes_ / t / 1e9, "hbm_frac": bytes_ / t / 1e9 / peak}
        if tc:
            row.update(binding="hbm", frac_of_binding_ceiling=ev / hbm_ceiling)
            if "mma_64x64x32_per_s_per_sm" in peaks:  # two 64x64x32 MMAs per matrix (K = 64)
                sms = torch.cuda.get_device_properties(0).multi_processor_count
                row["tensor_issue_frac"] = 2 * ev / (peaks["mma_64x64x32_per_s_per_sm"] * sms)
        else:
            popc_ceiling = peaks.get("popc_per_s", float("inf")) / ((m * (m - 1) // 2) * ((m + 31) // 32))
            binding = "hbm" if hbm_ceiling < popc_ceiling else "popc"
            row.update(binding=binding, frac_of_binding_ceiling=ev / min(hbm_ceiling, popc_ceiling))
        rows.append(row)
        del pop, out
        torch.cuda.empty_cache()
    return {"kernel": "hga_fitness_i8 (int8 (n,m,m) drop-in layout, F2)", "inputs": "larger than L2",
            "peaks": {k: v for k, v in peaks.items() if k != "probes"}, "rows": rows}


def run_generation_rows(args, engine, torch, lib, peaks):
    """The production loop at the config-3 / config-4 island sizes (BASELINE
    configs[2] / [3] split over 8 GPUs): one persistent launch of K
    generations after a warm-up launch, per-generation time, and its
    fraction of the HBM and POPC ceilings (algorithmic bytes of section 4
    of DESIGN.md; pair chain without column 0)."""
    from paper_2208_14961_b200._lib import RUN_FORCE, check

    sp = torch.cuda.current_stream().cuda_stream
    rows = []
    for tag, m, n_pairs, nc, nr, gens in (("C3 island (order 28, 1M / 8)", 28, 31_250, 1, 10, 200),
                                          ("C4 island (order 36, 10M / 8)", 36, 312_500, 1, 12, 40)):
        cfg = engine.GAConfig(order=m, population=n_pairs, seed=11, fitness="f2", mutation_cols=nc,
                              mutation_row_pairs=nr, max_iterations=engine.MAX_ITERATIONS)
        st = engine.initial_state(cfg)
        res = st._res
        res.ensure_trace(3 * gens + 8)
        a = res.run_args()
        a.gens_this_call = gens
        a.flags = RUN_FORCE
        check(lib.hga_run(a, sp), "hga_run")  # warm-up launch
        torch.cuda.synchronize()
        a = res.run_args()
        a.gens_this_call = gens
        a.flags = RUN_FORCE
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        check(lib.hga_run(a, sp), "hga_run")
        e.record()
        e.synchronize()
        t = s.elapsed_time(e) / 1e3 / gens
        alg = algorithmic_bytes_per_generation(m, n_pairs)
        pairs = (m - 1) * (m - 2) // 2
        popc = 2 * n_pairs * pairs * ((m + 31) // 32)
        rows.append({"config": tag, "m": m, "matrices": 4 * n_pairs, "nc": nc, "nr": nr, "us_per_generation": t * 1e6,
                     "offspring_evals_per_s": 2 * n_pairs / t, "algorithmic_bytes_per_generation": alg,
                     "hbm_frac": alg / t / 1e9 / float(peaks["hbm_gbs"]),
                     "popc_frac": popc / t / peaks["popc_per_s"] if "popc_per_s" in peaks else None})
        del st, res
        torch.cuda.empty_cache()
    return rows


# ---------------------------------------------------------------- cpu / reference arm


def cpu_baseline(args, budget_s: float = 12.0) -> dict:
    import oracle

    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    st = oracle.initial_state(ORDER, N_PAIRS, 2024, FITNESS, NC, NR, "multi", threads=threads)
    oracle.step(st, threads)
    t0 = time.perf_counter()
    n = 0
    while time.perf_counter() - t0 < budget_s and n < 400:
        oracle.step(st, threads)
        n += 1
    t = time.perf_counter() - t0
    return {"value": 2 * N_PAIRS * n / t, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{n} generations of the same workload (order 20, 40,000 matrices, f2, NC=4, NR=2) by the C "
                      f"oracle (oracle/hga_oracle.c, OpenMP fitness), {t:.1f} s"}


def numpy_reference_timing() -> list | dict:
    """The unmodified NumPy reference (hadamard_ga, installed under baseline/_ref
    when present) timed on this host: evaluate() with 1 / all workers and
    bench._timed_loop at the same workload (scripts/numpy_ref_timing.py).
    Reported beside the C-port arm; the arm's value stays the C port."""
    if not (ROOT / "baseline" / "_ref" / "hadamard_ga").exists():
        return {"unavailable": "baseline/_ref not installed"}
    env = dict(os.environ, OPENBLAS_NUM_THREADS="1")
    try:
        cp = subprocess.run([sys.executable, str(ROOT / "scripts" / "numpy_ref_timing.py"), "--gens", "3"], env=env,
                            capture_output=True, text=True, timeout=240)
        return [json.loads(ln) for ln in cp.stdout.splitlines() if ln.startswith("{")]
    except (OSError, subprocess.TimeoutExpired, ValueError) as exc:
        return {"unavailable": f"{type(exc).__name__}: {exc}"[:200]}


def run_reference(args, rank, world):
    if rank != 0:
        return None
    import oracle

    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    st = oracle.initial_state(ORDER, N_PAIRS, 2024, FITNESS, NC, NR, "multi", threads=threads)
    for _ in range(args.warmup):
        oracle.step(st, threads)
    steps = args.steps
    t0 = time.perf_counter()
    for _ in range(steps):
        oracle.step(st, threads)
    t = time.perf_counter() - t0
    value = 2 * N_PAIRS * steps / t
    numpy_ref = numpy_reference_timing()
    return {
        "numpy_reference": numpy_ref,
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": steps,
        "warmup": args.warmup,
        "ms_per_step": t / steps * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "int8 +-1 (int64 fitness)",
        "data": "synthetic: random balanced sign matrices (reference splitmix64 streams, seed 2024)",
        "config": {"workload": "BASELINE configs[1]: order-20 GA, population 40,000 matrices (N=10,000 pairs), "
                               "fitness f2, mutation multi NC=4 NR=2", "order": ORDER, "matrices": 4 * N_PAIRS,
                   "offspring_evals_per_step": 2 * N_PAIRS, "parallelism": "host threads (OpenMP)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{steps} generations of the full workload by the C oracle port of the reference "
                                   "(oracle/hga_oracle.c; the reference is pure Python/NumPy, nothing to compile)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank, world = env_int("RANK", 0), env_int("WORLD_SIZE", 1)
    local_rank = env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        out = run_reference(args, rank, world)
    else:
        out = run_ours(args, rank, world, local_rank)
    if rank == 0 and out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
