"""numpy-facing wrapper over liboracle.so (TEST INFRASTRUCTURE ONLY).

Names and argument meanings follow the reference package ``hadamard_ga``
(pkg/src/hadamard_ga/engine.py:34-55, rand.py:22) so the parity tests read
like the reference's own tests.  Heavy lifting is in hga_oracle.c; the
run_search driver below restates engine.py:472-538 in Python.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import time
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

__all__ = [
    "FITNESS_CODES",
    "STRATEGY_CODES",
    "load",
    "stream_key",
    "stream_words",
    "uniform_array",
    "permutation",
    "sid",
    "random_balanced",
    "init_population",
    "penalties",
    "evaluate",
    "select",
    "select_indices",
    "draw_crossover_points",
    "crossover",
    "make_mutation_plan",
    "mutate",
    "step",
    "OracleState",
    "initial_state",
    "run_search",
    "max_threads",
]

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "liboracle.so"

FITNESS_CODES = {"f1": 0, "f2": 1, "orth": 2, "sq": 3}
STRATEGY_CODES = {"shared": 0, "per-matrix": 1, "multi": 2}
MASK64 = (1 << 64) - 1

# stream purposes, engine.py:71-77
P_INIT, P_SELECT, P_CROSSOVER, P_MUT_COL, P_MUT_ROW_A, P_MUT_ROW_B, P_RESTART = 1, 2, 3, 4, 5, 6, 7

_lib = None

_i8p = np.ctypeslib.ndpointer(dtype=np.int8, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_u64 = ctypes.c_uint64
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32


def load() -> ctypes.CDLL:
    """Load (building on first use) oracle/liboracle.so."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    lib = ctypes.CDLL(str(LIB_PATH))
    sig = {
        "ora_mix64": (_u64, [_u64]),
        "ora_stream_key": (_u64, [_u64, _u64]),
        "ora_stream_words": (None, [_u64, _u64, _i64, _u64p]),
        "ora_uniform": (None, [_u64, _u64, _u64, _i64, _i64, _i64, _i64p]),
        "ora_permutation": (None, [_u64, _u64, _u64, _i64, _i64p]),
        "ora_sid": (_u64, [_u64, _u64, _u64, _u64]),
        "ora_random_balanced": (None, [_i32, _i64, _u64, _u64, _u64, _i64, _i8p]),
        "ora_penalties": (None, [_i8p, _i64, _i32, ctypes.c_void_p, ctypes.c_void_p,
                                 ctypes.c_void_p, ctypes.c_void_p, _i32]),
        "ora_evaluate": (None, [_i8p, _i64, _i32, _i32, _i64p, _i32]),
        "ora_select_indices": (None, [_i64p, _i64, _u64, _u64, _u64, _i64p]),
        "ora_select": (None, [_i8p, _i64p, _i64, _i32, _u64, _u64, _u64]),
        "ora_crossover": (ctypes.c_int, [_i8p, _i64, _i32, _i64p]),
        "ora_mutation_plan": (None, [_i32, _i64, _i32, _i32, _i32, _u64, _u64, _i64p, _i64p, _i64p]),
        "ora_mutate": (ctypes.c_int, [_i8p, _i64, _i32, _i64p, _i64p, _i64p, _i32, _i32]),
        "ora_step": (_i64, [_i8p, _i64p, _i64, _i32, _u64, _u64, _i32, _i32, _i32, _i32, _i32]),
        "ora_max_threads": (_i32, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def max_threads() -> int:
    return int(load().ora_max_threads())


def _threads(threads: int | None) -> int:
    if threads is None or threads <= 0:
        return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    return int(threads)


# ---------------------------------------------------------------------- rng


def stream_key(seed: int, stream_id: int) -> int:
    return int(load().ora_stream_key(seed & MASK64, stream_id & MASK64))


def stream_words(seed: int, stream_id: int, counter: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.uint64)
    load().ora_stream_words(stream_key(seed, stream_id), counter, n, out)
    return out


def uniform_array(seed: int, stream_id: int, counter: int, lo: int, hi: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.int64)
    load().ora_uniform(seed & MASK64, stream_id & MASK64, counter, lo, hi, n, out)
    return out


def permutation(seed: int, stream_id: int, counter: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.int64)
    load().ora_permutation(seed & MASK64, stream_id & MASK64, counter, n, out)
    return out


def sid(purpose: int, generation: int = 0, matrix: int = 0, column: int = 0) -> int:
    return int(load().ora_sid(purpose, generation, matrix, column))


# ---------------------------------------------------------------------- engine


def random_balanced(order: int, count: int, seed: int, purpose: int, generation: int,
                    first_slot: int) -> np.ndarray:
    out = np.empty((count, order, order), dtype=np.int8)
    load().ora_random_balanced(order, count, seed & MASK64, purpose, generation, first_slot, out)
    return out


def init_population(order: int, n_pairs: int, seed: int) -> np.ndarray:
    return random_balanced(order, 4 * n_pairs, seed, P_INIT, 0, 0)


def penalties(population: np.ndarray, threads: int | None = None) -> np.ndarray:
    """(n, 4) int64: columns f1, f2, orth, sq."""
    pop = np.ascontiguousarray(population, dtype=np.int8)
    n, m = pop.shape[0], pop.shape[1]
    out = np.empty((4, n), dtype=np.int64)
    ptrs = [out[i].ctypes.data_as(ctypes.c_void_p) for i in range(4)]
    load().ora_penalties(pop, n, m, *ptrs, _threads(threads))
    return out.T.copy()


def evaluate(population: np.ndarray, fitness: str = "f2", threads: int | None = None) -> np.ndarray:
    pop = np.ascontiguousarray(population, dtype=np.int8)
    out = np.empty(pop.shape[0], dtype=np.int64)
    load().ora_evaluate(pop, pop.shape[0], pop.shape[1] if pop.ndim == 3 else 0,
                        FITNESS_CODES[fitness], out, _threads(threads))
    return out


def select_indices(fitness_values: np.ndarray, seed: int, stream_id: int, counter: int = 0) -> np.ndarray:
    fit = np.ascontiguousarray(fitness_values, dtype=np.int64)
    out = np.empty(fit.shape[0] // 2, dtype=np.int64)
    load().ora_select_indices(fit, fit.shape[0], seed & MASK64, stream_id & MASK64, counter, out)
    return out


def select(population: np.ndarray, fitness_values: np.ndarray, seed: int, stream_id: int,
           counter: int = 0) -> None:
    assert population.flags.c_contiguous and fitness_values.flags.c_contiguous
    load().ora_select(population, fitness_values, population.shape[0], population.shape[1],
                      seed & MASK64, stream_id & MASK64, counter)


def draw_crossover_points(order: int, n_pairs: int, seed: int, generation: int) -> np.ndarray:
    return uniform_array(seed, sid(P_CROSSOVER, generation), 0, 1, order - 1, n_pairs)


def crossover(population: np.ndarray, points: np.ndarray) -> None:
    pts = np.ascontiguousarray(points, dtype=np.int64)
    if load().ora_crossover(population, population.shape[0], population.shape[1], pts) != 0:
        raise IndexError("crossover point out of range")


def make_mutation_plan(order: int, n_pairs: int, nc: int, nr: int, strategy: str, seed: int,
                       generation: int):
    n_off = 2 * n_pairs
    wc = nc if strategy == "multi" else 1
    wr = nr if strategy == "multi" else 1
    cols = np.empty((n_off, wc), dtype=np.int64)
    ra = np.empty((n_off, wr), dtype=np.int64)
    rb = np.empty((n_off, wr), dtype=np.int64)
    load().ora_mutation_plan(order, n_off, nc, nr, STRATEGY_CODES[strategy], seed & MASK64,
                             generation, cols, ra, rb)
    return cols, ra, rb


def mutate(population: np.ndarray, cols: np.ndarray, ra: np.ndarray, rb: np.ndarray) -> None:
    cols = np.ascontiguousarray(cols, dtype=np.int64)
    ra = np.ascontiguousarray(ra, dtype=np.int64)
    rb = np.ascontiguousarray(rb, dtype=np.int64)
    rc = load().ora_mutate(population, population.shape[0], population.shape[1], cols, ra, rb,
                           cols.shape[1], ra.shape[1])
    if rc != 0:
        raise IndexError("mutation plan index out of range")


# ---------------------------------------------------------------------- loop


@dataclass
class OracleState:
    order: int
    n_pairs: int
    seed: int
    fitness_name: str
    nc: int
    nr: int
    strategy: str
    population: np.ndarray
    fitness: np.ndarray
    iteration: int = 0
    best_fitness: int = 0
    best_matrix: np.ndarray | None = None
    trace: list = field(default_factory=list)


def initial_state(order: int, n_pairs: int, seed: int, fitness: str = "f2", nc: int = 1,
                  nr: int = 2, strategy: str = "multi", threads: int | None = None) -> OracleState:
    pop = init_population(order, n_pairs, seed)
    fit = evaluate(pop, fitness, threads)
    b = int(fit.argmin())
    return OracleState(order, n_pairs, seed & MASK64, fitness, nc, nr, strategy, pop, fit, 0,
                       int(fit[b]), pop[b].copy(), [int(fit[b])])


def step(st: OracleState, threads: int | None = None) -> OracleState:
    gen = st.iteration + 1
    b = int(load().ora_step(st.population, st.fitness, st.population.shape[0], st.order, st.seed,
                            gen, st.nc, st.nr, STRATEGY_CODES[st.strategy],
                            FITNESS_CODES[st.fitness_name], _threads(threads)))
    st.iteration = gen
    fmin = int(st.fitness[b])
    st.trace.append(fmin)
    if fmin < st.best_fitness:
        st.best_fitness = fmin
        st.best_matrix = st.population[b].copy()
    return st


def run_search(order: int, n_pairs: int, seed: int, fitness: str = "f2", nc: int = 1, nr: int = 2,
               strategy: str = "multi", max_iterations: int = 100_000, stall_window: int | None = None,
               time_budget_secs: float | None = None, threads: int | None = None) -> dict:
    """engine.run_search (engine.py:497-538) restated over the C step."""
    start = time.perf_counter()
    st = initial_state(order, n_pairs, seed, fitness, nc, nr, strategy, threads)
    complete, last_restart = True, 0
    while st.iteration < max_iterations and st.best_fitness > 0:
        if time_budget_secs is not None and time.perf_counter() - start > time_budget_secs:
            complete = False
            break
        step(st, threads)
        if (stall_window is not None and st.best_fitness > 0
                and st.iteration - last_restart >= stall_window):
            tail = st.trace[-stall_window:]
            if len(tail) == stall_window and tail[-1] != 0 and all(v == tail[0] for v in tail):
                half = 2 * n_pairs
                fresh = random_balanced(order, half, st.seed, P_RESTART, st.iteration, half)
                st.population[half:] = fresh
                st.fitness[half:] = evaluate(fresh, fitness, threads)
                b = int(st.fitness.argmin())
                if int(st.fitness[b]) < st.best_fitness:
                    st.best_fitness = int(st.fitness[b])
                    st.best_matrix = st.population[b].copy()
                last_restart = st.iteration
    return dict(success=st.best_fitness == 0, complete=complete or st.best_fitness == 0,
                iterations=st.iteration, best_fitness=st.best_fitness, best_matrix=st.best_matrix,
                trace=list(st.trace), wall_seconds=time.perf_counter() - start, seed=st.seed)
