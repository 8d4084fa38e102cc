"""GA inner loop on B200 -- drop-in for hadamard_ga.engine (engine.py:1-538).

Same names, argument order, return types and errors as the reference's
engine module (engine.py:34-55); the work runs in sm_100a kernels through
libhga (include/hga.h), with torch owning device memory.  No CPU fallback.

Population layouts
    * API edge: the reference's int8 (4N, m, m) row-major array, as numpy
      (copied to/from the GPU) or as a CUDA int8 tensor (used in place).
    * Resident (SearchState): bit-packed columns, m * ceil(m/32) uint32
      words per matrix (12.5-25x smaller than int8), ping-pong buffers.

Random streams (GAConfig.rng)
    * "reference": the reference's splitmix64 counter streams, reproduced on
      device bit-for-bit; a seeded run returns the identical RunRecord
      (trace, iterations, best matrix) as hadamard_ga.run_search.  Population
      limits are the reference's (its stream-id packing, engine.py:60-69).
    * "philox" (default): per-thread Philox4x32-10 draws inside ONE
      persistent kernel per batch of generations (csrc/generation.cu);
      same operators and selection rule, different random numbers, no
      host round trip per generation, populations up to 2^31 matrices.

Fitness choices are the reference's "f1" and "f2" plus "sq" (sum of squared
off-diagonal Gram entries); `evaluate` also returns "orth" (number of
orthogonal column pairs), and `penalties` returns all four from one pass.
"""

from __future__ import annotations

import ctypes
import os
import time
import weakref
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _dev
from ._dev import HgaError, check, lib, ptr, stream_ptr, words_for
from ._lib import (FLAG_FIT_RANGE, FLAG_NOT_GA, FLAG_NOT_SIGN, FLAG_PLAN_RANGE, FLAG_POINT_RANGE, HGA_E_UNSUPPORTED,
                   MUT_CODES, RUN_FORCE, RunArgs, VARIANT_BITS)
from .rand import MASK64, RngStream, random_seed

__all__ = [
    "FITNESS_CHOICES",
    "PENALTY_NAMES",
    "MUTATION_STRATEGIES",
    "RNG_MODES",
    "MAX_ORDER",
    "MAX_POPULATION",
    "MAX_POPULATION_PHILOX",
    "MAX_ITERATIONS",
    "GAConfig",
    "MutationPlan",
    "SearchState",
    "RunRecord",
    "init_population",
    "evaluate",
    "penalties",
    "select",
    "draw_crossover_points",
    "crossover",
    "make_mutation_plan",
    "mutate",
    "initial_state",
    "step",
    "detect_stall",
    "run_search",
]

FITNESS_CHOICES = ("f1", "f2", "sq")
PENALTY_NAMES = ("f1", "f2", "orth", "sq")
MUTATION_STRATEGIES = ("shared", "per-matrix", "multi")
RNG_MODES = ("philox", "reference")

_GEN_BITS, _MATRIX_BITS, _COL_BITS = 28, 20, 12
MAX_ORDER = 1 << _COL_BITS
MAX_POPULATION = (1 << _MATRIX_BITS) // 4       # reference-stream limit (engine.py:68)
MAX_POPULATION_PHILOX = ((1 << 31) - 1) // 4     # 32-bit slot ids in the select keys
MAX_ITERATIONS = (1 << _GEN_BITS) - 1
MAX_RESIDENT_ORDER = 128                         # register-resident column words (W <= 4)

_P_INIT, _P_SELECT, _P_CROSSOVER, _P_MUT_COL, _P_MUT_ROW_A, _P_MUT_ROW_B, _P_RESTART = 1, 2, 3, 4, 5, 6, 7

DEBUG_CHECKS = False
_RUN_FLAGS = 0  # extra hga_run_args.flags for every persistent-loop call (tests: RUN_TWO_BARRIER)


def _sid(purpose: int, generation: int = 0, matrix: int = 0, column: int = 0) -> int:
    """Stream id packing (engine.py:84-90)."""
    return (purpose << 60) | (generation << 32) | (matrix << 12) | column


# ============================================================== config


@dataclass(frozen=True)
class GAConfig:
    """All parameters of one search (engine.py:93-151) plus `rng`."""

    order: int
    population: int = 1000
    max_iterations: int = 100_000
    mutation_cols: int = 1
    mutation_row_pairs: int = 2
    fitness: str = "f2"
    mutation: str = "multi"
    seed: int | None = None
    stall_window: int | None = None
    time_budget_secs: float | None = None
    rng: str = "philox"

    def __post_init__(self):
        m = self.order
        if not isinstance(m, int) or m < 4 or m % 4 != 0:
            raise ValueError(f"order must be a positive multiple of 4, got {m}")
        if m > MAX_ORDER:
            raise ValueError(f"order {m} exceeds engine limit {MAX_ORDER}")
        if self.rng not in RNG_MODES:
            raise ValueError(f"rng must be one of {RNG_MODES}")
        cap = MAX_POPULATION if self.rng == "reference" else MAX_POPULATION_PHILOX
        if not 1 <= self.population <= cap:
            raise ValueError(f"population must be in [1, {cap}]")
        if not 0 <= self.max_iterations <= MAX_ITERATIONS:
            raise ValueError(f"max_iterations must be in [0, {MAX_ITERATIONS}]")
        if not 1 <= self.mutation_cols <= m - 1:
            raise ValueError(f"mutation_cols must be in [1, {m - 1}]")
        if not 1 <= self.mutation_row_pairs <= m // 2:
            raise ValueError(f"mutation_row_pairs must be in [1, {m // 2}]")
        if self.fitness not in FITNESS_CHOICES:
            raise ValueError(f"fitness must be one of {FITNESS_CHOICES}")
        if self.mutation not in MUTATION_STRATEGIES:
            raise ValueError(f"mutation must be one of {MUTATION_STRATEGIES}")
        if self.seed is not None and not isinstance(self.seed, int):
            raise ValueError("seed must be an integer or None")
        if self.stall_window is not None and self.stall_window < 1:
            raise ValueError("stall_window must be >= 1")
        if self.time_budget_secs is not None and self.time_budget_secs <= 0:
            raise ValueError("time_budget_secs must be positive")
        if self.fitness == "sq" and m > 64:
            raise ValueError("fitness 'sq' is limited to order <= 64 (24-bit selection keys)")

    @property
    def k(self) -> int:
        return self.order // 4

    @property
    def parents(self) -> int:
        return 2 * self.population

    @property
    def total(self) -> int:
        return 4 * self.population


# ============================================================== helpers


def _is_numpy(a) -> bool:
    return not isinstance(a, torch.Tensor)


def _check_flag(flag: torch.Tensor, what: str) -> None:
    v = int(flag.item())
    if v & FLAG_NOT_SIGN:
        raise ValueError(f"{what}: matrix entries must be +1 or -1")
    if v & FLAG_POINT_RANGE:
        raise IndexError(f"{what}: crossover point out of range")
    if v & FLAG_PLAN_RANGE:
        raise IndexError(f"{what}: mutation plan index out of range")
    if v & FLAG_FIT_RANGE:
        raise ValueError(f"{what}: fitness values span more than {int(lib.hga_select_max_range())}")


def _pop_shape(pop) -> tuple[int, int]:
    if pop.ndim != 3 or pop.shape[1] != pop.shape[2]:
        raise ValueError(f"expected a (n, m, m) population, got shape {tuple(pop.shape)}")
    return int(pop.shape[0]), int(pop.shape[1])


def _copy_back(host: np.ndarray, dev: torch.Tensor) -> None:
    host[...] = dev.cpu().numpy().reshape(host.shape)


# ============================================================== fitness


def _penalties_dev(pop: torch.Tensor, variants: int, check_sign: bool = True):
    n, m = _pop_shape(pop)
    dev = pop.device
    outs = {}
    for name, bit in VARIANT_BITS.items():
        outs[name] = torch.empty(n, dtype=torch.int64, device=dev) if variants & bit else None
    if n == 0:
        return outs
    flag = _dev.new_flag()
    wsb = int(lib.hga_fitness_i8_ws_bytes(n, m))
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev) if wsb else None
    check(lib.hga_fitness_i8(pop.data_ptr(), n, m, variants, ptr(outs["f1"]), ptr(outs["f2"]), ptr(outs["orth"]),
                             ptr(outs["sq"]), flag.data_ptr(), ptr(ws), wsb, stream_ptr()), "hga_fitness_i8")
    if check_sign:
        _check_flag(flag, "evaluate")
    return outs


def evaluate(population, fitness: str = "f2", workers: int = 1):
    """Fitness vector aligned with `population` (engine.py:216-230).

    numpy in -> numpy int64 out; CUDA int8 tensor in -> CUDA int64 tensor
    out.  `workers` is accepted for signature compatibility: the GPU grid
    replaces the reference's thread pool (results never depend on it).
    """
    if fitness not in PENALTY_NAMES:
        raise ValueError(f"fitness must be one of {FITNESS_CHOICES} (or 'orth')")
    host = _is_numpy(population)
    pop, _ = _dev.to_device(population, torch.int8)
    out = _penalties_dev(pop, VARIANT_BITS[fitness])[fitness]
    return out.cpu().numpy() if host else out


def penalties(population) -> dict:
    """All four penalties (f1, f2, orth, sq) from one fused pass."""
    host = _is_numpy(population)
    pop, _ = _dev.to_device(population, torch.int8)
    outs = _penalties_dev(pop, 15)
    return {k: (v.cpu().numpy() if host else v) for k, v in outs.items()}


# ============================================================== init


def _init_packed(config: GAConfig, seed: int, purpose: int, generation: int, first_slot: int, count: int,
                 out: torch.Tensor) -> None:
    """Reference-stream balanced matrices into packed `out` (engine.py:154-182)."""
    check(lib.hga_ref_init_packed(seed & MASK64, purpose, generation, first_slot, count, config.order,
                                  out.data_ptr(), stream_ptr()), "hga_ref_init_packed")


def _unpack(packed: torch.Tensor, n: int, m: int) -> torch.Tensor:
    out = torch.empty((n, m, m), dtype=torch.int8, device=packed.device)
    if n:
        check(lib.hga_unpack_i8(packed.data_ptr(), n, m, out.data_ptr(), stream_ptr()), "hga_unpack_i8")
    return out


def _pack(pop: torch.Tensor) -> torch.Tensor:
    n, m = _pop_shape(pop)
    out = torch.empty(n * m * words_for(m), dtype=torch.int32, device=pop.device)
    flag = _dev.new_flag()
    if n:
        check(lib.hga_pack_i8(pop.data_ptr(), n, m, out.data_ptr(), flag.data_ptr(), stream_ptr()), "hga_pack_i8")
        _check_flag(flag, "pack")
    return out


def init_population_device(config: GAConfig, seed: int | None = None) -> torch.Tensor:
    """(4N, m, m) int8 CUDA tensor of the initial population.

    rng="reference": the reference's streams, bit-identical to
    hadamard_ga.init_population; rng="philox": the production streams.
    """
    if seed is None:
        seed = config.seed
    if seed is None:
        raise ValueError("init_population needs an explicit seed")
    dev = _dev.require_cuda()
    m, total = config.order, config.total
    if config.rng == "philox" and m <= MAX_RESIDENT_ORDER:
        packed = torch.empty(total * m * words_for(m), dtype=torch.int32, device=dev)
        check(lib.hga_philox_init_packed(seed & MASK64, _P_INIT, 0, 0, total, m, packed.data_ptr(), stream_ptr()),
              "hga_philox_init_packed")
        return _unpack(packed, total, m)
    out = torch.empty((total, m, m), dtype=torch.int8, device=dev)
    if m <= MAX_RESIDENT_ORDER:
        check(lib.hga_ref_init_i8(seed & MASK64, _P_INIT, 0, 0, total, m, out.data_ptr(), stream_ptr()),
              "hga_ref_init_i8")
        return out
    packed = torch.empty(total * m * words_for(m), dtype=torch.int32, device=dev)
    _init_packed(config, seed, _P_INIT, 0, 0, total, packed)
    return _unpack(packed, total, m)


def init_population(config: GAConfig, seed: int | None = None) -> np.ndarray:
    """Initial population of 4N balanced matrices (engine.py:185-197); with
    rng="reference" bit-identical to the reference's for the same seed."""
    return init_population_device(config, seed).cpu().numpy()


# ============================================================== operators


def select(population, fitness_values, stream) -> None:
    """Move the 2N fittest into the parent slots in random order, in place
    (engine.py:233-248; ties toward lower index; `stream` is an RngStream,
    ours or the reference's, and advances by 2N-1 draws like the reference's).
    """
    half = population.shape[0] // 2
    host_pop, host_fit = _is_numpy(population), _is_numpy(fitness_values)
    pop, _ = _dev.to_device(population, torch.int8)
    fit, _ = _dev.to_device(fitness_values, torch.int64)
    if half == 0:
        return
    if not host_pop and pop.data_ptr() != population.data_ptr():
        raise ValueError("device population must be a contiguous int8 tensor")
    if not host_fit and fit.data_ptr() != fitness_values.data_ptr():
        raise ValueError("device fitness must be a contiguous int64 tensor")
    dev = pop.device
    total = fit.shape[0]
    order = torch.empty(half, dtype=torch.int64, device=dev)
    wsb = int(lib.hga_select_ws_bytes(total))
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    flag = _dev.new_flag()
    check(lib.hga_select_order(fit.data_ptr(), total, order.data_ptr(), flag.data_ptr(), ws.data_ptr(), wsb,
                               stream_ptr()), "hga_select_order")
    if int(flag.item()) & FLAG_FIT_RANGE:  # values span more than the histogram: stable radix sort
        _select_radix(fit, total, half, order)
    seed, sid, counter = int(stream.seed), int(stream.stream_id), int(stream.counter)
    perm = torch.empty(half, dtype=torch.int64, device=dev)
    pwsb = int(lib.hga_ref_permutation_ws_bytes(half))
    pws = torch.empty(max(pwsb, 1), dtype=torch.uint8, device=dev)
    check(lib.hga_ref_permutation(seed & MASK64, sid & MASK64, counter, half, perm.data_ptr(), pws.data_ptr(), pwsb,
                                  stream_ptr()), "hga_ref_permutation")
    stream.counter += half - 1
    m = pop.shape[1]
    tmp = torch.empty((half, m, m), dtype=torch.int8, device=dev)
    ftmp = torch.empty(half, dtype=torch.int64, device=dev)
    check(lib.hga_compose_gather(order.data_ptr(), perm.data_ptr(), half, pop.data_ptr(), tmp.data_ptr(), m * m,
                                 fit.data_ptr(), ftmp.data_ptr(), None, stream_ptr()), "hga_compose_gather")
    pop[:half].copy_(tmp)
    fit[:half].copy_(ftmp)
    if host_pop:
        _copy_back(population, pop)
    if host_fit:
        _copy_back(fitness_values, fit)


def _select_radix(fit: torch.Tensor, total: int, k: int, order: torch.Tensor) -> None:
    """order[:k] = the first k indices of the stable argsort of fit (any int64 values)."""
    wsb = int(lib.hga_select_radix_ws_bytes(total))
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=fit.device)
    check(lib.hga_select_smallest_radix(fit.data_ptr(), total, k, order.data_ptr(), ws.data_ptr(), wsb, stream_ptr()),
          "hga_select_smallest_radix")


def _fitness_bound(m: int, fit_var: int) -> int:
    """Largest value the GA fitness variant can take at order m."""
    return {1: m * m * (m - 1), 2: m * (m - 1), 8: m ** 3 * (m - 1)}[fit_var]


def draw_crossover_points(config: GAConfig, seed: int, generation: int) -> np.ndarray:
    """One split column per parent pair, uniform in [1, m-1] (engine.py:251-254)."""
    return RngStream(seed, _sid(_P_CROSSOVER, generation)).uniform_array(1, config.order - 1, config.population)


def crossover(population, points) -> None:
    """Rebuild all offspring from the parent pairs, in place (engine.py:257-277)."""
    n_pairs = population.shape[0] // 4
    m = population.shape[1]
    pts_np = points.cpu().numpy() if isinstance(points, torch.Tensor) else np.asarray(points)
    if pts_np.shape != (n_pairs,):
        raise ValueError(f"expected {n_pairs} crossover points, got {pts_np.shape}")
    if n_pairs and (pts_np.min() < 1 or pts_np.max() > m - 1):
        raise IndexError(f"crossover points must lie in [1, {m - 1}]")
    host = _is_numpy(population)
    pop, _ = _dev.to_device(population, torch.int8)
    pts, _ = _dev.to_device(pts_np.astype(np.int64), torch.int64)
    flag = _dev.new_flag()
    check(lib.hga_crossover_i8(pop.data_ptr(), pop.shape[0], m, pts.data_ptr(), flag.data_ptr(), stream_ptr()),
          "hga_crossover_i8")
    _check_flag(flag, "crossover")
    if host:
        _copy_back(population, pop)


@dataclass(frozen=True)
class MutationPlan:
    """Flip targets for the 2N offspring (engine.py:280-302)."""

    columns: np.ndarray
    rows_a: np.ndarray
    rows_b: np.ndarray

    def __post_init__(self):
        if self.columns.ndim != 2 or self.rows_a.ndim != 2 or self.rows_b.ndim != 2:
            raise ValueError("plan arrays must be 2-D")
        if self.rows_a.shape != self.rows_b.shape:
            raise ValueError("row index arrays must have equal shapes")
        if self.columns.shape[0] != self.rows_a.shape[0]:
            raise ValueError("plan arrays must agree on offspring count")
        if self.columns.size and self.columns.min() < 1:
            raise IndexError("column 0 may not be mutated")


def _plan_device(config: GAConfig, seed: int, generation: int):
    """(cols, ra, rb) int64 CUDA tensors of the reference plan (engine.py:305-336)."""
    m, n_off = config.order, config.parents
    sc, sa, sb = _sid(_P_MUT_COL, generation), _sid(_P_MUT_ROW_A, generation), _sid(_P_MUT_ROW_B, generation)
    from .rand import device_uniform

    if config.mutation == "shared":
        c = device_uniform(seed, sc, 0, 1, m - 1, 1)
        a = device_uniform(seed, sa, 0, 0, m - 1, 1)
        b = device_uniform(seed, sb, 0, 0, m - 1, 1)
        return (c.expand(n_off).reshape(n_off, 1).contiguous(), a.expand(n_off).reshape(n_off, 1).contiguous(),
                b.expand(n_off).reshape(n_off, 1).contiguous())
    nc = 1 if config.mutation == "per-matrix" else config.mutation_cols
    nr = 1 if config.mutation == "per-matrix" else config.mutation_row_pairs
    return (device_uniform(seed, sc, 0, 1, m - 1, n_off * nc).reshape(n_off, nc),
            device_uniform(seed, sa, 0, 0, m - 1, n_off * nr).reshape(n_off, nr),
            device_uniform(seed, sb, 0, 0, m - 1, n_off * nr).reshape(n_off, nr))


def make_mutation_plan(config: GAConfig, seed: int, generation: int) -> MutationPlan:
    """Draw the mutation plan for one generation (engine.py:305-336)."""
    c, a, b = _plan_device(config, seed, generation)
    return MutationPlan(columns=c.cpu().numpy(), rows_a=a.cpu().numpy(), rows_b=b.cpu().numpy())


def mutate(population, plan: MutationPlan) -> None:
    """Apply the plan to the offspring half, in place (engine.py:339-373)."""
    total, m = population.shape[0], population.shape[1]
    half = total // 2
    cols_np, ra_np, rb_np = (np.asarray(x) for x in (plan.columns, plan.rows_a, plan.rows_b))
    n_off = cols_np.shape[0]
    if n_off != half:
        raise ValueError(f"plan covers {n_off} offspring, population has {half}")
    if cols_np.size and cols_np.max() > m - 1:
        raise IndexError(f"plan column beyond order {m}")
    for arr in (ra_np, rb_np):
        if arr.size and (arr.min() < 0 or arr.max() > m - 1):
            raise IndexError("plan row index out of range")
    host = _is_numpy(population)
    pop, _ = _dev.to_device(population, torch.int8)
    c, _ = _dev.to_device(cols_np.astype(np.int64), torch.int64)
    a, _ = _dev.to_device(ra_np.astype(np.int64), torch.int64)
    b, _ = _dev.to_device(rb_np.astype(np.int64), torch.int64)
    flag = _dev.new_flag()
    check(lib.hga_mutate_i8(pop.data_ptr(), total, m, c.data_ptr(), a.data_ptr(), b.data_ptr(), cols_np.shape[1],
                            ra_np.shape[1], flag.data_ptr(), stream_ptr()), "hga_mutate_i8")
    _check_flag(flag, "mutate")
    if host:
        _copy_back(population, pop)


# ============================================================== search state


@dataclass
class RunRecord:
    """Outcome of one search run (engine.py:390-402)."""

    config: GAConfig
    seed: int
    success: bool
    complete: bool
    iterations: int
    best_fitness: int
    best_matrix: np.ndarray
    trace: list[int]
    wall_seconds: float


class _Resident:
    """Device side of a SearchState: packed ping-pong population + fitness."""

    def __init__(self, config: GAConfig, seed: int):
        self.config = config
        self.seed = seed
        self.dev = _dev.require_cuda()
        m, N = config.order, config.population
        self.m, self.N, self.W = m, N, words_for(m)
        self.mw = m * self.W
        total = 4 * N
        self.pop = [torch.empty(total * self.mw, dtype=torch.int32, device=self.dev) for _ in range(2)]
        self.fit = [torch.empty(total, dtype=torch.int64, device=self.dev) for _ in range(2)]
        self.cur = 0
        self.fit_var = VARIANT_BITS[config.fitness]
        self.best_packed = torch.zeros(self.mw, dtype=torch.int32, device=self.dev)
        self.dstate = torch.zeros(8, dtype=torch.int64, device=self.dev)
        self.trace_dev = torch.zeros(1024, dtype=torch.int64, device=self.dev)
        self.key = torch.zeros(1, dtype=torch.int64, device=self.dev)
        self.run_ws = None
        self.host_state = None
        self.sel_ws = None
        self.perm_ws = None

    # -- argmin over a fitness buffer, lowest index on ties
    def argmin(self, fit: torch.Tensor) -> tuple[int, int]:
        check(lib.hga_argmin_key(fit.data_ptr(), fit.shape[0], self.key.data_ptr(), 1, stream_ptr()), "argmin")
        k = int(self.key.item()) & MASK64
        return k >> 32, k & 0xFFFFFFFF

    def matrix(self, buf: int, idx: int) -> torch.Tensor:
        return self.pop[buf][idx * self.mw:(idx + 1) * self.mw]

    def run_args(self) -> RunArgs:
        cfg = self.config
        if self.run_ws is None:
            wsb = int(lib.hga_run_ws_bytes(self.N, self.m))
            self.run_ws = torch.zeros(wsb, dtype=torch.uint8, device=self.dev)
        a = RunArgs()
        a.pop[0], a.pop[1] = self.pop[0].data_ptr(), self.pop[1].data_ptr()
        a.fit[0], a.fit[1] = self.fit[0].data_ptr(), self.fit[1].data_ptr()
        a.n_pairs, a.m = self.N, self.m
        a.nc, a.nr = cfg.mutation_cols, cfg.mutation_row_pairs
        a.strategy = MUT_CODES[cfg.mutation]
        a.fit_var = self.fit_var
        a.stall_window = cfg.stall_window or 0
        a.seed = self.seed & MASK64
        a.max_generation = cfg.max_iterations
        a.gens_this_call = 0
        a.state = self.dstate.data_ptr()
        a.trace = self.trace_dev.data_ptr()
        a.trace_capacity = self.trace_dev.shape[0]
        a.best_matrix = self.best_packed.data_ptr()
        a.ws = self.run_ws.data_ptr()
        a.ws_bytes = self.run_ws.shape[0]
        a.flags = _RUN_FLAGS
        return a

    def ensure_trace(self, upto: int) -> None:
        cap = self.trace_dev.shape[0]
        if upto < cap:
            return
        new = max(upto + 1, 2 * cap)
        t = torch.zeros(new, dtype=torch.int64, device=self.dev)
        t[:cap].copy_(self.trace_dev)
        self.trace_dev = t


class SearchState:
    """Mutable state of a running search (engine.py:376-387).

    The population lives on the GPU (packed); `population`, `fitness` and
    `best_matrix` materialise reference-layout numpy copies on access.
    """

    def __init__(self, config: GAConfig, seed: int, res: _Resident, iteration: int, best_fitness: int,
                 trace: list[int], best_matrix: np.ndarray):
        self.config = config
        self.seed = seed
        self._res = res
        self.iteration = iteration
        self.best_fitness = best_fitness
        self.trace = trace
        self.best_matrix = best_matrix
        self._last_restart = 0

    @property
    def population(self) -> np.ndarray:
        return self.population_device.cpu().numpy()

    @property
    def population_device(self) -> torch.Tensor:
        r = self._res
        if isinstance(r, _ResidentI8):
            return r.pop[r.cur]
        return _unpack(r.pop[r.cur], 4 * r.N, r.m)

    @property
    def packed_population(self) -> torch.Tensor:
        r = self._res
        if isinstance(r, _ResidentI8):
            return _pack(r.pop[r.cur]).view(4 * r.N, r.m, r.W)
        return r.pop[r.cur].view(4 * r.N, r.m, r.W)

    @property
    def fitness(self) -> np.ndarray:
        r = self._res
        return r.fit[r.cur].cpu().numpy()

    @property
    def fitness_device(self) -> torch.Tensor:
        r = self._res
        return r.fit[r.cur]


def _best_from_packed(res: _Resident, packed: torch.Tensor) -> np.ndarray:
    return _unpack(packed, 1, res.m)[0].cpu().numpy()


def initial_state(config: GAConfig, seed: int | None = None, workers: int = 1) -> SearchState:
    """Initialise and evaluate the full population (engine.py:405-428)."""
    if seed is None:
        seed = config.seed if config.seed is not None else random_seed()
    seed &= MASK64
    if config.order > MAX_RESIDENT_ORDER:
        return _initial_state_i8(config, seed)
    res = _Resident(config, seed)
    m, total = config.order, config.total
    if config.rng == "reference":
        _init_packed(config, seed, _P_INIT, 0, 0, total, res.pop[0])
        fvar = res.fit_var
        out = res.fit[0]
        check(lib.hga_fitness_packed(res.pop[0].data_ptr(), total, m, fvar, ptr(out) if fvar == 1 else None,
                                     ptr(out) if fvar == 2 else None, None, ptr(out) if fvar == 8 else None,
                                     stream_ptr()), "hga_fitness_packed")
        best, idx = res.argmin(res.fit[0])
        res.best_packed.copy_(res.matrix(0, idx))
        res.dstate.copy_(torch.tensor([0, best, 0, 0, idx, int(best == 0), 1, best], dtype=torch.int64))
    else:
        a = res.run_args()
        check(lib.hga_run_init(a, stream_ptr()), "hga_run_init")
        st = res.dstate.cpu().tolist()
        best = int(st[1])
    return SearchState(config, seed, res, 0, int(best), [int(best)], _best_from_packed(res, res.best_packed))


class _ResidentI8:
    """Device side of a SearchState at orders above MAX_RESIDENT_ORDER (up to the
    reference's 4096, engine.py:57): the reference's own int8 (4N, m, m)
    layout in ping-pong buffers, advanced by the explicit-plan operator
    kernels (select / permutation / gather, crossover_i8, mutate_i8,
    fitness_i8) with the reference's counter streams, so a seeded run is the
    reference's run.  (Orders <= 128 use the packed resident loops.)"""

    def __init__(self, config: GAConfig, seed: int):
        self.config = config
        self.seed = seed
        self.dev = _dev.require_cuda()
        m, N = config.order, config.population
        self.m, self.N, self.W = m, N, words_for(m)
        total = 4 * N
        self.pop = [torch.empty((total, m, m), dtype=torch.int8, device=self.dev) for _ in range(2)]
        self.fit = [torch.empty(total, dtype=torch.int64, device=self.dev) for _ in range(2)]
        self.cur = 0
        self.fit_var = VARIANT_BITS[config.fitness]
        self.key = torch.zeros(1, dtype=torch.int64, device=self.dev)
        wsb = int(lib.hga_fitness_i8_ws_bytes(total, m))
        self.fws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=self.dev)
        self.sel_ws = torch.empty(int(lib.hga_select_ws_bytes(total)), dtype=torch.uint8, device=self.dev)
        pwsb = int(lib.hga_ref_permutation_ws_bytes(2 * N))
        self.perm_ws = torch.empty(max(pwsb, 1), dtype=torch.uint8, device=self.dev)

    argmin = _Resident.argmin

    def init_slots(self, buf: int, purpose: int, generation: int, first: int, count: int) -> None:
        """Reference-stream balanced matrices (engine.py:154-182) into slots [first, first+count)."""
        m, W = self.m, self.W
        step_ = max(1, min(count, (64 << 20) // (m * W * 4)))
        packed = torch.empty(step_ * m * W, dtype=torch.int32, device=self.dev)
        for a in range(first, first + count, step_):
            c = min(step_, first + count - a)
            # streams of slots [a, a + c), written from the start of `packed`
            check(lib.hga_ref_init_packed(self.seed & MASK64, purpose, generation, a, c, m, packed.data_ptr(),
                                          stream_ptr()),
                  "hga_ref_init_packed")
            check(lib.hga_unpack_i8(packed.data_ptr(), c, m, self.pop[buf][a].data_ptr(), stream_ptr()),
                  "hga_unpack_i8")

    def evaluate(self, buf: int, first: int, count: int) -> None:
        fv = self.fit_var
        out = self.fit[buf][first:first + count]
        check(lib.hga_fitness_i8(self.pop[buf][first].data_ptr(), count, self.m, fv, ptr(out) if fv == 1 else None,
                                 ptr(out) if fv == 2 else None, None, ptr(out) if fv == 8 else None, None,
                                 self.fws.data_ptr(), self.fws.shape[0], stream_ptr()), "hga_fitness_i8")


def _initial_state_i8(config: GAConfig, seed: int) -> SearchState:
    res = _ResidentI8(config, seed)
    total = config.total
    res.init_slots(0, _P_INIT, 0, 0, total)
    res.evaluate(0, 0, total)
    best, idx = res.argmin(res.fit[0])
    return SearchState(config, seed, res, 0, int(best), [int(best)], res.pop[0][idx].cpu().numpy())


def _step_i8(state: SearchState) -> None:
    """One reference generation on the int8 layout (engine.py:449-469)."""
    res, cfg = state._res, state.config
    gen = state.iteration + 1
    N, m, half, total = res.N, res.m, 2 * res.N, 4 * res.N
    cur, nxt = res.cur, res.cur ^ 1
    sp = stream_ptr()
    order = torch.empty(half, dtype=torch.int64, device=res.dev)
    if _fitness_bound(m, res.fit_var) < int(lib.hga_select_max_range()):
        flag = _dev.new_flag()
        check(lib.hga_select_order(res.fit[cur].data_ptr(), total, order.data_ptr(), flag.data_ptr(),
                                   res.sel_ws.data_ptr(), res.sel_ws.shape[0], sp), "hga_select_order")
    else:
        _select_radix(res.fit[cur], total, half, order)
    perm = torch.empty(half, dtype=torch.int64, device=res.dev)
    check(lib.hga_ref_permutation(state.seed, _sid(_P_SELECT, gen), 0, half, perm.data_ptr(), res.perm_ws.data_ptr(),
                                  res.perm_ws.shape[0], sp), "hga_ref_permutation")
    check(lib.hga_compose_gather(order.data_ptr(), perm.data_ptr(), half, res.pop[cur].data_ptr(),
                                 res.pop[nxt].data_ptr(), m * m, res.fit[cur].data_ptr(), res.fit[nxt].data_ptr(),
                                 None, sp), "hga_compose_gather")
    from .rand import device_uniform

    points = device_uniform(state.seed, _sid(_P_CROSSOVER, gen), 0, 1, m - 1, N)
    flag = _dev.new_flag()
    check(lib.hga_crossover_i8(res.pop[nxt].data_ptr(), total, m, points.data_ptr(), flag.data_ptr(), sp),
          "hga_crossover_i8")
    cols, ra, rb = _plan_device(cfg, state.seed, gen)
    check(lib.hga_mutate_i8(res.pop[nxt].data_ptr(), total, m, cols.data_ptr(), ra.data_ptr(), rb.data_ptr(),
                            cols.shape[1], ra.shape[1], flag.data_ptr(), sp), "hga_mutate_i8")
    res.evaluate(nxt, half, half)
    res.cur = nxt
    fmin, idx = res.argmin(res.fit[nxt])
    _check_flag(flag, "step")
    state.iteration = gen
    state.trace.append(fmin)
    if fmin < state.best_fitness:
        state.best_fitness = fmin
        state.best_matrix = res.pop[nxt][idx].cpu().numpy()


def _reinitialize_offspring_i8(state: SearchState) -> None:
    res = state._res
    half, total = 2 * res.N, 4 * res.N
    res.init_slots(res.cur, _P_RESTART, state.iteration, half, half)
    res.evaluate(res.cur, half, half)
    fmin, idx = res.argmin(res.fit[res.cur][:total])
    if fmin < state.best_fitness:
        state.best_fitness = fmin
        state.best_matrix = res.pop[res.cur][idx].cpu().numpy()


def _step_reference(state: SearchState) -> None:
    res, cfg = state._res, state.config
    gen = state.iteration + 1
    N, m, half, total = res.N, res.m, 2 * res.N, 4 * res.N
    cur, nxt = res.cur, res.cur ^ 1
    dev = res.dev
    sp = stream_ptr()
    # select (engine.py:233-248): stable order, reference permutation, gather
    order = torch.empty(half, dtype=torch.int64, device=dev)
    if res.sel_ws is None:
        wsb = int(lib.hga_select_ws_bytes(total))
        res.sel_ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
        pwsb = int(lib.hga_ref_permutation_ws_bytes(half))
        res.perm_ws = torch.empty(max(pwsb, 1), dtype=torch.uint8, device=dev)
    flag = _dev.new_flag()
    if _fitness_bound(m, res.fit_var) < int(lib.hga_select_max_range()):
        check(lib.hga_select_order(res.fit[cur].data_ptr(), total, order.data_ptr(), flag.data_ptr(),
                                   res.sel_ws.data_ptr(), res.sel_ws.shape[0], sp), "hga_select_order")
    else:  # SQ at large orders: the value span may exceed the histogram
        _select_radix(res.fit[cur], total, half, order)
    perm = torch.empty(half, dtype=torch.int64, device=dev)
    check(lib.hga_ref_permutation(state.seed, _sid(_P_SELECT, gen), 0, half, perm.data_ptr(), res.perm_ws.data_ptr(),
                                  res.perm_ws.shape[0], sp), "hga_ref_permutation")
    check(lib.hga_compose_gather(order.data_ptr(), perm.data_ptr(), half, res.pop[cur].data_ptr(),
                                 res.pop[nxt].data_ptr(), res.mw * 4, res.fit[cur].data_ptr(), res.fit[nxt].data_ptr(),
                                 None, sp), "hga_compose_gather")
    # crossover points + mutation plan (reference streams), fused generation
    from .rand import device_uniform

    points = device_uniform(state.seed, _sid(_P_CROSSOVER, gen), 0, 1, m - 1, N)
    cols, ra, rb = _plan_device(cfg, state.seed, gen)
    check(lib.hga_generation_explicit(res.pop[nxt].data_ptr(), res.fit[nxt].data_ptr(), N, m, points.data_ptr(),
                                      cols.data_ptr(), ra.data_ptr(), rb.data_ptr(), cols.shape[1], ra.shape[1],
                                      res.fit_var, None, sp), "hga_generation_explicit")
    res.cur = nxt
    fmin, idx = res.argmin(res.fit[nxt])
    _check_flag(flag, "select")
    state.iteration = gen
    state.trace.append(fmin)
    if fmin < state.best_fitness:
        state.best_fitness = fmin
        res.best_packed.copy_(res.matrix(nxt, idx))
        state.best_matrix = _best_from_packed(res, res.best_packed)


def _sync_from_device(state: SearchState) -> None:
    """Pull the 8-word device state (+ new trace entries) after hga_run: one
    small pinned D2H when a single generation ran (its trace value is
    state[7])."""
    res = state._res
    if res.host_state is None:
        res.host_state = torch.empty(8, dtype=torch.int64, pin_memory=True)
    res.host_state.copy_(res.dstate, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    st = res.host_state.tolist()
    it = int(st[0])
    if it == state.iteration + 1:
        state.trace.append(int(st[7]))
    elif it > state.iteration:
        state.trace.extend(int(v) for v in res.trace_dev[state.iteration + 1:it + 1].cpu().tolist())
    improved = int(st[1]) < state.best_fitness
    state.iteration = it
    state.best_fitness = int(st[1])
    state._last_restart = int(st[2])
    res.cur = int(st[3])
    if improved:
        state.best_matrix = _best_from_packed(res, res.best_packed)


def _run_device(state: SearchState, gens: int, force: bool = False) -> None:
    """`gens` generations in one persistent launch; `force` runs all of them
    even past a solution (the reference bench's fixed-length legs)."""
    res = state._res
    res.ensure_trace(state.iteration + gens)
    a = res.run_args()
    a.gens_this_call = gens
    if force:
        a.flags |= RUN_FORCE
    check(lib.hga_run(a, stream_ptr()), "hga_run")
    _sync_from_device(state)


def step(state, workers: int = 1):
    """Advance one generation (engine.py:449-469).

    `state` is a SearchState from initial_state (device resident), or any
    reference-style state whose population/fitness are numpy arrays (e.g.
    hadamard_ga.SearchState): that one is copied to the GPU, advanced and
    copied back in place, exactly like the reference's in-place step.
    """
    if not isinstance(state, SearchState):
        return _step_host(state)
    if isinstance(state._res, _ResidentI8):
        _step_i8(state)
    elif state.config.rng == "reference":
        _step_reference(state)
    else:
        res = state._res
        res.ensure_trace(state.iteration + 1)
        a = res.run_args()
        a.gens_this_call = 1
        a.flags |= RUN_FORCE
        check(lib.hga_run(a, stream_ptr()), "hga_run")
        _sync_from_device(state)
    if DEBUG_CHECKS:
        _check_state(state)
    return state


def _host_config(cfg) -> GAConfig:
    """Our GAConfig for a host state's config (ours or the reference's)."""
    if isinstance(cfg, GAConfig):
        return cfg
    return GAConfig(order=cfg.order, population=cfg.population, max_iterations=cfg.max_iterations,
                    mutation_cols=cfg.mutation_cols, mutation_row_pairs=cfg.mutation_row_pairs, fitness=cfg.fitness,
                    mutation=cfg.mutation, seed=cfg.seed, stall_window=cfg.stall_window,
                    time_budget_secs=cfg.time_budget_secs, rng=getattr(cfg, "rng", "reference"))


class _HostBridge:
    """Device buffers behind a host (numpy) search state; host arrays are
    page-locked in place (cudaHostRegister) so the per-step copies are DMA.
    Rebuilt whenever the state's config or seed changes (`key`)."""

    def __init__(self, state, cfg: GAConfig, key: tuple):
        self.cfg = cfg
        self.key = key
        self.res = _Resident(self.cfg, int(state.seed) & MASK64)
        m, total = self.cfg.order, self.cfg.total
        self.pop_i8 = torch.empty((total, m, m), dtype=torch.int8, device=self.res.dev)
        # page-locked host arrays (address -> array, kept alive while registered);
        # unregistered when the bridge (i.e. the host state) goes away
        self.registered: dict[int, np.ndarray] = {}
        self._finalizer = weakref.finalize(self, _unregister_all, self.registered)
        self.inner = SearchState(self.cfg, int(state.seed) & MASK64, self.res, 0, 0, [], None)
        self.copy_stream = torch.cuda.Stream(device=self.res.dev)
        self.host_state = torch.empty(8, dtype=torch.int64, pin_memory=True)
        self.host_state_in = torch.empty(8, dtype=torch.int64, pin_memory=True)  # pinned: no hidden stream sync
        self.host_flag = torch.zeros(1, dtype=torch.int32, pin_memory=True)
        self.args = None
        self._bits = None

    def bit_buffers(self):
        """(page-locked host, device) staging of hga_step_host_bits, or None
        when the order has no bit-stream path (or HGA_STEP_HOST=bytes)."""
        if self._bits is None:
            nb = int(lib.hga_step_host_bits_bytes(self.cfg.population, self.cfg.order))
            if nb == 0 or os.environ.get("HGA_STEP_HOST", "") == "bytes":
                self._bits = False
            else:
                self._bits = (torch.empty(nb, dtype=torch.uint8, pin_memory=True),
                              torch.empty(nb, dtype=torch.uint8, device=self.res.dev))
                self.bits_ptrs = (self._bits[0].data_ptr(), self._bits[1].data_ptr())
        return self._bits or None

    def pin(self, arr: np.ndarray) -> None:
        """Page-lock `arr` in place (shared, reference-counted registration,
        see _pin); not fatal when the runtime refuses (already pinned memory):
        the copies then go through the driver's staging path."""
        addr = arr.ctypes.data
        held = self.registered.get(addr)
        if arr.nbytes == 0 or (held is not None and held.nbytes >= arr.nbytes):
            return
        if held is not None:
            _unpin(addr)
            del self.registered[addr]
        if _pin(arr):
            self.registered[addr] = arr


# Page-locked host ranges, shared by every bridge: address -> [array, users].
# Two host states over the same arrays (or a new state reusing a freed
# state's address) share one registration; it is dropped with its last user.
_PINNED: dict[int, list] = {}


def _pin(arr: np.ndarray) -> bool:
    addr = arr.ctypes.data
    ent = _PINNED.get(addr)
    if ent is not None:
        if ent[0].nbytes >= arr.nbytes:
            ent[1] += 1
            return True
        return False  # a smaller live registration at this address: use staged copies
    try:
        rc = int(torch.cuda.cudart().cudaHostRegister(addr, arr.nbytes, 0))
    except Exception:  # noqa: BLE001 -- registration is an optimisation only
        rc = -1
    if rc != 0:
        lib.hga_clear_last_error()
        return False
    _PINNED[addr] = [arr, 1]
    return True


def _unpin(addr: int) -> None:
    ent = _PINNED.get(addr)
    if ent is None:
        return
    ent[1] -= 1
    if ent[1] <= 0:
        del _PINNED[addr]
        try:
            torch.cuda.cudart().cudaHostUnregister(addr)
            lib.hga_clear_last_error()
        except Exception:  # noqa: BLE001 -- interpreter shutdown
            pass


def _unregister_all(registered: dict) -> None:
    for addr in list(registered):
        _unpin(addr)
    registered.clear()


_BIT_CHUNKS = 4  # pieces of the bit-stream upload / download (hga_step_host_bits)
_HOST_CHUNKS = 8  # host <-> device population copies are pipelined against pack / unpack in this many pieces


def _chunks(total: int) -> list[tuple[int, int]]:
    k = max(1, min(_HOST_CHUNKS, total))
    return [(total * i // k, total * (i + 1) // k) for i in range(k)]


def _bridge_for(state) -> _HostBridge:
    cfg = _host_config(state.config)
    key = (cfg.order, cfg.population, cfg.mutation_cols, cfg.mutation_row_pairs, cfg.fitness, cfg.mutation,
           cfg.stall_window, cfg.rng, int(state.seed) & MASK64)
    bridge = getattr(state, "_hga_bridge", None)
    if bridge is None or bridge.key != key:
        bridge = _HostBridge(state, cfg, key)
        state._hga_bridge = bridge
    return bridge


def _host_arrays(state, cfg: GAConfig):
    """(population, fitness) as C-contiguous int8 / int64 arrays of the
    config's shapes: the caller's own arrays when they already are, else
    scratch copies that are written back (with the caller's dtype) after
    the step -- the native step reads and writes exactly these sizes."""
    pop, fit = state.population, state.fitness
    m, total = cfg.order, cfg.total
    if not isinstance(pop, np.ndarray) or not isinstance(fit, np.ndarray):
        raise ValueError("host state population and fitness must be numpy arrays")
    if pop.shape != (total, m, m):
        raise ValueError(f"population shape {pop.shape} does not match the config ({total}, {m}, {m})")
    if fit.shape != (total,):
        raise ValueError(f"fitness shape {fit.shape} does not match the config ({total},)")
    p = pop if (pop.dtype == np.int8 and pop.flags.c_contiguous) else np.ascontiguousarray(pop, dtype=np.int8)
    f = fit if (fit.dtype == np.int64 and fit.flags.c_contiguous) else np.ascontiguousarray(fit, dtype=np.int64)
    if p is not pop and not np.array_equal(p, pop):
        raise ValueError("step: matrix entries must be +1 or -1")
    return p, f


def _step_host(state):
    """One generation on a host (numpy) state, in place (engine.py:449-469).

    The int8 population goes up and comes back every step (the caller owns
    the arrays); the copies run on a side stream in chunks, each chunk packed
    (unpacked) on the compute stream as soon as it has landed (before it
    leaves), and in Philox mode the only host synchronisations are the
    validation after the upload and the final one.  A population that breaks
    the GA invariants (column 0 all +1, balanced columns) is stepped exactly
    by the explicit-plan generation (all column pairs, exact keys) instead of
    the Philox loop, whose fast paths rely on them.
    """
    bridge = _bridge_for(state)
    pop_np, fit_np = _host_arrays(state, bridge.cfg)
    res = bridge.res
    res.cur = 0  # the host arrays are authoritative: upload into buffer 0
    it0, best0 = int(state.iteration), int(state.best_fitness)
    last0 = int(state.trace[-1]) if state.trace else best0
    explicit = bridge.cfg.rng != "philox"
    if bridge.bit_buffers() is None:
        bridge.pin(pop_np)  # DMA copies of the int8 population (the bit-stream paths pack it on the host instead)
    bridge.pin(fit_np)
    if not explicit and res.m <= 64:
        # the whole step is enqueued natively (hga_step_host): chunked copies on a
        # side stream overlapped with pack / unpack, one synchronisation at the end
        if bridge.args is None:  # the trace buffer is not used by this path; args stay valid
            bridge.args = res.run_args()
            bridge.st_in = (ctypes.c_int64 * 8)()
            bridge.hs_np, bridge.hf_np = bridge.host_state.numpy(), bridge.host_flag.numpy()
            bridge.ptrs = (bridge.host_state.data_ptr(), bridge.host_flag.data_ptr(), bridge.copy_stream.cuda_stream)
        st_in = bridge.st_in
        st_in[0], st_in[1], st_in[2], st_in[6], st_in[7] = it0, best0, 0, 1, last0
        bits = bridge.bit_buffers()
        if bits is not None:
            # the population crosses PCIe as a bit stream (hga_step_host_bits: 8x fewer bytes)
            hs_p, hf_p, cs_p = bridge.ptrs
            rc = lib.hga_step_host_bits(bridge.args, pop_np.ctypes.data, fit_np.ctypes.data, bridge.bits_ptrs[0],
                                        bridge.bits_ptrs[1], st_in, hs_p, hf_p, _BIT_CHUNKS, stream_ptr(), cs_p)
        else:
            rc = lib.hga_step_host(bridge.args, pop_np.ctypes.data, fit_np.ctypes.data, bridge.pop_i8.data_ptr(),
                                   st_in, bridge.host_state.data_ptr(), bridge.host_flag.data_ptr(), _HOST_CHUNKS,
                                   stream_ptr(), bridge.copy_stream.cuda_stream)
        if rc == HGA_E_UNSUPPORTED:  # the v1 loop's configs (SQ above 32, m % 4 != 0, long plans): generic path
            _step_host_generic(state, bridge, pop_np, fit_np, it0, best0, last0, explicit)
            _write_back(state, pop_np, fit_np)
            return state
        check(rc, "hga_step_host")
        hf = int(bridge.hf_np[0])
        if hf & FLAG_NOT_SIGN:
            raise ValueError("step: matrix entries must be +1 or -1")
        if not hf & FLAG_NOT_GA:
            res.cur = 1
            _finish_host_step(state, pop_np, fit_np, int(bridge.hs_np[0]), int(bridge.hs_np[7]))
            _write_back(state, pop_np, fit_np)
            return state
        explicit = True  # host arrays untouched: take the exact path below
    _step_host_generic(state, bridge, pop_np, fit_np, it0, best0, last0, explicit)
    _write_back(state, pop_np, fit_np)
    return state


def _write_back(state, pop_np: np.ndarray, fit_np: np.ndarray) -> None:
    if state.population is not pop_np:
        state.population[...] = pop_np
    if state.fitness is not fit_np:
        state.fitness[...] = fit_np


def _step_host_generic(state, bridge: _HostBridge, pop_np, fit_np, it0: int, best0: int, last0: int,
                       explicit: bool) -> None:
    res, inner = bridge.res, bridge.inner
    cur = 0
    flag = _dev.new_flag()
    m, total, mw = res.m, 4 * res.N, res.mw
    comp, cs = torch.cuda.current_stream(), bridge.copy_stream
    pop_t, fit_t = torch.from_numpy(pop_np), torch.from_numpy(fit_np)
    parts = _chunks(total)
    bits = bridge.bit_buffers()  # orders 4..64: the population crosses PCIe as a bit stream
    nb = 4 * ((pop_np.size + 31) // 32)
    if bits is not None and lib.hga_host_pack_bits(pop_np.ctypes.data, pop_np.size, bits[0].data_ptr()) & FLAG_NOT_SIGN:
        raise ValueError("step: matrix entries must be +1 or -1")
    cs.wait_stream(comp)
    with torch.cuda.stream(cs):
        res.fit[cur].copy_(fit_t, non_blocking=True)
    if bits is not None:
        with torch.cuda.stream(cs):
            bits[1][:nb].copy_(bits[0][:nb], non_blocking=True)
        comp.wait_stream(cs)
        check(lib.hga_bits_to_cols(bits[1].data_ptr(), total, m, res.pop[cur].data_ptr(), flag.data_ptr(),
                                   comp.cuda_stream), "hga_bits_to_cols")
    for a, b in (parts if bits is None else ()):
        with torch.cuda.stream(cs):
            bridge.pop_i8[a:b].copy_(pop_t[a:b], non_blocking=True)
            landed = torch.cuda.Event()
            landed.record(cs)
        comp.wait_event(landed)
        check(lib.hga_pack_i8(bridge.pop_i8[a].data_ptr(), b - a, m, res.pop[cur][a * mw].data_ptr(),
                              flag.data_ptr(), comp.cuda_stream), "hga_pack_i8")
    comp.wait_stream(cs)
    # validate before anything is written back (the host arrays are in-place outputs)
    fl = int(flag.item())
    if fl & FLAG_NOT_SIGN:
        raise ValueError("step: matrix entries must be +1 or -1")
    if fl & FLAG_NOT_GA:
        explicit = True
    res.cur = cur
    if explicit:
        inner.iteration, inner.best_fitness, inner.trace, inner.best_matrix = it0, best0, [last0], None
        _step_reference(inner)
        new = res.cur
    else:
        bridge.host_state_in.copy_(torch.tensor([it0, best0, 0, cur, 0, 0, 1, last0], dtype=torch.int64))
        res.dstate.copy_(bridge.host_state_in, non_blocking=True)
        check(lib.hga_run_prepare(res.run_args(), stream_ptr()), "hga_run_prepare")
        res.ensure_trace(it0 + 1)
        args = res.run_args()
        args.gens_this_call = 1
        args.flags |= RUN_FORCE  # exactly one generation: the new population is in buffer cur ^ 1
        check(lib.hga_run(args, stream_ptr()), "hga_run")
        new = cur ^ 1
    if bits is not None:
        check(lib.hga_cols_to_bits(res.pop[new].data_ptr(), total, m, bits[1].data_ptr(), comp.cuda_stream),
              "hga_cols_to_bits")
    for a, b in (parts if bits is None else ()):
        check(lib.hga_unpack_i8(res.pop[new][a * mw].data_ptr(), b - a, m, bridge.pop_i8[a].data_ptr(),
                                comp.cuda_stream), "hga_unpack_i8")
        ready = torch.cuda.Event()
        ready.record(comp)
        cs.wait_event(ready)
        with torch.cuda.stream(cs):
            pop_t[a:b].copy_(bridge.pop_i8[a:b], non_blocking=True)
    cs.wait_stream(comp)
    with torch.cuda.stream(cs):
        if bits is not None:
            bits[0][:nb].copy_(bits[1][:nb], non_blocking=True)
        fit_t.copy_(res.fit[new], non_blocking=True)
        bridge.host_state.copy_(res.dstate, non_blocking=True)
    cs.synchronize()
    if bits is not None:
        lib.hga_host_unpack_bits(bits[0].data_ptr(), pop_np.size, pop_np.ctypes.data)
    if explicit:
        it1, fmin = inner.iteration, inner.trace[-1]
    else:
        it1, fmin = int(bridge.host_state[0]), int(bridge.host_state[7])
    _finish_host_step(state, pop_np, fit_np, it1, fmin)


def _finish_host_step(state, pop_np: np.ndarray, fit_np: np.ndarray, it1: int, fmin: int) -> None:
    """Trace / best bookkeeping of a host state (engine.py:430-437)."""
    state.iteration = it1
    state.trace.append(fmin)
    if fmin < state.best_fitness:
        state.best_fitness = fmin
        state.best_matrix = pop_np[int(np.argmin(fit_np))].copy()


def check_invariants(state: SearchState) -> tuple[int, int, int]:
    """(bad first columns, unbalanced columns, stale fitness values) of the
    device-resident population, counted on the GPU (hga_check_invariants)."""
    res = state._res
    total = 4 * res.N
    counts = torch.zeros(3, dtype=torch.int64, device=res.dev)
    wsb = int(lib.hga_check_invariants_ws_bytes(total))
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=res.dev)
    check(lib.hga_check_invariants(res.pop[res.cur].data_ptr(), res.fit[res.cur].data_ptr(), total, res.m,
                                   res.fit_var, counts.data_ptr(), ws.data_ptr(), wsb, stream_ptr()),
          "hga_check_invariants")
    c = counts.tolist()
    return int(c[0]), int(c[1]), int(c[2])


def _check_state(state: SearchState) -> None:
    """engine.py:440-446, on the device (no host copy of the population)."""
    c0, c1, c2 = check_invariants(state)
    assert c0 == 0, "first column lost its all-+1 contract"
    assert c1 == 0, "column balance broken"
    assert c2 == 0, "fitness vector is stale"


def detect_stall(state: SearchState, window: int) -> bool:
    """True when the min-fitness trace sat flat and positive for `window` steps (engine.py:472-479)."""
    if window < 1:
        raise ValueError("window must be >= 1")
    tail = state.trace[-window:]
    if len(tail) < window or tail[-1] == 0:
        return False
    return all(v == tail[0] for v in tail)


def _reinitialize_offspring(state: SearchState) -> None:
    """Fresh balanced offspring, parents retained (engine.py:482-494), reference streams."""
    res, cfg = state._res, state.config
    half, total, m = 2 * res.N, 4 * res.N, res.m
    cur = res.cur
    off = res.pop[cur][half * res.mw:]
    _init_packed(cfg, state.seed, _P_RESTART, state.iteration, half, half, off)
    fo = res.fit[cur][half:]
    fv = res.fit_var
    check(lib.hga_fitness_packed(off.data_ptr(), half, m, fv, ptr(fo) if fv == 1 else None,
                                 ptr(fo) if fv == 2 else None, None, ptr(fo) if fv == 8 else None, stream_ptr()),
          "hga_fitness_packed")
    fmin, idx = res.argmin(res.fit[cur][:total])
    if fmin < state.best_fitness:
        state.best_fitness = fmin
        res.best_packed.copy_(res.matrix(cur, idx))
        state.best_matrix = _best_from_packed(res, res.best_packed)


def run_search(config: GAConfig, workers: int = 1, poll_interval: int = 256) -> RunRecord:
    """Init, then step until fitness 0 or budgets run out (engine.py:497-538).

    Philox mode runs `poll_interval` generations per kernel launch (the
    device stops by itself on success or max_iterations; the host only
    reads an 8-word state block between launches for the time budget).
    """
    start = time.perf_counter()
    state = initial_state(config, workers=workers)
    complete = True
    if config.rng == "reference" or isinstance(state._res, _ResidentI8):
        last_restart = 0
        while state.iteration < config.max_iterations and state.best_fitness > 0:
            if config.time_budget_secs is not None and time.perf_counter() - start > config.time_budget_secs:
                complete = False
                break
            step(state)
            if (config.stall_window is not None and state.best_fitness > 0
                    and state.iteration - last_restart >= config.stall_window
                    and detect_stall(state, config.stall_window)):
                if isinstance(state._res, _ResidentI8):
                    _reinitialize_offspring_i8(state)
                else:
                    _reinitialize_offspring(state)
                last_restart = state.iteration
    else:
        while state.iteration < config.max_iterations and state.best_fitness > 0:
            if config.time_budget_secs is not None and time.perf_counter() - start > config.time_budget_secs:
                complete = False
                break
            gens = min(poll_interval, config.max_iterations - state.iteration)
            _run_device(state, gens)
    torch.cuda.synchronize()
    wall = time.perf_counter() - start
    success = state.best_fitness == 0
    return RunRecord(config=config, seed=state.seed, success=success, complete=complete or success,
                     iterations=state.iteration, best_fitness=state.best_fitness, best_matrix=state.best_matrix,
                     trace=list(state.trace), wall_seconds=wall)
