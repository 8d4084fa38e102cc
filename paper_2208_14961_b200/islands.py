"""Island model across GPUs (north star: population sharded as islands, NCCL
elite migration + best-fitness all-reduce).  No reference counterpart: the
reference GA is single-population (islands are a SPEC non-goal,
SPEC.md:312); with one island this reduces to engine.run_search.

One process per GPU (torchrun), torch.distributed over NCCL.  Each rank
evolves its own 4N population with the persistent generation kernel; every
`poll_interval` generations the ranks agree on the global best fitness and a
common stop decision with one 2-int64 all_reduce(MIN), and every
`migration_interval` generations each island sends its E best individuals
(packed columns + fitness, one all_gather) to the next island in the ring,
which writes them over the first E offspring slots -- so they compete in its
next selection -- and rebuilds its selection histogram.

The communication is backend-agnostic (`Exchange`), so the protocol is
exercised by the CPU tests with gloo and a host stand-in for the island.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

from . import _dev
from ._dev import check, lib, stream_ptr
from .engine import GAConfig, initial_state, _run_device, _best_from_packed, _sync_from_device
from .rand import MASK64, mix64

__all__ = ["IslandConfig", "Exchange", "GpuIsland", "IslandRecord", "island_seed", "run_islands",
           "shard_bounds", "evaluate_sharded"]


@dataclass(frozen=True)
class IslandConfig:
    migration_interval: int = 200   # generations between migrations
    migration_size: int = 16        # E elites sent to the next island
    poll_interval: int = 100        # generations per launch between global-best checks

    def __post_init__(self):
        if self.migration_interval < 1 or self.poll_interval < 1 or self.migration_size < 0:
            raise ValueError("island intervals must be >= 1 and migration_size >= 0")


def island_seed(seed: int, rank: int) -> int:
    """Independent stream seed per island (rank 0 keeps the run's seed)."""
    return seed & MASK64 if rank == 0 else mix64((seed ^ (rank * 0x9E3779B97F4A7C15)) & MASK64)


class Exchange:
    """The two collectives of the island model."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        backend = dist.get_backend(group) if dist.is_initialized() else "none"
        self.device = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")

    def agree(self, best: int, want_stop: bool) -> tuple[int, bool]:
        """(global best fitness, stop) -- identical on every rank."""
        if self.world == 1:
            return best, want_stop
        t = torch.tensor([best, 0 if want_stop else 1], dtype=torch.int64, device=self.device)
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)
        v = t.cpu().tolist()
        return int(v[0]), v[1] == 0

    def agree_tensor(self, best: torch.Tensor, want_stop: bool) -> torch.Tensor:
        """Enqueue the agreement on a 1-element int64 `best` tensor (device
        resident for NCCL: no host read before the collective) and return
        the reduced (best, continue) pair without reading it; the caller's
        next stream synchronisation covers it."""
        flag = torch.ones(1, dtype=torch.int64, device=best.device) if not want_stop else \
            torch.zeros(1, dtype=torch.int64, device=best.device)
        t = torch.cat([best.reshape(1).to(torch.int64), flag]).to(self.device)
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)
        return t

    @staticmethod
    def read(t: torch.Tensor) -> tuple[int, bool]:
        v = t.tolist()
        return int(v[0]), v[1] == 0

    def ring_shift(self, payload: torch.Tensor) -> torch.Tensor:
        """Every rank sends `payload` to rank+1 and returns what rank-1 sent."""
        if self.world == 1:
            return payload
        p = payload.to(self.device)
        parts = [torch.empty_like(p) for _ in range(self.world)]
        dist.all_gather(parts, p, group=self.group)
        return parts[(self.rank - 1) % self.world]

    def owner_of_best(self, best: int) -> int:
        """Lowest rank whose island holds the global best (for the final record)."""
        if self.world == 1:
            return 0
        t = torch.tensor([best * self.world + self.rank], dtype=torch.int64, device=self.device)
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)
        return int(t.item()) % self.world

    def broadcast(self, t: torch.Tensor, src: int) -> torch.Tensor:
        if self.world == 1:
            return t
        x = t.to(self.device).contiguous()
        dist.broadcast(x, src=src, group=self.group)
        return x


def pack_payload(packed: torch.Tensor, fit: torch.Tensor) -> torch.Tensor:
    """One int32 tensor: E packed records followed by E int64 fitness values."""
    return torch.cat([packed.reshape(-1).to(torch.int32), fit.to(torch.int64).view(torch.int32).reshape(-1)])


def unpack_payload(payload: torch.Tensor, e: int, mw: int) -> tuple[torch.Tensor, torch.Tensor]:
    rec = payload[: e * mw].reshape(e, mw)
    fit = payload[e * mw: e * mw + 2 * e].contiguous().view(torch.int64)
    return rec, fit


class GpuIsland:
    """One island: a device-resident SearchState advanced by hga_run."""

    def __init__(self, config: GAConfig, seed: int):
        if config.rng != "philox":
            raise ValueError("islands run on the production (philox) loop")
        self.state = initial_state(config, seed=seed)
        self.res = self.state._res
        self._ws = None
        self.last_received = None  # slots the last migrants were written to (tests)

    @property
    def iteration(self) -> int:
        return self.state.iteration

    @property
    def best(self) -> int:
        return self.state.best_fitness

    def advance(self, gens: int) -> None:
        _run_device(self.state, gens)

    def launch(self, gens: int) -> None:
        """Enqueue `gens` generations (one persistent launch), no host sync."""
        res, st = self.res, self.state
        res.ensure_trace(st.iteration + gens)
        a = res.run_args()
        a.gens_this_call = gens
        check(lib.hga_run(a, stream_ptr()), "hga_run")

    def best_tensor(self) -> torch.Tensor:
        """Device-resident best-so-far fitness (state word 1)."""
        return self.res.dstate[1:2]

    def sync(self) -> None:
        """Refresh the host view (best, iteration) from the device state."""
        _sync_from_device(self.state)

    def elites(self, e: int) -> tuple[torch.Tensor, torch.Tensor]:
        """The e best individuals (lowest fitness, lowest index first) of the current population."""
        res = self.res
        total = 4 * res.N
        cur = res.cur
        dev = res.dev
        if self._ws is None:
            wsb = int(lib.hga_select_ws_bytes(total))
            self._ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
        idx = torch.empty(max(e, 1), dtype=torch.int64, device=dev)
        flag = _dev.new_flag()
        check(lib.hga_select_smallest(res.fit[cur].data_ptr(), total, e, idx.data_ptr(), flag.data_ptr(),
                                      self._ws.data_ptr(), self._ws.shape[0], stream_ptr()), "hga_select_smallest")
        rec = torch.empty((max(e, 1), res.mw), dtype=torch.int32, device=dev)
        fit = torch.empty(max(e, 1), dtype=torch.int64, device=dev)
        check(lib.hga_compose_gather(idx.data_ptr(), None, e, res.pop[cur].data_ptr(), rec.data_ptr(), res.mw * 4,
                                     res.fit[cur].data_ptr(), fit.data_ptr(), None, stream_ptr()),
              "hga_compose_gather")
        return rec[:e], fit[:e]

    def receive(self, rec: torch.Tensor, fit: torch.Tensor) -> None:
        """Migrants overwrite the e WORST individuals of the current population
        (largest fitness, lowest index first among equals), so the island's
        own best always survives and its min fitness never rises; they then
        compete in the next selection.  Everything stays on the device (no
        host synchronisation): the selection histogram is rebuilt and the
        loop's best-so-far (state word 1 + best matrix) takes a better
        migrant, which the host sees at the next poll."""
        res = self.res
        e = rec.shape[0]
        if e == 0:
            return
        total, cur, mw = 4 * res.N, res.cur, res.mw
        if e >= total:
            raise ValueError("migration_size must be smaller than the island population")
        rec = rec.reshape(e, mw).to(device=res.dev, dtype=torch.int32)
        fit = fit.to(device=res.dev, dtype=torch.int64)
        if self._ws is None:
            self._ws = torch.empty(int(lib.hga_select_ws_bytes(total)), dtype=torch.uint8, device=res.dev)
        neg = torch.neg(res.fit[cur])
        worst = torch.empty(e, dtype=torch.int64, device=res.dev)
        flag = _dev.new_flag()
        check(lib.hga_select_smallest(neg.data_ptr(), total, e, worst.data_ptr(), flag.data_ptr(),
                                      self._ws.data_ptr(), self._ws.shape[0], stream_ptr()), "hga_select_smallest")
        res.pop[cur].view(total, mw).index_copy_(0, worst, rec)
        res.fit[cur].index_copy_(0, worst, fit)
        check(lib.hga_run_prepare(res.run_args(), stream_ptr()), "hga_run_prepare")
        k = torch.argmin(fit)
        better = fit[k] < res.dstate[1]
        res.best_packed.copy_(torch.where(better, rec[k], res.best_packed))
        res.dstate[1:2].copy_(torch.minimum(res.dstate[1:2], fit[k].reshape(1)))
        self.last_received = worst

    def best_matrix_packed(self) -> torch.Tensor:
        return self.res.best_packed


@dataclass
class IslandRecord:
    config: GAConfig
    island_config: IslandConfig
    seed: int
    world: int
    success: bool
    complete: bool
    iterations: int
    best_fitness: int
    best_matrix: np.ndarray
    winner_rank: int
    wall_seconds: float
    migrations: int
    trace: list = field(default_factory=list)


def run_islands(config: GAConfig, island_config: IslandConfig = IslandConfig(), group=None,
                island_factory=None) -> IslandRecord:
    """Island-model search; call on every rank (torchrun).  Returns the same
    record on every rank.  `island_factory(config, seed)` substitutes the
    island implementation (the CPU tests pass a host stand-in)."""
    start = time.perf_counter()
    ex = Exchange(group)
    seed = config.seed if config.seed is not None else 0
    make = island_factory or GpuIsland
    island = make(config, island_seed(seed, ex.rank))
    ic = island_config
    migrations = 0
    complete = True
    best, _ = ex.agree(island.best, False)
    trace = [best]
    pipelined = hasattr(island, "launch")
    while True:
        if best == 0 or island.iteration >= config.max_iterations:
            break
        to_mig = ic.migration_interval - (island.iteration % ic.migration_interval)
        gens = min(ic.poll_interval, to_mig, config.max_iterations - island.iteration)
        over = config.time_budget_secs is not None and time.perf_counter() - start > config.time_budget_secs
        if pipelined:
            # launch, agree on the device-resident best, then ONE host sync per poll
            island.launch(gens)
            t = ex.agree_tensor(island.best_tensor(), over)
            island.sync()
            best, stop = ex.read(t)
        else:
            island.advance(gens)
            best, stop = ex.agree(island.best, over)
        trace.append(best)
        if stop:
            complete = best == 0
            break
        if best > 0 and island.iteration % ic.migration_interval == 0 and ic.migration_size > 0 and ex.world > 1:
            e = min(ic.migration_size, 2 * config.population)
            rec, fit = island.elites(e)
            incoming = ex.ring_shift(pack_payload(rec, fit))
            r2, f2 = unpack_payload(incoming, e, rec.shape[1])
            island.receive(r2, f2)
            migrations += 1
    if pipelined:
        island.sync()  # migrants received after the last poll may hold the best
    owner = ex.owner_of_best(island.best)
    mat = ex.broadcast(island.best_matrix_packed().reshape(-1).to(torch.int32), owner)
    if isinstance(island, GpuIsland):
        res = island.res
        best_matrix = _best_from_packed(res, mat.to(res.dev))
    else:
        best_matrix = island.decode(mat.cpu())
    torch.cuda.synchronize() if torch.cuda.is_available() else None
    return IslandRecord(config=config, island_config=ic, seed=seed, world=ex.world, success=best == 0,
                        complete=complete, iterations=island.iteration, best_fitness=best, best_matrix=best_matrix,
                        winner_rank=owner, wall_seconds=time.perf_counter() - start, migrations=migrations,
                        trace=trace)


# ---------------------------------------------------------------- fitness-only sharding


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous slice [lo, hi) of n matrices owned by `rank` (SURVEY.md §8e:
    matrices are independent units; sizes differ by at most one)."""
    return n * rank // world, n * (rank + 1) // world


def evaluate_sharded(population, fitness: str = "f2", group=None, evaluator=None, local: bool = False):
    """`evaluate` across all ranks of a torch.distributed job: rank r scores
    only its contiguous slice on its own GPU and one all_gather returns the
    whole fitness vector on every rank; no other collective.

    * `local=False`: every rank passes the same population (numpy or a
      tensor) and scores `population[lo:hi]` (`shard_bounds`); only that
      slice is copied to the device.
    * `local=True`: each rank passes ONLY its own slice (config 5 at 10^7
      matrices need not exist on any one host); the slice sizes are agreed
      with one extra 8-byte all_gather.
    With NCCL the gather runs on device tensors (no host staging); the
    result is a CUDA int64 tensor for tensor input and numpy for numpy
    input.  `evaluator(pop, fitness)` replaces the GPU kernel (the CPU tests
    run the protocol on gloo with the oracle).  Without an initialised
    process group this is `evaluate`.
    """
    from . import engine

    host_in = not isinstance(population, torch.Tensor)
    evaluator = evaluator or engine.evaluate
    if not (dist.is_available() and dist.is_initialized()):
        return evaluator(population, fitness)
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    nccl = dist.get_backend(group) == "nccl"
    dev = torch.device("cuda", torch.cuda.current_device()) if nccl else torch.device("cpu")
    if local:
        mine_pop = population
        cnt = torch.tensor([int(population.shape[0])], dtype=torch.int64, device=dev)
        counts = [torch.empty_like(cnt) for _ in range(world)]
        dist.all_gather(counts, cnt, group=group)
        sizes = [int(c.item()) for c in counts]
    else:
        n = int(population.shape[0])
        sizes = [shard_bounds(n, world, r)[1] - shard_bounds(n, world, r)[0] for r in range(world)]
        lo, hi = shard_bounds(n, world, rank)
        mine_pop = population[lo:hi]
    mine = evaluator(mine_pop, fitness)
    mine = torch.as_tensor(mine).to(device=dev, dtype=torch.int64)
    width = max(max(sizes), 1)  # all_gather needs equal sizes: pad every slice to the largest
    buf = torch.zeros(width, dtype=torch.int64, device=dev)
    buf[: mine.shape[0]] = mine
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    out = torch.cat([part[:sz] for part, sz in zip(parts, sizes)])
    return out.cpu().numpy() if host_in else out.to(population.device)
