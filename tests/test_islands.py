"""Island-model protocol on CPU: two gloo ranks, a host stand-in island.

The collectives (global-best agreement, ring migration, winner broadcast)
are the ones run_islands uses with NCCL on GPUs; the stand-in evolves its
population with the CPU oracle (reference semantics), so the test covers
the host logic of the multi-GPU path without a GPU.
"""

from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def pack_np(pop: np.ndarray) -> np.ndarray:
    """int8 (n, m, m) -> packed (n, m * W) int32 columns (bit r = entry r is -1)."""
    n, m, _ = pop.shape
    w = (m + 31) // 32
    out = np.zeros((n, m, w), dtype=np.uint32)
    neg = (pop < 0).astype(np.uint32)
    for r in range(m):
        out[:, :, r // 32] |= neg[:, r, :] << np.uint32(r % 32)
    return out.reshape(n, m * w).view(np.int32)


def unpack_np(rec: np.ndarray, m: int) -> np.ndarray:
    w = (m + 31) // 32
    words = rec.view(np.uint32).reshape(-1, m, w)
    pop = np.ones((words.shape[0], m, m), dtype=np.int8)
    for r in range(m):
        bit = (words[:, :, r // 32] >> np.uint32(r % 32)) & 1
        pop[:, r, :] = np.where(bit == 1, -1, 1)
    return pop


class HostIsland:
    """CPU stand-in with GpuIsland's interface (test code only)."""

    def __init__(self, config, seed):
        sys.path.insert(0, str(ROOT))
        import oracle

        self.o = oracle
        self.cfg = config
        self.st = oracle.initial_state(config.order, config.population, seed, config.fitness, config.mutation_cols,
                                       config.mutation_row_pairs, config.mutation)
        self.received = 0

    @property
    def iteration(self):
        return self.st.iteration

    @property
    def best(self):
        return self.st.best_fitness

    def advance(self, gens):
        for _ in range(gens):
            self.o.step(self.st, threads=1)

    def elites(self, e):
        order = np.argsort(self.st.fitness, kind="stable")[:e]
        return torch.from_numpy(pack_np(self.st.population[order])), torch.from_numpy(self.st.fitness[order].copy())

    def receive(self, rec, fit):
        # same rule as GpuIsland.receive: migrants replace the e worst (largest
        # fitness, lowest index first among equals)
        e = rec.shape[0]
        worst = np.argsort(-self.st.fitness, kind="stable")[:e]
        self.st.population[worst] = unpack_np(rec.numpy(), self.cfg.order)
        self.st.fitness[worst] = fit.numpy()
        self.received += e
        b = int(self.st.fitness.min())
        if b < self.st.best_fitness:
            self.st.best_fitness = b
            self.st.best_matrix = self.st.population[int(self.st.fitness.argmin())].copy()

    def best_matrix_packed(self):
        return torch.from_numpy(pack_np(self.st.best_matrix[None])[0])

    def decode(self, packed):
        return unpack_np(packed.numpy().reshape(1, -1), self.cfg.order)[0]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, str(ROOT))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2208_14961_b200.engine import GAConfig
        from paper_2208_14961_b200.islands import Exchange, IslandConfig, run_islands

        ex = Exchange()
        got = ex.ring_shift(torch.tensor([rank * 10 + 1, rank], dtype=torch.int32))
        best, stop = ex.agree(100 + rank, rank == 1)
        cfg = GAConfig(order=8, population=20, seed=5, fitness="f1", max_iterations=60)
        rec = run_islands(cfg, IslandConfig(migration_interval=5, migration_size=4, poll_interval=5),
                          island_factory=HostIsland)
        q.put((rank, got.tolist(), best, stop, rec.success, rec.iterations, rec.best_fitness,
               rec.best_matrix.tolist(), rec.winner_rank, rec.migrations, rec.trace))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_island_protocol_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, got0, b0, s0, *rec0), (r1, got1, b1, s1, *rec1) = res
    assert got0 == [11, 1] and got1 == [1, 0]          # ring: rank r receives from r-1
    assert (b0, s0) == (100, True) and (b1, s1) == (100, True)  # MIN agreement, any rank stops all
    assert rec0 == rec1                                  # identical record on every rank
    success, iters, best, matrix, winner, migrations, trace = rec0
    assert all(a >= b for a, b in zip(trace, trace[1:]))
    assert winner in (0, 1)
    if success:
        q = np.array(matrix, dtype=np.int64)
        assert (q.T @ q == 8 * np.eye(8, dtype=np.int64)).all()
    else:
        assert migrations >= 1


def test_payload_roundtrip():
    sys.path.insert(0, str(ROOT))
    from paper_2208_14961_b200.islands import pack_payload, unpack_payload

    rec = torch.arange(3 * 20, dtype=torch.int32).reshape(3, 20)
    fit = torch.tensor([5, 1 << 40, 7], dtype=torch.int64)
    r2, f2 = unpack_payload(pack_payload(rec, fit), 3, 20)
    assert torch.equal(r2, rec) and torch.equal(f2, fit)
    pop = np.random.default_rng(0).choice(np.array([-1, 1], np.int8), size=(4, 36, 36))
    assert np.array_equal(unpack_np(pack_np(pop), 36), pop)


def _shard_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, str(ROOT))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2208_14961_b200.islands import evaluate_sharded, shard_bounds

        pop = oracle.init_population(12, 251, 3)  # 1004 matrices: not divisible by 3
        seen = []

        def ev(p, fit):
            seen.append(len(p))
            return oracle.evaluate(p, fit)

        got = evaluate_sharded(pop, "f1", evaluator=ev)
        lo, hi = shard_bounds(len(pop), world, rank)
        # local mode: each rank holds only its own (uneven) slice
        cut = [0, 100, 101, 1004]
        got_local = evaluate_sharded(pop[cut[rank]:cut[rank + 1]], "f1", evaluator=ev, local=True)
        t = evaluate_sharded(torch.from_numpy(pop), "f1", evaluator=lambda p, f: oracle.evaluate(p.numpy(), f))
        q.put((rank, got.tolist(), seen, (lo, hi), got_local.tolist(), t.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_sharded_fitness_gloo():
    """Fitness-only sharding: each rank scores only its slice,
    one all_gather returns the full, reference-equal vector on every rank."""
    import oracle

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = oracle.evaluate(oracle.init_population(12, 251, 3), "f1").tolist()
    bounds = []
    for rank, got, seen, (lo, hi), got_local, t in res:
        assert got == want, rank
        assert got_local == want and t == want, rank
        assert seen == [hi - lo, [100, 1, 903][rank]]
        bounds.append((lo, hi))
    assert bounds == [(0, 334), (334, 669), (669, 1004)]
