"""Production (Philox) loop at the sizes it is measured at, the host-state
step's invariant guard, and the real island path on one GPU.

* The generation loop partitions its histogram, survivor lists and tiles
  per CTA, and those partitions change with N, so the loop is checked at
  the bench config (m = 20, 4N = 40,000, NC = 4, NR = 2) and at the config-3
  and config-4 island sizes (m = 28, 4N = 125,000; m = 36, 4N = 1,250,000)
  for >= 50 generations: after every batch the GA invariants hold
  (engine.py:440-446 `_check_state`), the fitness vector equals the oracle
  (all of it, or a 20k sample at 1.25M), the trace is monotone, and single
  steps select exactly the 2N lowest under the stable tie rule
  (engine.py:245).
* engine.step on a host (numpy) state validates the population first: an
  entry that is not +-1 raises ValueError with the arrays untouched; a
  population that breaks the GA invariants (which the Philox loop's fast
  paths assume) is stepped exactly by the explicit-plan path -- identical
  to the reference's own step (oracle) for the same seed and generation.
* run_islands / GpuIsland at world size 2 (gloo, both ranks on cuda:0):
  migrants land on the receiver's worst slots, its best survives, the
  histogram is rebuilt, and the loop keeps its invariants afterwards.
"""

from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

import oracle
import paper_2208_14961_b200 as hga
from paper_2208_14961_b200 import engine

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def _hash_records(packed: torch.Tensor) -> torch.Tensor:
    """(n, words) int32 -> (n,) int64 hash (two independent weightings)."""
    x = packed.reshape(packed.shape[0], -1).to(torch.int64) & 0xFFFFFFFF
    g = torch.Generator(device="cpu").manual_seed(1234)
    w1 = torch.randint(1, 2**62, (x.shape[1],), generator=g, dtype=torch.int64).to(x.device)
    w2 = torch.randint(1, 2**62, (x.shape[1],), generator=g, dtype=torch.int64).to(x.device)
    return (x * w1).sum(1) ^ ((x * w2).sum(1) << 1)


def _device_invariants(st, sample: int | None, rng: np.random.Generator) -> None:
    """Column 0 all +1, other columns balanced (all matrices, on the device);
    fitness == oracle (all, or `sample` random matrices)."""
    cfg = st.config
    m, total = cfg.order, cfg.total
    res = st._res
    pop = engine._unpack(res.pop[res.cur], total, m)  # (4N, m, m) int8 on the device
    assert bool((pop[:, :, 0] == 1).all()), "first column lost its all-+1 contract"
    assert bool((pop[:, :, 1:].sum(dim=1) == 0).all()), "column balance broken"
    fit = st.fitness_device
    if sample is None or sample >= total:
        idx = np.arange(total)
    else:
        idx = np.sort(rng.choice(total, size=sample, replace=False))
    it = torch.from_numpy(idx).to(pop.device)
    want = oracle.evaluate(pop[it].cpu().numpy(), cfg.fitness)
    assert np.array_equal(fit[it].cpu().numpy(), want), "fitness vector is stale or wrong"
    del pop


def _check_selection_step(st) -> None:
    """One generation: the parent half afterwards is exactly the 2N lowest
    of the population before (stable argsort order), as a multiset of
    matrices and of fitness values."""
    res = st._res
    total, half, mw = 4 * res.N, 2 * res.N, res.mw
    before = res.pop[res.cur].view(total, mw).clone()
    fbefore = st.fitness_device.clone()
    hga.step(st)
    order = torch.sort(fbefore, stable=True).indices[:half]
    want_h = torch.sort(_hash_records(before[order])).values
    after = res.pop[res.cur].view(total, mw)[:half]
    got_h = torch.sort(_hash_records(after)).values
    assert torch.equal(want_h, got_h), "survivors are not the 2N lowest (stable tie rule)"
    assert torch.equal(torch.sort(fbefore[order]).values, torch.sort(st.fitness_device[:half]).values)


@pytest.mark.parametrize("m,N,nc,nr,fit,sample", [
    (20, 10_000, 4, 2, "f2", None),      # bench config (BASELINE configs[1])
    (20, 10_000, 4, 2, "f1", None),
    (28, 31_250, 1, 10, "f2", None),     # config-3 island (1M / 8)
    (28, 31_250, 1, 10, "sq", 40_000),
    (36, 312_500, 1, 12, "f2", 20_000),  # config-4 island (10M / 8)
    (36, 312_500, 1, 12, "f1", 20_000),
])
def test_production_loop_at_measured_sizes(m, N, nc, nr, fit, sample, cuda_device):
    cfg = engine.GAConfig(order=m, population=N, seed=2024 + m, fitness=fit, mutation_cols=nc, mutation_row_pairs=nr,
                          max_iterations=10_000)
    rng = np.random.default_rng(m * 7 + N)
    st = hga.initial_state(cfg)
    _device_invariants(st, sample, rng)
    gens = 0
    for batch in range(6):
        _check_selection_step(st)           # one generation, survivor set checked
        engine._run_device(st, 9, force=True)  # nine more in one persistent launch
        gens += 10
        _device_invariants(st, sample, rng)
        assert all(a >= b for a, b in zip(st.trace, st.trace[1:]))
        assert st.trace[-1] == int(st.fitness_device.min().item())
        assert st.best_fitness == min(st.trace)
    assert gens >= 50 and st.iteration == gens and len(st.trace) == gens + 1


def test_production_loop_with_stall_restarts_at_bench_size(cuda_device):
    """Stall restarts (engine.py:518-525) at the bench population: a window of
    2 restarts whenever the best stays flat for two generations; the
    restart refills offspring from fresh Philox streams and the invariants
    and fitness must still hold."""
    cfg = engine.GAConfig(order=20, population=10_000, seed=77, fitness="f2", mutation_cols=4, mutation_row_pairs=2,
                          max_iterations=10_000, stall_window=2)
    st = hga.initial_state(cfg)
    rng = np.random.default_rng(0)
    for _ in range(5):
        engine._run_device(st, 12)  # not forced: the device loop decides restarts itself
        _device_invariants(st, None, rng)
        assert all(a >= b for a, b in zip(st.trace, st.trace[1:]))
    assert st._last_restart > 0, "no stall restart happened"


# ------------------------------------------------------------ host-state guard


def _host_state(cfg, seed, pop, fit):
    from dataclasses import dataclass, field

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

    b = int(fit.argmin())
    return HostState(cfg, seed, pop, fit, 0, pop[b].copy(), int(fit[b]), [int(fit[b])])


@pytest.mark.parametrize("m,N,fit,breakage", [(12, 40, "f2", "unbalanced"), (20, 100, "f1", "first_column"),
                                              (36, 64, "f2", "random"), (8, 16, "f1", "random")])
def test_host_step_non_ga_population_is_exact(m, N, fit, breakage, cuda_device):
    """A Philox-config host state whose population breaks the GA invariants
    is stepped by the exact explicit-plan generation: the result equals the
    reference's step (oracle) on the same arrays, seed and generation."""
    cfg = engine.GAConfig(order=m, population=N, seed=31, fitness=fit, mutation_cols=2, mutation_row_pairs=3)
    rng = np.random.default_rng(m)
    pop = oracle.init_population(m, N, 31)
    # every matrix broken, so the breakage survives selection (columns move whole
    # and mutation swaps keep column sums): all three steps take the exact path
    if breakage == "unbalanced":
        pop[:, 0, 3] = -pop[:, 0, 3]
    elif breakage == "first_column":
        pop[:, 1, 0] = -1
    else:
        pop = rng.choice(np.array([-1, 1], dtype=np.int8), size=pop.shape)
    f = oracle.evaluate(pop, fit)
    hs = _host_state(cfg, 31, pop.copy(), f.copy())
    ref = oracle.OracleState(m, N, 31, fit, 2, 3, "multi", pop.copy(), f.copy(), 0, hs.best_fitness,
                             hs.best_matrix.copy(), [hs.best_fitness])
    for _ in range(3):
        hga.step(hs)
        oracle.step(ref)
        assert np.array_equal(hs.population, ref.population)
        assert np.array_equal(hs.fitness, ref.fitness)
    assert hs.trace == ref.trace and hs.best_fitness == ref.best_fitness
    assert np.array_equal(hs.best_matrix, ref.best_matrix)


def test_host_step_rejects_non_sign_and_bad_shapes_untouched(cuda_device):
    cfg = engine.GAConfig(order=20, population=50, seed=3, fitness="f2")
    pop = oracle.init_population(20, 50, 3)
    f = oracle.evaluate(pop, "f2")
    bad = pop.copy()
    bad[7, 3, 4] = 0
    hs = _host_state(cfg, 3, bad.copy(), f.copy())
    with pytest.raises(ValueError):
        hga.step(hs)
    assert np.array_equal(hs.population, bad) and np.array_equal(hs.fitness, f) and hs.iteration == 0
    # wrong shapes: ValueError before any native call
    hs2 = _host_state(cfg, 3, pop[:-4].copy(), f[:-4].copy())
    with pytest.raises(ValueError):
        hga.step(hs2)
    hs3 = _host_state(cfg, 3, pop.copy(), f[:-1].copy())
    with pytest.raises(ValueError):
        hga.step(hs3)
    # int32 fitness: stepped through scratch arrays, written back in the caller's dtype
    hs4 = _host_state(cfg, 3, pop.copy(), f.astype(np.int32))
    hs5 = _host_state(cfg, 3, pop.copy(), f.copy())
    hga.step(hs4)
    hga.step(hs5)
    assert hs4.fitness.dtype == np.int32
    assert np.array_equal(hs4.population, hs5.population) and np.array_equal(hs4.fitness, hs5.fitness)


def test_host_step_shared_arrays_and_config_change(cuda_device):
    """Two host states over the SAME arrays (the second registration of an
    address fails inside CUDA and must not break the step), then a config
    change on the same state object rebuilds the device bridge."""
    cfg = engine.GAConfig(order=20, population=200, seed=8, fitness="f2")
    pop = oracle.init_population(20, 200, 8)
    f = oracle.evaluate(pop, "f2")
    a = _host_state(cfg, 8, pop, f)
    b = _host_state(cfg, 8, pop, f)   # same numpy buffers
    hga.step(a)
    hga.step(b)
    assert np.array_equal(a.population, b.population)
    assert np.array_equal(a.fitness, oracle.evaluate(a.population, "f2"))
    big = np.concatenate([pop, oracle.init_population(20, 100, 9)])  # a larger array at a new address
    a.config = engine.GAConfig(order=20, population=300, seed=8, fitness="f1")
    a.population, a.fitness = big, oracle.evaluate(big, "f1")
    hga.step(a)
    assert np.array_equal(a.fitness, oracle.evaluate(a.population, "f1"))
    assert a._hga_bridge.cfg.population == 300
    # pinned torch memory viewed as numpy (cudaHostRegister refuses it)
    pt = torch.from_numpy(oracle.init_population(20, 200, 10)).pin_memory()
    c = _host_state(cfg, 8, pt.numpy(), oracle.evaluate(pt.numpy(), "f2"))
    hga.step(c)
    hga.step(c)
    assert np.array_equal(c.fitness, oracle.evaluate(c.population, "f2"))


# ------------------------------------------------------------ islands on one GPU


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _island_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, str(ROOT))
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as ora
        from paper_2208_14961_b200 import engine as eng
        from paper_2208_14961_b200.islands import (Exchange, GpuIsland, IslandConfig, island_seed, pack_payload,
                                                   run_islands, unpack_payload)

        torch.cuda.set_device(0)
        ex = Exchange()
        cfg = eng.GAConfig(order=20, population=500, seed=40, fitness="f2", mutation_cols=2, mutation_row_pairs=3,
                           max_iterations=100_000)
        isl = GpuIsland(cfg, island_seed(40, rank))
        isl.advance(7)
        total = cfg.total
        before_pop = isl.state.population
        before_fit = isl.state.fitness
        best_before = isl.best
        rec, fit = isl.elites(16)
        incoming = ex.ring_shift(pack_payload(rec, fit))
        r2, f2 = unpack_payload(incoming, 16, rec.shape[1])
        isl.receive(r2, f2)
        isl.sync()
        after_pop, after_fit = isl.state.population, isl.state.fitness
        slots = isl.last_received.cpu().numpy()
        worst = np.argsort(-before_fit, kind="stable")[:16]
        ok_slots = sorted(slots.tolist()) == sorted(worst.tolist())
        mig = eng._unpack(r2.reshape(-1).cuda(), 16, 20).cpu().numpy()
        ok_land = np.array_equal(after_pop[slots], mig) and np.array_equal(after_fit[slots], f2.cpu().numpy())
        keep = np.setdiff1d(np.arange(total), slots)
        ok_rest = np.array_equal(after_pop[keep], before_pop[keep])
        ok_best = isl.best == min(best_before, int(f2.min()))
        # the loop runs on from the new population (histogram rebuilt)
        fb = isl.state.fitness
        isl.advance(1)
        pop1 = isl.state.population
        order = np.argsort(fb, kind="stable")[:1000]
        ok_sel = sorted(p.tobytes() for p in pop1[:1000]) == sorted(after_pop[i].tobytes() for i in order)
        isl.advance(5)
        p2 = isl.state.population
        ok_inv = bool((p2[:, :, 0] == 1).all() and (p2[:, :, 1:].sum(axis=1) == 0).all())
        ok_fit = np.array_equal(isl.state.fitness, ora.evaluate(p2, "f2"))
        ok_trace = all(a >= b for a, b in zip(isl.state.trace, isl.state.trace[1:]))
        # the whole protocol with real GPU islands
        cfg2 = eng.GAConfig(order=20, population=500, seed=41, fitness="f2", mutation_cols=2, mutation_row_pairs=8,
                            max_iterations=400)
        rec2 = run_islands(cfg2, IslandConfig(migration_interval=20, migration_size=8, poll_interval=10))
        q.put((rank, ok_slots, ok_land, ok_rest, ok_best, ok_sel, ok_inv, ok_fit, ok_trace,
               (rec2.success, rec2.iterations, rec2.best_fitness, rec2.best_matrix.tolist(), rec2.winner_rank,
                rec2.migrations, rec2.trace)))
    except Exception as exc:  # noqa: BLE001 -- report to the parent
        import traceback

        q.put((rank, "error", traceback.format_exc()))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_two_gpu_islands_on_one_device(cuda_device):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_island_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=500) for _ in procs), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert r[1] != "error", r[2]
    for r in res:
        rank, *oks, rec = r
        assert all(oks), (rank, oks)
    assert res[0][-1] == res[1][-1]  # identical record on both ranks
    success, iters, best, matrix, winner, migrations, trace = res[0][-1]
    assert all(a >= b for a, b in zip(trace, trace[1:]))
    if success:
        q_ = np.array(matrix, dtype=np.int64)
        assert (q_.T @ q_ == 20 * np.eye(20, dtype=np.int64)).all()
    else:
        assert migrations >= 1 and iters == 400


# ------------------------------------------------------------ device invariant check (engine.py:440-446)


def test_device_invariant_check_counts_violations(cuda_device, monkeypatch):
    cfg = engine.GAConfig(order=28, population=2000, seed=3, fitness="f1", mutation_cols=2, mutation_row_pairs=3)
    st = hga.initial_state(cfg)
    engine._run_device(st, 5)
    assert engine.check_invariants(st) == (0, 0, 0)
    monkeypatch.setattr(engine, "DEBUG_CHECKS", True)
    hga.step(st)  # runs _check_state on the device after the generation
    res = st._res
    pop = res.pop[res.cur].view(cfg.total, cfg.order, res.W)
    saved = pop.clone()
    fsaved = res.fit[res.cur].clone()
    pop[7, 0, 0] ^= 1          # column 0 of matrix 7 gets a -1 (and becomes unbalanced-looking: counted once as c0)
    pop[9, 5, 0] ^= 0b11       # column 5 of matrix 9: popcount m/2 -> m/2 +- 2 (or unchanged when the bits differ)
    pop[11, 3, 0] ^= 1         # column 3 of matrix 11: popcount changes by one
    res.fit[res.cur][13] += 8  # stale fitness
    c0, c1, c2 = engine.check_invariants(st)
    assert c0 == 1 and c1 >= 1 and c2 >= 1  # the corrupted matrices' recomputed fitness also differs
    with pytest.raises(AssertionError):
        engine._check_state(st)
    pop.copy_(saved)
    res.fit[res.cur].copy_(fsaved)
    assert engine.check_invariants(st) == (0, 0, 0)


@pytest.mark.parametrize("m,N,fit,nc,nr", [(68, 300, "f2", 2, 3), (96, 200, "f1", 1, 4), (128, 150, "f2", 3, 2),
                                           (36, 500, "sq", 2, 3), (48, 300, "sq", 1, 5), (64, 200, "sq", 2, 2)])
def test_v1_loop_orders_and_sq(m, N, fit, nc, nr, cuda_device):
    """Orders 68..128 and SQ above order 32 run the round-1 loop kernel (k_run,
    generation.cu) instead of k_run_v3: invariants, fitness == oracle and the
    exact survivor set after single steps, plus a multi-generation launch."""
    cfg = engine.GAConfig(order=m, population=N, seed=19, fitness=fit, mutation_cols=nc, mutation_row_pairs=nr,
                          max_iterations=10_000)
    st = hga.initial_state(cfg)
    rng = np.random.default_rng(m)
    _device_invariants(st, None, rng)
    for _ in range(3):
        _check_selection_step(st)
        _device_invariants(st, None, rng)
    engine._run_device(st, 20, force=True)
    _device_invariants(st, None, rng)
    assert engine.check_invariants(st) == (0, 0, 0)
    assert all(a >= b for a, b in zip(st.trace, st.trace[1:])) and st.iteration == 23


def test_repeated_runs_are_bit_identical(cuda_device, monkeypatch):
    """Race smoke test (compute-sanitizer is closed on this pool): the
    hand-synchronised kernels -- the tcgen05 fitness pipeline (mbarrier rings,
    TMEM slots, shared-memory finalisation ring) and the persistent loop
    (one-atomic grid barrier, survivor lists) -- give bit-identical results
    over repeated runs on the same inputs, at sizes with many units / tiles
    per CTA."""
    monkeypatch.setenv("HGA_FITNESS_TC", "2")
    for m in (44, 48, 60, 64):
        pop = engine.init_population_device(engine.GAConfig(order=m, population=60_000, seed=m))
        ref = hga.penalties(pop)
        for _ in range(4):
            got = hga.penalties(pop)
            for k in ("f1", "f2", "orth", "sq"):
                assert torch.equal(got[k], ref[k]), (m, k)
    monkeypatch.delenv("HGA_FITNESS_TC")
    for m, N in ((20, 10_000), (36, 50_000)):
        outs = []
        for _ in range(3):
            st = hga.initial_state(engine.GAConfig(order=m, population=N, seed=5, fitness="f2", mutation_cols=2,
                                                   mutation_row_pairs=3, max_iterations=10_000))
            engine._run_device(st, 30, force=True)
            outs.append((list(st.trace), _hash_records(st._res.pop[st._res.cur].view(4 * N, -1)).sum().item(),
                         st.fitness_device.sum().item()))
        assert outs[0] == outs[1] == outs[2], m


@pytest.mark.parametrize("m,N,fit,mut", [(132, 24, "f2", "multi"), (160, 12, "f1", "per-matrix"),
                                         (256, 6, "f2", "shared")])
def test_orders_above_128_run_the_reference_generation(m, N, fit, mut, cuda_device):
    """Orders above the packed loops' 128 (the reference allows 4096,
    engine.py:57): the int8-layout path reproduces the reference step for
    step -- initial population, three generations and a stall restart."""
    cfg = engine.GAConfig(order=m, population=N, seed=23, fitness=fit, mutation=mut, mutation_cols=2,
                          mutation_row_pairs=3, max_iterations=6, stall_window=1)
    st = hga.initial_state(cfg)
    ref = oracle.initial_state(m, N, 23, fit, 2 if mut == "multi" else 1, 3 if mut == "multi" else 1, mut)
    assert np.array_equal(st.population, ref.population) and np.array_equal(st.fitness, ref.fitness)
    for _ in range(3):
        hga.step(st)
        oracle.step(ref)
        assert np.array_equal(st.population, ref.population) and np.array_equal(st.fitness, ref.fitness)
    assert st.trace == ref.trace and st.best_fitness == ref.best_fitness
    rec = hga.run_search(cfg)
    want = oracle.run_search(m, N, 23, fit, 2 if mut == "multi" else 1, 3 if mut == "multi" else 1, mut,
                             max_iterations=6, stall_window=1)
    assert rec.trace == want["trace"] and rec.iterations == want["iterations"]
    assert np.array_equal(rec.best_matrix, want["best_matrix"])


# ------------------------------------------------------------ bit-stream host step


@pytest.mark.parametrize("m,N,fit,nc,nr", [(4, 3, "f1", 1, 1), (16, 77, "f2", 1, 1), (20, 10_000, "f2", 4, 2), (36, 500, "f2", 1, 12),
                                           (48, 257, "f1", 2, 3), (64, 300, "f2", 3, 5), (12, 40, "sq", 2, 2),
                                           (36, 64, "sq", 2, 2)])
def test_host_step_bit_stream_matches_byte_path(m, N, fit, nc, nr, cuda_device, monkeypatch):
    """hga_step_host_bits (population moved as a bit stream, packed and
    unpacked on the host) gives exactly the populations, fitness and traces
    of the int8 path (hga_step_host) step after step; configs outside the
    loop's fast path (SQ above 32) take the generic path on both."""
    cfg = engine.GAConfig(order=m, population=N, seed=17, fitness=fit, mutation_cols=nc, mutation_row_pairs=nr)
    pop = oracle.init_population(m, N, 17)
    f = oracle.evaluate(pop, fit)
    a = _host_state(cfg, 17, pop.copy(), f.copy())
    b = _host_state(cfg, 17, pop.copy(), f.copy())
    monkeypatch.delenv("HGA_STEP_HOST", raising=False)
    hga.step(a)
    monkeypatch.setenv("HGA_STEP_HOST", "bytes")
    hga.step(b)
    monkeypatch.delenv("HGA_STEP_HOST")
    has_bits = int(engine.lib.hga_step_host_bits_bytes(N, m)) > 0
    assert bool(a._hga_bridge._bits) == has_bits and b._hga_bridge._bits is False
    for i in range(4):
        assert np.array_equal(a.population, b.population), i
        assert np.array_equal(a.fitness, b.fitness), i
        assert a.trace == b.trace and a.iteration == b.iteration == i + 1
        hga.step(a)
        hga.step(b)
    assert np.array_equal(a.population, b.population) and np.array_equal(a.fitness, b.fitness)
    p = a.population
    assert (p[:, :, 0] == 1).all() and (p[:, :, 1:].sum(axis=1) == 0).all()
    sample = np.arange(0, 4 * N, max(1, 4 * N // 4000))
    assert np.array_equal(a.fitness[sample], oracle.evaluate(p[sample], fit))
