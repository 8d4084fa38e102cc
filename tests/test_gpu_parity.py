"""CUDA path vs the oracle and the reference's golden vectors (B200 only).

Bit-exact is the bar everywhere: fitness values, stream draws, init,
select/crossover/mutate results, and -- in reference-stream mode -- whole
RunRecords (trace, iteration count, best matrix) of the reference itself.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from conftest import run_config

pytestmark = pytest.mark.gpu

hga = pytest.importorskip("paper_2208_14961_b200")
from paper_2208_14961_b200 import engine  # noqa: E402
from paper_2208_14961_b200.rand import RngStream  # noqa: E402


# ------------------------------------------------------------------ fitness


def test_fitness_golden_all_cases(golden, cuda_device):
    for name in golden["fit_names"]:
        pop = golden[f"fit_pop_{name}"]
        want = golden[f"fit_val_{name}"]
        got = hga.penalties(pop)
        for col, key in enumerate(("f1", "f2", "orth", "sq")):
            assert np.array_equal(got[key], want[:, col]), (name, key)
        for col, key in enumerate(("f1", "f2", "orth", "sq")):
            assert np.array_equal(hga.evaluate(pop, key), want[:, col]), (name, key)


@pytest.mark.parametrize("m", [4, 8, 12, 16, 20, 24, 28, 32, 36, 40, 44, 48, 64, 96, 100, 128, 132, 200])
def test_fitness_random_vs_oracle(m, cuda_device):
    rng = np.random.default_rng(1000 + m)
    n = 300 if m <= 64 else 24
    bal = oracle.random_balanced(m, n, 77 + m, 1, 0, 0)
    unb = rng.choice(np.array([-1, 1], dtype=np.int8), size=(n // 3, m, m))
    for pop in (bal, unb):
        want = oracle.penalties(pop, threads=4)
        got = hga.penalties(pop)
        for col, key in enumerate(("f1", "f2", "orth", "sq")):
            assert np.array_equal(got[key], want[:, col]), (m, key)


@pytest.mark.parametrize("m", [1, 2, 3, 5, 6, 7, 9, 10, 13, 31, 33, 63, 65, 127, 129])
def test_fitness_odd_and_unaligned_orders(m, cuda_device):
    rng = np.random.default_rng(m)
    pop = rng.choice(np.array([-1, 1], dtype=np.int8), size=(37, m, m))
    want = oracle.penalties(pop)
    got = hga.penalties(pop)
    for col, key in enumerate(("f1", "f2", "orth", "sq")):
        assert np.array_equal(got[key], want[:, col]), (m, key)


def test_fitness_device_tensor_and_empty(cuda_device):
    pop = oracle.random_balanced(20, 50, 5, 1, 0, 0)
    t = torch.from_numpy(pop).cuda()
    out = hga.evaluate(t, "f1")
    assert out.is_cuda and out.dtype == torch.int64
    assert np.array_equal(out.cpu().numpy(), oracle.evaluate(pop, "f1"))
    assert hga.evaluate(np.zeros((0, 12, 12), np.int8), "f2").shape == (0,)


def test_fitness_rejects_non_sign(cuda_device):
    pop = np.ones((3, 12, 12), dtype=np.int8)
    pop[1, 4, 7] = 0
    with pytest.raises(ValueError):
        hga.evaluate(pop, "f2")
    pop[1, 4, 7] = 3
    with pytest.raises(ValueError):
        hga.evaluate(pop, "f1")
    with pytest.raises(ValueError):
        hga.evaluate(np.ones((2, 4, 4), np.int8), "f3")


@pytest.mark.parametrize("m", [4, 16, 20, 32, 36, 40, 44, 48, 52, 56, 60, 64])
def test_fitness_tensor_core_path_matches_popc_path(m, cuda_device, monkeypatch):
    """HGA_FITNESS_TC=all runs the Gram on tcgen05 (kind::i8, TMEM) at every
    order, HGA_FITNESS_TC=0 on the XOR+POPC kernel (default: tensor cores
    from m = 48).  Both must equal the oracle bit for bit,
    for odd batch sizes (the last MMA pair half empty) and fixtures."""
    rng = np.random.default_rng(m)
    pops = [oracle.random_balanced(m, 2047, 5 + m, 1, 0, 0),
            rng.choice(np.array([-1, 1], dtype=np.int8), size=(3, m, m)),
            rng.choice(np.array([-1, 1], dtype=np.int8), size=(1, m, m))]
    if m in (48, 64):
        h = hga.sylvester(6)[:m, :m] if m == 64 else None
        if h is not None:
            pops.append(np.stack([h, -h, h.T]))
    for pop in pops:
        want = oracle.penalties(pop, threads=4)
        monkeypatch.setenv("HGA_FITNESS_TC", "all")  # round-1 tensor-core kernel at every order
        got_tc = hga.penalties(pop)
        monkeypatch.setenv("HGA_FITNESS_TC", "0")
        got_pc = hga.penalties(pop)
        monkeypatch.setenv("HGA_FITNESS_TC", "2")  # round-2 tensor-core kernel (orders 36..64)
        got_t2 = hga.penalties(pop)
        monkeypatch.delenv("HGA_FITNESS_TC")
        for col, key in enumerate(("f1", "f2", "orth", "sq")):
            assert np.array_equal(got_tc[key], want[:, col]), (m, key, len(pop))
            assert np.array_equal(got_pc[key], want[:, col]), (m, key, len(pop))
            assert np.array_equal(got_t2[key], want[:, col]), (m, key, len(pop), "tc2")
        for key in ("f1", "f2"):
            assert np.array_equal(hga.evaluate(pop, key), want[:, ("f1", "f2").index(key)])


@pytest.mark.parametrize("m", list(range(4, 68, 4)))
@pytest.mark.parametrize("path", ["all", "2"])
def test_fitness_tensor_core_rejects_non_sign(m, path, cuda_device, monkeypatch):
    # round 1 checks bytes in {-1, 0, +1} on the staged tiles and zeros through
    # the nonzero count; round 2 (orders 36..64) with the dp4a identity
    # 128 sum v^2 == sum(127 v + u), sum v^2 == m^2: cover zeros, +-2, -3, the
    # int8 extremes, and pairs that cancel in one sum but not the other
    monkeypatch.setenv("HGA_FITNESS_TC", path)
    base = oracle.random_balanced(m, 13, 3, 1, 0, 0)
    cases = [[(0, 0, 0, 0)], [(4, m - 1, m - 1, 2)], [(2, m // 2, m - 1, -3)], [(3, 7 % m, 17 % m, 0)],
             [(1, 1 % m, 1 % m, -2)], [(0, m - 1, 0, -128)], [(4, 0, m // 2, 127)], [(12, m - 1, m - 2, 0)],
             [(9, 2, 3, 0), (9, 3, 3, 2)], [(8, 0, 1, 3), (8, 1, 1, -3)], [(7, m - 1, m - 1, -1 * 0)]]
    for case in cases:
        pop = base.copy()
        for (k, r, c, v) in case:
            pop[k, r, c] = v
        with pytest.raises(ValueError):
            hga.evaluate(pop, "f2")
    assert np.array_equal(hga.evaluate(base, "f2"), oracle.evaluate(base, "f2"))


@pytest.mark.parametrize("m", list(range(36, 68, 4)))
def test_fitness_tc2_many_units_vs_oracle(m, cuda_device, monkeypatch):
    """Round-2 tensor-core kernel over many pipeline units per CTA (stage and
    TMEM-slot rings wrap many times, partial last unit), all four penalties
    bit-exact; balanced and unbalanced populations."""
    monkeypatch.setenv("HGA_FITNESS_TC", "2")
    n = 148 * 8 * 9 + 5
    pop = np.concatenate([oracle.random_balanced(m, n - 1000, 11 + m, 1, 0, 0),
                          np.random.default_rng(m).choice(np.array([-1, 1], dtype=np.int8), size=(1000, m, m))])
    want = oracle.penalties(pop)
    got = hga.penalties(pop)
    for col, key in enumerate(("f1", "f2", "orth", "sq")):
        assert np.array_equal(got[key], want[:, col]), (m, key)
    for key in ("f1", "f2", "sq"):
        assert np.array_equal(hga.evaluate(pop, key), want[:, ("f1", "f2", "orth", "sq").index(key)]), (m, key)


def test_fitness_large_population_sampled(cuda_device):
    m, n = 20, 1_000_000
    pop_t = engine.init_population_device(engine.GAConfig(order=m, population=n // 4, seed=2024, rng="reference"))
    got = hga.evaluate(pop_t, "f2").cpu().numpy()
    idx = np.random.default_rng(0).choice(n, 2000, replace=False)
    sample = pop_t[torch.from_numpy(idx).cuda()].cpu().numpy()
    assert np.array_equal(got[idx], oracle.evaluate(sample, "f2"))
    # size-independent properties on the whole batch
    assert (got >= 0).all() and (got % 2 == 0).all()


def test_pack_unpack_roundtrip(cuda_device):
    for m in (4, 12, 20, 33, 64, 100, 130):
        pop = np.random.default_rng(m).choice(np.array([-1, 1], dtype=np.int8), size=(17, m, m))
        t = torch.from_numpy(pop).cuda()
        packed = engine._pack(t)
        back = engine._unpack(packed, 17, m).cpu().numpy()
        assert np.array_equal(back, pop), m
        pf = torch.empty(17, dtype=torch.int64, device="cuda")
        hga._lib.lib.hga_fitness_packed(packed.data_ptr(), 17, m, 2, None, pf.data_ptr(), None, None,
                                        torch.cuda.current_stream().cuda_stream)
        assert np.array_equal(pf.cpu().numpy(), oracle.evaluate(pop, "f2")), m


# ------------------------------------------------------------------ streams


def test_reference_streams(golden, cuda_device):
    for a, s in enumerate(golden["rng_seeds"][:3]):
        w = torch.empty(64, dtype=torch.int64, device="cuda")
        hga._lib.lib.hga_ref_words(int(s), 17, 5, 64, w.data_ptr(), torch.cuda.current_stream().cuda_stream)
        assert np.array_equal(w.cpu().numpy().view(np.uint64), golden["rng_words_seed_sid17_c5"][a])
    assert np.array_equal(RngStream(99, 12).uniform_array(1, 11, 1000), golden["rng_uniform_99_12_1_11"])
    assert np.array_equal(RngStream(7, 3, counter=11).uniform_array(0, 35, 333), golden["rng_uniform_7_3_0_35"])
    for n in (1, 2, 5, 100, 1000, 4097):
        st = RngStream(3, engine._sid(2, 9), counter=2)
        assert np.array_equal(st.permutation(n), golden[f"rng_perm_{n}"]), n
        assert st.counter == 2 + n - 1


def test_permutation_large_matches_oracle(cuda_device):
    # serial replay below 8192 entries, parallel replay (k_pfy_*) from 8192 on
    for n in (8191, 8192, 8193, 20_000, 50_000, 60_000, 200_001):
        got = RngStream(11, 5, counter=3).permutation(n)
        assert np.array_equal(got, oracle.permutation(11, 5, 3, n)), n


@pytest.mark.parametrize("m", [4, 8, 12, 20, 36, 64])
def test_init_golden(golden, m, cuda_device):
    mm, count, seed, purpose, gen, first = [int(v) for v in golden[f"init_m{m}_args"]]
    cfg = engine.GAConfig(order=m, population=1, rng="reference")
    packed = torch.empty(count * m * ((m + 31) // 32), dtype=torch.int32, device="cuda")
    engine._init_packed(cfg, seed, purpose, gen, first, count, packed)
    assert np.array_equal(engine._unpack(packed, count, m).cpu().numpy(), golden[f"init_m{m}"])


def test_init_population_matches_oracle(cuda_device):
    for m, n_pairs, seed in [(12, 100, 3), (20, 250, 2024), (36, 10, 9), (128, 2, 1), (132, 1, 4)]:
        cfg = engine.GAConfig(order=m, population=n_pairs, seed=seed, rng="reference")
        assert np.array_equal(hga.init_population(cfg), oracle.init_population(m, n_pairs, seed)), m


# ------------------------------------------------------------------ operators


@pytest.mark.parametrize("m", [8, 12, 20])
def test_select_golden(golden, m, cuda_device):
    tag = f"select_m{m}"
    _, _, seed, gen = [int(v) for v in golden[f"{tag}_args"]]
    pop = golden[f"{tag}_pop_in"].copy()
    fit = golden[f"{tag}_fit_in"].copy()
    st = RngStream(seed, engine._sid(2, gen))
    hga.select(pop, fit, st)
    assert np.array_equal(pop, golden[f"{tag}_pop_out"])
    assert np.array_equal(fit, golden[f"{tag}_fit_out"])
    assert st.counter == int(golden[f"{tag}_counter_after"][0])


def test_select_device_ties_and_large(cuda_device):
    rng = np.random.default_rng(3)
    for total, m, spread in [(4000, 12, 3), (40_000, 20, 50), (400, 8, 1)]:
        pop = oracle.random_balanced(m, total, 5, 1, 0, 0)
        fit = rng.integers(0, spread, size=total).astype(np.int64) * 4 + 100
        want_p, want_f = pop.copy(), fit.copy()
        oracle.select(want_p, want_f, 9, engine._sid(2, 3))
        tp, tf = torch.from_numpy(pop).cuda(), torch.from_numpy(fit).cuda()
        hga.select(tp, tf, RngStream(9, engine._sid(2, 3)))
        assert np.array_equal(tp.cpu().numpy(), want_p)
        assert np.array_equal(tf.cpu().numpy(), want_f)


def test_select_any_int64_range_matches_reference(cuda_device):
    """The reference sorts any int64 fitness (stable argsort, engine.py:245);
    spans beyond the histogram fall back to a stable radix sort."""
    rng = np.random.default_rng(8)
    for total, m, lo, hi in [(4000, 12, -(1 << 40), 1 << 40), (1000, 8, 0, 1 << 23), (6000, 16, -(1 << 62), 1 << 62)]:
        pop = oracle.random_balanced(m, total, 5, 1, 0, 0)
        fit = rng.integers(lo, hi, size=total, dtype=np.int64)
        fit[::7] = fit[3]  # ties across the whole range
        want_p, want_f = pop.copy(), fit.copy()
        oracle.select(want_p, want_f, 9, engine._sid(2, 3))
        assert sorted(want_f[: total // 2].tolist()) == np.sort(fit)[: total // 2].tolist()
        for host in (True, False):
            p, f = (pop.copy(), fit.copy()) if host else (torch.from_numpy(pop).cuda(), torch.from_numpy(fit).cuda())
            hga.select(p, f, RngStream(9, engine._sid(2, 3)))
            p = p if host else p.cpu().numpy()
            f = f if host else f.cpu().numpy()
            assert np.array_equal(p, want_p) and np.array_equal(f, want_f), (total, host)


@pytest.mark.parametrize("m", [8, 12, 20, 36])
def test_crossover_mutation_golden(golden, m, cuda_device):
    tag = f"xo_m{m}"
    _, n_pairs, seed, gen, nc, nr = [int(v) for v in golden[f"{tag}_args"]]
    cfg = engine.GAConfig(order=m, population=n_pairs, seed=seed, mutation_cols=nc, mutation_row_pairs=nr,
                          rng="reference")
    pts = hga.draw_crossover_points(cfg, seed, gen)
    assert np.array_equal(pts, golden[f"{tag}_points"])
    pop = golden[f"{tag}_pop_in"].copy()
    hga.crossover(pop, pts)
    assert np.array_equal(pop, golden[f"{tag}_pop_out"])
    for strat in ("shared", "per-matrix", "multi"):
        s = strat.replace("-", "_")
        scfg = engine.GAConfig(order=m, population=n_pairs, seed=seed, mutation_cols=nc, mutation_row_pairs=nr,
                               mutation=strat, rng="reference")
        plan = hga.make_mutation_plan(scfg, seed, gen)
        assert np.array_equal(plan.columns, golden[f"{tag}_plan_{s}_cols"])
        assert np.array_equal(plan.rows_a, golden[f"{tag}_plan_{s}_ra"])
        assert np.array_equal(plan.rows_b, golden[f"{tag}_plan_{s}_rb"])
        mt = pop.copy()
        hga.mutate(mt, plan)
        assert np.array_equal(mt, golden[f"{tag}_mut_{s}"]), strat


def test_operator_errors(cuda_device):
    pop = oracle.init_population(8, 2, 1)
    with pytest.raises(ValueError):
        hga.crossover(pop, np.array([1, 2, 3]))
    with pytest.raises(IndexError):
        hga.crossover(pop, np.array([0, 3]))
    with pytest.raises(IndexError):
        hga.crossover(pop, np.array([3, 8]))
    plan = engine.MutationPlan(np.ones((4, 1), np.int64), np.zeros((4, 1), np.int64), np.zeros((4, 1), np.int64))
    with pytest.raises(ValueError):
        hga.mutate(oracle.init_population(8, 3, 1), plan)
    with pytest.raises(IndexError):
        engine.MutationPlan(np.zeros((4, 1), np.int64), np.zeros((4, 1), np.int64), np.zeros((4, 1), np.int64))
    bad = engine.MutationPlan(np.full((4, 1), 8, np.int64), np.zeros((4, 1), np.int64), np.zeros((4, 1), np.int64))
    with pytest.raises(IndexError):
        hga.mutate(pop, bad)


def test_figure2_crossover(golden, cuda_device):
    par = golden["fig2_parents"]
    pop = np.concatenate([par, np.zeros_like(par)])
    hga.crossover(pop, np.array([3]))
    assert np.array_equal(pop[2:], golden["fig2_offspring"])


# ------------------------------------------------------------------ whole loop, reference streams


def test_reference_mode_state_after_three_steps(golden, cuda_device):
    for i in range(int(golden["run_count"][0])):
        kw = run_config(golden, i)
        cfg = engine.GAConfig(**kw, rng="reference")
        st = hga.initial_state(cfg)
        for _ in range(min(3, kw["max_iterations"])):
            hga.step(st)
        assert np.array_equal(st.population, golden[f"run{i}_state3_pop"]), i
        assert np.array_equal(st.fitness, golden[f"run{i}_state3_fit"]), i


def test_reference_mode_run_records(golden, cuda_device):
    for i in range(int(golden["run_count"][0])):
        kw = run_config(golden, i)
        rec = hga.run_search(engine.GAConfig(**kw, rng="reference"))
        it, best, succ = golden[f"run{i}_meta"].tolist()
        assert rec.trace == golden[f"run{i}_trace"].tolist(), i
        assert (rec.iterations, rec.best_fitness, int(rec.success)) == (it, best, succ), i
        assert np.array_equal(rec.best_matrix, golden[f"run{i}_best"]), i


# ------------------------------------------------------------------ drop-in step on host (numpy) states


def _host_state(cfg, seed, pop, fit, best_matrix, best):
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

    return HostState(cfg, seed, pop, fit, 0, best_matrix, best, [best])


def test_host_state_step_reference_streams(golden, cuda_device):
    """engine.step on numpy arrays (chunked copies + pack/unpack around the
    generation) reproduces the reference's own state after three steps."""
    for i in (0, 2, 5):
        kw = run_config(golden, i)
        cfg = engine.GAConfig(**kw, rng="reference")
        o = oracle.initial_state(cfg.order, cfg.population, kw["seed"], cfg.fitness, cfg.mutation_cols,
                                 cfg.mutation_row_pairs, cfg.mutation)
        hs = _host_state(cfg, kw["seed"], o.population, o.fitness, o.best_matrix, o.best_fitness)
        for _ in range(min(3, kw["max_iterations"])):
            hga.step(hs)
        assert np.array_equal(hs.population, golden[f"run{i}_state3_pop"]), i
        assert np.array_equal(hs.fitness, golden[f"run{i}_state3_fit"]), i
        assert hs.trace == golden[f"run{i}_trace"].tolist()[:len(hs.trace)], i


def test_host_state_step_philox_matches_device_state(cuda_device):
    for m, N in ((20, 1000), (12, 37), (36, 301)):
        cfg = engine.GAConfig(order=m, population=N, seed=21, fitness="f2", mutation_cols=2, mutation_row_pairs=3)
        dev = hga.initial_state(cfg)
        hs = _host_state(cfg, dev.seed, dev.population.copy(), dev.fitness.copy(), dev.best_matrix.copy(),
                         dev.best_fitness)
        for _ in range(4):
            hga.step(dev)
            hga.step(hs)
            assert np.array_equal(hs.population, dev.population), m
            assert np.array_equal(hs.fitness, dev.fitness), m
        assert hs.trace == dev.trace and hs.iteration == dev.iteration == 4


# ------------------------------------------------------------------ production (Philox) loop


def _invariants(st):
    pop = st.population
    assert (pop[:, :, 0] == 1).all()
    assert (pop[:, :, 1:].sum(axis=1, dtype=np.int64) == 0).all()
    assert np.array_equal(st.fitness, oracle.evaluate(pop, st.config.fitness))


@pytest.mark.parametrize("m,fit", [(12, "f2"), (20, "f1"), (28, "f2"), (36, "f1"), (64, "f2"), (16, "sq")])
def test_philox_steps_keep_invariants(m, fit, cuda_device):
    cfg = engine.GAConfig(order=m, population=300, seed=11, fitness=fit, mutation_cols=2, mutation_row_pairs=3)
    st = hga.initial_state(cfg)
    _invariants(st)
    prev = st.trace[-1]
    for _ in range(5):
        hga.step(st)
        _invariants(st)
        assert st.trace[-1] <= prev
        prev = st.trace[-1]
        assert st.trace[-1] == int(st.fitness.min())
    assert len(st.trace) == 6


def test_philox_parents_are_the_selected_set(cuda_device):
    cfg = engine.GAConfig(order=20, population=500, seed=4, fitness="f2")
    st = hga.initial_state(cfg)
    before_pop, before_fit = st.population, st.fitness
    hga.step(st)
    after = st.population
    half = 2 * cfg.population
    order = np.argsort(before_fit, kind="stable")[:half]
    want = {before_pop[i].tobytes() for i in order}
    got = [after[s].tobytes() for s in range(half)]
    assert sorted(got) == sorted(before_pop[i].tobytes() for i in order)
    assert set(got) == want
    assert np.array_equal(np.sort(st.fitness[:half]), np.sort(before_fit[order]))


def _check_solution(rec):
    assert oracle.penalties(rec.best_matrix[None])[0, 1] == 0
    assert hga.core.is_hadamard(rec.best_matrix)
    assert hga.core.is_balanced(rec.best_matrix)
    assert all(a >= b for a, b in zip(rec.trace, rec.trace[1:]))
    assert rec.trace[-1] == 0 and len(rec.trace) == rec.iterations + 1


def test_philox_search_finds_and_verifies(cuda_device):
    for m in (8, 12):
        rec = hga.run_search(engine.GAConfig(order=m, population=1000, seed=5, fitness="f1", max_iterations=3000))
        assert rec.success, m
        _check_solution(rec)
    # order 16 stalls for about half of all seeds in the reference too (the
    # oracle sticks at F1 = 96 for seeds 0, 1, 3): require one success in 6
    wins = 0
    for seed in range(6):
        rec = hga.run_search(engine.GAConfig(order=16, population=1000, seed=seed, fitness="f1", max_iterations=1500))
        if rec.success:
            _check_solution(rec)
            wins += 1
    assert wins >= 1


def test_philox_stochastic_parity_order12(cuda_device):
    """Stochastic parity: the reference solves m = 12, N = 1000,
    NC = 1, NR = 2, F1 in 30/30 seeds with a mean of 89.9 generations (range
    53-125).  The Philox loop draws different random numbers but must show
    the same behaviour; its seeds are fixed, so the check is deterministic.
    (rng="reference" reproduces the reference's 30 runs exactly:
    profiles/r01_stochastic_parity.jsonl.)"""
    its = []
    for sd in range(30):
        rec = hga.run_search(engine.GAConfig(order=12, population=1000, max_iterations=3000, mutation_cols=1,
                                             mutation_row_pairs=2, fitness="f1", seed=sd))
        assert rec.success, sd
        _check_solution(rec)
        its.append(rec.iterations)
    mean = sum(its) / len(its)
    assert 70 <= mean <= 115, mean  # reference 89.9; the standard error of a 30-run mean is ~4


def test_philox_stall_restart_runs(cuda_device):
    cfg = engine.GAConfig(order=16, population=50, seed=2, fitness="f2", max_iterations=300, stall_window=5)
    rec = hga.run_search(cfg)
    assert all(a >= b for a, b in zip(rec.trace, rec.trace[1:]))
    assert rec.best_fitness == rec.trace[-1] or rec.best_fitness <= rec.trace[-1]


@pytest.mark.parametrize("m,N,fit,nc,nr,sw", [(20, 1000, "f2", 4, 2, None), (12, 300, "f1", 1, 2, 4),
                                               (28, 2000, "f2", 2, 3, None), (36, 600, "f1", 3, 3, None),
                                               (16, 100, "sq", 1, 1, 3), (8, 32768, "f2", 1, 2, None),
                                               (64, 257, "f2", 5, 4, None)])
def test_one_barrier_loop_matches_two_barrier(m, N, fit, nc, nr, sw, cuda_device, monkeypatch):
    """The one-barrier generation loop (4N <= 131072) selects the same
    survivors with the same ranks as the two-barrier loop: identical runs."""
    from paper_2208_14961_b200._lib import RUN_ONE_BARRIER

    out = []
    for flags in (0, RUN_ONE_BARRIER):
        monkeypatch.setattr(engine, "_RUN_FLAGS", flags)
        cfg = engine.GAConfig(order=m, population=N, seed=9, fitness=fit, mutation_cols=nc, mutation_row_pairs=nr,
                              stall_window=sw, max_iterations=400)
        st = hga.initial_state(cfg)
        engine._run_device(st, 60)
        for _ in range(3):
            if st.best_fitness == 0:
                break
            hga.step(st)
        _invariants(st)
        out.append((list(st.trace), st.population, st.fitness, st.best_matrix))
    a, b = out
    assert a[0] == b[0]
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2]) and np.array_equal(a[3], b[3])


@pytest.mark.parametrize("m,N,fit,nc,nr,mut,sw", [(24, 333, "sq", 2, 5, "multi", 4), (24, 20000, "f2", 1, 10, "multi", None),
                                                   (28, 1000, "f2", 2, 3, "multi", None), (36, 600, "f1", 3, 3, "multi", None),
                                                   (40, 300, "f2", 1, 12, "multi", 5), (32, 257, "f2", 1, 2, "shared", None),
                                                   (36, 129, "f1", 1, 1, "per-matrix", None), (28, 70, "sq", 5, 2, "multi", 3)])
def test_throughput_tiles_match_team_tiles(m, N, fit, nc, nr, mut, sw, cuda_device, monkeypatch):
    """Orders 24..40 use one thread per child (the whole pair chain per warp)
    by default; it must give the same runs as the team-of-four tiles (same
    survivors, points, plans, operator order)."""
    out = []
    for flags in (0, 1 << 16):  # internal kRunTeamTiles
        monkeypatch.setattr(engine, "_RUN_FLAGS", flags)
        cfg = engine.GAConfig(order=m, population=N, seed=13, fitness=fit, mutation_cols=nc, mutation_row_pairs=nr,
                              mutation=mut, stall_window=sw, max_iterations=500)
        st = hga.initial_state(cfg)
        engine._run_device(st, 40)
        _invariants(st)
        out.append((list(st.trace), st.population, st.fitness, st.best_matrix))
    a, b = out
    assert a[0] == b[0]
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2]) and np.array_equal(a[3], b[3])


def test_evaluate_sharded_single_process(cuda_device):
    from paper_2208_14961_b200.islands import evaluate_sharded

    pop = oracle.random_balanced(28, 777, 4, 1, 0, 0)
    assert np.array_equal(evaluate_sharded(pop, "f2"), oracle.evaluate(pop, "f2"))


def test_single_gpu_island_and_elites(cuda_device):
    from paper_2208_14961_b200.islands import GpuIsland, IslandConfig, run_islands

    rec = run_islands(engine.GAConfig(order=12, population=1000, seed=3, fitness="f1", max_iterations=3000),
                      IslandConfig(migration_interval=50, migration_size=8, poll_interval=25))
    assert rec.success and rec.world == 1
    q = rec.best_matrix.astype(np.int64)
    assert (q.T @ q == 12 * np.eye(12, dtype=np.int64)).all()
    isl = GpuIsland(engine.GAConfig(order=20, population=500, seed=9), seed=9)
    isl.advance(3)
    fit = isl.state.fitness
    rec_e, fit_e = isl.elites(16)
    order = np.argsort(fit, kind="stable")[:16]
    assert np.array_equal(fit_e.cpu().numpy(), fit[order])
    pop = isl.state.population
    assert np.array_equal(engine._unpack(rec_e.reshape(-1), 16, 20).cpu().numpy(), pop[order])
    # migrants replace the 16 worst (largest fitness, lowest index first) and the loop keeps running
    isl.receive(rec_e, fit_e)
    after = isl.state.population
    worst = np.argsort(-fit, kind="stable")[:16]
    slots = isl.last_received.cpu().numpy()
    assert sorted(slots.tolist()) == sorted(worst.tolist())
    assert np.array_equal(after[slots], pop[order])
    isl.advance(2)
    p2 = isl.state.population
    assert np.array_equal(isl.state.fitness, oracle.evaluate(p2, "f2"))


from hypothesis import given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402


@settings(max_examples=60, deadline=None)
@given(m=st.integers(1, 70), n=st.integers(1, 300), seed=st.integers(0, 2**31), balanced=st.booleans())
def test_fitness_fuzz_vs_oracle(m, n, seed, balanced):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if balanced and m % 4 == 0:
        pop = oracle.random_balanced(m, n, seed, 1, 0, 0)
    else:
        pop = np.random.default_rng(seed).choice(np.array([-1, 1], dtype=np.int8), size=(n, m, m))
    want = oracle.penalties(pop, threads=2)
    got = hga.penalties(pop)
    for col, key in enumerate(("f1", "f2", "orth", "sq")):
        assert np.array_equal(got[key], want[:, col]), (m, key)


@pytest.mark.parametrize("total,k", [(10, 1), (4000, 7), (40_000, 16), (40_000, 20_000), (123_457, 999)])
def test_select_smallest_is_stable_topk(total, k, cuda_device):
    rng = np.random.default_rng(total + k)
    fit = rng.integers(0, 64, size=total).astype(np.int64) * 2
    t = torch.from_numpy(fit).cuda()
    out = torch.empty(k, dtype=torch.int64, device="cuda")
    wsb = int(hga._lib.lib.hga_select_ws_bytes(total))
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    rc = hga._lib.lib.hga_select_smallest(t.data_ptr(), total, k, out.data_ptr(), flag.data_ptr(), ws.data_ptr(), wsb,
                                          torch.cuda.current_stream().cuda_stream)
    assert rc == 0 and int(flag.item()) == 0
    assert np.array_equal(out.cpu().numpy(), np.argsort(fit, kind="stable")[:k])
