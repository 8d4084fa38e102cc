"""Pin the CPU oracle against the reference's golden vectors (CPU only).

Golden values come from the unmodified reference package (see
tests/golden/make_golden.py); the hand-written cases mirror the
reference's own known-answer tests (pkg/tests/test_core.py:10-31, 78-88).
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from conftest import run_config


def test_stream_keys_and_words(golden):
    for a, s in enumerate(golden["rng_seeds"]):
        for b, i in enumerate(golden["rng_sids"]):
            assert oracle.stream_key(int(s), int(i)) == int(golden["rng_keys"][a, b])
    for a, s in enumerate(golden["rng_seeds"][:3]):
        w = oracle.stream_words(int(s), 17, 5, 64)
        assert np.array_equal(w, golden["rng_words_seed_sid17_c5"][a])


def test_uniform_and_permutation(golden):
    assert np.array_equal(oracle.uniform_array(99, 12, 0, 1, 11, 1000), golden["rng_uniform_99_12_1_11"])
    assert np.array_equal(oracle.uniform_array(7, 3, 11, 0, 35, 333), golden["rng_uniform_7_3_0_35"])
    for n in (1, 2, 5, 100, 1000, 4097):
        got = oracle.permutation(3, oracle.sid(2, 9), 2, n)
        assert np.array_equal(got, golden[f"rng_perm_{n}"]), n


def test_sid_packing():
    assert oracle.sid(2, 5) == (2 << 60) | (5 << 32)
    assert oracle.sid(1, 0, 3, 7) == (1 << 60) | (3 << 12) | 7


@pytest.mark.parametrize("m", [4, 8, 12, 20, 36, 64])
def test_random_balanced(golden, m):
    args = [int(v) for v in golden[f"init_m{m}_args"]]
    got = oracle.random_balanced(*args)
    assert np.array_equal(got, golden[f"init_m{m}"])


def test_fitness_all_cases(golden):
    for name in golden["fit_names"]:
        pop = golden[f"fit_pop_{name}"]
        want = golden[f"fit_val_{name}"]
        got = oracle.penalties(pop, threads=2)
        assert np.array_equal(got, want), name
        for col, fit in enumerate(("f1", "f2", "orth", "sq")):
            assert np.array_equal(oracle.evaluate(pop, fit, threads=1), want[:, col]), (name, fit)


def test_reference_known_answers(golden):
    # pkg/tests/test_core.py:78-88
    assert oracle.penalties(golden["fit_pop_all_ones_4"])[0, :2].tolist() == [48, 12]
    assert oracle.penalties(golden["fit_pop_h4"])[0, :2].tolist() == [0, 0]
    assert oracle.penalties(golden["fit_pop_known_case"])[0, :2].tolist() == [8, 2]
    for m in (20, 24, 28, 32):
        assert oracle.penalties(golden[f"fit_pop_fixture_{m}"])[:, :2].tolist() == [[0, 0], [0, 0]]
        # derived known answer: one sign flip of a Hadamard matrix
        assert oracle.penalties(golden[f"fit_pop_fixture_{m}_flip"])[0, :2].tolist() == [4 * (m - 1), 2 * (m - 1)]


@pytest.mark.parametrize("m", [8, 12, 20])
def test_select(golden, m):
    tag = f"select_m{m}"
    _, _, seed, gen = [int(v) for v in golden[f"{tag}_args"]]
    pop = golden[f"{tag}_pop_in"].copy()
    fit = golden[f"{tag}_fit_in"].copy()
    oracle.select(pop, fit, seed, oracle.sid(2, gen))
    assert np.array_equal(pop, golden[f"{tag}_pop_out"])
    assert np.array_equal(fit, golden[f"{tag}_fit_out"])


@pytest.mark.parametrize("m", [8, 12, 20, 36])
def test_crossover_and_mutation(golden, m):
    tag = f"xo_m{m}"
    _, n_pairs, seed, gen, nc, nr = [int(v) for v in golden[f"{tag}_args"]]
    pts = oracle.draw_crossover_points(m, n_pairs, seed, gen)
    assert np.array_equal(pts, golden[f"{tag}_points"])
    pop = golden[f"{tag}_pop_in"].copy()
    oracle.crossover(pop, pts)
    assert np.array_equal(pop, golden[f"{tag}_pop_out"])
    for strat in ("shared", "per-matrix", "multi"):
        s = strat.replace("-", "_")
        cols, ra, rb = oracle.make_mutation_plan(m, n_pairs, nc, nr, strat, seed, gen)
        assert np.array_equal(cols, golden[f"{tag}_plan_{s}_cols"]), strat
        assert np.array_equal(ra, golden[f"{tag}_plan_{s}_ra"]), strat
        assert np.array_equal(rb, golden[f"{tag}_plan_{s}_rb"]), strat
        mt = pop.copy()
        oracle.mutate(mt, cols, ra, rb)
        assert np.array_equal(mt, golden[f"{tag}_mut_{s}"]), strat


def test_figure2_crossover(golden):
    par = golden["fig2_parents"]
    pop = np.concatenate([par, np.zeros_like(par)])
    oracle.crossover(pop, np.array([3]))
    assert np.array_equal(pop[2:], golden["fig2_offspring"])


def test_whole_loop_records(golden):
    for i in range(int(golden["run_count"][0])):
        kw = run_config(golden, i)
        rec = oracle.run_search(
            kw["order"], kw["population"], kw["seed"], kw.get("fitness", "f2"),
            kw.get("mutation_cols", 1), kw.get("mutation_row_pairs", 2), kw.get("mutation", "multi"),
            kw.get("max_iterations", 100_000), kw.get("stall_window"), threads=2)
        it, best, succ = golden[f"run{i}_meta"].tolist()
        assert rec["trace"] == golden[f"run{i}_trace"].tolist(), i
        assert (rec["iterations"], rec["best_fitness"], int(rec["success"])) == (it, best, succ)
        assert np.array_equal(rec["best_matrix"], golden[f"run{i}_best"])


def test_three_step_state(golden):
    for i in range(int(golden["run_count"][0])):
        kw = run_config(golden, i)
        st = oracle.initial_state(kw["order"], kw["population"], kw["seed"], kw.get("fitness", "f2"),
                                  kw.get("mutation_cols", 1), kw.get("mutation_row_pairs", 2),
                                  kw.get("mutation", "multi"))
        for _ in range(min(3, kw["max_iterations"])):
            oracle.step(st)
        assert np.array_equal(st.population, golden[f"run{i}_state3_pop"]), i
        assert np.array_equal(st.fitness, golden[f"run{i}_state3_fit"]), i
