"""Generate the golden vectors that pin the oracle and the CUDA path.

Run ONLY in the build container, where the upstream reference package is
importable from /root/reference (it does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every array written here is produced by the unmodified reference package
(`hadamard_ga`, pkg/src/hadamard_ga/{rand,engine,core}.py) on fixed seeds,
plus the reference's own hand-written known-answer cases
(pkg/tests/test_core.py:10-31) and Hadamard fixtures
(pkg/tests/fixtures/hadamard_{20,24,28,32}.txt).  The output,
tests/golden/golden.npz, is committed; the tests read only that file.

The two extra penalty reductions the north star names (count of orthogonal
column pairs, sum of squared off-diagonal Gram entries) have no reference
implementation; their golden values are computed here from the reference's
exact int32 `core.gram` (core.py:59-67), i.e. they are pinned to the
reference Gram, not to our own code.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
REF_FIXTURES = Path("/root/reference/pkg/tests/fixtures")
OUT = Path(__file__).with_name("golden.npz")


def _import_reference():
    if str(REF_SRC) not in sys.path:
        sys.path.insert(0, str(REF_SRC))
    import hadamard_ga  # noqa: F401
    from hadamard_ga import core, engine, rand

    return core, engine, rand


def _parse_pm(text: str) -> np.ndarray:
    rows = [ln.strip() for ln in text.strip().splitlines() if ln.strip()]
    return np.array([[1 if ch == "+" else -1 for ch in r] for r in rows], dtype=np.int8)


def _load_fixture(path: Path) -> np.ndarray:
    lines = path.read_text().splitlines()
    assert lines[0].startswith("hadamard-ga matrix m=")
    return _parse_pm("\n".join(lines[1:]))


def gram_penalties(core, q: np.ndarray):
    """(f1, f2, orth, sq) of one matrix from the reference's exact Gram."""
    g = core.gram(q).astype(np.int64)
    m = g.shape[0]
    off = g[~np.eye(m, dtype=bool)]
    f1 = int(np.abs(g).sum()) - m * m
    f2 = int(np.count_nonzero(g)) - m
    iu = np.triu_indices(m, 1)
    orth = int((g[iu] == 0).sum())
    sq = int((off * off).sum())
    return f1, f2, orth, sq


def main() -> None:
    core, engine, rand = _import_reference()
    out: dict[str, np.ndarray] = {}

    # ---------------------------------------------------------------- rng
    seeds = [0, 1, 42, 2024, (1 << 64) - 1, 0x123456789ABCDEF0]
    sids = [0, 1, 17, 1 << 60, (1 << 64) - 1, engine._sid(2, 5), engine._sid(1, 0, 3, 7)]
    keys = np.array([[rand._stream_key(s, i) for i in sids] for s in seeds], dtype=np.uint64)
    out["rng_seeds"] = np.array(seeds, dtype=np.uint64)
    out["rng_sids"] = np.array(sids, dtype=np.uint64)
    out["rng_keys"] = keys
    words = []
    for s in seeds[:3]:
        st = rand.RngStream(s, 17, counter=5)
        words.append([st.next_u64() for _ in range(64)])
    out["rng_words_seed_sid17_c5"] = np.array(words, dtype=np.uint64)
    out["rng_uniform_99_12_1_11"] = rand.RngStream(99, 12).uniform_array(1, 11, 1000)
    out["rng_uniform_7_3_0_35"] = rand.RngStream(7, 3, counter=11).uniform_array(0, 35, 333)
    for n in (1, 2, 5, 100, 1000, 4097):
        out[f"rng_perm_{n}"] = rand.RngStream(3, engine._sid(2, 9), counter=2).permutation(n)

    # ---------------------------------------------------------------- init
    for m, count, seed, purpose, gen, first in [
        (4, 6, 5, 1, 0, 0),
        (8, 9, 11, 1, 0, 0),
        (12, 16, 2024, 1, 0, 0),
        (20, 12, 7, 7, 33, 40),
        (36, 5, (1 << 64) - 3, 1, 0, 0),
        (64, 3, 9, 7, 1000, 100),
    ]:
        pop = engine._random_balanced(m, count, seed, purpose, gen, first)
        out[f"init_m{m}"] = pop
        out[f"init_m{m}_args"] = np.array([m, count, seed, purpose, gen, first], dtype=np.uint64)

    # ---------------------------------------------------------------- fitness
    rng = np.random.default_rng(20240817)
    fit_cases = {}
    fit_cases["all_ones_4"] = np.ones((1, 4, 4), dtype=np.int8)
    fit_cases["h4"] = _parse_pm("++++\n+-+-\n++--\n+--+")[None]
    fit_cases["known_case"] = _parse_pm("-+++\n-+--\n+-+-\n+--+")[None]
    fit_cases["sylvester"] = np.stack([core.sylvester(5)])
    fixtures = []
    for m in (20, 24, 28, 32):
        h = _load_fixture(REF_FIXTURES / f"hadamard_{m}.txt")
        out[f"fixture_hadamard_{m}"] = h
        fixtures.append(h)
        fit_cases[f"fixture_{m}"] = np.stack([h, h.T.copy()])
        flip = h.copy()
        flip[3, 5] *= -1  # single sign flip: F1 = 4(m-1), F2 = 2(m-1)
        fit_cases[f"fixture_{m}_flip"] = flip[None]
    for m in (1, 2, 3, 5, 7, 9, 13, 31, 33):
        fit_cases[f"random_odd_m{m}"] = rng.choice(np.array([-1, 1], dtype=np.int8), size=(7, m, m))
    for m in (4, 8, 12, 16, 20, 24, 28, 32, 36, 40, 48, 64, 96, 100, 128):
        count = 40 if m <= 64 else 6
        fit_cases[f"balanced_m{m}"] = engine._random_balanced(m, count, 2024 + m, 1, 0, 0)
        fit_cases[f"unbalanced_m{m}"] = rng.choice(np.array([-1, 1], dtype=np.int8), size=(count // 2, m, m))
    fit_cases["all_ones_20"] = np.ones((2, 20, 20), dtype=np.int8)
    fit_cases["all_ones_65"] = np.ones((1, 65, 65), dtype=np.int8)
    names = sorted(fit_cases)
    out["fit_names"] = np.array(names)
    for name in names:
        pop = fit_cases[name]
        out[f"fit_pop_{name}"] = pop
        f1 = engine.evaluate(pop, "f1")
        f2 = engine.evaluate(pop, "f2")
        pen = np.array([gram_penalties(core, q) for q in pop], dtype=np.int64).reshape(-1, 4)
        assert np.array_equal(pen[:, 0], f1) and np.array_equal(pen[:, 1], f2), name
        out[f"fit_val_{name}"] = pen  # columns: f1, f2, orth, sq

    # ---------------------------------------------------------------- operators
    # select: identical population/fitness/stream in, population/fitness out
    for m, n_pairs, seed, gen, fitness in [(8, 5, 3, 1, "f2"), (12, 50, 77, 4, "f1"), (20, 33, 5, 123, "f2")]:
        cfg = engine.GAConfig(order=m, population=n_pairs, seed=seed, fitness=fitness)
        pop = engine.init_population(cfg, seed)
        fit = engine.evaluate(pop, fitness)
        if m == 8:  # force heavy ties to pin the stable tie-break
            fit = (fit // 8) * 8
        p2, f2v = pop.copy(), fit.copy()
        stream = rand.RngStream(seed, engine._sid(2, gen))
        engine.select(p2, f2v, stream)
        tag = f"select_m{m}"
        out[f"{tag}_args"] = np.array([m, n_pairs, seed, gen], dtype=np.uint64)
        out[f"{tag}_pop_in"], out[f"{tag}_fit_in"] = pop, fit
        out[f"{tag}_pop_out"], out[f"{tag}_fit_out"] = p2, f2v
        out[f"{tag}_counter_after"] = np.array([stream.counter], dtype=np.int64)

    # crossover points + crossover + mutation plans + mutate
    for m, n_pairs, seed, gen, nc, nr in [(8, 4, 9, 1, 3, 2), (12, 25, 31, 7, 1, 2), (20, 16, 5, 2, 4, 3), (36, 6, 1, 9, 2, 5)]:
        cfg = engine.GAConfig(order=m, population=n_pairs, seed=seed, mutation_cols=nc, mutation_row_pairs=nr)
        pop = engine.init_population(cfg, seed)
        pts = engine.draw_crossover_points(cfg, seed, gen)
        c1 = pop.copy()
        engine.crossover(c1, pts)
        tag = f"xo_m{m}"
        out[f"{tag}_args"] = np.array([m, n_pairs, seed, gen, nc, nr], dtype=np.uint64)
        out[f"{tag}_pop_in"], out[f"{tag}_points"], out[f"{tag}_pop_out"] = pop, pts, c1
        for strat in engine.MUTATION_STRATEGIES:
            scfg = engine.GAConfig(order=m, population=n_pairs, seed=seed, mutation_cols=nc,
                                   mutation_row_pairs=nr, mutation=strat)
            plan = engine.make_mutation_plan(scfg, seed, gen)
            mt = c1.copy()
            engine.mutate(mt, plan)
            s = strat.replace("-", "_")
            out[f"{tag}_plan_{s}_cols"] = plan.columns
            out[f"{tag}_plan_{s}_ra"] = plan.rows_a
            out[f"{tag}_plan_{s}_rb"] = plan.rows_b
            out[f"{tag}_mut_{s}"] = mt

    # paper Figure 2 crossover golden, c_cop = 3
    p1 = _parse_pm("-+++\n-+--\n+-+-\n+--+")
    p2 = _parse_pm("-+++\n+-++\n----\n++--")
    fig = np.stack([p1, p2, np.zeros_like(p1), np.zeros_like(p1)])
    engine.crossover(fig, np.array([3]))
    out["fig2_parents"] = np.stack([p1, p2])
    out["fig2_offspring"] = fig[2:]

    # ---------------------------------------------------------------- whole-loop records
    runs = [
        dict(order=8, population=20, max_iterations=200, fitness="f2", mutation="multi", seed=1),
        dict(order=12, population=100, max_iterations=400, fitness="f1", mutation="multi", seed=7, mutation_row_pairs=2),
        dict(order=12, population=250, max_iterations=60, fitness="f2", mutation="per-matrix", seed=11),
        dict(order=12, population=60, max_iterations=80, fitness="f2", mutation="shared", seed=13),
        dict(order=16, population=200, max_iterations=150, fitness="f1", mutation="multi", seed=5,
             mutation_cols=2, mutation_row_pairs=3, stall_window=6),
        dict(order=20, population=300, max_iterations=40, fitness="f2", mutation="multi", seed=2024,
             mutation_cols=2, mutation_row_pairs=4),
        dict(order=12, population=1000, max_iterations=3000, fitness="f1", mutation="multi", seed=3),
    ]
    for i, kw in enumerate(runs):
        rec = engine.run_search(engine.GAConfig(**kw))
        tag = f"run{i}"
        out[f"{tag}_cfg"] = np.array(repr(sorted(kw.items())))
        out[f"{tag}_trace"] = np.array(rec.trace, dtype=np.int64)
        out[f"{tag}_best"] = rec.best_matrix
        out[f"{tag}_meta"] = np.array([rec.iterations, rec.best_fitness, int(rec.success)], dtype=np.int64)
        # also pin the full state after 3 steps
        st = engine.initial_state(engine.GAConfig(**kw))
        for _ in range(min(3, kw["max_iterations"])):
            engine.step(st)
        out[f"{tag}_state3_pop"] = st.population
        out[f"{tag}_state3_fit"] = st.fitness
    out["run_count"] = np.array([len(runs)])

    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT} ({OUT.stat().st_size / 1e6:.2f} MB, {len(out)} arrays)")


if __name__ == "__main__":
    main()
