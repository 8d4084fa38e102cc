"""GAConfig validation and detect_stall (host logic, CPU): every error branch
of engine.GAConfig.__post_init__ (reference engine.py:114-137) and
detect_stall (engine.py:472-479) against the reference's own behaviour."""

from __future__ import annotations

from types import SimpleNamespace

import pytest

from paper_2208_14961_b200 import engine
from paper_2208_14961_b200.engine import GAConfig, detect_stall


@pytest.mark.parametrize("kw", [
    dict(order=0), dict(order=6), dict(order=-4), dict(order=4.0), dict(order=8192),
    dict(order=12, population=0), dict(order=12, population=engine.MAX_POPULATION + 1, rng="reference"),
    dict(order=12, population=engine.MAX_POPULATION_PHILOX + 1),
    dict(order=12, max_iterations=-1), dict(order=12, max_iterations=engine.MAX_ITERATIONS + 1),
    dict(order=12, mutation_cols=0), dict(order=12, mutation_cols=12),
    dict(order=12, mutation_row_pairs=0), dict(order=12, mutation_row_pairs=7),
    dict(order=12, fitness="f3"), dict(order=12, mutation="uniform"), dict(order=12, seed="7"),
    dict(order=12, stall_window=0), dict(order=12, time_budget_secs=0), dict(order=12, time_budget_secs=-1.0),
    dict(order=12, rng="mt19937"), dict(order=68, fitness="sq"),
])
def test_gaconfig_rejects(kw):
    with pytest.raises(ValueError):
        GAConfig(**kw)


def test_gaconfig_accepts_limits_and_properties():
    c = GAConfig(order=12, population=engine.MAX_POPULATION, rng="reference", mutation_cols=11, mutation_row_pairs=6,
                 max_iterations=0, stall_window=1, time_budget_secs=0.5, seed=3)
    assert (c.k, c.parents, c.total) == (3, 2 * c.population, 4 * c.population)
    # the production (Philox) loop widens N past the reference's stream-id cap (config 4 island)
    GAConfig(order=36, population=312_500)
    GAConfig(order=4096, population=1)


def _st(trace):
    return SimpleNamespace(trace=list(trace))


def test_detect_stall_rules():
    with pytest.raises(ValueError):
        detect_stall(_st([5, 5, 5]), 0)
    with pytest.raises(ValueError):
        detect_stall(_st([5, 5, 5]), -3)
    assert detect_stall(_st([9, 5, 5, 5]), 3)
    assert not detect_stall(_st([5, 5]), 3)          # trace shorter than the window
    assert not detect_stall(_st([6, 5, 5]), 3)       # not flat over the window
    assert not detect_stall(_st([0, 0, 0]), 3)       # solved: never a stall
    assert detect_stall(_st([7]), 1)
