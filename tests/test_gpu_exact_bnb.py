"""Exact parallel branch and bound (cubics_solve_optimize, AUTO engine).

The reference's solve_optimize (search.cpp:187-201) visits nodes in DFS order with the bound of
the last improving solution; its stats and its sequence of incumbents are what every test here
checks, against the goldens of the unmodified reference and the pinned oracle. The engine gets
them from a chain of parallel exact-first-solution phases with static bounds, each seeded with the
pending right branches of a guided replay of the previous incumbent's path (engine.cu exact_bnb).
"""
import pytest

import golden_cases as G
import oracle_binding as O
from paper_1909_09213_b200 import _abi as A
from paper_1909_09213_b200 import models
from paper_1909_09213_b200 import solver as S

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def engine_present():
    assert S.device_count() >= 1, "no CUDA device visible to libcubics"


@pytest.mark.parametrize("inst", ["golomb5", "golomb6", "golomb7", "golomb8", "golomb9", "golomb10"])
def test_golomb_exact_stats_and_ruler(inst):
    g = G.goldens()[inst]
    m = S.parse_model(G.model_text(inst))
    r = S.solve_optimize(m, S.SearchConfig(device=0))
    assert r.engine == A.ENGINE_PARALLEL
    assert r.stats.as_tuple() == G.expected_tuple(g)
    assert r.best.objective == g["objective"] and r.best.values == g["best"]
    assert r.complete


def test_optimization_corpus_exact():
    c = G.corpus()["optimization"]
    for seed, g in c.items():
        text, goal = models.optimization_instance(int(seed))
        m = S.parse_model(models.with_goal(text, goal))
        r = S.solve_optimize(m, S.SearchConfig(device=0))
        assert r.stats.as_tuple() == G.expected_tuple(g), seed
        if g.get("best") is not None:
            assert r.best is not None and r.best.values == g["best"], seed
        else:
            assert r.best is None, seed


@pytest.mark.parametrize("name", ["assign8", "assign9", "magic4_max"])
def test_other_objectives_match_oracle(name):
    if name == "magic4_max":  # a maximize goal: the corner value of a 4x4 magic square
        text = models.magic(4).replace("solve satisfy;", "solve maximize m0_0;")
    else:
        text = models.assignment(int(name[6:]), seed=3)
    m = S.parse_model(text)
    r = S.solve_optimize(m, S.SearchConfig(device=0))
    o = O.solve_optimize(m, S.SearchConfig())
    assert r.stats.as_tuple() == o.stats.as_tuple()
    assert r.best.objective == o.best.objective and r.best.values == o.best.values


def test_initial_bound_is_honoured_exactly():
    # Dfs::set_initial_bound (search.cpp:63, 282): a strict bound from the start
    m = S.parse_model(G.model_text("golomb8"))
    for b in (40, 36, 35, 34):
        r = S.solve_optimize(m, S.SearchConfig(device=0, initial_bound=b))
        o = O.solve_optimize(m, S.SearchConfig(initial_bound=b))
        assert r.stats.as_tuple() == o.stats.as_tuple(), b
        assert (r.best.values if r.best else None) == (o.best.values if o.best else None), b


@pytest.mark.parametrize("k", [1, 3, 5])
def test_solution_cap_stops_after_k_incumbents(k):
    m = S.parse_model(G.model_text("golomb8"))
    r = S.solve_optimize(m, S.SearchConfig(device=0, max_solutions=k))
    o = O.solve_optimize(m, S.SearchConfig(max_solutions=k))
    assert r.engine == A.ENGINE_PARALLEL
    assert r.stats.as_tuple() == o.stats.as_tuple()
    assert r.best.values == o.best.values and r.complete == o.complete


@pytest.mark.parametrize("k", [1, 4, 19, 20, 50])
def test_incumbent_stream_through_solve_satisfy(k):
    # fd::solve_satisfy on a model with an objective: the callback sees the reference's
    # incumbents in order (streamed phase by phase by the exact parallel B&B)
    m = S.parse_model(models.assignment(9, seed=3))
    seen, oseen = [], []
    r = S.solve_satisfy(m, S.SearchConfig(device=0), lambda s: seen.append(s.values) or len(seen) < k)
    o = O.solve_satisfy(m, S.SearchConfig(), lambda s: oseen.append(s.values) or len(oseen) < k)
    assert r.engine == A.ENGINE_PARALLEL
    assert seen == oseen
    assert r.stats.as_tuple() == o.stats.as_tuple()
