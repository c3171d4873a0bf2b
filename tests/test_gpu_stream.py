"""Streaming solution delivery (cubics_solve_satisfy with a callback) on the default config.

The reference hands every solution to the callback as it is found and stops the search when the
callback returns false, reporting the stats at that point (search.cpp:134-156, stop :147-154).
The engine streams solutions through a host-mapped ring while the kernel runs; the parallel
engine's segments put them back into DFS order, and a stop reaches the device at once.
Expectations: the pinned oracle (tests/test_oracle.py) on the same model and callback.
"""
import time

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


def stop_after(k, acc):
    return lambda s: acc.append(s.values) or len(acc) < k


def oracle_stop(m, k, cfg=None):
    acc = []
    r = O.solve_satisfy(m, cfg or S.SearchConfig(), stop_after(k, acc))
    return r, acc


def test_stop_at_5_on_a_huge_search_returns_at_once_default_config():
    # nq20: 39,029,188,884 solutions. The default (AUTO) config picks the parallel engine; a
    # callback that stops at 5 must end the device search, not run it to completion.
    m = S.parse_model(models.gen_nqueens(20))
    S.solve_satisfy(m, S.SearchConfig(), stop_after(1, []))  # warm (module load, arenas)
    seen = []
    t0 = time.perf_counter()
    r = S.solve_satisfy(m, S.SearchConfig(), stop_after(5, seen))
    dt = time.perf_counter() - t0
    ro, oseen = oracle_stop(m, 5)
    assert r.engine == A.ENGINE_PARALLEL
    assert seen == oseen and len(seen) == 5
    assert r.stats.as_tuple() == ro.stats.as_tuple()
    assert r.complete is False
    assert dt < 2.0, f"stop took {dt:.3f} s"


@pytest.mark.parametrize("k", [1, 2, 7, 100, 1000, 5000, 14199, 14200])
def test_parallel_stream_stop_at_k_has_reference_stats(k):
    m = S.parse_model(G.model_text("nq12"))
    seen = []
    r = S.solve_satisfy(m, S.SearchConfig(), stop_after(k, seen))
    ro, oseen = oracle_stop(m, k)
    assert r.engine == A.ENGINE_PARALLEL
    assert seen == oseen
    assert r.stats.as_tuple() == ro.stats.as_tuple()
    assert r.complete is (k > 14200)


def test_parallel_stream_all_in_dfs_order():
    m = S.parse_model(G.model_text("nq12"))
    got = []
    r = S.solve_satisfy(m, S.SearchConfig(), lambda s: got.append(s.values) or True)
    ost = S.SearchStats()
    want = [s.values for s in O.enumerate_solutions(m, S.SearchConfig(), ost)]
    assert r.engine == A.ENGINE_PARALLEL and r.complete
    assert r.stats.as_tuple() == ost.as_tuple()
    assert got == want


@pytest.mark.parametrize("inst,flags", [("magic4", "--all"), ("nq10", "--all --fc"), ("nq10", "--all --input")])
@pytest.mark.parametrize("k", [3, 50])
def test_stream_stop_other_models(inst, flags, k):
    m = S.parse_model(G.model_text(inst))
    cfg = G.cfg_from_flags(flags.split())
    seen = []
    r = S.solve_satisfy(m, cfg, stop_after(k, seen))
    ro, oseen = oracle_stop(m, k, G.cfg_from_flags(flags.split()))
    assert seen == oseen
    assert r.stats.as_tuple() == ro.stats.as_tuple()


@pytest.mark.parametrize("k", [1, 9, 92, 93])
def test_parity_stream_stop(k):
    m = S.parse_model(G.model_text("nq8"))
    seen = []
    r = S.solve_satisfy(m, S.SearchConfig(engine=A.ENGINE_PARITY), stop_after(k, seen))
    ro, oseen = oracle_stop(m, k)
    assert r.engine == A.ENGINE_PARITY
    assert seen == oseen
    assert r.stats.as_tuple() == ro.stats.as_tuple()


def test_parity_stream_more_solutions_than_the_ring():
    # nq10 has 724 solutions; nq11 2,680 - with the explicit parity engine every one goes through
    # the ring (no 4M-row device buffer, no rerun)
    m = S.parse_model(models.gen_nqueens(11))
    got = []
    r = S.solve_satisfy(m, S.SearchConfig(engine=A.ENGINE_PARITY), lambda s: got.append(s.values) or True)
    ost = S.SearchStats()
    want = [s.values for s in O.enumerate_solutions(m, S.SearchConfig(), ost)]
    assert r.stats.as_tuple() == ost.as_tuple() and got == want


def test_stream_of_incumbents_on_an_objective_model():
    # solve_satisfy on a model with a goal: the reference's DFS passes each improving solution
    # (branch and bound) to the callback; stop after the second one
    m = S.parse_model(models.golomb(6, 36))
    for k in (1, 2, 100):
        seen = []
        r = S.solve_satisfy(m, S.SearchConfig(), stop_after(k, seen))
        ro, oseen = oracle_stop(m, k)
        assert seen == oseen
        assert r.stats.as_tuple() == ro.stats.as_tuple()


def test_callback_starting_another_search_fails_loudly():
    m = S.parse_model(G.model_text("nq8"))
    inner = []

    def cb(s):
        try:
            S.solve_satisfy(m, S.SearchConfig())
        except ValueError as e:  # the device is busy with this very search
            inner.append(str(e))
        return False

    S.solve_satisfy(m, S.SearchConfig(), cb)
    assert inner and "callback" in inner[0]


def test_stream_after_stop_is_clean():
    # a stopped stream leaves the device ready: the next call is exact
    m = S.parse_model(G.model_text("nq10"))
    S.solve_satisfy(m, S.SearchConfig(), stop_after(3, []))
    st = S.SearchStats()
    sols = S.enumerate_solutions(m, S.SearchConfig(), st)
    ost = S.SearchStats()
    O.enumerate_solutions(m, S.SearchConfig(), ost)
    assert st.as_tuple() == ost.as_tuple() and len(sols) == 724


@pytest.mark.parametrize("k", [2, 10, 500, 14200, 20000])
def test_first_k_solutions_on_the_parallel_engine_are_exact(k):
    # AUTO with max_solutions = k: the parallel engine streams and stops at the k-th solution;
    # stats and rows equal the reference's first k (search.cpp:151-154)
    m = S.parse_model(G.model_text("nq12"))
    ost = S.SearchStats()
    want = [s.values for s in O.enumerate_solutions(m, S.SearchConfig(max_solutions=k), ost)]
    st = S.SearchStats()
    got = [s.values for s in S.enumerate_solutions(m, S.SearchConfig(max_solutions=k), st)]
    assert st.as_tuple() == ost.as_tuple() and got == want
    r = S.solve_satisfy(m, S.SearchConfig(max_solutions=k))  # no callback: counts only
    assert r.engine == A.ENGINE_PARALLEL
    assert r.stats.as_tuple() == ost.as_tuple()
    assert r.complete is (k > 14200)


def test_stream_from_the_grid_context_on_a_large_model():
    # AUTO on a 100k-variable model picks the grid-wide reference-order context; its solutions and
    # stop flag go through the same ring (search.cuh EvKind)
    key = "rcsp_100000|--max 1 --node-limit 200"
    g = G.goldens()[key]
    inst, flags = G.split_key(key)
    m = S.parse_model(G.model_text(inst))
    seen = []
    r = S.solve_satisfy(m, G.cfg_from_flags(flags), lambda s: seen.append(s.values) or True)
    assert r.engine == A.ENGINE_GRID
    assert r.stats.as_tuple() == G.expected_tuple(g)
    assert (seen[0] if seen else None) == g.get("first")


@pytest.mark.parametrize("k", [1, 5, 40])
def test_stream_stop_on_table_models(k):
    # extensional constraints (BASELINE config 5, checked against the oracle's table extension)
    m = S.parse_model(models.random_binary_csp(12, 4, 18, 0.35, seed=7))
    seen = []
    r = S.solve_satisfy(m, S.SearchConfig(), stop_after(k, seen))
    ro, oseen = oracle_stop(m, k)
    assert seen == oseen
    assert r.stats.as_tuple() == ro.stats.as_tuple()


def test_stream_stops_across_the_acceptance_corpus():
    # the 200-instance acceptance corpus (acceptance.cpp:47-54), each streamed on the default
    # config and stopped at a seeded random k: the delivered prefix and the stats equal the oracle's
    import random

    rnd = random.Random(20261019)
    c = G.corpus()["corpus"]
    checked = 0
    for seed in range(200):
        total = len(c[str(seed)]["all"]["all"])
        if total == 0:
            continue
        k = rnd.randint(1, total + 1)
        m = S.parse_model(models.corpus_instance(seed))
        seen = []
        r = S.solve_satisfy(m, S.SearchConfig(), stop_after(k, seen))
        ro, oseen = oracle_stop(m, k)
        assert seen == oseen, seed
        assert r.stats.as_tuple() == ro.stats.as_tuple(), seed
        checked += 1
    assert checked > 50  # the instances with at least one solution
