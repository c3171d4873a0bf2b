"""Batched branch-and-bound (cubics_solve_optimize_batch) and the LNS built on it.

The reference runs each LNS neighbourhood as its own Dfs on a sub-model whose kept variables are
fixed to the incumbent (search.cpp:207-217, 277-285). Here every neighbourhood of an iteration is
one thread block of ONE launch; each must reproduce the oracle's branch-and-bound on the same
sub-model exactly: stats, objective, incumbent values and completeness."""
import math

import numpy as np
import pytest

from paper_1909_09213_b200 import _abi as A
from paper_1909_09213_b200 import models
from paper_1909_09213_b200 import solver as S

import oracle_binding as O

pytestmark = pytest.mark.gpu


def _destroy_sets(n, count, rate, seed, it=0):
    destroy = min(n, max(1, math.ceil(rate * n)))
    out = []
    for nb in range(count):
        rng = models.Rng.derive(seed, nb, it)
        ids = list(range(n))
        d = [False] * n
        for i in range(destroy):
            j = i + rng.below(n - i)
            ids[i], ids[j] = ids[j], ids[i]
            d[ids[i]] = True
        out.append(d)
    return out


def _neighbourhood_words(m, inc, destroyed):
    nw = m.word_start[-1]
    base = np.ctypeslib.as_array(m.words_of(m.domains))[:nw].copy()
    rows = np.tile(base, (len(destroyed), 1))
    for r, d in enumerate(destroyed):
        for v in range(m.n_vars):
            if not d[v]:
                a, b = m.word_start[v], m.word_start[v + 1]
                rows[r, a:b] = 0
                bit = inc[v] - m.offsets[v]
                rows[r, a + bit // 64] = np.uint64(1 << (bit % 64))
    return rows


def _sub_model(m, inc, d):
    # exactly the reference's neighborhood_model: Domain(val, val) for every kept variable
    doms = [m.domains[v] if d[v] else S.Domain(inc[v], bits=1, width=1) for v in range(m.n_vars)]
    return m.with_domains(doms)


def _first(m):
    got = []
    S.solve_satisfy(m, S.SearchConfig(max_solutions=1), lambda s: (got.append(s), False)[1])
    return got[0].values


@pytest.mark.parametrize("name,count,rate,limit", [
    ("golomb7", 24, 0.3, 0),
    ("golomb8", 40, 0.8, 300),
    ("assign12", 24, 0.5, 0),
    ("assign20", 48, 0.4, 0),
    ("assign30", 64, 0.4, 1500),
])
def test_batch_matches_oracle_per_neighbourhood(name, count, rate, limit):
    m = S.parse_model(models.named_instance(name))
    inc = _first(m)
    obj = inc[m.goal_var]
    sets = _destroy_sets(m.n_vars, count, rate, seed=7)
    cfg = S.SearchConfig(node_limit=limit, engine=A.ENGINE_PARITY)
    got = S.optimize_batch(m, _neighbourhood_words(m, inc, sets), [obj] * count, cfg)
    assert len(got) == count
    for d, g in zip(sets, got):
        ref = O.solve_optimize(_sub_model(m, inc, d), S.SearchConfig(node_limit=limit, initial_bound=obj))
        assert g.stats.as_tuple() == ref.stats.as_tuple()
        assert g.complete == ref.complete
        assert (g.best is None) == (ref.best is None)
        if ref.best is not None:
            assert g.best.objective == ref.best.objective
            assert g.best.values == ref.best.values


def test_batch_without_bound_is_solve_optimize():
    m = S.parse_model(models.named_instance("golomb7"))
    nw = m.word_start[-1]
    base = np.ctypeslib.as_array(m.words_of(m.domains))[:nw].copy()
    got = S.optimize_batch(m, np.tile(base, (3, 1)), None, S.SearchConfig(engine=A.ENGINE_PARITY))
    ref = O.solve_optimize(m)
    for g in got:
        assert g.stats.as_tuple() == ref.stats.as_tuple()
        assert g.best.objective == ref.best.objective and g.best.values == ref.best.values


def test_batch_mixed_bounds_and_empty_domains():
    m = S.parse_model(models.named_instance("golomb6"))
    inc = _first(m)
    sets = _destroy_sets(m.n_vars, 6, 0.4, seed=3)
    rows = _neighbourhood_words(m, inc, sets)
    a, b = m.word_start[2], m.word_start[3]
    rows[4, a:b] = 0  # problem 4: an empty domain -> fails at the root
    bounds = [inc[m.goal_var], None, inc[m.goal_var] - 3, None, None, 10 ** 6]
    got = S.optimize_batch(m, rows, bounds, S.SearchConfig(engine=A.ENGINE_PARITY))
    for i, (d, g) in enumerate(zip(sets, got)):
        sub = _sub_model(m, inc, d)
        if i == 4:
            doms = list(sub.domains)
            doms[2] = S.Domain(m.offsets[2], bits=0, width=m.widths[2])
            sub = m.with_domains(doms)
        ref = O.solve_optimize(sub, S.SearchConfig(initial_bound=bounds[i]))
        assert g.stats.as_tuple() == ref.stats.as_tuple(), i
        assert (g.best is None) == (ref.best is None), i
        if ref.best:
            assert g.best.values == ref.best.values, i


def test_batch_errors():
    m = S.parse_model(models.gen_nqueens(6))
    with pytest.raises(S.LogicError):
        S.optimize_batch(m, np.zeros((1, m.word_start[-1]), dtype=np.uint64))
    assert S.optimize_batch(S.parse_model(models.named_instance("golomb5")), np.zeros((0, 1), np.uint64)) == []


def _oracle_lns(m, cfg):
    """search.cpp:225-314 restated over the oracle (one Dfs per neighbourhood)."""
    got = []
    first = O.solve_satisfy(m, S.SearchConfig(max_solutions=1), lambda s: (got.append(s), False)[1])
    stats = S.SearchStats(*first.stats.as_tuple())
    best = S.Solution(got[0].values, got[0].values[m.goal_var])
    traj = []
    minimizing = m.goal == A.MINIMIZE
    for it in range(cfg.iterations):
        inc = best
        for d in _destroy_sets(m.n_vars, cfg.neighborhoods, cfg.destroy_rate, cfg.seed, it):
            r = O.solve_optimize(_sub_model(m, inc.values, d),
                                 S.SearchConfig(node_limit=cfg.per_iteration_node_limit, initial_bound=inc.objective))
            stats.nodes += r.stats.nodes
            stats.failures += r.stats.failures
            stats.rounds += r.stats.rounds
            if r.best and (r.best.objective < best.objective if minimizing else r.best.objective > best.objective):
                best = r.best
        traj.append(best.objective)
    return best, stats, traj


@pytest.mark.parametrize("name,iters,nbs,rate,seed,limit", [
    ("golomb7", 4, 8, 0.3, 1, 0),
    ("assign20", 4, 16, 0.4, 1, 0),
    ("assign30", 3, 64, 0.35, 5, 1500),
])
def test_lns_matches_reference_loop(name, iters, nbs, rate, seed, limit):
    m = S.parse_model(models.named_instance(name))
    cfg = S.LnsConfig(destroy_rate=rate, iterations=iters, neighborhoods=nbs, seed=seed,
                      per_iteration_node_limit=limit)
    got = S.lns_optimize(m, cfg)
    best, stats, traj = _oracle_lns(m, cfg)
    assert got.trajectory == traj
    assert got.stats.as_tuple()[:3] == stats.as_tuple()[:3]
    assert got.best.objective == best.objective and got.best.values == best.values
