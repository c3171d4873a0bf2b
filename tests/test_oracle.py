"""Pin the CPU oracle port (oracle/cubics_oracle.c) against the unmodified reference.

Every expectation here was produced by the reference itself (oracle/_ref/fdref_driver, see
tests/golden/make_goldens.py). CPU only."""
import pytest

import golden_cases as G
import oracle_binding as O
from paper_1909_09213_b200 import models
from paper_1909_09213_b200 import solver as S


def run_case(key):
    inst, flags = G.split_key(key)
    m = S.parse_model(G.model_text(inst))
    cfg = G.cfg_from_flags(flags)
    if m.goal != 0:
        r = O.solve_optimize(m, cfg)
        return r.stats.as_tuple(), (r.best.values if r.best else None)
    first = []
    r = O.solve_satisfy(m, cfg, lambda s: (first.append(s.values) if not first else None) or True)
    return r.stats.as_tuple(), (first[0] if first else None)


@pytest.mark.parametrize("key", G.FAST_CASES)
def test_oracle_matches_reference_goldens(key):
    g = G.goldens()[key]
    stats, sol = run_case(key)
    assert stats == G.expected_tuple(g)
    assert sol == (g.get("best") if "best" in g else g.get("first"))


def test_oracle_corpus_all_solutions_and_fixpoints():
    c = G.corpus()["corpus"]
    for seed in range(200):
        rec = c[str(seed)]
        m = S.parse_model(models.corpus_instance(seed))
        stats = S.SearchStats()
        sols = O.enumerate_solutions(m, S.SearchConfig(), stats)
        assert [s.values for s in sols] == rec["all"]["all"], seed
        assert stats.as_tuple() == G.expected_tuple(rec["all"]), seed
        for name, cfg in (("all_fc", S.SearchConfig(alldiff=0)), ("all_input", S.SearchConfig(var_heuristic=0)),
                          ("first", S.SearchConfig(max_solutions=1))):
            st = S.SearchStats()
            O.enumerate_solutions(m, cfg, st)
            assert st.as_tuple() == G.expected_tuple(rec[name]), (seed, name)
        for name, level in (("fix_gac", 1), ("fix_fc", 0)):
            doms, fr = O.propagate_fixpoint(m, alldiff=level)
            exp = rec[name]
            assert fr.failed == exp["failed"] and fr.rounds == exp["rounds"], (seed, name)
            assert fr.failed_var == exp["failed_var"], (seed, name)
            assert [d.values() for d in doms] == exp["domains"], (seed, name)


def test_oracle_optimization_corpus():
    c = G.corpus()["optimization"]
    for seed in range(50):
        text, goal = models.optimization_instance(seed)
        m = S.parse_model(models.with_goal(text, goal))
        r = O.solve_optimize(m)
        exp = c[str(seed)]
        assert r.stats.as_tuple() == G.expected_tuple(exp), seed
        assert (r.best.values if r.best else None) == exp.get("best"), seed


def test_oracle_random_instances():
    c = G.corpus()["random"]
    for seed in range(100, 140):
        text, _ = models.random_instance(seed)
        m = S.parse_model(text)
        st = S.SearchStats()
        sols = O.enumerate_solutions(m, S.SearchConfig(), st)
        assert [s.values for s in sols] == c[str(seed)]["all"], seed
        assert st.as_tuple() == G.expected_tuple(c[str(seed)]), seed


@pytest.mark.parametrize("key", ["nq8|--all", "nq10|--all", "magic3|--all"])
def test_oracle_solution_stream_hash_matches_reference(key):
    """The oracle's full callback stream hashes to the reference's (tests/golden/stream_hashes.json,
    made by make_stream_hashes.py from oracle/_ref/fdref_driver --solutions-bin)."""
    import hashlib
    import json
    import os
    import struct

    with open(os.path.join(G.GOLDEN, "stream_hashes.json")) as f:
        h = json.load(f)[key]
    inst, flags = G.split_key(key)
    m = S.parse_model(G.model_text(inst))
    sols = O.enumerate_solutions(m, G.cfg_from_flags(flags))
    blob = b"".join(struct.pack("<%dq" % len(s.values), *s.values) for s in sols)
    assert len(sols) == h["rows"]
    assert hashlib.sha256(blob).hexdigest() == h["sha256"]


def test_stream_hash_fixture_consistent_with_goldens():
    import json
    import os

    with open(os.path.join(G.GOLDEN, "stream_hashes.json")) as f:
        hs = json.load(f)
    gold = G.goldens()
    assert "nq14|--all" in hs, "regenerate with make_stream_hashes.py --long"
    for key, h in hs.items():
        assert tuple(h["stats"]) == G.expected_tuple(gold[key]), key
        assert h["first"] == gold[key]["first"], key
        assert h["bytes"] == 8 * h["rows"] * h["n_vars"], key
