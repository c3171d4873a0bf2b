"""Parity of the CUDA engine (through the C ABI) with the reference / the pinned oracle.

Expectations come from the unmodified reference (tests/golden/*.json) or from the oracle port
that tests/test_oracle.py pins to it. Bit-exact: stats, solutions, solution order, domains.
"""
import itertools

import pytest

import golden_cases as G
import oracle_binding as O
from paper_1909_09213_b200 import _abi as A
from paper_1909_09213_b200 import models
from paper_1909_09213_b200 import solver as S

pytestmark = pytest.mark.gpu

PARITY = A.ENGINE_PARITY
PARALLEL = A.ENGINE_PARALLEL


@pytest.fixture(scope="module", autouse=True)
def engine_present():
    # fail loudly (never skip) when the native engine is absent on a GPU box
    assert S.device_count() >= 1, "no CUDA device visible to libcubics"


def gpu_case(key, engine):
    inst, flags = G.split_key(key)
    m = S.parse_model(G.model_text(inst))
    cfg = G.cfg_from_flags(flags)
    cfg.engine = engine
    if m.goal != 0:
        r = S.solve_optimize(m, cfg)
        return r.stats.as_tuple(), (r.best.values if r.best else None)
    first = []
    r = S.solve_satisfy(m, cfg, lambda s: (first.append(s.values) if not first else None) or True)
    return r.stats.as_tuple(), (first[0] if first else None)


@pytest.mark.parametrize("key", G.FAST_CASES + ["nq10|--all", "nq12|--all", "golomb9",
                                                 "magic4|--all --node-limit 20000",
                                                 "rcsp_100000|--max 1 --node-limit 200"])
def test_parity_engine_matches_reference(key):
    g = G.goldens()[key]
    stats, sol = gpu_case(key, PARITY)
    assert stats == G.expected_tuple(g)
    assert sol == (g.get("best") if "best" in g else g.get("first"))


@pytest.mark.parametrize("key", ["nq4|--all", "nq6|--all", "nq8|--all", "nq8|--all --fc", "nq8|--all --input",
                                 "nq10|--all", "nq12|--all", "magic3|--all"])
def test_parallel_engine_exact_on_complete_enumerations(key):
    g = G.goldens()[key]
    stats, sol = gpu_case(key, PARALLEL)
    assert stats == G.expected_tuple(g)
    assert sol == g["first"]


def test_parallel_solution_stream_in_reference_order():
    m = S.parse_model(G.model_text("nq8"))
    expect = [s.values for s in O.enumerate_solutions(m)]
    for eng in (PARITY, PARALLEL):
        got = [s.values for s in S.enumerate_solutions(m, S.SearchConfig(engine=eng))]
        assert got == expect


def test_corpus_solutions_fixpoints_and_first():
    c = G.corpus()["corpus"]
    for seed in range(200):
        rec = c[str(seed)]
        m = S.parse_model(models.corpus_instance(seed))
        for eng in (PARITY, PARALLEL):
            st = S.SearchStats()
            sols = S.enumerate_solutions(m, S.SearchConfig(engine=eng), st)
            assert [s.values for s in sols] == rec["all"]["all"], (seed, eng)
            assert st.as_tuple() == G.expected_tuple(rec["all"]), (seed, eng)
        for name, cfg in (("all_fc", S.SearchConfig(alldiff=0)), ("all_input", S.SearchConfig(var_heuristic=0)),
                          ("first", S.SearchConfig(max_solutions=1))):
            st = S.SearchStats()
            S.enumerate_solutions(m, cfg, st)
            assert st.as_tuple() == G.expected_tuple(rec[name]), (seed, name)
        for name, level in (("fix_gac", 1), ("fix_fc", 0)):
            doms, fr = S.propagate_fixpoint(m, alldiff=level)
            exp = rec[name]
            assert (fr.failed, fr.rounds, fr.failed_var) == (exp["failed"], exp["rounds"], exp["failed_var"]), (seed, name)
            assert [d.values() for d in doms] == exp["domains"], (seed, name)


def test_corpus_removals_per_constraint():
    for seed in range(200):
        m = S.parse_model(models.corpus_instance(seed))
        for level in (0, 1):
            for c in range(m.n_cons):
                assert S.removals(m, cons=[c], alldiff=level) == O.removals(m, cons=[c], alldiff=level), (seed, c)
            assert S.removals(m, alldiff=level) == O.removals(m, alldiff=level), seed


def test_optimization_corpus():
    c = G.corpus()["optimization"]
    for seed in range(50):
        text, goal = models.optimization_instance(seed)
        m = S.parse_model(models.with_goal(text, goal))
        exp = c[str(seed)]
        r = S.solve_optimize(m, S.SearchConfig(engine=PARITY))
        assert r.stats.as_tuple() == G.expected_tuple(exp), seed
        assert (r.best.values if r.best else None) == exp.get("best"), seed
        rp = S.solve_optimize(m, S.SearchConfig(engine=PARALLEL))
        assert (rp.best is None) == (r.best is None), seed
        if r.best:
            assert rp.best.objective == r.best.objective, seed


def test_random_instances():
    c = G.corpus()["random"]
    for seed in range(100, 140):
        text, _ = models.random_instance(seed)
        m = S.parse_model(text)
        st = S.SearchStats()
        sols = S.enumerate_solutions(m, S.SearchConfig(), st)
        assert [s.values for s in sols] == c[str(seed)]["all"], seed
        assert st.as_tuple() == G.expected_tuple(c[str(seed)]), seed


# ---- acceptance.cpp:184-301 (criterion 5) inputs: per-propagator removals vs the oracle
def _subset_domains(lo, hi, bits_list):
    doms = []
    for bits in bits_list:
        d = S.Domain(lo, hi)
        for b in range(hi - lo + 1):
            if not (bits >> b) & 1:
                d.remove(lo + b)
        doms.append(d)
    return doms


def test_relbin_exhaustive_small_domains():
    texts = []
    for op in ["<", "<=", ">", ">=", "=", "!="]:
        for off in (-1, 0, 2):
            rhs = "y" if off == 0 else (f"y + {off}" if off > 0 else f"y - {-off}")
            texts.append(f"var x in 1..4; var y in 1..4; constraint x {op} {rhs}; solve satisfy;")
        texts.append(f"var x in 1..4; var y in 1..4; constraint x {op} 2; solve satisfy;")
    for t in texts:
        m = S.parse_model(t)
        for bx in range(1, 16):
            for by in range(1, 16):
                doms = _subset_domains(1, 4, [bx, by])
                assert S.removals(m, doms) == O.removals(m, doms), (t, bx, by)


def test_alldiff_exhaustive_triples():
    m = S.parse_model("var x in 1..3; var y in 1..3; var z in 1..3; constraint alldifferent(x, y, z); solve satisfy;")
    for bx, by, bz in itertools.product(range(1, 8), repeat=3):
        doms = _subset_domains(1, 3, [bx, by, bz])
        for level in (0, 1):
            assert S.removals(m, doms, alldiff=level) == O.removals(m, doms, alldiff=level), (bx, by, bz, level)
            gd, gf = S.propagate_fixpoint(m, doms, alldiff=level)
            od, of = O.propagate_fixpoint(m, doms, alldiff=level)
            assert gd == od and gf == of, (bx, by, bz, level)


def test_random_linear_and_alldiff4():
    rng = models.Rng(5150)
    for trial in range(400):
        doms = []
        for v in range(4):
            d = S.Domain(1, 8)
            for x in range(1, 9):
                if d.size() > 1 and rng.below(2) == 0:
                    d.remove(x)
            doms.append(d)
        a0, a1, a2 = rng.range(-3, 3), rng.range(1, 3), rng.range(-2, 2)
        op = "<=" if rng.below(2) else "="
        bound = rng.range(-10, 25)
        a0, a2 = a0 or 1, a2 or 1
        t = (f"var a in 1..8; var b in 1..8; var c in 1..8; var d in 1..8; "
             f"constraint {a0}*a + {a1}*b + {a2}*c {op} {bound}; constraint alldifferent(a, b, c, d); solve satisfy;")
        t = t.replace("+ -", "- ")
        m = S.parse_model(t)
        for level in (0, 1):
            assert S.removals(m, doms, alldiff=level) == O.removals(m, doms, alldiff=level), (trial, t)


def test_pigeonhole_fails_at_root():
    m = S.parse_model("var a in 1..2;\nvar b in 1..2;\nvar c in 1..2;\nconstraint alldifferent(a, b, c);\nsolve satisfy;")
    st = S.SearchStats()
    assert S.enumerate_solutions(m, S.SearchConfig(), st) == []
    assert (st.nodes, st.failures) == (1, 1)


def test_overflow_raises_reference_exception():
    m = S.parse_model("var x in 1..5; var y in 1..5; constraint 4611686018427387904*x + 4611686018427387904*y <= 3; "
                      "solve satisfy;")
    with pytest.raises(S.ArithmeticOverflowError):
        S.solve_satisfy(m, S.SearchConfig())
    with pytest.raises(S.ArithmeticOverflowError):
        O.solve_satisfy(m, S.SearchConfig())


def test_optimize_without_objective_is_logic_error():
    m = S.parse_model("var x in 1..3; solve satisfy;")
    with pytest.raises(S.LogicError):
        S.solve_optimize(m, S.SearchConfig())


def test_callback_stop_truncates_stats_like_reference():
    # reference search.cpp:147-149: a callback returning false stops the search right there
    m = S.parse_model(G.model_text("nq8"))
    for k in (1, 5, 40):
        seen = []
        r = S.solve_satisfy(m, S.SearchConfig(engine=PARITY), lambda s: seen.append(s) or len(seen) < k)
        ro = O.solve_satisfy(m, S.SearchConfig(), (lambda acc: (lambda s: acc.append(s) or len(acc) < k))([]))
        assert r.stats.as_tuple() == ro.stats.as_tuple()
        assert r.complete is False and len(seen) == k


@pytest.mark.parametrize("key", ["nq8|--all", "nq10|--all", "nq12|--all", "magic3|--all", "nq8|--all --fc"])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_search_sums_exactly(key, world):
    # every rank's cubics_solve_shard, run one after another on this GPU; the sum of the shards'
    # stats is the reference's, and their key-merged solutions are the reference's stream
    from paper_1909_09213_b200 import distributed as D

    inst, flags = G.split_key(key)
    m = S.parse_model(G.model_text(inst))
    cfg = G.cfg_from_flags(flags)
    tot = [0, 0, 0, 0]
    streams = []
    for r in range(world):
        keyed = []
        res = S.solve_shard(m, cfg, r, world, lambda k, v, keyed=keyed: keyed.append((tuple(k), v)) or True)
        tot = [a + b for a, b in zip(tot, res.stats.as_tuple())]
        streams.append(keyed)
    g = G.goldens()[key]
    assert tuple(tot) == G.expected_tuple(g)
    merged = D.merge_keyed(streams)
    assert merged == [s.values for s in O.enumerate_solutions(m, cfg)]


# ---- generic alldifferent path (> 64 members or a value universe wider than 1024)
def _random_alldiff_model(rng, n, width, offsets=None):
    offs = offsets or [1] * n
    lines = [f"var v{i} in {offs[i]}..{offs[i] + width - 1};" for i in range(n)]
    lines.append("constraint alldifferent(" + ", ".join(f"v{i}" for i in range(n)) + ");")
    lines.append("solve satisfy;")
    return S.parse_model("\n".join(lines))


def test_big_alldiff_removals_and_fixpoints():
    rng = models.Rng(4242)
    for trial in range(40):
        n = 65 + rng.below(60)
        width = n + rng.below(8)
        m = _random_alldiff_model(rng, n, width)
        doms = []
        for v in range(n):
            d = S.Domain(1, width)
            for x in range(1, width + 1):
                if d.size() > 2 and rng.below(3) == 0:
                    d.remove(x)
            doms.append(d)
        for level in (0, 1):
            assert S.removals(m, doms, alldiff=level) == O.removals(m, doms, alldiff=level), (trial, level)
            gd, gf = S.propagate_fixpoint(m, doms, alldiff=level)
            od, of = O.propagate_fixpoint(m, doms, alldiff=level)
            assert gf == of and gd == od, (trial, level)


def test_wide_universe_alldiff():
    rng = models.Rng(99)
    for trial in range(40):
        n = 3 + rng.below(6)
        offs = [rng.range(-3000, 3000) for _ in range(n)]
        # two members share a range so pruning happens; the rest sit far apart
        offs[1] = offs[0]
        m = _random_alldiff_model(rng, n, 3, offs)
        doms = [S.Domain(o, o + 2) for o in offs]
        doms[0].remove(offs[0] + 2)
        doms[1].remove(offs[1] + 2)
        for level in (0, 1):
            assert S.removals(m, doms, alldiff=level) == O.removals(m, doms, alldiff=level), (trial, level)


def test_big_alldiff_search_matches_oracle():
    for n in (66, 70):
        m = S.parse_model(models.gen_nqueens(n))
        cfg = S.SearchConfig(max_solutions=1)
        got, exp = [], []
        r = S.solve_satisfy(m, cfg, lambda s: got.append(s.values) or True)
        ro = O.solve_satisfy(m, cfg, lambda s: exp.append(s.values) or True)
        assert r.stats.as_tuple() == ro.stats.as_tuple() and got == exp, n


@pytest.mark.parametrize("key", ["nq8|--max 1", "nq14|--max 1", "nq24|--max 1", "nq40|--max 1", "magic4|--max 1",
                                 "magic5|--max 1", "rcsp_1000|--max 1"])
def test_parallel_first_solution_exact(key):
    # many contexts, subtrees right of the best known solution abandoned, and still the
    # reference's exact nodes/failures/rounds up to its DFS-first solution
    g = G.goldens()[key]
    stats, sol = gpu_case(key, PARALLEL)
    assert stats == G.expected_tuple(g)
    assert sol == g["first"]


# ---- positive table constraints (extension; BASELINE config 5). Parity vs the oracle port and
# brute force (the reference has no table constraint).
def _brute_force(m, lo_hi):
    tabs = []
    for c in range(m.n_cons):
        k = m.con_start[c + 1] - m.con_start[c]
        vs = m.term_var[m.con_start[c]:m.con_start[c + 1]]
        tu = {tuple(m.table_data[m.table_start[c] + i * k:m.table_start[c] + (i + 1) * k]) for i in range(m.con_value[c])}
        tabs.append((vs, tu))
    return [list(a) for a in itertools.product(*[range(lo, hi + 1) for lo, hi in lo_hi])
            if all(tuple(a[v] for v in vs) in tu for vs, tu in tabs)]


def test_table_removals_binary_and_nary():
    rng = models.Rng(777)
    for trial in range(60):
        n, d = 4, 3 + rng.below(5)
        lines = [f"var v{i} in {i}..{i + d - 1};" for i in range(n)]
        for arity in (2, 3):
            scope = [rng.below(n) for _ in range(arity)]
            tuples = set()
            for _ in range(rng.below(d * d) + 1):
                tuples.add(tuple(scope[j] + rng.below(d + 1) - (1 if rng.below(5) == 0 else 0) for j in range(arity)))
            body = ", ".join(" ".join(str(x) for x in t) for t in sorted(tuples))
            lines.append(f"constraint table({', '.join(f'v{s}' for s in scope)} : {body});")
        lines.append("solve satisfy;")
        m = S.parse_model("\n".join(lines))
        doms = [d_.copy() for d_ in m.domains]
        for v in range(n):
            for x in doms[v].values():
                if doms[v].size() > 1 and rng.below(3) == 0:
                    doms[v].remove(x)
        for c in range(m.n_cons):
            assert S.removals(m, doms, cons=[c]) == O.removals(m, doms, cons=[c]), (trial, c)
        gd, gf = S.propagate_fixpoint(m, doms)
        od, of = O.propagate_fixpoint(m, doms)
        assert gd == od and gf == of, trial


def test_table_all_solutions_vs_brute_force():
    for seed in range(30):
        n, d = 5 + seed % 2, 3 + seed % 2
        text = models.random_binary_csp(n, d, 6 + seed % 4, 0.45, seed)
        m = S.parse_model(text)
        bf = _brute_force(m, [(1, d)] * n)
        exp = [s.values for s in O.enumerate_solutions(m)]
        assert sorted(exp) == sorted(bf), seed
        for eng in (PARITY, PARALLEL):
            st, ost = S.SearchStats(), S.SearchStats()
            got = [s.values for s in S.enumerate_solutions(m, S.SearchConfig(engine=eng), st)]
            O.enumerate_solutions(m, S.SearchConfig(), ost)
            assert got == exp and st.as_tuple() == ost.as_tuple(), (seed, eng)


def test_table_random_csp_search_matches_oracle():
    n = 200
    t = models.phase_transition_tightness(n, 10, 2 * n) - 0.06
    m = S.parse_model(models.random_binary_csp(n, 10, 2 * n, t, 5))
    for cfg in (S.SearchConfig(max_solutions=1, node_limit=1500, engine=PARITY),
                S.SearchConfig(max_solutions=1, node_limit=1500, var_heuristic=0, engine=PARITY)):
        r, ro = S.solve_satisfy(m, cfg), O.solve_satisfy(m, cfg)
        assert r.stats.as_tuple() == ro.stats.as_tuple()


@pytest.mark.parametrize("key", ["nq8|--all", "nq8|--max 1", "nq10|--all --node-limit 1000", "golomb7", "magic3|--all",
                                 "magic5|--max 1", "rcsp_10000|--max 1 --node-limit 200",
                                 "rcsp_100000|--max 1 --node-limit 200"])
def test_grid_context_matches_reference(key):
    # one search context spanning the GPU (cooperative launch, grid barriers between phases)
    g = G.goldens()[key]
    stats, sol = gpu_case(key, A.ENGINE_GRID)
    assert stats == G.expected_tuple(g)
    assert sol == (g.get("best") if "best" in g else g.get("first"))


def test_grid_context_tables_and_corpus():
    for seed in range(0, 200, 7):
        m = S.parse_model(models.corpus_instance(seed))
        st, ost = S.SearchStats(), S.SearchStats()
        got = [s.values for s in S.enumerate_solutions(m, S.SearchConfig(engine=A.ENGINE_GRID), st)]
        exp = [s.values for s in O.enumerate_solutions(m, S.SearchConfig(), ost)]
        assert got == exp and st.as_tuple() == ost.as_tuple(), seed
    n = 200
    t = models.phase_transition_tightness(n, 10, 2 * n) - 0.06
    m = S.parse_model(models.random_binary_csp(n, 10, 2 * n, t, 5))
    cfg = S.SearchConfig(max_solutions=1, node_limit=500, engine=A.ENGINE_GRID)
    assert S.solve_satisfy(m, cfg).stats.as_tuple() == O.solve_satisfy(m, cfg).stats.as_tuple()


@pytest.mark.parametrize("key", ["nq8|--all", "nq10|--all", "nq12|--all", "magic3|--all", "nq8|--all --fc"])
@pytest.mark.parametrize("world", [2, 8])
def test_shared_queue_shards_sum_exactly(key, world):
    # cubics_solve_shard_shared: every rank seeds all frontier subtrees and claims them through
    # one counter; run one after another here, so the first rank claims everything and the rest
    # only count (rank 0) or contribute nothing. Sums and key order are the reference's.
    from paper_1909_09213_b200 import distributed as D

    inst, flags = G.split_key(key)
    m = S.parse_model(G.model_text(inst))
    cfg = G.cfg_from_flags(flags)
    q = S.TaskQueue.create(0)
    try:
        for _ in range(2):  # the queue is reusable after a reset
            q.reset()
            assert q.claims() == 0
            tot = [0, 0, 0, 0]
            streams = []
            for r in range(world):
                keyed = []
                res = S.solve_shard(m, cfg, r, world, lambda k, v, keyed=keyed: keyed.append((tuple(k), v)) or True,
                                    queue=q)
                tot = [a + b for a, b in zip(tot, res.stats.as_tuple())]
                streams.append(keyed)
            assert tuple(tot) == G.expected_tuple(G.goldens()[key])
            assert D.merge_keyed(streams) == [s.values for s in O.enumerate_solutions(m, cfg)]
            if inst == "nq12":  # the smaller trees can close above the split depth (no subtrees)
                assert q.claims() > 0
    finally:
        q.close()


def _shared_queue_worker(rank, world, port, key, out):
    import os

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_1909_09213_b200 import distributed as D

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        inst, flags = G.split_key(key)
        m = S.parse_model(G.model_text(inst))
        cfg = G.cfg_from_flags(flags)
        q = D.shared_task_queue(rank, world, device=0)
        res = []
        for _ in range(2):
            stats, merged, _ = D.solve_distributed(m, cfg, rank, world, queue=q)
            res.append((stats, merged))
        dist.barrier()  # the owner frees the counter only after every mapping is done with it
        q.close()
        dist.barrier()
        out.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_shared_queue_across_processes_ipc():
    # two processes map one claim counter through CUDA IPC (the NVLink peer-memory path on a
    # multi-GPU box; here both sit on cuda:0 and never wait on each other's kernels)
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    key, world = "nq12|--all", 2
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    procs = [ctx.Process(target=_shared_queue_worker, args=(r, world, port, key, out)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(out.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    inst, flags = G.split_key(key)
    m = S.parse_model(G.model_text(inst))
    want = [s.values for s in O.enumerate_solutions(m, G.cfg_from_flags(flags))]
    for rank in range(world):
        for stats, merged in got[rank]:
            assert stats == G.expected_tuple(G.goldens()[key])
            assert (merged == want) if rank == 0 else merged is None
