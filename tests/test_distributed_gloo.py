"""Multi-rank plumbing of the sharded search on CPU: world_size 2, gloo backend.

The GPU shard is replaced by a deterministic fake that splits a known enumeration (the oracle's,
pinned to the reference) by DFS rank, so the test checks exactly what the ranks exchange: the
stats all-reduce and the key-ordered solution merge."""
import os
import socket

import pytest
import torch.multiprocessing as mp

import golden_cases as G


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    import oracle_binding as O
    from paper_1909_09213_b200 import distributed as D
    from paper_1909_09213_b200 import solver as S

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = S.parse_model(G.model_text("nq8"))
        full = O.enumerate_solutions(m)
        st = S.SearchStats()
        O.enumerate_solutions(m, S.SearchConfig(), st)

        def fake_shard(model, cfg, r, w, collect):
            mine = [((i,), s.values) for i, s in enumerate(full) if i % w == r]
            # stats: rank 0 carries the remainder so the sum is exact
            part = [x // w + (x % w if r == 0 else 0) for x in st.as_tuple()]
            res = S.SatisfyResult(S.SearchStats(*part), True, device_ms=float(r + 1))
            return res, list(reversed(mine))

        stats, merged, ms = D.solve_distributed(m, S.SearchConfig(), rank, world, shard_fn=fake_shard)
        q.put((rank, stats, merged, ms))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_allreduce_and_merge():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        rank, stats, merged, ms = q.get(timeout=120)
        out[rank] = (stats, merged, ms)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = G.goldens()["nq8|--all"]
    for rank in range(world):
        assert out[rank][0] == G.expected_tuple(g)
        assert out[rank][2] == 2.0  # max over ranks
    merged = out[0][1]
    assert len(merged) == 92 and merged[0] == g["first"]
    assert out[1][1] is None


def _worker_opt(rank, world, port, q, fail_rank):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    import oracle_binding as O
    from paper_1909_09213_b200 import distributed as D
    from paper_1909_09213_b200 import solver as S

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = S.parse_model(G.model_text("golomb6"))
        opt = O.solve_optimize(m)

        def fake_shard(model, cfg, r, w):
            if r == fail_rank:
                raise S.CapacityError("shard buffer overflow on rank %d" % r)
            # the optimum sits on the last rank; the others hold worse incumbents (or none)
            part = [x // w + (x % w if r == 0 else 0) for x in opt.stats.as_tuple()]
            if r == w - 1:
                best = opt.best
            elif r == 0:
                best = S.Solution(list(opt.best.values), opt.best.objective + 5)
            else:
                best = None
            return S.OptimizeResult(best, True, S.SearchStats(*part), device_ms=float(r))

        try:
            stats, best, ms = D.solve_distributed(m, S.SearchConfig(), rank, world, shard_fn=fake_shard)
            q.put((rank, "ok", stats, (best.objective, best.values) if best else None, ms, opt.stats.as_tuple(),
                   opt.best.objective))
        except Exception as e:  # noqa: BLE001
            q.put((rank, "raised", type(e).__name__, str(e), None, None, None))
    finally:
        dist.destroy_process_group()


def _run_opt(world, fail_rank):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker_opt, args=(r, world, port, q, fail_rank)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        rec = q.get(timeout=120)
        out[rec[0]] = rec[1:]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def test_two_rank_gloo_branch_and_bound_best_over_ranks():
    out = _run_opt(2, fail_rank=-1)
    for rank in range(2):
        status, stats, best, ms, exp_stats, exp_obj = out[rank]
        assert status == "ok"
        assert stats == exp_stats  # partial stats sum exactly
        assert best[0] == exp_obj == 17  # golomb6 optimum, from the rank that holds it
        assert ms == 1.0


def test_failing_rank_raises_on_every_rank_instead_of_hanging():
    out = _run_opt(2, fail_rank=1)
    assert out[1][0] == "raised" and out[1][1] == "CapacityError"
    assert out[0][0] == "raised" and "another rank" in out[0][2]


def _worker_first(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_1909_09213_b200 import distributed as D
    from paper_1909_09213_b200 import solver as S

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = S.parse_model(G.model_text("nq8"))

        class FakePart:  # the two-phase protocol of cubics_solve_first_shard
            def __init__(self, r):
                self.r = r
                self.result = S.SatisfyResult(S.SearchStats(), False, device_ms=float(r + 3))

            def best(self):  # rank 1 holds the DFS-first key [5], rank 0 a later one [9]
                return ([9], [0] * 8) if self.r == 0 else ([5], list(range(8)))

            def prefix(self, key):
                assert key == [5]  # every rank sees the global minimum
                return S.SearchStats(10 * (self.r + 1), self.r, 100, 1 if self.r == 0 else 0)

        stats, sols, ms = D.solve_distributed(m, S.SearchConfig(max_solutions=1), rank, world,
                                              shard_fn=lambda *a: FakePart(a[2]))
        q.put((rank, stats, sols, ms))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_first_solution_min_key_and_prefix_sum():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker_first, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        rank, stats, sols, ms = q.get(timeout=120)
        out[rank] = (stats, sols, ms)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank in range(world):
        stats, sols, ms = out[rank]
        assert stats == (30, 1, 200, 1)
        assert sols == [list(range(8))]
        assert ms == 4.0
