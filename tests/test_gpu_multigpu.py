"""Multi-GPU search paths on one B200: the ranks' shard calls run one after another on cuda:0
(or as two processes mapping one queue through CUDA IPC), which exercises every line of the
N-GPU code without ranks that wait on each other's kernels.

* Branch and bound across shards (cubics_solve_optimize_shard): Golomb m=10 must reach the
  reference's optimum 55 and its ruler 0 1 6 10 23 26 34 41 53 55 (the optimal ruler is unique
  once d1_2 < d9_10 breaks the mirror symmetry, so every complete B&B returns the reference's
  solution) for world 2, 3 and 8, static split and shared queue (shared incumbent).
* The same through distributed.solve_distributed in two processes (gloo plumbing, IPC queue).
"""
import socket

import pytest

import golden_cases as G
import oracle_binding as O
from paper_1909_09213_b200 import models
from paper_1909_09213_b200 import solver as S

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def engine_present():
    assert S.device_count() >= 1, "no CUDA device visible to libcubics"


def _best_over(results, minimize=True):
    best = None
    for r in results:
        if r.best is None:
            continue
        if best is None or (r.best.objective < best.objective if minimize else r.best.objective > best.objective):
            best = r.best
    return best


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("shared", [False, True])
@pytest.mark.parametrize("inst", ["golomb8", "golomb10"])
def test_branch_and_bound_across_shards(inst, world, shared):
    g = G.goldens()[inst]
    m = S.parse_model(G.model_text(inst))
    q = S.TaskQueue.create(0) if shared else None
    try:
        if q is not None:
            q.reset()
        res = [S.solve_optimize_shard(m, S.SearchConfig(device=0), r, world, queue=q) for r in range(world)]
    finally:
        if q is not None:
            q.close()
    best = _best_over(res)
    assert best is not None and best.objective == g["objective"]
    assert best.values == g["best"]
    assert all(r.complete for r in res)
    # every rank searched something or found the frontier closed; rank 0 counts the expansion
    assert sum(r.stats.nodes for r in res) > 0


def test_optimize_shard_single_rank_matches_reference_optimum():
    g = G.goldens()["golomb9"]
    m = S.parse_model(G.model_text("golomb9"))
    r = S.solve_optimize_shard(m, S.SearchConfig(device=0), 0, 1)
    assert r.best.objective == g["objective"] and r.best.values == g["best"]


def test_optimize_shard_rejects_satisfy_model():
    m = S.parse_model(G.model_text("nq8"))
    with pytest.raises(S.LogicError):
        S.solve_optimize_shard(m, S.SearchConfig(device=0), 0, 2)


def _bnb_worker(rank, world, port, inst, out):
    import os

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_1909_09213_b200 import distributed as D

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = S.parse_model(G.model_text(inst))
        q = D.shared_task_queue(rank, world, device=0)
        res = []
        for _ in range(2):
            stats, best, _ = D.solve_distributed(m, S.SearchConfig(device=0), rank, world, queue=q)
            res.append((stats, best.objective if best else None, best.values if best else None))
        dist.barrier()
        q.close()
        dist.barrier()
        out.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_distributed_branch_and_bound_two_processes_ipc():
    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    inst, world = "golomb9", 2
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    procs = [ctx.Process(target=_bnb_worker, args=(r, world, port, inst, out)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(out.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    g = G.goldens()[inst]
    for rank in range(world):
        for stats, obj, vals in got[rank]:
            assert obj == g["objective"] and vals == g["best"]
            assert stats[0] > 0


# ---- exact first solution across shards (cubics_solve_first_shard) ---------------------------
FIRST_KEYS = ["nq8|--max 1", "nq14|--max 1", "nq24|--max 1", "magic4|--max 1", "magic5|--max 1",
              "rcsp_1000|--max 1"]


# static split: no state shared between the ranks, so a rank searches its subtrees up to its OWN
# first solution (exact, but unbounded work on sparse models such as rcsp: those use the queue)
FIRST_CASES = [(k, False) for k in FIRST_KEYS if not k.startswith("rcsp")] + [(k, True) for k in FIRST_KEYS]


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("key,shared", FIRST_CASES)
def test_first_solution_across_shards_is_the_reference(key, world, shared):
    # every rank's part run one after another on this GPU; the two-phase merge (min key, summed
    # prefixes) must give the reference's first solution and its exact stats (search.cpp:174-186).
    # With the queue, subtrees are claimed in DFS order and the best key prefix is shared, so
    # every GPU abandons subtrees right of any GPU's solution.
    g = G.goldens()[key]
    inst, flags = G.split_key(key)
    m = S.parse_model(G.model_text(inst))
    cfg = G.cfg_from_flags(flags)
    cfg.device = 0
    q = S.TaskQueue.create(0) if shared else None
    try:
        if q is not None:
            q.reset()
        parts = [S.solve_first_shard(m, cfg, r, world, queue=q) for r in range(world)]
        stats, vals = S.merge_first(parts)
    finally:
        if q is not None:
            q.close()
    assert stats.as_tuple() == G.expected_tuple(g)
    assert vals == g["first"]


def test_first_solution_none_across_shards_counts_the_whole_search():
    # an infeasible model: no rank finds a solution, the shares sum to the complete search
    m = S.parse_model(models.gen_nqueens(3))
    ost = S.SearchStats()
    O.enumerate_solutions(m, S.SearchConfig(), ost)
    for world in (1, 2, 3):
        parts = [S.solve_first_shard(m, S.SearchConfig(max_solutions=1, device=0), r, world) for r in range(world)]
        stats, vals = S.merge_first(parts)
        assert vals is None and stats.as_tuple() == ost.as_tuple()


def _first_worker(rank, world, port, key, out):
    import os

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_1909_09213_b200 import distributed as D

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        inst, flags = G.split_key(key)
        m = S.parse_model(G.model_text(inst))
        cfg = G.cfg_from_flags(flags)
        cfg.device = 0
        q = D.shared_task_queue(rank, world, device=0)
        res = []
        for queue in (q, q):
            stats, sols, _ = D.solve_distributed(m, cfg, rank, world, queue=queue)
            res.append((stats, sols))
        dist.barrier()
        q.close()
        dist.barrier()
        out.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_distributed_first_solution_two_processes_ipc():
    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    key, world = "rcsp_1000|--max 1", 2
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    procs = [ctx.Process(target=_first_worker, args=(r, world, port, key, out)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(out.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    g = G.goldens()[key]
    for rank in range(world):
        for stats, sols in got[rank]:
            assert stats == G.expected_tuple(g)
            assert sols == [g["first"]]


# ---- cross-GPU stealing through the shared queue's global pool -------------------------------
def _steal_worker(rank, world, port, out):
    import os

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    from paper_1909_09213_b200 import distributed as D

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = S.parse_model(G.model_text("nq14"))
        q = D.shared_task_queue(rank, world, device=0)
        res = []
        for _ in range(4):
            if rank == 0:
                q.reset()
            dist.barrier()
            # few contexts per process, so both kernels are resident on this one GPU at once; the
            # process with many contexts runs out of work first and steals right branches from the
            # one with few
            ctxs = 256 if rank == 0 else 16
            r = S.solve_shard(m, S.SearchConfig(device=0, contexts=ctxs, count_only=True), rank, world, queue=q)
            t = torch.tensor(list(r.stats.as_tuple()) + [r.remote_in, r.remote_out], dtype=torch.int64)
            dist.all_reduce(t)
            res.append(t.tolist())
        dist.barrier()
        q.close()
        dist.barrier()
        out.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_cross_gpu_stealing_two_processes_ipc():
    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    world = 2
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    procs = [ctx.Process(target=_steal_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(out.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    g = G.goldens()["nq14|--all"]
    moved = 0
    for row in got[0]:
        assert tuple(row[:4]) == G.expected_tuple(g)  # every subtree searched exactly once
        assert row[4] == row[5]  # every subtree given to the pool was taken
        moved += row[4]
    print("subtrees moved between the two processes:", [row[4] for row in got[0]])
    assert moved > 0


# ---- one host process driving several devices (cubics_solve_multi; the C++ host's path) --------
@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0]])
def test_solve_multi_single_process(devices):
    m = S.parse_model(G.model_text("nq12"))
    got = []
    r = S.solve_multi(m, devices, S.SearchConfig(), lambda s: got.append(s.values) or True)
    ost = S.SearchStats()
    want = [s.values for s in O.enumerate_solutions(m, S.SearchConfig(), ost)]
    assert r.stats.as_tuple() == ost.as_tuple() and got == want
    g = G.goldens()["golomb8"]
    r = S.solve_multi(S.parse_model(G.model_text("golomb8")), devices)
    assert r.best.objective == g["objective"] and r.best.values == g["best"]
    for key in ("rcsp_1000|--max 1", "magic4|--max 1"):
        inst, flags = G.split_key(key)
        firsts = []
        r = S.solve_multi(S.parse_model(G.model_text(inst)), devices, G.cfg_from_flags(flags),
                          lambda s: firsts.append(s.values) or True)
        assert r.stats.as_tuple() == G.expected_tuple(G.goldens()[key]) and firsts == [G.goldens()[key]["first"]]


def test_fdsolve_multi_gpu_env_matches_reference_cli():
    # the unmodified reference CLI over the adapter with CUBICS_DEVICES naming two GPUs (here the
    # same one twice): identical output for enumerations, first solutions and optimization
    import os
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    ref, b200 = os.path.join(root, "oracle", "_ref", "fdsolve"), os.path.join(root, "adapter", "_build", "fdsolve_b200")
    mdir = os.path.join(root, "tests", "golden", "models")
    norm = __import__("re").compile(r'time_ms[=":]+\d+')
    for args in (["solve", f"{mdir}/nq8.fd", "--all", "--stats"], ["solve", f"{mdir}/nq10.fd", "--all", "--json"],
                 ["solve", f"{mdir}/golomb7.fd", "--stats"], ["solve", f"{mdir}/magic4.fd", "--stats"]):
        a = subprocess.run([b200] + args, capture_output=True, text=True, timeout=300,
                           env={**os.environ, "CUBICS_DEVICES": "0,0"})
        b = subprocess.run([ref] + args, capture_output=True, text=True, timeout=300)
        assert (a.returncode, norm.sub("T", a.stdout)) == (b.returncode, norm.sub("T", b.stdout)), args


def test_solve_multi_edge_cases():
    # an infeasible model: no first solution, the complete search's stats
    m = S.parse_model(models.gen_nqueens(3))
    ost = S.SearchStats()
    O.enumerate_solutions(m, S.SearchConfig(), ost)
    r = S.solve_multi(m, [0, 0], S.SearchConfig(max_solutions=1))
    assert r.stats.as_tuple() == ost.as_tuple() and r.complete
    # count only: no callback, exact counts
    m = S.parse_model(G.model_text("nq10"))
    seen = []
    r = S.solve_multi(m, [0, 0], S.SearchConfig(count_only=True), lambda s: seen.append(s) or True)
    assert r.stats.as_tuple() == G.expected_tuple(G.goldens()["nq10|--all"]) and seen == []
    # node limits are not sharded: a clear error
    with pytest.raises(S.UnsupportedInstance):
        S.solve_multi(m, [0, 0], S.SearchConfig(node_limit=100))
