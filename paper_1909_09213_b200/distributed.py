"""Multi-GPU search, one process per GPU.

Every rank calls cubics_solve_shard(rank, world): the search tree is expanded deterministically
to a frontier of open subtrees, numbered in DFS order, and rank r searches the subtrees
t with t % world == r with the in-GPU parallel engine (dynamic work sharing across its search
contexts). Nodes above the frontier are counted by rank 0 only, so a single all-reduce (sum) of
(nodes, failures, rounds, solutions) gives exactly the reference's stats. Solutions carry their
DFS path key; rank 0 merges the ranks' key-sorted streams into the reference's solution order.

With a shared TaskQueue (shared_task_queue) the split is dynamic instead: every rank seeds all
frontier subtrees and claims them one at a time through one counter in rank 0's HBM, mapped into
the other ranks with CUDA IPC and incremented with system-scope atomics over NVLink; the stats
still sum exactly because each subtree is claimed exactly once.
"""
from __future__ import annotations

import heapq

from . import solver as S


def _collect_shard(model, cfg, rank, world, collect, queue=None):
    sols = []

    def cb(key, values):
        sols.append((tuple(key), values))
        return True

    r = S.solve_shard(model, cfg, rank, world, cb if collect else None, queue=queue)
    return r, sols


def shared_task_queue(rank: int, world: int, device: int = -1):
    """Collective: rank 0 creates the shared subtree queue on its GPU and broadcasts the IPC
    handle over the default process group; every other rank maps it. Returns a TaskQueue."""
    import torch.distributed as dist

    q = S.TaskQueue.create(device) if rank == 0 else None
    if world == 1:
        return q
    box = [q.handle if q is not None else None]
    dist.broadcast_object_list(box, src=0)
    err = None
    if rank != 0:
        try:
            q = S.TaskQueue.open(box[0], device)
        except (S.EngineUnavailable, ValueError) as e:  # e.g. no peer access between these GPUs
            err = f"rank {rank}: {e}"
    errs = [None] * world
    dist.all_gather_object(errs, err)
    bad = [e for e in errs if e]
    if bad:  # every rank must agree, or subtrees would be searched twice
        if q is not None:
            q.close()
        raise S.EngineUnavailable("shared task queue unavailable: " + "; ".join(bad))
    return q


def merge_keyed(streams):
    """Merge per-rank lists of (key, values) into one list in key (= DFS) order."""
    return [v for _, v in heapq.merge(*[sorted(s) for s in streams], key=lambda kv: kv[0])]


def _optimize_shard(model, cfg, rank, world, queue=None):
    return S.solve_optimize_shard(model, cfg, rank, world, queue=queue)


def _first_distributed(model, cfg, rank, world, shard_fn=None, device=None, queue=None):
    """Exact first solution across ranks (cubics_solve_first_shard): one all-gather of the ranks'
    DFS-first keys picks K* (the minimum), one all-reduce sums each rank's share of the
    reference's prefix up to K* (nodes above the frontier, whole subtrees left of K*, and the
    snapshot of K*'s own subtree segment)."""
    import torch
    import torch.distributed as dist

    part, err = None, None
    if queue is not None:
        try:
            if rank == 0:
                queue.reset()
        except Exception as e:  # noqa: BLE001 - re-raised after the collectives
            err = e
        dist.barrier()
    if err is None:
        try:
            part = shard_fn(model, cfg, rank, world) if shard_fn else S.solve_first_shard(model, cfg, rank, world, queue)
        except Exception as e:  # noqa: BLE001 - re-raised after the collectives
            err = e
    mine = None
    if part is not None:
        try:
            mine = part.best()
        except Exception as e:  # noqa: BLE001
            err = e
    allb = [None] * world
    dist.all_gather_object(allb, (err is not None, mine))
    if any(f for f, _ in allb):
        if err is not None:
            raise err
        raise RuntimeError("solve_distributed: another rank's shard failed")
    cands = [b for _, b in allb if b is not None]
    key, vals = min(cands, key=lambda b: b[0]) if cands else (None, None)
    dev = device if device is not None else "cpu"
    stats, flag = [0, 0, 0, 0], 0
    try:
        stats = list(part.prefix(key).as_tuple())
    except Exception as e:  # noqa: BLE001
        err, flag = e, 1
    t = torch.tensor(stats + [flag], dtype=torch.int64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    ms = torch.tensor([part.result.device_ms], dtype=torch.float64, device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    if int(t[4].item()):
        if err is not None:
            raise err
        raise RuntimeError("solve_distributed: another rank's prefix failed")
    total = tuple(int(x) for x in t[:4].tolist())
    return total, ([vals] if vals is not None else []), float(ms.item())


def solve_distributed(model, cfg: S.SearchConfig, rank: int, world: int, collect: bool = True,
                      shard_fn=None, device=None, queue=None):
    """Run this rank's shard and combine over the default torch.distributed process group.

    Satisfy goals: returns (stats tuple, solutions in DFS order or None on ranks != 0, max device
    ms over ranks). max_solutions == 1: the exact first solution (cubics_solve_first_shard; the
    stats are the reference's prefix up to it, and the list holds that one solution on every rank). Minimize / maximize goals (branch and bound, cubics_solve_optimize_shard):
    returns (stats tuple, best Solution over all ranks or None, max device ms); with a queue the
    GPUs share the incumbent while they search.
    shard_fn(model, cfg, rank, world, collect) -> (SatisfyResult, [(key, values)]) (satisfy) or
    shard_fn(model, cfg, rank, world) -> OptimizeResult (optimize) may replace the GPU shard (tests
    use it to exercise the collective plumbing on CPU/gloo).
    queue (from shared_task_queue) switches to dynamic subtree claiming; it is reset here.
    A rank whose shard raises still joins every collective: the error flag travels with the stats
    all-reduce and every rank raises, instead of the others blocking forever.
    """
    import torch
    import torch.distributed as dist

    optimize = model.goal != 0
    if not optimize and cfg.max_solutions == 1:
        return _first_distributed(model, cfg, rank, world, shard_fn, device, queue)
    r, sols, err = None, [], None
    if queue is not None:
        try:
            if rank == 0:
                queue.reset()
        except Exception as e:  # noqa: BLE001 - re-raised after the collectives
            err = e
        dist.barrier()
    if err is None:
        try:
            if optimize:
                r = shard_fn(model, cfg, rank, world) if shard_fn else _optimize_shard(model, cfg, rank, world, queue)
            elif queue is not None:
                r, sols = _collect_shard(model, cfg, rank, world, collect, queue=queue)
            else:
                r, sols = (shard_fn or _collect_shard)(model, cfg, rank, world, collect)
        except Exception as e:  # noqa: BLE001 - re-raised after the collectives
            err = e
    dev = device if device is not None else "cpu"
    stats = list(r.stats.as_tuple()) if r is not None else [0, 0, 0, 0]
    t = torch.tensor(stats + [1 if err is not None else 0], dtype=torch.int64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    ms = torch.tensor([r.device_ms if r is not None else 0.0], dtype=torch.float64, device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    if int(t[4].item()):
        if err is not None:
            raise err
        raise RuntimeError("solve_distributed: another rank's shard failed")
    total = tuple(int(x) for x in t[:4].tolist())
    if optimize:
        mine = (r.best.objective, r.best.values) if r is not None and r.best is not None else None
        allb = [None] * world
        dist.all_gather_object(allb, mine)
        best = None
        for cand in allb:  # best objective; ties to the lowest rank (deterministic)
            if cand is None:
                continue
            if best is None or (cand[0] < best[0] if model.goal == 1 else cand[0] > best[0]):
                best = cand
        return total, (S.Solution(best[1], best[0]) if best else None), float(ms.item())
    merged = None
    if collect:
        gathered = [None] * world if rank == 0 else None
        dist.gather_object(sols, gathered, dst=0)
        if rank == 0:
            merged = merge_keyed(gathered)
    return total, merged, float(ms.item())
