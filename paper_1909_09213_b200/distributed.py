"""Multi-GPU search, one process per GPU.

Every rank calls cubics_solve_shard(rank, world): the search tree is expanded deterministically
to a frontier of open subtrees, numbered in DFS order, and rank r searches the subtrees
t with t % world == r with the in-GPU parallel engine (dynamic work sharing across its search
contexts). Nodes above the frontier are counted by rank 0 only, so a single all-reduce (sum) of
(nodes, failures, rounds, solutions) gives exactly the reference's stats. Solutions carry their
DFS path key; rank 0 merges the ranks' key-sorted streams into the reference's solution order.
"""
from __future__ import annotations

import heapq

from . import solver as S


def _collect_shard(model, cfg, rank, world, collect):
    sols = []

    def cb(key, values):
        sols.append((tuple(key), values))
        return True

    r = S.solve_shard(model, cfg, rank, world, cb if collect else None)
    return r, sols


def merge_keyed(streams):
    """Merge per-rank lists of (key, values) into one list in key (= DFS) order."""
    return [v for _, v in heapq.merge(*[sorted(s) for s in streams], key=lambda kv: kv[0])]


def solve_distributed(model, cfg: S.SearchConfig, rank: int, world: int, collect: bool = True,
                      shard_fn=None, device=None):
    """Run this rank's shard and combine over the default torch.distributed process group.

    Returns (stats tuple, solutions in DFS order or None on ranks != 0, max device ms over ranks).
    shard_fn(model, cfg, rank, world, collect) -> (SatisfyResult, [(key, values)]) may replace
    the GPU shard (tests use it to exercise the collective plumbing on CPU/gloo).
    """
    import torch
    import torch.distributed as dist

    fn = shard_fn or _collect_shard
    r, sols = fn(model, cfg, rank, world, collect)
    dev = device if device is not None else "cpu"
    t = torch.tensor(list(r.stats.as_tuple()), dtype=torch.int64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    ms = torch.tensor([r.device_ms], dtype=torch.float64, device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    merged = None
    if collect:
        gathered = [None] * world if rank == 0 else None
        dist.gather_object(sols, gathered, dst=0)
        if rank == 0:
            merged = merge_keyed(gathered)
    return tuple(int(x) for x in t.tolist()), merged, float(ms.item())
