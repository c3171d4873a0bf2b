"""B200 probes: (1) parity-engine per-node cost vs block size on golomb10 (node-limited);
(2) cost of the multi-GPU frontier expansion and of each rank's share (ranks run one after
another on this GPU, static and shared-queue split)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_09213_b200 import _abi as A  # noqa: E402
from paper_1909_09213_b200 import models  # noqa: E402
from paper_1909_09213_b200 import solver as S  # noqa: E402

m = S.parse_model(models.named_instance("golomb10"))
for bt in (0, 96, 128, 256, 512):
    cfg = S.SearchConfig(engine=A.ENGINE_PARITY, node_limit=10000, count_only=True, block_threads=bt)
    S.solve_optimize(m, S.SearchConfig(engine=A.ENGINE_PARITY, node_limit=50, count_only=True, block_threads=bt))
    r = S.solve_optimize(m, cfg)
    print(json.dumps({"probe": "golomb10_parity_block", "block_threads": bt, "stats": r.stats.as_tuple(),
                      "device_ms": round(r.device_ms, 3)}), flush=True)

nq = S.parse_model(models.named_instance("nq14"))
cfg = S.SearchConfig(engine=A.ENGINE_PARALLEL, count_only=True)
S.solve_satisfy(nq, cfg)
r1 = S.solve_satisfy(nq, cfg)
print(json.dumps({"probe": "nq14_1gpu", "device_ms": round(r1.device_ms, 3), "total_ms": round(r1.total_ms, 3)}))
for world in (2, 4, 8):
    for shared in (False, True):
        q = S.TaskQueue.create(0) if shared else None
        if q:
            q.reset()
        per = []
        for rank in range(world):
            r = S.solve_shard(nq, cfg, rank, world, queue=q)
            per.append((round(r.device_ms, 3), round(r.total_ms, 3), r.stats.nodes))
        print(json.dumps({"probe": "nq14_shards_sequential", "world": world, "shared": shared,
                          "per_rank_device_ms_total_ms_nodes": per,
                          "claims": q.claims() if q else None}), flush=True)
        if q:
            q.close()
