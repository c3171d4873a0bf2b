"""magic5 all solutions (BASELINE configs[3]): throughput on a uniform sample of the search.

The frontier is split into W static shards (subtree t goes to shard t % W, in DFS order); running
shards 0..k-1 searches about k/W of the tree. nodes/s on the sample is the engine's throughput on
this workload, and W/k x (time, nodes, solutions) estimates the complete enumeration (the
solution count is known: 8 x 275,305,224 = 2,202,441,792 with the reference's model)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import golden_cases as G  # noqa: E402
from paper_1909_09213_b200 import solver as S  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 512
K = int(sys.argv[2]) if len(sys.argv) > 2 else 4
STRIDE = int(sys.argv[3]) if len(sys.argv) > 3 else 1  # shards 0, STRIDE, 2*STRIDE, ...
m = S.parse_model(G.model_text("magic5"))
tot = [0, 0, 0, 0]
ms = 0.0
for r in range(0, K * STRIDE, STRIDE):
    t0 = time.perf_counter()
    res = S.solve_shard(m, S.SearchConfig(device=0, count_only=True), r, W)
    wall = (time.perf_counter() - t0) * 1e3
    tot = [a + b for a, b in zip(tot, res.stats.as_tuple())]
    ms += res.device_ms
    print(json.dumps({"shard": r, "of": W, "stats": res.stats.as_tuple(), "device_ms": res.device_ms,
                      "wall_ms": wall}), flush=True)
est = W / K
print(json.dumps({"sample": f"{K}/{W} shards", "stats": tot, "device_ms": ms, "nodes_per_s": tot[0] / (ms / 1e3),
                  "est_full": {"nodes": tot[0] * est, "solutions": tot[3] * est, "device_s": ms * est / 1e3},
                  "known_solutions": 2202441792}), flush=True)
