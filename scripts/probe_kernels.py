"""nq14 all: device time of the lean single-GPU kernel (solve_satisfy) vs the shard kernel
(solve_shard, world 1 with a queue: claims, stealing and B&B sharing compiled in), and the
cubics_enumerate end-to-end time."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import golden_cases as G  # noqa: E402
from paper_1909_09213_b200 import solver as S  # noqa: E402

inst = sys.argv[1] if len(sys.argv) > 1 else "nq14"
m = S.parse_model(G.model_text(inst))
cfg = S.SearchConfig(device=0, count_only=True)
q = S.TaskQueue.create(0)
for name, fn in [("lean solve_satisfy", lambda: S.solve_satisfy(m, cfg)),
                 ("shard world=1 + queue", lambda: (q.reset(), S.solve_shard(m, cfg, 0, 1, queue=q))[1]),
                 ("shard world=2 rank0 + queue", lambda: (q.reset(), S.solve_shard(m, cfg, 0, 2, queue=q))[1]),
                 ("shard world=1 static", lambda: S.solve_shard(m, cfg, 0, 2))]:
    ts = []
    for i in range(6):
        r = fn()
        ts.append(r.device_ms)
    print(f"{name:32s} device ms {min(ts[2:]):.2f} .. {max(ts[2:]):.2f}  nodes {r.stats.nodes}", flush=True)
for i in range(6):
    t0 = time.perf_counter()
    arr, r = S.enumerate_array(m, S.SearchConfig(device=0))
    dt = (time.perf_counter() - t0) * 1e3
    print(f"enumerate e2e {dt:.2f} ms (device {r.device_ms:.2f}, total_ms {r.total_ms:.2f})", flush=True)
q.close()
