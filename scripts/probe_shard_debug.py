"""CUBICS_DEBUG lines of the lean search vs the shard search (world 1, shared queue) on nq14."""
import os
import sys

os.environ["CUBICS_DEBUG"] = "1"
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import golden_cases as G  # noqa: E402
from paper_1909_09213_b200 import solver as S  # noqa: E402

m = S.parse_model(G.model_text(sys.argv[1] if len(sys.argv) > 1 else "nq14"))
cfg = S.SearchConfig(device=0, count_only=True)
q = S.TaskQueue.create(0)
for i in range(3):
    print("--- lean", flush=True)
    S.solve_satisfy(m, cfg)
    print("--- shard", flush=True)
    q.reset()
    S.solve_shard(m, cfg, 0, 1, queue=q)
q.close()
