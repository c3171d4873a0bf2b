"""Dev probe: large models (config 5 random binary CSP with tables; rcsp) - grid context vs one block."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_09213_b200 import _abi as A  # noqa: E402
from paper_1909_09213_b200 import models  # noqa: E402
from paper_1909_09213_b200 import solver as S  # noqa: E402

LIM = {"rbcsp_1000": 2000, "rbcsp_10000": 200, "rbcsp_100000": 200, "rcsp_10000": 200, "rcsp_100000": 200}
names = sys.argv[1:] or list(LIM)
for name in names:
    m = S.parse_model(models.named_instance(name))
    for eng in (A.ENGINE_PARITY, A.ENGINE_GRID):
        cfg = S.SearchConfig(engine=eng, max_solutions=1, count_only=True, node_limit=LIM[name])
        t = time.time()
        r = S.solve_satisfy(m, cfg)
        print(f"{name} eng={eng} ms={r.device_ms:.1f} wall={time.time() - t:.2f}s stats={r.stats.as_tuple()} "
              f"nodes/s={r.stats.nodes / r.device_ms * 1e3:.3e} rounds/s={r.stats.rounds / r.device_ms * 1e3:.3e}",
              flush=True)
