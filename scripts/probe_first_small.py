"""Exact first solution on small models: warp contexts (default) vs wider block contexts."""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import golden_cases as G  # noqa: E402
from paper_1909_09213_b200 import solver as S  # noqa: E402

for inst in ("magic5", "nq24", "magic4"):
    m = S.parse_model(G.model_text(inst))
    for bt in (0, 32, 64, 128, 256):
        ts = []
        for _ in range(3):
            r = S.solve_satisfy(m, S.SearchConfig(device=0, max_solutions=1, count_only=True, block_threads=bt))
            ts.append(r.device_ms)
        print(json.dumps({"instance": inst, "block": bt, "contexts": r.contexts, "ms": sorted(ts)[1],
                          "stats": r.stats.as_tuple()}), flush=True)
