"""Grid-wide context (rcsp_100000, 200 nodes; rbcsp_100000 tables): block size sweep."""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import golden_cases as G  # noqa: E402
from paper_1909_09213_b200 import models, solver as S  # noqa: E402

for inst in ("rcsp_100000", "rbcsp_100000"):
    text = G.model_text(inst) if inst.startswith("rcsp") else models.named_instance(inst)
    m = S.parse_model(text)
    for bt in (0, 256, 512, 1024):
        ts = []
        for _ in range(3):
            r = S.solve_satisfy(m, S.SearchConfig(device=0, max_solutions=1, node_limit=200, count_only=True,
                                                  block_threads=bt))
            ts.append(r.device_ms)
        print(json.dumps({"instance": inst, "block": bt, "engine": r.engine, "ms": sorted(ts)[1],
                          "stats": r.stats.as_tuple()}), flush=True)
