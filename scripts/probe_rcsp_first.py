"""Exact first solution on the larger random CSPs (BASELINE configs[4]): parallel engine, bounded."""
import json
import os
import sys
import time

os.environ.setdefault("CUBICS_DEBUG", "1")
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import golden_cases as G  # noqa: E402
from paper_1909_09213_b200 import solver as S  # noqa: E402

for inst in sys.argv[1:] or ["rcsp_1000", "rcsp_10000"]:
    m = S.parse_model(G.model_text(inst))
    t0 = time.perf_counter()
    try:
        r = S.solve_satisfy(m, S.SearchConfig(device=0, max_solutions=1, count_only=True))
        print(json.dumps({"instance": inst, "stats": r.stats.as_tuple(), "engine": r.engine, "contexts": r.contexts,
                          "device_ms": r.device_ms, "wall_ms": (time.perf_counter() - t0) * 1e3}), flush=True)
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"instance": inst, "error": repr(e), "wall_ms": (time.perf_counter() - t0) * 1e3}), flush=True)
