"""Exact B&B on golomb10: per-run wall vs device time (CUBICS_DEBUG)."""
import os
import sys
import time

os.environ["CUBICS_DEBUG"] = "1"
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import golden_cases as G  # noqa: E402
from paper_1909_09213_b200 import solver as S  # noqa: E402

m = S.parse_model(G.model_text("golomb10"))
for i in range(3):
    t0 = time.perf_counter()
    r = S.solve_optimize(m, S.SearchConfig(device=0))
    print(f"=== total wall {1e3*(time.perf_counter()-t0):.1f} ms device {r.device_ms:.1f} ms", flush=True)
