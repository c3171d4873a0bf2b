"""Exact B&B launch geometry sweep: threads per context x contexts, median of 5 searches each.
usage: python scripts/probe_bnb_geometry.py [INSTANCE]"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import golden_cases as G  # noqa: E402
from paper_1909_09213_b200 import solver as S  # noqa: E402

inst = sys.argv[1] if len(sys.argv) > 1 else "golomb10"
m = S.parse_model(G.model_text(inst))
want = S.solve_optimize(m, S.SearchConfig(device=0)).stats.as_tuple()
for bt in (0, 64, 96, 128, 192, 256):
    for ctx in (0, 592, 1184, 2368):
        ts, ok = [], True
        for _ in range(5):
            r = S.solve_optimize(m, S.SearchConfig(device=0, block_threads=bt, contexts=ctx))
            ok &= r.stats.as_tuple() == want
            ts.append(r.device_ms)
        print(json.dumps({"block_threads": bt, "contexts": ctx, "ms": round(statistics.median(ts), 2),
                          "min": round(min(ts), 2), "stats_ok": ok}), flush=True)
