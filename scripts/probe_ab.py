"""A/B timing of the parallel engine between two trees: probe_ab.py ROOT (imports ROOT's package)."""
import json
import os
import sys

root = os.path.abspath(sys.argv[1])
sys.path.insert(0, root)
from paper_1909_09213_b200 import _abi as A  # noqa: E402
from paper_1909_09213_b200 import models  # noqa: E402
from paper_1909_09213_b200 import solver as S  # noqa: E402

for name in ("nq14", "magic4", "golomb10"):
    m = S.parse_model(models.named_instance(name))
    ts = []
    for _ in range(5):
        cfg = S.SearchConfig(engine=A.ENGINE_PARALLEL, count_only=True)
        r = S.solve_optimize(m, cfg) if m.goal else S.solve_satisfy(m, cfg)
        ts.append(r.device_ms)
    print(json.dumps({"root": os.path.basename(root), "case": name, "ms": sorted(round(t, 2) for t in ts),
                      "nodes": r.stats.nodes}), flush=True)
