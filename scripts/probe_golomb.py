"""Per-node cost of the parity engine on Golomb rulers at growing node limits (B200 probe)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_09213_b200 import _abi as A  # noqa: E402
from paper_1909_09213_b200 import models  # noqa: E402
from paper_1909_09213_b200 import solver as S  # noqa: E402

runs = [("golomb8", 0), ("golomb9", 0), ("golomb10", 2000), ("golomb10", 20000), ("golomb10", 60000)]
if len(sys.argv) > 1:
    runs = [(a.split(":")[0], int(a.split(":")[1])) for a in sys.argv[1:]]
for name, limit in runs:
    m = S.parse_model(models.named_instance(name))
    cfg = S.SearchConfig(engine=A.ENGINE_PARITY, node_limit=limit, count_only=True)
    S.solve_optimize(m, S.SearchConfig(engine=A.ENGINE_PARITY, node_limit=50, count_only=True))
    r = S.solve_optimize(m, cfg)
    st = r.stats.as_tuple()
    print(json.dumps({"instance": name, "node_limit": limit, "stats": st, "device_ms": round(r.device_ms, 3),
                      "us_per_node": round(1e3 * r.device_ms / st[0], 2),
                      "us_per_round": round(1e3 * r.device_ms / st[2], 3), "threads": r.contexts}), flush=True)
