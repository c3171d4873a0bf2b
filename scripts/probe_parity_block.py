"""Reference-order engine: block size sweep on golomb10 (20000-node prefix) and assign9 B&B."""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import golden_cases as G  # noqa: E402
from paper_1909_09213_b200 import _abi as A, models, solver as S  # noqa: E402

for name, m in (("golomb10", S.parse_model(G.model_text("golomb10"))),
                ("assign9", S.parse_model(models.assignment(9, seed=3)))):
    for bt in (0, 64, 96, 128, 192, 256, 512):
        r = S.solve_optimize(m, S.SearchConfig(device=0, engine=A.ENGINE_PARITY, node_limit=20000, block_threads=bt))
        print(json.dumps({"instance": name, "block": bt, "ms": r.device_ms, "stats": r.stats.as_tuple()}), flush=True)
