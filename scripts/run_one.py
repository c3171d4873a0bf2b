"""One search of a named instance (for ncu captures): run_one.py NAME KIND LIMIT [ENGINE]
(ENGINE: parity (default) | parallel | auto)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_09213_b200 import _abi as A  # noqa: E402
from paper_1909_09213_b200 import models  # noqa: E402
from paper_1909_09213_b200 import solver as S  # noqa: E402

name, kind, limit = sys.argv[1], sys.argv[2], int(sys.argv[3])
m = S.parse_model(models.named_instance(name))
eng = {"parity": A.ENGINE_PARITY, "parallel": A.ENGINE_PARALLEL, "auto": A.ENGINE_AUTO}[sys.argv[4] if len(sys.argv) > 4 else "parity"]
cfg = S.SearchConfig(engine=eng, node_limit=limit, count_only=True)
r = S.solve_optimize(m, cfg) if kind == "opt" else S.solve_satisfy(m, cfg)
print(name, r.stats.as_tuple(), round(r.device_ms, 3), "ms")
