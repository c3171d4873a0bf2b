"""One golden case through the C ABI (for ncu captures): run_case.py KEY ENGINE [REPS]
KEY as in tests/golden/goldens.json (e.g. 'nq14|--all'); ENGINE parity|parallel|auto."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import golden_cases as G  # noqa: E402
from paper_1909_09213_b200 import _abi as A  # noqa: E402
from paper_1909_09213_b200 import solver as S  # noqa: E402

key, eng = sys.argv[1], sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
inst, flags = G.split_key(key)
m = S.parse_model(G.model_text(inst))
cfg = G.cfg_from_flags(flags)
cfg.engine = {"parity": A.ENGINE_PARITY, "parallel": A.ENGINE_PARALLEL, "auto": A.ENGINE_AUTO}[eng]
cfg.device = 0
for _ in range(reps):
    if m.goal != 0:
        r = S.solve_optimize(m, cfg)
    else:
        r = S.solve_satisfy(m, cfg, lambda s: True)
g = G.goldens().get(key)
print(key, eng, r.stats.as_tuple(), "ok" if g and r.stats.as_tuple() == G.expected_tuple(g) else "MISMATCH",
      round(r.device_ms, 3), "ms")
