"""Probe: streaming delivery on a few models (CUBICS_DEBUG prints the drain summary)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
os.environ.setdefault("CUBICS_DEBUG", "1")
import golden_cases as G
from paper_1909_09213_b200 import _abi as A, models, solver as S
for inst, n in [("nq40", 1), ("nq24", 1), ("nq40", 3), ("rcsp_10000", 1)]:
    m = S.parse_model(G.model_text(inst))
    for eng in (A.ENGINE_PARITY, A.ENGINE_AUTO):
        got = []
        cfg = S.SearchConfig(engine=eng, max_solutions=n)
        if inst.startswith("rcsp"):
            cfg.node_limit = 200
        r = S.solve_satisfy(m, cfg, lambda s: got.append(s.values) or True)
        print(inst, n, eng, r.engine, r.stats.as_tuple(), len(got), flush=True)
