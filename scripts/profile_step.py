"""One search of a bench workload, for `ncu --metrics ...` step counts (instructions, shared-memory
wavefronts, DRAM bytes summed over the step's launches).
usage: python scripts/profile_step.py INSTANCE"""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import golden_cases as G  # noqa: E402
from paper_1909_09213_b200 import solver as S  # noqa: E402

inst = sys.argv[1]
m = S.parse_model(G.model_text(inst))
if m.goal != 0:
    r = S.solve_optimize(m, S.SearchConfig(device=0))
else:
    r = S.solve_satisfy(m, S.SearchConfig(device=0, count_only=True,
                                          max_solutions=1 if inst.startswith("rcsp") else (1 << 64) - 1))
print(json.dumps({"instance": inst, "stats": r.stats.as_tuple(), "device_ms": r.device_ms,
                  "launches": r.kernel_launches}))
