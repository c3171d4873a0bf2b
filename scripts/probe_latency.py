"""Dev probe: per-call latency of the C ABI on small inputs (fixpoint and first-solution search)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_09213_b200 import models  # noqa: E402
from paper_1909_09213_b200 import solver as S  # noqa: E402

for name, text in [("nq24", models.gen_nqueens(24)), ("nq8", models.gen_nqueens(8))]:
    m = S.parse_model(text)
    S.propagate_fixpoint(m)
    t = time.perf_counter()
    for _ in range(50):
        S.propagate_fixpoint(m)
    print(f"{name} propagate_fixpoint: {(time.perf_counter() - t) / 50 * 1e3:.3f} ms/call")
    t = time.perf_counter()
    for _ in range(20):
        r = S.solve_satisfy(m, S.SearchConfig(max_solutions=1))
    print(f"{name} first solution: {(time.perf_counter() - t) / 20 * 1e3:.3f} ms/call (device {r.device_ms:.3f} ms)")
