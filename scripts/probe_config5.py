"""Dev probe: BASELINE config 5 sweep (random binary CSP with tables near the phase transition)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_09213_b200 import _abi as A  # noqa: E402
from paper_1909_09213_b200 import models  # noqa: E402
from paper_1909_09213_b200 import solver as S  # noqa: E402

LIM = {1000: 2000, 10000: 200, 100000: 200}
for n in (1000, 10000, 100000):
    t0 = time.time()
    m = S.parse_model(models.named_instance(f"rbcsp_{n}"))
    tp = time.time() - t0
    for eng, kw in ((A.ENGINE_PARITY, dict(node_limit=LIM[n])),):
        cfg = S.SearchConfig(engine=eng, max_solutions=1, count_only=True, **kw)
        t = time.time()
        r = S.solve_satisfy(m, cfg)
        print(f"rbcsp_{n} parse={tp:.1f}s eng={eng} {kw} ms={r.device_ms:.1f} wall={time.time() - t:.2f}s "
              f"stats={r.stats.as_tuple()} complete={r.complete} nodes/s={r.stats.nodes / r.device_ms * 1e3:.3e}",
              flush=True)
