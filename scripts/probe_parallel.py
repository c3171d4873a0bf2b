"""Dev probe: wall/device time of the engines over contexts/block sizes (run with CUBICS_DEBUG=1)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_09213_b200 import _abi as A  # noqa: E402
from paper_1909_09213_b200 import models  # noqa: E402
from paper_1909_09213_b200 import solver as S  # noqa: E402

inst = sys.argv[1] if len(sys.argv) > 1 else "nq12"
m = S.parse_model(models.named_instance(inst))
configs = [(A.ENGINE_PARITY, 0, 0)] if "--parity" in sys.argv else []
for ctx in (148, 592, 1184, 2368, 4736):
    for blk in (32, 64, 128):
        configs.append((A.ENGINE_PARALLEL, ctx, blk))
for eng, ctx, blk in configs:
    cfg = S.SearchConfig(engine=eng, contexts=ctx, block_threads=blk, count_only=True)
    if m.goal != 0:
        r = S.solve_optimize(m, cfg)
    else:
        r = S.solve_satisfy(m, cfg)
    print(f"{inst} eng={eng} ctx={ctx} blk={blk} used={r.contexts} ms={r.device_ms:.1f} "
          f"nodes/s={r.stats.nodes / r.device_ms * 1e3:.3e} stats={r.stats.as_tuple()}", flush=True)
