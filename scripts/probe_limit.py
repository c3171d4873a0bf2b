"""Dev probe: parity-engine stats and time on INSTANCE with a node limit (compare with the reference)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_09213_b200 import _abi as A  # noqa: E402
from paper_1909_09213_b200 import models  # noqa: E402
from paper_1909_09213_b200 import solver as S  # noqa: E402

inst, limit = sys.argv[1], int(sys.argv[2])
blk = int(sys.argv[3]) if len(sys.argv) > 3 else 0
m = S.parse_model(models.named_instance(inst))
cfg = S.SearchConfig(engine=A.ENGINE_PARITY, node_limit=limit, max_solutions=1, block_threads=blk, count_only=True)
t = time.time()
r = S.solve_satisfy(m, cfg)
print(f"{inst} limit={limit} blk={blk} ms={r.device_ms:.1f} wall={1e3*(time.time()-t):.0f} stats={r.stats.as_tuple()} "
      f"nodes/s={r.stats.nodes / r.device_ms * 1e3:.3e}", flush=True)
