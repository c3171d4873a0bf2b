"""One LNS run on assign20 (148 neighbourhoods per iteration, no node limit): the batched
reference-order kernel for ncu."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1909_09213_b200 import models, solver as S  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 2
m = S.parse_model(models.named_instance("assign20"))
t0 = time.perf_counter()
r = S.lns_optimize(m, S.LnsConfig(destroy_rate=0.4, iterations=iters, neighborhoods=148, seed=1))
print(json.dumps({"wall_ms": (time.perf_counter() - t0) * 1e3, "device_ms": r.device_ms, "nodes": r.stats.nodes,
                  "objective": r.best.objective if r.best else None}))
