"""Dev probe: device time of the engines over contexts/block sizes (run with CUBICS_DEBUG=1).

usage: probe_parallel.py INSTANCE [--parity] [--grid ctx,ctx,...] [--blocks b,b,...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_09213_b200 import _abi as A  # noqa: E402
from paper_1909_09213_b200 import models  # noqa: E402
from paper_1909_09213_b200 import solver as S  # noqa: E402

inst = sys.argv[1] if len(sys.argv) > 1 else "nq12"
args = sys.argv[2:]
grid = [0]
blocks = [0]
if "--grid" in args:
    grid = [int(x) for x in args[args.index("--grid") + 1].split(",")]
if "--blocks" in args:
    blocks = [int(x) for x in args[args.index("--blocks") + 1].split(",")]
m = S.parse_model(models.named_instance(inst))
configs = [(A.ENGINE_PARITY, 0, 0)] if "--parity" in args else []
if "--no-parallel" not in args:
    configs += [(A.ENGINE_PARALLEL, c, b) for c in grid for b in blocks]
for eng, ctx, blk in configs:
    cfg = S.SearchConfig(engine=eng, contexts=ctx, block_threads=blk, count_only=True,
                         max_solutions=1 if "--first" in args else A.UINT64_MAX)
    if m.goal != 0:
        r = S.solve_optimize(m, cfg)
        extra = f" obj={r.best.objective if r.best else None}"
    else:
        r = S.solve_satisfy(m, cfg)
        extra = ""
    print(f"{inst} eng={eng} ctx={ctx} blk={blk} used={r.contexts} ms={r.device_ms:.2f} "
          f"nodes/s={r.stats.nodes / max(r.device_ms, 1e-9) * 1e3:.3e} stats={r.stats.as_tuple()}{extra}", flush=True)
