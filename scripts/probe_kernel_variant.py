import sys, json
sys.path.insert(0, '/root/repo')
from paper_1909_09213_b200 import _abi as A, models, solver as S
for name, kind, lim in [("golomb9", "opt", 0), ("nq10", "all", 0), ("assign20", "opt", 20000)]:
    m = S.parse_model(models.named_instance(name))
    for block in (0, 128, 512, 544, 576):
        best = None
        for _ in range(2):
            cfg = S.SearchConfig(engine=A.ENGINE_PARITY, block_threads=block, node_limit=lim)
            r = S.solve_optimize(m, cfg) if kind == "opt" else S.solve_satisfy(m, cfg)
            best = r.device_ms if best is None else min(best, r.device_ms)
        print(json.dumps({"case": name, "block": block, "ms": round(best, 2), "us_per_node": round(1000 * best / r.stats.nodes, 2)}), flush=True)
