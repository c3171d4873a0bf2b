"""Per-node latency of the parity engine (one block, reference node order) vs block size, and
of the batched B&B (cubics_solve_optimize_batch) vs problem count: the quantities that bound
exact B&B and LNS on the device."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1909_09213_b200 import _abi as A  # noqa: E402
from paper_1909_09213_b200 import models  # noqa: E402
from paper_1909_09213_b200 import solver as S  # noqa: E402


def main():
    cases = [("assign20", "opt", 60000), ("golomb9", "opt", 0), ("nq10", "all", 0), ("magic4", "first", 0)]
    for name, kind, limit in cases:
        m = S.parse_model(models.named_instance(name))
        for block in (0, 32, 64, 128, 256):
            cfg = S.SearchConfig(engine=A.ENGINE_PARITY, block_threads=block, node_limit=limit)
            best = None
            for _ in range(2):
                if kind == "opt":
                    r = S.solve_optimize(m, cfg)
                else:
                    if kind == "first":
                        cfg.max_solutions = 1
                    r = S.solve_satisfy(m, cfg)
                if best is None or r.device_ms < best[0]:
                    best = (r.device_ms, r.stats.nodes, r.stats.rounds)
            ms, nodes, rounds = best
            print(json.dumps({"case": name, "block": block, "ms": round(ms, 3), "nodes": nodes, "rounds": rounds,
                              "us_per_node": round(1000 * ms / max(1, nodes), 3),
                              "us_per_round": round(1000 * ms / max(1, rounds), 3)}), flush=True)
    # batch: N copies of the same limited search -> throughput vs N
    m = S.parse_model(models.named_instance("assign20"))
    nw = m.word_start[-1]
    base = np.ctypeslib.as_array(m.words_of(m.domains))[:nw].copy()
    for block in (0, 32, 64):
        for count in (1, 148, 592, 2368):
            cfg = S.SearchConfig(engine=A.ENGINE_PARITY, node_limit=2000, block_threads=block)
            rs = S.optimize_batch(m, np.tile(base, (count, 1)), None, cfg)
            rs = S.optimize_batch(m, np.tile(base, (count, 1)), None, cfg)
            nodes = sum(r.stats.nodes for r in rs)
            print(json.dumps({"batch": count, "block": block, "ms": round(rs[0].device_ms, 3), "nodes": nodes,
                              "nodes_per_s": round(nodes / rs[0].device_ms * 1000)}), flush=True)


if __name__ == "__main__":
    main()
