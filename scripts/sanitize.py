"""Small searches for compute-sanitizer (one tool per run): nq8 on the parity and parallel
engines, a streamed stop, an exact parallel first solution, and a 2-shard shared-queue search."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1909_09213_b200 import _abi as A, models, solver as S  # noqa: E402

m = S.parse_model(models.gen_nqueens(8))
for eng in (A.ENGINE_PARITY, A.ENGINE_PARALLEL):
    st = S.SearchStats()
    S.enumerate_solutions(m, S.SearchConfig(engine=eng, contexts=64), st)
    assert st.as_tuple() == (695, 256, 1485, 92), st
seen = []
S.solve_satisfy(m, S.SearchConfig(contexts=64), lambda s: seen.append(s) or len(seen) < 5)
assert len(seen) == 5
r = S.solve_satisfy(S.parse_model(models.gen_nqueens(12)), S.SearchConfig(max_solutions=1, contexts=64))
assert r.stats.solutions == 1
q = S.TaskQueue.create(0)
q.reset()
tot = [0, 0, 0, 0]
for rank in range(2):
    res = S.solve_shard(m, S.SearchConfig(device=0, contexts=64), rank, 2, queue=q)
    tot = [a + b for a, b in zip(tot, res.stats.as_tuple())]
q.close()
assert tuple(tot) == (695, 256, 1485, 92), tot
g = S.solve_optimize(S.parse_model(models.golomb(6, 36)), S.SearchConfig(contexts=64))
assert g.best.objective == 17
print("sanitize workload ok")
