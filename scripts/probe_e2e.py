import sys, time
sys.path.insert(0, '/root/repo')
from paper_1909_09213_b200 import _abi as A, models, solver as S
m = S.parse_model(models.named_instance("nq14"))
cfg = S.SearchConfig(engine=A.ENGINE_PARALLEL)
for i in range(5):
    t = time.perf_counter()
    arr, r = S.enumerate_array(m, cfg)
    print("e2e ms", round((time.perf_counter() - t) * 1e3, 3), "device", round(r.device_ms, 3), arr.shape, flush=True)
    del arr
