"""nq14 e2e breakdown (cubics_enumerate) with and without an L2 flush before each call."""
import os
import sys
import time

os.environ["CUBICS_DEBUG"] = "1"
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import torch  # noqa: E402

import golden_cases as G  # noqa: E402
from paper_1909_09213_b200 import solver as S  # noqa: E402

m = S.parse_model(G.model_text("nq14"))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")
for flushing in (False, True):
    for i in range(5):
        if flushing:
            flush.zero_()
            torch.cuda.synchronize()
        t0 = time.perf_counter()
        arr, r = S.enumerate_array(m, S.SearchConfig(device=0))
        t1 = time.perf_counter()
        print(f"flush={flushing} e2e {1e3*(t1-t0):.2f} ms  total_ms {r.total_ms:.2f} device {r.device_ms:.2f}", flush=True)
