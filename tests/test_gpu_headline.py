"""The headline workloads at full size, asserted in the driver-run GPU suite.

Expectations are the unmodified reference's own outputs (tests/golden/goldens.json and
tests/golden/stream_hashes.json, made by tests/golden/make_goldens.py and
make_stream_hashes.py from oracle/_ref/fdref_driver):

* nq14 all solutions (BASELINE configs[1]) on the PARALLEL engine: the exact stats tuple
  (4,864,749 / 2,066,779 / 11,003,828 / 365,596), the first solution, and the sha256 of the
  whole 365,596 x 14 int64 solution stream that cubics_enumerate returns, which must equal the
  reference's callback stream byte for byte (search.cpp:134-156, DFS order).
* Golomb m=10 branch-and-bound on the PARITY engine: 198,279 / 99,133 / 1,223,000 / 7 and the
  reference's optimal ruler (search.cpp:87-101, 143-146).
* magic4 all, rcsp_1000 first (PARALLEL exact-first and PARITY), nq10/nq12/magic3/magic4 streams.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import golden_cases as G
from paper_1909_09213_b200 import _abi as A
from paper_1909_09213_b200 import solver as S

pytestmark = pytest.mark.gpu

HASHES = os.path.join(G.GOLDEN, "stream_hashes.json")


def stream_golden(key):
    with open(HASHES) as f:
        return json.load(f)[key]


@pytest.fixture(scope="module", autouse=True)
def engine_present():
    assert S.device_count() >= 1, "no CUDA device visible to libcubics"


def check_stream(key, engine):
    inst, flags = G.split_key(key)
    g = G.goldens()[key]
    h = stream_golden(key)
    m = S.parse_model(G.model_text(inst))
    cfg = G.cfg_from_flags(flags)
    cfg.engine = engine
    arr, r = S.enumerate_array(m, cfg)
    assert r.stats.as_tuple() == G.expected_tuple(g)
    assert arr.dtype == np.int64 and arr.shape == (h["rows"], h["n_vars"])
    assert arr[0].tolist() == g["first"]
    assert hashlib.sha256(np.ascontiguousarray(arr).astype("<i8").tobytes()).hexdigest() == h["sha256"]
    return r


def test_nq14_all_parallel_headline():
    r = check_stream("nq14|--all", A.ENGINE_PARALLEL)
    assert r.stats.as_tuple() == (4864749, 2066779, 11003828, 365596)
    assert r.engine == A.ENGINE_PARALLEL


def test_nq14_all_auto_engine_count_only():
    m = S.parse_model(G.model_text("nq14"))
    r = S.solve_satisfy(m, S.SearchConfig(count_only=True))
    assert r.stats.as_tuple() == (4864749, 2066779, 11003828, 365596)
    assert r.complete


@pytest.mark.parametrize("key", ["nq8|--all", "nq10|--all", "nq12|--all", "magic3|--all", "magic4|--all"])
def test_complete_streams_match_reference_hash(key):
    check_stream(key, A.ENGINE_PARALLEL)


@pytest.mark.parametrize("key", ["nq8|--all", "nq10|--all", "magic3|--all"])
def test_parity_engine_streams_match_reference_hash(key):
    check_stream(key, A.ENGINE_PARITY)


def test_golomb10_parity_exact():
    g = G.goldens()["golomb10"]
    m = S.parse_model(G.model_text("golomb10"))
    r = S.solve_optimize(m, S.SearchConfig(engine=A.ENGINE_PARITY))
    assert r.stats.as_tuple() == (198279, 99133, 1223000, 7) == G.expected_tuple(g)
    assert r.best.objective == 55
    marks = r.best.values[:10]
    assert marks == [0, 1, 6, 10, 23, 26, 34, 41, 53, 55]
    assert r.best.values == g["best"]
    assert r.complete


def test_golomb10_parallel_optimum():
    m = S.parse_model(G.model_text("golomb10"))
    r = S.solve_optimize(m, S.SearchConfig(engine=A.ENGINE_PARALLEL))
    assert r.best.objective == 55 and r.complete


def test_magic4_all_parallel_stats():
    g = G.goldens()["magic4|--all"]
    m = S.parse_model(G.model_text("magic4"))
    r = S.solve_satisfy(m, S.SearchConfig(engine=A.ENGINE_PARALLEL, count_only=True))
    assert r.stats.as_tuple() == G.expected_tuple(g) == (504819, 245370, 1786720, 7040)


@pytest.mark.parametrize("engine", [A.ENGINE_PARALLEL, A.ENGINE_PARITY])
def test_rcsp1000_first_exact(engine):
    g = G.goldens()["rcsp_1000|--max 1"]
    m = S.parse_model(G.model_text("rcsp_1000"))
    first = []
    r = S.solve_satisfy(m, S.SearchConfig(engine=engine, max_solutions=1), lambda s: first.append(s.values) or True)
    assert r.stats.as_tuple() == G.expected_tuple(g) == (114354, 57003, 777656, 1)
    assert first == [g["first"]]
