"""ctypes binding of the test-only CPU oracle (oracle/liboracle.so, oracle/cubics_oracle.c).

Exposes the same contracts as the product entry points so parity tests can call both on the
same model. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

from paper_1909_09213_b200 import _abi as A
from paper_1909_09213_b200 import solver as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
_OL = None


def oracle_lib():
    global _OL
    if _OL is None:
        if not os.path.exists(ORACLE_SO):
            subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "liboracle.so"], check=True,
                           capture_output=True)
        lib = C.CDLL(ORACLE_SO)
        P = C.POINTER
        lib.oracle_solve_satisfy.argtypes = [P(A.ModelDesc), P(A.SearchConfig), A.SOLUTION_CB, C.c_void_p, P(A.Result)]
        lib.oracle_solve_optimize.argtypes = [P(A.ModelDesc), P(A.SearchConfig), P(C.c_int64), P(A.Result)]
        lib.oracle_propagate.argtypes = [P(A.ModelDesc), P(C.c_uint64), C.c_int32, C.c_int32, P(A.FixpointResult)]
        lib.oracle_removals.argtypes = [P(A.ModelDesc), P(C.c_uint64), C.c_int32, P(C.c_int32), C.c_int32,
                                        P(C.c_uint64)]
        for f in (lib.oracle_solve_satisfy, lib.oracle_solve_optimize, lib.oracle_propagate, lib.oracle_removals):
            f.restype = C.c_int
        _OL = lib
    return _OL


def _raise(rc):
    if rc == A.E_OVERFLOW:
        raise S.ArithmeticOverflowError("overflow in linear propagation")
    if rc == A.E_NO_OBJECTIVE:
        raise S.LogicError("solve_optimize requires a minimize or maximize goal")
    if rc != A.OK:
        raise ValueError(f"oracle status {rc}")


def solve_satisfy(model: S.Model, cfg: S.SearchConfig | None = None, cb=None) -> S.SatisfyResult:
    cfg = cfg or S.SearchConfig()
    keep = model.desc_arrays()

    def tramp(_u, vals, n):
        return 1 if cb(S.Solution([vals[i] for i in range(n)])) else 0

    cf = A.SOLUTION_CB(tramp) if cb else A.SOLUTION_CB()
    res = A.Result()
    c = cfg.to_c()
    _raise(oracle_lib().oracle_solve_satisfy(C.byref(keep["desc"]), C.byref(c), cf, None, C.byref(res)))
    return S.SatisfyResult(S._stats(res), bool(res.complete))


def enumerate_solutions(model, cfg=None, stats=None):
    out = []
    r = solve_satisfy(model, cfg, lambda s: out.append(s) or True)
    if stats is not None:
        stats.nodes, stats.failures, stats.rounds, stats.solutions = r.stats.as_tuple()
    return out


def solve_optimize(model: S.Model, cfg: S.SearchConfig | None = None) -> S.OptimizeResult:
    cfg = cfg or S.SearchConfig()
    keep = model.desc_arrays()
    res = A.Result()
    best = (C.c_int64 * max(1, model.n_vars))()
    c = cfg.to_c()
    _raise(oracle_lib().oracle_solve_optimize(C.byref(keep["desc"]), C.byref(c), best, C.byref(res)))
    sol = S.Solution([best[i] for i in range(model.n_vars)], res.objective) if res.has_solution else None
    return S.OptimizeResult(sol, bool(res.complete), S._stats(res))


def propagate_fixpoint(model: S.Model, domains=None, alldiff=A.ARC_CONSISTENT, max_rounds=0):
    keep = model.desc_arrays()
    words = model.words_of(domains if domains is not None else model.domains)
    fr = A.FixpointResult()
    _raise(oracle_lib().oracle_propagate(C.byref(keep["desc"]), words, alldiff, max_rounds, C.byref(fr)))
    return model.domains_of(words), S.FixpointResult(bool(fr.failed), fr.failed_var, fr.rounds, fr.last_status)


def removals(model: S.Model, domains=None, cons=None, alldiff=A.ARC_CONSISTENT):
    keep = model.desc_arrays()
    words = model.words_of(domains if domains is not None else model.domains)
    out = (C.c_uint64 * max(1, model.word_start[-1]))()
    if cons is None:
        rc = oracle_lib().oracle_removals(C.byref(keep["desc"]), words, alldiff, None, 0, out)
    else:
        arr = (C.c_int32 * max(1, len(cons)))(*cons)
        rc = oracle_lib().oracle_removals(C.byref(keep["desc"]), words, alldiff, arr, len(cons), out)
    _raise(rc)
    return [d.values() for d in model.domains_of(out)]
