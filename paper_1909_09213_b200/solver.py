"""Python mirror of the reference solver interface (proj/include/fd/*.hpp) over libcubics.so.

Names, argument meaning and error behaviour follow the reference so the parity tests read like
the reference's own tests:

    fd::parse_model          -> parse_model(text)               (parser.hpp:38)
    fd::model_validate       -> Model.validate()                (model.hpp:93)
    fd::solve_satisfy        -> solve_satisfy(model, cfg, cb)   (search.hpp:62)
    fd::enumerate_solutions  -> enumerate_solutions(model, cfg) (search.hpp:65)
    fd::solve_optimize       -> solve_optimize(model, cfg)      (search.hpp:77)
    fd::lns_optimize         -> lns_optimize(model, LnsConfig)  (search.hpp:92; neighbourhoods
                                batched into one launch by optimize_batch)
    fd::propagate_fixpoint   -> propagate_fixpoint(model, doms) (propagation.hpp:114)
    fd::propagate_round      -> propagate_round(model, doms)    (propagation.hpp:102)
    fd::run_batch / prop_*   -> removals(model, doms, cons)     (propagation.hpp:78-89)

Errors are raised as the reference's exception types: ArithmeticOverflowError
(model.hpp:99-101), ValueError for a parse error, LogicError (std::logic_error) when optimising
without an objective. The CUDA engine is the only implementation: if libcubics.so is missing or
no B200 is present, calls raise EngineUnavailable - there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

from . import _abi as A


class EngineUnavailable(RuntimeError):
    """libcubics.so is not built or no usable sm_100 device is present."""


class ArithmeticOverflowError(RuntimeError):
    """fd::ArithmeticOverflowError (model.hpp:99-101)."""


class LogicError(RuntimeError):
    """std::logic_error raised by fd::solve_optimize without an objective (search.cpp:192)."""


class CapacityError(RuntimeError):
    pass


class UnsupportedInstance(RuntimeError):
    pass


_LIB = None


def lib():
    """Load the in-tree libcubics.so (built by __graft_entry__.build())."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(A.LIB_PATH):
            raise EngineUnavailable(f"{A.LIB_PATH} is not built; run __graft_entry__.build()")
        _LIB = A.declare(C.CDLL(A.LIB_PATH))
    return _LIB


def _check(rc, what=""):
    if rc == A.OK:
        return
    msg = (lib().cubics_last_error() or b"").decode()
    if rc == A.E_OVERFLOW:
        raise ArithmeticOverflowError(msg)
    if rc == A.E_NO_OBJECTIVE:
        raise LogicError(msg)
    if rc == A.E_CUDA:
        raise EngineUnavailable(msg)
    if rc == A.E_CAPACITY:
        raise CapacityError(msg)
    if rc == A.E_UNSUPPORTED:
        raise UnsupportedInstance(msg)
    raise ValueError(f"{what}: {A.STATUS_NAMES.get(rc, rc)}: {msg}")


# ------------------------------------------------------------------ configuration / results
@dataclass
class SearchConfig:
    """fd::SearchConfig (search.hpp:19-27) plus the engine selector."""
    var_heuristic: int = A.FIRST_FAIL
    value_heuristic: int = 0
    max_solutions: int = A.UINT64_MAX
    thread_count: int = 1
    seed: int = 0
    alldiff: int = A.ARC_CONSISTENT
    node_limit: int = 0
    engine: int = A.ENGINE_AUTO
    device: int = -1
    contexts: int = 0
    block_threads: int = 0
    count_only: bool = False
    initial_bound: int | None = None

    def to_c(self) -> A.SearchConfig:
        c = A.SearchConfig()
        for f in ("var_heuristic", "value_heuristic", "max_solutions", "thread_count", "seed", "alldiff",
                  "node_limit", "engine", "device", "contexts", "block_threads"):
            setattr(c, f, getattr(self, f))
        c.count_only = 1 if self.count_only else 0
        if self.initial_bound is not None:
            c.has_initial_bound = 1
            c.initial_bound = self.initial_bound
        return c


@dataclass
class SearchStats:
    nodes: int = 0
    failures: int = 0
    rounds: int = 0
    solutions: int = 0

    def as_tuple(self):
        return (self.nodes, self.failures, self.rounds, self.solutions)


@dataclass
class SatisfyResult:
    stats: SearchStats
    complete: bool
    engine: int = 0
    contexts: int = 1
    device_ms: float = 0.0
    total_ms: float = 0.0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    kernel_launches: int = 0
    remote_in: int = 0   # shared queue: subtrees taken from other GPUs
    remote_out: int = 0  # shared queue: subtrees given to other GPUs


@dataclass
class Solution:
    values: list
    objective: int | None = None


@dataclass
class OptimizeResult:
    best: Solution | None
    complete: bool
    stats: SearchStats
    engine: int = 0
    contexts: int = 1
    device_ms: float = 0.0
    total_ms: float = 0.0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    kernel_launches: int = 0
    remote_in: int = 0   # shared queue: subtrees taken from other GPUs
    remote_out: int = 0  # shared queue: subtrees given to other GPUs


@dataclass
class FixpointResult:
    failed: bool
    failed_var: int
    rounds: int
    last_status: int = 1  # fd::RoundResult::Status: 0 Changed, 1 Stable, 2 Failed


def _stats(r: A.Result) -> SearchStats:
    return SearchStats(r.stats.nodes, r.stats.failures, r.stats.rounds, r.stats.solutions)


# ------------------------------------------------------------------ model
class Domain:
    """A value set [offset, offset+width) as a Python int bitmask (bit i = offset + i)."""

    __slots__ = ("offset", "width", "bits")

    def __init__(self, lo: int, hi: int | None = None, bits: int | None = None, width: int | None = None):
        if hi is not None:
            if lo > hi:
                raise ValueError("empty range")
            if hi - lo >= 1024:
                raise ValueError("width exceeded")
            self.offset, self.width = lo, hi - lo + 1
            self.bits = (1 << self.width) - 1
        else:
            self.offset, self.width = lo, width
            self.bits = bits & ((1 << width) - 1)

    def values(self):
        b, out, i = self.bits, [], 0
        while b:
            if b & 1:
                out.append(self.offset + i)
            b >>= 1
            i += 1
        return out

    def size(self):
        return bin(self.bits).count("1")

    def empty(self):
        return self.bits == 0

    def contains(self, v):
        i = v - self.offset
        return 0 <= i < self.width and (self.bits >> i) & 1 == 1

    def remove(self, v):
        if self.contains(v):
            self.bits &= ~(1 << (v - self.offset))

    def copy(self):
        return Domain(self.offset, bits=self.bits, width=self.width)

    def __eq__(self, o):
        return (self.offset, self.width, self.bits) == (o.offset, o.width, o.bits)

    def __repr__(self):
        return f"Domain({self.values()})"

    def words(self):
        nw = (self.width + 63) // 64
        return [(self.bits >> (64 * i)) & ((1 << 64) - 1) for i in range(nw)]


class Model:
    """Owning handle of a cubics_model (fd::Model)."""

    def __init__(self, handle):
        self._h = handle
        d = A.ModelDesc()
        _check(lib().cubics_model_describe(self._h, C.byref(d)), "describe")
        self.n_vars = d.n_vars
        self.n_cons = d.n_cons
        self.goal = d.goal
        self.goal_var = d.goal_var
        n, mc = self.n_vars, self.n_cons
        self.offsets = d.var_offset[:n] if n else []
        self.widths = d.var_width[:n] if n else []
        self.word_start = [0]
        for w in self.widths:
            self.word_start.append(self.word_start[-1] + (w + 63) // 64)
        words = d.var_words[:self.word_start[-1]] if self.word_start[-1] else []
        self.domains = []
        for v in range(n):
            a, b = self.word_start[v], self.word_start[v + 1]
            bits = words[a] if b - a == 1 else sum(x << (64 * i) for i, x in enumerate(words[a:b]))
            self.domains.append(Domain(self.offsets[v], bits=bits, width=self.widths[v]))
        self.con_kind = d.con_kind[:mc] if mc else []
        self.con_op = d.con_op[:mc] if mc else []
        self.con_value = d.con_value[:mc] if mc else []
        self.con_start = d.con_start[:mc + 1] if mc else [0]
        nt = self.con_start[-1] if mc else 0
        self.term_var = d.term_var[:nt] if nt else []
        self.term_coeff = d.term_coeff[:nt] if nt else []
        # positive tables (extension): tuples of constraint c, flattened
        self.table_start = d.table_start[:mc] if mc else []
        tot = 0
        for c in range(mc):
            if self.con_kind[c] == A.TABLE:
                k = self.con_start[c + 1] - self.con_start[c]
                tot = max(tot, self.table_start[c] + self.con_value[c] * k)
        self.table_data = d.table_data[:tot] if tot else []
        self._names = None

    @property
    def names(self):
        if self._names is None:
            self._names = [lib().cubics_model_var_name(self._h, i).decode() for i in range(self.n_vars)]
        return self._names

    @property
    def handle(self):
        return self._h

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h and _LIB is not None:
            _LIB.cubics_model_free(h)

    def validate(self):
        """fd::model_validate: list of (kind, constraint_index); empty = valid."""
        cnt = C.c_int32(0)
        buf = (A.Diagnostic * 256)()
        _check(lib().cubics_model_validate(self._h, buf, 256, C.byref(cnt)), "validate")
        return [(buf[i].kind, buf[i].constraint_index) for i in range(min(cnt.value, 256))]

    def desc_arrays(self):
        """Flat arrays for building a cubics_model_desc (keeps them alive in the returned dict)."""
        return build_desc(self.offsets, self.widths, self.domains, self.con_kind, self.con_op, self.con_value,
                          self.con_start, self.term_var, self.term_coeff, self.goal, self.goal_var,
                          self.table_start, self.table_data)

    def words_of(self, domains):
        out = (C.c_uint64 * max(1, self.word_start[-1]))()
        for v, d in enumerate(domains):
            for i, x in enumerate(d.words()):
                out[self.word_start[v] + i] = x
        return out

    def domains_of(self, words):
        doms = []
        for v in range(self.n_vars):
            bits = 0
            for i in range(self.word_start[v + 1] - self.word_start[v]):
                bits |= int(words[self.word_start[v] + i]) << (64 * i)
            doms.append(Domain(self.offsets[v], bits=bits, width=self.widths[v]))
        return doms

    def with_goal(self, goal, var):
        arr = self.desc_arrays()
        arr["desc"].goal = goal
        arr["desc"].goal_var = var
        return model_from_desc(arr["desc"])

    def with_domains(self, domains):
        """A copy of this model with new initial domains (each keeps its own offset and width,
        as fd::Model::domains does, e.g. the Domain(val, val) of neighborhood_model)."""
        arr = build_desc([d.offset for d in domains], [d.width for d in domains], domains, self.con_kind, self.con_op, self.con_value,
                         self.con_start, self.term_var, self.term_coeff, self.goal, self.goal_var,
                         self.table_start, self.table_data)
        return model_from_desc(arr["desc"])


def build_desc(offsets, widths, domains, kinds, ops, values, starts, tvars, tcoeffs, goal=A.SATISFY, goal_var=0,
               table_start=None, table_data=None):
    n, m = len(offsets), len(kinds)
    nt = starts[-1] if m else 0
    ws = [0]
    for w in widths:
        ws.append(ws[-1] + (w + 63) // 64)
    keep = {
        "off": (C.c_int64 * max(1, n))(*offsets),
        "width": (C.c_int32 * max(1, n))(*widths),
        "words": (C.c_uint64 * max(1, ws[-1]))(),
        "kind": (C.c_int32 * max(1, m))(*kinds),
        "op": (C.c_int32 * max(1, m))(*ops),
        "value": (C.c_int64 * max(1, m))(*values),
        "start": (C.c_int32 * (m + 1))(*(starts if m else [0])),
        "tvar": (C.c_int32 * max(1, nt))(*tvars),
        "tcoeff": (C.c_int64 * max(1, nt))(*(tcoeffs or [1] * nt)),
        "tstart": (C.c_int64 * max(1, m))(*(table_start or [0] * m)),
        "tdata": (C.c_int64 * max(1, len(table_data or [])))(*(table_data or [])),
    }
    for v, d in enumerate(domains):
        for i, x in enumerate(d.words()):
            keep["words"][ws[v] + i] = x
    d = A.ModelDesc()
    d.n_vars = n
    d.var_offset = keep["off"]
    d.var_width = keep["width"]
    d.var_words = keep["words"]
    d.n_cons = m
    d.con_kind = keep["kind"]
    d.con_op = keep["op"]
    d.con_value = keep["value"]
    d.con_start = keep["start"]
    d.term_var = keep["tvar"]
    d.term_coeff = keep["tcoeff"]
    d.goal = goal
    d.goal_var = goal_var
    d.table_start = keep["tstart"]
    d.table_data = keep["tdata"]
    keep["desc"] = d
    return keep


def model_from_desc(desc: A.ModelDesc) -> Model:
    h = C.c_void_p()
    _check(lib().cubics_model_create(C.byref(desc), C.byref(h)), "model_create")
    return Model(h.value)


def parse_model(text: str) -> Model:
    """fd::parse_model; raises ValueError(message) with the reference's line/column format."""
    h = C.c_void_p()
    err = A.ParseError()
    raw = text.encode()
    rc = lib().cubics_model_parse(raw, len(raw), C.byref(h), C.byref(err))
    if rc == A.E_PARSE:
        e = ValueError(err.message.decode())
        e.kind, e.line, e.column = err.kind, err.line, err.column
        raise e
    _check(rc, "parse")
    return Model(h.value)


# ------------------------------------------------------------------ search
def solve_satisfy(model: Model, cfg: SearchConfig | None = None, cb=None) -> SatisfyResult:
    """fd::solve_satisfy: cb(Solution) -> bool is called per solution in the reference's DFS order."""
    cfg = cfg or SearchConfig()
    user_err = []

    def trampoline(_user, vals, n):
        try:
            keep = cb(Solution([vals[i] for i in range(n)]))
            return 1 if keep else 0
        except BaseException as e:  # noqa: BLE001 - re-raised below
            user_err.append(e)
            return 0

    cfun = A.SOLUTION_CB(trampoline) if cb else A.SOLUTION_CB()
    res = A.Result()
    c = cfg.to_c()
    _check(lib().cubics_solve_satisfy(model.handle, C.byref(c), cfun, None, C.byref(res)), "solve_satisfy")
    if user_err:
        raise user_err[0]
    return SatisfyResult(_stats(res), bool(res.complete), res.engine, res.contexts, res.device_ms, res.total_ms,
                         res.h2d_bytes, res.d2h_bytes, res.kernel_launches)


def enumerate_array(model: Model, cfg: SearchConfig | None = None):
    """cubics_enumerate: (numpy int64 array [count, n_vars] in DFS order, SatisfyResult)."""
    import numpy as np

    cfg = cfg or SearchConfig()
    res = A.Result()
    sols = C.POINTER(A.Solutions)()
    c = cfg.to_c()
    _check(lib().cubics_enumerate(model.handle, C.byref(c), C.byref(sols), C.byref(res)), "enumerate")
    cnt, nv = sols.contents.count, sols.contents.n_vars
    if cnt and nv:
        # zero-copy view of the library buffer; freed when the last view is collected
        arr = np.ctypeslib.as_array(sols.contents.values, shape=(cnt, nv))
        import weakref
        weakref.finalize(arr, lib().cubics_solutions_free, sols)
    else:
        lib().cubics_solutions_free(sols)
        arr = np.zeros((cnt, nv), dtype=np.int64)
    return arr, SatisfyResult(_stats(res), bool(res.complete), res.engine, res.contexts, res.device_ms,
                              res.total_ms, res.h2d_bytes, res.d2h_bytes, res.kernel_launches)


def enumerate_solutions(model: Model, cfg: SearchConfig | None = None, stats: SearchStats | None = None):
    """fd::enumerate_solutions: every solution (Solution objects) in DFS order."""
    arr, r = enumerate_array(model, cfg)
    if stats is not None:
        stats.nodes, stats.failures, stats.rounds, stats.solutions = r.stats.as_tuple()
    return [Solution(row) for row in arr.tolist()]


def solve_optimize(model: Model, cfg: SearchConfig | None = None) -> OptimizeResult:
    """fd::solve_optimize (branch and bound)."""
    cfg = cfg or SearchConfig()
    res = A.Result()
    best = (C.c_int64 * max(1, model.n_vars))()
    c = cfg.to_c()
    _check(lib().cubics_solve_optimize(model.handle, C.byref(c), best, C.byref(res)), "solve_optimize")
    sol = None
    if res.has_solution:
        sol = Solution([best[i] for i in range(model.n_vars)], res.objective)
    return OptimizeResult(sol, bool(res.complete), _stats(res), res.engine, res.contexts, res.device_ms, res.total_ms,
                          res.h2d_bytes, res.d2h_bytes, res.kernel_launches)


def optimize_batch(model: Model, domain_words, bounds=None, cfg: SearchConfig | None = None):
    """cubics_solve_optimize_batch: one branch-and-bound search per row of ``domain_words``
    (uint64 [count, model words], desc packing), all in one device launch. ``bounds`` (None or a
    sequence of int / None) gives each problem's strict initial bound. Returns [OptimizeResult]."""
    import numpy as np

    cfg = cfg or SearchConfig()
    nw = max(1, model.word_start[-1])
    words = np.ascontiguousarray(np.asarray(domain_words, dtype=np.uint64).reshape(-1, nw))
    count = words.shape[0]
    if count == 0:
        return []
    b = np.zeros(count, dtype=np.int64)
    hb = np.zeros(count, dtype=np.int32)
    if bounds is not None:
        for i, x in enumerate(bounds):
            if x is not None:
                b[i], hb[i] = x, 1
    n = model.n_vars
    best = np.zeros((count, max(1, n)), dtype=np.int64)
    res = (A.Result * count)()
    c = cfg.to_c()
    P = C.POINTER
    _check(lib().cubics_solve_optimize_batch(
        model.handle, C.byref(c), count, words.ctypes.data_as(P(C.c_uint64)), b.ctypes.data_as(P(C.c_int64)),
        hb.ctypes.data_as(P(C.c_int32)), best.ctypes.data_as(P(C.c_int64)), res), "solve_optimize_batch")
    out = []
    for i in range(count):
        r = res[i]
        sol = Solution(best[i, :n].tolist(), r.objective) if r.has_solution else None
        out.append(OptimizeResult(sol, bool(r.complete), _stats(r), r.engine, r.contexts, r.device_ms, r.total_ms))
    return out


@dataclass
class LnsConfig:
    """fd::LnsConfig (search.hpp:29-37)."""
    destroy_rate: float = 0.3
    iterations: int = 10
    neighborhoods: int = 1
    seed: int = 0
    per_iteration_node_limit: int = 0
    thread_count: int = 1
    alldiff: int = A.ARC_CONSISTENT


@dataclass
class LnsResult:
    """fd::LnsResult (search.hpp:79-84): best, summed stats, per-iteration trajectory."""
    best: Solution | None
    stats: SearchStats
    trajectory: list
    initial_complete: bool
    device_ms: float = 0.0


def lns_optimize(model: Model, cfg: LnsConfig | None = None) -> LnsResult:
    """fd::lns_optimize (search.cpp:225-314): first solution, then ``iterations`` rounds of
    ``neighborhoods`` destroy-and-repair searches against the frozen incumbent. Each iteration's
    neighbourhoods run as ONE batched device launch (optimize_batch); destroy sets follow
    Rng::derive(seed, nb, iter) with the reference's partial Fisher-Yates, merge is lowest-index-wins."""
    import math

    import numpy as np

    from .models import Rng

    cfg = cfg or LnsConfig()
    if model.goal == A.SATISFY:
        raise LogicError("lns_optimize requires a minimize or maximize goal")
    minimizing = model.goal == A.MINIMIZE
    found = []
    first = solve_satisfy(model, SearchConfig(max_solutions=1, thread_count=cfg.thread_count, alldiff=cfg.alldiff),
                          lambda s: (found.append(s), False)[1])
    stats = SearchStats(*first.stats.as_tuple())
    best = None
    if found:
        best = Solution(found[0].values, found[0].values[model.goal_var])
    res = LnsResult(None, stats, [], first.complete or best is not None)
    if best is None:
        return res
    n = model.n_vars
    destroy = min(n, max(1, math.ceil(cfg.destroy_rate * n)))
    nw = max(1, model.word_start[-1])
    base = np.zeros(nw, dtype=np.uint64)
    base_words = model.words_of(model.domains)
    base[:] = np.ctypeslib.as_array(base_words)[:nw]
    scfg = SearchConfig(alldiff=cfg.alldiff, node_limit=cfg.per_iteration_node_limit, engine=A.ENGINE_PARITY)
    for it in range(cfg.iterations):
        inc = best
        words = np.tile(base, (cfg.neighborhoods, 1))
        for nb in range(cfg.neighborhoods):
            rng = Rng.derive(cfg.seed, nb, it)
            ids = list(range(n))
            destroyed = [False] * n
            for i in range(destroy):
                j = i + rng.below(n - i)
                ids[i], ids[j] = ids[j], ids[i]
                destroyed[ids[i]] = True
            for v in range(n):
                if not destroyed[v]:  # neighborhood_model (search.cpp:207-217): fixed to the incumbent
                    ws, we = model.word_start[v], model.word_start[v + 1]
                    words[nb, ws:we] = 0
                    bit = inc.values[v] - model.offsets[v]
                    words[nb, ws + bit // 64] = np.uint64(1 << (bit % 64))
        out = optimize_batch(model, words, [inc.objective] * cfg.neighborhoods, scfg)
        res.device_ms += out[0].device_ms  # one launch for the whole iteration
        for r in out:
            stats.nodes += r.stats.nodes
            stats.failures += r.stats.failures
            stats.rounds += r.stats.rounds
            if r.best is not None and (r.best.objective < best.objective if minimizing
                                       else r.best.objective > best.objective):
                best = r.best
        res.trajectory.append(best.objective)
    res.best = best
    return res


class TaskQueue:
    """Shared subtree queue for cubics_solve_shard_shared: one claim counter in the owner GPU's
    HBM. The owner creates it and ships `handle` (64 bytes) to the other ranks, which `open` it
    (CUDA IPC; NVLink peer access). reset() (owner) + a barrier must precede every search."""

    def __init__(self, ptr, handle: bytes, owner: bool):
        self.ptr, self.handle, self.owner = ptr, handle, owner

    @classmethod
    def create(cls, device: int = -1) -> "TaskQueue":
        ptr = C.c_void_p()
        buf = C.create_string_buffer(A.TASK_QUEUE_HANDLE_BYTES)
        _check(lib().cubics_task_queue_create(device, C.byref(ptr), buf), "task_queue_create")
        return cls(ptr, buf.raw, True)

    @classmethod
    def open(cls, handle: bytes, device: int = -1) -> "TaskQueue":
        if len(handle) != A.TASK_QUEUE_HANDLE_BYTES:
            raise ValueError("task queue handle must be %d bytes" % A.TASK_QUEUE_HANDLE_BYTES)
        ptr = C.c_void_p()
        _check(lib().cubics_task_queue_open(device, handle, C.byref(ptr)), "task_queue_open")
        return cls(ptr, bytes(handle), False)

    def reset(self):
        _check(lib().cubics_task_queue_reset(self.ptr), "task_queue_reset")

    def claims(self) -> int:
        v = C.c_uint64()
        _check(lib().cubics_task_queue_claims(self.ptr, C.byref(v)), "task_queue_claims")
        return v.value

    def close(self):
        if self.ptr:
            lib().cubics_task_queue_destroy(self.ptr)
            self.ptr = None


def solve_shard(model: Model, cfg: SearchConfig, shard_index: int, shard_count: int, cb=None,
                queue: TaskQueue | None = None):
    """One rank's share of a multi-GPU search; cb(key_words, values).

    queue=None: cubics_solve_shard (static split of the frontier subtrees). With a TaskQueue:
    cubics_solve_shard_shared (subtrees claimed dynamically through the shared counter)."""
    def trampoline(_u, key, kw, vals, n):
        return 1 if cb([key[i] for i in range(kw)], [vals[i] for i in range(n)]) else 0

    cfun = A.KEYED_SOLUTION_CB(trampoline) if cb else A.KEYED_SOLUTION_CB()
    res = A.Result()
    c = cfg.to_c()
    if queue is None:
        rc = lib().cubics_solve_shard(model.handle, C.byref(c), shard_index, shard_count, cfun, None, C.byref(res))
    else:
        rc = lib().cubics_solve_shard_shared(model.handle, C.byref(c), shard_index, shard_count, queue.ptr, cfun,
                                             None, C.byref(res))
    _check(rc, "solve_shard")
    return SatisfyResult(_stats(res), bool(res.complete), res.engine, res.contexts, res.device_ms, res.total_ms,
                         res.h2d_bytes, res.d2h_bytes, res.kernel_launches, res.remote_tasks_in, res.remote_tasks_out)


def solve_optimize_shard(model: Model, cfg: SearchConfig, shard_index: int, shard_count: int,
                         queue: TaskQueue | None = None) -> OptimizeResult:
    """One rank's share of a multi-GPU branch and bound (cubics_solve_optimize_shard): partial
    stats (summed across ranks) and this rank's best incumbent (the best over ranks is the
    optimum). With a TaskQueue the subtrees are claimed dynamically and the incumbent objective is
    shared between the GPUs through the queue state (reset it before every search)."""
    res = A.Result()
    best = (C.c_int64 * max(1, model.n_vars))()
    c = cfg.to_c()
    _check(lib().cubics_solve_optimize_shard(model.handle, C.byref(c), shard_index, shard_count,
                                             queue.ptr if queue is not None else None, best, C.byref(res)),
           "solve_optimize_shard")
    sol = Solution([best[i] for i in range(model.n_vars)], res.objective) if res.has_solution else None
    return OptimizeResult(sol, bool(res.complete), _stats(res), res.engine, res.contexts, res.device_ms, res.total_ms,
                          res.h2d_bytes, res.d2h_bytes, res.kernel_launches, res.remote_tasks_in,
                          res.remote_tasks_out)


def solve_multi(model: Model, devices, cfg: SearchConfig | None = None, cb=None):
    """cubics_solve_multi: one host process drives every device in `devices` (a device may repeat).
    Returns (SatisfyResult or OptimizeResult, remote subtrees moved between the devices)."""
    cfg = cfg or SearchConfig()
    user_err = []

    def trampoline(_user, vals, n):
        try:
            return 1 if cb(Solution([vals[i] for i in range(n)])) else 0
        except BaseException as e:  # noqa: BLE001 - re-raised below
            user_err.append(e)
            return 0

    cfun = A.SOLUTION_CB(trampoline) if cb else A.SOLUTION_CB()
    devs = (C.c_int32 * len(devices))(*devices)
    best = (C.c_int64 * max(1, model.n_vars))()
    res = A.Result()
    c = cfg.to_c()
    _check(lib().cubics_solve_multi(model.handle, C.byref(c), len(devices), devs, cfun, None, best, C.byref(res)),
           "solve_multi")
    if user_err:
        raise user_err[0]
    if model.goal != 0:
        sol = Solution([best[i] for i in range(model.n_vars)], res.objective) if res.has_solution else None
        r = OptimizeResult(sol, bool(res.complete), _stats(res), res.engine, res.contexts, res.device_ms, res.total_ms,
                           res.h2d_bytes, res.d2h_bytes, res.kernel_launches, res.remote_tasks_in, res.remote_tasks_out)
    else:
        r = SatisfyResult(_stats(res), bool(res.complete), res.engine, res.contexts, res.device_ms, res.total_ms,
                          res.h2d_bytes, res.d2h_bytes, res.kernel_launches, res.remote_tasks_in, res.remote_tasks_out)
    return r


class FirstShard:
    """One rank's part of a multi-GPU exact first solution (cubics_solve_first_shard).

    best() -> (key_words, values) of this rank's DFS-first solution, or None; the caller takes the
    minimum key K* over ranks. prefix(K*) -> this rank's share of the reference's stats up to K*
    (shares sum across ranks to the reference's (nodes, failures, rounds, 1)); prefix(None) when
    no rank found a solution gives the complete search's share."""

    def __init__(self, ptr, result: SatisfyResult, n_vars: int):
        self.ptr = ptr
        self.result = result
        self.n_vars = n_vars

    def best(self):
        kw = C.c_int32(0)
        has = C.c_int32(0)
        _check(lib().cubics_first_shard_best(self.ptr, None, C.byref(kw), None, C.byref(has)), "first_shard_best")
        if not has.value:
            return None
        key = (C.c_uint32 * max(1, kw.value))()
        vals = (C.c_int64 * max(1, self.n_vars))()
        _check(lib().cubics_first_shard_best(self.ptr, key, C.byref(kw), vals, C.byref(has)), "first_shard_best")
        return [key[i] for i in range(kw.value)], [vals[i] for i in range(self.n_vars)]

    def prefix(self, key) -> SearchStats:
        st = A.Stats()
        if key is None:
            _check(lib().cubics_first_shard_prefix(self.ptr, None, 0, C.byref(st)), "first_shard_prefix")
        else:
            arr = (C.c_uint32 * len(key))(*key)
            _check(lib().cubics_first_shard_prefix(self.ptr, arr, len(key), C.byref(st)), "first_shard_prefix")
        return SearchStats(st.nodes, st.failures, st.rounds, st.solutions)

    def close(self):
        if self.ptr:
            lib().cubics_first_shard_free(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter teardown
            pass


def solve_first_shard(model: Model, cfg: SearchConfig, shard_index: int, shard_count: int,
                      queue: TaskQueue | None = None) -> FirstShard:
    """One rank's share of a multi-GPU exact first-solution search (cubics_solve_first_shard)."""
    res = A.Result()
    ptr = C.c_void_p()
    c = cfg.to_c()
    _check(lib().cubics_solve_first_shard(model.handle, C.byref(c), shard_index, shard_count,
                                          queue.ptr if queue is not None else None, C.byref(ptr), C.byref(res)),
           "solve_first_shard")
    r = SatisfyResult(_stats(res), bool(res.complete), res.engine, res.contexts, res.device_ms, res.total_ms,
                      res.h2d_bytes, res.d2h_bytes, res.kernel_launches)
    return FirstShard(ptr.value, r, model.n_vars)


def merge_first(shards):
    """Sequential driver of the two-phase protocol over FirstShard parts held in one process:
    (stats, values of the DFS-first solution or None) - what distributed.solve_distributed does
    with one all-gather and one all-reduce."""
    bests = [b for b in (s.best() for s in shards) if b is not None]
    key, vals = min(bests, key=lambda b: b[0]) if bests else (None, None)
    tot = [0, 0, 0, 0]
    for s in shards:
        p = s.prefix(key)
        tot = [a + b for a, b in zip(tot, p.as_tuple())]
    return SearchStats(*tot), vals


# ------------------------------------------------------------------ propagation
def propagate_fixpoint(model: Model, domains=None, alldiff=A.ARC_CONSISTENT, max_rounds=0):
    """fd::propagate_fixpoint over `domains` (default: the model's); returns (domains, FixpointResult)."""
    doms = domains if domains is not None else model.domains
    words = model.words_of(doms)
    fr = A.FixpointResult()
    _check(lib().cubics_propagate(model.handle, words, alldiff, max_rounds, C.byref(fr)), "propagate")
    return model.domains_of(words), FixpointResult(bool(fr.failed), fr.failed_var, fr.rounds, fr.last_status)


def propagate_round(model: Model, domains=None, alldiff=A.ARC_CONSISTENT):
    """fd::propagate_round: one bulk-synchronous round; returns (domains, status, failed_var)."""
    doms, fr = propagate_fixpoint(model, domains, alldiff, max_rounds=1)
    return doms, fr.last_status, fr.failed_var


def removals(model: Model, domains=None, cons=None, alldiff=A.ARC_CONSISTENT):
    """fd::run_batch / propagate_one: per-var removed value lists against the snapshot."""
    doms = domains if domains is not None else model.domains
    words = model.words_of(doms)
    out = (C.c_uint64 * max(1, model.word_start[-1]))()
    if cons is None:
        rc = lib().cubics_removals(model.handle, words, alldiff, None, 0, out)
    else:
        arr = (C.c_int32 * max(1, len(cons)))(*cons)
        rc = lib().cubics_removals(model.handle, words, alldiff, arr, len(cons), out)
    _check(rc, "removals")
    return [d.values() for d in model.domains_of(out)]


def device_count() -> int:
    return lib().cubics_device_count()


def build_info() -> str:
    return lib().cubics_build_info().decode()
