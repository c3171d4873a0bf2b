"""ctypes declarations of include/cubics.h (the C ABI of libcubics.so).

The structures here are shared by the product binding (``solver.py``) and the test-only oracle
binding (``tests/oracle_binding.py``), which exposes the same entry-point contracts.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# CUBICS_LIB: an alternative in-tree build of the engine (A/B probes only)
LIB_PATH = os.environ.get("CUBICS_LIB") or os.path.join(HERE, "lib", "libcubics.so")

# status codes (enum cubics_status)
OK, E_INVALID, E_PARSE, E_OVERFLOW, E_NO_OBJECTIVE, E_CUDA, E_CAPACITY, E_UNSUPPORTED = range(8)
STATUS_NAMES = {0: "OK", 1: "INVALID", 2: "PARSE", 3: "OVERFLOW", 4: "NO_OBJECTIVE", 5: "CUDA",
                6: "CAPACITY", 7: "UNSUPPORTED"}

RELBIN, LINEAR, ALLDIFF, TABLE = 0, 1, 2, 3
LT, LE, GT, GE, EQ, NE = range(6)
LIN_LE, LIN_EQ = 0, 1
SATISFY, MINIMIZE, MAXIMIZE = 0, 1, 2
INPUT_ORDER, FIRST_FAIL = 0, 1
FORWARD_CHECKING, ARC_CONSISTENT = 0, 1
ENGINE_AUTO, ENGINE_PARITY, ENGINE_PARALLEL, ENGINE_GRID = 0, 1, 2, 3
UINT64_MAX = (1 << 64) - 1


class ModelDesc(C.Structure):
    _fields_ = [
        ("n_vars", C.c_int32),
        ("var_offset", C.POINTER(C.c_int64)),
        ("var_width", C.POINTER(C.c_int32)),
        ("var_words", C.POINTER(C.c_uint64)),
        ("n_cons", C.c_int32),
        ("con_kind", C.POINTER(C.c_int32)),
        ("con_op", C.POINTER(C.c_int32)),
        ("con_value", C.POINTER(C.c_int64)),
        ("con_start", C.POINTER(C.c_int32)),
        ("term_var", C.POINTER(C.c_int32)),
        ("term_coeff", C.POINTER(C.c_int64)),
        ("goal", C.c_int32),
        ("goal_var", C.c_int32),
        ("table_start", C.POINTER(C.c_int64)),
        ("table_data", C.POINTER(C.c_int64)),
    ]


class ParseError(C.Structure):
    _fields_ = [("kind", C.c_int32), ("line", C.c_int32), ("column", C.c_int32), ("message", C.c_char * 256)]


class Diagnostic(C.Structure):
    _fields_ = [("kind", C.c_int32), ("constraint_index", C.c_int32)]


class SearchConfig(C.Structure):
    _fields_ = [
        ("var_heuristic", C.c_int32),
        ("value_heuristic", C.c_int32),
        ("max_solutions", C.c_uint64),
        ("thread_count", C.c_int32),
        ("seed", C.c_uint64),
        ("alldiff", C.c_int32),
        ("node_limit", C.c_uint64),
        ("engine", C.c_int32),
        ("device", C.c_int32),
        ("contexts", C.c_int32),
        ("block_threads", C.c_int32),
        ("count_only", C.c_int32),
        ("has_initial_bound", C.c_int32),
        ("initial_bound", C.c_int64),
    ]


class Stats(C.Structure):
    _fields_ = [("nodes", C.c_uint64), ("failures", C.c_uint64), ("rounds", C.c_uint64), ("solutions", C.c_uint64)]


class Result(C.Structure):
    _fields_ = [
        ("stats", Stats),
        ("complete", C.c_int32),
        ("has_solution", C.c_int32),
        ("objective", C.c_int64),
        ("engine", C.c_int32),
        ("contexts", C.c_int32),
        ("device_ms", C.c_double),
        ("total_ms", C.c_double),
        ("h2d_bytes", C.c_uint64),
        ("d2h_bytes", C.c_uint64),
        ("kernel_launches", C.c_uint64),
        ("remote_tasks_in", C.c_uint64),
        ("remote_tasks_out", C.c_uint64),
    ]


class Solutions(C.Structure):
    _fields_ = [("count", C.c_uint64), ("n_vars", C.c_int32), ("values", C.POINTER(C.c_int64))]


class FixpointResult(C.Structure):
    _fields_ = [("failed", C.c_int32), ("failed_var", C.c_int32), ("rounds", C.c_int32), ("last_status", C.c_int32)]


TASK_QUEUE_HANDLE_BYTES = 64  # CUBICS_TASK_QUEUE_HANDLE_BYTES

SOLUTION_CB = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.POINTER(C.c_int64), C.c_int32)
KEYED_SOLUTION_CB = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.POINTER(C.c_uint32), C.c_int32,
                                C.POINTER(C.c_int64), C.c_int32)

# every symbol the header declares (tests check the library exports all of them)
EXPORTED = [
    "cubics_model_create", "cubics_model_parse", "cubics_model_free", "cubics_model_describe",
    "cubics_model_var_name", "cubics_model_validate", "cubics_search_config_init",
    "cubics_solve_satisfy", "cubics_enumerate", "cubics_solutions_free", "cubics_solve_optimize",
    "cubics_solve_optimize_batch", "cubics_solve_shard", "cubics_solve_shard_shared", "cubics_solve_optimize_shard",
    "cubics_task_queue_create", "cubics_task_queue_open", "cubics_task_queue_reset", "cubics_task_queue_claims",
    "cubics_task_queue_destroy", "cubics_solve_first_shard", "cubics_first_shard_best", "cubics_first_shard_prefix",
    "cubics_first_shard_free", "cubics_solve_multi", "cubics_propagate",
    "cubics_removals", "cubics_last_error", "cubics_build_info", "cubics_device_count", "cubics_warmup",
]


def declare(lib):
    """Attach argtypes/restype to a loaded libcubics."""
    P = C.POINTER
    lib.cubics_model_create.argtypes = [P(ModelDesc), P(C.c_void_p)]
    lib.cubics_model_create.restype = C.c_int
    lib.cubics_model_parse.argtypes = [C.c_char_p, C.c_size_t, P(C.c_void_p), P(ParseError)]
    lib.cubics_model_parse.restype = C.c_int
    lib.cubics_model_free.argtypes = [C.c_void_p]
    lib.cubics_model_free.restype = None
    lib.cubics_model_describe.argtypes = [C.c_void_p, P(ModelDesc)]
    lib.cubics_model_describe.restype = C.c_int
    lib.cubics_model_var_name.argtypes = [C.c_void_p, C.c_int32]
    lib.cubics_model_var_name.restype = C.c_char_p
    lib.cubics_model_validate.argtypes = [C.c_void_p, P(Diagnostic), C.c_int32, P(C.c_int32)]
    lib.cubics_model_validate.restype = C.c_int
    lib.cubics_search_config_init.argtypes = [P(SearchConfig)]
    lib.cubics_search_config_init.restype = None
    lib.cubics_solve_satisfy.argtypes = [C.c_void_p, P(SearchConfig), SOLUTION_CB, C.c_void_p, P(Result)]
    lib.cubics_solve_satisfy.restype = C.c_int
    lib.cubics_enumerate.argtypes = [C.c_void_p, P(SearchConfig), P(P(Solutions)), P(Result)]
    lib.cubics_enumerate.restype = C.c_int
    lib.cubics_solutions_free.argtypes = [P(Solutions)]
    lib.cubics_solutions_free.restype = None
    lib.cubics_solve_optimize.argtypes = [C.c_void_p, P(SearchConfig), P(C.c_int64), P(Result)]
    lib.cubics_solve_optimize.restype = C.c_int
    lib.cubics_solve_optimize_batch.argtypes = [C.c_void_p, P(SearchConfig), C.c_int32, P(C.c_uint64), P(C.c_int64),
                                                P(C.c_int32), P(C.c_int64), P(Result)]
    lib.cubics_solve_optimize_batch.restype = C.c_int
    lib.cubics_solve_shard.argtypes = [C.c_void_p, P(SearchConfig), C.c_int32, C.c_int32, KEYED_SOLUTION_CB,
                                       C.c_void_p, P(Result)]
    lib.cubics_solve_shard.restype = C.c_int
    lib.cubics_solve_shard_shared.argtypes = [C.c_void_p, P(SearchConfig), C.c_int32, C.c_int32, C.c_void_p,
                                              KEYED_SOLUTION_CB, C.c_void_p, P(Result)]
    lib.cubics_solve_shard_shared.restype = C.c_int
    lib.cubics_solve_optimize_shard.argtypes = [C.c_void_p, P(SearchConfig), C.c_int32, C.c_int32, C.c_void_p,
                                                P(C.c_int64), P(Result)]
    lib.cubics_solve_optimize_shard.restype = C.c_int
    lib.cubics_task_queue_create.argtypes = [C.c_int32, P(C.c_void_p), C.c_char_p]
    lib.cubics_task_queue_create.restype = C.c_int
    lib.cubics_task_queue_open.argtypes = [C.c_int32, C.c_char_p, P(C.c_void_p)]
    lib.cubics_task_queue_open.restype = C.c_int
    lib.cubics_task_queue_reset.argtypes = [C.c_void_p]
    lib.cubics_task_queue_reset.restype = C.c_int
    lib.cubics_task_queue_claims.argtypes = [C.c_void_p, P(C.c_uint64)]
    lib.cubics_task_queue_claims.restype = C.c_int
    lib.cubics_task_queue_destroy.argtypes = [C.c_void_p]
    lib.cubics_task_queue_destroy.restype = C.c_int
    lib.cubics_solve_first_shard.argtypes = [C.c_void_p, P(SearchConfig), C.c_int32, C.c_int32, C.c_void_p,
                                             P(C.c_void_p), P(Result)]
    lib.cubics_solve_first_shard.restype = C.c_int
    lib.cubics_first_shard_best.argtypes = [C.c_void_p, P(C.c_uint32), P(C.c_int32), P(C.c_int64), P(C.c_int32)]
    lib.cubics_first_shard_best.restype = C.c_int
    lib.cubics_first_shard_prefix.argtypes = [C.c_void_p, P(C.c_uint32), C.c_int32, P(Stats)]
    lib.cubics_first_shard_prefix.restype = C.c_int
    lib.cubics_solve_multi.argtypes = [C.c_void_p, P(SearchConfig), C.c_int32, P(C.c_int32), SOLUTION_CB, C.c_void_p,
                                       P(C.c_int64), P(Result)]
    lib.cubics_solve_multi.restype = C.c_int
    lib.cubics_first_shard_free.argtypes = [C.c_void_p]
    lib.cubics_first_shard_free.restype = None
    lib.cubics_propagate.argtypes = [C.c_void_p, P(C.c_uint64), C.c_int32, C.c_int32, P(FixpointResult)]
    lib.cubics_propagate.restype = C.c_int
    lib.cubics_removals.argtypes = [C.c_void_p, P(C.c_uint64), C.c_int32, P(C.c_int32), C.c_int32, P(C.c_uint64)]
    lib.cubics_removals.restype = C.c_int
    lib.cubics_last_error.argtypes = []
    lib.cubics_last_error.restype = C.c_char_p
    lib.cubics_build_info.argtypes = []
    lib.cubics_build_info.restype = C.c_char_p
    lib.cubics_device_count.argtypes = []
    lib.cubics_device_count.restype = C.c_int
    lib.cubics_warmup.argtypes = [C.c_int32]
    lib.cubics_warmup.restype = C.c_int
    return lib
