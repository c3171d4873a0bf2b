/*
 * cubics.h - C ABI of the B200-native CUBICS search engine (libcubics.so).
 *
 * This is the drop-in boundary for the reference solver's hot path: depth-first labeling,
 * propagation to a fixpoint and backtracking. Nothing here uses C++ or torch types: plain
 * integers, pointers and sizes, so any FFI (ctypes, cgo, JNI, N-API) can bind it.
 * The C++ adapter in adapter/fd_b200.cpp implements the reference's own C++ API
 * (proj/include/fd/search.hpp, propagation.hpp) on top of these entry points; see
 * INTEGRATION.md for how a maintainer links it.
 *
 * Reference interface each entry point replaces (paths relative to /root/reference/proj):
 *   cubics_solve_satisfy       fd::solve_satisfy        include/fd/search.hpp:62, src/search.cpp:174-177
 *                              fd::enumerate_solutions  include/fd/search.hpp:65-66, src/search.cpp:179-189
 *   cubics_solve_optimize      fd::solve_optimize       include/fd/search.hpp:77, src/search.cpp:191-201
 *   cubics_solve_optimize_batch  fd::lns_optimize's neighbourhood loop  src/search.cpp:250-295
 *   cubics_propagate           fd::propagate_fixpoint   include/fd/propagation.hpp:114-118, src/propagation.cpp:516-532
 *                              fd::propagate_round      include/fd/propagation.hpp:102-104 (max_rounds = 1)
 *   cubics_removals            fd::run_batch / fd::propagate_one / fd::prop_*
 *                                                       include/fd/propagation.hpp:78-89
 *   cubics_model_parse         fd::parse_model          include/fd/parser.hpp:38 (host-side loader)
 *   cubics_model_validate      fd::model_validate       include/fd/model.hpp:93
 *   cubics_enumerate           fd::enumerate_solutions  include/fd/search.hpp:65-66 (one host array)
 *   cubics_solve_shard         (new) one rank's share of a multi-GPU search; SURVEY.md 8(e)
 *   cubics_solve_shard_shared  (new) the same, subtrees claimed dynamically from a shared
 *   cubics_task_queue_*              queue over NVLink peer memory, with cross-GPU stealing
 *   cubics_solve_optimize_shard (new) multi-GPU branch and bound, incumbent shared over NVLink
 *   cubics_solve_first_shard   (new) multi-GPU exact first solution (two-phase merge)
 *   cubics_solve_multi         (new) multi-GPU search driven from one host process
 *
 * Threading: every call is synchronous and blocks until the device finishes. Calls on
 * different models may run from different host threads. Error details for the last failing
 * call on the calling thread are in cubics_last_error().
 */
#ifndef CUBICS_H
#define CUBICS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CUBICS_ABI_VERSION 1

/* ---- status codes (no exception ever crosses the ABI) ---------------------------------- */
enum cubics_status {
    CUBICS_OK = 0,
    CUBICS_E_INVALID = 1,      /* bad argument or malformed model description                 */
    CUBICS_E_PARSE = 2,        /* model text rejected; details in cubics_parse_error            */
    CUBICS_E_OVERFLOW = 3,     /* fd::ArithmeticOverflowError (src/propagation.cpp:198-210)     */
    CUBICS_E_NO_OBJECTIVE = 4, /* std::logic_error: optimize without a goal (search.cpp:192)    */
    CUBICS_E_CUDA = 5,         /* CUDA runtime failure or no usable sm_100 device               */
    CUBICS_E_CAPACITY = 6,     /* device decision stack / solution buffer capacity exceeded     */
    CUBICS_E_UNSUPPORTED = 7   /* instance outside the device engine's limits   */
};

/* ---- model vocabulary, numerically identical to the reference enums --------------------- */
enum cubics_kind { CUBICS_RELBIN = 0, CUBICS_LINEAR = 1, CUBICS_ALLDIFF = 2, /* fd::ConstraintKind */
                   CUBICS_TABLE = 3 /* extension: positive extensional constraint (allowed tuples) */ };
enum cubics_relop { CUBICS_LT = 0, CUBICS_LE, CUBICS_GT, CUBICS_GE, CUBICS_EQ, CUBICS_NE }; /* fd::RelOp */
enum cubics_linop { CUBICS_LIN_LE = 0, CUBICS_LIN_EQ = 1 };                    /* fd::LinOp */
enum cubics_goal { CUBICS_SATISFY = 0, CUBICS_MINIMIZE = 1, CUBICS_MAXIMIZE = 2 }; /* fd::Goal */
enum cubics_var_heuristic { CUBICS_INPUT_ORDER = 0, CUBICS_FIRST_FAIL = 1 };   /* fd::VarHeuristic */
enum cubics_alldiff { CUBICS_FORWARD_CHECKING = 0, CUBICS_ARC_CONSISTENT = 1 }; /* fd::AlldiffLevel */

#define CUBICS_MAX_WIDTH 1024 /* fd::Domain::kMaxWidth (include/fd/domain.hpp:27) */

/*
 * Flat description of an fd::Model (include/fd/model.hpp:67-74).
 * Domains: var v covers [var_offset[v], var_offset[v] + var_width[v]); its bitset is
 *   ceil(width/64) little-endian u64 words (bit i = value offset+i, fd::Domain::words()),
 *   packed back to back in var order. var_words == NULL means every domain is full.
 * Constraints: constraint c owns terms [con_start[c], con_start[c+1]).
 *   RELBIN : terms = {lhs} (x op literal) or {lhs, rhs_var} (x op y + k); con_op = relop;
 *            con_value = rhs_value (the literal, or k).               (model.hpp:26-32)
 *   LINEAR : terms = (term_coeff, term_var) pairs; con_op = linop; con_value = bound. (:42-46)
 *   ALLDIFF: terms = member vars; con_op and con_value ignored.        (:48-50)
 *   TABLE  : terms = scope vars (k); con_value = number of allowed tuples t; the tuples are
 *            t*k int64 values at table_data[con_value_offset...]: tuple i of constraint c is
 *            table_data[table_start[c] + i*k .. + k). Extension beyond the reference (whose
 *            Constraint variant has no table kind, model.hpp:52): BASELINE config 5.
 * term_coeff may be NULL when there is no LINEAR constraint; table_start / table_data may be
 * NULL when there is no TABLE constraint.
 */
typedef struct cubics_model_desc {
    int32_t n_vars;
    const int64_t* var_offset;
    const int32_t* var_width;
    const uint64_t* var_words;
    int32_t n_cons;
    const int32_t* con_kind;
    const int32_t* con_op;
    const int64_t* con_value;
    const int32_t* con_start; /* n_cons + 1 entries */
    const int32_t* term_var;
    const int64_t* term_coeff;
    int32_t goal;     /* enum cubics_goal */
    int32_t goal_var; /* objective variable when goal != SATISFY */
    const int64_t* table_start; /* n_cons entries (used for TABLE constraints only) */
    const int64_t* table_data;
} cubics_model_desc;

typedef struct cubics_model cubics_model; /* opaque, host-side */

typedef struct cubics_parse_error { /* fd::ParseError (include/fd/parser.hpp:13-30) */
    int32_t kind; /* 0 Syntax, 1 UnknownVariable, 2 DuplicateVariable, 3 EmptyDomain,
                     4 DomainTooWide, 5 MissingSolveItem */
    int32_t line;
    int32_t column;
    char message[256];
} cubics_parse_error;

typedef struct cubics_diagnostic { /* fd::Diagnostic (include/fd/model.hpp:76-90) */
    int32_t kind; /* same order as fd::Diagnostic::Kind */
    int32_t constraint_index;
} cubics_diagnostic;

int cubics_model_create(const cubics_model_desc* desc, cubics_model** out);
int cubics_model_parse(const char* text, size_t len, cubics_model** out, cubics_parse_error* err);
void cubics_model_free(cubics_model* m);
/* Pointers in *out stay valid for the model's lifetime. */
int cubics_model_describe(const cubics_model* m, cubics_model_desc* out);
const char* cubics_model_var_name(const cubics_model* m, int32_t var);
/* Writes up to cap diagnostics; *count receives the total (0 = valid). */
int cubics_model_validate(const cubics_model* m, cubics_diagnostic* out, int32_t cap, int32_t* count);

/* ---- search ------------------------------------------------------------------------------ */
enum cubics_engine {
    CUBICS_ENGINE_AUTO = 0,     /* PARALLEL for complete enumerations, else PARITY              */
    CUBICS_ENGINE_PARITY = 1,   /* one device search context, reference node order: every stat
                                   identical to the CPU reference                              */
    CUBICS_ENGINE_PARALLEL = 2, /* many search contexts per GPU with work sharing: solutions and
                                   all stats exact for complete enumerations and for the first
                                   solution; optimum exact for branch-and-bound (node counts
                                   then schedule-dependent)                                     */
    CUBICS_ENGINE_GRID = 3      /* PARITY semantics with one search context spanning the whole GPU
                                   (cooperative launch): for models of 10k-100k+ variables.
                                   AUTO picks it for large parity searches                      */
};

typedef struct cubics_search_config { /* fd::SearchConfig (include/fd/search.hpp:19-27) + engine */
    int32_t var_heuristic;   /* enum cubics_var_heuristic, default FIRST_FAIL */
    int32_t value_heuristic; /* 0 = MinValue (the only one)                 */
    uint64_t max_solutions;  /* UINT64_MAX = unbounded (reference default)   */
    int32_t thread_count;    /* accepted for API parity; no effect on the device engine */
    uint64_t seed;           /* accepted for API parity; the DFS never reads it          */
    int32_t alldiff;         /* enum cubics_alldiff, default ARC_CONSISTENT  */
    uint64_t node_limit;     /* 0 = unbounded                                */
    /* engine extension */
    int32_t engine;          /* enum cubics_engine                           */
    int32_t device;          /* CUDA ordinal, -1 = current device            */
    int32_t contexts;        /* PARALLEL: search contexts (0 = auto)         */
    int32_t block_threads;   /* threads per search context (0 = auto)        */
    int32_t count_only;      /* 1 = do not materialise solutions (callback not called) */
    int32_t has_initial_bound; /* branch and bound starts from this objective bound      */
    int64_t initial_bound;     /* (Dfs::set_initial_bound, search.cpp:63,282)             */
} cubics_search_config;

void cubics_search_config_init(cubics_search_config* cfg); /* reference defaults */

typedef struct cubics_stats { /* fd::SearchStats (include/fd/state.hpp:18-23) */
    uint64_t nodes;
    uint64_t failures;
    uint64_t rounds;
    uint64_t solutions;
} cubics_stats;

typedef struct cubics_result {
    cubics_stats stats;
    int32_t complete;      /* SatisfyResult.complete / OptimizeResult.complete */
    int32_t has_solution;  /* >= 1 solution (satisfy) or an incumbent (optimize) */
    int64_t objective;     /* best objective when optimizing and has_solution */
    int32_t engine;        /* engine actually used */
    int32_t contexts;      /* search contexts actually launched */
    double device_ms;      /* search kernel time (CUDA events) */
    double total_ms;       /* wall time of the whole call: upload + search + download */
    uint64_t h2d_bytes;    /* bytes copied host -> device by this call */
    uint64_t d2h_bytes;    /* bytes copied device -> host by this call */
    uint64_t kernel_launches; /* CUDA kernels this call launched */
    uint64_t remote_tasks_in;  /* shared queue: subtrees this GPU took from other GPUs' donations */
    uint64_t remote_tasks_out; /* shared queue: subtrees this GPU gave to idle GPUs */
} cubics_result;

/* Receives each solution (values indexed by var id, as fd::Solution::values) in the
 * reference's DFS order, on the calling thread, WHILE the device search runs (search.cpp:134-156):
 * the kernel streams solutions through a ring in host-mapped pinned memory; the parallel engine's
 * subtree segments put them back into DFS order. Return 0 to stop the stream: the device search
 * stops at once and the result carries the reference's stats at that solution (search.cpp:147-149).
 * The callback must not start another search on the same device (CUBICS_E_INVALID). */
typedef int32_t (*cubics_solution_cb)(void* user, const int64_t* values, int32_t n_vars);

/* AUTO engine: complete enumerations and first-k searches (max_solutions = k, no node limit)
 * run on the parallel engine; the first k are streamed in DFS order and the search stops at the
 * k-th with the reference's stats. */
int cubics_solve_satisfy(const cubics_model* m, const cubics_search_config* cfg,
                         cubics_solution_cb cb, void* user, cubics_result* out);

/* fd::enumerate_solutions (search.hpp:65-66) in one call: every solution, in the reference's DFS
 * order, as one row-major int64 array (count x n_vars) owned by the library; free it with
 * cubics_solutions_free. No per-solution callback crosses the ABI. */
typedef struct cubics_solutions {
    uint64_t count;
    int32_t n_vars;
    int64_t* values;
} cubics_solutions;
int cubics_enumerate(const cubics_model* m, const cubics_search_config* cfg, cubics_solutions** out_solutions,
                     cubics_result* out);
void cubics_solutions_free(cubics_solutions* s);

/* best_values (n_vars entries, may be NULL) receives the optimal / last incumbent.
 * AUTO without node_limit / max_solutions: the exact parallel branch and bound - a chain of
 * static-bound exact-first searches, each seeded by a replay of the previous incumbent's path -
 * whose stats and incumbents are the reference's (search.cpp:87-101, 187-201). Otherwise, or
 * with CUBICS_ENGINE_PARITY, one reference-order search context; CUBICS_ENGINE_PARALLEL: a
 * shared-bound parallel B&B (exact optimum, schedule-dependent node count). */
int cubics_solve_optimize(const cubics_model* m, const cubics_search_config* cfg,
                          int64_t* best_values, cubics_result* out);

/* Many independent branch-and-bound searches of one model in ONE device launch (one thread block
 * per problem, the reference's node order in each): the neighbourhoods of one fd::lns_optimize
 * iteration (src/search.cpp:250-295, neighborhood_model :207-217, Dfs::set_initial_bound :282).
 * Problem i starts from the domains words + i * W (desc packing of this model, W = its total
 * 64-bit word count) and, when has_bounds == NULL ? bounds != NULL : has_bounds[i], the strict
 * initial bound bounds[i]; cfg->node_limit applies to each problem. results[i] receives problem
 * i's stats, complete, has_solution and objective (device_ms / transfers are the whole launch's);
 * best_values (count * n_vars, may be NULL) its last incumbent. */
int cubics_solve_optimize_batch(const cubics_model* m, const cubics_search_config* cfg, int32_t count,
                                const uint64_t* words, const int64_t* bounds, const int32_t* has_bounds,
                                int64_t* best_values, cubics_result* results);

/* One rank's share of a multi-GPU search: the search tree is expanded
 * deterministically to a frontier of open subtrees; this call searches every subtree t with
 * t % shard_count == shard_index (nodes above the frontier are counted by shard 0 only) and
 * returns partial stats that sum exactly across shards. Solutions reach cb with their
 * 64-bit-word DFS rank key (key_words words, lexicographic = reference DFS order). */
typedef int32_t (*cubics_keyed_solution_cb)(void* user, const uint32_t* key, int32_t key_words,
                                            const int64_t* values, int32_t n_vars);
int cubics_solve_shard(const cubics_model* m, const cubics_search_config* cfg,
                       int32_t shard_index, int32_t shard_count,
                       cubics_keyed_solution_cb cb, void* user, cubics_result* out);

/* Dynamic cross-GPU balancing: a shared task queue is one claim counter in the
 * owner GPU's HBM. Rank 0 creates it and sends the CUBICS_TASK_QUEUE_HANDLE_BYTES-byte handle
 * to the other ranks (any transport; torch.distributed in distributed.py), which open it: CUDA
 * IPC maps it into their address space and the driver enables NVLink peer access.
 * cubics_solve_shard_shared then seeds EVERY frontier subtree on every rank (DFS order) and an
 * idle search context claims the next one with a system-scope atomicAdd on the counter over
 * NVLink; once the counter passes the task count the contexts fall back to the in-GPU
 * work-sharing ring. Each subtree is searched exactly once across the ranks, so stats sum
 * exactly as for cubics_solve_shard. Once the counter drains, a GPU whose contexts are all idle
 * steals: it posts a demand in the queue state, busy contexts on the other GPUs write their
 * shallowest pending right branch into a global pool there (one per demand), and the idle GPU
 * republishes it in its own work-sharing ring; remote_tasks_in / _out count them. A GPU exits
 * when no GPU searches and the pool is empty. The counter must be reset (cubics_task_queue_reset on the
 * owner, then a barrier) before every search that uses it. A queue opened in the creating
 * process is not supported by CUDA IPC: pass the creator's queue to every local call instead;
 * a call on another device of that process enables peer access to the owner's GPU first
 * (CUBICS_E_UNSUPPORTED when the two GPUs have none). */
#define CUBICS_TASK_QUEUE_HANDLE_BYTES 64
typedef struct cubics_task_queue cubics_task_queue; /* opaque */
int cubics_task_queue_create(int32_t device, cubics_task_queue** out, uint8_t* handle /* may be NULL */);
int cubics_task_queue_open(int32_t device, const uint8_t* handle, cubics_task_queue** out);
/* reset: claim counter 0 and no shared incumbent; call on the owner, then barrier, before each search */
int cubics_task_queue_reset(cubics_task_queue* q);
int cubics_task_queue_claims(cubics_task_queue* q, uint64_t* claims); /* claim attempts so far */
int cubics_task_queue_destroy(cubics_task_queue* q);
int cubics_solve_shard_shared(const cubics_model* m, const cubics_search_config* cfg,
                              int32_t shard_index, int32_t shard_count, cubics_task_queue* queue,
                              cubics_keyed_solution_cb cb, void* user, cubics_result* out);

/* Multi-GPU branch and bound (fd::solve_optimize, search.hpp:77 / search.cpp:187-201, sharded):
 * the same deterministic frontier (expanded without the bound, so every rank builds the same
 * one; solutions above it seed the bound), this rank's subtrees searched by the parallel engine,
 * and - when queue != NULL - subtrees claimed dynamically AND the incumbent objective shared
 * through the queue state: a system-scope atomicMin on an order-preserving encoding in the
 * owner's HBM, merged into every GPU's bound every 16 nodes per search context (the B&B shrink
 * of search.cpp:87-101 then prunes with the best bound of ALL GPUs). queue == NULL: static split,
 * bounds not shared. out receives this rank's partial stats (they sum across ranks), and
 * has_solution / objective / best_values this rank's best incumbent; the caller takes the best
 * over ranks (distributed.solve_distributed). The optimum is exact; node counts depend on the
 * schedule (as for the single-GPU parallel engine). */
int cubics_solve_optimize_shard(const cubics_model* m, const cubics_search_config* cfg,
                                int32_t shard_index, int32_t shard_count, cubics_task_queue* queue,
                                int64_t* best_values, cubics_result* out);

/* Multi-GPU exact first solution (fd::solve_satisfy with max_solutions == 1, search.cpp:174-186,
 * sharded). Each rank runs cubics_solve_first_shard: the same deterministic frontier (with its
 * DFS segments recorded), then its subtrees (t % shard_count == shard_index, or claimed through
 * queue when non-NULL) by the parallel engine's exact-first search. Then:
 *   1. cubics_first_shard_best: this rank's DFS-first solution key (key_words u32 words,
 *      lexicographic = reference DFS order) and values; the caller takes the minimum key K* over
 *      ranks (distributed.solve_distributed: one all-gather);
 *   2. cubics_first_shard_prefix(K*): this rank's share of the reference's stats up to K*; the
 *      shares sum (one all-reduce) to exactly the reference's nodes / failures / rounds, and
 *      solutions == 1. key == NULL (no rank found one): the complete search's share.
 * out receives this rank's raw work. */
typedef struct cubics_first_shard cubics_first_shard; /* opaque */
int cubics_solve_first_shard(const cubics_model* m, const cubics_search_config* cfg,
                             int32_t shard_index, int32_t shard_count, cubics_task_queue* queue,
                             cubics_first_shard** out_shard, cubics_result* out);
/* *key_words: in = capacity of key (words), out = the key's length; *has = 0 when none */
int cubics_first_shard_best(const cubics_first_shard* s, uint32_t* key, int32_t* key_words,
                            int64_t* values, int32_t* has);
int cubics_first_shard_prefix(const cubics_first_shard* s, const uint32_t* key, int32_t key_words,
                              cubics_stats* out);
void cubics_first_shard_free(cubics_first_shard* s);

/* Multi-GPU search from ONE host process (a C/C++ host such as the drop-in fdsolve): one thread per
 * device runs that rank's shard (cubics_solve_shard_shared / _optimize_shard / _first_shard) with
 * the shared queue on devices[0] and peer access between the devices; the ranks' stats are summed
 * (no collective library needed inside one process). Satisfy goals: every solution goes to cb in
 * the reference's DFS order (key-merged; cb == NULL or count_only: counts only), or with
 * max_solutions == 1 the exact first solution and the reference's stats; optimize goals: the
 * optimum (best_values, and cb once). node_limit and other solution caps: CUBICS_E_UNSUPPORTED.
 * The same device may appear more than once (its ranks then run one after another). */
int cubics_solve_multi(const cubics_model* m, const cubics_search_config* cfg, int32_t n_devices,
                       const int32_t* devices, cubics_solution_cb cb, void* user, int64_t* best_values,
                       cubics_result* out);

/* ---- propagation (kernel-level API) ------------------------------------------------------ */
typedef struct cubics_fixpoint_result { /* fd::FixpointResult (propagation.hpp:106-110) */
    int32_t failed;
    int32_t failed_var; /* lowest empty var id when failed, else -1 */
    int32_t rounds;
    int32_t last_status; /* fd::RoundResult::Status of the last round: 0 Changed 1 Stable 2 Failed */
} cubics_fixpoint_result;

/* Bulk-synchronous rounds over `words` (desc packing, in/out) until Stable or Failed, or until
 * max_rounds rounds ran (max_rounds <= 0: unbounded = fd::propagate_fixpoint; 1 = one
 * fd::propagate_round). */
int cubics_propagate(const cubics_model* m, uint64_t* words, int32_t alldiff, int32_t max_rounds,
                     cubics_fixpoint_result* out);

/* Union of the removals the constraints `cons[0..n_cons)` (all constraints when cons == NULL)
 * compute against the snapshot `words`, without applying them: fd::run_batch / propagate_one.
 * removed (desc packing) receives the removal masks restricted to present values. */
int cubics_removals(const cubics_model* m, const uint64_t* words, int32_t alldiff,
                    const int32_t* cons, int32_t n_cons, uint64_t* removed);

/* ---- misc -------------------------------------------------------------------------------- */
const char* cubics_last_error(void);
const char* cubics_build_info(void);
int cubics_device_count(void);
/* Create the CUDA context on `device` (-1: current) and load the engine's kernels, so the first
 * solve does not pay for them (the reference's acceptance criterion 1 bounds that call at 1 s). */
int cubics_warmup(int32_t device);

#ifdef __cplusplus
}
#endif
#endif /* CUBICS_H */
