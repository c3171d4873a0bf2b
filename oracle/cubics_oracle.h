/*
 * cubics_oracle.h - TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference solver's hot path (/root/reference/proj/src:
 * propagation.cpp, state.cpp, search.cpp, domain.cpp), used as the parity checker for the
 * CUDA engine. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * it. It is pinned against the reference itself: tests/golden/*.json were produced by the
 * unmodified reference (oracle/_ref/fdref_driver) and tests/test_oracle.py checks this port
 * against every one of them.
 *
 * It consumes the same flat model description as the product ABI (include/cubics.h).
 */
#ifndef CUBICS_ORACLE_H
#define CUBICS_ORACLE_H

#include "cubics.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Same contracts as cubics_solve_satisfy / cubics_solve_optimize, computed by the
 * reference's single-threaded DFS (search.cpp:56-201). Return a cubics_status. */
int oracle_solve_satisfy(const cubics_model_desc* d, const cubics_search_config* cfg,
                         cubics_solution_cb cb, void* user, cubics_result* out);
int oracle_solve_optimize(const cubics_model_desc* d, const cubics_search_config* cfg,
                          int64_t* best_values, cubics_result* out);

/* Same contract as cubics_propagate. */
int oracle_propagate(const cubics_model_desc* d, uint64_t* words, int32_t alldiff,
                     int32_t max_rounds, cubics_fixpoint_result* out);

/* Same contract as cubics_removals. */
int oracle_removals(const cubics_model_desc* d, const uint64_t* words, int32_t alldiff,
                    const int32_t* cons, int32_t n_cons, uint64_t* removed);

#ifdef __cplusplus
}
#endif
#endif
