// Host-side model object behind the opaque cubics_model handle.
//
// Holds one flattened fd::Model (/root/reference/proj/include/fd/model.hpp:67-74): variables
// with [offset, offset+width) bitset domains (u64 words, the reference Domain layout), and the
// constraint list as kind/op/value plus a term CSR. The device layout (u32 words, per-kind
// SoA tables) is derived from this in engine.cu at upload time.
#pragma once

#include <cstdint>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "cubics.h"

namespace cubics {

struct HostModel {
    std::vector<std::string> names;
    std::vector<int64_t> offset;
    std::vector<int32_t> width;
    std::vector<int32_t> word_start; // u64 words, n+1 entries
    std::vector<uint64_t> words;
    std::vector<int32_t> con_kind, con_op, con_start{0}, term_var;
    std::vector<int64_t> con_value, term_coeff;
    std::vector<int64_t> table_start, table_data; // TABLE: tuples of constraint c at table_start[c]
    int32_t goal = CUBICS_SATISFY;
    int32_t goal_var = 0;

    int n_vars() const { return static_cast<int>(offset.size()); }
    int n_cons() const { return static_cast<int>(con_kind.size()); }
    void finish_vars(); // recompute word_start / size words after adding vars
    cubics_model_desc desc() const;
};

// fd::parse_model grammar (reference src/parser.cpp:68-493), restated.
int parse_model_text(const char* text, size_t len, HostModel& out, cubics_parse_error* err);

// Thread-local last-error message used by cubics_last_error().
void set_error(const std::string& msg);
const char* last_error();

} // namespace cubics

struct cubics_model {
    cubics::HostModel m;
    // sharded searches: the frontier split depth found for each shard count (the first of 8, 12,
    // 16, ... with enough open nodes); later calls start there instead of re-expanding from 8.
    // The result is the same depth, so every rank still builds the same frontier.
    mutable std::mutex hint_mu;
    mutable std::map<int, int> split_hint;
};

struct cubics_task_queue {
    void* counter; // device pointer in this process (owned allocation or IPC mapping)
    int device;    // device the calling process uses it from
    int owner;     // 1: cudaMalloc'd here; 0: opened from an IPC handle
};
