// Device-side model and search-state layout shared by the host orchestration (engine.cu) and
// the kernels (kernels.cuh). Plain structs of device pointers; no torch types.
//
// HBM / shared-memory layout:
//   domains  : n x W u32 words, var v at [v*W, v*W+W); bit i = value off[v] + i. W is a power of
//              two >= every domain's and every alldifferent universe's word count (u32 words).
//   RelBin   : one 16-byte record per constraint {x, y, op, s} with every 64-bit offset folded
//              on the host into a 32-bit bit offset s (model.hpp:26-32): var form x op y + k has
//              s = off[y] + k - off[x]; the literal form carries its threshold bit index in s.
//   Linear   : CSR {start[], op[], bound[]} over terms {var[], coeff[]}     (model.hpp:42-46)
//   AllDiff  : CSR over members {var[], shift[]}; shift = off[var] - universe_offset, so a
//              member's domain shifted left by `shift` bits lands in the common value universe.
#pragma once

#include <cstdint>

namespace cubics {

namespace dev {
struct Ctl;
}
using dev_ctl_t = dev::Ctl;

struct alignas(16) RelBinRec {
    int32_t x;
    int32_t y;   // -1 for the literal form
    int32_t op;  // fd::RelOp
    int32_t s;   // var form: off[y] + k - off[x]; literal form: threshold bit (see engine.cu)
};

struct DevModel {
    int32_t n;           // variables
    int32_t W;           // u32 words per domain (power of two)
    const int64_t* off;  // [n]
    const uint32_t* init_dom; // [n*W]
    const int32_t* vw;        // [n] words a variable's own width needs (<= W; bits beyond are 0)
    int32_t nr;
    const RelBinRec* rb;         // generic records first, then the var-form != records
    int32_t nr_gen;              // records [0, nr_gen) are not var-form !=
    const int32_t* ne_start;     // [n+1] var-form != incidence: when v becomes a singleton at bit b,
    const int2* ne_edge;         //   each edge (p, s) removes bit b + s from var p
    const uint32_t* ne_mask;     // [ceil(n/32)] bit v: v has var-form != edges
    const unsigned long long* neq; // [n*n] warp kernel (n <= 32, W = 1): the != edges u -> p folded
                                 //   into one mask, bit s + 32 per shift s in [-31, 31]; else null
    int32_t nl;
    const int32_t* lin_start; // [nl+1]
    const int32_t* lin_op;    // [nl]
    const int64_t* lin_bound; // [nl]
    const int32_t* lin_var;
    const int64_t* lin_coeff;
    int32_t lin_g;            // lanes per linear constraint (1: one thread each; 2..32: lane groups)
    int32_t na;
    uint32_t ad_full_mask;    // bit a (a < 32): alldifferent a's scope is every variable, so it is
                              // triggered in every round (the trigger scan is skipped)
    const int32_t* ad_start;  // [na+1]
    const int32_t* ad_var;
    const int32_t* ad_shift;
    const int32_t* ad_uw;        // [na] <= 0: fast warp path (<= 64 members), universe of -ad_uw words;
                                 //      > 0: generic path over a uw-word universe (big_words scratch)
    int32_t big_words;           // u32 words of per-warp scratch the generic path needs (0: none)
    // positive table constraints (extension, BASELINE config 5)
    int32_t ntb;                 // binary tables: bitwise arc consistency over support bitsets
    const int32_t* tb_xy;        // [2*ntb] scope (x, y)
    const int64_t* tb_off;       // [2*ntb] u32-word offsets of x's and y's support blocks in tb_sup
    const uint32_t* tb_sup;      // block of x: width_x rows of W words, row a = y bits allowed with x=a
    int32_t ntn;                 // n-ary tables (arity <= 8): tuple scan
    const int32_t* tn_start;     // [ntn+1] scope CSR
    const int32_t* tn_var;
    const int64_t* tn_nt;        // [ntn] tuples
    const int64_t* tn_off;       // [ntn] offset into tn_data
    const int16_t* tn_data;      // tuples as bit indices (-1: value outside the domain range)
    int32_t total_members;
    int32_t goal;
    int32_t goal_var;
};

enum KernelMode : int32_t { MODE_PARITY = 0, MODE_PARALLEL = 1 };

enum DeviceError : int32_t {
    DERR_NONE = 0,
    DERR_OVERFLOW = 1,
    DERR_CAPACITY = 2,
    DERR_GUIDE = 3, // a guided replay failed before its solution (internal error)
};

// Global coordination state for the parallel engine (one per launch, in HBM).
// `hot` is read by every busy context once per node (one 16-byte load, issued early and consumed
// late so its L2 latency hides behind the propagation rounds); the counters that take heavy
// atomic traffic live on other 128-byte lines.
struct alignas(16) HotState {
    uint32_t push_ticket; // tasks published into the ring
    uint32_t pop_ticket;  // idle contexts that took a ticket
    int32_t stop;         // 1 => every context unwinds (error / limit / solution cap)
    int32_t has_bound;    // branch-and-bound incumbent present (parallel)
};

struct WorkState {
    HotState hot;
    int64_t bound;        // branch-and-bound incumbent objective (parallel)
    int32_t inc_lock;
    int32_t pad0[25];     // -> 128 bytes
    int32_t outstanding;  // busy contexts + published tasks; 0 => search finished
    int32_t error;        // DeviceError
    int32_t limit_hit;
    int32_t user_stop;
    uint64_t sol_count;   // solutions recorded (parallel: atomic slot allocator)
    int32_t pad1[26];     // -> 256 bytes
    uint64_t stats[4];    // nodes, failures, rounds, solutions
    uint64_t donations;
    uint64_t steals;
    uint64_t busy_cycles;  // sum over contexts of clock64 cycles with work
    uint64_t idle_cycles;  // sum over contexts of clock64 cycles waiting for work
    uint64_t lock_fails;   // unused (kept for the debug line)
    int32_t max_depth;     // deepest solution leaf (parallel): key words that can differ
    int32_t best_lock;     // first mode: guards hot.has_bound, which then holds the best record
    int64_t n_tasks;       // frontier expansion: open nodes emitted at split_depth
    int32_t inc_found;     // parallel B&B: inc_vals holds an incumbent found by this launch
    int32_t pad2;
    uint64_t ev_head;      // streaming: event slots reserved
    uint64_t ev_tail;      // streaming: the host's consumed count as last read over PCIe
    int32_t xs_thief;      // cross-GPU stealing: a waiting context holds the thief role
    int32_t xs_idle;       // this GPU returned its busy token (all contexts idle)
    int32_t xs_done;       // global termination seen: every waiting context exits
    int32_t pad3;
    int64_t xs_since;      // clock64 when this GPU's thief started waiting (any context may hold the role)
    uint64_t xs_in;        // subtrees taken from the global pool
    uint64_t xs_out;       // subtrees given to the global pool
};

// Cross-GPU stealing control block (in the shared queue owner's HBM, system-scope atomics).
// work = GPUs still searching + subtrees in the pool; a GPU exits when it reads 0 (or abort).
struct XsCtl {
    uint32_t push;    // pool tickets handed out to donors
    uint32_t pop;     // pool tickets taken by thieves (pop <= push)
    int32_t work;
    int32_t demand;   // subtrees idle GPUs asked for that no donor has committed to yet
    int32_t abort;    // a GPU stopped (error / limit): nobody waits for work any more
    int32_t pad[3];
};

struct SearchParams {
    DevModel M;
    int32_t mode;          // KernelMode
    int32_t var_heuristic; // 0 input order, 1 first fail
    int32_t alldiff;       // 0 FC, 1 GAC
    int32_t exact_wipe;    // 1: GAC failure wipes the reference's (Kuhn-order) member
    uint64_t max_solutions;
    uint64_t node_limit;
    int32_t n_ctx;
    int32_t frame_cap;     // decision frames per context
    int32_t KW;            // u32 words of the DFS path key (parallel); 0 in parity mode
    int32_t record;        // 1: materialise solutions
    int32_t dom_in_smem;
    // per-context global scratch
    uint32_t* big_scratch; // [n_ctx * warps][M.big_words] generic alldifferent working sets
    uint32_t* frames;      // [n_ctx][frame_cap][NW]
    int32_t* frame_meta;   // [n_ctx][frame_cap][4] : var, bit, depth, pad
    uint32_t* gdom;        // [n_ctx][2*NW] when domains do not fit in shared memory
    // work sharing
    WorkState* ws;
    unsigned long long* ring; // [ring_cap] published tasks: ((ticket + 1) << 32) | donor ctx
    uint32_t ring_cap;
    int32_t* outbox_busy;  // [n_ctx]
    uint32_t* outbox;      // [n_ctx][NW + KW + 4]
    // solutions
    uint64_t sol_cap;
    uint16_t* sol_vals;    // [sol_cap][n] bit index of each var's value
    uint32_t* sol_keys;    // [sol_cap][KW]
    uint64_t* sol_stats;   // [sol_cap][3] nodes, failures, rounds at emission (parity)
    // per-context DFS-first solution (parallel, count-only friendly)
    uint32_t* ctx_first_key;  // [n_ctx][KW]
    uint16_t* ctx_first_vals; // [n_ctx][n]
    int32_t* ctx_has_first;   // [n_ctx]
    // branch-and-bound incumbent (parallel)
    uint16_t* inc_vals;       // [n]
    int64_t init_bound;
    int32_t has_init_bound;
    // frontier expansion (parity mode): open nodes at binary depth split_depth become tasks
    int32_t split_depth;      // -1: off
    int64_t task_cap;
    uint32_t* tasks;          // [task_cap][OS] same layout as an outbox slot
    // seeded parallel run: outbox slots [n_ctx, n_ctx + n_seed) hold pre-published tasks
    int32_t n_seed;
    // shared task queue (cubics_solve_shard_shared): the n_seed tasks are NOT pre-published;
    // an idle context claims seed i = atomicAdd_system(task_claim, 1) (a counter that may live
    // in a peer GPU's memory, mapped over NVLink) until i >= n_seed, then joins the ring
    unsigned int* task_claim;
    // exact parallel first solution (max_solutions == 1): every subtree handed out ("segment",
    // id = ring ticket + 1; the root is segment 0) records its root path key and its own stats;
    // solutions record their segment and segment-local stats; subtrees right of the best
    // solution key found so far are abandoned. The host then sums exactly the reference's prefix.
    // grid-wide context (search_kernel_grid): control scalars, vote/min slots, trigger bitmaps
    dev_ctl_t* grid_ctl;
    unsigned* grid_or;     // [3]
    unsigned* grid_min;    // [3]
    uint32_t* grid_chg;    // [2 * ceil(n/32)]
    // batch mode (parity engine): block c runs an independent search from its own initial domains
    // and bound (LNS neighbourhoods, cubics_solve_optimize_batch)
    int32_t batch;             // 0 off, else number of problems (= blocks)
    const uint32_t* batch_dom; // [batch][NWP]
    const int64_t* batch_bound;   // [batch] initial bounds
    const int32_t* batch_has_bound;
    uint64_t* batch_stats;     // [batch][4] nodes, failures, rounds, solutions
    int32_t* batch_flags;      // [batch] bit0 limit hit, bit1 has incumbent
    uint16_t* batch_inc;       // [batch][n] last incumbent (bit indices)
    int32_t first_mode;    // 1: exact first solution (segments + abandoning); 2: segments only
    int32_t seg_base;      // segment id of ring ticket t = t + 1 + seg_base (claimed seed i: 1 + i)
    uint64_t* task_snap;   // frontier expansion with segments: [task_cap][4] segment, nodes, failures, rounds
    int64_t seg_cap;
    uint32_t* seg_key;     // [seg_cap][KW]
    uint64_t* seg_stats;   // [seg_cap][3]
    int32_t* sol_seg;      // [sol_cap]
    int32_t frames_in_smem; // warp contexts: decision stack in the context's shared memory
    // multi-GPU branch-and-bound (cubics_solve_optimize_shard): the shared incumbent objective in
    // the queue owner's HBM (CUDA IPC, system-scope atomics over NVLink), order-preserving u64
    // encoding (see bound_enc); all ones = none. Null: single GPU.
    unsigned long long* g_inc;
    // sharded exact first solution (cubics_solve_first_shard with a queue): the first 64 path-key
    // bits of the best solution any rank found, system-scope atomicMin; a subtree whose key prefix
    // is above it lies right of that solution and is abandoned on every GPU. Null: not shared.
    unsigned long long* g_first;
    // streaming delivery (cubics_solve_satisfy with a callback): solutions, and in the parallel
    // engine the segment events that put them back into DFS order, go into a ring in host-mapped
    // pinned memory that the calling thread drains while the kernel runs (see search.cuh EvKind).
    // The host stops the search by setting ws->hot.stop from a second stream.
    // cross-GPU stealing (cubics_solve_shard_shared): a global pool of right branches in the queue
    // owner's HBM. A busy context donates its shallowest pending branch into it while some GPU's
    // thief waits; an idle GPU's thief copies one into its own outbox and republishes it in its
    // local ticket ring. Null: off.
    XsCtl* xs_ctl;
    uint8_t* xs_slots;                       // [xs_cap][xs_slot]: u32 seq (ticket + 1 when full) | pad | OS words
    uint32_t xs_cap, xs_slot;
    // exact parallel branch and bound (engine.cu exact_bnb): a phase keeps the bound it started
    // with (the reference's bound between two improving solutions); no incumbent sharing
    int32_t static_bound;
    // guided replay (reference-order kernels): follow guide_key from the root; at every left
    // decision on the path the still-pending right branch goes out as a task (outbox layout) into
    // tasks[]; the B&B shrink at depth d uses guide_bound[d] / guide_has[d], the bound the
    // reference had when it entered that node. Null: off.
    const uint32_t* guide_key;
    const int64_t* guide_bound;
    const int32_t* guide_has;
    int32_t stream;
    uint32_t ev_cap;                         // slots
    uint32_t ev_slot;                        // bytes per slot
    uint32_t ev_epoch;                       // per-call tag in the slots' sequence words
    uint8_t* ev_ring;                        // host-mapped [ev_cap][ev_slot]
    const unsigned long long* ev_tail_host;  // host-mapped: events the host has consumed
};

// streaming event kinds and slot header bytes (search.cuh ev_commit, engine.cu drain_stream)
enum EvKind : uint32_t { EV_SOL = 1, EV_NEW = 2, EV_END = 3 };
constexpr int kEvHeader = 40;

struct PropParams {
    DevModel M;
    int32_t alldiff;
    int32_t max_rounds;    // <= 0 unbounded
    int32_t removals_only; // 1: run propagators once, output rm & dom, do not apply
    const uint8_t* enabled; // per constraint kind-local enable flags [nr + nl + na] or null
    uint32_t* dom;         // [NW] in/out
    uint32_t* out;         // removals output (removals_only)
    uint32_t* big_scratch; // [warps][M.big_words]
    int32_t* result;       // failed, failed_var, rounds, last_status, error
    // grid-wide fixpoint (cooperative launch, large models): control, vote slots, triggers
    dev_ctl_t* grid_ctl;
    unsigned* grid_or;     // [3]
    unsigned* grid_min;    // [3]
    uint32_t* grid_chg;    // [2 * ceil(n/32)]
};

} // namespace cubics
