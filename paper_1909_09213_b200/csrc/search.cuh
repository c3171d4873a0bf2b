// Persistent search kernel, sm_100a: the reference's Dfs::descend (search.cpp:80-132) as an
// iterative loop in one thread block per search context.
//
// * Labeling: first-fail / input-order selection is a block argmin over (popc, var id)
//   (select_variable, search.cpp:13-28); the value is the domain minimum (__ffs, :30-32).
// * Propagation: block_fixpoint (propagators.cuh) - all constraints in parallel per round.
// * Backtracking: every left branch pushes a copy of the parent's post-propagation domains
//   into a per-context decision stack in HBM (vectorised uint4 copies); the right branch
//   restores it and removes the value. This is observationally identical to SearchStore's
//   save-on-modify trail (state.cpp:12-36): both reinstate the state on entering the level.
//   At most one frame per variable is live (each left branch fixes one more variable).
// * Parallel engine: many contexts per GPU. A busy context donates its shallowest pending right
//   branch to an idle one through a lock-free ticket ring in HBM (each idle context spins on its
//   own ring slot); nodes are visited exactly once,
//   so nodes/failures/rounds/solutions of a complete enumeration are exact sums. Each subtree
//   carries its DFS path bits, the key that restores the reference's solution order.
#pragma once

#include "layout.hpp"
#include "propagators.cuh"
#include "scope.cuh"
#include "warp_ctx.cuh"

namespace cubics {
namespace dev {

__device__ __forceinline__ int ld_volatile(const int32_t* p) { return *reinterpret_cast<const volatile int32_t*>(p); }

__device__ __forceinline__ long long ld_volatile_s64(const int64_t* p) {
    return *reinterpret_cast<const volatile long long*>(p);
}

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
    return *reinterpret_cast<const volatile unsigned long long*>(p);
}

__device__ __forceinline__ void st_volatile_u64(unsigned long long* p, unsigned long long v) {
    *reinterpret_cast<volatile unsigned long long*>(p) = v;
}

// one 16-byte L1-bypassing load of {push_ticket, pop_ticket, stop, has_bound}
__device__ __forceinline__ uint4 ld_volatile_v4(const uint4* p) {
    uint4 r;
    asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ int spin_lock(int32_t* l) {
    int ns = 16, fails = 0;
    while (atomicCAS(l, 0, 1) != 0) {
        ++fails;
        __nanosleep(ns);
        ns = ns < 512 ? ns * 2 : ns;
    }
    __threadfence();
    return fails;
}

__device__ __forceinline__ void spin_unlock(int32_t* l) {
    __threadfence();
    atomicExch(l, 0);
}

// block-wide copy of nwords/4 uint4 words
__device__ __forceinline__ void copy4(uint32_t* dst, const uint32_t* src, size_t nwords, int tid, int T) {
    uint4* d = reinterpret_cast<uint4*>(dst);
    const uint4* s = reinterpret_cast<const uint4*>(src);
    for (size_t i = tid; i < nwords / 4; i += T) d[i] = s[i];
}

__device__ __forceinline__ void copy4_cg(uint32_t* dst, const uint32_t* src, size_t nwords, int tid, int T) {
    uint4* d = reinterpret_cast<uint4*>(dst);
    const uint4* s = reinterpret_cast<const uint4*>(src);
    for (size_t i = tid; i < nwords / 4; i += T) d[i] = __ldcg(s + i);
}

// Shared task queue (cubics_solve_shard_shared): claim the next seeded subtree; the counter may
// live in a peer GPU's HBM (CUDA IPC mapping), hence the system-scope atomic over NVLink.
// Out of line: it runs once per claimed subtree and must not cost the search loop registers.
static __device__ __noinline__ int claim_task(unsigned int* counter, int n_seed, int n_ctx) {
    const unsigned i = atomicAdd_system(counter, 1u);
    return i < (unsigned)n_seed ? n_ctx + (int)i : -1;
}

// Shared incumbent across GPUs: objectives as u64 whose unsigned order is "better first", so one
// system-scope atomicMin keeps the best (minimise: v ^ 2^63; maximise: ~(v ^ 2^63)).
__device__ __forceinline__ unsigned long long bound_enc(long long v, bool minimizing) {
    const unsigned long long u = (unsigned long long)v ^ 0x8000000000000000ull;
    return minimizing ? u : ~u;
}
__device__ __forceinline__ long long bound_dec(unsigned long long e, bool minimizing) {
    return (long long)((minimizing ? e : ~e) ^ 0x8000000000000000ull);
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// out of line: runs every 16 nodes per context and must not cost the search loop registers
static __device__ __noinline__ void pull_global_bound(WorkState* ws, const unsigned long long* g_inc, bool minimizing) {
    const unsigned long long e = ld_relaxed_sys_u64(g_inc);
    if (e == ~0ull) return;
    const long long v = bound_dec(e, minimizing);
    if (minimizing)
        atomicMin(reinterpret_cast<long long*>(&ws->bound), v);
    else
        atomicMax(reinterpret_cast<long long*>(&ws->bound), v);
    __threadfence();
    if (!*reinterpret_cast<volatile int32_t*>(&ws->hot.has_bound)) atomicExch(&ws->hot.has_bound, 1);
}

// Streaming delivery (cubics_solve_satisfy with a callback; emit_solution, search.cpp:134-156):
// the kernel writes events into a ring in host-mapped pinned memory while the calling thread
// drains it and runs the callback. Slot t: u64 seq = epoch<<40 | t+1 (written last, after a
// system fence; the per-call epoch keeps a reused ring's old slots from reading as new) |
// u32 kind | u32 segment | u64 stats[3] | u32 key[KW] | u16 vals[n].
//   EV_SOL  a solution: its segment and the segment-local nodes/failures/rounds at emission
//           (parity engine: segment 0 = the whole search, so the stats are the reference's)
//   EV_NEW  a subtree handed out (parallel): its segment id and root path key, published by the
//           donor BEFORE the subtree enters the ticket ring, so the host knows every segment left
//           of a finished one before that one's EV_END
//   EV_END  a segment finished: its totals
// Segments are contiguous intervals of the DFS order (a donor only hands out branches right of
// everything it still visits), so the host releases solutions in DFS order segment by segment
// and the reference's stats at any solution are the finished segments left of it plus its
// snapshot: a callback that stops gets exactly the stats of search.cpp:147-149.
__device__ __forceinline__ uint8_t* ev_slot_ptr(const SearchParams& P, long long t) {
    return P.ev_ring + (size_t)((unsigned long long)t % P.ev_cap) * P.ev_slot;
}

// thread 0: reserve the next slot, waiting while the ring is full; -1 once the search is stopped
// (the host no longer drains then). The host's consumed count is read over PCIe only when the
// cached copy says the ring is full.
static __device__ __noinline__ long long ev_reserve(const SearchParams& P) {
    WorkState* ws = P.ws;
    const unsigned long long t = atomicAdd((unsigned long long*)&ws->ev_head, 1ull);
    int ns = 64;
    for (;;) {
        unsigned long long tail = ld_volatile_u64((const unsigned long long*)&ws->ev_tail);
        if (t - tail < P.ev_cap) return (long long)t;
        tail = *reinterpret_cast<const volatile unsigned long long*>(P.ev_tail_host);
        atomicMax((unsigned long long*)&ws->ev_tail, tail);
        if (t - tail < P.ev_cap) return (long long)t;
        if (ld_volatile(&ws->hot.stop)) return -1;
        __nanosleep(ns);
        ns = ns < 8192 ? ns * 2 : ns;
    }
}

// thread 0: header, stats, system fence, then the sequence word that hands the slot to the host
// (the writers of the key / values fenced before the barrier that precedes this call)
static __device__ __noinline__ void ev_commit(const SearchParams& P, long long t, uint32_t kind, uint32_t seg,
                                              unsigned long long a, unsigned long long b, unsigned long long c) {
    uint8_t* s = ev_slot_ptr(P, t);
    volatile uint32_t* h = reinterpret_cast<volatile uint32_t*>(s + 8);
    h[0] = kind;
    h[1] = seg;
    volatile unsigned long long* st = reinterpret_cast<volatile unsigned long long*>(s + 16);
    st[0] = a;
    st[1] = b;
    st[2] = c;
    __threadfence_system();
    *reinterpret_cast<volatile unsigned long long*>(s) = ((unsigned long long)P.ev_epoch << 40) | ((unsigned long long)t + 1ull);
}

// thread 0 of a donor: EV_NEW for the subtree about to be published (key from its outbox)
static __device__ __noinline__ void ev_new_segment(const SearchParams& P, uint32_t seg, const uint32_t* key) {
    const long long t = ev_reserve(P);
    if (t < 0) return;
    uint32_t* k = reinterpret_cast<uint32_t*>(ev_slot_ptr(P, t) + kEvHeader);
    for (int i = 0; i < P.KW; ++i) k[i] = key[i];
    ev_commit(P, t, EV_NEW, seg, 0, 0, 0);
}

static __device__ __noinline__ void ev_end_segment(const SearchParams& P, uint32_t seg, unsigned long long a,
                                                   unsigned long long b, unsigned long long c) {
    const long long t = ev_reserve(P);
    if (t >= 0) ev_commit(P, t, EV_END, seg, a, b, c);
}

// ---- cross-GPU stealing (a stealer takes the shallowest untried right branch) ----
__device__ __forceinline__ int ld_relaxed_sys_s32(const int32_t* p) {
    int v;
    asm volatile("ld.relaxed.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_acquire_sys_u32(const uint32_t* p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys_u32(uint32_t* p, unsigned v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long global_ns() { // one clock for every SM
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint32_t* xs_slot_ptr(const SearchParams& P, unsigned t) {
    return reinterpret_cast<uint32_t*>(P.xs_slots + (size_t)(t % P.xs_cap) * P.xs_slot);
}

// take one unit of demand (donor) or give one back (a thief that leaves unsatisfied)
static __device__ __noinline__ bool xs_dec_demand(XsCtl* c) {
    int d = ld_relaxed_sys_s32(&c->demand);
    while (d > 0) {
        const int o = atomicCAS_system(&c->demand, d, d - 1);
        if (o == d) return true;
        d = o;
    }
    return false;
}

// thread 0 of a donor: take a unit of demand (-1: another donor was faster), then a pool ticket
// (its subtree counts as work until a thief takes it), once the slot is free. The payload goes
// straight into the slot in the owner GPU's HBM. One call site, on the donation path only, so the
// search loop keeps its registers.
static __device__ __noinline__ long long xs_reserve(const SearchParams& P) {
    if (!xs_dec_demand(P.xs_ctl)) return -1;
    atomicAdd_system(&P.xs_ctl->work, 1);
    const unsigned t = atomicAdd_system(&P.xs_ctl->push, 1u);
    uint32_t* sl = xs_slot_ptr(P, t);
    int ns = 32;
    while (ld_acquire_sys_u32(sl) != 0u) {
        __nanosleep(ns);
        ns = ns < 1024 ? ns * 2 : ns;
    }
    return (long long)t;
}

// thread 0 of a waiting context holding the thief role, when this GPU has no work left:
// 1 = a stolen subtree was republished in the local ring; 0 = nothing yet; -1 = exit (no GPU
// searches and the pool is empty, a GPU aborted, or nothing arrived for `patience` cycles; a
// thief leaves with the pool non-empty only when another thief just took from it, so the last
// GPU standing drains the pool).
static __device__ __noinline__ int xs_thief_step(const SearchParams& P, WorkState* ws, int ctx, size_t OS) {
    XsCtl* c = P.xs_ctl;
    volatile int32_t* idle = &ws->xs_idle; // serialised by the xs_thief role
    if (!*idle) { // this GPU's busy token goes back; it asks for one subtree
        *idle = 1;
        atomicSub_system(&c->work, 1);
        atomicAdd_system(&c->demand, 1);
        *reinterpret_cast<volatile long long*>(&ws->xs_since) = (long long)global_ns();
    }
    if (ld_relaxed_sys_s32(&c->abort)) {
        xs_dec_demand(c);
        return -1;
    }
    const unsigned pop = ld_acquire_sys_u32(&c->pop), push = ld_acquire_sys_u32(&c->push);
    if (pop < push && atomicCAS_system(&c->pop, pop, pop + 1u) == pop) {
        uint32_t* sl = xs_slot_ptr(P, pop);
        int ns = 32;
        while (ld_acquire_sys_u32(sl) != pop + 1u) { // the donor is still writing it
            __nanosleep(ns);
            ns = ns < 1024 ? ns * 2 : ns;
        }
        const uint32_t* src = sl + 4;
        uint32_t* ob = P.outbox + (size_t)ctx * OS;
        for (size_t i = 0; i < OS; ++i) ob[i] = __ldcv(src + i);
        st_release_sys_u32(sl, 0u); // slot free for the donor of ticket pop + xs_cap
        *idle = 0;                   // the subtree's work token is now this GPU's busy token
        atomicAdd((unsigned long long*)&ws->xs_in, 1ull);
        P.outbox_busy[ctx] = 1; // publish it locally as this context's donation
        atomicAdd(&ws->outstanding, 1);
        const uint32_t s = atomicAdd(&ws->hot.push_ticket, 1u);
        __threadfence();
        st_volatile_u64(P.ring + (s % P.ring_cap), ((unsigned long long)(s + 1u) << 32) | (unsigned)ctx);
        return 1;
    }
    const long long patience = 2000000; // 2 ms without a subtree (global timer, ns)
    if (ld_relaxed_sys_s32(&c->work) == 0 ||
        (long long)global_ns() - *reinterpret_cast<volatile long long*>(&ws->xs_since) > patience) {
        xs_dec_demand(c);
        return -1;
    }
    return 0;
}

// Thread 0 of an idle context in a sharded search: the next subtree (outbox index, or -1 when the
// search is over). Shared queue first (a claiming context stays outstanding), then a ticket of the
// in-GPU ring; when this GPU has no work left, one waiting context at a time is the thief of
// cross-GPU stealing. Out of line: the sharded kernels' search loop keeps its registers (the lean
// kernels inline their plain ticket wait).
struct WaitOut {
    int got;
    int claim_open;
    long long seg; // segment id of the subtree
};
static __device__ __noinline__ WaitOut wait_sharded(const SearchParams& P, WorkState* ws, int ctx, size_t OS,
                                                    int claim_open, bool xs) {
    int got = claim_open ? claim_task(P.task_claim, P.n_seed, P.n_ctx) : -1;
    if (got >= 0) return WaitOut{got, 1, (long long)(got - P.n_ctx) + 1}; // claimed seed i: segment 1 + i
    atomicSub(&ws->outstanding, 1);
    const uint32_t t = atomicAdd(&ws->hot.pop_ticket, 1u);
    const unsigned long long* slot = P.ring + (t % P.ring_cap);
    int ns = 32;
    for (int it = 0;; ++it) {
        const unsigned long long v = ld_volatile_u64(slot);
        if ((uint32_t)(v >> 32) == t + 1u) {
            got = (int)(v & 0xffffffffu);
            break;
        }
        if ((it & 7) == 7) {
            if (ld_volatile(&ws->hot.stop) || ld_volatile(&ws->xs_done)) break;
            if (ld_volatile(&ws->outstanding) == 0) { // this GPU has no work left
                if (!xs || !P.xs_ctl) break;
                if (atomicCAS(&ws->xs_thief, 0, 1) == 0) { // steal from another GPU
                    // re-check under the role: the previous holder may have just republished a
                    // stolen subtree (this GPU is busy again then)
                    __threadfence();
                    int xr = 0;
                    if (ld_volatile(&ws->outstanding) == 0 && !ld_volatile(&ws->xs_done)) xr = xs_thief_step(P, ws, ctx, OS);
                    if (xr < 0) atomicExch(&ws->xs_done, 1);
                    __threadfence();
                    atomicExch(&ws->xs_thief, 0);
                    if (xr < 0) break;
                }
            }
        }
        __nanosleep(ns);
        ns = ns < 1024 ? ns * 2 : ns;
    }
    if (got >= 0) __threadfence();
    return WaitOut{got, 0, (long long)t + 1 + P.seg_base}; // the subtree published under ticket t
}

__device__ __forceinline__ unsigned long long key_prefix64(uint32_t w0, uint32_t w1) {
    return ((unsigned long long)w0 << 32) | w1;
}

// DFS path key: decision at depth d is bit (31 - d%32) of word d/32, so comparing the words as
// unsigned integers, most significant first, is the reference's DFS (preorder) order.
// path_right_word: word i of the key of the right child taken at depth d (prefix [0,d) kept,
// bit d set, deeper bits cleared).
__device__ __forceinline__ uint32_t path_right_word(uint32_t word, int i, int d) {
    const int c = d - i * 32; // prefix bits of this word that are kept
    uint32_t keep = c <= 0 ? 0u : (c >= 32 ? 0xffffffffu : ~(0xffffffffu >> c));
    uint32_t x = word & keep;
    if (c >= 0 && c < 32) x |= 0x80000000u >> c;
    return x;
}

// A busy context's shallowest pending right branch (frame fr, meta {var, bit, depth}) into the
// global pool, all threads of the context; false when the demand was already taken. Out of line:
// it runs once per subtree given away, and the search loop keeps its registers.
template <int W, class SC>
static __device__ __noinline__ bool xs_donate(const SearchParams& P, SC& sc, const uint32_t* fr, const int32_t* meta,
                                              const uint32_t* path, int KW, size_t NWP, long long& s_ll, int tid, int T) {
    if (tid == 0) s_ll = xs_reserve(P);
    sc.sync();
    const long long xt = s_ll;
    if (xt < 0) return false;
    const int fvar = meta[0], fbit = meta[1], fdepth = meta[2];
    uint32_t* ob = xs_slot_ptr(P, (unsigned)xt) + 4;
    const size_t clr = (size_t)fvar * W + (fbit >> 5);
    for (size_t i = tid; i < NWP; i += T) {
        uint32_t x = fr[i];
        if (i == clr) x &= ~(1u << (fbit & 31));
        ob[i] = x;
    }
    for (int i = tid; i < KW; i += T) ob[NWP + i] = path_right_word(path[i], i, fdepth);
    if (tid == 0) {
        ob[NWP + KW] = (uint32_t)(fdepth + 1);
        ob[NWP + KW + 1] = (uint32_t)fvar;
    }
    __threadfence_system();
    sc.sync();
    if (tid == 0) {
        st_release_sys_u32(xs_slot_ptr(P, (unsigned)xt), (unsigned)xt + 1u);
        atomicAdd((unsigned long long*)&P.ws->xs_out, 1ull);
    }
    return true;
}

// block argmin of (size, id) over unbound vars; -1 when every domain is a singleton
template <int W, class SC>
__device__ __forceinline__ int select_var(const DevModel& M, const uint32_t* dom, int first_fail, unsigned* red, SC& sc) {
    const int tid = sc.tid(), T = sc.nthreads();
    unsigned best = 0xffffffffu;
    for (int v = tid; v < M.n; v += T) {
        const int sz = dom_size_n<W>(dom + (size_t)v * W, vwords<W>(M, v));
        if (sz > 1) {
            const unsigned key = first_fail ? ((unsigned)sz << 21) | (unsigned)v : (unsigned)v;
            best = key < best ? key : best;
        }
    }
    best = sc.min_u32(best, red);
    return best == 0xffffffffu ? -1 : (int)(best & 0x1fffffu);
}

template <int W, int F, class SC>
__device__ __forceinline__ void search_body(const SearchParams& P, SC& sc, Ctl& C, unsigned* red, uint8_t* smem) {
    static_assert(!SC::kWarp || W == 1, "warp contexts hold one-word domains");
    int& s_err = C.err;
    int& s_min = C.min;
    int& s_flag = C.flag;
    int& s_src = C.src;
    long long& s_ll = C.ll;

    const DevModel& M = P.M;
    // a warp context is warp (threadIdx.x >> 5) of its block; bt/bT index its private shared memory
    const int ctx = SC::kGrid ? 0
                    : (SC::kWarp ? (int)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) : (int)blockIdx.x);
    const int tid = sc.tid(), T = sc.nthreads(), nw = sc.nwarps();
    const int bt = SC::kWarp ? (int)(threadIdx.x & 31) : (int)threadIdx.x, bT = SC::kWarp ? 32 : (int)blockDim.x;
    const bool parallel = (F & F_PARITY) == 0 && P.mode == MODE_PARALLEL;
    const int n = M.n;
    const size_t NW = (size_t)n * W, NWP = round4(NW);
    const int KW = P.KW;
    // shared memory is per block: its layout follows the block's warps, not the scope's
    const SmemLayout L = smem_layout(W, n, M.total_members, SC::kWarp ? 1 : (int)(blockDim.x >> 5), KW, P.dom_in_smem, M.na,
                                     P.frames_in_smem ? P.frame_cap : 0);
    if (SC::kWarp) smem += (size_t)(threadIdx.x >> 5) * ((L.total + 15) & ~size_t(15));
    uint32_t* dom = P.dom_in_smem ? reinterpret_cast<uint32_t*>(smem + L.dom) : P.gdom + (size_t)ctx * 2 * NWP;
    uint32_t* rm = P.dom_in_smem ? reinterpret_cast<uint32_t*>(smem + L.rm) : dom + NWP;
    int16_t* mates = reinterpret_cast<int16_t*>(smem + L.mates);
    uint32_t* path = reinterpret_cast<uint32_t*>(smem + L.path);
    uint32_t* bestkey = reinterpret_cast<uint32_t*>(smem + L.bestkey);
    uint32_t* post = L.has_post ? reinterpret_cast<uint32_t*>(smem + L.post) : nullptr;
    int8_t* post_ok = reinterpret_cast<int8_t*>(smem + L.post_ok);
    // the grid context keeps its trigger bitmaps in global memory (every block reads them)
    uint32_t* chg0 = SC::kGrid ? P.grid_chg : (L.has_chg ? reinterpret_cast<uint32_t*>(smem + L.chg) : nullptr);
    uint32_t* chg1 = chg0 ? chg0 + ((n + 31) >> 5) : nullptr;
    const int nbw = (n + 31) >> 5;
    RoundCtx R{dom,     rm,      mates,     post,
               post_ok, chg0,    chg1,      chg0 != nullptr,
               P.big_scratch ? P.big_scratch + (SC::kGrid ? 0 : (size_t)ctx * nw * M.big_words) : nullptr,
               smem + L.scratch, L.stride, nullptr, P.alldiff, P.exact_wipe};
    bool first_all = true; // the root's first round evaluates every propagator
    bool skip_node = false; // first mode: the task just taken lies right of the best solution
    int trig_var = -1;     // var changed by the branch that created the current node
    uint32_t* frames = P.frames_in_smem ? reinterpret_cast<uint32_t*>(smem + L.frames) : P.frames + (size_t)ctx * P.frame_cap * NWP;
    int32_t* meta = P.frames_in_smem ? reinterpret_cast<int32_t*>(smem + L.meta) : P.frame_meta + (size_t)ctx * P.frame_cap * 4;
    WorkState* ws = P.ws;
    const size_t OS = NWP + round4((size_t)KW + 2); // outbox: domains | path key | depth | branch var

    for (size_t i = tid; i < NWP; i += T) rm[i] = 0;
    // block-private shared memory is initialised with block-local indices
    for (int i = bt; i < M.total_members; i += bT) mates[i] = -1;
    if (L.has_post)
        for (int i = bt; i < M.na; i += bT) post_ok[i] = 0;
    for (int i = bt; i < KW; i += bT) {
        path[i] = 0;
        bestkey[i] = 0xffffffffu;
    }
    if (tid == 0) s_err = 0;
    if (SC::kGrid) sc.sync();

    unsigned long long nodes = 0, failures = 0, rounds = 0, sols = 0;
    int sp = 0, base = 0, depth = 0;
    const bool batch = (F & F_PARITY) != 0 && !SC::kWarp && P.batch != 0; // parity block kernels only
    // lean warp kernels compile out branch-and-bound and the frontier expansion / shared claims
    constexpr bool kOpt = (F & F_NOOPT) == 0, kSplit = (F & F_NOSPLIT) == 0;
#ifdef CUBICS_XS_OFF
    constexpr bool kXs = false; // A/B builds only
#else
    constexpr bool kXs = kSplit; // cross-GPU stealing rides on the sharded kernels
#endif
    // block kernels keep the frontier expansion; warp kernels only in F_FRONTIER instantiations
    constexpr bool kFrontier = kSplit && (!SC::kWarp || (F & F_FRONTIER) != 0);
    bool has_bound = batch ? P.batch_has_bound[ctx] != 0 : P.has_init_bound != 0;
    long long bound = batch ? P.batch_bound[ctx] : P.init_bound;
    bool has_first = false;
    const bool optimizing = kOpt && M.goal != 0, minimizing = M.goal == 1;
    const int obj = M.goal_var;
    // thread 0's view of the shared coordination state (parallel engine)
    // warp contexts prefetch it with cp.async into shared memory (no registers held across the
    // fixpoint); block contexts into registers
    uint4 hot_reg = make_uint4(0, 0, 0, 0);
    uint4& hot = SC::kWarp ? C.hot : hot_reg;
    if (SC::kWarp && tid == 0) hot = hot_reg;
    long long g_bound = P.init_bound;
    int g_has_bound = P.has_init_bound;
    int my_busy = 0;

    // sharded kernels keep thread 0's work-sharing counters in shared memory (registers are what
    // their search loop runs short of); the lean kernels keep them in registers
    struct { long long idle_cyc, steals, donations, t_start; } lc{0, 0, 0, 0};
    long long& idle_cyc = kSplit ? C.idle_cyc : lc.idle_cyc;
    long long& steals = kSplit ? C.steals : lc.steals;
    long long& donations = kSplit ? C.donations : lc.donations;
    long long& t_start = kSplit ? C.t_start : lc.t_start;
    if (tid == 0) idle_cyc = steals = donations = 0;
    int& xs_want = C.xs_want; // thread 0: some GPU waits for a subtree (refreshed every 16 nodes)
    if (tid == 0) xs_want = 0;
    if (kXs && P.xs_ctl && ctx == 0 && tid == 0) atomicAdd_system(&P.xs_ctl->work, 1); // this GPU searches
    if (tid == 0) t_start = clock64();
    // first mode: current segment and the counters at its start; thread 0 caches the best key
    // segment bookkeeping (F_FIRST kernels, P.first_mode != 0): every subtree handed out records
    // its root key and stats, solutions their segment-local snapshots. first_mode (== 1) also
    // abandons subtrees right of the best solution found; 2 = bookkeeping only (the frontier
    // expansion of a sharded first-solution search, whose task set must not depend on timing)
    const bool seg_book = (F & F_FIRST) != 0 && (F & F_PARITY) == 0 && P.first_mode != 0; // compile-time off in lean kernels
    const bool first_mode = seg_book && P.first_mode == 1;
    // guided replay of a recorded path (exact parallel B&B, reference-order kernels only)
    const bool guided = (F & F_PARITY) != 0 && P.guide_key != nullptr;
    // streaming delivery: compiled into the reference-order kernels and the parallel kernels
    // with segment bookkeeping (F_FIRST); the lean parallel kernels never stream
    const bool stream = (F & (F_FIRST | F_PARITY)) != 0 && P.stream != 0;
    long long seg = (!parallel || ctx == 0) && !P.n_seed ? 0 : -1;
    unsigned long long seg_n0 = 0, seg_f0 = 0, seg_r0 = 0;
    int gbest_idx = -1;
    auto flush_seg = [&]() {
        if (seg_book && tid == 0 && seg >= 0 && seg < P.seg_cap) {
            P.seg_stats[seg * 3 + 0] = nodes - seg_n0;
            P.seg_stats[seg * 3 + 1] = failures - seg_f0;
            P.seg_stats[seg * 3 + 2] = rounds - seg_r0;
        }
        if (stream && tid == 0 && seg >= 0) {
            ev_end_segment(P, (uint32_t)seg, nodes - seg_n0, failures - seg_f0, rounds - seg_r0);
            seg = -1; // once per segment (thread 0 is the only reader of seg in stream mode)
        }
    };
    // first mode: is the current path key right of the best solution key (thread 0 only)?
    // (sharded: or is its 64-bit prefix above the best any GPU found)
    auto right_of_best = [&]() -> bool {
        if (P.g_first && key_prefix64(path[0], KW > 1 ? path[1] : 0u) > ld_relaxed_sys_u64(P.g_first)) return true;
        const int bi = (int)hot.w;
        if (bi < 0) return false;
        if (bi != gbest_idx) {
            gbest_idx = bi;
            for (int i = 0; i < KW; ++i) bestkey[i] = __ldcg(P.sol_keys + (size_t)bi * KW + i);
        }
        for (int i = 0; i < KW; ++i)
            if (path[i] != bestkey[i]) return path[i] > bestkey[i];
        return false;
    };
    // first mode: is the right branch taken at depth d (key: path prefix, bit d) right of the best?
    auto frame_right_of_best = [&](int d) -> bool {
        if (P.g_first && key_prefix64(path_right_word(path[0], 0, d), KW > 1 ? path_right_word(path[1], 1, d) : 0u) >
                             ld_relaxed_sys_u64(P.g_first))
            return true;
        const int bi = (int)hot.w;
        if (bi < 0) return false;
        if (bi != gbest_idx) {
            gbest_idx = bi;
            for (int i = 0; i < KW; ++i) bestkey[i] = __ldcg(P.sol_keys + (size_t)bi * KW + i);
        }
        for (int i = 0; i < KW; ++i) {
            const uint32_t k = path_right_word(path[i], i, d);
            if (k != bestkey[i]) return k > bestkey[i];
        }
        return false;
    };

    // Idle: take a ticket and wait for the task published under it (lock-free ticket queue:
    // each waiter spins on its own ring slot, so there is no shared hot spot to contend on).
    bool claim_open = kSplit && P.task_claim != nullptr; // thread 0: shared queue not yet drained
    auto get_work = [&]() -> bool {
        if (tid == 0) {
            const long long t0 = clock64();
            int got = -1;
            if constexpr (kSplit) {
                const WaitOut w = wait_sharded(P, ws, ctx, OS, claim_open ? 1 : 0, kXs);
                claim_open = w.claim_open != 0;
                s_ll = w.seg;
                got = w.got;
            } else {
                atomicSub(&ws->outstanding, 1);
                const uint32_t t = atomicAdd(&ws->hot.pop_ticket, 1u);
                const unsigned long long* slot = P.ring + (t % P.ring_cap);
                int ns = 32;
                for (int it = 0;; ++it) {
                    const unsigned long long v = ld_volatile_u64(slot);
                    if ((uint32_t)(v >> 32) == t + 1u) {
                        got = (int)(v & 0xffffffffu);
                        break;
                    }
                    if ((it & 7) == 7 && (ld_volatile(&ws->hot.stop) || ld_volatile(&ws->outstanding) == 0)) break;
                    __nanosleep(ns);
                    ns = ns < 1024 ? ns * 2 : ns;
                }
                if (got >= 0) __threadfence();
                s_ll = (long long)t + 1 + P.seg_base; // segment id of the subtree published under ticket t
            }
            if (got >= 0) ++steals;
            idle_cyc += clock64() - t0;
            s_src = got;
        }
        sc.sync();
        const int got = s_src;
        if (got < 0) return false;
        seg = s_ll;
        seg_n0 = nodes;
        seg_f0 = failures;
        seg_r0 = rounds;
        const uint32_t* ob = P.outbox + (size_t)got * OS;
        copy4_cg(dom, ob, NWP, tid, T);
        for (int i = tid; i < KW; i += T) path[i] = __ldcg(ob + NWP + i);
        depth = (int)__ldcg(ob + NWP + KW);
        const int tvar = (int)__ldcg(ob + NWP + KW + 1);
        if (chg0)
            for (int i = tid; i < 2 * nbw; i += T) chg0[i] = 0;
        sc.sync();
        if (tid == 0) {
            if (chg0) chg0[tvar >> 5] |= 1u << (tvar & 31);
            __threadfence();
            atomicExch(&P.outbox_busy[got], 0);
        }
        sp = base = 0;
        first_all = false;
        trig_var = tvar;
        if (seg_book && seg < P.seg_cap)
            for (int i = tid; i < KW; i += T) P.seg_key[(size_t)seg * KW + i] = path[i];
        if (first_mode) {
            if (tid == 0) {
                hot = ld_volatile_v4(reinterpret_cast<const uint4*>(&ws->hot));
                s_flag = right_of_best(); // the whole subtree lies right of a known solution
            }
            sc.sync();
            if (s_flag) {
                flush_seg();
                skip_node = true; // zero nodes: the main loop's backtrack takes the next task
            }
        }
        return true;
    };

    bool have_work;
    if (!parallel || (ctx == 0 && !P.n_seed)) {
        copy4(dom, batch ? P.batch_dom + (size_t)ctx * NWP : M.init_dom, NWP, tid, T);
        have_work = true;
    } else {
        have_work = get_work();
    }
    sc.sync();

    while (have_work) {
        bool backtrack = false;
        if (skip_node) {
            skip_node = false;
            backtrack = true;
        } else if (kFrontier && P.split_depth >= 0 && depth >= P.split_depth) {
            // ============ frontier expansion: this open node becomes a task (counted by its shard)
            if (tid == 0) s_ll = (long long)atomicAdd((unsigned long long*)&ws->n_tasks, 1ull);
            sc.sync();
            const long long t = s_ll;
            if (t < P.task_cap) {
                uint32_t* tb = P.tasks + (size_t)t * OS;
                copy4(tb, dom, NWP, tid, T);
                for (int i = tid; i < KW; i += T) tb[NWP + i] = path[i];
                if (tid == 0) {
                    tb[NWP + KW] = (uint32_t)depth;
                    tb[NWP + KW + 1] = (uint32_t)trig_var;
                    if (seg_book) { // where the task sits in the frontier's DFS: segment + snapshot
                        uint64_t* ts = P.task_snap + (size_t)t * 4;
                        ts[0] = (unsigned long long)seg;
                        ts[1] = nodes - seg_n0;
                        ts[2] = failures - seg_f0;
                        ts[3] = rounds - seg_r0;
                    }
                }
            }
            backtrack = true;
        } else {
        // ================= node entry (descend, search.cpp:80-111)
        ++nodes;
        if (P.node_limit && nodes > P.node_limit) {
            if (tid == 0) {
                if (batch) { // per-problem flag: the other problems keep searching
                    P.batch_flags[ctx] |= 1;
                } else {
                    ws->limit_hit = 1;
                    ws->hot.stop = 1;
                }
            }
            break;
        }
        if (stream && !parallel && (nodes & 1023) == 0) { // has a callback stopped the stream?
            if (tid == 0) s_flag = ld_volatile(&ws->hot.stop);
            sc.sync();
            const int stp = s_flag;
            sc.sync();
            if (stp) {
                if (tid == 0) ws->user_stop = 1;
                break;
            }
        }
        if (parallel && tid == 0) { // prefetch; consumed after the fixpoint
            if constexpr (SC::kWarp)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(&C.hot)),
                             "l"(&ws->hot)
                             : "memory");
            else
                hot = ld_volatile_v4(reinterpret_cast<const uint4*>(&ws->hot));
            if (optimizing) {
                // other GPUs' incumbents: merged into this launch's bound every 16 nodes
                if (kSplit && P.g_inc && (nodes & 15) == 1) pull_global_bound(ws, P.g_inc, minimizing);
                g_bound = ld_volatile_s64(&ws->bound);
            }
            my_busy = ld_volatile(&P.outbox_busy[ctx]);
            if (kXs && P.xs_ctl && (nodes & 15) == 2) { // every 16 nodes: does a GPU ask for work?
                if constexpr (SC::kWarp) // asynchronous, consumed after the fixpoint with the hot word
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(&C.xs)),
                                 "l"(P.xs_ctl)
                                 : "memory");
                else
                    xs_want = ld_relaxed_sys_s32(&P.xs_ctl->demand) > 0;
            }
        }
        if (optimizing) { // branch-and-bound shrink (:87-101), done by thread 0
            if (tid == 0) {
                int empty = 0;
                // guided replay: the bound the reference had when it entered this node; a static
                // bound (exact B&B phase): the phase's; parallel: the shared incumbent
                const bool shared_b = parallel && !P.static_bound;
                const long long bnd = guided ? P.guide_bound[depth] : (shared_b ? g_bound : bound);
                const bool hb = guided ? P.guide_has[depth] != 0 : (shared_b ? g_has_bound != 0 : has_bound);
                if (hb) {
                    uint32_t* d = dom + (size_t)obj * W;
                    const long long off = M.off[obj];
                    const int lo = dom_first<W>(d), hi = dom_last<W>(d);
                    const bool shrink = minimizing ? (off + hi >= bnd) : (off + lo <= bnd);
                    if (shrink) {
                        // minimise: remove_above(bound-1) ; maximise: remove_below(bound+1)
                        const long long cut = clampbit((i128)bnd - off, W * 32);
                        uint32_t any = 0;
#pragma unroll
                        for (int w = 0; w < W; ++w) {
                            uint32_t m = minimizing ? range_word(w, cut, W * 32) : range_word(w, -1, cut);
                            d[w] &= ~m;
                            any |= d[w];
                        }
                        empty = any == 0;
                        if (chg0) chg0[obj >> 5] |= 1u << (obj & 31);
                    }
                }
                s_flag = empty;
            }
            sc.sync();
            backtrack = s_flag != 0;
            if (backtrack) ++failures;
        }
        if (!backtrack) {
            int r = 0;
            int st;
            if constexpr (SC::kWarp && W == 1)
                st = warp_fixpoint<F>(M, R, &r, first_all, chg0 ? chg0[0] : 0u, tid);
            else
                st = block_fixpoint<W, F>(M, R, &s_err, &s_min, 0, &r, nullptr, first_all, sc);
            first_all = false;
            rounds += (unsigned long long)r;
            if (st == R_ERROR) {
                if (tid == 0) {
                    ws->error = DERR_OVERFLOW;
                    ws->hot.stop = 1;
                }
                break;
            }
            if (st == R_FAILED) {
                ++failures;
                backtrack = true;
            }
        }
        if constexpr (SC::kWarp)
            if (parallel && tid == 0) asm volatile("cp.async.wait_all;" ::: "memory");
        if (parallel && tid == 0) g_has_bound = (int)hot.w; // the prefetched bound pairs with this flag
        if constexpr (SC::kWarp && kXs)
            if (parallel && tid == 0 && P.xs_ctl && (nodes & 15) == 2) xs_want = (int)C.xs.w > 0;
        if (!backtrack) {
            const int sel = select_var<W>(M, dom, P.var_heuristic, red, sc);
            if (sel < 0 && guided) break; // the replay reached its solution: every task is out
            if (sel < 0) {
                // ============ solution leaf (emit_solution, search.cpp:134-156)
                if (tid == 0) {
                    if (stream) // an event slot in the host-mapped ring
                        s_ll = ev_reserve(P);
                    else if (first_mode) // only a solution left of the best known one can matter
                        s_ll = right_of_best() ? -1 : (long long)atomicAdd((unsigned long long*)&ws->sol_count, 1ull);
                    else
                        s_ll = parallel ? (long long)atomicAdd((unsigned long long*)&ws->sol_count, 1ull) : (long long)sols;
                    if (parallel) atomicMax(&ws->max_depth, depth);
                }
                sc.sync();
                const long long sidx = s_ll;
                const unsigned long long idx = (unsigned long long)sidx;
                ++sols;
                if (stream && sidx >= 0) {
                    uint8_t* es = ev_slot_ptr(P, sidx);
                    uint32_t* ek = reinterpret_cast<uint32_t*>(es + kEvHeader);
                    uint16_t* ev = reinterpret_cast<uint16_t*>(es + kEvHeader + 4 * KW);
                    for (int v = tid; v < n; v += T) ev[v] = (uint16_t)dom_first<W>(dom + (size_t)v * W);
                    for (int i = tid; i < KW; i += T) ek[i] = path[i];
                    __threadfence_system();
                    sc.sync();
                    if (tid == 0)
                        ev_commit(P, sidx, EV_SOL, (uint32_t)(seg < 0 ? 0 : seg), nodes - seg_n0, failures - seg_f0,
                                  rounds - seg_r0);
                } else if (P.record && sidx >= 0 && idx < P.sol_cap) {
                    for (int v = tid; v < n; v += T) P.sol_vals[idx * n + v] = (uint16_t)dom_first<W>(dom + (size_t)v * W);
                    for (int i = tid; i < KW; i += T) P.sol_keys[idx * KW + i] = path[i];
                    if (tid == 0 && (!parallel || seg_book)) { // parity: global; segments: segment-local
                        P.sol_stats[idx * 3 + 0] = nodes - seg_n0;
                        P.sol_stats[idx * 3 + 1] = failures - seg_f0;
                        P.sol_stats[idx * 3 + 2] = rounds - seg_r0;
                        if (seg_book) P.sol_seg[idx] = (int32_t)seg;
                    }
                }
                if (first_mode) {
                    sc.sync();
                    if (tid == 0 && sidx >= 0 && idx < P.sol_cap) { // publish as the best if still the best
                        __threadfence();
                        spin_lock(&ws->best_lock);
                        volatile int32_t* gb = &ws->hot.has_bound;
                        const int cur = *gb;
                        bool better = cur < 0;
                        for (int i = 0; i < KW && !better; ++i) {
                            const uint32_t a = path[i], b = __ldcg(P.sol_keys + (size_t)cur * KW + i);
                            if (a != b) {
                                better = a < b;
                                break;
                            }
                        }
                        if (better) *gb = (int32_t)idx;
                        spin_unlock(&ws->best_lock);
                        if (better && P.g_first) atomicMin_system(P.g_first, key_prefix64(path[0], KW > 1 ? path[1] : 0u));
                    }
                    // everything this context would visit next lies right of this solution
                    sp = base;
                }
                if (parallel && KW > 0 && !first_mode) { // per-context DFS-first solution
                    if (tid == 0) {
                        int less = 0;
                        for (int i = 0; i < KW; ++i)
                            if (path[i] != bestkey[i]) {
                                less = path[i] < bestkey[i];
                                break;
                            }
                        s_flag = less || !has_first;
                    }
                    sc.sync();
                    if (s_flag) {
                        has_first = true;
                        for (int i = tid; i < KW; i += T) {
                            bestkey[i] = path[i];
                            P.ctx_first_key[(size_t)ctx * KW + i] = path[i];
                        }
                        for (int v = tid; v < n; v += T)
                            P.ctx_first_vals[(size_t)ctx * n + v] = (uint16_t)dom_first<W>(dom + (size_t)v * W);
                        if (tid == 0) P.ctx_has_first[ctx] = 1;
                    }
                }
                if (optimizing) {
                    const long long val = M.off[obj] + dom_first<W>(dom + (size_t)obj * W);
                    if (!P.static_bound) { // an exact B&B phase keeps its bound until it stops
                        has_bound = true;
                        bound = val;
                    }
                    if (batch) {
                        for (int v = tid; v < n; v += T)
                            P.batch_inc[(size_t)ctx * n + v] = (uint16_t)dom_first<W>(dom + (size_t)v * W);
                        if (tid == 0) P.batch_flags[ctx] |= 2;
                    }
                    if (parallel && !P.static_bound && tid == 0) {
                        spin_lock(&ws->inc_lock);
                        volatile long long* gb = reinterpret_cast<volatile long long*>(&ws->bound);
                        volatile int32_t* ghb = &ws->hot.has_bound;
                        if (!*ghb || (minimizing ? val < *gb : val > *gb)) {
                            for (int v = 0; v < n; ++v) P.inc_vals[v] = (uint16_t)dom_first<W>(dom + (size_t)v * W);
                            ws->inc_found = 1;
                            // atomic: a concurrent pull of another GPU's better bound must win
                            if (minimizing)
                                atomicMin(reinterpret_cast<long long*>(&ws->bound), val);
                            else
                                atomicMax(reinterpret_cast<long long*>(&ws->bound), val);
                            __threadfence();
                            *ghb = 1;
                            if (kSplit && P.g_inc) atomicMin_system(P.g_inc, bound_enc(val, minimizing));
                        }
                        spin_unlock(&ws->inc_lock);
                        g_bound = *gb; // our own incumbent is visible to us at once
                        g_has_bound = 1;
                    }
                }
                if (stream && !parallel && tid == 0) s_flag = ld_volatile(&ws->hot.stop);
                sc.sync();
                if (!parallel && (sols >= P.max_solutions || (stream && s_flag))) {
                    if (tid == 0) {
                        ws->user_stop = 1;
                        ws->hot.stop = 1;
                    }
                    break;
                }
                backtrack = true;
            } else if (guided) {
                // ============ replay one decision of the recorded path (bit `depth` of its key):
                // left = the reference went left here and its right branch is still pending when
                // it reaches the solution: emit that branch as a task (outbox layout)
                const int bit = dom_first<W>(dom + (size_t)sel * W);
                const int gbit = (int)((P.guide_key[depth >> 5] >> (31 - (depth & 31))) & 1u);
                if (!gbit) {
                    if (tid == 0) s_ll = (long long)atomicAdd((unsigned long long*)&ws->n_tasks, 1ull);
                    sc.sync();
                    const long long t = s_ll;
                    if (t < P.task_cap) {
                        uint32_t* tb = P.tasks + (size_t)t * OS;
                        const size_t clr = (size_t)sel * W + (bit >> 5);
                        for (size_t i = tid; i < NWP; i += T) {
                            uint32_t x = dom[i];
                            if (i == clr) x &= ~(1u << (bit & 31));
                            tb[i] = x;
                        }
                        for (int i = tid; i < KW; i += T) tb[NWP + i] = path_right_word(path[i], i, depth);
                        if (tid == 0) {
                            tb[NWP + KW] = (uint32_t)(depth + 1);
                            tb[NWP + KW + 1] = (uint32_t)sel;
                        }
                    }
                }
                if (chg0)
                    for (int i = tid; i < 2 * nbw; i += T) chg0[i] = 0;
                sc.sync();
                if (!gbit) {
                    if (tid < W) dom[(size_t)sel * W + tid] = (tid == (bit >> 5)) ? (1u << (bit & 31)) : 0u;
                } else if (tid == 0) { // the reference took the right branch here
                    dom[(size_t)sel * W + (bit >> 5)] &= ~(1u << (bit & 31));
                    for (int i = depth >> 5; i < KW; ++i) path[i] = path_right_word(path[i], i, depth);
                }
                if (tid == 0 && chg0) chg0[sel >> 5] |= 1u << (sel & 31);
                trig_var = sel;
                ++depth;
                sc.sync();
                continue;
            } else {
                // ============ left branch: push the frame, assign x = min(x) (:116-121)
                if (sp >= P.frame_cap) {
                    if (tid == 0) {
                        ws->error = DERR_CAPACITY;
                        ws->hot.stop = 1;
                    }
                    break;
                }
                const int bit = dom_first<W>(dom + (size_t)sel * W);
                if (SC::kWarp && P.frames_in_smem)
                    copy4_shared(frames + (size_t)sp * NWP, dom, NWP, tid);
                else
                    copy4(frames + (size_t)sp * NWP, dom, NWP, tid, T);
                if (chg0)
                    for (int i = tid; i < 2 * nbw; i += T) chg0[i] = 0;
                if (tid == 0) {
                    meta[sp * 4 + 0] = sel;
                    meta[sp * 4 + 1] = bit;
                    meta[sp * 4 + 2] = depth;
                    // donate the shallowest pending right branch when someone waits for work
                    int want = hot.z ? 2 : 0;
                    // a whole GPU is idle: the shallowest pending branch goes to the global pool
                    // first (one subtree per unit it asked for; local sharing resumes after)
                    if (kXs && xs_want && parallel && !want && sp + 1 > base) { // one unit: xs_reserve
                        xs_want = 0;
                        want = 4;
                    }
                    if (parallel && !want && sp + 1 > base && !my_busy && hot.y > hot.x) want = 1;
                    // first mode: pending branches right of the best solution are dropped, never
                    // handed out (the shallowest pending branch is the rightmost one)
                    if (first_mode && want == 1 && frame_right_of_best(meta[base * 4 + 2])) want = 3;
                    s_flag = want;
                }
                sc.sync();
                if (tid < W) dom[(size_t)sel * W + tid] = (tid == (bit >> 5)) ? (1u << (bit & 31)) : 0u;
                if (tid == 0 && chg0) chg0[sel >> 5] |= 1u << (sel & 31);
                trig_var = sel;
                ++sp;
                ++depth;
                const int want = s_flag;
                if (want == 2) break;
                if (want == 3) ++base;
                if (kXs && want == 4) { // out of line: a slot in the owner GPU's HBM, if the demand holds
                    if (xs_donate<W>(P, sc, frames + (size_t)base * NWP, meta + base * 4, path, KW, NWP, s_ll, tid, T))
                        ++base;
                } else if (want == 1) {
                    const int f = base++;
                    const int fvar = meta[f * 4 + 0], fbit = meta[f * 4 + 1], fdepth = meta[f * 4 + 2];
                    uint32_t* ob = P.outbox + (size_t)ctx * OS;
                    const uint32_t* fr = frames + (size_t)f * NWP;
                    const size_t clr = (size_t)fvar * W + (fbit >> 5);
                    for (size_t i = tid; i < NWP; i += T) {
                        uint32_t x = fr[i];
                        if (i == clr) x &= ~(1u << (fbit & 31));
                        ob[i] = x;
                    }
                    for (int i = tid; i < KW; i += T) ob[NWP + i] = path_right_word(path[i], i, fdepth);
                    if (tid == 0) {
                        ob[NWP + KW] = (uint32_t)(fdepth + 1);
                        ob[NWP + KW + 1] = (uint32_t)fvar;
                    }
                    sc.sync();
                    if (tid == 0) {
                        P.outbox_busy[ctx] = 1;
                        atomicAdd(&ws->outstanding, 1);
                        const uint32_t s = atomicAdd(&ws->hot.push_ticket, 1u);
                        if (stream) ev_new_segment(P, s + 1u + (uint32_t)P.seg_base, ob + NWP); // known to the host first
                        __threadfence();
                        st_volatile_u64(P.ring + (s % P.ring_cap), ((unsigned long long)(s + 1u) << 32) | (unsigned)ctx);
                        ++donations;
                    }
                }
                sc.sync();
                continue;
            }
        }
        } // node processing
        if (guided) { // a failure on the recorded path: the replay does not match the search
            if (tid == 0) ws->error = DERR_GUIDE;
            break;
        }
        // ================= backtrack: right branch of the deepest pending frame (:122-131)
        if (parallel) {
            if (tid == 0) s_flag = hot.z;
            sc.sync();
            if (s_flag) break;
        }
        if (sp == base) {
            if (!parallel) break;
            flush_seg();
            have_work = get_work();
            sc.sync();
            continue;
        }
        --sp;
        if (SC::kWarp && P.frames_in_smem)
            copy4_shared(dom, frames + (size_t)sp * NWP, NWP, tid);
        else
            copy4(dom, frames + (size_t)sp * NWP, NWP, tid, T);
        if (chg0)
            for (int i = tid; i < 2 * nbw; i += T) chg0[i] = 0;
        const int var = meta[sp * 4 + 0], bit = meta[sp * 4 + 1], d = meta[sp * 4 + 2];
        sc.sync();
        if (tid == 0) {
            dom[(size_t)var * W + (bit >> 5)] &= ~(1u << (bit & 31));
            if (chg0) chg0[var >> 5] |= 1u << (var & 31);
            if (KW > 0) { // path: bit d = 1, everything deeper cleared
                const int last = depth < KW * 32 ? depth : KW * 32 - 1;
                for (int i = d >> 5; i <= (last >> 5); ++i) path[i] = path_right_word(path[i], i, d);
            }
            if (first_mode) s_flag = right_of_best(); // this branch and all pending ones lie right of it
        }
        depth = d + 1;
        trig_var = var;
        sc.sync();
        if (first_mode && s_flag) {
            sp = base;
            skip_node = true;
        }
    }
    flush_seg();
    sc.sync();
    // a GPU that stops (error) releases the others from waiting for its work
    if (kXs && P.xs_ctl && tid == 0 && ld_volatile(&ws->hot.stop)) atomicExch_system(&P.xs_ctl->abort, 1);
    if (parallel && tid == 0 && have_work) {
        // unwound by stop: this context no longer counts as outstanding
        atomicSub(&ws->outstanding, 1);
    }
    if (tid == 0) {
        const long long total = clock64() - t_start;
        atomicAdd((unsigned long long*)&ws->busy_cycles, (unsigned long long)(total - idle_cyc));
        atomicAdd((unsigned long long*)&ws->idle_cycles, (unsigned long long)idle_cyc);
        atomicAdd((unsigned long long*)&ws->steals, (unsigned long long)steals);
        atomicAdd((unsigned long long*)&ws->donations, (unsigned long long)donations);
        if (batch) {
            P.batch_stats[(size_t)ctx * 4 + 0] = nodes;
            P.batch_stats[(size_t)ctx * 4 + 1] = failures;
            P.batch_stats[(size_t)ctx * 4 + 2] = rounds;
            P.batch_stats[(size_t)ctx * 4 + 3] = sols;
        }
        atomicAdd((unsigned long long*)&ws->stats[0], nodes);
        atomicAdd((unsigned long long*)&ws->stats[1], failures);
        atomicAdd((unsigned long long*)&ws->stats[2], rounds);
        atomicAdd((unsigned long long*)&ws->stats[3], sols);
    }
}

template <int W, int F>
__global__ void __launch_bounds__(1024) search_kernel(const SearchParams P) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ Ctl C;
    __shared__ unsigned red[32];
    BlockScope sc;
    search_body<W, F>(P, sc, C, red, smem);
}

// small models (n <= 32, W = 1; warp_ctx.cuh): one search context per warp, blockDim.x / 32
// contexts per block, each with its own slice of the dynamic shared memory
#ifndef CUBICS_WARP_MINB
#define CUBICS_WARP_MINB 16 // 16 x 64 threads per SM: 64 registers
#endif
template <int F>
__global__ void __launch_bounds__(64, CUBICS_WARP_MINB) search_kernel_warp(const SearchParams P) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ Ctl C[2];
    WarpScope sc;
    search_body<1, F>(P, sc, C[threadIdx.x >> 5], nullptr, smem);
}

// one search context spanning the GPU (cooperative launch); see scope.cuh
template <int W>
__global__ void __launch_bounds__(1024) search_kernel_grid(const SearchParams P) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ unsigned red[32];
    GridScope sc{P.grid_or, P.grid_min};
    search_body<W, F_ALL | F_PARITY>(P, sc, *P.grid_ctl, red, smem);
}

// the parity engine and batched B&B: one block per problem, reference node order; no parallel
// work sharing compiled in, and up to 128 registers per thread (<= 512 threads)
template <int W>
__global__ void __launch_bounds__(512, 1) search_kernel_parity(const SearchParams P) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ Ctl C;
    __shared__ unsigned red[32];
    BlockScope sc;
    search_body<W, F_ALL | F_PARITY | F_REGS>(P, sc, C, red, smem);
}

// cubics_propagate / cubics_removals: one block over caller-provided domains
template <int W>
__global__ void __launch_bounds__(1024) propagate_kernel(const PropParams P, uint32_t* gscratch, int dom_in_smem) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ int s_err, s_min;
    BlockScope sc;
    const DevModel& M = P.M;
    const int tid = threadIdx.x, T = blockDim.x, nw = T >> 5;
    const size_t NW = (size_t)M.n * W, NWP = round4(NW);
    const SmemLayout L = smem_layout(W, M.n, M.total_members, nw, 0, dom_in_smem, M.na);
    uint32_t* dom = dom_in_smem ? reinterpret_cast<uint32_t*>(smem + L.dom) : gscratch;
    uint32_t* rm = dom_in_smem ? reinterpret_cast<uint32_t*>(smem + L.rm) : gscratch + NWP;
    int16_t* mates = reinterpret_cast<int16_t*>(smem + L.mates);
    uint32_t* chg0 = L.has_chg ? reinterpret_cast<uint32_t*>(smem + L.chg) : nullptr;
    RoundCtx R{dom, rm, mates, nullptr, nullptr, chg0, L.has_chg ? chg0 + ((M.n + 31) >> 5) : nullptr, false,
               P.big_scratch, smem + L.scratch, L.stride, P.enabled, P.alldiff, 1};
    for (size_t i = tid; i < NWP; i += T) {
        dom[i] = P.dom[i];
        rm[i] = 0;
    }
    for (int i = tid; i < M.total_members; i += T) mates[i] = -1;
    if (tid == 0) s_err = 0;
    __syncthreads();
    if (P.removals_only) {
        run_propagators<W, F_ALL>(M, R, &s_err, nullptr, sc);
        __syncthreads();
        for (size_t i = tid; i < NWP; i += T) P.out[i] = rm[i] & dom[i];
        if (tid == 0) P.result[4] = s_err;
        return;
    }
    int rounds = 0, fv = -1;
    const int st = block_fixpoint<W, F_ALL>(M, R, &s_err, &s_min, P.max_rounds, &rounds, &fv, true, sc);
    for (size_t i = tid; i < NWP; i += T) P.dom[i] = dom[i];
    if (tid == 0) {
        P.result[0] = st == R_FAILED;
        P.result[1] = st == R_FAILED ? fv : -1;
        P.result[2] = rounds;
        P.result[3] = st == R_ERROR ? 0 : st;
        P.result[4] = s_err;
    }
}

// cubics_propagate / cubics_removals for large models: one fixpoint spanning the GPU
// (cooperative launch). Domains and removals live in L2/HBM (gscratch); every warp of the grid
// takes propagators, so hundreds of alldifferents run side by side instead of a few per block.
template <int W>
__global__ void __launch_bounds__(1024) propagate_kernel_grid(const PropParams P, uint32_t* gscratch) {
    extern __shared__ __align__(16) uint8_t smem[];
    GridScope sc{P.grid_or, P.grid_min};
    Ctl& C = *P.grid_ctl;
    const DevModel& M = P.M;
    const int tid = sc.tid(), T = sc.nthreads();
    const size_t NW = (size_t)M.n * W, NWP = round4(NW);
    const SmemLayout L = smem_layout(W, M.n, M.total_members, (int)(blockDim.x >> 5), 0, false, M.na);
    uint32_t* dom = gscratch;
    uint32_t* rm = gscratch + NWP;
    int16_t* mates = reinterpret_cast<int16_t*>(smem + L.mates);
    uint32_t* chg0 = P.grid_chg;
    RoundCtx R{dom, rm, mates, nullptr, nullptr, chg0, chg0 + ((M.n + 31) >> 5), false,
               P.big_scratch, smem + L.scratch, L.stride, P.enabled, P.alldiff, 1};
    for (size_t i = tid; i < NWP; i += T) {
        dom[i] = P.dom[i];
        rm[i] = 0;
    }
    for (int i = threadIdx.x; i < M.total_members; i += blockDim.x) mates[i] = -1;
    if (tid == 0) C.err = 0;
    sc.sync();
    if (P.removals_only) {
        run_propagators<W, F_ALL>(M, R, &C.err, nullptr, sc);
        sc.sync();
        for (size_t i = tid; i < NWP; i += T) P.out[i] = rm[i] & dom[i];
        if (tid == 0) P.result[4] = C.err;
        return;
    }
    int rounds = 0, fv = -1;
    const int st = block_fixpoint<W, F_ALL>(M, R, &C.err, &C.min, P.max_rounds, &rounds, &fv, true, sc);
    for (size_t i = tid; i < NWP; i += T) P.dom[i] = dom[i];
    if (tid == 0) {
        P.result[0] = st == R_FAILED;
        P.result[1] = st == R_FAILED ? fv : -1;
        P.result[2] = rounds;
        P.result[3] = st == R_ERROR ? 0 : st;
        P.result[4] = C.err;
    }
}

} // namespace dev
} // namespace cubics
