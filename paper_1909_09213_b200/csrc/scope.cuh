// Execution scopes of one search context.
//
// BlockScope: the context is one thread block (the parity engine on small/medium models, every
//             context of the parallel engine). Barriers are __syncthreads.
// GridScope:  the context is the whole GPU (cooperative launch, every SM): the north star's
//             grid-wide context for models whose domains and constraint tables exceed shared
//             memory (10k-100k variables). Domains live in L2/HBM; a phase boundary is a grid
//             barrier followed by a gpu-scope fence (ptxas emits CCTL.IVALL for it, so no SM keeps
//             stale L1 lines of domains another SM rewrote); block-level votes and reductions go
//             through rotating global slots, so each costs one grid barrier.
#pragma once

#include <cooperative_groups.h>

#include <cstdint>

namespace cubics {
namespace dev {

// control scalars broadcast from thread 0 (shared memory for a block, global for the grid)
struct Ctl {
    uint4 hot; // warp contexts: the prefetched HotState (cp.async target)
    int err, min, flag, src;
    long long ll;
    int xs_want, pad; // thread 0: some GPU asked for a subtree (cross-GPU stealing)
    uint4 xs;         // warp contexts: {push, pop, work, demand} of the pool, prefetched by cp.async
    // thread 0's work-sharing counters (the debug line / busy fraction): kept here, not in
    // registers, so the search loop has 8 more registers under the 64-register cap
    long long idle_cyc, steals, donations, t_start;
    unsigned red[32];
};

struct BlockScope {
    static constexpr bool kGrid = false;
    static constexpr bool kWarp = false;
    __device__ __forceinline__ int tid() const { return threadIdx.x; }
    __device__ __forceinline__ int nthreads() const { return blockDim.x; }
    __device__ __forceinline__ int warp() const { return threadIdx.x >> 5; }
    __device__ __forceinline__ int nwarps() const { return blockDim.x >> 5; }
    __device__ __forceinline__ void sync() { __syncthreads(); }
    __device__ __forceinline__ int sync_or(int x) { return __syncthreads_or(x); }
    // block-wide min; red: 32 words of shared memory
    __device__ __forceinline__ unsigned min_u32(unsigned v, unsigned* red) {
        v = __reduce_min_sync(0xffffffffu, v);
        if (blockDim.x > 32) {
            if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
            __syncthreads();
            const unsigned x = (threadIdx.x & 31) < (blockDim.x >> 5) ? red[threadIdx.x & 31] : 0xffffffffu;
            v = __reduce_min_sync(0xffffffffu, x);
            __syncthreads();
        }
        return v;
    }
};

// WarpScope: the context is one warp of a block that may hold several (search_kernel_warp, small
// models: n <= 32 variables of <= 32 values). Barriers are __syncwarp, votes are warp votes, and
// the fixpoint keeps each variable's domain in its lane's register (warp_ctx.cuh).
struct WarpScope {
    static constexpr bool kGrid = false;
    static constexpr bool kWarp = true;
    __device__ __forceinline__ int tid() const { return threadIdx.x & 31; }
    __device__ __forceinline__ int nthreads() const { return 32; }
    __device__ __forceinline__ int warp() const { return 0; }
    __device__ __forceinline__ int nwarps() const { return 1; }
    __device__ __forceinline__ void sync() { __syncwarp(); }
    __device__ __forceinline__ int sync_or(int x) { return __any_sync(0xffffffffu, x); }
    __device__ __forceinline__ unsigned min_u32(unsigned v, unsigned*) { return __reduce_min_sync(0xffffffffu, v); }
};

struct GridScope {
    static constexpr bool kGrid = true;
    static constexpr bool kWarp = false;
    unsigned* or_slots;  // [3] rotating vote slots (zero-initialised)
    unsigned* min_slots; // [3] rotating min slots (0xffffffff-initialised)
    unsigned or_seq = 0, min_seq = 0;
    __device__ __forceinline__ int tid() const { return blockIdx.x * blockDim.x + threadIdx.x; }
    __device__ __forceinline__ int nthreads() const { return gridDim.x * blockDim.x; }
    __device__ __forceinline__ int warp() const { return tid() >> 5; }
    __device__ __forceinline__ int nwarps() const { return nthreads() >> 5; }
    __device__ __forceinline__ void sync() {
        cooperative_groups::this_grid().sync();
        __threadfence(); // drop this SM's stale L1 lines of data other SMs wrote before the barrier
    }
    // Slot s of call i is reset (by block 0) during call i+2's predecessor: every thread has read
    // slot s of call i before passing the barrier of call i+1, and nobody writes it again before
    // the barrier of call i+2.
    __device__ __forceinline__ int sync_or(int x) {
        const unsigned s = or_seq % 3;
        ++or_seq;
        const int b = __syncthreads_or(x);
        if (threadIdx.x == 0) {
            if (b) atomicOr(or_slots + s, 1u);
            if (blockIdx.x == 0) or_slots[(s + 1) % 3] = 0;
        }
        sync();
        return (int)*reinterpret_cast<volatile unsigned*>(or_slots + s);
    }
    __device__ __forceinline__ unsigned min_u32(unsigned v, unsigned* red) {
        const unsigned s = min_seq % 3;
        ++min_seq;
        v = BlockScope().min_u32(v, red);
        if (threadIdx.x == 0) {
            atomicMin(min_slots + s, v);
            if (blockIdx.x == 0) min_slots[(s + 1) % 3] = 0xffffffffu;
        }
        sync();
        return *reinterpret_cast<volatile unsigned*>(min_slots + s);
    }
};

} // namespace dev
} // namespace cubics
