// Shared-memory layout of one search context; used by the kernels and by the host launcher.
#pragma once

#include <cstddef>
#include <cstdint>

#ifndef __CUDACC__
#define CUBICS_HD
#else
#define CUBICS_HD __host__ __device__
#endif

namespace cubics {
namespace dev {

// Compile-time propagator features of a kernel instantiation: a model without linear sums,
// tables or large alldifferents runs a kernel without that code (register pressure decides the
// occupancy of one-warp search contexts).
// F_PARITY marks a kernel that only runs the reference-order engines (parity block, batched
// B&B, grid context): the parallel engine's work sharing compiles out of it.
// F_REGS marks the 128-register parity kernel: register-hungry fast paths are compiled in only
// there (in the 64-register kernels they cost more in spills than they save).
// F_LONG: linear sums of more than 4 terms (lane-group form); lean kernels compile it out.
// F_NOOPT / F_NOSPLIT (lean warp kernels): branch-and-bound, and the shared-queue claims and
// cross-GPU stealing of sharded runs, are compiled out. F_FRONTIER: the frontier expansion of a
// sharded run (warp kernels compile it only into the instantiations that run the expansion; it
// costs the seeded search ~15% per node on nq14).
enum Feature : int {
    F_LINEAR = 1, F_TABLE = 2, F_BIGAD = 4, F_FIRST = 8, F_LONG = 64, F_ALL = 15 | 64, F_PARITY = 16, F_REGS = 32,
    F_NOOPT = 128, F_NOSPLIT = 256, F_FRONTIER = 512
};


CUBICS_HD constexpr size_t round4(size_t x) { return (x + 3) & ~size_t(3); }

// per-warp alldifferent scratch: BFS layers [66] + ancestor sets [64] (u64) + value owners [W*32] (u8)
CUBICS_HD constexpr int warp_scratch_bytes(int W) { return (66 + 64) * 8 + W * 32; }

// u32 words of per-warp scratch of the generic alldifferent path (propagators.cuh BigScratch)
CUBICS_HD inline size_t big_scratch_words(int n, int uw) {
    const size_t nwm = ((size_t)n + 31) / 32;
    return (size_t)n * uw + (size_t)n * nwm + (size_t)uw * 32 + (size_t)n + 2 * (size_t)n + 6 * (size_t)uw +
           2 * nwm + 4 + 8;
}

struct SmemLayout {
    size_t dom, rm, mates, scratch, path, bestkey, post, post_ok, chg, frames, meta, total;
    int stride;
    bool has_post, has_chg;
};

// GAC post-states are kept when they cost at most this many bytes of shared memory
constexpr size_t kPostBudget = 16384;
// changed-variable trigger bitmaps (two buffers of n bits) are kept up to this size
constexpr size_t kChgBudget = 65536;

// frame_cap > 0: the decision stack (frame_cap frames of NWP words + 4 meta words each) lives in
// shared memory too (warp contexts of small models)
CUBICS_HD inline SmemLayout smem_layout(int W, int n, int total_members, int nw, int KW, bool dom_in_smem,
                                        int na = 0, int frame_cap = 0) {
    SmemLayout L{};
    const size_t NWP = round4((size_t)n * W);
    size_t p = 0;
    L.dom = p;
    L.rm = p + (dom_in_smem ? NWP * 4 : 0);
    p += dom_in_smem ? 2 * NWP * 4 : 0;
    L.mates = p;
    p += ((size_t)total_members * 2 + 15) & ~size_t(15);
    L.stride = (warp_scratch_bytes(W) + 15) & ~15;
    L.scratch = p;
    p += (size_t)nw * L.stride;
    L.path = p;
    p += ((size_t)KW * 4 + 15) & ~size_t(15);
    L.bestkey = p;
    p += ((size_t)KW * 4 + 15) & ~size_t(15);
    const size_t post_bytes = (size_t)total_members * W * 4;
    L.has_post = na > 0 && post_bytes <= kPostBudget;
    L.post = p;
    p += L.has_post ? ((post_bytes + 15) & ~size_t(15)) : 0;
    L.post_ok = p;
    p += L.has_post ? (((size_t)na + 15) & ~size_t(15)) : 0;
    const size_t chg_bytes = (((size_t)n + 31) / 32) * 4;
    L.has_chg = 2 * chg_bytes <= kChgBudget;
    L.chg = p;
    p += L.has_chg ? ((2 * chg_bytes + 15) & ~size_t(15)) : 0;
    L.frames = p;
    p += (size_t)frame_cap * NWP * 4;
    L.meta = p;
    p += (size_t)frame_cap * 16;
    L.total = p;
    return L;
}

} // namespace dev
} // namespace cubics
