// Warp-resident search context for small models, sm_100a (search_kernel_warp).
//
// Eligible models: n <= 32 variables, every domain within one u32 word (W = 1), alldifferents of
// <= 32 members over a one-word value universe, no tables. nq8-nq14, magic3-magic5 and the small
// corpora are of this kind. One context is one warp; lane v owns variable v.
//
// propagate_fixpoint (propagation.cpp:516-532) runs with each domain in its lane's register:
//   * var-form x != y + k (prop_rel_bin Ne, propagation.cpp:186-192) is event driven: when u
//     becomes a singleton at bit b, lane p removes bits b + s for every edge (u -> p, shift s).
//     The shifts of all edges u -> p are folded on the host into one 64-bit mask neq[u*n + p]
//     (bit s + 32), so lane p's removal is (neq >> (32 - b)) - no atomics, no memory traffic.
//   * the other RelBins, linear sums and alldifferents read the round's frozen snapshot from
//     shared memory (ld.shared) and OR their removals into the context's rm words
//     (red.shared.or) - the RemovalSet union (propagation.cpp:26-99).
//   * apply (propagation.cpp:497-512): lane v folds its register and rm[v] into its domain; the
//     changed and empty sets are warp ballots, failed_var = lowest empty id.
// Rounds are Jacobi with the reference's snapshot semantics, exactly as block_fixpoint.
#pragma once

#include "propagators.cuh"

namespace cubics {
namespace dev {

__device__ __forceinline__ uint32_t lds_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(p)));
    return v;
}
__device__ __forceinline__ void sts_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}
__device__ __forceinline__ void red_or_shared(uint32_t* p, uint32_t v) {
    asm volatile("red.shared.or.b32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}
__device__ __forceinline__ int16_t lds_s16(const int16_t* p) {
    short v;
    asm volatile("ld.shared.s16 %0, [%1];" : "=h"(v) : "r"((unsigned)__cvta_generic_to_shared(p)));
    return v;
}
__device__ __forceinline__ void sts_s16(int16_t* p, int16_t v) {
    asm volatile("st.shared.s16 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "h"((short)v) : "memory");
}

// the same on 32-bit shared-window addresses (computed once per call, no per-access conversion)
__device__ __forceinline__ unsigned saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t lds_a(unsigned a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts_a(unsigned a, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void red_or_a(unsigned a, uint32_t v) {
    asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// shared -> shared copy of nwords/4 uint4 words by the lanes of one warp
__device__ __forceinline__ void copy4_shared(uint32_t* dst, const uint32_t* src, size_t nwords, int lane) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst), s = (unsigned)__cvta_generic_to_shared(src);
    for (unsigned i = lane; i < nwords / 4; i += 32) {
        uint4 v;
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(s + 16 * i));
        asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(d + 16 * i), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                     : "memory");
    }
}

// one-word domain helpers
__device__ __forceinline__ int w_first(uint32_t d) { return d ? __ffs(d) - 1 : -1; }
__device__ __forceinline__ int w_last(uint32_t d) { return d ? 31 - __clz(d) : -1; }
__device__ __forceinline__ uint32_t w_below(long long hi) { // bits [0, hi]
    return hi < 0 ? 0u : (hi >= 31 ? 0xffffffffu : ((1u << (hi + 1)) - 1u));
}
__device__ __forceinline__ uint32_t w_from(long long lo) { // bits [lo, 31]
    return lo <= 0 ? 0xffffffffu : (lo > 31 ? 0u : (0xffffffffu << lo));
}

// prop_rel_bin for W = 1 on the shared snapshot (the var-form != records are event driven)
__device__ __forceinline__ void warp_relbin(const RelBinRec r, const uint32_t* dom, uint32_t* rm) {
    const uint32_t dx = lds_u32(dom + r.x);
    const int s = r.s;
    uint32_t mx = 0;
    if (r.y < 0) {
        switch (r.op) {
        case 0:
        case 1: mx = dx & w_from(s); break;
        case 2:
        case 3: mx = dx & w_below(s); break;
        case 4: mx = dx & ~((s >= 0 && s < 32) ? (1u << s) : 0u); break;
        default: mx = (s >= 0 && s < 32) ? dx & (1u << s) : 0u; break;
        }
        if (mx) red_or_shared(rm + r.x, mx);
        return;
    }
    const uint32_t dy = lds_u32(dom + r.y);
    uint32_t my = 0;
    if (r.op == 5) { // only reached when the event path is off
        if (dy && !(dy & (dy - 1))) {
            const int bit = __ffs(dy) - 1 + s;
            if (bit >= 0 && bit < 32) mx = dx & (1u << bit);
        }
        if (dx && !(dx & (dx - 1))) {
            const int bit = __ffs(dx) - 1 - s;
            if (bit >= 0 && bit < 32) my = dy & (1u << bit);
        }
    } else if (dx && dy) {
        switch (r.op) {
        case 0:
            mx = dx & w_from((long long)w_last(dy) + s);
            my = dy & w_below((long long)w_first(dx) - s);
            break;
        case 1:
            mx = dx & w_from((long long)w_last(dy) + s + 1);
            my = dy & w_below((long long)w_first(dx) - s - 1);
            break;
        case 2:
            mx = dx & w_below((long long)w_first(dy) + s);
            my = dy & w_from((long long)w_last(dx) - s);
            break;
        case 3:
            mx = dx & w_below((long long)w_first(dy) + s - 1);
            my = dy & w_from((long long)w_last(dx) - s + 1);
            break;
        default: { // x = y + k: x keeps D(y) << s, y keeps D(x) >> s
            const uint32_t ys = s >= 32 || s <= -32 ? 0u : (s >= 0 ? dy << s : dy >> -s);
            const uint32_t xs = s >= 32 || s <= -32 ? 0u : (s >= 0 ? dx >> s : dx << -s);
            mx = dx & ~ys;
            my = dy & ~xs;
            break;
        }
        }
    }
    if (mx) red_or_shared(rm + r.x, mx);
    if (my) red_or_shared(rm + r.y, my);
}

// filter_linear_le (propagation.cpp:213-236) over a one-word snapshot; false on int64 overflow
__device__ __forceinline__ bool warp_filter_le(const DevModel& M, int b, int e, long long sign, long long bound,
                                               const uint32_t* dom, uint32_t* rm) {
    long long total = 0;
    for (int t = b; t < e; ++t) { // :217-224
        const int v = M.lin_var[t];
        const uint32_t d = lds_u32(dom + v);
        if (!d) return true;
        const long long a = sign * M.lin_coeff[t];
        const long long val = M.off[v] + (a > 0 ? w_first(d) : w_last(d));
        const i128 tm = (i128)a * val;
        if (!fits64(tm)) return false;
        const i128 s = (i128)total + tm;
        if (!fits64(s)) return false;
        total = (long long)s;
    }
    for (int t = b; t < e; ++t) { // :225-235
        const int v = M.lin_var[t];
        const uint32_t d = lds_u32(dom + v);
        const long long a = sign * M.lin_coeff[t];
        const long long offv = M.off[v];
        const long long tm = a * (offv + (a > 0 ? w_first(d) : w_last(d)));
        const i128 rest = (i128)total + (i128)wrap_add(0, -tm);
        if (!fits64(rest)) return false;
        const i128 budget = (i128)bound - rest;
        uint32_t m;
        if (a > 0) {
            const i128 thr = a == 1 ? budget : floor_div(budget, a);
            m = d & w_from(clampbit(thr + 1 - offv, 32));
        } else {
            const i128 thr = a == -1 ? -budget - 1 : ceil_div(budget, a) - 1;
            m = d & w_below(clampbit(thr - offv, 32));
        }
        if (m) red_or_shared(rm + v, m);
    }
    return true;
}

// 32 x 32 bit-matrix transpose across a warp: lane i holds row i (bit j = M[i][j]) and gets row i
// of the transpose (bit j = M[j][i]); five butterfly stages of one shuffle each
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, int lane) {
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
        const uint32_t lo = s == 16 ? 0x0000ffffu : s == 8 ? 0x00ff00ffu : s == 4 ? 0x0f0f0f0fu : s == 2 ? 0x33333333u : 0x55555555u;
        const uint32_t y = __shfl_xor_sync(FULL, x, s);
        x = (lane & s) ? ((x & ~lo) | ((y & ~lo) >> s)) : ((x & lo) | ((y & lo) << s));
    }
    return x;
}

// the reference wipes the first member Kuhn's matching leaves unmatched (propagation.cpp:379-386):
// a greedy matching in member order fails at the same member (cold path, kept out of line)
static __device__ __noinline__ int warp_gac_greedy_fail(int n, const uint32_t (&D0)[1], bool h0, int lane, int* m0_out) {
    const uint32_t D1[1] = {0u};
    int m0 = -1, m1 = -1, fail = -1;
    uint32_t MV[1] = {0u};
    for (int r = 0; r < n; ++r)
        if (!gac_augment<1, false>(r, D0, D1, h0, false, m0, m1, MV, lane)) {
            fail = r;
            break;
        }
    *m0_out = m0;
    return fail;
}

// prop_alldiff_gac (propagation.cpp:348-433) for <= 32 members over a one-word universe, member
// lane l holding D(l) in universe coordinates; same algorithm as prop_alldiff_gac<W, 1, false>
// (warm-started matching, bit-parallel BFS augmentation, Warshall closure, free-value reach).
static __device__ void warp_alldiff_gac(const DevModel& M, int a, const uint32_t* dom, uint32_t* rm, int16_t* mates,
                                 const WarpScratch& ws, int lane, int exact_wipe, uint32_t* post, int8_t* post_ok) {
    const int b = M.ad_start[a], n = M.ad_start[a + 1] - b;
    const bool h0 = lane < n;
    int v0 = -1, s0 = 0;
    uint32_t dv = 0;
    const unsigned arm = saddr(rm), apost = post ? saddr(post) + 4 * lane : 0u;
    if (h0) {
        v0 = M.ad_var[b + lane];
        s0 = M.ad_shift[b + lane];
        dv = lds_a(saddr(dom) + 4 * v0);
    }
    uint32_t D0[1] = {s0 ? (s0 < 32 ? dv << s0 : 0u) : dv}, D1[1] = {0u};
    if (post) { // idempotence: the post-state of the last evaluation is GAC-consistent
        const bool same = !h0 || dv == lds_a(apost);
        if (__all_sync(FULL, same) && *post_ok) return;
    }
    int m0 = h0 ? lds_s16(mates + lane) : -1, m1 = -1;
    if (m0 >= 0 && !((D0[0] >> m0) & 1u)) m0 = -1; // warm start: keep still-valid edges
    uint32_t MV[1] = {__reduce_or_sync(FULL, m0 >= 0 ? 1u << m0 : 0u)};
    unsigned unm = __ballot_sync(FULL, h0 && m0 < 0);
    int fail = -1;
    while (unm) {
        const int r = __ffs(unm) - 1;
        unm &= unm - 1;
        if (!gac_augment<1, false>(r, D0, D1, h0, false, m0, m1, MV, lane)) {
            fail = r;
            break;
        }
    }
    if (fail >= 0) {
        if (exact_wipe) fail = warp_gac_greedy_fail(n, D0, h0, lane, &m0);
        if (lane == fail && dv) red_or_a(arm + 4 * v0, dv);
        if (h0) sts_s16(mates + lane, (int16_t)m0);
        if (post && lane == 0) *post_ok = 0;
        __syncwarp();
        return;
    }
    if (h0) {
        sts_s16(mates + lane, (int16_t)m0);
        ws.owner[m0] = (uint8_t)lane;
    }
    __syncwarp();
    // free values F = U & ~MV ; pred(k) = { m : mate(m) in D(k) }
    const uint32_t F = __reduce_or_sync(FULL, D0[0]) & ~MV[0];
    const bool sd0 = (D0[0] & F) != 0;
    unsigned p0 = 0;
    for (uint32_t x0 = D0[0] & MV[0]; x0; x0 &= x0 - 1) p0 |= 1u << ws.owner[__ffs(x0) - 1];
    // Warshall over the non-singleton members (a singleton member has no in-edge)
    for (unsigned q = __ballot_sync(FULL, h0 && (D0[0] & (D0[0] - 1))); q; q &= q - 1) {
        const int p = __ffs(q) - 1;
        const unsigned ap = __shfl_sync(FULL, p0, p);
        if ((p0 >> p) & 1u) p0 |= ap;
    }
    // p0 is now desc(k): the members k reaches (k -> m when k can take mate(m))
    const unsigned S = __ballot_sync(FULL, h0 && sd0); // members holding a free value
    const bool r0 = h0 && (p0 & S);                    // k reaches one: mate(k) can be freed
    const uint32_t KEEP = F | __reduce_or_sync(FULL, r0 ? (1u << m0) : 0u);
    // An unmatched edge (k, j), j = mate(m), survives iff j is kept above or m and k share an SCC.
    // k -> m holds by construction, so that is "m reaches k": lane j takes desc(owner(j)) and one
    // warp transpose gives every lane k the values whose owner reaches it.
    const bool jm = (MV[0] >> lane) & 1u;
    const uint32_t X = __shfl_sync(FULL, p0, jm ? ws.owner[lane] : 0);
    const uint32_t reach = warp_transpose32(jm ? X : 0u, lane);
    if (h0) {
        const uint32_t cand = D0[0] & ~KEEP & ~(1u << m0) & ~reach;
        const uint32_t rv = s0 ? cand >> s0 : cand; // back to the member's own bit positions
        if (rv) red_or_a(arm + 4 * v0, rv);
        if (post) sts_a(apost, dv & ~rv);
    }
    if (post && lane == 0) *post_ok = 1;
    __syncwarp();
}

// prop_alldiff_fc (propagation.cpp:254-268), one-word universe
__device__ __forceinline__ void warp_alldiff_fc(const DevModel& M, int a, const uint32_t* dom, uint32_t* rm, int lane) {
    const int b = M.ad_start[a], n = M.ad_start[a + 1] - b;
    const bool h0 = lane < n;
    int v0 = -1, s0 = 0;
    uint32_t D = 0;
    if (h0) {
        v0 = M.ad_var[b + lane];
        s0 = M.ad_shift[b + lane];
        const uint32_t dv = lds_u32(dom + v0);
        D = s0 ? (s0 < 32 ? dv << s0 : 0u) : dv;
    }
    const bool g = h0 && D && !(D & (D - 1));
    const int x = g ? __ffs(D) - 1 : -1;
    const uint32_t once = __reduce_or_sync(FULL, g ? 1u << x : 0u);
    const unsigned q = __match_any_sync(FULL, g ? x : -(lane + 1));
    const bool dup = g && __popc(q) > 1;
    if (h0) {
        const uint32_t own = g ? 1u << x : 0u;
        const uint32_t r = (g ? ((once & ~own) | (dup ? own : 0u)) : once) & D;
        const uint32_t rv = s0 ? r >> s0 : r;
        if (rv) red_or_shared(rm + v0, rv);
    }
}

// propagate_fixpoint with register-resident domains (see the header). trig: variables changed
// since the last fixpoint (ignored when first_all). Leaves dom[] (shared) updated and rm clear.
template <int F>
__device__ int warp_fixpoint(const DevModel& M, const RoundCtx& R, int* rounds, bool first_all, uint32_t trig, int lane) {
    const int n = M.n;
    const uint32_t all = n >= 32 ? 0xffffffffu : ((1u << n) - 1u);
    uint32_t* dom = R.dom;
    uint32_t* rm = R.rm;
    const unsigned adom_lane = saddr(dom) + 4 * lane, arm_lane = saddr(rm) + 4 * lane;
    uint32_t dv = lane < n ? lds_a(adom_lane) : 0u;
    uint32_t chg = first_all ? all : trig;
    const bool has_ne = M.neq != nullptr && lane < n && M.ne_start[lane] < M.ne_start[lane + 1];
    const unsigned long long* neq_row = M.neq;
    const WarpScratch ws = warp_scratch<1>(R, 0);
    int r = 0;
    for (;;) {
        ++r;
        // var-form != : singleton events of the variables that changed (every singleton at first)
        uint32_t rmr = 0;
        if (M.neq) {
            // a lane with edges that just became a singleton is an event; every lane applies it
            unsigned ev = __ballot_sync(FULL, has_ne && ((chg >> lane) & 1u) && dv && !(dv & (dv - 1)));
            while (ev) {
                const int u = __ffs(ev) - 1;
                ev &= ev - 1;
                const int bit = __ffs(__shfl_sync(FULL, dv, u)) - 1;
                if (lane < n) rmr |= (uint32_t)(__ldg(neq_row + (size_t)u * n + lane) >> (32 - bit));
            }
        }
        // the other RelBins, one lane per record
        const int nr_loop = M.neq ? M.nr_gen : M.nr;
        for (int c = lane; c < nr_loop; c += 32) {
            const RelBinRec rec = M.rb[c];
            if (!((chg >> rec.x) & 1u) && (rec.y < 0 || !((chg >> rec.y) & 1u))) continue;
            warp_relbin(rec, dom, rm);
        }
        bool overflow = false;
        if constexpr ((F & F_LINEAR) != 0) {
            for (int c = lane; c < M.nl; c += 32) {
                const int b = M.lin_start[c], e = M.lin_start[c + 1];
                bool hit = false;
                for (int t = b; t < e && !hit; ++t) hit = (chg >> M.lin_var[t]) & 1u;
                if (!hit) continue;
                const long long bound = M.lin_bound[c];
                bool ok = warp_filter_le(M, b, e, 1, bound, dom, rm);
                if (ok && M.lin_op[c] == 1) ok = warp_filter_le(M, b, e, -1, -bound, dom, rm);
                overflow |= !ok;
            }
        }
        for (int a = 0; a < M.na; ++a) {
            const int b = M.ad_start[a], e = M.ad_start[a + 1];
            const bool hit = b + lane < e && ((chg >> M.ad_var[b + lane]) & 1u);
            if (!__any_sync(FULL, hit)) continue;
            if (R.alldiff)
                warp_alldiff_gac(M, a, dom, rm, R.mates + b, ws, lane, R.exact_wipe,
                                 R.post ? R.post + b : nullptr, R.post_ok + a);
            else
                warp_alldiff_fc(M, a, dom, rm, lane);
        }
        __syncwarp();
        // apply (propagation.cpp:497-512)
        uint32_t rem = rmr;
        if (lane < n) {
            const uint32_t rs = lds_a(arm_lane);
            if (rs) sts_a(arm_lane, 0u);
            rem |= rs;
        }
        const uint32_t nd = dv & ~rem;
        const bool vch = nd != dv;
        if (vch) sts_a(adom_lane, nd);
        dv = nd;
        chg = __ballot_sync(FULL, vch);
        if (__any_sync(FULL, overflow)) {
            *rounds = r;
            return R_ERROR;
        }
        if (!chg) {
            *rounds = r;
            return R_STABLE;
        }
        if (__ballot_sync(FULL, lane < n && !dv)) {
            *rounds = r;
            return R_FAILED;
        }
    }
}

} // namespace dev
} // namespace cubics
