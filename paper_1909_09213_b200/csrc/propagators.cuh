// Device propagators and the bulk-synchronous round, sm_100a.
//
// One search context = one thread block. Its domains live in shared memory (or in a per-context
// HBM/L2 slab when they do not fit) as W u32 words per variable. A round follows the
// reference's snapshot semantics exactly (propagation.cpp:480-514): every propagator reads the
// frozen domains and ORs its removals into a removal buffer `rm` with atomics (the RemovalSet
// union, :26-99, without materialising per-call sets); after a barrier, the apply step does
// dom &= ~rm, detects "changed" and emptiness with __syncthreads_or, and clears rm.
//
// Removal masks may contain bits of values that are absent: the apply step ANDs them with the
// domain, which is exactly the reference's "only values present in the snapshot are recorded"
// rule (add_value, propagation.cpp:42-48).
#pragma once

#include <cstdint>
#include <type_traits>

#include "device_model.hpp"
#include "layout.hpp"
#include "scope.cuh"

namespace cubics {
namespace dev {

constexpr unsigned FULL = 0xffffffffu;
typedef __int128 i128;

enum RoundStatus : int { R_CHANGED = 0, R_STABLE = 1, R_FAILED = 2, R_ERROR = 3 };


// ------------------------------------------------------------------ bitset helpers
template <int W>
__device__ __forceinline__ bool dom_empty(const uint32_t* d) {
    uint32_t o = 0;
#pragma unroll
    for (int i = 0; i < W; ++i) o |= d[i];
    return o == 0;
}

template <int W>
__device__ __forceinline__ int dom_size(const uint32_t* d) {
    int s = 0;
#pragma unroll
    for (int i = 0; i < W; ++i) s += __popc(d[i]);
    return s;
}

template <int W>
__device__ __forceinline__ int dom_first(const uint32_t* d) { // -1 when empty
    int r = -1;
#pragma unroll
    for (int i = W - 1; i >= 0; --i)
        if (d[i]) r = i * 32 + __ffs(d[i]) - 1;
    return r;
}

template <int W>
__device__ __forceinline__ int dom_last(const uint32_t* d) {
    int r = -1;
#pragma unroll
    for (int i = 0; i < W; ++i)
        if (d[i]) r = i * 32 + 31 - __clz(d[i]);
    return r;
}

__device__ __forceinline__ long long clampbit(i128 x, int nb) {
    return x < -1 ? -1LL : (x > (i128)nb ? (long long)nb : (long long)x);
}

// bits of [lo, hi] (global bit indices, may lie outside the word) inside word w
__device__ __forceinline__ uint32_t range_word(int w, long long lo, long long hi) {
    long long a = lo - (long long)w * 32, b = hi - (long long)w * 32;
    if (b < 0 || a > 31 || a > b) return 0u;
    int aa = a < 0 ? 0 : (int)a;
    int bb = b > 31 ? 31 : (int)b;
    uint32_t hiMask = bb == 31 ? 0xffffffffu : ((1u << (bb + 1)) - 1u);
    return hiMask & ~((1u << aa) - 1u);
}

// word i of (src << s): out bit j = src bit (j - s); s may be negative; out-of-range bits are 0
template <int W>
__device__ __forceinline__ uint32_t shifted_word(const uint32_t* src, int i, long long s) {
    long long b = (long long)i * 32 - s;
    long long q = b >> 5;
    int r = (int)(b & 31);
    uint32_t lo = (q >= 0 && q < W) ? src[q] : 0u;
    uint32_t hi = (q + 1 >= 0 && q + 1 < W) ? src[q + 1] : 0u;
    return r ? ((lo >> r) | (hi << (32 - r))) : lo;
}

template <int W>
__device__ __forceinline__ void or_range(uint32_t* rmv, const uint32_t* dv, long long lo, long long hi) {
#pragma unroll
    for (int w = 0; w < W; ++w) {
        uint32_t m = range_word(w, lo, hi) & dv[w];
        if (m) atomicOr(rmv + w, m);
    }
}

__device__ __forceinline__ void or_bit(uint32_t* rmv, const uint32_t* dv, int bit, int nb) {
    if (bit < 0 || bit >= nb) return;
    const int b = bit;
    uint32_t m = (1u << (b & 31)) & dv[b >> 5];
    if (m) atomicOr(rmv + (b >> 5), m);
}

// Runtime-width variants: a variable's bits live in its first vwords(v) <= W words (the rest
// stay 0), so mixed-width models (e.g. a wide objective next to narrow decision variables) do
// not pay W words per operation on every variable.
template <int W>
__device__ __forceinline__ int vwords(const DevModel& M, int v) {
    if constexpr (W <= 4) return W; // short unrolled loops beat a per-variable bound
    else return M.vw ? M.vw[v] : W; // vw == null: no variable is much narrower than W
}
template <int W>
__device__ __forceinline__ bool dom_empty_n(const uint32_t* d, int n) {
    if (W <= 4 || n == W) return dom_empty<W>(d);
    uint32_t o = 0;
    for (int i = 0; i < n; ++i) o |= d[i];
    return o == 0;
}
template <int W>
__device__ __forceinline__ int dom_first_n(const uint32_t* d, int n) {
    if (W <= 4 || n == W) return dom_first<W>(d);
    for (int i = 0; i < n; ++i)
        if (d[i]) return i * 32 + __ffs(d[i]) - 1;
    return -1;
}
template <int W>
__device__ __forceinline__ int dom_last_n(const uint32_t* d, int n) {
    if (W <= 4 || n == W) return dom_last<W>(d);
    for (int i = n - 1; i >= 0; --i)
        if (d[i]) return i * 32 + 31 - __clz(d[i]);
    return -1;
}
template <int W>
__device__ __forceinline__ int dom_size_n(const uint32_t* d, int n) {
    if (W <= 4 || n == W) return dom_size<W>(d);
    int s = 0;
    for (int i = 0; i < n; ++i) s += __popc(d[i]);
    return s;
}
template <int W>
__device__ __forceinline__ void or_range_n(uint32_t* rmv, const uint32_t* dv, long long lo, long long hi, int n) {
    if (W <= 4 || n == W) {
        or_range<W>(rmv, dv, lo, hi);
    } else {
        if (lo > hi) return;
        const int w0 = lo < 0 ? 0 : (int)(lo >> 5);
        const int w1 = (int)((hi >> 5) < (long long)(n - 1) ? (hi >> 5) : (long long)(n - 1));
        for (int w = w0; w <= w1; ++w) {
            const uint32_t m = range_word(w, lo, hi) & dv[w];
            if (m) atomicOr(rmv + w, m);
        }
    }
}

__device__ __forceinline__ long long wrap_add(long long a, long long b) {
    return (long long)((unsigned long long)a + (unsigned long long)b);
}

// ------------------------------------------------------------------ RelBin (propagation.cpp:120-194)
// All offsets are pre-folded into r.s (engine.cu), so every case is 32-bit bit arithmetic:
//   x <  y+k : x loses bits >= last(y)+s      y loses bits <= first(x)-s
//   x <= y+k : x loses bits >= last(y)+s+1    y loses bits <= first(x)-s-1
//   x >  y+k : x loses bits <= first(y)+s     y loses bits >= last(x)-s
//   x >= y+k : x loses bits <= first(y)+s-1   y loses bits >= last(x)-s+1
//   x =  y+k : x keeps D(y) << s, y keeps D(x) >> s      (domain consistency)
//   x != y+k : singleton y removes bit first(y)+s from x, singleton x removes first(x)-s from y
// Literal forms carry the threshold bit in s (x < lit: bits >= s; x <= lit: bits >= s with
// s = lit+1-off; x > lit: bits <= s; x >= lit: bits <= s with s = lit-1-off; = / != : bit s).
template <int W>
__device__ __forceinline__ void prop_relbin(const DevModel& M, int c, const uint32_t* dom, uint32_t* rm) {
    constexpr int NB = W * 32;
    const RelBinRec r = M.rb[c];
    const uint32_t* dx = dom + (size_t)r.x * W;
    uint32_t* rx = rm + (size_t)r.x * W;
    const int s = r.s;
    if (r.y < 0) {
        switch (r.op) {
        case 0:
        case 1: or_range<W>(rx, dx, s, NB); break;
        case 2:
        case 3: or_range<W>(rx, dx, -1, s); break;
        case 4: {
#pragma unroll
            for (int w = 0; w < W; ++w) {
                const uint32_t keep = (s >= w * 32 && s < w * 32 + 32) ? (1u << (s - w * 32)) : 0u;
                const uint32_t m = dx[w] & ~keep;
                if (m) atomicOr(rx + w, m);
            }
            break;
        }
        default: or_bit(rx, dx, s, NB); break;
        }
        return;
    }
    const uint32_t* dy = dom + (size_t)r.y * W;
    uint32_t* ry = rm + (size_t)r.y * W;
    if (r.op == 5) {
        if (W == 1) {
            const uint32_t ax = dx[0], ay = dy[0];
            if (ay && !(ay & (ay - 1))) { // y singleton
                const int bit = __ffs(ay) - 1 + s;
                if (bit >= 0 && bit < 32 && ((ax >> bit) & 1u)) atomicOr(rx, 1u << bit);
            }
            if (ax && !(ax & (ax - 1))) {
                const int bit = __ffs(ax) - 1 - s;
                if (bit >= 0 && bit < 32 && ((ay >> bit) & 1u)) atomicOr(ry, 1u << bit);
            }
            return;
        }
        if (dom_size<W>(dy) == 1) or_bit(rx, dx, dom_first<W>(dy) + s, NB);
        if (dom_size<W>(dx) == 1) or_bit(ry, dy, dom_first<W>(dx) - s, NB);
        return;
    }
    if (dom_empty<W>(dx) || dom_empty<W>(dy)) return;
    switch (r.op) {
    case 0:
        or_range<W>(rx, dx, dom_last<W>(dy) + s, NB);
        or_range<W>(ry, dy, -1, dom_first<W>(dx) - s);
        break;
    case 1:
        or_range<W>(rx, dx, dom_last<W>(dy) + s + 1, NB);
        or_range<W>(ry, dy, -1, dom_first<W>(dx) - s - 1);
        break;
    case 2:
        or_range<W>(rx, dx, -1, dom_first<W>(dy) + s);
        or_range<W>(ry, dy, dom_last<W>(dx) - s, NB);
        break;
    case 3:
        or_range<W>(rx, dx, -1, dom_first<W>(dy) + s - 1);
        or_range<W>(ry, dy, dom_last<W>(dx) - s + 1, NB);
        break;
    default:
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const uint32_t mx = dx[w] & ~shifted_word<W>(dy, w, s);
            if (mx) atomicOr(rx + w, mx);
            const uint32_t my = dy[w] & ~shifted_word<W>(dx, w, -s);
            if (my) atomicOr(ry + w, my);
        }
        break;
    }
}

// ------------------------------------------------------------------ Linear (propagation.cpp:196-252)
__device__ __forceinline__ bool fits64(i128 v) {
    return v >= (i128)(-9223372036854775807LL - 1) && v <= (i128)9223372036854775807LL;
}

// floor / ceil of a / b (b != 0). Unit coefficients (golomb, magic, most sums) skip the division;
// operands that fit 64 bits take one hardware-emulated 64-bit division instead of two 128-bit ones
// (|b| >= 2 there, so x / b cannot overflow).
__device__ __forceinline__ i128 floor_div(i128 a, long long b) {
    if (b == 1) return a;
    if (b == -1) return -a;
    if (fits64(a)) {
        const long long x = (long long)a, q = x / b, r = x - q * b;
        return (i128)((r != 0 && ((x < 0) != (b < 0))) ? q - 1 : q);
    }
    const i128 q = a / b, r = a - q * (i128)b;
    return (r != 0 && ((a < 0) != (b < 0))) ? q - 1 : q;
}
__device__ __forceinline__ i128 ceil_div(i128 a, long long b) {
    if (b == 1) return a;
    if (b == -1) return -a;
    if (fits64(a)) {
        const long long x = (long long)a, q = x / b, r = x - q * b;
        return (i128)((r != 0 && ((x < 0) == (b < 0))) ? q + 1 : q);
    }
    const i128 q = a / b, r = a - q * (i128)b;
    return (r != 0 && ((a < 0) == (b < 0))) ? q + 1 : q;
}

// filter_linear_le over terms [b, e) with coefficients sign*coeff; false on int64 overflow
template <int W>
__device__ bool filter_le(const DevModel& M, int b, int e, long long sign, long long bound,
                          const uint32_t* dom, uint32_t* rm) {
    constexpr int NB = W * 32;
    long long total = 0;
    for (int t = b; t < e; ++t) { // :217-224
        const int v = M.lin_var[t];
        const uint32_t* d = dom + (size_t)v * W;
        const int nv = vwords<W>(M, v);
        if (dom_empty_n<W>(d, nv)) return true;
        const long long a = sign * M.lin_coeff[t];
        const long long val = M.off[v] + (a > 0 ? dom_first_n<W>(d, nv) : dom_last_n<W>(d, nv));
        i128 tm = (i128)a * val;
        if (!fits64(tm)) return false;
        i128 s = (i128)total + tm;
        if (!fits64(s)) return false;
        total = (long long)s;
    }
    for (int t = b; t < e; ++t) { // :225-235
        const int v = M.lin_var[t];
        const uint32_t* d = dom + (size_t)v * W;
        const int nv = vwords<W>(M, v);
        const long long a = sign * M.lin_coeff[t];
        const long long offv = M.off[v];
        const long long tm = a * (offv + (a > 0 ? dom_first_n<W>(d, nv) : dom_last_n<W>(d, nv)));
        i128 rest = (i128)total + (i128)wrap_add(0, -tm); // checked_add(total, -term_min)
        if (!fits64(rest)) return false;
        const i128 budget = (i128)bound - rest;
        uint32_t* rv = rm + (size_t)v * W;
        if (a > 0) { // remove v > floor(budget / a)
            i128 thr = a == 1 ? budget : floor_div(budget, a);
            or_range_n<W>(rv, d, clampbit(thr + 1 - offv, NB), NB, nv);
        } else {     // remove v < budget / a, i.e. v <= ceil(budget / a) - 1
            i128 thr = a == -1 ? -budget - 1 : ceil_div(budget, a) - 1;
            or_range_n<W>(rv, d, -1, clampbit(thr - offv, NB), nv);
        }
    }
    return true;
}

// Sums of <= 4 terms, one thread: each term's bounds are read once, and the cuts of both
// directions of an equality become one keep-window per variable. Event order, overflow checks
// and thresholds are filter_le's (the first empty domain in term order makes a direction a
// no-op; any overflow returns false).
template <int W>
__device__ bool prop_linear_small(const DevModel& M, int c, const uint32_t* dom, uint32_t* rm) {
    constexpr int NB = W * 32;
    const int b = M.lin_start[c], k = M.lin_start[c + 1] - b;
    const long long bound = M.lin_bound[c];
    const int ndir = M.lin_op[c] == 1 ? 2 : 1;
    int v[4], lo[4], hi[4];
    long long co[4], of[4], cutlo[4], cuthi[4]; // remove bits <= cutlo and bits >= cuthi
    int first_empty = 4;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        v[t] = 0;
        co[t] = of[t] = 0;
        lo[t] = hi[t] = 0;
        cutlo[t] = -1;
        cuthi[t] = NB;
        if (t < k) {
            v[t] = M.lin_var[b + t];
            co[t] = M.lin_coeff[b + t];
            of[t] = M.off[v[t]];
            const uint32_t* d = dom + (size_t)v[t] * W;
            lo[t] = dom_first<W>(d);
            hi[t] = dom_last<W>(d);
            if (lo[t] < 0 && first_empty == 4) first_empty = t;
        }
    }
#pragma unroll
    for (int dir = 0; dir < 2; ++dir) {
        if (dir >= ndir) break;
        const long long sg = dir ? -1 : 1, bnd = dir ? -bound : bound;
        long long total = 0;
        bool noop = false;
#pragma unroll
        for (int t = 0; t < 4; ++t) { // :217-224
            if (t >= k || noop) continue;
            if (t == first_empty) {
                noop = true;
                continue;
            }
            const long long a = sg * co[t];
            const i128 tm = (i128)a * (of[t] + (a > 0 ? lo[t] : hi[t]));
            if (!fits64(tm)) return false;
            const i128 sum = (i128)total + tm;
            if (!fits64(sum)) return false;
            total = (long long)sum;
        }
        if (noop) continue;
#pragma unroll
        for (int t = 0; t < 4; ++t) { // :225-235
            if (t >= k) continue;
            const long long a = sg * co[t];
            const long long tm = a * (of[t] + (a > 0 ? lo[t] : hi[t]));
            const i128 rest = (i128)total + (i128)wrap_add(0, -tm);
            if (!fits64(rest)) return false;
            const i128 budget = (i128)bnd - rest;
            if (a > 0) {
                const i128 thr = a == 1 ? budget : floor_div(budget, a);
                const long long f = clampbit(thr + 1 - of[t], NB);
                cuthi[t] = f < cuthi[t] ? f : cuthi[t];
            } else {
                const i128 thr = a == -1 ? -budget - 1 : ceil_div(budget, a) - 1;
                const long long u = clampbit(thr - of[t], NB);
                cutlo[t] = u > cutlo[t] ? u : cutlo[t];
            }
        }
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        if (t >= k || (cutlo[t] < 0 && cuthi[t] >= NB)) continue;
        const uint32_t* dv = dom + (size_t)v[t] * W;
        uint32_t* rv = rm + (size_t)v[t] * W;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const uint32_t m = (range_word(w, -1, cutlo[t]) | range_word(w, cuthi[t], NB)) & dv[w];
            if (m) atomicOr(rv + w, m);
        }
    }
    return true;
}

__device__ __forceinline__ i128 shfl_up_i128(unsigned mask, i128 v, int d, int width) {
    const unsigned long long lo = __shfl_up_sync(mask, (unsigned long long)v, d, width);
    const long long hi = __shfl_up_sync(mask, (long long)(v >> 64), d, width);
    return (i128)(((unsigned __int128)(unsigned long long)hi << 64) | lo);
}
__device__ __forceinline__ i128 shfl_i128(unsigned mask, i128 v, int src, int width) {
    const unsigned long long lo = __shfl_sync(mask, (unsigned long long)v, src, width);
    const long long hi = __shfl_sync(mask, (long long)(v >> 64), src, width);
    return (i128)(((unsigned __int128)(unsigned long long)hi << 64) | lo);
}

// filter_le by a group of G lanes (G = 2..32, a power of two; the whole warp calls it, each
// group on its own constraint, gl = lane within the group). Terms are spread over the lanes; the
// running total is an exact i128 segmented scan, so the first event in term order decides the
// outcome exactly as the sequential loop does: an empty domain first -> no-op (true), an int64
// overflow of a term or of a prefix sum first -> false. Pass 2 filters every term in parallel.
// Returns false on overflow (the caller aborts the search, so partial removals do not matter).
template <int W>
__device__ bool filter_le_group(const DevModel& M, int b, int e, long long sign, long long bound,
                                const uint32_t* dom, uint32_t* rm, int G, int gl, unsigned gmask) {
    constexpr int NB = W * 32;
    i128 carry = 0;
    for (int base = b; base < e; base += G) { // pass 1 (:217-224)
        const int t = base + gl;
        i128 tm = 0;
        int kind = 0; // 1 empty, 2 overflow
        if (t < e) {
            const int v = M.lin_var[t];
            const uint32_t* d = dom + (size_t)v * W;
            const int nv = vwords<W>(M, v);
            if (dom_empty_n<W>(d, nv)) {
                kind = 1;
            } else {
                const long long a = sign * M.lin_coeff[t];
                tm = (i128)a * (M.off[v] + (a > 0 ? dom_first_n<W>(d, nv) : dom_last_n<W>(d, nv)));
                if (!fits64(tm)) kind = 2;
            }
        }
        i128 ps = kind ? (i128)0 : tm;
        for (int o = 1; o < G; o <<= 1) {
            const i128 y = shfl_up_i128(gmask, ps, o, G);
            if (gl >= o) ps += y;
        }
        ps += carry;
        if (!kind && t < e && !fits64(ps)) kind = 2;
        const unsigned ev = __ballot_sync(gmask, kind != 0) & gmask;
        if (ev) {
            const int first = __ffs(ev) - 1; // lowest lane = earliest term
            return __shfl_sync(gmask, kind, first & (G - 1), G) == 1;
        }
        carry = shfl_i128(gmask, ps, G - 1, G);
    }
    const long long total = (long long)carry;
    bool ok = true;
    for (int t = b + gl; t < e; t += G) { // pass 2 (:225-235)
        const int v = M.lin_var[t];
        const uint32_t* d = dom + (size_t)v * W;
        const int nv = vwords<W>(M, v);
        const long long a = sign * M.lin_coeff[t];
        const long long offv = M.off[v];
        const long long tm = a * (offv + (a > 0 ? dom_first_n<W>(d, nv) : dom_last_n<W>(d, nv)));
        const i128 rest = (i128)total + (i128)wrap_add(0, -tm);
        if (!fits64(rest)) {
            ok = false;
            continue;
        }
        const i128 budget = (i128)bound - rest;
        uint32_t* rv = rm + (size_t)v * W;
        if (a > 0) {
            const i128 thr = a == 1 ? budget : floor_div(budget, a);
            or_range_n<W>(rv, d, clampbit(thr + 1 - offv, NB), NB, nv);
        } else {
            const i128 thr = a == -1 ? -budget - 1 : ceil_div(budget, a) - 1;
            or_range_n<W>(rv, d, -1, clampbit(thr - offv, NB), nv);
        }
    }
    return !(__ballot_sync(gmask, !ok) & gmask);
}

template <int W>
__device__ __forceinline__ bool prop_linear_group(const DevModel& M, int c, const uint32_t* dom, uint32_t* rm, int G,
                                                  int gl, unsigned gmask) {
    const int b = M.lin_start[c], e = M.lin_start[c + 1];
    const long long bound = M.lin_bound[c];
    if (!filter_le_group<W>(M, b, e, 1, bound, dom, rm, G, gl, gmask)) return false;
    if (M.lin_op[c] == 1 && !filter_le_group<W>(M, b, e, -1, -bound, dom, rm, G, gl, gmask)) return false;
    return true;
}

template <int W>
__device__ __forceinline__ bool prop_linear(const DevModel& M, int c, const uint32_t* dom, uint32_t* rm) {
    const int b = M.lin_start[c], e = M.lin_start[c + 1];
    const long long bound = M.lin_bound[c];
    if (!filter_le<W>(M, b, e, 1, bound, dom, rm)) return false;
    // Eq: the >= direction as sum(-a x) <= -bound (:243-250); INT64_MIN coefficients / bounds
    // (whose negation overflows) are rejected on the host before launch.
    if (M.lin_op[c] == 1 && !filter_le<W>(M, b, e, -1, -bound, dom, rm)) return false;
    return true;
}

// ------------------------------------------------------------------ Table (extension, no reference counterpart)
// Positive extensional constraint, generalised arc consistency. Binary tables use support bitsets
// (bitwise AC): x keeps value a iff row a of x's support block meets D(y). N-ary tables scan
// their tuples: a tuple is valid when every component is in its domain; valid tuples support
// their values. Matches oracle/cubics_oracle.c prop_table.
template <int W>
__device__ __forceinline__ void prop_table2(const DevModel& M, int t, const uint32_t* dom, uint32_t* rm) {
    const int x = M.tb_xy[2 * t], y = M.tb_xy[2 * t + 1];
    const uint32_t* dx = dom + (size_t)x * W;
    const uint32_t* dy = dom + (size_t)y * W;
    if (dom_empty<W>(dx) || dom_empty<W>(dy)) return;
    const uint32_t* sx = M.tb_sup + M.tb_off[2 * t];
    const uint32_t* sy = M.tb_sup + M.tb_off[2 * t + 1];
#pragma unroll
    for (int w = 0; w < W; ++w) {
        uint32_t bits = dx[w], gone = 0;
        while (bits) {
            const int a = w * 32 + __ffs(bits) - 1;
            bits &= bits - 1;
            uint32_t any = 0;
#pragma unroll
            for (int i = 0; i < W; ++i) any |= sx[(size_t)a * W + i] & dy[i];
            if (!any) gone |= 1u << (a & 31);
        }
        if (gone) atomicOr(rm + (size_t)x * W + w, gone);
    }
#pragma unroll
    for (int w = 0; w < W; ++w) {
        uint32_t bits = dy[w], gone = 0;
        while (bits) {
            const int b = w * 32 + __ffs(bits) - 1;
            bits &= bits - 1;
            uint32_t any = 0;
#pragma unroll
            for (int i = 0; i < W; ++i) any |= sy[(size_t)b * W + i] & dx[i];
            if (!any) gone |= 1u << (b & 31);
        }
        if (gone) atomicOr(rm + (size_t)y * W + w, gone);
    }
}

template <int W>
__device__ void prop_tablen(const DevModel& M, int t, const uint32_t* dom, uint32_t* rm) {
    const int b = M.tn_start[t], k = M.tn_start[t + 1] - b;
    for (int j = 0; j < k; ++j)
        if (dom_empty<W>(dom + (size_t)M.tn_var[b + j] * W)) return;
    uint32_t sup[8][W];
    for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int w = 0; w < W; ++w) sup[j][w] = 0;
    const int16_t* tu = M.tn_data + M.tn_off[t];
    for (int64_t i = 0; i < M.tn_nt[t]; ++i, tu += k) {
        bool valid = true;
        for (int j = 0; j < k && valid; ++j) {
            const int bi = tu[j];
            valid = bi >= 0 && ((dom[(size_t)M.tn_var[b + j] * W + (bi >> 5)] >> (bi & 31)) & 1u);
        }
        if (!valid) continue;
        for (int j = 0; j < k; ++j) sup[j][tu[j] >> 5] |= 1u << (tu[j] & 31);
    }
    for (int j = 0; j < k; ++j) {
        const int v = M.tn_var[b + j];
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const uint32_t r = dom[(size_t)v * W + w] & ~sup[j][w];
            if (r) atomicOr(rm + (size_t)v * W + w, r);
        }
    }
}

// ------------------------------------------------------------------ AllDifferent (warp per constraint)
// Members are spread over the 32 lanes, two slots per lane (member l and l+32), so one warp
// handles up to 64 members. Member domains are loaded into a common value universe (W words).

struct WarpScratch {
    unsigned long long* layers; // [66] BFS frontier member sets
    unsigned long long* anc;    // [64] ancestor sets (Warshall closure)
    uint8_t* owner;             // [W*32] universe value -> matched member
};

template <int W>
__device__ __forceinline__ bool testbit_r(const uint32_t (&a)[W], int bit) {
    bool t = false;
#pragma unroll
    for (int w = 0; w < W; ++w) t |= (w == (bit >> 5)) && ((a[w] >> (bit & 31)) & 1u);
    return t;
}

__device__ __forceinline__ uint32_t bitword(int bit, int w) { // word w of the singleton {bit}; bit < 0 -> 0
    return (bit >= 0 && (bit >> 5) == w) ? (1u << (bit & 31)) : 0u;
}

__device__ __forceinline__ unsigned long long ballot64(bool a, bool b) {
    return (unsigned long long)__ballot_sync(FULL, a) | ((unsigned long long)__ballot_sync(FULL, b) << 32);
}

template <bool TWO>
using MemberSet = typename std::conditional<TWO, unsigned long long, unsigned>::type;

template <bool TWO>
__device__ __forceinline__ MemberSet<TWO> ballot_m(bool a, bool b) {
    if constexpr (TWO) return ballot64(a, b);
    else return __ballot_sync(FULL, a);
}

template <bool TWO>
__device__ __forceinline__ int ffs_m(MemberSet<TWO> x) {
    if constexpr (TWO) return __ffsll((long long)x) - 1;
    else return __ffs(x) - 1;
}

// Bit-parallel BFS augmenting path from member r (uniform). Updates mate[], MV. true on success.
// Each member remembers the BFS layer it entered (lay0/lay1, registers), so the walk back needs
// no shared memory: at layer l the predecessor of value j is a member of layer l containing j.
template <int W, bool TWO>
__device__ bool gac_augment(int r, const uint32_t (&D0)[W], const uint32_t (&D1)[W], bool h0, bool h1, int& m0,
                            int& m1, uint32_t (&MV)[W], int lane) {
    using MS = MemberSet<TWO>;
    uint32_t vis[W];
#pragma unroll
    for (int w = 0; w < W; ++w) vis[w] = 0;
    MS front = (MS)1 << r;
    int lay0 = lane == r ? 0 : -1, lay1 = (TWO && lane + 32 == r) ? 0 : -1;
    int L = 0;
    for (;;) {
        const bool f0 = h0 && ((front >> lane) & 1u);
        bool f1 = false;
        if constexpr (TWO) f1 = h1 && ((front >> (lane + 32)) & 1ull);
        uint32_t nv[W];
        uint32_t any = 0;
        int found = -1;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            uint32_t c = f0 ? D0[w] : 0u;
            if constexpr (TWO) c |= f1 ? D1[w] : 0u;
            nv[w] = __reduce_or_sync(FULL, c) & ~vis[w];
            vis[w] |= nv[w];
            any |= nv[w];
            const uint32_t fr = nv[w] & ~MV[w];
            if (fr && found < 0) found = w * 32 + __ffs(fr) - 1;
        }
        if (!any) return false;
        if (found >= 0) { // walk back through the layers, re-matching along the path
            int j = found;
            for (int l = L;; --l) {
                const bool c0 = h0 && lay0 == l && testbit_r<W>(D0, j);
                bool c1 = false;
                if constexpr (TWO) c1 = h1 && lay1 == l && testbit_r<W>(D1, j);
                const int k = ffs_m<TWO>(ballot_m<TWO>(c0, c1));
                const int kl = k & 31, ks = k >> 5;
                const int old = __shfl_sync(FULL, ks ? m1 : m0, kl);
                if (lane == kl) {
                    if (ks) m1 = j;
                    else m0 = j;
                }
                if (l == 0) break;
                j = old;
            }
#pragma unroll
            for (int w = 0; w < W; ++w) MV[w] |= bitword(found, w);
            return true;
        }
        ++L;
        const bool t0 = h0 && m0 >= 0 && lay0 < 0 && testbit_r<W>(nv, m0);
        bool t1 = false;
        if constexpr (TWO) t1 = h1 && m1 >= 0 && lay1 < 0 && testbit_r<W>(nv, m1);
        if (t0) lay0 = L;
        if (t1) lay1 = L;
        front = ballot_m<TWO>(t0, t1);
    }
}

// prop_alldiff_gac (propagation.cpp:348-433): removes exactly the values in no maximum matching;
// the result is unique, so this bit-parallel formulation (warm-started matching, Warshall
// closure of the member graph m -> k iff mate(m) in D(k)) equals the reference's Kuhn + Tarjan.
// On infeasibility the reference wipes the first member Kuhn leaves unmatched (:379-386); with
// exact_wipe we recompute the matching greedily in member order, which leaves the same first
// member unmatched (transversal-matroid greedy basis), and wipe it.
// TWO = false: <= 32 members, one per lane, 32-bit member sets; TWO = true: <= 64 members.
template <int W, int U, bool TWO>
__device__ void prop_alldiff_gac(const DevModel& M, int a, const uint32_t* dom, uint32_t* rm, int16_t* mates,
                                 const WarpScratch& ws, int lane, int exact_wipe, uint32_t* post, int8_t* post_ok) {
    using MS = MemberSet<TWO>;
    const int b = M.ad_start[a], n = M.ad_start[a + 1] - b;
    const bool h0 = lane < n, h1 = TWO && lane + 32 < n;
    uint32_t D0[U], D1[U]; // member domains in universe coordinates (U <= W words)
    int v0 = -1, v1 = -1, s0 = 0, s1 = 0;
    if (h0) {
        v0 = M.ad_var[b + lane];
        s0 = M.ad_shift[b + lane];
    }
    if (h1) {
        v1 = M.ad_var[b + lane + 32];
        s1 = M.ad_shift[b + lane + 32];
    }
#pragma unroll
    for (int w = 0; w < U; ++w) {
        D0[w] = h0 ? (s0 ? shifted_word<W>(dom + (size_t)v0 * W, w, s0) : dom[(size_t)v0 * W + w]) : 0u;
        D1[w] = h1 ? (s1 ? shifted_word<W>(dom + (size_t)v1 * W, w, s1) : dom[(size_t)v1 * W + w]) : 0u;
    }
    if (post) { // idempotence: the post-state of the last evaluation is GAC-consistent
        bool same = true;
        if constexpr (U == W) { // variable coordinates
#pragma unroll
            for (int w = 0; w < W; ++w) {
                if (h0) same &= dom[(size_t)v0 * W + w] == post[(size_t)lane * W + w];
                if (h1) same &= dom[(size_t)v1 * W + w] == post[(size_t)(lane + 32) * W + w];
            }
        } else { // universe coordinates (the shift is injective on member values)
#pragma unroll
            for (int w = 0; w < U; ++w) {
                if (h0) same &= D0[w] == post[(size_t)lane * W + w];
                if (h1) same &= D1[w] == post[(size_t)(lane + 32) * W + w];
            }
        }
        if (__all_sync(FULL, same) && *post_ok) return;
    }
    int m0 = h0 ? mates[lane] : -1, m1 = h1 ? mates[lane + 32] : -1;
    if (m0 >= 0 && !testbit_r<U>(D0, m0)) m0 = -1; // warm start: keep still-valid edges
    if (m1 >= 0 && !testbit_r<U>(D1, m1)) m1 = -1;
    uint32_t MV[U];
#pragma unroll
    for (int w = 0; w < U; ++w) MV[w] = __reduce_or_sync(FULL, bitword(m0, w) | bitword(m1, w));

    MS unm = ballot_m<TWO>(h0 && m0 < 0, h1 && m1 < 0);
    int fail = -1;
    while (unm) {
        const int r = ffs_m<TWO>(unm);
        unm &= unm - 1;
        if (!gac_augment<U, TWO>(r, D0, D1, h0, h1, m0, m1, MV, lane)) {
            fail = r;
            break;
        }
    }
    if (fail >= 0) {
        if (exact_wipe) { // greedy matching in member order: its first failure is Kuhn's
            m0 = m1 = -1;
#pragma unroll
            for (int w = 0; w < U; ++w) MV[w] = 0;
            for (int r = 0; r < n; ++r)
                if (!gac_augment<U, TWO>(r, D0, D1, h0, h1, m0, m1, MV, lane)) {
                    fail = r;
                    break;
                }
        }
        if (lane == (fail & 31)) {
            const int v = (fail >> 5) ? v1 : v0;
#pragma unroll
            for (int w = 0; w < W; ++w) {
                uint32_t d = dom[(size_t)v * W + w];
                if (d) atomicOr(rm + (size_t)v * W + w, d);
            }
        }
        if (h0) mates[lane] = (int16_t)m0;
        if (h1) mates[lane + 32] = (int16_t)m1;
        if (post && lane == 0) *post_ok = 0;
        __syncwarp();
        return;
    }
    if (h0) {
        mates[lane] = (int16_t)m0;
        ws.owner[m0] = (uint8_t)lane;
    }
    if (h1) {
        mates[lane + 32] = (int16_t)m1;
        ws.owner[m1] = (uint8_t)(lane + 32);
    }
    __syncwarp();
    // free values F = U & ~MV ; pred(k) = { m : mate(m) in D(k) }
    uint32_t F[U];
    MS p0 = 0, p1 = 0;
    bool sd0 = false, sd1 = false;
#pragma unroll
    for (int w = 0; w < U; ++w) {
        F[w] = __reduce_or_sync(FULL, D0[w] | D1[w]) & ~MV[w];
        sd0 |= (D0[w] & F[w]) != 0;
        sd1 |= (D1[w] & F[w]) != 0;
        // two owner lookups per step: independent shared-memory loads in flight together
        // (the reference-order kernels run few warps, so the lookup latency is the cost)
        uint32_t x0 = D0[w] & MV[w];
        while (x0) {
            const int b1 = __ffs(x0) - 1;
            x0 &= x0 - 1;
            const int b2 = x0 ? __ffs(x0) - 1 : b1;
            x0 &= x0 - 1;
            p0 |= ((MS)1 << ws.owner[w * 32 + b1]) | ((MS)1 << ws.owner[w * 32 + b2]);
        }
        if constexpr (TWO) {
            uint32_t x1 = D1[w] & MV[w];
            while (x1) {
                const int b1 = __ffs(x1) - 1;
                x1 &= x1 - 1;
                const int b2 = x1 ? __ffs(x1) - 1 : b1;
                x1 &= x1 - 1;
                p1 |= ((MS)1 << ws.owner[w * 32 + b1]) | ((MS)1 << ws.owner[w * 32 + b2]);
            }
        }
    }
    // Warshall: anc(k) = members that reach k. A singleton member has no in-edge (its only value
    // is its own mate), so it is never interior to a path: only non-singletons serve as pivots.
    const MS pivots = ballot_m<TWO>(h0 && dom_size<U>(D0) > 1, h1 && dom_size<U>(D1) > 1);
    for (MS q = pivots; q; q &= q - 1) {
        const int p = ffs_m<TWO>(q);
        const MS ap = __shfl_sync(FULL, (p >> 5) ? p1 : p0, p & 31);
        if ((p0 >> p) & 1u) p0 |= ap;
        if constexpr (TWO)
            if ((p1 >> p) & 1u) p1 |= ap;
    }
    // members reached from free values (seeds: D(k) meets F)
    const MS S = ballot_m<TWO>(h0 && sd0, h1 && sd1);
    const bool r0 = h0 && (p0 & S), r1 = h1 && (p1 & S);
    uint32_t KEEP[U];
#pragma unroll
    for (int w = 0; w < U; ++w) KEEP[w] = F[w] | __reduce_or_sync(FULL, (r0 ? bitword(m0, w) : 0u) | (r1 ? bitword(m1, w) : 0u));
    ws.anc[lane] = p0;
    if constexpr (TWO) ws.anc[lane + 32] = p1;
    __syncwarp();
    // an unmatched edge (k, j) survives iff j is kept above or owner(j) is in k's SCC
#pragma unroll
    for (int sl = 0; sl < (TWO ? 2 : 1); ++sl) {
        const bool h = sl ? h1 : h0;
        if (!h) continue;
        const int k = lane + 32 * sl, mk = sl ? m1 : m0, v = sl ? v1 : v0, sh = sl ? s1 : s0;
        const MS ak = sl ? p1 : p0;
        uint32_t rem[U];
        bool anyr = false;
#pragma unroll
        for (int w = 0; w < U; ++w) {
            uint32_t cand = (sl ? D1[w] : D0[w]) & ~KEEP[w] & ~bitword(mk, w);
            uint32_t x = cand;
            while (x) { // two candidates per step (independent owner / ancestor loads)
                const int bit = __ffs(x) - 1;
                x &= x - 1;
                const int bit2 = x ? __ffs(x) - 1 : bit;
                x &= x - 1;
                const int m = ws.owner[w * 32 + bit], m2 = ws.owner[w * 32 + bit2];
                const MS a1 = (MS)ws.anc[m], a2 = (MS)ws.anc[m2];
                if (((ak >> m) & 1u) && ((a1 >> k) & 1u)) cand &= ~(1u << bit);
                if (((ak >> m2) & 1u) && ((a2 >> k) & 1u)) cand &= ~(1u << bit2);
            }
            rem[w] = cand;
            anyr |= cand != 0;
        }
        if (anyr) {
            const int nvw = vwords<W>(M, v);
#pragma unroll
            for (int w = 0; w < W; ++w) { // back to the member's own bit positions
                if (w >= nvw) break;      // (unrolled: rem[] stays in registers)
                const uint32_t mword = sh ? shifted_word<U>(rem, w, -sh) : (w < U ? rem[w] : 0u);
                if (mword) atomicOr(rm + (size_t)v * W + w, mword);
            }
        }
        if (post) {
            if constexpr (U == W) {
#pragma unroll
                for (int w = 0; w < W; ++w)
                    post[(size_t)k * W + w] = dom[(size_t)v * W + w] & ~(sh ? shifted_word<U>(rem, w, -sh) : rem[w]);
            } else {
#pragma unroll
                for (int w = 0; w < U; ++w) post[(size_t)k * W + w] = (sl ? D1[w] : D0[w]) & ~rem[w];
            }
        }
    }
    if (post && lane == 0) *post_ok = 1;
    __syncwarp();
}

// prop_alldiff_fc (propagation.cpp:254-268): singleton values are removed from the other members
template <int W>
__device__ void prop_alldiff_fc(const DevModel& M, int a, const uint32_t* dom, uint32_t* rm, int lane) {
    const int b = M.ad_start[a], n = M.ad_start[a + 1] - b;
    const bool h0 = lane < n, h1 = lane + 32 < n;
    uint32_t D0[W], D1[W];
    int v0 = -1, v1 = -1, s0 = 0, s1 = 0;
    if (h0) {
        v0 = M.ad_var[b + lane];
        s0 = M.ad_shift[b + lane];
    }
    if (h1) {
        v1 = M.ad_var[b + lane + 32];
        s1 = M.ad_shift[b + lane + 32];
    }
#pragma unroll
    for (int w = 0; w < W; ++w) {
        D0[w] = h0 ? (s0 ? shifted_word<W>(dom + (size_t)v0 * W, w, s0) : dom[(size_t)v0 * W + w]) : 0u;
        D1[w] = h1 ? (s1 ? shifted_word<W>(dom + (size_t)v1 * W, w, s1) : dom[(size_t)v1 * W + w]) : 0u;
    }
    const bool g0 = h0 && dom_size<W>(D0) == 1, g1 = h1 && dom_size<W>(D1) == 1;
    const int x0 = g0 ? dom_first<W>(D0) : -1, x1 = g1 ? dom_first<W>(D1) : -1;
    uint32_t once0[W], once1[W];
#pragma unroll
    for (int w = 0; w < W; ++w) {
        once0[w] = __reduce_or_sync(FULL, bitword(x0, w));
        once1[w] = __reduce_or_sync(FULL, bitword(x1, w));
    }
    const unsigned q0 = __match_any_sync(FULL, g0 ? x0 : -(lane + 1));
    const unsigned q1 = __match_any_sync(FULL, g1 ? x1 : -(lane + 33));
    const bool dup0 = g0 && (__popc(q0) > 1 || testbit_r<W>(once1, x0));
    const bool dup1 = g1 && (__popc(q1) > 1 || testbit_r<W>(once0, x1));
#pragma unroll
    for (int sl = 0; sl < 2; ++sl) {
        const bool h = sl ? h1 : h0;
        if (!h) continue;
        const bool g = sl ? g1 : g0, dup = sl ? dup1 : dup0;
        const int x = sl ? x1 : x0, v = sl ? v1 : v0, sh = sl ? s1 : s0;
        uint32_t rem[W];
        bool anyr = false;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            uint32_t once = once0[w] | once1[w];
            uint32_t r = g ? ((once & ~bitword(x, w)) | (dup ? bitword(x, w) : 0u)) : once;
            rem[w] = r & (sl ? D1[w] : D0[w]);
            anyr |= rem[w] != 0;
        }
        if (anyr) {
#pragma unroll
            for (int w = 0; w < W; ++w) {
                uint32_t mword = sh ? shifted_word<W>(rem, w, -sh) : rem[w];
                if (mword) atomicOr(rm + (size_t)v * W + w, mword);
            }
        }
    }
}

// ------------------------------------------------------------------ AllDifferent, generic path
// Any member count / value-universe width (the fast path above covers <= 64 members and a
// universe of <= 1024 values). Same algorithm, working sets in a per-warp global scratch:
// BFS augmentation over explicit frontier lists, Warshall over n x n member bit rows.
struct BigScratch {
    uint32_t* D;     // [n][uw] member domains in the value universe
    uint32_t* anc;   // [n][nwm] ancestor sets
    int32_t* owner;  // [uw*32] matched value -> member
    int32_t* layer;  // [n]
    int32_t* fl;     // [2][n] BFS frontier lists
    uint32_t* vec;   // [6][uw] vis, nv, MV, F, KEEP, spare
    uint32_t* mset;  // [2][nwm] seed set, pivot set
    int32_t* cnt;    // [4]
};

__device__ inline BigScratch big_layout(uint32_t* base, int n, int uw) {
    const int nwm = (n + 31) / 32;
    BigScratch S;
    uint32_t* p = base;
    S.D = p;
    p += (size_t)n * uw;
    S.anc = p;
    p += (size_t)n * nwm;
    S.owner = reinterpret_cast<int32_t*>(p);
    p += (size_t)uw * 32;
    S.layer = reinterpret_cast<int32_t*>(p);
    p += n;
    S.fl = reinterpret_cast<int32_t*>(p);
    p += 2 * (size_t)n;
    S.vec = p;
    p += 6 * (size_t)uw;
    S.mset = p;
    p += 2 * (size_t)nwm;
    S.cnt = reinterpret_cast<int32_t*>(p);
    return S;
}

__device__ __forceinline__ bool bit_of(const uint32_t* v, int j) { return (v[j >> 5] >> (j & 31)) & 1u; }

// BFS augmenting path from member r over the generic layout; true on success
__device__ inline bool big_augment(int r, int n, int uw, const BigScratch& S, int16_t* mates, int lane) {
    uint32_t *vis = S.vec, *nv = S.vec + uw, *MV = S.vec + 2 * uw;
    for (int w = lane; w < uw; w += 32) vis[w] = 0;
    for (int k = lane; k < n; k += 32) S.layer[k] = -1;
    __syncwarp();
    if (lane == 0) {
        S.fl[0] = r;
        S.cnt[0] = 1;
        S.layer[r] = 0;
    }
    __syncwarp();
    int cur = 0, L = 0;
    for (;;) {
        const int c = S.cnt[cur];
        const int32_t* fr = S.fl + (size_t)cur * n;
        bool any = false;
        int found = 0x7fffffff;
        if (uw <= 4) { // narrow universe: frontier members over the lanes, one word at a time
            for (int w = 0; w < uw; ++w) {
                uint32_t acc = 0;
                for (int i = lane; i < c; i += 32) acc |= S.D[(size_t)fr[i] * uw + w];
                acc = __reduce_or_sync(FULL, acc);
                const uint32_t x = acc & ~vis[w];
                __syncwarp();
                if (lane == 0) {
                    nv[w] = x;
                    vis[w] |= x;
                }
                any |= x != 0;
                const uint32_t f = x & ~MV[w];
                if (f && found == 0x7fffffff) found = w * 32 + __ffs(f) - 1;
            }
        } else {
            for (int w = lane; w < uw; w += 32) {
                uint32_t acc = 0;
                for (int i = 0; i < c; ++i) acc |= S.D[(size_t)fr[i] * uw + w];
                const uint32_t x = acc & ~vis[w];
                nv[w] = x;
                vis[w] |= x;
                any |= x != 0;
                const uint32_t f = x & ~MV[w];
                if (f && found == 0x7fffffff) found = w * 32 + __ffs(f) - 1;
            }
        }
        any = __any_sync(FULL, any);
        found = __reduce_min_sync(FULL, (unsigned)found);
        if (!any) return false;
        if (found != 0x7fffffff) {
            int j = found;
            for (int l = L;; --l) {
                int best = 0x7fffffff;
                for (int k = lane; k < n; k += 32)
                    if (S.layer[k] == l && bit_of(S.D + (size_t)k * uw, j) && k < best) best = k;
                const int k = (int)__reduce_min_sync(FULL, (unsigned)best);
                const int old = mates[k];
                __syncwarp();
                if (lane == 0) {
                    mates[k] = (int16_t)j;
                    S.owner[j] = k;
                }
                __syncwarp();
                if (l == 0) break;
                j = old;
            }
            if (lane == 0) MV[found >> 5] |= 1u << (found & 31);
            __syncwarp();
            return true;
        }
        __syncwarp();
        if (lane == 0) S.cnt[cur ^ 1] = 0;
        __syncwarp();
        int32_t* nx = S.fl + (size_t)(cur ^ 1) * n;
        for (int w = lane; w < uw; w += 32) {
            uint32_t x = nv[w];
            while (x) {
                const int j = w * 32 + __ffs(x) - 1;
                x &= x - 1;
                const int k = S.owner[j];
                S.layer[k] = L + 1;
                nx[atomicAdd(&S.cnt[cur ^ 1], 1)] = k;
            }
        }
        __syncwarp();
        cur ^= 1;
        ++L;
    }
}

template <int W>
__device__ void big_load(const DevModel& M, int a, const uint32_t* dom, const BigScratch& S, int n, int uw, int lane) {
    const int b = M.ad_start[a];
    for (int k = lane; k < n; k += 32) {
        const uint32_t* dv = dom + (size_t)M.ad_var[b + k] * W;
        const int sh = M.ad_shift[b + k];
        for (int w = 0; w < uw; ++w) S.D[(size_t)k * uw + w] = shifted_word<W>(dv, w, sh);
    }
    __syncwarp();
}

// universe-space removals of member k back to its own bits
template <int W>
__device__ __forceinline__ void big_remove(uint32_t* rm, int v, int sh, int w, uint32_t cand) {
    while (cand) {
        const int vb = w * 32 + __ffs(cand) - 1 - sh;
        cand &= cand - 1;
        if (vb >= 0 && vb < W * 32) atomicOr(rm + (size_t)v * W + (vb >> 5), 1u << (vb & 31));
    }
}

template <int W>
__device__ void prop_alldiff_gac_big(const DevModel& M, int a, const uint32_t* dom, uint32_t* rm, int16_t* mates,
                                     uint32_t* scratch, int lane, int exact_wipe) {
    const int b = M.ad_start[a], n = M.ad_start[a + 1] - b, uw = M.ad_uw[a], nwm = (n + 31) / 32;
    const BigScratch S = big_layout(scratch, n, uw);
    uint32_t *MV = S.vec + 2 * uw, *F = S.vec + 3 * uw, *KEEP = S.vec + 4 * uw;
    uint32_t *SEED = S.mset, *PIV = S.mset + nwm;
    big_load<W>(M, a, dom, S, n, uw, lane);
    for (int w = lane; w < uw; w += 32) MV[w] = 0;
    __syncwarp();
    bool kept = false;
    for (int k = lane; k < n; k += 32) { // warm start: keep still-valid matched edges
        int m = mates[k];
        if (m >= 0 && !bit_of(S.D + (size_t)k * uw, m)) m = mates[k] = -1;
        if (m >= 0) {
            atomicOr(MV + (m >> 5), 1u << (m & 31));
            S.owner[m] = k;
            kept = true;
        }
    }
    // from an empty matching the loop below IS the greedy in member order (Kuhn's first failure)
    kept = __any_sync(FULL, kept);
    __syncwarp();
    int fail = -1;
    for (int base = 0; base < n && fail < 0; base += 32) {
        unsigned unm = __ballot_sync(FULL, base + lane < n && mates[base + lane] < 0);
        while (unm) {
            const int r = base + __ffs(unm) - 1;
            unm &= unm - 1;
            if (!big_augment(r, n, uw, S, mates, lane)) {
                fail = r;
                break;
            }
        }
    }
    if (fail >= 0) {
        if (exact_wipe && kept) { // greedy matching in member order: its first failure is Kuhn's
            for (int k = lane; k < n; k += 32) mates[k] = -1;
            for (int w = lane; w < uw; w += 32) MV[w] = 0;
            __syncwarp();
            for (int r = 0; r < n; ++r)
                if (!big_augment(r, n, uw, S, mates, lane)) {
                    fail = r;
                    break;
                }
        }
        if (lane == 0) {
            const int v = M.ad_var[b + fail];
            for (int w = 0; w < W; ++w) {
                const uint32_t d = dom[(size_t)v * W + w];
                if (d) atomicOr(rm + (size_t)v * W + w, d);
            }
        }
        __syncwarp();
        return;
    }
    // free values, predecessor rows, seeds, pivots
    if (uw <= 4) {
        for (int w = 0; w < uw; ++w) {
            uint32_t u = 0;
            for (int k = lane; k < n; k += 32) u |= S.D[(size_t)k * uw + w];
            u = __reduce_or_sync(FULL, u);
            if (lane == 0) {
                F[w] = u & ~MV[w];
                KEEP[w] = F[w];
            }
        }
    } else {
        for (int w = lane; w < uw; w += 32) {
            uint32_t u = 0;
            for (int k = 0; k < n; ++k) u |= S.D[(size_t)k * uw + w];
            F[w] = u & ~MV[w];
            KEEP[w] = F[w];
        }
    }
    for (int i = lane; i < 2 * nwm; i += 32) S.mset[i] = 0;
    __syncwarp();
    for (int k = lane; k < n; k += 32) {
        uint32_t* row = S.anc + (size_t)k * nwm;
        for (int i = 0; i < nwm; ++i) row[i] = 0;
        bool seed = false;
        int size = 0;
        for (int w = 0; w < uw; ++w) {
            const uint32_t d = S.D[(size_t)k * uw + w];
            size += __popc(d);
            seed |= (d & F[w]) != 0;
            uint32_t x = d & MV[w];
            while (x) {
                const int m = S.owner[w * 32 + __ffs(x) - 1];
                x &= x - 1;
                row[m >> 5] |= 1u << (m & 31);
            }
        }
        if (seed) atomicOr(SEED + (k >> 5), 1u << (k & 31));
        if (size > 1) atomicOr(PIV + (k >> 5), 1u << (k & 31));
    }
    __syncwarp();
    for (int pw = 0; pw < nwm; ++pw) { // Warshall over the non-singleton pivots
        uint32_t pm = PIV[pw];
        while (pm) {
            const int p = pw * 32 + __ffs(pm) - 1;
            pm &= pm - 1;
            const uint32_t* rp = S.anc + (size_t)p * nwm;
            for (int k = lane; k < n; k += 32) {
                uint32_t* rk = S.anc + (size_t)k * nwm;
                if (k != p && bit_of(rk, p))
                    for (int i = 0; i < nwm; ++i) rk[i] |= rp[i];
            }
            __syncwarp();
        }
    }
    for (int k = lane; k < n; k += 32) { // members reached from a free value keep their mate
        const uint32_t* rk = S.anc + (size_t)k * nwm;
        bool reached = bit_of(SEED, k);
        for (int i = 0; i < nwm && !reached; ++i) reached = (rk[i] & SEED[i]) != 0;
        const int m = mates[k];
        if (reached && m >= 0) atomicOr(KEEP + (m >> 5), 1u << (m & 31));
    }
    __syncwarp();
    for (int k = lane; k < n; k += 32) {
        const int v = M.ad_var[b + k], sh = M.ad_shift[b + k], mk = mates[k];
        const uint32_t* rk = S.anc + (size_t)k * nwm;
        for (int w = 0; w < uw; ++w) {
            uint32_t cand = S.D[(size_t)k * uw + w] & ~KEEP[w] & ~bitword(mk, w);
            uint32_t x = cand;
            while (x) {
                const int bit = __ffs(x) - 1;
                x &= x - 1;
                const int m = S.owner[w * 32 + bit];
                if (bit_of(rk, m) && bit_of(S.anc + (size_t)m * nwm, k)) cand &= ~(1u << bit);
            }
            if (cand) big_remove<W>(rm, v, sh, w, cand);
        }
    }
    __syncwarp();
}

template <int W>
__device__ void prop_alldiff_fc_big(const DevModel& M, int a, const uint32_t* dom, uint32_t* rm, uint32_t* scratch,
                                    int lane) {
    const int b = M.ad_start[a], n = M.ad_start[a + 1] - b, uw = M.ad_uw[a];
    const BigScratch S = big_layout(scratch, n, uw);
    uint32_t *once = S.vec, *twice = S.vec + uw;
    big_load<W>(M, a, dom, S, n, uw, lane);
    for (int w = lane; w < uw; w += 32) once[w] = twice[w] = 0;
    __syncwarp();
    for (int k = lane; k < n; k += 32) {
        int size = 0, j = -1;
        for (int w = 0; w < uw; ++w) {
            const uint32_t d = S.D[(size_t)k * uw + w];
            if (d && j < 0) j = w * 32 + __ffs(d) - 1;
            size += __popc(d);
        }
        if (size == 1) {
            const uint32_t old = atomicOr(once + (j >> 5), 1u << (j & 31));
            if (old & (1u << (j & 31))) atomicOr(twice + (j >> 5), 1u << (j & 31));
        }
        S.layer[k] = size == 1 ? j : -1;
    }
    __syncwarp();
    for (int k = lane; k < n; k += 32) {
        const int v = M.ad_var[b + k], sh = M.ad_shift[b + k], j = S.layer[k];
        for (int w = 0; w < uw; ++w) {
            const uint32_t own = bitword(j, w);
            uint32_t rem = (j >= 0 ? ((once[w] & ~own) | (twice[w] & own)) : once[w]) & S.D[(size_t)k * uw + w];
            if (rem) big_remove<W>(rm, v, sh, w, rem);
        }
    }
    __syncwarp();
}

// ------------------------------------------------------------------ one bulk-synchronous round
struct RoundCtx {
    uint32_t* dom;
    uint32_t* rm;
    int16_t* mates;     // [total_members] persistent warm-start matchings
    uint32_t* post;     // [total_members * W] GAC post-states (null: skip test disabled)
    int8_t* post_ok;    // [na]
    uint32_t* chg0;     // [ceil(n/32)] vars changed since the last fixpoint (round-1 triggers)
    uint32_t* chg1;     // [ceil(n/32)] second buffer (null: triggers disabled, full sweeps)
    bool ne_events;     // var-form != handled by the singleton-event path (search kernel)
    uint32_t* big;      // this block's generic-alldifferent scratch ([warps][M.big_words]) or null
    uint8_t* scratch;   // per-warp GAC scratch
    int scratch_stride; // bytes per warp
    const uint8_t* enabled;
    int alldiff;
    int exact_wipe;
};

template <int W>
__device__ __forceinline__ WarpScratch warp_scratch(const RoundCtx& R, int warp) {
    WarpScratch ws;
    uint8_t* base = R.scratch + (size_t)warp * R.scratch_stride;
    ws.layers = reinterpret_cast<unsigned long long*>(base);
    ws.anc = ws.layers + 66;
    ws.owner = reinterpret_cast<uint8_t*>(ws.anc + 64);
    return ws;
}


__device__ __forceinline__ bool trig_bit(const uint32_t* t, int v) { return (t[v >> 5] >> (v & 31)) & 1u; }

// Phase A: every triggered propagator against the frozen domains (trig == null: all of them).
// A propagator is triggered when a variable of its scope changed in the previous apply. An
// untriggered propagator sees exactly the domains of its last evaluation, whose removals are
// already applied, so skipping it changes no domain, no "changed" flag and no round count.
// *s_err receives DERR_OVERFLOW.
template <int W, int F, class SC>
__device__ __forceinline__ void run_propagators(const DevModel& M, const RoundCtx& R, volatile int* s_err,
                                                const uint32_t* trig, SC& sc) {
    const int tid = sc.tid(), T = sc.nthreads(), nw = sc.nwarps(), warp = sc.warp(), lane = threadIdx.x & 31;
    const int ad_warps = M.na < nw ? M.na : nw;
    const int prop_threads = nw > ad_warps ? (nw - ad_warps) * 32 : T;
    if (tid < prop_threads) {
        const int nr_loop = R.ne_events ? M.nr_gen : M.nr;
        for (int c = tid; c < nr_loop; c += prop_threads) {
            if (R.enabled && !R.enabled[c]) continue;
            if (trig) {
                const int2 xy = *reinterpret_cast<const int2*>(M.rb + c);
                if (!trig_bit(trig, xy.x) && (xy.y < 0 || !trig_bit(trig, xy.y))) continue;
            }
            prop_relbin<W>(M, c, R.dom, R.rm);
        }
        if (R.ne_events && M.nr_gen < M.nr) {
            // x != y + k prunes only from a singleton side, and a singleton that did not change in
            // the last apply has had its removals applied already: walk the incidence lists of the
            // variables that just became singletons (every singleton in the root's first round).
            const int pw = prop_threads >> 5;
            constexpr int NB = W * 32;
            for (int base = warp * 32; base < M.n; base += pw * 32) {
                // variables of this word that changed and have != edges (one word test per lane)
                const uint32_t cw = (trig ? trig[base >> 5] : 0xffffffffu) & M.ne_mask[base >> 5];
                if (cw == 0) continue;
                const int v = base + lane;
                int b = -1;
                if (v < M.n && ((cw >> lane) & 1u)) {
                    const uint32_t* dv = R.dom + (size_t)v * W;
                    const int nv = vwords<W>(M, v);
                    if (dom_size_n<W>(dv, nv) == 1) b = dom_first_n<W>(dv, nv);
                }
                unsigned ev = __ballot_sync(FULL, b >= 0);
                while (ev) {
                    const int l = __ffs(ev) - 1;
                    ev &= ev - 1;
                    const int vv = base + l, bb = __shfl_sync(FULL, b, l);
                    for (int e = M.ne_start[vv] + lane; e < M.ne_start[vv + 1]; e += 32) {
                        const int2 ps = M.ne_edge[e];
                        const int bit = bb + ps.y;
                        if (bit >= 0 && bit < NB) {
                            const uint32_t m = (1u << (bit & 31)) & R.dom[(size_t)ps.x * W + (bit >> 5)];
                            if (m) atomicOr(R.rm + (size_t)ps.x * W + (bit >> 5), m);
                        }
                    }
                }
            }
        }
        if constexpr ((F & F_LINEAR) != 0) {
            const int G = (F & F_LONG) != 0 ? M.lin_g : 1; // lean kernels: thread per sum, any arity
            if (G == 1) {
                for (int c = tid; c < M.nl; c += prop_threads) {
                    if (R.enabled && !R.enabled[M.nr + c]) continue;
                    if (trig) {
                        bool hit = false;
                        for (int t = M.lin_start[c]; t < M.lin_start[c + 1] && !hit; ++t) hit = trig_bit(trig, M.lin_var[t]);
                        if (!hit) continue;
                    }
                    const bool ok = (F & F_REGS) != 0 && M.lin_g == 1 ? prop_linear_small<W>(M, c, R.dom, R.rm)
                                                                         : prop_linear<W>(M, c, R.dom, R.rm);
                    if (!ok) *s_err = DERR_OVERFLOW;
                }
            } else { // lane groups of G: every lane of the warp iterates the same number of times
                const int gl = lane & (G - 1);
                const unsigned gmask = (G == 32 ? FULL : ((1u << G) - 1u)) << (lane & ~(G - 1));
                const int groups = prop_threads / G;
                for (int c0 = 0; c0 < M.nl; c0 += groups) {
                    const int c = c0 + tid / G;
                    bool run = c < M.nl && !(R.enabled && !R.enabled[M.nr + c]);
                    if (run && trig) {
                        bool hit = false;
                        for (int t = M.lin_start[c] + gl; t < M.lin_start[c + 1]; t += G) hit |= trig_bit(trig, M.lin_var[t]);
                        run = (__ballot_sync(gmask, hit) & gmask) != 0;
                    }
                    if (run && !prop_linear_group<W>(M, c, R.dom, R.rm, G, gl, gmask) && gl == 0) *s_err = DERR_OVERFLOW;
                }
            }
        }
        if constexpr ((F & F_TABLE) != 0)
        for (int c = tid; c < M.ntb; c += prop_threads) {
            if (trig && !trig_bit(trig, M.tb_xy[2 * c]) && !trig_bit(trig, M.tb_xy[2 * c + 1])) continue;
            prop_table2<W>(M, c, R.dom, R.rm);
        }
        if constexpr ((F & F_TABLE) != 0)
        for (int c = tid; c < M.ntn; c += prop_threads) {
            if (trig) {
                bool hit = false;
                for (int t = M.tn_start[c]; t < M.tn_start[c + 1] && !hit; ++t) hit = trig_bit(trig, M.tn_var[t]);
                if (!hit) continue;
            }
            prop_tablen<W>(M, c, R.dom, R.rm);
        }
    }
    if (warp >= nw - ad_warps) {
        const WarpScratch ws = warp_scratch<W>(R, threadIdx.x >> 5); // shared memory of this block
        for (int a = warp - (nw - ad_warps); a < M.na; a += ad_warps) {
            if (R.enabled && !R.enabled[M.nr + M.nl + a]) continue;
            // a round only runs after some variable changed, so an alldifferent over every
            // variable is always triggered
            if (trig && !(a < 32 && ((M.ad_full_mask >> a) & 1u))) {
                const int b = M.ad_start[a], e = M.ad_start[a + 1];
                bool hit = false;
                for (int t = b + lane; t < e; t += 32) hit |= trig_bit(trig, M.ad_var[t]);
                if (!__any_sync(FULL, hit)) continue;
            }
            if ((F & F_BIGAD) != 0 && M.ad_uw[a] > 0) { // generic path: many members or a wide universe
                uint32_t* scratch = R.big + (size_t)(SC::kGrid ? warp : (int)(threadIdx.x >> 5)) * M.big_words;
                if (R.alldiff) prop_alldiff_gac_big<W>(M, a, R.dom, R.rm, R.mates + M.ad_start[a], scratch, lane, R.exact_wipe);
                else prop_alldiff_fc_big<W>(M, a, R.dom, R.rm, scratch, lane);
            } else if (R.alldiff) {
                uint32_t* post = R.post ? R.post + (size_t)M.ad_start[a] * W : nullptr;
                const bool two = M.ad_start[a + 1] - M.ad_start[a] > 32;
                if (W > 1 && M.ad_uw[a] == -1) { // one-word universe under a wider W
                    if (!two)
                        prop_alldiff_gac<W, 1, false>(M, a, R.dom, R.rm, R.mates + M.ad_start[a], ws, lane, R.exact_wipe,
                                                      post, R.post_ok + a);
                    else
                        prop_alldiff_gac<W, 1, true>(M, a, R.dom, R.rm, R.mates + M.ad_start[a], ws, lane, R.exact_wipe,
                                                     post, R.post_ok + a);
                } else if (!two) {
                    prop_alldiff_gac<W, W, false>(M, a, R.dom, R.rm, R.mates + M.ad_start[a], ws, lane, R.exact_wipe, post,
                                                  R.post_ok + a);
                } else {
                    prop_alldiff_gac<W, W, true>(M, a, R.dom, R.rm, R.mates + M.ad_start[a], ws, lane, R.exact_wipe, post,
                                                 R.post_ok + a);
                }
            }
            else prop_alldiff_fc<W>(M, a, R.dom, R.rm, lane);
        }
    }
}

// Phase B: dom &= ~rm. Returns R_CHANGED / R_STABLE / R_FAILED / R_ERROR.
// failed_var (when non-null) receives the lowest empty var id on failure.
// full == false: every domain was non-empty when the round started (any node but the root's first
// round), so only a variable with removals can change or empty: the others are skipped on their
// removal words alone (one 16-byte load per four one-word variables), without touching dom.
template <int W, class SC>
__device__ __forceinline__ int apply_removals(const DevModel& M, const RoundCtx& R, volatile int* s_err,
                                              volatile int* s_min, int* failed_var, uint32_t* chg_out, SC& sc,
                                              bool full = true) {
    const int tid = sc.tid(), T = sc.nthreads();
    int changed = 0, empty_min = 0x7fffffff;
    auto one = [&](int v, uint32_t rw) { // one-word variable v with removals rw != 0
        uint32_t dw = R.dom[v];
        if (dw & rw) {
            dw &= ~rw;
            R.dom[v] = dw;
            changed = 1;
            if (chg_out) atomicOr(chg_out + (v >> 5), 1u << (v & 31));
        }
        R.rm[v] = 0;
        if (!dw && v < empty_min) empty_min = v;
    };
    if constexpr (W == 1) {
        if (!full) {
            const uint4* r4 = reinterpret_cast<const uint4*>(R.rm); // rows padded to 4 words
            for (int q = tid; q < ((M.n + 3) >> 2); q += T) {
                const uint4 rr = r4[q];
                if (!(rr.x | rr.y | rr.z | rr.w)) continue;
                const int v = q << 2;
                if (rr.x) one(v, rr.x);
                if (rr.y && v + 1 < M.n) one(v + 1, rr.y);
                if (rr.z && v + 2 < M.n) one(v + 2, rr.z);
                if (rr.w && v + 3 < M.n) one(v + 3, rr.w);
            }
        }
    }
    for (int v = tid; v < M.n && (full || W > 1); v += T) {
        uint32_t* d = R.dom + (size_t)v * W;
        uint32_t* r = R.rm + (size_t)v * W;
        uint32_t any = 0;
        bool vch = false;
        const int nv = vwords<W>(M, v);
        if (!full) { // no removal for this variable: nothing to apply, and it cannot be empty
            uint32_t rany = 0;
#pragma unroll
            for (int w = 0; w < W; ++w) {
                if (W > 4 && w >= nv) break;
                rany |= r[w];
            }
            if (!rany) continue;
        }
#pragma unroll
        for (int w = 0; w < W; ++w) {
            if (W > 4 && w >= nv) break;
            uint32_t rw = r[w], dw = d[w];
            if (rw) {
                if (dw & rw) {
                    vch = true;
                    dw &= ~rw;
                    d[w] = dw;
                }
                r[w] = 0;
            }
            any |= dw;
        }
        if (vch) {
            changed = 1;
            if (chg_out) atomicOr(chg_out + (v >> 5), 1u << (v & 31));
        }
        if (!any && v < empty_min) empty_min = v;
    }
    const int ch = sc.sync_or(changed);
    const int err = *s_err;
    if (err) return R_ERROR;
    if (!ch) return R_STABLE;
    const int em = sc.sync_or(empty_min != 0x7fffffff);
    if (!em) return R_CHANGED;
    if (failed_var) {
        if (tid == 0) *s_min = 0x7fffffff;
        sc.sync();
        if (empty_min != 0x7fffffff) atomicMin(const_cast<int*>(s_min), empty_min);
        sc.sync();
        *failed_var = *s_min;
        sc.sync();
    }
    return R_FAILED;
}

// propagate_fixpoint (propagation.cpp:516-532); *rounds counts every round including the last.
// first_all: evaluate every propagator in round 1; otherwise round 1 is triggered by the vars
// set in R.chg0 (the caller's branch decision). Both trigger buffers are left dirty.
template <int W, int F, class SC>
__device__ int block_fixpoint(const DevModel& M, const RoundCtx& R, volatile int* s_err, volatile int* s_min,
                              int max_rounds, int* rounds, int* failed_var, bool first_all, SC& sc) {
    const int tid = sc.tid(), T = sc.nthreads();
    const int nb = (M.n + 31) >> 5;
    uint32_t* cur = R.chg0;
    uint32_t* nxt = R.chg1;
    bool all = first_all || !R.chg1;
    int r = 0;
    for (;;) {
        if (nxt)
            for (int i = tid; i < nb; i += T) nxt[i] = 0;
        run_propagators<W, F>(M, R, s_err, all ? nullptr : cur, sc);
        sc.sync();
        const int st = apply_removals<W>(M, R, s_err, s_min, failed_var, nxt, sc, all && r == 0);
        ++r;
        if (st != R_CHANGED || (max_rounds > 0 && r >= max_rounds)) {
            *rounds = r;
            return st;
        }
        uint32_t* t = cur;
        cur = nxt;
        nxt = t;
        all = false;
    }
}

} // namespace dev
} // namespace cubics
