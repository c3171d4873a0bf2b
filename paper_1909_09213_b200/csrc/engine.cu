// Host orchestration of the device search engine and the solve / propagate entry points of the
// C ABI (include/cubics.h). The model is flattened once per call into the device layout of
// device_model.hpp, uploaded with one host->device copy, searched by one persistent kernel
// launch, and the results (stats, solutions) come back with a few device->host copies.
//
// There is no CPU fallback: without a usable sm_100 device every entry point returns
// CUBICS_E_CUDA with the CUDA error text in cubics_last_error().
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <map>
#include <memory>
#include <unordered_map>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include <cub/device/device_radix_sort.cuh>

#include "cubics.h"
#include "device_model.hpp"
#include "model.hpp"
#include "kernels.hpp"
#include "layout.hpp"

using namespace cubics;

namespace {

// NVTX ranges (Nsight timelines; near free without a tool attached): one per search launch,
// per exact-B&B phase, per shard and per bulk enumeration
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

#define CUBICS_CHECK_OK(call)                                                                      \
    do {                                                                                           \
        const int rc_ = (call);                                                                    \
        if (rc_ != CUBICS_OK) throw StatusError{rc_, #call};                                        \
    } while (0)

constexpr int kFastAllDiffMembers = 64;  // warp fast path; larger ones take the generic path
constexpr int kMaxAllDiffMembers = 4096;  // generic path limit (n x n member bit rows per warp)
constexpr long kMaxUniverseWords = 1024;  // generic path value universe (32768 values)
constexpr size_t kSmemBudget = 200 * 1024;
// shared task queue state (rank 0's HBM, IPC-mapped): 256-byte header + the cross-GPU pool
constexpr size_t kXsBytes = size_t(32) << 20;
constexpr size_t kQueueBytes = 256 + kXsBytes;

struct CudaError {
    std::string msg;
};

#define CU(call)                                                                               \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess) throw CudaError{std::string(#call) + ": " + cudaGetErrorString(e_)}; \
    } while (0)

struct StatusError {
    int code;
    std::string msg;
};

double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// ------------------------------------------------------------------ device arena (grow-only, per device)
struct Arena {
    void* ptr = nullptr;
    size_t cap = 0;
};
// one search at a time per device: the arenas below are reused by every call
std::recursive_mutex g_dev_mu[64];
Arena g_arena[3][64];
Arena g_pinned[2][64];

// slot 0: per-call search state; slot 1: solution-ordering scratch; slot 2: int64 solution rows
// (kept apart so growing one never invalidates another while both are live)
uint8_t* device_arena(int dev, size_t bytes, int slot = 0) {
    Arena& a = g_arena[slot][dev];
    if (a.cap < bytes) {
        if (a.ptr) cudaFree(a.ptr);
        a.ptr = nullptr;
        size_t want = std::max(bytes, a.cap * 3 / 2);
        CU(cudaMalloc(&a.ptr, want));
        a.cap = want;
    }
    return static_cast<uint8_t*>(a.ptr);
}

// slot 0: upload staging; slot 1: solution download (read by the caller under the device lock)
uint8_t* pinned_arena(int dev, size_t bytes, int slot = 0) {
    Arena& a = g_pinned[slot][dev];
    if (a.cap < bytes) {
        if (a.ptr) cudaFreeHost(a.ptr);
        a.ptr = nullptr;
        size_t want = std::max(bytes, a.cap * 3 / 2);
        CU(cudaMallocHost(&a.ptr, want));
        a.cap = want;
    }
    return static_cast<uint8_t*>(a.ptr);
}

// Pinned result arrays (cubics_enumerate): the int64 rows go from the device straight into one of
// these with a DMA copy, and cubics_solutions_free returns it here instead of freeing it, so the
// next call reuses it (a fresh 40 MB pinned allocation costs milliseconds).
class PinnedPool {
public:
    static PinnedPool& get() {
        static PinnedPool* p = new PinnedPool(); // never destroyed: buffers may outlive static teardown
        return *p;
    }
    int64_t* take(size_t bytes) {
        std::lock_guard<std::mutex> lk(mu_);
        size_t best = free_.size();
        for (size_t i = 0; i < free_.size(); ++i)
            if (free_[i].second >= bytes && (best == free_.size() || free_[i].second < free_[best].second)) best = i;
        void* p = nullptr;
        size_t cap = 0;
        if (best < free_.size()) {
            p = free_[best].first;
            cap = free_[best].second;
            free_.erase(free_.begin() + best);
        } else {
            cap = (std::max<size_t>(bytes, 8) + (size_t(2) << 20) - 1) & ~((size_t(2) << 20) - 1);
            if (cudaHostAlloc(&p, cap, cudaHostAllocPortable) != cudaSuccess) {
                cudaGetLastError();
                return nullptr;
            }
        }
        live_[p] = cap;
        return static_cast<int64_t*>(p);
    }
    bool give_back(void* p) {
        std::lock_guard<std::mutex> lk(mu_);
        auto it = live_.find(p);
        if (it == live_.end()) return false;
        free_.emplace_back(p, it->second);
        live_.erase(it);
        while (free_.size() > 3) { // keep a few for the calls to come
            cudaFreeHost(free_.front().first);
            free_.erase(free_.begin());
        }
        return true;
    }

private:
    std::mutex mu_;
    std::vector<std::pair<void*, size_t>> free_;
    std::unordered_map<void*, size_t> live_;
};

// Sum of the segments' stats (nodes, failures, rounds) whose root key is not right of K (all of
// them when K is null), except segment `skip`: the reference's DFS prefix up to K (search.cuh
// segments). On the device, so the host downloads three numbers, not every segment.
__global__ void seg_prefix_sum(const uint32_t* seg_key, const uint64_t* seg_st, uint64_t nseg, int KW,
                               const uint32_t* K, int64_t skip, unsigned long long* tot) {
    unsigned long long a = 0, b = 0, c = 0;
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < nseg; s += (uint64_t)gridDim.x * blockDim.x) {
        if ((int64_t)s == skip) continue;
        if (K) {
            int cmp = 0; // K vs root key of s
            for (int i = 0; i < KW && !cmp; ++i) {
                const uint32_t x = K[i], y = seg_key[s * KW + i];
                cmp = x < y ? -1 : (x > y ? 1 : 0);
            }
            if (cmp < 0) continue; // right of K
        }
        a += seg_st[s * 3 + 0];
        b += seg_st[s * 3 + 1];
        c += seg_st[s * 3 + 2];
    }
    for (int o = 16; o; o >>= 1) {
        a += __shfl_down_sync(0xffffffffu, a, o);
        b += __shfl_down_sync(0xffffffffu, b, o);
        c += __shfl_down_sync(0xffffffffu, c, o);
    }
    if ((threadIdx.x & 31) == 0 && (a | b | c)) {
        atomicAdd(tot + 0, a);
        atomicAdd(tot + 1, b);
        atomicAdd(tot + 2, c);
    }
}

__global__ void rows_to_int64(const uint16_t* rows, const int64_t* off, int nv, uint64_t count, int64_t* out) {
    const uint64_t total = count * (uint64_t)nv;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = off[i % nv] + (int64_t)rows[i];
}

// host-mapped pinned memory (streaming event ring), grow-only per device
Arena g_mapped[64];
uint8_t* mapped_arena(int dev, size_t bytes) {
    Arena& a = g_mapped[dev];
    if (a.cap < bytes) {
        if (a.ptr) cudaFreeHost(a.ptr);
        a.ptr = nullptr;
        a.cap = 0;
        CU(cudaHostAlloc(&a.ptr, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
        a.cap = bytes;
    }
    return static_cast<uint8_t*>(a.ptr);
}

// ------------------------------------------------------------------ flattening to the device layout
struct Blob { // host staging of every device array, packed with 16-byte alignment
    std::vector<uint8_t> bytes;
    template <class T>
    size_t add(const T* p, size_t n) {
        size_t at = (bytes.size() + 15) & ~size_t(15);
        bytes.resize(at + std::max<size_t>(n * sizeof(T), 16), 0);
        if (n) std::memcpy(bytes.data() + at, p, n * sizeof(T));
        return at;
    }
};

struct Prepared {
    int W = 1;
    int n = 0;
    size_t NWP = 4;
    int nr = 0, nl = 0, na = 0, total_members = 0;
    bool has_empty = false;
    uint64_t depth_bound = 0; // sum(|D| - 1): max binary-tree depth
    Blob blob;
    size_t o_vw = 0;
    size_t o_neq = 0;
    bool warp_ok = false;     // search_kernel_warp eligible: n <= 32, W = 1, small alldifferents, no tables
    bool mixed_width = false; // some variable needs <= W/4 words: per-variable word counts pay
    size_t o_off, o_dom, o_rb, o_ls, o_lo, o_lb, o_lv, o_lc, o_as, o_av, o_ash, o_nes, o_nee, o_auw, o_nem;
    size_t o_tbxy, o_tboff, o_tbsup, o_tns, o_tnv, o_tnn, o_tno, o_tnd;
    int ntb = 0, ntn = 0;
    size_t big_words = 0;
    int nr_gen = 0;
    int lin_g = 1;
    uint32_t ad_full_mask = 0;
    std::vector<int> kind_index; // constraint index -> kind-local index (rb | nr+lin | nr+nl+ad)
    std::vector<int64_t> offsets;
    DevModel bind(const uint8_t* base) const {
        DevModel M{};
        M.n = n;
        M.W = W;
        M.off = reinterpret_cast<const int64_t*>(base + o_off);
        M.init_dom = reinterpret_cast<const uint32_t*>(base + o_dom);
        M.vw = mixed_width ? reinterpret_cast<const int32_t*>(base + o_vw) : nullptr;
        M.nr = nr;
        M.rb = reinterpret_cast<const RelBinRec*>(base + o_rb);
        M.nr_gen = nr_gen;
        M.ne_start = reinterpret_cast<const int32_t*>(base + o_nes);
        M.ne_edge = reinterpret_cast<const int2*>(base + o_nee);
        M.ne_mask = reinterpret_cast<const uint32_t*>(base + o_nem);
        M.neq = warp_ok && nr_gen < nr ? reinterpret_cast<const unsigned long long*>(base + o_neq) : nullptr;
        M.nl = nl;
        M.lin_start = reinterpret_cast<const int32_t*>(base + o_ls);
        M.lin_op = reinterpret_cast<const int32_t*>(base + o_lo);
        M.lin_bound = reinterpret_cast<const int64_t*>(base + o_lb);
        M.lin_var = reinterpret_cast<const int32_t*>(base + o_lv);
        M.lin_coeff = reinterpret_cast<const int64_t*>(base + o_lc);
        M.lin_g = lin_g;
        M.na = na;
        M.ad_full_mask = ad_full_mask;
        M.ad_start = reinterpret_cast<const int32_t*>(base + o_as);
        M.ad_var = reinterpret_cast<const int32_t*>(base + o_av);
        M.ad_shift = reinterpret_cast<const int32_t*>(base + o_ash);
        M.ad_uw = reinterpret_cast<const int32_t*>(base + o_auw);
        M.big_words = static_cast<int32_t>(big_words);
        M.ntb = ntb;
        M.tb_xy = reinterpret_cast<const int32_t*>(base + o_tbxy);
        M.tb_off = reinterpret_cast<const int64_t*>(base + o_tboff);
        M.tb_sup = reinterpret_cast<const uint32_t*>(base + o_tbsup);
        M.ntn = ntn;
        M.tn_start = reinterpret_cast<const int32_t*>(base + o_tns);
        M.tn_var = reinterpret_cast<const int32_t*>(base + o_tnv);
        M.tn_nt = reinterpret_cast<const int64_t*>(base + o_tnn);
        M.tn_off = reinterpret_cast<const int64_t*>(base + o_tno);
        M.tn_data = reinterpret_cast<const int16_t*>(base + o_tnd);
        M.total_members = total_members;
        return M;
    }
};

void words_to_u32(const HostModel& m, int v, const uint64_t* src64, uint32_t* dst, int W) {
    const int nw64 = m.word_start[v + 1] - m.word_start[v];
    for (int w = 0; w < W; ++w) {
        uint64_t x = (w / 2 < nw64) ? src64[m.word_start[v] + w / 2] : 0;
        dst[(size_t)v * W + w] = static_cast<uint32_t>(w % 2 ? x >> 32 : x);
    }
}

// check_ranges: the device engine limits
void prepare(const HostModel& m, const uint64_t* words, Prepared& P) {
    const int n = m.n_vars();
    P.n = n;
    int need = 1;
    for (int v = 0; v < n; ++v) need = std::max(need, (m.width[v] + 31) / 32);
    // constraint tables
    std::vector<RelBinRec> rb;
    std::vector<int32_t> ls{0}, lo, lv, as{0}, av, ash;
    std::vector<int64_t> lb, lc;
    P.kind_index.assign(m.n_cons(), 0);
    std::vector<int> ad_cons, tables2;
    std::vector<int32_t> tn_start{0}, tn_var;
    std::vector<int64_t> tn_nt, tn_off;
    std::vector<int16_t> tn_data;
    for (int c = 0; c < m.n_cons(); ++c) {
        const int b = m.con_start[c], e = m.con_start[c + 1];
        switch (m.con_kind[c]) {
        case CUBICS_RELBIN: {
            // fold the int64 arithmetic of prop_rel_bin (propagation.cpp:126-192) into one clamped
            // bit offset; any value beyond +-4096 bits behaves identically on <= 1024-bit domains
            auto clampi = [](__int128 v, long lo, long hi) {
                return static_cast<int32_t>(v < lo ? lo : (v > hi ? hi : v));
            };
            auto wrap = [](int64_t a, int64_t b) { return (int64_t)((uint64_t)a + (uint64_t)b); };
            RelBinRec r{};
            r.x = m.term_var[b];
            r.y = e - b == 2 ? m.term_var[b + 1] : -1;
            r.op = m.con_op[c];
            const int64_t k = m.con_value[c];
            const __int128 offx = m.offset[r.x];
            if (r.y >= 0) {
                r.s = clampi((__int128)m.offset[r.y] + k - offx, -4096, 4096);
            } else {
                __int128 lit = k;
                if (r.op == CUBICS_LE) lit = wrap(k, 1);  // remove [lit+1, max]
                if (r.op == CUBICS_GE) lit = wrap(k, -1); // remove [min, lit-1]
                r.s = clampi(lit - offx, -1, 2048);
            }
            P.kind_index[c] = static_cast<int>(rb.size());
            rb.push_back(r);
            break;
        }
        case CUBICS_LINEAR: {
            if (m.con_op[c] == CUBICS_LIN_EQ) {
                bool bad = m.con_value[c] == std::numeric_limits<int64_t>::min();
                for (int t = b; t < e; ++t) bad = bad || m.term_coeff[t] == std::numeric_limits<int64_t>::min();
                if (bad) throw StatusError{CUBICS_E_OVERFLOW, "overflow in linear propagation"};
            }
            P.kind_index[c] = static_cast<int>(lo.size());
            lo.push_back(m.con_op[c]);
            lb.push_back(m.con_value[c]);
            for (int t = b; t < e; ++t) {
                lv.push_back(m.term_var[t]);
                lc.push_back(m.term_coeff[t]);
            }
            ls.push_back(static_cast<int32_t>(lv.size()));
            break;
        }
        case CUBICS_TABLE: {
            const int k = e - b;
            const int64_t nt = m.con_value[c];
            const int64_t* data = m.table_data.data() + m.table_start[c];
            if (k == 2) { // support bitsets: row a of x's block = the y bits allowed with x = a
                tables2.push_back(c);
            } else {
                if (k > 8) throw StatusError{CUBICS_E_UNSUPPORTED, "table constraint of arity > 8"};
                tn_off.push_back(static_cast<int64_t>(tn_data.size()));
                tn_nt.push_back(nt);
                for (int64_t i = 0; i < nt; ++i)
                    for (int j = 0; j < k; ++j) {
                        const int v = m.term_var[b + j];
                        const __int128 pos = (__int128)data[i * k + j] - m.offset[v];
                        tn_data.push_back(pos >= 0 && pos < m.width[v] ? static_cast<int16_t>(pos) : int16_t(-1));
                    }
                for (int j = 0; j < k; ++j) tn_var.push_back(m.term_var[b + j]);
                tn_start.push_back(static_cast<int32_t>(tn_var.size()));
            }
            break;
        }
        default:
            ad_cons.push_back(c);
            break;
        }
    }
    std::vector<int32_t> auw;
    size_t big_words = 0;
    for (int c : ad_cons) {
        const int b = m.con_start[c], e = m.con_start[c + 1];
        if (e - b > kMaxAllDiffMembers)
            throw StatusError{CUBICS_E_UNSUPPORTED, "alldifferent with more than 4096 members"};
        __int128 uoff = 0, uend = 0;
        for (int t = b; t < e; ++t) {
            const int v = m.term_var[t];
            __int128 o = m.offset[v], en = (__int128)m.offset[v] + m.width[v];
            if (t == b || o < uoff) uoff = o;
            if (t == b || en > uend) uend = en;
        }
        const __int128 span = uend - uoff;
        const long uwords = static_cast<long>((span + 31) / 32);
        if (uwords > kMaxUniverseWords)
            throw StatusError{CUBICS_E_UNSUPPORTED, "alldifferent value universe wider than 32768 values"};
        if (e - b <= kFastAllDiffMembers && span <= 32 * 32) {
            need = std::max(need, static_cast<int>(uwords));
            auw.push_back(-static_cast<int32_t>(std::max(1L, uwords))); // fast path, universe words
        } else {
            auw.push_back(static_cast<int32_t>(uwords));
            big_words = std::max(big_words, dev::big_scratch_words(e - b, static_cast<int>(uwords)));
        }
        P.kind_index[c] = static_cast<int>(as.size()) - 1;
        for (int t = b; t < e; ++t) {
            av.push_back(m.term_var[t]);
            ash.push_back(static_cast<int32_t>(m.offset[m.term_var[t]] - uoff));
        }
        as.push_back(static_cast<int32_t>(av.size()));
    }
    P.big_words = (big_words + 3) & ~size_t(3);
    int W = 1;
    while (W < need) W *= 2;
    if (W > 32) throw StatusError{CUBICS_E_UNSUPPORTED, "domain wider than 1024 values"};
    P.W = W;
    P.NWP = dev::round4((size_t)std::max(n, 1) * W);
    std::vector<int32_t> tb_xy;
    std::vector<int64_t> tb_off;
    std::vector<uint32_t> tb_sup;
    for (int c : tables2) {
        const int b = m.con_start[c], x = m.term_var[b], y = m.term_var[b + 1];
        const int64_t nt = m.con_value[c];
        const int64_t* data = m.table_data.data() + m.table_start[c];
        const size_t ox = tb_sup.size(), oy = ox + (size_t)m.width[x] * W;
        tb_sup.resize(oy + (size_t)m.width[y] * W, 0);
        for (int64_t i = 0; i < nt; ++i) {
            const __int128 a = (__int128)data[2 * i] - m.offset[x], bb = (__int128)data[2 * i + 1] - m.offset[y];
            if (a < 0 || a >= m.width[x] || bb < 0 || bb >= m.width[y]) continue;
            tb_sup[ox + (size_t)a * W + (size_t)(bb >> 5)] |= 1u << (int)(bb & 31);
            tb_sup[oy + (size_t)bb * W + (size_t)(a >> 5)] |= 1u << (int)(a & 31);
        }
        tb_xy.push_back(x);
        tb_xy.push_back(y);
        tb_off.push_back(static_cast<int64_t>(ox));
        tb_off.push_back(static_cast<int64_t>(oy));
    }
    P.ntb = static_cast<int>(tables2.size());
    P.ntn = static_cast<int>(tn_nt.size());
    P.nr = static_cast<int>(rb.size());
    P.nl = static_cast<int>(lo.size());
    // lanes per linear sum: one thread for short sums, else a lane group of pow2ceil(max terms)
    // (<= 32; longer sums loop over 32-term chunks) scanning its terms in parallel
    int max_terms = 0;
    for (int c = 0; c < P.nl; ++c) max_terms = std::max(max_terms, ls[c + 1] - ls[c]);
    P.lin_g = 1;
    if (max_terms > 4)
        while (P.lin_g < max_terms && P.lin_g < 32) P.lin_g *= 2;
    P.na = static_cast<int>(as.size()) - 1;
    P.ad_full_mask = 0;
    for (int a = 0; a < P.na && a < 32; ++a) {
        std::vector<char> seen(n, 0);
        int cnt = 0;
        for (int t = as[a]; t < as[a + 1]; ++t)
            if (!seen[av[t]]) {
                seen[av[t]] = 1;
                ++cnt;
            }
        if (cnt == n) P.ad_full_mask |= 1u << a;
    }
    P.total_members = static_cast<int>(av.size());
    std::vector<uint32_t> dom(P.NWP, 0);
    P.depth_bound = 0;
    P.has_empty = false;
    for (int v = 0; v < n; ++v) {
        words_to_u32(m, v, words, dom.data(), W);
        int sz = 0;
        for (int w = 0; w < W; ++w) sz += __builtin_popcount(dom[(size_t)v * W + w]);
        if (sz == 0) P.has_empty = true;
        P.depth_bound += sz > 0 ? (uint64_t)(sz - 1) : 0;
    }
    // generic RelBin records first; var-form != records last, mirrored into a per-variable
    // incidence list for the singleton-event path of the search kernel
    std::stable_partition(rb.begin(), rb.end(), [](const RelBinRec& r) { return !(r.y >= 0 && r.op == CUBICS_NE); });
    P.nr_gen = static_cast<int>(std::count_if(rb.begin(), rb.end(), [](const RelBinRec& r) { return !(r.y >= 0 && r.op == CUBICS_NE); }));
    std::vector<int32_t> nes(n + 1, 0);
    for (size_t i = P.nr_gen; i < rb.size(); ++i) {
        nes[rb[i].y + 1]++; // y singleton -> removes from x
        nes[rb[i].x + 1]++; // x singleton -> removes from y
    }
    for (int v = 0; v < n; ++v) nes[v + 1] += nes[v];
    std::vector<int2> nee(nes[n]);
    std::vector<int32_t> fill(nes.begin(), nes.end() - 1);
    for (size_t i = P.nr_gen; i < rb.size(); ++i) {
        nee[fill[rb[i].y]++] = make_int2(rb[i].x, rb[i].s);
        nee[fill[rb[i].x]++] = make_int2(rb[i].y, -rb[i].s);
    }
    P.offsets = m.offset;
    P.o_off = P.blob.add(m.offset.data(), m.offset.size());
    P.o_dom = P.blob.add(dom.data(), dom.size());
    {
        std::vector<int32_t> vw(std::max(n, 1), 1);
        for (int v = 0; v < n; ++v) {
            vw[v] = std::max(1, std::min(W, (m.width[v] + 31) / 32));
            if (W >= 8 && vw[v] * 4 <= W) P.mixed_width = true;
        }
        P.o_vw = P.blob.add(vw.data(), vw.size());
    }
    P.o_rb = P.blob.add(rb.data(), rb.size());
    P.o_ls = P.blob.add(ls.data(), ls.size());
    P.o_lo = P.blob.add(lo.data(), lo.size());
    P.o_lb = P.blob.add(lb.data(), lb.size());
    P.o_lv = P.blob.add(lv.data(), lv.size());
    P.o_lc = P.blob.add(lc.data(), lc.size());
    P.o_as = P.blob.add(as.data(), as.size());
    P.o_av = P.blob.add(av.data(), av.size());
    P.o_ash = P.blob.add(ash.data(), ash.size());
    P.o_auw = P.blob.add(auw.data(), auw.size());
    P.o_tbxy = P.blob.add(tb_xy.data(), tb_xy.size());
    P.o_tboff = P.blob.add(tb_off.data(), tb_off.size());
    P.o_tbsup = P.blob.add(tb_sup.data(), tb_sup.size());
    P.o_tns = P.blob.add(tn_start.data(), tn_start.size());
    P.o_tnv = P.blob.add(tn_var.data(), tn_var.size());
    P.o_tnn = P.blob.add(tn_nt.data(), tn_nt.size());
    P.o_tno = P.blob.add(tn_off.data(), tn_off.size());
    P.o_tnd = P.blob.add(tn_data.data(), tn_data.size());
    P.o_nes = P.blob.add(nes.data(), nes.size());
    P.o_nee = P.blob.add(nee.data(), nee.size());
    std::vector<uint32_t> nem(((size_t)n + 31) / 32 + 1, 0u); // variables with != edges, one bit each
    for (int v = 0; v < n; ++v)
        if (nes[v] < nes[v + 1]) nem[v >> 5] |= 1u << (v & 31);
    P.o_nem = P.blob.add(nem.data(), nem.size());
    // warp contexts (warp_ctx.cuh): one lane per variable, one-word domains and alldifferent
    // universes, <= 32 members per alldifferent, no tables or generic-path alldifferents
    int max_members = 0;
    for (int a = 0; a < P.na; ++a) max_members = std::max(max_members, as[a + 1] - as[a]);
    P.warp_ok = n >= 1 && n <= 32 && W == 1 && P.ntb + P.ntn == 0 && P.big_words == 0 && max_members <= 32;
    if (P.warp_ok && P.nr_gen < P.nr) {
        // the != edges u -> p with shift s in [-31, 31] as bit s + 32 of neq[u*n + p] (other shifts
        // can never hit a one-word domain)
        std::vector<unsigned long long> neq((size_t)n * n, 0);
        for (int u = 0; u < n; ++u)
            for (int e = nes[u]; e < nes[u + 1]; ++e)
                if (nee[e].y >= -31 && nee[e].y <= 31) neq[(size_t)u * n + nee[e].x] |= 1ull << (nee[e].y + 32);
        P.o_neq = P.blob.add(neq.data(), neq.size());
    }
}

// per-device state created once: capability check, one non-blocking stream, timing events
struct DevState {
    bool checked = false;
    bool ok = false;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr; // streaming: the stop flag is written on this stream mid-kernel
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    bool streaming = false;      // a callback of a streaming search is running on this device
};
DevState g_dev[64];
int g_count = -1;

int current_device(int want) {
    if (g_count < 0) {
        int count = 0;
        CU(cudaGetDeviceCount(&count));
        g_count = count;
    }
    if (g_count == 0) throw CudaError{"no CUDA device"};
    int dev = want;
    if (dev < 0) CU(cudaGetDevice(&dev));
    if (dev >= g_count || dev >= 64) throw CudaError{"device ordinal out of range"};
    CU(cudaSetDevice(dev));
    DevState& s = g_dev[dev];
    if (!s.checked) {
        int major = 0;
        CU(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
        s.ok = major >= 10;
        s.checked = true;
        if (s.ok) {
            CU(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
            CU(cudaStreamCreateWithFlags(&s.side, cudaStreamNonBlocking));
            CU(cudaEventCreate(&s.e0));
            CU(cudaEventCreate(&s.e1));
        }
    }
    if (!s.ok) throw CudaError{"device is not sm_100 class (Blackwell)"};
    return dev;
}

// ------------------------------------------------------------------ kernel dispatch over W
#define CUBICS_DISPATCH_W(W, CALL)                                                                  \
    switch (W) {                                                                                   \
    case 1: CU(CALL(1)); break;                                                                    \
    case 2: CU(CALL(2)); break;                                                                    \
    case 4: CU(CALL(4)); break;                                                                    \
    case 8: CU(CALL(8)); break;                                                                    \
    case 16: CU(CALL(16)); break;                                                                  \
    case 32: CU(CALL(32)); break;                                                                  \
    default: throw StatusError{CUBICS_E_UNSUPPORTED, "bad word count"};                            \
    }

int parity_block(const Prepared& P) {
    const int work = P.nr + P.nl + P.ntb + P.ntn;
    int prop_warps = std::min(16, std::max(1, (work + 31) / 32));
    int ad_warps = std::min(P.na, 8);
    int apply_warps = std::min(16, std::max(1, (P.n + 63) / 64));
    int warps = std::max(prop_warps + ad_warps, apply_warps);
    return std::min(1024, 32 * warps);
}

// ------------------------------------------------------------------ solution ordering on the device
__global__ void iota_kernel(uint32_t* p, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = (uint32_t)i;
}

__global__ void gather_key_word(const uint32_t* keys, int KW, int w, const uint32_t* perm, uint32_t* out, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = keys[(uint64_t)perm[i] * KW + w];
}

__global__ void permute_rows(const uint16_t* in, const uint32_t* perm, int nv, uint64_t n, uint16_t* out) {
    const uint64_t total = n * (uint64_t)nv;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = i / nv, c = i % nv;
        out[i] = in[(uint64_t)perm[r] * nv + c];
    }
}

// LSD radix sort of the path keys (only the words that can differ), then one gather of the
// solution rows: the reference's DFS order without any host-side sort.
const uint16_t* order_on_device(int dev, const uint32_t* keys, int KW, int used_words, const uint16_t* vals, int nv,
                                uint64_t count, cudaStream_t st, uint64_t* launches) {
    size_t temp = 0;
    CU(cub::DeviceRadixSort::SortPairs(nullptr, temp, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                       (uint32_t*)nullptr, (int)count, 0, 32, st));
    size_t off = 0;
    auto take = [&](size_t b) {
        size_t at = (off + 255) & ~size_t(255);
        off = at + std::max<size_t>(b, 16);
        return at;
    };
    const size_t a_p0 = take(4 * count), a_p1 = take(4 * count), a_k0 = take(4 * count), a_k1 = take(4 * count),
                 a_t = take(temp), a_out = take(sizeof(uint16_t) * nv * count);
    uint8_t* b = device_arena(dev, off, 1);
    uint32_t *p0 = (uint32_t*)(b + a_p0), *p1 = (uint32_t*)(b + a_p1), *k0 = (uint32_t*)(b + a_k0),
             *k1 = (uint32_t*)(b + a_k1);
    const int grid = (int)std::min<uint64_t>(4096, (count + 255) / 256);
    iota_kernel<<<grid, 256, 0, st>>>(p0, count);
    ++*launches;
    for (int w = used_words - 1; w >= 0; --w) {
        gather_key_word<<<grid, 256, 0, st>>>(keys, KW, w, p0, k0, count);
        ++*launches;
        CU(cub::DeviceRadixSort::SortPairs(b + a_t, temp, k0, k1, p0, p1, (int)count, 0, 32, st));
        std::swap(p0, p1);
    }
    const int g2 = (int)std::min<uint64_t>(8192, (count * nv + 255) / 256);
    uint16_t* out = (uint16_t*)(b + a_out);
    permute_rows<<<std::max(g2, 1), 256, 0, st>>>(vals, p0, nv, count, out);
    ++*launches;
    CU(cudaGetLastError());
    return out;
}

struct Records { // solutions copied back from the device
    uint64_t count = 0;
    bool ordered = false; // vals already in the reference's DFS order
    std::vector<uint16_t> vals;
    const uint16_t* pinned = nullptr; // when set, the rows live in pinned slot 1 instead of vals
    const uint16_t* rows() const { return pinned ? pinned : vals.data(); }
    void materialize(size_t n) {
        if (pinned) vals.assign(pinned, pinned + count * n);
        pinned = nullptr;
    }
    std::vector<uint32_t> keys;
    std::vector<uint64_t> stats;
    std::vector<int32_t> seg; // segment bookkeeping: each solution's segment (stats: segment-local)
};

struct RunOut {
    WorkState ws{};
    Records rec;
    int engine = CUBICS_ENGINE_PARITY;
    int contexts = 1;
    int KW = 0;
    double device_ms = 0;
    uint64_t h2d = 0, d2h = 0, launches = 0;
    bool pinned_rows = false; // in: download solution rows into pinned slot 1 (cubics_enumerate)
    bool int64_rows = false;  // in: rows converted to int64 on the device, DMA'd into values64
    int64_t* values64 = nullptr; // out: a PinnedPool buffer holding rec.count rows (int64_rows)
    std::vector<uint16_t> inc_vals;
    std::vector<uint32_t> first_key;  // parallel: DFS-first solution key/values
    std::vector<uint16_t> first_vals;
    bool has_first = false;
};

// Multi-GPU sharding plumbing.
struct ShardIO {
    int split_depth = -1;        // > 0: frontier expansion; open nodes at this depth become tasks
    uint64_t task_cap = 0;
    uint32_t* task_dev = nullptr; // [task_cap][OS] device buffer (arena slot 1)
    uint64_t n_tasks = 0;         // out: tasks emitted
    const std::vector<int32_t>* seeds = nullptr; // seeded run: task indices of this shard
    unsigned int* claim = nullptr; // shared queue: seeds are claimed through this counter instead
    unsigned long long* g_inc = nullptr; // multi-GPU B&B: shared incumbent (queue state, IPC-mapped)
    unsigned long long* g_first = nullptr; // sharded first solution: best key prefix of all ranks
    uint8_t* xs = nullptr; // cross-GPU stealing: the shared queue state (XsCtl at +128, pool at +256)
    // exact parallel B&B (exact_bnb): phase 0 is an exact first solution over the whole tree
    // (root_first); every phase keeps its starting bound (static_bound); a guided replay run
    // (guide_key, reference-order kernel) emits the pending right branches of a recorded path
    bool root_first = false;
    bool static_bound = false;
    bool prefix_sum = false; // seeded exact-first run: best solution and prefix stats as for first mode
    const std::vector<uint32_t>* guide_key = nullptr;
    std::vector<int64_t> guide_bound; // [KW * 32 + 1]
    std::vector<int32_t> guide_has;
    // sharded first solution: 1 = seeded run with the exact-first bookkeeping (segments,
    // abandoning right of this rank's best); 2 = frontier expansion with segments only
    int first = 0;
    // out (first != 0): segments [n_seg] (root keys, stats), solutions' segments / snapshots in
    // RunOut::rec, frontier tasks' [n_tasks][4] (segment, nodes, failures, rounds) in emission order
    uint64_t n_seg = 0;
    std::vector<uint32_t> seg_key;
    std::vector<uint64_t> seg_st;
    std::vector<uint64_t> task_snap;
};

// Batched B&B (cubics_solve_optimize_batch): problem i = block i, reference node order.
struct BatchIO {
    int count = 0;
    const uint64_t* words = nullptr; // [count][model words] desc packing
    std::vector<uint32_t> dom;      // [count][NWP] device layout (filled by run_search)
    std::vector<int64_t> bound;     // [count]
    std::vector<int32_t> has_bound; // [count]
    bool any_empty = false;
    // out
    std::vector<uint64_t> stats;    // [count][4]
    std::vector<int32_t> flags;     // [count] bit0 limit hit, bit1 incumbent
    std::vector<uint16_t> inc;      // [count][n]
};

// Streaming delivery (cubics_solve_satisfy with a callback; search.cpp:134-156): the kernel
// writes solution / segment events into a host-mapped ring (search.cuh EvKind) and the calling
// thread runs the callback while the search goes on. visit(row, stats) gets each solution's bit
// indices and the reference's (nodes, failures, rounds) at its emission; false stops the search.
struct StreamIO {
    std::function<bool(const uint16_t* row, const uint64_t* stats)> visit;
    // out
    bool stopped = false;
    uint64_t delivered = 0;
    uint64_t stop_stats[3] = {0, 0, 0};
};

// Puts the parallel engine's events back into DFS order. Segments (the root = 0, each handed-out
// subtree = ring ticket + 1) are contiguous DFS intervals ordered by root key; the cursor is the
// leftmost unfinished one. Its solutions go out as they arrive, the others' wait in host memory;
// when the cursor finishes, every segment left of the next one has been announced (a donor's
// EV_NEW precedes its EV_END), so the next key in the map is the next interval.
class SegmentOrder {
public:
    SegmentOrder(int KW, int n, StreamIO& io) : KW_(KW), n_(n), io_(io) {
        Seg& root = segs_[0];
        root.key.assign(KW, 0u);
        order_.emplace(root.key, 0u);
    }
    void on_new(uint32_t id, const uint32_t* key) {
        std::vector<uint32_t> k(key, key + KW_);
        if (!done_ && !(segs_.at(cursor_).key < k))
            throw StatusError{CUBICS_E_INVALID, "stream: segment announced left of the delivery cursor"};
        Seg& s = segs_[id];
        s.key = k;
        order_.emplace(std::move(k), id);
    }
    void on_sol(uint32_t id, const uint16_t* row, const uint64_t* snap) {
        if (io_.stopped) return;
        auto it = segs_.find(id);
        if (it == segs_.end()) throw StatusError{CUBICS_E_INVALID, "stream: solution of an unknown segment"};
        if (id == cursor_ && !done_) {
            deliver(row, snap);
            return;
        }
        Seg& s = it->second;
        buffered_ += sizeof(uint16_t) * n_ + sizeof(uint64_t) * 3;
        if (buffered_ > kMaxBuffered) // fail loudly rather than exhaust host memory
            throw StatusError{CUBICS_E_CAPACITY, "stream: solutions waiting right of the delivery cursor exceed 16 GiB"};
        s.rows.insert(s.rows.end(), row, row + n_);
        s.snaps.insert(s.snaps.end(), snap, snap + 3);
    }
    void on_end(uint32_t id, const uint64_t* st) {
        auto it = segs_.find(id);
        if (it == segs_.end()) return;
        it->second.done = true;
        std::copy_n(st, 3, it->second.st);
        while (!io_.stopped && !done_ && segs_.at(cursor_).done) {
            Seg& c = segs_.at(cursor_);
            for (int i = 0; i < 3; ++i) prefix_[i] += c.st[i];
            order_.erase(order_.begin());
            segs_.erase(cursor_);
            if (order_.empty()) {
                done_ = true;
                break;
            }
            cursor_ = order_.begin()->second;
            Seg& nx = segs_.at(cursor_);
            for (size_t r = 0; r * 3 < nx.snaps.size() && !io_.stopped; ++r)
                deliver(nx.rows.data() + r * n_, nx.snaps.data() + r * 3);
            buffered_ -= std::min<size_t>(buffered_, (nx.snaps.size() / 3) * (sizeof(uint16_t) * n_ + sizeof(uint64_t) * 3));
            nx.rows.clear();
            nx.rows.shrink_to_fit();
            nx.snaps.clear();
            nx.snaps.shrink_to_fit();
        }
    }

private:
    struct Seg {
        std::vector<uint32_t> key;
        bool done = false;
        uint64_t st[3] = {0, 0, 0};
        std::vector<uint16_t> rows;
        std::vector<uint64_t> snaps;
    };
    void deliver(const uint16_t* row, const uint64_t* snap) {
        uint64_t st[3];
        for (int i = 0; i < 3; ++i) st[i] = prefix_[i] + snap[i];
        ++io_.delivered;
        if (!io_.visit(row, st)) {
            io_.stopped = true;
            std::copy_n(st, 3, io_.stop_stats);
        }
    }
    static constexpr size_t kMaxBuffered = size_t(16) << 30;
    size_t buffered_ = 0;
    int KW_, n_;
    StreamIO& io_;
    std::unordered_map<uint32_t, Seg> segs_;
    std::map<std::vector<uint32_t>, uint32_t> order_;
    uint32_t cursor_ = 0;
    bool done_ = false;
    uint64_t prefix_[3] = {0, 0, 0};
};

// The calling thread's side of the stream: consume slots in ticket order until the kernel has
// finished and every reserved slot is drained, or until the callback stops the search (then the
// stop flag goes to the device on the side stream and the rest of the ring is ignored).
void drain_stream(uint8_t* ring, uint32_t cap, uint32_t slot_bytes, volatile unsigned long long* tail_host,
                  unsigned long long epoch, int KW, int n, bool parallel, cudaEvent_t done_ev, int32_t* dev_stop, const int32_t* host_one,
                  cudaStream_t side, StreamIO& io) {
    std::unique_ptr<SegmentOrder> order;
    if (parallel) order.reset(new SegmentOrder(KW, n, io));
    uint64_t tail = 0;
    bool kernel_done = false;
    int idle = 0;
    for (;;) {
        uint8_t* s = ring + (size_t)(tail % cap) * slot_bytes;
        const unsigned long long seq = *reinterpret_cast<volatile unsigned long long*>(s);
        if (seq == ((epoch << 40) | (tail + 1))) {
            std::atomic_thread_fence(std::memory_order_acquire);
            const uint32_t kind = *reinterpret_cast<volatile uint32_t*>(s + 8);
            const uint32_t seg = *reinterpret_cast<volatile uint32_t*>(s + 12);
            uint64_t st[3];
            std::memcpy(st, s + 16, sizeof st);
            const uint32_t* key = reinterpret_cast<const uint32_t*>(s + kEvHeader);
            const uint16_t* row = reinterpret_cast<const uint16_t*>(s + kEvHeader + 4 * KW);
            if (kind == EV_SOL) {
                if (order) {
                    order->on_sol(seg, row, st);
                } else if (!io.stopped) {
                    ++io.delivered;
                    if (!io.visit(row, st)) {
                        io.stopped = true;
                        std::copy_n(st, 3, io.stop_stats);
                    }
                }
            } else if (kind == EV_NEW && order) {
                order->on_new(seg, key);
            } else if (kind == EV_END && order) {
                order->on_end(seg, st);
            }
            ++tail;
            if ((tail & 255) == 0) *tail_host = tail;
            idle = 0;
            if (io.stopped) {
                CU(cudaMemcpyAsync(dev_stop, host_one, sizeof(int32_t), cudaMemcpyHostToDevice, side));
                CU(cudaStreamSynchronize(side));
                return;
            }
            continue;
        }
        *tail_host = tail;
        if (kernel_done) { // finished and nothing left: every reserved slot was written
            if (std::getenv("CUBICS_DEBUG"))
                std::fprintf(stderr, "[cubics] stream: %llu events, %llu delivered, next seq %llx want %llx\n",
                             (unsigned long long)tail, (unsigned long long)io.delivered, seq,
                             (epoch << 40) | (tail + 1));
            return;
        }
        const cudaError_t q = cudaEventQuery(done_ev);
        if (q == cudaSuccess) {
            kernel_done = true; // one more pass over what the last contexts wrote
            continue;
        }
        if (q != cudaErrorNotReady) CU(q);
        if (++idle > 64) std::this_thread::sleep_for(std::chrono::microseconds(20));
        else std::this_thread::yield();
    }
}

__global__ void gather_tasks(const uint32_t* src, const int32_t* idx, int n, size_t os, uint32_t* dst) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < (size_t)n * os; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[(size_t)idx[i / os] * os + i % os];
}

// One device search: upload, launch, download.
void run_search(const HostModel& hm, const cubics_search_config& cfg, int engine, bool record, uint64_t sol_cap,
                RunOut& out, bool want_keys = false, ShardIO* shard = nullptr, BatchIO* batch = nullptr,
                StreamIO* sio = nullptr) {
    const double rs_t0 = now_ms();
    const int dev = current_device(cfg.device);
    std::lock_guard<std::recursive_mutex> lock(g_dev_mu[dev]);
    NvtxRange nvtx(sio ? "cubics search (streaming)" : batch ? "cubics search (batch)" : shard ? "cubics search (shard)"
                                                                                       : "cubics search");
    // a solution callback runs while its search still owns this device's arenas and stream
    if (g_dev[dev].streaming)
        throw StatusError{CUBICS_E_INVALID, "a solution callback cannot start another search on the same device"};
    if (sio) {
        record = false;
        sol_cap = 0;
    }
    Prepared P;
    prepare(hm, hm.words.data(), P);
    const int n = P.n;
    // AUTO: a large model searched with reference node order gets the grid-wide context
    // (measured on B200: tables weigh ~4 RelBins; rbcsp_10000 / rcsp_100000 gain 1.7x / 6.8x,
    // rcsp_10000 with 20k cheap != constraints is faster in one block)
    if (batch) {
        engine = CUBICS_ENGINE_PARITY;
        record = false;
        const size_t nw64 = hm.words.size();
        batch->dom.assign(P.NWP * batch->count, 0);
        for (int i = 0; i < batch->count; ++i) {
            uint32_t* dst = batch->dom.data() + P.NWP * i;
            for (int v = 0; v < n; ++v) {
                words_to_u32(hm, v, batch->words + nw64 * i, dst, P.W);
                int sz = 0;
                for (int w = 0; w < P.W; ++w) sz += __builtin_popcount(dst[(size_t)v * P.W + w]);
                if (!sz) batch->any_empty = true;
            }
        }
    }
    if (engine == CUBICS_ENGINE_PARITY && cfg.engine == CUBICS_ENGINE_AUTO && !shard && !batch &&
        ((long)P.nr + P.nl + 4L * (P.ntb + P.ntn) >= 40000 || P.n >= 50000))
        engine = CUBICS_ENGINE_GRID;
    const bool grid = engine == CUBICS_ENGINE_GRID;
    const bool parallel = engine == CUBICS_ENGINE_PARALLEL;
    const bool keyed = parallel || (shard && (shard->split_depth > 0 || shard->guide_key));
    // exact parallel first solution: complete otherwise-equal search, max_solutions == 1
    const bool first_mode = (parallel && !shard && !sio && hm.goal == CUBICS_SATISFY && cfg.max_solutions == 1 &&
                             cfg.node_limit == 0) ||
                            (parallel && shard && shard->root_first);
    if (sio && (shard || batch || (parallel && hm.goal != CUBICS_SATISFY)))
        throw StatusError{CUBICS_E_INVALID, "streaming: reference-order engines, or the parallel engine on satisfy goals"};
    if (first_mode) {
        record = true;
        sol_cap = 65536;
    }
    const int seg_mode = first_mode ? 1 : (shard ? shard->first : 0);
    const int KW = keyed ? static_cast<int>((P.depth_bound + 1 + 31) / 32) : 0;
    const int n_seed = (shard && shard->seeds) ? static_cast<int>(shard->seeds->size()) : 0;
    if (parallel && KW > 4096) throw StatusError{CUBICS_E_UNSUPPORTED, "search tree too deep for ordered parallel keys"};
    out.KW = KW;
    // launch geometry
    // small models run warp contexts (warp_ctx.cuh): K contexts per block of 32K threads
    // (sharded first-solution runs need the frontier split with segment bookkeeping, which the
    // lean warp kernels compile out: they run block contexts)
    // (exact-first searches run block contexts too: fewer, wider contexts win there - magic5 first
    // 3.7 -> 2.7 ms at 128 threads)
    const bool use_warp = P.warp_ok && !grid && !batch && cfg.block_threads <= 0 && !(shard && (shard->first || shard->root_first)) &&
                          !first_mode &&
                          (parallel || engine == CUBICS_ENGINE_PARITY) && !std::getenv("CUBICS_NO_WARP");
    const int warp_k = use_warp && parallel ? std::max(1, std::min(2, std::getenv("CUBICS_WARP_K") ? std::atoi(std::getenv("CUBICS_WARP_K")) : 1)) : 1;
    int block = cfg.block_threads > 0 ? ((cfg.block_threads + 31) / 32) * 32 : 0;
    if (use_warp) block = 32 * warp_k;
    if (!block && grid) block = 512;
    if (!block) // parallel: one warp per context maximises resident contexts (32 per SM) for small models
        block = parallel ? (P.nr + P.nl + P.ntb + P.ntn > 1024 || P.n > 1024
                                ? 128
                                : (P.W >= 8 || P.nr + P.nl + P.ntb + P.ntn > 256 ? 64 : 32))
                         : parity_block(P);
    // exact-first searches (first solution, exact B&B phases, sharded first): fewer, wider
    // contexts - less speculation right of the answer, faster per node (B200: golomb10 exact B&B
    // 89 -> 65 ms at 128 threads, rcsp-1k first 137 -> 123 ms at 256)
    if (parallel && seg_mode == 1 && !use_warp && cfg.block_threads <= 0) block = std::min(256, std::max(128, 4 * block));
    block = std::min(std::max(block, 32), batch ? 512 : 1024);
    const int nw = use_warp ? 1 : block / 32;
    bool in_smem = !grid; // the grid context keeps its domains in L2/HBM
    int frame_cap = n + 1;
    if (cfg.node_limit && cfg.node_limit + 1 < (uint64_t)frame_cap) frame_cap = static_cast<int>(cfg.node_limit + 1);
    frame_cap = std::max(frame_cap, 1);
    // warp contexts keep their decision stack in shared memory when it is small (n <= 32: at
    // most 33 frames of 32 words)
    const bool frames_in_smem = use_warp && !std::getenv("CUBICS_WARP_GFRAMES") &&
                                (size_t)frame_cap * (P.NWP * 4 + 16) <= 4096;
    dev::SmemLayout L = dev::smem_layout(P.W, n, P.total_members, nw, KW, in_smem, P.na, frames_in_smem ? frame_cap : 0);
    // bytes of dynamic shared memory per block (warp contexts: one 16-byte aligned slice each)
    const size_t smem_block = use_warp ? (size_t)warp_k * ((L.total + 15) & ~size_t(15)) : L.total;
    if (use_warp && smem_block > kSmemBudget) throw StatusError{CUBICS_E_UNSUPPORTED, "warp context does not fit in shared memory"};
    if (L.total > kSmemBudget) {
        in_smem = false;
        L = dev::smem_layout(P.W, n, P.total_members, nw, KW, false, P.na);
        if (L.total > kSmemBudget) throw StatusError{CUBICS_E_UNSUPPORTED, "search context does not fit in shared memory"};
    }
    // propagator features the model needs: the lean kernel instantiations skip the rest
    // F_FIRST (8): segment bookkeeping, also what streaming needs (a reference-order search
    // wider than 512 threads runs the generic kernel, whose lean instantiations do not stream)
    const int feat = (P.nl ? 1 : 0) | (P.ntb + P.ntn ? 2 : 0) | (P.big_words ? 4 : 0) |
                     (seg_mode || sio ? 8 : 0) |
                     (P.lin_g > 1 ? dev::F_LONG : 0) |
                     (hm.goal == CUBICS_SATISFY ? dev::F_NOOPT : 0) | (!shard ? dev::F_NOSPLIT : 0) |
                     (shard && shard->split_depth > 0 ? dev::F_FRONTIER : 0);
    int n_ctx = batch ? batch->count : 1;
    if (parallel) {
        int per_sm = 0;
        if (use_warp) {
            CU(occupancy_search_warp(feat, false, block, smem_block, &per_sm));
        } else {
#define OCC(w) occupancy_search<w>(feat, block, L.total, &per_sm)
            CUBICS_DISPATCH_W(P.W, OCC)
#undef OCC
        }
        int sms = 0;
        CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        const int cap = std::max(1, per_sm) * sms * warp_k;
        n_ctx = cfg.contexts > 0 ? std::min(cfg.contexts, cap) : cap;
        n_ctx = std::max(warp_k, n_ctx / warp_k * warp_k); // whole blocks of warp contexts
        // decision stacks of many contexts in HBM: up to n+1 frames each, within a budget (large
        // models: rcsp-10k would need 400 MB per context); a stack that outgrows its share stops
        // the search with CUBICS_E_CAPACITY (the exact first solution then falls back to PARITY)
        if (!frames_in_smem) {
            const size_t per = sizeof(uint32_t) * P.NWP + 16, budget = size_t(24) << 30;
            size_t fit = budget / (per * (size_t)n_ctx);
            if (fit < 256) { // fewer contexts, each with at least 256 frames
                n_ctx = std::max(warp_k, (int)std::min<size_t>((size_t)n_ctx, budget / (per * 256)) / warp_k * warp_k);
                fit = budget / (per * (size_t)n_ctx);
            }
            if ((size_t)frame_cap > fit) frame_cap = (int)std::max<size_t>(fit, 1);
        }
    } else if (!frames_in_smem) { // one context (or one per batch problem): the same budget
        const size_t per = sizeof(uint32_t) * P.NWP + 16, budget = size_t(32) << 30;
        const size_t fit = std::max<size_t>(budget / (per * (size_t)n_ctx), 64);
        if ((size_t)frame_cap > fit) frame_cap = (int)fit; // rcsp-100k: 80k of its 100k+1 frames
    }
    int grid_blocks = 0;
    if (grid) { // co-resident blocks for the cooperative launch
        int per_sm = 0;
#define OCCG(w) occupancy_search_grid<w>(block, L.total, &per_sm)
        CUBICS_DISPATCH_W(P.W, OCCG)
#undef OCCG
        int sms = 0;
        CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        if (per_sm < 1) throw StatusError{CUBICS_E_UNSUPPORTED, "grid context does not fit on an SM"};
        grid_blocks = std::min(per_sm, 2) * sms;
    }
    out.contexts = n_ctx;
    out.engine = engine;
    const size_t NWP = P.NWP;
    const size_t OS = NWP + dev::round4((size_t)KW + 2);
    if (!record) sol_cap = 0;

    // one device allocation: [model blob | ws | queue | busy | has_first | frames | meta | gdom | outbox |
    //                          sol_vals | sol_keys | sol_stats | first keys | first vals | inc_vals]
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t at = (off + 255) & ~size_t(255);
        off = at + std::max<size_t>(bytes, 16);
        return at;
    };
    const size_t a_blob = take(P.blob.bytes.size());
    const size_t a_ws = take(sizeof(WorkState));
    const uint32_t ring_cap = 2u * (uint32_t)n_ctx + (uint32_t)n_seed;
    const size_t a_queue = take(sizeof(unsigned long long) * ring_cap);
    const size_t a_busy = take(sizeof(int32_t) * (n_ctx + n_seed));
    const size_t a_hf = take(sizeof(int32_t) * n_ctx);
    const size_t zero_end = off;
    const size_t a_big = take(sizeof(uint32_t) * P.big_words * (size_t)nw * (grid ? grid_blocks : n_ctx));
    const size_t a_gctl = take(grid ? 256 : 0);
    const size_t a_gslots = take(grid ? 6 * sizeof(unsigned) : 0);
    const size_t a_gchg = take(grid ? sizeof(uint32_t) * 2 * (((size_t)n + 31) / 32) : 0);
    const size_t a_frames = take(frames_in_smem ? 0 : sizeof(uint32_t) * NWP * frame_cap * n_ctx);
    const size_t a_meta = take(frames_in_smem ? 0 : sizeof(int32_t) * 4 * frame_cap * n_ctx);
    const size_t a_gdom = take(in_smem ? 0 : sizeof(uint32_t) * 2 * NWP * n_ctx);
    const size_t a_outbox = take(parallel ? sizeof(uint32_t) * OS * (n_ctx + n_seed) : 0);
    const size_t a_seedidx = take(sizeof(int32_t) * n_seed);
    const size_t a_svals = take(sizeof(uint16_t) * n * sol_cap);
    const size_t a_skeys = take(sizeof(uint32_t) * KW * sol_cap);
    const size_t a_sstats = take(parallel && !seg_mode ? 0 : sizeof(uint64_t) * 3 * sol_cap);
    const size_t a_fkey = take(sizeof(uint32_t) * KW * n_ctx);
    const size_t a_fval = take(parallel ? sizeof(uint16_t) * n * n_ctx : 0);
    const size_t a_inc = take(sizeof(uint16_t) * std::max(n, 1));
    // one segment per handed-out subtree; sized by memory (<= 1 GiB), parity fallback beyond
    const int64_t seg_cap = seg_mode ? std::max<int64_t>(n_seed + 1 + 2 * (int64_t)n_ctx,
                                                         std::min<int64_t>((int64_t)1 << 21, ((int64_t)1 << 30) / (4 * KW + 24)))
                                     : 0;
    const size_t a_tsnap = take(seg_mode && shard && shard->split_depth > 0 ? sizeof(uint64_t) * 4 * shard->task_cap : 0);
    const size_t a_segk = take(sizeof(uint32_t) * KW * seg_cap);
    const size_t a_segs = take(sizeof(uint64_t) * 3 * seg_cap);
    const size_t a_sseg = take(seg_mode ? sizeof(int32_t) * sol_cap : 0);
    const int nb = batch ? batch->count : 0;
    const size_t a_bdom = take(sizeof(uint32_t) * NWP * nb);
    const size_t a_bbound = take(sizeof(int64_t) * nb);
    const size_t a_bhas = take(sizeof(int32_t) * nb);
    const size_t a_bstats = take(sizeof(uint64_t) * 4 * nb);
    const size_t a_bflags = take(sizeof(int32_t) * nb);
    const size_t a_binc = take(sizeof(uint16_t) * n * nb);
    const bool guided = shard && shard->guide_key;
    const size_t gdepth = (size_t)KW * 32 + 1;
    const size_t a_gkey = take(guided ? sizeof(uint32_t) * KW : 0);
    const size_t a_gbnd = take(guided ? sizeof(int64_t) * gdepth : 0);
    const size_t a_ghas = take(guided ? sizeof(int32_t) * gdepth : 0);
    uint8_t* base = device_arena(dev, off);

    cudaStream_t st = g_dev[dev].stream;
    cudaEvent_t e0 = g_dev[dev].e0, e1 = g_dev[dev].e1;
    bool recorded_first_done = false;
    {
        // staging: blob + initial WorkState in pinned memory, one H2D copy
        WorkState w0{};
        const bool shared_q = shard && shard->claim;
        w0.outstanding = n_ctx + (shared_q ? 0 : n_seed);
        w0.hot.has_bound = seg_mode == 1 ? -1 : (cfg.has_initial_bound ? 1 : 0);
        // no initial bound: the worst value, so merging other GPUs' bounds is a plain atomic min/max
        w0.bound = cfg.has_initial_bound ? cfg.initial_bound
                                         : (hm.goal == CUBICS_MAXIMIZE ? std::numeric_limits<int64_t>::min()
                                                                       : std::numeric_limits<int64_t>::max());
        w0.hot.push_ticket = shared_q ? 0u : (uint32_t)n_seed;
        const size_t stage_bytes = a_ws + sizeof(WorkState);
        uint8_t* stage = pinned_arena(dev, stage_bytes);
        std::memset(stage, 0, stage_bytes);
        std::memcpy(stage + a_blob, P.blob.bytes.data(), P.blob.bytes.size());
        std::memcpy(stage + a_ws, &w0, sizeof w0);
        CU(cudaMemcpyAsync(base, stage, stage_bytes, cudaMemcpyHostToDevice, st));
        out.h2d += stage_bytes;
        CU(cudaMemsetAsync(base + a_queue, 0, zero_end - a_queue, st));
        if (seg_mode) {
            CU(cudaMemsetAsync(base + a_segk, 0, sizeof(uint32_t) * KW * seg_cap, st));
            CU(cudaMemsetAsync(base + a_segs, 0, sizeof(uint64_t) * 3 * seg_cap, st));
        }
        if (n_seed) { // pre-published tasks: ring tickets 0..n_seed-1 point at outbox slots n_ctx+i
            if (!shared_q) {
                std::vector<unsigned long long> ring0(n_seed);
                for (int i = 0; i < n_seed; ++i) ring0[i] = ((unsigned long long)(i + 1) << 32) | (unsigned)(n_ctx + i);
                CU(cudaMemcpyAsync(base + a_queue, ring0.data(), sizeof(unsigned long long) * n_seed, cudaMemcpyHostToDevice, st));
                out.h2d += sizeof(unsigned long long) * n_seed;
            }
            CU(cudaMemcpyAsync(base + a_seedidx, shard->seeds->data(), sizeof(int32_t) * n_seed, cudaMemcpyHostToDevice, st));
            out.h2d += sizeof(int32_t) * n_seed;
            const size_t total = (size_t)n_seed * OS;
            gather_tasks<<<(int)std::min<size_t>(4096, (total + 255) / 256), 256, 0, st>>>(
                shard->task_dev, reinterpret_cast<const int32_t*>(base + a_seedidx), n_seed, OS,
                reinterpret_cast<uint32_t*>(base + a_outbox) + (size_t)n_ctx * OS);
            CU(cudaGetLastError());
            out.launches += 1;
        }

        if (batch) {
            CU(cudaMemcpyAsync(base + a_bdom, batch->dom.data(), sizeof(uint32_t) * NWP * nb, cudaMemcpyHostToDevice, st));
            CU(cudaMemcpyAsync(base + a_bbound, batch->bound.data(), sizeof(int64_t) * nb, cudaMemcpyHostToDevice, st));
            CU(cudaMemcpyAsync(base + a_bhas, batch->has_bound.data(), sizeof(int32_t) * nb, cudaMemcpyHostToDevice, st));
            CU(cudaMemsetAsync(base + a_bflags, 0, sizeof(int32_t) * nb, st));
            out.h2d += (sizeof(uint32_t) * NWP + sizeof(int64_t) + sizeof(int32_t)) * nb;
        }
        SearchParams S{};
        S.M = P.bind(base + a_blob);
        S.M.goal = hm.goal;
        S.M.goal_var = hm.goal_var;
        S.mode = parallel ? MODE_PARALLEL : MODE_PARITY;
        S.var_heuristic = cfg.var_heuristic == CUBICS_FIRST_FAIL ? 1 : 0;
        S.alldiff = cfg.alldiff == CUBICS_FORWARD_CHECKING ? 0 : 1;
        S.exact_wipe = P.has_empty || (batch && batch->any_empty) ? 1 : 0;
        S.max_solutions = batch ? std::numeric_limits<uint64_t>::max() : cfg.max_solutions;
        S.node_limit = cfg.node_limit;
        S.n_ctx = n_ctx;
        S.frame_cap = frame_cap;
        S.KW = KW;
        S.record = record ? 1 : 0;
        S.dom_in_smem = in_smem ? 1 : 0;
        S.frames_in_smem = frames_in_smem ? 1 : 0;
        S.big_scratch = P.big_words ? reinterpret_cast<uint32_t*>(base + a_big) : nullptr;
        if (grid) {
            const unsigned init[6] = {0, 0, 0, 0xffffffffu, 0xffffffffu, 0xffffffffu};
            CU(cudaMemcpyAsync(base + a_gslots, init, sizeof init, cudaMemcpyHostToDevice, st));
            CU(cudaMemsetAsync(base + a_gctl, 0, 256, st));
            S.grid_ctl = reinterpret_cast<dev_ctl_t*>(base + a_gctl);
            S.grid_or = reinterpret_cast<unsigned*>(base + a_gslots);
            S.grid_min = S.grid_or + 3;
            S.grid_chg = reinterpret_cast<uint32_t*>(base + a_gchg);
        }
        S.frames = reinterpret_cast<uint32_t*>(base + a_frames);
        S.frame_meta = reinterpret_cast<int32_t*>(base + a_meta);
        S.gdom = reinterpret_cast<uint32_t*>(base + a_gdom);
        S.ws = reinterpret_cast<WorkState*>(base + a_ws);
        S.ring = reinterpret_cast<unsigned long long*>(base + a_queue);
        S.ring_cap = ring_cap;
        S.outbox_busy = reinterpret_cast<int32_t*>(base + a_busy);
        S.outbox = reinterpret_cast<uint32_t*>(base + a_outbox);
        S.sol_cap = sol_cap;
        S.sol_vals = reinterpret_cast<uint16_t*>(base + a_svals);
        S.sol_keys = reinterpret_cast<uint32_t*>(base + a_skeys);
        S.sol_stats = reinterpret_cast<uint64_t*>(base + a_sstats);
        S.ctx_first_key = reinterpret_cast<uint32_t*>(base + a_fkey);
        S.ctx_first_vals = reinterpret_cast<uint16_t*>(base + a_fval);
        S.ctx_has_first = reinterpret_cast<int32_t*>(base + a_hf);
        S.inc_vals = reinterpret_cast<uint16_t*>(base + a_inc);
        S.has_init_bound = cfg.has_initial_bound ? 1 : 0;
        S.init_bound = cfg.initial_bound;
        S.split_depth = shard ? shard->split_depth : -1;
        S.task_cap = shard ? (int64_t)shard->task_cap : 0;
        S.tasks = shard ? shard->task_dev : nullptr;
        S.n_seed = n_seed;
        S.task_claim = shard ? shard->claim : nullptr;
        S.g_inc = shard ? shard->g_inc : nullptr;
        S.g_first = shard ? shard->g_first : nullptr;
        S.static_bound = shard && shard->static_bound ? 1 : 0;
        if (guided) {
            if (shard->guide_key->size() != (size_t)KW || shard->guide_bound.size() != gdepth ||
                shard->guide_has.size() != gdepth)
                throw StatusError{CUBICS_E_INVALID, "guided replay: key / bound sizes"};
            CU(cudaMemcpyAsync(base + a_gkey, shard->guide_key->data(), sizeof(uint32_t) * KW, cudaMemcpyHostToDevice, st));
            CU(cudaMemcpyAsync(base + a_gbnd, shard->guide_bound.data(), sizeof(int64_t) * gdepth, cudaMemcpyHostToDevice, st));
            CU(cudaMemcpyAsync(base + a_ghas, shard->guide_has.data(), sizeof(int32_t) * gdepth, cudaMemcpyHostToDevice, st));
            out.h2d += sizeof(uint32_t) * KW + (sizeof(int64_t) + sizeof(int32_t)) * gdepth;
            S.guide_key = reinterpret_cast<const uint32_t*>(base + a_gkey);
            S.guide_bound = reinterpret_cast<const int64_t*>(base + a_gbnd);
            S.guide_has = reinterpret_cast<const int32_t*>(base + a_ghas);
        }
        if (shard && shard->xs && parallel && !seg_mode && !std::getenv("CUBICS_NO_XS")) { // pool slots: header + outbox
            const size_t slot = (16 + 4 * OS + 15) & ~size_t(15);
            const size_t cap = std::min<size_t>(4096, kXsBytes / slot);
            if (cap >= 8) {
                S.xs_ctl = reinterpret_cast<XsCtl*>(shard->xs + 128);
                S.xs_slots = shard->xs + 256;
                S.xs_cap = (uint32_t)cap;
                S.xs_slot = (uint32_t)slot;
            }
        }
        S.first_mode = seg_mode;
        S.seg_base = shard && shard->claim ? n_seed : 0;
        S.task_snap = reinterpret_cast<uint64_t*>(base + a_tsnap);
        S.seg_cap = seg_cap;
        S.seg_key = reinterpret_cast<uint32_t*>(base + a_segk);
        S.seg_stats = reinterpret_cast<uint64_t*>(base + a_segs);
        S.sol_seg = reinterpret_cast<int32_t*>(base + a_sseg);
        S.batch = nb;
        S.batch_dom = reinterpret_cast<const uint32_t*>(base + a_bdom);
        S.batch_bound = reinterpret_cast<const int64_t*>(base + a_bbound);
        S.batch_has_bound = reinterpret_cast<const int32_t*>(base + a_bhas);
        S.batch_stats = reinterpret_cast<uint64_t*>(base + a_bstats);
        S.batch_flags = reinterpret_cast<int32_t*>(base + a_bflags);
        S.batch_inc = reinterpret_cast<uint16_t*>(base + a_binc);
        // streaming: [host tail u64 | stop source i32 | pad to 64] [ring of cap slots]
        uint8_t* ev_host = nullptr;
        uint32_t ev_cap = 0, ev_slot = 0;
        static uint32_t epochs[64];
        if (sio) {
            ev_slot = (uint32_t)(((size_t)kEvHeader + 4 * (size_t)KW + 2 * (size_t)n + 15) & ~size_t(15));
            ev_cap = (uint32_t)std::max<size_t>(256, std::min<size_t>((size_t)1 << 20, ((size_t)64 << 20) / ev_slot));
            ev_host = mapped_arena(dev, 64 + (size_t)ev_cap * ev_slot);
            *reinterpret_cast<volatile unsigned long long*>(ev_host) = 0;
            *reinterpret_cast<volatile int32_t*>(ev_host + 8) = 1;
            void* dptr = nullptr;
            CU(cudaHostGetDevicePointer(&dptr, ev_host, 0));
            epochs[dev] = (epochs[dev] + 1) & 0xffffffu;
            S.stream = 1;
            S.ev_cap = ev_cap;
            S.ev_slot = ev_slot;
            S.ev_epoch = epochs[dev];
            S.ev_ring = static_cast<uint8_t*>(dptr) + 64;
            S.ev_tail_host = static_cast<const unsigned long long*>(dptr);
        }

        CU(cudaEventRecord(e0, st));
        if (grid) {
#define LG(w) launch_search_grid<w>(S, grid_blocks, block, L.total, st)
            CUBICS_DISPATCH_W(P.W, LG)
#undef LG
        } else if (use_warp) {
            CU(launch_search_warp(S, feat, n_ctx / warp_k, block, smem_block, st));
        } else {
#define LS(w) launch_search<w>(S, feat, n_ctx, block, L.total, st)
            CUBICS_DISPATCH_W(P.W, LS)
#undef LS
        }
        CU(cudaEventRecord(e1, st));
        out.launches += 1;
        if (sio) { // the calling thread runs the callback while the kernel searches on
            struct Flag {
                bool& f;
                explicit Flag(bool& x) : f(x) { f = true; }
                ~Flag() { f = false; }
            } busy(g_dev[dev].streaming);
            int32_t* dev_stop = &reinterpret_cast<WorkState*>(base + a_ws)->hot.stop;
            try {
                drain_stream(ev_host + 64, ev_cap, ev_slot, reinterpret_cast<volatile unsigned long long*>(ev_host),
                             S.ev_epoch, KW, n, parallel, e1, dev_stop, reinterpret_cast<const int32_t*>(ev_host + 8),
                             g_dev[dev].side, *sio);
            } catch (...) { // stop the device before unwinding (the callback or the ordering threw)
                cudaMemcpyAsync(dev_stop, ev_host + 8, sizeof(int32_t), cudaMemcpyHostToDevice, g_dev[dev].side);
                cudaStreamSynchronize(g_dev[dev].side);
                cudaStreamSynchronize(st);
                throw;
            }
        }
        CU(cudaMemcpyAsync(&out.ws, base + a_ws, sizeof(WorkState), cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        out.d2h += sizeof(WorkState);
        float ms = 0;
        CU(cudaEventElapsedTime(&ms, e0, e1));
        out.device_ms = ms;
        if (first_mode || (shard && shard->prefix_sum)) { // the reference's prefix up to the DFS-first solution
            const uint64_t nseg = (uint64_t)out.ws.hot.push_ticket + 1 + (uint64_t)S.seg_base, nsol = out.ws.sol_count;
            if (nseg > (uint64_t)seg_cap || nsol > sol_cap)
                throw StatusError{CUBICS_E_CAPACITY, "first-solution bookkeeping capacity"};
            std::vector<uint32_t> solk(nsol * KW);
            std::vector<uint64_t> sst(nsol * 3);
            std::vector<int32_t> sseg(nsol);
            if (nsol) {
                CU(cudaMemcpyAsync(solk.data(), base + a_skeys, sizeof(uint32_t) * KW * nsol, cudaMemcpyDeviceToHost, st));
                CU(cudaMemcpyAsync(sst.data(), base + a_sstats, sizeof(uint64_t) * 3 * nsol, cudaMemcpyDeviceToHost, st));
                CU(cudaMemcpyAsync(sseg.data(), base + a_sseg, sizeof(int32_t) * nsol, cudaMemcpyDeviceToHost, st));
            }
            CU(cudaStreamSynchronize(st));
            out.d2h += sizeof(uint32_t) * KW * nsol + sizeof(uint64_t) * 3 * nsol + 4 * nsol;
            auto less = [&](const uint32_t* a, const uint32_t* b) { return std::lexicographical_compare(a, a + KW, b, b + KW); };
            int64_t best = -1;
            for (uint64_t i = 0; i < nsol; ++i)
                if (best < 0 || less(&solk[i * KW], &solk[best * KW])) best = (int64_t)i;
            // every segment not right of the answer, its own segment aside: summed on the device
            uint64_t tot[3] = {0, 0, 0};
            {
                uint8_t* scratch = device_arena(dev, 256 + sizeof(uint32_t) * KW, 2);
                unsigned long long* dtot = reinterpret_cast<unsigned long long*>(scratch);
                uint32_t* dk = reinterpret_cast<uint32_t*>(scratch + 256);
                CU(cudaMemsetAsync(dtot, 0, 3 * sizeof(unsigned long long), st));
                if (best >= 0)
                    CU(cudaMemcpyAsync(dk, base + a_skeys + sizeof(uint32_t) * KW * best, sizeof(uint32_t) * KW,
                                       cudaMemcpyDeviceToDevice, st));
                const int g = (int)std::max<uint64_t>(1, std::min<uint64_t>(1184, (nseg + 255) / 256));
                seg_prefix_sum<<<g, 256, 0, st>>>(reinterpret_cast<const uint32_t*>(base + a_segk),
                                                 reinterpret_cast<const uint64_t*>(base + a_segs), nseg, KW,
                                                 best >= 0 ? dk : nullptr, best >= 0 ? (int64_t)sseg[best] : -1, dtot);
                CU(cudaGetLastError());
                out.launches += 1;
                unsigned long long h[3];
                CU(cudaMemcpyAsync(h, dtot, sizeof h, cudaMemcpyDeviceToHost, st));
                CU(cudaStreamSynchronize(st));
                out.d2h += sizeof h;
                for (int i = 0; i < 3; ++i) tot[i] = h[i];
            }
            if (best >= 0) {
                for (int i = 0; i < 3; ++i) tot[i] += sst[best * 3 + i];
                out.first_key.assign(solk.begin() + best * KW, solk.begin() + (best + 1) * KW);
                out.has_first = true;
                out.rec.count = 1;
                out.rec.ordered = true;
                out.rec.vals.resize(n);
                CU(cudaMemcpy(out.rec.vals.data(), base + a_svals + sizeof(uint16_t) * n * best, sizeof(uint16_t) * n,
                              cudaMemcpyDeviceToHost));
                out.d2h += sizeof(uint16_t) * n;
                out.ws.user_stop = 1; // max_solutions reached, as the reference reports it
            }
            out.ws.stats[0] = tot[0];
            out.ws.stats[1] = tot[1];
            out.ws.stats[2] = tot[2];
            out.ws.stats[3] = best >= 0 ? 1 : 0;
            recorded_first_done = true;
        }
        const uint64_t got = std::min<uint64_t>(out.ws.sol_count ? out.ws.sol_count : 0, sol_cap);
        uint64_t recorded = parallel ? got : std::min<uint64_t>(out.ws.stats[3], sol_cap);
        if (!recorded_first_done) out.rec.count = recorded;
        if (recorded && !recorded_first_done) {
            uint16_t* dst;
            if (out.pinned_rows) {
                dst = reinterpret_cast<uint16_t*>(pinned_arena(dev, sizeof(uint16_t) * n * recorded, 1));
                out.rec.pinned = dst;
            } else {
                out.rec.vals.resize(recorded * n);
                dst = out.rec.vals.data();
            }
            const uint16_t* src = reinterpret_cast<const uint16_t*>(base + a_svals);
            if (parallel && KW && n && recorded > 1 && !want_keys) {
                const int used = std::max(1, std::min(KW, (out.ws.max_depth + 31) / 32));
                src = order_on_device(dev, reinterpret_cast<const uint32_t*>(base + a_skeys), KW, used, src, n, recorded,
                                      st, &out.launches);
                out.rec.ordered = true;
            }
            int64_t* v64 = out.int64_rows && (!parallel || out.rec.ordered || recorded == 1)
                               ? PinnedPool::get().take(sizeof(int64_t) * n * recorded)
                               : nullptr;
            if (v64) { // offsets added on the device, one DMA of the final array
                int64_t* d64 = reinterpret_cast<int64_t*>(device_arena(dev, sizeof(int64_t) * n * recorded, 2));
                const int g2 = (int)std::max<uint64_t>(1, std::min<uint64_t>(8192, (recorded * n + 255) / 256));
                rows_to_int64<<<g2, 256, 0, st>>>(src, S.M.off, n, recorded, d64);
                CU(cudaGetLastError());
                out.launches += 1;
                CU(cudaMemcpyAsync(v64, d64, sizeof(int64_t) * n * recorded, cudaMemcpyDeviceToHost, st));
                out.d2h += sizeof(int64_t) * n * recorded;
                out.values64 = v64;
                out.rec.ordered = true;
            } else {
                CU(cudaMemcpyAsync(dst, src, sizeof(uint16_t) * n * recorded, cudaMemcpyDeviceToHost, st));
                out.d2h += sizeof(uint16_t) * n * recorded;
            }
            if (!parallel) out.rec.ordered = true;
            if (KW && want_keys) {
                out.rec.keys.resize(recorded * KW);
                CU(cudaMemcpyAsync(out.rec.keys.data(), base + a_skeys, sizeof(uint32_t) * KW * recorded,
                                   cudaMemcpyDeviceToHost, st));
                out.d2h += sizeof(uint32_t) * KW * recorded;
            }
            if (seg_mode) {
                out.rec.seg.resize(recorded);
                CU(cudaMemcpyAsync(out.rec.seg.data(), base + a_sseg, sizeof(int32_t) * recorded, cudaMemcpyDeviceToHost, st));
                out.d2h += sizeof(int32_t) * recorded;
            }
            if (!parallel || seg_mode) {
                out.rec.stats.resize(recorded * 3);
                CU(cudaMemcpyAsync(out.rec.stats.data(), base + a_sstats, sizeof(uint64_t) * 3 * recorded,
                                   cudaMemcpyDeviceToHost, st));
                out.d2h += sizeof(uint64_t) * 3 * recorded;
            }
        }
        if (parallel && KW && n && !first_mode) { // DFS-first solution over the contexts' firsts
            std::vector<int32_t> hf(n_ctx);
            std::vector<uint32_t> fk((size_t)KW * n_ctx);
            CU(cudaMemcpyAsync(hf.data(), base + a_hf, sizeof(int32_t) * n_ctx, cudaMemcpyDeviceToHost, st));
            CU(cudaMemcpyAsync(fk.data(), base + a_fkey, sizeof(uint32_t) * KW * n_ctx, cudaMemcpyDeviceToHost, st));
            CU(cudaStreamSynchronize(st));
            out.d2h += sizeof(int32_t) * n_ctx + sizeof(uint32_t) * KW * n_ctx;
            int best = -1;
            for (int c = 0; c < n_ctx; ++c) {
                if (!hf[c]) continue;
                if (best < 0 || std::lexicographical_compare(fk.begin() + (size_t)c * KW, fk.begin() + (size_t)(c + 1) * KW,
                                                             fk.begin() + (size_t)best * KW,
                                                             fk.begin() + (size_t)(best + 1) * KW))
                    best = c;
            }
            if (best >= 0) {
                out.has_first = true;
                out.first_key.assign(fk.begin() + (size_t)best * KW, fk.begin() + (size_t)(best + 1) * KW);
                out.first_vals.resize(n);
                CU(cudaMemcpyAsync(out.first_vals.data(), base + a_fval + sizeof(uint16_t) * n * best,
                                   sizeof(uint16_t) * n, cudaMemcpyDeviceToHost, st));
                out.d2h += sizeof(uint16_t) * n;
            }
        }
        if (batch) {
            batch->stats.resize((size_t)4 * nb);
            batch->flags.resize(nb);
            batch->inc.resize((size_t)n * nb);
            CU(cudaMemcpyAsync(batch->stats.data(), base + a_bstats, sizeof(uint64_t) * 4 * nb, cudaMemcpyDeviceToHost, st));
            CU(cudaMemcpyAsync(batch->flags.data(), base + a_bflags, sizeof(int32_t) * nb, cudaMemcpyDeviceToHost, st));
            if (n)
                CU(cudaMemcpyAsync(batch->inc.data(), base + a_binc, sizeof(uint16_t) * n * nb, cudaMemcpyDeviceToHost, st));
            out.d2h += (sizeof(uint64_t) * 4 + sizeof(int32_t) + sizeof(uint16_t) * n) * nb;
        }
        if (shard) shard->n_tasks = (uint64_t)out.ws.n_tasks;
        if (shard && seg_mode && !shard->prefix_sum) { // segments and the frontier tasks' positions, for the host's prefix sums
            const uint64_t nseg = (uint64_t)out.ws.hot.push_ticket + 1 + (uint64_t)S.seg_base;
            if (nseg > (uint64_t)seg_cap) throw StatusError{CUBICS_E_CAPACITY, "segment bookkeeping capacity"};
            shard->n_seg = nseg;
            shard->seg_key.resize(nseg * KW);
            shard->seg_st.resize(nseg * 3);
            CU(cudaMemcpyAsync(shard->seg_key.data(), base + a_segk, sizeof(uint32_t) * KW * nseg, cudaMemcpyDeviceToHost, st));
            CU(cudaMemcpyAsync(shard->seg_st.data(), base + a_segs, sizeof(uint64_t) * 3 * nseg, cudaMemcpyDeviceToHost, st));
            out.d2h += (sizeof(uint32_t) * KW + sizeof(uint64_t) * 3) * nseg;
            if (shard->split_depth > 0) {
                const uint64_t nt = std::min<uint64_t>((uint64_t)out.ws.n_tasks, shard->task_cap);
                shard->task_snap.resize(nt * 4);
                CU(cudaMemcpyAsync(shard->task_snap.data(), base + a_tsnap, sizeof(uint64_t) * 4 * nt, cudaMemcpyDeviceToHost, st));
                out.d2h += sizeof(uint64_t) * 4 * nt;
            }
        }
        if (parallel && hm.goal != CUBICS_SATISFY && n) {
            out.inc_vals.resize(n);
            CU(cudaMemcpyAsync(out.inc_vals.data(), base + a_inc, sizeof(uint16_t) * n, cudaMemcpyDeviceToHost, st));
            out.d2h += sizeof(uint16_t) * n;
        }
        CU(cudaStreamSynchronize(st));
    }
    if (sio && sio->stopped) { // the reference's stats where its callback stopped (search.cpp:147-149)
        for (int i = 0; i < 3; ++i) out.ws.stats[i] = sio->stop_stats[i];
        out.ws.stats[3] = sio->delivered;
        out.ws.user_stop = 1;
    }
    if (std::getenv("CUBICS_DEBUG")) {
        std::fprintf(stderr, "[cubics] run_search wall %.3f ms (device %.3f)\n", now_ms() - rs_t0, out.device_ms);
        const WorkState& w = out.ws;
        const double tot = (double)w.busy_cycles + (double)w.idle_cycles;
        std::fprintf(stderr,
                     "[cubics] engine=%s%s ctx=%d block=%d W=%d smem=%zu KW=%d ms=%.3f nodes=%llu donations=%llu "
                     "steals=%llu busy=%.3f xs_in=%llu xs_out=%llu\n",
                     parallel ? "parallel" : "parity", use_warp ? "(warp)" : "", n_ctx, block, P.W, smem_block, KW, out.device_ms,
                     (unsigned long long)w.stats[0], (unsigned long long)w.donations, (unsigned long long)w.steals,
                     tot > 0 ? w.busy_cycles / tot : 0.0, (unsigned long long)w.xs_in, (unsigned long long)w.xs_out);
    }
    if (out.ws.error == DERR_OVERFLOW) throw StatusError{CUBICS_E_OVERFLOW, "overflow in linear propagation"};
    if (out.ws.error == DERR_CAPACITY) throw StatusError{CUBICS_E_CAPACITY, "device decision stack capacity exceeded"};
    if (out.ws.error == DERR_GUIDE) throw StatusError{CUBICS_E_INVALID, "guided replay left its recorded path"};
}

void fill_result(const RunOut& r, cubics_result* out) {
    out->stats.nodes = r.ws.stats[0];
    out->stats.failures = r.ws.stats[1];
    out->stats.rounds = r.ws.stats[2];
    out->stats.solutions = r.ws.stats[3];
    out->engine = r.engine;
    out->contexts = r.contexts;
    out->device_ms = r.device_ms;
    out->h2d_bytes = r.h2d;
    out->d2h_bytes = r.d2h;
    out->kernel_launches = r.launches;
    out->remote_tasks_in = r.ws.xs_in;
    out->remote_tasks_out = r.ws.xs_out;
}

int pick_engine(const cubics_search_config& cfg, bool optimize_goal) {
    if (cfg.engine == CUBICS_ENGINE_GRID) return CUBICS_ENGINE_GRID;
    if (cfg.engine == CUBICS_ENGINE_PARITY || cfg.engine == CUBICS_ENGINE_PARALLEL) {
        if (cfg.engine == CUBICS_ENGINE_PARALLEL &&
            (cfg.node_limit != 0 ||
             (!optimize_goal && cfg.max_solutions != std::numeric_limits<uint64_t>::max() && cfg.max_solutions != 1)))
            throw StatusError{CUBICS_E_UNSUPPORTED,
                              "parallel engine needs a complete search (no node_limit, unbounded max_solutions)"};
        return cfg.engine;
    }
    if (!optimize_goal && cfg.node_limit == 0 &&
        (cfg.max_solutions == std::numeric_limits<uint64_t>::max() || cfg.max_solutions == 1))
        return CUBICS_ENGINE_PARALLEL; // complete enumeration, or the exact parallel first solution
    return CUBICS_ENGINE_PARITY;
}

template <class F>
int guarded(F&& f) {
    try {
        return f();
    } catch (const StatusError& e) {
        set_error(e.msg);
        return e.code;
    } catch (const CudaError& e) {
        set_error(e.msg);
        return CUBICS_E_CUDA;
    } catch (const std::bad_alloc&) {
        set_error("host allocation failed");
        return CUBICS_E_CAPACITY;
    }
}

uint64_t default_sol_cap(const HostModel& m, const cubics_search_config& cfg) {
    const uint64_t per = (uint64_t)m.n_vars() * 2 + 64;
    uint64_t cap = (uint64_t)1 << 22;
    cap = std::min<uint64_t>(cap, ((uint64_t)2 << 30) / per);
    if (cfg.max_solutions != std::numeric_limits<uint64_t>::max()) cap = std::min<uint64_t>(cap, cfg.max_solutions);
    return std::max<uint64_t>(cap, 1);
}

} // namespace

// ============================================================================ C ABI
extern "C" void cubics_search_config_init(cubics_search_config* c) {
    if (!c) return;
    std::memset(c, 0, sizeof *c);
    c->var_heuristic = CUBICS_FIRST_FAIL;
    c->value_heuristic = 0;
    c->max_solutions = std::numeric_limits<uint64_t>::max();
    c->thread_count = 1;
    c->seed = 0;
    c->alldiff = CUBICS_ARC_CONSISTENT;
    c->node_limit = 0;
    c->engine = CUBICS_ENGINE_AUTO;
    c->device = -1;
    c->contexts = 0;
    c->block_threads = 0;
    c->count_only = 0;
}

namespace {
// Search for every solution with records materialised (rerun once with an exact buffer when the
// first guess overflowed); the records come back in the reference's DFS order.
RunOut satisfy_run(const HostModel& m, const cubics_search_config& cfg, bool record, cubics_result* out,
                   bool pinned_rows = false, bool int64_rows = false) {
    std::memset(out, 0, sizeof *out);
    // an objective makes the stream a sequence of incumbents, whose order only the reference
    // node order reproduces: AUTO picks the parity engine then
    int engine = pick_engine(cfg, m.goal != CUBICS_SATISFY);
    uint64_t cap = default_sol_cap(m, cfg);
    RunOut r;
    r.pinned_rows = pinned_rows;
    r.int64_rows = int64_rows && m.goal == CUBICS_SATISFY;
    try {
        run_search(m, cfg, engine, record, cap, r);
    } catch (const StatusError& e) {
        // the exact parallel first solution ran out of bookkeeping space: the parity engine
        // gives the same answer and stats
        if (e.code != CUBICS_E_CAPACITY || engine != CUBICS_ENGINE_PARALLEL || cfg.max_solutions != 1) throw;
        engine = CUBICS_ENGINE_PARITY;
        r = RunOut{};
        r.pinned_rows = pinned_rows;
        r.int64_rows = int64_rows && m.goal == CUBICS_SATISFY;
        run_search(m, cfg, engine, record, cap, r);
    }
    if (record && r.ws.stats[3] > r.rec.count && r.rec.count == cap) { // buffer overflow: rerun exact
        RunOut r2;
        r2.pinned_rows = pinned_rows;
        r2.int64_rows = r.int64_rows;
        if (r.values64) PinnedPool::get().give_back(r.values64); // the truncated first attempt
        r.values64 = nullptr;
        run_search(m, cfg, engine, record, r.ws.stats[3], r2);
        r2.h2d += r.h2d;
        r2.d2h += r.d2h;
        r2.launches += r.launches;
        r = std::move(r2);
    }
    fill_result(r, out);
    const int n = m.n_vars();
    out->complete = !r.ws.limit_hit && !r.ws.user_stop;
    out->has_solution = r.ws.stats[3] > 0;
    if (m.goal != CUBICS_SATISFY && r.rec.count) {
        const size_t last = r.rec.count - 1;
        out->objective = m.offset[m.goal_var] + r.rec.rows()[last * n + m.goal_var];
    }
    if (record && r.rec.count && !r.rec.ordered && r.KW) { // keyed records: host-side DFS order
        r.rec.materialize(n);
        const int KW = r.KW;
        std::vector<uint64_t> order(r.rec.count);
        std::iota(order.begin(), order.end(), 0);
        const uint32_t* K = r.rec.keys.data();
        std::sort(order.begin(), order.end(), [&](uint64_t a, uint64_t b) {
            return std::lexicographical_compare(K + a * KW, K + (a + 1) * KW, K + b * KW, K + (b + 1) * KW);
        });
        std::vector<uint16_t> v(r.rec.vals.size());
        for (uint64_t i = 0; i < order.size(); ++i)
            std::copy_n(r.rec.vals.begin() + order[i] * n, n, v.begin() + i * n);
        r.rec.vals.swap(v);
        r.rec.ordered = true;
    }
    return r;
}

template <class Visit>
int satisfy_records(const HostModel& m, const cubics_search_config& cfg, bool record, cubics_result* out,
                    Visit&& visit) {
    const double t0 = now_ms();
    RunOut r = satisfy_run(m, cfg, record, out);
    const int n = m.n_vars();
    for (uint64_t i = 0; record && i < r.rec.count; ++i) {
        if (!visit(i, r.rec.vals.data() + i * n)) {
            if (!r.KW && !r.rec.stats.empty()) { // parity: the reference stops right here
                out->stats.nodes = r.rec.stats[i * 3 + 0];
                out->stats.failures = r.rec.stats[i * 3 + 1];
                out->stats.rounds = r.rec.stats[i * 3 + 2];
                out->stats.solutions = i + 1;
            }
            out->complete = 0;
            break;
        }
    }
    out->total_ms = now_ms() - t0;
    return CUBICS_OK;
}
} // namespace

namespace {
void exact_bnb(const HostModel& m, const cubics_search_config& cfg0, std::vector<uint16_t>& best, cubics_result* out,
               const std::function<bool(const uint16_t*)>* visit = nullptr);

// AUTO satisfy search capped at k > 1 solutions, no node limit: the parallel engine streams the
// solutions in DFS order (segments) and the host stops it at the k-th, whose stats are the
// reference's (search.cpp:151-154) - the exact first-k at parallel speed.
bool capped_stream(const HostModel& m, const cubics_search_config& cfg) {
    return cfg.engine == CUBICS_ENGINE_AUTO && m.goal == CUBICS_SATISFY && cfg.node_limit == 0 && cfg.max_solutions > 1 &&
           cfg.max_solutions != std::numeric_limits<uint64_t>::max() && m.n_vars() > 0 &&
           !std::getenv("CUBICS_NO_CAPPED_STREAM");
}

// One streamed satisfy search: visit(row) per solution in DFS order (false stops), at most
// `cap` solutions. Returns the objective of the last solution delivered (objective goals).
int64_t stream_satisfy(const HostModel& m, const cubics_search_config& cfg, int engine, uint64_t cap,
                       const std::function<bool(const uint16_t*)>& visit, cubics_result* out) {
    const double t0 = now_ms();
    std::memset(out, 0, sizeof *out);
    int64_t last_obj = 0;
    StreamIO io;
    io.visit = [&](const uint16_t* row, const uint64_t*) {
        if (m.goal != CUBICS_SATISFY) last_obj = m.offset[m.goal_var] + row[m.goal_var];
        return visit(row) && io.delivered < cap;
    };
    RunOut r;
    run_search(m, cfg, engine, false, 0, r, false, nullptr, nullptr, &io);
    fill_result(r, out);
    out->complete = !r.ws.limit_hit && !r.ws.user_stop;
    out->has_solution = r.ws.stats[3] > 0;
    if (m.goal != CUBICS_SATISFY && io.delivered) out->objective = last_obj;
    out->total_ms = now_ms() - t0;
    return last_obj;
}
} // namespace

extern "C" int cubics_solve_satisfy(const cubics_model* h, const cubics_search_config* cfg, cubics_solution_cb cb,
                                    void* user, cubics_result* out) {
    if (!h || !cfg || !out) return CUBICS_E_INVALID;
    return guarded([&] {
        const HostModel& m = h->m;
        const int n = m.n_vars();
        std::vector<int64_t> vals(n);
        const bool want = cb && !cfg->count_only;
        const int engine = want ? pick_engine(*cfg, m.goal != CUBICS_SATISFY) : CUBICS_ENGINE_PARITY;
        // streamed unless it is the exact parallel first solution (one row) or a parallel
        // branch-and-bound stream (reference-order incumbents need the parity engine)
        const bool par = engine == CUBICS_ENGINE_PARALLEL;
        // an objective: the reference's stream is its sequence of incumbents - the exact parallel
        // B&B delivers them in order (AUTO, no node limit)
        if (m.goal != CUBICS_SATISFY && cfg->engine == CUBICS_ENGINE_AUTO && cfg->node_limit == 0 && n > 0 &&
            cfg->max_solutions > 0 && !std::getenv("CUBICS_NO_EXACT_BNB")) {
            const double t0 = now_ms();
            std::memset(out, 0, sizeof *out);
            std::vector<uint16_t> best;
            uint64_t delivered = 0;
            const std::function<bool(const uint16_t*)> visit = [&](const uint16_t* row) {
                ++delivered;
                if (!want) return true;
                for (int v = 0; v < n; ++v) vals[v] = m.offset[v] + row[v];
                return cb(user, vals.data(), n) != 0;
            };
            try {
                exact_bnb(m, *cfg, best, out, &visit);
                out->has_solution = !best.empty();
                if (!best.empty()) out->objective = m.offset[m.goal_var] + best[m.goal_var];
                out->total_ms = now_ms() - t0;
                return (int)CUBICS_OK;
            } catch (const StatusError& e) {
                if (e.code != CUBICS_E_CAPACITY || delivered) throw; // incumbents already delivered
            }
        }
        const bool capped = capped_stream(m, *cfg);
        if (capped || (want && !(par && (cfg->max_solutions == 1 || m.goal != CUBICS_SATISFY)))) {
            stream_satisfy(m, *cfg, capped ? CUBICS_ENGINE_PARALLEL : engine, cfg->max_solutions,
                           [&](const uint16_t* row) {
                               if (!want) return true;
                               for (int v = 0; v < n; ++v) vals[v] = m.offset[v] + row[v];
                               return cb(user, vals.data(), n) != 0;
                           },
                           out);
            return (int)CUBICS_OK;
        }
        return satisfy_records(m, *cfg, want, out, [&](uint64_t, const uint16_t* row) {
            for (int v = 0; v < n; ++v) vals[v] = m.offset[v] + row[v];
            return cb(user, vals.data(), n) != 0;
        });
    });
}

// Host workers for the solution-array conversion, started once and kept: spawning 16 threads per
// cubics_enumerate call cost a visible part of the ~1 ms conversion. run(n, f) calls f(0..n-1),
// f(0) on the caller; calls are serialised (one job at a time).
class HostPool {
public:
    static HostPool& get() {
        // never destroyed: workers outlive static teardown. A forked child has none of the
        // parent's workers, so it starts its own pool.
        static std::mutex mu;
        static HostPool* p = nullptr;
        std::lock_guard<std::mutex> lk(mu);
        if (!p || p->pid_ != getpid()) p = new HostPool();
        return *p;
    }
    unsigned size() const { return (unsigned)threads_.size() + 1; }
    // f(i) for i < n; n must not exceed size() (callers partition by their own n)
    void run(unsigned n, const std::function<void(unsigned)>& f) {
        if (n > size()) throw StatusError{CUBICS_E_INVALID, "host pool: more parts than workers"};
        if (n <= 1) {
            if (n) f(0);
            return;
        }
        std::lock_guard<std::mutex> job(job_mu_);
        {
            std::lock_guard<std::mutex> lk(mu_);
            fn_ = &f;
            parts_ = n;
            pending_ = n - 1;
            ++gen_;
        }
        cv_.notify_all();
        f(0);
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [&] { return pending_ == 0; });
        fn_ = nullptr;
    }

private:
    HostPool() {
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        for (unsigned i = 1; i < std::min(16u, hw); ++i) threads_.emplace_back([this, i] { loop(i); });
        for (auto& t : threads_) t.detach();
    }
    void loop(unsigned id) {
        unsigned long long seen = 0;
        for (;;) {
            const std::function<void(unsigned)>* f;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
                if (id >= parts_) continue;
                f = fn_;
            }
            (*f)(id);
            std::lock_guard<std::mutex> lk(mu_);
            if (--pending_ == 0) done_.notify_one();
        }
    }
    pid_t pid_ = getpid();
    std::vector<std::thread> threads_;
    std::mutex mu_, job_mu_;
    std::condition_variable cv_, done_;
    const std::function<void(unsigned)>* fn_ = nullptr;
    unsigned parts_ = 0, pending_ = 0;
    unsigned long long gen_ = 0;
};

// Solution arrays: 2 MiB-aligned and advised as huge pages when large, so filling a 40 MB result
// costs tens of page faults instead of ten thousand. Freed with free() (cubics_solutions_free).
int64_t* alloc_values(uint64_t count) {
    const size_t bytes = sizeof(int64_t) * count;
    void* p = nullptr;
    if (bytes >= (size_t(4) << 20)) {
        const size_t huge = size_t(2) << 20;
        if (posix_memalign(&p, huge, (bytes + huge - 1) / huge * huge) != 0) p = nullptr;
        if (p) madvise(p, (bytes + huge - 1) / huge * huge, MADV_HUGEPAGE);
    }
    if (!p) p = std::malloc(std::max<size_t>(bytes, 8));
    if (!p) throw std::bad_alloc();
    return static_cast<int64_t*>(p);
}

extern "C" int cubics_enumerate(const cubics_model* h, const cubics_search_config* cfg, cubics_solutions** sols,
                                cubics_result* out) {
    if (!h || !cfg || !out || !sols) return CUBICS_E_INVALID;
    *sols = nullptr;
    return guarded([&] {
        const double t0 = now_ms();
        const HostModel& m = h->m;
        const int n = m.n_vars();
        if (capped_stream(m, *cfg)) { // the first k solutions, streamed from the parallel engine
            std::vector<uint16_t> rows;
            stream_satisfy(m, *cfg, CUBICS_ENGINE_PARALLEL, cfg->max_solutions,
                           [&](const uint16_t* row) {
                               if (!cfg->count_only) rows.insert(rows.end(), row, row + n);
                               return true;
                           },
                           out);
            const uint64_t count = n ? rows.size() / n : 0;
            int64_t* values = alloc_values(std::max<uint64_t>(rows.size(), 1));
            auto* S = new cubics_solutions{};
            S->n_vars = n;
            S->count = count;
            S->values = values;
            for (uint64_t i = 0; i < count; ++i)
                for (int v = 0; v < n; ++v) values[i * n + v] = m.offset[v] + rows[i * n + v];
            *sols = S;
            out->total_ms = now_ms() - t0;
            return (int)CUBICS_OK;
        }
        // the rows arrive in the device's pinned download buffer: hold the device until converted
        std::lock_guard<std::recursive_mutex> lock(g_dev_mu[current_device(cfg->device)]);
        RunOut r = satisfy_run(m, *cfg, !cfg->count_only, out, true, true);
        const double t1 = now_ms();
        if (r.values64) { // already int64 in a pinned buffer: no host conversion
            auto* S = new cubics_solutions{};
            S->n_vars = n;
            S->count = r.rec.count;
            S->values = r.values64;
            *sols = S;
            out->total_ms = now_ms() - t0;
            if (std::getenv("CUBICS_DEBUG"))
                std::fprintf(stderr, "[cubics] enumerate: search+download %.3f ms (device %.3f), int64 on the device, %llu rows\n",
                             t1 - t0, out->device_ms, (unsigned long long)r.rec.count);
            return (int)CUBICS_OK;
        }
        const uint64_t total = r.rec.count * (uint64_t)n;
        int64_t* values = alloc_values(std::max<uint64_t>(total, 1)); // before the struct: no leak on throw
        auto* S = new cubics_solutions{};
        S->n_vars = n;
        S->count = r.rec.count;
        S->values = values;
        // offset conversion straight into the returned buffer, split over host threads
        const unsigned nt = total > (1u << 20) ? HostPool::get().size() : 1u;
        const uint64_t count = r.rec.count;
        const uint16_t* rows = r.rec.rows();
        HostPool::get().run(nt, [&](unsigned t) {
            for (uint64_t i = count * t / nt; i < count * (t + 1) / nt; ++i) {
                const uint16_t* row = rows + i * n;
                int64_t* dst = S->values + i * n;
                for (int v = 0; v < n; ++v) dst[v] = m.offset[v] + row[v];
            }
        });
        *sols = S;
        out->total_ms = now_ms() - t0;
        if (std::getenv("CUBICS_DEBUG"))
            std::fprintf(stderr, "[cubics] enumerate: search+download %.3f ms (device %.3f), convert %.3f ms, %llu rows\n",
                         t1 - t0, out->device_ms, now_ms() - t1, (unsigned long long)r.rec.count);
        return (int)CUBICS_OK;
    });
}

extern "C" void cubics_solutions_free(cubics_solutions* s) {
    if (!s) return;
    if (!PinnedPool::get().give_back(s->values)) std::free(s->values);
    delete s;
}

namespace {
// Exact parallel branch and bound: the reference's solve_optimize (search.cpp:187-201) - node
// order, every stat, every incumbent - at parallel-engine speed. Between two improving solutions
// K_i and K_i+1 (DFS order) the reference's bound is constant, v_i. So the search is a chain of
// exact-first-solution searches, each with a static bound:
//   phase 0: the DFS-first solution of the whole tree (no bound): K_1, and the reference's stats
//            up to it (segment prefix sums, as for max_solutions == 1);
//   phase i: replay K_i's path from the root on the reference-order kernel, with the bound the
//            reference had when it entered each node on it (the last K_j left of that node), and
//            emit the right branch of every left decision on the path - exactly the branches the
//            reference still has pending when it reaches K_i; seed them (DFS order) into the
//            parallel engine's exact-first search under the static bound v_i: K_i+1 and the
//            stats from K_i to it. No K_i+1: that phase searched the rest of the tree.
// The stats are the sums over the phases; the solutions are the K_i.
// visit (may be null) receives each incumbent in order (the reference's solution stream of a
// B&B search); false stops, as does the cfg0.max_solutions-th incumbent (complete = 0).
void exact_bnb(const HostModel& m, const cubics_search_config& cfg0, std::vector<uint16_t>& best, cubics_result* out,
               const std::function<bool(const uint16_t*)>* visit) {
    NvtxRange nvtx("cubics exact B&B");
    const int n = m.n_vars();
    const bool minimizing = m.goal == CUBICS_MINIMIZE;
    cubics_search_config c = cfg0;
    c.engine = CUBICS_ENGINE_PARALLEL;
    uint64_t tot[3] = {0, 0, 0}, sols = 0;
    std::vector<std::vector<uint32_t>> keys; // K_1, K_2, ... (increasing DFS order)
    std::vector<int64_t> objs;
    auto add = [&](const RunOut& r) {
        out->device_ms += r.device_ms;
        out->h2d_bytes += r.h2d;
        out->d2h_bytes += r.d2h;
        out->kernel_launches += r.launches;
        out->contexts = std::max(out->contexts, r.contexts);
    };
    auto objective = [&](const uint16_t* row) { return m.offset[m.goal_var] + (int64_t)row[m.goal_var]; };
    int KW = 0;
    bool stopped = false;
    auto incumbent = [&]() { // deliver K_i; true: stop here
        if (visit && !(*visit)(best.data())) return stopped = true;
        return stopped = sols >= cfg0.max_solutions;
    };
    { // phase 0
        RunOut r;
        ShardIO io;
        io.root_first = true;
        io.first = 1;
        io.static_bound = true;
        run_search(m, c, CUBICS_ENGINE_PARALLEL, true, 65536, r, true, &io);
        add(r);
        KW = r.KW;
        for (int i = 0; i < 3; ++i) tot[i] += r.ws.stats[i];
        if (r.has_first) {
            keys.push_back(r.first_key);
            best.assign(r.rec.vals.begin(), r.rec.vals.begin() + n);
            objs.push_back(objective(best.data()));
            ++sols;
            incumbent();
        }
    }
    // the outbox layout of the replay's tasks (once: prepare() flattens the whole model)
    const int dev = current_device(c.device);
    size_t NWP = 0;
    if (!keys.empty() && !stopped) {
        Prepared P0;
        prepare(m, m.words.data(), P0);
        NWP = P0.NWP;
    }
    const size_t OS = NWP + dev::round4((size_t)KW + 2);
    while (!keys.empty() && !stopped) {
        const std::vector<uint32_t>& K = keys.back();
        // the bound in force when the reference entered the node at depth d of K's path
        const size_t gd = (size_t)KW * 32 + 1;
        ShardIO rp;
        rp.guide_key = &K;
        rp.guide_bound.assign(gd, 0);
        rp.guide_has.assign(gd, 0);
        std::vector<uint32_t> node(KW);
        for (size_t d = 0; d < gd; ++d) {
            for (int w = 0; w < KW; ++w) {
                const long c0 = (long)d - 32L * w; // prefix bits of word w that are kept
                node[w] = c0 <= 0 ? 0u : (c0 >= 32 ? K[w] : (K[w] & ~(0xffffffffu >> c0)));
            }
            int64_t b = cfg0.initial_bound;
            int32_t hb = cfg0.has_initial_bound ? 1 : 0;
            for (size_t j = 0; j < keys.size(); ++j)
                if (std::lexicographical_compare(keys[j].begin(), keys[j].end(), node.begin(), node.end())) {
                    b = objs[j];
                    hb = 1;
                }
            rp.guide_bound[d] = b;
            rp.guide_has[d] = hb;
        }
        rp.task_cap = gd;
        rp.task_dev = reinterpret_cast<uint32_t*>(device_arena(dev, sizeof(uint32_t) * OS * rp.task_cap, 1));
        cubics_search_config cr = c;
        cr.engine = CUBICS_ENGINE_PARITY;
        RunOut rr;
        run_search(m, cr, CUBICS_ENGINE_PARITY, false, 0, rr, false, &rp);
        add(rr);
        const uint64_t nt = rp.n_tasks;
        if (nt > rp.task_cap) throw StatusError{CUBICS_E_INVALID, "exact B&B: replay emitted more branches than its depth"};
        if (nt == 0) break; // nothing right of K_i: the search is complete
        std::vector<uint32_t> tkey(nt * KW);
        CU(cudaMemcpy2D(tkey.data(), sizeof(uint32_t) * KW, rp.task_dev + NWP, sizeof(uint32_t) * OS,
                        sizeof(uint32_t) * KW, nt, cudaMemcpyDeviceToHost));
        std::vector<int32_t> seeds(nt);
        std::iota(seeds.begin(), seeds.end(), 0);
        std::sort(seeds.begin(), seeds.end(), [&](int32_t x, int32_t y) {
            return std::lexicographical_compare(tkey.begin() + (size_t)x * KW, tkey.begin() + (size_t)(x + 1) * KW,
                                                tkey.begin() + (size_t)y * KW, tkey.begin() + (size_t)(y + 1) * KW);
        });
        ShardIO ph;
        ph.task_dev = rp.task_dev;
        ph.seeds = &seeds;
        ph.first = 1;
        ph.static_bound = true;
        ph.prefix_sum = true; // best solution + prefix stats summed on the device
        cubics_search_config cp = c;
        cp.has_initial_bound = 1;
        cp.initial_bound = objs.back();
        RunOut pr;
        run_search(m, cp, CUBICS_ENGINE_PARALLEL, true, 65536, pr, true, &ph);
        add(pr);
        // K_i+1 (the phase's DFS-first solution) and the reference's stats up to it, or the whole
        // rest of the tree when the phase found none
        for (int i = 0; i < 3; ++i) tot[i] += pr.ws.stats[i];
        if (!pr.has_first) break; // no improving solution right of K_i: complete
        keys.push_back(pr.first_key);
        best.assign(pr.rec.vals.begin(), pr.rec.vals.begin() + n);
        const int64_t v = objective(best.data());
        if (!(minimizing ? v < objs.back() : v > objs.back()))
            throw StatusError{CUBICS_E_INVALID, "exact B&B: a phase returned a non-improving solution"};
        objs.push_back(v);
        ++sols;
        incumbent();
    }
    out->stats.nodes = tot[0];
    out->stats.failures = tot[1];
    out->stats.rounds = tot[2];
    out->stats.solutions = sols;
    out->engine = CUBICS_ENGINE_PARALLEL;
    out->complete = stopped ? 0 : 1;
}
} // namespace

extern "C" int cubics_solve_optimize(const cubics_model* h, const cubics_search_config* cfg, int64_t* best_values,
                                     cubics_result* out) {
    if (!h || !cfg || !out) return CUBICS_E_INVALID;
    return guarded([&] {
        const double t0 = now_ms();
        std::memset(out, 0, sizeof *out);
        const HostModel& m = h->m;
        if (m.goal == CUBICS_SATISFY) throw StatusError{CUBICS_E_NO_OBJECTIVE, "solve_optimize requires a minimize or maximize goal"};
        cubics_search_config c = *cfg;
        const int n = m.n_vars();
        // AUTO: the exact parallel branch and bound (reference stats and incumbents); the
        // reference-order engine for node-limited / solution-capped searches
        if (c.engine == CUBICS_ENGINE_AUTO && c.node_limit == 0 && c.max_solutions > 0 && n > 0 &&
            !std::getenv("CUBICS_NO_EXACT_BNB")) {
            std::vector<uint16_t> best;
            bool done = false;
            try {
                exact_bnb(m, c, best, out);
                done = true;
            } catch (const StatusError& e) {
                if (e.code != CUBICS_E_CAPACITY) throw;
                std::memset(out, 0, sizeof *out); // bookkeeping capacity: the reference-order engine
            }
            if (done) {
                out->complete = 1; // fd::solve_optimize: complete = !limit_hit (search.cpp:197)
                out->has_solution = !best.empty();
                if (!best.empty()) {
                    out->objective = m.offset[m.goal_var] + best[m.goal_var];
                    if (best_values)
                        for (int v = 0; v < n; ++v) best_values[v] = m.offset[v] + best[v];
                }
                out->total_ms = now_ms() - t0;
                return (int)CUBICS_OK;
            }
        }
        if (c.engine == CUBICS_ENGINE_AUTO) c.engine = CUBICS_ENGINE_PARITY;
        const int engine = pick_engine(c, true);
        RunOut r;
        // parity: every incumbent is recorded in order (max_solutions bounds them); parallel: global incumbent
        const bool parallel = engine == CUBICS_ENGINE_PARALLEL;
        run_search(m, c, engine, !parallel, parallel ? 0 : default_sol_cap(m, c), r);
        fill_result(r, out);
        out->complete = !r.ws.limit_hit;
        std::vector<uint16_t> best;
        if (parallel) {
            if (r.ws.inc_found) best = r.inc_vals;
        } else if (r.rec.count) {
            best.assign(r.rec.vals.end() - n, r.rec.vals.end());
        }
        out->has_solution = !best.empty() || (n == 0 && r.ws.stats[3] > 0);
        if (!best.empty()) {
            out->objective = m.offset[m.goal_var] + best[m.goal_var];
            if (best_values)
                for (int v = 0; v < n; ++v) best_values[v] = m.offset[v] + best[v];
        }
        out->total_ms = now_ms() - t0;
        return (int)CUBICS_OK;
    });
}

extern "C" int cubics_solve_optimize_batch(const cubics_model* h, const cubics_search_config* cfg, int32_t count,
                                           const uint64_t* words, const int64_t* bounds, const int32_t* has_bounds,
                                           int64_t* best_values, cubics_result* results) {
    if (!h || !cfg || count < 0 || (count > 0 && (!words || !results))) return CUBICS_E_INVALID;
    return guarded([&] {
        const double t0 = now_ms();
        const HostModel& m = h->m;
        if (m.goal == CUBICS_SATISFY) throw StatusError{CUBICS_E_NO_OBJECTIVE, "solve_optimize requires a minimize or maximize goal"};
        if (count == 0) return CUBICS_OK;
        std::memset(results, 0, sizeof(cubics_result) * count);
        const int n = m.n_vars();
        BatchIO b;
        b.count = count;
        b.words = words;
        b.bound.assign(count, 0);
        b.has_bound.assign(count, 0);
        for (int i = 0; i < count; ++i) {
            b.has_bound[i] = has_bounds ? has_bounds[i] != 0 : (bounds != nullptr);
            b.bound[i] = bounds ? bounds[i] : 0;
        }
        // No per-problem node limit (fd::lns_optimize without per_iteration_node_limit): the batch
        // runs under a node budget, and a problem that exhausts it is searched again from scratch by
        // the exact parallel B&B - the whole GPU, the reference's stats and incumbent - so an LNS
        // iteration no longer waits for its slowest neighbourhood on one thread block.
        const bool handoff = cfg->node_limit == 0 && cfg->max_solutions == std::numeric_limits<uint64_t>::max() &&
                             n > 0 && !std::getenv("CUBICS_NO_BATCH_HANDOFF");
        cubics_search_config cbud = *cfg;
        if (handoff) {
            const char* b = std::getenv("CUBICS_BATCH_BUDGET"); // A/B only
            cbud.node_limit = b ? std::max(1, std::atoi(b)) : 4096;
        }
        RunOut r;
        run_search(m, cbud, CUBICS_ENGINE_PARITY, false, 0, r, false, nullptr, &b);
        const size_t nw64 = m.words.size();
        for (int i = 0; i < count; ++i) {
            cubics_result& o = results[i];
            fill_result(r, &o);
            if (handoff && (b.flags[i] & 1)) { // over budget: the exact parallel B&B instead
                HostModel mi = m;
                mi.words.assign(words + nw64 * i, words + nw64 * (i + 1));
                cubics_search_config ce = *cfg;
                ce.engine = CUBICS_ENGINE_AUTO;
                ce.has_initial_bound = b.has_bound[i];
                ce.initial_bound = b.bound[i];
                std::vector<uint16_t> best;
                cubics_result e{};
                exact_bnb(mi, ce, best, &e);
                o.stats = e.stats;
                o.complete = 1;
                o.has_solution = !best.empty();
                o.device_ms += e.device_ms;
                o.kernel_launches += e.kernel_launches;
                if (!best.empty()) {
                    o.objective = m.offset[m.goal_var] + best[m.goal_var];
                    if (best_values)
                        for (int v = 0; v < n; ++v) best_values[(size_t)n * i + v] = m.offset[v] + best[v];
                }
                o.contexts = count;
                o.total_ms = now_ms() - t0;
                continue;
            }
            o.stats.nodes = b.stats[4 * i + 0];
            o.stats.failures = b.stats[4 * i + 1];
            o.stats.rounds = b.stats[4 * i + 2];
            o.stats.solutions = b.stats[4 * i + 3];
            o.complete = !(b.flags[i] & 1);
            o.has_solution = (b.flags[i] & 2) != 0 || (n == 0 && o.stats.solutions > 0);
            if (b.flags[i] & 2) {
                const uint16_t* inc = b.inc.data() + (size_t)n * i;
                o.objective = m.offset[m.goal_var] + inc[m.goal_var];
                if (best_values)
                    for (int v = 0; v < n; ++v) best_values[(size_t)n * i + v] = m.offset[v] + inc[v];
            }
            o.contexts = count;
            o.total_ms = now_ms() - t0;
        }
        return CUBICS_OK;
    });
}

namespace {
// Shared queue state (256 bytes in the owner GPU's HBM, CUDA IPC-mapped by the other ranks):
//   [0]  u32 claim counter              (next frontier subtree to claim)
//   [8]  u64 shared incumbent, encoded   (bound_enc in search.cuh; all ones = none)
//   [16] u64 first 64 key bits of the best first solution any rank found (all ones = none)
//   [128] XsCtl: cross-GPU stealing counters (device_model.hpp)
//   [256] the global pool of stolen right branches: kXsBytes of slots, geometry per search
struct QueueState {
    uint32_t claim;
    uint32_t pad;
    unsigned long long g_inc;
    unsigned long long g_first;
};

// The search device must reach the queue owner's memory: peer access inside one process (CUDA
// IPC mappings from another process enable it themselves, cudaIpcMemLazyEnablePeerAccess).
void ensure_queue_access(int dev, const cubics_task_queue* q) {
    if (!q || q->device == dev || !q->owner) return;
    int ok = 0;
    CU(cudaDeviceCanAccessPeer(&ok, dev, q->device));
    if (!ok) throw StatusError{CUBICS_E_UNSUPPORTED, "search device cannot access the task queue's GPU (no peer access)"};
    CU(cudaSetDevice(dev));
    const cudaError_t e = cudaDeviceEnablePeerAccess(q->device, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
    } else {
        CU(e);
    }
}

// One rank's share of a multi-GPU search (satisfy: every solution, keyed; optimize: branch and
// bound with the incumbent shared through the queue state). queue == nullptr: static split
// (task t goes to shard t % shard_count); otherwise every shard seeds all tasks in DFS order
// and claims them dynamically through the shared counter.
int solve_shard_impl(const cubics_model* h, const cubics_search_config* cfg, int32_t shard_index,
                     int32_t shard_count, cubics_task_queue* queue, cubics_keyed_solution_cb cb, void* user,
                     cubics_result* out, bool optimize, int64_t* best_values) {
    if (!h || !cfg || !out || shard_count < 1 || shard_index < 0 || shard_index >= shard_count) return CUBICS_E_INVALID;
    return guarded([&]() -> int {
        const double t0 = now_ms();
        std::memset(out, 0, sizeof *out);
        const HostModel& m = h->m;
        if (optimize && m.goal == CUBICS_SATISFY)
            throw StatusError{CUBICS_E_NO_OBJECTIVE, "solve_optimize requires a minimize or maximize goal"};
        if (!optimize && m.goal != CUBICS_SATISFY)
            throw StatusError{CUBICS_E_UNSUPPORTED, "sharded enumeration needs a satisfy goal (use cubics_solve_optimize_shard)"};
        cubics_search_config c = *cfg;
        c.engine = CUBICS_ENGINE_PARALLEL;
        pick_engine(c, optimize);
        const bool record = !optimize && cb && !c.count_only;
        const int n = m.n_vars();
        const int dev = current_device(c.device);
        ensure_queue_access(dev, queue);
        QueueState* qs = queue ? reinterpret_cast<QueueState*>(queue->counter) : nullptr;
        std::vector<int64_t> vals(n);
        auto deliver = [&](const RunOut& r) {
            for (uint64_t s = 0; s < r.rec.count; ++s) {
                for (int v = 0; v < n; ++v) vals[v] = m.offset[v] + r.rec.vals[s * n + v];
                if (!cb(user, r.rec.keys.data() + s * r.KW, r.KW, vals.data(), n)) return false;
            }
            return true;
        };
        // a recorded run that found more solutions than its buffer: rerun with the exact size, or
        // fail loudly when it cannot be repeated (claims through the shared queue are spent)
        auto full_records = [&](RunOut& r, auto&& rerun, bool repeatable) {
            if (!record || r.ws.sol_count <= r.rec.count) return;
            if (!repeatable)
                throw StatusError{CUBICS_E_CAPACITY, "shard solution buffer overflow (shared-queue run cannot be repeated)"};
            const uint64_t want = r.ws.sol_count;
            r = RunOut{};
            rerun(want);
        };
        // best solution of this rank (optimize): objective and values
        bool has_best = false;
        int64_t best_obj = 0;
        std::vector<int64_t> best(n);
        auto offer = [&](const uint16_t* row) {
            const int64_t obj = m.offset[m.goal_var] + row[m.goal_var];
            if (has_best && (m.goal == CUBICS_MINIMIZE ? obj >= best_obj : obj <= best_obj)) return;
            has_best = true;
            best_obj = obj;
            for (int v = 0; v < n; ++v) best[v] = m.offset[v] + row[v];
        };
        auto finish = [&]() {
            if (optimize) {
                out->has_solution = has_best;
                if (has_best) {
                    out->objective = best_obj;
                    if (best_values) std::copy(best.begin(), best.end(), best_values);
                }
            } else {
                out->has_solution = out->stats.solutions > 0;
            }
            out->complete = 1;
            out->total_ms = now_ms() - t0;
            return CUBICS_OK;
        };
        if (shard_count == 1) {
            RunOut r;
            ShardIO one;
            one.g_inc = qs ? &qs->g_inc : nullptr;
            auto go = [&](uint64_t cap) {
                run_search(m, c, CUBICS_ENGINE_PARALLEL, record, record ? cap : 0, r, true, qs ? &one : nullptr);
            };
            go(record ? default_sol_cap(m, c) : 0);
            full_records(r, go, true);
            fill_result(r, out);
            if (optimize && r.ws.inc_found) offer(r.inc_vals.data());
            if (record) deliver(r);
            return finish();
        }
        // 1. deterministic frontier: expand the tree (in parallel; exact node semantics) until
        //    the open nodes at the split depth are plentiful; they are numbered in DFS order.
        //    Branch and bound expands without the bound (goal cleared), so every rank builds the
        //    same frontier whatever the timing; solutions above the frontier seed the bound.
        Prepared P;
        prepare(m, m.words.data(), P);
        const int KW = static_cast<int>((P.depth_bound + 1 + 31) / 32);
        const size_t OS = P.NWP + dev::round4((size_t)KW + 2);
        std::lock_guard<std::recursive_mutex> lock(g_dev_mu[dev]); // the task buffer lives across two runs
        HostModel sat_model;
        const HostModel* exp_model = &m;
        if (optimize) {
            sat_model = m;
            sat_model.goal = CUBICS_SATISFY;
            exp_model = &sat_model;
        }
        const bool exp_record = record || optimize;
        const uint64_t want = 256ull * (uint64_t)shard_count;
        RunOut ex;
        ShardIO io;
        int depth0 = 8;
        {
            std::lock_guard<std::mutex> hl(h->hint_mu);
            auto it = h->split_hint.find(shard_count);
            if (it != h->split_hint.end()) depth0 = it->second;
        }
        for (int depth = depth0;; depth += 4) {
            io = ShardIO{};
            io.split_depth = depth;
            io.task_cap = std::max<uint64_t>(4096, 8 * want);
            for (;;) {
                io.task_dev = reinterpret_cast<uint32_t*>(device_arena(dev, sizeof(uint32_t) * OS * io.task_cap, 1));
                ex = RunOut{};
                auto go = [&](uint64_t cap) {
                    run_search(*exp_model, c, CUBICS_ENGINE_PARALLEL, exp_record, exp_record ? cap : 0, ex, true, &io);
                };
                go(exp_record ? default_sol_cap(m, c) : 0);
                if (exp_record && ex.ws.sol_count > ex.rec.count) {
                    const uint64_t cap = ex.ws.sol_count;
                    ex = RunOut{};
                    go(cap);
                }
                if (io.n_tasks <= io.task_cap) break;
                io.task_cap = io.n_tasks;
            }
            if (io.n_tasks >= want || io.n_tasks == 0 || depth >= 64 || (uint64_t)depth >= P.depth_bound) {
                std::lock_guard<std::mutex> hl(h->hint_mu);
                h->split_hint[shard_count] = depth;
                break;
            }
        }
        if (optimize)
            for (uint64_t s = 0; s < ex.rec.count; ++s) offer(ex.rec.vals.data() + s * n);
        // 2. DFS rank of each task = order of its path key
        const uint64_t nt = io.n_tasks;
        std::vector<uint32_t> keys(nt * KW);
        if (nt)
            CU(cudaMemcpy2D(keys.data(), sizeof(uint32_t) * KW, io.task_dev + P.NWP, sizeof(uint32_t) * OS,
                            sizeof(uint32_t) * KW, nt, cudaMemcpyDeviceToHost));
        std::vector<int32_t> order(nt);
        std::iota(order.begin(), order.end(), 0);
        std::sort(order.begin(), order.end(), [&](int32_t x, int32_t y) {
            return std::lexicographical_compare(keys.begin() + (size_t)x * KW, keys.begin() + (size_t)(x + 1) * KW,
                                                keys.begin() + (size_t)y * KW, keys.begin() + (size_t)(y + 1) * KW);
        });
        std::vector<int32_t> mine;
        uint64_t extra_d2h = 0;
        if (qs) {
            // shared queue: claim the (estimated) largest subtrees first, so the last claims are
            // small and the GPUs finish together (list scheduling, largest first). Estimate =
            // log2 of the product of the task's domain sizes; every rank computes the same order.
            std::vector<uint32_t> tdom(nt * P.NWP);
            if (nt)
                CU(cudaMemcpy2D(tdom.data(), sizeof(uint32_t) * P.NWP, io.task_dev, sizeof(uint32_t) * OS,
                                sizeof(uint32_t) * P.NWP, nt, cudaMemcpyDeviceToHost));
            std::vector<double> est(nt, 0.0);
            for (uint64_t t = 0; t < nt; ++t)
                for (int v = 0; v < n; ++v) {
                    int sz = 0;
                    for (int w = 0; w < P.W; ++w) sz += __builtin_popcount(tdom[t * P.NWP + (size_t)v * P.W + w]);
                    if (sz > 1) est[t] += std::log2((double)sz);
                }
            mine = order;
            std::stable_sort(mine.begin(), mine.end(), [&](int32_t x, int32_t y) { return est[x] > est[y]; });
            extra_d2h = sizeof(uint32_t) * P.NWP * nt;
        } else
            for (uint64_t r = shard_index; r < nt; r += shard_count) mine.push_back(order[r]);
        // 3. this shard's subtrees, seeded into the parallel engine (B&B: starting from the best
        //    solution above the frontier, and sharing incumbents through the queue state)
        cubics_search_config cs = c;
        if (optimize && has_best &&
            (!cs.has_initial_bound || (m.goal == CUBICS_MINIMIZE ? best_obj < cs.initial_bound : best_obj > cs.initial_bound))) {
            cs.has_initial_bound = 1;
            cs.initial_bound = best_obj;
        }
        RunOut run;
        if (!mine.empty()) {
            ShardIO seeded;
            seeded.task_dev = io.task_dev;
            seeded.seeds = &mine;
            seeded.claim = qs ? &qs->claim : nullptr;
            seeded.g_inc = qs && optimize ? &qs->g_inc : nullptr;
            seeded.xs = qs ? reinterpret_cast<uint8_t*>(qs) : nullptr;
            auto go = [&](uint64_t cap) {
                run_search(m, cs, CUBICS_ENGINE_PARALLEL, record, record ? cap : 0, run, true, &seeded);
            };
            go(record ? default_sol_cap(m, c) : 0);
            full_records(run, go, qs == nullptr);
            if (optimize && run.ws.inc_found) offer(run.inc_vals.data());
        }
        fill_result(run, out);
        if (shard_index == 0) { // nodes above the frontier belong to shard 0
            out->stats.nodes += ex.ws.stats[0];
            out->stats.failures += ex.ws.stats[1];
            out->stats.rounds += ex.ws.stats[2];
            out->stats.solutions += ex.ws.stats[3];
        }
        out->device_ms = run.device_ms + ex.device_ms;
        out->h2d_bytes += ex.h2d;
        out->d2h_bytes += ex.d2h + sizeof(uint32_t) * KW * nt + extra_d2h;
        out->kernel_launches += ex.launches;
        if (record) {
            if (shard_index == 0 && !deliver(ex)) return finish();
            if (!mine.empty()) deliver(run);
        }
        return finish();
    });
}
} // namespace

// Sharded exact first solution (fd::solve_satisfy, max_solutions == 1, search.cpp:174-186, across
// GPUs). The reference's stats are those of the DFS prefix up to its first solution K*. Every
// part of the sharded search is a sequence of segments, contiguous intervals of the DFS order
// with a root key and stats: the frontier expansion's (intervals of the tree cut at the split
// depth; each task records where it sits in one of them) and each rank's seeded subtrees'
// (claimed / pre-published seeds and the right branches donated inside them). So the prefix up to
// K* is, summed over all ranks: the segments whose root key is below K*, except K*'s own, plus
// the snapshot of K*'s own segment taken at K* - in the frontier tree (rank 0) with K*'s task
// (or K* itself when it lies above the frontier) in place of K*.
struct cubics_first_shard {
    int KW = 0, n = 0;
    bool rank0 = false;
    std::vector<int64_t> offset;
    uint64_t raw[4] = {0, 0, 0, 0}; // this rank's own work (its stats when there is no solution)
    // frontier expansion (identical on every rank)
    uint64_t nfseg = 0;
    std::vector<uint32_t> fseg_key;
    std::vector<uint64_t> fseg_st;
    std::vector<uint32_t> task_key;  // [nt][KW] in emission order
    std::vector<uint64_t> task_snap; // [nt][4] segment, nodes, failures, rounds
    Records fsol;                    // solutions above the frontier (keys, segments, snapshots)
    // this rank's seeded run
    uint64_t nseg = 0;
    std::vector<uint32_t> seg_key;
    std::vector<uint64_t> seg_st;
    Records sol;

    bool less(const uint32_t* a, const uint32_t* b) const { return std::lexicographical_compare(a, a + KW, b, b + KW); }
    bool equal(const uint32_t* a, const uint32_t* b) const { return std::equal(a, a + KW, b); }
    // segments [0, count) with root key < K, except `skip`
    static void sum_left(const cubics_first_shard& s, uint64_t count, const std::vector<uint32_t>& keys,
                         const std::vector<uint64_t>& st, const uint32_t* K, int64_t skip, uint64_t* tot) {
        for (uint64_t i = 0; i < count; ++i)
            if ((int64_t)i != skip && s.less(&keys[i * s.KW], K))
                for (int j = 0; j < 3; ++j) tot[j] += st[i * 3 + j];
    }
};

namespace {
int first_shard_impl(const cubics_model* h, const cubics_search_config* cfg, int32_t shard_index, int32_t shard_count,
                     cubics_task_queue* queue, cubics_first_shard** res, cubics_result* out) {
    if (!h || !cfg || !out || !res || shard_count < 1 || shard_index < 0 || shard_index >= shard_count)
        return CUBICS_E_INVALID;
    *res = nullptr;
    return guarded([&]() -> int {
        const double t0 = now_ms();
        std::memset(out, 0, sizeof *out);
        const HostModel& m = h->m;
        if (m.goal != CUBICS_SATISFY)
            throw StatusError{CUBICS_E_UNSUPPORTED, "sharded first solution needs a satisfy goal"};
        cubics_search_config c = *cfg;
        c.engine = CUBICS_ENGINE_PARALLEL;
        c.max_solutions = 1;
        pick_engine(c, false); // rejects node_limit
        const int n = m.n_vars();
        const int dev = current_device(c.device);
        ensure_queue_access(dev, queue);
        QueueState* qs = queue ? reinterpret_cast<QueueState*>(queue->counter) : nullptr;
        std::unique_ptr<cubics_first_shard> fs(new cubics_first_shard);
        fs->n = n;
        fs->rank0 = shard_index == 0;
        fs->offset = m.offset;
        Prepared P;
        prepare(m, m.words.data(), P);
        const int KW = static_cast<int>((P.depth_bound + 1 + 31) / 32);
        fs->KW = KW;
        const size_t OS = P.NWP + dev::round4((size_t)KW + 2);
        std::lock_guard<std::recursive_mutex> lock(g_dev_mu[dev]);
        // 1. the deterministic frontier, with segment bookkeeping (no abandoning: the task set
        //    must not depend on timing) and its solutions recorded
        const uint64_t want = 256ull * (uint64_t)shard_count;
        RunOut ex;
        ShardIO io;
        for (int depth = 8;; depth += 4) {
            io = ShardIO{};
            io.split_depth = depth;
            io.first = 2;
            io.task_cap = std::max<uint64_t>(4096, 8 * want);
            for (;;) {
                io.task_dev = reinterpret_cast<uint32_t*>(device_arena(dev, sizeof(uint32_t) * OS * io.task_cap, 1));
                ex = RunOut{};
                cubics_search_config all = c;
                all.max_solutions = std::numeric_limits<uint64_t>::max();
                run_search(m, c, CUBICS_ENGINE_PARALLEL, true, default_sol_cap(m, all), ex, true, &io);
                if (ex.ws.sol_count > ex.rec.count)
                    throw StatusError{CUBICS_E_CAPACITY, "frontier solution buffer overflow"};
                if (io.n_tasks <= io.task_cap) break;
                io.task_cap = io.n_tasks;
            }
            if (io.n_tasks >= want || io.n_tasks == 0 || depth >= 64 || (uint64_t)depth >= P.depth_bound) break;
        }
        const uint64_t nt = io.n_tasks;
        fs->nfseg = io.n_seg;
        fs->fseg_key = std::move(io.seg_key);
        fs->fseg_st = std::move(io.seg_st);
        fs->task_snap = std::move(io.task_snap);
        fs->task_key.resize(nt * KW);
        if (nt)
            CU(cudaMemcpy2D(fs->task_key.data(), sizeof(uint32_t) * KW, io.task_dev + P.NWP, sizeof(uint32_t) * OS,
                            sizeof(uint32_t) * KW, nt, cudaMemcpyDeviceToHost));
        fs->fsol = std::move(ex.rec);
        // 2. this rank's subtrees in DFS order (static: t = shard_index mod shard_count of the
        //    DFS-ordered tasks; shared queue: all of them, claimed)
        std::vector<int32_t> order(nt);
        std::iota(order.begin(), order.end(), 0);
        std::sort(order.begin(), order.end(), [&](int32_t x, int32_t y) {
            return fs->less(&fs->task_key[(size_t)x * KW], &fs->task_key[(size_t)y * KW]);
        });
        std::vector<int32_t> mine;
        if (qs)
            mine = order;
        else
            for (uint64_t r = shard_index; r < nt; r += shard_count) mine.push_back(order[r]);
        // 3. the exact-first parallel search of those subtrees (abandoning right of this rank's best)
        RunOut run;
        if (!mine.empty()) {
            ShardIO seeded;
            seeded.task_dev = io.task_dev;
            seeded.seeds = &mine;
            seeded.claim = qs ? &qs->claim : nullptr;
            seeded.g_first = qs ? &qs->g_first : nullptr;
            seeded.first = 1;
            run_search(m, c, CUBICS_ENGINE_PARALLEL, true, 65536, run, true, &seeded);
            if (run.ws.sol_count > run.rec.count)
                throw StatusError{CUBICS_E_CAPACITY, "first-solution bookkeeping capacity"};
            fs->nseg = seeded.n_seg;
            fs->seg_key = std::move(seeded.seg_key);
            fs->seg_st = std::move(seeded.seg_st);
            fs->sol = std::move(run.rec);
        }
        fill_result(run, out);
        for (int i = 0; i < 4; ++i) fs->raw[i] = run.ws.stats[i] + (fs->rank0 ? ex.ws.stats[i] : 0);
        out->stats.nodes = fs->raw[0];
        out->stats.failures = fs->raw[1];
        out->stats.rounds = fs->raw[2];
        out->stats.solutions = fs->raw[3];
        out->device_ms = run.device_ms + ex.device_ms;
        out->h2d_bytes += ex.h2d;
        out->d2h_bytes += ex.d2h + sizeof(uint32_t) * KW * nt;
        out->kernel_launches += ex.launches;
        out->has_solution = fs->sol.count + fs->fsol.count > 0;
        out->complete = 0;
        out->total_ms = now_ms() - t0;
        *res = fs.release();
        return CUBICS_OK;
    });
}
} // namespace

extern "C" int cubics_solve_first_shard(const cubics_model* h, const cubics_search_config* cfg, int32_t shard_index,
                                        int32_t shard_count, cubics_task_queue* queue, cubics_first_shard** res,
                                        cubics_result* out) {
    return first_shard_impl(h, cfg, shard_index, shard_count, queue, res, out);
}

extern "C" int cubics_first_shard_best(const cubics_first_shard* s, uint32_t* key, int32_t* key_words, int64_t* values,
                                       int32_t* has) {
    if (!s || !key_words || !has) return CUBICS_E_INVALID;
    const uint32_t* best = nullptr;
    const uint16_t* row = nullptr;
    for (const Records* r : {&s->fsol, &s->sol})
        for (uint64_t i = 0; i < r->count; ++i)
            if (!best || s->less(&r->keys[i * s->KW], best)) {
                best = &r->keys[i * s->KW];
                row = r->rows() + i * s->n;
            }
    *has = best != nullptr;
    const int32_t cap = *key_words;
    *key_words = s->KW;
    if (!best) return CUBICS_OK;
    if (key) {
        if (cap < s->KW) return CUBICS_E_INVALID;
        std::copy_n(best, s->KW, key);
    }
    if (values)
        for (int v = 0; v < s->n; ++v) values[v] = s->offset[v] + row[v];
    return CUBICS_OK;
}

extern "C" int cubics_first_shard_prefix(const cubics_first_shard* s, const uint32_t* key, int32_t key_words,
                                         cubics_stats* out) {
    if (!s || !out) return CUBICS_E_INVALID;
    std::memset(out, 0, sizeof *out);
    if (!key) { // no solution on any rank: the complete search, this rank's share
        out->nodes = s->raw[0];
        out->failures = s->raw[1];
        out->rounds = s->raw[2];
        return CUBICS_OK;
    }
    if (key_words != s->KW) return CUBICS_E_INVALID;
    uint64_t tot[3] = {0, 0, 0};
    auto find = [&](const Records& r) -> int64_t { // K*'s record in r, or -1
        for (uint64_t i = 0; i < r.count; ++i)
            if (s->equal(&r.keys[i * s->KW], key)) return (int64_t)i;
        return -1;
    };
    auto take = [&](const Records& r, int64_t i) { // K*'s segment; its snapshot joins the sum
        for (int j = 0; j < 3; ++j) tot[j] += r.stats[i * 3 + j];
        return (int64_t)r.seg[i];
    };
    const int64_t fi = find(s->fsol); // K* above the frontier (every rank has those records)
    int64_t sseg = -1;
    if (fi < 0) {
        const int64_t si = find(s->sol);
        if (si >= 0) sseg = take(s->sol, si);
    }
    cubics_first_shard::sum_left(*s, s->nseg, s->seg_key, s->seg_st, key, sseg, tot);
    if (s->rank0) { // the frontier tree: K* itself when above the frontier, else the task holding it
        int64_t fseg = -1;
        const uint32_t* at = key;
        if (fi >= 0) {
            fseg = take(s->fsol, fi);
        } else {
            const uint64_t nt = s->task_snap.size() / 4;
            int64_t t = -1;
            for (uint64_t i = 0; i < nt; ++i)
                if (!s->less(key, &s->task_key[i * s->KW]) &&
                    (t < 0 || s->less(&s->task_key[(size_t)t * s->KW], &s->task_key[i * s->KW])))
                    t = (int64_t)i;
            if (t < 0) return CUBICS_E_INVALID; // a key from no task of this search
            fseg = (int64_t)s->task_snap[t * 4];
            for (int j = 0; j < 3; ++j) tot[j] += s->task_snap[t * 4 + 1 + j];
            at = &s->task_key[(size_t)t * s->KW];
        }
        cubics_first_shard::sum_left(*s, s->nfseg, s->fseg_key, s->fseg_st, at, fseg, tot);
        out->solutions = 1;
    }
    out->nodes = tot[0];
    out->failures = tot[1];
    out->rounds = tot[2];
    return CUBICS_OK;
}

extern "C" void cubics_first_shard_free(cubics_first_shard* s) { delete s; }

// Single-process multi-GPU search: one host thread per device runs that rank's shard (the same
// protocol as distributed.solve_distributed, without a collective library: the ranks share this
// process, so the "all-reduce" is a sum here). The shared queue lives on devices[0]; the other
// devices reach it with peer access. This is the multi-GPU path of a C++ host (the adapter's
// fd:: calls use it when CUBICS_DEVICES names several GPUs).
extern "C" int cubics_solve_multi(const cubics_model* h, const cubics_search_config* cfg, int32_t n_devices,
                                  const int32_t* devices, cubics_solution_cb cb, void* user, int64_t* best_values,
                                  cubics_result* out) {
    if (!h || !cfg || !out || n_devices < 1 || !devices) return CUBICS_E_INVALID;
    return guarded([&]() -> int {
        const double t0 = now_ms();
        std::memset(out, 0, sizeof *out);
        const HostModel& m = h->m;
        const int n = m.n_vars(), N = n_devices;
        const bool optimize = m.goal != CUBICS_SATISFY;
        const bool first = !optimize && cfg->max_solutions == 1;
        if (cfg->node_limit || (!optimize && !first && cfg->max_solutions != std::numeric_limits<uint64_t>::max()))
            throw StatusError{CUBICS_E_UNSUPPORTED,
                              "multi-GPU search: complete enumeration, first solution or optimization, no node limit"};
        cubics_task_queue* q = nullptr;
        int rc = cubics_task_queue_create(devices[0], &q, nullptr);
        if (rc) return rc;
        struct QueueGuard {
            cubics_task_queue* q;
            ~QueueGuard() { cubics_task_queue_destroy(q); }
        } qg{q};
        if ((rc = cubics_task_queue_reset(q))) return rc;
        using Row = std::pair<std::vector<uint32_t>, std::vector<int64_t>>;
        std::vector<cubics_result> res(N);
        std::vector<int> rcs(N, 0);
        std::vector<std::string> errs(N);
        std::vector<std::vector<Row>> rows(N);
        std::vector<std::vector<int64_t>> bests(N, std::vector<int64_t>(std::max(n, 1)));
        std::vector<std::unique_ptr<cubics_first_shard>> parts(N);
        const bool collect = !optimize && !first && cb && !cfg->count_only;
        cubics_keyed_solution_cb keyed = [](void* u, const uint32_t* key, int32_t kw, const int64_t* vals,
                                            int32_t nv) -> int32_t {
            static_cast<std::vector<Row>*>(u)->emplace_back(std::vector<uint32_t>(key, key + kw),
                                                            std::vector<int64_t>(vals, vals + nv));
            return 1;
        };
        std::vector<std::thread> th;
        for (int r = 0; r < N; ++r)
            th.emplace_back([&, r] {
                cubics_search_config c = *cfg;
                c.device = devices[r];
                if (first) {
                    cubics_first_shard* p = nullptr;
                    rcs[r] = first_shard_impl(h, &c, r, N, q, &p, &res[r]);
                    parts[r].reset(p);
                } else if (optimize) {
                    rcs[r] = solve_shard_impl(h, &c, r, N, q, nullptr, nullptr, &res[r], true, bests[r].data());
                } else {
                    rcs[r] = solve_shard_impl(h, &c, r, N, q, collect ? keyed : nullptr, &rows[r], &res[r], false, nullptr);
                }
                if (rcs[r]) errs[r] = cubics_last_error();
            });
        for (auto& t : th) t.join();
        for (int r = 0; r < N; ++r)
            if (rcs[r]) {
                set_error("rank " + std::to_string(r) + ": " + errs[r]);
                return rcs[r];
            }
        for (int r = 0; r < N; ++r) { // the "all-reduce"
            out->stats.nodes += res[r].stats.nodes;
            out->stats.failures += res[r].stats.failures;
            out->stats.rounds += res[r].stats.rounds;
            out->stats.solutions += res[r].stats.solutions;
            out->device_ms = std::max(out->device_ms, res[r].device_ms);
            out->h2d_bytes += res[r].h2d_bytes;
            out->d2h_bytes += res[r].d2h_bytes;
            out->kernel_launches += res[r].kernel_launches;
            out->remote_tasks_in += res[r].remote_tasks_in;
            out->remote_tasks_out += res[r].remote_tasks_out;
            out->contexts += res[r].contexts;
        }
        out->engine = CUBICS_ENGINE_PARALLEL;
        out->complete = 1;
        if (optimize) { // the best incumbent over the ranks (ties: the lowest rank)
            int br = -1;
            for (int r = 0; r < N; ++r)
                if (res[r].has_solution &&
                    (br < 0 || (m.goal == CUBICS_MINIMIZE ? res[r].objective < res[br].objective
                                                          : res[r].objective > res[br].objective)))
                    br = r;
            out->has_solution = br >= 0;
            if (br >= 0) {
                out->objective = res[br].objective;
                if (best_values) std::copy_n(bests[br].begin(), n, best_values);
                if (cb && !cfg->count_only) cb(user, bests[br].data(), n);
            }
        } else if (first) { // min key over the ranks, then the summed prefix shares
            std::vector<uint32_t> key;
            std::vector<int64_t> vals(std::max(n, 1));
            int32_t kw = 0, has = 0;
            for (int r = 0; r < N; ++r) {
                std::vector<uint32_t> k(parts[r]->KW);
                std::vector<int64_t> v(std::max(n, 1));
                kw = parts[r]->KW;
                CUBICS_CHECK_OK(cubics_first_shard_best(parts[r].get(), k.data(), &kw, v.data(), &has));
                if (has && (key.empty() || std::lexicographical_compare(k.begin(), k.end(), key.begin(), key.end()))) {
                    key = k;
                    vals = v;
                }
            }
            cubics_stats tot{};
            for (int r = 0; r < N; ++r) {
                cubics_stats st{};
                CUBICS_CHECK_OK(cubics_first_shard_prefix(parts[r].get(), key.empty() ? nullptr : key.data(),
                                                          (int32_t)key.size(), &st));
                tot.nodes += st.nodes;
                tot.failures += st.failures;
                tot.rounds += st.rounds;
                tot.solutions += st.solutions;
            }
            out->stats = tot;
            out->has_solution = !key.empty();
            out->complete = key.empty() ? 1 : 0; // stopped at max_solutions, as the reference reports
            if (!key.empty()) {
                if (best_values) std::copy_n(vals.begin(), n, best_values);
                if (cb && !cfg->count_only) cb(user, vals.data(), n);
            }
        } else {
            out->has_solution = out->stats.solutions > 0;
            if (collect) { // the ranks' key-ordered streams merged into the reference's DFS order
                std::vector<Row*> all;
                for (auto& v : rows)
                    for (auto& row : v) all.push_back(&row);
                std::sort(all.begin(), all.end(), [](const Row* a, const Row* b) { return a->first < b->first; });
                for (const Row* row : all)
                    if (!cb(user, row->second.data(), n)) break;
            }
        }
        out->total_ms = now_ms() - t0;
        return (int)CUBICS_OK;
    });
}

extern "C" int cubics_solve_shard(const cubics_model* h, const cubics_search_config* cfg, int32_t shard_index,
                                  int32_t shard_count, cubics_keyed_solution_cb cb, void* user, cubics_result* out) {
    return solve_shard_impl(h, cfg, shard_index, shard_count, nullptr, cb, user, out, false, nullptr);
}

extern "C" int cubics_solve_shard_shared(const cubics_model* h, const cubics_search_config* cfg, int32_t shard_index,
                                         int32_t shard_count, cubics_task_queue* queue, cubics_keyed_solution_cb cb,
                                         void* user, cubics_result* out) {
    if (!queue) return CUBICS_E_INVALID;
    return solve_shard_impl(h, cfg, shard_index, shard_count, queue, cb, user, out, false, nullptr);
}

extern "C" int cubics_solve_optimize_shard(const cubics_model* h, const cubics_search_config* cfg, int32_t shard_index,
                                           int32_t shard_count, cubics_task_queue* queue, int64_t* best_values,
                                           cubics_result* out) {
    return solve_shard_impl(h, cfg, shard_index, shard_count, queue, nullptr, nullptr, out, true, best_values);
}

// Shared task queue: one u32 claim counter in the owner GPU's HBM, mapped into the other ranks'
// address spaces with CUDA IPC (peer access over NVLink enabled lazily by the driver).
extern "C" int cubics_task_queue_create(int32_t device, cubics_task_queue** out, uint8_t* handle) {
    if (!out) return CUBICS_E_INVALID;
    *out = nullptr;
    return guarded([&]() -> int {
        const int dev = current_device(device);
        CU(cudaSetDevice(dev));
        void* p = nullptr;
        CU(cudaMalloc(&p, kQueueBytes));
        CU(cudaMemset(p, 0, kQueueBytes));
        QueueState init{};
        init.g_inc = ~0ull; // no incumbent
        init.g_first = ~0ull;
        CU(cudaMemcpy(p, &init, sizeof init, cudaMemcpyHostToDevice));
        if (handle) {
            cudaIpcMemHandle_t hd;
            cudaError_t e = cudaIpcGetMemHandle(&hd, p);
            if (e != cudaSuccess) {
                cudaFree(p);
                CU(e);
            }
            static_assert(sizeof hd == CUBICS_TASK_QUEUE_HANDLE_BYTES, "IPC handle size");
            std::memcpy(handle, &hd, sizeof hd);
        }
        *out = new cubics_task_queue{p, dev, 1};
        return CUBICS_OK;
    });
}

extern "C" int cubics_task_queue_open(int32_t device, const uint8_t* handle, cubics_task_queue** out) {
    if (!out || !handle) return CUBICS_E_INVALID;
    *out = nullptr;
    return guarded([&]() -> int {
        const int dev = current_device(device);
        CU(cudaSetDevice(dev));
        cudaIpcMemHandle_t hd;
        std::memcpy(&hd, handle, sizeof hd);
        void* p = nullptr;
        CU(cudaIpcOpenMemHandle(&p, hd, cudaIpcMemLazyEnablePeerAccess));
        *out = new cubics_task_queue{p, dev, 0};
        return CUBICS_OK;
    });
}

extern "C" int cubics_task_queue_reset(cubics_task_queue* q) {
    if (!q) return CUBICS_E_INVALID;
    return guarded([&]() -> int {
        CU(cudaSetDevice(q->device));
        QueueState init{};
        init.g_inc = ~0ull; // no incumbent
        init.g_first = ~0ull;
        CU(cudaMemset(q->counter, 0, kQueueBytes));
        CU(cudaMemcpy(q->counter, &init, sizeof init, cudaMemcpyHostToDevice));
        CU(cudaDeviceSynchronize());
        return CUBICS_OK;
    });
}

extern "C" int cubics_task_queue_claims(cubics_task_queue* q, uint64_t* claims) {
    if (!q || !claims) return CUBICS_E_INVALID;
    return guarded([&]() -> int {
        CU(cudaSetDevice(q->device));
        uint32_t v = 0;
        CU(cudaMemcpy(&v, q->counter, sizeof v, cudaMemcpyDeviceToHost));
        *claims = v;
        return CUBICS_OK;
    });
}

extern "C" int cubics_task_queue_destroy(cubics_task_queue* q) {
    if (!q) return CUBICS_OK;
    return guarded([&]() -> int {
        cudaSetDevice(q->device);
        if (q->owner)
            cudaFree(q->counter);
        else
            cudaIpcCloseMemHandle(q->counter);
        delete q;
        return CUBICS_OK;
    });
}

namespace {
int run_prop(const cubics_model* h, const uint64_t* words_in, uint64_t* words_out, int32_t alldiff, int32_t max_rounds,
             const int32_t* cons, int32_t n_cons, bool removals_only, cubics_fixpoint_result* fr) {
    const HostModel& m = h->m;
    const int dev = current_device(-1);
    std::lock_guard<std::recursive_mutex> lock(g_dev_mu[dev]);
    Prepared P;
    // the removal subset decides which constraints are evaluated (INT64_MIN pre-check included)
    HostModel sub;
    const HostModel* use = &m;
    std::vector<uint8_t> enabled;
    if (removals_only && cons) {
        std::vector<char> on(m.n_cons(), 0);
        for (int i = 0; i < n_cons; ++i) {
            if (cons[i] < 0 || cons[i] >= m.n_cons()) throw StatusError{CUBICS_E_INVALID, "constraint index out of range"};
            on[cons[i]] = 1;
        }
        sub = m;
        sub.con_kind.clear();
        sub.con_op.clear();
        sub.con_value.clear();
        sub.con_start.assign(1, 0);
        sub.term_var.clear();
        sub.term_coeff.clear();
        sub.table_start.clear();
        sub.table_data.clear();
        for (int c = 0; c < m.n_cons(); ++c) {
            if (!on[c]) continue;
            sub.con_kind.push_back(m.con_kind[c]);
            sub.con_op.push_back(m.con_op[c]);
            sub.con_value.push_back(m.con_value[c]);
            sub.table_start.push_back(static_cast<int64_t>(sub.table_data.size()));
            if (m.con_kind[c] == CUBICS_TABLE) {
                const int64_t* src = m.table_data.data() + m.table_start[c];
                sub.table_data.insert(sub.table_data.end(), src,
                                      src + m.con_value[c] * (m.con_start[c + 1] - m.con_start[c]));
            }
            for (int t = m.con_start[c]; t < m.con_start[c + 1]; ++t) {
                sub.term_var.push_back(m.term_var[t]);
                sub.term_coeff.push_back(m.term_coeff[t]);
            }
            sub.con_start.push_back(static_cast<int32_t>(sub.term_var.size()));
        }
        use = &sub;
    }
    const double tp0 = now_ms();
    prepare(*use, words_in, P);
    const double tp1 = now_ms();
    const size_t NWP = P.NWP;
    // many alldifferents (more than one block's warps) or a large model: a grid-wide fixpoint
    const bool grid = P.na > 8 || (long)P.nr + P.nl + 4L * (P.ntb + P.ntn) >= 40000 || P.n >= 50000;
    const int block = grid ? 512 : parity_block(P);
    bool in_smem = !grid;
    dev::SmemLayout L = dev::smem_layout(P.W, P.n, P.total_members, block / 32, 0, in_smem, P.na);
    if (L.total > kSmemBudget) {
        in_smem = false;
        L = dev::smem_layout(P.W, P.n, P.total_members, block / 32, 0, false, P.na);
        if (grid && L.total > kSmemBudget) throw StatusError{CUBICS_E_UNSUPPORTED, "propagation context does not fit in shared memory"};
    }
    int grid_blocks = 1;
    if (grid) {
        int per_sm = 0, sms = 0;
#define OPG(w) occupancy_propagate_grid<w>(block, L.total, &per_sm)
        CUBICS_DISPATCH_W(P.W, OPG)
#undef OPG
        CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        if (per_sm < 1) throw StatusError{CUBICS_E_UNSUPPORTED, "grid propagation does not fit on an SM"};
        grid_blocks = std::min(per_sm, 2) * sms;
    }
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t at = (off + 255) & ~size_t(255);
        off = at + std::max<size_t>(bytes, 16);
        return at;
    };
    const size_t a_blob = take(P.blob.bytes.size());
    const size_t a_dom = take(sizeof(uint32_t) * NWP);
    const size_t a_out = take(sizeof(uint32_t) * NWP);
    const size_t a_res = take(sizeof(int32_t) * 8);
    const size_t a_scr = take(in_smem ? 0 : sizeof(uint32_t) * 2 * NWP);
    const size_t a_big = take(sizeof(uint32_t) * P.big_words * (size_t)(block / 32) * grid_blocks);
    const size_t a_gctl = take(grid ? 256 : 0);
    const size_t a_gslots = take(grid ? 6 * sizeof(unsigned) : 0);
    const size_t a_gchg = take(grid ? sizeof(uint32_t) * 2 * (((size_t)P.n + 31) / 32) : 0);
    uint8_t* base = device_arena(dev, off);
    const size_t stage_bytes = a_dom + sizeof(uint32_t) * NWP;
    uint8_t* stage = pinned_arena(dev, stage_bytes);
    std::memcpy(stage + a_blob, P.blob.bytes.data(), P.blob.bytes.size());
    std::memcpy(stage + a_dom, P.blob.bytes.data() + P.o_dom, sizeof(uint32_t) * NWP);
    cudaStream_t st = g_dev[dev].stream;
    CU(cudaMemcpyAsync(base, stage, stage_bytes, cudaMemcpyHostToDevice, st));
    PropParams PP{};
    PP.M = P.bind(base + a_blob);
    PP.alldiff = alldiff == CUBICS_FORWARD_CHECKING ? 0 : 1;
    PP.max_rounds = max_rounds;
    PP.removals_only = removals_only ? 1 : 0;
    PP.enabled = nullptr;
    PP.dom = reinterpret_cast<uint32_t*>(base + a_dom);
    PP.out = reinterpret_cast<uint32_t*>(base + a_out);
    PP.result = reinterpret_cast<int32_t*>(base + a_res);
    PP.big_scratch = P.big_words ? reinterpret_cast<uint32_t*>(base + a_big) : nullptr;
    uint32_t* scr = reinterpret_cast<uint32_t*>(base + a_scr);
    if (grid) {
        const unsigned init[6] = {0, 0, 0, 0xffffffffu, 0xffffffffu, 0xffffffffu};
        CU(cudaMemcpyAsync(base + a_gslots, init, sizeof init, cudaMemcpyHostToDevice, st));
        CU(cudaMemsetAsync(base + a_gctl, 0, 256, st));
        PP.grid_ctl = reinterpret_cast<dev_ctl_t*>(base + a_gctl);
        PP.grid_or = reinterpret_cast<unsigned*>(base + a_gslots);
        PP.grid_min = PP.grid_or + 3;
        PP.grid_chg = reinterpret_cast<uint32_t*>(base + a_gchg);
    }
    CU(cudaEventRecord(g_dev[dev].e0, st));
    if (grid) {
#define LPG(w) launch_propagate_grid<w>(PP, grid_blocks, block, L.total, st, scr)
        CUBICS_DISPATCH_W(P.W, LPG)
#undef LPG
    } else {
#define LP(w) launch_propagate<w>(PP, block, L.total, st, scr, in_smem ? 1 : 0)
        CUBICS_DISPATCH_W(P.W, LP)
#undef LP
    }
    CU(cudaEventRecord(g_dev[dev].e1, st));
    std::vector<uint32_t> res32(NWP);
    int32_t res[8] = {0};
    CU(cudaMemcpyAsync(res32.data(), removals_only ? (void*)PP.out : (void*)PP.dom, sizeof(uint32_t) * NWP,
                       cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(res, PP.result, sizeof res, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    if (std::getenv("CUBICS_DEBUG")) {
        float kms = 0;
        CU(cudaEventElapsedTime(&kms, g_dev[dev].e0, g_dev[dev].e1));
        std::fprintf(stderr, "[cubics] propagate: %s blocks=%d block=%d prepare %.3f ms, kernel %.3f ms, rounds %d, total %.3f ms\n",
                     grid ? "grid" : "block", grid_blocks, block, tp1 - tp0, kms, res[2], now_ms() - tp0);
    }
    if (res[4] == DERR_OVERFLOW) throw StatusError{CUBICS_E_OVERFLOW, "overflow in linear propagation"};
    // back to the u64 reference layout
    for (int v = 0; v < m.n_vars(); ++v) {
        const int nw64 = m.word_start[v + 1] - m.word_start[v];
        for (int i = 0; i < nw64; ++i) {
            uint64_t lo = 2 * i < P.W ? res32[(size_t)v * P.W + 2 * i] : 0;
            uint64_t hi = 2 * i + 1 < P.W ? res32[(size_t)v * P.W + 2 * i + 1] : 0;
            words_out[m.word_start[v] + i] = lo | (hi << 32);
        }
    }
    if (fr) {
        fr->failed = res[0];
        fr->failed_var = res[1];
        fr->rounds = res[2];
        fr->last_status = res[3];
    }
    return CUBICS_OK;
}
} // namespace

extern "C" int cubics_propagate(const cubics_model* h, uint64_t* words, int32_t alldiff, int32_t max_rounds,
                                cubics_fixpoint_result* out) {
    if (!h || !words || !out) return CUBICS_E_INVALID;
    return guarded([&] { return run_prop(h, words, words, alldiff, max_rounds, nullptr, 0, false, out); });
}

extern "C" int cubics_removals(const cubics_model* h, const uint64_t* words, int32_t alldiff, const int32_t* cons,
                               int32_t n_cons, uint64_t* removed) {
    if (!h || !words || !removed) return CUBICS_E_INVALID;
    return guarded([&] { return run_prop(h, words, removed, alldiff, 1, cons, n_cons, true, nullptr); });
}

#define CUBICS_STR2(x) #x
#define CUBICS_STR(x) CUBICS_STR2(x)
extern "C" const char* cubics_build_info(void) {
    return "cubics-b200 abi=1 arch=sm_100a engine=persistent-dfs(parity|parallel) nvcc=" CUBICS_STR(__CUDACC_VER_MAJOR__) "." CUBICS_STR(__CUDACC_VER_MINOR__);
}

extern "C" int cubics_warmup(int32_t device) {
    return guarded([&] {
        current_device(device);
        CU(cudaFree(nullptr));
        // one tiny search and one tiny fixpoint per common word count load the kernels
        HostModel m;
        m.names = {"a", "b"};
        m.offset = {1, 1};
        m.width = {2, 2};
        m.finish_vars();
        m.words.assign(m.word_start.back(), 3);
        m.con_kind = {CUBICS_ALLDIFF};
        m.con_op = {0};
        m.con_value = {0};
        m.con_start = {0, 2};
        m.term_var = {0, 1};
        m.term_coeff = {1, 1};
        cubics_search_config c;
        cubics_search_config_init(&c);
        c.device = device;
        c.count_only = 1;
        for (int engine : {CUBICS_ENGINE_PARITY, CUBICS_ENGINE_PARALLEL}) {
            c.engine = engine;
            RunOut r;
            run_search(m, c, engine, false, 0, r);
        }
        cubics_model h{m};
        std::vector<uint64_t> w(m.words);
        cubics_fixpoint_result fr{};
        return cubics_propagate(&h, w.data(), CUBICS_ARC_CONSISTENT, 0, &fr);
    });
}

extern "C" int cubics_device_count(void) {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) return 0;
    return c;
}
