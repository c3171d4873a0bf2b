// One instantiation of the search / propagation kernels for domain word count CUBICS_W.
#include "kernels.hpp"
#include "search.cuh"

#ifndef CUBICS_W
#error "compile with -DCUBICS_W=<1|2|4|8|16|32>"
#endif
// CUBICS_PART splits one W into translation units by kernel family (the W=32 kernels take
// minutes each in ptxas): 0 generic search, 1 parity search, 2 grid search, 3 propagation.
#ifndef CUBICS_PART
#define CUBICS_PART -1 // everything
#endif
#define CUBICS_HAS_PART(p) (CUBICS_PART < 0 || CUBICS_PART == (p))

namespace cubics {

// internal linkage by `static`, not an anonymous namespace: nvcc names anonymous namespaces after
// the source file, and every (W, part) object is built from this same file
// cudaFuncSetAttribute only when a launch needs more dynamic shared memory than already granted
template <class K>
static cudaError_t grant_smem(K k, size_t smem, size_t& granted) {
    if (smem <= granted) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) granted = smem;
    return e;
}
static size_t g_search_smem = 48 * 1024, g_prop_smem = 48 * 1024, g_grid_smem = 48 * 1024;
static size_t g_search_smem0 = 48 * 1024, g_search_smem1 = 48 * 1024, g_parity_smem = 48 * 1024;
static size_t g_propgrid_smem = 48 * 1024;

#if CUBICS_HAS_PART(0)
// lean instantiations for narrow domains: {RelBin + small alldiff}, {+ linear}; everything else
// (tables, large alldifferents, the first-solution bookkeeping, wide domains) runs the full kernel
using SearchFn = void (*)(const SearchParams);

static SearchFn pick_search(int feat) {
    feat &= ~(dev::F_NOOPT | dev::F_NOSPLIT | dev::F_FRONTIER); // lean bits select warp kernels only
    if constexpr (CUBICS_W <= 4) {
        if (feat == 0) return dev::search_kernel<CUBICS_W, 0>;
        if (feat == dev::F_LINEAR) return dev::search_kernel<CUBICS_W, dev::F_LINEAR>;
    }
    return dev::search_kernel<CUBICS_W, dev::F_ALL>;
}

#if CUBICS_W == 1
// warp contexts (warp_ctx.cuh): parallel and parity engines on small models
// feat bit F_NOOPT | F_NOSPLIT (lean: satisfy goal, unsharded) selects the lean instantiations
static SearchFn pick_warp(int feat, bool parity) {
    using namespace dev;
    const bool lin = feat & F_LINEAR, first = feat & F_FIRST, lean = (feat & (F_NOOPT | F_NOSPLIT)) == (F_NOOPT | F_NOSPLIT);
    constexpr int L = F_NOOPT | F_NOSPLIT;
    if (parity) return lin ? search_kernel_warp<F_PARITY | F_LINEAR> : search_kernel_warp<F_PARITY>;
    if (first) return lin ? search_kernel_warp<F_LINEAR | F_FIRST | L> : search_kernel_warp<F_FIRST | L>;
    if (lean) return lin ? search_kernel_warp<F_LINEAR | L> : search_kernel_warp<L>;
    // the frontier expansion of a sharded search (always a satisfy goal: B&B expands without it)
    if (feat & F_FRONTIER)
        return lin ? search_kernel_warp<F_LINEAR | F_NOOPT | F_FRONTIER> : search_kernel_warp<F_NOOPT | F_FRONTIER>;
    // seeded sharded satisfy searches: shared-queue claims, cross-GPU stealing; no B&B
    if (feat & F_NOOPT) return lin ? search_kernel_warp<F_LINEAR | F_NOOPT> : search_kernel_warp<F_NOOPT>;
    return lin ? search_kernel_warp<F_LINEAR> : search_kernel_warp<0>;
}
static size_t g_warp_smem[12] = {48 * 1024, 48 * 1024, 48 * 1024, 48 * 1024, 48 * 1024, 48 * 1024,
                                  48 * 1024, 48 * 1024, 48 * 1024, 48 * 1024, 48 * 1024, 48 * 1024};
static int warp_slot(int feat, bool parity) {
    const bool lean = (feat & (dev::F_NOOPT | dev::F_NOSPLIT)) == (dev::F_NOOPT | dev::F_NOSPLIT);
    if (parity) return 6 | ((feat & dev::F_LINEAR) ? 1 : 0);
    if (!lean && !(feat & dev::F_FIRST) && (feat & dev::F_FRONTIER)) return 10 | ((feat & dev::F_LINEAR) ? 1 : 0);
    if (!lean && !(feat & dev::F_FIRST) && (feat & dev::F_NOOPT)) return 8 | ((feat & dev::F_LINEAR) ? 1 : 0);
    return ((feat & dev::F_LINEAR) ? 1 : 0) | ((feat & dev::F_FIRST) ? 2 : (lean ? 4 : 0));
}

cudaError_t launch_search_warp(const SearchParams& P, int feat, int grid, int block, size_t smem, cudaStream_t st) {
    const bool parity = P.mode == MODE_PARITY;
    SearchFn k = pick_warp(feat, parity);
    cudaError_t e = grant_smem(k, smem, g_warp_smem[warp_slot(feat, parity)]);
    if (e != cudaSuccess) return e;
    k<<<grid, block, smem, st>>>(P);
    return cudaGetLastError();
}

cudaError_t occupancy_search_warp(int feat, bool parity, int block, size_t smem, int* out) {
    SearchFn k = pick_warp(feat, parity);
    cudaError_t e = grant_smem(k, smem, g_warp_smem[warp_slot(feat, parity)]);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, k, block, smem);
}
#endif

template <>
cudaError_t launch_search<CUBICS_W>(const SearchParams& P, int feat, int grid, int block, size_t smem,
                                    cudaStream_t st) {
    // the generic block kernel also runs one-warp contexts: a __syncwarp-specialised variant
    // measured slower on B200 (19.3 vs 14.0 ms on nq14; register spills at the 64-register cap)
    if (P.mode == MODE_PARITY && block <= 512) return launch_search_parity<CUBICS_W>(P, grid, block, smem, st);
    if (P.batch) return cudaErrorInvalidConfiguration; // batched B&B runs in the parity kernel only
    SearchFn k = pick_search(feat);
    feat &= ~(dev::F_NOOPT | dev::F_NOSPLIT | dev::F_FRONTIER);
    cudaError_t e = grant_smem(k, smem, feat == 0 ? g_search_smem0 : (feat == dev::F_LINEAR ? g_search_smem1 : g_search_smem));
    if (e != cudaSuccess) return e;
    k<<<grid, block, smem, st>>>(P);
    return cudaGetLastError();
}

template <>
cudaError_t occupancy_search<CUBICS_W>(int feat, int block, size_t smem, int* out) {
    SearchFn k = pick_search(feat);
    feat &= ~(dev::F_NOOPT | dev::F_NOSPLIT | dev::F_FRONTIER);
    cudaError_t e = grant_smem(k, smem, feat == 0 ? g_search_smem0 : (feat == dev::F_LINEAR ? g_search_smem1 : g_search_smem));
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, k, block, smem);
}
#endif

#if CUBICS_HAS_PART(1)
template <>
cudaError_t launch_search_parity<CUBICS_W>(const SearchParams& P, int grid, int block, size_t smem, cudaStream_t st) {
    auto k = dev::search_kernel_parity<CUBICS_W>;
    cudaError_t e = grant_smem(k, smem, g_parity_smem);
    if (e != cudaSuccess) return e;
    k<<<grid, block, smem, st>>>(P);
    return cudaGetLastError();
}
#endif

#if CUBICS_HAS_PART(2)
template <>
cudaError_t launch_search_grid<CUBICS_W>(const SearchParams& P, int grid, int block, size_t smem, cudaStream_t st) {
    auto k = dev::search_kernel_grid<CUBICS_W>;
    cudaError_t e = grant_smem(k, smem, g_grid_smem);
    if (e != cudaSuccess) return e;
    SearchParams p = P;
    void* args[] = {&p};
    return cudaLaunchCooperativeKernel((const void*)k, dim3(grid), dim3(block), args, smem, st);
}

template <>
cudaError_t occupancy_search_grid<CUBICS_W>(int block, size_t smem, int* out) {
    auto k = dev::search_kernel_grid<CUBICS_W>;
    cudaError_t e = grant_smem(k, smem, g_grid_smem);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, k, block, smem);
}

#endif

#if CUBICS_HAS_PART(3)
template <>
cudaError_t launch_propagate<CUBICS_W>(const PropParams& P, int block, size_t smem, cudaStream_t st,
                                       uint32_t* scratch, int in_smem) {
    auto k = dev::propagate_kernel<CUBICS_W>;
    cudaError_t e = grant_smem(k, smem, g_prop_smem);
    if (e != cudaSuccess) return e;
    k<<<1, block, smem, st>>>(P, scratch, in_smem);
    return cudaGetLastError();
}

template <>
cudaError_t launch_propagate_grid<CUBICS_W>(const PropParams& P, int grid, int block, size_t smem, cudaStream_t st,
                                            uint32_t* scratch) {
    auto k = dev::propagate_kernel_grid<CUBICS_W>;
    cudaError_t e = grant_smem(k, smem, g_propgrid_smem);
    if (e != cudaSuccess) return e;
    PropParams p = P;
    void* args[] = {&p, &scratch};
    return cudaLaunchCooperativeKernel((const void*)k, dim3(grid), dim3(block), args, smem, st);
}

template <>
cudaError_t occupancy_propagate_grid<CUBICS_W>(int block, size_t smem, int* out) {
    auto k = dev::propagate_kernel_grid<CUBICS_W>;
    cudaError_t e = grant_smem(k, smem, g_propgrid_smem);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, k, block, smem);
}

#endif

} // namespace cubics
