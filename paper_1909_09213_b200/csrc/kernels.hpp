// Launch interface of the device kernels. Each domain word count W in {1,2,4,8,16,32} is
// instantiated in its own translation unit (kernels_inst.cu compiled with -DCUBICS_W=W).
#pragma once

#include <cuda_runtime.h>

#include "device_model.hpp"

namespace cubics {

// feat: the model's propagator features (dev::Feature bits); a lean instantiation is chosen
template <int W>
cudaError_t launch_search(const SearchParams& P, int feat, int grid, int block, size_t smem, cudaStream_t st);
template <int W>
cudaError_t occupancy_search(int feat, int block, size_t smem, int* blocks_per_sm);
// warp contexts for small models (n <= 32, W = 1): blockDim.x / 32 contexts per block
cudaError_t launch_search_warp(const SearchParams& P, int feat, int grid, int block, size_t smem, cudaStream_t st);
cudaError_t occupancy_search_warp(int feat, bool parity, int block, size_t smem, int* blocks_per_sm);
template <int W>
cudaError_t launch_search_parity(const SearchParams& P, int grid, int block, size_t smem, cudaStream_t st);
template <int W>
cudaError_t launch_search_grid(const SearchParams& P, int grid, int block, size_t smem, cudaStream_t st);
template <int W>
cudaError_t occupancy_search_grid(int block, size_t smem, int* blocks_per_sm);
template <int W>
cudaError_t launch_propagate_grid(const PropParams& P, int grid, int block, size_t smem, cudaStream_t st,
                                  uint32_t* scratch);
template <int W>
cudaError_t occupancy_propagate_grid(int block, size_t smem, int* blocks_per_sm);
template <int W>
cudaError_t launch_propagate(const PropParams& P, int block, size_t smem, cudaStream_t st, uint32_t* scratch,
                             int in_smem);

} // namespace cubics
