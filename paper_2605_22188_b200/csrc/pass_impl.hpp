// pass_impl.hpp -- per-width entry points of the persistent pass kernel; the
// definitions (pass_impl.cuh) are instantiated once per width in pass_e<E>.cu.
#pragma once
#include <cuda_runtime.h>

#include "launchers.hpp"

namespace bnbg {

template <int E>
cudaError_t pass_static_smem_t(size_t* bytes);
template <int E>
cudaError_t pass_setup_t(size_t smem, int* blocks_per_sm);
template <int E>
cudaError_t pass_launch_t(int grid, size_t smem, cudaStream_t st, PassArgs* a, int cluster);
template <int E>
bool pass_cluster_ok_t(size_t smem, int cs);

}  // namespace bnbg
