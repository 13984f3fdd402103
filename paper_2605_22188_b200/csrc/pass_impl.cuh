// pass_impl.cuh -- definitions behind pass_impl.hpp (included by pass_e<E>.cu).
#pragma once
#include "pass_impl.hpp"
#include "pass_kernel.cuh"

namespace bnbg {

template <int E>
cudaError_t pass_static_smem_t(size_t* bytes) {
  cudaFuncAttributes fa;
  const cudaError_t e = cudaFuncGetAttributes(&fa, k_pass<E>);
  *bytes = e == cudaSuccess ? fa.sharedSizeBytes : 0;
  return e;
}

template <int E>
cudaError_t pass_setup_t(size_t smem, int* blocks_per_sm) {
  cudaError_t e = cudaFuncSetAttribute(k_pass<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_pass<E>, kPassThreads, smem);
  return e;
}

template <int E>
cudaError_t pass_launch_t(int grid, size_t smem, cudaStream_t st, PassArgs* a, int cluster) {
  if (cluster > 0) {  // the grid is one cluster: co-resident by construction
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kPassThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_pass<E>, *a);
  }
  void* args[] = {a};
  return cudaLaunchCooperativeKernel((const void*)k_pass<E>, dim3(grid), dim3(kPassThreads), args,
                                     smem, st);
}

template <int E>
bool pass_cluster_ok_t(size_t smem, int cs) {
  if (cudaFuncSetAttribute(k_pass<E>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess ||
      cudaFuncSetAttribute(k_pass<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    (void)cudaGetLastError();
    return false;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs);
  cfg.blockDim = dim3(kPassThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int nc = 0;
  if (cudaOccupancyMaxActiveClusters(&nc, k_pass<E>, &cfg) != cudaSuccess) {
    (void)cudaGetLastError();
    return false;
  }
  return nc >= 1;
}

}  // namespace bnbg

#define BNBG_INSTANTIATE_PASS(E)                                                            \
  namespace bnbg {                                                                          \
  template cudaError_t pass_static_smem_t<E>(size_t*);                                      \
  template cudaError_t pass_setup_t<E>(size_t, int*);                                       \
  template cudaError_t pass_launch_t<E>(int, size_t, cudaStream_t, PassArgs*, int);         \
  template bool pass_cluster_ok_t<E>(size_t, int);                                          \
  }
