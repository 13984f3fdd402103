// pass_kernels.cu -- instantiations and cooperative launcher of k_pass.
#include "launchers.hpp"
#include "pass_kernel.cuh"

namespace bnbg {

#define DISPATCH_E(E_, ...)  \
  switch (E_) {              \
    case 1: {                \
      constexpr int EV = 1;  \
      __VA_ARGS__;           \
    } break;                 \
    case 2: {                \
      constexpr int EV = 2;  \
      __VA_ARGS__;           \
    } break;                 \
    case 4: {                \
      constexpr int EV = 4;  \
      __VA_ARGS__;           \
    } break;                 \
    default: {               \
      constexpr int EV = 0;  \
      __VA_ARGS__;           \
    } break;                 \
  }

size_t pass_smem(int p, int n2, int E) { return pass_smem_bytes(p, n2, E); }

cudaError_t pass_setup(int E, size_t smem, int* blocks_per_sm) {
  cudaError_t e = cudaSuccess;
  *blocks_per_sm = 0;
  DISPATCH_E(E, {
    e = cudaFuncSetAttribute(k_pass<EV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_pass<EV>, kPassThreads,
                                                        smem);
  });
  return e;
}

cudaError_t pass_launch(int E, int grid, size_t smem, cudaStream_t st, PassArgs* a) {
  void* args[] = {a};
  cudaError_t e = cudaSuccess;
  DISPATCH_E(E, e = cudaLaunchCooperativeKernel((const void*)k_pass<EV>, dim3(grid),
                                                dim3(kPassThreads), args, smem, st));
  return e;
}

}  // namespace bnbg
