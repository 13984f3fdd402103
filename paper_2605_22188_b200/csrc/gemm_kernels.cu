// gemm_kernels.cu -- instantiations and launcher of the DMMA GEMM kernels.
#include "gemm_big.cuh"
#include "launchers.hpp"

namespace bnbg {

template <bool TN, int FM, int FN, int EPI>
static cudaError_t set_attr() {
  return cudaFuncSetAttribute(k_gemm<TN, FM, FN, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)GemmShape<TN, FM, FN>::SMEM_BYTES);
}

#define FOR_GEMM_CFGS(X) \
  X(2, 1) X(2, 2) X(2, 4) X(4, 1) X(4, 2) X(4, 4) X(8, 1) X(8, 2) X(8, 4)

cudaError_t gemm_set_attrs() {
  cudaError_t e = cudaSuccess;
#define SETA(FM, FN)                                            \
  if (e == cudaSuccess) e = set_attr<false, FM, FN, EPI_DERIV>(); \
  if (e == cudaSuccess) e = set_attr<false, FM, FN, EPI_EVAL>();  \
  if (e == cudaSuccess) e = set_attr<false, FM, FN, EPI_STORE>(); \
  if (e == cudaSuccess) e = set_attr<true, FM, FN, EPI_STORE>();
  FOR_GEMM_CFGS(SETA)
#undef SETA
  const int big = (int)kBigSmemBytes;
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_gemm_big<false, EPI_DERIV>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_gemm_big<false, EPI_EVAL>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_gemm_big<false, EPI_STORE>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_gemm_big<true, EPI_STORE>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  return e;
}

int gemm_big_tile_m() { return kBigBM; }
int gemm_big_tile_n() { return kBigBN; }
int gemm_big_tile_k() { return kBigBK; }
void gemm_big_boxes(int* nn, int* tn) {
  nn[0] = kBigBoxNN0;
  nn[1] = kBigBoxNN1;
  tn[0] = kBigBoxTN0;
  tn[1] = kBigBoxTN1;
}

cudaError_t gemm_big_launch(bool tn, int epi, dim3 grid, cudaStream_t st, const GemmArgs& g) {
  const dim3 block(kBigThreads);
  if (tn)
    k_gemm_big<true, EPI_STORE><<<grid, block, kBigSmemBytes, st>>>(g);
  else if (epi == EPI_DERIV)
    k_gemm_big<false, EPI_DERIV><<<grid, block, kBigSmemBytes, st>>>(g);
  else if (epi == EPI_EVAL)
    k_gemm_big<false, EPI_EVAL><<<grid, block, kBigSmemBytes, st>>>(g);
  else
    k_gemm_big<false, EPI_STORE><<<grid, block, kBigSmemBytes, st>>>(g);
  return cudaGetLastError();
}

cudaError_t gemm_launch(bool tn, int epi, int fm, int fn, dim3 grid, cudaStream_t st,
                        const GemmArgs& g) {
  const dim3 block(kGemmThreads);
#define LAUNCH_ONE(FM, FN)                                                                      \
  if (fm == FM && fn == FN) {                                                                   \
    if (tn)                                                                                     \
      k_gemm<true, FM, FN, EPI_STORE><<<grid, block, GemmShape<true, FM, FN>::SMEM_BYTES, st>>>(g); \
    else if (epi == EPI_DERIV)                                                                  \
      k_gemm<false, FM, FN, EPI_DERIV>                                                          \
          <<<grid, block, GemmShape<false, FM, FN>::SMEM_BYTES, st>>>(g);                       \
    else if (epi == EPI_EVAL)                                                                   \
      k_gemm<false, FM, FN, EPI_EVAL><<<grid, block, GemmShape<false, FM, FN>::SMEM_BYTES, st>>>(g); \
    else                                                                                        \
      k_gemm<false, FM, FN, EPI_STORE>                                                          \
          <<<grid, block, GemmShape<false, FM, FN>::SMEM_BYTES, st>>>(g);                       \
  }
  FOR_GEMM_CFGS(LAUNCH_ONE)
#undef LAUNCH_ONE
  return cudaGetLastError();
}

}  // namespace bnbg
