// column_kernels.cu -- instantiations and launchers of the per-column kernels.
#include "launchers.hpp"

namespace bnbg {

// E = 8 (p <= 2048) was measured slower than the shared-memory network: the
// 2048-key network does not unroll and its arrays land in local memory
int column_E(int n2) { return n2 <= 256 ? 1 : n2 <= 512 ? 2 : n2 <= 1024 ? 4 : 0; }

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

template <int E>
static cudaError_t set_attrs(size_t smem) {
  const int s = (int)smem;
  cudaError_t e = cudaFuncSetAttribute(k_prox_fista<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, s);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_eval<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, s);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_round_select<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, s);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_prox_standalone<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, s);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_g_standalone<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, s);
  return e;
}

cudaError_t column_set_attrs(int E, size_t smem) {
  cudaError_t e = cudaSuccess;
  DISPATCH_E(E, e = set_attrs<EV>(smem));
  return e;
}

cudaError_t launch_prox_fista(int E, int m, size_t smem, cudaStream_t st, const RelaxDev& r) {
  DISPATCH_E(E, k_prox_fista<EV><<<m, kNodeThreads, smem, st>>>(r));
  return cudaGetLastError();
}

cudaError_t launch_eval(int E, int m, size_t smem, cudaStream_t st, const RelaxDev& r,
                        const EvalArgs& e) {
  DISPATCH_E(E, k_eval<EV><<<m, kNodeThreads, smem, st>>>(r, e));
  return cudaGetLastError();
}

cudaError_t launch_round_select(int E, int m, size_t smem, cudaStream_t st, int p, int n2, int k,
                                const double* beta, const uint8_t* state, const int* kbar,
                                const int* one_off, const int* one_idx, const int* one_len, int* sup,
                                int* len, int* jb, double* gscr, long long gstride) {
  DISPATCH_E(E, k_round_select<EV><<<m, kNodeThreads, smem, st>>>(p, n2, k, beta, state, kbar,
                                                                  one_off, one_idx, one_len, sup,
                                                                  len, jb, gscr, gstride));
  return cudaGetLastError();
}

cudaError_t launch_prox_standalone(int E, int m, size_t smem, cudaStream_t st, int mode, int p,
                                   int n2, const double* U, const uint8_t* state, const int* kbar,
                                   double w, double M, double* out, double* gscr,
                                   long long gstride) {
  DISPATCH_E(E, k_prox_standalone<EV><<<m, kNodeThreads, smem, st>>>(mode, p, n2, U, state, kbar,
                                                                     w, M, out, gscr, gstride));
  return cudaGetLastError();
}

cudaError_t launch_g_standalone(int E, int m, size_t smem, cudaStream_t st, int mode, int p, int n2,
                                const double* in, const uint8_t* state, const int* kbar, double M,
                                double* out, double* gscr, long long gstride) {
  DISPATCH_E(E, k_g_standalone<EV><<<m, kNodeThreads, smem, st>>>(mode, p, n2, in, state, kbar, M,
                                                                  out, gscr, gstride));
  return cudaGetLastError();
}

}  // namespace bnbg
