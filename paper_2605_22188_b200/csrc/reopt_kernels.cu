// reopt_kernels.cu -- instantiations and cluster launcher of k_reopt_cluster.
#include <cstdlib>

#include "launchers.hpp"
#include "reopt_kernels.cuh"

namespace bnbg {

template <int Q, int R>
static cudaError_t launch_q_r(int cs, int nsup, cudaStream_t st, int n, const double* X,
                              const double* y, int loss, double M, double lambda2, double step,
                              const int* off, const int* idx, double* coef, double* obj,
                              int* its) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nsup * cs);
  cfg.blockDim = dim3(kReoptClusterThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  static const bool mb = [] {
    const char* e = getenv("BNBG_REOPT_MB");  // 0: cluster-barrier exchange
    return !(e && e[0] == '0');
  }();
  if (cs > 8) {
    cudaError_t e = cudaFuncSetAttribute(mb ? (const void*)k_reopt_cluster_mb<Q, R>
                                            : (const void*)k_reopt_cluster<Q, R>,
                                         cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  if (mb)
    return cudaLaunchKernelEx(&cfg, k_reopt_cluster_mb<Q, R>, n, X, y, loss, M, lambda2, step, off,
                              idx, coef, obj, its);
  return cudaLaunchKernelEx(&cfg, k_reopt_cluster<Q, R>, n, X, y, loss, M, lambda2, step, off, idx,
                            coef, obj, its);
}

cudaError_t launch_reopt_cluster(int qmax, int rpt, int cs, int nsup, cudaStream_t st, int n,
                                 const double* X, const double* y, int loss, double M,
                                 double lambda2, double step, const int* off, const int* idx,
                                 double* coef, double* obj, int* its) {
  // the exchange maps one thread to each (destination, value) pair
  if (cs < 1 || cs > kReoptMaxCluster || cs * qmax > kReoptClusterThreads)
    return cudaErrorInvalidValue;
#define RQ(Q, R)                                                                              \
  if (qmax == Q && rpt == R)                                                                  \
    return launch_q_r<Q, R>(cs, nsup, st, n, X, y, loss, M, lambda2, step, off, idx, coef, obj, \
                            its);
  RQ(8, 1) RQ(8, 2) RQ(8, 4) RQ(8, 8) RQ(16, 1) RQ(16, 2) RQ(16, 4)
#undef RQ
  return cudaErrorInvalidValue;
}

size_t reopt_smem_bytes(int n, int qmax, int cs) {
  const int qm = qmax <= 8 ? 8 : 16;
  const size_t rows = (size_t)(n + cs - 1) / cs;
  return sizeof(double) * (rows * qm + rows);
}

template <int Q>
static cudaError_t launch_smem_q(int cs, int nsup, cudaStream_t st, int n, const double* X,
                                 const double* y, int loss, double M, double lambda2, double step,
                                 const int* off, const int* idx, double* coef, double* obj,
                                 int* its) {
  const size_t smem = reopt_smem_bytes(n, Q, cs);
  cudaError_t e = cudaFuncSetAttribute(k_reopt_cluster_smem<Q>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess && cs > 8)
    e = cudaFuncSetAttribute(k_reopt_cluster_smem<Q>,
                             cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nsup * cs);
  cfg.blockDim = dim3(kReoptSmemThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_reopt_cluster_smem<Q>, n, X, y, loss, M, lambda2, step, off,
                            idx, coef, obj, its);
}

cudaError_t launch_reopt_smem(int qmax, int cs, int nsup, cudaStream_t st, int n, const double* X,
                              const double* y, int loss, double M, double lambda2, double step,
                              const int* off, const int* idx, double* coef, double* obj,
                              int* its) {
  if (qmax <= 8)
    return launch_smem_q<8>(cs, nsup, st, n, X, y, loss, M, lambda2, step, off, idx, coef, obj,
                            its);
  return launch_smem_q<16>(cs, nsup, st, n, X, y, loss, M, lambda2, step, off, idx, coef, obj, its);
}

}  // namespace bnbg
