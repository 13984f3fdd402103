// Phase timing of the per-column prox kernel on one column (clock64 stamps).
#include <cstdio>
#include <vector>
#include <random>
#include "../../paper_2605_22188_b200/csrc/node_kernels.cuh"
using namespace bnbg;

__global__ void __launch_bounds__(kNodeThreads) k_phases(int p, int n2, const double* U, int kb, double rho, double M, long long* stamps, double* out) {
  extern __shared__ __align__(16) double sm[];
  double* key = sm; int* idx = reinterpret_cast<int*>(key + n2); double* u = reinterpret_cast<double*>(idx + n2); double* scan = u + p;
  __shared__ double wtot[kNodeThreads / 32];
  long long t0 = clock64();
  for (int j = threadIdx.x; j < n2; j += kNodeThreads) {
    if (j < p) { u[j] = U[j]; key[j] = rho * fabs(U[j]); } else key[j] = -2.0;
    idx[j] = j;
  }
  __syncthreads();
  long long t1 = clock64();
  bitonic_sort_desc<kNodeThreads>(key, idx, n2);
  long long t2 = clock64();
  int lo, hi; double pooled;
  block_pava<kNodeThreads>(key, p, kb, rho, M, scan, wtot, lo, hi, pooled);
  __syncthreads();
  long long t3 = clock64();
  const double inv_rho = 1.0 / rho;
  for (int rk = threadIdx.x; rk < p; rk += kNodeThreads) {
    const int j = idx[rk]; const double uj = u[j];
    const bool in_block = hi >= lo && rk >= lo && rk <= hi;
    double o = 0.0;
    if (!(rk >= kb && !in_block)) { const double v = in_block ? pooled : d_prox_huber(key[rk], rho, M); const double sign = uj > 0 ? 1.0 : (uj < 0 ? -1.0 : 0.0); o = uj - inv_rho * sign * v; }
    out[j] = o;
  }
  __syncthreads();
  long long t4 = clock64();
  if (threadIdx.x == 0) { stamps[0] = t1 - t0; stamps[1] = t2 - t1; stamps[2] = t3 - t2; stamps[3] = t4 - t3; stamps[4] = lo; stamps[5] = hi; }
}

int main() {
  for (int p : {100, 500, 2000, 5000}) {
    int n2 = 1; while (n2 < p) n2 <<= 1;
    std::vector<double> U(p); std::mt19937 g(1); std::normal_distribution<double> nd(0, 0.01);
    for (auto& x : U) x = nd(g);
    double *dU, *dout; long long* dst; cudaMalloc(&dU, 8 * p); cudaMalloc(&dout, 8 * p); cudaMalloc(&dst, 64);
    cudaMemcpy(dU, U.data(), 8 * p, cudaMemcpyHostToDevice);
    size_t smem = column_smem_bytes(p, n2);
    cudaFuncSetAttribute(k_phases, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int rep = 0; rep < 3; ++rep) k_phases<<<1, kNodeThreads, smem>>>(p, n2, dU, 8, 900.0, 2.0, dst, dout);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0); k_phases<<<1, kNodeThreads, smem>>>(p, n2, dU, 8, 900.0, 2.0, dst, dout); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long st[6]; cudaMemcpy(st, dst, 48, cudaMemcpyDeviceToHost);
    printf("p=%d n2=%d: load %lld sort %lld pava %lld scatter %lld cycles; lo=%lld hi=%lld; kernel %.2f us  err=%s\n", p, n2, st[0], st[1], st[2], st[3], st[4], st[5], ms * 1e3, cudaGetErrorString(cudaGetLastError()));
  }
}
