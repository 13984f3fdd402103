// Phase timing of the per-column prox kernel on one column (clock64 stamps).
#include <cstdio>
#include <vector>
#include <random>
__device__ long long g_probe[8];
#define BNBG_PAVA_PROBE(i) do { if (threadIdx.x == 0) g_probe[i] = clock64(); } while (0)
#include "../../paper_2605_22188_b200/csrc/node_kernels.cuh"
using namespace bnbg;

template <int EE> __global__ void __launch_bounds__(kNodeThreads) k_phases(int p, int n2, const double* U, int kb, double rho, double M, long long* stamps, double* out) {
  extern __shared__ __align__(16) double sm[];
  const ColSmem S = col_smem(sm, p, n2, EE);
  double* key = S.key; int* idx = S.idx; double* u = S.u;
  long long t0 = clock64();
  double kk[EE]; int ii[EE];
  for (int r = 0; r < EE; ++r) { int j = threadIdx.x * EE + r; kk[r] = j < p ? rho * fabs(U[j]) : -2.0; ii[r] = j; if (j < p) u[j] = U[j]; }
  __syncthreads();
  long long t1 = clock64();
  reg_bitonic<kNodeThreads, EE>(kk, ii, S.xk, S.xi);
  for (int r = 0; r < EE; ++r) { key[threadIdx.x * EE + r] = kk[r]; idx[threadIdx.x * EE + r] = ii[r]; }
  __syncthreads();
  long long t2 = clock64();
  int lo, hi; double pooled;
  block_pava<kNodeThreads>(key, p, kb, rho, M, S.scan, lo, hi, pooled);
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
  for (int p : {500}) {
    int n2 = 1; while (n2 < p) n2 <<= 1;
    std::vector<double> U(p); std::mt19937 g(1); std::normal_distribution<double> nd(0, 0.01);
    for (auto& x : U) x = nd(g);
    double *dU, *dout; long long* dst; cudaMalloc(&dU, 8 * p); cudaMalloc(&dout, 8 * p); cudaMalloc(&dst, 64);
    cudaMemcpy(dU, U.data(), 8 * p, cudaMemcpyHostToDevice);
    const int E = n2 <= 256 ? 1 : n2 <= 512 ? 2 : n2 <= 1024 ? 4 : 8;
    size_t smem = column_smem_bytes(p, n2, E);
    auto kern = E == 1 ? k_phases<1> : E == 2 ? k_phases<2> : E == 4 ? k_phases<4> : k_phases<8>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int rep = 0; rep < 3; ++rep) kern<<<148, kNodeThreads, smem>>>(p, n2, dU, 8, 900.0, 2.0, dst, dout);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0); kern<<<148, kNodeThreads, smem>>>(p, n2, dU, 8, 900.0, 2.0, dst, dout); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long st[6]; cudaMemcpy(st, dst, 48, cudaMemcpyDeviceToHost);
    long long pr[8]; cudaMemcpyFromSymbol(pr, g_probe, sizeof(pr));
    printf("  pava probes: scan %lld, walk %lld, final %lld\n", pr[1]-pr[0], pr[3]-pr[1], pr[4]-pr[3]);
    printf("p=%d n2=%d: load %lld sort %lld pava %lld scatter %lld cycles; lo=%lld hi=%lld; kernel %.2f us  err=%s\n", p, n2, st[0], st[1], st[2], st[3], st[4], st[5], ms * 1e3, cudaGetErrorString(cudaGetLastError()));
  }
}
