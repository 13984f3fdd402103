// Microbenchmark: FP64 DFMA vs DMMA (mma.sync m8n8k4 f64) issue throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_peak(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0+4, a5=a0+5, a6=a0+6, a7=a0+7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__global__ void dmma_peak(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 0.5;
  double c[8][2] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) dmma(c[u][0], c[u][1], a, b);
  }
  double s = 0; for (int u = 0; u < 8; ++u) s += c[u][0] + c[u][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__device__ __forceinline__ void dmma16(double* d, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
}
__global__ void dmma16_peak(double* out, int iters) {
  double a[2] = {threadIdx.x * 1e-3, 0.3}, b[1] = {0.5};
  double c[4][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) dmma16(c[u], a, b);
  }
  double s = 0; for (int u = 0; u < 4; ++u) s += c[u][0] + c[u][1] + c[u][2] + c[u][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, sizeof(double) * 1 << 24);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096;
  for (int threads : {256, 512}) for (int bps : {2, 4}) {
    int blocks = sms * bps;
    dfma_peak<<<blocks, threads>>>(out, 16); cudaDeviceSynchronize();
    cudaEventRecord(e0); dfma_peak<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 64 * iters * (double)blocks * threads;
    printf("DFMA   threads=%d blocks=%d: %.2f TFLOP/s\n", threads, blocks, flops / ms / 1e9);
    dmma_peak<<<blocks, threads>>>(out, 16); cudaDeviceSynchronize();
    cudaEventRecord(e0); dmma_peak<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 8 * 8 * 4 * 8 * (double)iters * blocks * (threads / 32);
    printf("DMMA884 threads=%d blocks=%d: %.2f TFLOP/s\n", threads, blocks, flops / ms / 1e9);
    dmma16_peak<<<blocks, threads>>>(out, 16); cudaDeviceSynchronize();
    cudaEventRecord(e0); dmma16_peak<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 16 * 8 * 4 * 4 * (double)iters * blocks * (threads / 32);
    printf("DMMA1684 threads=%d blocks=%d: %.2f TFLOP/s\n", threads, blocks, flops / ms / 1e9);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
