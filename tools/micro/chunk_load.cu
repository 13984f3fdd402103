// Latency of staging a 32 KB B chunk into shared memory (the resident pass
// kernel's per-tile load): 16-byte cp.async issue + wait, per CTA.
#include <cstdio>
__device__ __forceinline__ void cp16(void* s, const void* g) {
  unsigned a = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(a), "l"(g));
}
__global__ void k(const double* src, int distinct, int reps, long long* out) {
  extern __shared__ double sm[];
  const double* base = src + (distinct ? (size_t)blockIdx.x * 4096 : 0);
  long long ti = 0, tw = 0;
  for (int r = 0; r < reps; ++r) {
    __syncthreads();
    long long t0 = clock64();
    for (int e = threadIdx.x; e < 2048; e += blockDim.x) cp16(sm + 2 * e, base + 2 * e);
    asm volatile("cp.async.commit_group;\n");
    long long t1 = clock64();
    asm volatile("cp.async.wait_group 0;\n");
    __syncthreads();
    long long t2 = clock64();
    ti += t1 - t0;
    tw += t2 - t1;
  }
  if (threadIdx.x == 0) {
    out[2 * blockIdx.x] = ti / reps;
    out[2 * blockIdx.x + 1] = tw / reps;
  }
}
int main() {
  double* src; long long* out;
  cudaMalloc(&src, 8ull << 22); cudaMemset(src, 0, 8ull << 22);
  cudaMalloc(&out, 16 * 256);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  for (int grid : {1, 125}) for (int distinct : {0, 1}) {
    k<<<grid, 256, 33000>>>(src, distinct, 50, out);
    long long h[2]; cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    printf("grid %3d %s source: issue %lld cycles, wait %lld cycles (CTA 0)  %s\n", grid,
           distinct ? "distinct" : "shared  ", h[0], h[1], cudaGetErrorString(cudaGetLastError()));
  }
}
