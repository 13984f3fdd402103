// Chunk-load latency when the chunk was just written by other SMs (the pass
// kernel's pattern: prox CTAs write V, grid barrier, every CTA loads V).
#include <cstdio>
__device__ __forceinline__ void cp16(void* s, const void* g) {
  unsigned a = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(a), "l"(g));
}
__device__ __forceinline__ void gbar(unsigned* ctr, unsigned& target) {
  target += gridDim.x;
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(ctr) : "memory");
    unsigned v;
    do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(ctr) : "memory"); } while ((int)(v - target) < 0);
  }
  __syncthreads();
}
__global__ void k(double* buf, unsigned* ctr, int writers, int reps, long long* out) {
  extern __shared__ double sm[];
  unsigned target = 0;
  long long ti = 0, tw = 0;
  for (int r = 0; r < reps; ++r) {
    if ((int)blockIdx.x < writers)
      for (int c = blockIdx.x; c < 8; c += writers)
        for (int j = threadIdx.x; j < 500; j += blockDim.x) buf[c * 500 + j] = r + j;
    gbar(ctr, target);
    long long t0 = clock64();
    for (int e = threadIdx.x; e < 2000; e += blockDim.x) cp16(sm + 2 * e, buf + 2 * e);
    asm volatile("cp.async.commit_group;\n");
    long long t1 = clock64();
    asm volatile("cp.async.wait_group 0;\n");
    __syncthreads();
    long long t2 = clock64();
    ti += t1 - t0;
    tw += t2 - t1;
    gbar(ctr, target);
  }
  if (threadIdx.x == 0) { out[2 * blockIdx.x] = ti / reps; out[2 * blockIdx.x + 1] = tw / reps; }
}
int main() {
  double* buf; unsigned* ctr; long long* out;
  cudaMalloc(&buf, 8 * 4096); cudaMalloc(&ctr, 4); cudaMalloc(&out, 16 * 256);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  for (int writers : {0, 8, 1}) {
    cudaMemset(ctr, 0, 4);
    int reps = 200;
    void* args[] = {&buf, &ctr, &writers, &reps, &out};
    cudaLaunchCooperativeKernel((void*)k, dim3(125), dim3(256), args, 33000, 0);
    cudaDeviceSynchronize();
    long long h[250]; cudaMemcpy(h, out, 16 * 125, cudaMemcpyDeviceToHost);
    long long si = 0, sw = 0, mi = 0, mw = 0;
    for (int b = 0; b < 125; ++b) { si += h[2*b]; sw += h[2*b+1]; mi = h[2*b] > mi ? h[2*b] : mi; mw = h[2*b+1] > mw ? h[2*b+1] : mw; }
    printf("writers %d: issue avg %lld max %lld, wait avg %lld max %lld cycles  %s\n", writers, si / 125, mi, sw / 125, mw, cudaGetErrorString(cudaGetLastError()));
  }
}
