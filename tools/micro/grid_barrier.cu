// Grid-barrier latency on B200: 148 persistent CTAs x 256 threads, R barriers.
//   mode 0: red.release.gpu + ld.acquire.gpu poll (the pass kernel's barrier)
//   mode 1: red.release.gpu + ld.relaxed.gpu poll + fence.acq_rel.gpu
//   mode 2: cooperative_groups grid.sync()
//   mode 3: cluster (4 CTAs) barrier, leaders on the global counter, cluster barrier again
//   mode 4: the grid is ONE cluster (8 or 16 CTAs): barrier.cluster arrive.release / wait.acquire
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ void bar0(unsigned* ctr, unsigned& target, int relaxed) {
  target += gridDim.x;
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(ctr) : "memory");
    unsigned v;
    if (relaxed) {
      do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(ctr) : "memory"); } while ((int)(v - target) < 0);
      asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
    } else {
      do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(ctr) : "memory"); } while ((int)(v - target) < 0);
    }
  }
  __syncthreads();
}

__global__ void k_bar(unsigned* ctr, int reps, int mode, unsigned long long* out) {
  unsigned target = 0;
  unsigned long long t0 = clock64();
  if (mode == 2) {
    cg::grid_group g = cg::this_grid();
    for (int r = 0; r < reps; ++r) g.sync();
  } else if (mode == 3) {
    cg::cluster_group cl = cg::this_cluster();
    const int cs = cl.num_blocks();
    const int nclus = gridDim.x / cs;
    for (int r = 0; r < reps; ++r) {
      cl.sync();
      target += nclus;
      if (cl.block_rank() == 0 && threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(ctr) : "memory");
        unsigned v;
        do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(ctr) : "memory"); } while ((int)(v - target) < 0);
      }
      cl.sync();
    }
  } else if (mode == 4) {
    for (int r = 0; r < reps; ++r) {
      asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    }
  } else {
    for (int r = 0; r < reps; ++r) bar0(ctr, target, mode);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}

static void one_cluster(unsigned* ctr, unsigned long long* out, int reps) {
  cudaFuncSetAttribute(k_bar, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {2, 4, 8, 16}) for (int rep = 0; rep < 2; ++rep) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(cs); cfg.blockDim = dim3(256);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaEventRecord(a);
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_bar, ctr, reps, 4, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (rep) printf("mode 4 one cluster of %d: %.3f us per barrier (%s)\n", cs, ms * 1e3 / reps, cudaGetErrorString(e == cudaSuccess ? cudaGetLastError() : e));
  }
}

int main() {
  unsigned* ctr; unsigned long long* out;
  cudaMalloc(&ctr, 4); cudaMalloc(&out, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int reps = 20000;
  one_cluster(ctr, out, reps);
  for (int gsz : {sms, 128, 74, 37, 16}) for (int mode = 0; mode < 4; ++mode) {
    if (mode == 3 && gsz != sms) continue;
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(ctr, 0, 4);
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      int grid = mode == 3 ? (sms / 4) * 4 : gsz;
      cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(grid); cfg.blockDim = dim3(256);
      cudaLaunchAttribute at[2]; int na = 0;
      at[na].id = cudaLaunchAttributeCooperative; at[na].val.cooperative = 1; ++na;
      if (mode == 3) { at[na].id = cudaLaunchAttributeClusterDimension; at[na].val.clusterDim.x = 4; at[na].val.clusterDim.y = 1; at[na].val.clusterDim.z = 1; ++na; }
      cfg.attrs = at; cfg.numAttrs = na;
      cudaEventRecord(a);
      cudaError_t e = cudaLaunchKernelEx(&cfg, k_bar, ctr, reps, mode, out);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("mode %d grid %d: %.3f us per barrier (%s)\n", mode, grid, ms * 1e3 / reps, cudaGetErrorString(e == cudaSuccess ? cudaGetLastError() : e));
    }
  }
}
