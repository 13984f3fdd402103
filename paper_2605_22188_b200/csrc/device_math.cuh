// device_math.cuh -- scalar GLM math shared by every sm_100a kernel.
//
// Same formulas and branch structure as the reference scalars so device
// values agree with the CPU path to rounding:
//   log1p_exp / sigmoid / xlogx        losses.hpp:37-52
//   loss_value / derivative / conjugate losses.hpp:56-79
//   huber_value / prox_huber          prox_kernel.hpp:27-36
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace bnbg {

constexpr int kFree = 0, kFixedOne = 1, kFixedZero = 2;
constexpr int kSquared = 0, kLogistic = 1;
constexpr int kPrunable = 0, kConverged = 1, kCapped = 2;

__host__ __device__ __forceinline__ double d_inf() {
#ifdef __CUDA_ARCH__
  return __longlong_as_double(0x7ff0000000000000LL);
#else
  return __builtin_huge_val();
#endif
}

__device__ __forceinline__ double d_log1p_exp(double t) {
  if (t > 0.0) return t + log1p(exp(-t));
  return log1p(exp(t));
}

__device__ __forceinline__ double d_sigmoid(double t) {
  if (t >= 0.0) {
    const double e = exp(-t);
    return 1.0 / (1.0 + e);
  }
  const double e = exp(t);
  return e / (1.0 + e);
}

__device__ __forceinline__ double d_xlogx(double v) { return v > 0.0 ? v * log(v) : 0.0; }

__device__ __forceinline__ double d_loss_value(int loss, double s, double y) {
  if (loss == kSquared) {
    const double r = s - y;
    return 0.5 * r * r;
  }
  return d_log1p_exp(-y * s);
}

__device__ __forceinline__ double d_loss_deriv(int loss, double s, double y) {
  if (loss == kSquared) return s - y;
  return -y * d_sigmoid(-y * s);
}

__device__ __forceinline__ double d_loss_conj(int loss, double zeta, double y) {
  if (loss == kSquared) return 0.5 * zeta * zeta + zeta * y;
  const double a = -zeta * y;
  if (a < 0.0 || a > 1.0) return d_inf();
  return d_xlogx(a) + d_xlogx(1.0 - a);
}

__device__ __forceinline__ double d_huber(double q, double M) {
  const double a = fabs(q);
  return a <= M ? 0.5 * q * q : M * a - 0.5 * M * M;
}

__device__ __forceinline__ double d_prox_huber(double x, double w, double M) {
  if (fabs(x) <= (1.0 + w) * M) return x / (1.0 + w);
  return x - w * M * (x > 0.0 ? 1.0 : -1.0);
}

// FP64 tensor-core MMA, D(8x8) += A(8x4, row) * B(4x8, col).  Lowers to
// DMMA.8x8x4 on sm_100a (the FP64 tensor path; tcgen05 has no f64 kind).
// Fragments: a = A[lane>>2][lane&3], b = B[lane&3][lane>>2],
// d0/d1 = D[lane>>2][(lane&3)*2 + {0,1}].
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async_8(void* smem, const void* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int src_size = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem),
               "r"(src_size));
}
// 16-byte copy; src_bytes in {0, 8, 16}, the rest of the 16 bytes zero-filled
__device__ __forceinline__ void cp_async_16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---- mbarrier / bulk-async helpers (sm_90+ PTX) ----------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_arm(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ uint32_t cluster_map(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_f64(uint32_t addr, double v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];\n" ::"r"(
                   addr),
               "l"(__double_as_longlong(v)), "r"(bar)
               : "memory");
}

// Block-wide deterministic sum (fixed shuffle tree + fixed warp order).
// `red` must hold blockDim.x/32 doubles.  All threads receive the result.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < NT / 32; ++w) s += red[w];
  return s;
}

// Block-wide deterministic sums of NV values at once (one barrier pair).
// `red` must hold (blockDim.x/32) * NV doubles.  All threads receive the sums.
template <int NT, int NV>
__device__ __forceinline__ void block_sum_vec(double (&v)[NV], double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int r = 0; r < NV; ++r)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[r] += __shfl_xor_sync(0xffffffffu, v[r], o);
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int r = 0; r < NV; ++r) red[warp * NV + r] = v[r];
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < NV; ++r) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) s += red[w * NV + r];
    v[r] = s;
  }
}

template <int NT>
__device__ __forceinline__ int block_or(int v, int* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = __any_sync(0xffffffffu, v) ? 1 : 0;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  int s = 0;
#pragma unroll
  for (int w = 0; w < NT / 32; ++w) s |= red[w];
  return s;
}

template <int NT>
__device__ __forceinline__ int block_count(int v, int* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int c = __popc(__ballot_sync(0xffffffffu, v != 0));
  __syncthreads();
  if (lane == 0) red[warp] = c;
  __syncthreads();
  int s = 0;
#pragma unroll
  for (int w = 0; w < NT / 32; ++w) s += red[w];
  return s;
}

// In-place bitonic sort of n2 (a power of two) (key, idx) pairs in shared
// memory into the reference order: key descending, index ascending
// (prox_kernel.hpp:119-122, primal_heuristics.hpp:41-45).
template <int NT>
__device__ __forceinline__ void bitonic_sort_desc(double* key, int* idx, int n2) {
  for (int size = 2; size <= n2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int t = threadIdx.x; t < (n2 >> 1); t += NT) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const double ka = key[lo], kb = key[hi];
        const int ia = idx[lo], ib = idx[hi];
        const bool hi_first = (kb > ka) || (kb == ka && ib < ia);
        const bool up = (lo & size) == 0;
        if (hi_first == up) {
          key[lo] = kb;
          key[hi] = ka;
          idx[lo] = ib;
          idx[hi] = ia;
        }
      }
    }
  }
  __syncthreads();
}

}  // namespace bnbg
