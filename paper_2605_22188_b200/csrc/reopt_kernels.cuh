// reopt_kernels.cuh -- VK10 re-optimisation and the smoothness-constant GEMVs.
//
//   k_reopt / k_reopt_direct / k_reopt_gram   reoptimize_supports
//                                  (primal_heuristics.hpp:174-227)
//   k_pw_xv, k_pw_xtv, k_pw_step     smoothness_constant
//                                  power iteration (losses.hpp:86-112)
#pragma once
#include <cooperative_groups.h>

#include "device_math.cuh"

namespace bnbg {

// --------------------------------------------------------------------------
// VK10: box-constrained refit of each support by projected gradient,
// step 1/(L + 2 lambda2), stop at |beta - next|/step <= 1e-8 or 5000
// iterations; objective exact at the returned coefficients.
// --------------------------------------------------------------------------
constexpr int kReoptThreads = 256;

static __global__ void __launch_bounds__(kReoptThreads)
    k_reopt(int n, const double* __restrict__ X, const double* __restrict__ y, int loss, double M,
            double lambda2, double step, const int* off, const int* sidx, double* deriv_scratch,
            double* coef_out, double* obj_out, int* it_out) {
  extern __shared__ __align__(16) double sm[];
  constexpr int NW = kReoptThreads / 32;
  const int s = blockIdx.x;
  const int q = off[s + 1] - off[s];
  const int* S = sidx + off[s];
  double* beta = sm;            // q
  double* red = beta + q;       // NW * q
  double* nxt = red + NW * q;   // q
  __shared__ int s_stop;
  __shared__ double wred[NW];
  double* d = deriv_scratch + (size_t)s * n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int r = tid; r < q; r += kReoptThreads) beta[r] = 0.0;
  if (tid == 0) s_stop = 0;
  __syncthreads();
  int its = 0;
  if (q > 0) {
    for (int it = 0; it < 5000; ++it) {
      ++its;
      // scores and derivative for this thread's rows (primal_heuristics.hpp:194-209)
      for (int i = tid; i < n; i += kReoptThreads) {
        double sc = 0.0;
        for (int r = 0; r < q; ++r) sc += beta[r] * X[(size_t)S[r] * n + i];
        d[i] = d_loss_deriv(loss, sc, y[i]);
      }
      // grad_r = X_{S_r}' deriv (+ 2 lambda2 beta_r)  (:210-211)
      for (int r = 0; r < q; ++r) {
        const double* col = X + (size_t)S[r] * n;
        double a = 0.0;
        for (int i = tid; i < n; i += kReoptThreads) a += col[i] * d[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0) red[warp * q + r] = a;
      }
      __syncthreads();
      for (int r = tid; r < q; r += kReoptThreads) {
        double gr = 0.0;
        for (int w = 0; w < NW; ++w) gr += red[w * q + r];
        gr += 2.0 * lambda2 * beta[r];
        double v = beta[r] - step * gr;
        v = v < -M ? -M : v;
        v = v > M ? M : v;
        nxt[r] = v;
      }
      __syncthreads();
      if (tid == 0) {
        double gm2 = 0.0;
        for (int r = 0; r < q; ++r) {
          const double dl = beta[r] - nxt[r];
          gm2 += dl * dl;
        }
        s_stop = (sqrt(gm2) / step) <= 1e-8;
      }
      __syncthreads();
      for (int r = tid; r < q; r += kReoptThreads) beta[r] = nxt[r];
      const int stop = s_stop;
      __syncthreads();
      if (stop) break;
    }
  }
  // objective lambda2 |beta|^2 + sum l(X_S beta)  (:217-222)
  double acc = 0.0;
  for (int i = tid; i < n; i += kReoptThreads) {
    double sc = 0.0;
    for (int r = 0; r < q; ++r) sc += beta[r] * X[(size_t)S[r] * n + i];
    acc += d_loss_value(loss, sc, y[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) wred[warp] = acc;
  __syncthreads();
  if (tid == 0) {
    double sq = 0.0;
    for (int r = 0; r < q; ++r) sq += beta[r] * beta[r];
    double obj = lambda2 * sq;
    for (int w = 0; w < NW; ++w) obj += wred[w];
    obj_out[s] = obj;
    if (it_out) it_out[s] = its;
  }
  for (int r = tid; r < q; r += kReoptThreads) coef_out[off[s] + r] = beta[r];
}

// --------------------------------------------------------------------------
// VK10 fast paths (q <= QMAX).  Every thread of the CTA keeps the whole
// coefficient vector in registers and recomputes the update redundantly from
// the same shared partial sums, so one barrier per iteration suffices and all
// threads take the same stopping decision.
//
// k_reopt_direct: the reference's gather form (primal_heuristics.hpp:194-215):
//   scores = sum_r beta_r X[:,S_r] (r ascending), deriv = l'(scores),
//   grad_r = X[:,S_r]' deriv + 2 lambda2 beta_r, next = clip(beta - step grad).
// --------------------------------------------------------------------------
constexpr int kReoptFastThreads = 512;

template <int QMAX>
__global__ void __launch_bounds__(kReoptFastThreads)
    k_reopt_direct(int n, const double* __restrict__ X, const double* __restrict__ y, int loss,
                   double M, double lambda2, double step, const int* off, const int* sidx,
                   double* deriv_scratch, double* coef_out, double* obj_out, int* it_out) {
  constexpr int NW = kReoptFastThreads / 32;
  __shared__ double red[2][NW][QMAX];
  __shared__ const double* cols[QMAX];
  __shared__ double wred[NW];
  const int s = blockIdx.x;
  const int q = off[s + 1] - off[s];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < q) cols[tid] = X + (size_t)sidx[off[s] + tid] * n;
  __syncthreads();
  double* d = deriv_scratch + (size_t)s * n;
  double beta[QMAX];
#pragma unroll
  for (int r = 0; r < QMAX; ++r) beta[r] = 0.0;
  int buf = 0;
  int its = 0;
  if (q > 0) {
    for (int it = 0; it < 5000; ++it) {
      ++its;
      double part[QMAX];
#pragma unroll
      for (int r = 0; r < QMAX; ++r) part[r] = 0.0;
      for (int i = tid; i < n; i += kReoptFastThreads) {
        double sc = 0.0;
#pragma unroll
        for (int r = 0; r < QMAX; ++r)
          if (r < q) sc += beta[r] * cols[r][i];
        const double di = d_loss_deriv(loss, sc, y[i]);
#pragma unroll
        for (int r = 0; r < QMAX; ++r)
          if (r < q) part[r] += cols[r][i] * di;
      }
#pragma unroll
      for (int r = 0; r < QMAX; ++r) {
        if (r < q) {
          double a = part[r];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
          if (lane == 0) red[buf][warp][r] = a;
        }
      }
      __syncthreads();
      double gm2 = 0.0;
#pragma unroll
      for (int r = 0; r < QMAX; ++r) {
        if (r < q) {
          double g = 0.0;
          for (int w = 0; w < NW; ++w) g += red[buf][w][r];
          g += 2.0 * lambda2 * beta[r];
          double v = beta[r] - step * g;
          v = v < -M ? -M : v;
          v = v > M ? M : v;
          const double dl = beta[r] - v;
          gm2 += dl * dl;
          beta[r] = v;
        }
      }
      buf ^= 1;
      if (sqrt(gm2) / step <= 1e-8) break;
    }
  }
  (void)d;
  double acc = 0.0;
  for (int i = tid; i < n; i += kReoptFastThreads) {
    double sc = 0.0;
#pragma unroll
    for (int r = 0; r < QMAX; ++r)
      if (r < q) sc += beta[r] * cols[r][i];
    acc += d_loss_value(loss, sc, y[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) wred[warp] = acc;
  __syncthreads();
  if (tid == 0) {
    double sq = 0.0;
#pragma unroll
    for (int r = 0; r < QMAX; ++r)
      if (r < q) sq += beta[r] * beta[r];
    double obj = lambda2 * sq;
    for (int w = 0; w < NW; ++w) obj += wred[w];
    obj_out[s] = obj;
    if (it_out) it_out[s] = its;
#pragma unroll
    for (int r = 0; r < QMAX; ++r)
      if (r < q) coef_out[off[s] + r] = beta[r];
  }
}

// --------------------------------------------------------------------------
// k_reopt_cluster: the gather form split over a thread-block cluster of CS
// CTAs (CS = 1..8, chosen at launch).  CTA `rank` owns rows
// [rank*chunk, (rank+1)*chunk) and keeps its slice of X_S and y in registers
// for all 5000 iterations (RPT rows per thread), so an iteration touches no
// memory: per-row scores / l' / gradient partials, a warp-shuffle and
// cross-warp reduction, then the CTA partials are exchanged through
// distributed shared memory and one cluster barrier.  Every CTA sums the
// partials in rank order and redoes the q-vector update, so all CTAs hold the
// same beta and take the same stopping decision.  Partial buffers alternate
// per iteration, which makes one cluster barrier per iteration sufficient.
// --------------------------------------------------------------------------
constexpr int kReoptClusterThreads = 128;
constexpr int kReoptMaxCluster = 16;  // > 8 needs the non-portable cluster size

// Warp reduce-scatter of QMAX partial sums (QMAX in {8, 16}): log2(QMAX)
// halving exchanges, then a butterfly over the remaining lane bits -- 9
// shuffles for QMAX = 8 instead of 40.  On return v[0] of lane L holds the
// warp total of value reduce_scatter_index<QMAX>(L).
template <int QMAX>
__device__ __forceinline__ int reduce_scatter_index(int lane) {
  return QMAX == 8 ? (lane >> 2) & 7 : (lane >> 1) & 15;
}
template <int QMAX>
__device__ __forceinline__ void warp_reduce_scatter(double (&v)[QMAX], int lane) {
  constexpr int LOGQ = QMAX == 8 ? 3 : 4;
#pragma unroll
  for (int l = 0; l < LOGQ; ++l) {
    const int o = 16 >> l;
    const int half = QMAX >> (l + 1);
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int r = 0; r < half; ++r) {
      const double send = up ? v[r] : v[r + half];
      const double keep = up ? v[r + half] : v[r];
      v[r] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
#pragma unroll
  for (int o = 16 >> LOGQ; o > 0; o >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
}

template <int QMAX, int RPT>
__global__ void __launch_bounds__(kReoptClusterThreads)
    k_reopt_cluster(int n, const double* __restrict__ X, const double* __restrict__ y, int loss,
                    double M, double lambda2, double step, const int* off, const int* sidx,
                    double* coef_out, double* obj_out, int* it_out) {
  namespace cg = cooperative_groups;
  constexpr int NT = kReoptClusterThreads, NW = NT / 32;
  cg::cluster_group cl = cg::this_cluster();
  const int CS = (int)cl.num_blocks();
  const int rank = (int)cl.block_rank();
  const int s = blockIdx.x / CS;
  __shared__ double red[2][NW][QMAX];
  __shared__ __align__(16) double xsum[2][kReoptMaxCluster][QMAX];
  __shared__ double fin[kReoptMaxCluster];
  __shared__ double wred[NW];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = off[s + 1] - off[s];
  const int* S = sidx + off[s];
  const int chunk = (n + CS - 1) / CS;
  const int r0 = rank * chunk, r1 = min(n, r0 + chunk);
  double xs[RPT][QMAX], ys[RPT];
  bool valid[RPT];
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    const int i = r0 + j * NT + tid;
    valid[j] = i < r1;
    ys[j] = valid[j] ? y[i] : 0.0;
#pragma unroll
    for (int r = 0; r < QMAX; ++r) xs[j][r] = (valid[j] && r < q) ? X[(size_t)S[r] * n + i] : 0.0;
  }
  double beta[QMAX];
#pragma unroll
  for (int r = 0; r < QMAX; ++r) beta[r] = 0.0;
  const int ridx = reduce_scatter_index<QMAX>(lane);
  const bool writer = (lane & (32 / QMAX - 1)) == 0;
  int buf = 0, its = 0;
  if (q > 0) {
    for (int it = 0; it < 5000; ++it) {
      ++its;
      double part[QMAX];
#pragma unroll
      for (int r = 0; r < QMAX; ++r) part[r] = 0.0;
#pragma unroll
      for (int j = 0; j < RPT; ++j) {
        double sc = 0.0;  // scores, r ascending (primal_heuristics.hpp:194-198)
#pragma unroll
        for (int r = 0; r < QMAX; ++r) sc += beta[r] * xs[j][r];
        const double di = valid[j] ? d_loss_deriv(loss, sc, ys[j]) : 0.0;
#pragma unroll
        for (int r = 0; r < QMAX; ++r) part[r] += xs[j][r] * di;
      }
      warp_reduce_scatter<QMAX>(part, lane);
      if (writer) red[buf][warp][ridx] = part[0];
      __syncthreads();
      if (tid < CS * QMAX) {  // one DSMEM store per (destination, value)
        const int dst = tid / QMAX, r = tid % QMAX;
        double v = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) v += red[buf][w][r];
        *cl.map_shared_rank(&xsum[buf][rank][r], dst) = v;
      }
      cl.sync();
      double gs[QMAX];
#pragma unroll
      for (int r = 0; r < QMAX; ++r) gs[r] = 0.0;
      for (int c = 0; c < CS; ++c) {
        const double2* row = reinterpret_cast<const double2*>(xsum[buf][c]);
#pragma unroll
        for (int r2 = 0; r2 < QMAX / 2; ++r2) {
          const double2 t = row[r2];
          gs[2 * r2] += t.x;
          gs[2 * r2 + 1] += t.y;
        }
      }
      double gm2 = 0.0;
#pragma unroll
      for (int r = 0; r < QMAX; ++r) {
        double g = gs[r];
        g += 2.0 * lambda2 * beta[r];  // (:210-211)
        double v = beta[r] - step * g;
        v = v < -M ? -M : v;
        v = v > M ? M : v;
        const double dl = beta[r] - v;
        gm2 += dl * dl;
        beta[r] = r < q ? v : 0.0;
      }
      buf ^= 1;
      if (sqrt(gm2) / step <= 1e-8) break;  // (:212-215)
    }
  }
  // objective lambda2 |beta|^2 + sum l(X_S beta)  (:217-222)
  double acc = 0.0;
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    double sc = 0.0;
#pragma unroll
    for (int r = 0; r < QMAX; ++r) sc += beta[r] * xs[j][r];
    if (valid[j]) acc += d_loss_value(loss, sc, ys[j]);
  }
  const double cta = block_sum<NT>(acc, wred);
  if (tid == 0) *cl.map_shared_rank(&fin[rank], 0) = cta;
  cl.sync();
  if (rank == 0 && tid == 0) {
    double sq = 0.0;
#pragma unroll
    for (int r = 0; r < QMAX; ++r) sq += beta[r] * beta[r];
    double obj = lambda2 * sq;
    for (int c = 0; c < CS; ++c) obj += fin[c];
    obj_out[s] = obj;
    if (it_out) it_out[s] = its;
    for (int r = 0; r < q && r < QMAX; ++r) coef_out[off[s] + r] = beta[r];
  }
}

// k_reopt_cluster_mb: k_reopt_cluster with the per-iteration exchange done by
// st.async remote stores that complete transactions on the receiver's
// mbarrier (double-buffered), instead of a full cluster barrier: a CTA waits
// only for the bytes it needs, with no cluster-wide arrive/wait round trip.
// A buffer's barrier is re-armed (arrive.expect_tx) after the next iteration's
// first block barrier -- every thread has consumed it by then -- and before
// this CTA's sends of that iteration, which precede every sender's next write
// to it: one block barrier per iteration.
template <int QMAX, int RPT>
__global__ void __launch_bounds__(kReoptClusterThreads)
    k_reopt_cluster_mb(int n, const double* __restrict__ X, const double* __restrict__ y, int loss,
                       double M, double lambda2, double step, const int* off, const int* sidx,
                       double* coef_out, double* obj_out, int* it_out) {
  namespace cg = cooperative_groups;
  constexpr int NT = kReoptClusterThreads, NW = NT / 32;
  cg::cluster_group cl = cg::this_cluster();
  const int CS = (int)cl.num_blocks();
  const int rank = (int)cl.block_rank();
  const int s = blockIdx.x / CS;
  __shared__ double red[2][NW][QMAX];
  __shared__ __align__(16) double xsum[2][kReoptMaxCluster][QMAX];
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ double fin[kReoptMaxCluster];
  __shared__ double wred[NW];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = off[s + 1] - off[s];
  const int* S = sidx + off[s];
  const int chunk = (n + CS - 1) / CS;
  const int r0 = rank * chunk, r1 = min(n, r0 + chunk);
  const uint32_t bytes = (uint32_t)(CS * QMAX * sizeof(double));
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    mbar_arm(&mbar[0], bytes);
    mbar_arm(&mbar[1], bytes);
  }
  double xs[RPT][QMAX], ys[RPT];
  bool valid[RPT];
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    const int i = r0 + j * NT + tid;
    valid[j] = i < r1;
    ys[j] = valid[j] ? y[i] : 0.0;
#pragma unroll
    for (int r = 0; r < QMAX; ++r) xs[j][r] = (valid[j] && r < q) ? X[(size_t)S[r] * n + i] : 0.0;
  }
  cl.sync();  // barriers initialised and armed everywhere before any remote store
  // this CTA's slot in every receiver, and every receiver's barrier, as
  // shared::cluster addresses
  uint32_t dst_slot = 0, dst_bar = 0;
  const int my_dst = tid / QMAX, my_r = tid % QMAX;
  if (tid < CS * QMAX) {
    dst_slot = cluster_map(smem_addr(&xsum[0][rank][my_r]), (uint32_t)my_dst);
    dst_bar = cluster_map(smem_addr(&mbar[0]), (uint32_t)my_dst);
  }
  const uint32_t buf_stride = (uint32_t)(kReoptMaxCluster * QMAX * sizeof(double));
  double beta[QMAX];
#pragma unroll
  for (int r = 0; r < QMAX; ++r) beta[r] = 0.0;
  const int ridx = reduce_scatter_index<QMAX>(lane);
  const bool writer = (lane & (32 / QMAX - 1)) == 0;
  int its = 0;
  if (q > 0) {
    for (int it = 0; it < 5000; ++it) {
      ++its;
      const int buf = it & 1;
      double part[QMAX];
#pragma unroll
      for (int r = 0; r < QMAX; ++r) part[r] = 0.0;
#pragma unroll
      for (int j = 0; j < RPT; ++j) {
        double sc = 0.0;  // scores, r ascending (primal_heuristics.hpp:194-198)
#pragma unroll
        for (int r = 0; r < QMAX; ++r) sc += beta[r] * xs[j][r];
        const double di = valid[j] ? d_loss_deriv(loss, sc, ys[j]) : 0.0;
#pragma unroll
        for (int r = 0; r < QMAX; ++r) part[r] += xs[j][r] * di;
      }
      warp_reduce_scatter<QMAX>(part, lane);
      if (writer) red[buf][warp][ridx] = part[0];
      __syncthreads();
      // every thread has finished reading the other buffer (last iteration):
      // re-arm it for its next use, before this CTA's sends of this iteration
      if (tid == 0 && it > 0) mbar_arm(&mbar[buf ^ 1], bytes);
      if (tid < CS * QMAX) {
        double v = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) v += red[buf][w][my_r];
        st_async_f64(dst_slot + buf * buf_stride, v, dst_bar + buf * (uint32_t)sizeof(uint64_t));
      }
      mbar_wait(&mbar[buf], (uint32_t)((it >> 1) & 1));
      double gs[QMAX];
#pragma unroll
      for (int r = 0; r < QMAX; ++r) gs[r] = 0.0;
      for (int c = 0; c < CS; ++c) {
        const double2* row = reinterpret_cast<const double2*>(xsum[buf][c]);
#pragma unroll
        for (int r2 = 0; r2 < QMAX / 2; ++r2) {
          const double2 t = row[r2];
          gs[2 * r2] += t.x;
          gs[2 * r2 + 1] += t.y;
        }
      }
      double gm2 = 0.0;
#pragma unroll
      for (int r = 0; r < QMAX; ++r) {
        double g = gs[r];
        g += 2.0 * lambda2 * beta[r];  // (:210-211)
        double v = beta[r] - step * g;
        v = v < -M ? -M : v;
        v = v > M ? M : v;
        const double dl = beta[r] - v;
        gm2 += dl * dl;
        beta[r] = r < q ? v : 0.0;
      }
      if (sqrt(gm2) / step <= 1e-8) break;  // (:212-215)
    }
  }
  // objective lambda2 |beta|^2 + sum l(X_S beta)  (:217-222)
  double acc = 0.0;
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    double sc = 0.0;
#pragma unroll
    for (int r = 0; r < QMAX; ++r) sc += beta[r] * xs[j][r];
    if (valid[j]) acc += d_loss_value(loss, sc, ys[j]);
  }
  const double cta = block_sum<NT>(acc, wred);
  if (tid == 0) *cl.map_shared_rank(&fin[rank], 0) = cta;
  cl.sync();
  if (rank == 0 && tid == 0) {
    double sq = 0.0;
#pragma unroll
    for (int r = 0; r < QMAX; ++r) sq += beta[r] * beta[r];
    double obj = lambda2 * sq;
    for (int c = 0; c < CS; ++c) obj += fin[c];
    obj_out[s] = obj;
    if (it_out) it_out[s] = its;
    for (int r = 0; r < q && r < QMAX; ++r) coef_out[off[s] + r] = beta[r];
  }
}

// k_reopt_cluster_smem: the large-n variant (c4: n = 20000, where X_S no
// longer fits 8 CTAs' registers).  Each CTA keeps its X_S slice and y in
// shared memory, column-major so consecutive threads read consecutive rows
// (conflict-free), with up to 16 CTAs per support (non-portable cluster
// size); the exchange is k_reopt_cluster_mb's st.async + mbarrier scheme.
#ifndef BNBG_REOPT_SMEM_THREADS
#define BNBG_REOPT_SMEM_THREADS 256
#endif
constexpr int kReoptSmemThreads = BNBG_REOPT_SMEM_THREADS;
constexpr int kReoptSmemMaxCluster = 16;

template <int QMAX>
__global__ void __launch_bounds__(kReoptSmemThreads)
    k_reopt_cluster_smem(int n, const double* __restrict__ X, const double* __restrict__ y,
                         int loss, double M, double lambda2, double step, const int* off,
                         const int* sidx, double* coef_out, double* obj_out, int* it_out) {
  namespace cg = cooperative_groups;
  constexpr int NT = kReoptSmemThreads, NW = NT / 32;
  extern __shared__ __align__(16) double xsl[];  // QMAX columns of `chunk` rows, then y
  cg::cluster_group cl = cg::this_cluster();
  const int CS = (int)cl.num_blocks();
  const int rank = (int)cl.block_rank();
  const int s = blockIdx.x / CS;
  __shared__ double red[2][NW][QMAX];
  __shared__ __align__(16) double xsum[2][kReoptSmemMaxCluster][QMAX];
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ double fin[kReoptSmemMaxCluster];
  __shared__ double wred[NW];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = off[s + 1] - off[s];
  const int* S = sidx + off[s];
  const int chunk = (n + CS - 1) / CS;
  const int r0 = rank * chunk, r1 = min(n, r0 + chunk), rows = max(0, r1 - r0);
  double* ysl = xsl + (size_t)chunk * QMAX;
  const uint32_t bytes = (uint32_t)(CS * QMAX * sizeof(double));
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    mbar_arm(&mbar[0], bytes);
    mbar_arm(&mbar[1], bytes);
  }
  for (int r = 0; r < QMAX; ++r)
    for (int i = tid; i < rows; i += NT)
      xsl[(size_t)r * chunk + i] = r < q ? X[(size_t)S[r] * n + r0 + i] : 0.0;
  for (int i = tid; i < rows; i += NT) ysl[i] = y[r0 + i];
  cl.sync();
  uint32_t dst_slot = 0, dst_bar = 0;
  const int my_dst = tid / QMAX, my_r = tid % QMAX;
  if (tid < CS * QMAX) {
    dst_slot = cluster_map(smem_addr(&xsum[0][rank][my_r]), (uint32_t)my_dst);
    dst_bar = cluster_map(smem_addr(&mbar[0]), (uint32_t)my_dst);
  }
  const uint32_t buf_stride = (uint32_t)(kReoptSmemMaxCluster * QMAX * sizeof(double));
  double beta[QMAX];
#pragma unroll
  for (int r = 0; r < QMAX; ++r) beta[r] = 0.0;
  const int ridx = reduce_scatter_index<QMAX>(lane);
  const bool writer = (lane & (32 / QMAX - 1)) == 0;
  int its = 0;
  if (q > 0) {
    for (int it = 0; it < 5000; ++it) {
      ++its;
      const int buf = it & 1;
      double part[QMAX];
#pragma unroll
      for (int r = 0; r < QMAX; ++r) part[r] = 0.0;
      for (int i = tid; i < rows; i += NT) {
        double xv[QMAX];
#pragma unroll
        for (int r = 0; r < QMAX; ++r) xv[r] = xsl[(size_t)r * chunk + i];
        double sc = 0.0;  // scores, r ascending (primal_heuristics.hpp:194-198)
#pragma unroll
        for (int r = 0; r < QMAX; ++r) sc += beta[r] * xv[r];
        const double di = d_loss_deriv(loss, sc, ysl[i]);
#pragma unroll
        for (int r = 0; r < QMAX; ++r) part[r] += xv[r] * di;
      }
      warp_reduce_scatter<QMAX>(part, lane);
      if (writer) red[buf][warp][ridx] = part[0];
      __syncthreads();
      if (tid == 0 && it > 0) mbar_arm(&mbar[buf ^ 1], bytes);
      if (tid < CS * QMAX) {
        double v = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) v += red[buf][w][my_r];
        st_async_f64(dst_slot + buf * buf_stride, v, dst_bar + buf * (uint32_t)sizeof(uint64_t));
      }
      mbar_wait(&mbar[buf], (uint32_t)((it >> 1) & 1));
      double gs[QMAX];
#pragma unroll
      for (int r = 0; r < QMAX; ++r) gs[r] = 0.0;
      for (int c = 0; c < CS; ++c) {
        const double2* row = reinterpret_cast<const double2*>(xsum[buf][c]);
#pragma unroll
        for (int r2 = 0; r2 < QMAX / 2; ++r2) {
          const double2 t = row[r2];
          gs[2 * r2] += t.x;
          gs[2 * r2 + 1] += t.y;
        }
      }
      double gm2 = 0.0;
#pragma unroll
      for (int r = 0; r < QMAX; ++r) {
        double g = gs[r] + 2.0 * lambda2 * beta[r];  // (:210-211)
        double v = beta[r] - step * g;
        v = v < -M ? -M : v;
        v = v > M ? M : v;
        const double dl = beta[r] - v;
        gm2 += dl * dl;
        beta[r] = r < q ? v : 0.0;
      }
      if (sqrt(gm2) / step <= 1e-8) break;  // (:212-215)
    }
  }
  double acc = 0.0;  // objective (:217-222)
  for (int i = tid; i < rows; i += NT) {
    double sc = 0.0;
#pragma unroll
    for (int r = 0; r < QMAX; ++r) sc += beta[r] * xsl[(size_t)r * chunk + i];
    acc += d_loss_value(loss, sc, ysl[i]);
  }
  const double cta = block_sum<NT>(acc, wred);
  if (tid == 0) *cl.map_shared_rank(&fin[rank], 0) = cta;
  cl.sync();
  if (rank == 0 && tid == 0) {
    double sq = 0.0;
#pragma unroll
    for (int r = 0; r < QMAX; ++r) sq += beta[r] * beta[r];
    double obj = lambda2 * sq;
    for (int c = 0; c < CS; ++c) obj += fin[c];
    obj_out[s] = obj;
    if (it_out) it_out[s] = its;
    for (int r = 0; r < q && r < QMAX; ++r) coef_out[off[s] + r] = beta[r];
  }
}

// k_reopt_gram (squared loss): X_S'(X_S beta - y) = Gram beta - X_S'y, the
// same iterates in exact arithmetic.  The q x q Gram and
// X_S'y are built once per support; warp 0 then runs the projected-gradient
// loop with lane r owning beta_r.  q <= 32.
static __global__ void __launch_bounds__(kReoptFastThreads)
    k_reopt_gram(int n, const double* __restrict__ X, const double* __restrict__ y, double M,
                 double lambda2, double step, const int* off, const int* sidx, double* coef_out,
                 double* obj_out, int* it_out) {
  constexpr int NW = kReoptFastThreads / 32;
  __shared__ double gram[32][33];
  __shared__ double xty[32];
  __shared__ double bsh[32];
  __shared__ double wred[NW];
  __shared__ const double* cols[32];
  const int s = blockIdx.x;
  const int q = off[s + 1] - off[s];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < q) cols[tid] = X + (size_t)sidx[off[s] + tid] * n;
  if (tid < 32) bsh[tid] = 0.0;
  __syncthreads();
  // Gram entries (r <= c) and X_S'y: one warp per dot product
  const int npairs = q * (q + 1) / 2 + q;
  for (int t = warp; t < npairs; t += NW) {
    int r = 0, c = 0;
    const double* a;
    const double* bvec;
    if (t < q * (q + 1) / 2) {
      int tt = t;
      while (tt >= q - r) {
        tt -= q - r;
        ++r;
      }
      c = r + tt;
      a = cols[r];
      bvec = cols[c];
    } else {
      r = t - q * (q + 1) / 2;
      a = cols[r];
      bvec = y;
    }
    double acc = 0.0;
    for (int i = lane; i < n; i += 32) acc += a[i] * bvec[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      if (t < q * (q + 1) / 2) {
        gram[r][c] = acc;
        gram[c][r] = acc;
      } else {
        xty[r] = acc;
      }
    }
  }
  __syncthreads();
  int its = 0;
  if (warp == 0 && q > 0) {
    double b = 0.0;
    const bool own = lane < q;
    for (int it = 0; it < 5000; ++it) {
      ++its;
      double g = 0.0;
      for (int c = 0; c < q; ++c) {
        const double bc = __shfl_sync(0xffffffffu, b, c);
        if (own) g += gram[lane][c] * bc;
      }
      double dl2 = 0.0, nx = 0.0;
      if (own) {
        g = g - xty[lane] + 2.0 * lambda2 * b;
        double v = b - step * g;
        v = v < -M ? -M : v;
        v = v > M ? M : v;
        nx = v;
        const double dl = b - v;
        dl2 = dl * dl;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) dl2 += __shfl_xor_sync(0xffffffffu, dl2, o);
      b = nx;
      if (sqrt(dl2) / step <= 1e-8) break;
    }
    if (own) bsh[lane] = b;
  }
  __syncthreads();
  double acc = 0.0;
  for (int i = tid; i < n; i += kReoptFastThreads) {
    double sc = 0.0;
    for (int r = 0; r < q; ++r) sc += bsh[r] * cols[r][i];
    acc += d_loss_value(kSquared, sc, y[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) wred[warp] = acc;
  __syncthreads();
  if (tid == 0) {
    double sq = 0.0;
    for (int r = 0; r < q; ++r) sq += bsh[r] * bsh[r];
    double obj = lambda2 * sq;
    for (int w = 0; w < NW; ++w) obj += wred[w];
    obj_out[s] = obj;
    if (it_out) it_out[s] = its;
  }
  if (tid < q) coef_out[off[s] + tid] = bsh[tid];
}

// smoothness_constant (losses.hpp:86-112), one power-iteration round as
// three kernels, in EXACTLY the oracle's / the reference's sequential
// association (oracle.c orc_smoothness; losses.hpp:99-102 evaluated by plain
// loops): xv_i = sum_j X_ij v_j in j order, w_j = sum_i X_ij xv_i in i order,
// v.w and |w|^2 in j order, each product rounded before its add (no FMA), so
// L is bit-identical to the oracle's.
// ps = {done, estimate, result, rounds}: once `done` is set on the device the
// remaining kernels of a launched batch of rounds return at once.
// xv = X v, one thread per row, the row's sum in j order.  The row's X
// elements (coalesced across the warp) and v (a broadcast) are loaded 16
// columns ahead of the add chain.
static __global__ void __launch_bounds__(256) k_pw_xv(int n, int p, const double* __restrict__ X,
                                                      const double* __restrict__ v,
                                                      double* __restrict__ xv, const double* ps) {
  if (ps[0] != 0.0 || ps[3] >= 100.0) return;  // stopped, or past losses.hpp:98's 100 rounds
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  constexpr int U = 16;
  double bx[U], bv[U];
  double s = 0.0;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    bx[u] = u < p ? X[(size_t)u * n + i] : 0.0;
    bv[u] = u < p ? __ldg(v + u) : 0.0;
  }
  for (int j0 = 0; j0 < p; j0 += U) {
    double nx[U], nv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + U + u;
      nx[u] = j < p ? X[(size_t)j * n + i] : 0.0;
      nv[u] = j < p ? __ldg(v + j) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (j0 + u < p) s = __dadd_rn(s, __dmul_rn(bx[u], bv[u]));
#pragma unroll
    for (int u = 0; u < U; ++u) {
      bx[u] = nx[u];
      bv[u] = nv[u];
    }
  }
  xv[i] = s;
}

// w = X' xv, one warp per column: the lanes load 32 consecutive rows of the
// column (coalesced) and form the products, staged in shared memory; lane 0
// adds them in row order (the chain of n dependent adds is the floor).
static __global__ void __launch_bounds__(256) k_pw_xtv(int n, int p, const double* __restrict__ X,
                                                       const double* __restrict__ xv,
                                                       double* __restrict__ w, const double* ps) {
  __shared__ double prods[8][2][32];
  if (ps[0] != 0.0 || ps[3] >= 100.0) return;  // stopped, or past losses.hpp:98's 100 rounds
  const int wp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.x * (blockDim.x >> 5) + wp;
  if (j >= p) return;
  const double* col = X + (size_t)j * n;
  double s = 0.0;
  int buf = 0;
  prods[wp][0][lane] = lane < n ? __dmul_rn(col[lane], xv[lane]) : 0.0;
  for (int i0 = 0; i0 < n; i0 += 32, buf ^= 1) {
    const int in = i0 + 32 + lane;  // next chunk's products, ahead of the chain
    const double nprod = in < n ? __dmul_rn(col[in], xv[in]) : 0.0;
    __syncwarp();
    if (lane == 0) {
      const double* pr = prods[wp][buf];
      if (i0 + 32 <= n) {
#pragma unroll
        for (int q = 0; q < 32; ++q) s = __dadd_rn(s, pr[q]);
      } else {
        for (int q = 0; q < n - i0; ++q) s = __dadd_rn(s, pr[q]);
      }
    }
    prods[wp][buf ^ 1][lane] = nprod;
  }
  if (lane == 0) w[j] = s;
}

// next = v.w, wn = |w| (sequential), then the round's host logic of
// losses.hpp:96-110: stop on a zero or non-positive estimate (result 1e-12),
// else v = w / wn, and stop once the estimate moves by at most 1e-4 relative
// (after round 0).  One CTA.
static __global__ void k_pw_step(int p, const double* w, double* v, double* ps) {
  constexpr int CH = 2048;  // v, w staged through shared memory in chunks
  __shared__ double cv[CH], cw[CH];
  __shared__ int s_dec;
  __shared__ double s_wn;
  if (ps[0] != 0.0 || ps[3] >= 100.0) return;  // stopped, or past losses.hpp:98's 100 rounds
  double next = 0.0, nrm2 = 0.0;  // thread 0's sequential sums (the oracle's order)
  for (int c0 = 0; c0 < p; c0 += CH) {
    const int len = min(CH, p - c0);
    for (int j = threadIdx.x; j < len; j += blockDim.x) {
      cv[j] = v[c0 + j];
      cw[j] = w[c0 + j];
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int j = 0; j < len; ++j) next = __dadd_rn(next, __dmul_rn(cv[j], cw[j]));
    __syncthreads();
  }
  for (int c0 = 0; c0 < p; c0 += CH) {
    const int len = min(CH, p - c0);
    for (int j = threadIdx.x; j < len; j += blockDim.x) cw[j] = w[c0 + j];
    __syncthreads();
    if (threadIdx.x == 0)
      for (int j = 0; j < len; ++j) nrm2 = __dadd_rn(nrm2, __dmul_rn(cw[j], cw[j]));
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double wn = sqrt(nrm2);
    int dec = 0;  // 0: continue, 1: zero / non-positive, 2: converged
    if (wn == 0.0 || next <= 0.0)
      dec = 1;
    else if (ps[3] > 0.0 && fabs(next - ps[1]) <= 1e-4 * next)
      dec = 2;
    if (dec == 1) {
      ps[2] = 1e-12;
    } else {
      ps[1] = next;
    }
    s_dec = dec;
    s_wn = wn;
  }
  __syncthreads();
  const int dec = s_dec;
  const double wn = s_wn;
  if (dec != 1)
    for (int j = threadIdx.x; j < p; j += blockDim.x) v[j] = w[j] / wn;
  if (threadIdx.x == 0) {
    if (dec != 0) ps[0] = 1.0;
    ps[3] += 1.0;
  }
}

// The whole power iteration as ONE cooperative kernel (small p: every column
// of X'(X v) has its own warp in the grid): rounds loop on the device, the
// three steps of a round (X v by rows, X'(X v) by columns, the sequential
// v.w / |w| / stopping test on CTA 0) separated by grid barriers; the same
// arithmetic and order as k_pw_xv / k_pw_xtv / k_pw_step, so L stays
// bit-identical to the oracle's.  Values written by other CTAs are read
// through L2 (__ldcg): L1 is not coherent across the grid.
static __global__ void __launch_bounds__(256) k_pw_all(int n, int p, const double* __restrict__ X,
                                                       double* v, double* xv, double* w,
                                                       double* ps) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  constexpr int CH = 1024;
  __shared__ double cv[CH], cw[CH];
  constexpr int CW = 128;  // products per chain step: 4 loads per lane in flight
  __shared__ double prods[8][2][CW];
  __shared__ int s_dec;
  __shared__ double s_wn;
  const int G = gridDim.x, tid = threadIdx.x, wp = tid >> 5, lane = tid & 31;
  for (;;) {
    if (__ldcg(ps) != 0.0 || __ldcg(ps + 3) >= 100.0) break;  // losses.hpp:98-109
    // X v: thread per row, j in order (k_pw_xv)
    for (int i = blockIdx.x * 256 + tid; i < n; i += G * 256) {
      constexpr int U = 16;
      double bx[U], bv[U];
      double s = 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        bx[u] = u < p ? __ldg(X + (size_t)u * n + i) : 0.0;
        bv[u] = u < p ? __ldcg(v + u) : 0.0;
      }
      for (int j0 = 0; j0 < p; j0 += U) {
        double nx[U], nv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = j0 + U + u;
          nx[u] = j < p ? __ldg(X + (size_t)j * n + i) : 0.0;
          nv[u] = j < p ? __ldcg(v + j) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (j0 + u < p) s = __dadd_rn(s, __dmul_rn(bx[u], bv[u]));
#pragma unroll
        for (int u = 0; u < U; ++u) {
          bx[u] = nx[u];
          bv[u] = nv[u];
        }
      }
      xv[i] = s;
    }
    grid.sync();
    // X'(X v): warp per column, lane 0 adds the products in row order (k_pw_xtv)
    for (int j = blockIdx.x * 8 + wp; j < p; j += G * 8) {
      const double* col = X + (size_t)j * n;
      double s = 0.0;
      int buf = 0;
#pragma unroll
      for (int d = 0; d < CW / 32; ++d) {
        const int i = lane + 32 * d;
        prods[wp][0][i] = i < n ? __dmul_rn(__ldg(col + i), __ldcg(xv + i)) : 0.0;
      }
      for (int i0 = 0; i0 < n; i0 += CW, buf ^= 1) {
        double np[CW / 32];  // the next step's products, loaded during this chain
#pragma unroll
        for (int d = 0; d < CW / 32; ++d) {
          const int in = i0 + CW + lane + 32 * d;
          np[d] = in < n ? __dmul_rn(__ldg(col + in), __ldcg(xv + in)) : 0.0;
        }
        __syncwarp();
        if (lane == 0) {
          const double* pr = prods[wp][buf];
          if (i0 + CW <= n) {
#pragma unroll
            for (int q = 0; q < CW; ++q) s = __dadd_rn(s, pr[q]);
          } else {
            for (int q = 0; q < n - i0; ++q) s = __dadd_rn(s, pr[q]);
          }
        }
        __syncwarp();
#pragma unroll
        for (int d = 0; d < CW / 32; ++d) prods[wp][buf ^ 1][lane + 32 * d] = np[d];
      }
      if (lane == 0) w[j] = s;
      __syncwarp();
    }
    grid.sync();
    if (blockIdx.x == 0) {  // k_pw_step
      double next = 0.0, nrm2 = 0.0;
      for (int c0 = 0; c0 < p; c0 += CH) {
        const int len = min(CH, p - c0);
        for (int j = tid; j < len; j += 256) {
          cv[j] = __ldcg(v + c0 + j);
          cw[j] = __ldcg(w + c0 + j);
        }
        __syncthreads();
        if (tid == 0)
          for (int j = 0; j < len; ++j) next = __dadd_rn(next, __dmul_rn(cv[j], cw[j]));
        __syncthreads();
      }
      for (int c0 = 0; c0 < p; c0 += CH) {
        const int len = min(CH, p - c0);
        for (int j = tid; j < len; j += 256) cw[j] = __ldcg(w + c0 + j);
        __syncthreads();
        if (tid == 0)
          for (int j = 0; j < len; ++j) nrm2 = __dadd_rn(nrm2, __dmul_rn(cw[j], cw[j]));
        __syncthreads();
      }
      if (tid == 0) {
        const double wn = sqrt(nrm2);
        int dec = 0;  // 0: continue, 1: zero / non-positive, 2: converged
        if (wn == 0.0 || next <= 0.0)
          dec = 1;
        else if (ps[3] > 0.0 && fabs(next - ps[1]) <= 1e-4 * next)
          dec = 2;
        if (dec == 1)
          ps[2] = 1e-12;
        else
          ps[1] = next;
        s_dec = dec;
        s_wn = wn;
      }
      __syncthreads();
      const int dec = s_dec;
      const double wn = s_wn;
      if (dec != 1)
        for (int j = tid; j < p; j += 256) v[j] = __ldcg(w + j) / wn;
      __syncthreads();
      if (tid == 0) {
        if (dec != 0) ps[0] = 1.0;
        ps[3] += 1.0;
      }
    }
    grid.sync();
  }
}

}  // namespace bnbg
