// pass_kernel.cuh -- the whole batched relaxation of one BnB pass as a single
// persistent cooperative kernel (solve_batch_relaxation, relaxation.hpp:163-255).
//
// At narrow frontiers (m_a columns << SMs x tiles) every iteration is a chain
// of three dependent, latency-bound steps: S = X V (+ l' epilogue), G = X'R,
// prox + FISTA.  Launching them as separate kernels costs a launch gap and a
// ramp/drain per step and a host round trip per check interval.  Here one
// CTA per SM loops over the iterations on the device:
//
//   phase NN   row tiles of X (BM=16) x active columns     -> R = l'(X V)
//   grid.sync
//   phase TN   column tiles of X x active columns x split-K -> G slabs
//   grid.sync
//   phase prox one CTA per active column                  -> B, V
//   grid.sync
//   every check_interval: NN(eval) / TN / per-column bounds / compaction,
//   with the active count read back on the device (no host round trip).
//
// The per-phase code is exactly the standalone kernels' (gemm_tile,
// prox_column, eval_column, compact_active), so results are identical to the
// multi-kernel path; only the scheduling differs.
#pragma once
#include <cooperative_groups.h>

#include "gemm.cuh"
#include "launchers.hpp"
#include "node_kernels.cuh"

namespace bnbg {

namespace cg = cooperative_groups;

constexpr int kPassThreads = kNodeThreads;  // 8 warps
constexpr int kPassNW = kPassThreads / 32;

__device__ __forceinline__ int pass_fn(int ma) { return ma <= 8 ? 1 : (ma <= 16 ? 2 : 4); }

template <int EPI>
__device__ void pass_phase_nn(const PassArgs& a, const double* Bsrc, int ma, double* smem,
                              int* colmap) {
  GemmArgs g = a.nn;
  g.B = Bsrc;
  const int fn = pass_fn(ma);
  const int mt = (a.n + 15) / 16;
  const int nt = (ma + 8 * fn - 1) / (8 * fn);
  for (int t = blockIdx.x; t < mt * nt; t += gridDim.x) {
    const int i = t % mt, j = t / mt;
    if (fn == 1)
      gemm_tile<false, 2, 1, EPI, kPassNW>(g, ma, i, j, 0, smem, colmap);
    else if (fn == 2)
      gemm_tile<false, 2, 2, EPI, kPassNW>(g, ma, i, j, 0, smem, colmap);
    else
      gemm_tile<false, 2, 4, EPI, kPassNW>(g, ma, i, j, 0, smem, colmap);
  }
}

// returns the split-K factor used (the consumers sum that many slabs)
__device__ inline int pass_phase_tn(const PassArgs& a, int ma, double* smem, int* colmap) {
  GemmArgs g = a.tn;
  const int fn = pass_fn(ma);
  const int mt = (a.p + 15) / 16;
  const int nt = (ma + 8 * fn - 1) / (8 * fn);
  const int nkt = (a.n + kBK - 1) / kBK;
  int nsplit = 1;  // same rule as the host planner (engine.cu, Engine::plan)
  while (nsplit < kMaxSplit && mt * nt * nsplit * 2 <= 2 * (int)gridDim.x && nkt >= nsplit * 4)
    nsplit *= 2;
  const int kt_per = (nkt + nsplit - 1) / nsplit;
  g.ksplit = kt_per * kBK;
  nsplit = (a.n + g.ksplit - 1) / g.ksplit;
  const int ntiles = mt * nt * nsplit;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int i = t % mt, rest = t / mt;
    const int j = rest % nt, s = rest / nt;
    if (fn == 1)
      gemm_tile<true, 2, 1, EPI_STORE, kPassNW>(g, ma, i, j, s, smem, colmap);
    else if (fn == 2)
      gemm_tile<true, 2, 2, EPI_STORE, kPassNW>(g, ma, i, j, s, smem, colmap);
    else
      gemm_tile<true, 2, 4, EPI_STORE, kPassNW>(g, ma, i, j, s, smem, colmap);
  }
  return nsplit;
}

// dynamic shared memory of k_pass
__host__ inline size_t pass_smem_bytes(int p, int n2, int E) {
  size_t b = column_smem_bytes(p, n2, E);
  const size_t g1 = GemmShape<false, 2, 4, kPassNW>::SMEM_BYTES;
  const size_t g2 = GemmShape<true, 2, 4, kPassNW>::SMEM_BYTES;
  if (g1 > b) b = g1;
  if (g2 > b) b = g2;
  return b;
}

__device__ __forceinline__ unsigned long long pass_clock() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// phase wall-time accumulation (tools/profile_solve.py; off in the product)
enum { PH_NN = 0, PH_TN, PH_PROX, PH_EVNN, PH_EVTN, PH_EVCOL, PH_COMPACT, PH_COUNT };

template <int E>
__global__ void __launch_bounds__(kPassThreads, 1) k_pass(PassArgs a) {
  extern __shared__ __align__(16) double smem[];
  __shared__ int colmap[32];
  cg::grid_group grid = cg::this_grid();
  RelaxDev r = a.r;
  int iter = 0, last_eval = 0, n_evals = 0;
  long long node_its = 0;
  int ma = *(volatile int*)r.d_ma;
  const bool prof = a.prof != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
  unsigned long long t_last = prof ? pass_clock() : 0ull;
  auto mark = [&](int ph) {
    if (prof) {
      const unsigned long long t = pass_clock();
      a.prof[ph] += t - t_last;
      t_last = t;
    }
  };

  auto evaluate = [&](int it) {  // relaxation.hpp:194-221
    pass_phase_nn<EPI_EVAL>(a, r.B, ma, smem, colmap);
    grid.sync();
    mark(PH_EVNN);
    r.nsplit = pass_phase_tn(a, ma, smem, colmap);
    grid.sync();
    mark(PH_EVTN);
    EvalArgs e;
    e.part_loss = a.nn.part_loss;
    e.part_conj = a.nn.part_conj;
    e.nrb = (a.n + 15) / 16;
    e.part_ld = a.nn.part_ld;
    e.iter = it;
    e.prune_threshold = a.prune_thr;
    e.gap_tolerance = a.gap_tol;
    e.trace = a.trace;
    e.eval_idx = n_evals;
    for (int c = blockIdx.x; c < ma; c += gridDim.x) eval_column<E>(r, e, c, smem);
    grid.sync();
    mark(PH_EVCOL);
    if (blockIdx.x == 0) compact_active<kPassThreads>(r.act, r.d_ma, r.frozen);
    grid.sync();
    mark(PH_COMPACT);
    ma = *(volatile int*)r.d_ma;
    // non-finite iterate (numeric_error, relaxation.hpp:76-81): stop early;
    // the host reports the column from d_err
    if (*(volatile int*)r.d_err != 0x7fffffff) ma = 0;
    ++n_evals;
  };

  while (iter < a.max_it && ma > 0) {  // relaxation.hpp:224-249
    ++iter;
    pass_phase_nn<EPI_DERIV>(a, r.V, ma, smem, colmap);
    grid.sync();
    mark(PH_NN);
    r.nsplit = pass_phase_tn(a, ma, smem, colmap);
    grid.sync();
    mark(PH_TN);
    for (int c = blockIdx.x; c < ma; c += gridDim.x) prox_column<E>(r, c, smem);
    grid.sync();
    mark(PH_PROX);
    node_its += ma;
    if (iter % a.check == 0) {
      evaluate(iter);
      last_eval = iter;
    }
  }
  if (ma > 0 && last_eval != iter) evaluate(iter);  // relaxation.hpp:250
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.out[0] = iter;
    a.out[1] = n_evals;
    a.out[2] = node_its;
  }
}

}  // namespace bnbg
