// pass_kernel.cuh -- the whole batched relaxation of one BnB pass as a single
// persistent cooperative kernel (solve_batch_relaxation, relaxation.hpp:163-255).
//
// At narrow frontiers (m_a columns << SMs x tiles) every iteration is a chain
// of three dependent, latency-bound steps: S = X V (+ l' epilogue), G = X'R,
// prox + FISTA.  Launching them as separate kernels costs a launch gap and a
// ramp/drain per step and a host round trip per check interval.  Here one
// CTA per SM loops over the iterations on the device:
//
//   phase NN   row tiles of X x active columns           -> R = l'(X V)
//   grid barrier
//   phase TN   column tiles of X x active columns x split-K -> G slabs
//   grid barrier
//   phase prox one CTA per active column                  -> B, V
//   grid barrier
//   every check_interval: NN(eval) / TN / per-column bounds / compaction,
//   with the active count read back on the device (no host round trip).
//
// Two operand modes:
//   resident (ResLayout.on): when X fits in the SMs' shared memory (c1, c2:
//     8 MB over 148 x 227 KB), CTA b loads its NN row tile and its TN tile of
//     X once per pass and keeps them for every iteration; an iteration then
//     only moves V / R chunks (cp.async, all k at once) and the DMMA fragments
//     come straight from shared memory.
//   streaming: X tiles are staged through a cp.async ring per iteration
//     (gemm_tile, the standalone kernels' code) -- c3/c4 sizes.
//
// The grid barrier is a monotone arrival counter: CTA leaders add with
// red.release.gpu and poll with ld.acquire.gpu until the epoch target, one
// L2 round trip less than an atomic-return barrier.
//
// The column phases (prox_column, eval_column, compact_active) are the
// standalone kernels' code, so results do not depend on the scheduling mode.
#pragma once
#include <cooperative_groups.h>

#include "gemm.cuh"
#include "gemm_big.cuh"
#include "launchers.hpp"
#include "node_kernels.cuh"

namespace bnbg {

constexpr int kPassThreads = kNodeThreads;  // 8 warps
constexpr int kPassNW = kPassThreads / 32;

__device__ __forceinline__ int pass_fn(int ma) { return ma <= 8 ? 1 : (ma <= 16 ? 2 : 4); }

__device__ __forceinline__ void grid_barrier(unsigned* ctr, unsigned& target, int cluster) {
  if (cluster) {  // one-cluster grid: the hardware cluster barrier (0.2 us vs 1.2 us)
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    return;
  }
  target += gridDim.x;
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(ctr) : "memory");
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(ctr) : "memory");
    } while ((int)(v - target) < 0);
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// streaming-mode phases
// ---------------------------------------------------------------------------
// streaming mode uses the register-tiled GEMM tiles for wide batches: 128 x 64
// from kBigNarrowMax active columns on, 128 x 32 below
#ifndef BNBG_NARROW_MAX
#define BNBG_NARROW_MAX 48
#endif
constexpr int kBigNarrowMax = BNBG_NARROW_MAX;
__device__ __forceinline__ bool pass_big(const PassArgs& a, int ma) {
  return a.big > 0 && ma >= a.big;
}

template <int EPI>
__device__ void pass_phase_nn(const PassArgs& a, const double* Bsrc, int ma, double* smem,
                              int* colmap, const int* act) {
  GemmArgs g = a.nn;
  g.B = Bsrc;
  g.act = act;
  if (pass_big(a, ma)) {
    auto* epi = reinterpret_cast<double(*)[4][kBigBN]>(smem + kBigSmemBytes / sizeof(double));
    const int mt = (a.n + kBigBM - 1) / kBigBM;
    if (ma >= kBigNarrowMax) {
      const int nt = (ma + kBigBN - 1) / kBigBN;
      for (int t = blockIdx.x; t < mt * nt; t += gridDim.x)
        gemm_big_tile<false, EPI, 64>(g, ma, t % mt, t / mt, smem, colmap, epi);
    } else {
      const int nt = (ma + 31) / 32;
      for (int t = blockIdx.x; t < mt * nt; t += gridDim.x)
        gemm_big_tile<false, EPI, 32>(g, ma, t % mt, t / mt, smem, colmap, epi);
    }
    return;
  }
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

// Gram form of the iteration gradient (squared loss): G = Q V - c over
// 16-row tiles of Q streamed from L2 (engine.hpp, gram_)
static __device__ void pass_phase_gram(const PassArgs& a, int ma, double* smem, int* colmap,
                                       const int* act) {
  GemmArgs g = a.gq;
  g.act = act;
  const int fn = pass_fn(ma);
  const int mt = (a.p + 15) / 16;
  const int nt = (ma + 8 * fn - 1) / (8 * fn);
  for (int t = blockIdx.x; t < mt * nt; t += gridDim.x) {
    const int i = t % mt, j = t / mt;
    if (fn == 1)
      gemm_tile<false, 2, 1, EPI_DERIV, kPassNW>(g, ma, i, j, 0, smem, colmap);
    else if (fn == 2)
      gemm_tile<false, 2, 2, EPI_DERIV, kPassNW>(g, ma, i, j, 0, smem, colmap);
    else
      gemm_tile<false, 2, 4, EPI_DERIV, kPassNW>(g, ma, i, j, 0, smem, colmap);
  }
}

// returns the split-K factor used (the consumers sum that many slabs)
__device__ inline int pass_phase_tn(const PassArgs& a, int ma, double* smem, int* colmap,
                                    const int* act) {
  GemmArgs g = a.tn;
  g.act = act;
  if (pass_big(a, ma)) {
    auto* epi = reinterpret_cast<double(*)[4][kBigBN]>(smem + kBigSmemBytes / sizeof(double));
    const int mt = (a.p + kBigBM - 1) / kBigBM;
    const int bn = ma >= kBigNarrowMax ? kBigBN : 32;
    const int nt = (ma + bn - 1) / bn;
    // split K until every CTA has a tile (c3: p / 128 = 16 row tiles)
    const int nkt = (a.n + kBigBK - 1) / kBigBK;
    int ns = 1;
    while (ns < kMaxSplit && mt * nt * ns < (int)gridDim.x && nkt >= 2 * ns * 32) ns *= 2;
    g.ksplit = ((nkt + ns - 1) / ns) * kBigBK;
    ns = (a.n + g.ksplit - 1) / g.ksplit;
    for (int t = blockIdx.x; t < mt * nt * ns; t += gridDim.x) {
      const int i = t % mt, rest = t / mt;
      if (bn == kBigBN)
        gemm_big_tile<true, EPI_STORE, 64>(g, ma, i, rest % nt, smem, colmap, epi, rest / nt);
      else
        gemm_big_tile<true, EPI_STORE, 32>(g, ma, i, rest % nt, smem, colmap, epi, rest / nt);
    }
    return ns;
  }
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

// dynamic shared memory of the streaming-mode k_pass
__host__ inline size_t pass_smem_bytes(int p, int n2, int E) {
  size_t b = column_smem_bytes(p, n2, E);
  const size_t g1 = GemmShape<false, 2, 4, kPassNW>::SMEM_BYTES;
  const size_t g2 = GemmShape<true, 2, 4, kPassNW>::SMEM_BYTES;
  const size_t g3 = kBigSmemBytes + sizeof(double) * 2 * 4 * kBigBN;  // big tiles + epilogue sums
  if (g1 > b) b = g1;
  if (g2 > b) b = g2;
  if (g3 > b) b = g3;
  return b;
}

// ---------------------------------------------------------------------------
// resident mode
// ---------------------------------------------------------------------------
constexpr int kResBM = 16;  // FM = 2

__host__ __device__ inline int ld_mod16_4(int v) {  // smallest >= v with (x % 16) == 4
  int x = (v + 3) & ~3;
  while (x % 16 != 4) x += 4;
  return x;
}

// work region: staged B chunk (up to 16 columns x ldb), reused afterwards for
// the cross-warp reduction (NW x 2 x FN x 64) and the l / l* staging (2 x 16 rt x 16)
__host__ __device__ inline size_t res_work_doubles(const ResLayout& r) {
  size_t b = (size_t)16 * r.ldb;
  const size_t red = (size_t)kPassNW * 2 * 2 * 64 + 2 * 16 * r.rt * 16;
  return b > red ? b : red;
}

// Loads this CTA's resident tiles of X (once per pass).
static __device__ void res_load_x(const PassArgs& a, double* smem) {
  const ResLayout& L = a.res;
  const double* X = a.nn.A;
  const int n = a.n, p = a.p;
  if ((int)blockIdx.x < L.nn_tiles) {
    const int bm = kResBM * L.rt;
    const int m0 = blockIdx.x * bm;
    double* A = smem;
    for (int e = threadIdx.x; e < L.kpad_nn * bm; e += kPassThreads) {
      const int k = e / bm, m = e % bm;
      A[k * L.lda_nn + m] = (k < p && m0 + m < n) ? X[(size_t)k * n + m0 + m] : 0.0;
    }
  }
  if ((int)blockIdx.x < L.tn_mt * L.tn_split) {
    const int i = blockIdx.x % L.tn_mt, sp = blockIdx.x / L.tn_mt;
    const int c0 = i * kResBM, r0 = sp * L.tn_klen;
    double* A = smem + L.off_tn;
    for (int e = threadIdx.x; e < kResBM * L.tn_klen; e += kPassThreads) {
      const int m = e / L.tn_klen, k = e % L.tn_klen;
      const int row = r0 + k;
      A[m * L.ldk_tn + k] = (c0 + m < p && row < n) ? X[(size_t)(c0 + m) * n + row] : 0.0;
    }
  }
  __syncthreads();
}

// One output tile (16 RT rows x 8*FN compact columns starting at n0) from the
// resident A operand: NN  A[k*lda + m] (K = kpad_nn), TN  A[m*lda + k] (K = tn_klen).
// B chunk: column c at g.B + col*g.ldb + kbeg, kvalid valid rows (rest zero).
// RT 16-row sub-tiles share the staged B chunk; warp w computes sub-tile
// w % RT over the k-steps w / RT (mod NW / RT).
template <bool TN, int FN, int EPI, int RT = 1>
__device__ void res_tile(const GemmArgs& g, const double* Ares, int lda, int K, int kbeg,
                         int kvalid, int m0, int mt, int n0, int ncols, int split, double* work,
                         int ldb, int* colmap) {
  constexpr int FM = 2, BM = 16 * RT, BN = 8 * FN, NW = kPassNW, NT = kPassThreads, KW = NW / RT;
  static_assert(!TN || RT == 1, "TN tiles are 16 columns of X");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int sub = warp % RT, kw = warp / RT;
  ColProbe pr(g.probe);
  if (tid < BN) {
    const int c = n0 + tid;
    colmap[tid] = c < ncols ? (g.act ? g.act[c] : c) : -1;
  }
  __syncthreads();
  double* Bs = work;
  // B chunk: 16-byte copies when the rows are 16-byte aligned (even ld and
  // offset), else 8-byte; rows past kvalid are zero-filled
  if (((g.ldb | kbeg) & 1) == 0 && ((reinterpret_cast<size_t>(g.B) & 15) == 0)) {
    // NT / BN threads per column: no integer division in the issue loop
    constexpr int TPC = NT / BN;
    const int K2 = K >> 1;
    const int c = tid / TPC, col = colmap[c];
    const double* src = col >= 0 ? g.B + (size_t)col * g.ldb + kbeg : g.B;
    double* dst = Bs + c * ldb;
    for (int k2 = tid % TPC; k2 < K2; k2 += TPC) {
      const int k = 2 * k2;
      const int nb = col < 0 ? 0 : (k + 2 <= kvalid ? 16 : (k < kvalid ? 8 : 0));
      cp_async_16(dst + k, nb ? src + k : g.B, nb);
    }
  } else {
    for (int c = 0; c < BN; ++c) {
      const int col = colmap[c];
      const double* src = col >= 0 ? g.B + (size_t)col * g.ldb + kbeg : g.B;
      for (int k = tid; k < K; k += NT) {
        const bool valid = col >= 0 && k < kvalid;
        cp_async_8(Bs + c * ldb + k, valid ? src + k : g.B, valid);
      }
    }
  }
  cp_async_commit();
  pr.mark(0);
  cp_async_wait<0>();
  __syncthreads();
  pr.mark(1);
  // two accumulator sets (even / odd k-steps of the warp) halve the DMMA
  // dependency chain; they are added in a fixed order afterwards
  double acc[2][FM][FN][2];
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
      for (int j = 0; j < FN; ++j) acc[u][i][j][0] = acc[u][i][j][1] = 0.0;
  const int nks = K >> 2;
  auto kstep = [&](int u, int ks) {
    const int kk = ks * 4 + (lane & 3);
    double av[FM], bv[FN];
#pragma unroll
    for (int i = 0; i < FM; ++i) {
      const int row = sub * 16 + i * 8 + (lane >> 2);
      av[i] = TN ? Ares[row * lda + kk] : Ares[kk * lda + row];
    }
#pragma unroll
    for (int j = 0; j < FN; ++j) bv[j] = Bs[(j * 8 + (lane >> 2)) * ldb + kk];
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
      for (int j = 0; j < FN; ++j) dmma_8x8x4(acc[u][i][j][0], acc[u][i][j][1], av[i], bv[j]);
  };
  int ks = kw;
  for (; ks + KW < nks; ks += 2 * KW) {
    kstep(0, ks);
    kstep(1, ks + KW);
  }
  if (ks < nks) kstep(0, ks);
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) {
      acc[0][i][j][0] += acc[1][i][j][0];
      acc[0][i][j][1] += acc[1][i][j][1];
    }
  __syncthreads();  // Bs consumed: the work region becomes the reduction buffer
  pr.mark(2);
  double* red = work;
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) red[((warp * FM + i) * FN + j) * 64 + h * 32 + lane] = acc[0][i][j][h];
  __syncthreads();
  double* lv = work + NW * FM * 2 * 64;
  double* cv = lv + BM * BN;
  double* Cout = g.C + (size_t)split * g.split_stride;
  for (int e = tid; e < BM * BN; e += NT) {
    const int c = e / BM, r = e % BM;
    const int rs = r >> 4, rr = r & 15;
    const int i = rr >> 3, j = c >> 3;
    const int ln = (rr & 7) * 4 + ((c & 7) >> 1), h = c & 1;
    constexpr int stride_w = FM * FN * 64;
    const int off = (i * FN + j) * 64 + h * 32 + ln + rs * stride_w;
    double s = red[off];
#pragma unroll
    for (int w = 1; w < KW; ++w) s += red[off + w * RT * stride_w];
    const int gm = m0 + r;
    const int col = colmap[c];
    if (EPI == EPI_STORE) {
      if (gm < g.M && col >= 0) Cout[(size_t)col * g.ldc + gm] = s;
    } else {
      double rv = 0.0, l = 0.0, cj = 0.0;
      if (gm < g.M && col >= 0) {
        const double yv = g.y[gm];
        rv = d_loss_deriv(g.loss, s, yv);
        Cout[(size_t)col * g.ldc + gm] = rv;
        if (EPI == EPI_EVAL) {
          l = d_loss_value(g.loss, s, yv);
          cj = d_loss_conj(g.loss, rv, yv);
        }
      }
      if (EPI == EPI_EVAL) {
        lv[c * BM + r] = l;
        cv[c * BM + r] = cj;
      }
    }
  }
  if (EPI == EPI_EVAL) {
    __syncthreads();
    if (tid < BN && colmap[tid] >= 0) {
      double sl = 0.0, sc = 0.0;
      for (int r = 0; r < BM; ++r) {
        sl += lv[tid * BM + r];
        sc += cv[tid * BM + r];
      }
      g.part_loss[(size_t)mt * g.part_ld + colmap[tid]] = sl;
      g.part_conj[(size_t)mt * g.part_ld + colmap[tid]] = sc;
    }
  }
  __syncthreads();
  pr.mark(3);
}

template <int EPI>
__device__ void res_phase_nn(const PassArgs& a, const double* Bsrc, int ma, double* smem,
                             int* colmap, const int* act) {
  const ResLayout& L = a.res;
  if ((int)blockIdx.x >= L.nn_tiles) return;
  GemmArgs g = a.nn;
  g.B = Bsrc;
  g.act = act;
  double* work = smem + L.off_work;
  const int m0 = blockIdx.x * kResBM * L.rt;
  for (int n0 = 0; n0 < ma; n0 += 16) {
    if (L.rt == 4) {
      if (ma - n0 > 8)
        res_tile<false, 2, EPI, 4>(g, smem, L.lda_nn, L.kpad_nn, 0, a.p, m0, blockIdx.x, n0, ma,
                                   0, work, L.ldb, colmap);
      else
        res_tile<false, 1, EPI, 4>(g, smem, L.lda_nn, L.kpad_nn, 0, a.p, m0, blockIdx.x, n0, ma,
                                   0, work, L.ldb, colmap);
    } else if (ma - n0 > 8) {
      res_tile<false, 2, EPI>(g, smem, L.lda_nn, L.kpad_nn, 0, a.p, m0, blockIdx.x, n0, ma, 0,
                              work, L.ldb, colmap);
    } else {
      res_tile<false, 1, EPI>(g, smem, L.lda_nn, L.kpad_nn, 0, a.p, m0, blockIdx.x, n0, ma, 0,
                              work, L.ldb, colmap);
    }
  }
}

static __device__ void res_phase_tn(const PassArgs& a, int ma, double* smem, int* colmap,
                             const int* act) {
  const ResLayout& L = a.res;
  if ((int)blockIdx.x >= L.tn_mt * L.tn_split) return;
  GemmArgs g = a.tn;
  g.act = act;
  double* work = smem + L.off_work;
  const int i = blockIdx.x % L.tn_mt, sp = blockIdx.x / L.tn_mt;
  const int r0 = sp * L.tn_klen;
  const int kvalid = min(L.tn_klen, a.n - r0);
  for (int n0 = 0; n0 < ma; n0 += 16) {
    if (ma - n0 > 8)
      res_tile<true, 2, EPI_STORE>(g, smem + L.off_tn, L.ldk_tn, L.tn_klen, r0, kvalid,
                                   i * kResBM, i, n0, ma, sp, work, L.ldb, colmap);
    else
      res_tile<true, 1, EPI_STORE>(g, smem + L.off_tn, L.ldk_tn, L.tn_klen, r0, kvalid,
                                   i * kResBM, i, n0, ma, sp, work, L.ldb, colmap);
  }
}

__device__ __forceinline__ unsigned long long pass_clock() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// phase wall-time accumulation (tools/pass_phases.py; off in the product)
enum { PH_NN = 0, PH_TN, PH_PROX, PH_EVNN, PH_EVTN, PH_EVCOL, PH_COMPACT, PH_COUNT };

constexpr int kActCache = 256;

template <int E>
__global__ void __launch_bounds__(kPassThreads, 1) k_pass(const __grid_constant__ PassArgs a) {
  extern __shared__ __align__(128) double smem[];
  __shared__ int colmap[kBigBN];  // column map of the current GEMM tile (<= 64 columns)
  __shared__ int s_act[kActCache];  // the active list, refreshed after every compaction
  const RelaxDev& r = a.r;  // kernel-parameter space (no local copy)
  int nsplit = 1;            // split-K slabs of the current G
  const bool res = a.res.on != 0;
  double* colsm = res ? smem + a.res.off_work : smem;  // column phases' shared memory
  int iter = 0, last_eval = 0, n_evals = 0;
  long long node_its = 0;
  unsigned bar_target = 0;
  if (res) res_load_x(a, smem);
  else if (a.nn.tmap) gemm_big_tma_init();
  int ma = 0;
  const int* actp = r.act;
  // CTA c owns active column c between compactions: its B, V, states in
  // shared memory (ColCache), refreshed from global after every evaluation
  ColCache cc;
  bool cached = false;
  // local-Gram region (a.gram_local > 0): Q [p*p] c [p] G [p] | B [p] V [p] states [p]
  double* gl = (E == 1 && a.gram_local > 0) ? smem + a.gram_local : nullptr;
  const bool can_cache = (res && E != 0 && a.res.off_cc > 0) || (E != 0 && gl != nullptr);
  auto refresh = [&]() {
    ma = *(volatile int*)r.d_ma;
    for (int i = threadIdx.x; i < ma && i < kActCache; i += kPassThreads) s_act[i] = r.act[i];
    __syncthreads();
    actp = ma <= kActCache ? s_act : r.act;
    cached = can_cache && ma <= (int)gridDim.x && (int)blockIdx.x < ma;
    if (cached) {
      const int p = r.p;
      const int b = actp[blockIdx.x];
      cc.b = b;
      cc.kb = r.kbar[b];
      cc.pf = r.pf[b];
      cc.t = r.t[b];
      cc.B = gl ? gl + (size_t)p * p + 2 * p : smem + a.res.off_cc;
      cc.V = cc.B + p;
      uint8_t* stc = reinterpret_cast<uint8_t*>(cc.V + p);
      cc.st = stc;
      for (int j = threadIdx.x; j < p; j += kPassThreads) {
        cc.B[j] = r.B[(size_t)b * p + j];
        cc.V[j] = r.V[(size_t)b * p + j];
        stc[j] = r.state[(size_t)b * p + j];
      }
      __syncthreads();
    }
  };
  if (gl) {  // Q and c, once per launch
    const int p = r.p;
    for (int e = threadIdx.x; e < p * p; e += kPassThreads) gl[e] = a.gq.A[e];
    for (int j = threadIdx.x; j < p; j += kPassThreads) gl[(size_t)p * p + j] = a.gram_c[j];
    __syncthreads();
  }
  refresh();
  const bool prof = a.prof != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
  unsigned long long t_last = prof ? pass_clock() : 0ull;
  auto mark = [&](int ph) {  // phase end (after its grid barrier)
    if (prof) {
      const unsigned long long t = pass_clock();
      atomicAdd(a.prof + ph, t - t_last);  // RED: no load on CTA 0's path
      t_last = t;
    }
  };
  auto arrive = [&](int ph) {  // CTA 0 reaches the phase's barrier
    if (prof) atomicAdd(a.prof + 8 + ph, pass_clock() - t_last);
  };
  auto phase_nn = [&](const double* src, bool eval) {
    if (res) {
      if (eval)
        res_phase_nn<EPI_EVAL>(a, src, ma, smem, colmap, actp);
      else
        res_phase_nn<EPI_DERIV>(a, src, ma, smem, colmap, actp);
    } else {
      if (eval)
        pass_phase_nn<EPI_EVAL>(a, src, ma, smem, colmap, actp);
      else
        pass_phase_nn<EPI_DERIV>(a, src, ma, smem, colmap, actp);
    }
  };
  auto phase_tn = [&]() {
    if (res) {
      res_phase_tn(a, ma, smem, colmap, actp);
      return a.res.tn_split;
    }
    return pass_phase_tn(a, ma, smem, colmap, actp);
  };

  auto evaluate = [&](int it) {  // relaxation.hpp:194-221
    phase_nn(r.B, true);
    arrive(PH_EVNN);
    grid_barrier(a.bar, bar_target, a.res.cluster);
    mark(PH_EVNN);
    nsplit = phase_tn();
    arrive(PH_EVTN);
    grid_barrier(a.bar, bar_target, a.res.cluster);
    mark(PH_EVTN);
    EvalArgs e;
    e.part_loss = a.nn.part_loss;
    e.part_conj = a.nn.part_conj;
    e.nrb = res ? a.res.nn_tiles : (pass_big(a, ma) ? (a.n + kBigBM - 1) / kBigBM : (a.n + 15) / 16);
    e.part_ld = a.nn.part_ld;
    e.iter = it;
    e.prune_threshold = a.prune_thr;
    e.gap_tolerance = a.gap_tol;
    e.trace = a.trace;
    e.eval_idx = n_evals;
    if (cached)
      eval_column_impl<E, true>(r, nsplit, e, blockIdx.x, colsm, cc);
    else
      for (int c = blockIdx.x; c < ma; c += gridDim.x) eval_column<E>(r, nsplit, e, c, colsm);
    arrive(PH_EVCOL);
    grid_barrier(a.bar, bar_target, a.res.cluster);
    mark(PH_EVCOL);
    if (blockIdx.x == 0) compact_active<kPassThreads>(r.act, r.d_ma, r.frozen);
    arrive(PH_COMPACT);
    grid_barrier(a.bar, bar_target, a.res.cluster);
    mark(PH_COMPACT);
    refresh();
    // non-finite iterate (numeric_error, relaxation.hpp:76-81): stop early;
    // the host reports the column from d_err
    if (*(volatile int*)r.d_err != 0x7fffffff) ma = 0;
    ++n_evals;
  };

  while (iter < a.max_it && ma > 0) {  // relaxation.hpp:224-249
    if (E == 1 && gl && ma <= (int)gridDim.x) {  // p <= 128 implies E == 1
      // local Gram iterations up to the next evaluation: the CTA owning a
      // column forms G = Q V - c from shared memory (thread j: row j, k in
      // order) and runs the prox on it; no other CTA is involved
      const int nloc = min(a.check - iter % a.check, a.max_it - iter);
      if (cached) {
        const int p = r.p;
        const double* Qs = gl;
        const double* cs = gl + (size_t)p * p;
        double* Gs = gl + (size_t)p * p + p;
        RelaxDev rl = r;  // gsum(rl, 1, b, j) reads Gs[j]
        rl.G = Gs - (size_t)cc.b * p;
        rl.nsplit = 1;
        rl.split_stride = 0;
        for (int s2 = 0; s2 < nloc; ++s2) {
          {
            // p <= 128: thread t takes row t % 128 over the k half t / 128,
            // two independent chains each; the halves and chains are added
            // in a fixed order
            const int j = threadIdx.x & 127, h = threadIdx.x >> 7;
            const int kh = (p + 1) >> 1, kb = h * kh, ke = min(p, kb + kh);
            double a0 = 0.0, a1 = 0.0;
            if (j < p) {
              const double* qj = Qs + j;
              int k2 = kb;
              for (; k2 + 8 <= ke; k2 += 8) {  // 16 loads in flight, then the FMAs
                double q[8], vv[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                  q[u] = qj[(size_t)(k2 + u) * p];
                  vv[u] = cc.V[k2 + u];
                }
#pragma unroll
                for (int u = 0; u < 8; u += 2) {
                  a0 += q[u] * vv[u];
                  a1 += q[u + 1] * vv[u + 1];
                }
              }
              for (; k2 + 2 <= ke; k2 += 2) {
                a0 += qj[(size_t)k2 * p] * cc.V[k2];
                a1 += qj[(size_t)(k2 + 1) * p] * cc.V[k2 + 1];
              }
              if (k2 < ke) a0 += qj[(size_t)k2 * p] * cc.V[k2];
            }
            if (h == 1 && j < p) Gs[j] = a0 + a1;  // upper half's partial
            __syncthreads();
            if (h == 0 && j < p) Gs[j] = ((a0 + a1) + Gs[j]) - cs[j];  // l' of the squared loss
          }
          __syncthreads();
          cc.t = prox_column_impl<E, true>(rl, 1, blockIdx.x, colsm, cc);
        }
      }
      iter += nloc;
      node_its += (long long)ma * nloc;
      arrive(PH_PROX);
      grid_barrier(a.bar, bar_target, a.res.cluster);
      mark(PH_PROX);
      if (iter % a.check == 0) {
        evaluate(iter);
        last_eval = iter;
      }
      continue;
    }
    ++iter;
    if (a.gram && !res) {  // one product: G = Q V - c (resident mode keeps the X form)
      pass_phase_gram(a, ma, smem, colmap, actp);
      nsplit = 1;
      arrive(PH_TN);
      grid_barrier(a.bar, bar_target, a.res.cluster);
      mark(PH_TN);
    } else {
      phase_nn(r.V, false);
      arrive(PH_NN);
      grid_barrier(a.bar, bar_target, a.res.cluster);
      mark(PH_NN);
      nsplit = phase_tn();
      arrive(PH_TN);
      grid_barrier(a.bar, bar_target, a.res.cluster);
      mark(PH_TN);
    }
    if (cached)
      cc.t = prox_column_impl<E, true>(r, nsplit, blockIdx.x, colsm, cc);
    else
      for (int c = blockIdx.x; c < ma; c += gridDim.x) prox_column<E>(r, nsplit, c, colsm);
    arrive(PH_PROX);
    grid_barrier(a.bar, bar_target, a.res.cluster);
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
