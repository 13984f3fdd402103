// gemm_big.cuh -- register-tiled DMMA GEMM for wide batches (c3/c4 widths).
//
// Same contractions and epilogues as gemm.cuh (S = X V[:,act] with l', eval
// sums; G = X' R[:,act]), for m_a >= 64 active columns where the split-K
// kernel's cross-warp reductions cost more than they hide:
//   CTA tile 128 x 64, 8 warps in a 4 (M) x 2 (N) grid, warp tile 32 x 32
//   (4 x 4 DMMA.8x8x4 fragments, 16 independent accumulators per lane),
//   BK = 16 (four k-steps) staged through a 3-deep 16-byte cp.async ring
//   (90 KB: two CTAs, 16 warps per SM).
// Every output element is accumulated by one lane in k order, so results are
// deterministic.  Shared-memory strides are = 4 (mod 16) doubles, which makes
// the fragment loads conflict-free.  Needs n and p even (16-byte rows).
#pragma once
#include "gemm.cuh"

namespace bnbg {

constexpr int kBigThreads = 256;
#ifndef BNBG_BIG_BK
#define BNBG_BIG_BK 16
#endif
#ifndef BNBG_BIG_NS
#define BNBG_BIG_NS 3
#endif
constexpr int kBigBM = 128, kBigBN = 64, kBigBK = BNBG_BIG_BK, kBigNS = BNBG_BIG_NS;
constexpr int kBigLDA_NN = kBigBM + 4;  // NN A tile stored [k][m]
constexpr int kBigLDK = kBigBK + 4;     // [m][k] / [n][k] tiles
constexpr int kBigA = kBigBK * kBigLDA_NN > kBigBM * kBigLDK ? kBigBK * kBigLDA_NN : kBigBM * kBigLDK;
constexpr int kBigB = kBigBN * kBigLDK;
constexpr int kBigStage = kBigA + kBigB;
constexpr size_t kBigSmemBytes = sizeof(double) * (size_t)kBigNS * kBigStage;

// One 128 x BN output tile (row tile mt, column tile nt), BN = 64 (warp tile
// 32 x 32) or 32 (warp tile 32 x 16, for narrower batches).  All 256 threads
// of the CTA call; smem holds kBigSmemBytes; colmap kBigBN ints and epi_red
// 2 x 4 x kBigBN doubles of shared memory.  Ends with a block barrier.
template <bool TN, int EPI, int BN = kBigBN>
__device__ void gemm_big_tile(const GemmArgs& g, int ncols, int mt, int nt, double* smem,
                              int* colmap, double (*epi_red)[4][kBigBN]) {
  static_assert(BN == 64 || BN == 32, "BN");
  constexpr int FN = BN / 16, WN = BN / 2;  // fragments and columns per warp
  const int n0 = nt * BN;
  const int m0 = mt * kBigBM;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 3, wn = warp >> 2;
  if (tid < BN) {
    const int c = n0 + tid;
    colmap[tid] = c < ncols ? (g.act ? g.act[c] : c) : -1;
  }
  __syncthreads();
  const int K = g.K;
  const int nkt = (K + kBigBK - 1) / kBigBK;

  auto load_stage = [&](int stage, int kt) {
    double* As = smem + stage * kBigStage;
    double* Bs = As + kBigA;
    const int k0 = kt * kBigBK;
    // A: 128 x BK doubles in 16-byte chunks
    constexpr int KC = kBigBK / 2;  // chunks per k-row (TN) ...
    constexpr int MC = kBigBM / 2;  // ... and per m-row (NN)
#pragma unroll
    for (int it = 0; it < kBigBM * kBigBK / 2 / kBigThreads; ++it) {
      const int e = tid + it * kBigThreads;
      if (TN) {  // A(m, k) = X[(m0+m)*n + k0 + k], contiguous in k; stored [m][k]
        const int m = e / KC, kc = (e % KC) * 2;
        const int gm = m0 + m, gk = k0 + kc;
        const bool ok = gm < g.M && gk < K;
        cp_async_16(As + m * kBigLDK + kc, ok ? g.A + (size_t)gm * g.lda + gk : g.A, ok ? 16 : 0);
      } else {   // A(m, k) = X[(k0+k)*n + m0 + m], contiguous in m; stored [k][m]
        const int k = e / MC, mc = (e % MC) * 2;
        const int gm = m0 + mc, gk = k0 + k;
        const bool ok = gm < g.M && gk < K;
        cp_async_16(As + k * kBigLDA_NN + mc, ok ? g.A + (size_t)gk * g.lda + gm : g.A, ok ? 16 : 0);
      }
    }
    // B: BN columns x BK
#pragma unroll
    for (int it = 0; it < (BN * kBigBK / 2 + kBigThreads - 1) / kBigThreads; ++it) {
      const int e = tid + it * kBigThreads;
      if (e >= BN * KC) break;
      const int c = e / KC, kc = (e % KC) * 2;
      const int col = colmap[c];
      const int gk = k0 + kc;
      const bool ok = col >= 0 && gk < K;
      cp_async_16(Bs + c * kBigLDK + kc, ok ? g.B + (size_t)col * g.ldb + gk : g.B, ok ? 16 : 0);
    }
  };

  double acc[4][FN][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < kBigNS - 1; ++s) {
    if (s < nkt) load_stage(s, s);
    cp_async_commit();
  }
  for (int kt = 0; kt < nkt; ++kt) {
    cp_async_wait<kBigNS - 2>();
    __syncthreads();
    if (kt + kBigNS - 1 < nkt) load_stage((kt + kBigNS - 1) % kBigNS, kt + kBigNS - 1);
    cp_async_commit();
    const double* As = smem + (kt % kBigNS) * kBigStage;
    const double* Bs = As + kBigA;
#pragma unroll
    for (int ks = 0; ks < kBigBK / 4; ++ks) {
      const int kk = ks * 4 + (lane & 3);
      double a[4], b[FN];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int row = wm * 32 + i * 8 + (lane >> 2);
        a[i] = TN ? As[row * kBigLDK + kk] : As[kk * kBigLDA_NN + row];
      }
#pragma unroll
      for (int j = 0; j < FN; ++j) b[j] = Bs[(wn * WN + j * 8 + (lane >> 2)) * kBigLDK + kk];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  cp_async_wait<0>();

  // epilogue: lane holds D[row][col] for row = wm*32 + i*8 + lane/4 and
  // col = wn*32 + j*8 + 2*(lane%4) + h
  double lsum[FN][2], csum[FN][2];
#pragma unroll
  for (int j = 0; j < FN; ++j) lsum[j][0] = lsum[j][1] = csum[j][0] = csum[j][1] = 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + wm * 32 + i * 8 + (lane >> 2);
    const double yv = (EPI != EPI_STORE && gm < g.M) ? g.y[gm] : 0.0;
#pragma unroll
    for (int j = 0; j < FN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = wn * WN + j * 8 + (lane & 3) * 2 + h;
        const int col = colmap[c];
        if (gm >= g.M || col < 0) continue;
        const double s = acc[i][j][h];
        if (EPI == EPI_STORE) {
          g.C[(size_t)col * g.ldc + gm] = s;
        } else {
          const double rv = d_loss_deriv(g.loss, s, yv);
          g.C[(size_t)col * g.ldc + gm] = rv;
          if (EPI == EPI_EVAL) {
            lsum[j][h] += d_loss_value(g.loss, s, yv);
            csum[j][h] += d_loss_conj(g.loss, rv, yv);
          }
        }
      }
  }
  if (EPI == EPI_EVAL) {
    // column sums over the CTA's 128 rows: lanes sharing lane%4 (8 rows each),
    // then the 4 warp rows in order
#pragma unroll
    for (int j = 0; j < FN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
          lsum[j][h] += __shfl_xor_sync(0xffffffffu, lsum[j][h], o);
          csum[j][h] += __shfl_xor_sync(0xffffffffu, csum[j][h], o);
        }
    if (lane < 4) {
#pragma unroll
      for (int j = 0; j < FN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = wn * WN + j * 8 + lane * 2 + h;
          epi_red[0][wm][c] = lsum[j][h];
          epi_red[1][wm][c] = csum[j][h];
        }
    }
    __syncthreads();
    if (tid < BN && colmap[tid] >= 0) {
      double sl = 0.0, sc = 0.0;
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        sl += epi_red[0][w][tid];
        sc += epi_red[1][w][tid];
      }
      g.part_loss[(size_t)mt * g.part_ld + colmap[tid]] = sl;
      g.part_conj[(size_t)mt * g.part_ld + colmap[tid]] = sc;
    }
  }
  __syncthreads();  // smem / colmap reusable by the caller's next tile
}

template <bool TN, int EPI>
__global__ void __launch_bounds__(kBigThreads, 2) k_gemm_big(GemmArgs g) {
  extern __shared__ __align__(16) double smem[];
  __shared__ int colmap[kBigBN];
  __shared__ double epi_red[2][4][kBigBN];  // EVAL: per-warp-row column sums (l, l*)
  const int ncols = *g.d_ncols;
  if ((int)blockIdx.y * kBigBN >= ncols) return;
  gemm_big_tile<TN, EPI>(g, ncols, blockIdx.x, blockIdx.y, smem, colmap, epi_red);
}

}  // namespace bnbg
