// gemm_big.cuh -- register-tiled DMMA GEMM for wide batches (c3/c4 widths).
//
// Same contractions and epilogues as gemm.cuh (S = X V[:,act] with l', eval
// sums; G = X' R[:,act]), for m_a >= 64 active columns where the split-K
// kernel's cross-warp reductions cost more than they hide:
//   CTA tile 128 x 64, 8 warps in a 4 (M) x 2 (N) grid, warp tile 32 x 32
//   (4 x 4 DMMA.8x8x4 fragments, 16 independent accumulators per lane),
//   BK = 16 (four k-steps) staged through a 3-deep ring (90 KB: two CTAs,
//   16 warps per SM).
// Staging: the X tile of a stage (the A operand, 2/3 of the bytes) is one
// TMA box (cp.async.bulk.tensor.2d, UTMALDG) completing on the stage's
// mbarrier; the box is 4 elements wider than the tile so the shared-memory
// rows land on the conflict-free (= 4 mod 16 doubles) stride the fragment
// loads need, and TMA zero-fills past n and p.  The B operand (columns
// gathered through the active list) is cp.async 16-byte chunks.
// TN (G = X' R) splits K over blockIdx.z when the tiles alone leave SMs
// idle (c4: p / 128 = 40 row tiles); slab s holds rows [s*ksplit, ...) and
// the consumers sum the slabs in order.
// Every output element is accumulated by one lane in k order, so results are
// deterministic.  Needs n and p even (16-byte rows).
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

// TMA boxes (elements, innermost first) of X = n x p column-major:
//   NN  A(m, k) = X[k*n + m0 + m], stored [k][kBigLDA_NN]: box {kBigLDA_NN, kBigBK}
//   TN  A(m, k) = X[(m0+m)*n + k0 + k], stored [m][kBigLDK]: box {kBigLDK, kBigBM}
constexpr int kBigBoxNN0 = kBigLDA_NN, kBigBoxNN1 = kBigBK;
constexpr int kBigBoxTN0 = kBigLDK, kBigBoxTN1 = kBigBM;
constexpr unsigned kBigTxNN = sizeof(double) * kBigBoxNN0 * kBigBoxNN1;
constexpr unsigned kBigTxTN = sizeof(double) * kBigBoxTN0 * kBigBoxTN1;
static_assert(kBigBoxNN0 * kBigBoxNN1 <= kBigA && kBigBoxTN0 * kBigBoxTN1 <= kBigA, "box fits");
static_assert((kBigStage * sizeof(double)) % 128 == 0, "TMA destinations 128-byte aligned");

// one mbarrier per ring stage and the parity of each (bit s), per CTA
static __shared__ __align__(8) unsigned long long s_big_bar[kBigNS];
static __shared__ unsigned s_big_phase;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// Once per CTA before the first gemm_big_tile of a kernel (all threads call).
__device__ __forceinline__ void gemm_big_tma_init() {
  if (threadIdx.x == 0) {
    for (int s = 0; s < kBigNS; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&s_big_bar[s])));
    s_big_phase = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
}

__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int c0, int c1,
                                            unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// One 128 x BN output tile (row tile mt, column tile nt), BN = 64 (warp tile
// 32 x 32) or 32 (warp tile 32 x 16, for narrower batches).  All 256 threads
// of the CTA call; smem holds kBigSmemBytes; colmap kBigBN ints and epi_red
// 2 x 4 x kBigBN doubles of shared memory.  Ends with a block barrier.
template <bool TN, int EPI, int BN = kBigBN>
__device__ void gemm_big_tile(const GemmArgs& g, int ncols, int mt, int nt, double* smem,
                              int* colmap, double (*epi_red)[4][kBigBN], int split = 0) {
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
  // K range of this split (ksplit is a multiple of kBigBK: no stage straddles
  // two splits, so the zero-fill at K covers the last one)
  const int kbeg = TN ? split * g.ksplit : 0;
  const int K = TN ? min(g.K, kbeg + g.ksplit) : g.K;
  const int nkt = (K - kbeg + kBigBK - 1) / kBigBK;
  const bool tma = g.tmap != nullptr;
  unsigned phase = s_big_phase;

  auto load_stage = [&](int stage, int kt) {
    double* As = smem + stage * kBigStage;
    double* Bs = As + kBigA;
    const int k0 = kbeg + kt * kBigBK;
    constexpr int KC = kBigBK / 2;  // 16-byte chunks per k-row (TN) ...
    constexpr int MC = kBigBM / 2;  // ... and per m-row (NN)
    if (tma) {
      if (threadIdx.x == 0) {
        // the stage's previous contents were read by the generic proxy
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (TN)
          tma_load_2d(As, g.tmap, k0, m0, &s_big_bar[stage], kBigTxTN);
        else
          tma_load_2d(As, g.tmap, m0, k0, &s_big_bar[stage], kBigTxNN);
      }
    } else {
    // A: 128 x BK doubles in 16-byte chunks
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
    if (tma) {
      const int st = kt % kBigNS;
      mbar_wait(&s_big_bar[st], (phase >> st) & 1u);
      phase ^= 1u << st;
    }
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
          g.C[(size_t)split * g.split_stride + (size_t)col * g.ldc + gm] = s;
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
  if (tid == 0) s_big_phase = phase;
  __syncthreads();  // smem / colmap reusable by the caller's next tile
}

template <bool TN, int EPI>
__global__ void __launch_bounds__(kBigThreads, 2) k_gemm_big(const __grid_constant__ GemmArgs g) {
  extern __shared__ __align__(128) double smem[];
  __shared__ int colmap[kBigBN];
  __shared__ double epi_red[2][4][kBigBN];  // EVAL: per-warp-row column sums (l, l*)
  // blockIdx.x walks the column tiles of one row tile, so the CTAs sharing an
  // X tile run together and all but one read it from L2
  const int ncols = *g.d_ncols;
  if ((int)blockIdx.x * kBigBN >= ncols) return;
  if (g.tmap) gemm_big_tma_init();
  gemm_big_tile<TN, EPI>(g, ncols, blockIdx.y, blockIdx.x, smem, colmap, epi_red, blockIdx.z);
}

}  // namespace bnbg
