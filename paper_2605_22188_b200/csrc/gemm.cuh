// gemm.cuh -- the batched FP64 contractions of the relaxation on DMMA.
//
//   NN:  S = X * V[:, act]   (n x m_a), epilogue R = l'(S)        relaxation.hpp:82-92
//        (eval mode also reduces sum l(S) and sum l*(R) per column) relaxation.hpp:108-147
//   TN:  G = X' * R[:, act]  (p x m_a), split-K partial slabs      relaxation.hpp:102, :132
//
// X stays resident in HBM/L2 in its reference column-major layout; columns
// of the batch are gathered through the active list `act` (frozen columns are
// compacted out, which leaves every active column's arithmetic unchanged --
// each output column is a function of its own input column only).
//
// Tiling: a CTA of NW warps owns a BM x BN output tile (BM = 8*FM, BN = 8*FN)
// and the warps split the K dimension (k-steps interleaved inside each BK=64
// stage), so small batches still put every warp on the DMMA pipe.  Stages are
// filled by cp.async (zero-fill at the edges) NS deep; partial accumulators
// are combined in a fixed warp order (deterministic), then the fused epilogue
// runs.  gemm_tile() is shared by the standalone kernels (4 warps) and the
// persistent pass kernel (8 warps).
#pragma once
#include "device_math.cuh"

namespace bnbg {

enum { EPI_STORE = 0, EPI_DERIV = 1, EPI_EVAL = 2 };

struct GemmArgs {
  int M, K;              // output rows, reduction length
  const double* A;       // X (n x p col-major)
  int lda;               // n
  const double* B;       // input block, column c at B + col*ldb
  int ldb;
  double* C;             // output block, column c at C + col*ldc (+ split slab)
  int ldc;
  long long split_stride;  // elements between split-K slabs of C
  int ksplit;            // K range per split (multiple of BK)
  const int* act;        // compact -> physical column (nullptr: identity)
  const int* d_ncols;    // active column count (device)
  // epilogue (NN)
  const double* y;
  int loss;
  double* part_loss;     // [row_block * part_ld + col]
  double* part_conj;
  int part_ld;
  unsigned long long* probe;  // optional sub-phase timers (CTA 0), nullptr: off
  // TMA descriptor (CUtensorMap in global memory) of X for the 128 x 64
  // register-tiled kernel's A tiles (gemm_big.cuh); nullptr: cp.async staging
  const void* tmap;
};

constexpr int kGemmThreads = 128;
constexpr int kBK = 64;
constexpr int kBKP = kBK + 4;  // padded k-stride (2 wavefronts per fragment load)

template <bool TN, int FM, int FN, int NW = 4>
struct GemmShape {
  static constexpr int BM = 8 * FM, BN = 8 * FN;
  static constexpr int PADA = (BM % 16 == 0) ? 8 : 0;  // NN: (BM+PADA) = 8 mod 16
  static constexpr int A_ELEMS = TN ? BM * kBKP : kBK * (BM + PADA);
  static constexpr int B_ELEMS = BN * kBKP;
  static constexpr int STAGE = A_ELEMS + B_ELEMS;
  static constexpr int NS = (FM * FN >= 16) ? 3 : 4;
  static constexpr int RED = NW * FM * FN * 64;     // cross-warp reduction buffer
  static constexpr int EPI = 2 * BM * BN;           // l / l* staging for EVAL
  static constexpr int SMEM_ELEMS =
      (NS * STAGE > RED + EPI) ? NS * STAGE : RED + EPI;
  static constexpr size_t SMEM_BYTES = sizeof(double) * SMEM_ELEMS;
};

// One output tile (mt, nt) of K-split `split`.  All NW*32 threads call.
// colmap: 32 ints of shared memory.  Ends with a barrier (smem reusable).
template <bool TN, int FM, int FN, int EPI, int NW>
__device__ __forceinline__ void gemm_tile(const GemmArgs& g, int ncols, int mt, int nt, int split,
                                          double* smem, int* colmap) {
  using Sh = GemmShape<TN, FM, FN, NW>;
  constexpr int BM = Sh::BM, BN = Sh::BN, NS = Sh::NS, NT = NW * 32;
  static_assert(16 % NW == 0, "k-steps per stage must split evenly over the warps");
  const int n0 = nt * BN;
  const int m0 = mt * BM;
  const int kbeg = split * g.ksplit;
  const int kend = min(g.K, kbeg + g.ksplit);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  if (tid < BN) {  // physical columns of this tile (BN <= 32)
    const int c = n0 + tid;
    colmap[tid] = c < ncols ? (g.act ? g.act[c] : c) : -1;
  }
  __syncthreads();

  auto load_stage = [&](int stage, int kt) {
    double* As = smem + stage * Sh::STAGE;
    double* Bs = As + Sh::A_ELEMS;
    const int k0 = kbeg + kt * kBK;
#pragma unroll 4
    for (int e = tid; e < BM * kBK; e += NT) {
      int m, k;
      if (TN) {
        m = e / kBK;
        k = e % kBK;
      } else {
        k = e / BM;
        m = e % BM;
      }
      const int gm = m0 + m, gk = k0 + k;
      const bool valid = gm < g.M && gk < kend;
      const double* src =
          valid ? (TN ? g.A + (size_t)gm * g.lda + gk : g.A + (size_t)gk * g.lda + gm) : g.A;
      double* dst = TN ? As + m * kBKP + k : As + k * (BM + Sh::PADA) + m;
      cp_async_8(dst, src, valid);
    }
#pragma unroll 4
    for (int e = tid; e < BN * kBK; e += NT) {
      const int c = e / kBK, k = e % kBK;
      const int gk = k0 + k;
      const int col = colmap[c];
      const bool valid = col >= 0 && gk < kend;
      const double* src = valid ? g.B + (size_t)col * g.ldb + gk : g.B;
      cp_async_8(Bs + c * kBKP + k, src, valid);
    }
  };

  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int nk = (kend - kbeg + kBK - 1) / kBK;
#pragma unroll
  for (int s = 0; s < NS - 1; ++s) {
    if (s < nk) load_stage(s, s);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<NS - 2>();
    __syncthreads();
    if (kt + NS - 1 < nk) load_stage((kt + NS - 1) % NS, kt + NS - 1);
    cp_async_commit();
    const double* As = smem + (kt % NS) * Sh::STAGE;
    const double* Bs = As + Sh::A_ELEMS;
#pragma unroll
    for (int s4 = 0; s4 < 16 / NW; ++s4) {
      const int kk = (s4 * NW + warp) * 4 + (lane & 3);
      double a[FM], b[FN];
#pragma unroll
      for (int i = 0; i < FM; ++i) {
        const int row = i * 8 + (lane >> 2);
        a[i] = TN ? As[row * kBKP + kk] : As[kk * (BM + Sh::PADA) + row];
      }
#pragma unroll
      for (int j = 0; j < FN; ++j) b[j] = Bs[(j * 8 + (lane >> 2)) * kBKP + kk];
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();

  // cross-warp split-K reduction in fixed warp order
  double* red = smem;
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) red[((warp * FM + i) * FN + j) * 64 + h * 32 + lane] = acc[i][j][h];
  __syncthreads();

  double* lv = smem + Sh::RED;
  double* cv = lv + BM * BN;
  double* Cout = g.C + (size_t)split * g.split_stride;
  for (int e = tid; e < BM * BN; e += NT) {
    const int c = e / BM, r = e % BM;
    const int i = r >> 3, j = c >> 3;
    const int ln = (r & 7) * 4 + ((c & 7) >> 1), h = c & 1;
    const int off = (i * FN + j) * 64 + h * 32 + ln;
    constexpr int stride_w = FM * FN * 64;
    double s = red[off];
#pragma unroll
    for (int w = 1; w < NW; ++w) s += red[off + w * stride_w];
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
}

template <bool TN, int FM, int FN, int EPI>
__global__ void __launch_bounds__(kGemmThreads) k_gemm(GemmArgs g) {
  extern __shared__ __align__(128) double smem[];
  __shared__ int colmap[32];
  const int ncols = *g.d_ncols;
  if ((int)blockIdx.y * GemmShape<TN, FM, FN>::BN >= ncols) return;
  gemm_tile<TN, FM, FN, EPI, kGemmThreads / 32>(g, ncols, blockIdx.x, blockIdx.y, blockIdx.z, smem,
                                                colmap);
}

}  // namespace bnbg
