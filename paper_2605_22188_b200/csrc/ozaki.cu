// ozaki.cu -- Engine methods of the tcgen05 (kind::i8) emulated-FP64 products
// of the relaxation iteration (ozaki.cuh):
//   NN  R = l'(X V[:, act])   A = X  (rows i, k = j),  B = V  (k = j)
//   TN  G = X' R[:, act]      A = X' (rows j, k = i),  B = R  (k = i)
// X's digits are cut once per engine (both orientations, on first use);
// the batch operand's digits every iteration.  The bound evaluation keeps
// the DMMA kernels (Psi must be exact for the R it is evaluated at,
// relaxation.hpp:125-147).  On by default (BNBG_OZAKI=0 disables).
#include <algorithm>
#include <cstdlib>
#include <string>

#include "engine.hpp"
#include "ozaki.cuh"

namespace bnbg {

#define CK(call)                                          \
  do {                                                    \
    cudaError_t e_ = (call);                              \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);   \
  } while (0)

#define CKL(what)                                         \
  do {                                                    \
    ++launches;                                           \
    cudaError_t e_ = cudaGetLastError();                  \
    if (e_ != cudaSuccess) return cuda_fail(e_, what);    \
  } while (0)

// On by default; BNBG_OZAKI=0 keeps every product on the DMMA kernels.
bool Engine::ozaki_enabled() const {
  const char* e = getenv("BNBG_OZAKI");
  return !(e && e[0] == '0');
}

// side 0: NN (A = X rows, K = p), side 1: TN (A = X columns, K = n)
int Engine::ozaki_prepare_x(int side) {
  OzSide& S = oz_[side];
  if (S.dX) return 0;
  const int rows = side ? p : n, K = side ? n : p;
  S.nkb = (K + kOzBK - 1) / kOzBK;
  const int rows_pad = (rows + kOzBM - 1) / kOzBM * kOzBM;
  CK(cudaFuncSetAttribute(k_ozaki_gemm<EPI_STORE, 64>,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, OzShape<64>::SmemBytes));
  CK(cudaFuncSetAttribute(k_ozaki_gemm<EPI_DERIV, 64>,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, OzShape<64>::SmemBytes));
  CK(cudaFuncSetAttribute(k_ozaki_gemm<EPI_STORE, 32>,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, OzShape<32>::SmemBytes));
  CK(cudaFuncSetAttribute(k_ozaki_gemm<EPI_DERIV, 32>,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, OzShape<32>::SmemBytes));
  CK(cudaMallocAsync(&S.dX, (size_t)kOzS * rows_pad * S.nkb * kOzBK, stream_));
  CK(cudaMallocAsync(&S.dEx, sizeof(int) * rows, stream_));
  // NN reads X rows with stride n (once per engine); TN reads X columns
  k_oz_split_rows<<<rows_pad, 256, 0, stream_>>>(dX_, side ? n : 1, side ? 1 : n, nullptr, rows,
                                                 nullptr, K, S.nkb, kOzBM, kOzBM,
                                                 static_cast<signed char*>(S.dX), S.dEx);
  CKL("k_oz_split_rows(X)");
  return 0;
}

int Engine::ozaki_reserve_b(int side, int m) {
  OzSide& S = oz_[side];
  if (m <= S.bcap) return 0;
  const int cap = (std::max(m, std::max(64, 2 * S.bcap)) + 63) / 64 * 64;
  dfree(S.dB);
  dfree(S.dEb);
  CK(cudaMallocAsync(&S.dB, (size_t)kOzS * cap * S.nkb * kOzBK, stream_));
  CK(cudaMallocAsync(&S.dEb, sizeof(int) * cap, stream_));
  S.bcap = cap;
  return 0;
}

// C (+ split*split_stride) column act[c] (ldc) = op(X) * Bsrc[:, act[c]] for
// the ma active columns (Bsrc column c at Bsrc + act[c]*ldb; act nullptr:
// identity); deriv applies l' (NN: R = l'(X V)).  *nsplit receives the
// K-split count (TN; NN is never split, its epilogue needs whole sums).
int Engine::gemm_ozaki(bool tn, bool deriv, const double* Bsrc, int ldb, const int* act, int ma,
                       const int* d_ncols, double* C, int ldc, long long split_stride,
                       int* nsplit) {
  const int side = tn ? 1 : 0;
  if (int rc = ozaki_prepare_x(side)) return rc;
  if (int rc = ozaki_reserve_b(side, ma)) return rc;
  OzSide& S = oz_[side];
  const int M = tn ? p : n, K = tn ? n : p;
  // one CTA per SM (the digits ring fills shared memory and TMEM).  TN:
  // 64-column tiles, K split so that the CTAs make about one wave.  NN (no
  // split: the l' epilogue needs whole sums): the tile width with the fewer
  // wave-weighted tile costs.
  const int mt = (M + kOzBM - 1) / kOzBM;
  int bn = ma <= 32 ? 32 : 64;
  if (!tn && ma > 32) {  // waves x per-tile cost (a 32-column tile costs ~0.6 of a 64-column one:
              // the A digits it loads are the same)
    const int t64 = mt * ((ma + 63) / 64), t32 = mt * ((ma + 31) / 32);
    const double c64 = (double)((t64 + sms_ - 1) / sms_), c32 = 0.6 * ((t32 + sms_ - 1) / sms_);
    if (c32 < c64) bn = 32;
  }
  const int nt = (ma + bn - 1) / bn;
  const int nkb = S.nkb;
  // the batch digits in the tiling of this launch (bn-row tiles)
  k_oz_split_rows<<<nt * bn, 256, 0, stream_>>>(Bsrc, ldb, 1, act, ma, d_ncols, K, nkb, bn,
                                                kOzG, static_cast<signed char*>(S.dB), S.dEb);
  CKL("k_oz_split_rows(batch)");
  int ns = 1;
  if (tn) ns = std::max(1, std::min({nsplit_max_, sms_ / (mt * nt), nkb / 16}));
  OzArgs a{};
  a.A = static_cast<const signed char*>(S.dX);
  a.B = static_cast<const signed char*>(S.dB);
  a.nkb_total = nkb;
  a.ea = S.dEx;
  a.eb = S.dEb;
  a.M = M;
  a.K = K;
  a.ksplit = ((nkb + ns - 1) / ns) * kOzBK;
  ns = (K + a.ksplit - 1) / a.ksplit;
  a.d_ncols = d_ncols;
  a.act = act;
  a.C = C;
  a.ldc = ldc;
  a.split_stride = split_stride;
  a.y = dy_;
  a.loss = loss;
  const dim3 grid(nt, mt, ns);
  if (bn == 64) {
    if (!deriv)
      k_ozaki_gemm<EPI_STORE, 64><<<grid, kOzThreads, OzShape<64>::SmemBytes, stream_>>>(a);
    else
      k_ozaki_gemm<EPI_DERIV, 64><<<grid, kOzThreads, OzShape<64>::SmemBytes, stream_>>>(a);
  } else {
    if (!deriv)
      k_ozaki_gemm<EPI_STORE, 32><<<grid, kOzThreads, OzShape<32>::SmemBytes, stream_>>>(a);
    else
      k_ozaki_gemm<EPI_DERIV, 32><<<grid, kOzThreads, OzShape<32>::SmemBytes, stream_>>>(a);
  }
  CKL("k_ozaki_gemm");
  if (nsplit) *nsplit = ns;
  return 0;
}

}  // namespace bnbg
