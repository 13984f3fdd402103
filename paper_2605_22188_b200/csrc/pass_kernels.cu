// pass_kernels.cu -- host dispatch of the persistent pass kernel over the
// column-sort width E.  Each k_pass<E> instantiation lives in its own
// translation unit (pass_e<E>.cu) so the five compile in parallel.
#include "launchers.hpp"
#include "pass_kernel.cuh"
#include "pass_impl.hpp"

namespace bnbg {

#define DISPATCH_E(E_, ...)  \
  switch (E_) {              \
    case 1: {                \
      constexpr int EV = 1;  \
      __VA_ARGS__;           \
    } break;                 \
    case 2: {                \
      constexpr int EV = 2;  \
      __VA_ARGS__;           \
    } break;                 \
    case 4: {                \
      constexpr int EV = 4;  \
      __VA_ARGS__;           \
    } break;                 \
    default: {               \
      constexpr int EV = 0;  \
      __VA_ARGS__;           \
    } break;                 \
  }

size_t pass_smem(int p, int n2, int E) { return pass_smem_bytes(p, n2, E); }

size_t pass_res_plan(int n, int p, int n2, int E, int grid, size_t smem_limit, ResLayout* res,
                     int rt) {
  ResLayout L = {};
  L.rt = rt;
  L.nn_tiles = (n + kResBM * rt - 1) / (kResBM * rt);
  L.kpad_nn = (p + 3) & ~3;
  L.lda_nn = kResBM * rt + 4;
  L.tn_mt = (p + kResBM - 1) / kResBM;
  *res = L;
  if (L.nn_tiles > grid || L.tn_mt > grid) return 0;
  int split = grid / L.tn_mt;
  if (split > kMaxSplit) split = kMaxSplit;
  if (split < 1) split = 1;
  int klen = (n + split - 1) / split;
  klen = (klen + 3) & ~3;
  L.tn_klen = klen;
  L.tn_split = (n + klen - 1) / klen;
  L.ldk_tn = ld_mod16_4(klen);
  L.ldb = ld_mod16_4(L.kpad_nn > klen ? L.kpad_nn : klen);
  const long long nn = (long long)L.kpad_nn * L.lda_nn;
  L.off_tn = (nn + 1) & ~1LL;
  L.off_work = (L.off_tn + (long long)kResBM * L.ldk_tn + 1) & ~1LL;
  size_t work = res_work_doubles(L);
  const size_t col = column_smem_bytes(p, n2, E) / 8 + 1;
  if (col > work) work = col;
  size_t bytes = 8 * ((size_t)L.off_work + work);
  if (bytes > smem_limit) return 0;
  // column cache for the register-sort widths (E > 0)
  const size_t cc = 2 * (size_t)p + ((size_t)p + 7) / 8 + 2;
  if (E && bytes + 8 * cc <= smem_limit) {
    L.off_cc = (long long)(L.off_work + work + 1) & ~1LL;
    bytes = 8 * ((size_t)L.off_cc + cc);
  }
  L.on = 1;
  *res = L;
  return bytes;
}

cudaError_t pass_static_smem(int E, size_t* bytes) {
  cudaError_t e = cudaSuccess;
  DISPATCH_E(E, e = pass_static_smem_t<EV>(bytes));
  return e;
}

cudaError_t pass_setup(int E, size_t smem, int* blocks_per_sm) {
  cudaError_t e = cudaSuccess;
  *blocks_per_sm = 0;
  DISPATCH_E(E, e = pass_setup_t<EV>(smem, blocks_per_sm));
  return e;
}

cudaError_t pass_launch(int E, int grid, size_t smem, cudaStream_t st, PassArgs* a, int cluster) {
  cudaError_t e = cudaSuccess;
  DISPATCH_E(E, e = pass_launch_t<EV>(grid, smem, st, a, cluster));
  return e;
}

bool pass_cluster_ok(int E, size_t smem, int cs) {
  bool ok = false;
  DISPATCH_E(E, ok = pass_cluster_ok_t<EV>(smem, cs));
  return ok;
}

}  // namespace bnbg
