// pool.cu -- Engine methods of the device-resident node pool (pool_kernels.cuh).
#include <algorithm>
#include <cstring>

#include "engine.hpp"
#include "pool_kernels.cuh"

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

static PoolDev pool_view(void* const* mem, int p, int k, int cap) {
  PoolDev P;
  P.p = p;
  P.k = std::max(k, 1);
  P.cap = cap;
  P.state = static_cast<uint8_t*>(mem[0]);
  P.warm = static_cast<double*>(mem[1]);
  P.j0 = static_cast<int*>(mem[2]);
  P.j1 = static_cast<int*>(mem[3]);
  P.n0 = static_cast<int*>(mem[4]);
  P.n1 = static_cast<int*>(mem[5]);
  P.depth = static_cast<int*>(mem[6]);
  return P;
}

int Engine::pool_reserve(int cap) {
  if (cap <= pool_cap_) return 0;
  cap = std::max(cap, std::max(64, pool_cap_ * 2));
  const int kk = std::max(k, 1);
  const size_t per[7] = {(size_t)p, sizeof(double) * p, sizeof(int) * (size_t)p,
                         sizeof(int) * (size_t)kk, sizeof(int), sizeof(int), sizeof(int)};
  for (int a = 0; a < 7; ++a) {
    void* nb = nullptr;
    CK(cudaMallocAsync(&nb, per[a] * cap, stream_));
    if (pool_mem_[a]) {
      CK(cudaMemcpyAsync(nb, pool_mem_[a], per[a] * pool_cap_, cudaMemcpyDeviceToDevice, stream_));
      CK(cudaStreamSynchronize(stream_));
      dfree(pool_mem_[a]);
    }
    pool_mem_[a] = nb;
  }
  pool_cap_ = cap;
  return 0;
}

int Engine::pool_root(int slot) {
  if (int rc = pool_reserve(slot + 1)) return rc;
  k_pool_root<<<1, 256, 0, stream_>>>(pool_view(pool_mem_, p, k, pool_cap_), slot);
  CKL("k_pool_root");
  return 0;
}

int Engine::ensure_pool_batch(int m) {
  if (int rc = ensure(m)) return rc;
  if (m <= pool_batch_cap_) return 0;
  const int cap = std::max(m, std::max(16, pool_batch_cap_ * 2));
  const int kk = std::max(k, 1);
  dfree(dSlots_);
  dfree(dLbIn_);
  dfree(dLbOut_);
  dfree(dPos_);
  dfree(dTot_);
  dfree(dFree_);
  dfree(dRec_);
  dfree(dRecLb_);
  dfree(dOneLen_);
  dfree(dOneIdx_);
  dfree(dLists_);
  dLists_ = nullptr;
  CK(cudaMallocAsync(&dSlots_, sizeof(int) * cap, stream_));
  CK(cudaMallocAsync(&dLbIn_, sizeof(double) * cap, stream_));
  CK(cudaMallocAsync(&dLbOut_, sizeof(double) * cap, stream_));
  CK(cudaMallocAsync(&dPos_, sizeof(int) * cap, stream_));
  CK(cudaMallocAsync(&dTot_, sizeof(int) * 2, stream_));
  CK(cudaMallocAsync(&dFree_, sizeof(int) * 2 * (size_t)cap, stream_));
  CK(cudaMallocAsync(&dRec_, sizeof(int) * 2 * (size_t)cap * child_rec_ints(kk), stream_));
  CK(cudaMallocAsync(&dRecLb_, sizeof(double) * 2 * (size_t)cap, stream_));
  // small passes read every record slot back (branch_pool): defined bytes
  CK(cudaMemsetAsync(dRec_, 0xff, sizeof(int) * 2 * (size_t)cap * child_rec_ints(kk), stream_));
  CK(cudaMemsetAsync(dRecLb_, 0, sizeof(double) * 2 * (size_t)cap, stream_));
  CK(cudaMallocAsync(&dOneLen_, sizeof(int) * cap, stream_));
  CK(cudaMallocAsync(&dOneIdx_, sizeof(int) * (size_t)cap * kk, stream_));
  pool_batch_cap_ = cap;
  return 0;
}

int Engine::relax_pool(int m, const int* slots, const RelaxParams& cfg, double thr, bool trace,
                       PassResult& out, bool lists, std::vector<int>* n01, std::vector<int>* j0,
                       std::vector<int>* j1) {
  if (m <= 0) return fail(1, "solve_batch_relaxation: empty batch");
  if (int rc = ensure_pool_batch(m)) return rc;
  const int kk = std::max(k, 1);
  if (int rc_ = h2d(dSlots_, slots, sizeof(int) * m)) return rc_;
  const PoolDev P = pool_view(pool_mem_, p, k, pool_cap_);
  k_pack_pool<<<m, kPoolThreads, 0, stream_>>>(P, m, dSlots_, dState_, dKbar_, dPf_, dB_, dV_, dT_,
                                                dBest_, dLast_, dFrozen_, dStatus_, dIters_, dAct_,
                                                cfg.max_iterations, dOneLen_, dOneIdx_);
  CKL("k_pack_pool");
  if (lists) {
    const size_t ints = (size_t)m * (2 + p + kk);
    if (!dLists_) CK(cudaMallocAsync(&dLists_, sizeof(int) * (size_t)pool_batch_cap_ * (2 + p + kk), stream_));
    k_pool_lists<<<m, 128, 0, stream_>>>(P, m, dSlots_, dLists_, dLists_ + 2 * m,
                                         dLists_ + (size_t)m * (2 + p));
    CKL("k_pool_lists");
    std::vector<int> h(ints);
    if (int rc_ = d2h(h.data(), dLists_, sizeof(int) * ints)) return rc_;
    CK(cudaStreamSynchronize(stream_));
    n01->assign(h.begin(), h.begin() + 2 * m);
    j0->assign(h.begin() + 2 * m, h.begin() + (size_t)m * (2 + p));
    j1->assign(h.begin() + (size_t)m * (2 + p), h.end());
  }
  return relax_uploaded(m, cfg, thr, trace, out, true, nullptr, dOneIdx_, dOneLen_, false);
}

int Engine::branch_pool(int m, const int* slots, const double* lb_in, double post_thr,
                        const int* free_slots, int& survivors, int& bad_column,
                        std::vector<int>& rec, std::vector<double>& rec_lb) {
  survivors = 0;
  bad_column = -1;
  if (m <= 0) return 0;
  const int kk = std::max(k, 1);
  const int RI = child_rec_ints(kk);
  if (int rc_ = h2d(dLbIn_, lb_in, sizeof(double) * m)) return rc_;
  if (int rc_ = h2d(dFree_, free_slots, sizeof(int) * 2 * (size_t)m)) return rc_;
  k_branch_scan<<<1, 1024, 0, stream_>>>(m, dStatus_, dBest_, dLbIn_, post_thr, dJb_, dLbOut_,
                                          dPos_, dTot_);
  CKL("k_branch_scan");
  const PoolDev P = pool_view(pool_mem_, p, k, pool_cap_);
  k_branch_write<<<m, kPoolThreads, 0, stream_>>>(P, m, M, dSlots_, dState_, dB_, dJb_, dPos_,
                                                   dLbOut_, dFree_, dRec_, dRecLb_);
  CKL("k_branch_write");
  int tot[2];
  if (int rc_ = d2h_defer(tot, dTot_, sizeof(tot))) return rc_;
  // small passes: every possible child record comes back with the counts
  // (one synchronisation); large ones read the survivors' records only
  const size_t ncmax = 2 * (size_t)m;
  const bool whole = ncmax * (RI * sizeof(int) + sizeof(double)) <= (256u << 10);
  if (whole) {
    rec.resize(ncmax * RI);
    rec_lb.resize(ncmax);
    if (int rc_ = d2h_defer(rec.data(), dRec_, sizeof(int) * ncmax * RI)) return rc_;
    if (int rc_ = d2h_defer(rec_lb.data(), dRecLb_, sizeof(double) * ncmax)) return rc_;
  }
  if (int rc_ = sync_flush()) return rc_;
  survivors = tot[0];
  bad_column = tot[1];
  const size_t nc = 2 * (size_t)survivors;
  rec.resize(nc * RI);
  rec_lb.resize(nc);
  if (nc && !whole) {
    if (int rc_ = d2h_defer(rec.data(), dRec_, sizeof(int) * nc * RI)) return rc_;
    if (int rc_ = d2h_defer(rec_lb.data(), dRecLb_, sizeof(double) * nc)) return rc_;
    if (int rc_ = sync_flush()) return rc_;
  }
  (void)slots;
  return 0;
}

}  // namespace bnbg
