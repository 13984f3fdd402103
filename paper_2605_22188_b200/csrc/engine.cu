// engine.cu -- device engine: instance upload, GEMM planning, the relaxation
// loop (relaxation.hpp:163-255), rounding/branch selection and re-opt.
#include <algorithm>
#include <chrono>
#include <mutex>
#include <vector>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include <cuda.h>
#include <cudaTypedefs.h>  // PFN_cuTensorMapEncodeTiled

#include "engine.hpp"
#include "gemm.cuh"
#include "node_kernels.cuh"
#include "launchers.hpp"
#include "reopt_kernels.cuh"
#include "rng.hpp"

namespace bnbg {

// Small pinned host slots (4 ints) for the per-pass readbacks, kept for the
// process: page-locking a new block costs ~2 ms per engine creation, which
// would dominate creating an engine for a small instance.
static std::mutex g_pin_mu;
static std::vector<int*> g_pin_free;

static int* pinned_slot_acquire() {
  {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    if (!g_pin_free.empty()) {
      int* s = g_pin_free.back();
      g_pin_free.pop_back();
      return s;
    }
  }
  void* p = nullptr;
  // portable: a released slot may be reused by an engine on another device
  if (cudaHostAlloc(&p, 64, cudaHostAllocPortable) != cudaSuccess) return nullptr;
  return static_cast<int*>(p);
}

static void pinned_slot_release(int* s) {
  std::lock_guard<std::mutex> lk(g_pin_mu);
  g_pin_free.push_back(s);
}

// pinned readback staging buffers, pooled like the slots above
constexpr size_t kStageBytes = 4u << 20;
static std::vector<char*> g_stage_free;

static char* stage_acquire() {
  {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    if (!g_stage_free.empty()) {
      char* s = g_stage_free.back();
      g_stage_free.pop_back();
      return s;
    }
  }
  void* p = nullptr;
  if (cudaHostAlloc(&p, kStageBytes, cudaHostAllocPortable) != cudaSuccess) {
    (void)cudaGetLastError();
    return nullptr;  // readbacks then stay pageable
  }
  return static_cast<char*>(p);
}

static void stage_release(char* s) {
  std::lock_guard<std::mutex> lk(g_pin_mu);
  g_stage_free.push_back(s);
}

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

static int next_pow2(int v) {
  int r = 1;
  while (r < v) r <<= 1;
  return r;
}

Engine::~Engine() {
  dfree(dX_);
  dfree(dy_);
  dfree(dB_);
  dfree(dV_);
  dfree(dG_);
  dfree(dR_);
  dfree(dPL_);
  dfree(dPC_);
  dfree(dT_);
  dfree(dBest_);
  dfree(dLast_);
  dfree(dState_);
  dfree(dFrozen_);
  dfree(dKbar_);
  dfree(dPf_);
  dfree(dStatus_);
  dfree(dIters_);
  dfree(dAct_);
  dfree(dMa_);
  dfree(dErr_);
  dfree(dSup_);
  dfree(dLen_);
  dfree(dJb_);
  dfree(dAux_);
  dfree(dPassOut_);
  dfree(dPassProf_);
  dfree(dBar_);
  dfree(dTmap_);
  dfree(dTmapQ_);
  dfree(dQ_);
  dfree(dCq_);
  dfree(dGramCnt_);
  dfree(dColScr_);
  for (OzSide& S : oz_) {
    dfree(S.dX);
    dfree(S.dEx);
    dfree(S.dB);
    dfree(S.dEb);
  }
  comm_release();
  for (void* q : pool_mem_) dfree(q);
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
  // an error path may have left a d2h copy into hPin_ in flight: drain the
  // stream before the slot returns to the process-wide free list
  if (stream_) cudaStreamSynchronize(stream_);
  if (hPin_) pinned_slot_release(hPin_);
  if (hStage_) stage_release(hStage_);
  if (ev0_) cudaEventDestroy(ev0_);
  if (ev1_) cudaEventDestroy(ev1_);
  if (stream_) cudaStreamDestroy(stream_);
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link)
static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

// X (n x p column-major, resident) as a 2-D FLOAT64 tensor {n, p}: one map
// per A-tile box of the register-tiled GEMM (BNBG_TMA=0 keeps cp.async).
int Engine::make_tmaps() {
  const char* e = getenv("BNBG_TMA");
  if ((e && e[0] == '0') || (n % 2) || (p % 2)) return 0;
  auto enc = tmap_encoder();
  if (!enc) return fail(4, "cuTensorMapEncodeTiled unavailable");
  int nn[2], tn[2];
  gemm_big_boxes(nn, tn);
  CUtensorMap h[2];
  const cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)p};
  const cuuint64_t strides[1] = {(cuuint64_t)n * sizeof(double)};
  const cuuint32_t estr[2] = {1, 1};
  for (int t = 0; t < 2; ++t) {
    const cuuint32_t box[2] = {(cuuint32_t)(t ? tn[0] : nn[0]), (cuuint32_t)(t ? tn[1] : nn[1])};
    const CUresult r = enc(&h[t], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, dX_, dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
      return fail(4, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  }
  CK(cudaMallocAsync(&dTmap_, sizeof(h), stream_));
  CK(cudaMemcpyAsync(dTmap_, h, sizeof(h), cudaMemcpyHostToDevice, stream_));
  CK(cudaStreamSynchronize(stream_));
  tmNN_ = dTmap_;
  tmTN_ = static_cast<const char*>(dTmap_) + sizeof(CUtensorMap);
  return 0;
}

int Engine::fail(int code, const std::string& msg) {
  err = msg;
  defer_.clear();  // queued readbacks of the failed call are never copied out
  pass_pending_ = false;
  return code;
}

int Engine::cuda_fail(cudaError_t e, const char* what) {
  err = std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e);
  defer_.clear();
  pass_pending_ = false;
  return 4;  // BNBG_CUDA_ERROR
}

int Engine::init(const double* X, const double* y, int n_, int p_, int loss_, int k_, double M_,
                 double lambda2_, double L_, int device_) {
  n = n_;
  p = p_;
  k = k_;
  loss = loss_;
  M = M_;
  lambda2 = lambda2_;
  device = device_;
  // BNBG_INIT_PROF=1: wall time of each creation step on stderr (diagnostics)
  const char* ip = getenv("BNBG_INIT_PROF");
  const bool iprof = ip && ip[0] == '1';
  auto t_last = std::chrono::steady_clock::now();
  auto stamp = [&](const char* what) {
    if (!iprof) return;
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "init %-14s %8.3f ms\n", what,
            std::chrono::duration<double, std::milli>(t - t_last).count());
    t_last = t;
  };
  CK(cudaSetDevice(device));
  stamp("set_device");
  CK(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  stamp("stream");
  {  // stream-ordered allocations: keep freed blocks in the device pool for reuse
    cudaMemPool_t mp;
    CK(cudaDeviceGetDefaultMemPool(&mp, device));
    uint64_t keep = UINT64_MAX;
    CK(cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &keep));
  }
  CK(cudaEventCreate(&ev0_));
  CK(cudaEventCreate(&ev1_));
  CK(cudaDeviceGetAttribute(&sms_, cudaDevAttrMultiProcessorCount, device));
  hPin_ = pinned_slot_acquire();
  if (!hPin_) return cuda_fail(cudaErrorMemoryAllocation, "cudaMallocHost");
  {
    const char* de = getenv("BNBG_DEFER_D2H");
    defer_on_ = !(de && de[0] == '0');
    if (defer_on_) hStage_ = stage_acquire();
  }
  stamp("malloc_host");
  CK(cudaMallocAsync(&dX_, sizeof(double) * (size_t)n * p, stream_));
  CK(cudaMallocAsync(&dy_, sizeof(double) * (size_t)n, stream_));
  if (int rc_ = h2d(dX_, X, sizeof(double) * (size_t)n * p)) return rc_;
  if (int rc_ = h2d(dy_, y, sizeof(double) * (size_t)n)) return rc_;
  stamp("upload");
  if (int rc = make_tmaps()) return rc;
  CK(cudaMallocAsync(&dMa_, sizeof(int), stream_));
  CK(cudaMallocAsync(&dErr_, sizeof(int), stream_));
  CK(gemm_set_attrs());
  n2_ = next_pow2(std::max(p, 2));
  colE_ = column_E(n2_);
  csmem_ = column_smem_bytes(p, n2_, colE_);
  if (csmem_ > 220 * 1024) {
    // large p (> 7 680): a node's sort keys no longer fit one CTA's shared
    // memory; the column kernels keep them in a global scratch (L1/L2), one
    // slice per CTA, and the persistent pass kernel is off (its plan below
    // fails the shared-memory limit)
    colstride_ = (long long)((csmem_ + 255) / 256 * 32);  // doubles, 256-byte aligned slices
    csmem_ = 0;
  }
  CK(column_set_attrs(colE_, csmem_));
  stamp("attrs");
  // persistent pass kernel: one CTA per SM when it fits (BNBG_PERSISTENT=0
  // disables it; BNBG_RESIDENT=0 forces the streaming operand mode)
  {
    const char* env = getenv("BNBG_PERSISTENT");
    const char* renv = getenv("BNBG_RESIDENT");
    int coop = 0, optin = 0;
    CK(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device));
    CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    pass_grid_ = 0;
    res_ = ResLayout{};
    {
      const char* ge = getenv("BNBG_GRAM");
      gram_ = loss == kSquared && p <= n && !(ge && ge[0] == '0');
    }
    if (coop && !(env && env[0] == '0')) {
      size_t stat = 0;
      CK(pass_static_smem(colE_, &stat));
      const size_t limit = (size_t)optin - stat - 256;
      pass_smem_ = pass_smem(p, n2_, colE_);
      // small p (c1): Q, c and the column's B, V, states held in shared
      // memory past the streaming region; every CTA iterates its column
      // alone between evaluations (no grid barrier per iteration)
      gram_local_off_ = 0;
      const char* le = getenv("BNBG_GRAM_LOCAL");
      const bool want_local =
          gram_ && colE_ != 0 && !(le && le[0] == '0') && (size_t)p * p * 8 <= 128 * 1024;
      const size_t gl_bytes = want_local ? gram_local_bytes(p) + 16 : 0;
      // X residency: always tried without the Gram form; with it, only next to
      // the local region (the evaluations read the resident X, the local
      // iterations never touch it).  Streaming Gram iterations need the
      // shared memory for their Q tiles.
      if (!(renv && renv[0] == '0') && (!gram_ || want_local)) {
        ResLayout L;
        const size_t rb = pass_res_plan(n, p, n2_, colE_, sms_, limit - gl_bytes, &L);
        if (L.on) {
          const char* cenv = getenv("BNBG_COLCACHE");
          if (cenv && cenv[0] == '0') L.off_cc = 0;  // diagnostics: no column cache
          res_ = L;
          pass_smem_ = rb;
        }
      }
      if (want_local) {
        const long long off = (long long)((pass_smem_ + 15) / 16 * 2);  // doubles, 16-byte aligned
        const size_t bytes = 8 * (size_t)off + gram_local_bytes(p);
        if (bytes <= limit) {
          gram_local_off_ = off;
          pass_smem_ = bytes;
        }
      }
      // one-cluster variant for small X (c1): 16 CTAs of one cluster hold X
      // (64-row NN tiles) and meet at cluster barriers, 0.2 us against the
      // grid barrier's 1.2 us (profiles/r02_barriers.txt); narrow batches only,
      // as it has 16 SMs (BNBG_CLUSTER_PASS=0 disables it, BNBG_CLUSTER_MAXM
      // sets the widest batch)
      resc_ = ResLayout{};
      const char* cenv = getenv("BNBG_CLUSTER_PASS");
      if (res_.on && gram_local_off_ == 0 && !(cenv && cenv[0] == '0')) {
        constexpr int kCS = 16;
        ResLayout Lc;
        const size_t rbc = pass_res_plan(n, p, n2_, colE_, kCS, limit, &Lc, 4);
        if (Lc.on && Lc.off_cc > 0 && pass_cluster_ok(colE_, rbc, kCS)) {
          Lc.cluster = kCS;
          resc_ = Lc;
          pass_smem_c_ = rbc;
        }
        (void)cudaGetLastError();
        const char* me = getenv("BNBG_CLUSTER_MAXM");
        if (me) cluster_max_m_ = atoi(me);
      }
      if (pass_smem_ <= limit) {
        int nb = 0;
        CK(pass_setup(colE_, std::max(pass_smem_, pass_smem_c_), &nb));
        if (nb >= 1) pass_grid_ = sms_;
      }
    }
    CK(cudaMallocAsync(&dBar_, sizeof(unsigned), stream_));
    CK(cudaMallocAsync(&dPassOut_, 4 * sizeof(long long), stream_));
    const char* penv = getenv("BNBG_PASS_PROF");
    if (penv && penv[0] == '1') {
      CK(cudaMallocAsync(&dPassProf_, 32 * sizeof(unsigned long long), stream_));
      CK(cudaMemsetAsync(dPassProf_, 0, 32 * sizeof(unsigned long long), stream_));
    }
  }
  stamp("pass_plan");
  nrb_max_ = (n + 15) / 16;
  {  // per-iteration work above which streaming batches use the standalone kernels
    const char* e = getenv("BNBG_PERSIST_MAXFLOPS");
    persist_max_flops_ = e ? atof(e) : 4e9;
  }
  {  // active width from which the 128 x 64 GEMM tiles are used (BNBG_BIGGEMM=0: never)
    const char* e = getenv("BNBG_BIGGEMM");
    big_min_ = e ? std::max(0, atoi(e)) : 64;
    // ... and from which the standalone iteration GEMMs run on the tcgen05
    // emulation (measured at c4: 16 beats 32 and 64 by 3-4 %)
    const char* o = getenv("BNBG_OZAKI_MIN");
    oz_min_ = o ? std::max(1, atoi(o)) : 16;
  }
  // batch workspaces and the node pool sized for a typical narrow frontier up
  // front, so the first passes of a solve do not pay cudaMalloc/cudaFree
  // (cudaFree synchronises the device) while the batch width grows
  {
    const size_t col_bytes = (size_t)p * 40 + (size_t)n * 8;
    const int pre = (int)std::min<size_t>(128, std::max<size_t>(16, (256u << 20) / col_bytes));
    if (int rc = ensure(pre)) return rc;
    if (int rc = ensure_pool_batch(pre)) return rc;
    if (int rc = pool_reserve(4 * pre)) return rc;
    // re-opt / upload scratch for a pass of `pre` supports
    if (int rc = ensure_aux(sizeof(double) * ((size_t)p * pre + (size_t)8 * pre * std::max(k, 1)) +
                            (size_t)(64 << 10)))
      return rc;
  }
  CK(cudaStreamSynchronize(stream_));
  stamp("prealloc+sync");
  if (L_ > 0.0) {
    L = L_;
  } else {
    int rc = compute_smoothness(&L);
    if (rc) return rc;
  }
  stamp("smoothness");
  return 0;
}

int Engine::ensure(int m) {
  if (m <= mcap_) return 0;
  int cap = std::max(m, std::max(16, mcap_ * 2));
  dfree(dB_);
  dfree(dV_);
  dfree(dG_);
  dfree(dR_);
  dfree(dPL_);
  dfree(dPC_);
  dfree(dT_);
  dfree(dBest_);
  dfree(dLast_);
  dfree(dState_);
  dfree(dFrozen_);
  dfree(dKbar_);
  dfree(dPf_);
  dfree(dStatus_);
  dfree(dIters_);
  dfree(dAct_);
  dfree(dSup_);
  dfree(dLen_);
  dfree(dJb_);
  const size_t pm = (size_t)p * cap;
  if (colstride_) {
    dfree(dColScr_);
    CK(cudaMallocAsync(&dColScr_, sizeof(double) * (size_t)colstride_ * cap, stream_));
  }
  CK(cudaMallocAsync(&dB_, sizeof(double) * pm, stream_));
  CK(cudaMallocAsync(&dV_, sizeof(double) * pm, stream_));
  CK(cudaMallocAsync(&dG_, sizeof(double) * pm * nsplit_max_, stream_));
  CK(cudaMallocAsync(&dR_, sizeof(double) * (size_t)n * cap, stream_));
  CK(cudaMallocAsync(&dPL_, sizeof(double) * (size_t)nrb_max_ * cap, stream_));
  CK(cudaMallocAsync(&dPC_, sizeof(double) * (size_t)nrb_max_ * cap, stream_));
  CK(cudaMallocAsync(&dT_, sizeof(double) * cap, stream_));
  CK(cudaMallocAsync(&dBest_, sizeof(double) * cap, stream_));
  CK(cudaMallocAsync(&dLast_, sizeof(double) * cap, stream_));
  CK(cudaMallocAsync(&dState_, pm, stream_));
  CK(cudaMallocAsync(&dFrozen_, cap, stream_));
  CK(cudaMallocAsync(&dKbar_, sizeof(int) * cap, stream_));
  CK(cudaMallocAsync(&dPf_, sizeof(int) * cap, stream_));
  CK(cudaMallocAsync(&dStatus_, sizeof(int) * cap, stream_));
  CK(cudaMallocAsync(&dIters_, sizeof(int) * cap, stream_));
  CK(cudaMallocAsync(&dAct_, sizeof(int) * cap, stream_));
  CK(cudaMallocAsync(&dSup_, sizeof(int) * (size_t)cap * std::max(k, 1), stream_));
  CK(cudaMallocAsync(&dLen_, sizeof(int) * cap, stream_));
  CK(cudaMallocAsync(&dJb_, sizeof(int) * cap, stream_));
  mcap_ = cap;
  return 0;
}

int Engine::ensure_aux(size_t bytes) {
  if (bytes <= aux_bytes_) return 0;
  dfree(dAux_);
  dAux_ = nullptr;
  size_t cap = std::max(bytes, aux_bytes_ * 2);
  CK(cudaMallocAsync(&dAux_, cap, stream_));
  aux_bytes_ = cap;
  return 0;
}

cudaEvent_t Engine::get_event() {
  if (!ev_pool_.empty()) {
    cudaEvent_t e = ev_pool_.back();
    ev_pool_.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// Deferred CUDA-event timing of each kernel class on the engine stream: the
// pairs are resolved at the next stream synchronisation, so timing does not
// add host syncs to the loop.
void Engine::tic(int kc) {
  (void)kc;
  if (!timing) return;
  cur_a_ = get_event();
  cudaEventRecord(cur_a_, stream_);
}
void Engine::toc(int kc, double flops) {
  kc_launches[kc] += 1;
  kc_flops[kc] += flops;
  if (!timing) return;
  cudaEvent_t b = get_event();
  cudaEventRecord(b, stream_);
  pending_.push_back({cur_a_, b, kc});
}
void Engine::resolve_timing() {
  for (auto& pr : pending_) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, pr.a, pr.b) == cudaSuccess) kc_ms[pr.kc] += ms;
    ev_pool_.push_back(pr.a);
    ev_pool_.push_back(pr.b);
  }
  pending_.clear();
}

int Engine::h2d(void* dst, const void* src, size_t bytes) {
  if (!bytes) return 0;
  h2d_bytes += (long long)bytes;
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, stream_));
  return 0;
}
int Engine::d2h(void* dst, const void* src, size_t bytes) {
  if (!bytes) return 0;
  d2h_bytes += (long long)bytes;
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, stream_));
  return 0;
}
int Engine::d2h_defer(void* dst, const void* src, size_t bytes) {
  if (!bytes) return 0;
  if (!hStage_ || bytes > kStageBytes) return d2h(dst, src, bytes);
  size_t off = (stage_used_ + 15) & ~(size_t)15;
  if (off + bytes > kStageBytes) {
    if (int rc = sync_flush()) return rc;
    off = 0;
  }
  d2h_bytes += (long long)bytes;
  CK(cudaMemcpyAsync(hStage_ + off, src, bytes, cudaMemcpyDeviceToHost, stream_));
  defer_.push_back(Deferred{dst, off, bytes});
  stage_used_ = off + bytes;
  return 0;
}

int Engine::sync_flush() {
  const cudaError_t e = cudaStreamSynchronize(stream_);
  if (e != cudaSuccess) {
    defer_.clear();  // the destinations are not written on a failed stream
    return cuda_fail(e, "cudaStreamSynchronize");
  }
  for (const Deferred& d : defer_) std::memcpy(d.dst, hStage_ + d.off, d.bytes);
  defer_.clear();
  stage_used_ = 0;
  return 0;
}

// ---------------------------------------------------------------------------
// GEMM planning: BN from the active width, BM so the grid covers the SMs,
// split-K (TN only) when the tiles alone cannot.
// ---------------------------------------------------------------------------
Engine::GemmPlan Engine::plan(int Mr, int K, int ncols, bool allow_split, bool allow_big) const {
  GemmPlan pl;
  // wide batches: register-tiled 128 x 64 tiles, no split-K (BNBG_BIGGEMM=0 disables)
  if (allow_big && big_min_ > 0 && ncols >= big_min_ && (n % 2) == 0 && (p % 2) == 0) {
    const int bm = gemm_big_tile_m(), bn = gemm_big_tile_n(), bk = gemm_big_tile_k();
    pl.big = true;
    pl.fm = pl.fn = 0;
    const int mt = (Mr + bm - 1) / bm, nt = (ncols + bn - 1) / bn;
    // TN: split K until the tiles fill both CTA slots of every SM (c4 at
    // m_a <= 64: 40 tiles on 148 SMs unsplit), keeping >= 32 k-tiles a split
    int nsplit = 1;
    if (allow_split) {
      const int nkt = (K + bk - 1) / bk;
      while (nsplit < nsplit_max_ && mt * nt * nsplit < 2 * sms_ && nkt >= 2 * nsplit * 32)
        nsplit *= 2;
    }
    const int nkt = (K + bk - 1) / bk;
    pl.ksplit = ((nkt + nsplit - 1) / nsplit) * bk;
    pl.nsplit = (K + pl.ksplit - 1) / pl.ksplit;
    pl.grid = dim3(nt, mt, pl.nsplit);  // column tiles fastest (k_gemm_big)
    return pl;
  }
  pl.fn = ncols <= 8 ? 1 : (ncols <= 16 ? 2 : 4);
  const int nt = (ncols + 8 * pl.fn - 1) / (8 * pl.fn);
  pl.fm = 2;
  for (int fm : {8, 4}) {
    const int ctas = ((Mr + 8 * fm - 1) / (8 * fm)) * nt;
    if (ctas >= sms_) {
      pl.fm = fm;
      break;
    }
  }
  const int mt = (Mr + 8 * pl.fm - 1) / (8 * pl.fm);
  int nsplit = 1;
  if (allow_split) {
    const int nkt = (K + kBK - 1) / kBK;
    while (nsplit < nsplit_max_ && mt * nt * nsplit * 2 <= 2 * sms_ && nkt >= nsplit * 4)
      nsplit *= 2;
  }
  const int nkt = (K + kBK - 1) / kBK;
  const int kt_per = (nkt + nsplit - 1) / nsplit;
  pl.ksplit = kt_per * kBK;
  pl.nsplit = (K + pl.ksplit - 1) / pl.ksplit;
  if (pl.nsplit < 1) pl.nsplit = 1;
  pl.grid = dim3(mt, nt, pl.nsplit);
  return pl;
}

int Engine::launch_gemm(bool tn, int epi, const GemmPlan& pl, const double* Bsrc, int ldb,
                        double* C, int ldc, const int* act, const int* d_ncols,
                        long long split_stride, int part_ld) {
  GemmArgs g{};
  g.M = tn ? p : n;
  g.K = tn ? n : p;
  g.A = dX_;
  g.lda = n;
  g.B = Bsrc;
  g.ldb = ldb;
  g.C = C;
  g.ldc = ldc;
  g.split_stride = split_stride;
  g.ksplit = pl.ksplit;
  g.act = act;
  g.d_ncols = d_ncols;
  g.y = dy_;
  g.loss = loss;
  g.part_loss = dPL_;
  g.part_conj = dPC_;
  g.part_ld = part_ld;
  ++launches;
  g.tmap = pl.big ? (tn ? tmTN_ : tmNN_) : nullptr;
  if (pl.big)
    CK(gemm_big_launch(tn, epi, pl.grid, stream_, g));
  else
    CK(gemm_launch(tn, epi, pl.fm, pl.fn, pl.grid, stream_, g));
  return 0;
}

// Q = X'X and c = X'y for the Gram-form iteration gradient (once per engine;
// the TN product kernels, unsplit)
int Engine::gram_prepare() {
  if (dQ_) return 0;
  CK(cudaMallocAsync(&dQ_, sizeof(double) * (size_t)p * p, stream_));
  CK(cudaMallocAsync(&dCq_, sizeof(double) * (size_t)p, stream_));
  CK(cudaMallocAsync(&dGramCnt_, 2 * sizeof(int), stream_));
  const int cnt[2] = {p, 1};
  if (int rc = h2d(dGramCnt_, cnt, sizeof(cnt))) return rc;
  if (int rc = launch_gemm(true, EPI_STORE, plan(p, n, p, false), dX_, n, dQ_, p, nullptr, dGramCnt_,
                           0, mcap_))
    return rc;
  if (int rc = launch_gemm(true, EPI_STORE, plan(p, n, 1, false), dy_, n, dCq_, p, nullptr,
                           dGramCnt_ + 1, 0, mcap_))
    return rc;
  if (tmNN_ && p >= 132) {  // TMA descriptor of Q in the NN orientation
    auto enc = tmap_encoder();
    int nn[2], tn[2];
    gemm_big_boxes(nn, tn);
    CUtensorMap h;
    const cuuint64_t dims[2] = {(cuuint64_t)p, (cuuint64_t)p};
    const cuuint64_t strides[1] = {(cuuint64_t)p * sizeof(double)};
    const cuuint32_t box[2] = {(cuuint32_t)nn[0], (cuuint32_t)nn[1]};
    const cuuint32_t estr[2] = {1, 1};
    if (enc && enc(&h, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, dQ_, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS) {
      CK(cudaMallocAsync(&dTmapQ_, sizeof(h), stream_));
      CK(cudaMemcpyAsync(dTmapQ_, &h, sizeof(h), cudaMemcpyHostToDevice, stream_));
      CK(cudaStreamSynchronize(stream_));
    }
  }
  return 0;
}

// G[:, act] = Q V[:, act] - c (l' of the squared loss with y = c: EPI_DERIV)
int Engine::launch_gram(const GemmPlan& pl, const double* Bsrc, int ldb, double* C, int ldc,
                        const int* act, const int* d_ncols) {
  GemmArgs g{};
  g.M = p;
  g.K = p;
  g.A = dQ_;
  g.lda = p;
  g.B = Bsrc;
  g.ldb = ldb;
  g.C = C;
  g.ldc = ldc;
  g.split_stride = 0;
  g.ksplit = pl.ksplit;
  g.act = act;
  g.d_ncols = d_ncols;
  g.y = dCq_;
  g.loss = kSquared;
  g.part_ld = mcap_;
  ++launches;
  g.tmap = pl.big ? dTmapQ_ : nullptr;
  if (pl.big)
    CK(gemm_big_launch(false, EPI_DERIV, pl.grid, stream_, g));
  else
    CK(gemm_launch(false, EPI_DERIV, pl.fm, pl.fn, pl.grid, stream_, g));
  return 0;
}

// ---------------------------------------------------------------------------
// smoothness_constant (losses.hpp:86-112): start vector from xoshiro256++
// seeded 0x5eed5eed on the host, GEMVs and reductions on the device.
// ---------------------------------------------------------------------------
int Engine::compute_smoothness(double* out) {
  const double c = loss == kSquared ? 1.0 : 0.25;
  std::vector<double> v(p);
  Xoshiro256pp rng(0x5eed5eedULL);
  for (int j = 0; j < p; ++j) v[j] = rng.uniform() - 0.5;
  auto vnorm = [&](const std::vector<double>& a) {
    double s = 0.0;
    for (double x : a) s += x * x;
    return std::sqrt(s);
  };
  if (vnorm(v) == 0.0) v[0] = 1.0;
  {
    const double nv = vnorm(v);
    for (double& x : v) x /= nv;
  }
  if (int rc = ensure_aux(sizeof(double) * ((size_t)2 * p + n + 4))) return rc;
  double* dv = static_cast<double*>(dAux_);
  double* dw = dv + p;
  double* dxv = dw + p;
  double* dps = dxv + n;  // {done, estimate, result, rounds}
  if (int rc_ = h2d(dv, v.data(), sizeof(double) * p)) return rc_;
  const double ps0[4] = {0.0, 0.0, -1.0, 0.0};
  if (int rc_ = h2d(dps, ps0, sizeof(ps0))) return rc_;
  // rounds are launched in batches with the stopping test on the device, so
  // the host synchronises once per batch instead of once per round; the
  // arithmetic is the oracle's sequential order (bit-identical L)
  double ps[4] = {0.0, 0.0, -1.0, 0.0};
  // small p: one cooperative kernel loops the rounds on the device (every
  // column of X'(X v) gets its own warp; no host synchronisation between
  // rounds).  Larger p: the graph below (more columns in flight per round).
  // BNBG_PW_COOP=0 forces the graph.
  {
    const char* ce = getenv("BNBG_PW_COOP");
    int coop = 0, nb = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    if (coop && !(ce && ce[0] == '0') &&
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_pw_all, 256, 0) == cudaSuccess &&
        nb >= 1 && (p + 7) / 8 <= nb * sms_) {
      const int G = std::max((p + 7) / 8, std::min(sms_, (n + 255) / 256));
      int nn_ = n, pp_ = p;
      const double* Xc = dX_;
      void* args[] = {&nn_, &pp_, &Xc, &dv, &dxv, &dw, &dps};
      ++launches;
      CK(cudaLaunchCooperativeKernel((const void*)k_pw_all, dim3(G), dim3(256), args, 0, stream_));
      if (int rc_ = d2h(ps, dps, sizeof(ps))) return rc_;
      CK(cudaStreamSynchronize(stream_));
      double result = ps[2];
      if (result < 0.0) result = std::max(1.01 * c * ps[1], 1e-12);
      *out = result;
      return 0;
    }
    (void)cudaGetLastError();
  }
  // 8 rounds (24 kernels) captured once as a CUDA graph and replayed: the
  // kernels of rounds past the stop or past round 100 return at once
  constexpr int kRounds = 8;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  CK(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
  for (int b = 0; b < kRounds; ++b) {
    k_pw_xv<<<(n + 255) / 256, 256, 0, stream_>>>(n, p, dX_, dv, dxv, dps);
    k_pw_xtv<<<(p + 7) / 8, 256, 0, stream_>>>(n, p, dX_, dxv, dw, dps);  // a warp per column
    k_pw_step<<<1, 256, 0, stream_>>>(p, dw, dv, dps);
  }
  const cudaError_t ce = cudaStreamEndCapture(stream_, &graph);
  if (ce != cudaSuccess) return cuda_fail(ce, "power iteration: graph capture");
  cudaError_t ge = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ge != cudaSuccess) return cuda_fail(ge, "power iteration: graph instantiate");
  for (int launched = 0; launched < 100; launched += kRounds) {
    launches += 3 * kRounds;
    ge = cudaGraphLaunch(exec, stream_);
    if (ge != cudaSuccess) break;
    if (int rc_ = d2h(ps, dps, sizeof(ps))) {
      cudaGraphExecDestroy(exec);
      return rc_;
    }
    ge = cudaStreamSynchronize(stream_);
    if (ge != cudaSuccess || ps[0] != 0.0) break;
  }
  cudaGraphExecDestroy(exec);
  if (ge != cudaSuccess) return cuda_fail(ge, "power iteration");
  const double estimate = ps[1];
  double result = ps[2];
  if (result < 0.0) result = std::max(1.01 * c * estimate, 1e-12);
  *out = result;
  return 0;
}

// ---------------------------------------------------------------------------
// one proximal-gradient iteration over the active columns
// (relaxation.hpp:225-244)
// ---------------------------------------------------------------------------
int Engine::step(int ma, double eta, double rho, const RelaxParams& cfg) {
  int tn_split = 1;
  if (gram_) {  // G = Q V - c, one product, one slab
    tic(KC_GEMM_TN);
    if (int rc = launch_gram(plan(p, p, ma, false, dTmapQ_ != nullptr), dV_, p, dG_, p, dAct_, dMa_))
      return rc;
    toc(KC_GEMM_TN, 2.0 * p * p * ma);
  } else if (int rc = step_products(ma, tn_split)) {
    return rc;
  }
  return step_prox(ma, eta, rho, cfg, tn_split);
}

int Engine::step_products(int ma, int& tn_split) {
  const GemmPlan p1 = plan(n, p, ma, false);
  tic(KC_GEMM_NN);
  if (ma >= oz_min_ && ozaki_enabled()) {  // tcgen05 kind::i8 emulated FP64 + l' epilogue
    if (int rc = gemm_ozaki(false, true, dV_, p, dAct_, ma, dMa_, dR_, n, 0, nullptr)) return rc;
  } else if (int rc = launch_gemm(false, EPI_DERIV, p1, dV_, p, dR_, n, dAct_, dMa_, 0, mcap_)) {
    return rc;
  }
  toc(KC_GEMM_NN, 2.0 * n * p * ma);
  const GemmPlan p2 = plan(p, n, ma, true);
  tic(KC_GEMM_TN);
  tn_split = p2.nsplit;
  if (ma >= oz_min_ && ozaki_enabled()) {  // tcgen05 kind::i8 emulated FP64 (ozaki.cuh)
    if (int rc = gemm_ozaki(true, false, dR_, n, dAct_, ma, dMa_, dG_, p, (long long)p * mcap_, &tn_split))
      return rc;
  } else if (int rc = launch_gemm(true, EPI_STORE, p2, dR_, n, dG_, p, dAct_, dMa_,
                                  (long long)p * mcap_, mcap_)) {
    return rc;
  }
  toc(KC_GEMM_TN, 2.0 * n * p * ma);
  return 0;
}

int Engine::step_prox(int ma, double eta, double rho, const RelaxParams& cfg, int tn_split) {
  cur_nsplit_ = tn_split;
  RelaxDev r{};
  r.p = p;
  r.n2 = n2_;
  r.mcap = mcap_;
  r.B = dB_;
  r.V = dV_;
  r.G = dG_;
  r.split_stride = (long long)p * mcap_;
  r.nsplit = tn_split;
  r.state = dState_;
  r.kbar = dKbar_;
  r.pf = dPf_;
  r.t = dT_;
  r.best = dBest_;
  r.last_gap = dLast_;
  r.frozen = dFrozen_;
  r.status = dStatus_;
  r.iters = dIters_;
  r.act = dAct_;
  r.d_ma = dMa_;
  r.d_err = dErr_;
  r.eta = eta;
  r.rho = rho;
  r.M = M;
  r.lambda2 = lambda2;
  r.accel = cfg.acceleration;
  r.colscr = colstride_ ? dColScr_ : nullptr;
  r.colstride = colstride_;
  tic(KC_PROX);
  ++launches;
  CK(launch_prox_fista(colE_, ma, csmem_, stream_, r));
  toc(KC_PROX, 0.0);
  return 0;
}

// evaluate_bounds (relaxation.hpp:194-221) + active-list compaction
int Engine::evaluate(int ma, double eta, double rho, const RelaxParams& cfg, int iter, double thr,
                     double* trace, int eval_idx) {
  const GemmPlan p1 = plan(n, p, ma, false);
  tic(KC_GEMM_NN);
  if (int rc = launch_gemm(false, EPI_EVAL, p1, dB_, p, dR_, n, dAct_, dMa_, 0, mcap_)) return rc;
  toc(KC_GEMM_NN, 2.0 * n * p * ma);
  const GemmPlan p2 = plan(p, n, ma, true);
  tic(KC_GEMM_TN);
  if (int rc = launch_gemm(true, EPI_STORE, p2, dR_, n, dG_, p, dAct_, dMa_,
                           (long long)p * mcap_, mcap_))
    return rc;
  toc(KC_GEMM_TN, 2.0 * n * p * ma);
  RelaxDev r{};
  r.p = p;
  r.n2 = n2_;
  r.mcap = mcap_;
  r.B = dB_;
  r.V = dV_;
  r.G = dG_;
  r.split_stride = (long long)p * mcap_;
  r.nsplit = p2.nsplit;
  r.state = dState_;
  r.kbar = dKbar_;
  r.pf = dPf_;
  r.t = dT_;
  r.best = dBest_;
  r.last_gap = dLast_;
  r.frozen = dFrozen_;
  r.status = dStatus_;
  r.iters = dIters_;
  r.act = dAct_;
  r.d_ma = dMa_;
  r.d_err = dErr_;
  r.eta = eta;
  r.rho = rho;
  r.M = M;
  r.lambda2 = lambda2;
  r.accel = cfg.acceleration;
  r.colscr = colstride_ ? dColScr_ : nullptr;
  r.colstride = colstride_;
  EvalArgs e;
  e.part_loss = dPL_;
  e.part_conj = dPC_;
  e.nrb = p1.big ? p1.grid.y : p1.grid.x;  // row blocks of the NN partial sums
  e.part_ld = mcap_;
  e.iter = iter;
  e.prune_threshold = thr;
  e.gap_tolerance = cfg.gap_tolerance;
  e.trace = trace;
  e.eval_idx = eval_idx;
  tic(KC_EVAL);
  ++launches;
  CK(launch_eval(colE_, ma, csmem_, stream_, r, e));
  k_compact<<<1, 1024, 0, stream_>>>(dAct_, dMa_, dFrozen_);
  CKL("k_compact");
  toc(KC_EVAL, 0.0);
  if (int rc_ = d2h(hPin_, dMa_, sizeof(int))) return rc_;
  if (int rc_ = d2h(hPin_ + 1, dErr_, sizeof(int))) return rc_;
  CK(cudaStreamSynchronize(stream_));
  resolve_timing();
  if (hPin_[1] != 0x7fffffff) {
    return fail(2, "relaxation: non-finite iterate in column " + std::to_string(hPin_[1]));
  }
  return 0;
}

// The relaxation of a narrow batch as one persistent cooperative kernel
// (pass_kernel.cuh).  Same per-phase code as the multi-kernel path.
int Engine::run_pass(int m, const RelaxParams& cfg, double thr, double eta, double rho,
                     double* dTrace, int& iter, int& n_evals, long long& node_its) {
  PassArgs a{};
  RelaxDev& r = a.r;
  r.p = p;
  r.n2 = n2_;
  r.mcap = mcap_;
  r.B = dB_;
  r.V = dV_;
  r.G = dG_;
  r.split_stride = (long long)p * mcap_;
  r.nsplit = 1;
  r.state = dState_;
  r.kbar = dKbar_;
  r.pf = dPf_;
  r.t = dT_;
  r.best = dBest_;
  r.last_gap = dLast_;
  r.frozen = dFrozen_;
  r.status = dStatus_;
  r.iters = dIters_;
  r.act = dAct_;
  r.d_ma = dMa_;
  r.d_err = dErr_;
  r.eta = eta;
  r.rho = rho;
  r.M = M;
  r.lambda2 = lambda2;
  r.accel = cfg.acceleration;
  r.colscr = colstride_ ? dColScr_ : nullptr;
  r.colstride = colstride_;
  GemmArgs& g1 = a.nn;
  g1.M = n;
  g1.K = p;
  g1.A = dX_;
  g1.lda = n;
  g1.B = dV_;
  g1.ldb = p;
  g1.C = dR_;
  g1.ldc = n;
  g1.split_stride = 0;
  g1.ksplit = ((p + kBK - 1) / kBK) * kBK;
  g1.act = dAct_;
  g1.d_ncols = dMa_;
  g1.y = dy_;
  g1.loss = loss;
  g1.part_loss = dPL_;
  g1.part_conj = dPC_;
  g1.part_ld = mcap_;
  GemmArgs& g2 = a.tn;
  g2 = g1;
  g2.M = p;
  g2.K = n;
  g2.B = dR_;
  g2.ldb = n;
  g2.C = dG_;
  g2.ldc = p;
  g2.split_stride = (long long)p * mcap_;
  a.n = n;
  a.p = p;
  a.max_it = cfg.max_iterations;
  a.check = cfg.check_interval;
  a.gap_tol = cfg.gap_tolerance;
  a.prune_thr = thr;
  a.trace = dTrace;
  a.out = dPassOut_;
  a.prof = dPassProf_;
  r.probe = dPassProf_ ? dPassProf_ + 16 : nullptr;
  a.nn.probe = dPassProf_ ? dPassProf_ + 20 : nullptr;
  a.tn.probe = dPassProf_ ? dPassProf_ + 24 : nullptr;
  a.bar = dBar_;
  const bool clus = resc_.on && m <= cluster_max_m_;
  a.res = clus ? resc_ : res_;
  a.gram = gram_ ? 1 : 0;
  a.gram_local = gram_local_off_;
  a.gram_c = dCq_;
  if (gram_) {  // G = Q V - c (streaming 16-row tiles of Q, L2-resident)
    GemmArgs& gq = a.gq;
    gq = g1;
    gq.M = p;
    gq.K = p;
    gq.A = dQ_;
    gq.lda = p;
    gq.B = dV_;
    gq.ldb = p;
    gq.C = dG_;
    gq.ldc = p;
    gq.ksplit = ((p + kBK - 1) / kBK) * kBK;
    gq.y = dCq_;
    gq.loss = kSquared;
    gq.tmap = nullptr;
    gq.probe = nullptr;
  }
  a.big = ((n % 2) == 0 && (p % 2) == 0) ? big_min_ : 0;
  a.nn.tmap = res_.on ? nullptr : tmNN_;  // streaming mode's 128 x 64 tiles
  a.tn.tmap = res_.on ? nullptr : tmTN_;
  if (!clus) CK(cudaMemsetAsync(dBar_, 0, sizeof(unsigned), stream_));
  tic(KC_PASS);
  cudaError_t e = cudaSuccess;
  if (clus)
    e = pass_launch(colE_, resc_.cluster, pass_smem_c_, stream_, &a, resc_.cluster);
  else
    e = pass_launch(colE_, pass_grid_, pass_smem_, stream_, &a);
  ++launches;
  CK(e);
  toc(KC_PASS, 0.0);  // end event right behind the kernel, before the readback sync
  // the counters and the error word are read back with the pass's other
  // results (relax_uploaded: one synchronisation); a traced pass needs its
  // evaluation count first
  if (int rc = d2h_defer(pass_out_h_, dPassOut_, 3 * sizeof(long long))) return rc;
  if (int rc = d2h(hPin_ + 1, dErr_, sizeof(int))) return rc;
  pass_pending_ = true;
  if (dTrace) {
    if (int rc = sync_flush()) return rc;
    return finish_pass(iter, n_evals, node_its);
  }
  return 0;
}

int Engine::finish_pass(int& iter, int& n_evals, long long& node_its) {
  pass_pending_ = false;
  iter = (int)pass_out_h_[0];
  n_evals = (int)pass_out_h_[1];
  node_its = pass_out_h_[2];
  // FP64 work performed per node-iteration: X V and X'R (4np), or Q V (2p^2)
  // in the Gram form -- evaluations excluded
  kc_flops[KC_PASS] += (gram_ ? 2.0 * p * p : 4.0 * n * p) * (double)node_its;
  resolve_timing();
  if (hPin_[1] != 0x7fffffff)
    return fail(2, "relaxation: non-finite iterate in column " + std::to_string(hPin_[1]));
  return 0;
}

int Engine::relax_uploaded(int m, const RelaxParams& cfg, double thr, bool want_trace,
                           PassResult& out, bool round_select, const int* d_one_off,
                           const int* d_one_idx, const int* d_one_len, bool read_beta) {
  const double eta = 1.0 / L;  // relaxation.hpp:177-180
  const double rho = 1.0 / (2.0 * eta * lambda2);
  const int max_evals = cfg.max_iterations / std::max(1, cfg.check_interval) + 2;
  double* dTrace = nullptr;
  if (want_trace) {
    CK(cudaMallocAsync(&dTrace, sizeof(double) * (size_t)max_evals * mcap_, stream_));
    CK(cudaMemsetAsync(dTrace, 0xff, sizeof(double) * (size_t)max_evals * mcap_, stream_));
  }
  const int big = 0x7fffffff;
  if (int rc_ = h2d(dErr_, &big, sizeof(int))) return rc_;
  if (int rc_ = h2d(dMa_, &m, sizeof(int))) return rc_;
  int iter = 0, last_eval = 0, ma = m, n_evals = 0;
  long long node_its = 0;
  int rc = 0;
  // The persistent kernel wins when an iteration is latency-bound (narrow
  // batches, X resident); when one iteration's X V + X'R is large (c4-sized
  // X), the standalone GEMM kernels (two CTAs per SM) run faster and launch
  // gaps no longer matter.
  const double iter_flops = gram_ ? 2.0 * p * (double)p * m : 4.0 * n * (double)p * m;
  if (gram_)
    if ((rc = gram_prepare())) goto done;
  if (pass_grid_ > 0 && (res_.on || (m <= 2 * sms_ && iter_flops <= persist_max_flops_))) {
    // narrow batch: the whole relaxation as one persistent cooperative kernel
    if ((rc = run_pass(m, cfg, thr, eta, rho, dTrace, iter, n_evals, node_its))) goto done;
  } else {
    while (iter < cfg.max_iterations && ma > 0) {
      const int to_check = cfg.check_interval - iter % cfg.check_interval;
      const int nsteps = std::min(to_check, cfg.max_iterations - iter);
      for (int s = 0; s < nsteps; ++s) {
        if ((rc = step(ma, eta, rho, cfg))) goto done;
      }
      node_its += (long long)nsteps * ma;
      iter += nsteps;
      if (iter % cfg.check_interval == 0) {
        if ((rc = evaluate(ma, eta, rho, cfg, iter, thr, dTrace, n_evals))) goto done;
        ++n_evals;
        last_eval = iter;
        ma = hPin_[0];
      }
    }
    if (ma > 0 && last_eval != iter) {
      if ((rc = evaluate(ma, eta, rho, cfg, iter, thr, dTrace, n_evals))) goto done;
      ++n_evals;
    }
  }
  if (read_beta) out.beta.resize((size_t)p * m);
  out.bounds.resize(m);
  out.status.resize(m);
  out.iters.resize(m);
  if (round_select) {
    ++launches;
    CK(launch_round_select(colE_, m, csmem_, stream_, p, n2_, std::max(k, 1), dB_, dState_, dKbar_,
                           d_one_off, d_one_idx, d_one_len, dSup_, dLen_, dJb_,
                           colstride_ ? dColScr_ : nullptr, colstride_));
    out.sup.resize((size_t)m * std::max(k, 1));
    out.len.resize(m);
    out.jbranch.resize(m);
    if (int rc_ = d2h_defer(out.sup.data(), dSup_, sizeof(int) * out.sup.size())) return rc_;
    if (int rc_ = d2h_defer(out.len.data(), dLen_, sizeof(int) * m)) return rc_;
    if (int rc_ = d2h_defer(out.jbranch.data(), dJb_, sizeof(int) * m)) return rc_;
  }
  if (read_beta) {
    if (int rc_ = d2h_defer(out.beta.data(), dB_, sizeof(double) * (size_t)p * m)) return rc_;
  } else {
    out.beta.clear();
  }
  if (int rc_ = d2h_defer(out.bounds.data(), dBest_, sizeof(double) * m)) return rc_;
  if (int rc_ = d2h_defer(out.status.data(), dStatus_, sizeof(int) * m)) return rc_;
  if (int rc_ = d2h_defer(out.iters.data(), dIters_, sizeof(int) * m)) return rc_;
  if (want_trace) {
    out.trace.resize((size_t)n_evals * m);
    for (int e = 0; e < n_evals; ++e)
      if (int rc_ = d2h_defer(out.trace.data() + (size_t)e * m, dTrace + (size_t)e * mcap_,
                              sizeof(double) * m))
        return rc_;
  }
  if (int rc_ = sync_flush()) return rc_;
  if (pass_pending_)
    if ((rc = finish_pass(iter, n_evals, node_its))) goto done;
  out.iterations = iter;
  out.node_iterations = node_its;
  out.n_evals = n_evals;
  resolve_timing();
done:
  if (dTrace) dfree(dTrace);
  return rc;
}

int Engine::relax_raw(int m, const RelaxParams& cfg, double thr, const uint8_t* state,
                      const int32_t* kbar, const double* warm, bool trace, PassResult& out) {
  if (m <= 0) return fail(1, "solve_batch_relaxation: empty batch");
  if (int rc = ensure(m)) return rc;
  if (int rc_ = h2d(dState_, state, (size_t)p * m)) return rc_;
  if (int rc_ = h2d(dKbar_, kbar, sizeof(int) * m)) return rc_;
  if (int rc_ = h2d(dB_, warm, sizeof(double) * (size_t)p * m)) return rc_;
  k_init_cols<<<m, kNodeThreads, 0, stream_>>>(p, m, dState_, dPf_, dB_, dV_, dT_, dBest_, dLast_,
                                              dFrozen_, dStatus_, dIters_, dAct_,
                                              cfg.max_iterations);
  CKL("k_init_cols");
  return relax_uploaded(m, cfg, thr, trace, out, false, nullptr, nullptr, nullptr, true);
}

int Engine::relax_lists(const BatchLists& L_, const double* warm, const RelaxParams& cfg,
                        double thr, bool trace, PassResult& out) {
  const int m = L_.m;
  if (m <= 0) return fail(1, "solve_batch_relaxation: empty batch");
  if (int rc = ensure(m)) return rc;
  const size_t nz = L_.z_idx.size(), no = L_.o_idx.size();
  const size_t ints = (size_t)(m + 1) * 2 + nz + no;
  const size_t bytes = sizeof(double) * (size_t)p * m + sizeof(int) * (ints + 4);
  if (int rc = ensure_aux(bytes)) return rc;
  double* dWarm = static_cast<double*>(dAux_);
  int* dz_off = reinterpret_cast<int*>(dWarm + (size_t)p * m);
  int* do_off = dz_off + (m + 1);
  int* dz_idx = do_off + (m + 1);
  int* do_idx = dz_idx + nz;
  if (int rc_ = h2d(dWarm, warm, sizeof(double) * (size_t)p * m)) return rc_;
  if (int rc_ = h2d(dz_off, L_.z_off.data(), sizeof(int) * (m + 1))) return rc_;
  if (int rc_ = h2d(do_off, L_.o_off.data(), sizeof(int) * (m + 1))) return rc_;
  if (nz)
    if (int rc_ = h2d(dz_idx, L_.z_idx.data(), sizeof(int) * nz)) return rc_;
  if (no)
    if (int rc_ = h2d(do_idx, L_.o_idx.data(), sizeof(int) * no)) return rc_;
  k_pack<<<m, 256, 0, stream_>>>(p, k, m, dz_off, dz_idx, do_off, do_idx, dState_, dKbar_, dPf_,
                                 dWarm, dB_, dV_, dT_, dBest_, dLast_, dFrozen_, dStatus_, dIters_,
                                 dAct_, cfg.max_iterations);
  CKL("k_pack");
  return relax_uploaded(m, cfg, thr, trace, out, true, do_off, do_idx, nullptr, true);
}

int Engine::pack_lists(const BatchLists& L_, uint8_t* state_out, int* kbar_out, int* pf_out) {
  const int m = L_.m;
  if (m <= 0) return fail(1, "batch meta: empty batch");
  if (int rc = ensure(m)) return rc;
  const size_t nz = L_.z_idx.size(), no = L_.o_idx.size();
  const size_t ints = (size_t)(m + 1) * 2 + nz + no;
  const size_t bytes = sizeof(double) * (size_t)p * m + sizeof(int) * (ints + 4);
  if (int rc = ensure_aux(bytes)) return rc;
  double* dWarm = static_cast<double*>(dAux_);
  int* dz_off = reinterpret_cast<int*>(dWarm + (size_t)p * m);
  int* do_off = dz_off + (m + 1);
  int* dz_idx = do_off + (m + 1);
  int* do_idx = dz_idx + nz;
  CK(cudaMemsetAsync(dWarm, 0, sizeof(double) * (size_t)p * m, stream_));
  if (int rc_ = h2d(dz_off, L_.z_off.data(), sizeof(int) * (m + 1))) return rc_;
  if (int rc_ = h2d(do_off, L_.o_off.data(), sizeof(int) * (m + 1))) return rc_;
  if (nz)
    if (int rc_ = h2d(dz_idx, L_.z_idx.data(), sizeof(int) * nz)) return rc_;
  if (no)
    if (int rc_ = h2d(do_idx, L_.o_idx.data(), sizeof(int) * no)) return rc_;
  k_pack<<<m, 256, 0, stream_>>>(p, k, m, dz_off, dz_idx, do_off, do_idx, dState_, dKbar_, dPf_,
                                 dWarm, dB_, dV_, dT_, dBest_, dLast_, dFrozen_, dStatus_, dIters_,
                                 dAct_, 1);
  CKL("k_pack");
  if (int rc_ = d2h(state_out, dState_, (size_t)p * m)) return rc_;
  if (int rc_ = d2h(kbar_out, dKbar_, sizeof(int) * m)) return rc_;
  if (int rc_ = d2h(pf_out, dPf_, sizeof(int) * m)) return rc_;
  CK(cudaStreamSynchronize(stream_));
  return 0;
}

int Engine::round_select(int m, const double* beta, const uint8_t* state, const int32_t* kbar,
                         const int32_t* one_off, const int32_t* one_idx, int32_t* sup,
                         int32_t* len, int32_t* jb) {
  if (m <= 0) return 0;
  if (int rc = ensure(m)) return rc;
  const int no = one_off ? one_off[m] : 0;
  if (int rc = ensure_aux(sizeof(int) * ((size_t)m + 1 + no + 1))) return rc;
  int* d_off = static_cast<int*>(dAux_);
  int* d_idx = d_off + m + 1;
  if (int rc_ = h2d(dB_, beta, sizeof(double) * (size_t)p * m)) return rc_;
  if (int rc_ = h2d(dState_, state, (size_t)p * m)) return rc_;
  if (int rc_ = h2d(dKbar_, kbar, sizeof(int) * m)) return rc_;
  if (one_off) {
    if (int rc_ = h2d(d_off, one_off, sizeof(int) * (m + 1))) return rc_;
    if (no)
      if (int rc_ = h2d(d_idx, one_idx, sizeof(int) * no)) return rc_;
  }
  ++launches;
  CK(launch_round_select(colE_, m, csmem_, stream_, p, n2_, std::max(k, 1), dB_, dState_, dKbar_,
                         one_off ? d_off : nullptr, one_off ? d_idx : nullptr, nullptr, dSup_, dLen_,
                         dJb_, colstride_ ? dColScr_ : nullptr, colstride_));
  if (sup)
    if (int rc_ = d2h(sup, dSup_, sizeof(int) * (size_t)m * std::max(k, 1))) return rc_;
  if (len) if (int rc_ = d2h(len, dLen_, sizeof(int) * m)) return rc_;
  if (jb) if (int rc_ = d2h(jb, dJb_, sizeof(int) * m)) return rc_;
  CK(cudaStreamSynchronize(stream_));
  resolve_timing();
  return 0;
}

// reoptimize_supports (primal_heuristics.hpp:174-227)
int Engine::reoptimize(int nsup, const int* offsets, const int* idx, double* coef, double* obj) {
  if (nsup <= 0) return 0;
  const int tot = offsets[nsup];
  int qmax = 0;
  for (int s = 0; s < nsup; ++s) qmax = std::max(qmax, offsets[s + 1] - offsets[s]);
  const bool gram = loss == kSquared && qmax <= 32;
  // cluster gather form: X_S slice in registers, CS CTAs per support
  int cs = 0, rpt = 0;
  if (!gram && qmax <= 16) {
    const int qm = qmax <= 8 ? 8 : 16;
    const int rpt_max = 64 / qm;
    // every (destination, value) pair of the exchange needs its own thread
    const int cs_cap = std::min(kReoptMaxCluster, kReoptClusterThreads / qm);
    for (int c = 1; c <= cs_cap; c <<= 1) {
      const int rows = (n + c - 1) / c;
      const int need = (rows + kReoptClusterThreads - 1) / kReoptClusterThreads;
      if (need <= rpt_max) {
        cs = c;
        break;
      }
    }
    if (cs) {
      const char* env = getenv("BNBG_REOPT_CS");
      if (env && atoi(env) > 0) {
        cs = std::max(cs, std::min(cs_cap, atoi(env)));
      } else {
        while (cs < cs_cap && nsup * cs * 2 <= sms_) cs <<= 1;
      }
      const int rows = (n + cs - 1) / cs;
      const int need = (rows + kReoptClusterThreads - 1) / kReoptClusterThreads;
      rpt = need <= 1 ? 1 : need <= 2 ? 2 : need <= 4 ? 4 : 8;
    }
  }
  // large n: X_S slices in shared memory, 8 or 16 CTAs per support
  // (BNBG_REOPT_SMEM=0 falls back to the per-CTA gather form)
  int cs_smem = 0;
  static const bool smem_ok = [] {
    const char* e = getenv("BNBG_REOPT_SMEM");
    return !(e && e[0] == '0');
  }();
  if (smem_ok && !gram && !cs && qmax <= 16) {
    for (int c : {8, 16}) {
      if (reopt_smem_bytes(n, qmax, c) <= 200 * 1024) {
        cs_smem = c;
        break;
      }
    }
    // Very many supports: the shared-memory slices run only sms / cs
    // supports at a time, each on cs SMs; the per-CTA gather form runs them
    // all at once, reading X_S from L2.  Measured at c4 (30 s runs): gather
    // form everywhere 7.6 s of re-opt against 5.7 s for the slices, so the
    // switch is kept for batches of more than 16 waves of clusters.
    // BNBG_REOPT_MODE=smem|direct forces one (measurements).
    static const char* mode = getenv("BNBG_REOPT_MODE");
    const bool force_smem = mode && mode[0] == 's', force_direct = mode && mode[0] == 'd';
    if (cs_smem && (force_direct || (!force_smem && nsup > 16 * (sms_ / cs_smem)))) cs_smem = 0;
  }
  const bool direct = !gram && !cs && !cs_smem && qmax <= 16;
  // the deriv scratch is only used by the generic kernel
  const size_t scr = (gram || direct || cs || cs_smem) ? 0 : (size_t)nsup * n;
  const size_t bytes = sizeof(double) * (scr + tot + nsup + 2) +
                       sizeof(int) * ((size_t)2 * nsup + 1 + tot + 2);
  if (int rc = ensure_aux(bytes)) return rc;
  double* d_scr = static_cast<double*>(dAux_);
  double* d_coef = d_scr + scr;
  double* d_obj = d_coef + tot + 1;
  int* d_off = reinterpret_cast<int*>(d_obj + nsup + 1);
  int* d_idx = d_off + nsup + 1;
  int* d_its = d_idx + tot + 1;
  if (int rc_ = h2d(d_off, offsets, sizeof(int) * (nsup + 1))) return rc_;
  if (tot) if (int rc_ = h2d(d_idx, idx, sizeof(int) * tot)) return rc_;
  const double step = 1.0 / (L + 2.0 * lambda2);
  tic(KC_REOPT);
  if (gram) {
    k_reopt_gram<<<nsup, kReoptFastThreads, 0, stream_>>>(n, dX_, dy_, M, lambda2, step, d_off,
                                                          d_idx, d_coef, d_obj, d_its);
    CKL("k_reopt_gram");
  } else if (cs) {
    ++launches;
    cudaError_t le = launch_reopt_cluster(qmax <= 8 ? 8 : 16, rpt, cs, nsup, stream_, n, dX_, dy_,
                                          loss, M, lambda2, step, d_off, d_idx, d_coef, d_obj, d_its);
    if (le != cudaSuccess && cs > 8) {  // 16-CTA clusters not schedulable here: portable size
      (void)cudaGetLastError();
      cs = 8;
      const int rows = (n + cs - 1) / cs;
      const int need = (rows + kReoptClusterThreads - 1) / kReoptClusterThreads;
      rpt = need <= 1 ? 1 : need <= 2 ? 2 : need <= 4 ? 4 : 8;
      le = launch_reopt_cluster(qmax <= 8 ? 8 : 16, rpt, cs, nsup, stream_, n, dX_, dy_, loss, M,
                                lambda2, step, d_off, d_idx, d_coef, d_obj, d_its);
    }
    CK(le);
  } else if (cs_smem) {
    ++launches;
    CK(launch_reopt_smem(qmax, cs_smem, nsup, stream_, n, dX_, dy_, loss, M, lambda2, step, d_off,
                         d_idx, d_coef, d_obj, d_its));
  } else if (qmax <= 8) {
    k_reopt_direct<8><<<nsup, kReoptFastThreads, 0, stream_>>>(
        n, dX_, dy_, loss, M, lambda2, step, d_off, d_idx, d_scr, d_coef, d_obj, d_its);
    CKL("k_reopt_direct");
  } else if (qmax <= 16) {
    k_reopt_direct<16><<<nsup, kReoptFastThreads, 0, stream_>>>(
        n, dX_, dy_, loss, M, lambda2, step, d_off, d_idx, d_scr, d_coef, d_obj, d_its);
    CKL("k_reopt_direct");
  } else {
    const size_t smem = sizeof(double) * (size_t)(kReoptThreads / 32 + 2) * std::max(qmax, 1);
    if (smem > 48 * 1024) {
      CK(cudaFuncSetAttribute(k_reopt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    }
    k_reopt<<<nsup, kReoptThreads, smem, stream_>>>(n, dX_, dy_, loss, M, lambda2, step, d_off,
                                                    d_idx, d_scr, d_coef, d_obj, d_its);
    CKL("k_reopt");
  }
  toc(KC_REOPT, 0.0);
  std::vector<int> its(nsup);
  if (tot) if (int rc_ = d2h_defer(coef, d_coef, sizeof(double) * tot)) return rc_;
  if (int rc_ = d2h_defer(obj, d_obj, sizeof(double) * nsup)) return rc_;
  if (int rc_ = d2h_defer(its.data(), d_its, sizeof(int) * nsup)) return rc_;
  if (int rc_ = sync_flush()) return rc_;
  // algorithmic work of the reference iteration: 4 q n flops per support-iteration
  double flops = 0.0;
  for (int s = 0; s < nsup; ++s) {
    flops += 4.0 * (offsets[s + 1] - offsets[s]) * (double)n * its[s];
    reopt_iterations += its[s];
  }
  kc_flops[KC_REOPT] += flops;
  resolve_timing();
  return 0;
}

int Engine::pass_profile(double* ns, int count) {
  if (!dPassProf_) return 0;
  unsigned long long h[32];
  CK(cudaMemcpy(h, dPassProf_, sizeof(h), cudaMemcpyDeviceToHost));
  // [0..6] phase totals, [8..14] CTA 0's time to the phase barrier,
  // [16..19] prox sub-phases of CTA 0 (load+sort, PAVA, scatter, barrier)
  // [28..29] PAVA sub-phases of CTA 0 (scan, walk), [30] walk steps, [31] walks
  const int c = std::min(count, 32);
  for (int i = 0; i < c; ++i) ns[i] = (double)h[i];
  return c;
}

int Engine::gemm_probe(int trans, int m, const double* Bh, double* Ch) {
  if (m <= 0) return 0;
  if (int rc = ensure(m)) return rc;
  const int K = trans ? n : p, Mo = trans ? p : n;
  if (int rc = ensure_aux(sizeof(double) * ((size_t)K * m + (size_t)Mo * m * nsplit_max_) + 64))
    return rc;
  double* dBin = static_cast<double*>(dAux_);
  double* dC = dBin + (size_t)K * m;
  if (int rc_ = h2d(dBin, Bh, sizeof(double) * (size_t)K * m)) return rc_;
  if (int rc_ = h2d(dMa_, &m, sizeof(int))) return rc_;
  const GemmPlan pl = plan(Mo, K, m, trans != 0);
  int ns = pl.nsplit;
  if (m >= oz_min_ && ozaki_enabled()) {
    if (int rc = gemm_ozaki(trans != 0, false, dBin, K, nullptr, m, dMa_, dC, Mo,
                            (long long)Mo * m, &ns))
      return rc;
  } else if (int rc = launch_gemm(trans != 0, EPI_STORE, pl, dBin, K, dC, Mo, nullptr, dMa_,
                                  (long long)Mo * m, m)) {
    return rc;
  }
  std::vector<double> slabs((size_t)Mo * m * ns);
  if (int rc_ = d2h(slabs.data(), dC, sizeof(double) * slabs.size())) return rc_;
  CK(cudaStreamSynchronize(stream_));
  for (size_t e = 0; e < (size_t)Mo * m; ++e) {
    double s = slabs[e];
    for (int t = 1; t < ns; ++t) s += slabs[(size_t)t * Mo * m + e];
    Ch[e] = s;
  }
  return 0;
}

}  // namespace bnbg

// ===========================================================================
// stateless kernel entry points (prox_kernel.hpp test surface)
// ===========================================================================
#include "../../include/bnbg.h"

namespace {

struct DevScratch {
  std::vector<void*> ptrs;
  ~DevScratch() {
    for (void* q : ptrs) cudaFree(q);
  }
  template <class T>
  T* alloc(size_t count, cudaError_t& e) {
    void* q = nullptr;
    if (e == cudaSuccess) e = cudaMalloc(&q, sizeof(T) * std::max<size_t>(count, 1));
    if (e == cudaSuccess) ptrs.push_back(q);
    return static_cast<T*>(q);
  }
};

thread_local std::string g_stateless_err;

int stateless_column_op(int device, int kind, int mode, int p, int m, const double* in,
                        const uint8_t* state, const int32_t* kbar, double w, double M,
                        double* out) {
  using namespace bnbg;
  if (p <= 0 || m <= 0) return BNBG_OK;
  cudaError_t e = cudaSetDevice(device);
  DevScratch s;
  const int n2 = next_pow2(std::max(p, 2));
  const int E = column_E(n2);
  size_t smem = column_smem_bytes(p, n2, E);
  // large p: column buffers in global memory (see Engine::create)
  const long long gstride = smem > 220 * 1024 ? (long long)((smem + 255) / 256 * 32) : 0;
  if (gstride) smem = 0;
  if (e == cudaSuccess) e = column_set_attrs(E, smem);
  double* gscr = gstride ? s.alloc<double>((size_t)gstride * m, e) : nullptr;
  double* din = s.alloc<double>((size_t)p * m, e);
  uint8_t* dst = s.alloc<uint8_t>((size_t)p * m, e);
  int* dkb = s.alloc<int>(m, e);
  const size_t outn = kind == 0 ? (size_t)p * m : (size_t)m;
  double* dout = s.alloc<double>(outn, e);
  if (e == cudaSuccess) e = cudaMemcpy(din, in, sizeof(double) * (size_t)p * m, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(dst, state, (size_t)p * m, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(dkb, kbar, sizeof(int) * m, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && kind == 0)
    e = launch_prox_standalone(E, m, smem, 0, mode, p, n2, din, dst, dkb, w, M, dout, gscr,
                               gstride);
  else if (e == cudaSuccess)
    e = launch_g_standalone(E, m, smem, 0, mode, p, n2, din, dst, dkb, M, dout, gscr, gstride);
  if (e == cudaSuccess) e = cudaMemcpy(out, dout, sizeof(double) * outn, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) {
    g_stateless_err = std::string("CUDA error: ") + cudaGetErrorString(e);
    return BNBG_CUDA_ERROR;
  }
  return BNBG_OK;
}

}  // namespace

extern "C" {

int bnbg_prox_step(int device, int p, int m, const double* U, double eta, double lambda2,
                   const uint8_t* state, const int32_t* kbar, double M, double* out) {
  if (!(eta > 0.0) || !(lambda2 > 0.0)) return BNBG_INPUT_ERROR;  // prox_kernel.hpp:288-289
  const double rho = 1.0 / (2.0 * eta * lambda2);
  return stateless_column_op(device, 0, 0, p, m, U, state, kbar, rho, M, out);
}

int bnbg_conjugate_prox(int device, int p, int m, const double* U_scaled, double weight,
                        const uint8_t* state, const int32_t* kbar, double M, double* out) {
  return stateless_column_op(device, 0, 1, p, m, U_scaled, state, kbar, weight, M, out);
}

int bnbg_g_value(int device, int p, int m, const double* beta, const uint8_t* state,
                 const int32_t* kbar, double M, double* out) {
  return stateless_column_op(device, 1, 0, p, m, beta, state, kbar, 0.0, M, out);
}

int bnbg_g_conjugate(int device, int p, int m, const double* q, const uint8_t* state,
                     const int32_t* kbar, double M, double* out) {
  return stateless_column_op(device, 1, 1, p, m, q, state, kbar, 0.0, M, out);
}

}  // extern "C"
