// engine.hpp -- one GPU's node-processing engine (host side of the seam).
//
// Owns the device-resident instance (X column-major, y), the batch
// workspaces sized for the widest batch seen, and the stream.  The relaxation
// loop runs entirely on the device between bound evaluations; the host reads
// back one integer (the active-column count) per check_interval iterations,
// exactly when the reference's active count can change
// (relaxation.hpp:224-250).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/bnbg.h"
#include "launchers.hpp"

namespace bnbg {

struct RelaxParams {
  int max_iterations = 2000;
  double gap_tolerance = 1e-6;
  int check_interval = 10;
  int acceleration = 1;
};

// Host-side batch description in CSR form (one entry per node/column).
struct BatchLists {
  int m = 0;
  std::vector<int> z_off, z_idx;  // J0 lists
  std::vector<int> o_off, o_idx;  // J1 lists (construction order)
};

struct PassResult {
  std::vector<double> beta;   // p x m
  std::vector<double> bounds; // m
  std::vector<int> status, iters;
  std::vector<int> sup, len, jbranch;  // m x k, m, m
  std::vector<double> trace;  // n_evals x m (NaN where not evaluated)
  int n_evals = 0;
  long long iterations = 0;       // loop iterations run
  long long node_iterations = 0;  // sum over columns of iterations
};

enum KernelClass { KC_GEMM_NN = 0, KC_GEMM_TN, KC_PROX, KC_EVAL, KC_REOPT, KC_PASS, KC_COUNT };

class Engine {
 public:
  Engine() = default;
  ~Engine();
  int init(const double* X, const double* y, int n, int p, int loss, int k, double M,
           double lambda2, double L, int device);

  // losses.hpp:86-112 on the device
  int compute_smoothness(double* out);

  // solve_batch_relaxation over columns already uploaded (state/kbar/B)
  int relax_uploaded(int m, const RelaxParams& cfg, double prune_threshold, bool trace,
                     PassResult& out, bool round_select, const int* d_one_off,
                     const int* d_one_idx, const int* d_one_len, bool read_beta);
  // bnbg_relax_batch: raw state/kbar/warm from the host
  int relax_raw(int m, const RelaxParams& cfg, double prune_threshold, const uint8_t* state,
                const int32_t* kbar, const double* warm, bool trace, PassResult& out);
  // one BnB pass of lower bounds + rounding + branch selection from CSR lists
  int relax_lists(const BatchLists& lists, const double* warm, const RelaxParams& cfg,
                  double prune_threshold, bool trace, PassResult& out);
  // the packer alone (bnbg_pack_batch): CSR lists -> state, kbar, free count
  int pack_lists(const BatchLists& lists, uint8_t* state_out, int* kbar_out, int* pf_out);
  // reoptimize_supports (CSR)
  int reoptimize(int nsup, const int* offsets, const int* idx, double* coef, double* obj);
  int round_select(int m, const double* beta, const uint8_t* state, const int32_t* kbar,
                   const int32_t* one_off, const int32_t* one_idx, int32_t* sup, int32_t* len,
                   int32_t* jb);
  int gemm_probe(int trans, int m, const double* B, double* C);

  // ---- device-resident node pool (pool.cu, pool_kernels.cuh) ----
  int pool_reserve(int cap);  // grow the pool to >= cap slots (contents kept)
  int pool_root(int slot);    // root_node (node_model.hpp:47-52) in `slot`
  int pool_capacity() const { return pool_cap_; }
  // one pass of lower bounds + rounding + branch selection over pool slots;
  // no warm start or beta crosses PCIe.  With `lists`, the batch's J0/J1
  // lists are read back (DebugHooks): n01 m x 2, j0 m x p, j1 m x k.
  int relax_pool(int m, const int* slots, const RelaxParams& cfg, double prune_threshold,
                 bool trace, PassResult& out, bool lists, std::vector<int>* n01,
                 std::vector<int>* j0, std::vector<int>* j1);
  // prune test + branch (bnb_engine.hpp:242-256, node_model.hpp:57-105) of the
  // last relax_pool batch: children go to free_slots[0 .. 2 survivors); one
  // record per child (slot, leaf, |J1|, depth, J1 list) plus its lower bound.
  // bad_column >= 0 reports a survivor without a free coordinate.
  int branch_pool(int m, const int* slots, const double* lb_in, double post_threshold,
                  const int* free_slots, int& survivors, int& bad_column, std::vector<int>& rec,
                  std::vector<double>& rec_lb);

  // ---- multi-GPU node exchange (comm.cu) ----
  size_t node_record_bytes() const;
  // pack `cnt` pool slots (with their bounds) into the send staging buffer
  int pool_pack(int cnt, const int* slots, const double* lbs, uint8_t** d_send);
  // receive staging buffer of `cnt` records
  int pool_recv_buffer(int cnt, uint8_t** d_recv);
  // unpack `cnt` received records into pool `slots`; bounds to lbs (host)
  int pool_unpack(int cnt, const int* slots, double* lbs);
  int comm_allgather_nccl(const void* send, size_t bytes, void* recv);
  int comm_exchange_nccl(int world, const int64_t* send_nodes, const uint8_t* d_send,
                         const int64_t* recv_nodes, uint8_t* d_recv, size_t rec_bytes);
  int comm_exchange_host(const bnbg_comm_ops* ops, const int64_t* send_nodes,
                         const uint8_t* d_send, const int64_t* recv_nodes, uint8_t* d_recv,
                         size_t rec_bytes);
  int nccl_init(const uint8_t* uid, int rank, int world);
  void comm_release();
  void* nccl_comm = nullptr;  // ncclComm_t
  int nccl_rank = 0, nccl_world = 1;

  int n = 0, p = 0, k = 0, loss = 0, device = 0;
  double M = 1.0, lambda2 = 1.0, L = 0.0;
  long long launches = 0;
  long long h2d_bytes = 0, d2h_bytes = 0;
  long long reopt_iterations = 0;  // support-iterations run by the re-opt kernels
  bool timing = false;
  double kc_ms[KC_COUNT] = {0};
  double kc_flops[KC_COUNT] = {0};
  long long kc_launches[KC_COUNT] = {0};
  std::string err;

 private:
  int ensure(int m);
  // stream-ordered device allocations (cudaMallocAsync on the engine stream):
  // freeing does not synchronise the device
  void dfree(void* q) {
    if (q) cudaFreeAsync(q, stream_);
  }
  int pool_cap_ = 0;
  void* pool_mem_[7] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  int* dSlots_ = nullptr;    // batch slot ids (m)
  double* dLbIn_ = nullptr;  // parents' lower bounds (m)
  double* dLbOut_ = nullptr;
  int* dPos_ = nullptr;      // child position of each survivor (m)
  int* dTot_ = nullptr;      // [0] survivors, [1] first bad column
  int* dFree_ = nullptr;     // free slots for children (2m)
  int* dRec_ = nullptr;      // child records (2m x (4 + k))
  double* dRecLb_ = nullptr; // (2m)
  int* dOneLen_ = nullptr;   // padded J1 lists of the batch (m, m x k)
  int* dOneIdx_ = nullptr;
  int* dLists_ = nullptr;    // DebugHooks list readback scratch
  int pool_batch_cap_ = 0;
  int ensure_pool_batch(int m);
  uint8_t* dXSend_ = nullptr;  // node-exchange staging
  uint8_t* dXRecv_ = nullptr;
  size_t xsend_bytes_ = 0, xrecv_bytes_ = 0;
  int* dXSlots_ = nullptr;
  double* dXLb_ = nullptr;
  int xslots_cap_ = 0;
  void* dGather_ = nullptr;  // NCCL allgather scratch
  size_t gather_bytes_ = 0;
  int ensure_aux(size_t bytes);
  int fail(int code, const std::string& msg);
  int cuda_fail(cudaError_t e, const char* what);
  int step(int ma, double eta, double rho, const RelaxParams& cfg);
  int step_products(int ma, int& tn_split);
  int step_prox(int ma, double eta, double rho, const RelaxParams& cfg, int tn_split);
  int run_pass(int m, const RelaxParams& cfg, double thr, double eta, double rho, double* dTrace,
               int& iter, int& n_evals, long long& node_its);
  int finish_pass(int& iter, int& n_evals, long long& node_its);
  long long pass_out_h_[4] = {0, 0, 0, 0};  // deferred readback of the pass counters
  bool pass_pending_ = false;
  int pass_grid_ = 0;       // CTAs of the persistent pass kernel (0: disabled)
  size_t pass_smem_ = 0;
  long long* dPassOut_ = nullptr;
  unsigned* dBar_ = nullptr;  // grid barrier counter of the pass kernel
  // TMA descriptors of X (global memory) for the 128 x 64 tiles' A operand:
  // NN box and TN box (gemm_big.cuh); nullptr when TMA staging is off
  void* dTmap_ = nullptr;
  const void* tmNN_ = nullptr;
  const void* tmTN_ = nullptr;
  int make_tmaps();
  // tcgen05 kind::i8 emulated-FP64 TN product (ozaki.cu; BNBG_OZAKI=1)
  bool ozaki_enabled() const;
  int ozaki_prepare_x(int side);
  int ozaki_reserve_b(int side, int m);
  int gemm_ozaki(bool tn, bool deriv, const double* Bsrc, int ldb, const int* act, int ma,
                 const int* d_ncols, double* C, int ldc, long long split_stride, int* nsplit);
  struct OzSide {             // [0] NN (X rows), [1] TN (X columns)
    void* dX = nullptr;       // X digits, pre-tiled [row tile][K block][digit][128][64 B]
    int* dEx = nullptr;       // per-row exponent
    void* dB = nullptr;       // batch digits, pre-tiled [col tile][K block][digit][bn][64 B]
    int* dEb = nullptr;
    int nkb = 0, bcap = 0;    // K blocks (64 B), batch capacity (multiple of 64)
  } oz_[2];
  ResLayout res_{};           // X residency plan (res_.on = 0: streaming)
  ResLayout resc_{};          // one-cluster plan for narrow batches (resc_.on = 0: none)
  size_t pass_smem_c_ = 0;    // its dynamic shared memory
  int cluster_max_m_ = 16;    // widest batch run by the one-cluster pass kernel
 public:
  unsigned long long* dPassProf_ = nullptr;  // phase wall times (BNBG_PASS_PROF=1)
  int pass_profile(double* ns, int count);
 private:
  int evaluate(int ma, double eta, double rho, const RelaxParams& cfg, int iter, double thr,
               double* trace, int eval_idx);
  struct GemmPlan {
    int fm, fn, nsplit, ksplit;
    bool big = false;  // gemm_big.cuh tile (wide batches)
    dim3 grid;
  };
  GemmPlan plan(int M, int K, int ncols, bool allow_split, bool allow_big = true) const;
  // Squared loss with p <= n: the iteration gradient G = X'(X V - y) is
  // formed as Q V - c with Q = X'X (p x p) and c = X'y computed once per
  // engine (2 p^2 flops per column instead of 4 n p, one product instead of
  // two).  The bound evaluations keep the X products (Psi from R = X B - y).
  // BNBG_GRAM=0 disables.
  bool gram_ = false;
  double* dQ_ = nullptr;
  double* dCq_ = nullptr;
  int* dGramCnt_ = nullptr;  // device {p, 1}: column counts of the setup products
  void* dTmapQ_ = nullptr;   // TMA descriptor of Q for the 128 x 64 tiles (p even, >= 132)
  int gram_prepare();
  long long gram_local_off_ = 0;  // pass kernel: double offset of the local-Gram region (0: off)
  int launch_gram(const GemmPlan& pl, const double* Bsrc, int ldb, double* C, int ldc,
                  const int* act, const int* d_ncols);
  int launch_gemm(bool tn, int epi, const GemmPlan& pl, const double* Bsrc, int ldb, double* C,
                  int ldc, const int* act, const int* d_ncols, long long split_stride,
                  int part_ld);
  void tic(int kc);
  void toc(int kc, double flops);
  void resolve_timing();
  int h2d(void* dst, const void* src, size_t bytes);
  int d2h(void* dst, const void* src, size_t bytes);
  // Readbacks into pageable host memory go through a pinned staging buffer:
  // d2h_defer queues an asynchronous copy into it, sync_flush synchronises the
  // stream once and copies every queued block out.  (A pageable
  // cudaMemcpyAsync blocks the host per call: ~10 us each, several per pass.)
  int d2h_defer(void* dst, const void* src, size_t bytes);
  int sync_flush();
  struct Deferred {
    void* dst;
    size_t off, bytes;
  };
  std::vector<Deferred> defer_;
  char* hStage_ = nullptr;  // pinned, kStageBytes, from the process-wide pool
  size_t stage_used_ = 0;
  bool defer_on_ = true;
  struct EvPair {
    cudaEvent_t a, b;
    int kc;
  };
  std::vector<EvPair> pending_;
  std::vector<cudaEvent_t> ev_pool_;
  cudaEvent_t cur_a_ = nullptr;
  cudaEvent_t get_event();

  cudaStream_t stream_ = nullptr;
  cudaEvent_t ev0_ = nullptr, ev1_ = nullptr;
  int n2_ = 1;
  int colE_ = 0;        // elements per thread of the register column sort
  size_t csmem_ = 0;    // dynamic shared memory of the column kernels
  long long colstride_ = 0;     // large p: column buffers in global memory, doubles per CTA
  double* dColScr_ = nullptr;   // ... mcap_ slices of them
  int sms_ = 148;
  int mcap_ = 0;
  double* dX_ = nullptr;
  double* dy_ = nullptr;
  double *dB_ = nullptr, *dV_ = nullptr, *dG_ = nullptr, *dR_ = nullptr;
  double *dPL_ = nullptr, *dPC_ = nullptr;
  double *dT_ = nullptr, *dBest_ = nullptr, *dLast_ = nullptr;
  uint8_t *dState_ = nullptr, *dFrozen_ = nullptr;
  int *dKbar_ = nullptr, *dPf_ = nullptr, *dStatus_ = nullptr, *dIters_ = nullptr;
  int *dAct_ = nullptr, *dMa_ = nullptr, *dErr_ = nullptr;
  int *dSup_ = nullptr, *dLen_ = nullptr, *dJb_ = nullptr;
  void* dAux_ = nullptr;  // CSR uploads, reopt scratch, trace
  size_t aux_bytes_ = 0;
  int* hPin_ = nullptr;   // pinned: [0] ma, [1] err
  int nsplit_max_ = 8;
  int big_min_ = 64;  // m_a from which the 128 x 64 register-tiled GEMM is used
  int oz_min_ = 16;   // m_a from which the standalone iteration GEMMs use the tcgen05 emulation
  double persist_max_flops_ = 4e9;  // streaming mode: persistent kernel up to this work per iteration
  int nrb_max_ = 1;
  int cur_nsplit_ = 1;
  int cur_nrb_ = 1;
};

}  // namespace bnbg
