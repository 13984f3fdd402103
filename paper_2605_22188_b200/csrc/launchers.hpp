// launchers.hpp -- host launchers of the sm_100a kernels, one translation
// unit per kernel family (gemm_kernels.cu, column_kernels.cu, pass_kernels.cu)
// so the template instantiations compile in parallel.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "gemm.cuh"
#include "node_kernels.cuh"

namespace bnbg {

// Shared-memory residency plan of X for the persistent pass kernel: CTA b
// keeps NN row tile b (rows [16 rt b, 16 rt (b+1)) x all p, k-major, stride
// lda_nn) and TN tile b (X columns [16 (b % tn_mt), +16) x rows of split
// b / tn_mt, row-major, stride ldk_tn) for the whole pass; only V / R move per
// iteration.  cluster > 0: the grid is ONE thread-block cluster of that many
// CTAs (small X, rt = 4), synchronised by cluster barriers.
struct ResLayout {
  int on;        // 0: stream X tiles from L2/HBM (gemm_tile)
  int nn_tiles;  // ceil(n / (16 rt))
  int kpad_nn;   // p rounded up to 4
  int lda_nn;    // 16 rt + 4 (conflict-free DMMA fragment loads)
  int rt;        // 16-row sub-tiles per NN tile (1 or 4)
  int cluster;   // 0: grid barriers over one CTA per SM; else the cluster size
  int tn_mt;     // ceil(p / 16)
  int tn_split;  // K splits of the n rows
  int tn_klen;   // rows per split (multiple of 4)
  int ldk_tn;    // >= tn_klen, = 4 mod 16
  int ldb;       // k-stride of the staged B operand, >= max(kpad_nn, tn_klen), = 4 mod 16
  long long off_tn, off_work;  // double offsets of the TN tile and the work region
  long long off_cc;            // column cache (B, V, states of the CTA's column); 0: none
};

// arguments of the persistent pass kernel (pass_kernel.cuh)
struct PassArgs {
  RelaxDev r;
  GemmArgs nn;  // X * (V or B) -> R, with part_loss / part_conj for EVAL
  GemmArgs tn;  // X' * R -> G slabs
  int n, p;
  int max_it, check;
  double gap_tol, prune_thr;
  double* trace;
  long long* out;  // [0] iterations, [1] evaluations, [2] node-iterations
  unsigned long long* prof;  // optional phase wall times (ns, CTA 0's view); nullptr: off
  unsigned* bar;             // grid barrier counter (zeroed before the launch)
  ResLayout res;
  GemmArgs gq;  // gram: Q * V - c -> G (one slab), the iteration's only product
  int gram;
  long long gram_local;  // > 0: double offset of the local-Gram region (p <= 128): each
                         // CTA iterates its own column between evaluations
  const double* gram_c;  // c = X'y
  int big;                   // streaming mode: 128 x 64 register-tiled GEMM tiles when
                             // m_a >= big (gemm_big.cuh; needs n, p even); 0: never
};

// shared memory of the pass kernel's local-Gram region: Q (p x p), c, G, and
// the column cache (B, V, states)
inline size_t gram_local_bytes(int p) {
  return 8 * ((size_t)p * p + 4 * (size_t)p) + (size_t)p + 64;
}

// ---- gemm_kernels.cu -------------------------------------------------------
cudaError_t gemm_set_attrs();
cudaError_t gemm_launch(bool tn, int epi, int fm, int fn, dim3 grid, cudaStream_t st,
                        const GemmArgs& g);
// register-tiled 128 x 64 DMMA GEMM for wide batches (gemm_big.cuh); n, p even
int gemm_big_tile_m();
int gemm_big_tile_n();
int gemm_big_tile_k();
// TMA box sizes {inner, outer} of the NN and TN A tiles (X)
void gemm_big_boxes(int* nn, int* tn);
cudaError_t gemm_big_launch(bool tn, int epi, dim3 grid, cudaStream_t st, const GemmArgs& g);

// ---- column_kernels.cu -----------------------------------------------------
int column_E(int n2);  // register-sort elements per thread (0: shared-memory sort)
cudaError_t column_set_attrs(int E, size_t smem);
cudaError_t launch_prox_fista(int E, int m, size_t smem, cudaStream_t st, const RelaxDev& r);
cudaError_t launch_eval(int E, int m, size_t smem, cudaStream_t st, const RelaxDev& r,
                        const EvalArgs& e);
cudaError_t launch_round_select(int E, int m, size_t smem, cudaStream_t st, int p, int n2, int k,
                                const double* beta, const uint8_t* state, const int* kbar,
                                const int* one_off, const int* one_idx, const int* one_len, int* sup,
                                int* len, int* jb, double* gscr = nullptr, long long gstride = 0);
// gscr / gstride: column buffers in global memory (large p), see RelaxDev::colscr
cudaError_t launch_prox_standalone(int E, int m, size_t smem, cudaStream_t st, int mode, int p,
                                   int n2, const double* U, const uint8_t* state, const int* kbar,
                                   double w, double M, double* out, double* gscr = nullptr,
                                   long long gstride = 0);
cudaError_t launch_g_standalone(int E, int m, size_t smem, cudaStream_t st, int mode, int p, int n2,
                                const double* in, const uint8_t* state, const int* kbar, double M,
                                double* out, double* gscr = nullptr, long long gstride = 0);

// ---- reopt_kernels.cu ------------------------------------------------------
// k_reopt_cluster<qmax in {8,16}, rpt>: cs CTAs (one cluster) per support
cudaError_t launch_reopt_cluster(int qmax, int rpt, int cs, int nsup, cudaStream_t st, int n,
                                 const double* X, const double* y, int loss, double M,
                                 double lambda2, double step, const int* off, const int* idx,
                                 double* coef, double* obj, int* its);

// large-n variant: X_S slice in shared memory, cs <= 16 CTAs per support
size_t reopt_smem_bytes(int n, int qmax, int cs);
cudaError_t launch_reopt_smem(int qmax, int cs, int nsup, cudaStream_t st, int n, const double* X,
                              const double* y, int loss, double M, double lambda2, double step,
                              const int* off, const int* idx, double* coef, double* obj, int* its);

// ---- pass_kernels.cu -------------------------------------------------------
size_t pass_smem(int p, int n2, int E);
// residency plan for `grid` CTAs (res.on = 0 when X does not fit); returns the
// dynamic shared memory the resident kernel needs
size_t pass_res_plan(int n, int p, int n2, int E, int grid, size_t smem_limit, ResLayout* res,
                     int rt = 1);
// true when k_pass<E> launches as one cluster of `cs` CTAs with `smem` bytes
bool pass_cluster_ok(int E, size_t smem, int cs);
cudaError_t pass_setup(int E, size_t smem, int* blocks_per_sm);
cudaError_t pass_static_smem(int E, size_t* bytes);
cudaError_t pass_launch(int E, int grid, size_t smem, cudaStream_t st, PassArgs* a, int cluster = 0);

}  // namespace bnbg
