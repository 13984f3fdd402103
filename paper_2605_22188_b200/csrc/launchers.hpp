// launchers.hpp -- host launchers of the sm_100a kernels, one translation
// unit per kernel family (gemm_kernels.cu, column_kernels.cu, pass_kernels.cu)
// so the template instantiations compile in parallel.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "gemm.cuh"
#include "node_kernels.cuh"

namespace bnbg {

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
};

// ---- gemm_kernels.cu -------------------------------------------------------
cudaError_t gemm_set_attrs();
cudaError_t gemm_launch(bool tn, int epi, int fm, int fn, dim3 grid, cudaStream_t st,
                        const GemmArgs& g);

// ---- column_kernels.cu -----------------------------------------------------
int column_E(int n2);  // register-sort elements per thread (0: shared-memory sort)
cudaError_t column_set_attrs(int E, size_t smem);
cudaError_t launch_prox_fista(int E, int m, size_t smem, cudaStream_t st, const RelaxDev& r);
cudaError_t launch_eval(int E, int m, size_t smem, cudaStream_t st, const RelaxDev& r,
                        const EvalArgs& e);
cudaError_t launch_round_select(int E, int m, size_t smem, cudaStream_t st, int p, int n2, int k,
                                const double* beta, const uint8_t* state, const int* kbar,
                                const int* one_off, const int* one_idx, int* sup, int* len,
                                int* jb);
cudaError_t launch_prox_standalone(int E, int m, size_t smem, cudaStream_t st, int mode, int p,
                                   int n2, const double* U, const uint8_t* state, const int* kbar,
                                   double w, double M, double* out);
cudaError_t launch_g_standalone(int E, int m, size_t smem, cudaStream_t st, int mode, int p, int n2,
                                const double* in, const uint8_t* state, const int* kbar, double M,
                                double* out);

// ---- reopt_kernels.cu ------------------------------------------------------
// k_reopt_cluster<qmax in {8,16}, rpt>: cs CTAs (one cluster) per support
cudaError_t launch_reopt_cluster(int qmax, int rpt, int cs, int nsup, cudaStream_t st, int n,
                                 const double* X, const double* y, int loss, double M,
                                 double lambda2, double step, const int* off, const int* idx,
                                 double* coef, double* obj, int* its);

// ---- pass_kernels.cu -------------------------------------------------------
size_t pass_smem(int p, int n2, int E);
cudaError_t pass_setup(int E, size_t smem, int* blocks_per_sm);
cudaError_t pass_launch(int E, int grid, size_t smem, cudaStream_t st, PassArgs* a);

}  // namespace bnbg
