/*
 * bnbg.h -- C-ABI of the B200 batched branch-and-bound engine (libbnbg.so).
 *
 * Drop-in boundary for the node-processing path of the reference bnbglm
 * library (/root/reference/proj/include/bnbglm, "the reference" below).  Every
 * entry point names the reference interface it replaces (file:line).  Plain
 * pointers and sizes only; no exceptions cross this boundary.  Host buffers
 * are caller-owned and may be pinned.  A handle owns one GPU's copy of the
 * instance (X, y resident in HBM), the batch workspaces and the streams; it is
 * NOT thread-safe (single orchestrator, bnb_engine.hpp:3-9).
 *
 * Conventions (identical to the reference):
 *   matrices are column-major float64: X is n x p, a batch block is p x m
 *   (one column per node); coordinate states are uint8 {0 free, 1 fixed-one,
 *   2 fixed-zero} (node_model.hpp:20); indices are 0-based; loss 0 = squared
 *   (l = (s-y)^2/2), 1 = logistic (labels +-1) (losses.hpp:21-69).
 *
 * Status codes map to the reference's exception taxonomy (errors.hpp:9-24):
 *   BNBG_INPUT_ERROR   -> bnbglm::input_error
 *   BNBG_NUMERIC_ERROR -> bnbglm::numeric_error (non-finite iterate)
 *   BNBG_LOGIC_ERROR   -> std::logic_error (branch on a non-free coordinate)
 *   BNBG_CUDA_ERROR    -> new: a CUDA runtime failure (no CPU fallback exists)
 * The message of the last failure is available from bnbg_last_error().
 */
#ifndef BNBG_H
#define BNBG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  BNBG_OK = 0,
  BNBG_INPUT_ERROR = 1,
  BNBG_NUMERIC_ERROR = 2,
  BNBG_LOGIC_ERROR = 3,
  BNBG_CUDA_ERROR = 4
};
enum { BNBG_SQUARED = 0, BNBG_LOGISTIC = 1 };
enum { BNBG_FREE = 0, BNBG_FIXED_ONE = 1, BNBG_FIXED_ZERO = 2 };
/* relaxation.hpp:35 NodeStatus */
enum { BNBG_PRUNABLE = 0, BNBG_CONVERGED = 1, BNBG_ITERATION_CAPPED = 2 };
enum { BNBG_STATUS_OPTIMAL = 0, BNBG_STATUS_TIME_LIMIT = 1 };

/* relaxation.hpp:26-33 RelaxConfig (same fields, same defaults). */
typedef struct {
  int max_iterations;   /* 2000 */
  double gap_tolerance; /* 1e-6 relative duality gap */
  int check_interval;   /* 10 */
  int acceleration;     /* 1: restarted accelerated scheme */
  double smoothness;    /* <= 0: computed (losses.hpp:86-112) */
  int workers;          /* accepted for API parity; the device ignores it */
} bnbg_relax_cfg;

/* bnb_engine.hpp:28-36 SolverConfig (same fields, same defaults). */
typedef struct {
  int batch_size;         /* 0 = auto (bnb_engine.hpp:75-88) */
  uint64_t memory_budget; /* bytes for auto, 1 GiB */
  double time_limit;      /* seconds, +inf */
  double prune_slack;     /* delta = 1e-6, scaled by max(1,|UB|) */
  bnbg_relax_cfg relax;
  int profile;
  int workers;
} bnbg_solver_cfg;

/* bnb_engine.hpp:40-60 ComponentProfile + Certificate.  support and
 * coefficients are caller buffers of capacity k. */
typedef struct {
  double optimal_value;
  int support_len;
  int32_t* support;      /* sorted, 0-based */
  double* coefficients;  /* aligned with support */
  double gap_percent;
  double lower_bound;
  long long nodes_processed;
  long long lb_batches;
  long long reopt_batches;
  int batch_size_used;
  double lower_bound_seconds;
  double reoptimization_seconds;
  double transfer_seconds;
  double branch_generate_seconds;
  double total_seconds;
  int status; /* BNBG_STATUS_* */
  /* B200 additions (not in the reference Certificate) */
  long long relax_iterations;  /* sum over passes of the iterations run */
  long long node_iterations;   /* sum over columns of proximal steps taken */
  long long reopt_supports;    /* supports re-optimised */
  double device_seconds;       /* GPU time of the node-processing kernels */
} bnbg_certificate;

typedef void (*bnbg_trace_fn)(void* user, int column, double psi);
/* DebugHooks (bnb_engine.hpp:63-66).  on_dual_bound receives the node's J0/J1
 * lists instead of a NodeState reference. */
typedef void (*bnbg_dual_hook)(void* user, int n0, const int32_t* j0, int n1,
                               const int32_t* j1, double psi);
typedef void (*bnbg_boundary_hook)(void* user, double lb, double ub);

typedef struct bnbg_handle bnbg_handle;
typedef struct bnbg_pool bnbg_pool;

/* ---- defaults ------------------------------------------------------------ */
void bnbg_relax_cfg_default(bnbg_relax_cfg* cfg);   /* relaxation.hpp:26-33 */
void bnbg_solver_cfg_default(bnbg_solver_cfg* cfg); /* bnb_engine.hpp:28-36 */
/* bnb_engine.hpp:75-88 auto_batch_size; returns -1 on a zero budget */
int bnbg_auto_batch_size(uint64_t memory_budget, int n, int p, int k, int loss);

/* ---- instance ------------------------------------------------------------ */
/* problem.hpp:70-132 generate_synthetic (host fixture; same stream as the
 * reference: xoshiro256++/splitmix64, Box-Muller with cached spare). */
int bnbg_generate_synthetic(int n, int p, int k, double correlation, int loss, double snr,
                            uint64_t seed, double* X_out, double* y_out, int32_t* support_out);
/* problem.hpp:36-51 validate */
int bnbg_validate(const double* X, const double* y, int n, int p, int loss, int k, double M,
                  double lambda2);

/* Uploads X (n x p col-major) and y to `device` and validates the instance
 * (problem.hpp:36-51).  L <= 0 computes the smoothness constant on the device
 * by the reference power iteration (losses.hpp:86-112). */
int bnbg_create(const double* X, const double* y, int n, int p, int loss, int k, double M,
                double lambda2, double L, int device, bnbg_handle** out);
void bnbg_destroy(bnbg_handle* h);
const char* bnbg_last_error(const bnbg_handle* h); /* h may be NULL */
/* losses.hpp:86-112 smoothness_constant of the handle's instance */
double bnbg_smoothness(bnbg_handle* h);

/* ---- the node-processing seam (bnb_engine.hpp:179-256) -------------------- */
/* relaxation.hpp:163-255 solve_batch_relaxation.  state p x m, kbar m (the
 * reduced budgets, prox_kernel.hpp:87), warm p x m; outputs beta p x m, bounds
 * (best dual bound per column), status, iterations.  trace, when non-NULL,
 * receives every dual evaluation in the reference's order (relaxation.hpp:203). */
int bnbg_relax_batch(bnbg_handle* h, const bnbg_relax_cfg* cfg, int m, const uint8_t* state,
                     const int32_t* kbar, const double* warm, double prune_threshold,
                     double* beta_out, double* bounds_out, int32_t* status_out,
                     int32_t* iters_out, bnbg_trace_fn trace, void* user);

/* prox_kernel.hpp:52-90 BatchMeta::from_nodes -- the device packer (VK1)
 * alone.  J0 / J1 lists as CSR (j0_off[m+1], j0_idx; j1_off[m+1], j1_idx;
 * 0-based, disjoint per node) -> state_out p x m CoordState bytes (column b
 * = node b), kbar_out[m] = max(0, k - |J1|), free_count_out[m] = |Jf|. */
int bnbg_pack_batch(bnbg_handle* h, int m, const int32_t* j0_off, const int32_t* j0_idx,
                    const int32_t* j1_off, const int32_t* j1_idx, uint8_t* state_out,
                    int32_t* kbar_out, int32_t* free_count_out);

/* primal_heuristics.hpp:134-146 round_support, batched.  fixed_one lists in
 * construction order as CSR (one_off[m+1], one_idx).  support_out is m x k
 * (row b holds J1 ++ top-kbar free), len_out[m]. */
int bnbg_round_support(bnbg_handle* h, int m, const double* beta, const uint8_t* state,
                       const int32_t* kbar, const int32_t* one_off, const int32_t* one_idx,
                       int32_t* support_out, int32_t* len_out);

/* primal_heuristics.hpp:148-163 select_branch_variable, batched; j_out[b] = -1
 * when column b has no free coordinate (the reference's logic_error). */
int bnbg_select_branch(bnbg_handle* h, int m, const double* beta, const uint8_t* state,
                       int32_t* j_out);

/* primal_heuristics.hpp:174-227 reoptimize_supports.  Supports as CSR
 * (offsets[nsup+1], idx).  coef_out aligned with idx; obj_out[nsup]. */
int bnbg_reoptimize(bnbg_handle* h, int nsup, const int32_t* offsets, const int32_t* idx,
                    double* coef_out, double* obj_out);

/* ---- device-resident node pool: the per-pass successor of the seam ---------
 * (SURVEY 8(b) item 4).  Open nodes live in the handle's HBM pool, one slot
 * each (states, warm start, ordered J0/J1 lists); a caller keeping its own
 * best-bound queue over (bound, sequence, slot) runs run_bnb's node-processing
 * body (bnb_engine.hpp:179-256) with these calls, and no warm start or beta
 * crosses PCIe.  bnbg_solve is exactly this loop. */

/* root_node (node_model.hpp:47-52) into `slot` (the pool grows as needed) */
int bnbg_pool_root(bnbg_handle* h, int slot);
/* solve_batch_relaxation + round_support + select_branch_variable over the
 * nodes in slots[m] (relaxation.hpp:163-255, primal_heuristics.hpp:134-163).
 * Outputs: bounds (best dual), status, iterations per node; support_out m x k
 * (J1 in fixing order ++ top-kbar free) with lengths len_out.  The betas stay
 * on the device for bnbg_pool_branch. */
int bnbg_pool_relax(bnbg_handle* h, const bnbg_relax_cfg* cfg, int m, const int32_t* slots,
                    double prune_threshold, double* bounds_out, int32_t* status_out,
                    int32_t* iters_out, int32_t* support_out, int32_t* len_out);
/* The prune test and branch of the last bnbg_pool_relax batch
 * (bnb_engine.hpp:242-256, node_model.hpp:57-105): node b survives iff its
 * status is not prunable and max(lb_in[b], bound_b) < post_threshold; its two
 * children (J0 + j, J1 + j) go to free_slots[2i], free_slots[2i+1] for the
 * i-th survivor.  rec_out receives 2 x survivors records of (4 + k) ints:
 * slot, leaf flag, |J1|, depth, J1 list; child_lb_out 2 x survivors bounds.
 * Returns BNBG_LOGIC_ERROR when a survivor has no free coordinate. */
int bnbg_pool_branch(bnbg_handle* h, int m, const double* lb_in, double post_threshold,
                     const int32_t* free_slots, int32_t* survivors_out, int32_t* rec_out,
                     double* child_lb_out);

/* ---- stateless kernel entry points (prox_kernel.hpp) ---------------------- */
/* prox_kernel.hpp:284-301 prox_step: out = U - rho^-1 prox_{rho g*}(rho U). */
int bnbg_prox_step(int device, int p, int m, const double* U, double eta, double lambda2,
                   const uint8_t* state, const int32_t* kbar, double M, double* out);
/* prox_kernel.hpp:214-229 batched_conjugate_prox */
int bnbg_conjugate_prox(int device, int p, int m, const double* U_scaled, double weight,
                        const uint8_t* state, const int32_t* kbar, double M, double* out);
/* prox_kernel.hpp:310-347 / :351-370, batched over m columns */
int bnbg_g_value(int device, int p, int m, const double* beta, const uint8_t* state,
                 const int32_t* kbar, double M, double* out);
int bnbg_g_conjugate(int device, int p, int m, const double* q, const uint8_t* state,
                     const int32_t* kbar, double M, double* out);
/* GEMM probe (tests): C = X * B (trans=0, C n x m) or X' * B (trans=1, C p x m) */
int bnbg_gemm(bnbg_handle* h, int trans, int m, const double* B, double* C);

/* ---- the certified solve (bnb_engine.hpp:299-309, rashomon.hpp:149-218) --- */
int bnbg_solve(bnbg_handle* h, const bnbg_solver_cfg* cfg, bnbg_certificate* cert,
               bnbg_dual_hook on_dual, bnbg_boundary_hook on_boundary, void* user);

/* Rashomon pool: records sorted by (objective, sequence); sequences in
 * construction order (fixed-in first, then rounded by magnitude). */
int bnbg_collect_rashomon(bnbg_handle* h, const bnbg_solver_cfg* cfg, double epsilon,
                          long long cap, bnbg_certificate* cert, bnbg_pool** pool_out);
int bnbg_pool_size(const bnbg_pool* pool);
/* copies record i; returns the sequence length */
int bnbg_pool_record(const bnbg_pool* pool, int i, int32_t* seq_out, double* coef_out,
                     double* objective_out);
void bnbg_pool_free(bnbg_pool* pool);

/* ---- node-sharded multi-GPU solve (no reference counterpart:
 * the reference only describes node-parallel solving) --
 * X and y are replicated on every rank's handle; open nodes are sharded
 * across ranks; per pass only the incumbent, the termination state and (when
 * a rank starves) queue nodes cross between ranks.  One handle per rank
 * (one process per GPU). */

/* Host-staged transport supplied by the caller (e.g. torch.distributed over
 * gloo).  Callbacks return 0 on success. */
typedef struct {
  void* ctx;
  int rank, world;
  /* recv receives `world` blocks of `bytes` bytes in rank order */
  int (*allgather)(void* ctx, const void* send, int64_t bytes, void* recv);
  /* send holds one contiguous block per peer in rank order (send_bytes[peer]
   * bytes each, possibly 0); recv likewise with recv_bytes[peer] */
  int (*alltoallv)(void* ctx, const void* send, const int64_t* send_bytes, void* recv,
                   const int64_t* recv_bytes);
} bnbg_comm_ops;

/* NCCL bootstrap: rank 0 creates the id, the caller broadcasts its 128 bytes
 * (e.g. torch.distributed), then every rank binds its handle.  Communicators
 * are cached per process by (id, device, rank, world): binding a later handle
 * with the same id reuses the communicator. */
int bnbg_nccl_unique_id(uint8_t* uid_out /* 128 bytes */);
int bnbg_nccl_init(bnbg_handle* h, const uint8_t* uid /* 128 bytes */, int rank, int world);

/* The certified solve of bnbg_solve with nodes sharded over ranks.  ops ==
 * NULL uses the handle's NCCL communicator (bnbg_nccl_init).  Every rank
 * receives the same certificate; counters are sums over ranks.  Only the
 * solve policy (bnb_engine.hpp:304-307) is sharded. */
int bnbg_solve_sharded(bnbg_handle* h, const bnbg_solver_cfg* cfg, const bnbg_comm_ops* ops,
                       bnbg_certificate* cert);

/* The deterministic load-balancing plan used by bnbg_solve_sharded (exported
 * for tests): counts[world] queue sizes -> moves[world*world] (donor-major);
 * returns 1 when nodes move, 0 otherwise. */
int bnbg_balance_plan(int world, const int64_t* counts, int64_t* moves);

/* ---- diagnostics ---------------------------------------------------------- */
/* Number of kernel launches issued by this handle so far (bench gpu_launches). */
long long bnbg_kernel_launches(const bnbg_handle* h);
/* Device time (ms, CUDA events) spent in the dominant GEMM kernels and the
 * algorithmic FP64 flops they executed, since the handle was created. */
int bnbg_gemm_stats(const bnbg_handle* h, double* gemm_ms, double* gemm_flops,
                    long long* gemm_launches);
void bnbg_set_timing(bnbg_handle* h, int enabled);
/* Per kernel class (0 GEMM X*V, 1 GEMM X'*R, 2 prox/FISTA, 3 bound evaluation,
 * 4 re-optimisation): CUDA-event time (ms, only while timing is enabled),
 * algorithmic FP64 flops and launches. */
int bnbg_kernel_stats(const bnbg_handle* h, int kernel_class, double* ms, double* flops,
                      long long* launches);
/* Wall time (ns, CTA 0's view, including the grid barrier that ends each
 * phase) of the persistent pass kernel's phases since the handle was created:
 * [0] X*V, [1] X'*R, [2] prox/FISTA, [3] eval X*B, [4] eval X'*Z, [5] eval
 * columns, [6] compaction; [8..14] the same phases up to CTA 0's arrival at
 * the phase's grid barrier (the rest is barrier wait); [16..19] prox sub-phases of
 * CTA 0 (load+sort, PAVA, scatter, end barrier).  Recorded only when
 * BNBG_PASS_PROF=1 was set at bnbg_create; returns the number of values written. */
int bnbg_pass_profile(const bnbg_handle* h, double* ns_out, int count);
/* Host<->device bytes copied by this handle so far. */
int bnbg_transfer_bytes(const bnbg_handle* h, long long* h2d, long long* d2h);
/* Last bnbg_solve_sharded on this handle: out[0] node records sent, out[1]
 * received through the load-balance exchange, out[2] passes, then the local
 * relaxation batch width of each pass.  Returns the number of values (may
 * exceed cap; only cap are written). */
int bnbg_shard_stats(const bnbg_handle* h, long long* out, int cap);

#ifdef __cplusplus
}
#endif
#endif
