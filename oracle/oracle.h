/*
 * oracle.h -- CPU restatement of the bnbglm node-processing path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library,
 * and only as the checker or the timed CPU reference -- never as the product.
 *
 * This is a plain-C restatement of the reference headers under
 * /root/reference/proj/include/bnbglm (which cannot be compiled here: they
 * need Eigen, absent from the image -- see DESIGN.md "Oracle").  Every
 * function cites the reference file:line it follows.  Parity is pinned by the
 * SPEC.md known-answer vectors and the enumeration oracle (tests/test_oracle_*).
 *
 * Conventions (same as the reference):
 *   - matrices are column-major doubles; X is n x p, B is p x m;
 *   - coordinate states: 0 free, 1 fixed-one, 2 fixed-zero (node_model.hpp:20);
 *   - indices are 0-based.
 */
#ifndef BNBG_ORACLE_H
#define BNBG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_SQUARED = 0, ORC_LOGISTIC = 1 };
enum { ORC_FREE = 0, ORC_ONE = 1, ORC_ZERO = 2 };
enum { ORC_PRUNABLE = 0, ORC_CONVERGED = 1, ORC_CAPPED = 2 };
enum { ORC_OK = 0, ORC_INPUT_ERROR = 1, ORC_NUMERIC_ERROR = 2, ORC_LOGIC_ERROR = 3 };

/* ---- rng.hpp:13-64 ---------------------------------------------------- */
typedef struct {
  uint64_t s[4];
  double spare;
  int has_spare;
} orc_rng;
void orc_rng_seed(orc_rng* r, uint64_t seed);
uint64_t orc_rng_next(orc_rng* r);
double orc_rng_uniform(orc_rng* r);
double orc_rng_gaussian(orc_rng* r);

/* ---- losses.hpp:56-112 ------------------------------------------------- */
double orc_loss_value(int loss, double s, double y);
double orc_loss_derivative(int loss, double s, double y);
double orc_loss_conjugate(int loss, double zeta, double y);
double orc_smoothness(int loss, const double* X, int n, int p);

/* ---- problem.hpp:36-132 ------------------------------------------------ */
int orc_validate(const double* X, const double* y, int n, int p, int loss, int k,
                 double M, double lambda2);
/* Fills X (n x p col-major), y (n) and support (k).  Returns ORC_OK or
 * ORC_INPUT_ERROR.  Row i of X = chol(Sigma) g_i with g_i ~ N(0,I) drawn in
 * row order (problem.hpp:90-99). */
int orc_generate(int n, int p, int k, double rho, int loss, double snr, uint64_t seed,
                 double* X, double* y, int* support);

/* ---- prox_kernel.hpp:27-370 ------------------------------------------- */
double orc_huber(double q, double M);
double orc_prox_huber(double x, double w, double M);
void orc_prox_step_column(const double* u, const uint8_t* st, int p, int kbar, double rho,
                          double M, double* out);
void orc_conjugate_prox_column(const double* x, const uint8_t* st, int p, int kbar,
                               double w, double M, double* out);
/* generic full-scan PAVA ("kept as test oracle") */
void orc_conjugate_prox_column_generic(const double* x, const uint8_t* st, int p, int kbar,
                                       double w, double M, double* out);
double orc_g_value(const double* beta, const uint8_t* st, int p, int kbar, double M);
double orc_g_conjugate(const double* q, const uint8_t* st, int p, int kbar, double M);
/* primal_heuristics.hpp:60-130.  Returns 1 if ok (z filled), 0 if infeasible. */
int orc_recover(const double* beta, const uint8_t* st, int p, int kbar, double M, double* z,
                double* tau, int* cap_count);

/* ---- relaxation.hpp:163-255 -------------------------------------------- */
typedef struct {
  int max_iterations;   /* 2000 */
  double gap_tolerance; /* 1e-6 */
  int check_interval;   /* 10 */
  int acceleration;     /* 1 */
  double smoothness;    /* <=0 -> computed */
  int workers;          /* 1 */
} orc_relax_cfg;
void orc_relax_cfg_default(orc_relax_cfg* c);

typedef void (*orc_trace_fn)(void* user, int column, double psi);

/* state: p x m column-major CoordState bytes; kbar: m; warm: p x m.
 * Outputs: beta p x m, bounds m, status m, iters m.  Returns ORC_OK,
 * ORC_INPUT_ERROR or ORC_NUMERIC_ERROR (err_column set). */
int orc_relax_batch(const double* X, const double* y, int n, int p, int loss, double M,
                    double lambda2, const orc_relax_cfg* cfg, double prune_threshold, int m,
                    const uint8_t* state, const int* kbar, const double* warm, double* beta,
                    double* bounds, int* status, int* iters, orc_trace_fn trace, void* user,
                    int* err_column);

/* ---- primal_heuristics.hpp:134-227 -------------------------------------- */
/* support = fixed_one (construction order) ++ top-kbar free; returns length */
int orc_round_support(const double* beta, const uint8_t* st, int p, const int* fixed_one,
                      int n_one, int kbar, int* support_out);
/* returns index or -1 (logic error: no free coordinate) */
int orc_select_branch(const double* beta, const uint8_t* st, int p);
/* supports given CSR-style: offsets[nsup+1], idx[offsets[nsup]] */
void orc_reoptimize(const double* X, const double* y, int n, int p, int loss, double M,
                    double lambda2, double smoothness, int nsup, const int* offsets,
                    const int* idx, int workers, double* coef_out, double* obj_out);

/* ---- bnb_engine.hpp:28-309 / rashomon.hpp:149-218 ---------------------- */
typedef struct {
  int batch_size;          /* 0 = auto */
  uint64_t memory_budget;  /* 1 GiB */
  double time_limit;       /* +inf */
  double prune_slack;      /* 1e-6 */
  orc_relax_cfg relax;
  int workers;
} orc_solver_cfg;
void orc_solver_cfg_default(orc_solver_cfg* c);

int orc_auto_batch_size(uint64_t memory_budget, int n, int p, int k, int loss);

typedef struct {
  double optimal_value;
  int support_len;
  int* support;         /* caller buffer, capacity k (sorted, 0-based) */
  double* coefficients; /* caller buffer, capacity k */
  double gap_percent;
  double lower_bound;
  long long nodes_processed;
  long long lb_batches;
  long long reopt_batches;
  int batch_size_used;
  double prof_lower_bound, prof_reoptimization, prof_transfer, prof_branch_generate,
      prof_total;
  int status; /* 0 optimal, 1 time limit */
  int err_column;
} orc_certificate;

typedef void (*orc_dual_hook)(void* user, int n0, const int* j0, int n1, const int* j1,
                              double psi);
typedef void (*orc_boundary_hook)(void* user, double lb, double ub);

int orc_solve(const double* X, const double* y, int n, int p, int loss, int k, double M,
              double lambda2, const orc_solver_cfg* cfg, orc_certificate* cert,
              orc_dual_hook on_dual, orc_boundary_hook on_boundary, void* user);

/* Rashomon pool (rashomon.hpp:149-218): compacted records, sorted by
 * (objective, sequence).  Sequences are in insertion (construction) order. */
typedef struct orc_pool orc_pool;
int orc_collect_rashomon(const double* X, const double* y, int n, int p, int loss, int k,
                         double M, double lambda2, const orc_solver_cfg* cfg, double epsilon,
                         long long cap, orc_certificate* cert, orc_pool** pool_out);
int orc_pool_size(const orc_pool* pool);
int orc_pool_record(const orc_pool* pool, int i, int* seq_out, double* coef_out,
                    double* objective_out); /* returns sequence length */
void orc_pool_free(orc_pool* pool);

/* ---- BLAS plumbing (timing only) ---------------------------------------- */
/* Load an OpenBLAS shared object exporting scipy_cblas_dgemm64_ (numpy's
 * bundled scipy-openblas) for the GEMMs; threads <= 0 keeps its default.
 * Returns 1 on success.  Without it the oracle uses plain C loops. */
int orc_use_openblas(const char* path, int threads);
int orc_blas_active(void);

#ifdef __cplusplus
}
#endif
#endif
