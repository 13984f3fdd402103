// ref_capi.cpp -- the REFERENCE ITSELF behind oracle.h's C API.
//
// TEST INFRASTRUCTURE ONLY: built into oracle/_ref/libbnbref.so by
// oracle/ref/Makefile, loaded by oracle/oracle.py (backend "ref") from tests/,
// __graft_entry__.smoke() and bench.py's reference arm / cpu_baseline leg.
// Never linked into the product.
//
// The reference headers are compiled UNMODIFIED from
// /root/reference/proj/include/bnbglm (include path only; no source is
// copied), with Eigen replaced by the subset shim in oracle/ref/eigen_shim
// (SURVEY.md §8(c) option A).  Each entry point exports the same symbol and
// signature as oracle/oracle.c, so every oracle test can run against the real
// reference and oracle.c (the restatement) is pinned by it.
#include <dlfcn.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "bnbglm/bnb_engine.hpp"
#include "bnbglm/rashomon.hpp"

extern "C" {
#include "../oracle.h"
}

using namespace bnbglm;

namespace {

LossKind kind_of(int loss) { return loss == ORC_LOGISTIC ? LossKind::kLogistic : LossKind::kSquared; }

ProblemInstance make_instance(const double* X, const double* y, int n, int p, int loss, int k,
                              double M, double lambda2) {
  ProblemInstance inst;
  inst.X.resize(n, p);
  std::memcpy(inst.X.data(), X, sizeof(double) * static_cast<size_t>(n) * p);
  inst.y.resize(n);
  std::memcpy(inst.y.data(), y, sizeof(double) * static_cast<size_t>(n));
  inst.loss = kind_of(loss);
  inst.k = k;
  inst.M = M;
  inst.lambda2 = lambda2;
  return inst;
}

// CoordState bytes (index order) -> NodeState with J0/J1 in index order.
NodeState node_from_states(const uint8_t* st, int p, const double* warm) {
  NodeState node;
  node.warm_start = Eigen::VectorXd::Zero(p);
  for (int j = 0; j < p; ++j) {
    if (st[j] == ORC_ZERO) node.fixed_zero.push_back(j);
    if (st[j] == ORC_ONE) node.fixed_one.push_back(j);
    if (warm) node.warm_start[j] = warm[j];
  }
  return node;
}

int n_one(const uint8_t* st, int p) {
  int c = 0;
  for (int j = 0; j < p; ++j) c += st[j] == ORC_ONE;
  return c;
}

// relaxation.hpp:76-81 names the column in the message
int column_of(const char* what) {
  const char* s = std::strstr(what, "column ");
  return s ? std::atoi(s + 7) : -1;
}

template <class F>
int guarded(F&& f, int* err_column = nullptr) {
  try {
    f();
    return ORC_OK;
  } catch (const numeric_error& e) {
    if (err_column) *err_column = column_of(e.what());
    return ORC_NUMERIC_ERROR;
  } catch (const input_error&) {
    return ORC_INPUT_ERROR;
  } catch (const parse_error&) {
    return ORC_INPUT_ERROR;
  } catch (const std::logic_error&) {
    return ORC_LOGIC_ERROR;
  }
}

typedef void (*cblas_dgemm64_t)(int, int, int, int64_t, int64_t, int64_t, double, const double*,
                                int64_t, const double*, int64_t, double, double*, int64_t);
cblas_dgemm64_t g_dgemm = nullptr;

void blas_gemm(bool ta, bool tb, Eigen::Index m, Eigen::Index n, Eigen::Index k, const double* A,
               Eigen::Index lda, const double* B, Eigen::Index ldb, double* C, Eigen::Index ldc) {
  g_dgemm(102, ta ? 112 : 111, tb ? 112 : 111, m, n, k, 1.0, A, lda, B, ldb, 0.0, C, ldc);
}

void fill_cert(const Certificate& c, orc_certificate* out) {
  out->optimal_value = c.optimal_value;
  out->support_len = static_cast<int>(c.support.size());
  for (size_t i = 0; i < c.support.size(); ++i) {
    out->support[i] = c.support[i];
    out->coefficients[i] = c.coefficients[static_cast<Eigen::Index>(i)];
  }
  out->gap_percent = c.gap_percent;
  out->lower_bound = c.lower_bound;
  out->nodes_processed = c.nodes_processed;
  out->lb_batches = c.lb_batches;
  out->reopt_batches = c.reopt_batches;
  out->batch_size_used = c.batch_size_used;
  out->prof_lower_bound = c.profile.lower_bound_seconds;
  out->prof_reoptimization = c.profile.reoptimization_seconds;
  out->prof_transfer = c.profile.transfer_seconds;
  out->prof_branch_generate = c.profile.branch_generate_seconds;
  out->prof_total = c.profile.total_seconds;
  out->status = c.status == SolveStatus::kOptimal ? 0 : 1;
  out->err_column = -1;
}

SolverConfig solver_config(const orc_solver_cfg* c) {
  SolverConfig s;
  s.batch_size = c->batch_size;
  s.memory_budget = c->memory_budget;
  s.time_limit = c->time_limit;
  s.prune_slack = c->prune_slack;
  s.relax.max_iterations = c->relax.max_iterations;
  s.relax.gap_tolerance = c->relax.gap_tolerance;
  s.relax.check_interval = c->relax.check_interval;
  s.relax.acceleration = c->relax.acceleration != 0;
  s.relax.smoothness = c->relax.smoothness;
  s.relax.workers = c->relax.workers;
  s.workers = c->workers;
  return s;
}

}  // namespace

struct orc_pool {
  struct Rec {
    std::vector<int> seq;
    std::vector<double> coef;
    double objective;
  };
  std::vector<Rec> rec;
};

extern "C" {

// ---- losses.hpp ----------------------------------------------------------
double orc_loss_value(int loss, double s, double y) { return loss_value(kind_of(loss), s, y); }
double orc_loss_derivative(int loss, double s, double y) {
  return loss_derivative(kind_of(loss), s, y);
}
double orc_loss_conjugate(int loss, double zeta, double y) {
  return loss_conjugate(kind_of(loss), zeta, y);
}
double orc_smoothness(int loss, const double* X, int n, int p) {
  Eigen::MatrixXd Xm(n, p);
  std::memcpy(Xm.data(), X, sizeof(double) * static_cast<size_t>(n) * p);
  return smoothness_constant(kind_of(loss), Xm);
}

// ---- problem.hpp ---------------------------------------------------------
int orc_validate(const double* X, const double* y, int n, int p, int loss, int k, double M,
                 double lambda2) {
  return guarded([&] {
    ProblemInstance inst = make_instance(X, y, n, p, loss, k, M, lambda2);
    validate(inst);
  });
}

int orc_generate(int n, int p, int k, double rho, int loss, double snr, uint64_t seed, double* X,
                 double* y, int* support) {
  return guarded([&] {
    GeneratorSpec spec;
    spec.n = n;
    spec.p = p;
    spec.k = k;
    spec.correlation = rho;
    spec.loss = kind_of(loss);
    spec.snr = snr;
    spec.seed = seed;
    std::vector<int> sup;
    ProblemInstance inst = generate_synthetic(spec, &sup);
    std::memcpy(X, inst.X.data(), sizeof(double) * static_cast<size_t>(n) * p);
    std::memcpy(y, inst.y.data(), sizeof(double) * static_cast<size_t>(n));
    for (int t = 0; t < k; ++t) support[t] = sup[t];
  });
}

// ---- prox_kernel.hpp -----------------------------------------------------
double orc_huber(double q, double M) { return huber_value(q, M); }
double orc_prox_huber(double x, double w, double M) { return prox_huber(x, w, M); }

void orc_prox_step_column(const double* u, const uint8_t* st, int p, int kbar, double rho,
                          double M, double* out) {
  Eigen::VectorXd uv(p), ov(p);
  std::memcpy(uv.data(), u, sizeof(double) * p);
  PavaWorkspace ws;
  ws.resize(p, 1);
  detail::prox_step_column(uv, reinterpret_cast<const CoordState*>(st), p, kbar, rho, M, ov, ws,
                           0);
  std::memcpy(out, ov.data(), sizeof(double) * p);
}

void orc_conjugate_prox_column(const double* x, const uint8_t* st, int p, int kbar, double w,
                               double M, double* out) {
  Eigen::VectorXd xv(p), ov(p);
  std::memcpy(xv.data(), x, sizeof(double) * p);
  PavaWorkspace ws;
  ws.resize(p, 1);
  conjugate_prox_column(xv, reinterpret_cast<const CoordState*>(st), p, kbar, w, M, ov, ws, 0);
  std::memcpy(out, ov.data(), sizeof(double) * p);
}

// The reference has only the boundary-seeded PAVA; the generic full-scan
// variant is oracle.c's own cross-check.
void orc_conjugate_prox_column_generic(const double* x, const uint8_t* st, int p, int kbar,
                                       double w, double M, double* out) {
  orc_conjugate_prox_column(x, st, p, kbar, w, M, out);
}

double orc_g_value(const double* beta, const uint8_t* st, int p, int kbar, double M) {
  Eigen::VectorXd b(p);
  std::memcpy(b.data(), beta, sizeof(double) * p);
  return detail::g_value_core(b, reinterpret_cast<const CoordState*>(st), p, kbar, M);
}

double orc_g_conjugate(const double* q, const uint8_t* st, int p, int kbar, double M) {
  Eigen::VectorXd v(p);
  std::memcpy(v.data(), q, sizeof(double) * p);
  std::vector<double> scratch;
  return detail::g_conjugate_core(v, reinterpret_cast<const CoordState*>(st), p, kbar, M,
                                  scratch);
}

int orc_recover(const double* beta, const uint8_t* st, int p, int kbar, double M, double* z,
                double* tau, int* cap_count) {
  NodeState node = node_from_states(st, p, nullptr);
  Eigen::VectorXd b(p);
  std::memcpy(b.data(), beta, sizeof(double) * p);
  const int k = kbar + static_cast<int>(node.fixed_one.size());
  try {
    RecoveredIndicators r = recover_indicators(b, node, k, M);
    std::memcpy(z, r.z.data(), sizeof(double) * p);
    *tau = r.tau;
    *cap_count = r.cap_count;
    return 1;
  } catch (const input_error&) {
    return 0;
  }
}

// ---- relaxation.hpp ------------------------------------------------------
void orc_relax_cfg_default(orc_relax_cfg* c) {
  RelaxConfig r;
  c->max_iterations = r.max_iterations;
  c->gap_tolerance = r.gap_tolerance;
  c->check_interval = r.check_interval;
  c->acceleration = r.acceleration ? 1 : 0;
  c->smoothness = r.smoothness;
  c->workers = r.workers;
}

int orc_relax_batch(const double* X, const double* y, int n, int p, int loss, double M,
                    double lambda2, const orc_relax_cfg* cfg, double prune_threshold, int m,
                    const uint8_t* state, const int* kbar, const double* warm, double* beta,
                    double* bounds, int* status, int* iters, orc_trace_fn trace, void* user,
                    int* err_column) {
  if (m <= 0) return ORC_INPUT_ERROR;
  // BatchMeta::from_nodes takes one k for the batch (prox_kernel.hpp:52):
  // per-column kbar must agree with k - |J1|.
  const int k = kbar[0] + n_one(state, p);
  for (int b = 0; b < m; ++b)
    if (kbar[b] != std::max(0, k - n_one(state + static_cast<size_t>(b) * p, p)))
      return ORC_INPUT_ERROR;
  ProblemInstance inst = make_instance(X, y, n, p, loss, std::max(1, k), M, lambda2);
  std::vector<NodeState> batch;
  for (int b = 0; b < m; ++b)
    batch.push_back(node_from_states(state + static_cast<size_t>(b) * p, p,
                                     warm + static_cast<size_t>(b) * p));
  RelaxConfig rc;
  rc.max_iterations = cfg->max_iterations;
  rc.gap_tolerance = cfg->gap_tolerance;
  rc.check_interval = cfg->check_interval;
  rc.acceleration = cfg->acceleration != 0;
  rc.smoothness = cfg->smoothness;
  rc.workers = cfg->workers;
  std::function<void(int, double)> tr;
  if (trace) tr = [&](int b, double psi) { trace(user, b, psi); };
  RelaxationResult res;
  const int code =
      guarded([&] { res = solve_batch_relaxation(batch, inst, rc, prune_threshold, nullptr, tr); },
              err_column);
  if (code != ORC_OK) return code;
  std::memcpy(beta, res.beta.data(), sizeof(double) * static_cast<size_t>(p) * m);
  for (int b = 0; b < m; ++b) {
    bounds[b] = res.bounds[b];
    status[b] = res.status[b] == NodeStatus::kPrunable    ? ORC_PRUNABLE
                : res.status[b] == NodeStatus::kConverged ? ORC_CONVERGED
                                                          : ORC_CAPPED;
    iters[b] = res.iterations[b];
  }
  return ORC_OK;
}

// ---- primal_heuristics.hpp -----------------------------------------------
int orc_round_support(const double* beta, const uint8_t* st, int p, const int* fixed_one,
                      int n_one_, int kbar, int* support_out) {
  NodeState node = node_from_states(st, p, nullptr);
  node.fixed_one.assign(fixed_one, fixed_one + n_one_);  // construction order
  Eigen::VectorXd b(p);
  std::memcpy(b.data(), beta, sizeof(double) * p);
  const std::vector<int> s = round_support(b, node, kbar + n_one_);
  for (size_t t = 0; t < s.size(); ++t) support_out[t] = s[t];
  return static_cast<int>(s.size());
}

int orc_select_branch(const double* beta, const uint8_t* st, int p) {
  NodeState node = node_from_states(st, p, nullptr);
  Eigen::VectorXd b(p);
  std::memcpy(b.data(), beta, sizeof(double) * p);
  try {
    return select_branch_variable(b, node);
  } catch (const std::logic_error&) {
    return -1;
  }
}

void orc_reoptimize(const double* X, const double* y, int n, int p, int loss, double M,
                    double lambda2, double smoothness, int nsup, const int* offsets,
                    const int* idx, int workers, double* coef_out, double* obj_out) {
  ProblemInstance inst = make_instance(X, y, n, p, loss, 1, M, lambda2);
  std::vector<std::vector<int>> supports(nsup);
  for (int s = 0; s < nsup; ++s) supports[s].assign(idx + offsets[s], idx + offsets[s + 1]);
  ReoptResult r = reoptimize_supports(supports, inst, smoothness, workers);
  for (int s = 0; s < nsup; ++s) {
    for (int t = 0; t < offsets[s + 1] - offsets[s]; ++t)
      coef_out[offsets[s] + t] = r.coefficients[s][t];
    obj_out[s] = r.objectives[s];
  }
}

// ---- bnb_engine.hpp / rashomon.hpp ---------------------------------------
void orc_solver_cfg_default(orc_solver_cfg* c) {
  SolverConfig s;
  c->batch_size = s.batch_size;
  c->memory_budget = s.memory_budget;
  c->time_limit = s.time_limit;
  c->prune_slack = s.prune_slack;
  orc_relax_cfg_default(&c->relax);
  c->workers = s.workers;
}

int orc_auto_batch_size(uint64_t memory_budget, int n, int p, int k, int loss) {
  return auto_batch_size(memory_budget, n, p, k, kind_of(loss));
}

int orc_solve(const double* X, const double* y, int n, int p, int loss, int k, double M,
              double lambda2, const orc_solver_cfg* cfg, orc_certificate* cert,
              orc_dual_hook on_dual, orc_boundary_hook on_boundary, void* user) {
  ProblemInstance inst = make_instance(X, y, n, p, loss, k, M, lambda2);
  DebugHooks hooks;
  if (on_dual)
    hooks.on_dual_bound = [&](const NodeState& node, double psi) {
      on_dual(user, static_cast<int>(node.fixed_zero.size()), node.fixed_zero.data(),
              static_cast<int>(node.fixed_one.size()), node.fixed_one.data(), psi);
    };
  if (on_boundary) hooks.on_batch_boundary = [&](double lb, double ub) { on_boundary(user, lb, ub); };
  cert->err_column = -1;
  return guarded(
      [&] {
        Certificate c = solve(inst, solver_config(cfg), &hooks);
        fill_cert(c, cert);
      },
      &cert->err_column);
}

int orc_collect_rashomon(const double* X, const double* y, int n, int p, int loss, int k,
                         double M, double lambda2, const orc_solver_cfg* cfg, double epsilon,
                         long long cap, orc_certificate* cert, orc_pool** pool_out) {
  ProblemInstance inst = make_instance(X, y, n, p, loss, k, M, lambda2);
  RashomonConfig rcfg;
  rcfg.epsilon = epsilon;
  rcfg.cap = cap;
  orc_pool* pool = new orc_pool;
  *pool_out = pool;
  cert->err_column = -1;
  return guarded(
      [&] {
        RashomonResult r = collect_rashomon(inst, solver_config(cfg), rcfg);
        fill_cert(r.certificate, cert);
        for (int i = 0; i < r.pool.size(); ++i) {
          SupportTrie::Recovered rec = r.pool.recover(i);
          pool->rec.push_back({rec.path, rec.coefficients, rec.objective});
        }
      },
      &cert->err_column);
}

int orc_pool_size(const orc_pool* pool) { return pool ? static_cast<int>(pool->rec.size()) : 0; }
int orc_pool_record(const orc_pool* pool, int i, int* seq_out, double* coef_out,
                    double* objective_out) {
  const auto& r = pool->rec[i];
  std::memcpy(seq_out, r.seq.data(), sizeof(int) * r.seq.size());
  std::memcpy(coef_out, r.coef.data(), sizeof(double) * r.coef.size());
  *objective_out = r.objective;
  return static_cast<int>(r.seq.size());
}
void orc_pool_free(orc_pool* pool) { delete pool; }

// ---- BLAS plumbing (timing legs) -------------------------------------------
int orc_use_openblas(const char* path, int threads) {
  void* h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
  if (!h) return 0;
  auto f = reinterpret_cast<cblas_dgemm64_t>(dlsym(h, "scipy_cblas_dgemm64_"));
  if (!f) return 0;
  if (threads > 0) {
    auto set_threads =
        reinterpret_cast<void (*)(int)>(dlsym(h, "scipy_openblas_set_num_threads64_"));
    if (set_threads) set_threads(threads);
  }
  g_dgemm = f;
  Eigen::shim::gemm_hook() = blas_gemm;
  return 1;
}
int orc_blas_active(void) { return g_dgemm != nullptr; }

}  // extern "C"
