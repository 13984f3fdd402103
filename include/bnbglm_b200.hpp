// bnbglm_b200.hpp -- reference-side adapter: the bnbglm C++ API on the B200 engine.
//
// A maintainer of the reference (/root/reference/proj/include/bnbglm) adds this
// header next to bnb_engine.hpp and links libbnbg.so.  It keeps the reference's
// public types and signatures and rethrows its exception types, so a call site
// switches with a namespace change:
//
//   bnbglm::solve(inst, cfg)                  -> bnbglm::b200::solve(inst, cfg)
//   bnbglm::collect_rashomon(inst, cfg, rc)   -> bnbglm::b200::collect_rashomon(inst, cfg, rc)
//   bnbglm::solve_batch_relaxation(...)       -> bnbglm::b200::solve_batch_relaxation(...)
//   bnbglm::reoptimize_supports(...)          -> bnbglm::b200::reoptimize_supports(...)
//
// Signatures replaced (file:line under proj/include/bnbglm):
//   solve                    bnb_engine.hpp:299-309
//   collect_rashomon         rashomon.hpp:149-151
//   solve_batch_relaxation   relaxation.hpp:163-167
//   reoptimize_supports      primal_heuristics.hpp:174-176
// Exceptions (errors.hpp:9-24): BNBG_INPUT_ERROR -> input_error,
// BNBG_NUMERIC_ERROR -> numeric_error, BNBG_LOGIC_ERROR -> std::logic_error,
// CUDA failures -> std::runtime_error.
//
// Compiled against the unmodified reference headers by
// tests/test_adapter_cpu.py (CPU: compile, link, error mapping) and run by
// tests/test_gpu_adapter.py (B200: b200::solve == bnbglm::solve).
#pragma once

#include <cstdint>
#include <cstdlib>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "bnbg.h"
#include "bnbglm/bnb_engine.hpp"
#include "bnbglm/rashomon.hpp"
#include "bnbglm/relaxation.hpp"

namespace bnbglm::b200 {

// GPU used by the adapter's handles (default: BNBG_DEVICE or 0).
inline int& device() {
  static int d = std::getenv("BNBG_DEVICE") ? std::atoi(std::getenv("BNBG_DEVICE")) : 0;
  return d;
}

[[noreturn]] inline void raise(int rc, const std::string& msg) {
  switch (rc) {
    case BNBG_INPUT_ERROR: throw input_error(msg);
    case BNBG_NUMERIC_ERROR: throw numeric_error(msg);
    case BNBG_LOGIC_ERROR: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}
inline void check(int rc, const bnbg_handle* h) {
  if (rc != BNBG_OK) raise(rc, bnbg_last_error(h));
}

// One GPU copy of an instance (X, y resident in HBM); closes on destruction.
class Handle {
 public:
  Handle(const ProblemInstance& inst, double smoothness) {
    // Eigen::MatrixXd is column-major: X.data() is the layout bnbg expects.
    check(bnbg_create(inst.X.data(), inst.y.data(), inst.n(), inst.p(),
                      inst.loss == LossKind::kSquared ? BNBG_SQUARED : BNBG_LOGISTIC, inst.k,
                      inst.M, inst.lambda2, smoothness, device(), &h_),
          nullptr);
  }
  ~Handle() { bnbg_destroy(h_); }
  Handle(const Handle&) = delete;
  Handle& operator=(const Handle&) = delete;
  bnbg_handle* get() const { return h_; }

 private:
  bnbg_handle* h_ = nullptr;
};

inline bnbg_relax_cfg to_c(const RelaxConfig& r) {  // relaxation.hpp:26-33
  bnbg_relax_cfg o;
  bnbg_relax_cfg_default(&o);
  o.max_iterations = r.max_iterations;
  o.gap_tolerance = r.gap_tolerance;
  o.check_interval = r.check_interval;
  o.acceleration = r.acceleration ? 1 : 0;
  o.smoothness = r.smoothness;
  o.workers = r.workers;
  return o;
}

inline bnbg_solver_cfg to_c(const SolverConfig& c) {  // bnb_engine.hpp:28-36
  bnbg_solver_cfg o;
  bnbg_solver_cfg_default(&o);
  o.batch_size = c.batch_size;
  o.memory_budget = c.memory_budget;
  o.time_limit = c.time_limit;
  o.prune_slack = c.prune_slack;
  o.relax = to_c(c.relax);
  o.profile = c.profile ? 1 : 0;
  o.workers = c.workers;
  return o;
}

// bnbg_certificate -> Certificate (bnb_engine.hpp:40-60)
struct CertBuffers {
  explicit CertBuffers(int k) : sup(k), coef(k) {
    c.support = sup.data();
    c.coefficients = coef.data();
  }
  Certificate take() const {
    Certificate cert;
    cert.optimal_value = c.optimal_value;
    cert.support.assign(sup.begin(), sup.begin() + c.support_len);
    cert.coefficients = Eigen::VectorXd::Zero(c.support_len);
    for (int i = 0; i < c.support_len; ++i) cert.coefficients[i] = coef[i];
    cert.gap_percent = c.gap_percent;
    cert.lower_bound = c.lower_bound;
    cert.nodes_processed = c.nodes_processed;
    cert.lb_batches = c.lb_batches;
    cert.reopt_batches = c.reopt_batches;
    cert.batch_size_used = c.batch_size_used;
    cert.profile.lower_bound_seconds = c.lower_bound_seconds;
    cert.profile.reoptimization_seconds = c.reoptimization_seconds;
    cert.profile.transfer_seconds = c.transfer_seconds;
    cert.profile.branch_generate_seconds = c.branch_generate_seconds;
    cert.profile.total_seconds = c.total_seconds;
    cert.status =
        c.status == BNBG_STATUS_OPTIMAL ? SolveStatus::kOptimal : SolveStatus::kTimeLimit;
    return cert;
  }
  std::vector<int32_t> sup;
  std::vector<double> coef;
  bnbg_certificate c{};
};

// bnb_engine.hpp:299-309
inline Certificate solve(const ProblemInstance& inst, const SolverConfig& config,
                         const DebugHooks* hooks = nullptr) {
  validate(inst);  // input_error before any device work, as the reference
  Handle h(inst, config.relax.smoothness);
  CertBuffers out(inst.k);
  const bnbg_solver_cfg cfg = to_c(config);
  struct Ctx {
    const DebugHooks* hooks;
    int p;
  } ctx{hooks, inst.p()};
  bnbg_dual_hook on_dual = nullptr;
  bnbg_boundary_hook on_boundary = nullptr;
  if (hooks && hooks->on_dual_bound)
    on_dual = [](void* u, int n0, const int32_t* j0, int n1, const int32_t* j1, double psi) {
      auto* x = static_cast<Ctx*>(u);
      NodeState node;  // J0/J1 in fixing order; warm start not shipped back
      node.fixed_zero.assign(j0, j0 + n0);
      node.fixed_one.assign(j1, j1 + n1);
      node.warm_start = Eigen::VectorXd::Zero(x->p);
      x->hooks->on_dual_bound(node, psi);
    };
  if (hooks && hooks->on_batch_boundary)
    on_boundary = [](void* u, double lb, double ub) {
      static_cast<Ctx*>(u)->hooks->on_batch_boundary(lb, ub);
    };
  check(bnbg_solve(h.get(), &cfg, &out.c, on_dual, on_boundary, &ctx), h.get());
  return out.take();
}

// rashomon.hpp:149-218: records come back sorted by (objective, sequence)
// and are inserted into the reference's SupportTrie in that order.
inline RashomonResult collect_rashomon(const ProblemInstance& inst, const SolverConfig& config,
                                       const RashomonConfig& rconfig) {
  if (rconfig.epsilon < 0.0) throw input_error("rashomon: epsilon must be nonnegative");
  validate(inst);
  Handle h(inst, config.relax.smoothness);
  CertBuffers out(inst.k);
  const bnbg_solver_cfg cfg = to_c(config);
  bnbg_pool* pool = nullptr;
  check(bnbg_collect_rashomon(h.get(), &cfg, rconfig.epsilon, rconfig.cap, &out.c, &pool),
        h.get());
  std::unique_ptr<bnbg_pool, void (*)(bnbg_pool*)> guard(pool, bnbg_pool_free);
  RashomonResult result;
  result.certificate = out.take();
  std::vector<int32_t> seq(inst.k);
  std::vector<double> coef(inst.k);
  for (int i = 0; i < bnbg_pool_size(pool); ++i) {
    double obj = 0.0;
    const int len = bnbg_pool_record(pool, i, seq.data(), coef.data(), &obj);
    Eigen::VectorXd c = Eigen::VectorXd::Zero(len);
    for (int t = 0; t < len; ++t) c[t] = coef[t];
    result.pool.insert(std::vector<int>(seq.begin(), seq.begin() + len), c, obj);
  }
  return result;
}

// relaxation.hpp:163-255.  external_ws is accepted for signature parity; the
// workspace lives in HBM inside the handle.
inline RelaxationResult solve_batch_relaxation(
    const std::vector<NodeState>& batch, const ProblemInstance& inst, const RelaxConfig& config,
    double prune_threshold, BatchWorkspace* external_ws = nullptr,
    const std::function<void(int, double)>& dual_trace = nullptr) {
  (void)external_ws;
  if (batch.empty()) throw input_error("solve_batch_relaxation: empty batch");
  const int p = inst.p(), m = static_cast<int>(batch.size());
  const BatchMeta meta = BatchMeta::from_nodes(batch, inst.k);  // prox_kernel.hpp:52-90
  std::vector<double> warm(static_cast<size_t>(p) * m);
  for (int b = 0; b < m; ++b)
    for (int j = 0; j < p; ++j) warm[static_cast<size_t>(b) * p + j] = batch[b].warm_start[j];
  Handle h(inst, config.smoothness);
  const bnbg_relax_cfg cfg = to_c(config);
  std::vector<int32_t> status(m), iters(m);
  RelaxationResult res;
  res.beta = Eigen::MatrixXd::Zero(p, m);
  res.bounds.assign(m, 0.0);
  bnbg_trace_fn tr = nullptr;
  if (dual_trace)
    tr = [](void* u, int b, double psi) {
      (*static_cast<const std::function<void(int, double)>*>(u))(b, psi);
    };
  check(bnbg_relax_batch(h.get(), &cfg, m, reinterpret_cast<const uint8_t*>(meta.state.data()),
                         meta.reduced_budget.data(), warm.data(), prune_threshold,
                         res.beta.data(), res.bounds.data(), status.data(), iters.data(), tr,
                         const_cast<std::function<void(int, double)>*>(&dual_trace)),
        h.get());
  res.status.resize(m);
  res.iterations.assign(iters.begin(), iters.end());
  for (int b = 0; b < m; ++b)
    res.status[b] = status[b] == BNBG_PRUNABLE    ? NodeStatus::kPrunable
                    : status[b] == BNBG_CONVERGED ? NodeStatus::kConverged
                                                  : NodeStatus::kIterationCapped;
  return res;
}

// primal_heuristics.hpp:174-227 (workers accepted for signature parity)
inline ReoptResult reoptimize_supports(const std::vector<std::vector<int>>& supports,
                                       const ProblemInstance& inst, double smoothness = 0.0,
                                       int workers = 1) {
  (void)workers;
  Handle h(inst, smoothness);
  std::vector<int32_t> off(1, 0), idx;
  for (const auto& s : supports) {
    idx.insert(idx.end(), s.begin(), s.end());
    off.push_back(static_cast<int32_t>(idx.size()));
  }
  std::vector<double> coef(idx.size() + 1), obj(supports.size() + 1);
  check(bnbg_reoptimize(h.get(), static_cast<int>(supports.size()), off.data(), idx.data(),
                        coef.data(), obj.data()),
        h.get());
  ReoptResult out;
  for (size_t s = 0; s < supports.size(); ++s) {
    Eigen::VectorXd c = Eigen::VectorXd::Zero(off[s + 1] - off[s]);
    for (int t = off[s]; t < off[s + 1]; ++t) c[t - off[s]] = coef[t];
    out.coefficients.push_back(std::move(c));
    out.objectives.push_back(obj[s]);
  }
  return out;
}

}  // namespace bnbglm::b200
