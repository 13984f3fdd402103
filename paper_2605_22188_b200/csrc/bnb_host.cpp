// bnb_host.cpp -- host orchestration above the device engine and the C-ABI.
//
// The BnB loop keeps the reference's semantics (bnb_engine.hpp:116-291): a
// single orchestration thread owns the best-bound queue, the pending leaves
// and the incumbent; each pass ships one batch to the device, where the
// relaxation, rounding and branch selection run without per-node host
// synchronisation; re-optimisation of all candidate supports of the pass runs
// as one device batch.  Only the queue bookkeeping and child construction
// (node_model.hpp:77-105) stay on the host.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cmath>
#include <cstring>
#include <functional>
#include <limits>
#include <map>
#include <memory>
#include <queue>
#include <string>
#include <vector>

#include "../../include/bnbg.h"
#include "comm.hpp"
#include "engine.hpp"
#include "rng.hpp"

struct bnbg_handle {
  bnbg::Engine eng;
  int last_pool_m = 0;                 // batch of the last bnbg_pool_relax
  std::vector<int> last_pool_slots;
  // last sharded solve on this rank: node records sent / received through
  // the pool exchange, and the relaxation batch width of every pass
  long long shard_sent = 0, shard_recv = 0;
  std::vector<int> shard_batch;
};

struct bnbg_pool {
  struct Rec {
    std::vector<int> seq;
    std::vector<double> coef;
    double objective;
  };
  std::vector<Rec> recs;
};

static thread_local std::string g_last_error;

namespace {

using Clock = std::chrono::steady_clock;
constexpr double kInf = std::numeric_limits<double>::infinity();

int set_err(bnbg_handle* h, int code, const std::string& msg) {
  g_last_error = msg;
  if (h) h->eng.err = msg;
  return code;
}

// ---- node_model.hpp:114-172 -------------------------------------------------
// Open nodes live in the engine's device-resident pool (pool_kernels.cuh); the
// best-bound queue holds (lower bound, insertion sequence, pool slot) only.
// Ties on the bound pop in insertion order (FIFO), as in the reference.
struct QEntry {
  double bound;
  uint64_t seq;
  int slot;
  bool operator>(const QEntry& o) const {
    if (bound != o.bound) return bound > o.bound;
    return seq > o.seq;
  }
};

class NodeQueue {
 public:
  void push(double lb, int slot) { heap_.push(QEntry{lb, seq_++, slot}); }
  bool empty() const { return heap_.empty(); }
  size_t size() const { return heap_.size(); }
  double global_lb() const { return heap_.empty() ? kInf : heap_.top().bound; }
  QEntry pop() {
    QEntry e = heap_.top();
    heap_.pop();
    return e;
  }

 private:
  std::priority_queue<QEntry, std::vector<QEntry>, std::greater<QEntry>> heap_;
  uint64_t seq_ = 0;
};

// A leaf (kbar <= 0 or no free coordinate, node_model.hpp:33-36) skips the
// relaxation: only its fixed-in support and bound are needed (bnb_engine.hpp:164-175, :200).
struct Leaf {
  double lb;
  std::vector<int> j1;
};

// Pool slot allocator (host side of the device pool).
class SlotAllocator {
 public:
  int take() {
    if (!free_.empty()) {
      const int s = free_.back();
      free_.pop_back();
      return s;
    }
    return next_++;
  }
  void give(int s) { free_.push_back(s); }
  int high_water() const { return next_; }

 private:
  std::vector<int> free_;
  int next_ = 0;
};

// ---- search policies: solve (bnb_engine.hpp:304-307), rashomon (:169-196)
struct Policy {
  int kind = 0;
  double delta = 1e-6;
  double eps = 0.0;
  long long cap = -1;
  struct Staged {
    std::vector<int> seq;
    std::vector<double> coef;
    double objective;
  };
  std::vector<Staged> staged;
  std::map<std::vector<int>, int> staged_index;
  std::priority_queue<double> best_heap;
  double best_objective = kInf;

  double nth_best() const {
    if (cap < 0) return kInf;
    if ((long long)best_heap.size() < cap) return kInf;
    return best_heap.top();
  }
  double threshold(double ub) const {
    if (kind == 0) {
      if (!std::isfinite(ub)) return kInf;
      return ub - delta * std::max(1.0, std::fabs(ub));
    }
    const double tau = std::min(std::isfinite(ub) ? (1.0 + eps) * ub : kInf, nth_best());
    return std::nextafter(tau, kInf);
  }
  void on_model(const int* seq, int len, const double* coef, double objective) {
    if (kind != 1) return;
    best_objective = std::min(best_objective, objective);
    const double tau_now = std::min((1.0 + eps) * best_objective, nth_best()) + 1e-9;
    if (objective > tau_now) return;
    std::vector<int> key(seq, seq + len);
    std::sort(key.begin(), key.end());
    if (staged_index.count(key)) return;
    staged_index.emplace(std::move(key), (int)staged.size());
    staged.push_back({std::vector<int>(seq, seq + len), std::vector<double>(coef, coef + len),
                      objective});
    if (cap >= 0) {
      if ((long long)best_heap.size() < cap)
        best_heap.push(objective);
      else if (objective < best_heap.top()) {
        best_heap.pop();
        best_heap.push(objective);
      }
    }
  }
};

struct Timer {
  double& acc;
  Clock::time_point t0;
  explicit Timer(double& a) : acc(a), t0(Clock::now()) {}
  ~Timer() { acc += std::chrono::duration<double>(Clock::now() - t0).count(); }
};

int auto_batch(uint64_t budget, int n, int p, int k, int loss) {  // bnb_engine.hpp:75-88
  if (budget == 0) return -1;
  const double lb_bytes = 8.0 * 5.0 * p;
  const double loss_arrays = loss == BNBG_LOGISTIC ? 3.0 : 2.0;
  const double reopt_bytes = 8.0 * (loss_arrays * n + 2.0 * k);
  const double capacity = 0.9 * static_cast<double>(budget) / (lb_bytes + reopt_bytes);
  if (capacity < 2.0) return 1;
  int size = 1;
  while (2.0 * size <= capacity && size < (1 << 29)) size <<= 1;
  return size;
}

bnbg::RelaxParams relax_params(const bnbg_relax_cfg& c) {
  bnbg::RelaxParams r;
  r.max_iterations = c.max_iterations;
  r.gap_tolerance = c.gap_tolerance;
  r.check_interval = c.check_interval;
  r.acceleration = c.acceleration;
  return r;
}

// reoptimize_supports (primal_heuristics.hpp:174-227) is a pure function of
// each support SEQUENCE (indices in order: the order fixes the summation
// order of X_S beta) for a fixed instance and step, so a sequence's
// coefficients and objective never change within a solve.  Deep passes round
// many nodes to the same sequence, and later passes re-round sequences met
// before: each distinct sequence is re-optimised once per solve (ReoptMemo)
// and the results are handed out again.
struct ReoptMemo {
  static constexpr size_t kMaxEntries = 1 << 19;
  std::map<std::vector<int>, std::pair<std::vector<double>, double>> done;
  long long hits = 0;
};

static int reoptimize_unique(bnbg::Engine& eng, int nsup, const std::vector<int>& off,
                             const std::vector<int>& idx, double* coef, double* obj,
                             ReoptMemo& memo) {
  std::map<std::vector<int>, int> fresh;  // sequence -> slot in this launch
  std::vector<int> slot(nsup, -1), uoff(1, 0), uidx;
  for (int s = 0; s < nsup; ++s) {
    std::vector<int> key(idx.begin() + off[s], idx.begin() + off[s + 1]);
    auto hit = memo.done.find(key);
    if (hit != memo.done.end()) {
      std::copy(hit->second.first.begin(), hit->second.first.end(), coef + off[s]);
      obj[s] = hit->second.second;
      ++memo.hits;
      continue;
    }
    auto it = fresh.find(key);
    if (it == fresh.end()) {
      const int u = (int)uoff.size() - 1;
      it = fresh.emplace(std::move(key), u).first;
      uidx.insert(uidx.end(), idx.begin() + off[s], idx.begin() + off[s + 1]);
      uoff.push_back((int)uidx.size());
    }
    slot[s] = it->second;
  }
  const int nu = (int)uoff.size() - 1;
  if (nu == 0) return 0;
  std::vector<double> ucoef(uidx.size() + 1), uobj(nu + 1);
  if (int rc = eng.reoptimize(nu, uoff.data(), uidx.data(), ucoef.data(), uobj.data())) return rc;
  if (memo.done.size() + fresh.size() > ReoptMemo::kMaxEntries) memo.done.clear();  // bound host memory
  for (const auto& kv : fresh)
    memo.done.emplace(kv.first,
                      std::make_pair(std::vector<double>(ucoef.begin() + uoff[kv.second],
                                                         ucoef.begin() + uoff[kv.second + 1]),
                                     uobj[kv.second]));
  for (int s = 0; s < nsup; ++s) {
    const int u = slot[s];
    if (u < 0) continue;
    std::copy(ucoef.begin() + uoff[u], ucoef.begin() + uoff[u + 1], coef + off[s]);
    obj[s] = uobj[u];
  }
  return 0;
}

// Incumbent record exchanged between ranks: objective, |support|, support
// (sorted) and coefficients, as doubles.
struct IncRecord {
  static size_t doubles(int k) { return 3 + 2 * (size_t)k; }  // + the pass's error code
};

// bnb_engine.hpp:116-291 run_bnb.  With `comm` the nodes are sharded over
// ranks (comm.hpp): rank 0 starts with the root, every pass ends with the
// incumbent exchange, the termination/time-limit exchange and, when a rank
// starves, a node exchange between the ranks' device pools.
int run_bnb(bnbg_handle* h, const bnbg_solver_cfg& cfg, Policy& pol, bnbg_certificate* cert,
            bnbg_dual_hook on_dual, bnbg_boundary_hook on_boundary, void* user,
            bnbg::Comm* comm = nullptr) {
  bnbg::Engine& eng = h->eng;
  const int n = eng.n, p = eng.p, k = eng.k;
  const auto wall_start = Clock::now();
  auto elapsed = [&]() { return std::chrono::duration<double>(Clock::now() - wall_start).count(); };
  cert->optimal_value = kInf;
  cert->support_len = 0;
  cert->gap_percent = 0.0;
  cert->lower_bound = -kInf;
  cert->nodes_processed = cert->lb_batches = cert->reopt_batches = 0;
  cert->lower_bound_seconds = cert->reoptimization_seconds = cert->transfer_seconds = 0.0;
  cert->branch_generate_seconds = cert->total_seconds = 0.0;
  cert->relax_iterations = cert->node_iterations = cert->reopt_supports = 0;
  cert->device_seconds = 0.0;
  cert->status = BNBG_STATUS_OPTIMAL;
  if (cfg.relax.check_interval < 1 || cfg.relax.max_iterations < 1)
    return set_err(h, BNBG_INPUT_ERROR, "relax config: max_iterations, check_interval >= 1");
  bnbg::RelaxParams rp = relax_params(cfg.relax);
  {
    Timer t(cert->lower_bound_seconds);
    if (cfg.relax.smoothness > 0.0) eng.L = cfg.relax.smoothness;
  }
  const int batch_size =
      cfg.batch_size > 0 ? cfg.batch_size : auto_batch(cfg.memory_budget, n, p, k, eng.loss);
  if (batch_size < 1) return set_err(h, BNBG_INPUT_ERROR, "assemble_batch: batch_size >= 1");
  cert->batch_size_used = batch_size;

  NodeQueue queue;
  SlotAllocator slots;
  const int rank = comm ? comm->rank : 0, world = comm ? comm->world : 1;
  if (rank == 0) {
    const int root = slots.take();  // root_node (node_model.hpp:47-52)
    if (int rc = eng.pool_root(root)) return set_err(h, rc, eng.err);
    queue.push(-kInf, root);
  }
  int64_t global_open = 1;  // sharded: open nodes over all ranks after the last pass
  bool global_stop = false;
  std::vector<Leaf> pending;
  double inc_obj = kInf;
  std::vector<int> inc_sup;
  std::vector<double> inc_coef;
  int status = BNBG_STATUS_OPTIMAL;
  bnbg::PassResult pr;
  std::vector<int> batch_slots, n01, j0s, j1s, child_slots, rec;
  std::vector<double> batch_lb, rec_lb;
  const int kk = std::max(k, 1);
  // Sharded: a rank whose pass fails keeps taking part in the pass's
  // collectives with its error code, so every rank leaves together with a
  // non-OK status instead of blocking in the next allgather.
  int pass_rc = 0;
  std::string pass_msg;
  ReoptMemo memo;  // re-optimised sequences of this solve
  auto fail = [&](int rc, const std::string& msg) -> int {
    if (!comm) return set_err(h, rc, msg);
    if (!pass_rc) {
      pass_rc = rc;
      pass_msg = msg;
    }
    return 0;
  };
  // Test instrumentation (BNBG_FAULT="rank:pass"): that rank's pass fails
  // with a numeric error, exercising the error path of the collectives.
  int fault_rank = -1, fault_pass = -1;
  int64_t rotate = 0;
  if (comm) {
    if (const char* r = getenv("BNBG_BALANCE_ROTATE")) rotate = std::max(0, atoi(r));
    h->shard_sent = h->shard_recv = 0;
    h->shard_batch.clear();
    if (const char* f = getenv("BNBG_FAULT")) sscanf(f, "%d:%d", &fault_rank, &fault_pass);
  }
  int pass_no = 0;
  // After a collective: the lowest-ranked failure ends the solve on all ranks.
  auto collective_error = [&](const double* codes, size_t stride) -> int {
    for (int r = 0; r < world; ++r) {
      const int rc = (int)codes[(size_t)r * stride];
      if (!rc) continue;
      if (r == rank) return set_err(h, rc, pass_msg);
      return set_err(h, rc, "sharded solve: rank " + std::to_string(r) + " failed (code " +
                                std::to_string(rc) + ")");
    }
    return 0;
  };

  while (comm ? global_open > 0 : (!queue.empty() || !pending.empty())) {
    if (comm ? global_stop : elapsed() > cfg.time_limit) {
      status = BNBG_STATUS_TIME_LIMIT;
      break;
    }
    const double threshold = pol.threshold(inc_obj);
    std::vector<Leaf> leaves;
    {
      Timer t(cert->transfer_seconds);
      int popped = 0, discarded = 0;  // assemble_batch node_model.hpp:158-172
      batch_slots.clear();
      batch_lb.clear();
      while (!queue.empty() && popped < batch_size) {
        const QEntry e = queue.pop();
        if (e.bound >= threshold) {
          ++discarded;
          slots.give(e.slot);
          continue;
        }
        batch_slots.push_back(e.slot);
        batch_lb.push_back(e.bound);
        ++popped;
      }
      cert->nodes_processed += popped + discarded;
      for (Leaf& leaf : pending) {
        ++cert->nodes_processed;
        if (leaf.lb >= threshold) continue;
        leaves.push_back(std::move(leaf));
      }
      pending.clear();
    }
    const int m = (int)batch_slots.size();
    if (!comm && m == 0 && leaves.empty()) continue;
    if (comm) {
      h->shard_batch.push_back(m);
      if (rank == fault_rank && pass_no == fault_pass)
        if (int e = fail(BNBG_NUMERIC_ERROR, "injected fault (BNBG_FAULT)")) return e;
    }
    ++pass_no;

    if (m > 0) {
      Timer t(cert->lower_bound_seconds);
      const int rc = eng.relax_pool(m, batch_slots.data(), rp, threshold, on_dual != nullptr, pr,
                                    on_dual != nullptr, &n01, &j0s, &j1s);
      if (rc) {
        if (int e = fail(rc, eng.err)) return e;
      }
    }
    if (m > 0 && !pass_rc) {
      ++cert->lb_batches;
      cert->relax_iterations += pr.iterations;
      cert->node_iterations += pr.node_iterations;
      if (on_dual) {  // replay in the reference's order (relaxation.hpp:201-203)
        for (int e = 0; e < pr.n_evals; ++e)
          for (int b = 0; b < m; ++b) {
            const double psi = pr.trace[(size_t)e * m + b];
            if (std::isnan(psi)) continue;
            on_dual(user, n01[2 * b], j0s.data() + (size_t)b * p, n01[2 * b + 1],
                    j1s.data() + (size_t)b * kk, psi);
          }
      }
    }

    // one re-optimization batch: leaf supports, then rounded columns (:193-212)
    std::vector<int> offsets(1, 0), sidx;
    {
      Timer t(cert->reoptimization_seconds);
      for (const Leaf& leaf : leaves) {
        sidx.insert(sidx.end(), leaf.j1.begin(), leaf.j1.end());
        offsets.push_back((int)sidx.size());
      }
      for (int b = 0; b < m && !pass_rc; ++b) {
        if (pr.status[b] == BNBG_PRUNABLE) continue;
        const int* row = pr.sup.data() + (size_t)b * kk;
        sidx.insert(sidx.end(), row, row + pr.len[b]);
        offsets.push_back((int)sidx.size());
      }
    }
    const int nsup = (int)offsets.size() - 1;
    std::vector<double> coef(sidx.size() + 1), obj(nsup + 1);
    if (nsup > 0 && !pass_rc) {
      Timer t(cert->reoptimization_seconds);
      const int rc = reoptimize_unique(eng, nsup, offsets, sidx, coef.data(), obj.data(), memo);
      if (rc) {
        if (int e = fail(rc, eng.err)) return e;
      }
    }
    if (nsup > 0 && !pass_rc) {
      ++cert->reopt_batches;
      cert->reopt_supports += nsup;
    }
    {
      Timer t(cert->branch_generate_seconds);
      for (int s = 0; s < nsup && !pass_rc; ++s) {  // incumbent update (bnb_engine.hpp:216-240)
        const int len = offsets[s + 1] - offsets[s];
        const int* sq = sidx.data() + offsets[s];
        const double* cf = coef.data() + offsets[s];
        pol.on_model(sq, len, cf, obj[s]);
        if (obj[s] < inc_obj) {
          inc_obj = obj[s];
          std::vector<int> order(len);
          for (int i = 0; i < len; ++i) order[i] = i;
          std::sort(order.begin(), order.end(), [&](int a, int b) { return sq[a] < sq[b]; });
          inc_sup.resize(len);
          inc_coef.resize(len);
          for (int i = 0; i < len; ++i) {
            inc_sup[i] = sq[order[i]];
            inc_coef[i] = cf[order[i]];
          }
        }
      }
      if (comm) {  // global incumbent: lowest objective, ties to the lowest rank
        const size_t R = IncRecord::doubles(kk);
        std::vector<double> mine(R, 0.0), all(R * world);
        mine[R - 1] = (double)pass_rc;  // error code of this rank's pass
        mine[0] = inc_obj;
        mine[1] = (double)inc_sup.size();
        for (size_t i = 0; i < inc_sup.size(); ++i) {
          mine[2 + i] = (double)inc_sup[i];
          mine[2 + kk + i] = inc_coef[i];
        }
        if (int rc = comm->allgather(eng, mine.data(), sizeof(double) * R, all.data()))
          return set_err(h, rc, eng.err);
        if (int e = collective_error(all.data() + R - 1, R)) return e;
        int win = -1;
        for (int r = 0; r < world; ++r)
          if (win < 0 || all[R * r] < all[R * win]) win = r;
        const double* w = all.data() + R * win;
        if (w[0] < inc_obj || (w[0] == inc_obj && win < rank)) {
          inc_obj = w[0];
          const int len = (int)w[1];
          inc_sup.resize(len);
          inc_coef.resize(len);
          for (int i = 0; i < len; ++i) {
            inc_sup[i] = (int)w[2 + i];
            inc_coef[i] = w[2 + kk + i];
          }
        }
      }
      const double post_threshold = pol.threshold(inc_obj);
      if (m > 0) {
        // prune test, branch variable and children on the device (:243-256)
        child_slots.resize(2 * (size_t)m);
        for (int i = 0; i < 2 * m; ++i) child_slots[i] = slots.take();
        int surv = 0, bad = -1;
        int rc = eng.pool_reserve(slots.high_water());
        if (!rc)
          rc = eng.branch_pool(m, batch_slots.data(), batch_lb.data(), post_threshold,
                               child_slots.data(), surv, bad, rec, rec_lb);
        if (rc) {
          if (int e = fail(rc, eng.err)) return e;
          surv = 0;
        } else if (bad >= 0) {
          if (int e = fail(BNBG_LOGIC_ERROR, "select_branch_variable: no free coordinate"))
            return e;
          surv = 0;
        }
        for (int i = 2 * m - 1; i >= 2 * surv; --i) slots.give(child_slots[i]);
        const int RI = 4 + kk;
        for (int c = 0; c < 2 * surv; ++c) {
          const int* r = rec.data() + (size_t)c * RI;
          if (r[1]) {  // leaf child -> pending_leaves (node_model.hpp:33-36)
            pending.push_back(Leaf{rec_lb[c], std::vector<int>(r + 4, r + 4 + r[2])});
            slots.give(r[0]);
          } else {
            queue.push(rec_lb[c], r[0]);
          }
        }
        for (int s : batch_slots) slots.give(s);
      }
    }
    if (comm) {  // termination, time limit and load balance over the ranks
      Timer t(cert->transfer_seconds);
      double lb_local = queue.global_lb();
      for (const Leaf& leaf : pending) lb_local = std::min(lb_local, leaf.lb);
      const double mine[5] = {(double)queue.size(), (double)pending.size(), lb_local,
                              elapsed() > cfg.time_limit ? 1.0 : 0.0, (double)pass_rc};
      std::vector<double> all(5 * (size_t)world);
      if (int rc = comm->allgather(eng, mine, sizeof(mine), all.data()))
        return set_err(h, rc, eng.err);
      if (int e = collective_error(all.data() + 4, 5)) return e;
      global_open = 0;
      global_stop = false;
      std::vector<int64_t> counts(world), moves((size_t)world * world);
      for (int r = 0; r < world; ++r) {
        counts[r] = (int64_t)all[5 * r];
        global_open += counts[r] + (int64_t)all[5 * r + 1];
        global_stop = global_stop || all[5 * r + 3] != 0.0;
      }
      bool move = global_open > 0 && !global_stop &&
                  bnbg::balance_plan(world, counts.data(), moves.data());
      // Test instrumentation (BNBG_BALANCE_ROTATE=k): on top of the plan,
      // every rank hands min(k, queue / 2) nodes to the next rank each pass,
      // exercising pool_pack / exchange / pool_unpack on balanced searches.
      if (rotate > 0 && global_open > 0 && !global_stop && world > 1) {
        if (!move) std::fill(moves.begin(), moves.end(), 0);
        for (int r = 0; r < world; ++r) {
          int64_t left = counts[r];
          for (int q = 0; q < world; ++q) left -= moves[(size_t)r * world + q];
          const int64_t t = std::min<int64_t>(rotate, left / 2);
          if (t > 0) {
            moves[(size_t)r * world + (r + 1) % world] += t;
            move = true;
          }
        }
      }
      if (move) {
        // donors hand over every other node from the top of their queue
        std::vector<int64_t> send_n(world, 0), recv_n(world, 0);
        int64_t nsend = 0, nrecv = 0;
        for (int r = 0; r < world; ++r) {
          send_n[r] = moves[(size_t)rank * world + r];
          recv_n[r] = moves[(size_t)r * world + rank];
          nsend += send_n[r];
          nrecv += recv_n[r];
        }
        std::vector<int> send_slots;
        std::vector<double> send_lb;
        if (nsend > 0) {
          std::vector<QEntry> keep;
          int idx = 0;
          while ((int64_t)send_slots.size() < nsend && !queue.empty()) {
            const QEntry e = queue.pop();
            const int64_t need = nsend - (int64_t)send_slots.size();
            if (idx % 2 == 1 || (int64_t)queue.size() < need) {
              send_slots.push_back(e.slot);
              send_lb.push_back(e.bound);
            } else {
              keep.push_back(e);
            }
            ++idx;
          }
          for (const QEntry& e : keep) queue.push(e.bound, e.slot);
        }
        uint8_t* d_send = nullptr;
        uint8_t* d_recv = nullptr;
        if (int rc = eng.pool_pack((int)nsend, send_slots.data(), send_lb.data(), &d_send))
          return set_err(h, rc, eng.err);
        if (int rc = eng.pool_recv_buffer((int)nrecv, &d_recv)) return set_err(h, rc, eng.err);
        if (int rc = comm->exchange(eng, send_n, d_send, recv_n, d_recv, eng.node_record_bytes()))
          return set_err(h, rc, eng.err);
        for (int s : send_slots) slots.give(s);
        h->shard_sent += nsend;
        h->shard_recv += nrecv;
        if (nrecv > 0) {
          std::vector<int> rslots(nrecv);
          for (auto& s : rslots) s = slots.take();
          if (int rc = eng.pool_reserve(slots.high_water())) return set_err(h, rc, eng.err);
          std::vector<double> rlb(nrecv);
          if (int rc = eng.pool_unpack((int)nrecv, rslots.data(), rlb.data()))
            return set_err(h, rc, eng.err);
          for (int64_t i = 0; i < nrecv; ++i) queue.push(rlb[i], rslots[i]);
        }
      }
    }
    if (on_boundary) {  // :259-265
      double lb = queue.global_lb();
      for (const Leaf& leaf : pending) lb = std::min(lb, leaf.lb);
      on_boundary(user, std::min(lb, inc_obj), inc_obj);
    }
  }

  double lb_open = queue.global_lb();
  for (const Leaf& leaf : pending) lb_open = std::min(lb_open, leaf.lb);
  if (comm) {  // counters are sums over ranks; the open bound is the global minimum
    const double mine[7] = {(double)cert->nodes_processed, (double)cert->lb_batches,
                            (double)cert->reopt_batches,   (double)cert->relax_iterations,
                            (double)cert->node_iterations, (double)cert->reopt_supports,
                            lb_open};
    std::vector<double> all(7 * (size_t)world);
    if (int rc = comm->allgather(eng, mine, sizeof(mine), all.data()))
      return set_err(h, rc, eng.err);
    double tot[6] = {0, 0, 0, 0, 0, 0};
    lb_open = kInf;
    for (int r = 0; r < world; ++r) {
      for (int q = 0; q < 6; ++q) tot[q] += all[7 * r + q];
      lb_open = std::min(lb_open, all[7 * r + 6]);
    }
    cert->nodes_processed = (long long)tot[0];
    cert->lb_batches = (long long)tot[1];
    cert->reopt_batches = (long long)tot[2];
    cert->relax_iterations = (long long)tot[3];
    cert->node_iterations = (long long)tot[4];
    cert->reopt_supports = (long long)tot[5];
  }
  const double ub = inc_obj;  // certificate (:268-290)
  cert->status = status;
  cert->optimal_value = ub;
  cert->support_len = (int)inc_sup.size();
  for (size_t i = 0; i < inc_sup.size(); ++i) {
    if (cert->support) cert->support[i] = inc_sup[i];
    if (cert->coefficients) cert->coefficients[i] = inc_coef[i];
  }
  if (status == BNBG_STATUS_OPTIMAL) {
    cert->lower_bound = ub;
    cert->gap_percent = 0.0;
  } else {
    const double lb = std::min(lb_open, ub);
    cert->lower_bound = lb;
    cert->gap_percent =
        !std::isfinite(ub) ? 100.0 : 100.0 * (ub - lb) / std::max(std::fabs(ub), 1e-12);
  }
  cert->total_seconds = elapsed();
  return BNBG_OK;
}

}  // namespace

// ===========================================================================
// C-ABI
// ===========================================================================
// The pool pass seam is two calls (bnbg_pool_relax, then bnbg_pool_branch)
// sharing the batch workspaces (slots, states, betas, status, best bounds,
// branch variables).  Every other entry point that may write those buffers
// or the pool ends the pass: a later bnbg_pool_branch is rejected instead of
// branching on overwritten data.
static void end_pool_pass(bnbg_handle* h) {
  h->last_pool_m = 0;
  h->last_pool_slots.clear();
}

extern "C" {

void bnbg_relax_cfg_default(bnbg_relax_cfg* c) {
  c->max_iterations = 2000;
  c->gap_tolerance = 1e-6;
  c->check_interval = 10;
  c->acceleration = 1;
  c->smoothness = 0.0;
  c->workers = 1;
}

void bnbg_solver_cfg_default(bnbg_solver_cfg* c) {
  c->batch_size = 0;
  c->memory_budget = uint64_t(1) << 30;
  c->time_limit = kInf;
  c->prune_slack = 1e-6;
  bnbg_relax_cfg_default(&c->relax);
  c->profile = 0;
  c->workers = 1;
}

int bnbg_auto_batch_size(uint64_t memory_budget, int n, int p, int k, int loss) {
  return auto_batch(memory_budget, n, p, k, loss);
}

int bnbg_validate(const double* X, const double* y, int n, int p, int loss, int k, double M,
                  double lambda2) {  // problem.hpp:36-51
  if (n <= 0 || p <= 0) return set_err(nullptr, BNBG_INPUT_ERROR, "instance: empty design matrix");
  for (size_t i = 0; i < (size_t)n * p; ++i)
    if (!std::isfinite(X[i])) return set_err(nullptr, BNBG_INPUT_ERROR, "instance: non-finite entries");
  for (int i = 0; i < n; ++i)
    if (!std::isfinite(y[i])) return set_err(nullptr, BNBG_INPUT_ERROR, "instance: non-finite entries");
  if (k < 1 || k > p) return set_err(nullptr, BNBG_INPUT_ERROR, "instance: k must satisfy 1 <= k <= p");
  if (!(M > 0.0)) return set_err(nullptr, BNBG_INPUT_ERROR, "instance: M must be positive");
  if (!(lambda2 > 0.0)) return set_err(nullptr, BNBG_INPUT_ERROR, "instance: lambda2 must be positive");
  if (loss != BNBG_SQUARED && loss != BNBG_LOGISTIC)
    return set_err(nullptr, BNBG_INPUT_ERROR, "instance: unknown loss");
  if (loss == BNBG_LOGISTIC)
    for (int i = 0; i < n; ++i)
      if (y[i] != 1.0 && y[i] != -1.0)
        return set_err(nullptr, BNBG_INPUT_ERROR, "logistic label must be -1 or +1");
  return BNBG_OK;
}

// problem.hpp:70-132.  AR(1) Toeplitz Cholesky factor in closed form:
// L[j][0] = rho^j, L[j][l] = rho^(j-l) sqrt(1-rho^2); row i = L g_i summed in
// ascending l with fma (bit-identical to the oracle's restatement).
int bnbg_generate_synthetic(int n, int p, int k, double rho, int loss, double snr, uint64_t seed,
                            double* X, double* y, int32_t* support) {
  if (n < 1 || p < 1) return set_err(nullptr, BNBG_INPUT_ERROR, "generator: n, p >= 1");
  if (k < 1 || k > p) return set_err(nullptr, BNBG_INPUT_ERROR, "generator: k must satisfy 1 <= k <= p");
  if (rho < 0.0 || rho >= 1.0)
    return set_err(nullptr, BNBG_INPUT_ERROR, "generator: correlation must lie in [0, 1)");
  if (!(snr > 0.0)) return set_err(nullptr, BNBG_INPUT_ERROR, "generator: snr must be positive");
  bnbg::Xoshiro256pp rng(seed);
  std::vector<double> G((size_t)n * p);
  for (auto& g : G) g = rng.gaussian();
  if (rho > 0.0) {
    std::vector<double> pw(p);
    pw[0] = 1.0;
    for (int d = 1; d < p; ++d) pw[d] = pw[d - 1] * rho;
    const double sr = std::sqrt(1.0 - rho * rho);
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i) {
      const double* g = G.data() + (size_t)i * p;
      for (int j = 0; j < p; ++j) {
        double acc = pw[j] * g[0];
        for (int l = 1; l <= j; ++l) acc = std::fma(pw[j - l] * sr, g[l], acc);
        X[(size_t)j * n + i] = acc;
      }
    }
  } else {
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < p; ++j) X[(size_t)j * n + i] = G[(size_t)i * p + j];
  }
  const int step = p / k;
  for (int t = 1; t <= k; ++t) support[t - 1] = t * step - 1;
  std::vector<double> signal(n, 0.0);
  for (int t = 0; t < k; ++t) {
    const double* col = X + (size_t)support[t] * n;
    for (int i = 0; i < n; ++i) signal[i] += col[i];
  }
  if (loss == BNBG_SQUARED) {
    double s2 = 0.0;
    for (double v : signal) s2 += v * v;
    const double sigma2 = std::sqrt(s2) / snr;
    const double sd = std::sqrt(sigma2);
    for (int i = 0; i < n; ++i) y[i] = signal[i] + sd * rng.gaussian();
  } else {
    for (int i = 0; i < n; ++i) {
      const double t = signal[i];
      double prob;
      if (t >= 0.0) {
        const double e = std::exp(-t);
        prob = 1.0 / (1.0 + e);
      } else {
        const double e = std::exp(t);
        prob = e / (1.0 + e);
      }
      y[i] = rng.uniform() < prob ? 1.0 : -1.0;
    }
  }
  return BNBG_OK;
}

int bnbg_create(const double* X, const double* y, int n, int p, int loss, int k, double M,
                double lambda2, double L, int device, bnbg_handle** out) {
  *out = nullptr;
  if (int rc = bnbg_validate(X, y, n, p, loss, k, M, lambda2)) return rc;
  auto* h = new bnbg_handle();
  const int rc = h->eng.init(X, y, n, p, loss, k, M, lambda2, L, device);
  if (rc) {
    g_last_error = h->eng.err;
    delete h;
    return rc;
  }
  *out = h;
  return BNBG_OK;
}

void bnbg_destroy(bnbg_handle* h) { delete h; }

const char* bnbg_last_error(const bnbg_handle* h) {
  if (h && !h->eng.err.empty()) return h->eng.err.c_str();
  return g_last_error.c_str();
}

double bnbg_smoothness(bnbg_handle* h) { return h->eng.L; }

int bnbg_relax_batch(bnbg_handle* h, const bnbg_relax_cfg* cfg, int m, const uint8_t* state,
                     const int32_t* kbar, const double* warm, double prune_threshold,
                     double* beta_out, double* bounds_out, int32_t* status_out,
                     int32_t* iters_out, bnbg_trace_fn trace, void* user) {
  end_pool_pass(h);
  bnbg_relax_cfg c;
  if (cfg)
    c = *cfg;
  else
    bnbg_relax_cfg_default(&c);
  if (m <= 0) return set_err(h, BNBG_INPUT_ERROR, "solve_batch_relaxation: empty batch");
  if (c.check_interval < 1 || c.max_iterations < 1)
    return set_err(h, BNBG_INPUT_ERROR, "relax config: max_iterations, check_interval >= 1");
  const double saved_L = h->eng.L;
  if (c.smoothness > 0.0) h->eng.L = c.smoothness;
  bnbg::PassResult pr;
  const int rc =
      h->eng.relax_raw(m, relax_params(c), prune_threshold, state, kbar, warm, trace != nullptr, pr);
  h->eng.L = saved_L;
  if (rc) return set_err(h, rc, h->eng.err);
  std::memcpy(beta_out, pr.beta.data(), sizeof(double) * pr.beta.size());
  std::memcpy(bounds_out, pr.bounds.data(), sizeof(double) * m);
  std::memcpy(status_out, pr.status.data(), sizeof(int) * m);
  std::memcpy(iters_out, pr.iters.data(), sizeof(int) * m);
  if (trace) {
    for (int e = 0; e < pr.n_evals; ++e)
      for (int b = 0; b < m; ++b) {
        const double psi = pr.trace[(size_t)e * m + b];
        if (!std::isnan(psi)) trace(user, b, psi);
      }
  }
  return BNBG_OK;
}

int bnbg_pack_batch(bnbg_handle* h, int m, const int32_t* j0_off, const int32_t* j0_idx,
                    const int32_t* j1_off, const int32_t* j1_idx, uint8_t* state_out,
                    int32_t* kbar_out, int32_t* free_count_out) {
  end_pool_pass(h);
  if (m <= 0) return set_err(h, BNBG_INPUT_ERROR, "batch meta: empty batch");
  const int p = h->eng.p;
  bnbg::BatchLists L;
  L.m = m;
  std::vector<uint8_t> mark(p);
  for (int b = 0; b < m; ++b) {
    std::fill(mark.begin(), mark.end(), 0);
    for (int pass = 0; pass < 2; ++pass) {
      const int32_t* off = pass ? j1_off : j0_off;
      const int32_t* idx = pass ? j1_idx : j0_idx;
      if (off[b + 1] < off[b]) return set_err(h, BNBG_INPUT_ERROR, "batch meta: bad offsets");
      for (int t = off[b]; t < off[b + 1]; ++t) {
        if (idx[t] < 0 || idx[t] >= p)
          return set_err(h, BNBG_INPUT_ERROR, "batch meta: index out of range");
        if (mark[idx[t]]++)
          return set_err(h, BNBG_INPUT_ERROR, "batch meta: J0 and J1 must be disjoint sets");
      }
    }
  }
  L.z_off.assign(j0_off, j0_off + m + 1);
  L.o_off.assign(j1_off, j1_off + m + 1);
  L.z_idx.assign(j0_idx + j0_off[0], j0_idx + j0_off[m]);
  L.o_idx.assign(j1_idx + j1_off[0], j1_idx + j1_off[m]);
  for (auto& v : L.z_off) v -= j0_off[0];
  for (auto& v : L.o_off) v -= j1_off[0];
  const int rc = h->eng.pack_lists(L, state_out, kbar_out, free_count_out);
  return rc ? set_err(h, rc, h->eng.err) : BNBG_OK;
}

int bnbg_round_support(bnbg_handle* h, int m, const double* beta, const uint8_t* state,
                       const int32_t* kbar, const int32_t* one_off, const int32_t* one_idx,
                       int32_t* support_out, int32_t* len_out) {
  end_pool_pass(h);
  const int rc = h->eng.round_select(m, beta, state, kbar, one_off, one_idx, support_out, len_out,
                                     nullptr);
  return rc ? set_err(h, rc, h->eng.err) : BNBG_OK;
}

int bnbg_select_branch(bnbg_handle* h, int m, const double* beta, const uint8_t* state,
                       int32_t* j_out) {
  end_pool_pass(h);
  std::vector<int> kb(std::max(m, 1), 0);
  const int rc =
      h->eng.round_select(m, beta, state, kb.data(), nullptr, nullptr, nullptr, nullptr, j_out);
  return rc ? set_err(h, rc, h->eng.err) : BNBG_OK;
}

int bnbg_reoptimize(bnbg_handle* h, int nsup, const int32_t* offsets, const int32_t* idx,
                    double* coef_out, double* obj_out) {
  for (int s = 0; s < nsup; ++s)
    for (int t = offsets[s]; t < offsets[s + 1]; ++t)
      if (idx[t] < 0 || idx[t] >= h->eng.p)
        return set_err(h, BNBG_INPUT_ERROR, "reoptimize_supports: index out of range");
  const int rc = h->eng.reoptimize(nsup, offsets, idx, coef_out, obj_out);
  return rc ? set_err(h, rc, h->eng.err) : BNBG_OK;
}

int bnbg_pool_root(bnbg_handle* h, int slot) {
  end_pool_pass(h);
  if (slot < 0) return set_err(h, BNBG_INPUT_ERROR, "pool_root: slot must be nonnegative");
  const int rc = h->eng.pool_root(slot);
  return rc ? set_err(h, rc, h->eng.err) : BNBG_OK;
}

int bnbg_pool_relax(bnbg_handle* h, const bnbg_relax_cfg* cfg, int m, const int32_t* slots,
                    double prune_threshold, double* bounds_out, int32_t* status_out,
                    int32_t* iters_out, int32_t* support_out, int32_t* len_out) {
  bnbg_relax_cfg c;
  if (cfg)
    c = *cfg;
  else
    bnbg_relax_cfg_default(&c);
  if (m <= 0) return set_err(h, BNBG_INPUT_ERROR, "solve_batch_relaxation: empty batch");
  if (c.check_interval < 1 || c.max_iterations < 1)
    return set_err(h, BNBG_INPUT_ERROR, "relax config: max_iterations, check_interval >= 1");
  for (int b = 0; b < m; ++b)
    if (slots[b] < 0 || slots[b] >= h->eng.pool_capacity())
      return set_err(h, BNBG_INPUT_ERROR, "pool_relax: slot out of range");
  const double saved_L = h->eng.L;
  if (c.smoothness > 0.0) h->eng.L = c.smoothness;
  bnbg::PassResult pr;
  const int rc =
      h->eng.relax_pool(m, slots, relax_params(c), prune_threshold, false, pr, false, nullptr,
                        nullptr, nullptr);
  h->eng.L = saved_L;
  if (rc) return set_err(h, rc, h->eng.err);
  const int kk = std::max(h->eng.k, 1);
  std::memcpy(bounds_out, pr.bounds.data(), sizeof(double) * m);
  std::memcpy(status_out, pr.status.data(), sizeof(int) * m);
  std::memcpy(iters_out, pr.iters.data(), sizeof(int) * m);
  if (support_out) std::memcpy(support_out, pr.sup.data(), sizeof(int) * (size_t)m * kk);
  if (len_out) std::memcpy(len_out, pr.len.data(), sizeof(int) * m);
  h->last_pool_m = m;
  h->last_pool_slots.assign(slots, slots + m);
  return BNBG_OK;
}

int bnbg_pool_branch(bnbg_handle* h, int m, const double* lb_in, double post_threshold,
                     const int32_t* free_slots, int32_t* survivors_out, int32_t* rec_out,
                     double* child_lb_out) {
  if (m != h->last_pool_m || m <= 0)
    return set_err(h, BNBG_INPUT_ERROR, "pool_branch: m must match the last pool_relax batch");
  {
    // children are written while the parents' pool slots are read: the 2m
    // free slots must be distinct and disjoint from the batch's slots
    std::vector<int> seen(free_slots, free_slots + 2 * m);
    seen.insert(seen.end(), h->last_pool_slots.begin(), h->last_pool_slots.end());
    std::sort(seen.begin(), seen.end());
    if (!seen.empty() && seen.front() < 0)
      return set_err(h, BNBG_INPUT_ERROR, "pool_branch: free slots must be nonnegative");
    if (std::adjacent_find(seen.begin(), seen.end()) != seen.end())
      return set_err(h, BNBG_INPUT_ERROR,
                     "pool_branch: free slots must be distinct and not slots of the batch");
  }
  int hw = 0;
  for (int i = 0; i < 2 * m; ++i) hw = std::max(hw, free_slots[i] + 1);
  if (int rc = h->eng.pool_reserve(hw)) return set_err(h, rc, h->eng.err);
  int surv = 0, bad = -1;
  std::vector<int> rec;
  std::vector<double> rlb;
  const int rc = h->eng.branch_pool(m, h->last_pool_slots.data(), lb_in, post_threshold,
                                    free_slots, surv, bad, rec, rlb);
  end_pool_pass(h);  // one branch per relaxed batch
  if (rc) return set_err(h, rc, h->eng.err);
  if (bad >= 0) return set_err(h, BNBG_LOGIC_ERROR, "select_branch_variable: no free coordinate");
  *survivors_out = surv;
  if (rec_out && !rec.empty()) std::memcpy(rec_out, rec.data(), sizeof(int) * rec.size());
  if (child_lb_out && !rlb.empty()) std::memcpy(child_lb_out, rlb.data(), sizeof(double) * rlb.size());
  return BNBG_OK;
}

int bnbg_gemm(bnbg_handle* h, int trans, int m, const double* B, double* C) {
  end_pool_pass(h);
  const int rc = h->eng.gemm_probe(trans, m, B, C);
  return rc ? set_err(h, rc, h->eng.err) : BNBG_OK;
}

int bnbg_solve(bnbg_handle* h, const bnbg_solver_cfg* cfg, bnbg_certificate* cert,
               bnbg_dual_hook on_dual, bnbg_boundary_hook on_boundary, void* user) {
  end_pool_pass(h);
  bnbg_solver_cfg c;
  if (cfg)
    c = *cfg;
  else
    bnbg_solver_cfg_default(&c);
  Policy pol;
  pol.kind = 0;
  pol.delta = c.prune_slack;
  const double saved_L = h->eng.L;
  const int rc = run_bnb(h, c, pol, cert, on_dual, on_boundary, user);
  h->eng.L = saved_L;
  return rc;
}

int bnbg_nccl_init(bnbg_handle* h, const uint8_t* uid, int rank, int world) {
  if (world < 1 || rank < 0 || rank >= world)
    return set_err(h, BNBG_INPUT_ERROR, "nccl_init: rank must lie in [0, world)");
  const int rc = h->eng.nccl_init(uid, rank, world);
  return rc ? set_err(h, rc, h->eng.err) : BNBG_OK;
}

int bnbg_solve_sharded(bnbg_handle* h, const bnbg_solver_cfg* cfg, const bnbg_comm_ops* ops,
                       bnbg_certificate* cert) {
  end_pool_pass(h);
  bnbg_solver_cfg c;
  if (cfg)
    c = *cfg;
  else
    bnbg_solver_cfg_default(&c);
  Policy pol;
  pol.kind = 0;
  pol.delta = c.prune_slack;
  std::unique_ptr<bnbg::Comm> comm;
  if (ops) {
    if (ops->world < 1 || ops->rank < 0 || ops->rank >= ops->world || !ops->allgather ||
        !ops->alltoallv)
      return set_err(h, BNBG_INPUT_ERROR, "solve_sharded: invalid communicator");
    comm.reset(new bnbg::CallbackComm(ops));
  } else {
    if (!h->eng.nccl_comm)
      return set_err(h, BNBG_INPUT_ERROR, "solve_sharded: no communicator (bnbg_nccl_init)");
    auto* nc = new bnbg::NcclComm();
    nc->comm = h->eng.nccl_comm;
    nc->rank = h->eng.nccl_rank;
    nc->world = h->eng.nccl_world;
    comm.reset(nc);
  }
  const double saved_L = h->eng.L;
  const int rc = run_bnb(h, c, pol, cert, nullptr, nullptr, nullptr, comm.get());
  h->eng.L = saved_L;
  return rc;
}

int bnbg_collect_rashomon(bnbg_handle* h, const bnbg_solver_cfg* cfg, double epsilon, long long cap,
                          bnbg_certificate* cert, bnbg_pool** pool_out) {
  end_pool_pass(h);
  *pool_out = nullptr;
  if (epsilon < 0.0) return set_err(h, BNBG_INPUT_ERROR, "rashomon: epsilon must be nonnegative");
  bnbg_solver_cfg c;
  if (cfg)
    c = *cfg;
  else
    bnbg_solver_cfg_default(&c);
  Policy pol;
  pol.kind = 1;
  pol.eps = epsilon;
  pol.cap = cap;
  const double saved_L = h->eng.L;
  const int rc = run_bnb(h, c, pol, cert, nullptr, nullptr, nullptr);
  h->eng.L = saved_L;
  if (rc) return rc;
  // compaction against the final threshold (rashomon.hpp:201-216)
  const double tau_final = (1.0 + epsilon) * cert->optimal_value + 1e-9;
  std::vector<int> live;
  for (int i = 0; i < (int)pol.staged.size(); ++i)
    if (pol.staged[i].objective <= tau_final) live.push_back(i);
  std::sort(live.begin(), live.end(), [&](int a, int b) {
    if (pol.staged[a].objective != pol.staged[b].objective)
      return pol.staged[a].objective < pol.staged[b].objective;
    return pol.staged[a].seq < pol.staged[b].seq;
  });
  if (cap >= 0 && (long long)live.size() > cap) live.resize(cap);
  auto* pool = new bnbg_pool();
  for (int i : live)
    pool->recs.push_back({pol.staged[i].seq, pol.staged[i].coef, pol.staged[i].objective});
  *pool_out = pool;
  return BNBG_OK;
}

int bnbg_pool_size(const bnbg_pool* pool) { return pool ? (int)pool->recs.size() : 0; }

int bnbg_pool_record(const bnbg_pool* pool, int i, int32_t* seq_out, double* coef_out,
                     double* objective_out) {
  const auto& r = pool->recs[i];
  std::memcpy(seq_out, r.seq.data(), sizeof(int) * r.seq.size());
  std::memcpy(coef_out, r.coef.data(), sizeof(double) * r.coef.size());
  *objective_out = r.objective;
  return (int)r.seq.size();
}

void bnbg_pool_free(bnbg_pool* pool) { delete pool; }

long long bnbg_kernel_launches(const bnbg_handle* h) { return h->eng.launches; }

int bnbg_gemm_stats(const bnbg_handle* h, double* gemm_ms, double* gemm_flops,
                    long long* gemm_launches) {
  const auto& e = h->eng;
  if (gemm_ms) *gemm_ms = e.kc_ms[bnbg::KC_GEMM_NN] + e.kc_ms[bnbg::KC_GEMM_TN];
  if (gemm_flops) *gemm_flops = e.kc_flops[bnbg::KC_GEMM_NN] + e.kc_flops[bnbg::KC_GEMM_TN];
  if (gemm_launches)
    *gemm_launches = e.kc_launches[bnbg::KC_GEMM_NN] + e.kc_launches[bnbg::KC_GEMM_TN];
  return BNBG_OK;
}

void bnbg_set_timing(bnbg_handle* h, int enabled) { h->eng.timing = enabled != 0; }

int bnbg_kernel_stats(const bnbg_handle* h, int kc, double* ms, double* flops,
                      long long* launches) {
  if (kc < 0 || kc >= bnbg::KC_COUNT) return BNBG_INPUT_ERROR;
  const auto& e = h->eng;
  if (ms) *ms = e.kc_ms[kc];
  if (flops) *flops = e.kc_flops[kc];
  if (launches) *launches = e.kc_launches[kc];
  return BNBG_OK;
}

int bnbg_pass_profile(const bnbg_handle* h, double* ns_out, int count) {
  return const_cast<bnbg_handle*>(h)->eng.pass_profile(ns_out, count);
}

int bnbg_shard_stats(const bnbg_handle* h, long long* out, int cap) {
  const int np = (int)h->shard_batch.size();
  if (cap >= 1) out[0] = h->shard_sent;
  if (cap >= 2) out[1] = h->shard_recv;
  if (cap >= 3) out[2] = np;
  for (int i = 0; i < np && 3 + i < cap; ++i) out[3 + i] = h->shard_batch[i];
  return 3 + np;
}

int bnbg_transfer_bytes(const bnbg_handle* h, long long* h2d, long long* d2h) {
  if (h2d) *h2d = h->eng.h2d_bytes;
  if (d2h) *d2h = h->eng.d2h_bytes;
  return BNBG_OK;
}

}  // extern "C"
