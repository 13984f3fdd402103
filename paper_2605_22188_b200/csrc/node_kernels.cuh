// node_kernels.cuh -- per-node (column-local) sm_100a kernels of the pass.
//
//   k_pack          VK1  BatchMeta::from_nodes (prox_kernel.hpp:52-90)
//   k_prox_fista    VK5  U = V - eta G, prox_step_column + FISTA momentum
//                        (relaxation.hpp:227-244, prox_kernel.hpp:236-276)
//   k_eval          VK6-8 primal_values / dual_bounds / freeze-restart
//                        (relaxation.hpp:108-147, :194-221)
//   k_compact       active-column compaction (order preserving)
//   k_round_select  VK9+VK11 round_support / select_branch_variable
//                        (primal_heuristics.hpp:134-163)
//   k_reopt         VK10 reoptimize_supports (primal_heuristics.hpp:174-227)
//   k_conj_prox / k_g_value / k_g_conj   test entry points (prox_kernel.hpp)
//
// One CTA per column; the column's p coordinates live in shared memory and
// are sorted with a block bitonic sort in the reference order (key desc,
// index asc).  Every reduction has a fixed association order.
#pragma once
#include "device_math.cuh"

namespace bnbg {

constexpr int kNodeThreads = 256;

struct RelaxDev {
  int p, n2, mcap;
  double* B;
  double* V;
  const double* G;     // split-K slabs: G + s*split_stride + col*p
  long long split_stride;
  int nsplit;
  const uint8_t* state;
  const int* kbar;
  const int* pf;
  double* t;
  double* best;
  double* last_gap;
  uint8_t* frozen;
  int* status;
  int* iters;
  int* act;
  int* d_ma;
  int* d_err;
  double eta, rho, M, lambda2;
  int accel;
};

constexpr int kMaxSplit = 8;

// G = sum of the split-K slabs, added in slab order (loads issued together)
__device__ __forceinline__ double gsum(const RelaxDev& r, int b, int j) {
  double part[kMaxSplit];
#pragma unroll
  for (int s = 0; s < kMaxSplit; ++s)
    part[s] = s < r.nsplit ? r.G[(size_t)s * r.split_stride + (size_t)b * r.p + j] : 0.0;
  double g = part[0];
#pragma unroll
  for (int s = 1; s < kMaxSplit; ++s)
    if (s < r.nsplit) g += part[s];
  return g;
}

// --------------------------------------------------------------------------
// VK1 packer: dense CoordState column + reduced budget + free count, and the
// warm start copied into B and V.  Lists are CSR over the batch.
// --------------------------------------------------------------------------
__global__ void k_pack(int p, int k, int m, const int* z_off, const int* z_idx, const int* o_off,
                       const int* o_idx, uint8_t* state, int* kbar, int* pf, const double* warm,
                       double* B, double* V, double* t, double* best, double* last_gap,
                       uint8_t* frozen, int* status, int* iters, int* act, int max_it) {
  const int b = blockIdx.x;
  if (b >= m) return;
  uint8_t* col = state + (size_t)b * p;
  for (int j = threadIdx.x; j < p; j += blockDim.x) {
    col[j] = kFree;
    const double w = warm[(size_t)b * p + j];
    B[(size_t)b * p + j] = w;
    V[(size_t)b * p + j] = w;
  }
  __syncthreads();
  const int z0 = z_off[b], z1 = z_off[b + 1], q0 = o_off[b], q1 = o_off[b + 1];
  for (int t2 = z0 + threadIdx.x; t2 < z1; t2 += blockDim.x) col[z_idx[t2]] = kFixedZero;
  for (int t2 = q0 + threadIdx.x; t2 < q1; t2 += blockDim.x) col[o_idx[t2]] = kFixedOne;
  if (threadIdx.x == 0) {
    const int kb = k - (q1 - q0);
    kbar[b] = kb > 0 ? kb : 0;
    pf[b] = p - (z1 - z0) - (q1 - q0);
    t[b] = 1.0;
    best[b] = -d_inf();
    last_gap[b] = d_inf();
    frozen[b] = 0;
    status[b] = kCapped;
    iters[b] = max_it;
    act[b] = b;
  }
}

// init for the raw-state API (bnbg_relax_batch): state/kbar/B given.
__global__ void k_init_cols(int p, int m, const uint8_t* state, int* pf, const double* B, double* V,
                            double* t, double* best, double* last_gap, uint8_t* frozen, int* status,
                            int* iters, int* act, int max_it) {
  __shared__ double red[kNodeThreads / 32];
  const int b = blockIdx.x;
  if (b >= m) return;
  int cnt = 0;
  for (int j = threadIdx.x; j < p; j += kNodeThreads) {
    V[(size_t)b * p + j] = B[(size_t)b * p + j];
    cnt += state[(size_t)b * p + j] == kFree;
  }
  const int nfree = (int)block_sum<kNodeThreads>((double)cnt, red);
  if (threadIdx.x == 0) {
    pf[b] = nfree;
    t[b] = 1.0;
    best[b] = -d_inf();
    last_gap[b] = d_inf();
    frozen[b] = 0;
    status[b] = kCapped;
    iters[b] = max_it;
    act[b] = b;
  }
}

// --------------------------------------------------------------------------
// Block-wide inclusive scan of f(0..len-1) into out[] (each thread scans a
// contiguous chunk, chunk totals are combined with a warp scan).  Fixed
// association order, so the result is deterministic.
// --------------------------------------------------------------------------
template <int NT, class F>
__device__ __forceinline__ void block_scan_incl(int len, F f, double* out, double* wtot) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int chunk = (len + NT - 1) / NT;
  const int beg = min(len, tid * chunk), end = min(len, beg + chunk);
  double run = 0.0;
  for (int i = beg; i < end; ++i) {
    run += f(i);
    out[i] = run;
  }
  double incl = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  __syncthreads();
  if (lane == 31) wtot[warp] = incl;
  __syncthreads();
  double off = incl - run;
  for (int w = 0; w < warp; ++w) off += wtot[w];
  if (off != 0.0)
    for (int i = beg; i < end; ++i) out[i] += off;
  __syncthreads();
}

// --------------------------------------------------------------------------
// Boundary-seeded PAVA on the sorted keys (prox_kernel.hpp:132-170).
// v_r = prox_huber(key_r, w, M) for r < kbar and key_r otherwise; the only
// violation is at the kbar boundary and the pooled block [lo,hi] grows from
// [kbar-1, kbar] with the reference's rule (left first, then right).
//
// The reference re-sums the block after every expansion (O(len^2), one
// thread).  Here the block sums come from two prefix scans anchored at the
// boundary (left part SL, right part SR -- sums of block members only, so no
// cancellation), and warp 0 evaluates 32 consecutive expansion states per
// step, following the reference's decision sequence exactly: the first state
// whose left test fires (or whose right test fails) is found with a ballot.
// All threads call; lo/hi/pooled are returned to every thread.
// --------------------------------------------------------------------------
template <int NT>
__device__ void block_pava(const double* key, int pf, int kbar, double w, double M, double* scan,
                           double* wtot, int& blo, int& bhi, double& bval) {
  blo = 0;
  bhi = -1;
  bval = 0.0;
  if (kbar <= 0 || kbar >= pf) return;
  if (d_prox_huber(key[kbar - 1], w, M) >= key[kbar]) return;
  double* SL = scan;         // SL[i] = key[kbar-1] + ... + key[kbar-1-i]
  double* SR = scan + kbar;  // SR[e] = key[kbar] + ... + key[kbar+e]
  block_scan_incl<NT>(kbar, [&](int i) { return key[kbar - 1 - i]; }, SL, wtot);
  block_scan_incl<NT>(pf - kbar, [&](int e) { return key[kbar + e]; }, SR, wtot);
  auto pooled = [&](int lo, int hi) {
    const int len = hi - lo + 1;
    const double sum = SL[kbar - 1 - lo] + SR[hi - kbar];
    const double mean_w = w * (double)(kbar - lo) / len;
    return d_prox_huber(sum / len, mean_w, M);
  };
  auto v = [&](int r) { return r < kbar ? d_prox_huber(key[r], w, M) : key[r]; };
  // Each batch evaluates NT consecutive states of the current phase (thread
  // t owns state t); the first event is found with a ballot + per-warp min.
  // Shared scratch is double-buffered so one barrier per batch suffices.
  __shared__ int s_first[2][NT / 32];
  __shared__ unsigned char s_L[2][NT], s_R[2][NT];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int lo = kbar - 1, hi = kbar, buf = 0;
  bool left_phase = true;
  for (;;) {
    bool L = false, R = false, ev;
    if (left_phase) {  // state t = (lo - t, hi)
      const int cl = lo - tid;
      if (cl >= 0) {
        const double pv = pooled(cl, hi);
        L = cl > 0 && v(cl - 1) < pv;
        R = hi < pf - 1 && pv < v(hi + 1);
      }
      ev = !L;
    } else {  // state t = (lo, hi + t)
      const int ch = hi + tid;
      if (ch <= pf - 1) {
        const double pv = pooled(lo, ch);
        L = lo > 0 && v(lo - 1) < pv;
        R = ch < pf - 1 && pv < v(ch + 1);
      }
      ev = L || !R;
    }
    s_L[buf][tid] = L;
    s_R[buf][tid] = R;
    const unsigned bal = __ballot_sync(0xffffffffu, ev);
    if (lane == 0) s_first[buf][warp] = bal ? warp * 32 + __ffs(bal) - 1 : NT;
    __syncthreads();
    int first = NT;
#pragma unroll
    for (int w2 = 0; w2 < NT / 32; ++w2) first = min(first, s_first[buf][w2]);
    if (first == NT) {
      if (left_phase)
        lo -= NT;
      else
        hi += NT;
      buf ^= 1;
      continue;
    }
    const bool Lf = s_L[buf][first], Rf = s_R[buf][first];
    buf ^= 1;
    if (left_phase) {
      lo -= first;
      if (!Rf) break;
      ++hi;
      left_phase = false;
    } else {
      hi += first;
      if (!Lf) break;
      --lo;
      left_phase = true;
    }
  }
  blo = lo;
  bhi = hi;
  bval = pooled(lo, hi);
}

// shared-memory layout of the column kernels: key[n2] doubles, idx[n2] ints,
// u[p] doubles, scan[n2] doubles
__host__ __device__ inline size_t column_smem_bytes(int p, int n2) {
  return sizeof(double) * (size_t)n2 * 2 + sizeof(int) * (size_t)n2 + sizeof(double) * (size_t)p +
         sizeof(double) * 16;
}

// --------------------------------------------------------------------------
// VK5: proximal-gradient step + FISTA momentum for every active column.
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(kNodeThreads) k_prox_fista(RelaxDev r) {
  extern __shared__ __align__(16) double sm[];
  const int c = blockIdx.x;
  if (c >= *r.d_ma) return;
  const int b = r.act[c];
  const int p = r.p, n2 = r.n2;
  double* key = sm;
  int* idx = reinterpret_cast<int*>(key + n2);
  double* u = reinterpret_cast<double*>(idx + n2);
  double* scan = u + p;
  __shared__ double wtot[kNodeThreads / 32];

  const uint8_t* st = r.state + (size_t)b * p;
  double* Vb = r.V + (size_t)b * p;
  double* Bb = r.B + (size_t)b * p;
  const double tm = r.t[b];
  bool bad = false;
  for (int j = threadIdx.x; j < n2; j += kNodeThreads) {
    if (j < p) {
      const double v = Vb[j];
      bad |= !isfinite(v);
      const double uj = v - r.eta * gsum(r, b, j);  // U = V - eta G (relaxation.hpp:229)
      u[j] = uj;
      key[j] = st[j] == kFree ? r.rho * fabs(uj) : -1.0;
    } else {
      key[j] = -2.0;
    }
    idx[j] = j;
  }
  if (bad) atomicMin(r.d_err, b);  // refresh_predictions' finite check (relaxation.hpp:76-81)
  bitonic_sort_desc<kNodeThreads>(key, idx, n2);
  const int kb = r.kbar[b], pf = r.pf[b];
  int lo, hi;
  double pooled;
  block_pava<kNodeThreads>(key, pf, kb, r.rho, r.M, scan, wtot, lo, hi, pooled);
  const double inv_rho = 1.0 / r.rho;
  const double t_next = 0.5 * (1.0 + sqrt(1.0 + 4.0 * tm * tm));
  const double coef = (tm - 1.0) / t_next;
  // free coordinates by rank (prox_kernel.hpp:267-275)
  for (int rk = threadIdx.x; rk < pf; rk += kNodeThreads) {
    const int j = idx[rk];
    const double uj = u[j];
    double out;
    const bool in_block = hi >= lo && rk >= lo && rk <= hi;
    if (rk >= kb && !in_block) {
      out = 0.0;
    } else {
      const double v = in_block ? pooled : d_prox_huber(key[rk], r.rho, r.M);
      const double sign = uj > 0.0 ? 1.0 : (uj < 0.0 ? -1.0 : 0.0);
      out = uj - inv_rho * sign * v;
    }
    const double bo = Bb[j];
    Vb[j] = r.accel ? out + coef * (out - bo) : out;
    Bb[j] = out;
  }
  // fixed coordinates (prox_kernel.hpp:261-266)
  for (int j = threadIdx.x; j < p; j += kNodeThreads) {
    const uint8_t s = st[j];
    if (s == kFree) continue;
    const double uj = u[j];
    const double out = s == kFixedZero ? 0.0 : uj - inv_rho * d_prox_huber(r.rho * uj, r.rho, r.M);
    const double bo = Bb[j];
    Vb[j] = r.accel ? out + coef * (out - bo) : out;
    Bb[j] = out;
  }
  if (threadIdx.x == 0 && r.accel) r.t[b] = t_next;
}

// --------------------------------------------------------------------------
// g(beta) for one column already staged: returns +inf off the domain.
// (prox_kernel.hpp:310-347 + recover_core primal_heuristics.hpp:60-99)
// key/idx: scratch of n2 entries.  All threads return the same value.
// --------------------------------------------------------------------------
template <int NT>
__device__ double block_g_value(const double* beta, const uint8_t* st, int p, int n2, int kbar,
                                double M, double* key, int* idx, double* red, int* ired) {
  const double box_tol = M * (1.0 + 1e-9);
  double fixed = 0.0;
  int bad = 0, nz = 0;
  for (int j = threadIdx.x; j < n2; j += NT) {
    double kv = -2.0;
    if (j < p) {
      const double bj = beta[j];
      const uint8_t s = st[j];
      if (s == kFixedZero) {
        bad |= bj != 0.0;
        kv = -1.0;
      } else if (s == kFixedOne) {
        bad |= fabs(bj) > box_tol;
        fixed += bj * bj;
        kv = -1.0;
      } else {
        bad |= fabs(bj) > box_tol;
        nz += bj != 0.0;
        kv = fabs(bj);
      }
    }
    key[j] = kv;
    idx[j] = j;
  }
  const double fixed_part = block_sum<NT>(fixed, red);
  const int any_bad = block_or<NT>(bad, ired);
  const int nonzero = (int)block_sum<NT>((double)nz, red);
  if (any_bad) return d_inf();
  if (kbar <= 0) return nonzero > 0 ? d_inf() : 0.5 * fixed_part;
  bitonic_sort_desc<NT>(key, idx, n2);
  int pf = 0;
  {
    int cnt = 0;
    for (int j = threadIdx.x; j < n2; j += NT) cnt += key[j] >= 0.0;
    pf = (int)block_sum<NT>((double)cnt, red);
  }
  if (nonzero <= kbar) {
    double s = 0.0;
    for (int rk = threadIdx.x; rk < pf; rk += NT) s += key[rk] * key[rk];
    return 0.5 * (fixed_part + block_sum<NT>(s, red));
  }
  // binding case: suffix sums from the bottom; tail below kbar tree-summed
  double tl = 0.0;
  for (int rk = kbar + threadIdx.x; rk < pf; rk += NT) tl += key[rk];
  const double tail = block_sum<NT>(tl, red);
  __shared__ double s_tau;
  __shared__ int s_cap, s_ok;
  if (threadIdx.x == 0) {
    // suffix[s] for s < kbar, sequential from the bottom (primal_heuristics.hpp:82-84)
    double suffix[64];
    int ok = 0, cap = 0;
    double tau = 0.0;
    if (kbar <= 64) {
      double acc = tail;
      for (int s = kbar - 1; s >= 0; --s) {
        acc += key[s];
        suffix[s] = acc;
      }
      for (int s = 0; s < kbar; ++s) {
        const double tv = suffix[s] / (double)(kbar - s);
        const double upper = s == 0 ? d_inf() : key[s - 1];
        const double lower = key[s];
        if (upper >= tv && tv >= lower) {
          ok = 1;
          tau = tv;
          cap = s;
          break;
        }
      }
    } else {
      // kbar > 64: recompute suffixes on the fly (O(kbar^2) worst case, rare)
      for (int s = 0; s < kbar && !ok; ++s) {
        double acc = tail;
        for (int r2 = kbar - 1; r2 >= s; --r2) acc += key[r2];
        const double tv = acc / (double)(kbar - s);
        const double upper = s == 0 ? d_inf() : key[s - 1];
        const double lower = key[s];
        if (upper >= tv && tv >= lower) {
          ok = 1;
          tau = tv;
          cap = s;
        }
      }
    }
    s_ok = ok && !(tau > M * (1.0 + 1e-9));
    s_tau = tau;
    s_cap = cap;
  }
  __syncthreads();
  if (!s_ok) return d_inf();
  const double tau = s_tau;
  const int cap = s_cap;
  double fp = 0.0;
  for (int rk = threadIdx.x; rk < pf; rk += NT) fp += rk < cap ? key[rk] * key[rk] : tau * key[rk];
  return 0.5 * (fixed_part + block_sum<NT>(fp, red));
}

// g*(q): sum_{J1} H_M(q) + TopSum_kbar over free H_M(q) (prox_kernel.hpp:351-370)
template <int NT>
__device__ double block_g_conj(const double* q, double qscale, const uint8_t* st, int p, int n2,
                               int kbar, double M, double* key, int* idx, double* red) {
  double ones = 0.0;
  for (int j = threadIdx.x; j < n2; j += NT) {
    double kv = -2.0;
    if (j < p) {
      const double qj = q[j] * qscale;
      const uint8_t s = st[j];
      if (s == kFixedOne) {
        ones += d_huber(qj, M);
        kv = -1.0;
      } else if (s == kFree) {
        kv = d_huber(qj, M);
      } else {
        kv = -1.0;
      }
    }
    key[j] = kv;
    idx[j] = j;
  }
  const double total = block_sum<NT>(ones, red);
  if (kbar <= 0) return total;
  bitonic_sort_desc<NT>(key, idx, n2);
  double s = 0.0;
  for (int rk = threadIdx.x; rk < kbar && rk < n2; rk += NT) s += key[rk] >= 0.0 ? key[rk] : 0.0;
  return total + block_sum<NT>(s, red);
}

// --------------------------------------------------------------------------
// VK6-VK8: bound evaluation of every active column (relaxation.hpp:194-221).
// Expects fresh part_loss/part_conj (from the EVAL GEMM on B) and G = X'R(B).
// --------------------------------------------------------------------------
struct EvalArgs {
  const double* part_loss;
  const double* part_conj;
  int nrb;
  int part_ld;
  int iter;
  double prune_threshold;
  double gap_tolerance;
  double* trace;  // [eval_idx * mcap + b] or nullptr
  int eval_idx;
};

__global__ void __launch_bounds__(kNodeThreads) k_eval(RelaxDev r, EvalArgs e) {
  extern __shared__ __align__(16) double sm[];
  const int c = blockIdx.x;
  if (c >= *r.d_ma) return;
  const int b = r.act[c];
  const int p = r.p, n2 = r.n2;
  double* key = sm;
  int* idx = reinterpret_cast<int*>(key + n2);
  double* q = reinterpret_cast<double*>(idx + n2);
  __shared__ double red[kNodeThreads / 32];
  __shared__ int ired[kNodeThreads / 32];
  __shared__ int s_restart;
  const uint8_t* st = r.state + (size_t)b * p;
  const double* Bb = r.B + (size_t)b * p;

  const double inv2l = 1.0 / (2.0 * r.lambda2);
  bool bad = false;
  for (int j = threadIdx.x; j < p; j += kNodeThreads) {
    bad |= !isfinite(Bb[j]);
    q[j] = -gsum(r, b, j) * inv2l;  // Z = -R; Q = X'Z; Q *= 1/(2 lambda2)
  }
  if (bad) atomicMin(r.d_err, b);
  const int kb = r.kbar[b];
  // Phi = sum l(S) + 2 lambda2 g(B)  (relaxation.hpp:108-123)
  const double g = block_g_value<kNodeThreads>(Bb, st, p, n2, kb, r.M, key, idx, red, ired);
  // Psi = -sum l*(R) - 2 lambda2 g*(Q), Q = X'(-R) / (2 lambda2) (relaxation.hpp:127-147)
  const double gs = block_g_conj<kNodeThreads>(q, 1.0, st, p, n2, kb, r.M, key, idx, red);
  if (threadIdx.x == 0) {
    s_restart = 0;
    double loss = 0.0, conj = 0.0;
    for (int rb = 0; rb < e.nrb; ++rb) {
      loss += e.part_loss[(size_t)rb * e.part_ld + b];
      conj += e.part_conj[(size_t)rb * e.part_ld + b];
    }
    const double phi = loss + 2.0 * r.lambda2 * g;
    const double psi = -conj - 2.0 * r.lambda2 * gs;
    double best = r.best[b];
    if (psi > best) best = psi;
    r.best[b] = best;
    if (e.trace) e.trace[(size_t)e.eval_idx * r.mcap + b] = psi;
    const double gap = (phi - best) / fmax(1.0, fabs(phi));
    if (best >= e.prune_threshold) {
      r.frozen[b] = 1;
      r.status[b] = kPrunable;
      r.iters[b] = e.iter;
    } else if (gap <= e.gap_tolerance) {
      r.frozen[b] = 1;
      r.status[b] = kConverged;
      r.iters[b] = e.iter;
    } else if (r.accel && phi - psi > r.last_gap[b]) {
      r.t[b] = 1.0;
      s_restart = 1;
    }
    r.last_gap[b] = phi - psi;
  }
  __syncthreads();
  if (s_restart) {
    double* Vb = r.V + (size_t)b * p;
    for (int j = threadIdx.x; j < p; j += kNodeThreads) Vb[j] = Bb[j];
  }
}

// order-preserving compaction of the active list (single CTA)
__global__ void __launch_bounds__(1024) k_compact(int* act, int* d_ma, const uint8_t* frozen) {
  __shared__ int warp_tot[32];
  __shared__ int s_base;
  const int ma = *d_ma;
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
  for (int base = 0; base < ma; base += 1024) {
    const int i = base + threadIdx.x;
    int a = -1;
    int keep = 0;
    if (i < ma) {
      a = act[i];
      keep = !frozen[a];
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    const int pre = __popc(bal & ((1u << lane) - 1));
    if (lane == 0) warp_tot[warp] = __popc(bal);
    __syncthreads();
    int off = 0;
    for (int w = 0; w < warp; ++w) off += warp_tot[w];
    const int base_out = s_base;
    __syncthreads();
    if (keep) act[base_out + off + pre] = a;
    if (threadIdx.x == 1023) {
      int tot = 0;
      for (int w = 0; w < 32; ++w) tot += warp_tot[w];
      s_base = base_out + tot;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *d_ma = s_base;
}

// --------------------------------------------------------------------------
// VK9 + VK11: rounding support and branching variable from one sort of the
// free |beta| (key desc, index asc).  support row b = J1 ++ top-kbar free.
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(kNodeThreads)
    k_round_select(int p, int n2, int k, const double* beta, const uint8_t* state, const int* kbar,
                   const int* one_off, const int* one_idx, int* sup, int* len, int* jbranch) {
  extern __shared__ __align__(16) double sm[];
  const int b = blockIdx.x;
  double* key = sm;
  int* idx = reinterpret_cast<int*>(key + n2);
  const double* bb = beta + (size_t)b * p;
  const uint8_t* st = state + (size_t)b * p;
  for (int j = threadIdx.x; j < n2; j += kNodeThreads) {
    key[j] = j < p ? (st[j] == kFree ? fabs(bb[j]) : -1.0) : -2.0;
    idx[j] = j;
  }
  bitonic_sort_desc<kNodeThreads>(key, idx, n2);
  if (threadIdx.x == 0) {
    int l = 0;
    if (one_off) {
      for (int t = one_off[b]; t < one_off[b + 1]; ++t) sup[(size_t)b * k + l++] = one_idx[t];
    }
    const int kb = kbar[b];
    for (int rk = 0; rk < kb && rk < n2 && key[rk] >= 0.0; ++rk) sup[(size_t)b * k + l++] = idx[rk];
    if (len) len[b] = l;
    if (jbranch) jbranch[b] = key[0] >= 0.0 ? idx[0] : -1;
  }
}

// --------------------------------------------------------------------------
// VK10: box-constrained refit of each support by projected gradient,
// step 1/(L + 2 lambda2), stop at |beta - next|/step <= 1e-8 or 5000
// iterations; objective exact at the returned coefficients.
// --------------------------------------------------------------------------
constexpr int kReoptThreads = 256;

__global__ void __launch_bounds__(kReoptThreads)
    k_reopt(int n, const double* __restrict__ X, const double* __restrict__ y, int loss, double M,
            double lambda2, double step, const int* off, const int* sidx, double* deriv_scratch,
            double* coef_out, double* obj_out) {
  extern __shared__ __align__(16) double sm[];
  constexpr int NW = kReoptThreads / 32;
  const int s = blockIdx.x;
  const int q = off[s + 1] - off[s];
  const int* S = sidx + off[s];
  double* beta = sm;            // q
  double* red = beta + q;       // NW * q
  double* nxt = red + NW * q;   // q
  __shared__ int s_stop;
  __shared__ double wred[NW];
  double* d = deriv_scratch + (size_t)s * n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int r = tid; r < q; r += kReoptThreads) beta[r] = 0.0;
  if (tid == 0) s_stop = 0;
  __syncthreads();
  if (q > 0) {
    for (int it = 0; it < 5000; ++it) {
      // scores and derivative for this thread's rows (primal_heuristics.hpp:194-209)
      for (int i = tid; i < n; i += kReoptThreads) {
        double sc = 0.0;
        for (int r = 0; r < q; ++r) sc += beta[r] * X[(size_t)S[r] * n + i];
        d[i] = d_loss_deriv(loss, sc, y[i]);
      }
      // grad_r = X_{S_r}' deriv (+ 2 lambda2 beta_r)  (:210-211)
      for (int r = 0; r < q; ++r) {
        const double* col = X + (size_t)S[r] * n;
        double a = 0.0;
        for (int i = tid; i < n; i += kReoptThreads) a += col[i] * d[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0) red[warp * q + r] = a;
      }
      __syncthreads();
      for (int r = tid; r < q; r += kReoptThreads) {
        double gr = 0.0;
        for (int w = 0; w < NW; ++w) gr += red[w * q + r];
        gr += 2.0 * lambda2 * beta[r];
        double v = beta[r] - step * gr;
        v = v < -M ? -M : v;
        v = v > M ? M : v;
        nxt[r] = v;
      }
      __syncthreads();
      if (tid == 0) {
        double gm2 = 0.0;
        for (int r = 0; r < q; ++r) {
          const double dl = beta[r] - nxt[r];
          gm2 += dl * dl;
        }
        s_stop = (sqrt(gm2) / step) <= 1e-8;
      }
      __syncthreads();
      for (int r = tid; r < q; r += kReoptThreads) beta[r] = nxt[r];
      const int stop = s_stop;
      __syncthreads();
      if (stop) break;
    }
  }
  // objective lambda2 |beta|^2 + sum l(X_S beta)  (:217-222)
  double acc = 0.0;
  for (int i = tid; i < n; i += kReoptThreads) {
    double sc = 0.0;
    for (int r = 0; r < q; ++r) sc += beta[r] * X[(size_t)S[r] * n + i];
    acc += d_loss_value(loss, sc, y[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) wred[warp] = acc;
  __syncthreads();
  if (tid == 0) {
    double sq = 0.0;
    for (int r = 0; r < q; ++r) sq += beta[r] * beta[r];
    double obj = lambda2 * sq;
    for (int w = 0; w < NW; ++w) obj += wred[w];
    obj_out[s] = obj;
  }
  for (int r = tid; r < q; r += kReoptThreads) coef_out[off[s] + r] = beta[r];
}

// --------------------------------------------------------------------------
// VK10 fast paths (q <= QMAX).  Every thread of the CTA keeps the whole
// coefficient vector in registers and recomputes the update redundantly from
// the same shared partial sums, so one barrier per iteration suffices and all
// threads take the same stopping decision.
//
// k_reopt_direct: the reference's gather form (primal_heuristics.hpp:194-215):
//   scores = sum_r beta_r X[:,S_r] (r ascending), deriv = l'(scores),
//   grad_r = X[:,S_r]' deriv + 2 lambda2 beta_r, next = clip(beta - step grad).
// --------------------------------------------------------------------------
constexpr int kReoptFastThreads = 512;

template <int QMAX>
__global__ void __launch_bounds__(kReoptFastThreads)
    k_reopt_direct(int n, const double* __restrict__ X, const double* __restrict__ y, int loss,
                   double M, double lambda2, double step, const int* off, const int* sidx,
                   double* deriv_scratch, double* coef_out, double* obj_out) {
  constexpr int NW = kReoptFastThreads / 32;
  __shared__ double red[2][NW][QMAX];
  __shared__ const double* cols[QMAX];
  __shared__ double wred[NW];
  const int s = blockIdx.x;
  const int q = off[s + 1] - off[s];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < q) cols[tid] = X + (size_t)sidx[off[s] + tid] * n;
  __syncthreads();
  double* d = deriv_scratch + (size_t)s * n;
  double beta[QMAX];
#pragma unroll
  for (int r = 0; r < QMAX; ++r) beta[r] = 0.0;
  int buf = 0;
  if (q > 0) {
    for (int it = 0; it < 5000; ++it) {
      double part[QMAX];
#pragma unroll
      for (int r = 0; r < QMAX; ++r) part[r] = 0.0;
      for (int i = tid; i < n; i += kReoptFastThreads) {
        double sc = 0.0;
#pragma unroll
        for (int r = 0; r < QMAX; ++r)
          if (r < q) sc += beta[r] * cols[r][i];
        const double di = d_loss_deriv(loss, sc, y[i]);
#pragma unroll
        for (int r = 0; r < QMAX; ++r)
          if (r < q) part[r] += cols[r][i] * di;
      }
#pragma unroll
      for (int r = 0; r < QMAX; ++r) {
        if (r < q) {
          double a = part[r];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
          if (lane == 0) red[buf][warp][r] = a;
        }
      }
      __syncthreads();
      double gm2 = 0.0;
#pragma unroll
      for (int r = 0; r < QMAX; ++r) {
        if (r < q) {
          double g = 0.0;
          for (int w = 0; w < NW; ++w) g += red[buf][w][r];
          g += 2.0 * lambda2 * beta[r];
          double v = beta[r] - step * g;
          v = v < -M ? -M : v;
          v = v > M ? M : v;
          const double dl = beta[r] - v;
          gm2 += dl * dl;
          beta[r] = v;
        }
      }
      buf ^= 1;
      if (sqrt(gm2) / step <= 1e-8) break;
    }
  }
  (void)d;
  double acc = 0.0;
  for (int i = tid; i < n; i += kReoptFastThreads) {
    double sc = 0.0;
#pragma unroll
    for (int r = 0; r < QMAX; ++r)
      if (r < q) sc += beta[r] * cols[r][i];
    acc += d_loss_value(loss, sc, y[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) wred[warp] = acc;
  __syncthreads();
  if (tid == 0) {
    double sq = 0.0;
#pragma unroll
    for (int r = 0; r < QMAX; ++r)
      if (r < q) sq += beta[r] * beta[r];
    double obj = lambda2 * sq;
    for (int w = 0; w < NW; ++w) obj += wred[w];
    obj_out[s] = obj;
#pragma unroll
    for (int r = 0; r < QMAX; ++r)
      if (r < q) coef_out[off[s] + r] = beta[r];
  }
}

// k_reopt_gram (squared loss): X_S'(X_S beta - y) = Gram beta - X_S'y, the
// same iterates in exact arithmetic.  The q x q Gram and
// X_S'y are built once per support; warp 0 then runs the projected-gradient
// loop with lane r owning beta_r.  q <= 32.
__global__ void __launch_bounds__(kReoptFastThreads)
    k_reopt_gram(int n, const double* __restrict__ X, const double* __restrict__ y, double M,
                 double lambda2, double step, const int* off, const int* sidx, double* coef_out,
                 double* obj_out) {
  constexpr int NW = kReoptFastThreads / 32;
  __shared__ double gram[32][33];
  __shared__ double xty[32];
  __shared__ double bsh[32];
  __shared__ double wred[NW];
  __shared__ const double* cols[32];
  const int s = blockIdx.x;
  const int q = off[s + 1] - off[s];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < q) cols[tid] = X + (size_t)sidx[off[s] + tid] * n;
  if (tid < 32) bsh[tid] = 0.0;
  __syncthreads();
  // Gram entries (r <= c) and X_S'y: one warp per dot product
  const int npairs = q * (q + 1) / 2 + q;
  for (int t = warp; t < npairs; t += NW) {
    int r = 0, c = 0;
    const double* a;
    const double* bvec;
    if (t < q * (q + 1) / 2) {
      int tt = t;
      while (tt >= q - r) {
        tt -= q - r;
        ++r;
      }
      c = r + tt;
      a = cols[r];
      bvec = cols[c];
    } else {
      r = t - q * (q + 1) / 2;
      a = cols[r];
      bvec = y;
    }
    double acc = 0.0;
    for (int i = lane; i < n; i += 32) acc += a[i] * bvec[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      if (t < q * (q + 1) / 2) {
        gram[r][c] = acc;
        gram[c][r] = acc;
      } else {
        xty[r] = acc;
      }
    }
  }
  __syncthreads();
  if (warp == 0 && q > 0) {
    double b = 0.0;
    const bool own = lane < q;
    for (int it = 0; it < 5000; ++it) {
      double g = 0.0;
      for (int c = 0; c < q; ++c) {
        const double bc = __shfl_sync(0xffffffffu, b, c);
        if (own) g += gram[lane][c] * bc;
      }
      double dl2 = 0.0, nx = 0.0;
      if (own) {
        g = g - xty[lane] + 2.0 * lambda2 * b;
        double v = b - step * g;
        v = v < -M ? -M : v;
        v = v > M ? M : v;
        nx = v;
        const double dl = b - v;
        dl2 = dl * dl;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) dl2 += __shfl_xor_sync(0xffffffffu, dl2, o);
      b = nx;
      if (sqrt(dl2) / step <= 1e-8) break;
    }
    if (own) bsh[lane] = b;
  }
  __syncthreads();
  double acc = 0.0;
  for (int i = tid; i < n; i += kReoptFastThreads) {
    double sc = 0.0;
    for (int r = 0; r < q; ++r) sc += bsh[r] * cols[r][i];
    acc += d_loss_value(kSquared, sc, y[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) wred[warp] = acc;
  __syncthreads();
  if (tid == 0) {
    double sq = 0.0;
    for (int r = 0; r < q; ++r) sq += bsh[r] * bsh[r];
    double obj = lambda2 * sq;
    for (int w = 0; w < NW; ++w) obj += wred[w];
    obj_out[s] = obj;
  }
  if (tid < q) coef_out[off[s] + tid] = bsh[tid];
}

// --------------------------------------------------------------------------
// stateless test kernels (prox_kernel.hpp:177-229, :284-301, :310-370)
// --------------------------------------------------------------------------
// mode 0: prox_step (out = U - rho^-1 prox_{rho g*}(rho U)); mode 1: conjugate prox
__global__ void __launch_bounds__(kNodeThreads)
    k_prox_standalone(int mode, int p, int n2, const double* U, const uint8_t* state, const int* kbar,
                      double w, double M, double* out) {
  extern __shared__ __align__(16) double sm[];
  const int b = blockIdx.x;
  double* key = sm;
  int* idx = reinterpret_cast<int*>(key + n2);
  double* scan = reinterpret_cast<double*>(idx + n2);
  __shared__ double red[kNodeThreads / 32];
  const double* u = U + (size_t)b * p;
  const uint8_t* st = state + (size_t)b * p;
  double* o = out + (size_t)b * p;
  const double scale = mode == 0 ? w : 1.0;  // mode 0: w = rho
  int cnt = 0;
  for (int j = threadIdx.x; j < n2; j += kNodeThreads) {
    if (j < p) {
      const bool fr = st[j] == kFree;
      key[j] = fr ? scale * fabs(u[j]) : -1.0;
      cnt += fr;
    } else {
      key[j] = -2.0;
    }
    idx[j] = j;
  }
  const int pf = (int)block_sum<kNodeThreads>((double)cnt, red);
  bitonic_sort_desc<kNodeThreads>(key, idx, n2);
  const int kb = kbar[b];
  int lo, hi;
  double pooled;
  block_pava<kNodeThreads>(key, pf, kb, w, M, scan, red, lo, hi, pooled);
  for (int rk = threadIdx.x; rk < pf; rk += kNodeThreads) {
    const int j = idx[rk];
    const bool in_block = hi >= lo && rk >= lo && rk <= hi;
    const double v = in_block ? pooled : (rk < kb ? d_prox_huber(key[rk], w, M) : key[rk]);
    const double sign = u[j] > 0.0 ? 1.0 : (u[j] < 0.0 ? -1.0 : 0.0);
    if (mode == 0) {
      o[j] = (rk >= kb && !in_block) ? 0.0 : u[j] - (1.0 / w) * sign * v;
    } else {
      o[j] = sign * v;
    }
  }
  for (int j = threadIdx.x; j < p; j += kNodeThreads) {
    const uint8_t s = st[j];
    if (s == kFree) continue;
    if (mode == 0)
      o[j] = s == kFixedZero ? 0.0 : u[j] - (1.0 / w) * d_prox_huber(w * u[j], w, M);
    else
      o[j] = s == kFixedZero ? u[j] : d_prox_huber(u[j], w, M);
  }
}

__global__ void __launch_bounds__(kNodeThreads)
    k_g_standalone(int mode, int p, int n2, const double* in, const uint8_t* state, const int* kbar,
                   double M, double* out) {
  extern __shared__ __align__(16) double sm[];
  const int b = blockIdx.x;
  double* key = sm;
  int* idx = reinterpret_cast<int*>(key + n2);
  __shared__ double red[kNodeThreads / 32];
  __shared__ int ired[kNodeThreads / 32];
  const double v = mode == 0 ? block_g_value<kNodeThreads>(in + (size_t)b * p, state + (size_t)b * p,
                                                           p, n2, kbar[b], M, key, idx, red, ired)
                             : block_g_conj<kNodeThreads>(in + (size_t)b * p, 1.0,
                                                          state + (size_t)b * p, p, n2, kbar[b], M,
                                                          key, idx, red);
  if (threadIdx.x == 0) out[b] = v;
}

// --------------------------------------------------------------------------
// smoothness constant (losses.hpp:86-112): power-iteration GEMVs
// --------------------------------------------------------------------------
__global__ void k_gemv_n(int n, int p, const double* __restrict__ X, const double* __restrict__ v,
                         double* __restrict__ xv) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int j = 0; j < p; ++j) s += X[(size_t)j * n + i] * v[j];
  xv[i] = s;
}

__global__ void k_gemv_t(int n, int p, const double* __restrict__ X, const double* __restrict__ xv,
                         double* __restrict__ w) {
  const int j = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= p) return;
  const double* col = X + (size_t)j * n;
  double s = 0.0;
  for (int i = lane; i < n; i += 32) s += col[i] * xv[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) w[j] = s;
}

// out[0] = v.w, out[1] = |w|; single CTA of 256 threads
__global__ void k_power_stats(int p, const double* v, const double* w, double* out) {
  __shared__ double red[8];
  double a = 0.0, c = 0.0;
  for (int j = threadIdx.x; j < p; j += 256) {
    a += v[j] * w[j];
    c += w[j] * w[j];
  }
  const double dot = block_sum<256>(a, red);
  const double nrm2 = block_sum<256>(c, red);
  if (threadIdx.x == 0) {
    out[0] = dot;
    out[1] = sqrt(nrm2);
  }
}

__global__ void k_scale(int p, const double* w, double wn, double* v) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < p) v[j] = w[j] / wn;
}

}  // namespace bnbg
