// pool_kernels.cuh -- the device-resident node pool (SURVEY 8(f) row 1, VK1 + VK12).
//
// Open nodes live in HBM, one slot each: coordinate states (p bytes), warm
// start (p doubles), the ordered J0 list (p ints) and J1 list (k ints), and
// the list lengths and depth.  The host queue holds only (lower bound,
// insertion sequence, slot); a pass ships slot ids to the device and gets
// back per-child records, never a warm start.
//
//   k_pool_root       root_node (node_model.hpp:47-52)
//   k_pack_pool       BatchMeta::from_nodes from pool slots (prox_kernel.hpp:52-90):
//                     dense state column, kbar, free count, warm start -> B, V,
//                     padded J1 lists for round_support
//   k_pool_lists      J0 / J1 lists of a batch (DebugHooks only)
//   k_branch_scan     survivors of the prune test (bnb_engine.hpp:243-247):
//                     lb = max(lb, bound), keep iff not prunable and
//                     lb < post-threshold; exclusive prefix sum -> child positions
//   k_branch_write    branch + restore_budget (node_model.hpp:57-105) for every
//                     survivor, children written straight into free pool slots,
//                     compact child records for the host
#pragma once
#include "device_math.cuh"

namespace bnbg {

struct PoolDev {
  int p, k, cap;
  uint8_t* state;  // cap x p
  double* warm;    // cap x p
  int* j0;         // cap x p   (construction order)
  int* j1;         // cap x k   (construction order)
  int* n0;         // cap
  int* n1;         // cap
  int* depth;      // cap
};

// child record for the host: slot, leaf flag, |J1|, J1 list (k ints)
__host__ __device__ inline int child_rec_ints(int k) { return 4 + k; }

constexpr int kPoolThreads = 256;

static __global__ void k_pool_root(PoolDev P, int slot) {
  for (int j = threadIdx.x; j < P.p; j += blockDim.x) {
    P.state[(size_t)slot * P.p + j] = kFree;
    P.warm[(size_t)slot * P.p + j] = 0.0;
  }
  if (threadIdx.x == 0) {
    P.n0[slot] = 0;
    P.n1[slot] = 0;
    P.depth[slot] = 0;
  }
}

static __global__ void __launch_bounds__(kPoolThreads)
    k_pack_pool(PoolDev P, int m, const int* slots, uint8_t* state, int* kbar, int* pf, double* B,
                double* V, double* t, double* best, double* last_gap, uint8_t* frozen,
                int* status, int* iters, int* act, int max_it, int* one_len, int* one_idx) {
  const int b = blockIdx.x;
  if (b >= m) return;
  const int s = slots[b], p = P.p;
  const uint8_t* sst = P.state + (size_t)s * p;
  const double* sw = P.warm + (size_t)s * p;
  uint8_t* col = state + (size_t)b * p;
  for (int j = threadIdx.x; j < p; j += kPoolThreads) {
    col[j] = sst[j];
    const double w = sw[j];
    B[(size_t)b * p + j] = w;
    V[(size_t)b * p + j] = w;
  }
  const int n1 = P.n1[s];
  for (int q = threadIdx.x; q < n1; q += kPoolThreads)
    one_idx[(size_t)b * P.k + q] = P.j1[(size_t)s * P.k + q];
  if (threadIdx.x == 0) {
    const int kb = P.k - n1;
    kbar[b] = kb > 0 ? kb : 0;
    pf[b] = p - P.n0[s] - n1;
    one_len[b] = n1;
    t[b] = 1.0;
    best[b] = -d_inf();
    last_gap[b] = d_inf();
    frozen[b] = 0;
    status[b] = kCapped;
    iters[b] = max_it;
    act[b] = b;
  }
}

// n0/n1 then J0 (m x p) and J1 (m x k) of the batch slots
static __global__ void k_pool_lists(PoolDev P, int m, const int* slots, int* n01, int* j0, int* j1) {
  const int b = blockIdx.x;
  if (b >= m) return;
  const int s = slots[b];
  const int a0 = P.n0[s], a1 = P.n1[s];
  for (int q = threadIdx.x; q < a0; q += blockDim.x) j0[(size_t)b * P.p + q] = P.j0[(size_t)s * P.p + q];
  for (int q = threadIdx.x; q < a1; q += blockDim.x) j1[(size_t)b * P.k + q] = P.j1[(size_t)s * P.k + q];
  if (threadIdx.x == 0) {
    n01[2 * b] = a0;
    n01[2 * b + 1] = a1;
  }
}

// One CTA: flags, updated lower bounds and the exclusive scan of survivors.
// out_total[0] = survivors, out_total[1] = first column with no free
// coordinate among survivors (logic_error) or -1.
static __global__ void __launch_bounds__(1024)
    k_branch_scan(int m, const int* status, const double* bound, const double* lb_in,
                  double post_thr, const int* jb, double* lb_out, int* pos, int* out_total) {
  __shared__ int warp_tot[32];
  __shared__ int s_base, s_bad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    s_base = 0;
    s_bad = 0x7fffffff;
  }
  __syncthreads();
  for (int base = 0; base < m; base += 1024) {
    const int b = base + tid;
    int keep = 0;
    if (b < m) {
      const double lb = fmax(lb_in[b], bound[b]);  // nd.lb = max(nd.lb, bound_b)
      lb_out[b] = lb;
      keep = status[b] != kPrunable && lb < post_thr;
      if (keep && jb[b] < 0) {
        atomicMin(&s_bad, b);
        keep = 0;
      }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    const int pre = __popc(bal & ((1u << lane) - 1));
    if (lane == 0) warp_tot[warp] = __popc(bal);
    __syncthreads();
    int off = 0;
    for (int w = 0; w < warp; ++w) off += warp_tot[w];
    const int bo = s_base;
    if (b < m) pos[b] = keep ? bo + off + pre : -1;
    __syncthreads();
    if (tid == 1023) {
      int tot = 0;
      for (int w = 0; w < 32; ++w) tot += warp_tot[w];
      s_base = bo + tot;
    }
    __syncthreads();
  }
  if (tid == 0) {
    out_total[0] = s_base;
    out_total[1] = s_bad == 0x7fffffff ? -1 : s_bad;
  }
}

// restore_budget (node_model.hpp:57-68) of one child column held in w[]/cs[]
// (free entries scaled in place when their l1 mass exceeds kbar * M)
template <int NT>
__device__ __forceinline__ void restore_budget_col(double* w, const uint8_t* cs, int p, int kb,
                                                   double M, double* red) {
  double sum = 0.0;
  for (int j = threadIdx.x; j < p; j += NT)
    if (cs[j] == kFree) sum += fabs(w[j]);
  sum = block_sum<NT>(sum, red);
  const double budget = (double)kb * M;
  if (sum <= budget) return;
  const double scale = budget / sum * (1.0 - 1e-12);
  for (int j = threadIdx.x; j < p; j += NT)
    if (cs[j] == kFree) w[j] *= scale;
  __syncthreads();
}

// branch(nd, j, beta) for every survivor (node_model.hpp:77-105).  Batch
// column b holds the parent's states and final beta; the parent's lists come
// from its pool slot (never one of the child slots: the host frees the batch
// slots only after this kernel).
static __global__ void __launch_bounds__(kPoolThreads)
    k_branch_write(PoolDev P, int m, double M, const int* slots, const uint8_t* state,
                   const double* beta, const int* jb, const int* pos, const double* lb,
                   const int* free_slots, int* rec, double* rec_lb) {
  const int b = blockIdx.x;
  if (b >= m) return;
  const int ps = pos[b];
  if (ps < 0) return;
  __shared__ double red[kPoolThreads / 32];
  __shared__ int warp_tot[kPoolThreads / 32];
  __shared__ int s_base;
  const int p = P.p, k = P.k, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int par = slots[b], j = jb[b];
  const int pn0 = P.n0[par], pn1 = P.n1[par];
  const int c0 = free_slots[2 * ps], c1 = free_slots[2 * ps + 1];
  const uint8_t* pst = state + (size_t)b * p;
  const double* bb = beta + (size_t)b * p;
  uint8_t* s0 = P.state + (size_t)c0 * p;
  uint8_t* s1 = P.state + (size_t)c1 * p;
  double* w0 = P.warm + (size_t)c0 * p;
  double* w1 = P.warm + (size_t)c1 * p;
  const int kb1 = k - (pn1 + 1);
  const bool sweep = kb1 <= 0;  // child1 exhausts the budget: every other free -> J0
  for (int r = tid; r < p; r += kPoolThreads) {
    const uint8_t st = pst[r];
    const double v = bb[r];
    s0[r] = r == j ? (uint8_t)kFixedZero : st;
    w0[r] = r == j ? 0.0 : v;
    const bool swept = sweep && st == kFree && r != j;
    s1[r] = r == j ? (uint8_t)kFixedOne : (swept ? (uint8_t)kFixedZero : st);
    w1[r] = swept ? 0.0 : v;
  }
  // lists: child0 J0 = parent J0 + [j]; child1 J1 = parent J1 + [j]
  int* j00 = P.j0 + (size_t)c0 * p;
  int* j01 = P.j0 + (size_t)c1 * p;
  const int* pj0 = P.j0 + (size_t)par * p;
  for (int q = tid; q < pn0; q += kPoolThreads) {
    const int v = pj0[q];
    j00[q] = v;
    j01[q] = v;
  }
  for (int q = tid; q < pn1; q += kPoolThreads) {
    const int v = P.j1[(size_t)par * k + q];
    P.j1[(size_t)c0 * k + q] = v;
    P.j1[(size_t)c1 * k + q] = v;
  }
  if (tid == 0) {
    j00[pn0] = j;
    P.j1[(size_t)c1 * k + pn1] = j;
    s_base = pn0;
  }
  __syncthreads();
  // child1's budget sweep appends the remaining free indices in index order
  int n0c1 = pn0;
  if (sweep) {
    for (int base = 0; base < p; base += kPoolThreads) {
      const int r = base + tid;
      const bool f = r < p && pst[r] == kFree && r != j;
      const unsigned bal = __ballot_sync(0xffffffffu, f);
      const int pre = __popc(bal & ((1u << lane) - 1));
      if (lane == 0) warp_tot[warp] = __popc(bal);
      __syncthreads();
      int off = 0;
      for (int w = 0; w < warp; ++w) off += warp_tot[w];
      const int bo = s_base;
      if (f) j01[bo + off + pre] = r;
      __syncthreads();
      if (tid == 0) {
        int tot = 0;
        for (int w = 0; w < kPoolThreads / 32; ++w) tot += warp_tot[w];
        s_base = bo + tot;
      }
      __syncthreads();
    }
    n0c1 = s_base;
  }
  __syncthreads();
  restore_budget_col<kPoolThreads>(w0, s0, p, k - pn1, M, red);
  restore_budget_col<kPoolThreads>(w1, s1, p, kb1, M, red);
  if (tid == 0) {
    const int dep = P.depth[par] + 1;
    P.n0[c0] = pn0 + 1;
    P.n1[c0] = pn1;
    P.depth[c0] = dep;
    P.n0[c1] = n0c1;
    P.n1[c1] = pn1 + 1;
    P.depth[c1] = dep;
    const int RI = child_rec_ints(k);
    int* r0 = rec + (size_t)(2 * ps) * RI;
    int* r1 = r0 + RI;
    // is_leaf (node_model.hpp:33-36): kbar <= 0 or no free coordinate
    r0[0] = c0;
    r0[1] = (k - pn1 <= 0) || (pn0 + 1 + pn1 >= p);
    r0[2] = pn1;
    r0[3] = dep;
    r1[0] = c1;
    r1[1] = (kb1 <= 0) || (n0c1 + pn1 + 1 >= p);
    r1[2] = pn1 + 1;
    r1[3] = dep;
    rec_lb[2 * ps] = lb[b];
    rec_lb[2 * ps + 1] = lb[b];
  }
  const int RI = child_rec_ints(k);
  int* r0 = rec + (size_t)(2 * ps) * RI;
  // J1 lists; the unused tail of each k-slot list is -1 (every byte of the
  // record read back to the host is defined)
  for (int q = tid; q < k; q += kPoolThreads) {
    const int v = q < pn1 ? P.j1[(size_t)par * k + q] : (q == pn1 ? j : -1);
    r0[4 + q] = q < pn1 ? v : -1;
    r0[RI + 4 + q] = v;
  }
}

// ---------------------------------------------------------------------------
// node exchange between ranks (multi-GPU load balancing):
// a node travels as one fixed-size record
//   [lb f64][n0 i32 n1 i32 depth i32 pad][state p B, padded to 8][warm p f64]
//   [J0 p i32][J1 k i32, padded to 8]
// ---------------------------------------------------------------------------
__host__ __device__ inline size_t node_rec_bytes(int p, int k) {
  const size_t pad8 = ((size_t)p + 7) & ~(size_t)7;
  const size_t j1 = ((size_t)4 * k + 7) & ~(size_t)7;
  return 24 + pad8 + 8 * (size_t)p + 4 * (size_t)p + j1;
}

static __global__ void k_pool_pack(PoolDev P, int cnt, const int* slots, const double* lbs,
                                   uint8_t* out) {
  const int i = blockIdx.x;
  if (i >= cnt) return;
  const int s = slots[i], p = P.p, k = P.k;
  uint8_t* r = out + (size_t)i * node_rec_bytes(p, k);
  const size_t pad8 = ((size_t)p + 7) & ~(size_t)7;
  uint8_t* st = r + 24;
  double* w = reinterpret_cast<double*>(st + pad8);
  int* j0 = reinterpret_cast<int*>(w + p);
  int* j1 = j0 + p;
  const int n0 = P.n0[s], n1 = P.n1[s];
  for (int j = threadIdx.x; j < p; j += blockDim.x) {
    st[j] = P.state[(size_t)s * p + j];
    w[j] = P.warm[(size_t)s * p + j];
  }
  for (int q = threadIdx.x; q < n0; q += blockDim.x) j0[q] = P.j0[(size_t)s * p + q];
  for (int q = threadIdx.x; q < n1; q += blockDim.x) j1[q] = P.j1[(size_t)s * k + q];
  if (threadIdx.x == 0) {
    *reinterpret_cast<double*>(r) = lbs[i];
    int* hd = reinterpret_cast<int*>(r + 8);
    hd[0] = n0;
    hd[1] = n1;
    hd[2] = P.depth[s];
  }
}

static __global__ void k_pool_unpack(PoolDev P, int cnt, const uint8_t* in, const int* slots,
                                     double* lbs) {
  const int i = blockIdx.x;
  if (i >= cnt) return;
  const int s = slots[i], p = P.p, k = P.k;
  const uint8_t* r = in + (size_t)i * node_rec_bytes(p, k);
  const size_t pad8 = ((size_t)p + 7) & ~(size_t)7;
  const uint8_t* st = r + 24;
  const double* w = reinterpret_cast<const double*>(st + pad8);
  const int* j0 = reinterpret_cast<const int*>(w + p);
  const int* j1 = j0 + p;
  const int* hd = reinterpret_cast<const int*>(r + 8);
  const int n0 = hd[0], n1 = hd[1];
  for (int j = threadIdx.x; j < p; j += blockDim.x) {
    P.state[(size_t)s * p + j] = st[j];
    P.warm[(size_t)s * p + j] = w[j];
  }
  for (int q = threadIdx.x; q < n0; q += blockDim.x) P.j0[(size_t)s * p + q] = j0[q];
  for (int q = threadIdx.x; q < n1; q += blockDim.x) P.j1[(size_t)s * k + q] = j1[q];
  if (threadIdx.x == 0) {
    P.n0[s] = n0;
    P.n1[s] = n1;
    P.depth[s] = hd[2];
    lbs[i] = *reinterpret_cast<const double*>(r);
  }
}

}  // namespace bnbg
