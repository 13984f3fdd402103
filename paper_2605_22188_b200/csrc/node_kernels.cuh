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
//   k_prox_standalone / k_g_standalone   test entry points (prox_kernel.hpp)
//
// One CTA (256 threads) per column.  Each column's keys are sorted in the
// reference order (key descending, index ascending: prox_kernel.hpp:119-122,
// primal_heuristics.hpp:41-45) by a register-resident bitonic network: thread
// t holds E consecutive elements, strides below E are register swaps, strides
// below 32E are warp shuffles, and only the cross-warp strides go through
// shared memory (6 barriers for 512 keys instead of 45).  E = 0 selects the
// shared-memory network for p > 1024.  Every reduction has a fixed
// association order (deterministic results).
#pragma once
#include "device_math.cuh"

#ifndef BNBG_PAVA_WA  // PAVA walk window: left x right moves per step
#define BNBG_PAVA_WA 8
#endif
#ifndef BNBG_PAVA_WB
#define BNBG_PAVA_WB 4
#endif
#ifndef BNBG_PAVA_RQ  // right-run states per lane and step
#define BNBG_PAVA_RQ 2
#endif
// Optional timing probe for the PAVA phases (tools/micro); empty in the product.
#ifndef BNBG_PAVA_PROBE
#define BNBG_PAVA_PROBE(i)
#endif

namespace bnbg {

constexpr int kNodeThreads = 256;
constexpr int kMaxSplit = 8;

struct RelaxDev {
  int p, n2, mcap;
  double* B;
  double* V;
  const double* G;  // split-K slabs: G + s*split_stride + col*p
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
  unsigned long long* probe;  // optional sub-phase timers of CTA 0's column work (nullptr: off)
  // large p (column buffers above the shared-memory limit): the column
  // kernels' key/index/scan buffers live in global memory instead, colstride
  // doubles per CTA (nullptr: dynamic shared memory)
  double* colscr;
  long long colstride;
};

// the column buffers of CTA blockIdx.x: global scratch (large p) or shared memory
__device__ __forceinline__ double* col_base(double* gscr, long long gstride, double* sm) {
  return gscr ? gscr + (size_t)blockIdx.x * gstride : sm;
}

// CTA 0's sub-phase timer (tools/pass_phases.py); compiled in, off unless r.probe is set
struct ColProbe {
  unsigned long long* p;
  unsigned long long t;
  __device__ __forceinline__ explicit ColProbe(unsigned long long* q)
      : p(q && blockIdx.x == 0 && threadIdx.x == 0 ? q : nullptr), t(0) {
    if (p) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  }
  __device__ __forceinline__ void mark(int i) {
    if (!p) return;
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    atomicAdd(p + i, now - t);  // RED: no load on the timed thread's path
    t = now;
  }
};

// G = sum of the split-K slabs, added in slab order (loads issued together)
__device__ __forceinline__ double gsum(const RelaxDev& r, int ns, int b, int j) {
  double part[kMaxSplit];
#pragma unroll
  for (int s = 0; s < kMaxSplit; ++s)
    part[s] = s < ns ? r.G[(size_t)s * r.split_stride + (size_t)b * r.p + j] : 0.0;
  double g = part[0];
#pragma unroll
  for (int s = 1; s < kMaxSplit; ++s)
    if (s < ns) g += part[s];
  return g;
}

// ---------------------------------------------------------------------------
// column sort
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool kv_before(double ka, int ia, double kb, int ib) {
  return ka > kb || (ka == kb && ia < ib);
}

// number of sorted slots of the key/idx arrays
__host__ __device__ inline int sort_slots(int n2, int E) { return E ? kNodeThreads * E : n2; }

// dynamic shared memory: key[NS] idx[NS] u[p] scan[NS] (+ exchange buffers
// 2x(NS doubles + NS ints)) bo[p] (staged previous iterate) st[p] (staged states)
__host__ __device__ inline size_t column_smem_bytes(int p, int n2, int E) {
  const size_t ns = (size_t)sort_slots(n2, E);
  size_t b = ns * 8 + ns * 4 + (size_t)p * 8 + ns * 8;
  if (E) b += 2 * ns * 12 + (size_t)p * 8 + (size_t)p + 16;  // staging only for register sorts
  return b + 64;
}

// Register bitonic network over N = NT*E elements (thread t: elements t*E+r).
template <int NT, int E>
__device__ __forceinline__ void reg_bitonic(double (&k)[E], int (&ix)[E], double* xk, int* xi) {
  constexpr int N = NT * E;
  const int t = threadIdx.x, lane = t & 31;
  int buf = 0;
#pragma unroll
  for (int size = 2; size <= N; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride < E) {
#pragma unroll
        for (int r = 0; r < E; ++r) {
          const int pr = r ^ stride;
          if (pr > r) {
            const bool up = ((t * E + r) & size) == 0;
            if (kv_before(k[pr], ix[pr], k[r], ix[r]) == up) {
              const double tk = k[r];
              k[r] = k[pr];
              k[pr] = tk;
              const int ti = ix[r];
              ix[r] = ix[pr];
              ix[pr] = ti;
            }
          }
        }
      } else if (stride < 32 * E) {
        const int ld = stride / E;
        const bool lower = (lane & ld) == 0;
#pragma unroll
        for (int r = 0; r < E; ++r) {
          const double ok = __shfl_xor_sync(0xffffffffu, k[r], ld);
          const int oi = __shfl_xor_sync(0xffffffffu, ix[r], ld);
          const bool up = ((t * E + r) & size) == 0;
          const bool keep_first = lower == up;
          if (keep_first != kv_before(k[r], ix[r], ok, oi)) {
            k[r] = ok;
            ix[r] = oi;
          }
        }
      } else {
        double* bk = xk + buf * N;
        int* bi = xi + buf * N;
#pragma unroll
        for (int r = 0; r < E; ++r) {
          bk[t * E + r] = k[r];
          bi[t * E + r] = ix[r];
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < E; ++r) {
          const int e = t * E + r;
          const double ok = bk[e ^ stride];
          const int oi = bi[e ^ stride];
          const bool up = (e & size) == 0;
          const bool keep_first = ((e & stride) == 0) == up;
          if (keep_first != kv_before(k[r], ix[r], ok, oi)) {
            k[r] = ok;
            ix[r] = oi;
          }
        }
        buf ^= 1;
      }
    }
  }
}

// Shared-memory bitonic network over n2 elements already in key/idx.
template <int NT>
__device__ __forceinline__ void smem_bitonic(double* key, int* idx, int n2) {
  for (int size = 2; size <= n2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int t = threadIdx.x; t < (n2 >> 1); t += NT) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const double ka = key[lo], kb = key[hi];
        const int ia = idx[lo], ib = idx[hi];
        const bool hi_first = kv_before(kb, ib, ka, ia);
        const bool up = (lo & size) == 0;
        if (hi_first == up) {
          key[lo] = kb;
          key[hi] = ka;
          idx[lo] = ib;
          idx[hi] = ia;
        }
      }
    }
  }
  __syncthreads();
}

// Sorts kf(j) for j < p (pads beyond p get -2) into key[]/idx[] in the
// reference order.  kf may have side effects (called once per j < p).
template <int NT, int E, class KF>
__device__ __forceinline__ void column_sort(int p, int n2, KF kf, double* key, int* idx, double* xk,
                                            int* xi) {
  if constexpr (E == 0) {
    for (int j = threadIdx.x; j < n2; j += NT) {
      key[j] = j < p ? kf(j) : -2.0;
      idx[j] = j;
    }
    smem_bitonic<NT>(key, idx, n2);
  } else {
    double k[E];
    int ix[E];
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const int j = threadIdx.x * E + r;
      k[r] = j < p ? kf(j) : -2.0;
      ix[r] = j;
    }
    reg_bitonic<NT, E>(k, ix, xk, xi);
#pragma unroll
    for (int r = 0; r < E; ++r) {
      key[threadIdx.x * E + r] = k[r];
      idx[threadIdx.x * E + r] = ix[r];
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Boundary-seeded PAVA on the sorted keys (prox_kernel.hpp:132-170).
// v_r = prox_huber(key_r, w, M) for r < kbar and key_r otherwise; the only
// violation is at the kbar boundary and the pooled block [lo,hi] grows from
// [kbar-1, kbar] with the reference's rule (left test first, then right).
//
// The reference re-sums the block after every expansion (O(len^2), one
// thread).  Here block sums come from two scans anchored at the boundary (SL:
// suffix sums of ranks < kbar, SR: prefix sums of ranks >= kbar -- sums of
// block members only, no cancellation), built in one pass with two barriers,
// and the expansion evaluates NT consecutive states per step, following the
// reference's decision sequence: the first state whose left test fires (or
// whose right test fails) is located with ballots.  All threads call; lo/hi/
// pooled are returned to every thread.
// ---------------------------------------------------------------------------
template <int NT>
__device__ void block_pava(const double* key, int pf, int kbar, double w, double M, double* scan,
                           int& blo, int& bhi, double& bval, unsigned long long* probe = nullptr) {
  blo = 0;
  bhi = -1;
  bval = 0.0;
  if (kbar <= 0 || kbar >= pf) return;
  if (d_prox_huber(key[kbar - 1], w, M) >= key[kbar]) return;
  BNBG_PAVA_PROBE(0);
  // sub-phase timers of CTA 0 (scan, walk) and walk statistics (steps, calls)
  ColProbe pp(probe);
  constexpr int NW = NT / 32;
  __shared__ double s_ftot[NW], s_btot[NW];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* SL = scan;         // SL[i] = key[kbar-1] + ... + key[kbar-1-i]
  double* SR = scan + kbar;  // SR[e] = key[kbar] + ... + key[kbar+e]
  {
    const int chunk = (pf + NT - 1) / NT;
    const int beg = min(pf, tid * chunk), end = min(pf, beg + chunk);
    double f = 0.0, bsum = 0.0;
#pragma unroll 2
    for (int r = beg; r < end; ++r)
      if (r >= kbar) f += key[r];
#pragma unroll 2
    for (int r = end - 1; r >= beg; --r)
      if (r < kbar) bsum += key[r];
    double fi = f, bi = bsum;  // inclusive warp scans: forward (up), backward (down)
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double tf = __shfl_up_sync(0xffffffffu, fi, o);
      const double tb = __shfl_down_sync(0xffffffffu, bi, o);
      if (lane >= o) fi += tf;
      if (lane + o < 32) bi += tb;
    }
    if (lane == 31) s_ftot[warp] = fi;
    if (lane == 0) s_btot[warp] = bi;
    __syncthreads();
    double foff = fi - f, boff = bi - bsum;
    // warp offsets in the same order as a loop to `warp`, with the loads
    // issued together (adding nothing for the other warps)
#pragma unroll
    for (int w2 = 0; w2 < NW; ++w2) {
      const double v = s_ftot[w2];
      if (w2 < warp) foff += v;
    }
#pragma unroll
    for (int w2 = NW - 1; w2 >= 0; --w2) {
      const double v = s_btot[w2];
      if (w2 > warp) boff += v;
    }
    double run = foff;
#pragma unroll 2
    for (int r = beg; r < end; ++r)
      if (r >= kbar) {
        run += key[r];
        SR[r - kbar] = run;
      }
    run = boff;
#pragma unroll 2
    for (int r = end - 1; r >= beg; --r)
      if (r < kbar) {
        run += key[r];
        SL[kbar - 1 - r] = run;
      }
    __syncthreads();
  BNBG_PAVA_PROBE(1);
  }
  pp.mark(0);
  // Values are kept as fractions num/den (den > 0) so the expansion tests
  // need no division: pooled(lo,hi) = prox_huber(S/len, w(kbar-lo)/len, M)
  // = S/(len + W) inside the box (|S| <= (len + W) M, W = w (kbar-lo)) and
  // (S - W M)/len outside (S >= 0: keys are magnitudes); head values
  // v_r = prox_huber(key_r, w, M) likewise.  Only the final pooled value is
  // divided out (prox_kernel.hpp:145-151 evaluates the same quantity).
  // Left and right tests of state (cl, ch), branch-free so that several
  // states per lane overlap their loads (indices clamped; states outside
  // [0, pf) test false and are never reached).  v(cl-1) is always a head
  // value (cl <= kbar - 1) and v(ch+1) a raw key (ch >= kbar).
  const double hb = (1.0 + w) * M, wM = w * M;
  auto test = [&](int cl, int ch, bool& L, bool& R) {
    const bool ok = cl >= 0 && ch <= pf - 1;
    const int c0 = max(cl, 0), c1 = min(ch, pf - 1);
    const double len = (double)(c1 - c0 + 1);
    const double S = SL[kbar - 1 - c0] + SR[c1 - kbar];
    const double W = w * (double)(kbar - c0);
    const bool box = S <= (len + W) * M;
    const double pn = box ? S : S - W * M, pd = box ? len + W : len;
    const double a = key[max(c0 - 1, 0)];
    const bool hbox = a <= hb;
    const double vn = hbox ? a : a - wM, vd = hbox ? 1.0 + w : 1.0;
    const double b = key[min(c1 + 1, pf - 1)];
    L = ok && c0 > 0 && vn * pd < pn * vd;
    R = ok && c1 < pf - 1 && pn * 1.0 < b * pd;
  };
  auto pooled = [&](int lo, int hi) {
    const int len = hi - lo + 1;
    const double sum = SL[kbar - 1 - lo] + SR[hi - kbar];
    const double mean_w = w * (double)(kbar - lo) / len;
    return d_prox_huber(sum / len, mean_w, M);
  };
  // The expansion is replayed by warp 0 alone (no block barrier inside the
  // walk).  From state (lo, hi) the reference moves left while the left test
  // fires, else right while the right test fires, else stops; each step
  // evaluates a window of states in one pass:
  //  - 2-D window: lane (a, b) < (WA, WB) tests state (lo - a, hi + b); the
  //    path through the window is traced from the ballots of both tests;
  //  - after a window left by a straight run, a 1-D run along it (left:
  //    (lo - t, hi), 32 states; right: (lo, hi + t), 32 * RQ states), ending
  //    at the first state whose decision differs.
  // Both follow the reference's decision order exactly (left test first).
  // Left moves number at most kbar - 1, so long walks are right runs.
  constexpr int WA = BNBG_PAVA_WA, WB = BNBG_PAVA_WB, RQ = BNBG_PAVA_RQ;
  static_assert(WA * WB <= 32, "PAVA window");
  __shared__ int s_lohi[2];
  int lo = kbar - 1, hi = kbar;
  if (warp == 0) {
    int mode = 0;  // 0: 2-D window, 1: left run, 2: right run
    unsigned steps = 0;
    const int la = lane / WB, lb = lane - (lane / WB) * WB;
    for (;;) {
      ++steps;
      if (mode == 0) {
        bool L, R;
        test(lo - la, hi + lb, L, R);
        L = L && lane < WA * WB;
        R = R && lane < WA * WB;
        const unsigned bl = __ballot_sync(0xffffffffu, L);
        const unsigned br = __ballot_sync(0xffffffffu, R);
        int a = 0, b = 0, idx = 0;
        bool done = false;
        for (;;) {
          if ((bl >> idx) & 1u) {
            if (++a == WA) break;
            idx += WB;
          } else if ((br >> idx) & 1u) {
            if (++b == WB) break;
            ++idx;
          } else {
            done = true;
            break;
          }
        }
        lo -= a;
        hi += b;
        if (done) break;
        mode = b == 0 ? 1 : (a == 0 ? 2 : 0);
        continue;
      }
      if (mode == 1) {  // state t = (lo - t, hi): runs while L
        bool L, R;
        test(lo - lane, hi, L, R);
        const unsigned bev = __ballot_sync(0xffffffffu, !L);
        const unsigned br = __ballot_sync(0xffffffffu, R);
        if (!bev) {
          lo -= 32;
          continue;
        }
        const int first = __ffs(bev) - 1;
        lo -= first;
        if (!((br >> first) & 1u)) break;
        ++hi;
        mode = 0;
        continue;
      }
      // state t = (lo, hi + t) for t = q * 32 + lane: runs while !L && R
      unsigned bev[RQ], bl[RQ];
#pragma unroll
      for (int q = 0; q < RQ; ++q) {
        bool L, R;
        test(lo, hi + q * 32 + lane, L, R);
        bev[q] = __ballot_sync(0xffffffffu, L || !R);
        bl[q] = __ballot_sync(0xffffffffu, L);
      }
      int adv = 32 * RQ;
      bool Lf = false;
#pragma unroll
      for (int q = RQ - 1; q >= 0; --q)
        if (bev[q]) {
          const int f = __ffs(bev[q]) - 1;
          adv = q * 32 + f;
          Lf = (bl[q] >> f) & 1u;
        }
      hi += adv;
      if (adv == 32 * RQ) continue;
      if (!Lf) break;
      --lo;
      mode = 0;
    }
    if (lane == 0) {
      s_lohi[0] = lo;
      s_lohi[1] = hi;
    }
    if (pp.p) {
      atomicAdd(pp.p + 2, (unsigned long long)steps);
      atomicAdd(pp.p + 3, 1ull);
    }
  }
  __syncthreads();
  lo = s_lohi[0];
  hi = s_lohi[1];
  blo = lo;
  bhi = hi;
  pp.mark(1);
  BNBG_PAVA_PROBE(3);
  bval = pooled(lo, hi);
  BNBG_PAVA_PROBE(4);
}

// Column shared-memory carve-up used by every column kernel.
struct ColSmem {
  double* key;
  int* idx;
  double* u;
  double* scan;
  double* xk;
  int* xi;
  double* bo;   // p: staged previous iterate B (prox) / beta (eval)
  uint8_t* st;  // p: staged coordinate states
};
__device__ __forceinline__ ColSmem col_smem(double* sm, int p, int n2, int E) {
  const int ns = sort_slots(n2, E);
  ColSmem c;
  c.key = sm;
  c.idx = reinterpret_cast<int*>(c.key + ns);
  c.u = reinterpret_cast<double*>(c.idx + ns + (ns & 1));
  c.scan = c.u + p;
  c.xk = c.scan + ns;
  c.xi = reinterpret_cast<int*>(c.xk + 2 * ns);
  // staged B / states after xk[2 ns] and xi[2 ns]; the shared-memory sort
  // (E = 0, p > 1024) reads them from global memory instead
  c.bo = E ? c.xk + 3 * ns : nullptr;
  c.st = E ? reinterpret_cast<uint8_t*>(c.bo + p) : nullptr;
  return c;
}

// ---------------------------------------------------------------------------
// VK1 packer: dense CoordState column + reduced budget + free count, and the
// warm start copied into B and V.  Lists are CSR over the batch.
// ---------------------------------------------------------------------------
static __global__ void k_pack(int p, int k, int m, const int* z_off, const int* z_idx, const int* o_off,
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
  __syncthreads();  // J1 after J0, as prox_kernel.hpp:73-80
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
static __global__ void k_init_cols(int p, int m, const uint8_t* state, int* pf, const double* B, double* V,
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

// ---------------------------------------------------------------------------
// VK5: proximal-gradient step + FISTA momentum for every active column.
//
// ColCache: a CTA that owns the same column across iterations (the
// persistent pass kernel, between compactions) keeps the column's B, V and
// states in shared memory and its scalars in registers, so an iteration only
// reads the gradient slabs from global memory.  Global B / V / t are still
// written every iteration (the GEMMs and the evaluation read them).
// ---------------------------------------------------------------------------
struct ColCache {
  int b, kb, pf;
  double t;
  double* B;          // p, shared
  double* V;          // p, shared
  const uint8_t* st;  // p, shared
};

template <int E, bool CACHED>
__device__ __forceinline__ double prox_column_impl(const RelaxDev& r, int ns, int c, double* sm,
                                                   const ColCache cc0) {
  const ColCache* cc = &cc0;
  const int b = CACHED ? cc->b : r.act[c];
  const int p = r.p;
  const ColSmem S = col_smem(sm, p, r.n2, E);
  const uint8_t* st = CACHED ? cc->st : r.state + (size_t)b * p;
  double* Vb = r.V + (size_t)b * p;
  double* Bb = r.B + (size_t)b * p;
  const double* Vsrc = CACHED ? cc->V : Vb;
  const double tm = CACHED ? cc->t : r.t[b];
  ColProbe pr(r.probe);
  bool bad = false;
  column_sort<kNodeThreads, E>(
      p, r.n2,
      [&](int j) {
        const double v = Vsrc[j];
        const uint8_t sj = st[j];
        if (E && !CACHED) {
          S.bo[j] = Bb[j];
          S.st[j] = sj;
        }
        bad |= !isfinite(v);
        const double uj = v - r.eta * gsum(r, ns, b, j);  // U = V - eta G (relaxation.hpp:229)
        S.u[j] = uj;
        const double key = sj == kFree ? r.rho * fabs(uj) : -1.0;
        // a NaN key would break the sorting network's order (and the rank ->
        // index map); the column is reported as numeric_error, so any total
        // order will do
        return key == key ? key : -1.0;
      },
      S.key, S.idx, S.xk, S.xi);
  if (bad) atomicMin(r.d_err, b);  // refresh_predictions' finite check (relaxation.hpp:76-81)
  const int kb = CACHED ? cc->kb : r.kbar[b];
  const int pf = CACHED ? cc->pf : r.pf[b];
  const double* bo_src = CACHED ? cc->B : (E ? S.bo : Bb);
  const uint8_t* st_src = CACHED ? cc->st : (E ? S.st : st);
  int lo, hi;
  double pooled;
  pr.mark(0);
  block_pava<kNodeThreads>(S.key, pf, kb, r.rho, r.M, S.scan, lo, hi, pooled,
                           r.probe ? r.probe + 12 : nullptr);
  pr.mark(1);
  const double inv_rho = 1.0 / r.rho;
  const double t_next = 0.5 * (1.0 + sqrt(1.0 + 4.0 * tm * tm));
  const double coef = (tm - 1.0) / t_next;
  auto put = [&](int j, double out) {
    const double bo = bo_src[j];
    const double vn = r.accel ? out + coef * (out - bo) : out;
    Vb[j] = vn;
    Bb[j] = out;
    if (CACHED) {
      cc->V[j] = vn;
      cc->B[j] = out;
    }
  };
  // free coordinates by rank (prox_kernel.hpp:267-275)
  for (int rk = threadIdx.x; rk < pf; rk += kNodeThreads) {
    const int j = S.idx[rk];
    const double uj = S.u[j];
    double out;
    const bool in_block = hi >= lo && rk >= lo && rk <= hi;
    if (rk >= kb && !in_block) {
      out = 0.0;
    } else {
      const double v = in_block ? pooled : d_prox_huber(S.key[rk], r.rho, r.M);
      const double sign = uj > 0.0 ? 1.0 : (uj < 0.0 ? -1.0 : 0.0);
      out = uj - inv_rho * sign * v;
    }
    put(j, out);
  }
  // fixed coordinates (prox_kernel.hpp:261-266)
  for (int j = threadIdx.x; j < p; j += kNodeThreads) {
    const uint8_t s = st_src[j];
    if (s == kFree) continue;
    const double uj = S.u[j];
    const double out = s == kFixedZero ? 0.0 : uj - inv_rho * d_prox_huber(r.rho * uj, r.rho, r.M);
    put(j, out);
  }
  if (r.accel && threadIdx.x == 0) r.t[b] = t_next;
  pr.mark(2);
  __syncthreads();
  pr.mark(3);
  return r.accel ? t_next : tm;  // the column's new momentum scalar
}

template <int E>
__device__ void prox_column(const RelaxDev& r, int ns, int c, double* sm) {
  prox_column_impl<E, false>(r, ns, c, sm, ColCache{});
}

template <int E>
__global__ void __launch_bounds__(kNodeThreads) k_prox_fista(RelaxDev r) {
  extern __shared__ __align__(16) double sm[];
  if ((int)blockIdx.x >= *r.d_ma) return;
  prox_column<E>(r, r.nsplit, blockIdx.x, col_base(r.colscr, r.colstride, sm));
}

// ---------------------------------------------------------------------------
// g(beta) for one column: +inf off the domain
// (prox_kernel.hpp:310-347 + recover_core primal_heuristics.hpp:60-99).
// All threads return the same value.
// ---------------------------------------------------------------------------
template <int NT, int E>
__device__ double block_g_value(const double* beta, const uint8_t* st, int p, int n2, int kbar,
                                double M, const ColSmem& S, double* red, int* ired) {
  const double box_tol = M * (1.0 + 1e-9);
  double fixed = 0.0;
  int bad = 0, nz = 0, nfree = 0;
  for (int j = threadIdx.x; j < p; j += NT) {
    const double bj = beta[j];
    const uint8_t s = st[j];
    if (s == kFixedZero) {
      bad |= bj != 0.0;
    } else if (s == kFixedOne) {
      bad |= fabs(bj) > box_tol;
      fixed += bj * bj;
    } else {
      bad |= fabs(bj) > box_tol;
      nz += bj != 0.0;
      ++nfree;
    }
  }
  const double fixed_part = block_sum<NT>(fixed, red);
  const int any_bad = block_or<NT>(bad, ired);
  const int nonzero = (int)block_sum<NT>((double)nz, red);
  const int pf = (int)block_sum<NT>((double)nfree, red);
  if (any_bad) return d_inf();
  if (kbar <= 0) return nonzero > 0 ? d_inf() : 0.5 * fixed_part;
  if (nonzero <= kbar) {
    double s = 0.0;
    for (int j = threadIdx.x; j < p; j += NT)
      if (st[j] == kFree) s += beta[j] * beta[j];
    return 0.5 * (fixed_part + block_sum<NT>(s, red));
  }
  column_sort<NT, E>(
      p, n2, [&](int j) { return st[j] == kFree ? fabs(beta[j]) : -1.0; }, S.key, S.idx, S.xk,
      S.xi);
  const double* key = S.key;
  // binding case: suffix sums from the bottom; tail below kbar tree-summed
  double tl = 0.0;
  for (int rk = kbar + threadIdx.x; rk < pf; rk += NT) tl += key[rk];
  const double tail = block_sum<NT>(tl, red);
  __shared__ double s_tau;
  __shared__ int s_cap, s_ok;
  if (threadIdx.x == 0) {
    // suffix[s] for s < kbar, sequential from the bottom (primal_heuristics.hpp:82-84)
    int ok = 0, cap = 0;
    double tau = 0.0;
    double acc = tail;
    // scan s upward needs suffix[s]; accumulate the head once from the bottom
    double head[64];
    const int kh = kbar < 64 ? kbar : 64;
    for (int s = kbar - 1; s >= 0; --s) {
      acc += key[s];
      if (s < kh) head[s] = acc;
    }
    for (int s = 0; s < kbar; ++s) {
      double suf;
      if (s < kh) {
        suf = head[s];
      } else {  // kbar > 64 (rare): recompute this suffix
        suf = tail;
        for (int r2 = kbar - 1; r2 >= s; --r2) suf += key[r2];
      }
      const double tv = suf / (double)(kbar - s);
      const double upper = s == 0 ? d_inf() : key[s - 1];
      const double lower = key[s];
      if (upper >= tv && tv >= lower) {
        ok = 1;
        tau = tv;
        cap = s;
        break;
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
template <int NT, int E>
__device__ double block_g_conj(const double* q, const uint8_t* st, int p, int n2, int kbar,
                               double M, const ColSmem& S, double* red) {
  double ones = 0.0, all_free = 0.0;
  int nfree = 0;
  for (int j = threadIdx.x; j < p; j += NT) {
    const uint8_t s = st[j];
    if (s == kFixedOne) {
      ones += d_huber(q[j], M);
    } else if (s == kFree) {
      all_free += d_huber(q[j], M);
      ++nfree;
    }
  }
  const double total = block_sum<NT>(ones, red);
  if (kbar <= 0) return total;
  const int pf = (int)block_sum<NT>((double)nfree, red);
  if (pf <= kbar) return total + block_sum<NT>(all_free, red);  // TopSum over all entries
  column_sort<NT, E>(
      p, n2, [&](int j) { return st[j] == kFree ? d_huber(q[j], M) : -1.0; }, S.key, S.idx, S.xk,
      S.xi);
  double s = 0.0;
  for (int rk = threadIdx.x; rk < kbar; rk += NT) s += S.key[rk];
  return total + block_sum<NT>(s, red);
}

// ---------------------------------------------------------------------------
// VK6-VK8: bound evaluation of every active column (relaxation.hpp:194-221).
// Expects fresh part_loss/part_conj (from the EVAL GEMM on B) and G = X'R(B).
// ---------------------------------------------------------------------------
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

// One pass over the column gathers every statistic the bound needs (finite
// check, g(beta) domain / nonzero / budget sums, g*(Q) Huber sums, the
// row-block loss and conjugate partials) and reduces them together; only the
// binding g(beta) case and the TopSum of g*(Q) sort.  With a ColCache the
// column's B and states come from shared memory.
template <int E, bool CACHED>
__device__ void eval_column_impl(const RelaxDev& r, int ns, const EvalArgs& e, int c, double* sm,
                                 const ColCache cc0) {
  const ColCache* cc = CACHED ? &cc0 : nullptr;
  const int b = cc ? cc->b : r.act[c];
  const int p = r.p;
  const ColSmem S = col_smem(sm, p, r.n2, E);
  double* q = S.u;
  constexpr int NV = 10;
  __shared__ double red[(kNodeThreads / 32) * NV];
  __shared__ int s_restart;
  const uint8_t* st = cc ? cc->st : r.state + (size_t)b * p;
  const double* Bb = cc ? cc->B : r.B + (size_t)b * p;
  const int kb = cc ? cc->kb : r.kbar[b];
  const double inv2l = 1.0 / (2.0 * r.lambda2);
  const double M = r.M, box_tol = M * (1.0 + 1e-9);
  // v: 0 finite-bad, 1 domain-bad, 2 fixed-one sum b^2, 3 free nonzeros, 4 free count,
  //    5 free sum b^2, 6 sum_{J1} H_M(q), 7 sum_free H_M(q), 8 sum l(S), 9 sum l*(R)
  double v[NV];
#pragma unroll
  for (int t = 0; t < NV; ++t) v[t] = 0.0;
  for (int j = threadIdx.x; j < p; j += kNodeThreads) {
    const double bj = Bb[j];
    const uint8_t sj = st[j];
    const double qj = -gsum(r, ns, b, j) * inv2l;  // Z = -R; Q = X'Z; Q *= 1/(2 lambda2)
    q[j] = qj;
    v[0] += !isfinite(bj) ? 1.0 : 0.0;
    if (sj == kFixedZero) {
      v[1] += bj != 0.0 ? 1.0 : 0.0;
    } else if (sj == kFixedOne) {
      v[1] += fabs(bj) > box_tol ? 1.0 : 0.0;
      v[2] += bj * bj;
      v[6] += d_huber(qj, M);
    } else {
      v[1] += fabs(bj) > box_tol ? 1.0 : 0.0;
      v[3] += bj != 0.0 ? 1.0 : 0.0;
      v[4] += 1.0;
      v[5] += bj * bj;
      v[7] += d_huber(qj, M);
    }
  }
  for (int rb = threadIdx.x; rb < e.nrb; rb += kNodeThreads) {
    v[8] += e.part_loss[(size_t)rb * e.part_ld + b];
    v[9] += e.part_conj[(size_t)rb * e.part_ld + b];
  }
  block_sum_vec<kNodeThreads, NV>(v, red);
  if (v[0] != 0.0 && threadIdx.x == 0) atomicMin(r.d_err, b);
  const int nonzero = (int)v[3], pf = (int)v[4];
  // g(beta) (prox_kernel.hpp:310-347, recover_core primal_heuristics.hpp:60-99)
  double g;
  if (v[1] != 0.0) {
    g = d_inf();
  } else if (kb <= 0) {
    g = nonzero > 0 ? d_inf() : 0.5 * v[2];
  } else if (nonzero <= kb) {
    g = 0.5 * (v[2] + v[5]);
  } else {
    column_sort<kNodeThreads, E>(
        p, r.n2, [&](int j) { return st[j] == kFree ? fabs(Bb[j]) : -1.0; }, S.key, S.idx, S.xk,
        S.xi);
    const double* key = S.key;
    double tl = 0.0;  // ranks below kbar
    for (int rk = kb + threadIdx.x; rk < pf; rk += kNodeThreads) tl += key[rk];
    const double tail = block_sum<kNodeThreads>(tl, red);
    __shared__ double s_tau;
    __shared__ int s_cap, s_ok;
    if (threadIdx.x == 0) {
      // smallest s with key[s-1] >= tau_s >= key[s], tau_s = suffix_s / (kbar - s)
      int ok = 0, cap = 0;
      double tau = 0.0;
      // suffix sums accumulated from the bottom, as the reference does
      // (primal_heuristics.hpp:82-84); kbar <= k is small
      for (int s2 = 0; s2 < kb; ++s2) {
        double sf = tail;
        for (int t = kb - 1; t >= s2; --t) sf += key[t];
        const double tv = sf / (double)(kb - s2);
        const double upper = s2 == 0 ? d_inf() : key[s2 - 1];
        const double lower = key[s2];
        if (upper >= tv && tv >= lower) {
          ok = 1;
          tau = tv;
          cap = s2;
          break;
        }
      }
      s_ok = ok && !(tau > M * (1.0 + 1e-9));
      s_tau = tau;
      s_cap = cap;
    }
    __syncthreads();
    if (!s_ok) {
      g = d_inf();
    } else {
      const double tau = s_tau;
      const int cap = s_cap;
      double fp = 0.0;
      for (int rk = threadIdx.x; rk < pf; rk += kNodeThreads)
        fp += rk < cap ? key[rk] * key[rk] : tau * key[rk];
      g = 0.5 * (v[2] + block_sum<kNodeThreads>(fp, red));
    }
  }
  // g*(Q): sum_{J1} H_M(q) + TopSum_kbar over free H_M(q) (prox_kernel.hpp:351-370)
  double gs;
  if (kb <= 0) {
    gs = v[6];
  } else if (pf <= kb) {
    gs = v[6] + v[7];
  } else {
    column_sort<kNodeThreads, E>(
        p, r.n2, [&](int j) { return st[j] == kFree ? d_huber(q[j], M) : -1.0; }, S.key, S.idx,
        S.xk, S.xi);
    double s2 = 0.0;
    for (int rk = threadIdx.x; rk < kb; rk += kNodeThreads) s2 += S.key[rk];
    gs = v[6] + block_sum<kNodeThreads>(s2, red);
  }
  if (threadIdx.x == 0) {
    s_restart = 0;
    const double phi = v[8] + 2.0 * r.lambda2 * g;      // relaxation.hpp:108-123
    const double psi = -v[9] - 2.0 * r.lambda2 * gs;    // relaxation.hpp:127-147
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
  __syncthreads();
}

template <int E>
__device__ void eval_column(const RelaxDev& r, int ns, const EvalArgs& e, int c, double* sm) {
  eval_column_impl<E, false>(r, ns, e, c, sm, ColCache{});
}

template <int E>
__global__ void __launch_bounds__(kNodeThreads) k_eval(RelaxDev r, EvalArgs e) {
  extern __shared__ __align__(16) double sm[];
  if ((int)blockIdx.x >= *r.d_ma) return;
  eval_column<E>(r, r.nsplit, e, blockIdx.x, col_base(r.colscr, r.colstride, sm));
}

// order-preserving compaction of the active list by one CTA of NT threads
template <int NT>
__device__ void compact_active(int* act, int* d_ma, const uint8_t* frozen) {
  __shared__ int warp_tot[32];
  __shared__ int s_base;
  const int ma = *(volatile int*)d_ma;
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
  for (int base = 0; base < ma; base += NT) {
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
    if (threadIdx.x == NT - 1) {
      int tot = 0;
      for (int w = 0; w < NT / 32; ++w) tot += warp_tot[w];
      s_base = base_out + tot;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *d_ma = s_base;
  __syncthreads();
}

static __global__ void __launch_bounds__(1024) k_compact(int* act, int* d_ma, const uint8_t* frozen) {
  compact_active<1024>(act, d_ma, frozen);
}

// ---------------------------------------------------------------------------
// VK9 + VK11: rounding support and branching variable from one sort of the
// free |beta| (key desc, index asc).  support row b = J1 ++ top-kbar free.
// ---------------------------------------------------------------------------
template <int E>
__global__ void __launch_bounds__(kNodeThreads)
    k_round_select(int p, int n2, int k, const double* beta, const uint8_t* state, const int* kbar,
                   const int* one_off, const int* one_idx, const int* one_len, int* sup, int* len,
                   int* jbranch, double* gscr, long long gstride) {
  extern __shared__ __align__(16) double sm[];
  const int b = blockIdx.x;
  const ColSmem S = col_smem(col_base(gscr, gstride, sm), p, n2, E);
  const double* bb = beta + (size_t)b * p;
  const uint8_t* st = state + (size_t)b * p;
  column_sort<kNodeThreads, E>(
      p, n2, [&](int j) { return st[j] == kFree ? fabs(bb[j]) : -1.0; }, S.key, S.idx, S.xk, S.xi);
  if (threadIdx.x == 0) {
    int l = 0;
    if (one_len) {  // padded lists: column b's J1 at one_idx[b*k, b*k + one_len[b])
      for (int t = 0; t < one_len[b]; ++t) sup[(size_t)b * k + l++] = one_idx[(size_t)b * k + t];
    } else if (one_off) {  // CSR lists
      for (int t = one_off[b]; t < one_off[b + 1]; ++t) sup[(size_t)b * k + l++] = one_idx[t];
    }
    const int kb = kbar[b];
    for (int rk = 0; rk < kb && rk < p && S.key[rk] >= 0.0; ++rk) sup[(size_t)b * k + l++] = S.idx[rk];
    if (len) len[b] = l;
    if (jbranch) jbranch[b] = S.key[0] >= 0.0 ? S.idx[0] : -1;
  }
}

// ---------------------------------------------------------------------------
// stateless test kernels (prox_kernel.hpp:177-229, :284-301, :310-370)
// mode 0: prox_step (out = U - rho^-1 prox_{rho g*}(rho U), w = rho);
// mode 1: conjugate prox of weight*g* at U (w = weight)
// ---------------------------------------------------------------------------
template <int E>
__global__ void __launch_bounds__(kNodeThreads)
    k_prox_standalone(int mode, int p, int n2, const double* U, const uint8_t* state, const int* kbar,
                      double w, double M, double* out, double* gscr, long long gstride) {
  extern __shared__ __align__(16) double sm[];
  const int b = blockIdx.x;
  const ColSmem S = col_smem(col_base(gscr, gstride, sm), p, n2, E);
  __shared__ double red[kNodeThreads / 32];
  const double* u = U + (size_t)b * p;
  const uint8_t* st = state + (size_t)b * p;
  double* o = out + (size_t)b * p;
  const double scale = mode == 0 ? w : 1.0;
  int cnt = 0;
  for (int j = threadIdx.x; j < p; j += kNodeThreads) cnt += st[j] == kFree;
  const int pf = (int)block_sum<kNodeThreads>((double)cnt, red);
  column_sort<kNodeThreads, E>(
      p, n2,
      [&](int j) {
        const double key = st[j] == kFree ? scale * fabs(u[j]) : -1.0;
        return key == key ? key : -1.0;
      },
      S.key, S.idx, S.xk, S.xi);
  const int kb = kbar[b];
  int lo, hi;
  double pooled;
  block_pava<kNodeThreads>(S.key, pf, kb, w, M, S.scan, lo, hi, pooled);
  for (int rk = threadIdx.x; rk < pf; rk += kNodeThreads) {
    const int j = S.idx[rk];
    const bool in_block = hi >= lo && rk >= lo && rk <= hi;
    const double v = in_block ? pooled : (rk < kb ? d_prox_huber(S.key[rk], w, M) : S.key[rk]);
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

template <int E>
__global__ void __launch_bounds__(kNodeThreads)
    k_g_standalone(int mode, int p, int n2, const double* in, const uint8_t* state, const int* kbar,
                   double M, double* out, double* gscr, long long gstride) {
  extern __shared__ __align__(16) double sm[];
  const int b = blockIdx.x;
  const ColSmem S = col_smem(col_base(gscr, gstride, sm), p, n2, E);
  __shared__ double red[kNodeThreads / 32];
  __shared__ int ired[kNodeThreads / 32];
  const double v =
      mode == 0 ? block_g_value<kNodeThreads, E>(in + (size_t)b * p, state + (size_t)b * p, p, n2,
                                                 kbar[b], M, S, red, ired)
                : block_g_conj<kNodeThreads, E>(in + (size_t)b * p, state + (size_t)b * p, p, n2,
                                                kbar[b], M, S, red);
  if (threadIdx.x == 0) out[b] = v;
}

}  // namespace bnbg
