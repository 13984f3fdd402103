/*
 * oracle.c -- CPU restatement of the bnbglm node-processing path.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Not linked into the product.
 *
 * Each function restates the reference header it names, file:line relative to
 * /root/reference/proj/include/bnbglm/.  The reference itself cannot be built
 * in this image (Eigen absent), so the restatement keeps every constant,
 * tie-break and evaluation order visible in the source; only Eigen's GEMM /
 * GEMV / reduction association order is not reproducible.
 */
#define _GNU_SOURCE
#include "oracle.h"

#include <dlfcn.h>
#include <float.h>
#include <math.h>
#include <omp.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define INF (1.0 / 0.0)
#define SENTINEL (-DBL_MAX) /* prox_kernel.hpp:112 numeric_limits<double>::lowest() */

/* ======================================================================= */
/* rng.hpp:13-64                                                           */
/* ======================================================================= */
static inline uint64_t rotl64(uint64_t v, int s) { return (v << s) | (v >> (64 - s)); }

void orc_rng_seed(orc_rng* r, uint64_t seed) { /* rng.hpp:15-24 */
  uint64_t x = seed;
  for (int w = 0; w < 4; ++w) {
    x += 0x9e3779b97f4a7c15ULL;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    r->s[w] = z ^ (z >> 31);
  }
  r->spare = 0.0;
  r->has_spare = 0;
}

uint64_t orc_rng_next(orc_rng* r) { /* rng.hpp:26-35 */
  uint64_t* s = r->s;
  const uint64_t result = rotl64(s[0] + s[3], 23) + s[0];
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return result;
}

double orc_rng_uniform(orc_rng* r) { /* rng.hpp:39 */
  return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53;
}

double orc_rng_gaussian(orc_rng* r) { /* rng.hpp:42-55 */
  if (r->has_spare) {
    r->has_spare = 0;
    return r->spare;
  }
  const double u1 = (double)((orc_rng_next(r) >> 11) + 1) * 0x1.0p-53;
  const double u2 = orc_rng_uniform(r);
  const double radius = sqrt(-2.0 * log(u1));
  const double angle = 2.0 * M_PI * u2;
  r->spare = radius * sin(angle);
  r->has_spare = 1;
  return radius * cos(angle);
}

/* ======================================================================= */
/* losses.hpp:37-112                                                       */
/* ======================================================================= */
static inline double log1p_exp(double t) { /* losses.hpp:37-40 */
  if (t > 0.0) return t + log1p(exp(-t));
  return log1p(exp(t));
}
static inline double sigmoid(double t) { /* losses.hpp:43-50 */
  if (t >= 0.0) {
    const double e = exp(-t);
    return 1.0 / (1.0 + e);
  }
  const double e = exp(t);
  return e / (1.0 + e);
}
static inline double xlogx(double v) { return v > 0.0 ? v * log(v) : 0.0; } /* :52 */

double orc_loss_value(int loss, double s, double y) { /* losses.hpp:56-63 */
  if (loss == ORC_SQUARED) {
    const double r = s - y;
    return 0.5 * r * r;
  }
  return log1p_exp(-y * s);
}
double orc_loss_derivative(int loss, double s, double y) { /* losses.hpp:65-69 */
  if (loss == ORC_SQUARED) return s - y;
  return -y * sigmoid(-y * s);
}
double orc_loss_conjugate(int loss, double zeta, double y) { /* losses.hpp:74-79 */
  if (loss == ORC_SQUARED) return 0.5 * zeta * zeta + zeta * y;
  const double a = -zeta * y;
  if (a < 0.0 || a > 1.0) return INF;
  return xlogx(a) + xlogx(1.0 - a);
}

static double vnorm(const double* v, int len) {
  double s = 0.0;
  for (int i = 0; i < len; ++i) s += v[i] * v[i];
  return sqrt(s);
}

double orc_smoothness(int loss, const double* X, int n, int p) { /* losses.hpp:86-112 */
  if (n <= 0 || p <= 0) return -1.0;
  const double c = loss == ORC_SQUARED ? 1.0 : 0.25;
  orc_rng rng;
  orc_rng_seed(&rng, 0x5eed5eedULL);
  double* v = (double*)malloc(sizeof(double) * p);
  double* w = (double*)malloc(sizeof(double) * p);
  double* xv = (double*)malloc(sizeof(double) * n);
  for (int j = 0; j < p; ++j) v[j] = orc_rng_uniform(&rng) - 0.5;
  const double v0 = vnorm(v, p);
  if (v0 == 0.0) v[0] = 1.0;
  {
    const double nv = vnorm(v, p);
    for (int j = 0; j < p; ++j) v[j] /= nv;
  }
  double estimate = 0.0;
  double result = -1.0;
  for (int it = 0; it < 100; ++it) {
    for (int i = 0; i < n; ++i) xv[i] = 0.0; /* xv = X v */
    for (int j = 0; j < p; ++j) {
      const double vj = v[j];
      const double* col = X + (size_t)j * n;
      for (int i = 0; i < n; ++i) xv[i] += col[i] * vj;
    }
    for (int j = 0; j < p; ++j) { /* w = X' xv */
      const double* col = X + (size_t)j * n;
      double s = 0.0;
      for (int i = 0; i < n; ++i) s += col[i] * xv[i];
      w[j] = s;
    }
    double next = 0.0;
    for (int j = 0; j < p; ++j) next += v[j] * w[j];
    const double wn = vnorm(w, p);
    if (wn == 0.0 || next <= 0.0) {
      result = 1e-12;
      break;
    }
    for (int j = 0; j < p; ++j) v[j] = w[j] / wn;
    if (it > 0 && fabs(next - estimate) <= 1e-4 * next) {
      estimate = next;
      break;
    }
    estimate = next;
  }
  if (result < 0.0) result = fmax(1.01 * c * estimate, 1e-12);
  free(v);
  free(w);
  free(xv);
  return result;
}

/* ======================================================================= */
/* problem.hpp:36-132                                                      */
/* ======================================================================= */
int orc_validate(const double* X, const double* y, int n, int p, int loss, int k, double M,
                 double lambda2) { /* problem.hpp:36-51 */
  if (n <= 0 || p <= 0) return ORC_INPUT_ERROR;
  for (size_t i = 0; i < (size_t)n * p; ++i)
    if (!isfinite(X[i])) return ORC_INPUT_ERROR;
  for (int i = 0; i < n; ++i)
    if (!isfinite(y[i])) return ORC_INPUT_ERROR;
  if (k < 1 || k > p) return ORC_INPUT_ERROR;
  if (!(M > 0.0) || !(lambda2 > 0.0)) return ORC_INPUT_ERROR;
  if (loss == ORC_LOGISTIC)
    for (int i = 0; i < n; ++i)
      if (y[i] != 1.0 && y[i] != -1.0) return ORC_INPUT_ERROR;
  return ORC_OK;
}

/* problem.hpp:70-132.  The Cholesky factor of the AR(1) Toeplitz matrix
 * Sigma_jl = rho^|j-l| (problem.hpp:83-87) is used in closed form:
 * L[j][0] = rho^j, L[j][l] = rho^(j-l) sqrt(1-rho^2) for 1 <= l <= j
 * (exact in real arithmetic; rho^d by repeated multiplication).  Row i of X is
 * L g_i (problem.hpp:96) accumulated in ascending l with fma. */
int orc_generate(int n, int p, int k, double rho, int loss, double snr, uint64_t seed,
                 double* X, double* y, int* support) {
  if (n < 1 || p < 1) return ORC_INPUT_ERROR;
  if (k < 1 || k > p) return ORC_INPUT_ERROR;
  if (rho < 0.0 || rho >= 1.0) return ORC_INPUT_ERROR;
  if (!(snr > 0.0)) return ORC_INPUT_ERROR;
  orc_rng rng;
  orc_rng_seed(&rng, seed);
  double* G = (double*)malloc(sizeof(double) * (size_t)n * p); /* row-major draws */
  for (size_t t = 0; t < (size_t)n * p; ++t) G[t] = orc_rng_gaussian(&rng);
  if (rho > 0.0) {
    double* pw = (double*)malloc(sizeof(double) * p);
    pw[0] = 1.0;
    for (int d = 1; d < p; ++d) pw[d] = pw[d - 1] * rho;
    const double sr = sqrt(1.0 - rho * rho);
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i) {
      const double* g = G + (size_t)i * p;
      for (int j = 0; j < p; ++j) {
        double acc = pw[j] * g[0];
        for (int l = 1; l <= j; ++l) acc = fma(pw[j - l] * sr, g[l], acc);
        X[(size_t)j * n + i] = acc;
      }
    }
    free(pw);
  } else {
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < p; ++j) X[(size_t)j * n + i] = G[(size_t)i * p + j];
  }
  free(G);
  const int step = p / k; /* problem.hpp:101-107 */
  for (int t = 1; t <= k; ++t) support[t - 1] = t * step - 1;
  double* signal = (double*)calloc(n, sizeof(double));
  for (int t = 0; t < k; ++t) { /* X * beta_true, beta_true = 1 on support */
    const double* col = X + (size_t)support[t] * n;
    for (int i = 0; i < n; ++i) signal[i] += col[i];
  }
  if (loss == ORC_SQUARED) { /* problem.hpp:112-115 */
    const double sigma2 = vnorm(signal, n) / snr;
    const double sd = sqrt(sigma2);
    for (int i = 0; i < n; ++i) y[i] = signal[i] + sd * orc_rng_gaussian(&rng);
  } else { /* problem.hpp:116-121 */
    for (int i = 0; i < n; ++i) {
      const double prob = sigmoid(signal[i]);
      y[i] = orc_rng_uniform(&rng) < prob ? 1.0 : -1.0;
    }
  }
  free(signal);
  return ORC_OK;
}

/* ======================================================================= */
/* prox_kernel.hpp:27-370                                                  */
/* ======================================================================= */
double orc_huber(double q, double M) { /* prox_kernel.hpp:27-30 */
  const double a = fabs(q);
  return a <= M ? 0.5 * q * q : M * a - 0.5 * M * M;
}
double orc_prox_huber(double x, double w, double M) { /* prox_kernel.hpp:33-36 */
  if (fabs(x) <= (1.0 + w) * M) return x / (1.0 + w);
  return x - w * M * (x > 0.0 ? 1.0 : -1.0);
}

typedef struct {
  double key;
  int idx;
} keyed_t;

/* (key desc, idx asc): prox_kernel.hpp:119-122, primal_heuristics.hpp:41-45 */
static inline int keyed_before(const keyed_t* a, const keyed_t* b) {
  if (a->key != b->key) return a->key > b->key;
  return a->idx < b->idx;
}

/* bottom-up merge sort; the comparator is a total order so the result equals
 * std::sort's (sort_column, prox_kernel.hpp:116-124). */
static void sort_keyed(keyed_t* a, int len, keyed_t* tmp) {
  for (int i = 1; i < len; ++i) { /* insertion sort runs of 16 */
    if ((i & 15) == 0) continue;
    keyed_t v = a[i];
    int j = i - 1;
    const int lo = i & ~15;
    while (j >= lo && keyed_before(&v, &a[j])) {
      a[j + 1] = a[j];
      --j;
    }
    a[j + 1] = v;
  }
  keyed_t* src = a;
  keyed_t* dst = tmp;
  for (int width = 16; width < len; width *= 2) {
    for (int lo = 0; lo < len; lo += 2 * width) {
      int mid = lo + width < len ? lo + width : len;
      int hi = lo + 2 * width < len ? lo + 2 * width : len;
      int i = lo, j = mid, o = lo;
      while (i < mid && j < hi) dst[o++] = keyed_before(&src[j], &src[i]) ? src[j++] : src[i++];
      while (i < mid) dst[o++] = src[i++];
      while (j < hi) dst[o++] = src[j++];
    }
    keyed_t* t = src;
    src = dst;
    dst = t;
  }
  if (src != a) memcpy(a, src, sizeof(keyed_t) * len);
}

/* prox_kernel.hpp:132-170 boundary-seeded PAVA over one sorted column. */
static void run_pava(const double* sorted, int pf, int kbar, double w, double M, double* v,
                     int* blk_lo, int* blk_hi, double* blk_value) {
  *blk_lo = 0;
  *blk_hi = -1;
  *blk_value = 0.0;
  for (int r = 0; r < pf; ++r) v[r] = r < kbar ? orc_prox_huber(sorted[r], w, M) : sorted[r];
  if (kbar <= 0 || kbar >= pf) return;
  if (v[kbar - 1] >= v[kbar]) return;
  int lo = kbar - 1, hi = kbar;
  double pooled = 0.0;
#define RECOMPUTE()                                            \
  do {                                                         \
    double sum_ = 0.0;                                         \
    for (int r_ = lo; r_ <= hi; ++r_) sum_ += sorted[r_];      \
    const int len_ = hi - lo + 1;                              \
    const double mean_w_ = w * (double)(kbar - lo) / len_;     \
    pooled = orc_prox_huber(sum_ / len_, mean_w_, M);          \
  } while (0)
  RECOMPUTE();
  for (;;) {
    if (lo > 0 && v[lo - 1] < pooled) {
      --lo;
      RECOMPUTE();
      continue;
    }
    if (hi < pf - 1 && pooled < v[hi + 1]) {
      ++hi;
      RECOMPUTE();
      continue;
    }
    break;
  }
#undef RECOMPUTE
  for (int r = lo; r <= hi; ++r) v[r] = pooled;
  *blk_lo = lo;
  *blk_hi = hi;
  *blk_value = pooled;
}

/* sorted free keys -> keyed array (free coordinates only; non-free carry the
 * sentinel in the reference and sort strictly below every free key). */
static int collect_free_keys(const double* x, const uint8_t* st, int p, double scale,
                             keyed_t* kv, keyed_t* tmp) {
  int pf = 0;
  for (int j = 0; j < p; ++j)
    if (st[j] == ORC_FREE) {
      kv[pf].key = scale * fabs(x[j]);
      kv[pf].idx = j;
      ++pf;
    }
  sort_keyed(kv, pf, tmp);
  return pf;
}

/* prox_kernel.hpp:236-276 */
void orc_prox_step_column(const double* u, const uint8_t* st, int p, int kbar, double rho,
                          double M, double* out) {
  keyed_t* kv = (keyed_t*)malloc(sizeof(keyed_t) * 2 * (p + 1));
  keyed_t* tmp = kv + p + 1;
  double* sorted = (double*)calloc(2 * (p + 1), sizeof(double));
  double* v = sorted + p + 1;
  const int pf = collect_free_keys(u, st, p, rho, kv, tmp);
  for (int r = 0; r < pf; ++r) sorted[r] = kv[r].key;
  int lo, hi;
  double pooled;
  run_pava(sorted, pf, kbar, rho, M, v, &lo, &hi, &pooled);
  const double inv_rho = 1.0 / rho;
  for (int j = 0; j < p; ++j) {
    if (st[j] == ORC_ZERO)
      out[j] = 0.0;
    else if (st[j] == ORC_ONE)
      out[j] = u[j] - inv_rho * orc_prox_huber(rho * u[j], rho, M);
  }
  for (int r = 0; r < pf; ++r) {
    const int j = kv[r].idx;
    if (r >= kbar && (hi < lo || r < lo || r > hi)) {
      out[j] = 0.0;
      continue;
    }
    const double sign = u[j] > 0.0 ? 1.0 : (u[j] < 0.0 ? -1.0 : 0.0);
    out[j] = u[j] - inv_rho * sign * v[r];
  }
  free(kv);
  free(sorted);
}

/* prox_kernel.hpp:177-212 */
void orc_conjugate_prox_column(const double* x, const uint8_t* st, int p, int kbar, double w,
                               double M, double* out) {
  keyed_t* kv = (keyed_t*)malloc(sizeof(keyed_t) * 2 * (p + 1));
  keyed_t* tmp = kv + p + 1;
  double* sorted = (double*)calloc(2 * (p + 1), sizeof(double));
  double* v = sorted + p + 1;
  const int pf = collect_free_keys(x, st, p, 1.0, kv, tmp);
  for (int r = 0; r < pf; ++r) sorted[r] = kv[r].key;
  int lo, hi;
  double pooled;
  run_pava(sorted, pf, kbar, w, M, v, &lo, &hi, &pooled);
  for (int j = 0; j < p; ++j) {
    if (st[j] == ORC_ZERO)
      out[j] = x[j];
    else if (st[j] == ORC_ONE)
      out[j] = orc_prox_huber(x[j], w, M);
  }
  for (int r = 0; r < pf; ++r) {
    const int j = kv[r].idx;
    const double sign = x[j] > 0.0 ? 1.0 : (x[j] < 0.0 ? -1.0 : 0.0);
    out[j] = sign * v[r];
  }
  free(kv);
  free(sorted);
}

/* Generic left-to-right PAVA (SPEC.md:307 test oracle): nonincreasing fit of
 * sorted keys with per-rank weights w (r < kbar) / 0, block value =
 * prox_huber(mean key, mean weight, M). */
void orc_conjugate_prox_column_generic(const double* x, const uint8_t* st, int p, int kbar,
                                       double w, double M, double* out) {
  keyed_t* kv = (keyed_t*)malloc(sizeof(keyed_t) * 2 * (p + 1));
  keyed_t* tmp = kv + p + 1;
  const int pf = collect_free_keys(x, st, p, 1.0, kv, tmp);
  double* bsum = (double*)malloc(sizeof(double) * (pf + 1));
  double* bw = (double*)malloc(sizeof(double) * (pf + 1));
  double* bval = (double*)malloc(sizeof(double) * (pf + 1));
  int* blen = (int*)malloc(sizeof(int) * (pf + 1));
  int nb = 0;
  for (int r = 0; r < pf; ++r) {
    bsum[nb] = kv[r].key;
    bw[nb] = r < kbar ? w : 0.0;
    blen[nb] = 1;
    bval[nb] = orc_prox_huber(bsum[nb], bw[nb], M);
    ++nb;
    while (nb > 1 && bval[nb - 2] < bval[nb - 1]) {
      bsum[nb - 2] += bsum[nb - 1];
      bw[nb - 2] += bw[nb - 1];
      blen[nb - 2] += blen[nb - 1];
      --nb;
      bval[nb - 1] =
          orc_prox_huber(bsum[nb - 1] / blen[nb - 1], bw[nb - 1] / blen[nb - 1], M);
    }
  }
  for (int j = 0; j < p; ++j) {
    if (st[j] == ORC_ZERO)
      out[j] = x[j];
    else if (st[j] == ORC_ONE)
      out[j] = orc_prox_huber(x[j], w, M);
  }
  int r = 0;
  for (int b = 0; b < nb; ++b)
    for (int t = 0; t < blen[b]; ++t, ++r) {
      const int j = kv[r].idx;
      const double sign = x[j] > 0.0 ? 1.0 : (x[j] < 0.0 ? -1.0 : 0.0);
      out[j] = sign * bval[b];
    }
  free(kv);
  free(bsum);
  free(bw);
  free(bval);
  free(blen);
}

/* primal_heuristics.hpp:35-47 sorted_free_indices: (|beta| desc, idx asc) */
static int sorted_free(const double* beta, const uint8_t* st, int p, keyed_t* kv,
                       keyed_t* tmp) {
  return collect_free_keys(beta, st, p, 1.0, kv, tmp);
}

typedef struct {
  int ok, binding, cap_count;
  double tau;
} recovered_t;

/* primal_heuristics.hpp:60-99 recover_core; kv holds the sorted free set. */
static recovered_t recover_core(const double* beta, const keyed_t* kv, int pf, int kbar,
                                double M, double* suffix) {
  recovered_t core = {0, 0, 0, 0.0};
  if (kbar <= 0) {
    core.ok = 1;
    core.tau = M;
    return core;
  }
  int nonzero = 0;
  for (int r = 0; r < pf; ++r)
    if (beta[kv[r].idx] != 0.0) ++nonzero;
  if (nonzero <= kbar) {
    core.ok = 1;
    core.tau = M;
    core.cap_count = nonzero;
    return core;
  }
  core.binding = 1;
  suffix[pf] = 0.0;
  for (int r = pf - 1; r >= 0; --r) suffix[r] = suffix[r + 1] + fabs(beta[kv[r].idx]);
  for (int s = 0; s < kbar; ++s) {
    const double tau = suffix[s] / (double)(kbar - s);
    const double upper = s == 0 ? INF : fabs(beta[kv[s - 1].idx]);
    const double lower = fabs(beta[kv[s].idx]);
    if (upper >= tau && tau >= lower) {
      core.ok = 1;
      core.tau = tau;
      core.cap_count = s;
      return core;
    }
  }
  return core;
}

int orc_recover(const double* beta, const uint8_t* st, int p, int kbar, double M, double* z,
                double* tau, int* cap_count) { /* primal_heuristics.hpp:103-130 */
  keyed_t* kv = (keyed_t*)malloc(sizeof(keyed_t) * 2 * (p + 1));
  double* suffix = (double*)malloc(sizeof(double) * (p + 2));
  const int pf = sorted_free(beta, st, p, kv, kv + p + 1);
  recovered_t core = recover_core(beta, kv, pf, kbar, M, suffix);
  int ok = core.ok && !(core.tau > M * (1.0 + 1e-9));
  if (ok) {
    *tau = core.tau;
    *cap_count = core.cap_count;
    for (int j = 0; j < p; ++j) z[j] = st[j] == ORC_ONE ? 1.0 : 0.0;
    if (kbar > 0) {
      if (!core.binding) {
        for (int r = 0; r < pf; ++r)
          if (beta[kv[r].idx] != 0.0) z[kv[r].idx] = 1.0;
      } else {
        for (int r = 0; r < pf; ++r) {
          const int j = kv[r].idx;
          z[j] = r < core.cap_count ? 1.0 : fabs(beta[j]) / core.tau;
        }
      }
    }
  }
  free(kv);
  free(suffix);
  return ok;
}

/* prox_kernel.hpp:310-347 g_value_core (scratch: kv 2(p+1), suffix p+2) */
static double g_value_ws(const double* beta, const uint8_t* st, int p, int kbar, double M,
                         keyed_t* kv, double* suffix) {
  const double box_tol = M * (1.0 + 1e-9);
  double fixed_part = 0.0;
  for (int j = 0; j < p; ++j) {
    switch (st[j]) {
      case ORC_ZERO:
        if (beta[j] != 0.0) return INF;
        break;
      case ORC_ONE:
        if (fabs(beta[j]) > box_tol) return INF;
        fixed_part += beta[j] * beta[j];
        break;
      default:
        if (fabs(beta[j]) > box_tol) return INF;
        break;
    }
  }
  if (kbar <= 0) {
    for (int j = 0; j < p; ++j)
      if (st[j] == ORC_FREE && beta[j] != 0.0) return INF;
    return 0.5 * fixed_part;
  }
  const int pf = sorted_free(beta, st, p, kv, kv + p + 1);
  recovered_t core = recover_core(beta, kv, pf, kbar, M, suffix);
  if (!core.ok || core.tau > M * (1.0 + 1e-9)) return INF;
  double free_part = 0.0;
  if (!core.binding) {
    for (int r = 0; r < pf; ++r) free_part += beta[kv[r].idx] * beta[kv[r].idx];
  } else {
    for (int r = 0; r < pf; ++r) {
      const double mag = fabs(beta[kv[r].idx]);
      free_part += r < core.cap_count ? mag * mag : core.tau * mag;
    }
  }
  return 0.5 * (fixed_part + free_part);
}

double orc_g_value(const double* beta, const uint8_t* st, int p, int kbar, double M) {
  keyed_t* kv = (keyed_t*)malloc(sizeof(keyed_t) * 2 * (p + 1));
  double* suffix = (double*)malloc(sizeof(double) * (p + 2));
  const double g = g_value_ws(beta, st, p, kbar, M, kv, suffix);
  free(kv);
  free(suffix);
  return g;
}

static int cmp_desc_double(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return x < y ? 1 : (x > y ? -1 : 0);
}

/* prox_kernel.hpp:351-370 g_conjugate_core.  The top-kbar subset is summed in
 * descending order (the reference's nth_element order is unspecified). */
static double g_conjugate_ws(const double* q, const uint8_t* st, int p, int kbar, double M,
                             double* scratch) {
  double total = 0.0;
  int ns = 0;
  for (int j = 0; j < p; ++j) {
    if (st[j] == ORC_ONE)
      total += orc_huber(q[j], M);
    else if (st[j] == ORC_FREE)
      scratch[ns++] = orc_huber(q[j], M);
  }
  if (kbar <= 0) return total;
  if (ns > kbar) {
    qsort(scratch, ns, sizeof(double), cmp_desc_double);
    ns = kbar;
  }
  for (int t = 0; t < ns; ++t) total += scratch[t];
  return total;
}

double orc_g_conjugate(const double* q, const uint8_t* st, int p, int kbar, double M) {
  double* scratch = (double*)malloc(sizeof(double) * (p + 1));
  const double v = g_conjugate_ws(q, st, p, kbar, M, scratch);
  free(scratch);
  return v;
}

/* ======================================================================= */
/* GEMM plumbing (Eigen's products at relaxation.hpp:82, :102, :132)       */
/* ======================================================================= */
typedef void (*cblas_dgemm64_t)(int, int, int, int64_t, int64_t, int64_t, double,
                                const double*, int64_t, const double*, int64_t, double,
                                double*, int64_t);
static cblas_dgemm64_t g_blas_dgemm = NULL;

int orc_use_openblas(const char* path, int threads) {
  void* h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
  if (!h) return 0;
  cblas_dgemm64_t f = (cblas_dgemm64_t)dlsym(h, "scipy_cblas_dgemm64_");
  if (!f) return 0;
  if (threads > 0) {
    void (*set_threads)(int) = (void (*)(int))dlsym(h, "scipy_openblas_set_num_threads64_");
    if (set_threads) set_threads(threads);
  }
  g_blas_dgemm = f;
  return 1;
}
int orc_blas_active(void) { return g_blas_dgemm != NULL; }

/* C (n x m) = X (n x p) * B (p x m) */
static void gemm_nn(const double* X, int n, int p, const double* B, int m, double* C,
                    int workers) {
  if (g_blas_dgemm) {
    g_blas_dgemm(102, 111, 111, n, m, p, 1.0, X, n, B, p, 0.0, C, n);
    return;
  }
#pragma omp parallel for num_threads(workers) schedule(static)
  for (int b = 0; b < m; ++b) {
    double* c = C + (size_t)b * n;
    const double* bb = B + (size_t)b * p;
    for (int i = 0; i < n; ++i) c[i] = 0.0;
    for (int j = 0; j < p; ++j) {
      const double s = bb[j];
      const double* x = X + (size_t)j * n;
      for (int i = 0; i < n; ++i) c[i] += x[i] * s;
    }
  }
}

/* C (p x m) = X' (p x n) * R (n x m) */
static void gemm_tn(const double* X, int n, int p, const double* R, int m, double* C,
                    int workers) {
  if (g_blas_dgemm) {
    g_blas_dgemm(102, 112, 111, p, m, n, 1.0, X, n, R, n, 0.0, C, p);
    return;
  }
#pragma omp parallel for num_threads(workers) schedule(static)
  for (int b = 0; b < m; ++b) {
    const double* r = R + (size_t)b * n;
    for (int j = 0; j < p; ++j) {
      const double* x = X + (size_t)j * n;
      double s = 0.0;
      for (int i = 0; i < n; ++i) s += x[i] * r[i];
      C[(size_t)b * p + j] = s;
    }
  }
}

/* ======================================================================= */
/* relaxation.hpp:163-255                                                  */
/* ======================================================================= */
void orc_relax_cfg_default(orc_relax_cfg* c) { /* relaxation.hpp:26-33 */
  c->max_iterations = 2000;
  c->gap_tolerance = 1e-6;
  c->check_interval = 10;
  c->acceleration = 1;
  c->smoothness = 0.0;
  c->workers = 1;
}

typedef struct {
  int n, p, m;
  double *B, *Bnext, *V, *S, *R, *G, *Q, *primal, *dual;
  keyed_t** kv;    /* per worker scratch */
  double** dscr;   /* per worker scratch, 4(p+2) doubles */
  int nworkers;
} relax_ws;

static void ws_alloc(relax_ws* w, int n, int p, int m, int workers) {
  w->n = n;
  w->p = p;
  w->m = m;
  const size_t pm = (size_t)p * m, nm = (size_t)n * m;
  w->B = (double*)malloc(sizeof(double) * pm);
  w->Bnext = (double*)malloc(sizeof(double) * pm);
  w->V = (double*)malloc(sizeof(double) * pm);
  w->G = (double*)malloc(sizeof(double) * pm);
  w->Q = (double*)malloc(sizeof(double) * pm);
  w->S = (double*)malloc(sizeof(double) * nm);
  w->R = (double*)malloc(sizeof(double) * nm);
  w->primal = (double*)malloc(sizeof(double) * m);
  w->dual = (double*)malloc(sizeof(double) * m);
  w->nworkers = workers < 1 ? 1 : workers;
  w->kv = (keyed_t**)malloc(sizeof(keyed_t*) * w->nworkers);
  w->dscr = (double**)malloc(sizeof(double*) * w->nworkers);
  for (int t = 0; t < w->nworkers; ++t) {
    w->kv[t] = (keyed_t*)malloc(sizeof(keyed_t) * 2 * (p + 1));
    w->dscr[t] = (double*)malloc(sizeof(double) * 5 * (p + 2));
  }
}

static void ws_free(relax_ws* w) {
  free(w->B);
  free(w->Bnext);
  free(w->V);
  free(w->G);
  free(w->Q);
  free(w->S);
  free(w->R);
  free(w->primal);
  free(w->dual);
  for (int t = 0; t < w->nworkers; ++t) {
    free(w->kv[t]);
    free(w->dscr[t]);
  }
  free(w->kv);
  free(w->dscr);
}

/* prox_step_column with caller scratch (prox_kernel.hpp:236-276) */
static void prox_step_ws(const double* u, const uint8_t* st, int p, int kbar, double rho,
                         double M, double* out, keyed_t* kv, double* dscr) {
  double* sorted = dscr;
  double* v = dscr + (p + 1);
  const int pf = collect_free_keys(u, st, p, rho, kv, kv + p + 1);
  for (int r = 0; r < pf; ++r) sorted[r] = kv[r].key;
  int lo, hi;
  double pooled;
  run_pava(sorted, pf, kbar, rho, M, v, &lo, &hi, &pooled);
  const double inv_rho = 1.0 / rho;
  for (int j = 0; j < p; ++j) {
    if (st[j] == ORC_ZERO)
      out[j] = 0.0;
    else if (st[j] == ORC_ONE)
      out[j] = u[j] - inv_rho * orc_prox_huber(rho * u[j], rho, M);
  }
  for (int r = 0; r < pf; ++r) {
    const int j = kv[r].idx;
    if (r >= kbar && (hi < lo || r < lo || r > hi)) {
      out[j] = 0.0;
      continue;
    }
    const double sign = u[j] > 0.0 ? 1.0 : (u[j] < 0.0 ? -1.0 : 0.0);
    out[j] = u[j] - inv_rho * sign * v[r];
  }
}

/* relaxation.hpp:70-93 refresh_predictions.  Returns -1 or the first
 * non-frozen column with a non-finite entry. */
static int refresh_predictions(const double* Bmat, const double* X, const double* y, int n,
                               int p, int loss, relax_ws* w, const uint8_t* frozen,
                               int workers) {
  const int m = w->m;
  for (int b = 0; b < m; ++b) {
    if (frozen && frozen[b]) continue;
    const double* col = Bmat + (size_t)b * p;
    for (int j = 0; j < p; ++j)
      if (!isfinite(col[j])) return b;
  }
  gemm_nn(X, n, p, Bmat, m, w->S, workers);
#pragma omp parallel for num_threads(workers) schedule(static)
  for (int b = 0; b < m; ++b) {
    if (frozen && frozen[b]) continue;
    const double* s = w->S + (size_t)b * n;
    double* r = w->R + (size_t)b * n;
    if (loss == ORC_SQUARED) {
      for (int i = 0; i < n; ++i) r[i] = s[i] - y[i];
    } else {
      for (int i = 0; i < n; ++i) r[i] = -y[i] * sigmoid(-y[i] * s[i]);
    }
  }
  return -1;
}

int orc_relax_batch(const double* X, const double* y, int n, int p, int loss, double M,
                    double lambda2, const orc_relax_cfg* cfg, double prune_threshold, int m,
                    const uint8_t* state, const int* kbar, const double* warm, double* beta,
                    double* bounds, int* status, int* iters, orc_trace_fn trace, void* user,
                    int* err_column) {
  if (m <= 0) return ORC_INPUT_ERROR; /* relaxation.hpp:168 */
  const int workers = cfg->workers < 1 ? 1 : cfg->workers;
  relax_ws w;
  ws_alloc(&w, n, p, m, workers);
  double lips = cfg->smoothness;
  if (!(lips > 0.0)) lips = orc_smoothness(loss, X, n, p);
  const double eta = 1.0 / lips; /* relaxation.hpp:177-180 */
  const double rho = 1.0 / (2.0 * eta * lambda2);
  memcpy(w.B, warm, sizeof(double) * (size_t)p * m);
  memcpy(w.V, w.B, sizeof(double) * (size_t)p * m);
  uint8_t* frozen = (uint8_t*)calloc(m, 1);
  double* momentum = (double*)malloc(sizeof(double) * m);
  double* best_dual = (double*)malloc(sizeof(double) * m);
  double* last_gap = (double*)malloc(sizeof(double) * m);
  for (int b = 0; b < m; ++b) {
    momentum[b] = 1.0;
    best_dual[b] = -INF;
    last_gap[b] = INF;
    status[b] = ORC_CAPPED;
    iters[b] = cfg->max_iterations;
  }
  int active = m;
  int rc = ORC_OK;
  const double inv2l = 1.0 / (2.0 * lambda2);

  /* relaxation.hpp:194-221 evaluate_bounds */
#define EVALUATE(ITER)                                                                    \
  do {                                                                                    \
    int bad_ = refresh_predictions(w.B, X, y, n, p, loss, &w, frozen, workers);           \
    if (bad_ >= 0) {                                                                      \
      *err_column = bad_;                                                                 \
      rc = ORC_NUMERIC_ERROR;                                                             \
      goto done;                                                                          \
    }                                                                                     \
    /* primal_values relaxation.hpp:108-123 (all m columns) */                            \
    _Pragma("omp parallel for num_threads(workers) schedule(static)")                     \
    for (int b = 0; b < m; ++b) {                                                         \
      const int t_ = omp_get_thread_num();                                                \
      double loss_ = 0.0;                                                                 \
      const double* s_ = w.S + (size_t)b * n;                                             \
      for (int i = 0; i < n; ++i) loss_ += orc_loss_value(loss, s_[i], y[i]);             \
      const double g_ = g_value_ws(w.B + (size_t)b * p, state + (size_t)b * p, p,        \
                                   kbar[b], M, w.kv[t_], w.dscr[t_]);                     \
      w.primal[b] = loss_ + 2.0 * lambda2 * g_;                                           \
    }                                                                                     \
    /* dual_bounds relaxation.hpp:127-147: Q = X'(-R)/(2 lambda2) */                      \
    gemm_tn(X, n, p, w.R, m, w.Q, workers);                                               \
    _Pragma("omp parallel for num_threads(workers) schedule(static)")                     \
    for (int b = 0; b < m; ++b) {                                                         \
      const int t_ = omp_get_thread_num();                                                \
      double* q_ = w.Q + (size_t)b * p;                                                   \
      for (int j = 0; j < p; ++j) q_[j] = -q_[j] * inv2l;                                 \
      double conj_ = 0.0;                                                                 \
      const double* r_ = w.R + (size_t)b * n;                                             \
      for (int i = 0; i < n; ++i) conj_ += orc_loss_conjugate(loss, r_[i], y[i]);         \
      const double gc_ = g_conjugate_ws(q_, state + (size_t)b * p, p, kbar[b], M,         \
                                        w.dscr[t_]);                                      \
      w.dual[b] = -conj_ - 2.0 * lambda2 * gc_;                                           \
    }                                                                                     \
    for (int b = 0; b < m; ++b) {                                                         \
      if (frozen[b]) continue;                                                            \
      const double psi_ = w.dual[b];                                                      \
      const double phi_ = w.primal[b];                                                    \
      if (psi_ > best_dual[b]) best_dual[b] = psi_;                                       \
      if (trace) trace(user, b, psi_);                                                    \
      const double gap_ = (phi_ - best_dual[b]) / fmax(1.0, fabs(phi_));                  \
      if (best_dual[b] >= prune_threshold) {                                              \
        frozen[b] = 1;                                                                    \
        status[b] = ORC_PRUNABLE;                                                         \
        iters[b] = (ITER);                                                                \
        --active;                                                                         \
      } else if (gap_ <= cfg->gap_tolerance) {                                            \
        frozen[b] = 1;                                                                    \
        status[b] = ORC_CONVERGED;                                                        \
        iters[b] = (ITER);                                                                \
        --active;                                                                         \
      } else if (cfg->acceleration && phi_ - psi_ > last_gap[b]) {                        \
        momentum[b] = 1.0;                                                                \
        memcpy(w.V + (size_t)b * p, w.B + (size_t)b * p, sizeof(double) * p);             \
      }                                                                                   \
      last_gap[b] = phi_ - psi_;                                                          \
    }                                                                                     \
  } while (0)

  int iter = 0, last_eval = 0;
  while (iter < cfg->max_iterations && active > 0) { /* relaxation.hpp:224-249 */
    ++iter;
    int bad = refresh_predictions(w.V, X, y, n, p, loss, &w, frozen, workers);
    if (bad >= 0) {
      *err_column = bad;
      rc = ORC_NUMERIC_ERROR;
      goto done;
    }
    gemm_tn(X, n, p, w.R, m, w.G, workers); /* batched_gradient :102 */
#pragma omp parallel for num_threads(workers) schedule(static)
    for (int b = 0; b < m; ++b) {
      if (frozen[b]) continue;
      const int t = omp_get_thread_num();
      double* dscr = w.dscr[t];
      double* U = dscr + 2 * (p + 1);
      const double* Vb = w.V + (size_t)b * p;
      const double* Gb = w.G + (size_t)b * p;
      for (int j = 0; j < p; ++j) U[j] = Vb[j] - eta * Gb[j];
      double* Bn = w.Bnext + (size_t)b * p;
      prox_step_ws(U, state + (size_t)b * p, p, kbar[b], rho, M, Bn, w.kv[t], dscr);
      double* Bb = w.B + (size_t)b * p;
      double* Vw = w.V + (size_t)b * p;
      if (cfg->acceleration) {
        const double tm = momentum[b];
        const double t_next = 0.5 * (1.0 + sqrt(1.0 + 4.0 * tm * tm));
        const double coef = (tm - 1.0) / t_next;
        for (int j = 0; j < p; ++j) Vw[j] = Bn[j] + coef * (Bn[j] - Bb[j]);
        momentum[b] = t_next;
      } else {
        for (int j = 0; j < p; ++j) Vw[j] = Bn[j];
      }
      memcpy(Bb, Bn, sizeof(double) * p);
    }
    if (iter % cfg->check_interval == 0) {
      EVALUATE(iter);
      last_eval = iter;
    }
  }
  if (active > 0 && last_eval != iter) EVALUATE(iter);
#undef EVALUATE

  memcpy(beta, w.B, sizeof(double) * (size_t)p * m);
  for (int b = 0; b < m; ++b) bounds[b] = best_dual[b];
done:
  free(frozen);
  free(momentum);
  free(best_dual);
  free(last_gap);
  ws_free(&w);
  return rc;
}

/* ======================================================================= */
/* primal_heuristics.hpp:134-227                                           */
/* ======================================================================= */
int orc_round_support(const double* beta, const uint8_t* st, int p, const int* fixed_one,
                      int n_one, int kbar, int* support_out) { /* :134-146 */
  int len = 0;
  for (int t = 0; t < n_one; ++t) support_out[len++] = fixed_one[t];
  if (kbar > 0) {
    keyed_t* kv = (keyed_t*)malloc(sizeof(keyed_t) * 2 * (p + 1));
    const int pf = sorted_free(beta, st, p, kv, kv + p + 1);
    const int take = kbar < pf ? kbar : pf;
    for (int r = 0; r < take; ++r) support_out[len++] = kv[r].idx;
    free(kv);
  }
  return len;
}

int orc_select_branch(const double* beta, const uint8_t* st, int p) { /* :148-163 */
  int best = -1;
  double best_mag = -1.0;
  for (int j = 0; j < p; ++j) {
    if (st[j] != ORC_FREE) continue;
    const double mag = fabs(beta[j]);
    if (mag > best_mag) {
      best_mag = mag;
      best = j;
    }
  }
  return best;
}

void orc_reoptimize(const double* X, const double* y, int n, int p, int loss, double M,
                    double lambda2, double smoothness, int nsup, const int* offsets,
                    const int* idx, int workers, double* coef_out, double* obj_out) {
  double lips = smoothness; /* :178-180 */
  if (!(lips > 0.0)) lips = orc_smoothness(loss, X, n, p);
  const double step = 1.0 / (lips + 2.0 * lambda2);
  if (workers < 1) workers = 1;
#pragma omp parallel num_threads(workers)
  {
    double* scores = (double*)malloc(sizeof(double) * n);
    double* deriv = (double*)malloc(sizeof(double) * n);
    double* probs = (double*)malloc(sizeof(double) * n);
    double* bt = (double*)malloc(sizeof(double) * (p + 1));
    double* grad = (double*)malloc(sizeof(double) * (p + 1));
    double* next = (double*)malloc(sizeof(double) * (p + 1));
#pragma omp for schedule(static)
    for (int b = 0; b < nsup; ++b) { /* :186-225 */
      const int* S = idx + offsets[b];
      const int q = offsets[b + 1] - offsets[b];
      for (int r = 0; r < q; ++r) bt[r] = 0.0;
#define COMPUTE_SCORES()                                              \
  do {                                                                \
    for (int i = 0; i < n; ++i) scores[i] = 0.0;                      \
    for (int r = 0; r < q; ++r) {                                     \
      const double br = bt[r];                                        \
      const double* col = X + (size_t)S[r] * n;                       \
      for (int i = 0; i < n; ++i) scores[i] += br * col[i];           \
    }                                                                 \
  } while (0)
      if (q > 0) {
        for (int it = 0; it < 5000; ++it) {
          COMPUTE_SCORES();
          if (loss == ORC_LOGISTIC) {
            for (int i = 0; i < n; ++i) probs[i] = sigmoid(-y[i] * scores[i]);
            for (int i = 0; i < n; ++i) deriv[i] = -y[i] * probs[i];
          } else {
            for (int i = 0; i < n; ++i) deriv[i] = scores[i] - y[i];
          }
          for (int r = 0; r < q; ++r) {
            const double* col = X + (size_t)S[r] * n;
            double d = 0.0;
            for (int i = 0; i < n; ++i) d += col[i] * deriv[i];
            grad[r] = d + 2.0 * lambda2 * bt[r];
          }
          double gm2 = 0.0;
          for (int r = 0; r < q; ++r) {
            double v = bt[r] - step * grad[r];
            v = v < -M ? -M : v; /* cwiseMax(-M) */
            v = v > M ? M : v;   /* cwiseMin(M) */
            next[r] = v;
            const double dlt = bt[r] - v;
            gm2 += dlt * dlt;
          }
          const double gm = sqrt(gm2) / step;
          for (int r = 0; r < q; ++r) bt[r] = next[r];
          if (gm <= 1e-8) break;
        }
        COMPUTE_SCORES();
      } else {
        for (int i = 0; i < n; ++i) scores[i] = 0.0;
      }
#undef COMPUTE_SCORES
      double sq = 0.0;
      for (int r = 0; r < q; ++r) sq += bt[r] * bt[r];
      double obj = lambda2 * sq;
      for (int i = 0; i < n; ++i) obj += orc_loss_value(loss, scores[i], y[i]);
      for (int r = 0; r < q; ++r) coef_out[offsets[b] + r] = bt[r];
      obj_out[b] = obj;
    }
    free(scores);
    free(deriv);
    free(probs);
    free(bt);
    free(grad);
    free(next);
  }
}

/* ======================================================================= */
/* node_model.hpp:20-172                                                   */
/* ======================================================================= */
typedef struct {
  int n0, n1;
  int* j0; /* capacity p */
  int* j1; /* capacity p */
  double* warm;
  double lb;
  int depth;
} node_t;

static node_t* node_new(int p) {
  node_t* nd = (node_t*)malloc(sizeof(node_t));
  nd->n0 = nd->n1 = 0;
  nd->j0 = (int*)malloc(sizeof(int) * p);
  nd->j1 = (int*)malloc(sizeof(int) * p);
  nd->warm = (double*)calloc(p, sizeof(double));
  nd->lb = -INF;
  nd->depth = 0;
  return nd;
}
static void node_free(node_t* nd) {
  if (!nd) return;
  free(nd->j0);
  free(nd->j1);
  free(nd->warm);
  free(nd);
}
static node_t* node_copy(const node_t* src, int p) {
  node_t* nd = node_new(p);
  nd->n0 = src->n0;
  nd->n1 = src->n1;
  memcpy(nd->j0, src->j0, sizeof(int) * src->n0);
  memcpy(nd->j1, src->j1, sizeof(int) * src->n1);
  memcpy(nd->warm, src->warm, sizeof(double) * p);
  nd->lb = src->lb;
  nd->depth = src->depth;
  return nd;
}
static void node_states(const node_t* nd, int p, uint8_t* st) { /* node_model.hpp:40-45 */
  memset(st, ORC_FREE, p);
  for (int t = 0; t < nd->n0; ++t) st[nd->j0[t]] = ORC_ZERO;
  for (int t = 0; t < nd->n1; ++t) st[nd->j1[t]] = ORC_ONE;
}
static int node_is_leaf(const node_t* nd, int k, int p) { /* node_model.hpp:33-36 */
  return k - nd->n1 <= 0 || nd->n0 + nd->n1 >= p;
}
static void restore_budget(node_t* nd, int k, double M, int p, uint8_t* st) {
  /* node_model.hpp:57-68 */
  const int kb = k - nd->n1;
  node_states(nd, p, st);
  double sum = 0.0;
  for (int j = 0; j < p; ++j)
    if (st[j] == ORC_FREE) sum += fabs(nd->warm[j]);
  const double budget = (double)kb * M;
  if (sum <= budget) return;
  const double scale = budget / sum * (1.0 - 1e-12);
  for (int j = 0; j < p; ++j)
    if (st[j] == ORC_FREE) nd->warm[j] *= scale;
}
/* node_model.hpp:77-105 */
static void branch_node(const node_t* nd, int j, const double* beta, int k, double M, int p,
                        uint8_t* st, uint8_t* st2, node_t** c0, node_t** c1) {
  node_states(nd, p, st);
  node_t* a = node_copy(nd, p);
  a->j0[a->n0++] = j;
  memcpy(a->warm, beta, sizeof(double) * p);
  a->warm[j] = 0.0;
  a->depth = nd->depth + 1;
  restore_budget(a, k, M, p, st2);
  node_t* b = node_copy(nd, p);
  b->j1[b->n1++] = j;
  memcpy(b->warm, beta, sizeof(double) * p);
  b->depth = nd->depth + 1;
  if (k - b->n1 <= 0) {
    for (int r = 0; r < p; ++r)
      if (r != j && st[r] == ORC_FREE) {
        b->j0[b->n0++] = r;
        b->warm[r] = 0.0;
      }
  }
  restore_budget(b, k, M, p, st2);
  *c0 = a;
  *c1 = b;
}

/* best-bound min-heap keyed (bound, seq): node_model.hpp:114-148 */
typedef struct {
  double bound;
  uint64_t seq;
  node_t* node;
} qentry;
typedef struct {
  qentry* h;
  size_t size, cap;
  uint64_t next_seq;
} nqueue;
static int qe_less(const qentry* a, const qentry* b) {
  if (a->bound != b->bound) return a->bound < b->bound;
  return a->seq < b->seq;
}
static void q_push(nqueue* q, node_t* nd) {
  if (q->size == q->cap) {
    q->cap = q->cap ? q->cap * 2 : 64;
    q->h = (qentry*)realloc(q->h, sizeof(qentry) * q->cap);
  }
  size_t i = q->size++;
  qentry e = {nd->lb, q->next_seq++, nd};
  while (i > 0) {
    size_t par = (i - 1) / 2;
    if (!qe_less(&e, &q->h[par])) break;
    q->h[i] = q->h[par];
    i = par;
  }
  q->h[i] = e;
}
static node_t* q_pop(nqueue* q) {
  node_t* top = q->h[0].node;
  qentry last = q->h[--q->size];
  size_t i = 0;
  for (;;) {
    size_t l = 2 * i + 1, r = l + 1, best = i;
    const qentry* cand = &last;
    if (l < q->size && qe_less(&q->h[l], cand)) {
      best = l;
      cand = &q->h[l];
    }
    if (r < q->size && qe_less(&q->h[r], cand)) best = r;
    if (best == i) break;
    q->h[i] = q->h[best];
    i = best;
  }
  if (q->size > 0) q->h[i] = last;
  return top;
}
static double q_global_lb(const nqueue* q) { return q->size ? q->h[0].bound : INF; }

/* ======================================================================= */
/* bnb_engine.hpp:28-309, rashomon.hpp:149-218                             */
/* ======================================================================= */
void orc_solver_cfg_default(orc_solver_cfg* c) { /* bnb_engine.hpp:28-36 */
  c->batch_size = 0;
  c->memory_budget = (uint64_t)1 << 30;
  c->time_limit = INF;
  c->prune_slack = 1e-6;
  orc_relax_cfg_default(&c->relax);
  c->workers = 1;
}

int orc_auto_batch_size(uint64_t memory_budget, int n, int p, int k, int loss) {
  if (memory_budget == 0) return -1; /* bnb_engine.hpp:75-88 */
  const double lb_bytes = 8.0 * 5.0 * p;
  const double loss_arrays = loss == ORC_LOGISTIC ? 3.0 : 2.0;
  const double reopt_bytes = 8.0 * (loss_arrays * n + 2.0 * k);
  const double capacity = 0.9 * (double)memory_budget / (lb_bytes + reopt_bytes);
  if (capacity < 2.0) return 1;
  int size = 1;
  while (2.0 * size <= capacity && size < (1 << 29)) size <<= 1;
  return size;
}

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

/* ---- Rashomon staging (rashomon.hpp:156-196) --------------------------- */
typedef struct {
  int len;
  int* seq;
  double* coef;
  double objective;
  int* key; /* sorted */
} staged_t;

struct orc_pool {
  int count;
  staged_t* rec;
};

typedef struct {
  int kind; /* 0 solve, 1 rashomon */
  double delta;
  double eps;
  long long cap;
  /* rashomon */
  staged_t* staged;
  int nstaged, capstaged;
  int* hash; /* open addressing into staged, -1 empty */
  int hcap;
  double* heap; /* max-heap of best objectives */
  long long heapn;
  double best_objective;
} policy_t;

static double nth_best(const policy_t* pol) {
  if (pol->cap < 0) return INF;
  if (pol->heapn < pol->cap) return INF;
  return pol->heap[0];
}

static double policy_threshold(const policy_t* pol, double ub) {
  if (pol->kind == 0) { /* bnb_engine.hpp:304-307 */
    if (!isfinite(ub)) return INF;
    return ub - pol->delta * fmax(1.0, fabs(ub));
  }
  /* rashomon.hpp:169-174 */
  double tau = isfinite(ub) ? (1.0 + pol->eps) * ub : INF;
  const double nb = nth_best(pol);
  if (nb < tau) tau = nb;
  return nextafter(tau, INF);
}

static uint64_t key_hash(const int* key, int len) {
  uint64_t h = 1469598103934665603ULL;
  for (int t = 0; t < len; ++t) {
    h ^= (uint64_t)(uint32_t)key[t];
    h *= 1099511628211ULL;
  }
  h ^= (uint64_t)len;
  return h;
}

static int cmp_int(const void* a, const void* b) {
  const int x = *(const int*)a, y = *(const int*)b;
  return (x > y) - (x < y);
}

static void heap_push_max(double* h, long long* n, double v) {
  long long i = (*n)++;
  while (i > 0) {
    long long par = (i - 1) / 2;
    if (h[par] >= v) break;
    h[i] = h[par];
    i = par;
  }
  h[i] = v;
}
static void heap_pop_max(double* h, long long* n) {
  double last = h[--(*n)];
  long long i = 0;
  for (;;) {
    long long l = 2 * i + 1, r = l + 1, best = i;
    double bv = last;
    if (l < *n && h[l] > bv) {
      best = l;
      bv = h[l];
    }
    if (r < *n && h[r] > bv) best = r;
    if (best == i) break;
    h[i] = h[best];
    i = best;
  }
  if (*n > 0) h[i] = last;
}

static void policy_on_model(policy_t* pol, const int* seq, int len, const double* coef,
                            double objective) { /* rashomon.hpp:175-196 */
  if (pol->kind != 1) return;
  if (objective < pol->best_objective) pol->best_objective = objective;
  const double nb = nth_best(pol);
  const double base = (1.0 + pol->eps) * pol->best_objective;
  const double tau_now = (nb < base ? nb : base) + 1e-9;
  if (objective > tau_now) return;
  int* key = (int*)malloc(sizeof(int) * (len + 1));
  memcpy(key, seq, sizeof(int) * len);
  qsort(key, len, sizeof(int), cmp_int);
  if (pol->hcap == 0 || 2 * (pol->nstaged + 1) > pol->hcap) { /* rehash */
    int ncap = pol->hcap ? pol->hcap * 2 : 1024;
    int* nh = (int*)malloc(sizeof(int) * ncap);
    for (int t = 0; t < ncap; ++t) nh[t] = -1;
    for (int s = 0; s < pol->nstaged; ++s) {
      uint64_t h = key_hash(pol->staged[s].key, pol->staged[s].len) & (ncap - 1);
      while (nh[h] >= 0) h = (h + 1) & (ncap - 1);
      nh[h] = s;
    }
    free(pol->hash);
    pol->hash = nh;
    pol->hcap = ncap;
  }
  uint64_t h = key_hash(key, len) & (pol->hcap - 1);
  while (pol->hash[h] >= 0) {
    const staged_t* s = &pol->staged[pol->hash[h]];
    if (s->len == len && memcmp(s->key, key, sizeof(int) * len) == 0) {
      free(key);
      return;
    }
    h = (h + 1) & (pol->hcap - 1);
  }
  if (pol->nstaged == pol->capstaged) {
    pol->capstaged = pol->capstaged ? pol->capstaged * 2 : 256;
    pol->staged = (staged_t*)realloc(pol->staged, sizeof(staged_t) * pol->capstaged);
  }
  staged_t* s = &pol->staged[pol->nstaged];
  s->len = len;
  s->seq = (int*)malloc(sizeof(int) * (len + 1));
  memcpy(s->seq, seq, sizeof(int) * len);
  s->coef = (double*)malloc(sizeof(double) * (len + 1));
  memcpy(s->coef, coef, sizeof(double) * len);
  s->objective = objective;
  s->key = key;
  pol->hash[h] = pol->nstaged++;
  if (pol->cap >= 0) {
    if (pol->heapn < pol->cap) {
      pol->heap = (double*)realloc(pol->heap, sizeof(double) * (pol->heapn + 1));
      heap_push_max(pol->heap, &pol->heapn, objective);
    } else if (pol->heapn > 0 && objective < pol->heap[0]) {
      heap_pop_max(pol->heap, &pol->heapn);
      heap_push_max(pol->heap, &pol->heapn, objective);
    }
  }
}

/* DebugHooks::on_dual_bound wiring (bnb_engine.hpp:182-187) */
typedef struct {
  orc_dual_hook fn;
  void* user;
  node_t** nodes;
} trace_ctx;
static void trace_tramp(void* u, int b, double psi) {
  trace_ctx* c = (trace_ctx*)u;
  const node_t* nd = c->nodes[b];
  c->fn(c->user, nd->n0, nd->j0, nd->n1, nd->j1, psi);
}

/* bnb_engine.hpp:116-291 run_bnb */
static int run_bnb(const double* X, const double* y, int n, int p, int loss, int k, double M,
                   double lambda2, const orc_solver_cfg* cfg, policy_t* pol,
                   orc_certificate* cert, orc_dual_hook on_dual, orc_boundary_hook on_boundary,
                   void* user) {
  if (orc_validate(X, y, n, p, loss, k, M, lambda2) != ORC_OK) return ORC_INPUT_ERROR;
  const double wall_start = now_s();
  cert->optimal_value = INF;
  cert->support_len = 0;
  cert->gap_percent = 0.0;
  cert->lower_bound = -INF;
  cert->nodes_processed = cert->lb_batches = cert->reopt_batches = 0;
  cert->prof_lower_bound = cert->prof_reoptimization = cert->prof_transfer = 0.0;
  cert->prof_branch_generate = cert->prof_total = 0.0;
  cert->status = 0;
  cert->err_column = -1;
  const int workers = cfg->workers < 1 ? 1 : cfg->workers;
  orc_relax_cfg rcfg = cfg->relax;
  rcfg.workers = workers;
  {
    const double t0 = now_s();
    if (!(rcfg.smoothness > 0.0)) rcfg.smoothness = orc_smoothness(loss, X, n, p);
    cert->prof_lower_bound += now_s() - t0;
  }
  const int batch_size =
      cfg->batch_size > 0 ? cfg->batch_size
                          : orc_auto_batch_size(cfg->memory_budget, n, p, k, loss);
  cert->batch_size_used = batch_size;

  nqueue queue = {NULL, 0, 0, 0};
  q_push(&queue, node_new(p));
  node_t** pending = NULL;
  size_t npending = 0, cappending = 0;
  double inc_obj = INF;
  int* inc_sup = (int*)malloc(sizeof(int) * (k + 1));
  double* inc_coef = (double*)malloc(sizeof(double) * (k + 1));
  int inc_len = 0;
  int status = 0;
  int rc = ORC_OK;

  node_t** relax_nodes = (node_t**)malloc(sizeof(node_t*) * (size_t)batch_size);
  node_t** leaves = NULL;
  size_t capleaves = 0;
  uint8_t* st = (uint8_t*)malloc(p);
  uint8_t* st2 = (uint8_t*)malloc(p);

  while (queue.size > 0 || npending > 0) {
    if (now_s() - wall_start > cfg->time_limit) {
      status = 1;
      break;
    }
    const double threshold = policy_threshold(pol, inc_obj);
    int nrelax = 0;
    size_t nleaves = 0;
    {
      const double t0 = now_s();
      /* assemble_batch node_model.hpp:158-172 */
      int popped = 0, discarded = 0;
      node_t** batch = (node_t**)malloc(sizeof(node_t*) * (size_t)batch_size);
      while (queue.size > 0 && popped < batch_size) {
        node_t* nd = q_pop(&queue);
        if (nd->lb >= threshold) {
          ++discarded;
          node_free(nd);
          continue;
        }
        batch[popped++] = nd;
      }
      cert->nodes_processed += popped + discarded;
      if (capleaves < npending + popped) {
        capleaves = npending + popped + 16;
        leaves = (node_t**)realloc(leaves, sizeof(node_t*) * capleaves);
      }
      for (size_t t = 0; t < npending; ++t) {
        ++cert->nodes_processed;
        if (pending[t]->lb >= threshold) {
          node_free(pending[t]);
          continue;
        }
        leaves[nleaves++] = pending[t];
      }
      npending = 0;
      for (int t = 0; t < popped; ++t) {
        if (node_is_leaf(batch[t], k, p))
          leaves[nleaves++] = batch[t];
        else
          relax_nodes[nrelax++] = batch[t];
      }
      free(batch);
      cert->prof_transfer += now_s() - t0;
    }
    if (nrelax == 0 && nleaves == 0) continue;

    double* beta = NULL;
    double* bounds = NULL;
    int* rstatus = NULL;
    int* riters = NULL;
    if (nrelax > 0) {
      const double t0 = now_s();
      uint8_t* state = (uint8_t*)malloc((size_t)p * nrelax);
      int* kb = (int*)malloc(sizeof(int) * nrelax);
      double* warm = (double*)malloc(sizeof(double) * (size_t)p * nrelax);
      beta = (double*)malloc(sizeof(double) * (size_t)p * nrelax);
      bounds = (double*)malloc(sizeof(double) * nrelax);
      rstatus = (int*)malloc(sizeof(int) * nrelax);
      riters = (int*)malloc(sizeof(int) * nrelax);
      for (int b = 0; b < nrelax; ++b) { /* BatchMeta::from_nodes prox_kernel.hpp:52-90 */
        node_states(relax_nodes[b], p, state + (size_t)b * p);
        const int kk = k - relax_nodes[b]->n1;
        kb[b] = kk > 0 ? kk : 0;
        memcpy(warm + (size_t)b * p, relax_nodes[b]->warm, sizeof(double) * p);
      }
      trace_ctx tctx = {on_dual, user, relax_nodes};
      int errc = -1;
      rc = orc_relax_batch(X, y, n, p, loss, M, lambda2, &rcfg, threshold, nrelax, state, kb,
                           warm, beta, bounds, rstatus, riters, on_dual ? trace_tramp : NULL,
                           &tctx, &errc);
      free(state);
      free(kb);
      free(warm);
      ++cert->lb_batches;
      cert->prof_lower_bound += now_s() - t0;
      if (rc != ORC_OK) {
        cert->err_column = errc;
        goto cleanup_pass;
      }
    }
    {
      /* one re-optimization batch: leaves then rounded columns (:193-212) */
      const double t0 = now_s();
      const int nsup_max = (int)nleaves + nrelax;
      int* offsets = (int*)malloc(sizeof(int) * (nsup_max + 1));
      int* sidx = (int*)malloc(sizeof(int) * ((size_t)nsup_max * k + 1));
      double* coef = (double*)malloc(sizeof(double) * ((size_t)nsup_max * k + 1));
      double* obj = (double*)malloc(sizeof(double) * (nsup_max + 1));
      int nsup = 0;
      offsets[0] = 0;
      for (size_t t = 0; t < nleaves; ++t) {
        memcpy(sidx + offsets[nsup], leaves[t]->j1, sizeof(int) * leaves[t]->n1);
        offsets[nsup + 1] = offsets[nsup] + leaves[t]->n1;
        ++nsup;
      }
      for (int b = 0; b < nrelax; ++b) {
        if (rstatus[b] == ORC_PRUNABLE) continue;
        node_states(relax_nodes[b], p, st);
        const int kk = k - relax_nodes[b]->n1;
        const int len = orc_round_support(beta + (size_t)b * p, st, p, relax_nodes[b]->j1,
                                          relax_nodes[b]->n1, kk, sidx + offsets[nsup]);
        offsets[nsup + 1] = offsets[nsup] + len;
        ++nsup;
      }
      if (nsup > 0) {
        orc_reoptimize(X, y, n, p, loss, M, lambda2, rcfg.smoothness, nsup, offsets, sidx,
                       workers, coef, obj);
        ++cert->reopt_batches;
      }
      cert->prof_reoptimization += now_s() - t0;

      const double t1 = now_s();
      for (int s = 0; s < nsup; ++s) { /* bnb_engine.hpp:216-240 */
        const int len = offsets[s + 1] - offsets[s];
        policy_on_model(pol, sidx + offsets[s], len, coef + offsets[s], obj[s]);
        if (obj[s] < inc_obj) {
          inc_obj = obj[s];
          inc_len = len;
          /* stored sorted with coefficients aligned */
          for (int t = 0; t < len; ++t) {
            inc_sup[t] = sidx[offsets[s] + t];
            inc_coef[t] = coef[offsets[s] + t];
          }
          for (int a = 1; a < len; ++a) { /* insertion sort by index */
            int ks = inc_sup[a];
            double kc = inc_coef[a];
            int b2 = a - 1;
            while (b2 >= 0 && inc_sup[b2] > ks) {
              inc_sup[b2 + 1] = inc_sup[b2];
              inc_coef[b2 + 1] = inc_coef[b2];
              --b2;
            }
            inc_sup[b2 + 1] = ks;
            inc_coef[b2 + 1] = kc;
          }
        }
      }
      free(offsets);
      free(sidx);
      free(coef);
      free(obj);
      for (size_t t = 0; t < nleaves; ++t) node_free(leaves[t]);
      nleaves = 0;

      const double post_threshold = policy_threshold(pol, inc_obj);
      for (int b = 0; b < nrelax; ++b) { /* :243-256 */
        node_t* nd = relax_nodes[b];
        if (rstatus[b] == ORC_PRUNABLE) continue;
        if (bounds[b] > nd->lb) nd->lb = bounds[b];
        if (nd->lb >= post_threshold) continue;
        node_states(nd, p, st);
        const int j = orc_select_branch(beta + (size_t)b * p, st, p);
        if (j < 0) {
          rc = ORC_LOGIC_ERROR;
          goto cleanup_pass;
        }
        node_t *c0, *c1;
        branch_node(nd, j, beta + (size_t)b * p, k, M, p, st, st2, &c0, &c1);
        node_t* ch[2] = {c0, c1};
        for (int t = 0; t < 2; ++t) {
          if (node_is_leaf(ch[t], k, p)) {
            if (npending == cappending) {
              cappending = cappending ? cappending * 2 : 64;
              pending = (node_t**)realloc(pending, sizeof(node_t*) * cappending);
            }
            pending[npending++] = ch[t];
          } else {
            q_push(&queue, ch[t]);
          }
        }
      }
      cert->prof_branch_generate += now_s() - t1;
    }
    if (on_boundary) { /* :259-265 */
      double lb = q_global_lb(&queue);
      for (size_t t = 0; t < npending; ++t)
        if (pending[t]->lb < lb) lb = pending[t]->lb;
      on_boundary(user, lb < inc_obj ? lb : inc_obj, inc_obj);
    }
  cleanup_pass:
    for (int b = 0; b < nrelax; ++b) node_free(relax_nodes[b]);
    for (size_t t = 0; t < nleaves; ++t) node_free(leaves[t]);
    free(beta);
    free(bounds);
    free(rstatus);
    free(riters);
    if (rc != ORC_OK) break;
  }

  { /* certificate :268-290 */
    const double ub = inc_obj;
    cert->status = status;
    cert->optimal_value = ub;
    cert->support_len = inc_len;
    for (int t = 0; t < inc_len; ++t) {
      cert->support[t] = inc_sup[t];
      cert->coefficients[t] = inc_coef[t];
    }
    if (status == 0) {
      cert->lower_bound = ub;
      cert->gap_percent = 0.0;
    } else {
      double lb = q_global_lb(&queue);
      for (size_t t = 0; t < npending; ++t)
        if (pending[t]->lb < lb) lb = pending[t]->lb;
      if (ub < lb) lb = ub;
      cert->lower_bound = lb;
      cert->gap_percent = !isfinite(ub) ? 100.0 : 100.0 * (ub - lb) / fmax(fabs(ub), 1e-12);
    }
    cert->prof_total = now_s() - wall_start;
  }
  while (queue.size > 0) node_free(q_pop(&queue));
  free(queue.h);
  for (size_t t = 0; t < npending; ++t) node_free(pending[t]);
  free(pending);
  free(leaves);
  free(relax_nodes);
  free(st);
  free(st2);
  free(inc_sup);
  free(inc_coef);
  return rc;
}

int orc_solve(const double* X, const double* y, int n, int p, int loss, int k, double M,
              double lambda2, const orc_solver_cfg* cfg, orc_certificate* cert,
              orc_dual_hook on_dual, orc_boundary_hook on_boundary, void* user) {
  policy_t pol;
  memset(&pol, 0, sizeof(pol));
  pol.kind = 0;
  pol.delta = cfg->prune_slack;
  pol.cap = -1;
  return run_bnb(X, y, n, p, loss, k, M, lambda2, cfg, &pol, cert, on_dual, on_boundary, user);
}

static int cmp_staged(const staged_t* a, const staged_t* b) {
  if (a->objective != b->objective) return a->objective < b->objective ? -1 : 1;
  const int l = a->len < b->len ? a->len : b->len; /* vector lexicographic < */
  for (int t = 0; t < l; ++t)
    if (a->seq[t] != b->seq[t]) return a->seq[t] < b->seq[t] ? -1 : 1;
  return (a->len > b->len) - (a->len < b->len);
}
static const staged_t* g_sort_base;
static int cmp_staged_idx(const void* x, const void* y) {
  return cmp_staged(&g_sort_base[*(const int*)x], &g_sort_base[*(const int*)y]);
}

int orc_collect_rashomon(const double* X, const double* y, int n, int p, int loss, int k,
                         double M, double lambda2, const orc_solver_cfg* cfg, double epsilon,
                         long long cap, orc_certificate* cert, orc_pool** pool_out) {
  if (epsilon < 0.0) return ORC_INPUT_ERROR; /* rashomon.hpp:152-153 */
  policy_t pol;
  memset(&pol, 0, sizeof(pol));
  pol.kind = 1;
  pol.eps = epsilon;
  pol.cap = cap;
  pol.best_objective = INF;
  int rc = run_bnb(X, y, n, p, loss, k, M, lambda2, cfg, &pol, cert, NULL, NULL, NULL);
  orc_pool* pool = (orc_pool*)calloc(1, sizeof(orc_pool));
  if (rc == ORC_OK) { /* compaction rashomon.hpp:201-216 */
    const double tau_final = (1.0 + epsilon) * cert->optimal_value + 1e-9;
    int* live = (int*)malloc(sizeof(int) * (pol.nstaged + 1));
    int nlive = 0;
    for (int i = 0; i < pol.nstaged; ++i)
      if (pol.staged[i].objective <= tau_final) live[nlive++] = i;
    g_sort_base = pol.staged;
    qsort(live, nlive, sizeof(int), cmp_staged_idx);
    if (cap >= 0 && nlive > cap) nlive = (int)cap;
    pool->count = nlive;
    pool->rec = (staged_t*)malloc(sizeof(staged_t) * (nlive + 1));
    for (int t = 0; t < nlive; ++t) {
      pool->rec[t] = pol.staged[live[t]];
      pol.staged[live[t]].seq = NULL; /* ownership moved */
      pol.staged[live[t]].coef = NULL;
      pol.staged[live[t]].key = NULL;
    }
    free(live);
  }
  for (int i = 0; i < pol.nstaged; ++i) {
    free(pol.staged[i].seq);
    free(pol.staged[i].coef);
    free(pol.staged[i].key);
  }
  free(pol.staged);
  free(pol.hash);
  free(pol.heap);
  *pool_out = pool;
  return rc;
}

int orc_pool_size(const orc_pool* pool) { return pool ? pool->count : 0; }
int orc_pool_record(const orc_pool* pool, int i, int* seq_out, double* coef_out,
                    double* objective_out) {
  const staged_t* s = &pool->rec[i];
  memcpy(seq_out, s->seq, sizeof(int) * s->len);
  memcpy(coef_out, s->coef, sizeof(double) * s->len);
  *objective_out = s->objective;
  return s->len;
}
void orc_pool_free(orc_pool* pool) {
  if (!pool) return;
  for (int t = 0; t < pool->count; ++t) {
    free(pool->rec[t].seq);
    free(pool->rec[t].coef);
    free(pool->rec[t].key);
  }
  free(pool->rec);
  free(pool);
}
