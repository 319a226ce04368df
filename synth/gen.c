/* synth/gen.c -- seeded synthetic user/item-set generator.
 *
 * This module is shared test/bench infrastructure: it produces the input CSR
 * (offsets[n+1], items[nnz], int32, rows strictly ascending) that BOTH the CPU
 * oracle (oracle/) and the CUDA path consume.  It holds none of the method's
 * arithmetic (no item hash, no FastRandomHash, no Jaccard): only a counter-based
 * RNG, a profile-size distribution and a Zipf item-popularity sampler.
 *
 * Recipe:
 *   size(u)  = lognormal(median, sigma) rounded, clipped [lo, hi]      (dist 0)
 *            | bounded Pareto on [lo, hi], alpha fitted to a mean, floor (dist 1)
 *   draw j of user u: x = mix64(seed, u, j); rank = min r with x < T[r],
 *            T[r] = floor(2^64 * sum_{j<=r} (j+1)^-s / Z);  item = perm[rank]
 *   duplicates rejected until size(u) distinct items; row sorted ascending.
 *   perm = Fisher-Yates permutation of [0,m) seeded from (seed ^ PERM_SALT), so
 *   popularity does not correlate with item id.
 * Everything after the one-time table build is integer, so the output is a pure
 * function of the parameters and independent of the thread count.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define SIZE_SALT 0x5a17e5eedULL
#define PERM_SALT 0x9e3779b97f4a7c15ULL

static inline uint64_t fmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
static inline uint64_t mix64(uint64_t seed, uint64_t u, uint64_t j) {
  return fmix64(fmix64(fmix64(seed) ^ u) ^ j);
}
static inline double u01(uint64_t x) { return (double)(x >> 11) * (1.0 / 9007199254740992.0); }

/* Inverse standard normal CDF: Acklam's rational approximation + one Halley step. */
static double norm_ppf(double p) {
  static const double a[] = {-3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,
                             1.383577518672690e+02, -3.066479806614716e+01, 2.506628277459239e+00};
  static const double b[] = {-5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,
                             6.680131188771972e+01, -1.328068155288572e+01};
  static const double c[] = {-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00,
                             -2.549732539343734e+00, 4.374664141464968e+00, 2.938163982698783e+00};
  static const double d[] = {7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00,
                             3.754408661907416e+00};
  if (p <= 0) p = 1e-300;
  if (p >= 1) p = 1 - 1e-16;
  double q, r, x;
  if (p < 0.02425) {
    q = sqrt(-2 * log(p));
    x = (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
        ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1);
  } else if (p > 1 - 0.02425) {
    q = sqrt(-2 * log(1 - p));
    x = -(((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
        ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1);
  } else {
    q = p - 0.5;
    r = q * q;
    x = (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * q /
        (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1);
  }
  double e = 0.5 * erfc(-x / sqrt(2.0)) - p; /* Halley refinement */
  double uu = e * sqrt(2 * M_PI) * exp(x * x / 2);
  return x - uu / (1 + x * uu / 2);
}

/* Mean of a bounded Pareto(L, H, alpha). */
static double bp_mean(double L, double H, double al) {
  if (fabs(al - 1.0) < 1e-12) return (H * L / (H - L)) * log(H / L);
  double la = pow(L, al);
  return la / (1 - pow(L / H, al)) * (al / (al - 1)) * (1 / pow(L, al - 1) - 1 / pow(H, al - 1));
}
/* alpha such that E[X] - 0.5 = target (the -0.5 accounts for the floor). */
double synth_fit_pareto_alpha(double L, double H, double target) {
  double lo = 1e-3, hi = 20.0;
  for (int it = 0; it < 200; ++it) {
    double mid = 0.5 * (lo + hi);
    if (bp_mean(L, H, mid) - 0.5 > target) lo = mid; else hi = mid; /* mean decreases with alpha */
  }
  return 0.5 * (lo + hi);
}

/* dist 0: lognormal(p1 = median, p2 = sigma); dist 1: bounded Pareto (p1 = alpha). */
int synth_sizes(int64_t n, int dist, double p1, double p2, int lo, int hi, uint64_t seed, int32_t *sizes) {
  if (n < 0 || lo < 1 || hi < lo) return -1;
  for (int64_t u = 0; u < n; ++u) {
    double U = u01(mix64(seed ^ SIZE_SALT, (uint64_t)u, 0));
    double x;
    if (dist == 0) {
      x = floor(p1 * exp(p2 * norm_ppf(U)) + 0.5);
    } else {
      double L = lo, H = hi, al = p1;
      x = floor(L * pow(1 - U * (1 - pow(L / H, al)), -1.0 / al));
    }
    if (x < lo) x = lo;
    if (x > hi) x = hi;
    sizes[u] = (int32_t)x;
  }
  return 0;
}

typedef struct {
  const int32_t *offsets;
  int32_t *items;
  const uint64_t *T;
  const int32_t *perm;
  int64_t m;
  uint64_t seed;
  int64_t u0, u1;
  int status;
} job_t;

static int cmp_i32(const void *a, const void *b) {
  int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  return (x > y) - (x < y);
}

static void *fill_rows(void *arg) {
  job_t *J = (job_t *)arg;
  int64_t nw = (J->m + 63) / 64;
  uint64_t *seen = (uint64_t *)calloc((size_t)nw, 8);
  if (!seen) { J->status = -3; return NULL; }
  for (int64_t u = J->u0; u < J->u1; ++u) {
    int32_t *row = J->items + J->offsets[u];
    int32_t sz = J->offsets[u + 1] - J->offsets[u];
    if (sz > J->m) { J->status = -2; break; }
    int32_t got = 0;
    uint64_t j = 0, cap = 100000000ULL;
    while (got < sz && j < cap) {
      uint64_t x = mix64(J->seed, (uint64_t)u, j++);
      int64_t lo = 0, hi = J->m - 1; /* smallest r with x < T[r] (T[m-1] = UINT64_MAX) */
      while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (x < J->T[mid]) hi = mid; else lo = mid + 1;
      }
      int32_t it = J->perm[lo];
      uint64_t bit = 1ULL << (it & 63);
      if (seen[it >> 6] & bit) continue;
      seen[it >> 6] |= bit;
      row[got++] = it;
    }
    if (got < sz) { J->status = -4; break; }
    for (int32_t q = 0; q < sz; ++q) seen[row[q] >> 6] &= ~(1ULL << (row[q] & 63));
    qsort(row, (size_t)sz, sizeof(int32_t), cmp_i32);
  }
  free(seen);
  return NULL;
}

/* Fill items[offsets[u]..offsets[u+1]) for every user; offsets = exclusive scan of sizes. */
int synth_fill(int64_t n, int64_t m, double zipf_s, uint64_t seed, const int32_t *offsets, int32_t *items,
               int nthreads) {
  if (m < 1 || n < 0) return -1;
  uint64_t *T = (uint64_t *)malloc((size_t)m * 8);
  int32_t *perm = (int32_t *)malloc((size_t)m * 4);
  long double *w = (long double *)malloc((size_t)m * sizeof(long double));
  if (!T || !perm || !w) { free(T); free(perm); free(w); return -3; }
  long double Z = 0;
  for (int64_t r = 0; r < m; ++r) { w[r] = powl((long double)(r + 1), -(long double)zipf_s); Z += w[r]; }
  long double acc = 0;
  for (int64_t r = 0; r < m; ++r) {
    acc += w[r];
    long double v = ldexpl(acc / Z, 64);
    T[r] = (v >= ldexpl(1.0L, 64)) ? UINT64_MAX : (uint64_t)v;
  }
  T[m - 1] = UINT64_MAX;
  free(w);
  for (int64_t i = 0; i < m; ++i) perm[i] = (int32_t)i;
  uint64_t st = seed ^ PERM_SALT;
  for (int64_t i = m - 1; i > 0; --i) {
    st = fmix64(st);
    int64_t j = (int64_t)(st % (uint64_t)(i + 1));
    int32_t tmp = perm[i]; perm[i] = perm[j]; perm[j] = tmp;
  }
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  job_t jobs[256];
  for (int q = 0; q < nthreads; ++q) {
    jobs[q] = (job_t){offsets, items, T, perm, m, seed, n * q / nthreads, n * (q + 1) / nthreads, 0};
    pthread_create(&th[q], NULL, fill_rows, &jobs[q]);
  }
  int status = 0;
  for (int q = 0; q < nthreads; ++q) {
    pthread_join(th[q], NULL);
    if (jobs[q].status) status = jobs[q].status;
  }
  free(T);
  free(perm);
  return status;
}
