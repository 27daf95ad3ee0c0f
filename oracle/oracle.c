/* CPU oracle for the sobench hot path -- TEST INFRASTRUCTURE ONLY.
 *
 * This file restates, in plain C, the arithmetic of the reference package
 * (arXiv 2404.11631 artifact "sobench", /root/reference/pkg/src/sobench) so the
 * CUDA product can be checked bit-for-bit at sizes where the Python reference
 * would be slow.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it.  It is never on the product path.
 *
 * Pinning: every routine here is checked against golden vectors produced by
 * importing the real reference (tests/golden/gen_golden.py) -- see
 * tests/test_oracle.py.
 *
 * Third-party arithmetic the reference delegates (restated here):
 *   - numpy 2.3.5 Philox-4x64-10 bit generator + Generator.random
 *     (call site sobench/sampling.py:74-80, :95-98),
 *   - glibc 2.39 libm log1p/sin/cos/exp/erf through numba
 *     (sobench/_kernels.py:159-223) -- called directly here, exactly as numba does.
 * Build: see oracle/Makefile  (gcc -O2 -ffp-contract=off: no FMA contraction,
 * matching the numba kernels, which contain no vfmadd -- SURVEY.md sec. 0.4).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------- Philox4x64-10 (numpy _philox.h) ---------------- */
static void mulhilo64(uint64_t a, uint64_t b, uint64_t *hi, uint64_t *lo) {
  unsigned __int128 p = (unsigned __int128)a * b;
  *lo = (uint64_t)p;
  *hi = (uint64_t)(p >> 64);
}

static void philox4x64_10(const uint64_t ctr[4], const uint64_t key[2], uint64_t out[4]) {
  uint64_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint64_t k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; ++r) {
    uint64_t hi0, lo0, hi1, lo1;
    mulhilo64(0xD2E7470EE14C6C93ULL, c0, &hi0, &lo0);
    mulhilo64(0xCA5A826395121157ULL, c2, &hi1, &lo1);
    uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B97F4A7C15ULL;
    k1 += 0xBB67AE8584CAA73BULL;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* 256-bit counter increment (numpy philox_next: ++ctr with carry). */
static void ctr_inc(uint64_t c[4]) {
  if (++c[0]) return;
  if (++c[1]) return;
  if (++c[2]) return;
  ++c[3];
}

/* uniform01 (sampling.py:87-102): u[i] = (w >> 11) * 2^-53 where w is word
 * i%4 of numpy Philox's block stream.  The reference fills spans of 65536
 * doubles (SAMPLE_SPAN, sampling.py:46) from a fresh generator whose counter is
 * set to (counter + lo/4) mod 2^128 (RngStream._generator_at masks to two
 * words); numpy then pre-increments the full 256-bit counter before each block. */
void orc_uniform01(uint64_t seed, uint64_t sid, uint64_t ctr_lo, uint64_t ctr_hi,
                   int64_t n, double *out) {
  uint64_t key[2] = {seed, sid}, w[4];
  for (int64_t lo = 0; lo < n; lo += 65536) {
    uint64_t off = (uint64_t)(lo / 4);
    uint64_t c[4];
    c[0] = ctr_lo + off;
    c[1] = ctr_hi + (c[0] < ctr_lo ? 1 : 0);
    c[2] = 0;
    c[3] = 0;
    int64_t hi = lo + 65536 < n ? lo + 65536 : n;
    for (int64_t i = lo; i < hi; i += 4) {
      ctr_inc(c);
      philox4x64_10(c, key, w);
      for (int k = 0; k < 4 && i + k < hi; ++k)
        out[i + k] = (double)(w[k] >> 11) * (1.0 / 9007199254740992.0);
    }
  }
}

void orc_philox_block(const uint64_t ctr[4], const uint64_t key[2], uint64_t out[4]) {
  philox4x64_10(ctr, key, out);
}

/* boxmuller_block (_kernels.py:178-190) over m (even) uniforms. */
void orc_boxmuller(const double *u, double *z, int64_t m) {
  const double TAU = 6.283185307179586;
  for (int64_t p = 0; p < m / 2; ++p) {
    double u1 = u[2 * p], u2 = u[2 * p + 1];
    double r = sqrt(-2.0 * log1p(-u1));
    double th = TAU * u2;
    z[2 * p] = r * cos(th);
    z[2 * p + 1] = r * sin(th);
  }
}

/* standard_normal (sampling.py:105-120): m = 2*ceil(n/2) uniforms, keep n. */
void orc_standard_normal(uint64_t seed, uint64_t sid, uint64_t ctr_lo, uint64_t ctr_hi,
                         int64_t n, double *out) {
  int64_t m = 2 * ((n + 1) / 2);
  double *u = (double *)malloc(sizeof(double) * m);
  double *z = (double *)malloc(sizeof(double) * m);
  orc_uniform01(seed, sid, ctr_lo, ctr_hi, m, u);
  orc_boxmuller(u, z, m);
  memcpy(out, z, sizeof(double) * n);
  free(u);
  free(z);
}

/* ---------------- fixed reduction tree (_kernels.py:1-156) ---------------- */
double orc_fold_pairwise(double *p, int64_t m) {  /* _kernels.py:30-42 */
  if (m == 0) return 0.0;
  while (m > 1) {
    int64_t h = m / 2;
    for (int64_t i = 0; i < h; ++i) p[i] = p[2 * i] + p[2 * i + 1];
    if (m & 1) { p[h] = p[m - 1]; m = h + 1; } else { m = h; }
  }
  return p[0];
}

/* Backend.dot (backend.py:80-96) with strided operands. */
static double dot_strided(const double *x, int64_t sx, const double *y, int64_t sy,
                          int64_t n, int64_t chunk) {
  if (n == 0) return 0.0;
  int64_t nch = (n + chunk - 1) / chunk;
  double *p = (double *)malloc(sizeof(double) * nch);
  for (int64_t c = 0; c < nch; ++c) {
    int64_t lo = c * chunk, hi = lo + chunk < n ? lo + chunk : n;
    double s = 0.0;
    for (int64_t i = lo; i < hi; ++i) s += x[i * sx] * y[i * sy];
    p[c] = s;
  }
  double r = orc_fold_pairwise(p, nch);
  free(p);
  return r;
}

double orc_dot(const double *x, const double *y, int64_t n, int64_t chunk) {
  return dot_strided(x, 1, y, 1, n, chunk);
}

double orc_vec_sum(const double *x, int64_t n, int64_t chunk) {  /* backend.py:98-111 */
  if (n == 0) return 0.0;
  int64_t nch = (n + chunk - 1) / chunk;
  double *p = (double *)malloc(sizeof(double) * nch);
  for (int64_t c = 0; c < nch; ++c) {
    int64_t lo = c * chunk, hi = lo + chunk < n ? lo + chunk : n;
    double s = 0.0;
    for (int64_t i = lo; i < hi; ++i) s += x[i];
    p[c] = s;
  }
  double r = orc_fold_pairwise(p, nch);
  free(p);
  return r;
}

/* matvec_rows (_kernels.py:85-121): row r = fixed-tree dot(a[r], x). */
void orc_matvec(const double *a, int64_t rows, int64_t cols, const double *x, double *out,
                int64_t chunk) {
  for (int64_t r = 0; r < rows; ++r) out[r] = dot_strided(a + r * cols, 1, x, 1, cols, chunk);
}

/* matvec_t_cols (_kernels.py:124-156): column j, row chunks, p[c,j] += x[i]*a[i,j]. */
void orc_matvec_t(const double *a, int64_t rows, int64_t cols, const double *x, double *out,
                  int64_t chunk) {
  for (int64_t j = 0; j < cols; ++j) {
    if (rows == 0) { out[j] = 0.0; continue; }
    int64_t nch = (rows + chunk - 1) / chunk;
    double *p = (double *)malloc(sizeof(double) * nch);
    for (int64_t c = 0; c < nch; ++c) {
      int64_t lo = c * chunk, hi = lo + chunk < rows ? lo + chunk : rows;
      double s = 0.0;
      for (int64_t i = lo; i < hi; ++i) s += x[i] * a[i * cols + j];
      p[c] = s;
    }
    out[j] = orc_fold_pairwise(p, nch);
    free(p);
  }
}

/* ---------------- elementwise kernels (_kernels.py:159-259) ---------------- */
void orc_sigmoid(const double *x, double *out, int64_t n) {  /* :159-169 */
  for (int64_t i = 0; i < n; ++i) {
    double t = x[i];
    if (t >= 0.0) { double e = exp(-t); out[i] = 1.0 / (1.0 + e); }
    else { double e = exp(t); out[i] = e / (1.0 + e); }
  }
}

void orc_exp(const double *x, double *out, int64_t n) {  /* :172-175 */
  for (int64_t i = 0; i < n; ++i) out[i] = exp(x[i]);
}

void orc_logistic_loss_terms(const double *t, const double *z, double *out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {  /* :193-201 */
    double ti = t[i];
    if (ti >= 0.0) out[i] = log1p(exp(-ti)) + (1.0 - z[i]) * ti;
    else out[i] = log1p(exp(ti)) - z[i] * ti;
  }
}

void orc_normal_cdf(const double *z, double *out, int64_t n) {  /* :204-207 */
  for (int64_t i = 0; i < n; ++i) out[i] = 0.5 * (1.0 + erf(z[i] * 0.7071067811865476));
}

void orc_newsvendor_cost(const double *x, const double *mu, const double *sigma,
                         const double *unit, const double *hold, const double *sell,
                         double *out, int64_t n) {  /* :210-223 */
  const double INV_SQRT_TAU = 0.3989422804014327, SQRT1_2 = 0.7071067811865476;
  for (int64_t j = 0; j < n; ++j) {
    double zj = (x[j] - mu[j]) / sigma[j];
    double pdf = INV_SQRT_TAU * exp(-0.5 * zj * zj);
    double cdf = 0.5 * (1.0 + erf(zj * SQRT1_2));
    double over = sigma[j] * (zj * cdf + pdf);
    double under = sigma[j] * (pdf - zj * (1.0 - cdf));
    out[j] = unit[j] * x[j] + hold[j] * over + sell[j] * under;
  }
}

/* ecdf_count_block (:245-259): upper-bound binary search on sorted rows. */
void orc_ecdf_count(const double *samples, int64_t rows, int64_t s, const double *x,
                    int64_t *out) {
  for (int64_t j = 0; j < rows; ++j) {
    int64_t lo = 0, hi = s;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (samples[j * s + mid] <= x[j]) lo = mid + 1; else hi = mid;
    }
    out[j] = lo;
  }
}

/* bfgs_rank2_block (:226-242) over all rows. */
void orc_bfgs_rank2(double *h, const double *s, const double *u, double coef_su,
                    double coef_ss, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {
    double si = s[i], ui = u[i];
    for (int64_t j = 0; j < n; ++j)
      h[i * n + j] += coef_su * (si * u[j]) + coef_su * (ui * s[j]) + coef_ss * (si * s[j]);
  }
}

/* Sorting helper for sample_demands (sampling.py:192): numpy sort result is the
 * unique ascending order, so any correct sort reproduces it. */
static int dcmp(const void *a, const void *b) {
  double x = *(const double *)a, y = *(const double *)b;
  return (x > y) - (x < y);
}
void orc_sort_rows(double *a, int64_t rows, int64_t cols) {
  for (int64_t r = 0; r < rows; ++r) qsort(a + r * cols, (size_t)cols, sizeof(double), dcmp);
}
