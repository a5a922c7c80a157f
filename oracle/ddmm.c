/* oracle/ddmm.c — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). Plain, slow, obviously-correct
 * CPU kernels for the oracle: a naive double-double matrix product and a __float128 cyclic Jacobi
 * eigensolver. Shares no code with the CUDA path. Compile with -ffp-contract=off so that the
 * error-free transformations below are evaluated exactly as written.
 *
 *   TwoSum   : PAPER.md §2.2 (Knuth), lines 143-153.
 *   TwoProd  : x = fl(a*b), y = a*b - x, via fma (exact; the error term is unique).
 *   dd accumulation: PAPER.md §2.2 pair arithmetic, lines 155-161, with both parts kept.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline void two_sum(double a, double b, double *x, double *y) {
  double s = a + b;
  double z = s - a;
  *x = s;
  *y = (a - (s - z)) + (b - z);
}

static inline void fast_two_sum(double a, double b, double *x, double *y) { /* |a| >= |b| */
  double s = a + b;
  *x = s;
  *y = b - (s - a);
}

static inline void two_prod(double a, double b, double *x, double *y) {
  double p = a * b;
  *x = p;
  *y = fma(a, b, -p);
}

/* (sh, sl) += (ph, pl), accurate double-double addition */
static inline void dd_add(double *sh, double *sl, double ph, double pl) {
  double s, e, t, f;
  two_sum(*sh, ph, &s, &e);
  two_sum(*sl, pl, &t, &f);
  e += t;
  fast_two_sum(s, e, &s, &e);
  e += f;
  fast_two_sum(s, e, sh, sl);
}

/* C[i*n + j] = sum_k (P[i*K+k] (+ Pl)) * (Q[j*K+k] (+ Ql)), i<m, j<n, in double-double.
 * P, Q row-major (contraction index contiguous). Pl/Ql may be NULL (operand exactly fp64).
 * The lo*lo term (< 2^-104 relative) is included for completeness. */
void oracle_dd_gemm_nt(int64_t m, int64_t n, int64_t K, const double *P, const double *Pl, const double *Q,
                       const double *Ql, double *Ch, double *Cl) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t i = 0; i < m; ++i) {
    const double *p = P + i * K;
    const double *pl = Pl ? Pl + i * K : NULL;
    for (int64_t j = 0; j < n; ++j) {
      const double *q = Q + j * K;
      const double *ql = Ql ? Ql + j * K : NULL;
      double sh = 0.0, sl = 0.0;
      for (int64_t k = 0; k < K; ++k) {
        double x, y;
        two_prod(p[k], q[k], &x, &y);
        if (pl) y += pl[k] * q[k];
        if (ql) y += p[k] * ql[k];
        if (pl && ql) y += pl[k] * ql[k];
        dd_add(&sh, &sl, x, y);
      }
      Ch[i * n + j] = sh;
      Cl[i * n + j] = sl;
    }
  }
}

/* Cyclic Jacobi in __float128 on a symmetric n x n matrix (row-major doubles, hi + lo parts).
 * Output: eigenvalues (hi, lo) ascending and eigenvectors as columns of V (row-major, hi+lo),
 * each column sign-fixed so that its largest-|.| entry is positive (lowest index on ties).
 * Sweeps until off(A) <= tol * ||A||_F. Returns the number of sweeps, or -1 if not converged. */
typedef __float128 q_t;

static q_t q_abs(q_t x) { return x < 0 ? -x : x; }
static q_t q_sqrt(q_t x) { /* Newton in quad from a double seed */
  if (x <= 0) return 0;
  q_t y = (q_t)sqrt((double)x);
  for (int i = 0; i < 6; ++i) y = 0.5Q * (y + x / y);
  return y;
}

int oracle_jacobi_q(int n, const double *Ah, const double *Al, double tol, double *wh, double *wl, double *Vh,
                    double *Vl) {
  q_t *a = (q_t *)malloc(sizeof(q_t) * n * n);
  q_t *v = (q_t *)malloc(sizeof(q_t) * n * n);
  for (int i = 0; i < n * n; ++i) a[i] = (q_t)Ah[i] + (Al ? (q_t)Al[i] : 0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) v[i * n + j] = (i == j) ? 1 : 0;
  q_t fro = 0;
  for (int i = 0; i < n * n; ++i) fro += a[i] * a[i];
  fro = q_sqrt(fro);
  int sweeps = -1;
  for (int sw = 0; sw < 100; ++sw) {
    q_t off = 0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j)
        if (i != j) off += a[i * n + j] * a[i * n + j];
    off = q_sqrt(off);
    if (off <= (q_t)tol * fro) {
      sweeps = sw;
      break;
    }
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        q_t apq = a[p * n + q];
        if (apq == 0) continue;
        q_t app = a[p * n + p], aqq = a[q * n + q];
        q_t theta = (aqq - app) / (2 * apq);
        q_t t = (theta >= 0 ? 1 : -1) / (q_abs(theta) + q_sqrt(theta * theta + 1));
        q_t c = 1 / q_sqrt(t * t + 1), s = t * c;
        for (int k = 0; k < n; ++k) { /* A <- J^T A J, columns p,q then rows p,q */
          q_t akp = a[k * n + p], akq = a[k * n + q];
          a[k * n + p] = c * akp - s * akq;
          a[k * n + q] = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          q_t apk = a[p * n + k], aqk = a[q * n + k];
          a[p * n + k] = c * apk - s * aqk;
          a[q * n + k] = s * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) {
          q_t vkp = v[k * n + p], vkq = v[k * n + q];
          v[k * n + p] = c * vkp - s * vkq;
          v[k * n + q] = s * vkp + c * vkq;
        }
      }
  }
  /* sort ascending (selection sort on indices) */
  int *idx = (int *)malloc(sizeof(int) * n);
  for (int i = 0; i < n; ++i) idx[i] = i;
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j)
      if (a[idx[j] * n + idx[j]] < a[idx[i] * n + idx[i]]) {
        int t = idx[i];
        idx[i] = idx[j];
        idx[j] = t;
      }
  for (int c = 0; c < n; ++c) {
    int src = idx[c];
    q_t lam = a[src * n + src];
    wh[c] = (double)lam;
    wl[c] = (double)(lam - (q_t)wh[c]);
    int imax = 0;
    q_t vmax = -1;
    for (int r = 0; r < n; ++r)
      if (q_abs(v[r * n + src]) > vmax) {
        vmax = q_abs(v[r * n + src]);
        imax = r;
      }
    q_t sg = v[imax * n + src] < 0 ? -1 : 1;
    for (int r = 0; r < n; ++r) {
      q_t x = sg * v[r * n + src];
      Vh[r * n + c] = (double)x;
      Vl[r * n + c] = (double)(x - (q_t)Vh[r * n + c]);
    }
  }
  free(idx);
  free(a);
  free(v);
  return sweeps;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}
