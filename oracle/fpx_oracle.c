/* fpx_oracle.c -- CPU ORACLE for the findpts hot path (TEST INFRASTRUCTURE).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
 * `--impl reference`) may load this library; it is the checker, never the
 * product.  Built by oracle/Makefile with -ffp-contract=off so every sum is
 * evaluated as the reference's numpy code does: separate multiply and add,
 * sequential accumulation along the contracted (outer) axis.
 *
 * Every function cites the reference line it restates.  Reference files are
 * /root/reference/pkg/src/fpx/{basis,bounds}.py and /root/reference/SPEC.md.
 */
#include "fpx_oracle.h"

#include <math.h>
#ifdef FPXO_TRACE
#include <stdio.h>
#endif
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ZERO_EXTENT_REL 1e-12     /* bounds.py:43 */
#define INTERIOR_TOL 1e-12
/* D8 resolvability floor of the predicted decrease (DESIGN.md §3 D8) */
#define UNRES_REL 1e-13
#define UNRES_ABS 1e-14

/* ------------------------------------------------------------------ basis */

/* Legendre P_p with two derivatives by the three-term recurrence
 * (basis.py:42-66). */
static void legendre_eval(int p, double x, double* v, double* d, double* s) {
  double v0 = 1.0, d0 = 0.0, s0 = 0.0;
  if (p == 0) { *v = v0; *d = d0; *s = s0; return; }
  double v1 = v0, d1 = d0, s1 = s0;
  v0 = x; d0 = 1.0; s0 = 0.0;
  for (int k = 2; k <= p; ++k) {
    double a = (double)(2 * k - 1) / k;
    double b = (double)(k - 1) / k;
    double v2 = v1, d2 = d1, s2 = s1;
    v1 = v0; d1 = d0; s1 = s0;
    v0 = a * x * v1 - b * v2;
    d0 = a * (v1 + x * d1) - b * d2;
    s0 = a * (2 * d1 + x * s1) - b * s2;
  }
  *v = v0; *d = d0; *s = s0;
}

/* GLL nodes: Newton on P_p' from Chebyshev-Lobatto seeds, <=100 sweeps,
 * stop when max|dx| < 1e-15, then antisymmetrise (basis.py:69-90). */
int fpxo_gll_nodes(int p, double* z) {
  if (p < 1 || p > 29) return -1;
  z[0] = -1.0;
  z[p] = 1.0;
  if (p >= 2) {
    double x[FPXO_MAXN], y[FPXO_MAXN];
    int m = p - 1;
    for (int k = 1; k < p; ++k) x[k - 1] = -cos(M_PI * k / p);
    for (int it = 0; it < 100; ++it) {
      double mx = 0.0;
      for (int k = 0; k < m; ++k) {
        double v, d, s;
        legendre_eval(p, x[k], &v, &d, &s);
        double dx = d / s;
        x[k] -= dx;
        if (fabs(dx) > mx) mx = fabs(dx);
      }
      if (mx < 1e-15) break;
    }
    for (int k = 0; k < m; ++k) y[k] = 0.5 * (x[k] - x[m - 1 - k]);
    for (int k = 0; k < m; ++k) z[k + 1] = y[k];
  }
  return 0;
}

/* eta_j = -cos(j pi / (M-1)) (basis.py:93-97). */
static void chebyshev_points(int m, double* eta) {
  for (int j = 0; j < m; ++j) eta[j] = -cos(j * M_PI / (m - 1));
}

/* Unscaled prefix/suffix products and their derivatives (basis.py:138-180).
 * Outputs N values each; d2 may be NULL. */
static void raw_products(const double* z, int n, double r, double* val,
                         double* d1, double* d2) {
  double pv[FPXO_MAXN + 1], pd[FPXO_MAXN + 1], ps[FPXO_MAXN + 1];
  double sv[FPXO_MAXN + 1], sd[FPXO_MAXN + 1], ss[FPXO_MAXN + 1];
  double u[FPXO_MAXN];
  for (int k = 0; k < n; ++k) u[k] = r - z[k];
  pv[0] = 1.0; pd[0] = 0.0; ps[0] = 0.0;
  sv[n] = 1.0; sd[n] = 0.0; ss[n] = 0.0;
  for (int k = 0; k < n; ++k) {
    ps[k + 1] = ps[k] * u[k] + 2.0 * pd[k];
    pd[k + 1] = pd[k] * u[k] + pv[k];
    pv[k + 1] = pv[k] * u[k];
  }
  for (int k = n - 1; k >= 0; --k) {
    ss[k] = ss[k + 1] * u[k] + 2.0 * sd[k + 1];
    sd[k] = sd[k + 1] * u[k] + sv[k + 1];
    sv[k] = sv[k + 1] * u[k];
  }
  for (int i = 0; i < n; ++i) {
    double a = pv[i], b = sv[i + 1], da = pd[i], db = sd[i + 1];
    val[i] = a * b;
    d1[i] = da * b + a * db;
    if (d2) d2[i] = ps[i] * b + 2.0 * da * db + a * ss[i + 1];
  }
}

/* lagrange_eval at one point (basis.py:183-198). */
void fpxo_lagrange1(const fpxo_basis* B, double r, double* v, double* d1, double* d2) {
  double a[FPXO_MAXN], b[FPXO_MAXN], c[FPXO_MAXN];
  raw_products(B->z, B->N, r, a, b, d2 ? c : NULL);
  for (int i = 0; i < B->N; ++i) {
    v[i] = a[i] * B->scale[i];
    d1[i] = b[i] * B->scale[i];
    if (d2) d2[i] = c[i] * B->scale[i];
  }
}

/* Batched lagrange_eval; outputs [n][N]. */
void fpxo_lagrange(const fpxo_basis* B, int64_t n, const double* r, double* v,
                   double* d1, double* d2) {
  int N = B->N;
  for (int64_t k = 0; k < n; ++k)
    fpxo_lagrange1(B, r[k], v + k * N, d1 + k * N, d2 ? d2 + k * N : NULL);
}

/* Gauss-Legendre rule on nq points, ascending (restates the published
 * numpy.polynomial.legendre.leggauss: roots of P_nq, weights
 * 2/((1-x^2)P'^2), symmetrised, weights scaled to sum 2). */
static void gauss_legendre(int nq, double* x, double* w) {
  double xs[64], ws[64];
  for (int i = 0; i < nq; ++i) {
    double t = cos(M_PI * (i + 0.75) / (nq + 0.5));
    for (int it = 0; it < 100; ++it) {
      double v, d, s;
      legendre_eval(nq, t, &v, &d, &s);
      double dt = v / d;
      t -= dt;
      if (fabs(dt) < 1e-17) break;
    }
    double v, d, s;
    legendre_eval(nq, t, &v, &d, &s);
    xs[nq - 1 - i] = t;
    ws[nq - 1 - i] = 2.0 / ((1.0 - t * t) * d * d);
  }
  double sum = 0.0;
  for (int i = 0; i < nq; ++i) {
    x[i] = 0.5 * (xs[i] - xs[nq - 1 - i]);
    w[i] = 0.5 * (ws[i] + ws[nq - 1 - i]);
  }
  for (int i = 0; i < nq; ++i) sum += w[i];
  for (int i = 0; i < nq; ++i) w[i] *= 2.0 / sum;
}

/* Envelope sample + dense self-check (basis.py:229-238, 275-281). */
static double envelope_violation(const fpxo_basis* B, int samples) {
  int N = B->N, M = B->M;
  double worst = -INFINITY;
  double step = 2.0 / (samples - 1);
  for (int k = 0; k < samples; ++k) {
    double r = (k == samples - 1) ? 1.0 : -1.0 + k * step;
    /* searchsorted(eta, r, 'right') - 1, clipped to [0, M-2] */
    int idx = 0;
    while (idx < M && B->eta[idx] <= r) ++idx;
    idx -= 1;
    if (idx < 0) idx = 0;
    if (idx > M - 2) idx = M - 2;
    double t = (r - B->eta[idx]) / (B->eta[idx + 1] - B->eta[idx]);
    double v[FPXO_MAXN], d1[FPXO_MAXN];
    fpxo_lagrange1(B, r, v, d1, NULL);
    for (int i = 0; i < N; ++i) {
      double lo = B->lo[i * M + idx] * (1.0 - t) + B->lo[i * M + idx + 1] * t;
      double hi = B->hi[i * M + idx] * (1.0 - t) + B->hi[i * M + idx + 1] * t;
      if (lo - v[i] > worst) worst = lo - v[i];
      if (v[i] - hi > worst) worst = v[i] - hi;
    }
  }
  return worst;
}

/* ReferenceBasis + build_basis_envelope (basis.py:100-136, 241-282).
 * Returns 0, -1 (bad order), -2 (M < N), -3 (envelope invalid). */
int fpxo_basis_init(fpxo_basis* B, int p, int M, int validate) {
  memset(B, 0, sizeof(*B));
  if (fpxo_gll_nodes(p, B->z)) return -1;
  int N = p + 1;
  if (M <= 0) M = 2 * N;
  if (M < N) return -2;
  if (M < 2 || M > FPXO_MAXM) return -2;
  B->p = p; B->N = N; B->M = M;
  chebyshev_points(M, B->eta);
  for (int i = 0; i < N; ++i) B->scale[i] = 1.0;
  for (int i = 0; i < N; ++i) {
    double v[FPXO_MAXN], d1[FPXO_MAXN];
    raw_products(B->z, N, B->z[i], v, d1, NULL);
    B->scale[i] = 1.0 / v[i];
  }
  int nq = (p + 3) / 2 + 1;
  double qx[64], qw[64];
  gauss_legendre(nq, qx, qw);
  for (int i = 0; i < N; ++i) { B->proj0[i] = 0.0; B->proj1[i] = 0.0; }
  for (int q = 0; q < nq; ++q) {
    double v[FPXO_MAXN], d1[FPXO_MAXN];
    fpxo_lagrange1(B, qx[q], v, d1, NULL);
    for (int i = 0; i < N; ++i) {
      B->proj0[i] += (0.5 * v[i]) * qw[q];
      B->proj1[i] += (1.5 * v[i]) * (qw[q] * qx[q]);
    }
  }
  /* envelope: candidates {phi(eta_j), midpoint tangents extended by half a
   * gap} (basis.py:255-273; the half-gap is the code's choice, X1) */
  for (int j = 0; j < M; ++j) {
    double ve[FPXO_MAXN], de[FPXO_MAXN];
    fpxo_lagrange1(B, B->eta[j], ve, de, NULL);
    for (int i = 0; i < N; ++i) { B->lo[i * M + j] = ve[i]; B->hi[i * M + j] = ve[i]; }
  }
  double at_right[FPXO_MAXN * FPXO_MAXM], at_left[FPXO_MAXN * FPXO_MAXM];
  for (int j = 0; j + 1 < M; ++j) {
    double mid = 0.5 * (B->eta[j] + B->eta[j + 1]);
    double gap = B->eta[j + 1] - B->eta[j];
    double pm[FPXO_MAXN], dpm[FPXO_MAXN];
    fpxo_lagrange1(B, mid, pm, dpm, NULL);
    for (int i = 0; i < N; ++i) {
      at_right[i * M + j] = pm[i] + 0.5 * gap * dpm[i];
      at_left[i * M + j] = pm[i] - 0.5 * gap * dpm[i];
    }
  }
  for (int i = 0; i < N; ++i) {
    for (int j = 1; j + 1 < M; ++j) {
      double c0 = B->lo[i * M + j], c1 = at_right[i * M + j - 1], c2 = at_left[i * M + j];
      double mn = c0, mx = c0;
      if (c1 < mn) mn = c1;
      if (c2 < mn) mn = c2;
      if (c1 > mx) mx = c1;
      if (c2 > mx) mx = c2;
      B->lo[i * M + j] = mn;
      B->hi[i * M + j] = mx;
    }
    B->lo[i * M + 0] = B->hi[i * M + 0] = (i == 0) ? 1.0 : 0.0;
    B->lo[i * M + M - 1] = B->hi[i * M + M - 1] = (i == N - 1) ? 1.0 : 0.0;
  }
  if (validate && envelope_violation(B, 10000) > 1e-12) return -3;
  return 0;
}

double fpxo_envelope_violation(const fpxo_basis* B, int samples) {
  return envelope_violation(B, samples);
}

/* legendre_coeffs (basis.py:201-212); sequential dot. */
void fpxo_legendre_coeffs(const fpxo_basis* B, const double* u, double* a0, double* a1) {
  double s0 = 0.0, s1 = 0.0;
  for (int i = 0; i < B->N; ++i) { s0 += u[i] * B->proj0[i]; s1 += u[i] * B->proj1[i]; }
  *a0 = s0; *a1 = s1;
}

/* ----------------------------------------------------------------- bounds */

/* bound_function_1d (bounds.py:155-171): Legendre-compacted 1D bound. */
void fpxo_bound1d(const fpxo_basis* B, const double* u, double* lower, double* upper) {
  int N = B->N, M = B->M;
  double a0, a1, w[FPXO_MAXN];
  fpxo_legendre_coeffs(B, u, &a0, &a1);
  for (int i = 0; i < N; ++i) w[i] = u[i] - a0 - a1 * B->z[i];
  for (int j = 0; j < M; ++j) {
    double slo = 0.0, shi = 0.0;
    for (int i = 0; i < N; ++i) {
      double tl = w[i] * B->lo[i * M + j], th = w[i] * B->hi[i * M + j];
      double mn = tl < th ? tl : th, mx = tl > th ? tl : th;
      if (i == 0) { slo = mn; shi = mx; } else { slo += mn; shi += mx; }
    }
    double lin = a0 + a1 * B->eta[j];
    lower[j] = lin + slo;
    upper[j] = lin + shi;
  }
}

/* bound_function_2d (bounds.py:174-201): uncompacted two-sweep bound.
 * u[i + N*j] with i along r, j along s; lower/upper[k*M + l]. */
void fpxo_bound2d(const fpxo_basis* B, const double* u, double* lower, double* upper) {
  int N = B->N, M = B->M;
  double alo[FPXO_MAXN * FPXO_MAXM], ahi[FPXO_MAXN * FPXO_MAXM];
  /* sweep 1: a[j][k] = sum_i min/max(u_ij vlo_ik, u_ij vhi_ik) */
  for (int j = 0; j < N; ++j)
    for (int k = 0; k < M; ++k) {
      double slo = 0.0, shi = 0.0;
      for (int i = 0; i < N; ++i) {
        double uij = u[i + N * j];
        double tl = uij * B->lo[i * M + k], th = uij * B->hi[i * M + k];
        double mn = tl < th ? tl : th, mx = tl > th ? tl : th;
        if (i == 0) { slo = mn; shi = mx; } else { slo += mn; shi += mx; }
      }
      alo[j * M + k] = slo;
      ahi[j * M + k] = shi;
    }
  /* sweep 2: contract j against the s-direction envelope, 4 products */
  for (int k = 0; k < M; ++k)
    for (int l = 0; l < M; ++l) {
      double slo = 0.0, shi = 0.0;
      for (int j = 0; j < N; ++j) {
        double al = alo[j * M + k], ah = ahi[j * M + k];
        double vl = B->lo[j * M + l], vh = B->hi[j * M + l];
        double c0 = al * vl, c1 = al * vh, c2 = ah * vl, c3 = ah * vh;
        double mn = c0, mx = c0;
        if (c1 < mn) mn = c1;
        if (c2 < mn) mn = c2;
        if (c3 < mn) mn = c3;
        if (c1 > mx) mx = c1;
        if (c2 > mx) mx = c2;
        if (c3 > mx) mx = c3;
        if (j == 0) { slo = mn; shi = mx; } else { slo += mn; shi += mx; }
      }
      lower[k * M + l] = slo;
      upper[k * M + l] = shi;
    }
}

static void absorb1(const fpxo_basis* B, const double* u, double* lo, double* hi) {
  double L[FPXO_MAXM], U[FPXO_MAXM];
  fpxo_bound1d(B, u, L, U);
  for (int j = 0; j < B->M; ++j) {
    if (L[j] < *lo) *lo = L[j];
    if (U[j] > *hi) *hi = U[j];
  }
}

static void absorb2(const fpxo_basis* B, const double* u, double* lo, double* hi) {
  double L[FPXO_MAXM * FPXO_MAXM], U[FPXO_MAXM * FPXO_MAXM];
  fpxo_bound2d(B, u, L, U);
  int M = B->M;
  for (int j = 0; j < M * M; ++j) {
    if (L[j] < *lo) *lo = L[j];
    if (U[j] > *hi) *hi = U[j];
  }
}

/* _coordinate_bounds (bounds.py:253-289).  X is [d][N^dr], first reference
 * axis fastest. */
void fpxo_coord_bounds(const fpxo_basis* B, int d, int dr, const double* X,
                       double* lo, double* hi) {
  int N = B->N;
  int K = dr == 1 ? N : (dr == 2 ? N * N : N * N * N);
  double buf[FPXO_MAXN * FPXO_MAXN];
  for (int c = 0; c < d; ++c) { lo[c] = INFINITY; hi[c] = -INFINITY; }
  if (dr == 1) {
    for (int c = 0; c < d; ++c) absorb1(B, X + c * K, lo + c, hi + c);
  } else if (dr == 2 && d == 2) {
    /* quad: edges tens[:,0,:], tens[:,-1,:], tens[:,:,0], tens[:,:,-1] */
    for (int e = 0; e < 4; ++e)
      for (int c = 0; c < d; ++c) {
        const double* Xc = X + c * K;
        for (int t = 0; t < N; ++t) {
          if (e == 0) buf[t] = Xc[t];
          else if (e == 1) buf[t] = Xc[t + N * (N - 1)];
          else if (e == 2) buf[t] = Xc[N * t];
          else buf[t] = Xc[N * t + N - 1];
        }
        absorb1(B, buf, lo + c, hi + c);
      }
  } else if (dr == 2) {
    for (int c = 0; c < d; ++c) absorb2(B, X + c * K, lo + c, hi + c);
  } else {
    /* hex faces in the order k=0, k=N-1, j=0, j=N-1, i=0, i=N-1 */
    for (int f = 0; f < 6; ++f)
      for (int c = 0; c < d; ++c) {
        const double* Xc = X + c * K;
        int fix = (f & 1) ? N - 1 : 0;
        for (int b = 0; b < N; ++b)
          for (int a = 0; a < N; ++a) {
            int idx;
            if (f < 2) idx = a + N * b + N * N * fix;          /* (r=i, s=j) */
            else if (f < 4) idx = a + N * fix + N * N * b;     /* (r=i, s=k) */
            else idx = fix + N * a + N * N * b;                /* (r=j, s=k) */
            buf[a + N * b] = Xc[idx];
          }
        absorb2(B, buf, lo + c, hi + c);
      }
  }
}

/* _expand_box (bounds.py:236-250).  Returns -1 for a degenerate element. */
int fpxo_expand_box(int d, double* lo, double* hi, double factor) {
  double ext[3], pad[3];
  double mx = -INFINITY;
  for (int c = 0; c < d; ++c) { ext[c] = hi[c] - lo[c]; if (ext[c] > mx) mx = ext[c]; }
  if (mx <= 0.0) return -1;
  int anyflat = 0;
  double minlive = INFINITY;
  for (int c = 0; c < d; ++c) {
    pad[c] = factor * ext[c];
    if (ext[c] < ZERO_EXTENT_REL * mx) anyflat = 1;
    else if (ext[c] < minlive) minlive = ext[c];
  }
  if (anyflat)
    for (int c = 0; c < d; ++c)
      if (ext[c] < ZERO_EXTENT_REL * mx) pad[c] = factor * minlive;
  for (int c = 0; c < d; ++c) { lo[c] -= 0.5 * pad[c]; hi[c] += 0.5 * pad[c]; }
  return 0;
}

/* Sequential sum-factorised contraction of one nodal block with per-axis
 * factor vectors, axis 0 (fastest) first (basis.py:285-303). */
static double contract(const double* X, int N, int dr, const double* f0,
                       const double* f1, const double* f2) {
  if (dr == 1) {
    double s = 0.0;
    for (int i = 0; i < N; ++i) s += X[i] * f0[i];
    return s;
  }
  if (dr == 2) {
    double t = 0.0;
    for (int j = 0; j < N; ++j) {
      double s = 0.0;
      for (int i = 0; i < N; ++i) s += X[i + N * j] * f0[i];
      t += s * f1[j];
    }
    return t;
  }
  double q = 0.0;
  for (int k = 0; k < N; ++k) {
    double t = 0.0;
    for (int j = 0; j < N; ++j) {
      double s = 0.0;
      for (int i = 0; i < N; ++i) s += X[i + N * j + N * N * k] * f0[i];
      t += s * f1[j];
    }
    q += t * f2[k];
  }
  return q;
}

static double det3(const double m[3][3]) {
  return m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1]) -
         m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0]) +
         m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]);
}

static double detn(int d, const double m[3][3]) {
  if (d == 2) return m[0][0] * m[1][1] - m[0][1] * m[1][0];
  return det3(m);
}

static void invn(int d, const double m[3][3], double o[3][3]) {
  double det = detn(d, m);
  if (d == 2) {
    o[0][0] = m[1][1] / det; o[0][1] = -m[0][1] / det;
    o[1][0] = -m[1][0] / det; o[1][1] = m[0][0] / det;
    return;
  }
  o[0][0] = (m[1][1] * m[2][2] - m[1][2] * m[2][1]) / det;
  o[0][1] = (m[0][2] * m[2][1] - m[0][1] * m[2][2]) / det;
  o[0][2] = (m[0][1] * m[1][2] - m[0][2] * m[1][1]) / det;
  o[1][0] = (m[1][2] * m[2][0] - m[1][0] * m[2][2]) / det;
  o[1][1] = (m[0][0] * m[2][2] - m[0][2] * m[2][0]) / det;
  o[1][2] = (m[0][2] * m[1][0] - m[0][0] * m[1][2]) / det;
  o[2][0] = (m[1][0] * m[2][1] - m[1][1] * m[2][0]) / det;
  o[2][1] = (m[0][1] * m[2][0] - m[0][0] * m[2][1]) / det;
  o[2][2] = (m[0][0] * m[1][1] - m[0][1] * m[1][0]) / det;
}

static void matmul3(int d, const double a[3][3], const double b[3][3], double o[3][3]) {
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) {
      double s = 0.0;
      for (int k = 0; k < d; ++k) s += a[i][k] * b[k][j];
      o[i][j] = s;
    }
}

/* Rodrigues rotation carrying t onto +x (bounds.py:300-323). */
static int rotation_to_x(int d, const double* tin, double R[3][3]) {
  double nt = 0.0;
  for (int c = 0; c < d; ++c) nt += tin[c] * tin[c];
  nt = sqrt(nt);
  if (nt == 0.0) return -1;
  double t[3];
  for (int c = 0; c < d; ++c) t[c] = tin[c] / nt;
  memset(R, 0, sizeof(double) * 9);
  if (d == 2) {
    R[0][0] = t[0]; R[0][1] = t[1]; R[1][0] = -t[1]; R[1][1] = t[0];
    return 0;
  }
  /* k = t x e1 */
  double k[3] = {0.0, t[2], -t[1]};
  double sk = sqrt(k[0] * k[0] + k[1] * k[1] + k[2] * k[2]);
  double ck = t[0];
  if (sk < 1e-14) {
    if (ck > 0.0) { R[0][0] = R[1][1] = R[2][2] = 1.0; }
    else { R[0][0] = -1.0; R[1][1] = -1.0; R[2][2] = 1.0; }
    return 0;
  }
  for (int c = 0; c < 3; ++c) k[c] /= sk;
  double kx[3][3] = {{0, -k[2], k[1]}, {k[2], 0, -k[0]}, {-k[1], k[0], 0}};
  double kk[3][3];
  matmul3(3, kx, kx, kk);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      R[i][j] = (i == j ? 1.0 : 0.0) + sk * kx[i][j] + (1.0 - ck) * kk[i][j];
  return 0;
}

/* Rotation carrying the normal onto +z (bounds.py:326-338). */
static int rotation_normal_to_z(const double* nin, double R[3][3]) {
  double nn = sqrt(nin[0] * nin[0] + nin[1] * nin[1] + nin[2] * nin[2]);
  if (nn == 0.0) return -1;
  double n[3] = {nin[0] / nn, nin[1] / nn, nin[2] / nn};
  double k[3] = {n[1], -n[0], 0.0}; /* n x e3 */
  double sk = sqrt(k[0] * k[0] + k[1] * k[1] + k[2] * k[2]);
  double ck = n[2];
  memset(R, 0, sizeof(double) * 9);
  if (sk < 1e-14) {
    if (ck > 0.0) { R[0][0] = R[1][1] = R[2][2] = 1.0; }
    else { R[0][0] = 1.0; R[1][1] = -1.0; R[2][2] = -1.0; }
    return 0;
  }
  for (int c = 0; c < 3; ++c) k[c] /= sk;
  double kx[3][3] = {{0, -k[2], k[1]}, {k[2], 0, -k[0]}, {-k[1], k[0], 0}};
  double kk[3][3];
  matmul3(3, kx, kx, kk);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      R[i][j] = (i == j ? 1.0 : 0.0) + sk * kx[i][j] + (1.0 - ck) * kk[i][j];
  return 0;
}

/* center_map_and_jacobian + _center_frame (bounds.py:97-107, 341-363).
 * Returns 0 and (x_c, M) or -1 for SingularTransformError. */
static int center_frame(const fpxo_basis* B, int d, int dr, const double* X,
                        double* xc, double Mf[3][3]) {
  int N = B->N;
  int K = dr == 1 ? N : (dr == 2 ? N * N : N * N * N);
  double v0[FPXO_MAXN], d0[FPXO_MAXN];
  fpxo_lagrange1(B, 0.0, v0, d0, NULL);
  double jac[3][3] = {{0}};
  for (int c = 0; c < d; ++c) {
    xc[c] = contract(X + c * K, N, dr, v0, v0, v0);
    for (int a = 0; a < dr; ++a) {
      const double* f[3] = {v0, v0, v0};
      f[a] = d0;
      jac[c][a] = contract(X + c * K, N, dr, f[0], f[1], f[2]);
    }
  }
  memset(Mf, 0, sizeof(double) * 9);
  if (dr == d) {
    double det = detn(d, jac);
    double scale = 1.0;
    for (int a = 0; a < d; ++a) {
      double s = 0.0;
      for (int c = 0; c < d; ++c) s += jac[c][a] * jac[c][a];
      scale *= sqrt(s);
    }
    if (fabs(det) < 1e-13 * (scale > 1e-300 ? scale : 1e-300)) return -1;
    for (int i = 0; i < d; ++i)
      for (int j = 0; j < d; ++j) Mf[i][j] = jac[i][j];
    return 0;
  }
  double rot[3][3];
  if (dr == 1) {
    double t[3] = {jac[0][0], jac[1][0], d == 3 ? jac[2][0] : 0.0};
    if (rotation_to_x(d, t, rot)) return -1;
    invn(d, rot, Mf);
    return 0;
  }
  /* curved quad in 3D (bounds.py:354-363) */
  double t1[3] = {jac[0][0], jac[1][0], jac[2][0]};
  double t2[3] = {jac[0][1], jac[1][1], jac[2][1]};
  double nv[3] = {t1[1] * t2[2] - t1[2] * t2[1], t1[2] * t2[0] - t1[0] * t2[2],
                  t1[0] * t2[1] - t1[1] * t2[0]};
  double r1[3][3];
  if (rotation_normal_to_z(nv, r1)) return -1;
  double a[3][3];
  for (int i = 0; i < 3; ++i) {
    a[i][0] = r1[i][0] * t1[0] + r1[i][1] * t1[1] + r1[i][2] * t1[2];
    a[i][1] = r1[i][0] * t2[0] + r1[i][1] * t2[1] + r1[i][2] * t2[2];
    a[i][2] = (i == 2) ? 1.0 : 0.0;
  }
  if (fabs(det3(a)) < 1e-14) return -1;
  double ai[3][3];
  invn(3, a, ai);
  matmul3(3, ai, r1, rot);
  invn(3, rot, Mf);
  return 0;
}

/* Per-element setup: element_aabb + element_obb (bounds.py:292-297,
 * 366-384) plus the hash box of decision D5: the AABB_ref
 * intersected with the axis-aligned enclosure of the OBB.
 * status[e]: 0 ok, 1 degenerate AABB (setup error), 2 OBB unusable (AABB only).
 * Returns the number of degenerate elements. */
int64_t fpxo_element_boxes(const fpxo_basis* B, int d, int dr, int64_t E,
                           const double* nodes, double expansion, double* aabb,
                           double* obb_c, double* obb_inv, double* hbox,
                           uint8_t* obb_ok, int32_t* status, double* frame) {
  int N = B->N;
  int K = dr == 1 ? N : (dr == 2 ? N * N : N * N * N);
  int64_t bad = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(+ : bad)
  for (int64_t e = 0; e < E; ++e) {
    const double* X = nodes + e * d * K;
    double lo[3], hi[3];
    fpxo_coord_bounds(B, d, dr, X, lo, hi);
    status[e] = 0;
    if (fpxo_expand_box(d, lo, hi, expansion)) { status[e] = 1; ++bad; }
    for (int c = 0; c < d; ++c) { aabb[e * 2 * d + c] = lo[c]; aabb[e * 2 * d + d + c] = hi[c]; }
    double xc[3], Mf[3][3], Mi[3][3];
    int ok = center_frame(B, d, dr, X, xc, Mf) == 0;
    double olo[3], ohi[3];
    if (ok) {
      invn(d, Mf, Mi);
      double* loc = (double*)malloc(sizeof(double) * 3 * (size_t)K);
      for (int c = 0; c < d; ++c)
        for (int n = 0; n < K; ++n) {
          double s = 0.0;
          for (int b = 0; b < d; ++b) s += Mi[c][b] * (X[b * K + n] - xc[b]);
          loc[c * K + n] = s;
        }
      fpxo_coord_bounds(B, d, dr, loc, olo, ohi);
      free(loc);
      if (fpxo_expand_box(d, olo, ohi, expansion)) ok = 0;
    }
    if (ok) {
      double half[3], bc[3];
      for (int c = 0; c < d; ++c) { half[c] = 0.5 * (ohi[c] - olo[c]); bc[c] = 0.5 * (ohi[c] + olo[c]); }
      for (int c = 0; c < d; ++c) {
        double s = 0.0;
        for (int b = 0; b < d; ++b) s += Mf[c][b] * bc[b];
        obb_c[e * d + c] = xc[c] + s;
        for (int b = 0; b < d; ++b) obb_inv[(e * d + c) * d + b] = Mi[c][b] / half[c];
      }
      for (int c = 0; c < d; ++c) {
        double h = 0.0;
        for (int b = 0; b < d; ++b) h += fabs(Mf[c][b] * half[b]);
        double cc = obb_c[e * d + c];
        h = h * (1.0 + 1e-9) + 4.0 * 2.220446049250313e-16 * fabs(cc);
        double l = cc - h, u = cc + h;
        hbox[e * 2 * d + c] = l > lo[c] ? l : lo[c];
        hbox[e * 2 * d + d + c] = u < hi[c] ? u : hi[c];
      }
      obb_ok[e] = 1;
    } else {
      for (int c = 0; c < d; ++c) {
        obb_c[e * d + c] = NAN;
        for (int b = 0; b < d; ++b) obb_inv[(e * d + c) * d + b] = NAN;
        hbox[e * 2 * d + c] = lo[c];
        hbox[e * 2 * d + d + c] = hi[c];
      }
      obb_ok[e] = 0;
      if (status[e] == 0) status[e] = 2;
    }
    if (frame) {  /* centre frame (x_c, M^-1; zero when unusable): the D7' seed */
      double* fr = frame + e * (d + d * d);
      for (int c = 0; c < d; ++c) fr[c] = xc[c];
      for (int c = 0; c < d; ++c)
        for (int b = 0; b < d; ++b) fr[d + c * d + b] = ok ? Mi[c][b] : 0.0;
    }
  }
  return bad;
}

/* aabb_contains / obb_contains (bounds.py:387-396). */
static int aabb_contains(int d, const double* box, const double* x) {
  for (int c = 0; c < d; ++c)
    if (!((x[c] - box[c]) * (box[d + c] - x[c]) >= 0.0)) return 0;
  return 1;
}

static int obb_contains(int d, const double* cen, const double* inv, const double* x) {
  double dx[3];
  for (int c = 0; c < d; ++c) dx[c] = x[c] - cen[c];
  for (int c = 0; c < d; ++c) {
    double y = 0.0;
    for (int b = 0; b < d; ++b) y += inv[c * d + b] * dx[b];
    if (!(fabs(y) <= 1.0)) return 0;
  }
  return 1;
}

void fpxo_contains(int d, int64_t n, const double* box, const double* cen,
                   const double* inv, const double* x, uint8_t* in_aabb, uint8_t* in_obb) {
  for (int64_t k = 0; k < n; ++k) {
    in_aabb[k] = (uint8_t)aabb_contains(d, box, x + k * d);
    in_obb[k] = (uint8_t)obb_contains(d, cen, inv, x + k * d);
  }
}

/* --------------------------------------------------------- spatial hash */

/* Grid over the union of boxes: grid = lo[3], hi[3], h[3]. */
void fpxo_hash_grid(int d, int64_t E, const double* box, int ncell, double* grid) {
  for (int c = 0; c < 3; ++c) { grid[c] = 0.0; grid[3 + c] = 0.0; grid[6 + c] = 1.0; }
  for (int c = 0; c < d; ++c) {
    double lo = INFINITY, hi = -INFINITY;
    for (int64_t e = 0; e < E; ++e) {
      if (box[e * 2 * d + c] < lo) lo = box[e * 2 * d + c];
      if (box[e * 2 * d + d + c] > hi) hi = box[e * 2 * d + d + c];
    }
    grid[c] = lo;
    grid[3 + c] = hi;
    grid[6 + c] = (hi - lo) / ncell;
  }
}

/* cell_of: floor((x-lo)/h); upper boundary -> last cell;
 * outside -> -1.  Per-axis coordinates written to ax (may be NULL). */
static int64_t cell_of(int d, const double* grid, int n, const double* x, int* ax) {
  int64_t idx = 0, mul = 1;
  for (int c = 0; c < d; ++c) {
    if (!(x[c] >= grid[c] && x[c] <= grid[3 + c])) return -1;
    double t = (x[c] - grid[c]) / grid[6 + c];
    int64_t q = (int64_t)floor(t);
    if (q > n - 1) q = n - 1;
    if (q < 0) q = 0;
    if (ax) ax[c] = (int)q;
    idx += q * mul;
    mul *= n;
  }
  return idx;
}

int64_t fpxo_cell_of(int d, const double* grid, int n, const double* x) {
  return cell_of(d, grid, n, x, NULL);
}

/* Conservative cell-vs-OBB overlap (decision D5b): the cell
 * centre mapped into the OBB frame must lie within the unit cube grown by the
 * cell's half-extent seen in that frame, with a 1e-9 relative margin.  Never
 * drops a cell containing a point of the OBB, so the filtered candidate set
 * of every point is unchanged. */
static int cell_meets_obb(int d, const double* grid, const int* q, const double* cen,
                          const double* inv) {
  double dx[3];
  for (int b = 0; b < d; ++b) {
    double cc = grid[b] + ((double)q[b] + 0.5) * grid[6 + b];
    dx[b] = cc - cen[b];
  }
  for (int a = 0; a < d; ++a) {
    double y = 0.0, e = 0.0;
    for (int b = 0; b < d; ++b) {
      y += inv[a * d + b] * dx[b];
      e += fabs(inv[a * d + b]) * (0.5 * grid[6 + b]);
    }
    if (!(fabs(y) <= (1.0 + e) * (1.0 + 1e-9))) return 0;
  }
  return 1;
}

/* build_local_map: CSR of cell -> ascending element ids
 * over the rectangular cell range of each box's two corners; with OBBs
 * (obb_ok != NULL) cells that cannot meet the element's OBB are skipped.
 * Call with elems == NULL to get the total entry count in offsets[ncell^d]. */
int64_t fpxo_hash_build(int d, int64_t E, const double* box, const double* obb_c,
                        const double* obb_inv, const uint8_t* obb_ok, const double* grid, int n,
                        int32_t* offsets, int32_t* elems) {
  int64_t nc = 1;
  for (int c = 0; c < d; ++c) nc *= n;
  int64_t* cnt = (int64_t*)calloc((size_t)nc + 1, sizeof(int64_t));
  for (int64_t e = 0; e < E; ++e) {
    int a[3] = {0, 0, 0}, b[3] = {0, 0, 0};
    cell_of(d, grid, n, box + e * 2 * d, a);
    cell_of(d, grid, n, box + e * 2 * d + d, b);
    const int cull = obb_ok && obb_ok[e];
    for (int k = a[2]; k <= (d == 3 ? b[2] : 0); ++k)
      for (int j = a[1]; j <= b[1]; ++j)
        for (int i = a[0]; i <= b[0]; ++i) {
          int q[3] = {i, j, k};
          if (cull && !cell_meets_obb(d, grid, q, obb_c + e * d, obb_inv + e * d * d)) continue;
          int64_t cell = i + (int64_t)n * (j + (int64_t)n * k);
          if (elems) elems[offsets[cell] + cnt[cell]] = (int32_t)e;
          cnt[cell]++;
        }
  }
  int64_t total = 0;
  if (!elems) {
    for (int64_t c = 0; c < nc; ++c) { offsets[c] = (int32_t)total; total += cnt[c]; }
    offsets[nc] = (int32_t)total;
  } else {
    total = offsets[nc];
  }
  free(cnt);
  return total;
}

/* ---------------------------------------------------------------- invmap */

typedef struct {
  double x[3];
  double G[3][3];   /* G[c][a] = dx_c / dr_a */
  double H2[3][6];  /* (rr, ss, tt, rs, rt, st) */
} fmap_t;

/* forward_map: x(r), G and optionally second
 * derivatives by sum factorisation, axis 0 contracted first. */
static void fmap(const fpxo_basis* B, int d, int dr, const double* X, const double* r,
                 int want2, fmap_t* o) {
  int N = B->N;
  int K = dr == 1 ? N : (dr == 2 ? N * N : N * N * N);
  double v[3][FPXO_MAXN], g[3][FPXO_MAXN], h[3][FPXO_MAXN];
  for (int a = 0; a < dr; ++a) fpxo_lagrange1(B, r[a], v[a], g[a], want2 ? h[a] : NULL);
  memset(o, 0, sizeof(*o));
  for (int c = 0; c < d; ++c) {
    const double* Xc = X + c * K;
    if (dr == 1) {
      double s0 = 0, s1 = 0, s2 = 0;
      for (int i = 0; i < N; ++i) {
        s0 += Xc[i] * v[0][i];
        s1 += Xc[i] * g[0][i];
        if (want2) s2 += Xc[i] * h[0][i];
      }
      o->x[c] = s0; o->G[c][0] = s1; o->H2[c][0] = s2;
    } else if (dr == 2) {
      double t00 = 0, t10 = 0, t01 = 0, t20 = 0, t11 = 0, t02 = 0;
      for (int j = 0; j < N; ++j) {
        double s0 = 0, s1 = 0, s2 = 0;
        for (int i = 0; i < N; ++i) {
          double xv = Xc[i + N * j];
          s0 += xv * v[0][i];
          s1 += xv * g[0][i];
          if (want2) s2 += xv * h[0][i];
        }
        t00 += s0 * v[1][j]; t10 += s1 * v[1][j]; t01 += s0 * g[1][j];
        if (want2) { t20 += s2 * v[1][j]; t11 += s1 * g[1][j]; t02 += s0 * h[1][j]; }
      }
      o->x[c] = t00; o->G[c][0] = t10; o->G[c][1] = t01;
      /* sym index for dr=2: (rr, ss, -, rs) */
      o->H2[c][0] = t20; o->H2[c][1] = t02; o->H2[c][3] = t11;
    } else {
      double q[10] = {0};
      for (int k = 0; k < N; ++k) {
        double t00 = 0, t10 = 0, t01 = 0, t20 = 0, t11 = 0, t02 = 0;
        for (int j = 0; j < N; ++j) {
          double s0 = 0, s1 = 0, s2 = 0;
          for (int i = 0; i < N; ++i) {
            double xv = Xc[i + N * j + N * N * k];
            s0 += xv * v[0][i];
            s1 += xv * g[0][i];
            if (want2) s2 += xv * h[0][i];
          }
          t00 += s0 * v[1][j]; t10 += s1 * v[1][j]; t01 += s0 * g[1][j];
          if (want2) { t20 += s2 * v[1][j]; t11 += s1 * g[1][j]; t02 += s0 * h[1][j]; }
        }
        q[0] += t00 * v[2][k];           /* x   */
        q[1] += t10 * v[2][k];           /* x_r */
        q[2] += t01 * v[2][k];           /* x_s */
        q[3] += t00 * g[2][k];           /* x_t */
        if (want2) {
          q[4] += t20 * v[2][k];         /* rr */
          q[5] += t02 * v[2][k];         /* ss */
          q[6] += t00 * h[2][k];         /* tt */
          q[7] += t11 * v[2][k];         /* rs */
          q[8] += t10 * g[2][k];         /* rt */
          q[9] += t01 * g[2][k];         /* st */
        }
      }
      o->x[c] = q[0]; o->G[c][0] = q[1]; o->G[c][1] = q[2]; o->G[c][2] = q[3];
      for (int m = 0; m < 6; ++m) o->H2[c][m] = q[4 + m];
    }
  }
}

void fpxo_forward_map(const fpxo_basis* B, int d, int dr, const double* X, const double* r,
                      double* x, double* G, double* H2) {
  fmap_t o;
  fmap(B, d, dr, X, r, H2 != NULL, &o);
  for (int c = 0; c < d; ++c) {
    x[c] = o.x[c];
    for (int a = 0; a < dr; ++a) G[c * dr + a] = o.G[c][a];
    if (H2) for (int m = 0; m < 6; ++m) H2[c * 6 + m] = o.H2[c][m];
  }
}

static const int SYM[3][3] = {{0, 3, 4}, {3, 1, 5}, {4, 5, 2}};

/* Cholesky solve of the principal submatrix A[idx][idx] (n <= 3), pivot
 * test p > 1e-14 |trace| (decision D8: non-positive pivot -> not PD). */
static int chol_solve(int n, const int* idx, const double A[3][3], const double* b, double* x) {
  double L[3][3] = {{0}}, y[3], iL[3];
  double tr = 0.0;
  for (int k = 0; k < n; ++k) tr += A[idx[k]][idx[k]];
  double thr = 1e-14 * fabs(tr);
  for (int k = 0; k < n; ++k) {
    double s = A[idx[k]][idx[k]];
    for (int m = 0; m < k; ++m) s -= L[k][m] * L[k][m];
    if (!(s > thr)) return -1;
    L[k][k] = sqrt(s);
    iL[k] = 1.0 / L[k][k];
    for (int i = k + 1; i < n; ++i) {
      double t = A[idx[i]][idx[k]];
      for (int m = 0; m < k; ++m) t -= L[i][m] * L[k][m];
      L[i][k] = t * iL[k];
    }
  }
  for (int k = 0; k < n; ++k) {
    double t = b[k];
    for (int m = 0; m < k; ++m) t -= L[k][m] * y[m];
    y[k] = t * iL[k];
  }
  for (int k = n - 1; k >= 0; --k) {
    double t = y[k];
    for (int m = k + 1; m < n; ++m) t -= L[m][k] * x[m];
    x[k] = t * iL[k];
  }
  return 0;
}

/* Projected trust-region Newton step (decision D8 as frozen
 * in DESIGN.md §3.4).  freem[] enters as the axes not held by an active
 * bound (on a face with the gradient pushing out).
 *   1. Newton direction on the free axes: Hm_FF s_F = -J_F, s_A = 0;
 *   2. a free axis sitting on a face whose Newton component points out of
 *      the box is made active and the direction re-solved (<= dr times);
 *   3. the step is the direction truncated at the trust radius alpha
 *      (|s|_inf <= alpha) and at the first face it reaches: s = t s_N.
 * *hit gets a bitmask of the axes whose face limits t (they land exactly on
 * +-1).  A positive multiple of a Newton direction of a positive definite
 * model is a descent step, so the predicted decrease is > 0 unless s = 0.
 * Returns -1 if the free block is not positive definite. */
static int constrained_step(int dr, const double Hm[3][3], const double* J, const double* r,
                            int* freem, double alpha, double* s, int* hit) {
  double x[3] = {0, 0, 0};
  *hit = 0;
  for (int a = 0; a < dr; ++a) s[a] = 0.0;
  for (int pass = 0; pass <= dr; ++pass) {
    int fidx[3], nf = 0;
    for (int a = 0; a < dr; ++a) if (freem[a]) fidx[nf++] = a;
    if (nf == 0) return 0;
    double rhs[3] = {0, 0, 0}, y[3] = {0, 0, 0};
    for (int k = 0; k < nf; ++k) rhs[k] = -J[fidx[k]];
    if (chol_solve(nf, fidx, Hm, rhs, y)) return -1;
    int blocked = 0;
    for (int a = 0; a < dr; ++a) x[a] = 0.0;
    for (int k = 0; k < nf; ++k) {
      int a = fidx[k];
      x[a] = y[k];
      if ((r[a] == 1.0 && y[k] > 0.0) || (r[a] == -1.0 && y[k] < 0.0)) { freem[a] = 0; blocked = 1; }
    }
    if (!blocked) break;
    if (pass == dr) return 0;
  }
  double m = 0.0;
  for (int a = 0; a < dr; ++a) if (freem[a] && fabs(x[a]) > m) m = fabs(x[a]);
  if (m == 0.0) return 0;
  double t = m > alpha ? alpha / m : 1.0;
  double ta[3] = {INFINITY, INFINITY, INFINITY};
  for (int a = 0; a < dr; ++a) {
    if (!freem[a] || x[a] == 0.0) continue;
    ta[a] = x[a] > 0.0 ? (1.0 - r[a]) / x[a] : (-1.0 - r[a]) / x[a];
    if (ta[a] < t) t = ta[a];
  }
  for (int a = 0; a < dr; ++a) {
    if (!freem[a]) continue;
    s[a] = t * x[a];
    if (ta[a] == t) *hit |= 1 << a;
  }
  return 0;
}

static int on_boundary(int dr, const double* r) {
  for (int a = 0; a < dr; ++a) if (r[a] == -1.0 || r[a] == 1.0) return 1;
  return 0;
}

/* invert_point with the frozen
 * mechanics of decision D8. */
static void invert_core(const fpxo_basis* B, int d, int dr, const double* X, const double* xs,
                        const fpxo_newton* S, const double* r0, int abort_r2, double* r_out,
                        double* dist, int* iters, int* conv, int* aborted);

void fpxo_invert(const fpxo_basis* B, int d, int dr, const double* X, const double* xs,
                 const fpxo_newton* S, double* r_out, double* dist, int* iters, int* conv) {
  invert_core(B, d, dr, X, xs, S, NULL, 0, r_out, dist, iters, conv, NULL);
}

/* invert_point with an explicit initial guess r0 (NULL -> the
 * D7 nearest-node seed), clamped to [-1, 1]. */
void fpxo_invert_from(const fpxo_basis* B, int d, int dr, const double* X, const double* xs,
                      const fpxo_newton* S, const double* r0, double* r_out, double* dist,
                      int* iters, int* conv) {
  invert_core(B, d, dr, X, xs, S, r0, 0, r_out, dist, iters, conv, NULL);
}

/* The trust-region solve.  abort_r2: stop (*aborted = 1) when the iterate is
 * held on a face -- on it, with the descent direction -J leaving through it
 * -- at two consecutive iterations (it >= 1; rule R2, DESIGN.md §3 D7'). */
static void invert_core(const fpxo_basis* B, int d, int dr, const double* X, const double* xs,
                        const fpxo_newton* S, const double* r0, int abort_r2, double* r_out,
                        double* dist, int* iters, int* conv, int* aborted) {
  int held_prev = 0;
  if (aborted) *aborted = 0;
  int N = B->N;
  int K = dr == 1 ? N : (dr == 2 ? N * N : N * N * N);
  /* seed: nearest GLL node, ties -> lowest lexicographic index (D7) */
  double best = INFINITY;
  int bi = 0;
  for (int n = 0; n < (r0 ? 0 : K); ++n) {
    double dd = 0.0;
    for (int c = 0; c < d; ++c) { double t = xs[c] - X[c * K + n]; dd = fma(t, t, dd); }
    if (dd < best) { best = dd; bi = n; }
  }
  double r[3] = {0, 0, 0};
  r[0] = B->z[bi % N];
  if (dr > 1) r[1] = B->z[(bi / N) % N];
  if (dr > 2) r[2] = B->z[bi / (N * N)];
  if (r0)
    for (int a = 0; a < dr; ++a) r[a] = fmin(1.0, fmax(-1.0, r0[a]));
  fmap_t cur, nxt;
  fmap(B, d, dr, X, r, on_boundary(dr, r), &cur);
  double dx[3], f = 0.0;
  for (int c = 0; c < d; ++c) { dx[c] = xs[c] - cur.x[c]; f += dx[c] * dx[c]; }
  double alpha = S->alpha0;
  int it = 0, converged = 0;
  while (it < S->max_iters) {
    int beta = it > 0 && on_boundary(dr, r);
    double J[3], H0[3][3], Hb[3][3];
    for (int a = 0; a < dr; ++a) {
      double s = 0.0;
      for (int c = 0; c < d; ++c) s += cur.G[c][a] * dx[c];
      J[a] = -s;
      for (int b = 0; b < dr; ++b) {
        double g = 0.0, q = 0.0;
        for (int c = 0; c < d; ++c) { g += cur.G[c][a] * cur.G[c][b]; q += dx[c] * cur.H2[c][SYM[a][b]]; }
        H0[a][b] = g;
        Hb[a][b] = g - q;
      }
    }
    /* active bounds: on a face with the descent direction -J pointing out */
    int freem[3] = {1, 1, 1};
    for (int a = 0; a < dr; ++a)
      if ((r[a] == 1.0 && J[a] < 0.0) || (r[a] == -1.0 && J[a] > 0.0)) freem[a] = 0;
    if (abort_r2 && it >= 1) {
      const int held = !(freem[0] && freem[1] && freem[2]);
      if (held && held_prev) {
        if (aborted) *aborted = 1;
        break;
      }
      held_prev = held;
    }
    double s[3] = {0, 0, 0};
    const double(*Hm)[3] = H0;
    double Hr[3][3];
    int fr[3], hit = 0;
    for (int a = 0; a < 3; ++a) fr[a] = freem[a];
    if (beta && constrained_step(dr, Hb, J, r, fr, alpha, s, &hit) == 0) {
      Hm = Hb;
    } else {
      for (int a = 0; a < 3; ++a) fr[a] = freem[a];
      if (constrained_step(dr, H0, J, r, fr, alpha, s, &hit) != 0) {
        double tr = 0.0;
        for (int a = 0; a < dr; ++a) tr += H0[a][a];
        double lam = 1e-10 * tr / dr;
        if (!(lam > 0.0)) lam = 1e-300;
        for (int a = 0; a < dr; ++a)
          for (int b = 0; b < dr; ++b) Hr[a][b] = H0[a][b] + (a == b ? lam : 0.0);
        Hm = Hr;
        for (int a = 0; a < 3; ++a) fr[a] = freem[a];
        if (constrained_step(dr, Hr, J, r, fr, alpha, s, &hit) != 0)
          for (int a = 0; a < dr; ++a) s[a] = 0.0;
      }
    }
    ++it;
    double js = 0.0, shs = 0.0, smax = 0.0;
    for (int a = 0; a < dr; ++a) {
      js += J[a] * s[a];
      double t = 0.0;
      for (int b = 0; b < dr; ++b) t += Hm[a][b] * s[b];
      shs += s[a] * t;
      if (fabs(s[a]) > smax) smax = fabs(s[a]);
    }
    double pred = -(2.0 * js + shs);
    double rn[3] = {0, 0, 0};
    for (int a = 0; a < dr; ++a) {
      double v = r[a] + s[a];
      if (hit & (1 << a)) v = s[a] > 0.0 ? 1.0 : -1.0;  /* lands on the face */
      if (v < -1.0) v = -1.0;
      if (v > 1.0) v = 1.0;
      rn[a] = v;
    }
    /* D8 resolvability: |dx|^2 = f carries a rounding noise of about
     * eps f + 2 d* eps |x|.  A predicted decrease below that floor cannot be
     * checked against the actual one, so the step is taken on the model's
     * word: pred = -inf (accepted, alpha grows); a step below tol is the last
     * one and is applied without a trial evaluation (d* stays that of the
     * last evaluated iterate; the difference is second order).  r* is thus
     * the root of the projected gradient to roundoff, not wherever f
     * stopped resolving steps. */
    double xsc = 0.0;
    for (int c = 0; c < d; ++c) xsc = fmax(xsc, fabs(xs[c]));
    const int unres = !(pred > UNRES_REL * f + UNRES_ABS * sqrt(f) * xsc);
#ifdef FPXO_TRACE
    if (unres) fprintf(stderr, "unres it %d pred %.3e f %.3e s=(%.3e %.3e %.3e) J=(%.3e %.3e %.3e) free %d%d%d alpha %.3e\n", it, pred, f, s[0], s[1], s[2], J[0], J[1], J[2], freem[0], freem[1], freem[2], alpha);
#endif
    if (unres) {
      if (smax < S->tol) {
        for (int a = 0; a < dr; ++a) r[a] = rn[a];
        converged = 1;
        break;
      }
      pred = -INFINITY;
    }
    fmap(B, d, dr, X, rn, on_boundary(dr, rn), &nxt);
    double dxn[3], fn = 0.0;
    for (int c = 0; c < d; ++c) { dxn[c] = xs[c] - nxt.x[c]; fn += dxn[c] * dxn[c]; }
    double decr = f - fn;
#ifdef FPXO_TRACE
    fprintf(stderr, "it %2d beta %d free %d%d%d r=(%.6f %.6f %.6f) s=(%.3e %.3e %.3e) f=%.6e fn=%.6e pred=%.3e decr=%.3e alpha=%.3e\n", it, beta, freem[0], freem[1], freem[2], r[0], r[1], r[2], s[0], s[1], s[2], f, fn, pred, decr, alpha);
#endif
    if (decr >= S->accept * pred) {
      if (decr >= S->keep * pred) alpha *= S->grow;
      for (int a = 0; a < dr; ++a) r[a] = rn[a];
      cur = nxt;
      for (int c = 0; c < d; ++c) dx[c] = dxn[c];
      f = fn;
    } else {
      alpha *= S->shrink;
    }
    if (smax < S->tol) { converged = 1; break; }
  }
  for (int a = 0; a < dr; ++a) r_out[a] = r[a];
  *dist = sqrt(f);
  *iters = it;
  *conv = converged;
}

/* classify (surface eps_d SPEC.md:329). */
static int classify(int d, int dr, const double* r, double dist, double eps_d) {
  for (int a = 0; a < dr; ++a)
    if (!(fabs(r[a]) < 1.0 - INTERIOR_TOL)) return FPXO_BORDER;
  if (dr < d && !(dist < eps_d)) return FPXO_BORDER;
  return FPXO_INTERIOR;
}

/* One candidate's solve, decision D7': for volume elements
 * with a centre frame, first from the affine seed r0 = clamp(J_c^-1 (x* -
 * x_c)) with the abort rule R2; that result stands if it is INTERIOR (the
 * unique zero of the injective element map, whatever the seed).  Otherwise
 * -- aborted or BORDER -- the solve from the D7 nearest-node seed (SPEC.md:
 * 327) is the candidate's result.  Surfaces and lines use D7 only.  The
 * seed is formed with separate multiply and add exactly as the kernels do. */
static void candidate_solve(const fpxo_mesh* m, int32_t e, const double* xs, double* rr,
                            double* dd, int* it, int* cv) {
  int d = m->d, dr = m->dr, N = m->B->N;
  int K = dr == 1 ? N : (dr == 2 ? N * N : N * N * N);
  const double* X = m->nodes + (int64_t)e * d * K;
  if (m->frame && d == dr) {
    const double* fr = m->frame + (int64_t)e * (d + d * d);
    double r0[3] = {0, 0, 0}, dx[3];
    for (int c = 0; c < d; ++c) dx[c] = xs[c] - fr[c];
    for (int a = 0; a < d; ++a) {
      double y = 0.0;
      for (int b = 0; b < d; ++b) y = y + fr[d + a * d + b] * dx[b];
      r0[a] = isfinite(y) ? fmin(1.0, fmax(-1.0, y)) : 0.0;
    }
    int ab = 0, it1 = 0;
    invert_core(m->B, d, dr, X, xs, &m->newton, r0, 1, rr, dd, &it1, cv, &ab);
    int inside = !ab;
    for (int a = 0; a < dr; ++a) inside &= fabs(rr[a]) < 1.0 - INTERIOR_TOL;
    if (inside) { *it = it1; return; }
    invert_core(m->B, d, dr, X, xs, &m->newton, NULL, 0, rr, dd, it, cv, NULL);
    *it += it1;
    return;
  }
  invert_core(m->B, d, dr, X, xs, &m->newton, NULL, 0, rr, dd, it, cv, NULL);
}

/* engine.find Phase A: candidates from
 * the local map in ascending element id, AABB then OBB filter, Newton,
 * first INTERIOR wins, else min-d* BORDER (ties -> lower id), else
 * NOT_FOUND.  Records: code, elem, r[dr], dist; diagnostics: iters (sum
 * over Newton-ed candidates), ncand (Newton-ed candidates), nbox (box
 * tests). */
void fpxo_find(const fpxo_mesh* m, int64_t n, const double* x, int32_t* code, int32_t* elem,
               double* r, double* dist, int32_t* iters, int32_t* ncand, int32_t* nbox,
               int nthreads) {
  int d = m->d, dr = m->dr;
  
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t k = 0; k < n; ++k) {
    const double* xs = x + k * d;
    int bc = FPXO_NOT_FOUND, be = -1, tot = 0, nc = 0, nb = 0;
    double br[3] = {NAN, NAN, NAN}, bd = INFINITY;
    int64_t cell = cell_of(d, m->grid, m->ncell, xs, NULL);
    if (cell >= 0) {
      for (int32_t q = m->offsets[cell]; q < m->offsets[cell + 1]; ++q) {
        int32_t e = m->elems[q];
        ++nb;
        if (!aabb_contains(d, m->aabb + (int64_t)e * 2 * d, xs)) continue;
        if (m->obb_ok[e] && !obb_contains(d, m->obb_c + (int64_t)e * d,
                                          m->obb_inv + (int64_t)e * d * d, xs)) continue;
        double rr[3], dd;
        int it, cv;
        candidate_solve(m, e, xs, rr, &dd, &it, &cv);
        tot += it;
        ++nc;
        double eps_d = 0.0;
        if (dr < d) {
          if (m->eps_d_abs >= 0.0) eps_d = m->eps_d_abs;
          else {
            const double* bx = m->aabb + (int64_t)e * 2 * d;
            double s = 0.0;
            for (int c = 0; c < d; ++c) s += (bx[d + c] - bx[c]) * (bx[d + c] - bx[c]);
            eps_d = m->eps_d_rel * sqrt(s);
          }
        }
        int c = classify(d, dr, rr, dd, eps_d);
        if (c == FPXO_INTERIOR) {
          bc = c; be = e; bd = dd;
          for (int a = 0; a < dr; ++a) br[a] = rr[a];
          break;
        }
        if (dd < bd) {
          bc = FPXO_BORDER; be = e; bd = dd;
          for (int a = 0; a < dr; ++a) br[a] = rr[a];
        }
      }
    }
    code[k] = bc;
    elem[k] = be;
    for (int a = 0; a < dr; ++a) r[k * dr + a] = bc == FPXO_NOT_FOUND ? NAN : br[a];
    dist[k] = bc == FPXO_NOT_FOUND ? NAN : bd;
    if (iters) iters[k] = tot;
    if (ncand) ncand[k] = nc;
    if (nbox) nbox[k] = nb;
  }
}

/* engine.interpolate, local part (basis.py:285-303):
 * field [E][C][Nf^dr]; NOT_FOUND -> NaN (D12). */
void fpxo_eval(const fpxo_basis* Bf, int dr, int C, const double* field, int64_t n,
               const int32_t* code, const int32_t* elem, const double* r, double* out,
               int nthreads) {
  int N = Bf->N;
  int K = dr == 1 ? N : (dr == 2 ? N * N : N * N * N);
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < n; ++k) {
    if (code[k] == FPXO_NOT_FOUND || elem[k] < 0) {
      for (int c = 0; c < C; ++c) out[k * C + c] = NAN;
      continue;
    }
    double v[3][FPXO_MAXN], g[FPXO_MAXN];
    for (int a = 0; a < dr; ++a) fpxo_lagrange1(Bf, r[k * dr + a], v[a], g, NULL);
    const double* u = field + (int64_t)elem[k] * C * K;
    for (int c = 0; c < C; ++c)
      out[k * C + c] = contract(u + c * K, N, dr, v[0], dr > 1 ? v[1] : NULL, dr > 2 ? v[2] : NULL);
  }
}

int fpxo_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
