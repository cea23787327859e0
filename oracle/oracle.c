/*
 * oracle.c -- CPU fp64 reference of the eNMF hot path.  TEST INFRASTRUCTURE ONLY
 * (see oracle.h for the rules: no code shared with the CUDA path, plain loops,
 * sequential sums in index order, results independent of the thread count).
 *
 * Parity status: every function below is pinned by a `-m "not gpu"`
 * test in tests/test_oracle_pins.py, except the whole multi-sweep trajectory of
 * or_enmf beyond those pins ("parity unpinned" for the trajectory as such: the
 * paper prints no per-iteration values).
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define IDX(i, j, ld) ((int64_t)(i) * (int64_t)(ld) + (int64_t)(j))

/* ------------------------------------------------------------------------- */
/* Products: the cross terms XV, X^T U and the Grams.   */
/* ------------------------------------------------------------------------- */

/* P = X V: P_ik = sum_j X_ij V_jk, j ascending. */
void or_xv(const float* X, int64_t m, int64_t n, const double* V, int r, double* P) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i) {
    for (int k = 0; k < r; ++k) {
      double s = 0.0;
      for (int64_t j = 0; j < n; ++j) s += (double)X[IDX(i, j, n)] * V[IDX(j, k, r)];
      P[IDX(i, k, r)] = s;
    }
  }
}

/* Q = X^T U: Q_jk = sum_i X_ij U_ik, i ascending. */
void or_xtu(const float* X, int64_t m, int64_t n, const double* U, int r, double* Q) {
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < n; ++j) {
    for (int k = 0; k < r; ++k) {
      double s = 0.0;
      for (int64_t i = 0; i < m; ++i) s += (double)X[IDX(i, j, n)] * U[IDX(i, k, r)];
      Q[IDX(j, k, r)] = s;
    }
  }
}

/* G = A^T A: G_kl = sum_i A_ik A_il, i ascending. */
void or_gram(const double* A, int64_t rows, int r, double* G) {
  for (int k = 0; k < r; ++k)
    for (int l = 0; l < r; ++l) {
      double s = 0.0;
      for (int64_t i = 0; i < rows; ++i) s += A[IDX(i, k, r)] * A[IDX(i, l, r)];
      G[IDX(k, l, r)] = s;
    }
}

/* ------------------------------------------------------------------------- */
/* Objective, Eq.(1) PAPER.md:108-110.  Reported as ||X - U V^T||_F^2.       */
/* ------------------------------------------------------------------------- */

double or_xnorm2(const float* X, int64_t m, int64_t n) {
  double s = 0.0;
  for (int64_t e = 0; e < m * n; ++e) s += (double)X[e] * (double)X[e];
  return s;
}

/* Direct definition: sum_ij (X_ij - sum_k U_ik V_jk)^2.  Row sums run in parallel
 * (each sequential in j) and are added in row order afterwards. */
double or_frob2_direct(const float* X, int64_t m, int64_t n, const double* U,
                       const double* V, int r) {
  double* rows = (double*)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i) {
    double s = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      double uv = 0.0;
      for (int k = 0; k < r; ++k) uv += U[IDX(i, k, r)] * V[IDX(j, k, r)];
      double e = (double)X[IDX(i, j, n)] - uv;
      s += e * e;
    }
    rows[i] = s;
  }
  double f = 0.0;
  for (int64_t i = 0; i < m; ++i) f += rows[i];
  free(rows);
  return f;
}

/* Trace form ||X||^2 - 2<U, XV> + <U^T U, V^T V> (BASELINE.json:5). */
double or_frob2_trace(const float* X, int64_t m, int64_t n, const double* U,
                      const double* V, int r) {
  double* P = (double*)malloc(sizeof(double) * (size_t)m * r);
  double* GU = (double*)malloc(sizeof(double) * (size_t)r * r);
  double* GV = (double*)malloc(sizeof(double) * (size_t)r * r);
  or_xv(X, m, n, V, r, P);
  or_gram(U, m, r, GU);
  or_gram(V, n, r, GV);
  double cross = 0.0, gg = 0.0;
  for (int64_t e = 0; e < m * r; ++e) cross += U[e] * P[e];
  for (int64_t e = 0; e < (int64_t)r * r; ++e) gg += GU[e] * GV[e];
  double f = or_xnorm2(X, m, n) - 2.0 * cross + gg;
  free(P);
  free(GU);
  free(GV);
  return f;
}

/* sum_ij h(A_ij), h(q) = max(0, -q). */
double or_negativity(const double* A, int64_t count) {
  double s = 0.0;
  for (int64_t e = 0; e < count; ++e) s += A[e] < 0.0 ? -A[e] : 0.0;
  return s;
}

/* PAPER.md:2096-2099 (Table ablation_projection, variant (ii)): "direct projection onto the
 * nonnegative orthant" -- the Euclidean projection, entrywise max{0, a}. */
void or_project(double* A, int64_t count) {
  for (int64_t e = 0; e < count; ++e)
    if (A[e] < 0.0) A[e] = 0.0;
}

/* ------------------------------------------------------------------------- */
/* Dense small linear algebra.                                               */
/* ------------------------------------------------------------------------- */

/* Hestenes one-sided Jacobi: rotate column pairs of B = A (a copy) until all pairs are
 * orthogonal to 1e-15 relative; J accumulates the rotations, so A J = B, and
 * A = (B diag(1/s)) diag(s) J^T with s_k = ||B_:k||. */
int or_svd_jacobi(const double* A, int64_t rows, int k, double* Uo, double* s, double* Vo) {
  double* B = (double*)malloc(sizeof(double) * (size_t)rows * k);
  double* J = (double*)malloc(sizeof(double) * (size_t)k * k);
  memcpy(B, A, sizeof(double) * (size_t)rows * k);
  for (int a = 0; a < k; ++a)
    for (int b = 0; b < k; ++b) J[IDX(a, b, k)] = a == b ? 1.0 : 0.0;
  int sweep;
  for (sweep = 1; sweep <= 100; ++sweep) {
    int rotated = 0;
    for (int p = 0; p < k - 1; ++p)
      for (int q = p + 1; q < k; ++q) {
        double alpha = 0.0, beta = 0.0, gamma = 0.0;
        for (int64_t i = 0; i < rows; ++i) {
          double bp = B[IDX(i, p, k)], bq = B[IDX(i, q, k)];
          alpha += bp * bp;
          beta += bq * bq;
          gamma += bp * bq;
        }
        if (gamma == 0.0 || fabs(gamma) <= 1e-15 * sqrt(alpha * beta)) continue;
        rotated = 1;
        double zeta = (beta - alpha) / (2.0 * gamma);
        double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        double c = 1.0 / sqrt(1.0 + t * t);
        double sn = c * t;
        for (int64_t i = 0; i < rows; ++i) {
          double bp = B[IDX(i, p, k)], bq = B[IDX(i, q, k)];
          B[IDX(i, p, k)] = c * bp - sn * bq;
          B[IDX(i, q, k)] = sn * bp + c * bq;
        }
        for (int a = 0; a < k; ++a) {
          double jp = J[IDX(a, p, k)], jq = J[IDX(a, q, k)];
          J[IDX(a, p, k)] = c * jp - sn * jq;
          J[IDX(a, q, k)] = sn * jp + c * jq;
        }
      }
    if (!rotated) break;
  }
  /* column norms, then a stable selection sort into descending order */
  double* nrm = (double*)malloc(sizeof(double) * (size_t)k);
  int* ord = (int*)malloc(sizeof(int) * (size_t)k);
  for (int c = 0; c < k; ++c) {
    double t = 0.0;
    for (int64_t i = 0; i < rows; ++i) t += B[IDX(i, c, k)] * B[IDX(i, c, k)];
    nrm[c] = sqrt(t);
    ord[c] = c;
  }
  for (int a = 0; a < k; ++a) {
    int best = a;
    for (int b = a + 1; b < k; ++b)
      if (nrm[ord[b]] > nrm[ord[best]]) best = b;
    int tmp = ord[a];
    ord[a] = ord[best];
    ord[best] = tmp;
  }
  for (int a = 0; a < k; ++a) {
    int c = ord[a];
    if (s) s[a] = nrm[c];
    if (Vo)
      for (int b = 0; b < k; ++b) Vo[IDX(b, a, k)] = J[IDX(b, c, k)];
    if (Uo)
      for (int64_t i = 0; i < rows; ++i)
        Uo[IDX(i, a, k)] = nrm[c] > 0.0 ? B[IDX(i, c, k)] / nrm[c] : 0.0;
  }
  if (Uo) {
    /* complete the left basis for zero singular values (rank-deficient A) */
    for (int a = 0; a < k; ++a) {
      if (nrm[ord[a]] > 0.0) continue;
      for (int64_t e = 0; e < rows; ++e) {
        for (int64_t i = 0; i < rows; ++i) Uo[IDX(i, a, k)] = i == e ? 1.0 : 0.0;
        for (int pass = 0; pass < 2; ++pass)
          for (int b = 0; b < k; ++b) {
            if (b == a || (nrm[ord[b]] <= 0.0 && b > a)) continue;
            double d = 0.0;
            for (int64_t i = 0; i < rows; ++i) d += Uo[IDX(i, b, k)] * Uo[IDX(i, a, k)];
            for (int64_t i = 0; i < rows; ++i) Uo[IDX(i, a, k)] -= d * Uo[IDX(i, b, k)];
          }
        double t = 0.0;
        for (int64_t i = 0; i < rows; ++i) t += Uo[IDX(i, a, k)] * Uo[IDX(i, a, k)];
        if (t > 1e-6) {
          t = sqrt(t);
          for (int64_t i = 0; i < rows; ++i) Uo[IDX(i, a, k)] /= t;
          break;
        }
      }
    }
  }
  free(nrm);
  free(ord);
  free(B);
  free(J);
  return sweep;
}

/* Modified Gram-Schmidt, applied twice ("twice is enough"). */
void or_orthonormalise(double* Y, int64_t rows, int l) {
  for (int pass = 0; pass < 2; ++pass)
    for (int c = 0; c < l; ++c) {
      for (int b = 0; b < c; ++b) {
        double d = 0.0;
        for (int64_t i = 0; i < rows; ++i) d += Y[IDX(i, b, l)] * Y[IDX(i, c, l)];
        for (int64_t i = 0; i < rows; ++i) Y[IDX(i, c, l)] -= d * Y[IDX(i, b, l)];
      }
      double t = 0.0;
      for (int64_t i = 0; i < rows; ++i) t += Y[IDX(i, c, l)] * Y[IDX(i, c, l)];
      t = sqrt(t);
      for (int64_t i = 0; i < rows; ++i) Y[IDX(i, c, l)] = t > 0.0 ? Y[IDX(i, c, l)] / t : 0.0;
    }
}

/* X Z for Z (n x l): Y (m x l). */
static void mul_x(const float* X, int64_t m, int64_t n, const double* Z, int l, double* Y) {
  or_xv(X, m, n, Z, l, Y);
}
static void mul_xt(const float* X, int64_t m, int64_t n, const double* Qm, int l, double* Z) {
  or_xtu(X, m, n, Qm, l, Z);
}

/* ------------------------------------------------------------------------- */
/* Truncated SVD with balanced scaling: PAPER.md:135 and Alg. 3 line 331.     */
/* ------------------------------------------------------------------------- */
int or_truncated_svd(const float* X, int64_t m, int64_t n, int r, int p, double tol,
                     int max_iter, double* Ustar, double* Vstar, double* sigma) {
  int64_t mn = m < n ? m : n;
  int l = r + p;
  if (l > mn) l = (int)mn;
  if (r < 1 || r > l) return -1000000;
  double* Qm = (double*)malloc(sizeof(double) * (size_t)m * l);
  double* Z = (double*)malloc(sizeof(double) * (size_t)n * l);
  double* Bt = (double*)malloc(sizeof(double) * (size_t)n * l);   /* B^T = X^T Q */
  double* Ub = (double*)malloc(sizeof(double) * (size_t)n * l);   /* left sv of B^T */
  double* Jv = (double*)malloc(sizeof(double) * (size_t)l * l);
  double* s = (double*)malloc(sizeof(double) * (size_t)l);
  double* sprev = (double*)calloc((size_t)l, sizeof(double));
  /* deterministic start block (any full-rank start converges; reading R3) */
  uint64_t st = 0x9E3779B97F4A7C15ull;
  for (int64_t e = 0; e < m * l; ++e) {
    st ^= st << 13; st ^= st >> 7; st ^= st << 17;
    Qm[e] = (double)(st >> 11) * (1.0 / 9007199254740992.0) - 0.5;
  }
  or_orthonormalise(Qm, m, l);
  int it, conv = 0;
  for (it = 1; it <= max_iter; ++it) {
    /* subspace iteration: Z = orth(X^T Q), Q = orth(X Z) */
    mul_xt(X, m, n, Qm, l, Z);
    or_orthonormalise(Z, n, l);
    mul_x(X, m, n, Z, l, Qm);
    or_orthonormalise(Qm, m, l);
    /* Rayleigh-Ritz: B^T = X^T Q (n x l) = Ub diag(s) Jv^T */
    mul_xt(X, m, n, Qm, l, Bt);
    or_svd_jacobi(Bt, n, l, Ub, s, Jv);
    double dmax = 0.0;
    for (int k = 0; k < r; ++k) {
      double d = fabs(s[k] - sprev[k]);
      if (d > dmax) dmax = d;
    }
    memcpy(sprev, s, sizeof(double) * (size_t)l);
    if (it > 1 && dmax <= tol * s[0]) { conv = 1; break; }
  }
  /* X ~= Q B = Q Jv diag(s) Ub^T: left vectors Q Jv, right vectors Ub. */
  for (int k = 0; k < r; ++k) {
    /* sign rule R5: largest |.| entry of the left vector positive (ties: lowest index) */
    double best = -1.0, bval = 0.0;
    for (int64_t i = 0; i < m; ++i) {
      double u = 0.0;
      for (int c = 0; c < l; ++c) u += Qm[IDX(i, c, l)] * Jv[IDX(c, k, l)];
      if (fabs(u) > best) { best = fabs(u); bval = u; }
    }
    double sg = bval < 0.0 ? -1.0 : 1.0;
    double sq = sqrt(s[k]);
    for (int64_t i = 0; i < m; ++i) {
      double u = 0.0;
      for (int c = 0; c < l; ++c) u += Qm[IDX(i, c, l)] * Jv[IDX(c, k, l)];
      Ustar[IDX(i, k, r)] = sg * u * sq;
    }
    for (int64_t j = 0; j < n; ++j) Vstar[IDX(j, k, r)] = sg * Ub[IDX(j, k, l)] * sq;
    if (sigma) sigma[k] = s[k];
  }
  free(Qm); free(Z); free(Bt); free(Ub); free(Jv); free(s); free(sprev);
  return conv ? it : -(it - 1);
}

/* ------------------------------------------------------------------------- */
/* Alg. 1: ADMM for min sum h(Z) s.t. Z = W R, R^T R = I. */
/* Scaled dual Yh = Y / rho.                                                 */
/* ------------------------------------------------------------------------- */
/* Eq.(7): argmin_z h(z) + (rho/2)(z - b)^2, h(q) = max(0, -q). */
double or_zprox(double b, double rho) {
  if (b > 0.0) return b;
  if (b >= -1.0 / rho) return 0.0;
  return b + 1.0 / rho;
}

/* Orthogonal Procrustes: R = C D^T with W^T B = C S D^T. */
void or_procrustes(const double* W, const double* B, int64_t rows, int r, double* R) {
  double* M = (double*)malloc(sizeof(double) * (size_t)r * r);
  double* C = (double*)malloc(sizeof(double) * (size_t)r * r);
  double* D = (double*)malloc(sizeof(double) * (size_t)r * r);
  double* sv = (double*)malloc(sizeof(double) * (size_t)r);
  for (int a = 0; a < r; ++a)
    for (int b = 0; b < r; ++b) {
      double sacc = 0.0;
      for (int64_t i = 0; i < rows; ++i) sacc += W[IDX(i, a, r)] * B[IDX(i, b, r)];
      M[IDX(a, b, r)] = sacc;
    }
  or_svd_jacobi(M, r, r, C, sv, D);
  for (int a = 0; a < r; ++a)
    for (int b = 0; b < r; ++b) {
      double sacc = 0.0;
      for (int c = 0; c < r; ++c) sacc += C[IDX(a, c, r)] * D[IDX(b, c, r)];
      R[IDX(a, b, r)] = sacc;
    }
  free(M); free(C); free(D); free(sv);
}

int64_t or_admm_rotate(const double* W, int64_t rows, int r, double rho, int T, double* R,
                       double* neg_trace) {
  if (rho <= 0.0) {                         /* reading R7 */
    double wmax = 0.0;
    for (int64_t e = 0; e < rows * r; ++e) wmax = fabs(W[e]) > wmax ? fabs(W[e]) : wmax;
    rho = wmax > 0.0 ? 1e-3 / wmax : 1.0;
  }
  const double inv_rho = 1.0 / rho;
  double* Yh = (double*)calloc((size_t)(rows * r), sizeof(double));
  double* Z = (double*)malloc(sizeof(double) * (size_t)rows * r);
  double* WR = (double*)malloc(sizeof(double) * (size_t)rows * r);
  double* Bm = (double*)malloc(sizeof(double) * (size_t)rows * r);
  int64_t third = 0;
  for (int a = 0; a < r; ++a)
    for (int b = 0; b < r; ++b) R[IDX(a, b, r)] = a == b ? 1.0 : 0.0;   /* R^0 = I (R6) */
  for (int t = 1; t <= T; ++t) {
    /* b = W R^(k) - Y^(k)/rho ; Z-update, Eq.(7) */
    for (int64_t i = 0; i < rows; ++i)
      for (int b = 0; b < r; ++b) {
        double wr = 0.0;
        for (int c = 0; c < r; ++c) wr += W[IDX(i, c, r)] * R[IDX(c, b, r)];
        double bb = wr - Yh[IDX(i, b, r)];
        if (bb < -inv_rho) ++third;
        Z[IDX(i, b, r)] = or_zprox(bb, rho);
      }
    /* R-update: B = Z + Y/rho */
    for (int64_t e = 0; e < rows * r; ++e) Bm[e] = Z[e] + Yh[e];
    or_procrustes(W, Bm, rows, r, R);
    /* dual update Y^(k+1) = Y^(k) + rho (Z^(k+1) - W R^(k+1)), scaled */
    double neg = 0.0;
    for (int64_t i = 0; i < rows; ++i)
      for (int b = 0; b < r; ++b) {
        double wr = 0.0;
        for (int c = 0; c < r; ++c) wr += W[IDX(i, c, r)] * R[IDX(c, b, r)];
        WR[IDX(i, b, r)] = wr;
        Yh[IDX(i, b, r)] += Z[IDX(i, b, r)] - wr;
        neg += wr < 0.0 ? -wr : 0.0;
      }
    if (neg_trace) neg_trace[t - 1] = neg;
  }
  free(Yh); free(Z); free(WR); free(Bm);
  return third;
}

/* ------------------------------------------------------------------------- */
/* Feasibility stage.                                     */
/* ------------------------------------------------------------------------- */

/* Eq.(6)/(7): A_ij += rho*delta for A_ij < 0; only the product lam = rho*delta matters. */
void or_lift(double* A, int64_t count, double lam) {
  for (int64_t e = 0; e < count; ++e)
    if (A[e] < 0.0) A[e] += lam;
}

double or_lift_constant(const double* A, int64_t count, int L) {
  double mn = 0.0;
  for (int64_t e = 0; e < count; ++e) mn = A[e] < mn ? A[e] : mn;
  return mn < 0.0 ? (1.0 + 1e-3) * (-mn) / (double)L : 0.0;
}

/* ||M o (F G - C)||_F, rows in order. */
static double masked_grad_norm(const double* F, int64_t rows, int r, const double* C,
                               const double* G, const unsigned char* M) {
  double s = 0.0;
  for (int64_t i = 0; i < rows; ++i)
    for (int j = 0; j < r; ++j) {
      if (!M[IDX(i, j, r)]) continue;
      double g = -C[IDX(i, j, r)];
      for (int l = 0; l < r; ++l) g += F[IDX(i, l, r)] * G[IDX(l, j, r)];
      s += g * g;
    }
  return sqrt(s);
}

/* Alg. 2 PBCD with Eq.(8) row update and Eq.(10) step.
 * grad_U f = (U V^T - X) V = U (V^T V) - X V  (cross terms 1866-1868). */
int or_pbcd(double* F, int64_t rows, int r, const double* C, const double* G,
            const unsigned char* M, double eps, int max_iter, double* pg0_out,
            double* pg_out) {
  return or_pbcd_step(F, rows, r, C, G, M, eps, max_iter, 0.0, pg0_out, pg_out);
}

/* Alg. 2 with the step rule as a parameter: step <= 0 is Eq.(10)'s optimal row step d_i;
 * step > 0 a fixed step for every row -- the "fixed step size" feasibility variant of the
 * ablation (Table ablation_stepsize; reading R29: step = 1 / lambda_max(G)). */
int or_pbcd_step(double* F, int64_t rows, int r, const double* C, const double* G,
                 const unsigned char* M, double eps, int max_iter, double step, double* pg0_out,
                 double* pg_out) {
  double* grad = (double*)malloc(sizeof(double) * (size_t)r);
  double* g = (double*)malloc(sizeof(double) * (size_t)r);
  double pg0 = masked_grad_norm(F, rows, r, C, G, M);   /* line 235 */
  double pg = pg0;
  int it;
  for (it = 1; it <= max_iter; ++it) {                   /* line 237 (do-while, R10) */
    for (int64_t i = 0; i < rows; ++i) {                 /* line 238 */
      for (int j = 0; j < r; ++j) {
        double s = -C[IDX(i, j, r)];
        for (int l = 0; l < r; ++l) s += F[IDX(i, l, r)] * G[IDX(l, j, r)];
        grad[j] = s;
        g[j] = M[IDX(i, j, r)] ? s : 0.0;
      }
      /* Eq.(10): d_i = ||g_i||^2 / ||g_i V^T||^2, with ||g V^T||^2 = g (V^T V) g^T */
      double num = 0.0, den = 0.0;
      for (int j = 0; j < r; ++j) num += g[j] * g[j];
      for (int j = 0; j < r; ++j) {
        double gg = 0.0;
        for (int l = 0; l < r; ++l) gg += g[l] * G[IDX(l, j, r)];
        den += gg * g[j];
      }
      double d = step > 0.0 ? step : (den > 0.0 ? num / den : 0.0);
      /* Eq.(8): U_ij <- (U_ij - d_i grad_ij)_+ on I_+ */
      for (int j = 0; j < r; ++j)
        if (M[IDX(i, j, r)]) {
          double v = F[IDX(i, j, r)] - d * grad[j];
          F[IDX(i, j, r)] = v > 0.0 ? v : 0.0;
        }
    }
    pg = masked_grad_norm(F, rows, r, C, G, M);          /* line 241 */
    if (pg < eps * pg0) break;
  }
  if (it > max_iter) it = max_iter;
  if (pg0_out) *pg0_out = pg0;
  if (pg_out) *pg_out = pg;
  free(grad);
  free(g);
  return it;
}

/* HALS (Alg. 3): for k = 1..r,
 * F_:k <- max(0, F_:k + (C_:k - F G_:k) / G_kk), Gauss-Seidel over columns (R12). */
void or_hals(double* F, int64_t rows, int r, const double* C, const double* G) {
  for (int k = 0; k < r; ++k) {
    double gkk = G[IDX(k, k, r)];
    if (!(gkk > 0.0)) continue;
    for (int64_t i = 0; i < rows; ++i) {
      double fg = 0.0;
      for (int l = 0; l < r; ++l) fg += F[IDX(i, l, r)] * G[IDX(l, k, r)];
      double v = F[IDX(i, k, r)] + (C[IDX(i, k, r)] - fg) / gkk;
      F[IDX(i, k, r)] = v > 0.0 ? v : 0.0;
    }
  }
}

/* "Standard gradient descent" of the ablation (variants (iv)/(v); reading
 * R29): one projected-gradient step on the block, all entries of a row from the old row,
 * F <- max(0, F - step (F G - C)). */
void or_pgd(double* F, int64_t rows, int r, const double* C, const double* G, double step) {
  double* grad = (double*)malloc(sizeof(double) * (size_t)r);
  for (int64_t i = 0; i < rows; ++i) {
    for (int j = 0; j < r; ++j) {
      double s = -C[IDX(i, j, r)];
      for (int l = 0; l < r; ++l) s += F[IDX(i, l, r)] * G[IDX(l, j, r)];
      grad[j] = s;
    }
    for (int j = 0; j < r; ++j) {
      double v = F[IDX(i, j, r)] - step * grad[j];
      F[IDX(i, j, r)] = v > 0.0 ? v : 0.0;
    }
  }
  free(grad);
}

/* lambda_max of the symmetric PSD Gram G (r x r) = its largest singular value (Jacobi SVD). */
double or_lambda_max(const double* G, int r) {
  double* s = (double*)malloc(sizeof(double) * (size_t)r);
  or_svd_jacobi(G, r, r, NULL, s, NULL);
  double lm = s[0];
  free(s);
  return lm;
}

/* Reading R26: the C-ABI keeps U and V in fp32 between block updates. */
static void round_state(double* A, int64_t count, int on) {
  if (!on) return;
  for (int64_t e = 0; e < count; ++e) A[e] = (double)(float)A[e];
}

static double min_entry(const double* A, int64_t count) {
  double mn = INFINITY;
  for (int64_t e = 0; e < count; ++e) mn = A[e] < mn ? A[e] : mn;
  return mn;
}

/* One iteration of Alg. 3's loop (lines 334-340) or, once U,V >= 0, one HALS sweep
 * (line 341).  The stage is decided from the factors at entry. */
int or_sweep(const float* X, int64_t m, int64_t n, double* U, double* V,
             const or_options_t* opt, or_state_t* st, int* iters) {
  const int r = opt->r;
  double* C = (double*)malloc(sizeof(double) * (size_t)(m > n ? m : n) * r);
  double* G = (double*)malloc(sizeof(double) * (size_t)r * r);
  unsigned char* M = (unsigned char*)malloc((size_t)(m > n ? m : n) * r);
  if (st->stage == 0 && min_entry(U, m * r) >= 0.0 && min_entry(V, n * r) >= 0.0) st->stage = 1;
  int stage = st->stage;
  if (stage == 0) {
    /* U block: lift (line 335), mask (336), PBCD (337) */
    or_lift(U, m * r, st->lambda_u);
    for (int64_t e = 0; e < m * r; ++e) M[e] = U[e] >= 0.0;   /* reading R14 */
    or_xv(X, m, n, V, r, C);
    or_gram(V, n, r, G);
    int iu = or_pbcd_step(U, m, r, C, G, M, opt->pbcd_eps, opt->pbcd_max_iter,
                          opt->step_rule ? 1.0 / or_lambda_max(G, r) : 0.0, NULL, NULL);
    round_state(U, m * r, opt->round_f32);
    /* V block with X^T and the new U (lines 338-340; Eq.(11) uses U^(k+1)) */
    or_lift(V, n * r, st->lambda_v);
    for (int64_t e = 0; e < n * r; ++e) M[e] = V[e] >= 0.0;
    or_xtu(X, m, n, U, r, C);
    or_gram(U, m, r, G);
    int iv = or_pbcd_step(V, n, r, C, G, M, opt->pbcd_eps, opt->pbcd_max_iter,
                          opt->step_rule ? 1.0 / or_lambda_max(G, r) : 0.0, NULL, NULL);
    round_state(V, n * r, opt->round_f32);
    if (iters) { iters[0] = iu; iters[1] = iv; }
  } else {
    or_xv(X, m, n, V, r, C);
    or_gram(V, n, r, G);
    if (opt->descent) or_pgd(U, m, r, C, G, 1.0 / or_lambda_max(G, r));
    else or_hals(U, m, r, C, G);
    round_state(U, m * r, opt->round_f32);
    or_xtu(X, m, n, U, r, C);
    or_gram(U, m, r, G);
    if (opt->descent) or_pgd(V, n, r, C, G, 1.0 / or_lambda_max(G, r));
    else or_hals(V, n, r, C, G);
    round_state(V, n * r, opt->round_f32);
    if (iters) { iters[0] = 0; iters[1] = 0; }
  }
  st->sweeps_done += 1;
  free(C);
  free(G);
  free(M);
  return stage;
}

int or_enmf(const float* X, int64_t m, int64_t n, const or_options_t* opt, int n_sweeps,
            double* U, double* V, double* sigma, double* f_trace, or_state_t* st_out) {
  const int r = opt->r;
  for (int64_t e = 0; e < m * n; ++e)
    if (!(X[e] >= 0.0f)) return -3;                      /* X >= 0 */
  double* Us = (double*)malloc(sizeof(double) * (size_t)m * r);
  double* Vs = (double*)malloc(sizeof(double) * (size_t)n * r);
  double* W = (double*)malloc(sizeof(double) * (size_t)(m + n) * r);
  double* R = (double*)malloc(sizeof(double) * (size_t)r * r);
  /* line 331: U*, V* = SVD(X, r) */
  or_truncated_svd(X, m, n, r, opt->oversample, opt->svd_tol, opt->svd_max_iter, Us, Vs, sigma);
  /* line 332: rotation, W = [U*; V*] (Eq.3) */
  memcpy(W, Us, sizeof(double) * (size_t)m * r);
  memcpy(W + m * r, Vs, sizeof(double) * (size_t)n * r);
  or_admm_rotate(W, m + n, r, opt->admm_rho, opt->admm_iters, R, NULL);
  /* line 333: (U, V) = (U* R, V* R) */
  for (int64_t i = 0; i < m + n; ++i)
    for (int b = 0; b < r; ++b) {
      double s = 0.0;
      for (int c = 0; c < r; ++c) s += W[IDX(i, c, r)] * R[IDX(c, b, r)];
      if (i < m) U[IDX(i, b, r)] = s;
      else V[IDX(i - m, b, r)] = s;
    }
  or_state_t st;
  st.stage = 0;
  st.sweeps_done = 0;
  round_state(U, m * r, opt->round_f32);
  round_state(V, n * r, opt->round_f32);
  st.lambda_u = or_lift_constant(U, m * r, opt->lift_steps);   /* reading R9 */
  st.lambda_v = or_lift_constant(V, n * r, opt->lift_steps);
  for (int t = 0; t < n_sweeps; ++t) {
    or_sweep(X, m, n, U, V, opt, &st, NULL);
    if (f_trace) f_trace[t] = or_frob2_direct(X, m, n, U, V, r);
  }
  if (st_out) *st_out = st;
  free(Us); free(Vs); free(W); free(R);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* KKT conditions and Table 10's tuple (1486).           */
/* ------------------------------------------------------------------------- */
void or_kkt(const float* X, int64_t m, int64_t n, const double* U, const double* V, int r,
            double* out) {
  double* P = (double*)malloc(sizeof(double) * (size_t)m * r);
  double* Q = (double*)malloc(sizeof(double) * (size_t)n * r);
  double* GU = (double*)malloc(sizeof(double) * (size_t)r * r);
  double* GV = (double*)malloc(sizeof(double) * (size_t)r * r);
  or_xv(X, m, n, V, r, P);
  or_xtu(X, m, n, U, r, Q);
  or_gram(U, m, r, GU);
  or_gram(V, n, r, GV);
  double minu = min_entry(U, m * r), minv = min_entry(V, n * r);
  double cmax = 0.0, csum = 0.0, dmax = -INFINITY, dsum = 0.0, gmin = INFINITY, pq2 = 0.0;
  for (int blk = 0; blk < 2; ++blk) {
    const double* F = blk == 0 ? U : V;
    const double* Cc = blk == 0 ? P : Q;
    const double* G = blk == 0 ? GV : GU;
    int64_t rows = blk == 0 ? m : n;
    for (int64_t i = 0; i < rows; ++i)
      for (int j = 0; j < r; ++j) {
        /* grad_U f = U G_V - X V ; grad_V f = V G_U - X^T U */
        double g = -Cc[IDX(i, j, r)];
        for (int l = 0; l < r; ++l) g += F[IDX(i, l, r)] * G[IDX(l, j, r)];
        double c = g * F[IDX(i, j, r)];
        cmax = fabs(c) > cmax ? fabs(c) : cmax;
        csum += fabs(c);
        dmax = c > dmax ? c : dmax;
        dsum += c;
        gmin = g < gmin ? g : gmin;
        pq2 += Cc[IDX(i, j, r)] * Cc[IDX(i, j, r)];
      }
  }
  out[0] = minu;
  out[1] = minv;
  out[2] = cmax;
  out[3] = csum;
  out[4] = dmax;
  out[5] = dsum;
  out[6] = gmin < 0.0 ? -gmin : 0.0;
  out[7] = or_xnorm2(X, m, n);
  out[8] = sqrt(pq2 / (double)((m + n) * r));
  free(P); free(Q); free(GU); free(GV);
}
