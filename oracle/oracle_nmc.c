/*
 * oracle_nmc.c -- CPU fp64 reference of eNMC, the exterior method for nonnegative matrix
 * COMPLETION (App. C "Exterior NMC algorithm", lines 1011-1042; Alg. NMC).
 * TEST INFRASTRUCTURE ONLY (oracle.h rules: no code shared with the CUDA path, plain loops,
 * sums in index order, results independent of the thread count).
 *
 * Problem: minimise f^(U,V) = 1/2 || M_E o (X - U V^T) ||_F^2 over the
 * observed entries E of X; reported un-halved like Eq.(1) (reading R2).  The observed entries
 * are given as CSR lists (row_ptr, col_idx ascending within a row, val): a stored value is an
 * observed x_ij (possibly 0); entries not stored are MISSING (not zeros).
 *
 * Readings: R30 -- the PBCD row step for the masked problem is the exact line
 * minimiser of f^ along the masked gradient (App. B's derivation with the observed-entry
 * norm: d_i = ||g_i||^2 / sum_{j in E_i} (g_i . v_j)^2); R31 -- softImpute-ALS
 * (Hastie et al. 2015, Alg. 3.1, the paper's cited init) with lambda = 0 (the
 * unregularised f^ the paper states), a fixed iteration count, and output A = U D, B = V D
 * (balanced like U* = U S^1/2) with the sign rule R5 and D descending; R32 --
 * Alg. NMC's loop is lift + mask + PBCD on both blocks every sweep (no HALS stage: the
 * pseudocode has none; the lift changes nothing once a factor is nonnegative).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

#define IDX(i, j, ld) ((int64_t)(i) * (int64_t)(ld) + (int64_t)(j))

static double dotr(const double* a, const double* b, int r) {
  double s = 0.0;
  for (int k = 0; k < r; ++k) s += a[k] * b[k];
  return s;
}

/* f^ = sum over observed (i, j) of (x_ij - u_i . v_j)^2, rows in order, entries in order. */
double or_nmc_objective(const int64_t* ptr, const int32_t* idx, const float* val, int64_t m,
                        const double* U, const double* V, int r) {
  double s = 0.0;
  for (int64_t i = 0; i < m; ++i)
    for (int64_t e = ptr[i]; e < ptr[i + 1]; ++e) {
      const double d = (double)val[e] - dotr(U + IDX(i, 0, r), V + IDX(idx[e], 0, r), r);
      s += d * d;
    }
  return s;
}

/* grad_U f^ = (M_E o (U V^T - X)) V, written out over the observed
 * entries: row i = sum_{j in E_i} (u_i . v_j - x_ij) v_j.  For grad_V pass the transposed
 * lists (CSC of X) and swap U and V. */
void or_nmc_grad(const int64_t* ptr, const int32_t* idx, const float* val, int64_t rows,
                 const double* F, const double* O, int r, double* grad) {
  for (int64_t i = 0; i < rows; ++i) {
    double* g = grad + IDX(i, 0, r);
    for (int k = 0; k < r; ++k) g[k] = 0.0;
    for (int64_t e = ptr[i]; e < ptr[i + 1]; ++e) {
      const double* o = O + IDX(idx[e], 0, r);
      const double res = dotr(F + IDX(i, 0, r), o, r) - (double)val[e];
      for (int k = 0; k < r; ++k) g[k] += res * o[k];
    }
  }
}

/* || M o grad f^ ||_F (Alg. 2 line 241 with the masked gradient). */
static double nmc_masked_grad_norm(const int64_t* ptr, const int32_t* idx, const float* val,
                                   int64_t rows, const double* F, const double* O, int r,
                                   const unsigned char* M, double* grad) {
  or_nmc_grad(ptr, idx, val, rows, F, O, r, grad);
  double s = 0.0;
  for (int64_t e = 0; e < rows * r; ++e)
    if (M[e]) s += grad[e] * grad[e];
  return sqrt(s);
}

/* Alg. 2 with the eNMC gradient (Alg. NMC lines
 * "PBCD(X, U, V, eps, max_iter, M_U+, M_E)"): F (rows x r) is updated with the other factor
 * O fixed; M = 1 marks the free entries (M_{U+}).  Per inner iteration, for every row i:
 * grad_i over the observed entries of row i, g_i = M_i o grad_i, step d_i (reading R30),
 * F_ij <- max(0, F_ij - d_i grad_ij) on M (Eq.(8)); after all rows the masked gradient norm
 * decides the stop (do-while, reading R10).  Returns the inner iterations performed. */
int or_nmc_pbcd(const int64_t* ptr, const int32_t* idx, const float* val, int64_t rows,
                double* F, const double* O, int r, const unsigned char* M, double eps,
                int max_iter, double* pg0_out, double* pg_out) {
  double* grad = (double*)malloc(sizeof(double) * (size_t)(rows > 0 ? rows : 1) * r);
  double* gi = (double*)malloc(sizeof(double) * (size_t)r);
  double* g = (double*)malloc(sizeof(double) * (size_t)r);
  const double pg0 = nmc_masked_grad_norm(ptr, idx, val, rows, F, O, r, M, grad);
  double pg = pg0;
  int it;
  for (it = 1; it <= max_iter; ++it) {
    for (int64_t i = 0; i < rows; ++i) {
      double* f = F + IDX(i, 0, r);
      for (int k = 0; k < r; ++k) gi[k] = 0.0;
      for (int64_t e = ptr[i]; e < ptr[i + 1]; ++e) {
        const double* o = O + IDX(idx[e], 0, r);
        const double res = dotr(f, o, r) - (double)val[e];
        for (int k = 0; k < r; ++k) gi[k] += res * o[k];
      }
      double num = 0.0;
      for (int k = 0; k < r; ++k) {
        g[k] = M[IDX(i, k, r)] ? gi[k] : 0.0;
        num += g[k] * g[k];
      }
      /* exact line minimiser of f^ along -g_i: ||g_i||^2 / sum_{j in E_i} (g_i . o_j)^2 */
      double den = 0.0;
      for (int64_t e = ptr[i]; e < ptr[i + 1]; ++e) {
        const double t = dotr(g, O + IDX(idx[e], 0, r), r);
        den += t * t;
      }
      const double d = den > 0.0 ? num / den : 0.0;
      for (int k = 0; k < r; ++k)
        if (M[IDX(i, k, r)]) {
          const double v = f[k] - d * gi[k];
          f[k] = v > 0.0 ? v : 0.0;
        }
    }
    pg = nmc_masked_grad_norm(ptr, idx, val, rows, F, O, r, M, grad);
    if (pg < eps * pg0) break;
  }
  if (it > max_iter) it = max_iter;
  if (pg0_out) *pg0_out = pg0;
  if (pg_out) *pg_out = pg;
  free(grad);
  free(gi);
  free(g);
  return it;
}

/* Transposed lists (CSC of X: for every column j its observed rows ascending). */
void or_csr_transpose(const int64_t* ptr, const int32_t* idx, const float* val, int64_t m,
                      int64_t n, int64_t* tptr, int32_t* tidx, float* tval) {
  for (int64_t j = 0; j <= n; ++j) tptr[j] = 0;
  for (int64_t e = 0; e < ptr[m]; ++e) tptr[idx[e] + 1] += 1;
  for (int64_t j = 0; j < n; ++j) tptr[j + 1] += tptr[j];
  int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  for (int64_t j = 0; j < n; ++j) fill[j] = tptr[j];
  for (int64_t i = 0; i < m; ++i)
    for (int64_t e = ptr[i]; e < ptr[i + 1]; ++e) {
      const int64_t p = fill[idx[e]]++;
      tidx[p] = (int32_t)i;
      tval[p] = val[e];
    }
  free(fill);
}

static void round_f32(double* A, int64_t count, int on) {
  if (!on) return;
  for (int64_t e = 0; e < count; ++e) A[e] = (double)(float)A[e];
}

/* One eNMC sweep (Alg. NMC loop body, reading R32): lift U (Eq.(6)), mask M_{U+}, PBCD of U
 * with V fixed over the rows' observed entries; the same for V with the new U over the
 * columns' observed entries (tptr, tidx, tval: CSC of X).  iters[2] (optional) receives the
 * inner iteration counts.  The factor state is rounded to fp32 between blocks if round_f32
 * (reading R26). */
void or_nmc_sweep(const int64_t* ptr, const int32_t* idx, const float* val,
                  const int64_t* tptr, const int32_t* tidx, const float* tval, int64_t m,
                  int64_t n, double* U, double* V, int r, double lambda_u, double lambda_v,
                  double eps, int max_iter, int round32, int* iters) {
  const int64_t big = m > n ? m : n;
  unsigned char* M = (unsigned char*)malloc((size_t)(big > 0 ? big : 1) * r);
  or_lift(U, m * r, lambda_u);
  for (int64_t e = 0; e < m * r; ++e) M[e] = U[e] >= 0.0;
  const int iu = or_nmc_pbcd(ptr, idx, val, m, U, V, r, M, eps, max_iter, NULL, NULL);
  round_f32(U, m * r, round32);
  or_lift(V, n * r, lambda_v);
  for (int64_t e = 0; e < n * r; ++e) M[e] = V[e] >= 0.0;
  const int iv = or_nmc_pbcd(tptr, tidx, tval, n, V, U, r, M, eps, max_iter, NULL, NULL);
  round_f32(V, n * r, round32);
  if (iters) {
    iters[0] = iu;
    iters[1] = iv;
  }
  free(M);
}

/* softImpute-ALS (Hastie et al. 2015, Alg. 3.1) with lambda = 0 (reading R31), written out
 * with the completed matrix X* = P_E(X) + P_E-perp(A B^T) formed densely (m x n) at every
 * half step:
 *   1. U = orthonormalised U0 (m x r, the caller's random start), D = I, V = 0; A = U D,
 *      B = V D.
 *   2. B~ = X*^T U D (D^2)^-1 = X*^T U D^-1;  SVD  B~ D = V~ D~^2 R^T;  V <- V~, D <- D~,
 *      U <- U R;  B = V D, A = U D.
 *   3. A~ = X* V D^-1;  SVD  A~ D = U~ D~^2 R^T;  U <- U~, D <- D~, V <- V R;  A = U D,
 *      B = V D.
 *   4. Steps 2-3 `iters` times.
 * Output A (m x r), B (n x r) -- so that A B^T is the rank-r model -- and d = diag(D),
 * columns ordered by d descending, column signs by the rule of reading R5 (the largest-|.|
 * entry of each column of A positive, ties to the lowest row; A and B flipped together).
 * Returns 0, or -1 if a singular value of the half-step product is 0. */
int or_softimpute(const int64_t* ptr, const int32_t* idx, const float* val, int64_t m,
                  int64_t n, int r, const double* U0, int iters, double* A, double* B,
                  double* d) {
  double* U = (double*)malloc(sizeof(double) * (size_t)m * r);
  double* V = (double*)calloc((size_t)n * r, sizeof(double));
  double* D = (double*)malloc(sizeof(double) * (size_t)r);
  double* Xs = (double*)malloc(sizeof(double) * (size_t)m * n);
  double* T = (double*)malloc(sizeof(double) * (size_t)(m > n ? m : n) * r);
  double* Ls = (double*)malloc(sizeof(double) * (size_t)(m > n ? m : n) * r);
  double* Rm = (double*)malloc(sizeof(double) * (size_t)r * r);
  double* s = (double*)malloc(sizeof(double) * (size_t)r);
  double* W = (double*)malloc(sizeof(double) * (size_t)(m > n ? m : n) * r);
  int rc = 0;
  memcpy(U, U0, sizeof(double) * (size_t)m * r);
  or_orthonormalise(U, m, r);
  for (int k = 0; k < r; ++k) D[k] = 1.0;
  for (int t = 0; t < iters && rc == 0; ++t) {
    for (int half = 0; half < 2 && rc == 0; ++half) {
      /* X* = P_E(X) + P_E-perp(A B^T), A B^T = U D^2 V^T */
      for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) {
          double ab = 0.0;
          for (int k = 0; k < r; ++k) ab += U[IDX(i, k, r)] * D[k] * D[k] * V[IDX(j, k, r)];
          Xs[IDX(i, j, n)] = ab;
        }
      for (int64_t i = 0; i < m; ++i)
        for (int64_t e = ptr[i]; e < ptr[i + 1]; ++e) Xs[IDX(i, idx[e], n)] = (double)val[e];
      if (half == 0) {
        /* B~ D = X*^T U  (n x r) */
        for (int64_t j = 0; j < n; ++j)
          for (int k = 0; k < r; ++k) {
            double acc = 0.0;
            for (int64_t i = 0; i < m; ++i) acc += Xs[IDX(i, j, n)] * U[IDX(i, k, r)];
            T[IDX(j, k, r)] = acc;
          }
        or_svd_jacobi(T, n, r, Ls, s, Rm);                 /* T = V~ diag(s) R^T */
        for (int k = 0; k < r; ++k) {
          if (!(s[k] > 0.0)) rc = -1;
          D[k] = sqrt(s[k]);
        }
        memcpy(V, Ls, sizeof(double) * (size_t)n * r);
        /* U <- U R */
        for (int64_t i = 0; i < m; ++i)
          for (int k = 0; k < r; ++k) {
            double acc = 0.0;
            for (int l = 0; l < r; ++l) acc += U[IDX(i, l, r)] * Rm[IDX(l, k, r)];
            W[IDX(i, k, r)] = acc;
          }
        memcpy(U, W, sizeof(double) * (size_t)m * r);
      } else {
        /* A~ D = X* V  (m x r) */
        for (int64_t i = 0; i < m; ++i)
          for (int k = 0; k < r; ++k) {
            double acc = 0.0;
            for (int64_t j = 0; j < n; ++j) acc += Xs[IDX(i, j, n)] * V[IDX(j, k, r)];
            T[IDX(i, k, r)] = acc;
          }
        or_svd_jacobi(T, m, r, Ls, s, Rm);                 /* T = U~ diag(s) R^T */
        for (int k = 0; k < r; ++k) {
          if (!(s[k] > 0.0)) rc = -1;
          D[k] = sqrt(s[k]);
        }
        memcpy(U, Ls, sizeof(double) * (size_t)m * r);
        /* V <- V R */
        for (int64_t j = 0; j < n; ++j)
          for (int k = 0; k < r; ++k) {
            double acc = 0.0;
            for (int l = 0; l < r; ++l) acc += V[IDX(j, l, r)] * Rm[IDX(l, k, r)];
            W[IDX(j, k, r)] = acc;
          }
        memcpy(V, W, sizeof(double) * (size_t)n * r);
      }
    }
  }
  /* A = U D, B = V D; sign rule R5 on A */
  for (int k = 0; k < r; ++k) {
    int64_t arg = 0;
    double best = -1.0;
    for (int64_t i = 0; i < m; ++i)
      if (fabs(U[IDX(i, k, r)]) > best) {
        best = fabs(U[IDX(i, k, r)]);
        arg = i;
      }
    const double sg = U[IDX(arg, k, r)] < 0.0 ? -1.0 : 1.0;
    for (int64_t i = 0; i < m; ++i) A[IDX(i, k, r)] = sg * U[IDX(i, k, r)] * D[k];
    for (int64_t j = 0; j < n; ++j) B[IDX(j, k, r)] = sg * V[IDX(j, k, r)] * D[k];
    if (d) d[k] = D[k];
  }
  free(U);
  free(V);
  free(D);
  free(Xs);
  free(T);
  free(Ls);
  free(Rm);
  free(s);
  free(W);
  return rc;
}
