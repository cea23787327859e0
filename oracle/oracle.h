/*
 * oracle.h -- plain, slow, obviously-correct CPU reference of the eNMF hot path
 * (arxiv 2605.19325, "An Exterior Method for Nonnegative Matrix Factorization").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load liboracle.so.  It shares no code,
 * header, table or helper with the CUDA product path (paper_2605_19325_b200/).
 *
 * Arithmetic: IEEE fp64 throughout (X is read as fp32 bytes and promoted per
 * element).  Plain loops, no BLAS, no blocking; every sum runs sequentially in
 * index order, so results do not depend on the OpenMP thread count.
 *
 * Orientation (SURVEY.md reading R1): X is m x n row-major, U is m x r, V is n x r,
 * all row-major.  P := X V (m x r), Q := X^T U (n x r), G_U := U^T U, G_V := V^T V.
 *
 * Every function cites the PAPER.md passage it writes out.  Readings of silent or
 * ambiguous passages (R-numbers) are listed in DESIGN.md §3.
 */
#ifndef ENMF_ORACLE_H
#define ENMF_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- products (cross terms XV, X^T U and the Grams) ---- */
void or_xv(const float* X, int64_t m, int64_t n, const double* V, int r, double* P);
void or_xtu(const float* X, int64_t m, int64_t n, const double* U, int r, double* Q);
void or_gram(const double* A, int64_t rows, int r, double* G);

/* ---- objective, Eq.(1) PAPER.md:108-110 (reported un-halved, reading R2) ---- */
double or_frob2_direct(const float* X, int64_t m, int64_t n, const double* U,
                       const double* V, int r);
double or_frob2_trace(const float* X, int64_t m, int64_t n, const double* U,
                      const double* V, int r);
double or_xnorm2(const float* X, int64_t m, int64_t n);
double or_negativity(const double* A, int64_t count);   /* sum h(a), h(q)=max(0,-q) */

/* ---- dense small linear algebra ---- */
/* One-sided Jacobi SVD of A (rows x k, row-major, rows >= k): A = Uo diag(s) Vo^T,
 * s descending.  Uo (rows x k) and Vo (k x k) may be NULL.  Returns sweeps used. */
int or_svd_jacobi(const double* A, int64_t rows, int k, double* Uo, double* s, double* Vo);
/* Orthonormalise the columns of Y (rows x l) in place: modified Gram-Schmidt, twice. */
void or_orthonormalise(double* Y, int64_t rows, int l);

/* ---- truncated SVD with balanced scaling, PAPER.md:135 (U*=U S^1/2, V*=V S^1/2) ----
 * Block subspace iteration (block l = min(r+p, m, n)) + Rayleigh-Ritz until the r
 * leading Ritz values change by < tol * sigma_1 (reading R3).  Sign rule R5.
 * Returns the iteration count (negative if max_iter was hit without convergence). */
int or_truncated_svd(const float* X, int64_t m, int64_t n, int r, int p, double tol,
                     int max_iter, double* Ustar, double* Vstar, double* sigma);

/* ---- Alg. 1 ADMM rotation, PAPER.md:164-193 (Z-update Eq.7, Procrustes R=CD^T) ----
 * W: rows x r (rows = m+n), R out r x r.  rho <= 0 selects reading R7
 * (1/rho = 1000 max|W|).  neg_trace[t] = negativity(W R^(t)) if not NULL.
 * Returns the number of Z entries that took the third branch of Eq.(7). */
double or_zprox(double b, double rho);                               /* Eq.(7) */
void or_procrustes(const double* W, const double* B, int64_t rows, int r, double* R);
int64_t or_admm_rotate(const double* W, int64_t rows, int r, double rho, int T, double* R,
                       double* neg_trace);

/* ---- post-rotation variant "direct projection onto the nonnegative orthant" (ablation,
 * PAPER.md:2096-2099, Table ablation_projection (ii)): A <- max(0, A) elementwise ---- */
void or_project(double* A, int64_t count);

/* ---- feasibility stage, Alg. 2 PAPER.md:230-244 ---- */
void or_lift(double* A, int64_t count, double lam);             /* Eq.(6)/(7) */
/* PBCD on F (rows x r) with fixed cross term C (rows x r) and Gram G (r x r):
 * grad = F G - C (= (U V^T - X) V for the U block), masked by M (1 = free).
 * Returns inner iterations performed; pg0/pg_last out (may be NULL). */
int or_pbcd(double* F, int64_t rows, int r, const double* C, const double* G,
            const unsigned char* M, double eps, int max_iter, double* pg0, double* pg_last);
/* Same with the step rule as a parameter: step <= 0 Eq.(10), step > 0 fixed (ablation
 * "fixed step size"; reading R29). */
int or_pbcd_step(double* F, int64_t rows, int r, const double* C, const double* G,
                 const unsigned char* M, double eps, int max_iter, double step, double* pg0,
                 double* pg_last);
/* One projected-gradient step F <- max(0, F - step (F G - C)) ("standard gradient descent"
 * of the ablation; reading R29), and lambda_max of a PSD Gram. */
void or_pgd(double* F, int64_t rows, int r, const double* C, const double* G, double step);
double or_lambda_max(const double* G, int r);
/* HALS column sweep (cited PAPER.md:322-324, 341; reading R12). */
void or_hals(double* F, int64_t rows, int r, const double* C, const double* G);

/* ---- Alg. 3 eNMF, PAPER.md:326-345 ---- */
typedef struct {
  int r;
  int oversample;      /* p (reading R3), default 10 */
  double svd_tol;      /* default 1e-13 */
  int svd_max_iter;    /* default 500 */
  int admm_iters;      /* T_admm (reading R8), default 100 */
  double admm_rho;     /* <=0: reading R7 */
  int lift_steps;      /* L (reading R9), default 10 */
  double pbcd_eps;     /* default 1e-2 (R10) */
  int pbcd_max_iter;   /* default 50 (R10) */
  int round_f32;       /* 1: the factor state is stored in fp32 at block boundaries, as the
                          C-ABI stores U and V (reading R26); 0: fp64 state throughout */
  int step_rule;       /* ascent step: 0 Eq.(10) optimal d_i, 1 fixed 1 / lambda_max(G) (R29) */
  int descent;         /* descent stage: 0 HALS, 1 projected gradient, step 1 / lambda_max (R29) */
} or_options_t;

typedef struct {
  int stage;           /* 0 ascent, 1 HALS */
  double lambda_u, lambda_v;
  int sweeps_done;
} or_state_t;

/* lambda = (1 + 1e-3) |min A| / L, 0 if A has no negative entry (reading R9). */
double or_lift_constant(const double* A, int64_t count, int L);

/* One sweep (U block then V block), ascent or HALS by stage control.
 * Writes pbcd inner counts (U, V) to iters[2] if not NULL.  Returns the stage used. */
int or_sweep(const float* X, int64_t m, int64_t n, double* U, double* V,
             const or_options_t* opt, or_state_t* st, int* iters);

/* Full Alg. 3: truncated SVD, rotation, n_sweeps sweeps.  f_trace[t] = direct f
 * after sweep t (may be NULL).  sigma out (r) may be NULL.  Returns 0 on success. */
int or_enmf(const float* X, int64_t m, int64_t n, const or_options_t* opt, int n_sweeps,
            double* U, double* V, double* sigma, double* f_trace, or_state_t* st_out);

/* ---- KKT residuals, App. G PAPER.md:1475-1487 ----
 * out[0] min U, [1] min V, [2] comp_max = max|grad (.) W|, [3] comp_sum = sum|grad (.) W|,
 * [4] delta_W = max(grad (.) W), [5] sigma_W = sum(grad (.) W) (Table 10's tuple),
 * [6] dual_viol = max(0, -min grad), [7] ||X||_F^2, [8] rms of [XV; X^T U]. */
void or_kkt(const float* X, int64_t m, int64_t n, const double* U, const double* V, int r,
            double* out);

/* ---- eNMC, exterior nonnegative matrix completion (App. C; Alg. NMC)
 * -- oracle_nmc.c.  Observed entries of X as CSR lists (ptr: rows + 1, idx ascending within
 * a row, val); unlisted entries are missing.  Readings R30-R32. ---- */
double or_nmc_objective(const int64_t* ptr, const int32_t* idx, const float* val, int64_t m,
                        const double* U, const double* V, int r);
void or_nmc_grad(const int64_t* ptr, const int32_t* idx, const float* val, int64_t rows,
                 const double* F, const double* O, int r, double* grad);
int or_nmc_pbcd(const int64_t* ptr, const int32_t* idx, const float* val, int64_t rows,
                double* F, const double* O, int r, const unsigned char* M, double eps,
                int max_iter, double* pg0_out, double* pg_out);
void or_csr_transpose(const int64_t* ptr, const int32_t* idx, const float* val, int64_t m,
                      int64_t n, int64_t* tptr, int32_t* tidx, float* tval);
void or_nmc_sweep(const int64_t* ptr, const int32_t* idx, const float* val,
                  const int64_t* tptr, const int32_t* tidx, const float* tval, int64_t m,
                  int64_t n, double* U, double* V, int r, double lambda_u, double lambda_v,
                  double eps, int max_iter, int round32, int* iters);
int or_softimpute(const int64_t* ptr, const int32_t* idx, const float* val, int64_t m,
                  int64_t n, int r, const double* U0, int iters, double* A, double* B,
                  double* d);

#ifdef __cplusplus
}
#endif
#endif
