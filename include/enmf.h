/*
 * enmf.h -- C-ABI of the B200 (sm_100a) eNMF hot path.
 *
 * Method: "An Exterior Method for Nonnegative Matrix Factorization" (arxiv 2605.19325),
 * PAPER.md = /root/reference/PAPER.md of the build environment.  Problem (Eq.(1),
 * PAPER.md:107-110): minimise f(U,V) = 1/2 ||X - U V^T||_F^2 over U >= 0, V >= 0 for a
 * nonnegative X.  Pipeline (Alg. 3): truncated SVD with balanced scaling
 * -> ADMM orthogonal rotation toward the orthant (Alg. 1)
 * -> exterior ascent: lift + PBCD with optimal row steps (Eqs.(6)-(11), Alg. 2,
 * PAPER.md:197-244) until U, V >= 0 -> HALS descent.
 *
 * Conventions
 *   - Orientation (reading R1): X is m x n, U is m x r, V is n x r.  All
 *     matrices are fp32, row-major, with a leading dimension (elements) >= #columns.
 *   - Every pointer named without a _host suffix is a DEVICE pointer on the handle's
 *     device, except in enmf_solve_host.  X, U, V are caller-owned; U and V are updated in
 *     place; X is read only and must not change while it is bound to a handle.
 *   - Multi-GPU (SPMD, one process per GPU): rank s owns X rows [row_begin, row_begin +
 *     row_count) and the same U rows; V is replicated.  Every rank makes the same calls
 *     in the same order.  On return V is bitwise identical on all ranks.
 *   - The objective is REPORTED un-halved, ||X - U V^T||_F^2 (reading R2); gradients keep
 *     the 1/2 convention of PAPER.md:217, grad_U f = (U V^T - X) V.
 *   - All calls are ordered on the problem's CUDA stream.  Calls that return host values
 *     (arguments ending in _host) synchronise that stream before returning.
 *   - Errors: every call returns an enmf_status_t; nothing throws across the ABI.  After
 *     ENMF_ERR_CUDA / ENMF_ERR_NCCL the handle must be destroyed.
 *   - The handle owns every workspace (allocated in enmf_create / enmf_set_data), so
 *     enmf_iterate performs no allocation -- except, once per handle, the PBCD state of the
 *     ascent stage it first runs.
 */
#ifndef ENMF_H
#define ENMF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct enmf_handle_s* enmf_handle_t;

typedef enum {
  ENMF_OK = 0,
  ENMF_ERR_INVALID_ARG = -1,   /* NULL pointer, bad option value, leading dim too small */
  ENMF_ERR_SHAPE = -2,         /* r < 1, r > min(m, n), r > ENMF_MAX_RANK, bad row range */
  ENMF_ERR_NEGATIVE_X = -3,    /* X has a negative entry (PAPER.md:110 requires X >= 0) */
  ENMF_ERR_RANK_DEFICIENT = -4,/* sigma_1 = 0 (X = 0) */
  ENMF_ERR_NONFINITE = -5,     /* NaN/Inf in X or produced by an update */
  ENMF_ERR_CUDA = -6,
  ENMF_ERR_NCCL = -7,
  ENMF_ERR_OOM = -8,
  ENMF_ERR_STATE = -9          /* call out of order (e.g. iterate before set_data) */
} enmf_status_t;

#define ENMF_MAX_RANK 128

typedef struct {
  int64_t m_global;        /* rows of X */
  int64_t n;               /* columns of X */
  int64_t r;               /* factor rank, 1 <= r <= min(m, n, ENMF_MAX_RANK) */
  int64_t row_begin;       /* first X/U row owned by this rank */
  int64_t row_count;       /* X/U rows owned by this rank (m_global when world_size == 1) */
  int world_size;          /* ranks (GPUs) */
  int rank;                /* this rank */
  const void* nccl_unique_id; /* 128-byte ncclUniqueId from rank 0; NULL with world_size > 1
                              to use enmf_set_host_allreduce.  Non-NULL at world_size == 1:
                              a one-rank communicator and the sharded code path (V slice,
                              sliced pass 2, collectives) -- results equal the plain
                              single-rank path bitwise; NULL at world_size == 1: no
                              collectives at all */
  void* cuda_stream;       /* cudaStream_t for every call; NULL = legacy default stream */
} enmf_problem_t;

typedef enum {
  ENMF_PREC_AUTO = 0,      /* TC when the average rank holds >= 2.5e8 entries of X and
                              max|X| <= 64 rms(X) (decided from global statistics, the same on
                              every rank), else FP64 */
  ENMF_PREC_FP64 = 1,      /* SIMT contractions with fp64 accumulation */
  ENMF_PREC_TC = 2         /* tcgen05 kind::i8: X, V, U as three int8 digits (radix 8/8/7) of
                              a power-of-two-scaled fp32 value (one scale per X row for X V,
                              per X column for X^T U, per factor column), six digit products
                              accumulated exactly in int32 TMEM and combined in fp64; ~2^-22 of
                              each scale group's maximum per operand entry */
} enmf_precision_t;

typedef struct {
  uint64_t seed;           /* Philox key of the Gaussian test matrix Omega (randomised SVD) */
  int oversample;          /* p, block size l = r + p (reading R3); default 10 */
  int power_iters;         /* q power iterations of the range finder; default 2 */
  int admm_iters;          /* T_admm fixed ADMM steps, last iterate output (R8); default 100 */
  double admm_rho;         /* rho of Alg. 1; <= 0: 1/rho = 1000 max|W| (reading R7) */
  int lift_steps;          /* L: lift = 1.001 |min| / L, fixed at the rotated point (R9); 10 */
  double pbcd_eps;         /* epsilon of Alg. 2 (R10); default 1e-2 */
  int pbcd_max_iter;       /* max_iter of Alg. 2 (R10); default 50 */
  int precision;           /* enmf_precision_t */
  int step_rule;           /* ascent (Alg. 2) step: 0 = Eq.(10)'s optimal row step (default),
                              1 = fixed step 1 / lambda_max(G) -- the "fixed step size"
                              ablation variant (reading R29) */
  int descent;             /* descent stage: 0 = HALS (default), 1 = projected gradient with
                              step 1 / lambda_max(G) -- the "gradient descent" ablation
                              variants (reading R29) */
} enmf_options_t;

typedef struct {
  double sigma[ENMF_MAX_RANK]; /* leading singular values of X */
  int rank_deficient;      /* columns with sigma_k <= 1e-7 sigma_1 (zero-filled in U*, V*) */
  double negativity_svd;   /* sum h over [U*; V*] */
  double negativity_rot;   /* sum h over [U* R; V* R] after the last ADMM step */
  double orth_residual;    /* max |R^T R - I| */
  int64_t admm_third_branch; /* Z entries that took the third branch of Eq.(7) */
  double lambda_u, lambda_v; /* lift constants rho_u delta_u, rho_v delta_v (R9) */
  double xnorm2;           /* ||X||_F^2 */
} enmf_init_info_t;

typedef struct {
  int ascent_sweeps;       /* sweeps of this call spent in the ascent stage */
  int hals_sweeps;         /* sweeps of this call spent in HALS */
  int feasible;            /* 1 if U, V >= 0 on return */
  int pbcd_iters_u;        /* PBCD inner iterations of the last ascent U block (k*) */
  int pbcd_iters_v;        /* same for the V block */
  int hals_fallback_rows;  /* tensor-core HALS: row updates finished by the sequential fp64
                              fallback because u outgrew its digit scale (diagnostic) */
} enmf_iter_info_t;

typedef struct {
  double min_u, min_v;     /* KKT: U >= 0, V >= 0 */
  double comp_max;         /* max |grad (.) W| over W = [U; V] */
  double comp_sum;         /* sum |grad (.) W| */
  double delta_w;          /* Table 10: max(grad (.) W) */
  double sigma_w;          /* Table 10: sum(grad (.) W) */
  double dual_viol;        /* max(0, -min grad): violation of grad >= 0 */
  double xnorm2;           /* ||X||_F^2 (normaliser of comp_*) */
  double rms_cross;        /* rms of [X V; X^T U] (normaliser of dual_viol) */
} enmf_kkt_t;

/* Fill *opt with the defaults listed above. */
void enmf_default_options(enmf_options_t* opt);

/* Create a handle for one problem shape.  Validates shapes (ENMF_ERR_SHAPE), sets up the
 * NCCL communicator when nccl_unique_id is set (ENMF_ERR_NCCL), allocates workspaces
 * (ENMF_ERR_OOM).  *out is NULL on failure. */
enmf_status_t enmf_create(const enmf_problem_t* prob, const enmf_options_t* opt,
                          enmf_handle_t* out);
enmf_status_t enmf_destroy(enmf_handle_t h);

/* Bind this rank's rows of X (device, row_count x n, leading dim ldx >= n).  Computes
 * ||X||_F^2 and checks X >= 0 and finite (ENMF_ERR_NEGATIVE_X / ENMF_ERR_NONFINITE), then
 * selects the contraction path (enmf_precision_t).  On the tensor-core path it also builds the
 * handle-owned int8 digit copies of X (3 B per element) and, when device memory allows, of X^T
 * (another 3 B per element; without it X^T U gathers from the X copy, ~40 % slower) -- X
 * itself is not read again by enmf_iterate (ENMF_ERR_OOM if the X copy does not fit).
 * Resets the stage machine. */
enmf_status_t enmf_set_data(enmf_handle_t h, const float* X, int64_t ldx);

/* Sparse X (the paper's sparse Reuters experiment):
 * bind this rank's rows of X as CSR instead of a dense matrix.  row_ptr (row_count + 1,
 * int64, row_ptr[0] = 0, row_ptr[row_count] = nnz, non-decreasing), col_idx (nnz, int32,
 * strictly ascending within a row, in [0, n))
 * and vals (nnz, fp32, >= 0, finite) are DEVICE pointers, caller-owned, read-only and kept
 * (not copied) until the next set_data call or destroy; zeros not stored are zeros of X.
 * The handle builds a CSC copy for X^T U (deterministic: entries of a column in ascending
 * row order) and computes ||X||^2 over the stored values.  Every later call treats X through
 * P = X V and Q = X^T U (fp64-accumulating SpMM), so init / iterate / objective / kkt work
 * unchanged; enmf_objective(exact = 1) evaluates ||X||^2 - 2 sum_stored x_ij u_i.v_j +
 * <U^T U, V^T V>.  Block updates run on the tensor-core row kernels unless the precision
 * option is ENMF_PREC_FP64.  Errors: ENMF_ERR_INVALID_ARG (NULL pointers, a row_ptr that
 * does not start at 0 / end at nnz / decrease, column order), ENMF_ERR_SHAPE (nnz or n above 2^31 - 1), ENMF_ERR_NEGATIVE_X,
 * ENMF_ERR_NONFINITE, ENMF_ERR_OOM. */
enmf_status_t enmf_set_data_csr(enmf_handle_t h, const int64_t* row_ptr, const int32_t* col_idx,
                                const float* vals, int64_t nnz);

/* eNMC, the exterior method for nonnegative matrix COMPLETION (App. C, lines
 * 1011-1042; Alg. NMC): bind the OBSERVED entries of X as CSR lists (same layout, checks,
 * ownership and errors as enmf_set_data_csr); entries not stored are missing, and the
 * objective becomes f^ = ||M_E o (X - U V^T)||_F^2 over the observed entries (reported
 * un-halved).  Then: enmf_softimpute (the init, line 1027), enmf_rotate (Alg. 1 on its output,
 * line 1028), enmf_iterate (every sweep: lift + mask + PBCD of U over the rows' observed
 * entries, then of V over the columns', with the masked gradient (M_E o (U V^T - X)) V and
 * the exact line-minimising row step, readings R30/R32; f_trace_host receives f^),
 * enmf_objective (f^; `exact` ignored).  enmf_kkt_residual returns ENMF_ERR_STATE on such a
 * handle.  Single rank, r <= 64 (ENMF_ERR_SHAPE otherwise). */
enmf_status_t enmf_set_data_masked(enmf_handle_t h, const int64_t* row_ptr,
                                   const int32_t* col_idx, const float* vals, int64_t nnz);

/* softImpute-ALS with lambda = 0 (Hastie et al. 2015, Alg. 3.1; the eNMC init of PAPER.md:1017,
 * reading R31) on a handle bound by enmf_set_data_masked: `iters` iterations (>= 1) from the
 * start U0 (row_count x r, device, ld ldu0; orthonormalised first -- the caller supplies the
 * random start so that runs are reproducible), each a V-side and a U-side half step on the
 * completed matrix P_E(X) + P_E-perp(A B^T).  Writes A = U D into U and B = V D into V (fp32;
 * A B^T is the rank-r model, columns by D descending, sign rule R5 on A) and keeps [A; B] for
 * enmf_rotate; d_host (r values, may be NULL) receives D.  ENMF_ERR_STATE unless bound by
 * enmf_set_data_masked. */
enmf_status_t enmf_softimpute(enmf_handle_t h, const float* U0, int64_t ldu0, int iters,
                              float* U, int64_t ldu, float* V, int64_t ldv, double* d_host);

/* Rank-r truncated SVD with balanced scaling U* = U S^1/2, V* = V S^1/2 by
 * a randomised range finder (reading R3); sign rule R5.  Writes U* (this
 * rank's rows) into U and V* into V; sigma_host (r values) may be NULL. */
enmf_status_t enmf_svd(enmf_handle_t h, float* U, int64_t ldu, float* V, int64_t ldv,
                       double* sigma_host);

/* Alg. 1: rotate (U, V) <- (U R, V R) by T_admm ADMM steps from
 * R0 = I, Y0 = 0 (reading R6), then fix the lift constants from the rotated point (R9)
 * and enter the ascent stage.  info_host may be NULL. */
enmf_status_t enmf_rotate(enmf_handle_t h, float* U, int64_t ldu, float* V, int64_t ldv,
                          enmf_init_info_t* info_host);

/* RSR-ADMM (App. A, Alg. alg:rsr): the general
 * rotation-scale-rotation form of the rotation step for exact-NMF instances -- orthogonal R1,
 * R2 and a positive diagonal Lambda with U* R1 Lambda R2 >= 0 and V* R1 Lambda^-1 R2 >= 0 (Eq.
 * eq5), admm_iters iterations of the split-variable ADMM (readings R34-R37: penalties
 * rho = gamma = t = 1e-3 / max|W| unless admm_rho > 0, identity start, last iterate, the
 * lambda update's positive quartic root of least cost).  Input: (U, V) = (U*, V*) as enmf_svd
 * writes them; output U <- U* R1 Lambda R2, V <- V* R1 Lambda^-1 R2 (so U V^T is unchanged),
 * lift constants fixed from them and the ascent stage entered, as enmf_rotate.  info_host
 * (may be NULL): negativity before / after and the lift constants; lambda_host (r doubles, may
 * be NULL): Lambda.  Single rank (ENMF_ERR_STATE otherwise). */
enmf_status_t enmf_rotate_rsr(enmf_handle_t h, float* U, int64_t ldu, float* V, int64_t ldv,
                              enmf_init_info_t* info_host, double* lambda_host);

/* enmf_set_data + enmf_svd + enmf_rotate (Alg. 3). */
enmf_status_t enmf_init(enmf_handle_t h, const float* X, int64_t ldx, float* U, int64_t ldu,
                        float* V, int64_t ldv, enmf_init_info_t* info_host);

/* Post-rotation variant (ii) of the paper's ablation (Table
 * ablation_projection): "direct projection onto the nonnegative orthant followed by HALS
 * descent".  U (this rank's row_count x r, ld ldu) and V (n x r, ld ldv), device pointers,
 * caller-owned, are replaced in place by max(0, .) and the handle enters the HALS stage, so
 * the next enmf_iterate runs HALS sweeps from the projected point instead of the ascent
 * (lift + PBCD, the method's own feasibility stage).  Stream-ordered, synchronises before
 * returning.  ENMF_ERR_INVALID_ARG on NULL pointers or ld < r; V is replicated, so every rank
 * projects the same V identically. */
enmf_status_t enmf_project(enmf_handle_t h, float* U, int64_t ldu, float* V, int64_t ldv);

/* Switch the ablation variants of an existing handle (the enmf_options_t fields step_rule and
 * descent, reading R29) without rebuilding it -- a handle bound to a large X holds repacked
 * copies of X, so comparing variants on one handle avoids a second copy.  Takes effect at the
 * next enmf_iterate.  ENMF_ERR_INVALID_ARG unless both values are 0 or 1. */
enmf_status_t enmf_set_ablation(enmf_handle_t h, int step_rule, int descent);

/* Stage machine access (checkpoint/resume and shared-init parity runs): stage 0 = ascent,
 * 1 = HALS; lambda_u / lambda_v are the lift constants (reading R9). */
enmf_status_t enmf_set_stage(enmf_handle_t h, int stage, double lambda_u, double lambda_v);
enmf_status_t enmf_get_stage(enmf_handle_t h, int* stage, double* lambda_u, double* lambda_v);

/* n_iters sweeps of Alg. 3's loop: each sweep is one U block and one
 * V block, ascent (lift + mask + PBCD) while min(U) < 0 or min(V) < 0, HALS afterwards.
 * f_trace_host (n_iters doubles, may be NULL) receives ||X - U V^T||_F^2 after every
 * sweep in trace form ||X||^2 - 2<X^T U, V> + <U^T U, V^T V> (fp64 terms); on the
 * tensor-core path the terms are those of the quantised operands the X pass multiplied,
 * ||X~||^2 - 2<X~^T U~, V> + <U~^T U~, V^T V> = ||X~ - U~ V^T||^2 up to the dropped digit
 * products, which keeps the ||X||^2 / f conditioning of the trace form out of f.
 * Cache-resident problems (single rank, dense X, fp64 path, m n <= 2^26: the small
 * BASELINE configurations): every HALS sweep runs in one persistent
 * cooperative kernel (all remaining sweeps of the call in one launch), the ascent sweeps as
 * a CUDA graph each with a host check of the stage in between; the result does not depend
 * on how the caller chunks its calls.  That kernel's workspace is allocated when X is bound
 * (enmf_set_data / enmf_init).  ENMF_SMALL_FUSED=0 in the environment keeps
 * the separate launches (the path the multi-rank handle runs). */
enmf_status_t enmf_iterate(enmf_handle_t h, float* U, int64_t ldu, float* V, int64_t ldv,
                           int n_iters, double* f_trace_host, enmf_iter_info_t* info_host);

/* ||X - U V^T||_F^2 for the bound X: exact = 0 trace form (one X pass), exact = 1 direct
 * definition sum (X - U V^T)^2 (one X pass, 2mnr flops, fp64 accumulation). */
enmf_status_t enmf_objective(enmf_handle_t h, const float* U, int64_t ldu, const float* V,
                             int64_t ldv, int exact, double* f_host);

/* KKT residuals of App. G at (U, V) for the bound X. */
enmf_status_t enmf_kkt_residual(enmf_handle_t h, const float* U, int64_t ldu, const float* V,
                                int64_t ldv, enmf_kkt_t* out_host);

/* The two X passes of a sweep on their own: P = X V (this rank's
 * row_count x r, fp64, ld r) and Q = X^T U (n x r, fp64, ld r, summed over ranks), on the
 * contraction path the handle selected.  P or Q may be NULL to skip that pass. */
enmf_status_t enmf_cross_terms(enmf_handle_t h, const float* U, int64_t ldu, const float* V,
                               int64_t ldv, double* P, double* Q);

/* enmf_iterate with the factor state in HOST memory: U_host (this rank's row_count x r, ld r)
 * and V_host (n x r, ld r), updated in place (page-locked buffers make the copies
 * asynchronous).  Per call: V is uploaded on the handle's stream (the first X V pass needs
 * it), U on an internal copy stream overlapping that pass; U is downloaded behind the last V
 * block and V at the end.  Uses handle-owned device copies of U and V (allocated on the first
 * call).  Same semantics, errors and f_trace_host / info_host as enmf_iterate; synchronises. */
enmf_status_t enmf_iterate_host(enmf_handle_t h, float* U_host, float* V_host, int n_iters,
                                double* f_trace_host, enmf_iter_info_t* info_host);

/* End-to-end solve from HOST buffers (single GPU): X_host (m x n, ld = n), U_host
 * (m x r), V_host (n x r) and f_trace_host (n_iters) are host pointers.  Copies X to the
 * device through a pinned staging buffer, runs init + n_iters sweeps, copies U, V back. */
enmf_status_t enmf_solve_host(enmf_handle_t h, const float* X_host, float* U_host,
                              float* V_host, int n_iters, double* f_trace_host,
                              enmf_init_info_t* info_host);

/* Kernel launches issued by this handle since creation (instrumentation). */
int64_t enmf_launch_count(enmf_handle_t h);

/* Instrumentation of the two X passes: with profiling on, every X V and X^T U contraction
 * is bracketed by CUDA events on the handle's stream; enmf_get_profile returns the summed
 * device milliseconds ms_host[2] and pass counts count_host[2] ({X V, X^T U}) since the last
 * enmf_set_profiling call (synchronises the stream). */
enmf_status_t enmf_set_profiling(enmf_handle_t h, int on);
enmf_status_t enmf_get_profile(enmf_handle_t h, double* ms_host, int64_t* count_host);

/* Host-mediated collectives for a multi-rank handle created without an NCCL id: every
 * allreduce of the method (fp64) stages its buffer through pinned host memory and calls
 * fn(ctx, buf_host, count, op) with op 0 = sum, 1 = min, 2 = max; fn must reduce in place
 * across the ranks (same call order on every rank) and return 0.  Meant for validating the
 * sharded path (e.g. gloo ranks sharing one GPU in tests); NCCL is the production path.
 * ENMF_ERR_STATE if the handle already has an NCCL communicator. */
typedef int (*enmf_host_allreduce_fn)(void* ctx, double* buf_host, int64_t count, int op);
enmf_status_t enmf_set_host_allreduce(enmf_handle_t h, enmf_host_allreduce_fn fn, void* ctx);

/* 128-byte ncclUniqueId for a multi-GPU job (call on rank 0, broadcast the bytes, pass them
 * in enmf_problem_t.nccl_unique_id on every rank). */
enmf_status_t enmf_nccl_unique_id(void* out128);

/* Name of the contraction path selected by enmf_set_data ("fp64-simt", "tc-i8x3-exact",
 * "csr-f64-spmm", "csr-f64-spmm+tc-rows" or, for eNMC, "nmc-f64"). */
const char* enmf_precision_name(enmf_handle_t h);

const char* enmf_status_string(enmf_status_t s);

#ifdef __cplusplus
}
#endif
#endif
