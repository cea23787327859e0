// internal.h -- launchers shared by the translation units of libenmf.so (not installed).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "enmf.h"

namespace enmf {

constexpr int kSMs = 148;
constexpr int kMaxRankPad = 128;    // r padded to 32*CPL <= 128 in the row-block kernels

// Counts kernel launches issued by the library (reported by enmf_launch_count).
extern thread_local int64_t* g_launch_counter;
inline void count_launch(int n = 1) {
  if (g_launch_counter) *g_launch_counter += n;
}

// ---------------------------------------------------------------- SIMT fp64 GEMMs
// C = op(A) * B accumulated in fp64, op(A) = A (M x K, row-major, lda) or A^T where A is
// (K x M, row-major, lda).  B is K x N (row-major, ldb).  TA/TB are float or double.
// The K range is split over `splits` CTAs layers; partial results go to
// work[s*M*N + i*N + j] and are summed in split order (deterministic).  The final result
// is written to C (fp64, ldc) or, if Cf != nullptr, converted to fp32 into Cf (ldcf)
// after multiplication by colscale[j] (may be null).
struct GemmOut {
  double* C = nullptr;
  int64_t ldc = 0;
  float* Cf = nullptr;
  int64_t ldcf = 0;
  const double* colscale = nullptr;
};
template <typename TA, typename TB>
void gemm(bool transA, const TA* A, int64_t lda, const TB* B, int64_t ldb, int64_t M,
          int64_t N, int64_t K, GemmOut out, double* work, size_t work_elems,
          cudaStream_t st);

// G = A^T A (r x r fp64, ld r) of an fp32 rows x r matrix, upper-triangle tiles, fixed-order
// reduction of per-SM partials: parts >= gram_parts() * 128^2 doubles, Gu >= 128^2.
// qscale (device, r powers of two, may be null): Gram of the quantised A, entries
// rint(a s 2^15) / (s 2^15) -- the operand the tensor-core X pass multiplied.
bool gram_supported(int r);
int gram_parts();
void gram_sym(const float* A, int64_t lda, int64_t rows, int r, double* parts, double* Gu,
              double* G, cudaStream_t st, const double* qscale = nullptr);

// Deterministic sum of `parts` contiguous blocks of `len` doubles into out.
void reduce_parts(const double* parts, int nparts, int64_t len, double* out, cudaStream_t st);

// ---------------------------------------------------------------- elementwise / reductions
// sum of squares, min, non-finite count and max |.| of X (rows x n), one pass:
// writes out4 = {sum, min, nonfinite, max|X|}; parts >= 4 * nparts.
void x_stats(const float* X, int64_t ldx, int64_t rows, int64_t n, double* parts, int nparts,
             double* out4, cudaStream_t st);
int x_stats_parts(int64_t rows);
// Sparse X (kernels_sparse.cu): out (rows x ncols, ld ldo, fp64) = A B for a CSR / CSC block
// A (ptr rows + 1, idx, val) and a dense B (ld ldb); ncols any (128-column launches).
template <typename T>
void spmm(const int64_t* ptr, const int32_t* idx, const float* val, int64_t rows, const T* B,
          int64_t ldb, int ncols, double* out, int64_t ldo, cudaStream_t st);
// nonzero *bad_dev if a row range is invalid or its columns are not strictly ascending in [0, n)
int csr_check(const int64_t* ptr, const int32_t* col, int64_t rows, int64_t n, int64_t nnz,
              int* bad_dev, cudaStream_t st);
// CSC copy (colptr n + 1, rowidx, cval: nnz) of a CSR block; 0 ok, 2 out of memory / too big.
int csr_to_csc(const int64_t* ptr, const int32_t* col, const float* val, int64_t rows, int64_t n,
               int64_t nnz, int64_t* colptr, int32_t* rowidx, float* cval, cudaStream_t st);
// out = sum over stored entries x_ij (u_i . v_j); parts >= sddmm_parts(rows) doubles.
int sddmm_parts(int64_t rows);
void sddmm_dot(const int64_t* ptr, const int32_t* idx, const float* val, int64_t rows,
               const float* U, int64_t ldu, const float* V, int64_t ldv, int r, double* parts,
               double* out, cudaStream_t st);
// A <- max(0, A) in place (rows x cols, ld): post-rotation projection.
void project_f32(float* A, int64_t ld, int64_t rows, int64_t cols, cudaStream_t st);
// min over an fp32 matrix (rows x cols, ld): partials then out[0].
void min_f32(const float* A, int64_t ld, int64_t rows, int64_t cols, double* parts,
             double* out, cudaStream_t st);
// out = <A, B> (A fp64 rows x cols ld=cols, B fp32 ld) via partials.
void dot_f64_f32(const double* A, const float* B, int64_t ldb, int64_t rows, int64_t cols,
                 double* parts, double* out, cudaStream_t st);
// fp64 (ld=cols) -> fp32 strided copy with optional per-column scale.
void f64_to_f32(const double* A, int64_t rows, int64_t cols, const double* colscale,
                float* B, int64_t ldb, cudaStream_t st);
void f32_to_f64(const float* A, int64_t lda, int64_t rows, int64_t cols, double* B,
                cudaStream_t st);
// Gaussian test matrix Omega (rows x cols, fp64) from Philox4x32-10 keyed by seed.
void gaussian_fill(double* A, int64_t rows, int64_t cols, uint64_t seed, cudaStream_t st);

// ---------------------------------------------------------------- row-block updates
// HALS on F (rows x r fp32) with cross term C (rows x r fp64) and Gram G (r x r fp64).
// Runs only if *stage == want (device flag).  min partials to minparts[kRowGrid].
// colmax (optional, u64[r], zeroed by the caller): atomicMax of the fp64 bits of max |F| per
// column over the rows written -- the next X pass's digit scales without a separate scan.
constexpr int kRowGrid = 2 * kSMs;
constexpr int kRowWarps = 8;
void hals_rows(float* F, int64_t ldf, int64_t rows, int r, const double* C, const double* G,
               const int* stage, double* minparts, cudaStream_t st,
               unsigned long long* colmax = nullptr, const int* gate = nullptr);
// (gate: run only if *gate != 0 -- the device-side fallback of tc_hals_rows)
// PBCD phase A (all max_iter inner iterations, snapshots of every iterate, per-warp
// partial ||M o grad||^2 for each iteration 0..max_iter), runs only in the ascent stage.
void pbcd_rows(const float* F, int64_t ldf, int64_t rows, int r, const double* C,
               const double* G, const double* lam, int max_iter, float* snaps,
               double* pgparts, const int* stage, cudaStream_t st,
               const double* fixed_step = nullptr);   // fixed_step: device, > 0 -> fixed step
// Projected-gradient step F <- max(0, F - step (F G - C)) (ablation, R29); runs if *stage == 1.
void pgd_rows(float* F, int64_t ldf, int64_t rows, int r, const double* C, const double* G,
              const int* stage, const double* step, double* minparts, cudaStream_t st,
              unsigned long long* colmax = nullptr);
// *out = 1 / lambda_max(G) by power iteration warm-started from v (r values, updated) -- the
// fixed step of the ablation variants (R29); one CTA, r <= 128.
void lambda_power(const double* G, int r, double* v, bool warm, double* out, cudaStream_t st);
// *out = 1 / s[0] (0 if s[0] <= 0): the fixed step 1 / lambda_max from a singular-value list.
void recip_first(const double* s, double* out, cudaStream_t st);
int pbcd_parts();
// Selects k* from the partials (eps rule of Alg. 2), copies snapshot k* (row-major rows x r)
// into F and writes min partials; records k* into *kstar.
void pbcd_commit(float* F, int64_t ldf, int64_t rows, int r, const float* snaps,
                 const double* pgparts, double eps, int max_iter, int* kstar,
                 const int* stage, double* minparts, cudaStream_t st);
// Staged PBCD (tc_pbcd_chunk): the stopping rule on iterations [it0, it1] of the stage that
// read state src and wrote dst (sets *kstar, *done and the replay / commit control ctl[4]
// once it fires, or at it1 == max_iter), and the commit of the fp64 state ust[ctl[3]] into F
// with min partials / column maxima; both no-ops unless *stage == 0.
void pbcd_select_stage(const double* pgsum, int it0, int it1, int src, int dst, int max_iter,
                       double eps, int* kstar, int* done, int* ctl, const int* stage,
                       cudaStream_t st);
// (ctl == nullptr: ust0; want_stage 1: the tensor-core projected-gradient step, R29)
void pbcd_commit_state(float* F, int64_t ldf, int64_t rows, int r, const double* ust0,
                       const double* ust1, const int* ctl, const int* stage, double* minparts,
                       cudaStream_t st, unsigned long long* colmax, int want_stage = 0);
// eNMC PBCD of one block (App. C; kernels_rows.cu nmc_pbcd_kernel): F (rows x r, ld) with the
// other factor O (ld ldo) fixed, the block's observed entries as CSR lists (ptr rows + 1,
// idx, val); lift, mask, all max_iter inner iterations with snapshots and per-iteration
// ||M o grad||^2 partials into pgparts[nmc_pbcd_parts()][max_iter + 1] -- commit with
// pbcd_commit(..., tiled = false).  r <= 64.
bool nmc_supported(int r);
int nmc_pbcd_parts();
void nmc_pbcd_rows(const float* F, int64_t ldf, int64_t rows, int r, const int64_t* ptr,
                   const int32_t* idx, const float* val, const float* O, int64_t ldo,
                   const double* lam, int max_iter, float* snaps, double* pgparts,
                   cudaStream_t st);
// eNMC (nmc.cu): a softImpute-ALS half step T = S^T U + B o D (or S V + A o D) with the
// residual S = x - A B^T on the observed entries of the CSR / CSC lists (r <= 64); the
// masked objective sum (x_ij - u_i . v_j)^2 into *out (parts >= nmc_objective_parts());
// D~ = sqrt(sigma), 1 / sigma from the eigenvalues sigma^2 of T^T T.
void nmc_resid_spmm(const int64_t* ptr, const int32_t* idx, const float* val, int64_t rows,
                    int r, const double* Fr, const double* O1, const double* O2,
                    const double* dsc, double* out, cudaStream_t st);
int nmc_objective_parts();
void nmc_objective(const int64_t* ptr, const int32_t* idx, const float* val, int64_t rows, int r,
                   const float* U, int64_t ldu, const float* V, int64_t ldv, double* parts,
                   double* out, cudaStream_t st);
void nmc_svals(const double* sv, int r, double* d, double* inv, cudaStream_t st);
// RSR-ADMM (rsr.cu; App. A): per-entry updates of the split variables of
// Alg. alg:rsr over (rows x r) arrays whose first mu rows are the U block, the lambda solve
// (parts >= rsr_colsum_parts() * 4 r, abcd >= 4 r), the multiplier step and the final scaling.
int rsr_colsum_parts();
void rsr_w13(const double* WsR1, const double* W2R2, const double* M, const double* N,
             const double* W2, const double* P, const double* lam, int64_t rows, int64_t mu,
             int r, double rho, double gamma, double t, double* W1, double* W3, cudaStream_t st);
void rsr_w2(const double* W1, const double* N, const double* G, const double* lam, int64_t rows,
            int64_t mu, int r, double gamma, double t, double* W2, cudaStream_t st);
void rsr_add(const double* A, const double* B, int64_t count, double* out, cudaStream_t st);
void rsr_transpose(const double* R, int r, double* Rt, cudaStream_t st);
void rsr_lambda(const double* W1, const double* W2, const double* N, int64_t rows, int64_t mu,
                int r, double* parts, double* abcd, double* lam, cudaStream_t st);
void rsr_dual(const double* W1, const double* WsR1, const double* W2, const double* W3,
              const double* W2R2, const double* lam, int64_t rows, int64_t mu, int r, double* M,
              double* N, double* P, cudaStream_t st);
void rsr_scale(double* A, const double* lam, int64_t rows, int64_t mu, int r, cudaStream_t st);
// KKT partial statistics of one block (F, C = cross term, G): 8 values per warp slot.
void kkt_rows(const float* F, int64_t ldf, int64_t rows, int r, const double* C,
              const double* G, double* parts, cudaStream_t st);
int kkt_parts();
// Direct objective sum (X - U V^T)^2 partials.
void frob_direct(const float* X, int64_t ldx, int64_t rows, int64_t n, const float* U,
                 int64_t ldu, const float* V, int64_t ldv, int r, double* parts, int* nparts,
                 cudaStream_t st);

// ---------------------------------------------------------------- cache-resident sweeps
// small_sweep.cu: `count` HALS sweeps of a dense problem whose X
// stays cache resident (C1-C4) in one cooperative persistent kernel, fp64 on the
// fp32 state: U, V updated in place; GV in = V^T V of the V passed in, GV / GU out = the Grams
// of the final factors; one trace-form objective per sweep appended at ftrace[(*fcnt)++];
// *minu, *minv = the factor minima, *stage = 1, *cnt_hals += count.  ws >=
// small_sweeps_workspace() doubles.  Returns nonzero if the launch failed.
bool small_sweeps_supported(int64_t m, int64_t n, int r);
size_t small_sweeps_workspace(int64_t m, int64_t n, int r);
int small_sweeps_launch(const float* X, int64_t ldx, int64_t m, int64_t n, int r, float* U,
                        int64_t ldu, float* V, int64_t ldv, double* GV, double* GU,
                        const double* xnorm2, double* ftrace, int* fcnt, double* minu,
                        double* minv, int* stage, int* cnt_hals, double* ws, int count,
                        cudaStream_t st);

// ---------------------------------------------------------------- small dense (one CTA)
// Upper Cholesky G = R^T R of a k x k SPD matrix (row-major, ld k) with diagonal shift,
// and Rinv = R^{-1}.  *bad = number of non-positive pivots (replaced by tiny values).
void chol_inv(const double* G, int k, double shift_rel, double* R, double* Rinv, int* bad,
              cudaStream_t st);
// One-sided Jacobi SVD of a k x k matrix A (row-major): A = U diag(s) V^T, s descending.
// Uo, Vo are k x k row-major.  work >= 2*k*k doubles.  J0 (k x k row-major orthogonal, may be
// null): warm start, the rotations are accumulated onto J0 (B = A J0 initially).
// gate (device int, may be null): the kernel runs only if *gate != 0.
void jacobi_svd(const double* A, int k, double* Uo, double* s, double* Vo, double* work,
                cudaStream_t st, const double* J0 = nullptr, const int* gate = nullptr);
// R = C D^T from the SVD W^T B = C S D^T (orthogonal Procrustes), completing C's basis
// (in place) for zero singular values.
void procrustes_from_svd(double* Cm, const double* s, const double* Dm, int k, double* R,
                         cudaStream_t st, const int* gate = nullptr);
// Orthogonal polar factor of a nonsingular k x k row-major M (k <= 128) by scaled Newton
// iteration: R = C D^T for M = C S D^T.  *fail (device) = 1 if M is numerically singular or
// the iteration did not converge (R untouched) -- then gate the Jacobi path on it.
bool polar_supported(int k);
void polar_newton(const double* M, int k, double* R, int* fail, cudaStream_t st,
                  int* iters = nullptr, const int* gate = nullptr);
// Polar factor by the Newton-Schulz iteration (multi-CTA, device-side convergence, no host
// sync): state[2] (device) = {done, fail}; fail = 1 if |X^T X - I| did not reach tolerance in
// max_iter steps (gate polar_newton on state + 1).  work >= 3 k^2 + 16 doubles.
void polar_ns(const double* M, int k, double* R, int* state, double* work, int max_iter,
              cudaStream_t st);

// ---------------------------------------------------------------- stage / scalars
// stage[0]: 0 ascent, 1 HALS.  Switches to HALS when min U >= 0 and min V >= 0.
void stage_update(int* stage, const double* minu, const double* minv, int* counters,
                  cudaStream_t st);
// f = xnorm2 - 2 cross + gg, stored to *fout -- or, with slot (device int), to fout[*slot]
// and ++*slot (the objective trace: one launch sequence per sweep, replayable as a graph).
void objective_finish(const double* xnorm2, const double* cross, const double* gu,
                      const double* gv, int r, double* fout, cudaStream_t st,
                      int* slot = nullptr);
// dst[*slot] = *src; ++*slot.
void append_scalar(const double* src, double* dst, int* slot, cudaStream_t st);
// min over partial buffers.
void reduce_min(const double* parts, int n, double* out, cudaStream_t st);
// ADMM elementwise step (see kernels_small.cu).
void admm_z(const double* WR, double* Yh, double* Z, double* B, int64_t count, double inv_rho,
            int first, double* negparts, unsigned long long* third, cudaStream_t st);
// sum of h(A) = max(0, -A) over count entries into *out (device).
void negsum(const double* A, int64_t count, double* parts, double* out, cudaStream_t st);
// sign rule R5 helpers
void colabsmax(const double* A, int64_t rows, int r, int64_t row_offset, double* parts,
               cudaStream_t st);
int colabsmax_parts();
void colabsmax_finish(const double* parts, int r, double* sign_out, cudaStream_t st);
void scale_cols_f64(double* A, int64_t rows, int r, const double* s, cudaStream_t st);

}  // namespace enmf
