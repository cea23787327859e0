// tc.h -- tensor-core (tcgen05) contraction path for large X.
//
// X is repacked once (enmf_set_data) into a handle-owned copy of three int8 digit planes
// (mixed radix 8/8/7) (3 bytes per element, a power-of-two scale per X row), laid out in UMMA
// canonical tiles that bulk copies move straight into shared memory, plus a K-major copy of
// X^T (a scale per X column) for pass 2 when memory allows.  The two X passes of a sweep run
// as tcgen05.mma kind::i8 with exact int32 accumulation in TMEM (six digit products in four
// accumulators), combined exactly in fp64 by the epilogue (tc_gemm.cu).  The ascent stage's
// PBCD (Alg. 2) and the HALS sweep run their r x r products the same way (tc_pbcd.cu, with
// their own base-2^7 digits).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace enmf {

struct TcState;

// True when the shape is handled by the tensor-core kernels.
bool tc_supported(int64_t rows, int64_t n, int64_t r);
// Build the digit-plane copies of X (rows x n, ld, X >= 0).  q2parts: device scratch of
// q2cap >= 1 doubles (partials of ||X~||^2).  Returns 0, 1 (CUDA error) or 2 (OOM).
int tc_create(TcState** out, const float* X, int64_t ldx, int64_t rows, int64_t n, int64_t r,
              cudaStream_t st, double* q2parts, int q2cap);
// Device pointer to ||X~||^2 of the quantised X that pass 2 (Q = X^T U) reads: with it and
// the Gram of the quantised U (tc_factor_scales) the trace-form objective is exactly
// ||X~ - U~ V^T||^2.
const double* tc_xq_norm2(const TcState* s);
// Device pointer to the digit scales s_k (power of two, r entries) of the factor packed by the
// last tc_xv / tc_xtu call: its quantised columns are rint(F s_k 2^15) / (s_k 2^15).
const double* tc_factor_scales(const TcState* s);
void tc_destroy(TcState* s);
// P (rows x r fp64) = X V ; Q (n x r fp64) = X^T U  (this rank's rows only).  vmax / umax
// (optional, device u64[r]): fp64 bits of the factor's column maxima |F| when the kernel that
// wrote the factor already computed them (hals / pbcd copy); else a scan computes them.
int tc_xv(TcState* s, const float* V, int64_t ldv, double* P, cudaStream_t st,
          const unsigned long long* vmax = nullptr, unsigned* band_ready = nullptr,
          bool stamp = false);
// stamp: the X V kernel records its own start / end (%globaltimer); tc_stamp_accum (enqueue
// after the pass, anywhere later in the stream) adds end - start to a device total that
// tc_stamp_read returns (ms, passes; synchronous) and resets.  For timing the pass when its
// successor overlaps it (no CUDA event can sit between the two launches).
int tc_stamp_accum(TcState* s, cudaStream_t st);
int tc_stamp_read(TcState* s, double* ms, int64_t* count);
// Band flags for overlapping the U-block update with P = X V (programmatic dependent launch):
// null unless pass 1 writes P directly (no K split, single-CTA kernel).  Enqueues the epoch
// increment on st; pass the result to tc_xv (the X pass then publishes each finished
// 128-row band) and to tc_hals_launch.  tc_bands: the number of 128-row bands (Mt).
unsigned* tc_band_flags(TcState* s, cudaStream_t st);
int64_t tc_bands(const TcState* s);
int tc_xtu(TcState* s, const float* U, int64_t ldu, double* Q, cudaStream_t st,
           const unsigned long long* umax = nullptr);
// Pass 2 over the 128-column bands [b0, b1) of X only: Q rows [128 b0, min(n, 128 b1)).
// pack: repack U's digits first (the first range of a pass; later ranges reuse them).
// tc_xtu_band_count: ceil(n / 128).  Returns 0, 1 (error) or 2 (OOM).
int tc_xtu_bands(TcState* s, const float* U, int64_t ldu, double* Q, int64_t b0, int64_t b1,
                 cudaStream_t st, const unsigned long long* umax, bool pack);
int64_t tc_xtu_band_count(const TcState* s);
// G (r x r fp64) = U~^T U~ of the digits the last tc_xtu / tc_xtu_bands packed (the Gram of
// the quantised U, scales tc_factor_scales), exact on the tensor cores up to the final
// rounding to fp64.  Returns 0, 1 (error) or 2 (unsupported size: use the SIMT Gram).
int tc_gram_quantised(TcState* s, double* G, cudaStream_t st);
// Column-block products for the randomised SVD (fp64 factors of any width):
// out (ld ldo) = X F (F: n x ncols) or, transposed, X^T F (F: this rank's rows x ncols).
// Returns 0, 1 (CUDA error) or 2 (OOM).
int tc_xf(TcState* s, bool transposed, const double* F, int64_t ldf, int ncols, double* out,
          int64_t ldo, cudaStream_t st);

// Alg. 2 PBCD on the tensor cores, staged: tc_pbcd_prepare turns G into the B-operand digits
// (gd_work >= 4*128*128 bytes, gscale_work >= 128), then each tc_pbcd_chunk runs iterations
// [it0, it1) for every row -- lift + mask of F (src < 0) or resume from the fp64 state
// ust[src] -- and leaves u_it1 in ust[dst] (each >= ceil(rows / 128) * 128 * r doubles,
// tile-major), with the partials of ||M o grad||^2 for iterations it0 .. it1 in pgparts
// (tc_pbcd_parts() x (max_iter + 1)).  No per-iteration snapshots: when the stopping rule
// fires inside a stage, pbcd_select_stage fills rctl = {1, it0, src, dst} and a launch with
// rctl (and kst = the k* slot) replays that stage up to k*.  A stage returns at once if
// *stage != 0 or *done != 0, a replay unless rctl[0] != 0.  kprev (optional): the block's k*
// of the previous sweep; if it equals max_iter, the first stage (it0 = 0) runs to max_iter.
// Returns 0, or 1 on a launch / configuration error.
bool tc_pbcd_supported(int r);
int tc_pbcd_parts();
// fstep (optional, device): the ablation's fixed step 1 / lambda_max(G) instead of Eq.(10)
// (round B skipped); want_stage = 1 with fstep and [0, 1): one projected-gradient step of the
// descent stage (runs only if *stage == 1; commit with pbcd_commit_state(..., want_stage 1)).
void tc_pbcd_prepare(const double* G, int r, int8_t* gd_work, double* gscale_work,
                     const int* stage, cudaStream_t st, int want_stage = 0);
int tc_pbcd_chunk(const float* F, int64_t ldf, int64_t rows, int r, const double* C,
                  const double* lam, int max_iter, int it0, int it1, int src, int dst,
                  double* ust0, double* ust1, double* pgparts, const int8_t* gd_work,
                  const double* gscale_work, const int* stage, const int* done,
                  const int* kprev, const int* rctl, const int* kst, cudaStream_t st,
                  const double* fstep = nullptr, int want_stage = 0);
// HALS sweep of the rows with t = C - u G from exact int8-digit tcgen05
// rounds, 32-column Gauss-Seidel blocks in registers (tc_pbcd.cu).  Runs only if *stage == 1.
// Writes minparts[0, nparts) (nparts >= tc_hals_parts()); colmax (u64[r]) as hals_rows;
// fallbacks (optional) counts rows redone in fp64 because u outgrew its digit scale.
// gd_work / gscale_work as tc_pbcd_prepare (the two never run in the same stage).  ill
// (optional, device int): set nonzero when some column of G is too ill-conditioned for the
// digit coupling (the kernel then returns at once; run hals_rows gated on *ill).  0 = launched.
int tc_hals_parts();
// tc_hals_rows in two steps: the G digits (and the ill flag), then the kernel.  band_ready /
// bands (optional, tc_band_flags / tc_bands): the kernel takes tiles as the X V pass just
// enqueued before it publishes their bands, launched with programmatic dependent launch, so
// it must directly follow that pass in the stream.
int tc_hals_prepare(const double* G, int r, int8_t* gd_work, double* gscale_work,
                    const int* stage, int* ill, cudaStream_t st);
int tc_hals_launch(float* F, int64_t ldf, int64_t rows, int r, const double* C, const double* G,
                   const int8_t* gd_work, const double* gscale_work, const int* stage,
                   double* minparts, int nparts, unsigned long long* colmax, int* fallbacks,
                   const int* ill, unsigned* band_ready, int64_t bands, cudaStream_t st);
int tc_hals_rows(float* F, int64_t ldf, int64_t rows, int r, const double* C, const double* G,
                 int8_t* gd_work, double* gscale_work, const int* stage, double* minparts,
                 int nparts, unsigned long long* colmax, int* fallbacks, int* ill,
                 cudaStream_t st);

}  // namespace enmf
