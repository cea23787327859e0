// kernels_rows.cu -- row-block factor updates of the exterior method.
//
// Rows of U (and of V) are independent given the cross term C (= X V or X^T U) and the
// Gram G ("we can leverage this to update the rows of U and V
// independently"), so every kernel here maps RB rows to one warp: lane L owns columns
// L, L+32, ... (CPL = ceil(r/32) of them), the r x r Gram sits in shared memory (fp64,
// zero-padded to 32*CPL), and the row vectors live in registers in fp64.  One G row
// load serves RB rows, which keeps the fp64 FMA pipe (not shared-memory bandwidth) the
// bound.
//
//   hals_kernel   HALS column sweep, Gauss-Seidel over k with an
//                 incrementally updated residual t = C - u G.
//   pbcd_kernel   Alg. 2: lift (Eq.6/7), mask (line 336), then all
//                 max_iter inner iterations of Eq.(8) with the Eq.(10) step, snapshotting
//                 each iterate and accumulating ||M o grad||^2 per iteration; the global
//                 stopping rule is applied afterwards by pbcd_select (k*), see DESIGN.md.
//   kkt_kernel    App. G residual statistics.
#include <float.h>

#include "internal.h"
#include "rows_dev.cuh"

namespace enmf {
namespace {

using namespace rows_dev;

template <int CPL, int RB>
__global__ void __launch_bounds__(32 * kRowWarps)
hals_kernel(float* __restrict__ F, int64_t ldf, int64_t rows, int r, const double* __restrict__ C,
            const double* __restrict__ G, const int* __restrict__ stage, double* minparts,
            unsigned long long* colmax, const int* __restrict__ gate) {
  constexpr int RP = 32 * CPL;
  extern __shared__ double smem[];
  double* Gs = smem;
  double* Ss = smem + RP * RP + (threadIdx.x >> 5) * RB * RP;
  __shared__ double wmin_s[kRowWarps];
  __shared__ double ginv[RP];                 // 1 / G_kk, 0 where G_kk <= 0 (column skipped)
  const bool active = (stage == nullptr || *stage == 1) && (gate == nullptr || *gate != 0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double wmin = DBL_MAX;
  double cmax[CPL];                  // max |F| of my columns lane + 32 c over my rows
#pragma unroll
  for (int c = 0; c < CPL; ++c) cmax[c] = 0.0;
  if (active) {
    load_gram<CPL>(G, r, Gs);
    for (int k = threadIdx.x; k < RP; k += blockDim.x) {
      const double gkk = k < r ? G[k * r + k] : 0.0;
      ginv[k] = gkk > 0.0 ? 1.0 / gkk : 0.0;
    }
    __syncthreads();
    const int64_t nblk = (rows + RB - 1) / RB;
    for (int64_t rb = (int64_t)blockIdx.x * kRowWarps + warp; rb < nblk;
         rb += (int64_t)gridDim.x * kRowWarps) {
      double u[RB][CPL], t[RB][CPL];
#pragma unroll
      for (int b = 0; b < RB; ++b)
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          const int64_t row = rb * RB + b;
          const int col = lane + 32 * c;
          const bool ok = row < rows && col < r;
          u[b][c] = ok ? (double)F[row * ldf + col] : 0.0;
          t[b][c] = ok ? C[row * r + col] : 0.0;
        }
      row_times_gram<CPL, RB>(u, Gs, Ss, r, lane, -1.0, t);      // t = C - u G
#pragma unroll
      for (int s = 0; s < CPL; ++s) {
        const int kmax = r - 32 * s < 32 ? r - 32 * s : 32;
        for (int kk = 0; kk < kmax; ++kk) {
          const int k = 32 * s + kk;
          const double ig = ginv[k];
          if (ig == 0.0) continue;                  // G_kk <= 0: column skipped (warp-uniform)
          double gk[CPL];
#pragma unroll
          for (int c = 0; c < CPL; ++c) gk[c] = Gs[k * RP + lane + 32 * c];
#pragma unroll
          for (int b = 0; b < RB; ++b) {
            // U_ik <- max(0, U_ik + (C_ik - sum_l U_il G_lk) / G_kk).
            // Lane kk owns (u_k, t_k): every lane evaluates the update on its own pair (only
            // lane kk's is meaningful) and lane kk's change d is broadcast -- one shuffle.
            // (a compare-select instead of fmax: no NaN-quieting sequence in the inner loop)
            const double uo = u[b][s];
            const double v = fma(t[b][s], ig, uo);
            const double nu = v > 0.0 ? v : 0.0;
            if (lane == kk) u[b][s] = nu;
            const double d = __shfl_sync(FULL, nu - uo, kk);
#pragma unroll
            for (int c = 0; c < CPL; ++c) t[b][c] = fma(-d, gk[c], t[b][c]);
          }
        }
      }
#pragma unroll
      for (int b = 0; b < RB; ++b)
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          const int64_t row = rb * RB + b;
          const int col = lane + 32 * c;
          if (row < rows && col < r) {
            const float v = (float)u[b][c];
            F[row * ldf + col] = v;
            wmin = fmin(wmin, (double)v);
            cmax[c] = fmax(cmax[c], fabs((double)v));
          }
        }
    }
  }
  // column maxima for the next pass's digit packing (tc path): bits of non-negative doubles
  // order like the values, so an integer atomicMax is exact and order independent; reduced in
  // shared memory first (one global atomic per column per block)
  if (colmax && active) {
    __shared__ unsigned long long cm_s[32 * CPL];
    for (int c = threadIdx.x; c < 32 * CPL; c += blockDim.x) cm_s[c] = 0ull;
    __syncthreads();
#pragma unroll
    for (int c = 0; c < CPL; ++c)
      if (lane + 32 * c < r)
        atomicMax(&cm_s[lane + 32 * c], (unsigned long long)__double_as_longlong(cmax[c]));
    __syncthreads();
    for (int c = threadIdx.x; c < r; c += blockDim.x)
      if (cm_s[c]) atomicMax(&colmax[c], cm_s[c]);
  }
  if (minparts) {
    wmin = warp_min(wmin);
    if (lane == 0) wmin_s[warp] = wmin;
    __syncthreads();
    if (threadIdx.x == 0) {
      double m = DBL_MAX;
      for (int w = 0; w < kRowWarps; ++w) m = fmin(m, wmin_s[w]);
      if (active) minparts[blockIdx.x] = m;
    }
  }
}

template <int CPL, int RB>
__global__ void __launch_bounds__(32 * kRowWarps)
pbcd_kernel(const float* __restrict__ F, int64_t ldf, int64_t rows, int r,
            const double* __restrict__ C, const double* __restrict__ G,
            const double* __restrict__ lam_ptr, int max_iter, float* __restrict__ snaps,
            double* __restrict__ pgparts, const int* __restrict__ stage,
            const double* __restrict__ fixed_step) {
  constexpr int RP = 32 * CPL;
  if (stage != nullptr && *stage != 0) return;
  const double fstep = fixed_step ? *fixed_step : 0.0;   // > 0: fixed step (ablation, R29)
  extern __shared__ double smem[];
  double* Gs = smem;
  double* Ss = smem + RP * RP + (threadIdx.x >> 5) * RB * RP;
  double* pgw = smem + RP * RP + kRowWarps * RB * RP;   // [kRowWarps][max_iter + 1]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double lam = *lam_ptr;
  load_gram<CPL>(G, r, Gs);
  for (int e = threadIdx.x; e < kRowWarps * (max_iter + 1); e += blockDim.x) pgw[e] = 0.0;
  __syncthreads();
  double* mypg = pgw + warp * (max_iter + 1);
  const int64_t nblk = (rows + RB - 1) / RB;
  const int64_t snap_stride = rows * (int64_t)r;
  for (int64_t rb = (int64_t)blockIdx.x * kRowWarps + warp; rb < nblk;
       rb += (int64_t)gridDim.x * kRowWarps) {
    double u[RB][CPL], cc[RB][CPL], gr[RB][CPL];
    bool msk[RB][CPL];
#pragma unroll
    for (int b = 0; b < RB; ++b)
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int64_t row = rb * RB + b;
        const int col = lane + 32 * c;
        const bool ok = row < rows && col < r;
        double v = ok ? (double)F[row * ldf + col] : 0.0;
        if (v < 0.0) v += lam;                      // Eq.(6)/(7) lift of I_-
        u[b][c] = v;
        msk[b][c] = ok && v >= 0.0;                 // M_{U+} after the lift (R14)
        cc[b][c] = ok ? C[row * r + col] : 0.0;
        gr[b][c] = -cc[b][c];
      }
    row_times_gram<CPL, RB>(u, Gs, Ss, r, lane, 1.0, gr);   // grad = u G - C
    {
      double s = 0.0;
#pragma unroll
      for (int b = 0; b < RB; ++b)
#pragma unroll
        for (int c = 0; c < CPL; ++c) s += msk[b][c] ? gr[b][c] * gr[b][c] : 0.0;
      s = warp_sum(s);
      if (lane == 0) mypg[0] += s;
    }
    for (int it = 1; it <= max_iter; ++it) {
      double g[RB][CPL], gG[RB][CPL];
      double num[RB], den[RB];
#pragma unroll
      for (int b = 0; b < RB; ++b) {
        double sn = 0.0;
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          g[b][c] = msk[b][c] ? gr[b][c] : 0.0;
          sn += g[b][c] * g[b][c];
          gG[b][c] = 0.0;
        }
        num[b] = warp_sum(sn);
      }
      row_times_gram<CPL, RB>(g, Gs, Ss, r, lane, 1.0, gG);  // g V^T V
#pragma unroll
      for (int b = 0; b < RB; ++b) {
        double sd = 0.0;
#pragma unroll
        for (int c = 0; c < CPL; ++c) sd += gG[b][c] * g[b][c];
        den[b] = warp_sum(sd);
      }
#pragma unroll
      for (int b = 0; b < RB; ++b) {
        // Eq.(10): d_i = ||g_i||^2 / ||g_i V^T||^2 ; 0 on a zero denominator (R10)
        const double d = fstep > 0.0 ? fstep : (den[b] > 0.0 ? num[b] / den[b] : 0.0);
        const int64_t row = rb * RB + b;
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          if (msk[b][c]) u[b][c] = fmax(0.0, u[b][c] - d * gr[b][c]);   // Eq.(8)
          const int col = lane + 32 * c;
          if (row < rows && col < r)
            snaps[(int64_t)(it - 1) * snap_stride + row * r + col] = (float)u[b][c];
          gr[b][c] = -cc[b][c];
        }
      }
      row_times_gram<CPL, RB>(u, Gs, Ss, r, lane, 1.0, gr);
      double s = 0.0;
#pragma unroll
      for (int b = 0; b < RB; ++b)
#pragma unroll
        for (int c = 0; c < CPL; ++c) s += msk[b][c] ? gr[b][c] * gr[b][c] : 0.0;
      s = warp_sum(s);
      if (lane == 0) mypg[it] += s;
    }
  }
  __syncwarp();
  for (int it = lane; it <= max_iter; it += 32)
    pgparts[((int64_t)blockIdx.x * kRowWarps + warp) * (max_iter + 1) + it] = mypg[it];
}

// Projected-gradient descent step (ablation variants (iv)/(v); reading
// R29): F <- max(0, F - step (F G - C)), all columns of a row from the old row (Jacobi), the
// step 1/lambda_max(G) read from the device.  Same row layout as hals_kernel.
template <int CPL, int RB>
__global__ void __launch_bounds__(32 * kRowWarps)
pgd_kernel(float* __restrict__ F, int64_t ldf, int64_t rows, int r, const double* __restrict__ C,
           const double* __restrict__ G, const int* __restrict__ stage, const double* step_ptr,
           double* minparts, unsigned long long* colmax) {
  extern __shared__ double smem[];
  double* Gs = smem;
  double* Ss = smem + 32 * CPL * 32 * CPL + (threadIdx.x >> 5) * RB * 32 * CPL;
  __shared__ double wmin_s[kRowWarps];
  const bool active = stage == nullptr || *stage == 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double wmin = DBL_MAX;
  double cmax[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) cmax[c] = 0.0;
  if (active) {
    const double step = *step_ptr;
    load_gram<CPL>(G, r, Gs);
    __syncthreads();
    const int64_t nblk = (rows + RB - 1) / RB;
    for (int64_t rb = (int64_t)blockIdx.x * kRowWarps + warp; rb < nblk;
         rb += (int64_t)gridDim.x * kRowWarps) {
      double u[RB][CPL], t[RB][CPL];
#pragma unroll
      for (int b = 0; b < RB; ++b)
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          const int64_t row = rb * RB + b;
          const int col = lane + 32 * c;
          const bool ok = row < rows && col < r;
          u[b][c] = ok ? (double)F[row * ldf + col] : 0.0;
          t[b][c] = ok ? C[row * r + col] : 0.0;
        }
      row_times_gram<CPL, RB>(u, Gs, Ss, r, lane, -1.0, t);      // t = C - u G = -grad
#pragma unroll
      for (int b = 0; b < RB; ++b)
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          const int64_t row = rb * RB + b;
          const int col = lane + 32 * c;
          const double v = fma(step, t[b][c], u[b][c]);
          const float nu = (float)(v > 0.0 ? v : 0.0);
          if (row < rows && col < r) {
            F[row * ldf + col] = nu;
            wmin = fmin(wmin, (double)nu);
            cmax[c] = fmax(cmax[c], (double)nu);
          }
        }
    }
  }
  if (colmax && active) {
    __shared__ unsigned long long cm_s[32 * CPL];
    for (int c = threadIdx.x; c < 32 * CPL; c += blockDim.x) cm_s[c] = 0ull;
    __syncthreads();
#pragma unroll
    for (int c = 0; c < CPL; ++c)
      if (lane + 32 * c < r)
        atomicMax(&cm_s[lane + 32 * c], (unsigned long long)__double_as_longlong(cmax[c]));
    __syncthreads();
    for (int c = threadIdx.x; c < r; c += blockDim.x)
      if (cm_s[c]) atomicMax(&colmax[c], cm_s[c]);
  }
  if (minparts) {
    wmin = warp_min(wmin);
    if (lane == 0) wmin_s[warp] = wmin;
    __syncthreads();
    if (threadIdx.x == 0 && active) {
      double m = DBL_MAX;
      for (int w = 0; w < kRowWarps; ++w) m = fmin(m, wmin_s[w]);
      minparts[blockIdx.x] = m;
    }
  }
}

// lambda_max of the block's Gram G (r x r, symmetric PSD) by power iteration, warm-started from
// the previous sweep's eigenvector v (r values, kept by the caller; all ones if !warm): thread k
// owns component k; stop when the Rayleigh quotient changes by <= 1e-15 relative in 3
// consecutive steps (the Grams change little between sweeps: a few steps) or after max_it.
// out = 1 / lambda_max (0 if lambda_max <= 0): the fixed step of reading R29.
__global__ void __launch_bounds__(128) lambda_power_kernel(const double* __restrict__ G, int r,
                                                           double* v, int warm, int max_it,
                                                           double* out) {
  __shared__ double x[128];
  __shared__ double red[4], red2[4];
  const int k = threadIdx.x, lane = k & 31, w = k >> 5;
  x[k] = k < r ? (warm ? v[k] : 1.0) : 0.0;
  __syncthreads();
  double rq_prev = 0.0, rq = 0.0;
  int stable = 0;
  for (int it = 0; it < max_it && stable < 3; ++it) {
    double y = 0.0;
    if (k < r)
      for (int l = 0; l < r; ++l) y = fma(G[(int64_t)k * r + l], x[l], y);
    double a = x[k] * y, b = y * y;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    if (lane == 0) { red[w] = a; red2[w] = b; }
    __syncthreads();
    const double xy = (red[0] + red[1]) + (red[2] + red[3]);
    const double yy = (red2[0] + red2[1]) + (red2[2] + red2[3]);
    double xx = 0.0;
    for (int l = 0; l < r; ++l) xx = fma(x[l], x[l], xx);
    rq = xx > 0.0 ? xy / xx : 0.0;
    stable = fabs(rq - rq_prev) <= 1e-15 * fabs(rq) ? stable + 1 : 0;
    rq_prev = rq;
    __syncthreads();
    if (!(yy > 0.0)) break;
    x[k] = y / sqrt(yy);
    __syncthreads();
  }
  if (k < r) v[k] = x[k];
  if (k == 0) *out = rq > 0.0 ? 1.0 / rq : 0.0;
}

__global__ void recip_first_kernel(const double* s, double* out) {
  if (threadIdx.x == 0) *out = s[0] > 0.0 ? 1.0 / s[0] : 0.0;
}

// k* = first inner iteration whose projected gradient drops below eps * initial
// (Alg. 2), or max_iter.
// pgsum[it] = ||M o grad||_F^2 after `it` inner iterations, summed over all rows (and ranks).
__global__ void pbcd_select_kernel(const double* __restrict__ pgsum, int max_iter, double eps,
                                   int* kstar, const int* stage) {
  if (stage != nullptr && *stage != 0) return;
  if (threadIdx.x == 0) {
    const double pg0 = sqrt(pgsum[0]);
    int k = max_iter;
    for (int it = 1; it <= max_iter; ++it)
      if (sqrt(pgsum[it]) < eps * pg0) { k = it; break; }
    *kstar = k;
  }
}

// Alg. 2's stopping rule on a stage [it0, it1) of the staged tensor-core PBCD: the first
// it in [max(1, it0), it1] with ||M o grad_it|| < eps ||M o grad_0|| is k* (as in
// pbcd_select_kernel); none and it1 == max_iter: k* = max_iter.  Either way *done = 1, which
// makes the later stages of this block update return at once, and ctl[3] = dst (the state
// buffer holding the result); a stop before the stage's end (k* < it1) sets
// ctl[0..2] = {1, it0, src}: replay the stage from its start up to k* (no per-iteration
// snapshots are kept).  *kstar holds the previous sweep's k* on entry to the first stage:
// max_iter there means that stage ran to the end (tc_pbcd_chunk's kprev rule).
__global__ void pbcd_select_stage_kernel(const double* __restrict__ pgsum, int it0, int it1,
                                         int src, int dst, int max_iter, double eps,
                                         int* kstar, int* done, int* ctl, const int* stage) {
  if (stage != nullptr && *stage != 0) return;
  if (threadIdx.x == 0 && *done == 0) {
    if (it0 == 0 && *kstar == max_iter) it1 = max_iter;
    const double pg0 = sqrt(pgsum[0]);
    int k = -1;
    for (int it = it0 > 1 ? it0 : 1; it <= it1; ++it)
      if (sqrt(pgsum[it]) < eps * pg0) {
        k = it;
        break;
      }
    if (k < 0 && it1 == max_iter) k = max_iter;
    if (k < 0) return;
    *kstar = k;
    *done = 1;
    ctl[0] = k < it1 ? 1 : 0;
    ctl[1] = it0;
    ctl[2] = src;
    ctl[3] = dst;
  }
}

// The committed PBCD result: the fp64 state ust[ctl[3]] of the staged tensor-core PBCD
// (tile-major, element (i, j) at (i / 128) 128 r + j 128 + i % 128) rounded into F (fp32, the
// factor state, R26), with min partials and column maxima.  A (tile, 32-column chunk) unit is
// transposed through shared memory so that both the state reads and the F writes coalesce.
__global__ void pbcd_commit_state_kernel(float* __restrict__ F, int64_t ldf, int64_t rows,
                                         int r, const double* __restrict__ ust0,
                                         const double* __restrict__ ust1,
                                         const int* __restrict__ ctl, const int* stage,
                                         double* minparts, unsigned long long* colmax,
                                         int want_stage) {
  __shared__ float t[128][33];
  __shared__ double red[256];
  __shared__ unsigned long long cm[128];
  for (int c = threadIdx.x; c < 128; c += blockDim.x) cm[c] = 0ull;
  __syncthreads();
  const bool active = stage == nullptr || *stage == want_stage;
  double mn = DBL_MAX;
  if (active) {
    const double* src = (ctl != nullptr && ctl[3]) ? ust1 : ust0;   // no ctl: ust0
    const int64_t tiles = (rows + 127) / 128;
    const int chunks = (r + 31) / 32;
    for (int64_t unit = blockIdx.x; unit < tiles * chunks; unit += gridDim.x) {
      const int64_t tile = unit / chunks;
      const int j0 = (int)(unit - tile * chunks) * 32;
      const double* ts = src + tile * 128 * (int64_t)r;
      const int nt = (int)(rows - tile * 128 < 128 ? rows - tile * 128 : 128);
      __syncthreads();
      for (int e = threadIdx.x; e < 32 * 128; e += blockDim.x) {
        const int jl = e >> 7, il = e & 127;
        if (j0 + jl < r && il < nt) t[il][jl] = (float)ts[(int64_t)(j0 + jl) * 128 + il];
      }
      __syncthreads();
      for (int e = threadIdx.x; e < 128 * 32; e += blockDim.x) {
        const int il = e >> 5, jl = e & 31;
        const int64_t i = tile * 128 + il;
        if (i < rows && j0 + jl < r) {
          const float v = t[il][jl];
          F[i * ldf + j0 + jl] = v;
          mn = fmin(mn, (double)v);
          if (colmax)
            atomicMax(&cm[j0 + jl], (unsigned long long)__double_as_longlong(fabs((double)v)));
        }
      }
    }
  }
  red[threadIdx.x] = mn;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] = fmin(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0 && active) minparts[blockIdx.x] = red[0];
  if (colmax && active)
    for (int c = threadIdx.x; c < r; c += blockDim.x)
      if (cm[c]) atomicMax(&colmax[c], cm[c]);
}

__global__ void pbcd_copy_kernel(float* __restrict__ F, int64_t ldf, int64_t rows, int r,
                                 const float* __restrict__ snaps, const int* __restrict__ kstar,
                                 const int* stage, double* minparts) {
  __shared__ double red[256];
  const bool active = stage == nullptr || *stage == 0;
  double mn = DBL_MAX;
  if (active) {
    const float* src = snaps + (int64_t)(*kstar - 1) * rows * r;
    const int64_t total = rows * (int64_t)r;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
      const int64_t i = e / r, j = e - i * r;
      const float v = src[e];
      F[i * ldf + j] = v;
      mn = fmin(mn, (double)v);
    }
  }
  red[threadIdx.x] = mn;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] = fmin(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0 && active) minparts[blockIdx.x] = red[0];
}

// KKT statistics per warp slot: {max|c|, sum|c|, max c, sum c, min grad, min F, sum C^2, 0}
template <int CPL, int RB>
__global__ void __launch_bounds__(32 * kRowWarps)
kkt_kernel(const float* __restrict__ F, int64_t ldf, int64_t rows, int r,
           const double* __restrict__ C, const double* __restrict__ G, double* parts) {
  constexpr int RP = 32 * CPL;
  extern __shared__ double smem[];
  double* Gs = smem;
  double* Ss = smem + RP * RP + (threadIdx.x >> 5) * RB * RP;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  load_gram<CPL>(G, r, Gs);
  __syncthreads();
  double cmax = 0.0, csum = 0.0, dmax = -DBL_MAX, dsum = 0.0, gmin = DBL_MAX, fmn = DBL_MAX,
         c2 = 0.0;
  const int64_t nblk = (rows + RB - 1) / RB;
  for (int64_t rb = (int64_t)blockIdx.x * kRowWarps + warp; rb < nblk;
       rb += (int64_t)gridDim.x * kRowWarps) {
    double u[RB][CPL], gr[RB][CPL];
    bool ok[RB][CPL];
#pragma unroll
    for (int b = 0; b < RB; ++b)
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int64_t row = rb * RB + b;
        const int col = lane + 32 * c;
        ok[b][c] = row < rows && col < r;
        u[b][c] = ok[b][c] ? (double)F[row * ldf + col] : 0.0;
        const double cv = ok[b][c] ? C[row * r + col] : 0.0;
        gr[b][c] = -cv;
        c2 += cv * cv;
      }
    row_times_gram<CPL, RB>(u, Gs, Ss, r, lane, 1.0, gr);
#pragma unroll
    for (int b = 0; b < RB; ++b)
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        if (!ok[b][c]) continue;
        const double cv = gr[b][c] * u[b][c];
        cmax = fmax(cmax, fabs(cv));
        csum += fabs(cv);
        dmax = fmax(dmax, cv);
        dsum += cv;
        gmin = fmin(gmin, gr[b][c]);
        fmn = fmin(fmn, u[b][c]);
      }
  }
  cmax = warp_max(cmax);
  csum = warp_sum(csum);
  dmax = warp_max(dmax);
  dsum = warp_sum(dsum);
  gmin = warp_min(gmin);
  fmn = warp_min(fmn);
  c2 = warp_sum(c2);
  if (lane == 0) {
    double* p = parts + ((int64_t)blockIdx.x * kRowWarps + warp) * 8;
    p[0] = cmax; p[1] = csum; p[2] = dmax; p[3] = dsum; p[4] = gmin; p[5] = fmn; p[6] = c2;
    p[7] = 0.0;
  }
}

// eNMC PBCD (App. C, Alg. NMC): Alg. 2 with the masked gradient
// grad_i = sum_{j in E_i} (u_i . o_j - x_ij) o_j = u_i G_i - c_i, where G_i = sum_{j in E_i}
// o_j o_j^T and c_i = sum_{j in E_i} x_ij o_j run over the OBSERVED entries E_i of row i
// (CSR lists ptr / idx / val; o_j = row j of the other factor O).  One warp per row: G_i is
// accumulated in the warp's shared slice from the row's observed entries (each lane owns
// columns lane + 32 c, no two lanes write one word), then the inner iterations run exactly as
// pbcd_kernel's with G_i in place of the block Gram -- including the Eq.(10)-type step, which
// for the masked objective is ||g_i||^2 / sum_{j in E_i} (g_i . o_j)^2 = ||g_i||^2 / g_i G_i
// g_i^T (reading R30).  Lift, mask, snapshots and the per-iteration ||M o grad||^2 partials
// as pbcd_kernel (the global stopping rule is applied by pbcd_commit).
template <int CPL, int WARPS>
__global__ void __launch_bounds__(32 * WARPS)
nmc_pbcd_kernel(const float* __restrict__ F, int64_t ldf, int64_t rows, int r,
                const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                const float* __restrict__ val, const float* __restrict__ O, int64_t ldo,
                const double* __restrict__ lam_ptr, int max_iter, float* __restrict__ snaps,
                double* __restrict__ pgparts) {
  constexpr int RP = 32 * CPL;
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* Gs = smem + warp * (RP * RP + RP);
  double* Ss = Gs + RP * RP;
  double* pgw = smem + WARPS * (RP * RP + RP);        // [WARPS][max_iter + 1]
  const double lam = *lam_ptr;
  for (int e = threadIdx.x; e < WARPS * (max_iter + 1); e += blockDim.x) pgw[e] = 0.0;
  __syncthreads();
  double* mypg = pgw + warp * (max_iter + 1);
  const int64_t snap_stride = rows * (int64_t)r;
  for (int64_t row = (int64_t)blockIdx.x * WARPS + warp; row < rows;
       row += (int64_t)gridDim.x * WARPS) {
    for (int e = lane; e < RP * RP; e += 32) Gs[e] = 0.0;
    double cc[1][CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) cc[0][c] = 0.0;
    for (int64_t e = ptr[row]; e < ptr[row + 1]; ++e) {
      const int64_t j = idx[e];
      const double x = (double)val[e];
      double o[CPL];
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int col = lane + 32 * c;
        o[c] = col < r ? (double)O[j * ldo + col] : 0.0;
      }
      __syncwarp();
#pragma unroll
      for (int c = 0; c < CPL; ++c) Ss[lane + 32 * c] = o[c];
      __syncwarp();
      for (int l = 0; l < r; ++l) {
        const double ol = Ss[l];
#pragma unroll
        for (int c = 0; c < CPL; ++c) Gs[l * RP + lane + 32 * c] = fma(ol, o[c], Gs[l * RP + lane + 32 * c]);
      }
#pragma unroll
      for (int c = 0; c < CPL; ++c) cc[0][c] = fma(x, o[c], cc[0][c]);
    }
    __syncwarp();
    double u[1][CPL], gr[1][CPL];
    bool msk[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const int col = lane + 32 * c;
      const bool ok = col < r;
      double v = ok ? (double)F[row * ldf + col] : 0.0;
      if (v < 0.0) v += lam;                      // Eq.(6)/(7) lift of I_-
      u[0][c] = v;
      msk[c] = ok && v >= 0.0;                    // M_{U+} after the lift (R14)
      gr[0][c] = -cc[0][c];
    }
    row_times_gram<CPL, 1>(u, Gs, Ss, r, lane, 1.0, gr);   // grad = u G_i - c_i
    {
      double sg = 0.0;
#pragma unroll
      for (int c = 0; c < CPL; ++c) sg += msk[c] ? gr[0][c] * gr[0][c] : 0.0;
      sg = warp_sum(sg);
      if (lane == 0) mypg[0] += sg;
    }
    for (int it = 1; it <= max_iter; ++it) {
      double g[1][CPL], gG[1][CPL];
      double sn = 0.0;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        g[0][c] = msk[c] ? gr[0][c] : 0.0;
        sn += g[0][c] * g[0][c];
        gG[0][c] = 0.0;
      }
      const double num = warp_sum(sn);
      row_times_gram<CPL, 1>(g, Gs, Ss, r, lane, 1.0, gG);  // g G_i
      double sd = 0.0;
#pragma unroll
      for (int c = 0; c < CPL; ++c) sd += gG[0][c] * g[0][c];
      const double den = warp_sum(sd);
      const double d = den > 0.0 ? num / den : 0.0;          // reading R30
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        if (msk[c]) u[0][c] = fmax(0.0, u[0][c] - d * gr[0][c]);   // Eq.(8)
        const int col = lane + 32 * c;
        if (col < r) snaps[(int64_t)(it - 1) * snap_stride + row * r + col] = (float)u[0][c];
        gr[0][c] = -cc[0][c];
      }
      row_times_gram<CPL, 1>(u, Gs, Ss, r, lane, 1.0, gr);
      double s2 = 0.0;
#pragma unroll
      for (int c = 0; c < CPL; ++c) s2 += msk[c] ? gr[0][c] * gr[0][c] : 0.0;
      s2 = warp_sum(s2);
      if (lane == 0) mypg[it] += s2;
    }
  }
  __syncwarp();
  for (int it = lane; it <= max_iter; it += 32)
    pgparts[((int64_t)blockIdx.x * WARPS + warp) * (max_iter + 1) + it] = mypg[it];
}

template <int CPL>
size_t row_smem(int extra_doubles, int rb = 4) {
  return sizeof(double) * (size_t)(32 * CPL * 32 * CPL + kRowWarps * rb * 32 * CPL + extra_doubles);
}

template <typename K>
void set_smem(K kernel, size_t bytes) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

}  // namespace

#define ENMF_CPL_DISPATCH(r, CALL) \
  do {                             \
    if ((r) <= 32) { CALL(1); }    \
    else if ((r) <= 64) { CALL(2); } \
    else if ((r) <= 96) { CALL(3); } \
    else { CALL(4); }              \
  } while (0)

void hals_rows(float* F, int64_t ldf, int64_t rows, int r, const double* C, const double* G,
               const int* stage, double* minparts, cudaStream_t st,
               unsigned long long* colmax, const int* gate) {
#define CALL(CPL)                                                                      \
  {                                                                                    \
    auto k = hals_kernel<CPL, 8>;                                                      \
    size_t sm = row_smem<CPL>(0, 8);                                                   \
    set_smem(k, sm);                                                                   \
    k<<<kRowGrid, 32 * kRowWarps, sm, st>>>(F, ldf, rows, r, C, G, stage, minparts, colmax, gate); \
  }
  ENMF_CPL_DISPATCH(r, CALL);
#undef CALL
  count_launch();
}

void pgd_rows(float* F, int64_t ldf, int64_t rows, int r, const double* C, const double* G,
              const int* stage, const double* step, double* minparts, cudaStream_t st,
              unsigned long long* colmax) {
#define CALL(CPL)                                                                      \
  {                                                                                    \
    auto k = pgd_kernel<CPL, 8>;                                                       \
    size_t sm = row_smem<CPL>(0, 8);                                                   \
    set_smem(k, sm);                                                                   \
    k<<<kRowGrid, 32 * kRowWarps, sm, st>>>(F, ldf, rows, r, C, G, stage, step, minparts, colmax); \
  }
  ENMF_CPL_DISPATCH(r, CALL);
#undef CALL
  count_launch();
}

void lambda_power(const double* G, int r, double* v, bool warm, double* out, cudaStream_t st) {
  lambda_power_kernel<<<1, 128, 0, st>>>(G, r, v, warm ? 1 : 0, 2000, out);
  count_launch();
}

void recip_first(const double* s, double* out, cudaStream_t st) {
  recip_first_kernel<<<1, 32, 0, st>>>(s, out);
  count_launch();
}

int pbcd_parts() { return kRowGrid * kRowWarps; }

void pbcd_rows(const float* F, int64_t ldf, int64_t rows, int r, const double* C,
               const double* G, const double* lam, int max_iter, float* snaps,
               double* pgparts, const int* stage, cudaStream_t st, const double* fixed_step) {
#define CALL(CPL)                                                                           \
  {                                                                                         \
    auto k = pbcd_kernel<CPL, 4>;                                                           \
    size_t sm = row_smem<CPL>(kRowWarps * (max_iter + 1));                                  \
    set_smem(k, sm);                                                                        \
    k<<<kRowGrid, 32 * kRowWarps, sm, st>>>(F, ldf, rows, r, C, G, lam, max_iter, snaps,    \
                                           pgparts, stage, fixed_step);                     \
  }
  ENMF_CPL_DISPATCH(r, CALL);
#undef CALL
  count_launch();
}

bool nmc_supported(int r) { return r >= 1 && r <= 64; }
int nmc_pbcd_parts() { return kRowGrid * 8; }

void nmc_pbcd_rows(const float* F, int64_t ldf, int64_t rows, int r, const int64_t* ptr,
                   const int32_t* idx, const float* val, const float* O, int64_t ldo,
                   const double* lam, int max_iter, float* snaps, double* pgparts,
                   cudaStream_t st) {
  // rows beyond the grid's warps are strided; blocks x warps = nmc_pbcd_parts() slots (the
  // 4-warp CPL = 2 form leaves the upper half of the slots zero)
  cudaMemsetAsync(pgparts, 0, sizeof(double) * (size_t)nmc_pbcd_parts() * (max_iter + 1), st);
  if (r <= 32) {
    auto k = nmc_pbcd_kernel<1, 8>;
    const size_t sm = sizeof(double) * (size_t)(8 * (32 * 32 + 32) + 8 * (max_iter + 1));
    set_smem(k, sm);
    k<<<kRowGrid, 256, sm, st>>>(F, ldf, rows, r, ptr, idx, val, O, ldo, lam, max_iter, snaps,
                                 pgparts);
  } else {
    auto k = nmc_pbcd_kernel<2, 4>;
    const size_t sm = sizeof(double) * (size_t)(4 * (64 * 64 + 64) + 4 * (max_iter + 1));
    set_smem(k, sm);
    k<<<kRowGrid, 128, sm, st>>>(F, ldf, rows, r, ptr, idx, val, O, ldo, lam, max_iter, snaps,
                                 pgparts);
  }
  count_launch(2);
}

void pbcd_commit(float* F, int64_t ldf, int64_t rows, int r, const float* snaps,
                 const double* pgsum, double eps, int max_iter, int* kstar, const int* stage,
                 double* minparts, cudaStream_t st) {
  pbcd_select_kernel<<<1, 32, 0, st>>>(pgsum, max_iter, eps, kstar, stage);
  pbcd_copy_kernel<<<kRowGrid, 256, 0, st>>>(F, ldf, rows, r, snaps, kstar, stage, minparts);
  count_launch(2);
}

void pbcd_select_stage(const double* pgsum, int it0, int it1, int src, int dst, int max_iter,
                       double eps, int* kstar, int* done, int* ctl, const int* stage,
                       cudaStream_t st) {
  pbcd_select_stage_kernel<<<1, 32, 0, st>>>(pgsum, it0, it1, src, dst, max_iter, eps, kstar,
                                             done, ctl, stage);
  count_launch();
}

void pbcd_commit_state(float* F, int64_t ldf, int64_t rows, int r, const double* ust0,
                       const double* ust1, const int* ctl, const int* stage, double* minparts,
                       cudaStream_t st, unsigned long long* colmax, int want_stage) {
  pbcd_commit_state_kernel<<<kRowGrid, 256, 0, st>>>(F, ldf, rows, r, ust0, ust1, ctl, stage,
                                                     minparts, colmax, want_stage);
  count_launch();
}

int kkt_parts() { return kRowGrid * kRowWarps; }

void kkt_rows(const float* F, int64_t ldf, int64_t rows, int r, const double* C,
              const double* G, double* parts, cudaStream_t st) {
#define CALL(CPL)                                                                 \
  {                                                                               \
    auto k = kkt_kernel<CPL, 4>;                                                  \
    size_t sm = row_smem<CPL>(0);                                                 \
    set_smem(k, sm);                                                              \
    k<<<kRowGrid, 32 * kRowWarps, sm, st>>>(F, ldf, rows, r, C, G, parts);        \
  }
  ENMF_CPL_DISPATCH(r, CALL);
#undef CALL
  count_launch();
}

}  // namespace enmf
