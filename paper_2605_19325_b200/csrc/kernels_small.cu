// kernels_small.cu -- reductions, scalar bookkeeping, the ADMM elementwise step, the
// randomised-SVD helpers and the single-CTA fp64 dense kernels (Cholesky, one-sided Jacobi
// SVD, Procrustes) used at init.
#include <float.h>

#include "grid_barrier.cuh"
#include "internal.h"

namespace enmf {
namespace {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// Block-wide reduction of one double with a fixed tree (deterministic).
template <int OP>  // 0 sum, 1 min, 2 max
__device__ double block_reduce(double v, double* red) {
  red[threadIdx.x] = v;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      const double a = red[threadIdx.x], b = red[threadIdx.x + o];
      red[threadIdx.x] = OP == 0 ? a + b : (OP == 1 ? fmin(a, b) : fmax(a, b));
    }
    __syncthreads();
  }
  const double out = red[0];
  __syncthreads();
  return out;
}

constexpr int kStatGrid = 4 * kSMs;

// ||X||^2, min X, #non-finite and max |X| of this rank's rows in one pass (4 partials per
// block).  Rows by blocks, a row's columns by threads (float4 when aligned): no 64-bit division
// per element.
__global__ void __launch_bounds__(256)
x_stats_kernel(const float* __restrict__ X, int64_t ldx, int64_t rows, int64_t n,
               double* parts) {
  __shared__ double red[256];
  double s = 0.0, mn = DBL_MAX, bad = 0.0, mx = 0.0;
  const bool vec = (ldx & 3) == 0 && (n & 3) == 0 && ((uintptr_t)X & 15) == 0;
  auto take = [&](float v) {
    if (!isfinite(v)) {
      bad += 1.0;
      return;
    }
    s = fma((double)v, (double)v, s);
    mn = fmin(mn, (double)v);
    mx = fmax(mx, fabs((double)v));
  };
  for (int64_t i = blockIdx.x; i < rows; i += gridDim.x) {
    const float* xr = X + i * ldx;
    if (vec) {
      for (int64_t j = 4 * (int64_t)threadIdx.x; j < n; j += 4 * (int64_t)blockDim.x) {
        const float4 f = *reinterpret_cast<const float4*>(xr + j);
        take(f.x);
        take(f.y);
        take(f.z);
        take(f.w);
      }
    } else {
      for (int64_t j = threadIdx.x; j < n; j += blockDim.x) take(xr[j]);
    }
  }
  s = block_reduce<0>(s, red);
  mn = block_reduce<1>(mn, red);
  bad = block_reduce<0>(bad, red);
  mx = block_reduce<2>(mx, red);
  if (threadIdx.x == 0) {
    parts[4 * blockIdx.x] = s;
    parts[4 * blockIdx.x + 1] = mn;
    parts[4 * blockIdx.x + 2] = bad;
    parts[4 * blockIdx.x + 3] = mx;
  }
}

__global__ void x_stats_finish(const double* parts, int nparts, double* out4) {
  if (threadIdx.x != 0) return;
  double s = 0.0, mn = DBL_MAX, bad = 0.0, mx = 0.0;
  for (int p = 0; p < nparts; ++p) {
    s += parts[4 * p];
    mn = fmin(mn, parts[4 * p + 1]);
    bad += parts[4 * p + 2];
    mx = fmax(mx, parts[4 * p + 3]);
  }
  out4[0] = s;
  out4[1] = mn;
  out4[2] = bad;
  out4[3] = mx;
}

__global__ void min_f32_kernel(const float* __restrict__ A, int64_t ld, int64_t rows,
                               int64_t cols, double* parts) {
  __shared__ double red[256];
  double mn = DBL_MAX;
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / cols, j = e - i * cols;
    mn = fmin(mn, (double)A[i * ld + j]);
  }
  mn = block_reduce<1>(mn, red);
  if (threadIdx.x == 0) parts[blockIdx.x] = mn;
}

// The same over a contiguous factor (ld == cols), 16-byte loads, the minimum in fp32 (exact
// for fp32 data) and one conversion: HBM-bound instead of one division per element.
__global__ void min_f32_flat4_kernel(const float4* __restrict__ A, int64_t n4, double* parts) {
  __shared__ double red[256];
  float mn = INFINITY;             // factors are finite (checked at bind / by the updates)
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n4;
       e += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = A[e];
    mn = fminf(fminf(mn, fminf(v.x, v.y)), fminf(v.z, v.w));
  }
  const double m = block_reduce<1>(mn == INFINITY ? DBL_MAX : (double)mn, red);
  if (threadIdx.x == 0) parts[blockIdx.x] = m;
}

// Post-rotation variant (ii) of the ablation: A <- max(0, A) in place,
// float4 along rows when the rows are 16-byte aligned (HBM-bound: 8 B per element).
__global__ void project_f32_kernel(float* __restrict__ A, int64_t ld, int64_t rows, int64_t cols,
                                   bool vec) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (vec) {
    const int64_t c4 = cols / 4, total = rows * c4;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += stride) {
      const int64_t i = e / c4, j = e - i * c4;
      float4* p = reinterpret_cast<float4*>(A + i * ld) + j;
      float4 v = *p;
      v.x = v.x < 0.f ? 0.f : v.x;
      v.y = v.y < 0.f ? 0.f : v.y;
      v.z = v.z < 0.f ? 0.f : v.z;
      v.w = v.w < 0.f ? 0.f : v.w;
      *p = v;
    }
  } else {
    const int64_t total = rows * cols;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += stride) {
      const int64_t i = e / cols, j = e - i * cols;
      float* p = A + i * ld + j;
      if (*p < 0.f) *p = 0.f;
    }
  }
}

__global__ void reduce_min_kernel(const double* parts, int n, double* out) {
  __shared__ double red[256];
  double mn = DBL_MAX;
  for (int p = threadIdx.x; p < n; p += blockDim.x) mn = fmin(mn, parts[p]);   // exact in any order
  mn = block_reduce<1>(mn, red);
  if (threadIdx.x == 0) *out = mn;
}

__global__ void dot_kernel(const double* __restrict__ A, const float* __restrict__ B,
                           int64_t ldb, int64_t rows, int64_t cols, double* parts) {
  __shared__ double red[256];
  double s = 0.0;
  // rows by blocks, a row's columns by threads (no per-element 64-bit division); narrow rows
  // (cols <= 128, the factor width) take blockDim / 128 rows per step so no thread idles
  const int per = cols <= 128 ? (int)(blockDim.x / 128) : 1;
  const int sub = cols <= 128 ? (int)(threadIdx.x / 128) : 0;
  const int j0 = cols <= 128 ? (int)(threadIdx.x % 128) : (int)threadIdx.x;
  const int js = cols <= 128 ? 128 : (int)blockDim.x;
#pragma unroll 4
  for (int64_t i = (int64_t)blockIdx.x * per + sub; i < rows; i += (int64_t)gridDim.x * per)
    for (int64_t j = j0; j < cols; j += js) s += A[i * cols + j] * (double)B[i * ldb + j];
  s = block_reduce<0>(s, red);
  if (threadIdx.x == 0) parts[blockIdx.x] = s;
}

// Philox4x32-10 (Salmon et al. 2011) for the Gaussian test matrix of the range finder.
__device__ __forceinline__ uint4 philox10(uint4 c, uint2 k) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const unsigned lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const unsigned lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

__global__ void gaussian_kernel(double* A, int64_t total, uint64_t seed) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint4 w = philox10(make_uint4((unsigned)e, (unsigned)(e >> 32), 0x4F6D6567u, 0u),
                             make_uint2((unsigned)seed, (unsigned)(seed >> 32)));
    const double u1 = ((double)(w.x >> 8) + 1.0) * (1.0 / 16777216.0);
    const double u2 = (double)(w.y >> 8) * (1.0 / 16777216.0);
    A[e] = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
  }
}

__global__ void stage_update_kernel(int* stage, const double* minu, const double* minv,
                                    int* counters) {
  if (threadIdx.x != 0) return;
  if (*stage == 0 && *minu >= 0.0 && *minv >= 0.0) *stage = 1;
  if (counters) counters[*stage] += 1;                            // [ascent, hals] sweeps
}

__global__ void objective_finish_kernel(const double* xnorm2, const double* cross,
                                        const double* gu, const double* gv, int r,
                                        double* fout, int* slot) {
  __shared__ double red[256];
  double s = 0.0;
  const int nn = r * r;     // <= 128^2 = 64 x 256
  // 16 products' loads in flight before they are summed (in the same order as before)
  for (int q0 = 0; q0 < 64 && q0 * 256 < nn; q0 += 16) {
    double a[16], b[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int e = threadIdx.x + (q0 + q) * 256;
      a[q] = e < nn ? gu[e] : 0.0;
      b[q] = e < nn ? gv[e] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) s += a[q] * b[q];
  }
  s = block_reduce<0>(s, red);
  if (threadIdx.x == 0) fout[slot ? (*slot)++ : 0] = *xnorm2 - 2.0 * (*cross) + s;
}

__global__ void append_scalar_kernel(const double* src, double* dst, int* slot) {
  if (threadIdx.x == 0) dst[(*slot)++] = *src;
}

// ADMM elementwise part of one step (Alg. 1 lines 171-173 with scaled dual Yh = Y/rho):
//   [first == 0] Yh += Z - W R          (dual update of the previous step)
//   b = W R - Yh ; Z = Eq.(7)(b) ; B = Z + Yh
// and the negativity sum h(W R) of the current rotation.
__global__ void admm_z_kernel(const double* __restrict__ WR, double* __restrict__ Yh,
                              double* __restrict__ Z, double* __restrict__ B, int64_t count,
                              double inv_rho, int first, double* negparts,
                              unsigned long long* third) {
  __shared__ double red[256];
  double neg = 0.0;
  unsigned long long th = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double wr = WR[e];
    double yh = first ? 0.0 : Yh[e] + Z[e] - wr;
    const double b = wr - yh;
    double z;
    if (b > 0.0) z = b;
    else if (b >= -inv_rho) z = 0.0;
    else { z = b + inv_rho; ++th; }
    Yh[e] = yh;
    Z[e] = z;
    B[e] = z + yh;
    neg += wr < 0.0 ? -wr : 0.0;
  }
  neg = block_reduce<0>(neg, red);
  if (threadIdx.x == 0) negparts[blockIdx.x] = neg;
  if (th) atomicAdd(third, th);
}

// Column-wise arg max |A_ik| (ties: lowest row) -> parts[block][k] = (|v|, row, v).
__global__ void colabsmax_kernel(const double* __restrict__ A, int64_t rows, int r,
                                 int64_t row_offset, double* parts) {
  for (int k = threadIdx.x; k < r; k += blockDim.x) {
    double best = -1.0, bv = 0.0, bi = 0.0;
    for (int64_t i = blockIdx.x; i < rows; i += gridDim.x) {
      const double v = A[i * r + k];
      if (fabs(v) > best) { best = fabs(v); bv = v; bi = (double)(i + row_offset); }
    }
    double* p = parts + ((int64_t)blockIdx.x * r + k) * 3;
    p[0] = best; p[1] = bi; p[2] = bv;
  }
}

__global__ void colabsmax_finish_kernel(const double* parts, int nparts, int r, double* sg) {
  for (int k = threadIdx.x; k < r; k += blockDim.x) {
    double best = -1.0, bi = 0.0, bv = 0.0;
    for (int p = 0; p < nparts; ++p) {
      const double* q = parts + ((int64_t)p * r + k) * 3;
      if (q[0] > best || (q[0] == best && q[1] < bi)) { best = q[0]; bi = q[1]; bv = q[2]; }
    }
    sg[k] = bv < 0.0 ? -1.0 : 1.0;                 // sign rule R5
  }
}

__global__ void scale_cols_kernel(double* A, int64_t rows, int r, const double* s) {
  const int64_t total = rows * r;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x)
    A[e] *= s[e % r];
}

// ---------------------------------------------------------------- single-CTA dense fp64
// Upper Cholesky G = R^T R (row j of R from rows < j), then R^{-1} by back substitution,
// one column per thread.
__global__ void __launch_bounds__(1024)
chol_inv_kernel(const double* __restrict__ G, int k, double shift_rel, double* R, double* Rinv,
                int* bad) {
  __shared__ double diag_s;
  __shared__ double tr_s;
  if (threadIdx.x == 0) {
    double tr = 0.0;
    for (int i = 0; i < k; ++i) tr += G[i * k + i];
    tr_s = tr;
    *bad = 0;
  }
  __syncthreads();
  const double shift = shift_rel * tr_s / (k > 0 ? k : 1);
  for (int j = 0; j < k; ++j) {
    if (threadIdx.x == 0) {
      double s = G[j * k + j] + shift;
      for (int p = 0; p < j; ++p) s -= R[p * k + j] * R[p * k + j];
      if (!(s > 1e-300)) { ++*bad; s = 1e-300; }
      diag_s = sqrt(s);
      R[j * k + j] = diag_s;
    }
    __syncthreads();
    for (int i = j + 1 + threadIdx.x; i < k; i += blockDim.x) {
      double s = G[j * k + i];
      for (int p = 0; p < j; ++p) s -= R[p * k + j] * R[p * k + i];
      R[j * k + i] = s / diag_s;
    }
    for (int i = threadIdx.x; i < j; i += blockDim.x) R[j * k + i] = 0.0;
    __syncthreads();
  }
  // R^{-1}: column c solves R x = e_c (x_i = 0 for i > c)
  for (int c = threadIdx.x; c < k; c += blockDim.x) {
    for (int i = k - 1; i > c; --i) Rinv[i * k + c] = 0.0;
    for (int i = c; i >= 0; --i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int p = i + 1; p <= c; ++p) s -= R[i * k + p] * Rinv[p * k + c];
      Rinv[i * k + c] = s / R[i * k + i];
    }
  }
}

// One-sided (Hestenes) Jacobi SVD of a k x k matrix, parallel round-robin pair ordering.
// B = A J is orthogonalised column-pairwise; J accumulates the rotations (J = J0 or I at start).
// A warm start J0 (the previous ADMM step's D: consecutive Procrustes matrices differ little)
// leaves B nearly column-orthogonal, so 1-3 sweeps replace ~8 from the identity.  B lives in
// shared memory when k <= 128 (128 KB), J in `work`.
__global__ void __launch_bounds__(1024)
jacobi_svd_kernel(const double* __restrict__ A, int k, const double* J0,
                  double* Uo, double* s, double* Vo, double* work, const int* gate) {
  if (gate && *gate == 0) return;
  extern __shared__ double smB[];
  const bool in_smem = k <= 128;
  double* B = in_smem ? smB : work;               // column c at B + c*k
  double* J = work + (int64_t)k * k;
  __shared__ int rotated;
  __shared__ double nrm[512];
  __shared__ int ord[512];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
    const int i = e / k, c = e % k;             // A row-major (i, c); J column-major
    J[c * k + i] = J0 ? J0[i * k + c] : (i == c ? 1.0 : 0.0);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
    const int i = e / k, c = e % k;
    double acc;
    if (J0) {
      acc = 0.0;                                  // B = A J0
      for (int l = 0; l < k; ++l) acc = fma(A[i * k + l], J[c * k + l], acc);
    } else {
      acc = A[e];
    }
    B[c * k + i] = acc;
  }
  const int kk = (k + 1) & ~1;      // even number of players (one dummy if k is odd)
  const double tol = 2.0 * sqrt((double)k) * DBL_EPSILON;
  __syncthreads();
  for (int sweep = 0; sweep < 60; ++sweep) {
    if (threadIdx.x == 0) rotated = 0;
    __syncthreads();
    for (int rd = 0; rd < kk - 1; ++rd) {
      // round-robin: player 0 fixed, others rotate ((x - 1 + rd) < 2 (kk - 1): no modulo)
      auto pos = [&](int x) {
        if (x == 0) return 0;
        int v = x - 1 + rd;
        if (v >= kk - 1) v -= kk - 1;
        return 1 + v;
      };
      if (in_smem) {
        // k <= 128: every load of a pair (B in shared memory, J in global) is issued before the
        // dependent arithmetic, so a pair costs one L2 round trip instead of a chain of four
        for (int pr = warp; pr < kk / 2; pr += nw) {
          int p = pos(pr), q = pos(kk - 1 - pr);
          if (p > q) { const int t = p; p = q; q = t; }
          if (q >= k) continue;
          double bp[4], bq[4], jp[4], jq[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int i = lane + 32 * t;
            const bool ok = i < k;
            bp[t] = ok ? B[p * k + i] : 0.0;
            bq[t] = ok ? B[q * k + i] : 0.0;
            jp[t] = ok ? J[p * k + i] : 0.0;
            jq[t] = ok ? J[q * k + i] : 0.0;
          }
          double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            al += bp[t] * bp[t];
            be += bq[t] * bq[t];
            ga += bp[t] * bq[t];
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            al += __shfl_xor_sync(0xffffffffu, al, o);
            be += __shfl_xor_sync(0xffffffffu, be, o);
            ga += __shfl_xor_sync(0xffffffffu, ga, o);
          }
          if (ga == 0.0 || ga * ga <= tol * tol * (al * be)) continue;
          // rotation angle (Rutishauser): zeta = (be - al) / (2 ga), t = sign / (|zeta| +
          // sqrt(1 + zeta^2)), c = 1 / sqrt(1 + t^2), s = c t
          const double zeta = (be - al) * (0.5 / ga);
          const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
          const double c = rsqrt(fma(t, t, 1.0)), sn = c * t;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int i = lane + 32 * u;
            if (i < k) {
              B[p * k + i] = c * bp[u] - sn * bq[u];
              B[q * k + i] = sn * bp[u] + c * bq[u];
              J[p * k + i] = c * jp[u] - sn * jq[u];
              J[q * k + i] = sn * jp[u] + c * jq[u];
            }
          }
          if (lane == 0) rotated = 1;
        }
        __syncthreads();
        continue;
      }
      for (int pr = warp; pr < kk / 2; pr += nw) {
        int p = pos(pr), q = pos(kk - 1 - pr);
        if (p > q) { const int t = p; p = q; q = t; }
        if (q >= k) continue;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int i = lane; i < k; i += 32) {
          const double bp = B[p * k + i], bq = B[q * k + i];
          al += bp * bp; be += bq * bq; ga += bp * bq;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {        // three independent butterflies
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        // converged pair: |cos| at the rounding level of a length-k dot product (2 sqrt(k) eps,
        // as LAPACK's one-sided Jacobi uses sqrt(m) eps); a fixed 1e-15 sits below that noise
        // for k >= ~64 and kept every sweep rotating until the 60-sweep cap
        if (ga == 0.0 || fabs(ga) <= tol * sqrt(al * be)) continue;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), sn = c * t;
        for (int i = lane; i < k; i += 32) {
          const double bp = B[p * k + i], bq = B[q * k + i];
          const double jp = J[p * k + i], jq = J[q * k + i];
          B[p * k + i] = c * bp - sn * bq;
          B[q * k + i] = sn * bp + c * bq;
          J[p * k + i] = c * jp - sn * jq;
          J[q * k + i] = sn * jp + c * jq;
        }
        if (lane == 0) rotated = 1;
      }
      __syncthreads();
    }
    if (!rotated) break;
    __syncthreads();
  }
  // column norms and a descending order (ties: lower index first)
  for (int c = warp; c < k; c += nw) {
    double t = 0.0;
    for (int i = lane; i < k; i += 32) t += B[c * k + i] * B[c * k + i];
    t = warp_sum(t);
    if (lane == 0) nrm[c] = sqrt(t);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < k; c += blockDim.x) {
    int rank = 0;
    for (int d = 0; d < k; ++d)
      if (nrm[d] > nrm[c] || (nrm[d] == nrm[c] && d < c)) ++rank;
    ord[rank] = c;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
    const int i = e / k, a = e % k;
    const int c = ord[a];
    const double sc = nrm[c];
    Uo[i * k + a] = sc > 0.0 ? B[c * k + i] / sc : 0.0;
    Vo[i * k + a] = J[c * k + i];
  }
  for (int a = threadIdx.x; a < k; a += blockDim.x) s[a] = nrm[ord[a]];
}


// Orthogonal polar factor R of a nonsingular k x k matrix M (k <= 128; R = C D^T for
// M = C S D^T, i.e. the Procrustes rotation) by the scaled Newton iteration
// X <- (zeta X + X^{-T} / zeta) / 2, X0 = M, Frobenius scaling zeta = (|X^-1|_F / |X|_F)^1/2
// while far from convergence.  One CTA of 1024 threads; X lives in R (global, L2) between
// iterations; X^{-1} by Gauss-Jordan with partial pivoting held in REGISTERS: thread
// (row ei = tid / 8, columns ec0 + 8 t, ec0 = tid % 8, t < 16) owns 16 entries, and each
// elimination step exchanges only the pivot column and row through shared memory (shared-
// memory traffic of an in-place smem elimination bounded it at ~0.3 ms per inverse).
// *fail = 1 when M is numerically singular or the iteration does not converge (R is then
// garbage): the caller gates the Jacobi-SVD Procrustes on it (rank deficiency).
constexpr int kPolarLd = 129;
constexpr int kPolarTPR = 4;                    // threads per row
constexpr int kPolarCPT = 128 / kPolarTPR;      // columns per thread
constexpr int kPolarThreads = 128 * kPolarTPR;  // 512: 128 registers per thread
__global__ void __launch_bounds__(kPolarThreads)
polar_newton_kernel(const double* __restrict__ M, int k, double* R, int* fail, int* iters,
                    const int* gate) {
  if (gate && *gate == 0) {                     // an earlier method already produced R
    if (threadIdx.x == 0) *fail = 0;
    return;
  }
  extern __shared__ double Inv[];               // k x kPolarLd: X^{-1} of the iteration
  __shared__ double red[kPolarThreads];
  __shared__ double colb[2][128];               // pivot column (double-buffered by step)
  __shared__ double rowJ[128], rowP[128], rowN[128];
  __shared__ int perm[128], dst[128], src[128];
  __shared__ int bad_s;
  const int tid = threadIdx.x, lane = tid & 31;
  const int ei = tid / kPolarTPR, ec0 = tid % kPolarTPR;
  const bool mine = ei < k;
  for (int e = tid; e < k * k; e += blockDim.x) R[e] = M[e];
  if (tid == 0) bad_s = 0;
  __syncthreads();
  bool scaling = true, done = false;
  int it = 0;
  for (; it < 40 && !done; ++it) {
    double a[kPolarCPT];
    double amax = 0.0;
#pragma unroll
    for (int t = 0; t < kPolarCPT; ++t) {
      const int c = ec0 + kPolarTPR * t;
      a[t] = (mine && c < k) ? R[ei * k + c] : 0.0;
      amax = fmax(amax, fabs(a[t]));
    }
    amax = block_reduce<2>(amax, red);
    for (int j = 0; j < k; ++j) {
      double* col = colb[j & 1];
      const int tj = j / kPolarTPR;
      if (mine && ec0 == j % kPolarTPR) {
        double v = 0.0;
#pragma unroll
        for (int t = 0; t < kPolarCPT; ++t) v = t == tj ? a[t] : v;
        col[ei] = v;
      }
      __syncthreads();
      // every warp finds the pivot (max |col[i]|, i >= j; ties: lowest i) redundantly
      double bv = -1.0;
      int bi = j;
      for (int i = j + lane; i < k; i += 32) {
        const double v = fabs(col[i]);
        if (v > bv) { bv = v; bi = i; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
      }
      if (!(bv > 1e-13 * amax)) {                   // numerically singular: give up
        if (tid == 0) bad_s = 1;
        break;
      }
      const int pr = bi;
      if (tid == 0) perm[j] = pr;
      // publish rows j and pr (pre-swap)
      if (ei == j || ei == pr) {
#pragma unroll
        for (int t = 0; t < kPolarCPT; ++t) {
          const int c = ec0 + kPolarTPR * t;
          if (c < k) (ei == j ? rowJ : rowP)[c] = a[t];
        }
      }
      __syncthreads();
      const double piv = col[pr];
      const double ip = 1.0 / piv;
      // swap rows j <-> pr in registers; the new row j is normalised and published
      if (ei == j) {
        const double* srow = pr == j ? rowJ : rowP;   // no interchange: row j itself
#pragma unroll
        for (int t = 0; t < kPolarCPT; ++t) {
          const int c = ec0 + kPolarTPR * t;
          if (c < k) {
            const double v = c == j ? ip : srow[c] * ip;
            a[t] = v;
            rowN[c] = v;
          }
        }
      } else if (ei == pr) {
#pragma unroll
        for (int t = 0; t < kPolarCPT; ++t) {
          const int c = ec0 + kPolarTPR * t;
          if (c < k) a[t] = rowJ[c];
        }
      }
      __syncthreads();
      if (mine && ei != j) {
        // f = A[ei][j] after the swap: row pr now holds old row j's entry
        const double f = ei == pr ? col[j] : col[ei];
#pragma unroll
        for (int t = 0; t < kPolarCPT; ++t) {
          const int c = ec0 + kPolarTPR * t;
          if (c < k) a[t] = c == j ? -f * ip : fma(-f, rowN[c], a[t]);
        }
      }
    }
    __syncthreads();
    if (bad_s) break;
    // column unpermutation: swaps (j, perm[j]) for j = k-1 .. 0  ->  Inv[i][dst[c]] = a[i][c]
    if (tid == 0) {
      for (int c = 0; c < k; ++c) src[c] = c;
      for (int j = k - 1; j >= 0; --j) {
        const int t = src[j];
        src[j] = src[perm[j]];
        src[perm[j]] = t;
      }
      for (int q = 0; q < k; ++q) dst[src[q]] = q;
    }
    __syncthreads();
    if (mine) {
#pragma unroll
      for (int t = 0; t < kPolarCPT; ++t) {
        const int c = ec0 + kPolarTPR * t;
        if (c < k) Inv[ei * kPolarLd + dst[c]] = a[t];
      }
    }
    __syncthreads();
    // ---- X <- (zeta X + X^{-T} / zeta) / 2 ----
    double zeta = 1.0;
    if (scaling) {
      double nx = 0.0, ni = 0.0;
      if (mine) {
#pragma unroll
        for (int t = 0; t < kPolarCPT; ++t) {
          const int c = ec0 + kPolarTPR * t;
          if (c < k) {
            const double xv = R[ei * k + c], iv = Inv[ei * kPolarLd + c];
            nx += xv * xv;
            ni += iv * iv;
          }
        }
      }
      nx = block_reduce<0>(nx, red);
      ni = block_reduce<0>(ni, red);
      zeta = sqrt(sqrt(ni / nx));
    }
    double dif = 0.0, nn = 0.0;
    if (mine) {
#pragma unroll
      for (int t = 0; t < kPolarCPT; ++t) {
        const int c = ec0 + kPolarTPR * t;
        if (c < k) {
          const double xo = R[ei * k + c];
          const double xn = 0.5 * (zeta * xo + Inv[c * kPolarLd + ei] / zeta);   // X^{-T}
          dif += (xn - xo) * (xn - xo);
          nn += xn * xn;
          R[ei * k + c] = xn;
        }
      }
    }
    dif = block_reduce<0>(dif, red);
    nn = block_reduce<0>(nn, red);
    if (dif <= 1e-4 * nn) scaling = false;          // quadratic phase: unscaled steps
    if (dif <= 1e-28 * nn) done = true;             // |dX| <= 1e-14 |X|
  }
  if (tid == 0) {
    *fail = (bad_s || !done) ? 1 : 0;
    if (iters) *iters = it;
  }
}


// ---------------------------------------------------------------- Newton-Schulz polar factor
// R = polar(M) by the Newton-Schulz iteration X <- X (3 I - X^T X) / 2 from X0 = M / |M|_F
// (all singular values in (0, 1]; each step maps a small sigma to ~1.5 sigma, then converges
// quadratically).  Two small multi-CTA kernels per iteration (32 x 32 output tiles of the
// k x k products, k <= 128), no host synchronisation: ns_gram_kernel forms Y = X^T X and the
// per-tile partials of |Y - I|_F^2; ns_step_kernel sums the partials in a fixed order and, when
// |Y - I|_F <= tol, copies X to R and raises the done flag (every later kernel of the sequence
// returns at once), else writes X (1.5 I - 0.5 Y) to the other buffer.  state = {done, fail}.
constexpr int kNsTile = 16;              // 16 x 16 output tiles: 64 CTAs at k = 128

__global__ void ns_init_kernel(const double* __restrict__ M, int k, double* X, int* state,
                               unsigned* bar) {
  if (threadIdx.x == 0) *bar = 0u;
  __shared__ double red[256];
  double s = 0.0;
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) s += M[e] * M[e];
  s = block_reduce<0>(s, red);
  const double inv = s > 0.0 ? 1.0 / sqrt(s) : 0.0;
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) X[e] = M[e] * inv;
  if (threadIdx.x == 0) {
    state[0] = s > 0.0 ? 0 : 1;       // done (nothing to do for M = 0: left to the fallback)
    state[1] = s > 0.0 ? 1 : 1;       // fail until converged
  }
}

// Y[I, J] tile = sum_l X[l][I] X[l][J]; partial |Y - I|^2 of the tile
__device__ __forceinline__ void ns_gram_tile(const double* X, int k, double* Y, double* part,
                                             double* buf, double* red) {
  double (*Xi)[kNsTile + 1] = reinterpret_cast<double (*)[kNsTile + 1]>(buf);
  double (*Xj)[kNsTile + 1] = reinterpret_cast<double (*)[kNsTile + 1]>(buf + 128 * (kNsTile + 1));
  const int nt = (k + kNsTile - 1) / kNsTile;
  const int ti = blockIdx.x / nt, tj = blockIdx.x % nt;
  for (int e = threadIdx.x; e < k * kNsTile; e += blockDim.x) {
    const int l = e / kNsTile, c = e % kNsTile;
    const int ci = ti * kNsTile + c, cj = tj * kNsTile + c;
    Xi[l][c] = ci < k ? X[l * k + ci] : 0.0;
    Xj[l][c] = cj < k ? X[l * k + cj] : 0.0;
  }
  __syncthreads();
  double dev = 0.0;
  for (int o = threadIdx.x; o < kNsTile * kNsTile; o += blockDim.x) {
    const int a = o / kNsTile, b = o % kNsTile;
    double acc = 0.0;
    for (int l = 0; l < k; ++l) acc = fma(Xi[l][a], Xj[l][b], acc);
    const int i = ti * kNsTile + a, j = tj * kNsTile + b;
    if (i < k && j < k) {
      Y[i * k + j] = acc;
      const double d = acc - (i == j ? 1.0 : 0.0);
      dev = fma(d, d, dev);
    }
  }
  dev = block_reduce<0>(dev, red);
  if (threadIdx.x == 0) part[blockIdx.x] = dev;
}

// X_out[I, J] = sum_l X[I][l] (1.5 delta_lJ - 0.5 Y[l][J]), or R = X when converged (returns
// true: the same decision on every CTA, the partials are summed in one fixed order)
__device__ __forceinline__ bool ns_step_tile(const double* X, int k, const double* Y,
                                             const double* part, int nparts, double tol2,
                                             double* Xout, double* R, int* state, double* buf) {
  double (*Xr)[128 + 1] = reinterpret_cast<double (*)[128 + 1]>(buf);
  double (*Yc)[kNsTile + 1] = reinterpret_cast<double (*)[kNsTile + 1]>(buf + kNsTile * 129);
  double dev = 0.0;
  for (int q = 0; q < nparts; ++q) dev += part[q];          // fixed order: same on every CTA
  if (dev <= tol2) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < k * k; e += gridDim.x * blockDim.x)
      R[e] = X[e];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      state[1] = 0;
      state[0] = 1;
      __threadfence();
    }
    return true;
  }
  const int nt = (k + kNsTile - 1) / kNsTile;
  const int ti = blockIdx.x / nt, tj = blockIdx.x % nt;
  for (int e = threadIdx.x; e < kNsTile * k; e += blockDim.x) {
    const int a = e / k, l = e % k;
    const int i = ti * kNsTile + a;
    Xr[a][l] = i < k ? X[i * k + l] : 0.0;
  }
  for (int e = threadIdx.x; e < k * kNsTile; e += blockDim.x) {
    const int l = e / kNsTile, b = e % kNsTile;
    const int j = tj * kNsTile + b;
    Yc[l][b] = j < k ? (l == j ? 1.5 : 0.0) - 0.5 * Y[l * k + j] : 0.0;
  }
  __syncthreads();
  for (int o = threadIdx.x; o < kNsTile * kNsTile; o += blockDim.x) {
    const int a = o / kNsTile, b = o % kNsTile;
    double acc = 0.0;
    for (int l = 0; l < k; ++l) acc = fma(Xr[a][l], Yc[l][b], acc);
    const int i = ti * kNsTile + a, j = tj * kNsTile + b;
    if (i < k && j < k) Xout[i * k + j] = acc;
  }
  return false;
}

// The whole iteration in one cooperative launch (one CTA per 16 x 16 output tile, <= 64 CTAs):
// Gram phase | grid barrier | step phase | grid barrier, until |X^T X - I|_F <= tol or max_iter.
// (Round 1-2c issued 3 launches per iteration, 121 per ADMM step whether or not the iteration
// had converged: 12000 launches = 40 ms of a 100-step rotation, most of the init of the small
// configurations; profiles/r02e_small_C3_launches_summary.txt.)
__global__ void __launch_bounds__(256) ns_polar_kernel(int k, double* X0, double* X1, double* Y,
                                                       double* part, int nparts, double tol2,
                                                       double* R, int* state, unsigned* bar,
                                                       int max_iter) {
  // one buffer for both phases: (Xi, Xj) of the Gram tile, (Xr, Yc) of the step tile
  __shared__ double buf[2 * 128 * (kNsTile + 1)];
  __shared__ double red[256];
  if (state[0]) return;                        // M = 0: left to the fallback (uniform)
  unsigned target = 0;
  for (int it = 0; it < max_iter; ++it) {
    const double* Xc = (it & 1) ? X1 : X0;
    double* Xn = (it & 1) ? X0 : X1;
    ns_gram_tile(Xc, k, Y, part, buf, red);
    grid_barrier(bar, target);
    if (ns_step_tile(Xc, k, Y, part, nparts, tol2, Xn, R, state, buf)) return;
    grid_barrier(bar, target);
  }
}

// Columns of C with s = 0 are completed to an orthonormal basis (rank-deficient M only).
__global__ void complete_basis_kernel(double* Cm, const double* __restrict__ s, int k,
                                      const int* gate) {
  if (threadIdx.x != 0 || (gate && *gate == 0)) return;
  for (int a = 0; a < k; ++a) {
    if (s[a] > 0.0) continue;
    for (int e = 0; e < k; ++e) {
      for (int i = 0; i < k; ++i) Cm[i * k + a] = (i == e) ? 1.0 : 0.0;
      for (int pass = 0; pass < 2; ++pass)
        for (int b = 0; b < k; ++b) {
          if (b == a || (s[b] <= 0.0 && b > a)) continue;
          double d = 0.0;
          for (int i = 0; i < k; ++i) d += Cm[i * k + b] * Cm[i * k + a];
          for (int i = 0; i < k; ++i) Cm[i * k + a] -= d * Cm[i * k + b];
        }
      double t = 0.0;
      for (int i = 0; i < k; ++i) t += Cm[i * k + a] * Cm[i * k + a];
      if (t > 1e-6) {
        t = sqrt(t);
        for (int i = 0; i < k; ++i) Cm[i * k + a] /= t;
        break;
      }
    }
  }
}

// R = C D^T: block a computes row a (C row staged in shared memory).
__global__ void procrustes_kernel(const double* __restrict__ Cm, const double* __restrict__ Dm,
                                  int k, double* R, const int* gate) {
  if (gate && *gate == 0) return;
  __shared__ double crow[512];
  const int a = blockIdx.x;
  for (int c = threadIdx.x; c < k; c += blockDim.x) crow[c] = Cm[a * k + c];
  __syncthreads();
  for (int b = threadIdx.x; b < k; b += blockDim.x) {
    double acc = 0.0;
    for (int c = 0; c < k; ++c) acc = fma(crow[c], Dm[b * k + c], acc);
    R[a * k + b] = acc;
  }
}

inline int grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  return (int)(g < kStatGrid ? (g < 1 ? 1 : g) : kStatGrid);
}

}  // namespace

int x_stats_parts(int64_t rows) { (void)rows; return kStatGrid; }

void x_stats(const float* X, int64_t ldx, int64_t rows, int64_t n, double* parts, int nparts,
             double* out4, cudaStream_t st) {
  x_stats_kernel<<<nparts, 256, 0, st>>>(X, ldx, rows, n, parts);
  x_stats_finish<<<1, 32, 0, st>>>(parts, nparts, out4);
  count_launch(2);
}

void min_f32(const float* A, int64_t ld, int64_t rows, int64_t cols, double* parts, double* out,
             cudaStream_t st) {
  if (ld == cols && (rows * cols) % 4 == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0)
    min_f32_flat4_kernel<<<kStatGrid, 256, 0, st>>>(reinterpret_cast<const float4*>(A),
                                                    rows * cols / 4, parts);
  else
    min_f32_kernel<<<kStatGrid, 256, 0, st>>>(A, ld, rows, cols, parts);
  reduce_min_kernel<<<1, 256, 0, st>>>(parts, kStatGrid, out);
  count_launch(2);
}

void project_f32(float* A, int64_t ld, int64_t rows, int64_t cols, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  const bool vec = cols % 4 == 0 && ld % 4 == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0;
  project_f32_kernel<<<kStatGrid, 256, 0, st>>>(A, ld, rows, cols, vec);
  count_launch();
}

void reduce_min(const double* parts, int n, double* out, cudaStream_t st) {
  reduce_min_kernel<<<1, 256, 0, st>>>(parts, n, out);
  count_launch();
}

void dot_f64_f32(const double* A, const float* B, int64_t ldb, int64_t rows, int64_t cols,
                 double* parts, double* out, cudaStream_t st) {
  dot_kernel<<<kStatGrid, 256, 0, st>>>(A, B, ldb, rows, cols, parts);
  reduce_parts(parts, kStatGrid, 1, out, st);
  count_launch();
}

void gaussian_fill(double* A, int64_t rows, int64_t cols, uint64_t seed, cudaStream_t st) {
  gaussian_kernel<<<grid_for(rows * cols), 256, 0, st>>>(A, rows * cols, seed);
  count_launch();
}

void stage_update(int* stage, const double* minu, const double* minv, int* counters,
                  cudaStream_t st) {
  stage_update_kernel<<<1, 32, 0, st>>>(stage, minu, minv, counters);
  count_launch();
}

void objective_finish(const double* xnorm2, const double* cross, const double* gu,
                      const double* gv, int r, double* fout, cudaStream_t st, int* slot) {
  objective_finish_kernel<<<1, 256, 0, st>>>(xnorm2, cross, gu, gv, r, fout, slot);
  count_launch();
}

void append_scalar(const double* src, double* dst, int* slot, cudaStream_t st) {
  append_scalar_kernel<<<1, 32, 0, st>>>(src, dst, slot);
  count_launch();
}

void admm_z(const double* WR, double* Yh, double* Z, double* B, int64_t count, double inv_rho,
            int first, double* negparts, unsigned long long* third, cudaStream_t st) {
  admm_z_kernel<<<kStatGrid, 256, 0, st>>>(WR, Yh, Z, B, count, inv_rho, first, negparts, third);
  count_launch();
}

int colabsmax_parts() { return kStatGrid; }

void colabsmax(const double* A, int64_t rows, int r, int64_t row_offset, double* parts,
               cudaStream_t st) {
  colabsmax_kernel<<<kStatGrid, 128, 0, st>>>(A, rows, r, row_offset, parts);
  count_launch();
}

void colabsmax_finish(const double* parts, int r, double* sign_out, cudaStream_t st) {
  colabsmax_finish_kernel<<<1, 128, 0, st>>>(parts, kStatGrid, r, sign_out);
  count_launch();
}

void scale_cols_f64(double* A, int64_t rows, int r, const double* s, cudaStream_t st) {
  scale_cols_kernel<<<grid_for(rows * r), 256, 0, st>>>(A, rows, r, s);
  count_launch();
}

void chol_inv(const double* G, int k, double shift_rel, double* R, double* Rinv, int* bad,
              cudaStream_t st) {
  chol_inv_kernel<<<1, 1024, 0, st>>>(G, k, shift_rel, R, Rinv, bad);
  count_launch();
}

void jacobi_svd(const double* A, int k, double* Uo, double* s, double* Vo, double* work,
                cudaStream_t st, const double* J0, const int* gate) {
  const size_t sm = k <= 128 ? sizeof(double) * k * k : 0;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(jacobi_svd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(sizeof(double) * 128 * 128));
    attr = true;
  }
  jacobi_svd_kernel<<<1, 1024, sm, st>>>(A, k, J0, Uo, s, Vo, work, gate);
  count_launch();
}

void procrustes_from_svd(double* Cm, const double* s, const double* Dm, int k, double* R,
                         cudaStream_t st, const int* gate) {
  complete_basis_kernel<<<1, 32, 0, st>>>(Cm, s, k, gate);
  procrustes_kernel<<<k, 128, 0, st>>>(Cm, Dm, k, R, gate);
  count_launch(2);
}

bool polar_supported(int k) { return k >= 1 && k <= 128; }

void polar_ns(const double* M, int k, double* R, int* state, double* work, int max_iter,
              cudaStream_t st) {
  const int nt = (k + kNsTile - 1) / kNsTile;
  double* X0 = work;
  double* X1 = work + (size_t)k * k;
  double* Y = work + (size_t)2 * k * k;
  double* part = work + (size_t)3 * k * k;
  const double tol2 = 1e-26 * k;          // |X^T X - I|_F <= 1e-13 sqrt(k)
  unsigned* bar = reinterpret_cast<unsigned*>(work + (size_t)3 * k * k + 128);
  ns_init_kernel<<<1, 256, 0, st>>>(M, k, X0, state, bar);
  int nparts = nt * nt;
  void* args[] = {&k, &X0, &X1, &Y, &part, &nparts, const_cast<double*>(&tol2), &R, &state, &bar,
                  &max_iter};
  cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(ns_polar_kernel), dim3(nt * nt),
                              dim3(256), args, 0, st);
  count_launch(2);
}

void polar_newton(const double* M, int k, double* R, int* fail, cudaStream_t st, int* iters,
                  const int* gate) {
  const size_t sm = sizeof(double) * (size_t)k * kPolarLd;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(polar_newton_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(sizeof(double) * 128 * kPolarLd));
    attr = true;
  }
  polar_newton_kernel<<<1, kPolarThreads, sm, st>>>(M, k, R, fail, iters, gate);
  count_launch();
}

}  // namespace enmf

namespace enmf {
namespace {
__global__ void negsum_kernel(const double* __restrict__ A, int64_t count, double* parts) {
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x)
    s += A[e] < 0.0 ? -A[e] : 0.0;
  s = block_reduce<0>(s, red);
  if (threadIdx.x == 0) parts[blockIdx.x] = s;
}
}  // namespace

// sum h(A), h(q) = max(0, -q)
void negsum(const double* A, int64_t count, double* parts, double* out, cudaStream_t st) {
  negsum_kernel<<<kStatGrid, 256, 0, st>>>(A, count, parts);
  reduce_parts(parts, kStatGrid, 1, out, st);
  count_launch();
}
}  // namespace enmf
