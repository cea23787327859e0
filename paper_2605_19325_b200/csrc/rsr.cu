// rsr.cu -- elementwise and small kernels of RSR-ADMM, the rotation-scale-rotation ADMM of
// App. A (Alg. alg:rsr) that looks for orthogonal R1, R2 and a positive
// diagonal Lambda with U* R1 Lambda R2 >= 0 and V* R1 Lambda^-1 R2 >= 0 (Eq. eq5).  The skinny
// products (W R, W^T B) and the Procrustes polar factors run on the kernels the rotation of
// Alg. 1 uses (enmf_init.cu rsr_core); this file holds the per-entry updates of the split
// variables, the per-column reductions and the lambda solve (readings R34-R37).
// Rows [0, mu) of every (m + n) x r array are the U block (scaled by Lambda), the rest the V
// block (scaled by Lambda^-1).
#include <float.h>

#include "internal.h"

namespace enmf {
namespace {

__device__ __forceinline__ double zprox_t(double b, double inv_t) {
  // W3 update: argmin_z h(z) + t/2 (z - b)^2, h(q) = max(0, -q)
  return b > 0.0 ? b : (b >= -inv_t ? 0.0 : b + inv_t);
}

// (W1, W3) <- argmin f1:
//   W3 = zprox(W2 R2 - P);  W11 = (rho (U* R1 - M1) + gamma lam (W21 + N1)) / (rho + gamma lam^2),
//   W12 = (rho (V* R1 - M2) + gamma / lam (W22 + N2)) / (rho + gamma / lam^2)
__global__ void rsr_w13_kernel(const double* __restrict__ WsR1, const double* __restrict__ W2R2,
                               const double* __restrict__ M, const double* __restrict__ N,
                               const double* __restrict__ W2, const double* __restrict__ P,
                               const double* __restrict__ lam, int64_t rows, int64_t mu, int r,
                               double rho, double gamma, double inv_t, double* __restrict__ W1,
                               double* __restrict__ W3) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * r;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / r;
    const int j = (int)(e - i * r);
    W3[e] = zprox_t(W2R2[e] - P[e], inv_t);
    const double l = i < mu ? lam[j] : 1.0 / lam[j];
    W1[e] = (rho * (WsR1[e] - M[e]) + gamma * l * (W2[e] + N[e])) / (rho + gamma * l * l);
  }
}

// W2 <- argmin f2: (gamma W1 L - gamma N + t G) / (gamma + t), G = (W3 + P) R2^T,
// L = lam on the U block, 1 / lam on the V block
__global__ void rsr_w2_kernel(const double* __restrict__ W1, const double* __restrict__ N,
                              const double* __restrict__ G, const double* __restrict__ lam,
                              int64_t rows, int64_t mu, int r, double gamma, double t,
                              double* __restrict__ W2) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * r;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / r;
    const int j = (int)(e - i * r);
    const double l = i < mu ? lam[j] : 1.0 / lam[j];
    W2[e] = (gamma * W1[e] * l - gamma * N[e] + t * G[e]) / (gamma + t);
  }
}

// out = A + B (elementwise)
__global__ void rsr_add_kernel(const double* __restrict__ A, const double* __restrict__ B,
                               int64_t count, double* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x)
    out[e] = A[e] + B[e];
}

// R^T of an r x r matrix
__global__ void rsr_transpose_kernel(const double* __restrict__ R, int r, double* __restrict__ Rt) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < r * r; e += gridDim.x * blockDim.x)
    Rt[(e % r) * r + e / r] = R[e];
}

// per-block column partials of the quartic's coefficients:
//   a = ||W11(:,i)||^2, b = (W21 + N1)(:,i)^T W11(:,i), c = (W22 + N2)(:,i)^T W12(:,i),
//   d = ||W12(:,i)||^2 ; parts[block][4 r]
__global__ void rsr_colsums_kernel(const double* __restrict__ W1, const double* __restrict__ W2,
                                   const double* __restrict__ N, int64_t rows, int64_t mu, int r,
                                   double* __restrict__ parts) {
  // thread (c, slice): column c = threadIdx.x % r, rows strided by blockDim / r slices
  extern __shared__ double red[];
  const int slices = blockDim.x / r;
  const int c = threadIdx.x % r, sl = threadIdx.x / r;
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  if (sl < slices) {
    for (int64_t i = (int64_t)blockIdx.x * slices + sl; i < rows; i += (int64_t)gridDim.x * slices) {
      const int64_t e = i * r + c;
      const double w1 = W1[e], q = W2[e] + N[e];
      if (i < mu) {
        s[0] = fma(w1, w1, s[0]);
        s[1] = fma(q, w1, s[1]);
      } else {
        s[2] = fma(q, w1, s[2]);
        s[3] = fma(w1, w1, s[3]);
      }
    }
  }
  for (int k = 0; k < 4; ++k) red[threadIdx.x * 4 + k] = sl < slices ? s[k] : 0.0;
  __syncthreads();
  if (threadIdx.x < r) {
    double t[4] = {0.0, 0.0, 0.0, 0.0};
    for (int q = 0; q < slices; ++q)
      for (int k = 0; k < 4; ++k) t[k] += red[(q * r + threadIdx.x) * 4 + k];
    for (int k = 0; k < 4; ++k) parts[(int64_t)blockIdx.x * 4 * r + k * r + threadIdx.x] = t[k];
  }
}

// phi(lam) up to a constant: gamma / 2 (a lam^2 - 2 b lam + d / lam^2 - 2 c / lam)
__device__ __forceinline__ double rsr_phi(double l, double a, double b, double c, double d) {
  return a * l * l - 2.0 * b * l + d / (l * l) - 2.0 * c / l;
}
__device__ __forceinline__ double rsr_quartic(double l, double a, double b, double c, double d) {
  return (((a * l - b) * l) * l + c) * l - d;        // a l^4 - b l^3 + c l - d
}

// lambda_i (reading R37): the positive real root of the quartic with the smallest phi.  Every
// positive root lies in [1 / (1 + max(a, |b|, |c|) / d), 1 + max(|b|, |c|, d) / a] (Cauchy's
// bound on the polynomial and on its reverse); the interval is scanned on a 1024-point
// geometric grid for sign changes, each refined by 200 bisection steps (to the last ulp).
// lam is kept when a or d is 0 (no minimiser in (0, inf)).
__global__ void rsr_lambda_kernel(const double* __restrict__ abcd, int r, double* lam) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < r; i += gridDim.x * blockDim.x) {
    const double a = abcd[i], b = abcd[r + i], c = abcd[2 * r + i], d = abcd[3 * r + i];
    if (!(a > 0.0) || !(d > 0.0)) continue;
    const double lo = 1.0 / (1.0 + fmax(a, fmax(fabs(b), fabs(c))) / d);
    const double hi = 1.0 + fmax(fabs(b), fmax(fabs(c), d)) / a;
    const int NG = 1024;
    const double ratio = pow(hi / lo, 1.0 / NG);
    double best = lam[i], bestv = DBL_MAX;
    double x0 = lo, p0 = rsr_quartic(lo, a, b, c, d);
    for (int k = 1; k <= NG; ++k) {
      const double x1 = k == NG ? hi : lo * pow(ratio, (double)k);
      const double p1 = rsr_quartic(x1, a, b, c, d);
      if ((p0 <= 0.0) != (p1 <= 0.0)) {
        double l = x0, h = x1, pl = p0;
        for (int it = 0; it < 200 && l < h; ++it) {
          const double mid = 0.5 * (l + h);
          if (mid <= l || mid >= h) break;
          const double pm = rsr_quartic(mid, a, b, c, d);
          if ((pm <= 0.0) == (pl <= 0.0)) { l = mid; pl = pm; } else { h = mid; }
        }
        const double root = 0.5 * (l + h);
        const double v = rsr_phi(root, a, b, c, d);
        if (v < bestv) { bestv = v; best = root; }
      }
      x0 = x1;
      p0 = p1;
    }
    lam[i] = best;
  }
}

// multipliers: M += W1 - W_svd R1 ; N += W2 - [W11 Lambda; W12 Lambda^-1] ;
// P += W3 - W2 R2
__global__ void rsr_dual_kernel(const double* __restrict__ W1, const double* __restrict__ WsR1,
                                const double* __restrict__ W2, const double* __restrict__ W3,
                                const double* __restrict__ W2R2, const double* __restrict__ lam,
                                int64_t rows, int64_t mu, int r, double* __restrict__ M,
                                double* __restrict__ N, double* __restrict__ P) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * r;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / r;
    const int j = (int)(e - i * r);
    const double l = i < mu ? lam[j] : 1.0 / lam[j];
    M[e] += W1[e] - WsR1[e];
    N[e] += W2[e] - W1[e] * l;
    P[e] += W3[e] - W2R2[e];
  }
}

// A <- A diag(lam) on the U block, A diag(1 / lam) on the V block
__global__ void rsr_scale_kernel(double* __restrict__ A, const double* __restrict__ lam,
                                 int64_t rows, int64_t mu, int r) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * r;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / r;
    const int j = (int)(e - i * r);
    A[e] *= i < mu ? lam[j] : 1.0 / lam[j];
  }
}

inline int grid_of(int64_t count) {
  return (int)std::min<int64_t>((count + 255) / 256, 8 * kSMs);
}

}  // namespace

constexpr int kRsrColGrid = 2 * kSMs;

int rsr_colsum_parts() { return kRsrColGrid; }

void rsr_w13(const double* WsR1, const double* W2R2, const double* M, const double* N,
             const double* W2, const double* P, const double* lam, int64_t rows, int64_t mu,
             int r, double rho, double gamma, double t, double* W1, double* W3, cudaStream_t st) {
  rsr_w13_kernel<<<grid_of(rows * r), 256, 0, st>>>(WsR1, W2R2, M, N, W2, P, lam, rows, mu, r, rho,
                                                    gamma, 1.0 / t, W1, W3);
  count_launch();
}

void rsr_w2(const double* W1, const double* N, const double* G, const double* lam, int64_t rows,
            int64_t mu, int r, double gamma, double t, double* W2, cudaStream_t st) {
  rsr_w2_kernel<<<grid_of(rows * r), 256, 0, st>>>(W1, N, G, lam, rows, mu, r, gamma, t, W2);
  count_launch();
}

void rsr_add(const double* A, const double* B, int64_t count, double* out, cudaStream_t st) {
  rsr_add_kernel<<<grid_of(count), 256, 0, st>>>(A, B, count, out);
  count_launch();
}

void rsr_transpose(const double* R, int r, double* Rt, cudaStream_t st) {
  rsr_transpose_kernel<<<(r * r + 255) / 256, 256, 0, st>>>(R, r, Rt);
  count_launch();
}

void rsr_lambda(const double* W1, const double* W2, const double* N, int64_t rows, int64_t mu,
                int r, double* parts, double* abcd, double* lam, cudaStream_t st) {
  const int threads = std::max(r, (256 / r) * r);
  rsr_colsums_kernel<<<kRsrColGrid, threads, sizeof(double) * 4 * threads, st>>>(W1, W2, N, rows,
                                                                              mu, r, parts);
  reduce_parts(parts, kRsrColGrid, 4 * r, abcd, st);
  rsr_lambda_kernel<<<1, 128, 0, st>>>(abcd, r, lam);
  count_launch(2);
}

void rsr_dual(const double* W1, const double* WsR1, const double* W2, const double* W3,
              const double* W2R2, const double* lam, int64_t rows, int64_t mu, int r, double* M,
              double* N, double* P, cudaStream_t st) {
  rsr_dual_kernel<<<grid_of(rows * r), 256, 0, st>>>(W1, WsR1, W2, W3, W2R2, lam, rows, mu, r, M,
                                                     N, P);
  count_launch();
}

void rsr_scale(double* A, const double* lam, int64_t rows, int64_t mu, int r, cudaStream_t st) {
  rsr_scale_kernel<<<grid_of(rows * r), 256, 0, st>>>(A, lam, rows, mu, r);
  count_launch();
}

}  // namespace enmf
