// nmc.cu -- kernels of eNMC, the exterior method for nonnegative matrix COMPLETION (PAPER.md
// App. C; Alg. NMC), on the observed entries of X bound by
// enmf_set_data_masked (CSR lists, plus the handle's CSC copy for the V side):
//
//   nmc_resid_spmm   one half step of softImpute-ALS (Hastie et al. 2015, Alg. 3.1, the
//                    paper's init, lambda = 0: reading R31): T = S^T U + B D (V side) or
//                    T = S V + A D (U side), with S = P_E(X - A B^T) formed entry by entry
//                    from the observed values -- the completed matrix X* = S + A B^T is never
//                    materialised (X*^T U = S^T U + B A^T U = S^T U + B D, U orthonormal)
//   nmc_objective    f^ = sum over observed (i, j) of (x_ij - u_i . v_j)^2 (reported
//                    un-halved like Eq.(1), reading R2)
//   nmc_svals        D~ = sqrt(sigma) and 1 / sigma from the eigenvalues sigma^2 of T^T T
//
// The masked PBCD of the sweeps is nmc_pbcd_kernel (kernels_rows.cu).  All fp64, SIMT: the
// observed entries are ~4.5 % of X at the C4 / MovieLens shape, so a sweep is
// bound by the per-row Gram build (nnz_i r^2 fp64 FMAs) and the PBCD iterations, not by bytes.
#include <float.h>

#include "internal.h"

namespace enmf {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kNmcWarps = 8;

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// out[row] = sum_{e in row} (val_e - Fr[row] . O1[idx_e]) O2[idx_e] + Fr[row] o dsc
// (r <= 64: lanes own columns lane, lane + 32).  One warp per row, entries in list order.
__global__ void __launch_bounds__(32 * kNmcWarps)
nmc_resid_spmm_kernel(const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                      const float* __restrict__ val, int64_t rows, int r,
                      const double* __restrict__ Fr, const double* __restrict__ O1,
                      const double* __restrict__ O2, const double* __restrict__ dsc,
                      double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < rows;
       row += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    double f[2], acc[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int col = lane + 32 * c;
      f[c] = col < r ? Fr[row * r + col] : 0.0;
      acc[c] = col < r ? f[c] * dsc[col] : 0.0;
    }
    for (int64_t e = ptr[row]; e < ptr[row + 1]; ++e) {
      const int64_t j = idx[e];
      double d = 0.0;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int col = lane + 32 * c;
        if (col < r) d = fma(f[c], O1[j * r + col], d);
      }
      const double s = (double)val[e] - warp_sum_d(d);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int col = lane + 32 * c;
        if (col < r) acc[c] = fma(s, O2[j * r + col], acc[c]);
      }
    }
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int col = lane + 32 * c;
      if (col < r) out[row * r + col] = acc[c];
    }
  }
}

// per-warp partial sums of (x_ij - u_i . v_j)^2 over the observed entries (fp32 factors)
__global__ void __launch_bounds__(32 * kNmcWarps)
nmc_objective_kernel(const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                     const float* __restrict__ val, int64_t rows, int r,
                     const float* __restrict__ U, int64_t ldu, const float* __restrict__ V,
                     int64_t ldv, double* __restrict__ parts) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < rows;
       row += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    double u[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int col = lane + 32 * c;
      u[c] = col < r ? (double)U[row * ldu + col] : 0.0;
    }
    for (int64_t e = ptr[row]; e < ptr[row + 1]; ++e) {
      const int64_t j = idx[e];
      double d = 0.0;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int col = lane + 32 * c;
        if (col < r) d = fma(u[c], (double)V[j * ldv + col], d);
      }
      const double res = (double)val[e] - warp_sum_d(d);
      s = fma(res, res, s);              // identical on every lane: lane 0 keeps it
    }
  }
  __shared__ double ws[kNmcWarps];
  if (lane == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kNmcWarps; ++w) t += ws[w];
    parts[blockIdx.x] = t;
  }
}

// sv: eigenvalues sigma^2 of T^T T (descending, jacobi_svd) -> d = sqrt(sigma) (the D~ of
// B~ D = V~ D~^2 R^T) and inv = 1 / sigma (0 for sigma <= 1e-14 sigma_1: rank deficiency)
__global__ void nmc_svals_kernel(const double* __restrict__ sv, int r, double* d, double* inv) {
  const double s1 = sqrt(fmax(sv[0], 0.0));
  for (int k = threadIdx.x; k < r; k += blockDim.x) {
    const double s = sqrt(fmax(sv[k], 0.0));
    const bool ok = s > 1e-14 * s1 && s > 0.0;
    d[k] = ok ? sqrt(s) : 0.0;
    inv[k] = ok ? 1.0 / s : 0.0;
  }
}

}  // namespace

constexpr int kNmcGrid = 2 * kSMs;

void nmc_resid_spmm(const int64_t* ptr, const int32_t* idx, const float* val, int64_t rows,
                    int r, const double* Fr, const double* O1, const double* O2,
                    const double* dsc, double* out, cudaStream_t st) {
  nmc_resid_spmm_kernel<<<kNmcGrid, 32 * kNmcWarps, 0, st>>>(ptr, idx, val, rows, r, Fr, O1, O2,
                                                             dsc, out);
  count_launch();
}

int nmc_objective_parts() { return kNmcGrid; }

void nmc_objective(const int64_t* ptr, const int32_t* idx, const float* val, int64_t rows, int r,
                   const float* U, int64_t ldu, const float* V, int64_t ldv, double* parts,
                   double* out, cudaStream_t st) {
  nmc_objective_kernel<<<kNmcGrid, 32 * kNmcWarps, 0, st>>>(ptr, idx, val, rows, r, U, ldu, V,
                                                            ldv, parts);
  reduce_parts(parts, kNmcGrid, 1, out, st);
  count_launch();
}

void nmc_svals(const double* sv, int r, double* d, double* inv, cudaStream_t st) {
  nmc_svals_kernel<<<1, 128, 0, st>>>(sv, r, d, inv);
  count_launch();
}

}  // namespace enmf
