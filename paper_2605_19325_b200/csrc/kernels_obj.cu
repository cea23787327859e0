// kernels_obj.cu -- direct objective sum_ij (X_ij - U_i . V_j)^2 (Eq.(1)),
// the validator of the trace form (reading R16).  64x64 tiles of X, the matching U and V
// rows staged transposed in shared memory (fp64), fp64 residuals, one partial per CTA in
// a fixed tile order (deterministic).
#include "internal.h"

namespace enmf {
namespace {

constexpr int T = 64;

__global__ void __launch_bounds__(256)
frob_direct_kernel(const float* __restrict__ X, int64_t ldx, int64_t rows, int64_t n,
                   const float* __restrict__ U, int64_t ldu, const float* __restrict__ V,
                   int64_t ldv, int r, double* parts) {
  extern __shared__ double sm[];
  double* Ut = sm;            // [r][T]
  double* Vt = sm + r * T;    // [r][T]
  __shared__ double red[256];
  const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
  const int64_t tiles_i = (rows + T - 1) / T, tiles_j = (n + T - 1) / T;
  double acc = 0.0;
  for (int64_t tile = blockIdx.x; tile < tiles_i * tiles_j; tile += gridDim.x) {
    const int64_t i0 = (tile / tiles_j) * T, j0 = (tile % tiles_j) * T;
    for (int e = t; e < r * T; e += 256) {
      const int row = e / r, l = e % r;
      Ut[l * T + row] = (i0 + row < rows) ? (double)U[(i0 + row) * ldu + l] : 0.0;
      Vt[l * T + row] = (j0 + row < n) ? (double)V[(j0 + row) * ldv + l] : 0.0;
    }
    __syncthreads();
    double d[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) d[a][b] = 0.0;
    for (int l = 0; l < r; ++l) {
      double uv[4], vv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) uv[a] = Ut[l * T + ty + 16 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) vv[b] = Vt[l * T + tx + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) d[a][b] = fma(uv[a], vv[b], d[a][b]);
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int64_t i = i0 + ty + 16 * a;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int64_t j = j0 + tx + 16 * b;
        if (i < rows && j < n) {
          const double e = (double)X[i * ldx + j] - d[a][b];
          acc = fma(e, e, acc);
        }
      }
    }
    __syncthreads();
  }
  red[t] = acc;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (t < o) red[t] += red[t + o];
    __syncthreads();
  }
  if (t == 0) parts[blockIdx.x] = red[0];
}

}  // namespace

void frob_direct(const float* X, int64_t ldx, int64_t rows, int64_t n, const float* U,
                 int64_t ldu, const float* V, int64_t ldv, int r, double* parts, int* nparts,
                 cudaStream_t st) {
  const int grid = 4 * kSMs;
  const size_t sm = sizeof(double) * 2 * (size_t)r * T;
  cudaFuncSetAttribute(frob_direct_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)sm);
  frob_direct_kernel<<<grid, 256, sm, st>>>(X, ldx, rows, n, U, ldu, V, ldv, r, parts);
  count_launch();
  *nparts = grid;
}

}  // namespace enmf
