// synth_gpu.cu -- device side of the synthetic-input generator (see synth_core.h).
// Bench / test infrastructure, not the eNMF product path: writes X row ranges
// directly into HBM, bit-identical to synth_cpu.c.  Build with --fmad=false.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>
#include "synth_core.h"

namespace {

__global__ void factor_kernel(int recipe, uint64_t seed, int which, int64_t begin,
                              int64_t count, int k, float* out) {
  int64_t total = count * (int64_t)k;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e / k;
    int c = (int)(e - r * k);
    out[e] = which == 0 ? syn_rowf(recipe, seed, (uint64_t)(begin + r), k, c)
                        : syn_colf(recipe, seed, (uint64_t)(begin + r), k, c);
  }
}

constexpr int TM = 64, TN = 64, KC = 32;

// mode 0: write X; mode 1: max of S into *smax_bits (positive doubles order as uint64).
template <int MODE>
__global__ void __launch_bounds__(256) x_kernel(int recipe, uint64_t seed, int64_t n, int k,
                                                double noise, double smax, int64_t row_begin,
                                                int64_t row_count, const float* __restrict__ A,
                                                const float* __restrict__ B, float* X, int64_t ldx,
                                                unsigned long long* smax_bits) {
  __shared__ float sA[TM][KC + 1];
  __shared__ float sB[TN][KC + 1];
  const int t = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.y * TM;
  const int64_t c0 = (int64_t)blockIdx.x * TN;
  const int tr = (t / 16) * 4, tc = (t % 16) * 4;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  if (recipe != SYN_RATINGS) {
    for (int kc = 0; kc < k; kc += KC) {
      for (int e = t; e < TM * KC; e += 256) {
        int rr = e / KC, cc = e % KC;
        int64_t gr = r0 + rr;
        sA[rr][cc] = (gr < row_count && kc + cc < k) ? A[gr * k + kc + cc] : 0.0f;
        int64_t gc = c0 + rr;
        sB[rr][cc] = (gc < n && kc + cc < k) ? B[gc * k + kc + cc] : 0.0f;
      }
      __syncthreads();
      int kend = k - kc < KC ? k - kc : KC;
      for (int c = 0; c < kend; ++c) {
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b)
            acc[a][b] = acc[a][b] + (double)sA[tr + a][c] * (double)sB[tc + b][c];
      }
      __syncthreads();
    }
  }
  double local_max = 0.0;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    int64_t gr = r0 + tr + a;
    if (gr >= row_count) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      int64_t gc = c0 + tc + b;
      if (gc >= n) continue;
      if (MODE == 0) {
        X[gr * ldx + gc] = syn_x_from_s(recipe, seed, (uint64_t)(row_begin + gr), (uint64_t)gc,
                                        (uint64_t)n, acc[a][b], noise, smax);
      } else {
        local_max = acc[a][b] > local_max ? acc[a][b] : local_max;
      }
    }
  }
  if (MODE == 1) atomicMax(smax_bits, (unsigned long long)__double_as_longlong(local_max));
}

// SPARSE recipe, warp per row: entry counts (fill == false) or the CSR fill (columns
// ascending; positions from a ballot prefix).  A: rows of this range, B: all columns.
template <bool FILL>
__global__ void __launch_bounds__(256) csr_kernel(uint64_t seed, int64_t n, int k, double noise,
                                                  double density, int64_t row_begin,
                                                  int64_t row_count, const float* __restrict__ A,
                                                  const float* __restrict__ B, int64_t* counts,
                                                  const int64_t* rowptr, int32_t* colidx,
                                                  float* vals) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (r >= row_count) return;
  const uint64_t i = (uint64_t)(row_begin + r);
  int64_t pos = FILL ? rowptr[r] : 0;
  for (int64_t j0 = 0; j0 < n; j0 += 32) {
    const int64_t j = j0 + lane;
    const int keep = j < n && syn_sparse_keep(seed, i, (uint64_t)j, (uint64_t)n, density);
    const unsigned mask = __ballot_sync(0xffffffffu, keep);
    if (FILL && keep) {
      const int64_t p = pos + __popc(mask & ((1u << lane) - 1u));
      const double s = syn_dot(A + r * k, B + j * k, k);
      colidx[p] = (int32_t)j;
      vals[p] = syn_x_from_s(SYN_SPARSE, seed, i, (uint64_t)j, (uint64_t)n, s, noise, density);
    }
    pos += __popc(mask);
  }
  if (!FILL && lane == 0) counts[r] = pos;
}

}  // namespace

extern "C" {

// SPARSE recipe on the device: counts (row_count entries) when rowptr == NULL, else the CSR
// fill of colidx / vals given rowptr (row_count + 1, exclusive prefix of the counts).
int synth_gpu_csr_rows(uint64_t seed, int64_t m, int64_t n, int k, double noise, double density,
                       int64_t row_begin, int64_t row_count, int64_t* counts,
                       const int64_t* rowptr, int32_t* colidx, float* vals, void* stream_ptr) {
  if (row_begin < 0 || row_count < 0 || row_begin + row_count > m) return 1;
  if (row_count == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream_ptr;
  const unsigned grid = (unsigned)((row_count * 32 + 255) / 256);
  if (!rowptr) {
    csr_kernel<false><<<grid, 256, 0, st>>>(seed, n, k, noise, density, row_begin, row_count,
                                            nullptr, nullptr, counts, nullptr, nullptr, nullptr);
    return cudaGetLastError();
  }
  float* A = nullptr;
  float* B = nullptr;
  cudaError_t err;
  if ((err = cudaMallocAsync(&A, sizeof(float) * row_count * k, st))) return err;
  if ((err = cudaMallocAsync(&B, sizeof(float) * n * k, st))) return err;
  factor_kernel<<<1184, 256, 0, st>>>(SYN_SPARSE, seed, 0, row_begin, row_count, k, A);
  factor_kernel<<<1184, 256, 0, st>>>(SYN_SPARSE, seed, 1, 0, n, k, B);
  csr_kernel<true><<<grid, 256, 0, st>>>(seed, n, k, noise, density, row_begin, row_count, A, B,
                                         nullptr, rowptr, colidx, vals);
  err = cudaGetLastError();
  cudaFreeAsync(A, st);
  cudaFreeAsync(B, st);
  return err;
}

// Returns a cudaError_t value (0 = success).
int synth_gpu_x_rows(int recipe, uint64_t seed, int64_t m, int64_t n, int k, double noise,
                     double smax, int64_t row_begin, int64_t row_count, float* dX, int64_t ldx,
                     void* stream_ptr) {
  if (row_begin < 0 || row_count < 0 || row_begin + row_count > m || ldx < n) return 1;
  if (row_count == 0 || n == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream_ptr;
  float* A = nullptr;
  float* B = nullptr;
  cudaError_t err = cudaSuccess;
  if (recipe != SYN_RATINGS) {
    if ((err = cudaMallocAsync(&A, sizeof(float) * row_count * k, st))) return err;
    if ((err = cudaMallocAsync(&B, sizeof(float) * n * k, st))) return err;
    factor_kernel<<<1184, 256, 0, st>>>(recipe, seed, 0, row_begin, row_count, k, A);
    factor_kernel<<<1184, 256, 0, st>>>(recipe, seed, 1, 0, n, k, B);
  }
  // grid.y is limited to 65535: walk the rows in slabs.
  const int64_t slab = (int64_t)65535 * TM;
  for (int64_t s = 0; s < row_count; s += slab) {
    int64_t cnt = row_count - s < slab ? row_count - s : slab;
    dim3 grid((unsigned)((n + TN - 1) / TN), (unsigned)((cnt + TM - 1) / TM));
    x_kernel<0><<<grid, 256, 0, st>>>(recipe, seed, n, k, noise, smax, row_begin + s, cnt,
                                      A ? A + s * k : nullptr, B, dX + s * ldx, ldx, nullptr);
  }
  err = cudaGetLastError();
  if (A) cudaFreeAsync(A, st);
  if (B) cudaFreeAsync(B, st);
  return err;
}

// Global max of S = A B^T (IMAGE recipe normalisation), computed on the device.
int synth_gpu_smax(int recipe, uint64_t seed, int64_t m, int64_t n, int k, double* smax_out,
                   void* stream_ptr) {
  cudaStream_t st = (cudaStream_t)stream_ptr;
  float *A, *B;
  unsigned long long* bits;
  cudaError_t err;
  if ((err = cudaMallocAsync(&A, sizeof(float) * m * k, st))) return err;
  if ((err = cudaMallocAsync(&B, sizeof(float) * n * k, st))) return err;
  if ((err = cudaMallocAsync(&bits, sizeof(unsigned long long), st))) return err;
  cudaMemsetAsync(bits, 0, sizeof(unsigned long long), st);
  factor_kernel<<<1184, 256, 0, st>>>(recipe, seed, 0, 0, m, k, A);
  factor_kernel<<<1184, 256, 0, st>>>(recipe, seed, 1, 0, n, k, B);
  const int64_t slab = (int64_t)65535 * TM;
  for (int64_t s = 0; s < m; s += slab) {
    int64_t cnt = m - s < slab ? m - s : slab;
    dim3 grid((unsigned)((n + TN - 1) / TN), (unsigned)((cnt + TM - 1) / TM));
    x_kernel<1><<<grid, 256, 0, st>>>(recipe, seed, n, k, 0.0, 0.0, s, cnt, A + s * k, B,
                                      nullptr, n, bits);
  }
  unsigned long long h = 0;
  cudaMemcpyAsync(&h, bits, sizeof(h), cudaMemcpyDeviceToHost, st);
  err = cudaStreamSynchronize(st);
  cudaFreeAsync(A, st);
  cudaFreeAsync(B, st);
  cudaFreeAsync(bits, st);
  double d;
  memcpy(&d, &h, sizeof(d));
  *smax_out = d;
  return err;
}

}  // extern "C"
