// kernels_sparse.cu -- the X passes for a sparse X held as CSR (the
// paper's ultra-large sparse Reuters experiment, PAPER.md:418 and Table reuters).
//
// eNMF touches X only through P = X V and Q = X^T U and ||X||^2; the
// block updates, Grams and the trace-form objective are unchanged.  A sparse X therefore only
// swaps the two contractions for sparse-times-dense products (SpMM):
//   * P = X V from the caller's CSR (rows of this rank), Q = X^T U from a CSC copy built once
//     per enmf_set_data_csr (stable radix sort of the column indices, so every column lists
//     its entries in ascending row order and Q is summed in a fixed order: deterministic);
//   * one warp per output row, lane l owns columns l, l + 32, l + 64, l + 96 of a <= 128-wide
//     column block; the warp loads 32 (index, value) pairs at once (coalesced, then shuffled),
//     keeps 8 factor rows in flight per step, and for each stored entry reads the
//     factor row coalesced (128 x 4 B from L2: the factor is 25-100 MB and stays resident in
//     the 126 MB L2 far better than X streams), and accumulates x * f in fp64 (the objective's
//     conditioning needs P, Q to ~1e-12, as the dense fp64 path provides).
// Bound: fp64 FMA (128 per stored entry) with the CSR bytes (8-12 B per entry) streamed once.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <float.h>

#include <algorithm>

#include "internal.h"

namespace enmf {
namespace {

constexpr int kSpWarps = 8;                  // warps (rows) per block

template <typename T>
__global__ void __launch_bounds__(32 * kSpWarps)
spmm_kernel(const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
            const float* __restrict__ val, int64_t rows, const T* __restrict__ B, int64_t ldb,
            int ncols, double* __restrict__ out, int64_t ldo) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * kSpWarps + (threadIdx.x >> 5);
  if (row >= rows) return;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const int64_t e0 = ptr[row], e1 = ptr[row + 1];
  // 32 (index, value) pairs per coalesced load, then 8 factor rows in flight per step; the
  // accumulation order is the entry order (deterministic); padding entries add x = 0
  for (int64_t base = e0; base < e1; base += 32) {
    const int cnt = (int)(e1 - base < 32 ? e1 - base : 32);
    int myj = 0;
    double myx = 0.0;
    if (lane < cnt) {
      myj = idx[base + lane];
      myx = (double)val[base + lane];
    }
    const int j_pad = __shfl_sync(0xffffffffu, myj, 0);
    for (int q = 0; q < cnt; q += 8) {
      int jj[8];
      double xx[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int jv = __shfl_sync(0xffffffffu, myj, (q + u) & 31);
        const double xv = __shfl_sync(0xffffffffu, myx, (q + u) & 31);
        jj[u] = q + u < cnt ? jv : j_pad;
        xx[u] = q + u < cnt ? xv : 0.0;
      }
      T f[8][4];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const T* bu = B + (int64_t)jj[u] * ldb;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int col = lane + 32 * c;
          f[u][c] = col < ncols ? bu[col] : T(0);
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[c] = fma(xx[u], (double)f[u][c], acc[c]);
    }
  }
  double* o = out + row * ldo;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int col = lane + 32 * c;
    if (col < ncols) o[col] = acc[c];
  }
}

// row id of every stored entry (input of the CSC sort)
__global__ void csr_rowid_kernel(const int64_t* __restrict__ ptr, int64_t rows, int32_t* rowid) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * kSpWarps + (threadIdx.x >> 5);
  if (row >= rows) return;
  for (int64_t e = ptr[row] + lane; e < ptr[row + 1]; e += 32) rowid[e] = (int32_t)row;
}

__global__ void iota_kernel(int32_t* a, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    a[e] = (int32_t)e;
}

__global__ void col_count_kernel(const int32_t* __restrict__ col, int64_t nnz, int64_t n,
                                 unsigned long long* cnt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = col[e];
    if (c >= 0 && c < n) atomicAdd(&cnt[c], 1ull);
  }
}

// CSC arrays from the stably sorted entry permutation
__global__ void csc_gather_kernel(const int32_t* __restrict__ perm, const int32_t* __restrict__ rowid,
                                  const float* __restrict__ val, int64_t nnz, int32_t* crow,
                                  float* cval) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = perm[e];
    crow[e] = rowid[p];
    cval[e] = val[p];
  }
}

// column indices in range and ascending within each row, row_ptr[0] = 0 and
// row_ptr[rows] = nnz (the layout the paths assume: every stored entry belongs to a row)
__global__ void csr_check_kernel(const int64_t* __restrict__ ptr, const int32_t* __restrict__ col,
                                 int64_t rows, int64_t n, int64_t nnz, int* bad) {
  if (blockIdx.x == 0 && threadIdx.x == 0 && (ptr[0] != 0 || ptr[rows] != nnz)) atomicOr(bad, 1);
  for (int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; row < rows;
       row += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e0 = ptr[row], e1 = ptr[row + 1];
    if (e0 < 0 || e1 < e0 || e1 > nnz) {
      atomicOr(bad, 1);
      continue;
    }
    int32_t prev = -1;
    for (int64_t e = e0; e < e1; ++e) {
      const int32_t c = col[e];
      if (c <= prev || c >= n) {
        atomicOr(bad, 1);
        break;
      }
      prev = c;
    }
  }
}

// sum over stored entries of x_ij (u_i . v_j): the cross term of the exact objective
__global__ void __launch_bounds__(32 * kSpWarps)
sddmm_dot_kernel(const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                 const float* __restrict__ val, int64_t rows, const float* __restrict__ U,
                 int64_t ldu, const float* __restrict__ V, int64_t ldv, int r, double* parts) {
  __shared__ double wsum[kSpWarps];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t row = (int64_t)blockIdx.x * kSpWarps + w;
  double s = 0.0;
  if (row < rows) {
    const float* u = U + row * ldu;
    for (int64_t e = ptr[row]; e < ptr[row + 1]; ++e) {
      const float* v = V + (int64_t)idx[e] * ldv;
      double d = 0.0;
      for (int c = lane; c < r; c += 32) d = fma((double)u[c], (double)v[c], d);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
      s = fma((double)val[e], d, s);
    }
  }
  if (lane == 0) wsum[w] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < kSpWarps; ++k) t += wsum[k];
    parts[blockIdx.x] = t;
  }
}

int blocks_for_rows(int64_t rows) { return (int)((rows + kSpWarps - 1) / kSpWarps); }

}  // namespace

template <typename T>
void spmm(const int64_t* ptr, const int32_t* idx, const float* val, int64_t rows, const T* B,
          int64_t ldb, int ncols, double* out, int64_t ldo, cudaStream_t st) {
  if (rows <= 0) return;
  for (int c0 = 0; c0 < ncols; c0 += 128) {
    const int nc = ncols - c0 < 128 ? ncols - c0 : 128;
    spmm_kernel<T><<<blocks_for_rows(rows), 32 * kSpWarps, 0, st>>>(ptr, idx, val, rows, B + c0,
                                                                    ldb, nc, out + c0, ldo);
    count_launch();
  }
}
template void spmm<float>(const int64_t*, const int32_t*, const float*, int64_t, const float*,
                          int64_t, int, double*, int64_t, cudaStream_t);
template void spmm<double>(const int64_t*, const int32_t*, const float*, int64_t, const double*,
                           int64_t, int, double*, int64_t, cudaStream_t);

int csr_check(const int64_t* ptr, const int32_t* col, int64_t rows, int64_t n, int64_t nnz,
              int* bad_dev, cudaStream_t st) {
  if (cudaMemsetAsync(bad_dev, 0, sizeof(int), st) != cudaSuccess) return 1;
  if (rows > 0) {
    csr_check_kernel<<<4 * kSMs, 256, 0, st>>>(ptr, col, rows, n, nnz, bad_dev);
    count_launch();
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

// CSC (colptr n + 1, rowidx nnz, cval nnz) of a CSR block; scratch from cudaMallocAsync.
int csr_to_csc(const int64_t* ptr, const int32_t* col, const float* val, int64_t rows, int64_t n,
               int64_t nnz, int64_t* colptr, int32_t* rowidx, float* cval, cudaStream_t st) {
  if (nnz > INT32_MAX || n > INT32_MAX) return 2;
  int32_t *rowid = nullptr, *perm_in = nullptr, *perm_out = nullptr, *keys_out = nullptr;
  unsigned long long* cnt = nullptr;
  void* tmp = nullptr;
  size_t tmp_sort = 0, tmp_scan = 0;
  const int nn = (int)nnz;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_sort, col, keys_out, perm_in, perm_out, nn, 0,
                                  32, st);
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_scan, cnt, reinterpret_cast<unsigned long long*>(colptr),
                                (int)(n + 1), st);
  const size_t tmp_bytes = std::max(tmp_sort, tmp_scan) + 256;
  const size_t e = (size_t)std::max<int64_t>(nnz, 1);
  if (cudaMallocAsync(&rowid, 4 * e, st) || cudaMallocAsync(&perm_in, 4 * e, st) ||
      cudaMallocAsync(&perm_out, 4 * e, st) || cudaMallocAsync(&keys_out, 4 * e, st) ||
      cudaMallocAsync(&cnt, 8 * (size_t)(n + 1), st) || cudaMallocAsync(&tmp, tmp_bytes, st)) {
    cudaGetLastError();
    return 2;
  }
  if (rows > 0) csr_rowid_kernel<<<blocks_for_rows(rows), 32 * kSpWarps, 0, st>>>(ptr, rows, rowid);
  iota_kernel<<<4 * kSMs, 256, 0, st>>>(perm_in, nnz);
  // stable LSD radix sort by column: within a column the entries keep their CSR (row) order
  size_t tb = tmp_bytes;
  cub::DeviceRadixSort::SortPairs(tmp, tb, col, keys_out, perm_in, perm_out, nn, 0, 32, st);
  csc_gather_kernel<<<4 * kSMs, 256, 0, st>>>(perm_out, rowid, val, nnz, rowidx, cval);
  cudaMemsetAsync(cnt, 0, 8 * (size_t)(n + 1), st);
  col_count_kernel<<<4 * kSMs, 256, 0, st>>>(col, nnz, n, cnt);
  tb = tmp_bytes;
  cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, reinterpret_cast<unsigned long long*>(colptr),
                                (int)(n + 1), st);
  count_launch(6);
  cudaFreeAsync(rowid, st);
  cudaFreeAsync(perm_in, st);
  cudaFreeAsync(perm_out, st);
  cudaFreeAsync(keys_out, st);
  cudaFreeAsync(cnt, st);
  cudaFreeAsync(tmp, st);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int sddmm_parts(int64_t rows) { return std::max(1, blocks_for_rows(rows)); }

void sddmm_dot(const int64_t* ptr, const int32_t* idx, const float* val, int64_t rows,
               const float* U, int64_t ldu, const float* V, int64_t ldv, int r, double* parts,
               double* out, cudaStream_t st) {
  const int np = sddmm_parts(rows);
  if (rows > 0) {
    sddmm_dot_kernel<<<np, 32 * kSpWarps, 0, st>>>(ptr, idx, val, rows, U, ldu, V, ldv, r, parts);
    count_launch();
  } else {
    cudaMemsetAsync(parts, 0, sizeof(double), st);
  }
  reduce_parts(parts, np, 1, out, st);
}

}  // namespace enmf
