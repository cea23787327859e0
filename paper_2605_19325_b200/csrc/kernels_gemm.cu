// kernels_gemm.cu -- SIMT GEMMs with fp64 accumulation (the ENMF_PREC_FP64 path and the
// small dense products of init / ADMM).
//
// Used for the cross terms X V and X^T U, the Grams U^T U, V^T V, the
// range-finder products X Omega, X^T Q and the ADMM products W R,
// W^T B.  64x64 output tiles, 16-deep K slabs staged in shared memory
// as fp64, 16 x 32 warp tiles on the fp64 tensor cores (DMMA m8n8k4), split-K layers reduced
// in a fixed order.
#include "internal.h"

namespace enmf {
namespace {

constexpr int BM = 64, BN = 64, BK = 16;
constexpr int LDS = BM + 4;   // padded slab rows: the DMMA fragment loads (4 k x 8 rows) hit 16 banks

// D(8x8) += A(8x4) B(4x8) on the fp64 tensor cores: lane holds A[lane/4][lane%4],
// B[lane%4][lane/4] and D[lane/4][2 (lane%4) + {0, 1}].
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// 64 x 64 output tile, 16-deep K slabs staged in shared memory as fp64 (k-major), next slab
// prefetched into registers; the 8 warps are a 4 x 2 grid of 16 x 32 warp tiles on the fp64
// tensor cores (DMMA m8n8k4: 8 per 4-deep k step from 6 operand loads per lane).  Round 1-2c
// used 4 x 4 SIMT register tiles: 35 % of the fp64 rate, bound by shared-memory wavefronts
// (profiles/r02d_small_notes.md); DMMA has the same peak and ~1/5 of the operand traffic.
template <typename TA, typename TB, bool TRANS>
__global__ void __launch_bounds__(256)
gemm_kernel(const TA* __restrict__ A, int64_t lda, const TB* __restrict__ B, int64_t ldb,
            int64_t M, int64_t N, int64_t K, int64_t kchunk, double* __restrict__ out,
            int64_t ldo, int64_t split_stride) {
  __shared__ double As[BK][LDS];
  __shared__ double Bs[BK][LDS];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int wr = warp >> 1, wc = warp & 1;
  const int64_t i0 = (int64_t)blockIdx.y * BM, j0 = (int64_t)blockIdx.x * BN;
  const int64_t kb = (int64_t)blockIdx.z * kchunk;
  const int64_t ke = K < kb + kchunk ? K : kb + kchunk;
  double acc[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  double ar[4], br[4];
  auto fetch = [&](int64_t k0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = t + 256 * q;
      int ii, kk;
      if (TRANS) { kk = e / BM; ii = e % BM; }
      else { ii = e / BK; kk = e % BK; }
      const int64_t gi = i0 + ii, gk = k0 + kk;
      ar[q] = (gi < M && gk < ke) ? (double)(TRANS ? A[gk * lda + gi] : A[gi * lda + gk]) : 0.0;
      const int kb2 = e / BN, jj = e % BN;
      const int64_t gj = j0 + jj, gk2 = k0 + kb2;
      br[q] = (gj < N && gk2 < ke) ? (double)B[gk2 * ldb + gj] : 0.0;
    }
  };
  fetch(kb);
  const double* xa = &As[lane & 3][16 * wr + (lane >> 2)];
  const double* xb = &Bs[lane & 3][32 * wc + (lane >> 2)];
  for (int64_t k0 = kb; k0 < ke; k0 += BK) {
    __syncthreads();                       // the previous slab's MMAs are done
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = t + 256 * q;
      int ii, kk;
      if (TRANS) { kk = e / BM; ii = e % BM; }
      else { ii = e / BK; kk = e % BK; }
      As[kk][ii] = ar[q];
      Bs[e / BN][e % BN] = br[q];
    }
    __syncthreads();
    if (k0 + BK < ke) fetch(k0 + BK);      // next slab's loads in flight during the MMAs
#pragma unroll
    for (int k4 = 0; k4 < BK; k4 += 4) {
      const double a0 = xa[k4 * LDS], a1 = xa[k4 * LDS + 8];
      double bv[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = xb[k4 * LDS + 8 * j];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        dmma884(acc[0][j][0], acc[0][j][1], a0, bv[j]);
        dmma884(acc[1][j][0], acc[1][j][1], a1, bv[j]);
      }
    }
  }
  double* o = out + (int64_t)blockIdx.z * split_stride;
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const int64_t gi = i0 + 16 * wr + 8 * a + (lane >> 2);
    if (gi >= M) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t gj = j0 + 32 * wc + 8 * b + 2 * (lane & 3) + e;
        if (gj < N) o[gi * ldo + gj] = acc[a][b][e];
      }
  }
}

__global__ void reduce_parts_kernel(const double* __restrict__ parts, int nparts, int64_t len,
                                    double* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < len;
       e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
#pragma unroll 8
    for (int p = 0; p < nparts; ++p) s += parts[(int64_t)p * len + e];   // loads batched, order kept
    out[e] = s;
  }
}

// long outputs (the pass-2 split-K partials, n x r): 16-byte loads, 4 independent double2 per
// thread and iteration so that enough loads are in flight (the scalar loop ran at ~1 TB/s);
// the same per-element summation order as reduce_parts_kernel (bitwise equal results)
__global__ void __launch_bounds__(256) reduce_parts_vec_kernel(const double2* __restrict__ parts,
                                                               int nparts, int64_t len2,
                                                               double2* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e0 < len2; e0 += 4 * stride) {
    double2 s[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) s[u] = make_double2(0.0, 0.0);
    for (int p = 0; p < nparts; ++p) {
      double2 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t e = e0 + u * stride;
        v[u] = e < len2 ? parts[(int64_t)p * len2 + e] : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        s[u].x += v[u].x;
        s[u].y += v[u].y;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t e = e0 + u * stride;
      if (e < len2) out[e] = s[u];
    }
  }
}

// short outputs (len <= 64: scalars, the PBCD stopping vector): one block per element, the
// parts strided over 256 threads and a fixed-order tree -- deterministic, and no single
// thread walking hundreds of dependent loads
__global__ void __launch_bounds__(256) reduce_parts_short_kernel(const double* __restrict__ parts,
                                                                 int nparts, int64_t len,
                                                                 double* __restrict__ out) {
  __shared__ double red[256];
  const int64_t e = blockIdx.x;
  double s = 0.0;
  for (int p = threadIdx.x; p < nparts; p += 256) s += parts[(int64_t)p * len + e];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[e] = red[0];
}

__global__ void f64_to_f32_kernel(const double* __restrict__ A, int64_t rows, int64_t cols,
                                  const double* __restrict__ colscale, float* __restrict__ B,
                                  int64_t ldb) {
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / cols, j = e - i * cols;
    double v = A[e];
    if (colscale) v *= colscale[j];
    B[i * ldb + j] = (float)v;
  }
}

__global__ void f32_to_f64_kernel(const float* __restrict__ A, int64_t lda, int64_t rows,
                                  int64_t cols, double* __restrict__ B) {
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / cols, j = e - i * cols;
    B[e] = (double)A[i * lda + j];
  }
}

inline int grid_for(int64_t n, int per = 256) {
  int64_t g = (n + per - 1) / per;
  return (int)(g < 4 * kSMs ? (g < 1 ? 1 : g) : 4 * kSMs);
}

}  // namespace

template <typename TA, typename TB>
void gemm(bool transA, const TA* A, int64_t lda, const TB* B, int64_t ldb, int64_t M,
          int64_t N, int64_t K, GemmOut out, double* work, size_t work_elems,
          cudaStream_t st) {
  if (M <= 0 || N <= 0) return;
  const int64_t tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  int64_t splits = (2 * kSMs + tiles - 1) / tiles;
  const int64_t kmax = (K + 255) / 256;
  if (splits > kmax) splits = kmax;
  if (splits < 1) splits = 1;
  const int64_t need_extra = (out.Cf || (out.C && out.ldc != N)) ? 1 : 0;
  while (splits > 1 && (size_t)((splits + need_extra) * M * N) > work_elems) --splits;
  int64_t kchunk = (K + splits - 1) / splits;
  kchunk = ((kchunk + BK - 1) / BK) * BK;
  if (kchunk < BK) kchunk = BK;
  splits = (K + kchunk - 1) / kchunk;
  if (splits < 1) splits = 1;
  const bool direct = splits == 1 && out.C != nullptr;
  double* dst = direct ? out.C : work;
  const int64_t ldo = direct ? out.ldc : N;
  dim3 grid((unsigned)((N + BN - 1) / BN), (unsigned)((M + BM - 1) / BM), (unsigned)splits);
  if (K <= 0) {
    // empty contraction: C = 0
    cudaMemsetAsync(work, 0, sizeof(double) * M * N, st);
    splits = 1;
    dst = work;
  } else if (transA) {
    gemm_kernel<TA, TB, true><<<grid, 256, 0, st>>>(A, lda, B, ldb, M, N, K, kchunk, dst, ldo,
                                                    M * N);
    count_launch();
  } else {
    gemm_kernel<TA, TB, false><<<grid, 256, 0, st>>>(A, lda, B, ldb, M, N, K, kchunk, dst, ldo,
                                                     M * N);
    count_launch();
  }
  if (direct && K > 0) return;
  double* res = work;
  if (splits > 1) {
    res = out.Cf ? work + splits * M * N : nullptr;
    if (out.C && !out.Cf && out.ldc == N) {
      reduce_parts(work, (int)splits, M * N, out.C, st);
      return;
    }
    if (!res) res = work + splits * M * N;
    reduce_parts(work, (int)splits, M * N, res, st);
  }
  if (out.Cf) {
    f64_to_f32(res, M, N, out.colscale, out.Cf, out.ldcf, st);
  } else if (out.C) {
    cudaMemcpy2DAsync(out.C, sizeof(double) * out.ldc, res, sizeof(double) * N,
                      sizeof(double) * N, M, cudaMemcpyDeviceToDevice, st);
  }
}

template void gemm<float, float>(bool, const float*, int64_t, const float*, int64_t, int64_t,
                                 int64_t, int64_t, GemmOut, double*, size_t, cudaStream_t);
template void gemm<float, double>(bool, const float*, int64_t, const double*, int64_t, int64_t,
                                  int64_t, int64_t, GemmOut, double*, size_t, cudaStream_t);
template void gemm<double, double>(bool, const double*, int64_t, const double*, int64_t,
                                   int64_t, int64_t, int64_t, GemmOut, double*, size_t,
                                   cudaStream_t);
template void gemm<double, float>(bool, const double*, int64_t, const float*, int64_t, int64_t,
                                  int64_t, int64_t, GemmOut, double*, size_t, cudaStream_t);

void reduce_parts(const double* parts, int nparts, int64_t len, double* out, cudaStream_t st) {
  if (len <= 0) return;
  if (len <= 64 && nparts > 64)
    reduce_parts_short_kernel<<<(unsigned)len, 256, 0, st>>>(parts, nparts, len, out);
  else if (len < (int64_t)kSMs * 256)   // e.g. the Gram partials (16384 x 296): 64-thread
    reduce_parts_kernel<<<grid_for(len, 64), 64, 0, st>>>(parts, nparts, len, out);   // blocks
  else if (len % 2 == 0 && ((reinterpret_cast<uintptr_t>(parts) | reinterpret_cast<uintptr_t>(out)) & 15) == 0)
    reduce_parts_vec_kernel<<<2 * kSMs, 256, 0, st>>>(reinterpret_cast<const double2*>(parts), nparts,
                                                       len / 2, reinterpret_cast<double2*>(out));
  else
    reduce_parts_kernel<<<grid_for(len), 256, 0, st>>>(parts, nparts, len, out);
  count_launch();
}

void f64_to_f32(const double* A, int64_t rows, int64_t cols, const double* colscale, float* B,
                int64_t ldb, cudaStream_t st) {
  f64_to_f32_kernel<<<grid_for(rows * cols), 256, 0, st>>>(A, rows, cols, colscale, B, ldb);
  count_launch();
}

void f32_to_f64(const float* A, int64_t lda, int64_t rows, int64_t cols, double* B,
                cudaStream_t st) {
  f32_to_f64_kernel<<<grid_for(rows * cols), 256, 0, st>>>(A, lda, rows, cols, B);
  count_launch();
}

}  // namespace enmf
