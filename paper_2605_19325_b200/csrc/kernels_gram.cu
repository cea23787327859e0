// kernels_gram.cu -- the r x r Gram matrices G = F^T F of the fp32 factors (SURVEY §8(a) rows
// a5/a6: G_U for the V-block update, G_V for the U-block update, both for the trace-form
// objective).  The objective's third term <G_U, G_V> is ~||X||^2 while f can be ~3e-8 of it, so
// the Grams stay fp64-exact products of the fp32 entries (no digit split here).
//
// With qscale (the tensor-core path's digit scales of the factor, tc_factor_scales) the Gram
// is that of the quantised factor the X pass multiplied, so that the trace-form objective is
// ||X~ - U~ V^T||^2 of the same operands (tc_gemm.cu).
//
// Only the upper triangle is computed: the 128 x 128 output is a 16 x 16 grid of 8 x 8 tiles,
// and the 136 tiles with ti <= tj go to 136 threads (64 fp64 accumulators each).  Rows are
// split across a persistent grid (two CTAs per SM); a CTA stages 32 rows at a time in shared
// memory as fp64 and every thread runs 64 FMAs per row from 16 shared loads.  Per-CTA partials
// are summed in a fixed order (reduce_parts) and mirrored: deterministic.
#include <algorithm>

#include "internal.h"

namespace enmf {
namespace {

constexpr int kGramThreads = 160;            // 136 tile threads (5 warps)
constexpr int kGramRows = 32;                // rows staged per step
constexpr int kGramLd = 128 + 2;             // padded fp64 row stride

__global__ void __launch_bounds__(kGramThreads, 2)
gram_upper_kernel(const float* __restrict__ A, int64_t lda, int64_t rows, int r,
                  const double* __restrict__ qscale, double* __restrict__ parts) {
  __shared__ __align__(16) double S[kGramRows * kGramLd];
  const int tid = threadIdx.x;
  // tile t -> (ti, tj), ti <= tj, row-major over the upper triangle
  int ti = 0, tj = 0;
  {
    int t = tid, row = 0;
    while (row < 16 && t >= 16 - row) {
      t -= 16 - row;
      ++row;
    }
    ti = row;
    tj = row + t;
  }
  const bool tile_on = tid < 136;
  double acc[8][8];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b) acc[a][b] = 0.0;
  const int64_t per = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * per;
  const int64_t r1 = r0 + per < rows ? r0 + per : rows;
  for (int64_t base = r0; base < r1; base += kGramRows) {
    __syncthreads();
    for (int e = tid; e < kGramRows * 128; e += blockDim.x) {
      const int i = e >> 7, c = e & 127;
      const int64_t row = base + i;
      double v = (row < r1 && c < r) ? (double)A[row * lda + c] : 0.0;
      if (qscale && c < r) {
        // the value the tensor-core X pass multiplies: rint(v s 2^15) / (s 2^15), s = 2^k
        const double s = qscale[c] * 32768.0;
        v = rint(v * s) / s;
      }
      S[i * kGramLd + c] = v;
    }
    __syncthreads();
    if (tile_on) {
#pragma unroll 2
      for (int i = 0; i < kGramRows; ++i) {
        const double* srow = S + i * kGramLd;
        double x[8], y[8];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const double2 p = *reinterpret_cast<const double2*>(srow + 8 * ti + 2 * a);
          const double2 q = *reinterpret_cast<const double2*>(srow + 8 * tj + 2 * a);
          x[2 * a] = p.x;
          x[2 * a + 1] = p.y;
          y[2 * a] = q.x;
          y[2 * a + 1] = q.y;
        }
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
          for (int b = 0; b < 8; ++b) acc[a][b] = fma(x[a], y[b], acc[a][b]);
      }
    }
  }
  if (tile_on) {
    double* out = parts + (int64_t)blockIdx.x * 128 * 128;
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = 0; b < 8; ++b) out[(8 * ti + a) * 128 + 8 * tj + b] = acc[a][b];
  }
}

// G (r x r, ld r) from the reduced 128 x 128 upper tiles: G[i][j] = Gu[min][max]
__global__ void gram_mirror_kernel(const double* __restrict__ Gu, int r, double* __restrict__ G) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < r * r; e += gridDim.x * blockDim.x) {
    const int i = e / r, j = e % r;
    const int lo = i < j ? i : j, hi = i < j ? j : i;
    // within a diagonal tile both triangles were computed; take the upper one for symmetry
    G[e] = Gu[lo * 128 + hi];
  }
}

}  // namespace

constexpr int kGramGrid = 2 * kSMs;          // two CTAs (10 warps) per SM

int gram_parts() { return kGramGrid; }

bool gram_supported(int r) { return r >= 1 && r <= 128; }

void gram_sym(const float* A, int64_t lda, int64_t rows, int r, double* parts, double* Gu,
              double* G, cudaStream_t st, const double* qscale) {
  // every CTA writes a 128 x 128 partial (131 KB) that the reduction reads back: with few rows
  // (a rank's U block at 8 GPUs, the V block) 296 partials cost more than the Gram itself,
  // so the grid shrinks to one CTA per 128 rows (deterministic for a given row count)
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(kGramGrid, (rows + 127) / 128));
  gram_upper_kernel<<<grid, kGramThreads, 0, st>>>(A, lda, rows, r, qscale, parts);
  reduce_parts(parts, grid, 128 * 128, Gu, st);
  gram_mirror_kernel<<<(r * r + 255) / 256, 256, 0, st>>>(Gu, r, G);
  count_launch(2);
}

}  // namespace enmf
