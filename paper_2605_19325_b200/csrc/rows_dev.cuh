// rows_dev.cuh -- device helpers of the row-block kernels (kernels_rows.cu, small_sweep.cu):
// warp reductions, the row-times-Gram product with the rows lane-distributed, the Gram load.
// Lane L owns columns L, L+32, ... (CPL = ceil(r/32) of them); the r x r Gram sits in shared
// memory in fp64, zero-padded to 32*CPL (rows of U and V update independently).
#pragma once
#include <cuda_runtime.h>

namespace enmf {
namespace rows_dev {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, o));
  return v;
}

// out[b][c] += sign * sum_l S[b][l] G[l][lane + 32c]   (S held lane-distributed like out).
// S is staged through the warp's shared buffer Ss (RB x 32*CPL doubles) and read back as
// broadcast 16-byte loads, two l at a time: no shuffles, so the fp64 FMA pipe is the bound.
template <int CPL, int RB>
__device__ __forceinline__ void row_times_gram(const double (&S)[RB][CPL], const double* Gs,
                                               double* Ss, int r, int lane, double sign,
                                               double (&out)[RB][CPL]) {
  constexpr int RP = 32 * CPL;
  __syncwarp();
#pragma unroll
  for (int b = 0; b < RB; ++b)
#pragma unroll
    for (int c = 0; c < CPL; ++c) Ss[b * RP + lane + 32 * c] = sign * S[b][c];
  __syncwarp();
  const int rr = (r + 1) & ~1;                // entries >= r are zero in S and in G
#pragma unroll 2
  for (int l = 0; l < rr; l += 2) {
    double g0[CPL], g1[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      g0[c] = Gs[l * RP + lane + 32 * c];
      g1[c] = Gs[(l + 1) * RP + lane + 32 * c];
    }
#pragma unroll
    for (int b = 0; b < RB; ++b) {
      const double2 sv = *reinterpret_cast<const double2*>(Ss + b * RP + l);
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        out[b][c] = fma(sv.x, g0[c], out[b][c]);
        out[b][c] = fma(sv.y, g1[c], out[b][c]);
      }
    }
  }
}

template <int CPL>
__device__ __forceinline__ void load_gram(const double* G, int r, double* Gs) {
  constexpr int RP = 32 * CPL;
#pragma unroll 8                              // eight loads in flight per thread
  for (int e = threadIdx.x; e < RP * RP; e += blockDim.x) {
    const int l = e / RP, j = e % RP;
    Gs[e] = (l < r && j < r) ? G[l * r + j] : 0.0;
  }
}

}  // namespace rows_dev
}  // namespace enmf
