// tc_gemm.cu -- tcgen05 tensor-core path for the two X passes of a sweep (see tc.h).
//
// Per-iteration cost of eNMF is dominated by X V and X^T U.  At r = 128
// these are compute-bound on SIMT units (64 flop per X byte), so they run on the 5th-gen
// tensor cores:
//
//   * X is repacked ONCE (enmf_set_data) into two fp16 planes, X*sX = Xhi + Xlo (sX a power
//     of two), 4 bytes per element -- the same HBM bytes per pass as fp32 X.  Tiles of
//     128 rows x 64 columns are stored in the UMMA no-swizzle canonical layout with the
//     8x8 core matrix (g, kc) at byte (kc*16 + g)*128, so that ONE packed copy is
//       - a K-major A operand for P = X V   (SBO 128 B between 8-row groups, LBO 2048 B), and
//       - an MN-major A operand for Q = X^T U (two column-adjacent tiles form 128 contiguous
//         MN groups at a uniform 2048 B stride).
//   * The factor (V for pass 1, U for pass 2) is packed per pass into the same form (B operand,
//     K-major), with a power-of-two scale per column.
//   * Per 64-deep K stage the MMA warp issues 4 k-steps x 3 products
//       Xhi*Fhi + Xhi*Flo + Xlo*Fhi   (tcgen05.mma kind::f16, M=128, N=r padded to 16)
//     into one fp32 TMEM accumulator; every PROMOTE stages (K = 512) the accumulator is drained
//     by 8 epilogue warps into fp64 registers (double-buffered TMEM, 2 x 128 columns), which
//     bounds the fp32 accumulation error.
//   * Warp roles: warp 0 = producer (cp.async.bulk into a 3-stage smem ring, mbarrier
//     complete_tx), warp 1 = TMEM allocator + single-thread MMA issuer, warps 2..9 = epilogue.
//     Persistent grid: one CTA per SM walks the work units.
#include <cuda_fp16.h>
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>

#include "internal.h"
#include "tc.h"

namespace enmf {
namespace tcg {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int STAGES = 3;
constexpr int PROMOTE = 8;
constexpr int EPI_WARPS = 8;
constexpr int THREADS = 32 * (2 + EPI_WARPS);
constexpr int TILE_A = BM * BK * 2;              // bytes per X tile per plane (16 KB)
constexpr int MAX_TILE_B = 128 * BK * 2;         // bytes per factor tile per plane (<= 16 KB)
constexpr int STAGE_BYTES = 2 * TILE_A + 2 * MAX_TILE_B;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024;
constexpr int TMEM_COLS = 256;

struct Params {
  const uint8_t* xhi;
  const uint8_t* xlo;
  const uint8_t* fhi;
  const uint8_t* flo;
  double* out;
  int64_t out_ld;
  int64_t split_stride;
  const double* colscale;    // r values: 1 / (sX * sF_k)
  int mode;                  // 0: P = X V ; 1: Q = X^T U
  int num_units;
  int ksplit;
  int stages_total;          // 64-deep K stages of the full contraction
  int64_t tiles_per_row;     // packed X: 64-column tiles per 128-row band
  int rp;                    // padded N (multiple of 16, <= 128)
  int r;                     // valid output columns
  int64_t out_rows;          // valid output rows
  int promote;               // 64-deep stages per fp32 TMEM accumulation chunk
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  long long t0 = 0;
  int spins = 0;
  while (true) {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) return;
    if (++spins == 1024) t0 = clock64();
    if (spins > 1024 && (spins & 1023) == 0 && clock64() - t0 > 40000000000LL) {
      printf("enmf tc: mbarrier wait timeout (block %d thread %d)\n", blockIdx.x, threadIdx.x);
      __trap();
    }
  }
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(dst), "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::
                   "r"(bar)
               : "memory");
}
__device__ __forceinline__ void tc_mma_f16(uint32_t dtmem, uint64_t adesc, uint64_t bdesc,
                                           uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// UMMA shared-memory descriptor, no swizzle (layout type 0), Blackwell version 1.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

#define TMEM_LD32(taddr, v)                                                                    \
  asm volatile(                                                                                \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13," \
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"       \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),   \
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),            \
        "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),         \
        "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),         \
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),         \
        "=r"(v[31])                                                                            \
      : "r"(taddr))

__device__ __forceinline__ void unit_range(const Params& p, int u, int& tile, int& s0, int& s1,
                                           int& split) {
  if (p.mode == 0) {
    tile = u;
    split = 0;
    s0 = 0;
    s1 = p.stages_total;
  } else {
    tile = u / p.ksplit;
    split = u % p.ksplit;
    const int per = (p.stages_total + p.ksplit - 1) / p.ksplit;
    s0 = split * per;
    s1 = min(p.stages_total, s0 + per);
    if (s1 < s0) s1 = s0;
  }
}

__global__ void __launch_bounds__(THREADS, 1) tc_gemm_kernel(const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bars[2 * STAGES + 4];
  __shared__ uint32_t tmem_base_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bar_full = smem_u32(&bars[0]);
  const uint32_t bar_empty = smem_u32(&bars[STAGES]);
  const uint32_t bar_tfull = smem_u32(&bars[2 * STAGES]);
  const uint32_t bar_tempty = smem_u32(&bars[2 * STAGES + 2]);
  const uint32_t tile_b = (uint32_t)p.rp * BK * 2;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(bar_full + 8 * s, 1);
      mbar_init(bar_empty + 8 * s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(bar_tfull + 8 * b, 1);
      mbar_init(bar_tempty + 8 * b, EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_s)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_s;

  if (warp == 0) {
    // ===================== producer: bulk copies into the smem ring =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < p.num_units; u += gridDim.x) {
        int tile, s0, s1, split;
        unit_range(p, u, tile, s0, s1, split);
        for (int ks = s0; ks < s1; ++ks) {
          mbar_wait(bar_empty + 8 * stage, phase ^ 1);
          const uint32_t fb = bar_full + 8 * stage;
          mbar_expect_tx(fb, 2 * TILE_A + 2 * tile_b);
          uint8_t* st = smem + (size_t)stage * STAGE_BYTES;
          const uint32_t a_hi = smem_u32(st), a_lo = a_hi + TILE_A;
          const uint32_t b_hi = a_hi + 2 * TILE_A, b_lo = b_hi + tile_b;
          if (p.mode == 0) {
            const int64_t off = ((int64_t)tile * p.tiles_per_row + ks) * TILE_A;
            bulk_g2s(a_hi, p.xhi + off, TILE_A, fb);
            bulk_g2s(a_lo, p.xlo + off, TILE_A, fb);
          } else {
            // A = X^T: 128 output rows (j) = column tiles 2*tile, 2*tile+1 of row band
            // ks/2; the K stage is the 64-row half (ks & 1) of that band.
            const int64_t band = ks >> 1;
            const int half = ks & 1;
            for (int t = 0; t < 2; ++t) {
              const int64_t base = (band * p.tiles_per_row + 2 * tile + t) * TILE_A;
              for (int kc = 0; kc < 8; ++kc) {
                const int64_t src = base + (int64_t)(kc * 16 + 8 * half) * 128;
                const uint32_t dst = (uint32_t)((t * 8 + kc) * 1024);
                bulk_g2s(a_hi + dst, p.xhi + src, 1024, fb);
                bulk_g2s(a_lo + dst, p.xlo + src, 1024, fb);
              }
            }
          }
          const int64_t foff = (int64_t)ks * tile_b;
          bulk_g2s(b_hi, p.fhi + foff, tile_b, fb);
          bulk_g2s(b_lo, p.flo + foff, tile_b, fb);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (one thread) =====================
    if (lane == 0) {
      // instruction descriptor: F32 accumulate, F16 x F16, A K-major (mode 0) or MN-major
      // (mode 1), B K-major, N = rp, M = 128
      const uint32_t idesc = (1u << 4) | ((uint32_t)p.mode << 15) |
                             ((uint32_t)(p.rp >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
      const uint32_t a_lbo = p.mode == 0 ? 2048u : 128u;
      const uint32_t a_sbo = p.mode == 0 ? 128u : 1024u;
      const uint32_t a_kstep = p.mode == 0 ? 4096u : 256u;
      const uint32_t b_lbo = (uint32_t)p.rp * 16u, b_sbo = 128u;
      const uint32_t b_kstep = (uint32_t)p.rp * 32u;
      int stage = 0;
      uint32_t phase = 0;
      uint32_t chunk = 0;
      for (int u = blockIdx.x; u < p.num_units; u += gridDim.x) {
        int tile, s0, s1, split;
        unit_range(p, u, tile, s0, s1, split);
        uint32_t buf = 0;
        for (int ks = s0; ks < s1; ++ks) {
          const int t = ks - s0;
          const bool first = (t % p.promote) == 0;
          if (first) {
            buf = chunk & 1;
            mbar_wait(bar_tempty + 8 * buf, ((chunk >> 1) & 1) ^ 1);
            tc_fence_after();
          }
          mbar_wait(bar_full + 8 * stage, phase);
          tc_fence_after();
          const uint32_t a_hi = smem_u32(smem + (size_t)stage * STAGE_BYTES);
          const uint32_t a_lo = a_hi + TILE_A;
          const uint32_t b_hi = a_hi + 2 * TILE_A, b_lo = b_hi + tile_b;
          const uint32_t dt = tmem_base + buf * 128;
#pragma unroll
          for (int j = 0; j < BK / 16; ++j) {
            const uint64_t ah = umma_desc(a_hi + j * a_kstep, a_lbo, a_sbo);
            const uint64_t al = umma_desc(a_lo + j * a_kstep, a_lbo, a_sbo);
            const uint64_t bh = umma_desc(b_hi + j * b_kstep, b_lbo, b_sbo);
            const uint64_t bl = umma_desc(b_lo + j * b_kstep, b_lbo, b_sbo);
            tc_mma_f16(dt, ah, bh, idesc, (first && j == 0) ? 0u : 1u);
            tc_mma_f16(dt, ah, bl, idesc, 1u);
            tc_mma_f16(dt, al, bh, idesc, 1u);
          }
          tc_commit(bar_empty + 8 * stage);          // frees the smem slot when MMAs retire
          if ((t % p.promote) == p.promote - 1 || ks == s1 - 1) {
            tc_commit(bar_tfull + 8 * buf);          // accumulator chunk ready
            ++chunk;
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else {
    // ===================== epilogue: TMEM fp32 chunks -> fp64 registers =====================
    const int e = warp - 2;
    const int q = warp & 3;                 // TMEM lane quadrant of this warp
    const int hcol = e >> 2;                // columns [64*hcol, 64*hcol + 64)
    const int row_in_tile = 32 * q + lane;
    uint32_t chunk = 0;
    for (int u = blockIdx.x; u < p.num_units; u += gridDim.x) {
      int tile, s0, s1, split;
      unit_range(p, u, tile, s0, s1, split);
      if (s1 <= s0) continue;
      double acc[64];
#pragma unroll
      for (int c = 0; c < 64; ++c) acc[c] = 0.0;
      const int nchunks = (s1 - s0 + p.promote - 1) / p.promote;
      for (int c = 0; c < nchunks; ++c) {
        const uint32_t buf = chunk & 1;
        mbar_wait(bar_tfull + 8 * buf, (chunk >> 1) & 1);
        tc_fence_after();
        const uint32_t taddr = tmem_base + ((uint32_t)(32 * q) << 16) + buf * 128 + 64 * hcol;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t v[32];
          TMEM_LD32(taddr + 32 * h, v);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int i = 0; i < 32; ++i) acc[32 * h + i] += (double)__uint_as_float(v[i]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_tempty + 8 * buf);
        ++chunk;
      }
      const int64_t row = (int64_t)tile * BM + row_in_tile;
      if (row < p.out_rows) {
        double* o = p.out + (int64_t)split * p.split_stride + row * p.out_ld;
#pragma unroll
        for (int c = 0; c < 64; ++c) {
          const int col = 64 * hcol + c;
          if (col < p.r) o[col] = acc[c] * p.colscale[col];
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(TMEM_COLS));
  }
}

// ------------------------------------------------------------------ packing
__device__ __forceinline__ void split16(float v, __half& hi, __half& lo) {
  hi = __float2half_rn(v);
  lo = __float2half_rn(v - __half2float(hi));
}

// X (rows x n, ld) * sx -> hi/lo planes of [Mt][tiles_per_row] tiles.  One thread writes one
// 16-byte row chunk (8 consecutive columns) of each plane; consecutive threads read
// consecutive chunks of an X row (coalesced reads).
__global__ void pack_x_kernel(const float* __restrict__ X, int64_t ldx, int64_t rows, int64_t n,
                              float sx, int64_t tiles_per_row, int64_t Mt, uint4* hi, uint4* lo) {
  const int64_t cpr = tiles_per_row * 8;                 // 16-byte chunks per padded row
  const int64_t total = Mt * BM * cpr;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < total;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = c / cpr, jc = c - i * cpr;
    const int64_t j0 = jc * 8;
    __align__(16) __half h[8], l[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int64_t j = j0 + k;
      const float v = (i < rows && j < n) ? X[i * ldx + j] * sx : 0.0f;
      split16(v, h[k], l[k]);
    }
    const int64_t mt = i / BM, g = (i % BM) / 8, ri = i % 8;
    const int64_t kt = j0 / BK, kc = (j0 % BK) / 8;
    const int64_t byte = (mt * tiles_per_row + kt) * TILE_A + (kc * 16 + g) * 128 + ri * 16;
    hi[byte / 16] = *reinterpret_cast<uint4*>(h);
    lo[byte / 16] = *reinterpret_cast<uint4*>(l);
  }
}

// Factor F (K x r, ld) * colscale -> B tiles [Kt][rp x 64]: chunk (kc*(rp/8) + g)*128 + ri*16
// holds F[kt*64 + kc*8 + 0..7][g*8 + ri].
__global__ void pack_factor_kernel(const float* __restrict__ F, int64_t ldf, int64_t K, int r,
                                   int rp, const float* __restrict__ fscale, int64_t Kt,
                                   uint4* hi, uint4* lo) {
  const int64_t chunks_per_tile = (int64_t)rp * BK / 8;
  const int64_t total = Kt * chunks_per_tile;
  const int gpt = rp / 8;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < total;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t kt = c / chunks_per_tile;
    const int64_t w = c - kt * chunks_per_tile;            // 16-byte chunk index in the tile
    const int kc = (int)(w / (gpt * 8));
    const int rem = (int)(w % (gpt * 8));
    const int g = rem / 8, ri = rem % 8;
    const int col = g * 8 + ri;
    const float s = col < r ? fscale[col] : 0.0f;
    __align__(16) __half h[8], l[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int64_t kk = kt * BK + kc * 8 + k;
      const float v = (col < r && kk < K) ? F[kk * ldf + col] * s : 0.0f;
      split16(v, h[k], l[k]);
    }
    hi[c] = *reinterpret_cast<uint4*>(h);
    lo[c] = *reinterpret_cast<uint4*>(l);
  }
}

// Per-column max |F| (F rows x r) into maxbits[r] (float bits; max is order independent).
__global__ void colmax_kernel(const float* __restrict__ F, int64_t ldf, int64_t rows, int r,
                              unsigned* maxbits) {
  __shared__ float m[128];
  for (int k = threadIdx.x; k < r; k += blockDim.x) m[k] = 0.0f;
  __syncthreads();
  const int64_t total = rows * (int64_t)r;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / r;
    const int k = (int)(e - i * r);
    const float a = fabsf(F[i * ldf + k]);
    atomicMax(reinterpret_cast<unsigned*>(&m[k]), __float_as_uint(a));
  }
  __syncthreads();
  for (int k = threadIdx.x; k < r; k += blockDim.x) atomicMax(&maxbits[k], __float_as_uint(m[k]));
}

// fscale[k] = 2^(14 - floor(log2 max|F_k|)) ; colscale[k] = 1 / (sx * fscale[k])  (exact).
__global__ void scales_kernel(const unsigned* maxbits, int r, double sx, float* fscale,
                              double* colscale) {
  for (int k = threadIdx.x; k < r; k += blockDim.x) {
    const float mx = __uint_as_float(maxbits[k]);
    int e = 0;
    if (mx > 0.0f) {
      frexpf(mx, &e);                   // mx in [2^(e-1), 2^e)
      e = 14 - (e - 1);
    }
    const float s = ldexpf(1.0f, e);
    fscale[k] = s;
    colscale[k] = 1.0 / (sx * (double)s);
  }
}

__global__ void maxabs_x_kernel(const float* __restrict__ X, int64_t ldx, int64_t rows, int64_t n,
                                unsigned* maxbits) {
  unsigned m = 0;
  const int64_t total = rows * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e - i * n;
    m = max(m, __float_as_uint(fabsf(X[i * ldx + j])));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(maxbits, m);
}

}  // namespace tcg

using namespace tcg;

struct TcState {
  int64_t rows = 0, n = 0, r = 0;
  int rp = 0;
  int64_t Mt = 0;              // 128-row bands of X
  int64_t tiles_per_row = 0;   // 64-column tiles per band (even: 128-column pairs)
  int64_t Kt2 = 0;             // 64-row K stages of pass 2 (= 2 Mt)
  double sx = 1.0;
  uint8_t* xhi = nullptr;
  uint8_t* xlo = nullptr;
  uint8_t* fhi = nullptr;
  uint8_t* flo = nullptr;
  unsigned* maxbits = nullptr; // r + 1
  float* fscale = nullptr;     // r
  double* colscale = nullptr;  // r
  double* partial = nullptr;   // ksplit x (tiles_per_row/2 * 128) x r
  int ksplit = 1;
  int sms = kSMs;
  int promote = PROMOTE;
};

bool tc_supported(int64_t rows, int64_t n, int64_t r) {
  return r >= 1 && r <= 128 && rows >= 1 && n >= 1;
}

void tc_destroy(TcState* s) {
  if (!s) return;
  void* bufs[] = {s->xhi, s->xlo, s->fhi, s->flo, s->maxbits, s->fscale, s->colscale, s->partial};
  for (void* b : bufs)
    if (b) cudaFree(b);
  delete s;
}

int tc_create(TcState** out, const float* X, int64_t ldx, int64_t rows, int64_t n, int64_t r,
              cudaStream_t st) {
  *out = nullptr;
  TcState* s = new TcState();
  s->rows = rows;
  s->n = n;
  s->r = r;
  s->rp = (int)((r + 15) / 16 * 16);
  s->Mt = (rows + BM - 1) / BM;
  s->tiles_per_row = ((n + 127) / 128) * 2;
  s->Kt2 = 2 * s->Mt;
  if (const char* e = getenv("ENMF_TC_PROMOTE")) s->promote = std::max(1, atoi(e));
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&s->sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t plane = (size_t)s->Mt * s->tiles_per_row * TILE_A;
  const int64_t fK = std::max<int64_t>(s->tiles_per_row, s->Kt2);
  const size_t fplane = (size_t)fK * s->rp * BK * 2;
  const int64_t n_pad = s->tiles_per_row / 2 * 128;
  const int64_t units2 = s->tiles_per_row / 2;
  int ks = (int)((4 * s->sms + units2 - 1) / units2);
  ks = std::max(1, std::min<int>(ks, (int)s->Kt2));
  const int per = (int)((s->Kt2 + ks - 1) / ks);
  ks = (int)((s->Kt2 + per - 1) / per);          // no empty split ranges
  s->ksplit = ks;
  cudaError_t e = cudaSuccess;
  if (!e) e = cudaMalloc(&s->xhi, plane);
  if (!e) e = cudaMalloc(&s->xlo, plane);
  if (!e) e = cudaMalloc(&s->fhi, fplane);
  if (!e) e = cudaMalloc(&s->flo, fplane);
  if (!e) e = cudaMalloc(&s->maxbits, sizeof(unsigned) * (r + 1));
  if (!e) e = cudaMalloc(&s->fscale, sizeof(float) * r);
  if (!e) e = cudaMalloc(&s->colscale, sizeof(double) * r);
  if (!e) e = cudaMalloc(&s->partial, sizeof(double) * (size_t)ks * n_pad * r);
  if (e) {
    cudaGetLastError();
    tc_destroy(s);
    return e == cudaErrorMemoryAllocation ? 2 : 1;
  }
  // global power-of-two scale of X: max|X| * sx in [2^14, 2^15)
  cudaMemsetAsync(s->maxbits, 0, sizeof(unsigned), st);
  maxabs_x_kernel<<<4 * s->sms, 256, 0, st>>>(X, ldx, rows, n, s->maxbits);
  unsigned mb = 0;
  cudaMemcpyAsync(&mb, s->maxbits, sizeof(unsigned), cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) {
    tc_destroy(s);
    return 1;
  }
  float mx;
  memcpy(&mx, &mb, sizeof(mx));
  int ex = 0;
  if (mx > 0.0f) {
    frexpf(mx, &ex);
    ex = 14 - (ex - 1);
  }
  s->sx = ldexp(1.0, ex);
  pack_x_kernel<<<8 * s->sms, 256, 0, st>>>(X, ldx, rows, n, (float)s->sx, s->tiles_per_row, s->Mt,
                                            (uint4*)s->xhi, (uint4*)s->xlo);
  count_launch(2);
  if (cudaGetLastError() != cudaSuccess) {
    tc_destroy(s);
    return 1;
  }
  *out = s;
  return 0;
}

static void pack_factor(TcState* s, const float* F, int64_t ldf, int64_t K, int64_t Kt,
                        cudaStream_t st) {
  const int r = (int)s->r;
  cudaMemsetAsync(s->maxbits, 0, sizeof(unsigned) * r, st);
  colmax_kernel<<<2 * s->sms, 256, 0, st>>>(F, ldf, K, r, s->maxbits);
  scales_kernel<<<1, 128, 0, st>>>(s->maxbits, r, s->sx, s->fscale, s->colscale);
  pack_factor_kernel<<<4 * s->sms, 256, 0, st>>>(F, ldf, K, r, s->rp, s->fscale, Kt,
                                                 (uint4*)s->fhi, (uint4*)s->flo);
  count_launch(3);
}

static int launch_gemm(TcState* s, int mode, double* out, int64_t out_ld, int64_t split_stride,
                       int num_units, int ksplit, int stages_total, int64_t out_rows,
                       cudaStream_t st) {
  Params p;
  p.xhi = s->xhi;
  p.xlo = s->xlo;
  p.fhi = s->fhi;
  p.flo = s->flo;
  p.out = out;
  p.out_ld = out_ld;
  p.split_stride = split_stride;
  p.colscale = s->colscale;
  p.mode = mode;
  p.num_units = num_units;
  p.ksplit = ksplit;
  p.stages_total = stages_total;
  p.tiles_per_row = s->tiles_per_row;
  p.rp = s->rp;
  p.r = (int)s->r;
  p.out_rows = out_rows;
  p.promote = s->promote;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tc_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    attr = true;
  }
  const int grid = std::min(num_units, s->sms);
  tc_gemm_kernel<<<grid, THREADS, SMEM_BYTES, st>>>(p);
  count_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int tc_xv(TcState* s, const float* V, int64_t ldv, double* P, cudaStream_t st) {
  // B = V (K = n), packed over all 64-column stages of X
  pack_factor(s, V, ldv, s->n, s->tiles_per_row, st);
  return launch_gemm(s, 0, P, s->r, 0, (int)s->Mt, 1, (int)s->tiles_per_row, s->rows, st);
}

int tc_xtu(TcState* s, const float* U, int64_t ldu, double* Q, cudaStream_t st) {
  // B = U (K = rows of X), split-K partials reduced in a fixed order
  pack_factor(s, U, ldu, s->rows, s->Kt2, st);
  const int units = (int)(s->tiles_per_row / 2) * s->ksplit;
  if (launch_gemm(s, 1, s->partial, s->r, s->n * s->r, units, s->ksplit, (int)s->Kt2, s->n, st))
    return 1;
  reduce_parts(s->partial, s->ksplit, s->n * s->r, Q, st);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace enmf
