// tc_gemm.cu -- tcgen05 tensor-core path for the two X passes of a sweep (see tc.h).
//
// Per-iteration cost of eNMF is dominated by X V and X^T U.  At r = 128
// each X pass carries 64 flop per fp32 byte, far beyond SIMT reach, so the passes run on the
// 5th-gen tensor cores.  The accumulation must be EXACT: measured on B200, kind::f16 MMAs with
// fp32 TMEM accumulation lose ~3e-7 relative per 64-deep K stage (not round-to-nearest fp32),
// which the HALS update amplifies ~r-fold past BASELINE's 1e-5.  This path uses
// integer MMAs instead:
//
//   * Operands become three int8 digits in mixed radix (8, 8, 7), t = a s = d0 + d1/2^8 +
//     d2/2^15 (t rounded to the 2^-15 grid, |d0| <= 126, d1 in [-128, 127], d2 symmetric in
//     [-64, 64]: tc_ptx.cuh digits3_n) with s a power of two, max|a| s in [63, 126): one scale
//     per ROW of X for P = X V (the output row), one per COLUMN of X for Q = X^T U (the output
//     row of the transposed product), one per column of the factor.  22 bits relative to the
//     scale group's maximum.  X is repacked ONCE (enmf_set_data) into 3 byte planes per copy --
//     3 bytes per element, 3/4 of the fp32 X bytes; the factor is repacked per pass.
//   * tcgen05.mma kind::i8 (M = 128, N = r rounded to 16, K = 32) accumulates exactly in int32
//     TMEM.  The six products of weight >= 2^-16 are issued as 4 MMAs per 32-deep k-step into
//     4 accumulators (4 x 128 TMEM columns), one per weight:
//         acc0 = A0 B0 (1), acc1 = A0 B1 + A1 B0 (2^-8), acc2 = A1 B1 (2^-16),
//         acc3 = A0 B2 + A2 B0 (2^-15)
//     (B planes 0 and 1 are adjacent, so A0 [B0;B1] and A1 [B0;B1] are N = 2r MMAs writing
//     adjacent accumulators; A1 [B0;B1] accumulates into acc1 and acc2 together, so the
//     epilogue zeroes acc2 for the next unit; |acc| <= 2 * 126 * 128 * K < 2^31 for unit
//     K <= 65536).  The epilogue forms acc0 + 2^-8 (acc1 + 2^-8 (acc2 + 2 acc3)) EXACTLY in
//     fp64 (49 bits) and applies 1/(s_row s_col), a power of two.  The dropped products
//     (weight 2^-23 and below) each contain a symmetric last digit: unbiased, ~2^-23 of |X||F|
//     per term.  Measured in tools/digit_sim.py at a C5-recipe shape: Q ~6e-9 relative, one
//     HALS V block ~4e-7 from the fp64 update; the trace-form objective is formed from the
//     SAME quantised operands (||X~||^2 of the pass-2 copy, the Gram of the quantised U:
//     tc_xq_norm2, tc_factor_scales) so it equals ||X~ - U~ V^T||^2 up to the dropped
//     products' noise, and its error does not scale with ||X||^2 / f.
//   * Layout: tiles of 128 rows x 64 columns per plane in the UMMA no-swizzle canonical layout,
//     core matrix (g, kc) at byte (kc*16 + g)*128 (8 rows x 16 bytes): a K-major A operand for
//     P = X V (SBO 128 B, LBO 2048 B).  Q = X^T U reads a second packed copy of X^T in the same
//     K-major layout (mode 2); without it (ENMF_TC_XT=0 or not enough memory) the X copy is
//     gathered as an MN-major A operand (mode 1: two column-adjacent tiles give 8 MN groups at a
//     uniform 2048 B stride, 1 KB bulk copies into SBO 1024 B / LBO 128 B), ~40 % slower; the
//     X copy then uses one scale for all rows (a per-row scale would vary along K).
//   * Warp roles: warp 0 = producer (cp.async.bulk into a 4-stage ring, mbarrier complete_tx),
//     warp 1 = TMEM allocator + single-thread MMA issuer, warps 2..9 = epilogue.  Persistent
//     grid, one CTA per SM.  Units: pass 1 = one 128-row band over all of K; pass 2 = one
//     128-column band over a K range (split-K, fixed-order fp64 reduction).
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include "internal.h"
#include "tc.h"
#include "tc_ptx.cuh"

namespace enmf {
namespace tci {

constexpr int BM = 128;
constexpr int BK = 64;                          // K elements (= bytes) per stage per row
constexpr int EPI_WARPS = 8;
constexpr int THREADS = 32 * (2 + EPI_WARPS);
constexpr int PLANES = 3;                       // digit planes of X and of the factor
constexpr int NACC = 4;                         // TMEM accumulators
constexpr int TILE_A = BM * BK;                 // bytes per X tile per plane (8 KB)
constexpr int MAX_TILE_B = 128 * BK;            // bytes per factor tile per plane (<= 8 KB)
constexpr int STAGE_BYTES = PLANES * TILE_A + PLANES * MAX_TILE_B;   // 48 KB
constexpr int NST = 4;                          // pipeline stages
constexpr int SMEM_BYTES = NST * STAGE_BYTES + 1024;
constexpr int TMEM_COLS = 512;                  // 4 x 128
constexpr int64_t MAX_UNIT_K = 65536;           // |acc| <= 2 * 126 * 128 * K < 2^31
constexpr double TOP = 126.0;                   // max |t| of a scale group (digits3_n bound)

struct Params {
  const int8_t* xp[PLANES];
  const int8_t* xtp[PLANES];   // transposed packed copy (mode 2), may be null
  const int8_t* fp[PLANES];
  int64_t tiles_per_row_t;     // transposed copy: 64-row K tiles per 128-column band
  double* out;
  int64_t out_ld;
  int64_t split_stride;
  const double* colscale;    // r values: 1 / s_k of the factor column
  const double* rowinv;      // out_rows values: 1 / s of the X row (mode 0) / column (1, 2)
  int mode;                  // 0: P = X V ; 1: Q = X^T U (MN-major gather) ; 2: Q from X^T copy
  int num_units;
  int ksplit;
  int stages_total;          // 64-deep K stages of the full contraction
  int64_t tiles_per_row;     // packed X: 64-column tiles per 128-row band
  int rp;                    // padded N (multiple of 16, <= 128)
  int r;                     // valid output columns
  int64_t out_rows;          // valid output rows
  int tiles;                 // 128-row output tiles (pair kernel: tile 2 t + rank may not exist)
  // single-CTA kernel: units cover output tiles tile0 .. tile0 + tiles - 1 (a band range of
  // pass 2, tc_xtu_bands); output row i is stored at out row i - row0
  int tile0;
  int64_t row0;
  // mode 0, no K split: after a band's output rows are stored each epilogue warp adds 1 to
  // band_ready[tile] (release), so a consumer launched behind this kernel with programmatic
  // dependent launch (tc_hals_kernel) can take the band while later bands are still running
  unsigned* band_ready;
  // optional: {earliest CTA start, latest CTA end} in %globaltimer ns (atomicMin / atomicMax):
  // the pass's own device time when its successor overlaps it (no event can sit between them)
  unsigned long long* tstamp;
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

using namespace tcp;

__device__ __forceinline__ void unit_range(const Params& p, int u, int& tile, int& s0, int& s1,
                                           int& split) {
  tile = u / p.ksplit + p.tile0;
  split = u % p.ksplit;
  const int per = (p.stages_total + p.ksplit - 1) / p.ksplit;
  s0 = split * per;
  s1 = min(p.stages_total, s0 + per);
  if (s1 < s0) s1 = s0;
}

// The six digit products of weight >= 2^-16, issued per 32-deep k-step as 4 MMAs
// {a-plane, first b-plane, accumulator, wide}.  A wide MMA multiplies A_i by the adjacent
// planes [B0; B1] (N = 2 rp) into the adjacent accumulators acc_c | acc_c+1.  The first FRESH
// MMAs of a unit initialise acc0|acc1 and acc3; acc2 (written only by the accumulating wide
// A1 [B0;B1]) is zeroed by the epilogue before the unit (ZERO_ACC).
struct Mma {
  static constexpr int N = 4, FRESH = 2, ZERO_ACC = 2;
  __device__ static __forceinline__ int t(int q, int f) {
    constexpr int tab[4][4] = {{0, 0, 0, 1}, {0, 2, 3, 0}, {2, 0, 3, 0}, {1, 0, 1, 1}};
    return tab[q][f];
  }
};

// acc0 + 2^-8 (acc1 + 2^-8 (acc2 + 2 acc3)), exact in fp64 (|acc| < 2^31: <= 49 bits)
__device__ __forceinline__ double combine(uint32_t v0, uint32_t v1, uint32_t v2, uint32_t v3) {
  const double lo = (double)(int)v2 + 2.0 * (double)(int)v3;
  return (double)(int)v0 + ((double)(int)v1 + lo * 0x1p-8) * 0x1p-8;
}

// Zero the rows (TMEM lanes 32 q .. 32 q + 31) x columns [64 hcol, 64 hcol + 64) of the
// accumulator ZERO_ACC that this epilogue warp owns, before the MMAs of the next unit.
__device__ __forceinline__ void zero_acc_slice(uint32_t tmem_base, int q, int hcol, int rp) {
  const uint32_t lane_addr = tmem_base + ((uint32_t)(32 * q) << 16);
#pragma unroll 1
  for (int h = 0; h < 4; ++h) {
    const int c0 = 64 * hcol + 16 * h;
    if (c0 >= rp) break;
    TMEM_ST16_ZERO(lane_addr + Mma::ZERO_ACC * rp + c0);
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__global__ void __launch_bounds__(THREADS, 1) tc_i8_kernel(const Params p) {
  constexpr int STAGE = STAGE_BYTES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bars[2 * NST + 2];
  __shared__ uint32_t tmem_base_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bar_full = smem_u32(&bars[0]);
  const uint32_t bar_empty = smem_u32(&bars[NST]);
  const uint32_t bar_tfull = smem_u32(&bars[2 * NST]);
  const uint32_t bar_tempty = smem_u32(&bars[2 * NST + 1]);
  const uint32_t tile_b = (uint32_t)p.rp * BK;
  // a dependent grid (programmatic dependent launch) may start as soon as SMs free up: it
  // synchronises on band_ready, not on this grid's completion
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (p.tstamp != nullptr && threadIdx.x == 0) atomicMin(&p.tstamp[0], gtimer());

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(bar_full + 8 * s, 1);
      mbar_init(bar_empty + 8 * s, 1);
    }
    mbar_init(bar_tfull, 1);
    mbar_init(bar_tempty, EPI_WARPS);
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
  if (warp >= 2) zero_acc_slice(tmem_base, warp & 3, (warp - 2) >> 2, p.rp);   // first unit
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (warp == 0) {
    // ===================== producer: the whole warp issues a stage's bulk copies =====================
    int stage = 0;
    uint32_t phase = 0;
    for (int u = blockIdx.x; u < p.num_units; u += gridDim.x) {
      int tile, s0, s1, split;
      unit_range(p, u, tile, s0, s1, split);
      for (int ks = s0; ks < s1; ++ks) {
        mbar_wait(bar_empty + 8 * stage, phase ^ 1);
        const uint32_t fb = bar_full + 8 * stage;
        if (lane == 0) mbar_expect_tx(fb, PLANES * TILE_A + PLANES * tile_b);
        __syncwarp();
        const uint32_t st = smem_u32(smem + (size_t)stage * STAGE);
        if (p.mode == 0) {
          // the planes of a tile are contiguous: one bulk copy
          const int64_t off = ((int64_t)tile * p.tiles_per_row + ks) * PLANES * TILE_A;
          if (lane == 0) bulk_g2s(st, p.xp[0] + off, PLANES * TILE_A, fb);
        } else if (p.mode == 2) {
          // A = X^T from the transposed packed copy: K-major tiles
          const int64_t off = ((int64_t)tile * p.tiles_per_row_t + ks) * PLANES * TILE_A;
          if (lane == 0) bulk_g2s(st, p.xtp[0] + off, PLANES * TILE_A, fb);
        } else {
          // A = X^T: output rows j = column tiles 2*tile, 2*tile+1 of row band ks/2; the K stage
          // is the 64-row half (ks & 1) of that band: 8 chunks of 1 KB per plane, one per lane
          const int64_t band = ks >> 1;
          const int half = ks & 1;
          const int t = (lane >> 2) & 1, kc = lane & 3;
          const int64_t src = (band * p.tiles_per_row + 2 * tile + t) * PLANES * TILE_A +
                              (int64_t)(kc * 16 + 8 * half) * 128;
          const uint32_t dst = (uint32_t)((t * 4 + kc) * 1024);
          for (int pl = lane >> 3; pl < PLANES; pl += 4)
            bulk_g2s(st + pl * TILE_A + dst, p.xp[pl] + src, 1024, fb);
        }
        // the factor planes of a stage are contiguous too
        const int64_t foff = (int64_t)ks * PLANES * tile_b;
        if (lane == 31) bulk_g2s(st + PLANES * TILE_A, p.fp[0] + foff, PLANES * tile_b, fb);
        if (++stage == NST) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (one thread) =====================
    if (lane == 0) {
      // idesc: S32 accumulate (c_format 2), signed int8 A and B, A K-major (mode 0, 2) or
      // MN-major (mode 1), B K-major, M = 128, N = rp (one digit plane) or 2 rp (two planes)
      const bool mn = p.mode == 1;
      const uint32_t idesc_base = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)mn << 15) |
                                  ((uint32_t)(BM >> 4) << 24);
      const uint32_t idesc1 = idesc_base | ((uint32_t)(p.rp >> 3) << 17);
      const uint32_t idesc2 = idesc_base | ((uint32_t)(2 * p.rp >> 3) << 17);
      const uint32_t a_lbo = !mn ? 2048u : 128u;
      const uint32_t a_sbo = !mn ? 128u : 1024u;
      const uint32_t a_kstep = !mn ? 4096u : 512u;
      const uint32_t b_lbo = 128u, b_sbo = 512u, b_kstep = 256u;
      const uint32_t rpc = (uint32_t)p.rp;     // accumulator c lives at TMEM column c * rp
      int stage = 0;
      uint32_t phase = 0;
      uint32_t nunit = 0;
      for (int u = blockIdx.x; u < p.num_units; u += gridDim.x) {
        int tile, s0, s1, split;
        unit_range(p, u, tile, s0, s1, split);
        if (s1 <= s0) continue;
        mbar_wait(bar_tempty, (nunit & 1) ^ 1);    // epilogue drained the previous unit
        tc_fence_after();
        for (int ks = s0; ks < s1; ++ks) {
          mbar_wait(bar_full + 8 * stage, phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(smem + (size_t)stage * STAGE);
          const uint32_t b0 = a0 + PLANES * TILE_A;
#pragma unroll
          for (int j = 0; j < BK / 32; ++j) {
#pragma unroll
            for (int q = 0; q < Mma::N; ++q) {
              const int pa = Mma::t(q, 0), pb = Mma::t(q, 1), ac = Mma::t(q, 2), wide = Mma::t(q, 3);
              const uint64_t ad = umma_desc(a0 + pa * TILE_A + j * a_kstep, a_lbo, a_sbo);
              const uint64_t bd = umma_desc(b0 + pb * tile_b + j * b_kstep, b_lbo, b_sbo);
              const bool fresh = ks == s0 && j == 0 && q < Mma::FRESH;
              tc_mma_i8(tmem_base + ac * rpc, ad, bd, wide ? idesc2 : idesc1, fresh ? 0u : 1u);
            }
          }
          tc_commit(bar_empty + 8 * stage);          // frees the smem slot when MMAs retire
          if (++stage == NST) { stage = 0; phase ^= 1; }
        }
        tc_commit(bar_tfull);                        // unit's accumulators complete
        ++nunit;
      }
    }
  } else {
    // ===================== epilogue: exact int32 -> fp64 =====================
    const int e = warp - 2;
    const int q = warp & 3;                 // TMEM lane quadrant of this warp
    const int hcol = e >> 2;                // columns [64*hcol, 64*hcol + 64)
    const int row_in_tile = 32 * q + lane;
    uint32_t nunit = 0;
    for (int u = blockIdx.x; u < p.num_units; u += gridDim.x) {
      int tile, s0, s1, split;
      unit_range(p, u, tile, s0, s1, split);
      if (s1 <= s0) continue;
      mbar_wait_sleep(bar_tfull, nunit & 1);
      tc_fence_after();
      const int64_t row = (int64_t)tile * BM + row_in_tile;
      double* o = p.out + (int64_t)split * p.split_stride + (row - p.row0) * p.out_ld;
      const double rinv = row < p.out_rows ? p.rowinv[row] : 0.0;
      const uint32_t lane_addr = tmem_base + ((uint32_t)(32 * q) << 16);
#pragma unroll 1
      for (int h = 0; h < 4; ++h) {
        const int c0 = 64 * hcol + 16 * h;
        if (c0 >= p.rp) break;
        uint32_t v[NACC][16];
#pragma unroll
        for (int c = 0; c < NACC; ++c) TMEM_LD16(lane_addr + c * p.rp + c0, v[c]);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (row < p.out_rows) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int col = c0 + i;
            if (col < p.r)       // 1/(s_row s_col) is a power of two: one rounding
              o[col] = combine(v[0][i], v[1][i], v[2][i], v[3][i]) * (p.colscale[col] * rinv);
          }
        }
      }
      zero_acc_slice(tmem_base, q, hcol, p.rp);   // acc2 starts at 0 for the next unit
      if (p.band_ready != nullptr) __threadfence();  // this lane's rows before the flag
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(bar_tempty);
        if (p.band_ready != nullptr) atomicAdd(&p.band_ready[tile], 1u);
      }
      ++nunit;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (p.tstamp != nullptr && threadIdx.x == 0) atomicMax(&p.tstamp[1], gtimer());
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(TMEM_COLS));
  }
}

// ------------------------------------------------------------------ CTA-pair kernel
// cta_group::2: a cluster of two CTAs (two SMs of a TPC) computes a 256-row output band with
// M = 256 MMAs issued by the even CTA.  Each CTA stages its own 128 rows of A (X or X^T digits,
// tile 2 t + rank) and HALF of every B operand, at the same shared-memory offsets: for the wide
// MMA [B0; B1] (N = 2 rp) CTA 0 holds plane 0 and CTA 1 plane 1; for a narrow one (B2, B0) each
// holds rp/2 rows of the plane (a contiguous half of the canonical tile).  Per SM this halves
// the B-operand shared-memory reads.
// Synchronisation: each CTA's producer fills its own stage (cp.async.bulk, local mbarrier);
// CTA 1's idle MMA warp relays its stage completion to the leader (remote mbarrier arrive);
// the leader's commits are multicast to both CTAs (stage empty, accumulators full); both CTAs'
// epilogues release the accumulators on the leader's barrier.
constexpr int PAIR_SMEM = 230400;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    tc_i8_pair_kernel(const Params p) {
  constexpr int STAGE = PLANES * TILE_A + 2 * MAX_TILE_B;         // A planes | [B0|B1] | 2 halves
  constexpr int PNST = (PAIR_SMEM - 1024) / STAGE;                // 5
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bars[3 * 8 + 2];
  __shared__ uint32_t tmem_base_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const uint32_t bar_full = smem_u32(&bars[0]);
  const uint32_t bar_empty = smem_u32(&bars[PNST]);
  const uint32_t bar_peer = smem_u32(&bars[2 * PNST]);       // leader: CTA 1's stage is full
  const uint32_t bar_tfull = smem_u32(&bars[3 * PNST]);
  const uint32_t bar_tempty = smem_u32(&bars[3 * PNST + 1]);  // leader: both epilogues drained
  const uint32_t tile_b = (uint32_t)p.rp * BK;
  const uint32_t half_b = tile_b / 2;
  const uint32_t b_bytes = tile_b + 2 * half_b;

  if (threadIdx.x == 0) {
    for (int s = 0; s < PNST; ++s) {
      mbar_init(bar_full + 8 * s, 1);
      mbar_init(bar_empty + 8 * s, 1);
      mbar_init(bar_peer + 8 * s, 1);
    }
    mbar_init(bar_tfull, 1);
    mbar_init(bar_tempty, 2 * EPI_WARPS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_s)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_s;
  if (warp >= 2) zero_acc_slice(tmem_base, warp & 3, (warp - 2) >> 2, p.rp);   // first unit
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();

  if (warp == 0) {
    // ===================== producer (both CTAs): own A rows, own half of B =====================
    int stage = 0;
    uint32_t phase = 0;
    for (int u = cid; u < p.num_units; u += ncl) {
      int pt, s0, s1, split;
      unit_range(p, u, pt, s0, s1, split);
      const int tile = min(2 * pt + (int)rank, p.tiles - 1);   // a missing odd tile re-reads
      for (int ks = s0; ks < s1; ++ks) {                       // the last one; not stored
        mbar_wait(bar_empty + 8 * stage, phase ^ 1);
        const uint32_t fb = bar_full + 8 * stage;
        if (lane == 0) mbar_expect_tx(fb, PLANES * TILE_A + b_bytes);
        __syncwarp();
        const uint32_t st = smem_u32(smem + (size_t)stage * STAGE);
        if (lane == 0) {
          const int8_t* src =
              p.mode == 0 ? p.xp[0] + ((int64_t)tile * p.tiles_per_row + ks) * PLANES * TILE_A
                          : p.xtp[0] + ((int64_t)tile * p.tiles_per_row_t + ks) * PLANES * TILE_A;
          bulk_g2s(st, src, PLANES * TILE_A, fb);
        }
        const int64_t foff = (int64_t)ks * PLANES * tile_b;
        const uint32_t bst = st + PLANES * TILE_A;
        if (lane == 28) bulk_g2s(bst, p.fp[rank] + foff, tile_b, fb);                  // B0|B1
        if (lane == 30)                                                                // B2 half
          bulk_g2s(bst + tile_b, p.fp[2] + foff + rank * half_b, half_b, fb);
        if (lane == 31)                                                                // B0 half
          bulk_g2s(bst + tile_b + half_b, p.fp[0] + foff + rank * half_b, half_b, fb);
        if (++stage == PNST) { stage = 0; phase ^= 1; }
      }
    }
    // drain: the leader's last commits arrive on this CTA's empty barriers before it exits
    for (int i = 0; i < PNST; ++i) {
      mbar_wait(bar_empty + 8 * stage, phase ^ 1);
      if (++stage == PNST) { stage = 0; phase ^= 1; }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ===================== MMA issuer (leader CTA, one thread) =====================
      const uint32_t idesc_base = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(256 >> 4) << 24);
      const uint32_t idesc1 = idesc_base | ((uint32_t)(p.rp >> 3) << 17);
      const uint32_t idesc2 = idesc_base | ((uint32_t)(2 * p.rp >> 3) << 17);
      const uint32_t a_lbo = 2048u, a_sbo = 128u, a_kstep = 4096u;
      const uint32_t b_lbo = 128u, b_sbo = 512u, b_kstep = 256u;
      const uint32_t rpc = (uint32_t)p.rp;
      int stage = 0;
      uint32_t phase = 0;
      uint32_t nunit = 0;
      for (int u = cid; u < p.num_units; u += ncl) {
        int pt, s0, s1, split;
        unit_range(p, u, pt, s0, s1, split);
        if (s1 <= s0) continue;
        mbar_wait_cluster(bar_tempty, (nunit & 1) ^ 1);
        tc_fence_after();
        for (int ks = s0; ks < s1; ++ks) {
          mbar_wait(bar_full + 8 * stage, phase);
          mbar_wait_cluster(bar_peer + 8 * stage, phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(smem + (size_t)stage * STAGE);
          const uint32_t b0 = a0 + PLANES * TILE_A;
#pragma unroll
          for (int j = 0; j < BK / 32; ++j) {
#pragma unroll
            for (int q = 0; q < Mma::N; ++q) {
              const int pa = Mma::t(q, 0), pb = Mma::t(q, 1), ac = Mma::t(q, 2), wide = Mma::t(q, 3);
              // B region: wide [B0;B1] at 0; narrow B2 / B0 halves after it
              const uint32_t breg = wide ? 0u : tile_b + (pb == 0 ? half_b : 0u);
              const uint64_t ad = umma_desc(a0 + pa * TILE_A + j * a_kstep, a_lbo, a_sbo);
              const uint64_t bd = umma_desc(b0 + breg + j * b_kstep, b_lbo, b_sbo);
              const bool fresh = ks == s0 && j == 0 && q < Mma::FRESH;
              tc_mma_i8_pair(tmem_base + ac * rpc, ad, bd, wide ? idesc2 : idesc1,
                             fresh ? 0u : 1u);
            }
          }
          tc_commit_pair(bar_empty + 8 * stage, 3);     // frees the slot in both CTAs
          if (++stage == PNST) { stage = 0; phase ^= 1; }
        }
        tc_commit_pair(bar_tfull, 3);                   // accumulators complete in both CTAs
        ++nunit;
      }
    } else if (lane == 0) {
      // ===================== relay (CTA 1): my stage is full -> leader =====================
      const uint32_t peer0 = mapa_shared(bar_peer, 0);
      int stage = 0;
      uint32_t phase = 0;
      for (int u = cid; u < p.num_units; u += ncl) {
        int pt, s0, s1, split;
        unit_range(p, u, pt, s0, s1, split);
        for (int ks = s0; ks < s1; ++ks) {
          mbar_wait(bar_full + 8 * stage, phase);
          mbar_arrive_cluster(peer0 + 8 * stage);
          if (++stage == PNST) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else {
    // ===================== epilogue (both CTAs): exact int32 -> fp64 of my 128 rows ==========
    const int e = warp - 2;
    const int q = warp & 3;
    const int hcol = e >> 2;
    const int row_in_tile = 32 * q + lane;
    const uint32_t tempty0 = mapa_shared(bar_tempty, 0);
    uint32_t nunit = 0;
    for (int u = cid; u < p.num_units; u += ncl) {
      int pt, s0, s1, split;
      unit_range(p, u, pt, s0, s1, split);
      if (s1 <= s0) continue;
      mbar_wait_sleep(bar_tfull, nunit & 1);     // commit from the leader's tensor core
      tc_fence_after();
      const int tile = 2 * pt + (int)rank;
      const int64_t row = (int64_t)tile * BM + row_in_tile;
      const bool store = tile < p.tiles && row < p.out_rows;
      double* o = p.out + (int64_t)split * p.split_stride + row * p.out_ld;
      const double rinv = store ? p.rowinv[row] : 0.0;
      const uint32_t lane_addr = tmem_base + ((uint32_t)(32 * q) << 16);
#pragma unroll 1
      for (int h = 0; h < 4; ++h) {
        const int c0 = 64 * hcol + 16 * h;
        if (c0 >= p.rp) break;
        uint32_t v[NACC][16];
#pragma unroll
        for (int c = 0; c < NACC; ++c) TMEM_LD16(lane_addr + c * p.rp + c0, v[c]);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (store) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int col = c0 + i;
            if (col < p.r)
              o[col] = combine(v[0][i], v[1][i], v[2][i], v[3][i]) * (p.colscale[col] * rinv);
          }
        }
      }
      zero_acc_slice(tmem_base, q, hcol, p.rp);   // acc2 starts at 0 for the next unit
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty0);
      ++nunit;
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(TMEM_COLS));
  }
}

// ------------------------------------------------------------------ packing

// 16 consecutive values t(k) (|t| < TOP) -> the 16-byte chunks of the 3 digit planes,
// w[plane][k / 4] byte k % 4, built in registers (no addressable local arrays).  Returns
// sum_k n_k^2 (n = rint(t 2^15), exact: < 2^49) for the norm of the quantised operand.
template <typename F>
__device__ __forceinline__ double pack_digits16(F val, uint32_t (&w)[PLANES][4]) {
#pragma unroll
  for (int pl = 0; pl < PLANES; ++pl)
#pragma unroll
    for (int q = 0; q < 4; ++q) w[pl][q] = 0u;
  double n2 = 0.0;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int n = __double2int_rn(val(k) * 32768.0);
    n2 += (double)n * (double)n;
    const uint32_t dw = digits3_n(n);
#pragma unroll
    for (int pl = 0; pl < PLANES; ++pl) w[pl][k >> 2] |= ((dw >> (8 * pl)) & 255u) << (8 * (k & 3));
  }
  return n2;
}

// Block sum of v (blockDim.x <= 1024, a multiple of 32) into *out by thread 0.
__device__ __forceinline__ void block_sum_to(double v, double* out) {
  __shared__ double red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) *out = v;
  }
}

// X (rows x n, ld) -> 3 digit planes of [Mt][tiles_per_row] tiles, row i scaled by
// 1 / rinv[i] (a power of two).  One 128-row x 64-column tile at a time: coalesced row reads
// into shared memory, then the tile's 512 16-byte chunks per plane in memory order (chunk
// w = (kc*16 + g)*8 + ri), so the writes are contiguous too.  q2parts (optional, one per
// block): sum of the squared quantised values, ||X~||^2 of this copy.
__global__ void __launch_bounds__(256)
pack_x_kernel(const float* __restrict__ X, int64_t ldx, int64_t rows, int64_t n,
              const double* __restrict__ rinv, int64_t tiles_per_row, int64_t Mt, uint4* out,
              double* q2parts) {
  __shared__ float tx[BM][BK + 1];
  const bool vec = (ldx & 3) == 0 && ((uintptr_t)X & 15) == 0;
  double q2 = 0.0;
  for (int64_t t = blockIdx.x; t < Mt * tiles_per_row; t += gridDim.x) {
    const int64_t mt = t / tiles_per_row, kt = t - mt * tiles_per_row;
    __syncthreads();
    for (int e = threadIdx.x; e < BM * BK / 4; e += blockDim.x) {
      const int il = e / (BK / 4), jq = e % (BK / 4);
      const int64_t i = mt * BM + il, j = kt * BK + 4 * jq;
      float4 f = make_float4(0.f, 0.f, 0.f, 0.f);
      if (i < rows) {
        const float* xr = X + i * ldx;
        if (vec && j + 4 <= n) {
          f = *reinterpret_cast<const float4*>(xr + j);
        } else {
          if (j < n) f.x = xr[j];
          if (j + 1 < n) f.y = xr[j + 1];
          if (j + 2 < n) f.z = xr[j + 2];
          if (j + 3 < n) f.w = xr[j + 3];
        }
      }
      tx[il][4 * jq] = f.x;
      tx[il][4 * jq + 1] = f.y;
      tx[il][4 * jq + 2] = f.z;
      tx[il][4 * jq + 3] = f.w;
    }
    __syncthreads();
    for (int w = threadIdx.x; w < BM * BK / 16; w += blockDim.x) {
      const int kc = w >> 7, g = (w >> 3) & 15, ri = w & 7;
      const int il = g * 8 + ri;
      const int64_t i = mt * BM + il;
      const double s = i < rows ? 1.0 / rinv[i] : 0.0;        // exact: a power of two
      uint32_t wd[PLANES][4];
      const double n2 = pack_digits16([&](int k) { return (double)tx[il][kc * 16 + k] * s; }, wd);
      if (i < rows) q2 += n2 * (rinv[i] * rinv[i]);
      // planes interleaved per tile: tile t, plane pl at (t * PLANES + pl) * TILE_A
      const int64_t idx = (t * PLANES * TILE_A) / 16 + w;
#pragma unroll
      for (int pl = 0; pl < PLANES; ++pl)
        out[idx + pl * (TILE_A / 16)] = make_uint4(wd[pl][0], wd[pl][1], wd[pl][2], wd[pl][3]);
    }
  }
  if (q2parts) block_sum_to(q2 * 0x1p-30, q2parts + blockIdx.x);
}

// X^T copy: tiles [jt][it] of 128 columns (j, the M side of Q = X^T U) x 64 rows (i, the K
// side), K-major core matrices (kc*16 + g)*128 like pass 1's tiles, column j scaled by
// 1 / cinv[j].  A block stages a 64 x 128 block of X in shared memory (coalesced reads) and
// writes 16-byte chunks of 16 rows.  q2parts as pack_x_kernel.
__global__ void __launch_bounds__(256)
pack_xt_kernel(const float* __restrict__ X, int64_t ldx, int64_t rows, int64_t n,
               const double* __restrict__ cinv, int64_t jtiles, int64_t itiles, uint4* out,
               double* q2parts) {
  __shared__ float tx[64][129];
  double q2 = 0.0;
  for (int64_t t = blockIdx.x; t < jtiles * itiles; t += gridDim.x) {
    const int64_t jt = t / itiles, it = t % itiles;
    for (int e = threadIdx.x; e < 64 * 128; e += blockDim.x) {
      const int il = e / 128, jl = e % 128;
      const int64_t i = it * 64 + il, j = jt * 128 + jl;
      tx[il][jl] = (i < rows && j < n) ? X[i * ldx + j] : 0.0f;
    }
    __syncthreads();
    for (int w = threadIdx.x; w < 512; w += blockDim.x) {
      const int kc = w / 128, g = (w / 8) % 16, ri = w % 8;
      const int jl = g * 8 + ri;
      const int64_t j = jt * 128 + jl;
      const double s = j < n ? 1.0 / cinv[j] : 0.0;
      uint32_t wd[PLANES][4];
      const double n2 = pack_digits16([&](int k) { return (double)tx[kc * 16 + k][jl] * s; }, wd);
      if (j < n) q2 += n2 * (cinv[j] * cinv[j]);
      const int64_t idx = (t * PLANES * TILE_A) / 16 + w;   // planes interleaved per tile
#pragma unroll
      for (int pl = 0; pl < PLANES; ++pl)
        out[idx + pl * (TILE_A / 16)] = make_uint4(wd[pl][0], wd[pl][1], wd[pl][2], wd[pl][3]);
    }
    __syncthreads();
  }
  if (q2parts) block_sum_to(q2 * 0x1p-30, q2parts + blockIdx.x);
}

// Factor F (K x r, ld) * fscale[col] -> B tiles [Kt][PLANES][rp x 64]: 16-byte chunk w of a
// tile holds F[kt*64 + kc*16 + 0..15][g*8 + ri] with g = w/32, kc = (w/8)%4, ri = w%8, i.e.
// byte (g*4 + kc)*128 + ri*16 (SBO 512, LBO 128), so the planes B0, B1 stored back to back
// form one uniform 2 rp-row operand.  A block stages 64 factor rows in shared memory so global
// reads are coalesced.
template <typename T>
__global__ void __launch_bounds__(256)
pack_factor_kernel(const T* __restrict__ F, int64_t ldf, int64_t K, int r, int rp,
                   const double* __restrict__ fscale, int64_t Kt, uint4* out) {
  extern __shared__ __align__(16) unsigned char pf_smem[];
  T(*tileF)[129] = reinterpret_cast<T(*)[129]>(pf_smem);   // BK x 129
  const int gpt = rp / 8;
  const int chunks = 4 * gpt * 8;                        // 16-byte chunks per tile per plane
  for (int64_t kt = blockIdx.x; kt < Kt; kt += gridDim.x) {
    for (int e = threadIdx.x; e < BK * rp; e += blockDim.x) {
      const int kk = e / rp, col = e % rp;
      const int64_t row = kt * BK + kk;
      tileF[kk][col] = (row < K && col < r) ? F[row * ldf + col] : (T)0;
    }
    __syncthreads();
    for (int w = threadIdx.x; w < chunks; w += blockDim.x) {
      const int g = w / 32, kc = (w / 8) % 4;
      const int col = g * 8 + w % 8;
      const double s = col < r ? fscale[col] : 0.0;
      uint32_t wd[PLANES][4];
      pack_digits16([&](int k) { return (double)tileF[kc * 16 + k][col] * s; }, wd);
      const int64_t idx = kt * PLANES * chunks + w;       // planes interleaved per stage
#pragma unroll
      for (int pl = 0; pl < PLANES; ++pl)
        out[idx + pl * chunks] = make_uint4(wd[pl][0], wd[pl][1], wd[pl][2], wd[pl][3]);
    }
    __syncthreads();
  }
}

// Per-column max |F| (F rows x r) into maxbits[r] (bits of the fp64 |value|: non-negative
// doubles order like their bit patterns, so the max is order independent).
template <typename T>
__global__ void colmax_kernel(const T* __restrict__ F, int64_t ldf, int64_t rows, int r,
                              unsigned long long* maxbits) {
  // thread t owns column t % r of rows t / r, t / r + g, ... (g = 256 / r rows per block step):
  // a register maximum per thread, one shared-memory atomic per thread at the end (the
  // element-wise shared atomics of round 1 made this a 60 us kernel for a 25 MB factor)
  __shared__ unsigned long long m[128];
  for (int k = threadIdx.x; k < r; k += blockDim.x) m[k] = 0ull;
  __syncthreads();
  const int g = (int)blockDim.x / r;
  const int t = threadIdx.x, k = t % r;
  if (t < g * r) {
    double mx = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * g + t / r; i < rows; i += (int64_t)gridDim.x * g)
      mx = fmax(mx, fabs((double)F[i * ldf + k]));
    if (mx > 0.0) atomicMax(&m[k], (unsigned long long)__double_as_longlong(mx));
  }
  __syncthreads();
  for (int k2 = threadIdx.x; k2 < r; k2 += blockDim.x)
    if (m[k2]) atomicMax(&maxbits[k2], m[k2]);
}

// out[i, c0 + j] = buf[i, j] (rows x nb contiguous -> column block of a row-major ldo matrix)
__global__ void scatter_cols_kernel(const double* __restrict__ buf, int64_t rows, int nb,
                                    double* out, int64_t ldo, int c0) {
  const int64_t total = rows * nb;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / nb;
    out[i * ldo + c0 + (e - i * nb)] = buf[e];
  }
}

// Power of two s with mx * s in [63, 126) (TOP / 2 .. TOP), 1 for mx = 0: the largest scale
// whose top digit stays within int8 (digits3_n).
__host__ __device__ inline double pow2_scale(double mx) {
  if (!(mx > 0.0)) return 1.0;
  int e = 0;
  const double f = frexp(mx, &e);     // mx = f 2^e, f in [0.5, 1)
  return ldexp(1.0, (f < TOP / 128.0 ? 7 : 6) - e);
}

// fscale[k] = power of two with max|F_k| fscale in [63, 126); colscale[k] = 1 / fscale[k].
__global__ void scales_kernel(const unsigned long long* maxbits, int r, double* fscale,
                              double* colscale) {
  for (int k = threadIdx.x; k < r; k += blockDim.x) {
    const double s = pow2_scale(__longlong_as_double((long long)maxbits[k]));
    fscale[k] = s;
    colscale[k] = 1.0 / s;
  }
}

// Row maxima of X (rows x n): one warp per row; bits of the non-negative fp32 maxima.
__global__ void x_rowmax_kernel(const float* __restrict__ X, int64_t ldx, int64_t rows,
                                int64_t n, unsigned* rowbits) {
  const int lane = threadIdx.x & 31;
  const bool vec = (ldx & 3) == 0 && ((uintptr_t)X & 15) == 0;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < rows;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const float* xr = X + i * ldx;
    unsigned m = 0;
    if (vec) {
      const int64_t n4 = n >> 2;
      for (int64_t q = lane; q < n4; q += 32) {
        const float4 f = reinterpret_cast<const float4*>(xr)[q];
        m = max(max(m, __float_as_uint(fabsf(f.x))), max(__float_as_uint(fabsf(f.y)),
                max(__float_as_uint(fabsf(f.z)), __float_as_uint(fabsf(f.w)))));
      }
      for (int64_t j = 4 * n4 + lane; j < n; j += 32) m = max(m, __float_as_uint(fabsf(xr[j])));
    } else {
      for (int64_t j = lane; j < n; j += 32) m = max(m, __float_as_uint(fabsf(xr[j])));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) rowbits[i] = m;
  }
}

// Column maxima of X: a block covers 256 columns of a band of `band` rows, one global atomic
// per column per block.
__global__ void x_colmax_kernel(const float* __restrict__ X, int64_t ldx, int64_t rows,
                                int64_t n, int64_t band, unsigned* colbits) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int64_t i0 = blockIdx.y * band, i1 = min(rows, i0 + band);
  unsigned m = 0;
  for (int64_t i = i0; i < i1; ++i) m = max(m, __float_as_uint(fabsf(X[i * ldx + j])));
  atomicMax(colbits + j, m);
}

// inv[i] = 1 / pow2_scale(max): the epilogue's row factor; uniform (optional): every entry
// takes the scale of the maximum over all of bits[0, count).
__global__ void inv_scales_kernel(const unsigned* bits, int64_t count, double* inv,
                                  const unsigned* uniform) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    inv[i] = 1.0 / pow2_scale((double)__uint_as_float(uniform ? *uniform : bits[i]));
}

__global__ void max_u32_kernel(const unsigned* bits, int64_t count, unsigned* out) {
  unsigned m = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, bits[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

}  // namespace tci

using namespace tci;

struct TcState {
  int64_t rows = 0, n = 0, r = 0;
  int rp = 0;
  int64_t Mt = 0;              // 128-row bands of X
  int64_t tiles_per_row = 0;   // 64-column tiles per band (even: 128-column pairs)
  int64_t Kt2 = 0;             // 64-row K stages of pass 2 (= 2 Mt)
  int8_t* xp[PLANES] = {nullptr, nullptr, nullptr};
  int8_t* xtp[PLANES] = {nullptr, nullptr, nullptr};   // X^T copy (pass 2), optional
  int8_t* fp[PLANES] = {nullptr, nullptr, nullptr};
  double* xinv_r = nullptr;    // rows: 1 / s of each X row (pass 1 output rows)
  double* xinv_c = nullptr;    // n: 1 / s of each X column (pass 2 output rows)
  unsigned* xbits = nullptr;   // rows + n + 1: row / column / global maxima (fp32 bits)
  double* xq2 = nullptr;       // ||X~||^2 of the copy pass 2 reads
  unsigned long long* fmaxbits = nullptr;   // 128 factor column maxima (fp64 bits)
  double* fscale = nullptr;    // 128
  double* colscale = nullptr;  // 128
  double* colbuf = nullptr;    // max(rows, n) x 128: column-block products (tc_xf), lazy
  double* partial = nullptr;   // ksplit2 x n x r  (pass 2)  /  ksplit1 x rows x r (pass 1)
  int ksplit1 = 1, ksplit2 = 1;
  bool pair = false;           // cta_group::2 kernel (ENMF_TC_PAIR=1 enables)
  int ksplit1p = 1, ksplit2p = 1;
  int sms = kSMs;
  unsigned* band_flags = nullptr;   // Mt + 2: pass-1 band flags, epoch, consumer tile counter
  unsigned long long* stamps = nullptr;   // 4: pass-1 kernel timestamps (tc_stamp_*)
  double* chunk_partial = nullptr;        // split-K partials of a pass-2 band range
  size_t chunk_cap = 0;
  unsigned long long* gram64 = nullptr;   // 128 x 128 int64: the exact quantised Gram
};

bool tc_supported(int64_t rows, int64_t n, int64_t r) {
  return r >= 1 && r <= 128 && rows >= 1 && n >= 1;
}

void tc_destroy(TcState* s) {
  if (!s) return;
  if (s->xp[0]) cudaFree(s->xp[0]);     // planes 1..2 point into the same allocation
  if (s->xtp[0]) cudaFree(s->xtp[0]);
  if (s->fp[0]) cudaFree(s->fp[0]);
  void* bufs[] = {s->xinv_r, s->xinv_c, s->xbits, s->xq2, s->fmaxbits, s->fscale,
                  s->colscale, s->partial, s->colbuf, s->band_flags, s->stamps,
                  s->chunk_partial, s->gram64};
  for (void* b : bufs)
    if (b) cudaFree(b);
  delete s;
}

const double* tc_factor_scales(const TcState* s) { return s ? s->fscale : nullptr; }
const double* tc_xq_norm2(const TcState* s) { return s ? s->xq2 : nullptr; }

// K split of a pass: units = tiles x ks are dealt round-robin to `sms` persistent CTAs, so
// the pass takes ceil(units / sms) units of ceil(stages / ks) stages each.  Pick the ks that
// minimises that makespan (the old rule, ks = ceil(4 sms / tiles), left pass 2 at C5 with
// 782 units = 5.28 waves, i.e. 12 % of the SMs idle in the last wave), with a small per-split
// charge for the fp64 partials and their reduction (`split_cost` per extra split); every unit
// K <= MAX_UNIT_K, no empty unit.
static int choose_split(int64_t tiles, int64_t stages, int sms, double split_cost) {
  const int kmin = std::max(1, (int)((stages * BK + MAX_UNIT_K - 1) / MAX_UNIT_K));
  int best = kmin;
  double best_t = 1e300;
  for (int ks = kmin; ks <= std::max(kmin, 16) && ks <= stages; ++ks) {
    const int64_t per = (stages + ks - 1) / ks;
    const int64_t kse = (stages + per - 1) / per;
    const double t = (double)((tiles * kse + sms - 1) / sms) * (double)per *
                     (1.0 + split_cost * (double)(kse - 1));
    if (t < best_t * (1.0 - 1e-9)) {
      best_t = t;
      best = (int)kse;
    }
  }
  return best;
}

static int choose_split_waves(int64_t tiles, int64_t stages, int sms) {
  int ks = (int)((4 * sms + tiles - 1) / tiles);
  const int kmin = (int)((stages * BK + MAX_UNIT_K - 1) / MAX_UNIT_K);
  ks = std::max(std::max(ks, kmin), 1);
  ks = std::min<int64_t>(ks, stages);
  const int64_t per = (stages + ks - 1) / ks;
  return (int)((stages + per - 1) / per);
}

int tc_create(TcState** out, const float* X, int64_t ldx, int64_t rows, int64_t n, int64_t r,
              cudaStream_t st, double* q2parts, int q2cap) {
  *out = nullptr;
  TcState* s = new TcState();
  s->rows = rows;
  s->n = n;
  s->r = r;
  s->rp = (int)((r + 15) / 16 * 16);
  s->Mt = (rows + BM - 1) / BM;
  s->tiles_per_row = ((n + 127) / 128) * 2;
  s->Kt2 = 2 * s->Mt;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&s->sms, cudaDevAttrMultiProcessorCount, dev);
  // pass 1 writes P directly unless splitting pays for its fp64 partials (rows x r x ks,
  // written and reduced: charged 5 % per extra split) -- at C5 / 8 ranks 196 row bands take
  // ks = 3.  Pass 2 keeps its measured rule, ks = ceil(4 SMs / tiles): the makespan choice
  // (ks = 3 at C5) ran 2 % slower in an alternating 1-GPU A/B -- under the power cap idle SMs
  // in the last wave lend their power to the others, while extra partials cost bandwidth.
  s->ksplit1 = choose_split(s->Mt, s->tiles_per_row, s->sms, 0.05);
  s->ksplit2 = choose_split_waves(s->tiles_per_row / 2, s->Kt2, s->sms);
  {
    // cta_group::2 kernel: correct, but measured slower than the single-CTA kernel at C5
    // (DESIGN.md §5.1); ENMF_TC_PAIR=1 selects it
    const char* ev = getenv("ENMF_TC_PAIR");
    s->pair = ev && atoi(ev) == 1 && s->sms >= 2;
    const int64_t pairs1 = (s->Mt + 1) / 2, pairs2 = (s->tiles_per_row / 2 + 1) / 2;
    s->ksplit1p = 1;
    if (s->tiles_per_row * BK > MAX_UNIT_K || pairs1 < s->sms / 2)
      s->ksplit1p = choose_split(pairs1, s->tiles_per_row, s->sms / 2, 0.05);
    s->ksplit2p = choose_split_waves(pairs2, s->Kt2, s->sms / 2);
  }
  const size_t plane = (size_t)s->Mt * s->tiles_per_row * TILE_A;
  const int64_t fK = std::max<int64_t>(s->tiles_per_row, s->Kt2);
  const size_t fplane = (size_t)fK * 128 * BK;          // any factor block of <= 128 columns
  const size_t part = std::max<size_t>(
      (size_t)std::max(s->ksplit2, s->ksplit2p) * n * 128,
      std::max(s->ksplit1, s->ksplit1p) > 1
          ? (size_t)std::max(s->ksplit1, s->ksplit1p) * rows * 128
          : 0);
  cudaError_t e = cudaSuccess;
  // one allocation per packed copy; planes interleaved per tile (plane p at + p * tile bytes)
  e = cudaMalloc(&s->xp[0], PLANES * plane);
  if (!e) e = cudaMalloc(&s->fp[0], PLANES * fplane);
  for (int p = 1; p < PLANES && !e; ++p) {
    s->xp[p] = s->xp[0] + p * TILE_A;
    s->fp[p] = nullptr;    // factor planes: fp[0] + q * rp * BK for the block's rp (per launch)
  }
  if (!e) e = cudaMalloc(&s->xinv_r, sizeof(double) * rows);
  if (!e) e = cudaMalloc(&s->xinv_c, sizeof(double) * n);
  if (!e) e = cudaMalloc(&s->xbits, sizeof(unsigned) * (rows + n + 1));
  if (!e) e = cudaMalloc(&s->xq2, sizeof(double));
  if (!e) e = cudaMalloc(&s->fmaxbits, sizeof(unsigned long long) * 128);
  if (!e) e = cudaMalloc(&s->fscale, sizeof(double) * 128);
  if (!e) e = cudaMalloc(&s->colscale, sizeof(double) * 128);
  if (!e) e = cudaMalloc(&s->partial, sizeof(double) * std::max<size_t>(part, 1));
  if (e) {
    cudaGetLastError();
    tc_destroy(s);
    return e == cudaErrorMemoryAllocation ? 2 : 1;
  }
  // A second, transposed copy makes pass 2 a K-major stream of whole tiles like pass 1 (the
  // MN-major gather of 1 KB pieces measured ~2x slower).  It costs another 3 bytes per element
  // of HBM capacity and is skipped (ENMF_TC_XT=0, or not enough free memory) in favour of the
  // gather path.
  {
    const char* ev = getenv("ENMF_TC_XT");
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    const bool want = !(ev && atoi(ev) == 0) && free_b > PLANES * plane + ((size_t)8 << 30);
    if (want && cudaMalloc(&s->xtp[0], PLANES * plane) != cudaSuccess) {
      cudaGetLastError();
      s->xtp[0] = nullptr;
    }
    for (int p = 1; p < PLANES && s->xtp[0]; ++p) s->xtp[p] = s->xtp[0] + p * TILE_A;
  }
  // digit scales: per X row for pass 1 and per X column for pass 2 (the output rows of each
  // product); without the X^T copy pass 2 gathers the X copy along K, so every row of it (and
  // every output row of pass 2) takes the global scale
  unsigned* rowbits = s->xbits;
  unsigned* colbits = s->xbits + rows;
  unsigned* allbits = s->xbits + rows + n;
  cudaMemsetAsync(s->xbits, 0, sizeof(unsigned) * (rows + n + 1), st);
  x_rowmax_kernel<<<8 * s->sms, 256, 0, st>>>(X, ldx, rows, n, rowbits);
  max_u32_kernel<<<2 * s->sms, 256, 0, st>>>(rowbits, rows, allbits);
  count_launch(2);
  const bool uniform = s->xtp[0] == nullptr;
  if (!uniform) {
    const int64_t band = 4096;
    dim3 g((unsigned)((n + 255) / 256), (unsigned)((rows + band - 1) / band));
    x_colmax_kernel<<<g, 256, 0, st>>>(X, ldx, rows, n, band, colbits);
    count_launch();
  }
  inv_scales_kernel<<<2 * s->sms, 256, 0, st>>>(rowbits, rows, s->xinv_r,
                                                uniform ? allbits : nullptr);
  inv_scales_kernel<<<2 * s->sms, 256, 0, st>>>(colbits, n, s->xinv_c,
                                                uniform ? allbits : nullptr);
  count_launch(2);
  const int pgrid = std::min(8 * s->sms, q2cap);
  pack_x_kernel<<<pgrid, 256, 0, st>>>(X, ldx, rows, n, s->xinv_r, s->tiles_per_row, s->Mt,
                                       (uint4*)s->xp[0], uniform ? q2parts : nullptr);
  count_launch();
  if (s->xtp[0]) {
    const int64_t jt = s->tiles_per_row / 2;
    pack_xt_kernel<<<pgrid, 256, 0, st>>>(X, ldx, rows, n, s->xinv_c, jt, s->Kt2,
                                          (uint4*)s->xtp[0], q2parts);
    count_launch();
  }
  reduce_parts(q2parts, pgrid, 1, s->xq2, st);
  if (cudaGetLastError() != cudaSuccess) {
    tc_destroy(s);
    return 1;
  }
  *out = s;
  return 0;
}

// Packed factor block of rp (<= 128) padded columns: plane q of stage kt at
// fp[0] + (kt * PLANES + q) * rp * BK.
static int8_t* fplane(TcState* s, int q, int rp) { return s->fp[0] + (size_t)q * rp * BK; }

template <typename T>
static void pack_factor(TcState* s, const T* F, int64_t ldf, int64_t K, int64_t Kt, int ncols,
                        int rp, cudaStream_t st, const unsigned long long* premax = nullptr) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(pack_factor_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(BK * 129 * sizeof(T)));
    attr = true;
  }
  if (!premax) {                  // column maxima not provided by the producing kernel
    cudaMemsetAsync(s->fmaxbits, 0, sizeof(unsigned long long) * ncols, st);
    colmax_kernel<T><<<2 * s->sms, 256, 0, st>>>(F, ldf, K, ncols, s->fmaxbits);
    count_launch();
  }
  scales_kernel<<<1, 128, 0, st>>>(premax ? premax : s->fmaxbits, ncols, s->fscale,
                                   s->colscale);
  pack_factor_kernel<T><<<(int)std::min<int64_t>(Kt, 8 * s->sms), 256, BK * 129 * sizeof(T), st>>>(
      F, ldf, K, ncols, rp, s->fscale, Kt, (uint4*)fplane(s, 0, rp));
  count_launch(2);
}

static int launch_gemm(TcState* s, int mode, bool pair, double* out, int64_t out_ld,
                       int64_t split_stride, int tiles, int ksplit, int stages_total,
                       int64_t out_rows, int ncols, int rp, cudaStream_t st,
                       unsigned* band_ready = nullptr, unsigned long long* tstamp = nullptr,
                       int tile0 = 0, int64_t row0 = 0) {
  Params p;
  p.tile0 = pair ? 0 : tile0;    // band ranges: single-CTA kernel only
  p.row0 = pair ? 0 : row0;
  if (pair && (tile0 != 0 || row0 != 0)) return 1;
  p.band_ready = (mode == 0 && ksplit == 1 && !pair) ? band_ready : nullptr;
  p.tstamp = pair ? nullptr : tstamp;
  for (int q = 0; q < PLANES; ++q) {
    p.xp[q] = s->xp[q];
    p.xtp[q] = s->xtp[q];
    p.fp[q] = fplane(s, q, rp);
  }
  p.tiles_per_row_t = s->Kt2;
  p.out = out;
  p.out_ld = out_ld;
  p.split_stride = split_stride;
  p.colscale = s->colscale;
  p.rowinv = mode == 0 ? s->xinv_r : s->xinv_c;
  p.mode = mode;
  p.tiles = tiles;
  p.num_units = (pair ? (tiles + 1) / 2 : tiles) * ksplit;
  p.ksplit = ksplit;
  p.stages_total = stages_total;
  p.tiles_per_row = s->tiles_per_row;
  p.rp = rp;
  p.r = ncols;
  p.out_rows = out_rows;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tc_i8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    cudaFuncSetAttribute(tc_i8_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         PAIR_SMEM);
    attr = true;
  }
  if (pair) {
    const int grid = 2 * std::min(p.num_units, s->sms / 2);
    tc_i8_pair_kernel<<<grid, THREADS, PAIR_SMEM, st>>>(p);
  } else {
    const int grid = std::min(p.num_units, s->sms);
    tc_i8_kernel<<<grid, THREADS, SMEM_BYTES, st>>>(p);
  }
  count_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

// band flags: Mt counters, then the epoch (flagged passes so far) and a tile counter for the
// consumer's dynamic schedule
__global__ void band_epoch_kernel(unsigned* flags, int64_t Mt) {
  flags[Mt] += 1u;
  flags[Mt + 1] = 0u;
}

unsigned* tc_band_flags(TcState* s, cudaStream_t st) {
  if (s->pair || s->ksplit1 != 1) return nullptr;
  if (!s->band_flags) {
    if (cudaMalloc(&s->band_flags, sizeof(unsigned) * (s->Mt + 2)) != cudaSuccess) {
      s->band_flags = nullptr;
      cudaGetLastError();
      return nullptr;
    }
    if (cudaMemsetAsync(s->band_flags, 0, sizeof(unsigned) * (s->Mt + 2), st) != cudaSuccess)
      return nullptr;
  }
  band_epoch_kernel<<<1, 1, 0, st>>>(s->band_flags, s->Mt);
  count_launch();
  return s->band_flags;
}

int64_t tc_bands(const TcState* s) { return s ? s->Mt : 0; }

// pass-1 device time from the kernel's own timestamps: {start, end, accumulated ns, count}
__global__ void stamp_accum_kernel(unsigned long long* ts) {
  if (ts[1] > ts[0]) {
    ts[2] += ts[1] - ts[0];
    ts[3] += 1ull;
  }
  ts[0] = ~0ull;
  ts[1] = 0ull;
}

static int ensure_stamps(TcState* s) {
  if (s->stamps) return 0;
  if (cudaMalloc(&s->stamps, 4 * sizeof(unsigned long long)) != cudaSuccess) return 1;
  const unsigned long long init[4] = {~0ull, 0ull, 0ull, 0ull};
  return cudaMemcpy(s->stamps, init, sizeof(init), cudaMemcpyHostToDevice) == cudaSuccess ? 0 : 1;
}

int tc_stamp_accum(TcState* s, cudaStream_t st) {
  if (!s->stamps) return 0;
  stamp_accum_kernel<<<1, 1, 0, st>>>(s->stamps);
  count_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int tc_stamp_read(TcState* s, double* ms, int64_t* count) {
  *ms = 0.0;
  *count = 0;
  if (!s || !s->stamps) return 0;
  unsigned long long h[4];
  if (cudaMemcpy(h, s->stamps, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
  *ms = (double)h[2] * 1e-6;
  *count = (int64_t)h[3];
  const unsigned long long init[4] = {~0ull, 0ull, 0ull, 0ull};
  return cudaMemcpy(s->stamps, init, sizeof(init), cudaMemcpyHostToDevice) == cudaSuccess ? 0 : 1;
}

int tc_xv(TcState* s, const float* V, int64_t ldv, double* P, cudaStream_t st,
          const unsigned long long* vmax, unsigned* band_ready, bool stamp) {
  if (stamp && ensure_stamps(s)) return 1;
  // B = V (K = n), over all 64-column stages of X
  const int r = (int)s->r;
  pack_factor<float>(s, V, ldv, s->n, s->tiles_per_row, r, s->rp, st, vmax);
  const bool pair = s->pair;
  const int ks = pair ? s->ksplit1p : s->ksplit1;
  if (ks == 1)
    return launch_gemm(s, 0, pair, P, r, 0, (int)s->Mt, 1, (int)s->tiles_per_row, s->rows, r,
                       s->rp, st, band_ready, stamp ? s->stamps : nullptr);
  if (launch_gemm(s, 0, pair, s->partial, r, s->rows * r, (int)s->Mt, ks, (int)s->tiles_per_row,
                  s->rows, r, s->rp, st))
    return 1;
  reduce_parts(s->partial, ks, s->rows * r, P, st);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int tc_xtu(TcState* s, const float* U, int64_t ldu, double* Q, cudaStream_t st,
           const unsigned long long* umax) {
  // B = U (K = rows of X), split-K partials reduced in a fixed order
  const int r = (int)s->r;
  pack_factor<float>(s, U, ldu, s->rows, s->Kt2, r, s->rp, st, umax);
  const int mode = s->xtp[0] ? 2 : 1;
  const bool pair = s->pair && mode == 2;   // the pair kernel reads K-major A only
  const int ks = pair ? s->ksplit2p : s->ksplit2;
  if (launch_gemm(s, mode, pair, s->partial, r, s->n * r, (int)(s->tiles_per_row / 2), ks,
                  (int)s->Kt2, s->n, r, s->rp, st))
    return 1;
  reduce_parts(s->partial, ks, s->n * r, Q, st);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

// ------------------------------------------------------------------ quantised Gram
// G = U~^T U~ of the factor digits the last pass packed (the Gram the trace-form objective
// and the V update use, tc_factor_scales), EXACTLY, on the tensor cores.  A packed K-stage
// (64 factor rows x rp columns, 3 digit planes, K-major, core matrix (g, kc) at
// (4 g + kc) 128 B) serves as both operands: A = U~^T (M = rp rows of the Gram) and B = U~
// (N = rp), so every digit product d_i(u_k) d_j(u_l) of the stage is one kind::i8 MMA.  The
// digit weights 2^15, 2^7, 1 (mixed radix 8/8/7) give six product weights; TMEM holds four
// 128-column accumulators, so PHASE 0 accumulates 2^30 | 2^22 | 2^14 | 2^15 (products 00 |
// 01+10 | 11 | 02+20, the X passes' MMA list) and PHASE 1 2^7 | 1 (12+21 | 22).  Each CTA
// takes a contiguous K range (<= 65536 rows: |class| < 2^31), combines its classes into one
// int64 per entry (< 2^62) and adds it to the global int64 Gram with atomics (exact, order
// independent); gram_finish_kernel scales by 2^-30 / (s_k s_l).  Replaces gram_sym's fp64
// SIMT accumulation of the quantised factor (0.36 ms at C5, ~0.03 ms here).
constexpr int GRAM_STAGE = PLANES * 128 * BK;      // 24 KB at rp = 128

template <int PHASE>
__global__ void __launch_bounds__(128, 1)
tc_gram_kernel(const int8_t* __restrict__ planes, int64_t Kt, int rp, int per,
               unsigned long long* __restrict__ G64) {
  extern __shared__ __align__(1024) uint8_t gsm_raw[];
  uint8_t* gsm = (uint8_t*)(((uintptr_t)gsm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bars[5];
  __shared__ uint32_t tmem_base_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ks0 = (int64_t)blockIdx.x * per, ks1 = ks0 + per < Kt ? ks0 + per : Kt;
  const uint32_t bar_full[2] = {smem_u32(&bars[0]), smem_u32(&bars[1])};
  const uint32_t bar_mma[2] = {smem_u32(&bars[2]), smem_u32(&bars[3])};
  const uint32_t bar_done = smem_u32(&bars[4]);
  const uint32_t stage_bytes = (uint32_t)PLANES * rp * BK;
  if (threadIdx.x == 0) {
    for (int b = 0; b < 5; ++b) mbar_init(smem_u32(&bars[b]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_s)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_s;
  const uint32_t lane_addr = tmem_base + ((uint32_t)(32 * warp) << 16);
  if (PHASE == 0) {   // accumulator 2 is only ever accumulated into (wide A1 [B0;B1])
#pragma unroll 1
    for (int c0 = 0; c0 < rp; c0 += 16) TMEM_ST16_ZERO(lane_addr + 2 * rp + c0);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0 && ks1 > ks0) {
    const uint32_t base = smem_u32(gsm);
    const uint32_t idesc_base = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BM >> 4) << 24);
    const uint32_t idesc1 = idesc_base | ((uint32_t)(rp >> 3) << 17);
    const uint32_t idesc2 = idesc_base | ((uint32_t)(2 * rp >> 3) << 17);
    const uint32_t plane = (uint32_t)rp * BK;
    auto load = [&](int64_t ks, int slot) {
      mbar_expect_tx(bar_full[slot], stage_bytes);
      bulk_g2s(base + slot * GRAM_STAGE, planes + ks * stage_bytes, stage_bytes, bar_full[slot]);
    };
    load(ks0, 0);
    for (int64_t ks = ks0; ks < ks1; ++ks) {
      const int i = (int)(ks - ks0), slot = i & 1;
      if (ks + 1 < ks1) {
        if (i >= 1) mbar_wait(bar_mma[slot ^ 1], ((i - 1) >> 1) & 1);   // slot free again
        load(ks + 1, slot ^ 1);
      }
      mbar_wait(bar_full[slot], (i >> 1) & 1);
      tc_fence_after();
      const uint32_t st = base + slot * GRAM_STAGE;
#pragma unroll
      for (int j = 0; j < BK / 32; ++j) {
        const bool first = ks == ks0 && j == 0;
        auto mma = [&](int pa, int pb, int acc, bool wide, bool fresh) {
          const uint64_t ad = umma_desc(st + pa * plane + j * 256, 128, 512);
          const uint64_t bd = umma_desc(st + pb * plane + j * 256, 128, 512);
          tc_mma_i8(tmem_base + acc * rp, ad, bd, wide ? idesc2 : idesc1, fresh ? 0u : 1u);
        };
        if (PHASE == 0) {
          mma(0, 0, 0, true, first);    // 00 -> acc0, 01 -> acc1
          mma(0, 2, 3, false, first);   // 02 -> acc3
          mma(2, 0, 3, false, false);   // 20 -> acc3
          mma(1, 0, 1, true, false);    // 10 -> acc1, 11 -> acc2 (zeroed above)
        } else {
          mma(1, 2, 0, false, first);   // 12 -> acc0
          mma(2, 1, 0, false, false);   // 21 -> acc0
          mma(2, 2, 1, false, first);   // 22 -> acc1
        }
      }
      tc_commit(bar_mma[slot]);
    }
    tc_commit(bar_done);
  }
  __syncwarp();
  if (ks1 > ks0) {
    mbar_wait_sleep(bar_done, 0);
    tc_fence_after();
    const int k = 32 * warp + lane;            // Gram row (TMEM lane)
#pragma unroll 1
    for (int c0 = 0; c0 < rp; c0 += 16) {
      uint32_t v[4][16];
      TMEM_LD16(lane_addr + 0 * rp + c0, v[0]);
      TMEM_LD16(lane_addr + 1 * rp + c0, v[1]);
      if (PHASE == 0) {
        TMEM_LD16(lane_addr + 2 * rp + c0, v[2]);
        TMEM_LD16(lane_addr + 3 * rp + c0, v[3]);
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (k < rp) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          long long val;
          if (PHASE == 0)
            val = ((long long)(int)v[0][i] << 30) + ((long long)(int)v[1][i] << 22) +
                  ((long long)(int)v[2][i] << 14) + ((long long)(int)v[3][i] << 15);
          else
            val = ((long long)(int)v[0][i] << 7) + (long long)(int)v[1][i];
          if (val != 0)
            atomicAdd(&G64[(int64_t)k * rp + c0 + i], (unsigned long long)val);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
  }
}

// G (r x r fp64) = G64 2^-30 / (s_k s_l): colscale holds 1 / s of the factor's columns
__global__ void gram_finish_kernel(const unsigned long long* __restrict__ G64, int r, int rp,
                                   const double* __restrict__ colscale, double* __restrict__ G) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < r * r; e += gridDim.x * blockDim.x) {
    const int k = e / r, l = e % r;
    G[e] = (double)(long long)G64[(int64_t)k * rp + l] * 0x1p-30 * colscale[k] * colscale[l];
  }
}

int tc_gram_quantised(TcState* s, double* G, cudaStream_t st) {
  const int rp = s->rp, r = (int)s->r;
  if (rp != 128 && rp % 16 != 0) return 1;
  const int64_t Kt = s->Kt2;
  // <= 1024 stages (65536 rows) per CTA keeps every class below 2^31; the int64 total below
  // 2^63 needs rows < 2^63 / (126 2^15)^2, i.e. m < 5.2e5 per rank (else: SIMT path)
  int grid = (int)std::min<int64_t>(Kt, s->sms);
  int per = (int)((Kt + grid - 1) / grid);
  if (per > 1024 || s->rows > 500000) return 2;
  grid = (int)((Kt + per - 1) / per);
  if (!s->gram64) {
    if (cudaMalloc(&s->gram64, sizeof(unsigned long long) * 128 * 128) != cudaSuccess) {
      cudaGetLastError();
      return 1;
    }
  }
  static bool attr = false;
  const int smem = 2 * GRAM_STAGE + 1024;
  if (!attr) {
    cudaFuncSetAttribute(tc_gram_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(tc_gram_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  if (cudaMemsetAsync(s->gram64, 0, sizeof(unsigned long long) * 128 * 128, st) != cudaSuccess)
    return 1;
  const int8_t* planes = fplane(s, 0, rp);
  tc_gram_kernel<0><<<grid, 128, smem, st>>>(planes, Kt, rp, per, s->gram64);
  tc_gram_kernel<1><<<grid, 128, smem, st>>>(planes, Kt, rp, per, s->gram64);
  gram_finish_kernel<<<(r * r + 255) / 256, 256, 0, st>>>(s->gram64, r, rp, s->colscale, G);
  count_launch(3);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

// Q rows of the 128-column bands [b0, b1) of X (pass 2 over a band range: the chunks of the
// multi-rank V block, each reduced to its owner while the next one runs).  pack: repack the
// factor's digits (the first range of a pass).  The K split fills the SMs for the range alone
// (a chunk has few bands); its partials live in a range-sized buffer.
int tc_xtu_bands(TcState* s, const float* U, int64_t ldu, double* Q, int64_t b0, int64_t b1,
                 cudaStream_t st, const unsigned long long* umax, bool pack) {
  const int r = (int)s->r;
  const int64_t bands = s->tiles_per_row / 2;
  if (b0 < 0 || b1 > bands || b0 >= b1) return 1;
  if (pack) pack_factor<float>(s, U, ldu, s->rows, s->Kt2, r, s->rp, st, umax);
  const int mode = s->xtp[0] ? 2 : 1;
  const int64_t row0 = b0 * BM, rows = std::min<int64_t>(s->n, b1 * BM) - row0;
  const int nb = (int)(b1 - b0);
  const int ks = choose_split_waves(nb, s->Kt2, s->sms);
  if (ks == 1)
    return launch_gemm(s, mode, false, Q, r, 0, nb, 1, (int)s->Kt2, s->n, r, s->rp, st, nullptr,
                       nullptr, (int)b0, 0);
  const size_t need = (size_t)ks * rows * r;
  if (need > s->chunk_cap) {
    if (s->chunk_partial) cudaFree(s->chunk_partial);
    s->chunk_partial = nullptr;
    s->chunk_cap = 0;
    if (cudaMalloc(&s->chunk_partial, sizeof(double) * need) != cudaSuccess) {
      cudaGetLastError();
      return 2;
    }
    s->chunk_cap = need;
  }
  if (launch_gemm(s, mode, false, s->chunk_partial, r, rows * r, nb, ks, (int)s->Kt2, s->n, r,
                  s->rp, st, nullptr, nullptr, (int)b0, row0))
    return 1;
  reduce_parts(s->chunk_partial, ks, rows * r, Q + row0 * r, st);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int64_t tc_xtu_band_count(const TcState* s) { return s ? s->tiles_per_row / 2 : 0; }

int tc_xf(TcState* s, bool transposed, const double* F, int64_t ldf, int ncols, double* out,
          int64_t ldo, cudaStream_t st) {
  const int64_t out_rows = transposed ? s->n : s->rows;
  if (!s->colbuf) {
    if (cudaMalloc(&s->colbuf, sizeof(double) * std::max(s->rows, s->n) * 128) != cudaSuccess) {
      cudaGetLastError();
      s->colbuf = nullptr;
      return 2;
    }
  }
  for (int c0 = 0; c0 < ncols; c0 += 128) {
    const int nb = std::min(128, ncols - c0);
    const int rp = (nb + 15) / 16 * 16;
    int mode, tiles, ks, stages;
    if (!transposed) {
      pack_factor<double>(s, F + c0, ldf, s->n, s->tiles_per_row, nb, rp, st);
      mode = 0;
      tiles = (int)s->Mt;
      ks = s->ksplit1;
      stages = (int)s->tiles_per_row;
    } else {
      pack_factor<double>(s, F + c0, ldf, s->rows, s->Kt2, nb, rp, st);
      mode = s->xtp[0] ? 2 : 1;
      tiles = (int)(s->tiles_per_row / 2);
      ks = s->ksplit2;
      stages = (int)s->Kt2;
    }
    if (ks == 1) {
      if (launch_gemm(s, mode, false, out + c0, ldo, 0, tiles, 1, stages, out_rows, nb, rp, st))
        return 1;
      continue;
    }
    if (launch_gemm(s, mode, false, s->partial, nb, out_rows * nb, tiles, ks, stages, out_rows,
                    nb, rp, st))
      return 1;
    reduce_parts(s->partial, ks, out_rows * nb, s->colbuf, st);
    scatter_cols_kernel<<<2 * s->sms, 256, 0, st>>>(s->colbuf, out_rows, nb, out, ldo, c0);
    count_launch();
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace enmf
