// tc_pbcd.cu -- Alg. 2 PBCD on the tensor cores, for the tensor-core path.
//
// Per inner iteration every row i of a block needs two r x r products with the fixed Gram G:
//   grad_i = u_i G - c_i            (the masked gradient, Eq.(8) / line 241)
//   h_i    = g_i G,  g = M o grad   (the Eq.(10) denominator ||g V^T||^2 = g G g^T)
// i.e. 2 r^2 MACs per row-iteration -- 33 GFMA per U block at C5, 50 iterations.  The SIMT fp64
// kernel (kernels_rows.cu) is bound by the fp64 pipe; here a CTA holds a 128-row tile and runs
// all max_iter iterations with both products as exact int8-digit tcgen05 MMAs (same 4-digit,
// 4-class scheme as tc_gemm.cu: A = digits of u or g with a power-of-two scale per row, B =
// digits of G with a power-of-two scale per column, 4 exact int32 TMEM accumulators, combined
// exactly in fp64).  u stays in fp64 registers; g is never stored: it is rebuilt from its digit
// planes in shared memory, which represent it to 2^-22 of its row maximum.
//
// Warp roles: 8 warps, thread (row, half) owns 64 columns of one row (TMEM lane quadrant =
// warp % 4, column half = warp / 4).  Warp 0 allocates TMEM; thread 0 issues each round's MMAs
// after the named barrier that publishes the A planes (a ninth, issuer-only warp would cap the
// register file at 168 per thread and spill the 64 fp64 row values).
// Everything else follows pbcd_kernel: lift + mask at entry, a snapshot of every iterate, and the
// per-iteration ||M o grad||^2 partials for the global stopping rule (pbcd_select / pbcd_copy).
#include <float.h>
#include <math.h>
#include <stdint.h>

#include "internal.h"
#include "tc_ptx.cuh"

namespace enmf {
namespace tpb {

using namespace tcp;

constexpr int BM = 128;
constexpr int COMPUTE_WARPS = 8;
constexpr int THREADS = 32 * COMPUTE_WARPS;   // 8 warps: 255 registers per thread available
constexpr int KR = 128;                     // K (= r) padded to the MMA depth multiple
constexpr int PLANE_A = BM * KR;            // 16 KB
constexpr int PLANE_B = 128 * KR;           // 16 KB (G padded to 128 rows)
constexpr int CQ_LD = KR + 1;               // padded row stride (words): conflict-free row reads
constexpr int CQ_BYTES = BM * CQ_LD * 4;    // the tile's c rows as int32 fixed point
constexpr int SMEM_BYTES = 4 * PLANE_A + 4 * PLANE_B + CQ_BYTES;

struct Params {
  const float* F;
  int64_t ldf;
  int64_t rows;
  int r, rp;
  const double* C;           // rows x r, ld r
  const int8_t* gd;          // 4 planes of G digits, each rp x KR (B operand layout)
  const double* gscale;      // r: 1 / t_j
  const double* lam;
  int max_iter;
  float* snaps;
  double* pgparts;           // gridDim x (max_iter + 1)
  const int* stage;
};

__device__ __forceinline__ double pow2s(double mx) {
  if (!(mx > 0.0)) return 1.0;
  int e;
  frexp(mx, &e);
  return ldexp(1.0, 6 - e);
}

// pow2s from the high word of |x| (sign masked): only the exponent matters, so the maximum of
// the high words of a row selects the same power of two as pow2s(max |x|).  Zero / subnormal
// rows get 1 (their digits are zero anyway at 2^-22 resolution).
__device__ __forceinline__ int hiabs(double x) { return __double2hiint(x) & 0x7fffffff; }
__device__ __forceinline__ double pow2s_hi(int h) {
  if (h < 0x00100000) return 1.0;
  const int E = h >> 20;                       // biased exponent; frexp exponent e = E - 1022
  return __hiloint2double((2051 - E) << 20, 0); // 2^(6 - e)
}
// The 4 weight classes of an accumulator column combined exactly: v0 2^21 + v1 2^14 + v2 2^7 + v3
// (< 2^53, so the conversion to double is exact); callers fold 2^-21 into their scales.
__device__ __forceinline__ double comb4(uint32_t v0, uint32_t v1, uint32_t v2, uint32_t v3) {
  const long long a = (long long)(int)v0 * 2097152ll + (long long)(int)v1 * 16384ll +
                      (long long)(int)v2 * 128ll + (long long)(int)v3;
  return (double)a;
}

__device__ __forceinline__ void bar_compute() {
  asm volatile("bar.sync 1, %0;" ::"n"(32 * COMPUTE_WARPS) : "memory");
}

// digits_word(t): tc_ptx.cuh
struct Pack16 { uint32_t w[4][4]; };   // [plane][word]: 16 columns of the 4 digit planes
__device__ __forceinline__ void pack_put(Pack16& pk, int k, uint32_t dw) {
#pragma unroll
  for (int pl = 0; pl < 4; ++pl) pk.w[pl][k >> 2] |= ((dw >> (8 * pl)) & 255u) << (8 * (k & 3));
}
__device__ __forceinline__ void pack_clear(Pack16& pk) {
#pragma unroll
  for (int pl = 0; pl < 4; ++pl)
#pragma unroll
    for (int q = 0; q < 4; ++q) pk.w[pl][q] = 0u;
}
__device__ __forceinline__ void pack_store(const Pack16& pk, uint8_t* Ad, int off) {
#pragma unroll
  for (int pl = 0; pl < 4; ++pl)
    *reinterpret_cast<uint4*>(Ad + pl * PLANE_A + off) =
        make_uint4(pk.w[pl][0], pk.w[pl][1], pk.w[pl][2], pk.w[pl][3]);
}
// mask bit c of a thread's 64 columns; opaque() stops the compiler from hoisting the 64 bit
// tests out of the iteration loop (they would occupy 64 registers)
__device__ __forceinline__ bool mbit(uint32_t lo, uint32_t hi, int c) {
  return ((c < 32 ? lo >> c : hi >> (c - 32)) & 1u) != 0u;
}
__device__ __forceinline__ void opaque(uint32_t& a, uint32_t& b) {
  asm volatile("" : "+r"(a), "+r"(b));
}
__device__ __forceinline__ int digit_at(const uint4& v, int k) {
  const uint32_t w = (k >> 2) == 0 ? v.x : ((k >> 2) == 1 ? v.y : ((k >> 2) == 2 ? v.z : v.w));
  return (int)(int8_t)(uint8_t)(w >> (8 * (k & 3)));
}
// the value the digit planes hold for column k of a 16-column chunk (exact)
__device__ __forceinline__ double rebuild(const uint4 (&dq)[4], int k) {
  const int n = (digit_at(dq[0], k) << 21) + (digit_at(dq[1], k) << 14) +
                (digit_at(dq[2], k) << 7) + digit_at(dq[3], k);
  return (double)n * 0x1p-21;
}

// The 4-class digit products of one round as 6 MMAs (see tc_gemm.cu MmaList<4>), issued by one
// thread after the named barrier that publishes the A planes; completion arrives on bar_d.
__device__ __forceinline__ void issue_round(uint32_t a0, uint32_t b0, uint32_t tmem_base, int rp,
                                            int r, uint32_t bar_d) {
  const uint32_t idesc_base = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BM >> 4) << 24);
  const uint32_t idesc1 = idesc_base | ((uint32_t)(rp >> 3) << 17);
  const uint32_t idesc2 = idesc_base | ((uint32_t)(2 * rp >> 3) << 17);
  const uint32_t a_lbo = 2048, a_sbo = 128, a_kstep = 4096;
  const uint32_t b_lbo = 128, b_sbo = 8 * KR, b_kstep = 256;
  const int ksteps = (r + 31) / 32;
  constexpr int tab[6][4] = {{0, 0, 0, 1}, {0, 2, 2, 1}, {1, 0, 1, 1},
                             {1, 2, 3, 0}, {2, 0, 2, 1}, {3, 0, 3, 0}};
  tc_fence_after();
  for (int j = 0; j < ksteps; ++j) {
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      const uint64_t ad = umma_desc(a0 + tab[q][0] * PLANE_A + j * a_kstep, a_lbo, a_sbo);
      const uint64_t bd = umma_desc(b0 + tab[q][1] * rp * KR + j * b_kstep, b_lbo, b_sbo);
      tc_mma_i8(tmem_base + tab[q][2] * rp, ad, bd, tab[q][3] ? idesc2 : idesc1,
                (j == 0 && q < 2) ? 0u : 1u);
    }
  }
  tc_commit(bar_d);
}

__global__ void __launch_bounds__(THREADS, 1) tc_pbcd_kernel(const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;                  // no-swizzle operands need 16-byte alignment only
  uint8_t* Ad = smem;                        // 4 planes of A digits (128 x KR, K-major)
  uint8_t* Bd = smem + 4 * PLANE_A;          // 4 planes of G digits (rp x KR, K-major)
  __shared__ __align__(8) uint64_t bars[1];
  __shared__ uint32_t tmem_base_s;
  __shared__ double xch[2][BM];              // row exchange between the two column halves
  __shared__ int xchi[2][BM];
  __shared__ double xch2[2][BM];
  __shared__ double wsum[COMPUTE_WARPS];
  __shared__ double gsc_s[128];
  if (p.stage != nullptr && *p.stage != 0) return;
  // 2^-21 / t_j: the column scale with comb4's 2^-21 folded in (exact)
  for (int j = threadIdx.x; j < 128; j += blockDim.x)
    gsc_s[j] = j < p.r ? p.gscale[j] * 0x1p-21 : 0.0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bar_d = smem_u32(&bars[0]);     // MMA -> all warps: accumulators ready
  constexpr int rp = KR;                         // G padded to 128 columns (p.rp == KR)
  const int tiles = (int)((p.rows + BM - 1) / BM);
  int32_t* Cq = reinterpret_cast<int32_t*>(Bd + 4 * PLANE_B);    // c tile, fixed point per row
  double* pgsm = reinterpret_cast<double*>(Bd + 4 * PLANE_B + CQ_BYTES);   // max_iter + 1 sums

  // G digits -> shared memory (once per CTA); zero the A planes' padding once
  for (int e = threadIdx.x; e < 4 * rp * KR / 16; e += blockDim.x)
    reinterpret_cast<uint4*>(Bd)[e] = reinterpret_cast<const uint4*>(p.gd)[e];
  for (int e = threadIdx.x; e < 4 * PLANE_A / 16; e += blockDim.x)
    reinterpret_cast<uint4*>(Ad)[e] = make_uint4(0, 0, 0, 0);
  for (int e = threadIdx.x; e <= p.max_iter; e += blockDim.x) pgsm[e] = 0.0;
  if (threadIdx.x == 0) {
    mbar_init(bar_d, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
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
  const uint32_t a_s = smem_u32(Ad), b_s = smem_u32(Bd);

  {
    // ===================== compute warps =====================
    const int w = warp;
    const int q = warp & 3;                    // TMEM lane quadrant
    const int hc = warp >> 2;                  // column half
    const int rt = 32 * q + lane;              // row in tile
    const int c0 = 64 * hc;
    // my TMEM lane quadrant and column half; class k of the accumulators at column k * KR
    const uint32_t tcol = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)c0;
    const double lam = *p.lam;
    const int64_t snap_stride = p.rows * (int64_t)p.r;
    const int g8 = rt >> 3, ri = rt & 7;
    // my 16-byte digit chunks in the A planes: chunk b of my half at abase + b * 16 * 128
    uint8_t* const abase = Ad + ((c0 >> 4) * 16 + g8) * 128 + ri * 16;
    uint32_t round = 0;
    const double* gsc = gsc_s + c0;            // 1 / t_j for my columns (shared memory)

    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      const int64_t row = (int64_t)t * BM + rt;
      const bool rok = row < p.rows;
      double u[64];
      uint32_t mlo = 0, mhi = 0;   // M_{U+} bits of my 64 columns
#pragma unroll
      for (int c = 0; c < 64; ++c) {
        const int col = c0 + c;
        double v = (rok && col < p.r) ? (double)p.F[row * p.ldf + col] : 0.0;
        if (v < 0.0) v += lam;                                     // Eq.(6)/(7) lift
        u[c] = v;
        if (rok && col < p.r && v >= 0.0) {                        // M_{U+} (R14)
          if (c < 32) mlo |= 1u << c; else mhi |= 1u << (c - 32);
        }
      }
      // c_i (row of P or Q) -> shared memory as int32 fixed point with a power-of-two row scale:
      // c = cq * csc, |error| <= 2^-27 max_j |c_ij| (the same resolution as the u / g digits)
      double cs;
      {
        const double* crow = p.C + row * p.r;
        double cm = 0.0;
        for (int c = 0; c < 64; ++c)
          if (rok && c0 + c < p.r) cm = fmax(cm, fabs(crow[c0 + c]));
        xch2[hc][rt] = cm;
        bar_compute();
        const double sc = pow2s(fmax(cm, xch2[1 - hc][rt]));
        cs = 0x1p-21 / sc;
        for (int c = 0; c < 64; ++c)
          Cq[rt * CQ_LD + c0 + c] =
              (rok && c0 + c < p.r) ? __double2int_rn(crow[c0 + c] * sc * 0x1p21) : 0;
      }
      const int32_t* cqrow = Cq + rt * CQ_LD + c0;
      for (int it = 0; it <= p.max_iter; ++it) {
        // ---------------- round A: T1 = u G ----------------
        int mh = 0;
#pragma unroll
        for (int c = 0; c < 64; ++c) mh = max(mh, hiabs(u[c]));
        xchi[hc][rt] = mh;
        bar_compute();
        const double su = pow2s_hi(max(mh, xchi[1 - hc][rt]));
        // digits of u * su into the A planes: chunk (kc, g8, ri), 16 columns each
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          Pack16 pk;
          pack_clear(pk);
#pragma unroll
          for (int k = 0; k < 16; ++k) pack_put(pk, k, digits_word(u[16 * ch + k] * su));
          pack_store(pk, abase, ch * 16 * 128);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        bar_compute();
        if (threadIdx.x == 0) issue_round(a_s, b_s, tmem_base, rp, p.r, bar_d);
        mbar_wait(bar_d, round & 1);
        ++round;
        tc_fence_after();
        // pass 1: grad = T1 / su - c ; ||M o grad||^2 (pg of iteration it), num, max|g|
        double num = 0.0;
        int gmh = 0;
        opaque(mlo, mhi);
        const double isu = 1.0 / su;
#pragma unroll 1
        for (int b = 0; b < 8; ++b) {       // rolled: keeps the kernel inside the icache
          uint32_t v[4][8];
#pragma unroll
          for (int cls = 0; cls < 4; ++cls) TMEM_LD8(tcol + cls * KR + 8 * b, v[cls]);
          const uint32_t mb = ((b < 4 ? mlo : mhi) >> (8 * (b & 3))) & 255u;
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int c = 8 * b + k;
            const double a = comb4(v[0][k], v[1][k], v[2][k], v[3][k]);
            const double gr = a * isu * gsc[c] - (double)cqrow[c] * cs;
            const double gm = ((mb >> k) & 1u) ? gr : 0.0;     // M o grad
            num = fma(gm, gm, num);
            gmh = max(gmh, hiabs(gm));
          }
        }
        // per-iteration partial of ||M o grad||^2 (fixed-order block reduction)
        double pg = num;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) pg += __shfl_xor_sync(0xffffffffu, pg, o);
        if (lane == 0) wsum[w] = pg;
        xchi[hc][rt] = gmh;
        xch2[hc][rt] = num;
        bar_compute();
        if (threadIdx.x == 32) {
          double s = 0.0;
          for (int k = 0; k < COMPUTE_WARPS; ++k) s += wsum[k];
          pgsm[it] += s;
        }
        if (it == p.max_iter) {
          tc_fence_before();
          // the final round A has no round B; TMEM reads finish before the next tile's MMAs
          bar_compute();
          break;
        }
        const double numr = hc == 0 ? num + xch2[1][rt] : xch2[0][rt] + num;
        const double sg = pow2s_hi(max(gmh, xchi[1 - hc][rt]));
        // pass 2: digits of g * sg (g = M o grad) into the A planes (T1 re-read from TMEM)
        opaque(mlo, mhi);
#pragma unroll 1
        for (int b = 0; b < 4; ++b) {
          Pack16 pk;
          pack_clear(pk);
          const uint32_t mb = ((b < 2 ? mlo : mhi) >> (16 * (b & 1))) & 65535u;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            uint32_t v[4][8];
#pragma unroll
            for (int cls = 0; cls < 4; ++cls) TMEM_LD8(tcol + cls * KR + 16 * b + 8 * h, v[cls]);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int c = 16 * b + 8 * h + k;
              const double a = comb4(v[0][k], v[1][k], v[2][k], v[3][k]);
              const double gr = a * isu * gsc[c] - (double)cqrow[c] * cs;
              const double g = ((mb >> (8 * h + k)) & 1u) ? gr : 0.0;
              pack_put(pk, 8 * h + k, digits_word(g * sg));
            }
          }
          pack_store(pk, abase, b * 16 * 128);
        }
        tc_fence_before();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        bar_compute();
        if (threadIdx.x == 0) issue_round(a_s, b_s, tmem_base, rp, p.r, bar_d);
        // ---------------- round B: T2 = g G ----------------
        mbar_wait(bar_d, round & 1);
        ++round;
        tc_fence_after();
        // den = sum_j g_j h_j with g = rebuild / sg, h = T2 gsc / sg: accumulate rebuild * T2 gsc
        // and apply the exact power-of-two 1 / sg^2 once
        double den = 0.0;
        const double isg = 1.0 / sg;
#pragma unroll 1
        for (int b = 0; b < 4; ++b) {
          uint4 dq[4];
#pragma unroll
          for (int pl = 0; pl < 4; ++pl)
            dq[pl] = *reinterpret_cast<const uint4*>(abase + pl * PLANE_A + b * 16 * 128);
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            uint32_t v[4][8];
#pragma unroll
            for (int cls = 0; cls < 4; ++cls) TMEM_LD8(tcol + cls * KR + 16 * b + 8 * hh, v[cls]);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int c = 16 * b + 8 * hh + k;
              const double a = comb4(v[0][k], v[1][k], v[2][k], v[3][k]);
              den = fma(rebuild(dq, 8 * hh + k), a * gsc[c], den);
            }
          }
        }
        den *= isg * isg;
        tc_fence_before();
        xch[hc][rt] = den;
        bar_compute();
        const double denr = hc == 0 ? den + xch[1][rt] : xch[0][rt] + den;
        // Eq.(10): d_i = ||g_i||^2 / ||g_i V^T||^2 (0 on a zero denominator, R10); Eq.(8)
        const double dstep = denr > 0.0 ? numr / denr : 0.0;
        opaque(mlo, mhi);
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          uint4 dq[4];
#pragma unroll
          for (int pl = 0; pl < 4; ++pl)
            dq[pl] = *reinterpret_cast<const uint4*>(abase + pl * PLANE_A + b * 16 * 128);
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            const int c = 16 * b + k;
            const double un = fmax(0.0, u[c] - dstep * (rebuild(dq, k) * isg));
            u[c] = mbit(mlo, mhi, c) ? un : u[c];     // entries outside M_{U+} stay fixed
          }
        }
        if (rok) {
          // snapshot, tile-major (pbcd_copy_tiled_kernel): a warp's 32 rows are contiguous
          const int nt = (int)(p.rows - (int64_t)t * BM < BM ? p.rows - (int64_t)t * BM : BM);
          float* sn = p.snaps + (int64_t)it * snap_stride + (int64_t)t * BM * p.r + rt;
#pragma unroll
          for (int c = 0; c < 64; ++c)
            if (c0 + c < p.r) sn[(int64_t)(c0 + c) * nt] = (float)u[c];
        }
        bar_compute();          // everyone has read the g digits before they are overwritten
      }
    }
    bar_compute();
    if (threadIdx.x == 32)
      for (int it = 0; it <= p.max_iter; ++it)
        p.pgparts[(int64_t)blockIdx.x * (p.max_iter + 1) + it] = pgsm[it];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
  }
}

// G (r x r fp64, symmetric) -> 4 digit planes of the B operand (row j of B = column j of G,
// power-of-two scale t_j per column), layout (g * (KR/16) + kc) * 128 + ri * 16 + ki.
__global__ void gdigits_kernel(const double* __restrict__ G, int r, int rp, int8_t* gd,
                               double* gscale, const int* stage) {
  if (stage != nullptr && *stage != 0) return;
  __shared__ double t[128];
  for (int j = threadIdx.x; j < rp; j += blockDim.x) {
    double mx = 0.0;
    if (j < r)
      for (int l = 0; l < r; ++l) mx = fmax(mx, fabs(G[l * r + j]));
    t[j] = pow2s(mx);
    if (j < r) gscale[j] = 1.0 / t[j];
  }
  __syncthreads();
  const int plane = rp * KR;
  for (int e = threadIdx.x; e < rp * KR; e += blockDim.x) {
    const int j = e / KR, l = e % KR;
    const double v = (j < r && l < r) ? G[l * r + j] * t[j] : 0.0;
    const Dig4 z = digits4(v);
    const int off = ((j >> 3) * (KR / 16) + (l >> 4)) * 128 + (j & 7) * 16 + (l & 15);
#pragma unroll
    for (int pl = 0; pl < 4; ++pl) gd[pl * plane + off] = z.d[pl];
  }
}

}  // namespace tpb

int tc_pbcd_parts() { return kSMs; }

bool tc_pbcd_supported(int r) { return r >= 1 && r <= 128; }

// Same contract as pbcd_rows (kernels_rows.cu); pgparts holds gridDim x (max_iter + 1).
int tc_pbcd_rows(const float* F, int64_t ldf, int64_t rows, int r, const double* C,
                  const double* G, const double* lam, int max_iter, float* snaps,
                  double* pgparts, int8_t* gd_work, double* gscale_work, const int* stage,
                  cudaStream_t st) {
  using namespace tpb;
  const int rp = KR;   // G padded to 128 columns: class k of the accumulators at column k * 128
  gdigits_kernel<<<1, 256, 0, st>>>(G, r, rp, gd_work, gscale_work, stage);
  Params p;
  p.F = F;
  p.ldf = ldf;
  p.rows = rows;
  p.r = r;
  p.rp = rp;
  p.C = C;
  p.gd = gd_work;
  p.gscale = gscale_work;
  p.lam = lam;
  p.max_iter = max_iter;
  p.snaps = snaps;
  p.pgparts = pgparts;
  p.stage = stage;
  const size_t smem = SMEM_BYTES + sizeof(double) * (max_iter + 1);
  // the dynamic size grows with max_iter; static shared memory (row exchanges) counts against
  // the same 227 KB, so the attribute is the exact dynamic request, raised when it grows
  static size_t attr = 0;
  if (smem > attr) {
    if (cudaFuncSetAttribute(tc_pbcd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
      return 1;
    cudaFuncSetAttribute(tc_pbcd_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    attr = smem;
  }
  const int tiles = (int)((rows + BM - 1) / BM);
  const int grid = tiles < kSMs ? tiles : kSMs;
  // unused CTAs of the persistent grid still write their (zero) partials: launch kSMs always
  tc_pbcd_kernel<<<kSMs, THREADS, smem, st>>>(p);
  (void)grid;
  count_launch(2);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace enmf
