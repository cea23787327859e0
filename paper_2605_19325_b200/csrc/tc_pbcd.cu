// tc_pbcd.cu -- Alg. 2 PBCD on the tensor cores, for the tensor-core path.
//
// Per inner iteration every row i of a block needs two r x r products with the fixed Gram G:
//   grad_i = u_i G - c_i            (the masked gradient, Eq.(8) / line 241)
//   h_i    = g_i G,  g = M o grad   (the Eq.(10) denominator ||g V^T||^2 = g G g^T)
// i.e. 2 r^2 MACs per row-iteration -- 33 GFMA per U block at C5, 50 iterations.  The SIMT fp64
// kernel (kernels_rows.cu) is bound by the fp64 pipe; here a CTA holds a 128-row tile and runs
// the iterations with both products as exact int8-digit tcgen05 MMAs: A = u or g on the 2^-24
// grid of a power-of-two row scale (|t| < 64), B = G on the same grid per column, each as FOUR
// BALANCED BASE-2^8 DIGITS -- the bytes of (n + 0x808080) ^ 0x808080, n the grid integer (bdig;
// round 2b: the base-2^7 split cost ~30 integer ops per element and encoding, the byte form 2
// plus a 4 x 4 byte transpose per 4 columns) -- 10 digit products in 4 weight classes, i.e. 4
// exact int32 TMEM accumulators combined exactly in fp64 (comb8).  Resolution 2^-30 .. 2^-29 of
// the row maximum; the dropped classes (>= 4) are unbiased.  u stays in fp64 registers; g is
// never stored: its grid integers are read back from the digit planes in shared memory.
//
// Warp roles: 4 NH warps, NH threads per row, each owning 128 / NH columns (TMEM lane quadrant =
// warp % 4, column part = warp / 4).  Warp 0 allocates TMEM; thread 0 issues each round's MMAs
// after the named barrier that publishes the A planes.
// Everything else follows pbcd_kernel -- lift + mask at entry and the per-iteration
// ||M o grad||^2 partials for the global stopping rule -- but run in stages (tc_pbcd_chunk,
// pbcd_select_stage) that hand the fp64 iterate over through two state buffers, with a replay
// instead of pbcd_kernel's per-iterate snapshots (pbcd_commit_state commits the result).
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include "internal.h"
#include "tc_ptx.cuh"

namespace enmf {
namespace tpb {

using namespace tcp;

constexpr int BM = 128;
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
  double* pgparts;           // gridDim x (max_iter + 1); this launch writes [it0, it1]
  const int* stage;
  // Staged Alg. 2 (tc_pbcd_chunk): this launch runs iterations [it0, it1) -- round A of
  // it0 .. it1 (the ||M o grad||^2 of u_it0 .. u_it1) and the steps to u_{it0+1} .. u_{it1}
  // -- starting from the lifted F (src < 0) or from the fp64 state ust[src], and leaves u_it1
  // in ust[dst] (tile-major: element (row, col) of tile t at t 128 r + col 128 + row % 128).
  // No per-iteration snapshots: a stop inside a stage is replayed (rctl).  done != 0 (the
  // stopping rule already fired): nothing to do.  kprev: this block's k* of the previous
  // sweep; when it was max_iter (Alg. 2 ran to the end) the first stage runs all iterations
  // at once (it1 := max_iter), as pbcd_select_stage does.  rctl (a replay launch):
  // rctl = {replay?, it0, src, dst} written by pbcd_select_stage, it1 = *kst.
  int it0, it1, src, dst;
  double* ust[2];
  const int* done;
  const int* kprev;
  const int* rctl;
  const int* kst;
  // ablation variants (R29): fstep (device, optional) -- the fixed step 1 / lambda_max(G)
  // replaces Eq.(10)'s d_i (round B, the denominator, is skipped); want_stage 1 with fstep
  // and [0, 1) is one projected-gradient step of the descent stage (no stopping rule, no
  // final gradient).  want_stage 0: the ascent stage (Alg. 2).
  const double* fstep;
  int want_stage;
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
// The 4 weight classes of an accumulator column combined exactly: v0 2^21 + v1 2^14 + v2 2^7 + v3;
// callers fold 2^-21 into their scales.  With K <= 128 and |digits| <= 64 (97 for the HALS
// corrections) every |v_c| < 2^21, so v0 2^7 + v1 and v2 2^7 + v3 are exact int32 and the final
// hi 2^14 + lo (< 2^42) is exact in fp64: 2 int32 IMADs, 2 conversions, 1 DFMA.
__device__ __forceinline__ double comb4(uint32_t v0, uint32_t v1, uint32_t v2, uint32_t v3) {
  const int hi = (int)v0 * 128 + (int)v1;
  const int lo = (int)v2 * 128 + (int)v3;
  return fma((double)hi, 16384.0, (double)lo);
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

// ---- byte digits (tc_pbcd_kernel) ----
// t (|t| < 64) on the 2^-24 grid, n = rint(t 2^24) (|n| < 2^30), as four balanced signed
// base-2^8 digits n = d0 2^24 + d1 2^16 + d2 2^8 + d3 (d1..d3 in [-128, 127], |d0| <= 64): the
// bytes of w = (n + 0x808080) ^ 0x808080 (byte 3 = d0 ... byte 0 = d3).  With b the bytes of
// n + 0x808080, n = b0 2^24 + (b1 - 128) 2^16 + (b2 - 128) 2^8 + (b3 - 128), and b - 128 is
// the byte b ^ 0x80 read as int8.  2 integer ops instead of the 4-step base-2^7 split; every
// digit signed and balanced, so the dropped weight classes (>= 4) stay unbiased.
// Conversions without the XU pipe (quarter rate; ncu: 37 % busy, I2F the top stall after the
// MMA waits): rint(x) for |x| < 2^31 is the low word of x + 1.5 2^52 (one DFMA, round to
// nearest even like __double2int_rn), and an int32 k is the double with high word 0x43300000
// and low word k ^ 2^31 (= 2^52 + 2^31 + k) minus 2^52 + 2^31 (one LOP3 and one DADD).
__device__ __forceinline__ int rint_lo(double t, double scale) {
  return __double2loint(fma(t, scale, 0x1.8p52));
}
__device__ __forceinline__ double i2d(int k) {
  return __hiloint2double(0x43300000, k ^ (int)0x80000000) - 4503601774854144.0;
}
// bdig(t, s): the digit word of t s 2^24 (s a power of two)
__device__ __forceinline__ uint32_t bdig(double t, double s24) {
  return ((uint32_t)rint_lo(t, s24) + 0x00808080u) ^ 0x00808080u;
}
__device__ __forceinline__ uint32_t bdig(double t) { return bdig(t, 0x1p24); }
// 4 x 4 byte transpose (an involution): o[j] byte i = byte j of input i
__device__ __forceinline__ void bt4(uint32_t a, uint32_t b, uint32_t c, uint32_t d,
                                    uint32_t (&o)[4]) {
  const uint32_t t0 = __byte_perm(a, b, 0x5140), t1 = __byte_perm(a, b, 0x7362);
  const uint32_t t2 = __byte_perm(c, d, 0x5140), t3 = __byte_perm(c, d, 0x7362);
  o[0] = __byte_perm(t0, t2, 0x5410);
  o[1] = __byte_perm(t0, t2, 0x7632);
  o[2] = __byte_perm(t1, t3, 0x5410);
  o[3] = __byte_perm(t1, t3, 0x7632);
}
// 16 columns' digit words -> the 16-byte chunks of the 4 A planes (plane pl = digit d_pl =
// byte 3 - pl), one 16-byte store per plane
__device__ __forceinline__ void bstore16(const uint32_t (&w)[16], uint8_t* Ad, int off) {
  uint32_t pl[4][4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t o[4];
    bt4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3], o);
#pragma unroll
    for (int j = 0; j < 4; ++j) pl[3 - j][q] = o[j];
  }
#pragma unroll
  for (int k = 0; k < 4; ++k)
    *reinterpret_cast<uint4*>(Ad + k * PLANE_A + off) =
        make_uint4(pl[k][0], pl[k][1], pl[k][2], pl[k][3]);
}
// The 4 weight classes of an accumulator column combined exactly: v0 2^24 + v1 2^16 + v2 2^8
// + v3; callers fold 2^-24 into their scales.  With K <= 128 and |digits| <= 128 a product
// sum is < 2^21 in magnitude and class c holds c + 1 products, so v0 2^8 + v1 (< 2^29.1) and
// v2 2^8 + v3 (< 1.62e9) are exact int32 and hi 2^16 + lo (< 2^46) is exact in int64 and in
// fp64.  One int64 -> fp64 conversion: the conversions share the quarter-rate XU pipe, which
// ncu showed 38 % busy in the round-2 kernel (13 conversions per element and iteration).
__device__ __forceinline__ double comb8(uint32_t v0, uint32_t v1, uint32_t v2, uint32_t v3) {
  const int hi = (int)v0 * 256 + (int)v1;
  const int lo = (int)v2 * 256 + (int)v3;
  return __longlong_as_double(0x4338000000000000LL + ((long long)hi << 16) + (long long)lo) -
         0x1p52 * 1.5;
}
// 8 doubles of this thread's lanes as two 32-bit TMEM words each (lo words at taddr_lo,
// hi words at taddr_hi, 8 consecutive columns)
__device__ __forceinline__ void tmem_st8d(uint32_t taddr_lo, uint32_t taddr_hi,
                                          const double (&d)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr_lo),
      "r"(__double2loint(d[0])), "r"(__double2loint(d[1])), "r"(__double2loint(d[2])),
      "r"(__double2loint(d[3])), "r"(__double2loint(d[4])), "r"(__double2loint(d[5])),
      "r"(__double2loint(d[6])), "r"(__double2loint(d[7]))
      : "memory");
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr_hi),
      "r"(__double2hiint(d[0])), "r"(__double2hiint(d[1])), "r"(__double2hiint(d[2])),
      "r"(__double2hiint(d[3])), "r"(__double2hiint(d[4])), "r"(__double2hiint(d[5])),
      "r"(__double2hiint(d[6])), "r"(__double2hiint(d[7]))
      : "memory");
}

// The digit products of one round, issued by one thread after the named barrier that publishes
// the A planes; completion arrives on bar_d.  Round A (u G, the gradient: cancellation against
// c) keeps the 4 weight classes -- 10 products as 6 MMAs; round B (g G, only the Eq.(10)
// denominator g G g^T, no cancellation) keeps classes <= 2 -- 6 products as 4 MMAs, 2^-22 of
// the row maximum, like the X passes' operands (round 2b: -40 % of round B's tensor work and
// one TMEM load per column less in its epilogue).
__device__ __forceinline__ void issue_round(uint32_t a0, uint32_t b0, uint32_t tmem_base, int rp,
                                            int r, uint32_t bar_d, bool three = false) {
  const uint32_t idesc_base = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BM >> 4) << 24);
  const uint32_t idesc1 = idesc_base | ((uint32_t)(rp >> 3) << 17);
  const uint32_t idesc2 = idesc_base | ((uint32_t)(2 * rp >> 3) << 17);
  const uint32_t a_lbo = 2048, a_sbo = 128, a_kstep = 4096;
  const uint32_t b_lbo = 128, b_sbo = 8 * KR, b_kstep = 256;
  const int ksteps = (r + 31) / 32;
  constexpr int tab[6][4] = {{0, 0, 0, 1}, {0, 2, 2, 1}, {1, 0, 1, 1},
                             {1, 2, 3, 0}, {2, 0, 2, 1}, {3, 0, 3, 0}};
  // classes <= 2: A0 [B0;B1] -> 0|1, A0 B2 -> 2 (both fresh), A1 [B0;B1] -> 1|2, A2 B0 -> 2
  constexpr int tab3[4][4] = {{0, 0, 0, 1}, {0, 2, 2, 0}, {1, 0, 1, 1}, {2, 0, 2, 0}};
  tc_fence_after();
  for (int j = 0; j < ksteps; ++j) {
    if (three) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint64_t ad = umma_desc(a0 + tab3[q][0] * PLANE_A + j * a_kstep, a_lbo, a_sbo);
        const uint64_t bd = umma_desc(b0 + tab3[q][1] * rp * KR + j * b_kstep, b_lbo, b_sbo);
        tc_mma_i8(tmem_base + tab3[q][2] * rp, ad, bd, tab3[q][3] ? idesc2 : idesc1,
                  (j == 0 && q < 2) ? 0u : 1u);
      }
    } else {
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        const uint64_t ad = umma_desc(a0 + tab[q][0] * PLANE_A + j * a_kstep, a_lbo, a_sbo);
        const uint64_t bd = umma_desc(b0 + tab[q][1] * rp * KR + j * b_kstep, b_lbo, b_sbo);
        tc_mma_i8(tmem_base + tab[q][2] * rp, ad, bd, tab[q][3] ? idesc2 : idesc1,
                  (j == 0 && q < 2) ? 0u : 1u);
      }
    }
  }
  tc_commit(bar_d);
}

// NH threads per row (NH = 2: 8 warps, 64 columns each -- round 1; NH = 4: 16 warps, 32
// columns each -- twice the warps to hide the MMA round trips and the TMEM / shared-memory
// latencies of the epilogue passes, and half the registers for u).  Warp w reads TMEM lane
// quadrant w % 4 (tcgen05.ld's rule) and owns columns [CW (w / 4), CW (w / 4 + 1)).
template <int NH>
__device__ __forceinline__ void bar_pbcd() {
  asm volatile("bar.sync 1, %0;" ::"n"(128 * NH) : "memory");
}

template <int NH>
__global__ void __launch_bounds__(128 * NH, 1) tc_pbcd_kernel(const Params p) {
  constexpr int CW = 128 / NH;               // columns per thread
  constexpr int NWARP = 4 * NH;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;                  // no-swizzle operands need 16-byte alignment only
  uint8_t* Ad = smem;                        // 4 planes of A digits (128 x KR, K-major)
  uint8_t* Bd = smem + 4 * PLANE_A;          // 4 planes of G digits (rp x KR, K-major)
  __shared__ __align__(8) uint64_t bars[1];
  __shared__ uint32_t tmem_base_s;
  __shared__ double xch[NH][BM];             // row exchange between the column parts
  __shared__ int xchi[NH][BM];
  __shared__ double xch2[NH][BM];
  __shared__ double wsum[NWARP];
  __shared__ double gsc_s[128];
  if (p.stage != nullptr && *p.stage != p.want_stage) return;
  int it0 = p.it0, it1 = p.it1, src = p.src, dst = p.dst;
  if (p.rctl != nullptr) {                   // replay of the stage in which the rule fired
    if (p.rctl[0] == 0) return;
    it0 = p.rctl[1];
    it1 = *p.kst;
    src = p.rctl[2];
    dst = p.rctl[3];
  } else {
    if (p.done != nullptr && *p.done != 0) return;
    if (it0 == 0 && p.kprev != nullptr && *p.kprev == p.max_iter) it1 = p.max_iter;
  }
  // 2^-24 / t_j: the column scale with comb8's 2^-24 folded in (exact)
  for (int j = threadIdx.x; j < 128; j += blockDim.x)
    gsc_s[j] = j < p.r ? p.gscale[j] * 0x1p-24 : 0.0;
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
  const bool resume = src >= 0;
  const double* const ust_in = resume ? p.ust[src] : nullptr;
  double* const ust_out = p.ust[dst];
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
    const int hc = warp >> 2;                  // column part
    const int rt = 32 * q + lane;              // row in tile
    const int c0 = CW * hc;
    // my TMEM lane quadrant and columns; class k of the accumulators at column k * KR
    const uint32_t tcol = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)c0;
    const double lam = *p.lam;
    const double fstep = p.fstep != nullptr ? *p.fstep : 0.0;
    const int g8 = rt >> 3, ri = rt & 7;
    // my 16-byte digit chunks in the A planes: chunk b of my part at abase + b * 16 * 128
    uint8_t* const abase = Ad + ((c0 >> 4) * 16 + g8) * 128 + ri * 16;
    uint32_t round = 0;
    const double* gsc = gsc_s + c0;            // 1 / t_j for my columns (shared memory)

    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      const int64_t row = (int64_t)t * BM + rt;
      const bool rok = row < p.rows;
      double u[CW];
      uint32_t mlo = 0, mhi = 0;   // M_{U+} bits of my columns
      // my state slots: column c0 + c of my row at [c * BM] (coalesced across the warp)
      const int64_t sto = (int64_t)t * BM * p.r + (int64_t)c0 * BM + rt;
#pragma unroll
      for (int c = 0; c < CW; ++c) {
        const int col = c0 + c;
        double v;
        if (resume) {
          // u_it0 of an earlier launch: entries outside M_{U+} kept their (negative) lifted
          // value and the projected ones are >= 0, so the mask is again [u >= 0]
          v = (rok && col < p.r) ? ust_in[sto + (int64_t)c * BM] : 0.0;
        } else {
          v = (rok && col < p.r) ? (double)p.F[row * p.ldf + col] : 0.0;
          if (v < 0.0) v += lam;                                   // Eq.(6)/(7) lift
        }
        u[c] = v + 0.0;            // -0 -> +0: the update below tells M_{U+} by the sign bit
        if (rok && col < p.r && v >= 0.0) {                        // M_{U+} (R14)
          if (c < 32) mlo |= 1u << c; else mhi |= 1u << (c - 32);
        }
      }
      // c_i (row of P or Q) -> shared memory as int32 fixed point with a power-of-two row scale:
      // c = cq * csc, |error| <= 2^-30 max_j |c_ij| (the resolution of the u / g digits)
      double cs;
      {
        const double* crow = p.C + row * p.r;
        double cm = 0.0;
        for (int c = 0; c < CW; ++c)
          if (rok && c0 + c < p.r) cm = fmax(cm, fabs(crow[c0 + c]));
        xch2[hc][rt] = cm;
        bar_pbcd<NH>();
        double cmx = 0.0;
#pragma unroll
        for (int h = 0; h < NH; ++h) cmx = fmax(cmx, xch2[h][rt]);
        const double sc = pow2s(cmx);
        cs = 0x1p-24 / sc;
        for (int c = 0; c < CW; ++c)
          Cq[rt * CQ_LD + c0 + c] =
              (rok && c0 + c < p.r) ? __double2int_rn(crow[c0 + c] * sc * 0x1p24) : 0;
      }
      const int32_t* cqrow = Cq + rt * CQ_LD + c0;
      for (int it = it0; it <= it1; ++it) {
        if (it == it1 && p.want_stage == 1) {   // projected-gradient step: u_1 is the result
          if (rok) {
            const int ncol = p.r - c0 < CW ? p.r - c0 : CW;
#pragma unroll
            for (int c = 0; c < CW; ++c)
              if (c < ncol) ust_out[sto + (int64_t)c * BM] = u[c];
          }
          break;
        }
        // ---------------- round A: T1 = u G ----------------
        int mh = 0;
#pragma unroll
        for (int c = 0; c < CW; ++c) mh = max(mh, hiabs(u[c]));
        xchi[hc][rt] = mh;
        bar_pbcd<NH>();
        int mhx = 0;
#pragma unroll
        for (int h = 0; h < NH; ++h) mhx = max(mhx, xchi[h][rt]);
        const double su = pow2s_hi(mhx);
        // digits of u * su into the A planes: chunk (kc, g8, ri), 16 columns each
#pragma unroll
        for (int ch = 0; ch < CW / 16; ++ch) {
          uint32_t wd[16];
#pragma unroll
          for (int k = 0; k < 16; ++k) wd[k] = bdig(u[16 * ch + k], su * 0x1p24);
          bstore16(wd, abase, ch * 16 * 128);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        bar_pbcd<NH>();
        if (threadIdx.x == 0) issue_round(a_s, b_s, tmem_base, rp, p.r, bar_d);
        mbar_wait_hint(bar_d, round & 1);
        ++round;
        tc_fence_after();
        // pass 1: grad = T1 / su - c ; ||M o grad||^2 (pg of iteration it), num, max|g|
        double num = 0.0;
        int gmh = 0;
        opaque(mlo, mhi);
        const double isu = 1.0 / su;
#pragma unroll 1
        for (int b = 0; b < CW / 8; ++b) {  // rolled: keeps the kernel inside the icache
          uint32_t v[4][8];
          double gk[8];
#pragma unroll
          for (int cls = 0; cls < 4; ++cls) TMEM_LD8(tcol + cls * KR + 8 * b, v[cls]);
          const uint32_t mb = ((b < 4 ? mlo : mhi) >> (8 * (b & 3))) & 255u;
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int c = 8 * b + k;
            const double a = comb8(v[0][k], v[1][k], v[2][k], v[3][k]);
            const double gr = a * isu * gsc[c] - i2d(cqrow[c]) * cs;
            const double gm = ((mb >> k) & 1u) ? gr : 0.0;     // M o grad
            gk[k] = gm;
            num = fma(gm, gm, num);
            gmh = max(gmh, hiabs(gm));
          }
          // M o grad back into the classes-0/1 columns just read (lo / hi words): pass 2
          // reads it instead of recombining T1 (round B rewrites all four classes)
          tmem_st8d(tcol + 8 * b, tcol + KR + 8 * b, gk);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        // per-iteration partial of ||M o grad||^2 (fixed-order block reduction)
        double pg = num;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) pg += __shfl_xor_sync(0xffffffffu, pg, o);
        if (lane == 0) wsum[w] = pg;
        xchi[hc][rt] = gmh;
        xch2[hc][rt] = num;
        bar_pbcd<NH>();
        if (threadIdx.x == 32) {
          double s = 0.0;
          for (int k = 0; k < NWARP; ++k) s += wsum[k];
          pgsm[it] += s;
        }
        if (it == it1) {
          tc_fence_before();
          // the final round A has no round B; TMEM reads finish before the next tile's MMAs
          if (rok) {               // u_it1: the next stage's start, or the committed result
            const int ncol = p.r - c0 < CW ? p.r - c0 : CW;
#pragma unroll
            for (int c = 0; c < CW; ++c)
              if (c < ncol) ust_out[sto + (int64_t)c * BM] = u[c];
          }
          bar_pbcd<NH>();
          break;
        }
        if (fstep > 0.0) {
          // fixed step (R29): u <- max(0, u - step M o grad) from the TMEM words of pass 1
          // (unrolled: u must stay in registers)
          opaque(mlo, mhi);
#pragma unroll
          for (int b = 0; b < CW / 8; ++b) {
            uint32_t lo[8], hi[8];
            TMEM_LD8(tcol + 8 * b, lo);
            TMEM_LD8(tcol + KR + 8 * b, hi);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            const uint32_t mb = ((b < 4 ? mlo : mhi) >> (8 * (b & 3))) & 255u;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int c = 8 * b + k;
              const double un = fmax(0.0, u[c] - fstep * __hiloint2double((int)hi[k], (int)lo[k]));
              u[c] = ((mb >> k) & 1u) ? un : u[c];
            }
          }
          tc_fence_before();
          bar_pbcd<NH>();
          continue;
        }
        double numr = 0.0;
        int gmx = 0;
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          numr += xch2[h][rt];
          gmx = max(gmx, xchi[h][rt]);
        }
        const double sg = pow2s_hi(gmx);
        // pass 2: digits of g * sg (g = M o grad, from the TMEM words pass 1 left) into the A
        // planes
        const double sg24 = sg * 0x1p24;
#pragma unroll 1
        for (int b = 0; b < CW / 16; ++b) {
          uint32_t wd[16];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            uint32_t lo[8], hi[8];
            TMEM_LD8(tcol + 16 * b + 8 * h, lo);
            TMEM_LD8(tcol + KR + 16 * b + 8 * h, hi);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            uint32_t nq[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int n = rint_lo(__hiloint2double((int)hi[k], (int)lo[k]), sg24);
              nq[k] = (uint32_t)n;
              wd[8 * h + k] = ((uint32_t)n + 0x00808080u) ^ 0x00808080u;
            }
            // the grid integers of g also go to my class-3 TMEM columns, which round B (classes
            // <= 2) leaves alone: its epilogue and the update read them there instead of
            // transposing the digit planes back out of shared memory
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                    tcol + 3 * KR + 16 * b + 8 * h),
                "r"(nq[0]), "r"(nq[1]), "r"(nq[2]), "r"(nq[3]), "r"(nq[4]), "r"(nq[5]),
                "r"(nq[6]), "r"(nq[7])
                : "memory");
          }
          bstore16(wd, abase, b * 16 * 128);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        bar_pbcd<NH>();
        if (threadIdx.x == 0) issue_round(a_s, b_s, tmem_base, rp, p.r, bar_d, true);
        // ---------------- round B: T2 = g G ----------------
        mbar_wait_hint(bar_d, round & 1);
        ++round;
        tc_fence_after();
        // den = sum_j g_j h_j with g = n 2^-24 / sg (n: the digits' grid integer), h = T2 gsc / sg:
        // accumulate n * T2 gsc and apply the exact power of two 2^-24 / sg^2 once
        double den = 0.0;
        const double isg = 1.0 / sg;
#pragma unroll 1
        for (int b = 0; b < CW / 16; ++b) {
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            uint32_t v[4][8];        // classes 0..2 of T2, and g's grid integers (class 3)
#pragma unroll
            for (int cls = 0; cls < 4; ++cls) TMEM_LD8(tcol + cls * KR + 16 * b + 8 * hh, v[cls]);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int c = 16 * b + 8 * hh + k;
              const double a = comb8(v[0][k], v[1][k], v[2][k], 0u);   // classes <= 2
              den = fma(i2d((int)v[3][k]), a * gsc[c], den);
            }
          }
        }
        den *= 0x1p-24 * isg * isg;
        tc_fence_before();
        xch[hc][rt] = den;
        bar_pbcd<NH>();
        double denr = 0.0;
#pragma unroll
        for (int h = 0; h < NH; ++h) denr += xch[h][rt];
        // Eq.(10): d_i = ||g_i||^2 / ||g_i V^T||^2 (0 on a zero denominator, R10); Eq.(8)
        const double dstep = denr > 0.0 ? numr / denr : 0.0;
        opaque(mlo, mhi);
        const double dsg = dstep * 0x1p-24 * isg;     // step on the grid integers of g
#pragma unroll
        for (int b = 0; b < CW / 16; ++b) {
          uint32_t gn[2][8];
          TMEM_LD8(tcol + 3 * KR + 16 * b, gn[0]);
          TMEM_LD8(tcol + 3 * KR + 16 * b + 8, gn[1]);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          // Eq.(8) with the projection: entries of M_{U+} are exactly those with a clear sign
          // bit (>= +0 after the lift, kept there by the projection; the others stay < 0 and
          // see g = 0, so t = u for them), hence max(0, t) on M_{U+} is "t < 0 <= u -> 0"
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            const int c = 16 * b + k;
            const double t = fma(-dsg, i2d((int)gn[k >> 3][k & 7]), u[c]);
            u[c] = (__double2hiint(t) & ~__double2hiint(u[c])) < 0 ? 0.0 : t;
          }
        }
        tc_fence_before();       // TMEM reads done before the next round's MMAs
        bar_pbcd<NH>();          // everyone has read the g digits before they are overwritten
      }
    }
    bar_pbcd<NH>();
    if (threadIdx.x == 32)
      for (int it = it0; it <= it1; ++it)
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
// BYTE8: the byte digits of tc_pbcd_kernel (bdig: 4 balanced base-2^8 digits on the 2^-24
// grid); else the balanced base-2^7 digits on the 2^-21 grid of tc_hals_kernel.
template <bool BYTE8>
__global__ void __launch_bounds__(KR) gdigits_kernel(const double* __restrict__ G, int r, int rp,
                                                     int8_t* gd, double* gscale, const int* stage,
                                                     int want, int* ill) {
  // one block per B row j (= column j of G), one thread per k index l
  if (stage != nullptr && *stage != want) return;
  __shared__ double wmax[KR / 32], wsum[KR / 32];
  const int j = blockIdx.x, l = threadIdx.x;
  const double g = (j < r && l < r) ? G[(int64_t)l * r + j] : 0.0;
  double mx = fabs(g), sm = fabs(g);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    sm += __shfl_xor_sync(0xffffffffu, sm, o);
  }
  if ((l & 31) == 0) {
    wmax[l >> 5] = mx;
    wsum[l >> 5] = sm;
  }
  __syncthreads();
  mx = fmax(fmax(wmax[0], wmax[1]), fmax(wmax[2], wmax[3]));
  // HALS conditioning guard: the digit coupling errs by ~2^-26 max|u| sum_l |G_lj| in t_j,
  // i.e. 2^-26 sum_l |G_lj| / G_jj relative in the update of u_j.  A column whose diagonal is
  // 2^16 below its absolute column sum (a nearly-zero factor column still coupled to the
  // others) would lose all accuracy, so the SIMT fp64 kernel takes the sweep (*ill != 0).
  if (ill != nullptr && l == 0 && j < r) {
    const double colsum = (wsum[0] + wsum[1]) + (wsum[2] + wsum[3]);
    const double gjj = G[(int64_t)j * r + j];
    if (gjj > 0.0 && colsum > 65536.0 * gjj) atomicOr(ill, 1);
  }
  const double t = pow2s(mx);
  if (l == 0 && j < r) gscale[j] = 1.0 / t;
  const int plane = rp * KR;
  const int off = ((j >> 3) * (KR / 16) + (l >> 4)) * 128 + (j & 7) * 16 + (l & 15);
  if (BYTE8) {
    const uint32_t w = bdig(g * t);
#pragma unroll
    for (int pl = 0; pl < 4; ++pl) gd[pl * plane + off] = (int8_t)(w >> (8 * (3 - pl)));
  } else {
    const Dig4 z = digits4(g * t);
#pragma unroll
    for (int pl = 0; pl < 4; ++pl) gd[pl * plane + off] = z.d[pl];
  }
}

// ------------------------------------------------------------------------------ HALS
// HALS (reading R12) on the tensor cores, blocked Gauss-Seidel: a CTA holds
// a 128-row tile, one thread per row.  t = c - u G for the remaining columns comes from an
// exact int8-digit MMA round (u digits x G digits, 4 weight classes, as in PBCD) against the
// CURRENT u; the sequential column updates then run in registers 32 columns at a time:
//   for k in block:  u_k <- max(0, u_k + t_k / G_kk);  t_j -= (u_k' - u_k) G_kj  (j > k in block)
// after which the block's new u is final (written to F), and a correction round adds
// (u_new - u_old) G for the columns to its right (K = 32: the first round is the only full-K
// product; the change is taken on the digit grid, so T = digits(u_new) G as if recomputed).
// Same update as hals_kernel (the cross-block coupling is exact up to the digit rounding of u,
// 2^-26 of its row maximum); r^2 of the 2 r^2 fp64 FMAs per row move to the tensor pipe, and
// the per-(row, column) shuffles of the SIMT kernel disappear.  A row's c and the block's old
// u are prefetched one block ahead with cp.async into the row's shared-memory slot (coalesced
// per warp; consumers wait and __syncwarp), and the tile's digits are encoded a row per warp
// step with coalesced loads.  A row
// whose updated u outgrows its digit scale (|u| su >= 64, two bits of headroom) finishes the
// columns right of that block with the plain sequential fp64 update (counted in *fallbacks).
constexpr int HT = 128;                       // threads: one per row of the tile
constexpr int HB = 32;                        // columns per Gauss-Seidel block
constexpr int GT_BLK = HB * (HB + 1) / 2;     // packed upper triangle of a diagonal G block
constexpr int CS_LD = 34;                     // doubles per thread slot (16-byte aligned rows)
constexpr int US_LD = 36;                     // floats per thread slot
constexpr int H_SMEM = 4 * PLANE_A + 4 * PLANE_B + (KR / HB) * GT_BLK * 8 + HT * CS_LD * 8 +
                       HT * US_LD * 4;

struct HParams {
  float* F;
  int64_t ldf;
  int64_t rows;
  int r;
  const double* C;
  const double* G;
  const int8_t* gd;
  const double* gscale;
  const int* stage;
  double* minparts;                           // nparts >= gridDim (the rest set to DBL_MAX)
  int nparts;
  unsigned long long* colmax;                 // optional, u64[r]
  int* fallbacks;                             // optional
  const int* ill;                             // optional: nonzero -> the SIMT kernel runs
  // optional (tc_band_flags): tiles taken in order from the counter band_ready[bands + 1],
  // each once its pass-1 band is published (band_ready[t] >= 8 x epoch band_ready[bands]):
  // this kernel then runs behind the X V pass with programmatic dependent launch
  unsigned* band_ready;
  int64_t bands;
};

// the next tile of a dynamically scheduled launch, once its P rows are published (thread 0
// polls with acquire loads; the CTA barrier then orders everyone's reads after them)
__device__ __forceinline__ int next_band_tile(unsigned* band_ready, int64_t bands, int tiles,
                                              int* tile_s) {
  if (threadIdx.x == 0) {
    const int t = (int)atomicAdd(&band_ready[bands + 1], 1u);
    if (t < tiles) {
      const unsigned want = 8u * *((volatile unsigned*)&band_ready[bands]);
      unsigned v;
      long long t0 = clock64();
      while (true) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(band_ready + t)
                     : "memory");
        if (v >= want) break;
        __nanosleep(256);
        if (clock64() - t0 > 40000000000LL) {
          printf("enmf tc: band %d never published (%u < %u)\n", t, v, want);
          __trap();
        }
      }
    }
    *tile_s = t;
  }
  asm volatile("bar.sync 1, %0;" ::"n"(HT) : "memory");
  const int t = *tile_s;
  asm volatile("bar.sync 1, %0;" ::"n"(HT) : "memory");   // *tile_s is reused by the next call
  return t;
}

// (k, j), j >= k, of a packed upper-triangular 32 x 32 block; (k, k) holds 1 / G_kk (the
// diagonal itself is never needed: t_k is dead once u_k is updated)
__host__ __device__ constexpr int tri(int k, int j) { return HB * k - k * (k - 1) / 2 + (j - k); }

__device__ __forceinline__ void cp_async(uint32_t dst, const void* src, int bytes, int src_bytes) {
  if (bytes == 16)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
                 "r"(src_bytes) : "memory");
  else if (bytes == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src),
                 "r"(src_bytes) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src),
                 "r"(src_bytes) : "memory");
}

// my row's c[cs, cs+32) and u[cs, cs+32) -> my slots (zero beyond r or for an idle row)
__device__ __forceinline__ void prefetch_block(const HParams& p, int64_t row, bool rok, int cs,
                                               bool vc, bool vu, uint32_t cslot, uint32_t uslot) {
  const double* crow = p.C + (rok ? row : 0) * p.r;
  const float* frow = p.F + (rok ? row : 0) * p.ldf;
  if (vc && vu && rok && cs + HB <= p.r) {             // the common case: whole block, 16 B
#pragma unroll
    for (int q = 0; q < HB / 2; ++q) cp_async(cslot + 16 * q, crow + cs + 2 * q, 16, 16);
#pragma unroll
    for (int q = 0; q < HB / 4; ++q) cp_async(uslot + 16 * q, frow + cs + 4 * q, 16, 16);
    asm volatile("cp.async.commit_group;" ::: "memory");
    return;
  }
  if (vc) {
#pragma unroll
    for (int q = 0; q < HB / 2; ++q) {
      const int c = cs + 2 * q;
      const int nb = rok ? (c + 2 <= p.r ? 16 : (c < p.r ? 8 : 0)) : 0;
      cp_async(cslot + 16 * q, crow + (nb ? c : 0), 16, nb);
    }
  } else {
    for (int q = 0; q < HB; ++q) {
      const int c = cs + q;
      const int nb = rok && c < p.r ? 8 : 0;
      cp_async(cslot + 8 * q, crow + (nb ? c : 0), 8, nb);
    }
  }
  if (vu) {
#pragma unroll
    for (int q = 0; q < HB / 4; ++q) {
      const int c = cs + 4 * q;
      const int nb = rok && c < p.r ? 16 : 0;            // vu implies r % 4 == 0
      cp_async(uslot + 16 * q, frow + (nb ? c : 0), 16, nb);
    }
  } else {
    for (int q = 0; q < HB; ++q) {
      const int c = cs + q;
      const int nb = rok && c < p.r ? 4 : 0;
      cp_async(uslot + 4 * q, frow + (nb ? c : 0), 4, nb);
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// The same for the 32 rows of a warp, coalesced (2 rows of c / 4 rows of u per instruction):
// only when all 32 rows and the whole block exist and the 16-byte copies are allowed.  The
// slots are then written by other lanes: consumers wait (cp.async.wait_all) and __syncwarp.
__device__ __forceinline__ void prefetch_block_warp(const HParams& p, int64_t roww, int cs,
                                                    uint32_t cs_w, uint32_t us_w, int lane) {
#pragma unroll
  for (int i = 0; i < HB / 2; ++i) {
    const int rr = 2 * i + (lane >> 4), c2 = 2 * (lane & 15);
    cp_async(cs_w + (rr * CS_LD + c2) * 8, p.C + (roww + rr) * p.r + cs + c2, 16, 16);
  }
#pragma unroll
  for (int i = 0; i < HB / 4; ++i) {
    const int rr = 4 * i + (lane >> 3), c4 = 4 * (lane & 7);
    cp_async(us_w + (rr * US_LD + c4) * 4, p.F + (roww + rr) * p.ldf + cs + c4, 16, 16);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// MMAs of the first round: T[:, cs:128] = u G[:, cs:128] (4 classes, 10 narrow products)
__device__ __forceinline__ void issue_hals_round(uint32_t a0, uint32_t b0, uint32_t tmem_base,
                                                 int r, int cs, uint32_t bar_d) {
  const int rem = KR - cs;
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BM >> 4) << 24) |
                         ((uint32_t)(rem >> 3) << 17);
  const uint32_t a_lbo = 2048, a_sbo = 128, a_kstep = 4096;
  const uint32_t b_lbo = 128, b_sbo = 8 * KR, b_kstep = 256;
  const uint32_t bcol = (uint32_t)(cs / 8) * (8 * KR);     // first output column's row group
  const int ksteps = (r + 31) / 32;
  constexpr int prs[10][2] = {{0, 0}, {0, 1}, {1, 0}, {0, 2}, {1, 1},
                              {2, 0}, {0, 3}, {1, 2}, {2, 1}, {3, 0}};
  tc_fence_after();
  for (int j = 0; j < ksteps; ++j) {
#pragma unroll
    for (int q = 0; q < 10; ++q) {
      const int ia = prs[q][0], ib = prs[q][1], cls = ia + ib;
      const uint64_t ad = umma_desc(a0 + ia * PLANE_A + j * a_kstep, a_lbo, a_sbo);
      const uint64_t bd = umma_desc(b0 + ib * KR * KR + bcol + j * b_kstep, b_lbo, b_sbo);
      // first product of each class at k-step 0 initialises its accumulator
      const bool fresh = j == 0 && (q == 0 || q == 1 || q == 3 || q == 6);
      tc_mma_i8(tmem_base + cls * KR + cs, ad, bd, idesc, fresh ? 0u : 1u);
    }
  }
  tc_commit(bar_d);
}

// Correction round: T[:, cs:128] += du G[kb-slice, cs:128], du = the digit-integer change of
// block kb's u (K = 32, one k-step, 10 narrow products accumulating onto round 0's sums)
__device__ __forceinline__ void issue_hals_corr(uint32_t a0, uint32_t b0, uint32_t tmem_base,
                                                int kb, int cs, uint32_t bar_d) {
  const int rem = KR - cs;
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BM >> 4) << 24) |
                         ((uint32_t)(rem >> 3) << 17);
  const uint32_t bcol = (uint32_t)(cs / 8) * (8 * KR);
  constexpr int prs[10][2] = {{0, 0}, {0, 1}, {1, 0}, {0, 2}, {1, 1},
                              {2, 0}, {0, 3}, {1, 2}, {2, 1}, {3, 0}};
  tc_fence_after();
#pragma unroll
  for (int q = 0; q < 10; ++q) {
    const int ia = prs[q][0], ib = prs[q][1], cls = ia + ib;
    const uint64_t ad = umma_desc(a0 + ia * PLANE_A + kb * 4096, 2048, 128);
    const uint64_t bd = umma_desc(b0 + ib * KR * KR + bcol + kb * 256, 128, 8 * KR);
    tc_mma_i8(tmem_base + cls * KR + cs, ad, bd, idesc, 1u);
  }
  tc_commit(bar_d);
}

__device__ __forceinline__ int rebuild_n(const uint4 (&dq)[4], int k) {
  return (digit_at(dq[0], k) << 21) + (digit_at(dq[1], k) << 14) + (digit_at(dq[2], k) << 7) +
         digit_at(dq[3], k);
}

__device__ __forceinline__ void bar_hals() {
  asm volatile("bar.sync 1, %0;" ::"n"(HT) : "memory");
}

__global__ void __launch_bounds__(HT, 1) tc_hals_kernel(const HParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* Ad = smem_raw;                                        // u digits, 4 planes
  uint8_t* Bd = smem_raw + 4 * PLANE_A;                          // G digits, 4 planes
  double* Gt = reinterpret_cast<double*>(Bd + 4 * PLANE_B);      // diagonal G blocks (packed)
  double* Cs = Gt + (KR / HB) * GT_BLK;                          // per-thread c slots
  float* Us = reinterpret_cast<float*>(Cs + HT * CS_LD);         // per-thread u slots
  __shared__ __align__(8) uint64_t bars[1];
  __shared__ uint32_t tmem_base_s;
  __shared__ double gsc_s[KR];
  __shared__ unsigned cm_s[KR];                                  // fp32 bits of max |u|
  __shared__ double wmin_s[HT / 32];
  // Launched as the programmatic dependent of the X V pass (band_ready), this grid may finish
  // before that pass does; griddepcontrol.wait (a no-op otherwise) on every exit keeps the
  // stream order for what follows (the PBCD stages and the SIMT fallback read P).
  if ((p.stage != nullptr && *p.stage != 1) || (p.ill != nullptr && *p.ill != 0)) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    return;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = p.r;
  const int nblk = (r + HB - 1) / HB;
  for (int j = threadIdx.x; j < KR; j += blockDim.x) {
    gsc_s[j] = j < r ? p.gscale[j] * 0x1p-21 : 0.0;
    cm_s[j] = 0u;
  }
  for (int e = threadIdx.x; e < (KR / HB) * HB * HB; e += blockDim.x) {
    const int b = e / (HB * HB), k = (e / HB) % HB, j = e % HB;
    if (j < k) continue;
    const int gk = HB * b + k, gj = HB * b + j;
    double v = 0.0;
    if (gk < r && gj < r) {
      v = p.G[(int64_t)gk * r + gj];
      if (j == k) v = v > 0.0 ? 1.0 / v : 0.0;                   // column skipped if G_kk <= 0
    }
    Gt[b * GT_BLK + tri(k, j)] = v;
  }
  for (int e = threadIdx.x; e < 4 * KR * KR / 16; e += blockDim.x)
    reinterpret_cast<uint4*>(Bd)[e] = reinterpret_cast<const uint4*>(p.gd)[e];
  const uint32_t bar_d = smem_u32(&bars[0]);
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
  const int rt = threadIdx.x;                                     // row in tile
  const uint32_t tlane = tmem_base + ((uint32_t)(32 * warp) << 16);
  uint8_t* const abase = Ad + (rt >> 3) * 128 + (rt & 7) * 16;    // chunk kc at + kc * 2048
  double* const cslot = Cs + rt * CS_LD;
  float* const uslot = Us + rt * US_LD;
  const uint32_t cslot_s = smem_u32(cslot), uslot_s = smem_u32(uslot);
  // 16-byte copies where rows and columns allow (uniform)
  const bool vc = (r % 2) == 0 && (reinterpret_cast<uintptr_t>(p.C) & 15) == 0;
  const bool vu = (r % 4) == 0 && (p.ldf % 4) == 0 && (reinterpret_cast<uintptr_t>(p.F) & 15) == 0;
  const int tiles = (int)((p.rows + BM - 1) / BM);
  uint32_t round = 0;
  double wmin = DBL_MAX;
  int nfall = 0;
  __shared__ int tile_s;
  const bool dyn = p.band_ready != nullptr;
  for (int t = dyn ? next_band_tile(p.band_ready, p.bands, tiles, &tile_s) : (int)blockIdx.x;
       t < tiles;
       t = dyn ? next_band_tile(p.band_ready, p.bands, tiles, &tile_s) : t + (int)gridDim.x) {
    const int64_t row0 = (int64_t)t * BM;
    const int nt = (int)(p.rows - row0 < BM ? p.rows - row0 : BM);
    const bool rok = rt < nt;
    const int64_t row = row0 + rt;
    float* const frow = p.F + (rok ? row : 0) * p.ldf;
    const int64_t roww = row0 + 32 * warp;                        // my warp's first row
    const bool wfull = 32 * warp + 32 <= nt;                      // all 32 rows exist
    const uint32_t cs_w = smem_u32(Cs + 32 * warp * CS_LD), us_w = smem_u32(Us + 32 * warp * US_LD);
    auto prefetch = [&](int cs) {
      if (vc && vu && wfull && cs + HB <= r) prefetch_block_warp(p, roww, cs, cs_w, us_w, lane);
      else prefetch_block(p, row, rok, cs, vc, vu, cslot_s, uslot_s);
    };
    prefetch(0);
    // digits of the warp's rows, one row per step, coalesced (lane: columns 4 lane .. + 3):
    // scale with two bits of headroom, max |u| su in [16, 32); lane i keeps row i's scale
    double su = 0.5;
    {
      // all 32 rows' loads in flight first (one 16-byte load per lane and row)
      float4 q[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int rr = 32 * warp + i;
        const float* fr = p.F + (row0 + rr) * p.ldf;
        q[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (rr < nt) {
          if (vu) {
            if (4 * lane < r) q[i] = *reinterpret_cast<const float4*>(fr + 4 * lane);
          } else {
            if (4 * lane < r) q[i].x = fr[4 * lane];
            if (4 * lane + 1 < r) q[i].y = fr[4 * lane + 1];
            if (4 * lane + 2 < r) q[i].z = fr[4 * lane + 2];
            if (4 * lane + 3 < r) q[i].w = fr[4 * lane + 3];
          }
        }
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int rr = 32 * warp + i;
        const float v[4] = {q[i].x, q[i].y, q[i].z, q[i].w};
        unsigned mb = 0u;
#pragma unroll
        for (int k = 0; k < 4; ++k) mb = max(mb, __float_as_uint(v[k]) & 0x7fffffffu);
        mb = __reduce_max_sync(0xffffffffu, mb);
        const double sr = 0.5 * pow2s_hi(hiabs((double)__uint_as_float(mb)));
        if (lane == i) su = sr;
        uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t dw = digits_word((double)v[k] * sr);
#pragma unroll
          for (int pl = 0; pl < 4; ++pl) w[pl] |= ((dw >> (8 * pl)) & 255u) << (8 * k);
        }
        uint8_t* dst = Ad + (lane >> 2) * 2048 + (rr >> 3) * 128 + (rr & 7) * 16 + 4 * (lane & 3);
#pragma unroll
        for (int pl = 0; pl < 4; ++pl) *reinterpret_cast<uint32_t*>(dst + pl * PLANE_A) = w[pl];
      }
    }
    const double isu = 1.0 / su;
    const double snap = 0x1p-18 * isu;            // max |u| su in [16, 32): 2^-22..2^-23 of it
    const int ovf_hi = __double2hiint(64.0 * isu);
    int bover = -1;                    // first block whose new u outgrew the digit scale
#pragma unroll 1
    for (int b = 0; b < nblk; ++b) {
      const int cs = HB * b;
      // publish the digits (and finish reading the previous round's TMEM), then the round
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      bar_hals();
      if (threadIdx.x == 0) {
        if (b == 0) issue_hals_round(a_s, b_s, tmem_base, r, 0, bar_d);
        else issue_hals_corr(a_s, b_s, tmem_base, b - 1, cs, bar_d);
      }
      mbar_wait(bar_d, round & 1);
      ++round;
      tc_fence_after();
      asm volatile("cp.async.wait_all;" ::: "memory");
      __syncwarp();
      // t = c - u G on this block's columns (exact class combine, 2^-21 / t_j folded in gsc)
      double tt[HB], uu[HB];
#pragma unroll
      for (int h = 0; h < HB / 8; ++h) {
        uint32_t v[4][8];
#pragma unroll
        for (int cls = 0; cls < 4; ++cls) TMEM_LD8(tlane + cls * KR + cs + 8 * h, v[cls]);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const double a = comb4(v[0][k], v[1][k], v[2][k], v[3][k]);
          tt[8 * h + k] = cslot[8 * h + k] - a * isu * gsc_s[cs + 8 * h + k];
          uu[8 * h + k] = (double)uslot[8 * h + k];
        }
      }
      // the slot's values are in registers (tt, uu depend on them): prefetch the next block
      __syncwarp();                    // every lane of the warp has read its slot
      if (b + 1 < nblk) prefetch(cs + HB);
      // sequential Gauss-Seidel over the block's columns
      const double* gt = Gt + b * GT_BLK;
#pragma unroll
      for (int k = 0; k < HB; ++k) {
        const double ig = gt[tri(k, k)];
        const double vn = fma(tt[k], ig, uu[k]);
        // projection; below `snap` (2^-22 of the row's maximum, 16x the coupling's ~2^-26
        // error) an update counts as zero, so a column the exact update drives to zero stays
        // exactly zero (R28); G_kk <= 0: column skipped
        const double nu = ig == 0.0 ? uu[k] : (vn > snap ? vn : 0.0);
        const double d = nu - uu[k];
        uu[k] = nu;
#pragma unroll
        for (int j = k + 1; j < HB; ++j) tt[j] = fma(-d, gt[tri(k, j)], tt[j]);
      }
      // the block is final for this sweep: store (unless an earlier block overflowed: then the
      // fallback redoes these columns), column maxima, minimum; digits for the next rounds
      const bool keep = rok && bover < 0;
      int hmax = 0;                    // u >= 0: |u| su >= 64 <=> high word >= that of 64 / su
#pragma unroll
      for (int k = 0; k < HB; ++k) hmax = max(hmax, __double2hiint(uu[k]));
      const bool ovf = hmax >= ovf_hi;
      float uo[HB];
#pragma unroll
      for (int k = 0; k < HB; ++k) uo[k] = (float)uu[k];
      if (keep) {
        if (vu) {
#pragma unroll
          for (int q = 0; q < HB / 4; ++q)
            if (cs + 4 * q < r)
              *reinterpret_cast<float4*>(frow + cs + 4 * q) =
                  make_float4(uo[4 * q], uo[4 * q + 1], uo[4 * q + 2], uo[4 * q + 3]);
        } else {
#pragma unroll
          for (int k = 0; k < HB; ++k)
            if (cs + k < r) frow[cs + k] = uo[k];
        }
        float mn[HB / 2];
#pragma unroll
        for (int k = 0; k < HB / 2; ++k)
          mn[k] = cs + HB <= r ? fminf(uo[k], uo[k + HB / 2])
                               : fminf(cs + k < r ? uo[k] : FLT_MAX,
                                       cs + k + HB / 2 < r ? uo[k + HB / 2] : FLT_MAX);
#pragma unroll
        for (int w = HB / 4; w > 0; w >>= 1)
#pragma unroll
          for (int k = 0; k < w; ++k) mn[k] = fminf(mn[k], mn[k + w]);
        wmin = fmin(wmin, (double)mn[0]);
      }
      // u >= 0 (HALS projects), so the fp32 bits order like the values
      unsigned mine = 0u;
#pragma unroll
      for (int k = 0; k < HB; ++k) {
        const unsigned m = __reduce_max_sync(0xffffffffu, keep ? __float_as_uint(uo[k]) : 0u);
        if (lane == k) mine = m;
      }
      if (mine) atomicMax(&cm_s[cs + lane], mine);
      if (bover < 0 && ovf) bover = b;
      if (b + 1 < nblk) {
        // the block's slice of the A planes now holds the digits of du = n(u_new) - n(u_old)
        // (integers on the 2^-21 / su grid; |du| < 96 * 2^21 keeps d0 within int8), so the
        // correction round leaves T = digits(u_new) G up to the dropped weight classes
#pragma unroll
        for (int ch = 0; ch < HB / 16; ++ch) {
          const int off = (cs / 16 + ch) * 16 * 128;
          uint4 dq[4];
#pragma unroll
          for (int pl = 0; pl < 4; ++pl)
            dq[pl] = *reinterpret_cast<const uint4*>(abase + pl * PLANE_A + off);
          Pack16 pk;
          pack_clear(pk);
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            const int nn = __double2int_rn(uu[16 * ch + k] * su * 0x1p21);
            pack_put(pk, k, digits_n(nn - rebuild_n(dq, k)));
          }
          pack_store(pk, abase, off);
        }
      }
    }
    // rows whose u outgrew the digit scale: the columns right of that block, sequentially in
    // fp64 against F (columns left of k already hold this sweep's values, as in hals_kernel)
    if (rok && bover >= 0 && HB * (bover + 1) < r) {
      ++nfall;
      for (int k = HB * (bover + 1); k < r; ++k) {
        double s = p.C[row * r + k];
        for (int l = 0; l < r; ++l) s -= (double)frow[l] * p.G[(int64_t)l * r + k];
        const double gkk = p.G[(int64_t)k * r + k];
        if (!(gkk > 0.0)) continue;
        const double uo = (double)frow[k];
        const double vn = fma(s, 1.0 / gkk, uo);
        const float nu = (float)(vn > 0.0 ? vn : 0.0);
        frow[k] = nu;
        wmin = fmin(wmin, (double)nu);
        atomicMax(&cm_s[k], __float_as_uint(nu));
      }
    }
  }
  if (p.fallbacks && nfall) atomicAdd(p.fallbacks, nfall);
  // block minimum and column maxima
  double m = wmin;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) wmin_s[warp] = m;
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0 && p.minparts) {
    double mm = DBL_MAX;
    for (int w = 0; w < HT / 32; ++w) mm = fmin(mm, wmin_s[w]);
    p.minparts[blockIdx.x] = mm;
    for (int q = blockIdx.x + gridDim.x; q < p.nparts; q += gridDim.x) p.minparts[q] = DBL_MAX;
  }
  if (p.colmax)
    for (int j = threadIdx.x; j < r; j += blockDim.x)
      if (cm_s[j])
        atomicMax(&p.colmax[j],
                  (unsigned long long)__double_as_longlong((double)__uint_as_float(cm_s[j])));
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

}  // namespace tpb

int tc_pbcd_parts() { return kSMs; }

bool tc_pbcd_supported(int r) { return r >= 1 && r <= 128; }

// G (r x r) -> the B-operand digits and column scales of tc_pbcd_chunk (ascent stage only).
void tc_pbcd_prepare(const double* G, int r, int8_t* gd_work, double* gscale_work,
                     const int* stage, cudaStream_t st, int want_stage) {
  using namespace tpb;
  gdigits_kernel<true><<<KR, KR, 0, st>>>(G, r, KR, gd_work, gscale_work, stage, want_stage,
                                          nullptr);
  count_launch();
}

// One stage [it0, it1) of Alg. 2 on the tensor cores (see Params), or (rctl != nullptr) the
// replay of the stage in which the stopping rule fired; pgparts holds gridDim x
// (max_iter + 1), a launch writes columns it0 .. it1.  The caller reduces the partials and
// applies the stopping rule between stages (pbcd_select_stage), which sets *done.
int tc_pbcd_chunk(const float* F, int64_t ldf, int64_t rows, int r, const double* C,
                  const double* lam, int max_iter, int it0, int it1, int src, int dst,
                  double* ust0, double* ust1, double* pgparts, const int8_t* gd_work,
                  const double* gscale_work, const int* stage, const int* done,
                  const int* kprev, const int* rctl, const int* kst, cudaStream_t st,
                  const double* fstep, int want_stage) {
  using namespace tpb;
  Params p;
  p.fstep = fstep;
  p.want_stage = want_stage;
  p.F = F;
  p.ldf = ldf;
  p.rows = rows;
  p.r = r;
  p.rp = KR;   // G padded to 128 columns: class k of the accumulators at column k * 128
  p.C = C;
  p.gd = gd_work;
  p.gscale = gscale_work;
  p.lam = lam;
  p.max_iter = max_iter;
  p.pgparts = pgparts;
  p.stage = stage;
  p.it0 = it0;
  p.it1 = it1;
  p.src = src;
  p.dst = dst;
  p.ust[0] = ust0;
  p.ust[1] = ust1;
  p.done = done;
  p.kprev = kprev;
  p.rctl = rctl;
  p.kst = kst;
  if (!ust0 || !ust1 || dst < 0 || dst > 1 || src > 1 ||
      (!rctl && (it0 < 0 || it1 <= it0 || it1 > max_iter)) || (rctl && !kst))
    return 1;
  const size_t smem = SMEM_BYTES + sizeof(double) * (max_iter + 1);
  // the dynamic size grows with max_iter; static shared memory (row exchanges) counts against
  // the same 227 KB, so the attribute is the exact dynamic request, raised when it grows
  // NH = 4: 16 warps, 32 columns per thread (round 1's NH = 2, 64 columns per thread, was
  // 15 % slower: fewer warps to hide the MMA round trips and TMEM / shared-memory latencies)
  static size_t attr = 0;
  if (smem > attr) {
    auto k = tc_pbcd_kernel<4>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return 1;
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    attr = smem;
  }
  // unused CTAs of the persistent grid still write their (zero) partials: launch kSMs always
  tc_pbcd_kernel<4><<<kSMs, 512, smem, st>>>(p);
  count_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int tc_hals_parts() { return kSMs; }

int tc_hals_prepare(const double* G, int r, int8_t* gd_work, double* gscale_work,
                    const int* stage, int* ill, cudaStream_t st) {
  using namespace tpb;
  if (ill != nullptr && cudaMemsetAsync(ill, 0, sizeof(int), st) != cudaSuccess) return 1;
  gdigits_kernel<false><<<KR, KR, 0, st>>>(G, r, KR, gd_work, gscale_work, stage, 1, ill);
  count_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int tc_hals_launch(float* F, int64_t ldf, int64_t rows, int r, const double* C, const double* G,
                   const int8_t* gd_work, const double* gscale_work, const int* stage,
                   double* minparts, int nparts, unsigned long long* colmax, int* fallbacks,
                   const int* ill, unsigned* band_ready, int64_t bands, cudaStream_t st) {
  using namespace tpb;
  HParams p;
  p.F = F;
  p.ldf = ldf;
  p.rows = rows;
  p.r = r;
  p.C = C;
  p.G = G;
  p.gd = gd_work;
  p.gscale = gscale_work;
  p.stage = stage;
  p.minparts = minparts;
  p.nparts = nparts;
  p.colmax = colmax;
  p.fallbacks = fallbacks;
  p.ill = ill;
  p.band_ready = band_ready;
  p.bands = bands;
  if (band_ready != nullptr && bands != (rows + BM - 1) / BM) return 1;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(tc_hals_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             H_SMEM) != cudaSuccess)
      return 1;
    attr = true;
  }
  if (band_ready == nullptr) {
    tc_hals_kernel<<<kSMs, HT, H_SMEM, st>>>(p);
  } else {
    // programmatic dependent launch behind the X V pass (which triggers at its start): CTAs
    // take SMs as pass-1 CTAs retire and consume bands as they are published
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kSMs);
    cfg.blockDim = dim3(HT);
    cfg.dynamicSmemBytes = H_SMEM;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, tc_hals_kernel, p) != cudaSuccess) return 1;
  }
  count_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int tc_hals_rows(float* F, int64_t ldf, int64_t rows, int r, const double* C, const double* G,
                 int8_t* gd_work, double* gscale_work, const int* stage, double* minparts,
                 int nparts, unsigned long long* colmax, int* fallbacks, int* ill,
                 cudaStream_t st) {
  if (tc_hals_prepare(G, r, gd_work, gscale_work, stage, ill, st)) return 1;
  return tc_hals_launch(F, ldf, rows, r, C, G, gd_work, gscale_work, stage, minparts, nparts,
                        colmax, fallbacks, ill, nullptr, 0, st);
}

}  // namespace enmf
