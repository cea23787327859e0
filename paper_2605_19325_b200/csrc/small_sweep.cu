// small_sweep.cu -- HALS sweeps of a cache-resident problem in ONE persistent kernel.
//
// the small BASELINE configurations (C1-C4, X <= 90 MB) are bound by launch and
// synchronisation latency, not by HBM: a HALS sweep issued as separate kernels is ~25 launches
// of a few microseconds each around ~10 us of arithmetic.  Here a cooperative grid runs
// `count` whole sweeps (U block with P = X V and G_V, V block with
// Q = X^T U_new and G_U, then the trace-form objective, BASELINE.json:5) with four grid
// barriers per sweep and no host involvement:
//
//   A   partial products of P = X V over (64-row block) x (K chunk) tiles        | barrier
//   A'  per row: P = sum of its partials, HALS column sweep, U written (fp32),
//       per-CTA partial of G_U = U^T U, min U                                    | barrier
//   B   G_U = fixed-order sum of the partials; partial products of Q = X^T U     | barrier
//   B'  per row of V: Q, HALS, V written, partials of G_V, <Q, V>, min V         | barrier
//   (next A: G_V and <Q, V> summed; next A': f = ||X||^2 - 2 <Q, V> + <G_U, G_V>)
//
// All arithmetic is fp64 on the fp32 state (the ENMF_PREC_FP64 path); every sum has a fixed
// order given the grid, so results are deterministic.  The grid is sized to the problem (a
// barrier over 8 CTAs is cheaper than over 296).  Single rank, dense X, HALS stage only.
#include <float.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>

#include "grid_barrier.cuh"
#include "internal.h"
#include "rows_dev.cuh"

namespace enmf {
namespace {

using namespace rows_dev;

constexpr int kT = 256;     // threads per CTA
constexpr int kW = kT / 32;
constexpr int kTM = 64;     // output rows of a product tile
constexpr int kKS = 32;     // K slab
constexpr int kXP = kTM + 4;   // padded slab row: the DMMA A-fragment loads (4 k x 8 rows) hit 16 banks
constexpr int kRB = 4;      // rows per warp in the HALS phases

struct SmallArgs {
  const float* X;
  int64_t ldx, m, n;
  int r;
  float* U;
  int64_t ldu;
  float* V;
  int64_t ldv;
  double* GV;        // in: V^T V of the V passed in; out: of the final V
  double* GU;        // out: U^T U of the final U
  const double* xnorm2;
  double* ftrace;
  int* fcnt;
  double* minu;
  double* minv;
  int* stage;
  int* cnt_hals;
  double* pp;        // tile partials: max(ksA m, ksB n) r
  double* gp;        // Gram partials: gridDim x r^2
  double* sc;        // scalar partials: cross[grid], min[grid], then 2 reduced scalars
  int ksA, ksB;
  int64_t kcA, kcB;  // K chunk of a tile
  unsigned* bar;     // grid barrier counter (zeroed before the launch)
  int count;
  int debug;         // ENMF_SMALL_DEBUG=1: CTA 0 prints the last sweep's phase times
};

// ---------------------------------------------------------------------------------------------
// D(8x8) += A(8x4) B(4x8) on the fp64 tensor cores: lane holds A[lane/4][lane%4],
// B[lane%4][lane/4] and D[lane/4][2 (lane%4) + {0, 1}].
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int RCOLS>
struct TileShape {
  static constexpr int NB = RCOLS / 8;                 // 8-column B fragments of the tile
  static constexpr int WNB = NB < 8 ? NB : 8;          // ... of a warp
  static constexpr int CW = NB / WNB;                  // warps across the columns (1 or 2)
  static constexpr int NG = kW / (4 * CW);             // k groups (2 or 1)
  static constexpr int GT = kT / NG;                   // threads per group
  static constexpr int NA = 4 * WNB;                   // accumulators per thread
  static constexpr int FP = RCOLS + 4;                 // padded row of the factor slab
  static constexpr int SLABD = kKS * kXP + kKS * FP;   // doubles of the fp64 slabs
  static constexpr int REDD = (NG - 1) * NA * GT;      // doubles of the group hand-over
  static constexpr int PRODD = SLABD > REDD ? SLABD : REDD;
  static constexpr int SLAB32 = kTM * kKS + RCOLS * kKS;   // floats per staged slab
};

// One product tile: out[row][c] = sum_{k in [k0, k1)} op(X)[row][k] F[k][c] for the 64 output
// rows r0.. (rows of X if !TRANS, columns of X if TRANS) and all r <= RCOLS columns, fp64 on
// the tensor cores (DMMA m8n8k4: 256 FMA per instruction from two operand registers per lane,
// so shared memory carries ~1/5 of the SIMT register-tile traffic; the SIMT 4 x 4 tile ran at
// 35 % of the fp64 rate, bound by shared-memory wavefronts -- ncu, profiles/r02d notes).
// Warp (wr, wc) of a k group owns rows 16 wr .. +15 and columns 8 WNB wc .. ; the NG groups take
// the 4-deep k steps of a slab alternately and their sums are added in group order through
// shared memory at the end (fixed order).
template <int RCOLS, bool TRANS>
__device__ __forceinline__ void product_tile(const float* __restrict__ X, int64_t ldx, int64_t M,
                                             const float* F, int64_t ldf, int r, int64_t r0,
                                             int64_t k0, int64_t k1, double* out, double* Xs,
                                             double* Fs, float* St) {
  using TS = TileShape<RCOLS>;
  constexpr int NB = TS::NB, WNB = TS::WNB, CW = TS::CW, NG = TS::NG, GT = TS::GT, NA = TS::NA;
  constexpr int FP = TS::FP, SLAB32 = TS::SLAB32;
  constexpr int XQ = kTM * kKS / kT;       // X elements per thread and slab (8)
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int g = warp / (4 * CW), wr = (warp % (4 * CW)) / CW, wc = warp % CW;
  double acc[2][WNB][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < WNB; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  // Per-thread element maps of a slab:
  //   X, !TRANS: row t/16 + 16 (q%4), k t%16 + 16 (q/4)  (a warp reads 2 rows x 64 bytes);
  //      TRANS:  k t/64 + 4 q, row t%64;      F: k t/8, columns t%8 + 8 q, q < NB.
  // Slabs arrive as fp32 through cp.async into a two-deep staging ring (no registers held, two
  // slabs of FMAs to cover the L2 / HBM latency); every thread converts the elements it
  // requested itself into the fp64 slab the tensor cores read.
  const int xi = TRANS ? t % kTM : t / 16, xk = TRANS ? t / kTM : t % 16;
  const float* xp = TRANS ? X + (k0 + xk) * ldx + r0 + xi : X + (r0 + xi) * ldx + k0 + xk;
  const int64_t xrows = M - r0 - xi;             // rows left from this thread's first row
  const int fc = t % 8, fk = t / 8;
  const float* fp = F + (k0 + fk) * ldf + fc;
  const unsigned st_base = (unsigned)__cvta_generic_to_shared(St) + 4u * t;
  auto request = [&](int64_t ks, int buf) {
    const int64_t kleft = k1 - ks;               // valid k of this slab: kk < kleft
    const unsigned dst = st_base + 4u * SLAB32 * buf;
#pragma unroll
    for (int q = 0; q < XQ; ++q) {
      bool ok;
      const float* src;
      if (TRANS) {
        ok = xrows > 0 && xk + 4 * q < kleft;
        src = xp + (int64_t)(4 * q) * ldx;
      } else {
        ok = 16 * (q % 4) < xrows && xk + 16 * (q / 4) < kleft;
        src = xp + (int64_t)(16 * (q % 4)) * ldx + 16 * (q / 4);
      }
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst + 4u * kT * q),
                   "l"(ok ? src : X), "r"(ok ? 4 : 0));
    }
#pragma unroll
    for (int q = 0; q < NB; ++q) {
      const bool ok = fc + 8 * q < r && fk < kleft;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst + 4u * kT * (XQ + q)),
                   "l"(ok ? fp + 8 * q : F), "r"(ok ? 4 : 0));
    }
    xp += TRANS ? (int64_t)kKS * ldx : kKS;
    fp += (int64_t)kKS * ldf;
  };
  auto convert = [&](int buf) {
    const float* src = St + SLAB32 * buf + t;
#pragma unroll
    for (int q = 0; q < XQ; ++q) {
      const int kk = TRANS ? xk + 4 * q : xk + 16 * (q / 4);
      const int ii = TRANS ? xi : xi + 16 * (q % 4);
      Xs[kk * kXP + ii] = (double)src[kT * q];
    }
#pragma unroll
    for (int q = 0; q < NB; ++q) Fs[fk * FP + fc + 8 * q] = (double)src[kT * (XQ + q)];
  };
  request(k0, 0);
  asm volatile("cp.async.commit_group;");
  if (k0 + kKS < k1) request(k0 + kKS, 1);
  asm volatile("cp.async.commit_group;");
  int buf = 0;
  const double* xa = Xs + (lane & 3) * kXP + 16 * wr + (lane >> 2);
  const double* fb = Fs + (lane & 3) * FP + 8 * WNB * wc + (lane >> 2);
  for (int64_t ks = k0; ks < k1; ks += kKS, buf ^= 1) {
    asm volatile("cp.async.wait_group 1;" ::: "memory");   // this thread's requests of slab ks
    __syncthreads();                       // the previous slab's MMAs are done with Xs / Fs
    convert(buf);
    __syncthreads();
    if (ks + 2 * kKS < k1) request(ks + 2 * kKS, buf);
    asm volatile("cp.async.commit_group;");
#pragma unroll
    for (int kq = 0; kq < kKS / 4 / NG; ++kq) {
      const int k4 = 4 * (kq * NG + g);
      const double a0 = xa[k4 * kXP], a1 = xa[k4 * kXP + 8];
      double bv[WNB];
#pragma unroll
      for (int j = 0; j < WNB; ++j) bv[j] = fb[k4 * FP + 8 * j];
#pragma unroll
      for (int j = 0; j < WNB; ++j) {
        dmma884(acc[0][j][0], acc[0][j][1], a0, bv[j]);
        dmma884(acc[1][j][0], acc[1][j][1], a1, bv[j]);
      }
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  // groups 1 .. NG-1 hand their sums to group 0 through shared memory (over the slabs)
  const int w = t % GT;
  if (NG > 1) {
    double* red = Xs;                      // (NG - 1) x NA x GT doubles
    __syncthreads();
    if (g > 0) {
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < WNB; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e)
            red[((g - 1) * NA + (i * WNB + j) * 2 + e) * GT + w] = acc[i][j][e];
    }
    __syncthreads();
    if (g == 0) {
      for (int gg = 0; gg < NG - 1; ++gg)
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < WNB; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e)
              acc[i][j][e] += red[(gg * NA + (i * WNB + j) * 2 + e) * GT + w];
    }
  }
  if (g == 0) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int64_t row = r0 + 16 * wr + 8 * i + (lane >> 2);
      if (row >= M) continue;
#pragma unroll
      for (int j = 0; j < WNB; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = 8 * WNB * wc + 8 * j + 2 * (lane & 3) + e;
          if (c < r) out[row * r + c] = acc[i][j][e];
        }
    }
  }
  __syncthreads();                         // the next tile's slabs overwrite red
}

// All tiles of one pass: tile = (row block, K chunk); partial of chunk q at pp[q M r ...].
template <int RCOLS, bool TRANS>
__device__ __forceinline__ void product_pass(const float* __restrict__ X, int64_t ldx, int64_t M,
                                             int64_t K, const float* F, int64_t ldf, int r,
                                             int ksplit, int64_t kchunk, double* pp, double* Xs,
                                             double* Fs, float* St) {
  const int64_t nrb = (M + kTM - 1) / kTM;
  const int64_t tiles = nrb * ksplit;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int64_t rb = tile % nrb, q = tile / nrb;
    const int64_t k0 = q * kchunk, k1 = K < k0 + kchunk ? K : k0 + kchunk;
    product_tile<RCOLS, TRANS>(X, ldx, M, F, ldf, r, rb * kTM, k0, k1, pp + q * M * r, Xs, Fs, St);
  }
}

// G (r x r) = sum over the first nparts per-CTA partials, one entry per warp at a time: the
// lanes take the partials strided, then a fixed xor tree.
__device__ __forceinline__ void reduce_gram(const double* gp, int nparts, int r, double* G) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * kW + (threadIdx.x >> 5);
  const int nn = r * r;
  for (int64_t e = gw; e < nn; e += (int64_t)gridDim.x * kW) {
    double s = 0.0;
    for (int p = lane; p < nparts; p += 32) s += gp[(int64_t)p * nn + e];
    s = warp_sum(s);
    if (lane == 0) G[e] = s;
  }
}

// one warp (of the last CTA, the least likely to own HALS rows): sum (or min) of n partials
__device__ __forceinline__ double reduce_scalar(const double* parts, int n, bool is_min) {
  const int lane = threadIdx.x & 31;
  double s = is_min ? DBL_MAX : 0.0;
  for (int p = lane; p < n; p += 32) s = is_min ? fmin(s, parts[p]) : s + parts[p];
  return is_min ? warp_min(s) : warp_sum(s);
}

// (Dealing the 4-row blocks over the CTAs first -- one working warp per SM in a phase with few
// rows -- made the column sweep faster (C3 U 5.5 -> 3.8 us) but the partial sums slower
// (C2 U 6.3 -> 18.4 us, one warp per SM exposes every L2 round trip): 89 -> 107 us per C2 sweep,
// rejected.  Warps without rows now skip the sweep instead of running it on zeros.)
// (A lane-per-row form -- 32 rows per warp, rows k-major in shared memory, the column sweep
// blocked left-looking with 16 residuals in registers -- was built and measured: the sweep part
// took 14.7 / 6.5 / 4.7 us at C2 / C3 / C4 against 9.5 / 5.6 / 3.6 us here, one warp bound by
// the shared-memory wavefronts of the broadcast G rows; rejected, profiles/r02d_small_notes.md.)
// HALS on the rows of F (rows x r): C = sum of the ksplit tile partials, t = C - u G, then the
// Gauss-Seidel column sweep U_ik <- max(0, U_ik + (C_ik - sum_l U_il G_lk) / G_kk)
// (PAPER.md:322-324), F written in fp32; per-CTA partial Gram of the written rows, optional
// partial <C, F_new>, partial min.  Gs: the Gram in shared memory; Ss: kW x kRB x RP doubles.
template <int CPL, bool DBG>
__device__ __forceinline__ void hals_phase(float* F, int64_t ldf, int64_t rows, int r,
                                           const double* pp, int ksplit, const double* G,
                                           double* gpart, double* crosspart, double* minpart,
                                           double* Gs, double* Ss, double* ginv, double* red,
                                           unsigned long long* dbg) {
  constexpr int RP = 32 * CPL;
  auto hstamp = [&](int i) {               // ENMF_SMALL_DEBUG: phase-internal times of CTA 0
    if constexpr (DBG) {
      if (dbg && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(dbg[i]));
    }
  };
  hstamp(0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nblk = (rows + kRB - 1) / kRB;
  const bool cta_active = (int64_t)blockIdx.x * kW < nblk;
  double wmin = DBL_MAX, wcross = 0.0;
  if (cta_active) {
    load_gram<CPL>(G, r, Gs);
    for (int k = threadIdx.x; k < RP; k += kT) {
      const double gkk = k < r ? G[k * r + k] : 0.0;
      ginv[k] = gkk > 0.0 ? 1.0 / gkk : 0.0;
    }
    __syncthreads();
    hstamp(1);
    double* Sw = Ss + warp * kRB * RP;
    double* Cw = Ss + (kW + warp) * kRB * RP;      // this warp's C rows
    bool first = true;
    for (int64_t base = (int64_t)blockIdx.x * kW; base < nblk; base += (int64_t)gridDim.x * kW) {
      const int64_t rb = base + warp;
      double u[kRB][CPL], t[kRB][CPL];
      if (rb < nblk) {                              // (a warp without rows only zeroes its slot)
      // C rows of this warp: kRB consecutive rows are ONE contiguous span of cnt = rows * r
      // doubles in every K-chunk partial, so the lanes sum it flat (coalesced, 4 CPL loads in
      // flight per chunk, chunk order fixed) and scatter the sums into the warp's Cw[b][col]
      {
        const int64_t row0 = rb * kRB;
        const int64_t left = rb < nblk ? rows - row0 : 0;
        const int cnt = (int)(left < kRB ? left : kRB) * r;
        const double* src = pp + row0 * r + lane;
        const int64_t stride = rows * (int64_t)r;
        double sacc[kRB * CPL];
#pragma unroll
        for (int j = 0; j < kRB * CPL; ++j) sacc[j] = 0.0;
#pragma unroll 4
        for (int q = 0; q < ksplit; ++q) {
          double pv[kRB * CPL];
#pragma unroll
          for (int j = 0; j < kRB * CPL; ++j)
            pv[j] = lane + 32 * j < cnt ? __ldcg(src + q * stride + 32 * j) : 0.0;
#pragma unroll
          for (int j = 0; j < kRB * CPL; ++j) sacc[j] += pv[j];
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < kRB * CPL; ++j) {
          const int idx = lane + 32 * j;
          if (idx < cnt) Cw[(idx / r) * RP + idx % r] = sacc[j];
        }
        __syncwarp();
      }
#pragma unroll
      for (int b = 0; b < kRB; ++b)
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          const int64_t row = rb * kRB + b;
          const int col = lane + 32 * c;
          const bool ok = rb < nblk && row < rows && col < r;
          u[b][c] = ok ? (double)F[row * ldf + col] : 0.0;
          t[b][c] = ok ? Cw[b * RP + col] : 0.0;
        }
      hstamp(2);
      row_times_gram<CPL, kRB>(u, Gs, Sw, r, lane, -1.0, t);      // t = C - u G
      hstamp(3);
#pragma unroll
      for (int s = 0; s < CPL; ++s) {
        const int kmax = r - 32 * s < 32 ? r - 32 * s : 32;
        for (int kk = 0; kk < kmax; ++kk) {
          const int k = 32 * s + kk;
          const double ig = ginv[k];
          if (ig == 0.0) continue;                  // G_kk <= 0: column skipped (warp-uniform)
          double gk[CPL];
#pragma unroll
          for (int c = 0; c < CPL; ++c) gk[c] = Gs[k * RP + lane + 32 * c];
#pragma unroll
          for (int b = 0; b < kRB; ++b) {
            // lane kk owns (u_k, t_k); its change d is broadcast and the residual follows
            // u_k <- max(0, u_k + t_k / G_kk) as the change d = max(-u_k, t_k / G_kk) and
            // u_k + d: a multiply, a max and an add per row (the loop is bound by its
            // instruction count; forming v = fma(t, 1/G_kk, u), testing v > 0 and selecting
            // took ~25 instructions per row and step).  u_k + d is 0 exactly when the bound
            // is active; otherwise it differs from the fused form by <= 1/2 ulp of fp64.
            const double uo = u[b][s];
            const double dn = fmax(t[b][s] * ig, -uo);
            if (lane == kk) u[b][s] = uo + dn;
            const double d = __shfl_sync(FULL, dn, kk);
#pragma unroll
            for (int c = 0; c < CPL; ++c) t[b][c] = fma(-d, gk[c], t[b][c]);
          }
        }
      }
      }
      hstamp(4);
      // write the rows (fp32: the state), keep their rounded values for the Gram partial
      __syncwarp();
#pragma unroll
      for (int b = 0; b < kRB; ++b)
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          const int64_t row = rb * kRB + b;
          const int col = lane + 32 * c;
          double w = 0.0;
          if (rb < nblk && row < rows && col < r) {
            const float v = (float)u[b][c];
            F[row * ldf + col] = v;
            w = (double)v;
            wmin = fmin(wmin, w);
            wcross = fma(Cw[b * RP + col], w, wcross);
          }
          Sw[b * RP + col] = w;
        }
      __syncthreads();
      hstamp(5);
      // partial Gram of this round's kW * kRB rows: 4 x 4 blocks of the upper block triangle
      {
        const int nb4 = (r + 3) / 4;
        const int npair = nb4 * (nb4 + 1) / 2;
        for (int p = threadIdx.x; p < npair; p += kT) {
          // p -> (a, b), a <= b, row-major over the upper triangle
          int a = 0, rem = p;
          while (rem >= nb4 - a) { rem -= nb4 - a; ++a; }
          const int b = a + rem;
          double g[4][4];
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) g[i][j] = 0.0;
          for (int row = 0; row < kW * kRB; ++row) {
            const double2 a01 = *reinterpret_cast<const double2*>(Ss + row * RP + 4 * a);
            const double2 a23 = *reinterpret_cast<const double2*>(Ss + row * RP + 4 * a + 2);
            const double2 b01 = *reinterpret_cast<const double2*>(Ss + row * RP + 4 * b);
            const double2 b23 = *reinterpret_cast<const double2*>(Ss + row * RP + 4 * b + 2);
            const double av[4] = {a01.x, a01.y, a23.x, a23.y};
            const double bv[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
              for (int j = 0; j < 4; ++j) g[i][j] = fma(av[i], bv[j], g[i][j]);
          }
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int ci = 4 * a + i, cj = 4 * b + j;
              if (ci < r && cj < r) {
                const double val = first ? g[i][j] : gpart[ci * r + cj] + g[i][j];
                gpart[ci * r + cj] = val;
                if (a != b) gpart[cj * r + ci] = val;
              }
            }
        }
      }
      first = false;
      __syncthreads();
      hstamp(6);
    }
  }
  // per-CTA scalars (every CTA writes: the reductions read all gridDim slots)
  wmin = warp_min(wmin);
  wcross = warp_sum(wcross);
  if (lane == 0) {
    red[warp] = wmin;
    red[kW + warp] = wcross;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double mn = DBL_MAX, cr = 0.0;
    for (int w = 0; w < kW; ++w) {
      mn = fmin(mn, red[w]);
      cr += red[kW + w];
    }
    minpart[blockIdx.x] = mn;
    if (crosspart) crosspart[blockIdx.x] = cr;
  }
  __syncthreads();
  hstamp(7);
}

// f = ||X||^2 - 2 <Q, V> + <G_U, G_V> (one CTA: the last), appended to the trace
__device__ __forceinline__ void objective_append(const SmallArgs& a, double cross, double* red) {
  const int nn = a.r * a.r;
  double s = 0.0;
  for (int e = threadIdx.x; e < nn; e += kT) s = fma(a.GU[e], a.GV[e], s);
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double g = 0.0;
    for (int w = 0; w < kW; ++w) g += red[w];
    a.ftrace[(*a.fcnt)++] = *a.xnorm2 - 2.0 * cross + g;
  }
  __syncthreads();
}

template <int CPL, int RCOLS, bool DBG>
__global__ void __launch_bounds__(kT, CPL <= 2 ? 2 : 1) small_hals_kernel(SmallArgs a) {
  constexpr int RP = 32 * CPL;
  extern __shared__ double smem[];
  // product phases: Xs (kKS x kXP) + Fs (kKS x FP) [+ staging]; HALS phases: Gs + Ss + ginv
  double* Xs = smem;
  double* Fs = smem + kKS * kXP;
  double* Gs = smem;
  double* Ss = smem + RP * RP;
  double* ginv = Ss + 2 * kW * kRB * RP;
  constexpr int PRODD = TileShape<RCOLS>::PRODD;
  float* St = reinterpret_cast<float*>(smem + PRODD);   // 2 staged fp32 slabs
  __shared__ double red[2 * kW];
  unsigned bar_target = 0;
  unsigned* bar = a.bar;
  auto grid_sync = [&]() { grid_barrier(bar, bar_target); };
  const int G = (int)gridDim.x;
  const int r = a.r;
  const int64_t nblkU = (a.m + kRB - 1) / kRB, nblkV = (a.n + kRB - 1) / kRB;
  const int64_t ctaU = (nblkU + kW - 1) / kW, ctaV = (nblkV + kW - 1) / kW;
  const int actU = ctaU < G ? (int)ctaU : G;      // CTAs that write a Gram partial
  const int actV = ctaV < G ? (int)ctaV : G;
  double* crossp = a.sc;
  double* minp = a.sc + G;
  double* scal = a.sc + 2 * G;               // [0] cross, [1] min U, [2] min V
  unsigned long long tl[6] = {0, 0, 0, 0, 0, 0}, hu[8] = {0}, hv[8] = {0};
  const bool dbg0 = DBG && a.debug && blockIdx.x == 0;
  auto stamp = [&](int i) {
    if constexpr (DBG) {
      if (a.debug && blockIdx.x == 0 && threadIdx.x == 0)
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tl[i]));
    }
  };
  unsigned long long gt0 = 0;
  long long ck0 = 0;
  if (DBG && dbg0 && threadIdx.x == 0) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt0));
    ck0 = clock64();
  }
  for (int t = 0; t < a.count; ++t) {
    stamp(0);
    // ---- A: (G_V, <Q, V>, min V of the previous sweep;) partial products of P = X V
    if (t > 0) {
      reduce_gram(a.gp, actV, r, a.GV);
      if (blockIdx.x == gridDim.x - 1 && threadIdx.x < 32) {
        const double cr = reduce_scalar(crossp, G, false);
        const double mv = reduce_scalar(minp, G, true);
        if (threadIdx.x == 0) {
          scal[0] = cr;
          scal[2] = mv;
        }
      }
    }
    product_pass<RCOLS, false>(a.X, a.ldx, a.m, a.n, a.V, a.ldv, r, a.ksA, a.kcA, a.pp, Xs, Fs, St);
    stamp(5);
    grid_sync();
    stamp(1);
    // ---- A': (objective of the previous sweep;) HALS on U
    if (t > 0 && blockIdx.x == gridDim.x - 1) objective_append(a, scal[0], red);
    hals_phase<CPL, DBG>(a.U, a.ldu, a.m, r, a.pp, a.ksA, a.GV, a.gp + (int64_t)blockIdx.x * r * r,
                    nullptr, minp, Gs, Ss, ginv, red, dbg0 ? hu : nullptr);
    grid_sync();
    stamp(2);
    // ---- B: G_U, min U; partial products of Q = X^T U
    reduce_gram(a.gp, actU, r, a.GU);
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x < 32) {
      const double mu = reduce_scalar(minp, G, true);
      if (threadIdx.x == 0) scal[1] = mu;
    }
    product_pass<RCOLS, true>(a.X, a.ldx, a.n, a.m, a.U, a.ldu, r, a.ksB, a.kcB, a.pp, Xs, Fs, St);
    grid_sync();
    stamp(3);
    // ---- B': HALS on V with the cross-term partial <Q, V_new>
    hals_phase<CPL, DBG>(a.V, a.ldv, a.n, r, a.pp, a.ksB, a.GU, a.gp + (int64_t)blockIdx.x * r * r,
                    crossp, minp, Gs, Ss, ginv, red, dbg0 ? hv : nullptr);
    grid_sync();
    stamp(4);
  }
  if (DBG && a.debug && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long gt1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt1));
    printf("  SM clock %.0f MHz over %d sweeps\n", 1e3 * (double)(clock64() - ck0) / (double)(gt1 - gt0),
           a.count);
  }
  if (DBG && a.debug && blockIdx.x == 0 && threadIdx.x == 0)
    printf("small_hals grid %d ksA %d kcA %d ksB %d kcB %d: A %llu (own work %llu) A' %llu B %llu B' %llu ns\n",
           G, a.ksA, (int)a.kcA, a.ksB, (int)a.kcB, tl[1] - tl[0], tl[5] - tl[0], tl[2] - tl[1],
           tl[3] - tl[2], tl[4] - tl[3]);
  if (DBG && a.debug && blockIdx.x == 0 && threadIdx.x == 0)
    printf("  CTA 0 HALS U: gram %llu partials %llu uG %llu sweep %llu write %llu Gpart %llu tail %llu | "
           "V: gram %llu partials %llu uG %llu sweep %llu write %llu Gpart %llu tail %llu ns\n",
           hu[1] - hu[0], hu[2] - hu[1], hu[3] - hu[2], hu[4] - hu[3], hu[5] - hu[4], hu[6] - hu[5],
           hu[7] - hu[6], hv[1] - hv[0], hv[2] - hv[1], hv[3] - hv[2], hv[4] - hv[3], hv[5] - hv[4],
           hv[6] - hv[5], hv[7] - hv[6]);
  // ---- tail: G_V, <Q, V>, min V of the last sweep, its objective, the handle's scalars
  reduce_gram(a.gp, actV, r, a.GV);
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x < 32) {
    const double cr = reduce_scalar(crossp, G, false);
    const double mv = reduce_scalar(minp, G, true);
    if (threadIdx.x == 0) {
      scal[0] = cr;
      scal[2] = mv;
    }
  }
  grid_sync();
  if (blockIdx.x == gridDim.x - 1) {
    objective_append(a, scal[0], red);
    if (threadIdx.x == 0) {
      *a.minu = scal[1];
      *a.minv = scal[2];
      *a.stage = 1;
      *a.cnt_hals += a.count;
    }
  }
}

template <int CPL, int RCOLS>
size_t smem_bytes() {
  constexpr int RP = 32 * CPL;
  using TS = TileShape<RCOLS>;
  const size_t prod = (size_t)TS::PRODD + (size_t)TS::SLAB32;     // fp64 slabs + 2 staged fp32
  const size_t hals = (size_t)(RP * RP + 2 * kW * kRB * RP + RP);
  return sizeof(double) * std::max(prod, hals);
}

// K split of a product pass: tiles = row blocks x ksplit on G CTAs; the cost of a pass is
// (waves of tiles) x (chunk length + a fixed per-tile latency, in K units)
void choose_split(int64_t M, int64_t K, int G, int* ksplit, int64_t* kchunk) {
  const int64_t nrb = (M + kTM - 1) / kTM;
  const int64_t kmax = std::max<int64_t>(1, (K + 63) / 64);
  double best = 1e300;
  int64_t bk = 1;
  for (int64_t ks = 1; ks <= kmax && ks <= 4096; ++ks) {
    int64_t kc = ((K + ks - 1) / ks + kKS - 1) / kKS * kKS;
    if (kc < kKS) kc = kKS;
    const int64_t real = (K + kc - 1) / kc;
    const int64_t waves = (nrb * real + G - 1) / G;
    // (+ ~0.25 us per chunk in the row phase that sums the chunk partials: ~8 k of FMAs)
    const double cost = (double)waves * ((double)kc + 96.0) + 8.0 * (double)real;
    if (cost < best) {
      best = cost;
      bk = ks;
    }
    if (nrb * ks > 8 * (int64_t)G) break;
  }
  int64_t kc = ((K + bk - 1) / bk + kKS - 1) / kKS * kKS;
  if (kc < kKS) kc = kKS;
  *kchunk = kc;
  *ksplit = (int)std::max<int64_t>(1, (K + kc - 1) / kc);
}

struct Plan {
  int grid = 0, ksA = 1, ksB = 1;
  int64_t kcA = 0, kcB = 0;
  size_t smem = 0;
  const void* fn = nullptr;
};

bool timeline_requested() {                 // ENMF_SMALL_DEBUG=1: the instrumented instantiation
  const char* dbg = getenv("ENMF_SMALL_DEBUG");
  return dbg && dbg[0] == '1';
}

template <int CPL, int RCOLS>
bool make_plan_t(int64_t m, int64_t n, Plan* p) {
  auto k = timeline_requested() ? small_hals_kernel<CPL, RCOLS, true>
                                : small_hals_kernel<CPL, RCOLS, false>;
  const size_t sm = smem_bytes<CPL, RCOLS>();
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kT, sm) != cudaSuccess || occ < 1) {
    cudaGetLastError();
    return false;
  }
  if (occ > 2) occ = 2;
  int dev = 0, sms = kSMs;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int gmax = occ * sms;
  choose_split(m, n, gmax, &p->ksA, &p->kcA);
  choose_split(n, m, gmax, &p->ksB, &p->kcB);
  const int64_t tilesA = (m + kTM - 1) / kTM * p->ksA, tilesB = (n + kTM - 1) / kTM * p->ksB;
  const int64_t hu = ((m + kRB - 1) / kRB + kW - 1) / kW, hv = ((n + kRB - 1) / kRB + kW - 1) / kW;
  const int64_t want = std::max(std::max(tilesA, tilesB), std::max(hu, hv));
  p->grid = (int)std::max<int64_t>(1, std::min<int64_t>(gmax, want));
  p->smem = sm;
  p->fn = reinterpret_cast<const void*>(k);
  return true;
}

bool make_plan(int64_t m, int64_t n, int r, Plan* p) {
  if (r <= 16) return make_plan_t<1, 16>(m, n, p);
  if (r <= 24) return make_plan_t<1, 24>(m, n, p);
  if (r <= 32) return make_plan_t<1, 32>(m, n, p);
  if (r <= 64) return make_plan_t<2, 64>(m, n, p);
  if (r <= 96) return make_plan_t<3, 128>(m, n, p);
  if (r <= 128) return make_plan_t<4, 128>(m, n, p);
  return false;
}

}  // namespace

bool small_sweeps_supported(int64_t m, int64_t n, int r) {
  // cache-resident problems (C1-C4, X <= 90 MB); larger ones are bound by the X
  // passes, which have their own kernels
  return r >= 1 && r <= 128 && m >= 1 && n >= 1 && m * n <= (int64_t)64 * 1024 * 1024;
}

size_t small_sweeps_workspace(int64_t m, int64_t n, int r) {
  Plan p;
  if (!make_plan(m, n, r, &p)) return 0;
  const size_t pp = (size_t)std::max(p.ksA * m, p.ksB * n) * r;
  return pp + (size_t)p.grid * r * r + 2 * (size_t)p.grid + 8 + 16;
}

int small_sweeps_launch(const float* X, int64_t ldx, int64_t m, int64_t n, int r, float* U,
                        int64_t ldu, float* V, int64_t ldv, double* GV, double* GU,
                        const double* xnorm2, double* ftrace, int* fcnt, double* minu,
                        double* minv, int* stage, int* cnt_hals, double* ws, int count,
                        cudaStream_t st) {
  if (count <= 0) return 0;
  Plan p;
  if (!make_plan(m, n, r, &p)) return 1;
  SmallArgs a;
  a.X = X; a.ldx = ldx; a.m = m; a.n = n; a.r = r;
  a.U = U; a.ldu = ldu; a.V = V; a.ldv = ldv;
  a.GV = GV; a.GU = GU; a.xnorm2 = xnorm2; a.ftrace = ftrace; a.fcnt = fcnt;
  a.minu = minu; a.minv = minv; a.stage = stage; a.cnt_hals = cnt_hals;
  a.pp = ws;
  a.gp = ws + (size_t)std::max(p.ksA * m, p.ksB * n) * r;
  a.sc = a.gp + (size_t)p.grid * r * r;
  a.bar = reinterpret_cast<unsigned*>(a.sc + 2 * (size_t)p.grid + 8);
  a.ksA = p.ksA; a.ksB = p.ksB; a.kcA = p.kcA; a.kcB = p.kcB;
  a.count = count;
  a.debug = timeline_requested() ? 1 : 0;
  // (the barrier counter advances by 4 grid sizes per sweep: launches of <= 2^18 sweeps)
  for (int done = 0; done < count; done += 1 << 18) {
    a.count = count - done < (1 << 18) ? count - done : 1 << 18;
    if (cudaMemsetAsync(a.bar, 0, 16 * sizeof(double), st) != cudaSuccess) return 1;
    void* args[] = {&a};
    if (cudaLaunchCooperativeKernel(p.fn, dim3(p.grid), dim3(kT), args, p.smem, st) != cudaSuccess)
      return 1;
    count_launch();
  }
  return 0;
}

}  // namespace enmf
