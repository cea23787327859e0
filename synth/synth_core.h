/*
 * synth_core.h -- seeded, counter-based synthetic-input recipes.
 *
 * This module is the ONLY code shared by the CPU oracle tests and the GPU
 * product path: it draws the synthetic matrices X of BASELINE.json:7-11 and
 * holds none of the eNMF method's arithmetic.  The same source is compiled
 * for the host (gcc, -ffp-contract=off) and the device (nvcc, --fmad=false),
 * and every floating-point step is a single IEEE +,-,*,/ or sqrt (no libm),
 * so both sides produce bit-identical X.
 *
 * Generator: Philox4x32-10 (Salmon et al., SC'11), key = seed, counter =
 * (element index lo, element index hi, stream id, 0).  Streams are indexed
 * by the GLOBAL element index, so any row range (any shard) is generated
 * identically on any device and for any GPU count.
 *
 * Recipes (SURVEY.md §8(d) and readings R21-R24):
 *   PLANTED  X = A B^T + noise*|z|, A (m x k), B (n x k) ~ U[0,1)   (C1, C5)
 *   IMAGE    X = clip(S/max S + 0.05|z|, 0, 1), S = A B^T,
 *            A = u*[u'<0.3], B = Exp(1)                              (C2, R21)
 *   SPECTRO  X = A B^T + 0.01|z|, A = z^2/2 (Gamma(.5,1)),
 *            B = Exp(1)*[u>=0.7]                                     (C3, R22)
 *   RATINGS  X_ij = c in {1..5} w.p. 0.045, cat(.06,.11,.26,.35,.22);
 *            else 0                                                  (C4, R23)
 *   SPARSE   X_ij = (A B^T)_ij + noise*|z| w.p. density (A, B as PLANTED), else 0:
 *            the stand-in for the sparse Reuters matrix (
 *            density is passed in the smax argument)                 (C6, R27)
 * Factor entries are rounded to fp32 before the inner product, so every
 * product A_ic*B_jc is exact in fp64; the k-sum runs in ascending c order.
 */
#ifndef SYNTH_CORE_H
#define SYNTH_CORE_H

#include <stdint.h>
#include <math.h>

#ifdef __CUDACC__
#define SYN_FN static __host__ __device__ __forceinline__
#else
#define SYN_FN static inline
#endif

enum { SYN_PLANTED = 1, SYN_IMAGE = 2, SYN_SPECTRO = 3, SYN_RATINGS = 4, SYN_SPARSE = 5 };
enum { SYN_STREAM_ROWF = 1, SYN_STREAM_COLF = 2, SYN_STREAM_NOISE = 3, SYN_STREAM_X = 4 };

typedef struct { uint32_t v[4]; } syn_u32x4;

SYN_FN uint32_t syn_mulhilo(uint32_t a, uint32_t b, uint32_t* hi) {
  uint64_t p = (uint64_t)a * (uint64_t)b;
  *hi = (uint32_t)(p >> 32);
  return (uint32_t)p;
}

/* Philox4x32 with 10 rounds. */
SYN_FN syn_u32x4 syn_philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                            uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, hi1;
    uint32_t lo0 = syn_mulhilo(0xD2511F53u, c0, &hi0);
    uint32_t lo1 = syn_mulhilo(0xCD9E8D57u, c2, &hi1);
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
  syn_u32x4 out; out.v[0] = c0; out.v[1] = c1; out.v[2] = c2; out.v[3] = c3;
  return out;
}

SYN_FN syn_u32x4 syn_draw(uint64_t seed, uint32_t stream, uint64_t idx) {
  return syn_philox((uint32_t)idx, (uint32_t)(idx >> 32), stream, 0u,
                    (uint32_t)seed, (uint32_t)(seed >> 32));
}

/* u in [0,1) with 24 random bits: exact in fp32. */
SYN_FN double syn_u01(uint32_t w) { return (double)(w >> 8) * (1.0 / 16777216.0); }
/* u in (0,1]. */
SYN_FN double syn_u01_open0(uint32_t w) { return (double)((w >> 8) + 1u) * (1.0 / 16777216.0); }

/* Natural log for x in (0, 1] from +,-,*,/ only (atanh series after an
 * exact binary-exponent split).  Accurate to ~1e-15 relative; what matters
 * here is that host and device evaluate the identical operation sequence. */
SYN_FN double syn_log(double x) {
  int e = 0;
  /* x in (0,1]: scale into [1,2) by exact multiplications by 2. */
  while (x < 1.0) { x = x * 2.0; e -= 1; }
  if (x > 1.4142135623730951) { x = x * 0.5; e += 1; }
  double s = (x - 1.0) / (x + 1.0);
  double s2 = s * s;
  double p = 1.0 / 27.0;
  p = p * s2 + 1.0 / 25.0;
  p = p * s2 + 1.0 / 23.0;
  p = p * s2 + 1.0 / 21.0;
  p = p * s2 + 1.0 / 19.0;
  p = p * s2 + 1.0 / 17.0;
  p = p * s2 + 1.0 / 15.0;
  p = p * s2 + 1.0 / 13.0;
  p = p * s2 + 1.0 / 11.0;
  p = p * s2 + 1.0 / 9.0;
  p = p * s2 + 1.0 / 7.0;
  p = p * s2 + 1.0 / 5.0;
  p = p * s2 + 1.0 / 3.0;
  p = p * s2 + 1.0;
  return (double)e * 0.6931471805599453 + 2.0 * s * p;
}

/* sin and cos of t in [0, pi/2] by Taylor series (Horner). */
SYN_FN double syn_sin_q(double t) {
  double t2 = t * t;
  double p = 1.0 / 355687428096000.0;             /* 1/17! */
  p = p * t2 - 1.0 / 1307674368000.0;             /* -1/15! */
  p = p * t2 + 1.0 / 6227020800.0;                /* 1/13!  */
  p = p * t2 - 1.0 / 39916800.0;                  /* 1/11!  */
  p = p * t2 + 1.0 / 362880.0;
  p = p * t2 - 1.0 / 5040.0;
  p = p * t2 + 1.0 / 120.0;
  p = p * t2 - 1.0 / 6.0;
  p = p * t2 + 1.0;
  return t * p;
}
SYN_FN double syn_cos_q(double t) {
  double t2 = t * t;
  double p = -1.0 / 6402373705728000.0;           /* -1/18! */
  p = p * t2 + 1.0 / 20922789888000.0;            /* 1/16! */
  p = p * t2 - 1.0 / 87178291200.0;               /* 1/14! */
  p = p * t2 + 1.0 / 479001600.0;
  p = p * t2 - 1.0 / 3628800.0;
  p = p * t2 + 1.0 / 40320.0;
  p = p * t2 - 1.0 / 720.0;
  p = p * t2 + 1.0 / 24.0;
  p = p * t2 - 1.0 / 2.0;
  p = p * t2 + 1.0;
  return p;
}
/* cos(2*pi*u) for u in [0,1) (u has 24 bits, so 4u and its split are exact). */
SYN_FN double syn_cos2pi(double u) {
  double f4 = u * 4.0;
  int q = (int)f4;
  double t = (f4 - (double)q) * 1.5707963267948966;
  switch (q & 3) {
    case 0: return syn_cos_q(t);
    case 1: return -syn_sin_q(t);
    case 2: return -syn_cos_q(t);
    default: return syn_sin_q(t);
  }
}

/* Standard normal by Box-Muller from one Philox draw. */
SYN_FN double syn_normal(uint64_t seed, uint32_t stream, uint64_t idx) {
  syn_u32x4 w = syn_draw(seed, stream, idx);
  double u1 = syn_u01_open0(w.v[0]);
  double u2 = syn_u01(w.v[1]);
  double l = syn_log(u1);
  double rad = -2.0 * l;
  double sq = rad > 0.0 ? sqrt(rad) : 0.0;
  return sq * syn_cos2pi(u2);
}

SYN_FN double syn_exp1(uint32_t w) {           /* Exp(1) = -ln(1-u) */
  double u = syn_u01(w);
  return -syn_log(1.0 - u);
}

/* Row-factor entry A[i][c] (global row i). */
SYN_FN float syn_rowf(int recipe, uint64_t seed, uint64_t i, int k, int c) {
  uint64_t idx = i * (uint64_t)k + (uint64_t)c;
  syn_u32x4 w = syn_draw(seed, SYN_STREAM_ROWF, idx);
  switch (recipe) {
    case SYN_IMAGE: {
      double u = syn_u01(w.v[0]);
      double keep = syn_u01(w.v[1]);
      return keep < 0.3 ? (float)u : 0.0f;
    }
    case SYN_SPECTRO: {
      double z = syn_normal(seed, SYN_STREAM_ROWF, idx);
      return (float)(z * z * 0.5);
    }
    default:
      return (float)syn_u01(w.v[0]);
  }
}

/* Column-factor entry B[j][c]. */
SYN_FN float syn_colf(int recipe, uint64_t seed, uint64_t j, int k, int c) {
  uint64_t idx = j * (uint64_t)k + (uint64_t)c;
  syn_u32x4 w = syn_draw(seed, SYN_STREAM_COLF, idx);
  switch (recipe) {
    case SYN_IMAGE:
      return (float)syn_exp1(w.v[0]);
    case SYN_SPECTRO: {
      double keep = syn_u01(w.v[1]);
      return keep >= 0.7 ? (float)syn_exp1(w.v[0]) : 0.0f;
    }
    default:
      return (float)syn_u01(w.v[0]);
  }
}

/* S_ij = sum_c A_ic B_jc in fp64, ascending c (products exact). */
SYN_FN double syn_dot(const float* a, const float* b, int k) {
  double s = 0.0;
  for (int c = 0; c < k; ++c) s = s + (double)a[c] * (double)b[c];
  return s;
}

/* SPARSE support: entry (i, j) is stored w.p. density (X stream, word 0). */
SYN_FN int syn_sparse_keep(uint64_t seed, uint64_t i, uint64_t j, uint64_t n, double density) {
  syn_u32x4 w = syn_draw(seed, SYN_STREAM_X, i * n + j);
  return syn_u01(w.v[0]) < density;
}

/* Final X_ij from the planted inner product S (ignored for RATINGS).
 * smax: global max of S (IMAGE recipe, normalised reading R21; <=0 selects
 * the literal unnormalised reading). */
SYN_FN float syn_x_from_s(int recipe, uint64_t seed, uint64_t i, uint64_t j,
                          uint64_t n, double s, double noise, double smax) {
  uint64_t e = i * n + j;
  switch (recipe) {
    case SYN_RATINGS: {
      syn_u32x4 w = syn_draw(seed, SYN_STREAM_X, e);
      double u = syn_u01(w.v[0]);
      if (!(u < 0.045)) return 0.0f;
      double c = syn_u01(w.v[1]);
      if (c < 0.06) return 1.0f;
      if (c < 0.17) return 2.0f;
      if (c < 0.43) return 3.0f;
      if (c < 0.78) return 4.0f;
      return 5.0f;
    }
    case SYN_SPARSE: {
      if (!syn_sparse_keep(seed, i, j, n, smax)) return 0.0f;
      double z = syn_normal(seed, SYN_STREAM_NOISE, e);
      double az = z < 0.0 ? -z : z;
      return (float)(s + noise * az);
    }
    case SYN_IMAGE: {
      double z = syn_normal(seed, SYN_STREAM_NOISE, e);
      double az = z < 0.0 ? -z : z;
      double base = smax > 0.0 ? s / smax : s;
      double v = base + noise * az;
      if (v < 0.0) v = 0.0;
      if (v > 1.0) v = 1.0;
      return (float)v;
    }
    default: {
      double z = syn_normal(seed, SYN_STREAM_NOISE, e);
      double az = z < 0.0 ? -z : z;
      return (float)(s + noise * az);
    }
  }
}

#endif
