/*
 * synth_cpu.c -- host side of the synthetic-input generator (see synth_core.h).
 * Test / bench infrastructure: produces X row ranges bit-identical to
 * synth_gpu.cu.  Compile with -ffp-contract=off (no FMA contraction).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include "synth_core.h"

/* Philox known-answer access for tests. */
void synth_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  syn_u32x4 r = syn_philox(ctr[0], ctr[1], ctr[2], ctr[3], key[0], key[1]);
  for (int i = 0; i < 4; ++i) out[i] = r.v[i];
}

double synth_normal(uint64_t seed, uint32_t stream, uint64_t idx) {
  return syn_normal(seed, stream, idx);
}
double synth_log(double x) { return syn_log(x); }
double synth_cos2pi(double u) { return syn_cos2pi(u); }

/* Row factor rows [begin, begin+count) x k, or column factor (which=1). */
void synth_factor(int recipe, uint64_t seed, int which, int64_t begin, int64_t count,
                  int k, float* out) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < count; ++r)
    for (int c = 0; c < k; ++c)
      out[r * k + c] = which == 0 ? syn_rowf(recipe, seed, (uint64_t)(begin + r), k, c)
                                  : syn_colf(recipe, seed, (uint64_t)(begin + r), k, c);
}

/* max over all (i,j) of S_ij = A_i . B_j (IMAGE normalisation, reading R21). */
double synth_smax(int recipe, uint64_t seed, int64_t m, int64_t n, int k) {
  float* A = (float*)malloc(sizeof(float) * (size_t)m * k);
  float* B = (float*)malloc(sizeof(float) * (size_t)n * k);
  synth_factor(recipe, seed, 0, 0, m, k, A);
  synth_factor(recipe, seed, 1, 0, n, k, B);
  double best = 0.0;
#pragma omp parallel for schedule(static) reduction(max : best)
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double s = syn_dot(A + i * k, B + j * k, k);
      if (s > best) best = s;
    }
  free(A);
  free(B);
  return best;
}

/* Block X[r0:r0+rc, c0:c0+cc] of an m x n matrix into out (ld = ldo). */
int synth_x_block(int recipe, uint64_t seed, int64_t m, int64_t n, int k, double noise,
                  double smax, int64_t r0, int64_t rc, int64_t c0, int64_t cc, float* out,
                  int64_t ldo) {
  if (r0 < 0 || rc < 0 || r0 + rc > m || c0 < 0 || cc < 0 || c0 + cc > n || ldo < cc) return -1;
  float* A = NULL;
  float* B = NULL;
  if (recipe != SYN_RATINGS) {
    A = (float*)malloc(sizeof(float) * (size_t)(rc > 0 ? rc : 1) * k);
    B = (float*)malloc(sizeof(float) * (size_t)(cc > 0 ? cc : 1) * k);
    synth_factor(recipe, seed, 0, r0, rc, k, A);
    synth_factor(recipe, seed, 1, c0, cc, k, B);
  }
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < rc; ++r)
    for (int64_t c = 0; c < cc; ++c) {
      double s = recipe == SYN_RATINGS ? 0.0 : syn_dot(A + r * k, B + c * k, k);
      out[r * ldo + c] = syn_x_from_s(recipe, seed, (uint64_t)(r0 + r), (uint64_t)(c0 + c),
                                      (uint64_t)n, s, noise, smax);
    }
  free(A);
  free(B);
  return 0;
}

/* X rows [row_begin, row_begin+row_count) of an m x n matrix into out (ld = ldo). */
int synth_x_rows(int recipe, uint64_t seed, int64_t m, int64_t n, int k, double noise,
                 double smax, int64_t row_begin, int64_t row_count, float* out, int64_t ldo) {
  if (row_begin < 0 || row_count < 0 || row_begin + row_count > m || ldo < n) return -1;
  float* A = NULL;
  float* B = NULL;
  if (recipe != SYN_RATINGS) {
    A = (float*)malloc(sizeof(float) * (size_t)(row_count > 0 ? row_count : 1) * k);
    B = (float*)malloc(sizeof(float) * (size_t)n * k);
    synth_factor(recipe, seed, 0, row_begin, row_count, k, A);
    synth_factor(recipe, seed, 1, 0, n, k, B);
  }
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < row_count; ++r) {
    uint64_t i = (uint64_t)(row_begin + r);
    for (int64_t j = 0; j < n; ++j) {
      double s = recipe == SYN_RATINGS ? 0.0 : syn_dot(A + r * k, B + j * k, k);
      out[r * ldo + j] = syn_x_from_s(recipe, seed, i, (uint64_t)j, (uint64_t)n, s, noise, smax);
    }
  }
  free(A);
  free(B);
  return 0;
}

/* SPARSE recipe as CSR rows [row_begin, row_begin + row_count) (columns ascending).
 * rowptr == NULL: returns the entry count of the range; else fills rowptr (row_count + 1,
 * rowptr[0] = 0), colidx and vals (capacity cap) and returns the count (-1 on overflow). */
int64_t synth_csr_rows(uint64_t seed, int64_t m, int64_t n, int k, double noise, double density,
                       int64_t row_begin, int64_t row_count, int64_t* rowptr, int32_t* colidx,
                       float* vals, int64_t cap) {
  if (row_begin < 0 || row_count < 0 || row_begin + row_count > m) return -1;
  int64_t nnz = 0;
  float* A = NULL;
  float* B = NULL;
  if (rowptr) {
    A = (float*)malloc(sizeof(float) * (size_t)(row_count > 0 ? row_count : 1) * k);
    B = (float*)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1) * k);
    synth_factor(SYN_SPARSE, seed, 0, row_begin, row_count, k, A);
    synth_factor(SYN_SPARSE, seed, 1, 0, n, k, B);
    rowptr[0] = 0;
  }
  for (int64_t r = 0; r < row_count; ++r) {
    uint64_t i = (uint64_t)(row_begin + r);
    for (int64_t j = 0; j < n; ++j) {
      if (!syn_sparse_keep(seed, i, (uint64_t)j, (uint64_t)n, density)) continue;
      if (rowptr) {
        if (nnz >= cap) { free(A); free(B); return -1; }
        double s = syn_dot(A + r * k, B + j * k, k);
        colidx[nnz] = (int32_t)j;
        vals[nnz] = syn_x_from_s(SYN_SPARSE, seed, i, (uint64_t)j, (uint64_t)n, s, noise, density);
      }
      ++nnz;
    }
    if (rowptr) rowptr[r + 1] = nnz;
  }
  free(A);
  free(B);
  return nnz;
}
