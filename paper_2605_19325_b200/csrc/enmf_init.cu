// enmf_init.cu -- initialisation of Alg. 3: randomised truncated SVD with
// balanced scaling and the ADMM rotation of Alg. 1,
// plus the host-buffer end-to-end entry point.
#include <math.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "handle.h"

using namespace enmf;

namespace {

// Init workspaces: a handle-owned arena (h->arena, grown on demand and kept until
// enmf_destroy) handed out bump-style per call -- the rotation alone needs ~1 GB at C5, and a
// cudaMalloc / cudaFree of that per call costs more than the 100 ADMM steps' Procrustes work.
// The arena is grown only between calls; a call that needs more than the current capacity
// allocates the full requirement first (first-fit by size recorded in h->arena_need).
struct DevBuf {
  enmf_handle_t h;
  size_t used = 0;
  bool overflow = false;
  explicit DevBuf(enmf_handle_t hh) : h(hh) {}
  ~DevBuf() {
    if (used > h->arena_need) h->arena_need = used;
  }
  template <typename T>
  enmf_status_t get(T** p, size_t count) {
    const size_t bytes = ((sizeof(T) * (count ? count : 1)) + 255) & ~(size_t)255;
    if (used + bytes > h->arena_bytes) {
      // grow: free the old arena (the stream is idle at the start of an init call) and
      // allocate the larger of the recorded need and what this call needs so far
      if (used != 0) {
        // buffers already handed out live in the old arena: fall back to a private allocation
        overflow = true;
        enmf_status_t s = dalloc(p, count);
        if (s == ENMF_OK) h->arena_extra.push_back((void*)*p);
        return s;
      }
      if (h->arena) cudaFree(h->arena);
      h->arena = nullptr;
      h->arena_bytes = 0;
      const size_t want = std::max(h->arena_need, bytes);
      enmf_status_t s = dalloc_bytes((void**)&h->arena, want);
      if (s != ENMF_OK) return s;
      h->arena_bytes = want;
    }
    *p = reinterpret_cast<T*>(h->arena + used);
    used += bytes;
    return ENMF_OK;
  }
};

// CholeskyQR2 (first pass shifted): A (rows x l, fp64, ld l) <- A R^{-1}, columns orthonormal.
enmf_status_t cholqr(enmf_handle_t h, double* A, double* tmp, int64_t rows, int l,
                     bool sharded, double* G, double* R, double* Rinv, int* bad) {
  for (int pass = 0; pass < 2; ++pass) {
    GemmOut o;
    o.C = G;
    o.ldc = l;
    gemm<double, double>(true, A, l, A, l, l, l, rows, o, h->work, h->work_elems, h->st);
    if (sharded) ENMF_TRY(ar(h, G, (size_t)l * l, CommOp::Sum));
    chol_inv(G, l, pass == 0 ? 1e-13 : 0.0, R, Rinv, bad, h->st);
    GemmOut o2;
    o2.C = tmp;
    o2.ldc = l;
    gemm<double, double>(false, A, l, Rinv, l, rows, l, l, o2, h->work, h->work_elems, h->st);
    CUDA_TRY(cudaMemcpyAsync(A, tmp, sizeof(double) * rows * l, cudaMemcpyDeviceToDevice, h->st));
  }
  return check_launch();
}

// Global column-wise arg max |A_ik| (ties: lowest global row) -> sign of that entry (R5).
enmf_status_t column_signs(enmf_handle_t h, const double* A, int64_t rows, int r,
                           int64_t row_offset, std::vector<double>& sign) {
  colabsmax(A, rows, r, row_offset, h->parts, h->st);
  const int np = colabsmax_parts();
  std::vector<double> hp((size_t)np * r * 3);
  CUDA_TRY(cudaMemcpyAsync(hp.data(), h->parts, sizeof(double) * hp.size(),
                           cudaMemcpyDeviceToHost, h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  std::vector<double> best(r, -1.0), bidx(r, 0.0), bval(r, 0.0);
  for (int p = 0; p < np; ++p)
    for (int k = 0; k < r; ++k) {
      const double* q = &hp[((size_t)p * r + k) * 3];
      if (q[0] > best[k] || (q[0] == best[k] && q[1] < bidx[k])) {
        best[k] = q[0]; bidx[k] = q[1]; bval[k] = q[2];
      }
    }
  sign.assign(r, 1.0);
  if (h->sharded) {
    double* d = h->work;   // [best | idx | sign]
    std::vector<double> tmp(best);
    CUDA_TRY(cudaMemcpyAsync(d, tmp.data(), sizeof(double) * r, cudaMemcpyHostToDevice, h->st));
    ENMF_TRY(ar(h, d, r, CommOp::Max));
    std::vector<double> gbest(r);
    CUDA_TRY(cudaMemcpyAsync(gbest.data(), d, sizeof(double) * r, cudaMemcpyDeviceToHost, h->st));
    CUDA_TRY(cudaStreamSynchronize(h->st));
    for (int k = 0; k < r; ++k) tmp[k] = best[k] == gbest[k] ? bidx[k] : 1e300;
    CUDA_TRY(cudaMemcpyAsync(d, tmp.data(), sizeof(double) * r, cudaMemcpyHostToDevice, h->st));
    ENMF_TRY(ar(h, d, r, CommOp::Min));
    std::vector<double> gidx(r);
    CUDA_TRY(cudaMemcpyAsync(gidx.data(), d, sizeof(double) * r, cudaMemcpyDeviceToHost, h->st));
    CUDA_TRY(cudaStreamSynchronize(h->st));
    for (int k = 0; k < r; ++k)
      tmp[k] = (best[k] == gbest[k] && bidx[k] == gidx[k]) ? (bval[k] < 0 ? -1.0 : 1.0) : 0.0;
    CUDA_TRY(cudaMemcpyAsync(d, tmp.data(), sizeof(double) * r, cudaMemcpyHostToDevice, h->st));
    ENMF_TRY(ar(h, d, r, CommOp::Sum));
    CUDA_TRY(cudaMemcpyAsync(tmp.data(), d, sizeof(double) * r, cudaMemcpyDeviceToHost, h->st));
    CUDA_TRY(cudaStreamSynchronize(h->st));
    for (int k = 0; k < r; ++k) sign[k] = tmp[k] < 0 ? -1.0 : 1.0;
  } else {
    for (int k = 0; k < r; ++k) sign[k] = bval[k] < 0 ? -1.0 : 1.0;
  }
  return ENMF_OK;
}

// Sum of h(A) = max(0, -A) over `count` fp64 entries.
enmf_status_t negativity(enmf_handle_t h, const double* A, int64_t count, double* out_host) {
  negsum(A, count, h->parts, h->dscal + S_NEG, h->st);
  CUDA_TRY(cudaMemcpyAsync(out_host, h->dscal + S_NEG, sizeof(double), cudaMemcpyDeviceToHost,
                           h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  return check_launch();
}

// Randomised range finder + Rayleigh-Ritz; writes U*, V* into W64 (fp64) and U, V (fp32).
enmf_status_t svd_core(enmf_handle_t h, float* U, int64_t ldu, float* V, int64_t ldv,
                       double* sigma_host, enmf_init_info_t* info) {
  const int64_t m = h->prob.m_global, n = h->n, mr = h->m_loc;
  const int r = (int)h->r;
  int64_t l64 = std::min<int64_t>(std::min(m, n), r + h->opt.oversample);
  l64 = std::min<int64_t>(l64, 512);
  const int l = (int)l64;
  const bool sh = h->sharded;
  DevBuf db(h);
  double *Om, *Y, *Z, *Qt, *tmp, *G, *R, *Rinv, *Ue, *Ve, *sv, *jw, *Us;
  int* bad;
  const int64_t big = std::max(mr, n);
  ENMF_TRY(db.get(&Om, (size_t)(n * l)));
  ENMF_TRY(db.get(&Y, (size_t)(mr * l)));
  ENMF_TRY(db.get(&Z, (size_t)(n * l)));
  ENMF_TRY(db.get(&Qt, (size_t)(n * l)));
  ENMF_TRY(db.get(&tmp, (size_t)(big * l)));
  ENMF_TRY(db.get(&G, (size_t)l * l));
  ENMF_TRY(db.get(&R, (size_t)l * l));
  ENMF_TRY(db.get(&Rinv, (size_t)l * l));
  ENMF_TRY(db.get(&Ue, (size_t)l * l));
  ENMF_TRY(db.get(&Ve, (size_t)l * l));
  ENMF_TRY(db.get(&sv, (size_t)l));
  ENMF_TRY(db.get(&jw, (size_t)2 * l * l));
  ENMF_TRY(db.get(&Us, (size_t)(big * r)));
  ENMF_TRY(db.get(&bad, 1));
  if (!h->W64) ENMF_TRY(dalloc(&h->W64, (size_t)((mr + n) * r)));
  // Y = X Omega ; orth                                   (Krylov-type, 1827-1835)
  gaussian_fill(Om, n, l, h->opt.seed, h->st);
  GemmOut o;
  o.ldc = l;
  // the 2q + 2 X passes: the range finder's on the tensor-core path as int8-digit products in
  // blocks of <= 128 columns (tc_xf; any basis that captures the range serves, so its ~2^-22
  // operand rounding is harmless), else -- and for the final Rayleigh-Ritz pass B^T = X^T Q,
  // which fixes sigma and the factors (X's 2^-22 rounding alone moves the balanced factors of
  // a C5-shape problem by 1e-5, tools/digit_sim.py) -- the SIMT fp64-accumulating GEMM on the
  // caller's fp32 X
  auto xprod = [&](bool trans, const double* F, double* out, bool exact = false) -> enmf_status_t {
    if (h->sparse) {                 // CSR / CSC SpMM in fp64 (kernels_sparse.cu)
      if (trans)
        spmm<double>(h->csc_ptr, h->csc_row, h->csc_val, n, F, l, l, out, l, h->st);
      else
        spmm<double>(h->csr_ptr, h->csr_col, h->csr_val, mr, F, l, l, out, l, h->st);
      return ENMF_OK;
    }
    if (h->tc && !exact) {
      const int rc = tc_xf(h->tc, trans, F, l, l, out, l, h->st);
      return rc == 0 ? ENMF_OK : (rc == 2 ? ENMF_ERR_OOM : ENMF_ERR_CUDA);
    }
    GemmOut oo;
    oo.ldc = l;
    oo.C = out;
    if (trans)
      gemm<float, double>(true, h->X, h->ldx, F, l, n, l, mr, oo, h->work, h->work_elems, h->st);
    else
      gemm<float, double>(false, h->X, h->ldx, F, l, mr, l, n, oo, h->work, h->work_elems, h->st);
    return ENMF_OK;
  };
  ENMF_TRY(xprod(false, Om, Y));                                     // Y = X Omega
  ENMF_TRY(cholqr(h, Y, tmp, mr, l, sh, G, R, Rinv, bad));
  for (int q = 0; q < h->opt.power_iters; ++q) {
    ENMF_TRY(xprod(true, Y, Z));                                     // Z = X^T Q
    ENMF_TRY(ar(h, Z, (size_t)(n * l), CommOp::Sum));
    ENMF_TRY(cholqr(h, Z, tmp, n, l, false, G, R, Rinv, bad));
    ENMF_TRY(xprod(false, Z, Y));                                    // Y = X Z
    ENMF_TRY(cholqr(h, Y, tmp, mr, l, sh, G, R, Rinv, bad));
  }
  // B^T = X^T Q (n x l); B B^T = Qt^T Qt = Ve diag(s) Ve^T; sigma = sqrt(s)
  ENMF_TRY(xprod(true, Y, Qt, true));
  ENMF_TRY(ar(h, Qt, (size_t)(n * l), CommOp::Sum));
  o.C = G;
  gemm<double, double>(true, Qt, l, Qt, l, l, l, n, o, h->work, h->work_elems, h->st);
  jacobi_svd(G, l, Ue, sv, Ve, jw, h->st);
  std::vector<double> hs(l);
  CUDA_TRY(cudaMemcpyAsync(hs.data(), sv, sizeof(double) * l, cudaMemcpyDeviceToHost, h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  ENMF_TRY(check_launch());
  std::vector<double> sig(r);
  for (int k = 0; k < r; ++k) sig[k] = sqrt(std::max(hs[k], 0.0));
  if (!(sig[0] > 0.0)) return ENMF_ERR_RANK_DEFICIENT;
  int deficient = 0;
  // left singular vectors Q Ve_r (unscaled) for the sign rule R5
  o.C = Us;
  o.ldc = r;
  gemm<double, double>(false, Y, l, Ve, l, mr, r, l, o, h->work, h->work_elems, h->st);
  std::vector<double> sgn;
  ENMF_TRY(column_signs(h, Us, mr, r, h->prob.row_begin, sgn));
  std::vector<double> cu(r), cv(r);
  for (int k = 0; k < r; ++k) {
    const bool zero = sig[k] <= 1e-7 * sig[0];
    deficient += zero;
    cu[k] = zero ? 0.0 : sgn[k] * sqrt(sig[k]);          // U* = U S^1/2
    cv[k] = zero ? 0.0 : sgn[k] / sqrt(sig[k]);          // V* = B^T U S^-1 S^1/2
  }
  double* dcs = h->work;   // 2r column scales
  CUDA_TRY(cudaMemcpyAsync(dcs, cu.data(), sizeof(double) * r, cudaMemcpyHostToDevice, h->st));
  CUDA_TRY(cudaMemcpyAsync(dcs + r, cv.data(), sizeof(double) * r, cudaMemcpyHostToDevice, h->st));
  scale_cols_f64(Us, mr, r, dcs, h->st);
  CUDA_TRY(cudaMemcpyAsync(h->W64, Us, sizeof(double) * mr * r, cudaMemcpyDeviceToDevice, h->st));
  o.C = Us;
  gemm<double, double>(false, Qt, l, Ve, l, n, r, l, o, h->work + 2 * r, h->work_elems - 2 * r,
                       h->st);
  scale_cols_f64(Us, n, r, dcs + r, h->st);
  CUDA_TRY(cudaMemcpyAsync(h->W64 + mr * r, Us, sizeof(double) * n * r,
                           cudaMemcpyDeviceToDevice, h->st));
  f64_to_f32(h->W64, mr, r, nullptr, U, ldu, h->st);
  f64_to_f32(h->W64 + mr * r, n, r, nullptr, V, ldv, h->st);
  CUDA_TRY(cudaStreamSynchronize(h->st));
  ENMF_TRY(check_launch());
  if (sigma_host)
    for (int k = 0; k < r; ++k) sigma_host[k] = sig[k];
  if (info) {
    memset(info->sigma, 0, sizeof(info->sigma));
    for (int k = 0; k < r; ++k) info->sigma[k] = sig[k];
    info->rank_deficient = deficient;
  }
  return ENMF_OK;
}

// Alg. 1 from W64 = [U*; V*] (this rank's U rows, all V rows); writes U = U* R, V = V* R.
enmf_status_t rotate_core(enmf_handle_t h, float* U, int64_t ldu, float* V, int64_t ldv,
                          enmf_init_info_t* info) {
  const int64_t mr = h->m_loc, n = h->n, rows = mr + n;
  const int r = (int)h->r;
  const int64_t count = rows * r;
  const bool sh = h->sharded;
  DevBuf db(h);
  double *WR, *Yh, *Z, *B, *R, *M, *Cs, *Ds, *sv, *jw;
  unsigned long long* third;
  ENMF_TRY(db.get(&WR, (size_t)count));
  ENMF_TRY(db.get(&Yh, (size_t)count));
  ENMF_TRY(db.get(&Z, (size_t)count));
  ENMF_TRY(db.get(&B, (size_t)count));
  ENMF_TRY(db.get(&R, (size_t)r * r));
  ENMF_TRY(db.get(&M, (size_t)2 * r * r));
  ENMF_TRY(db.get(&Cs, (size_t)r * r));
  ENMF_TRY(db.get(&Ds, (size_t)r * r));
  ENMF_TRY(db.get(&sv, (size_t)r));
  ENMF_TRY(db.get(&jw, (size_t)2 * r * r));
  ENMF_TRY(db.get(&third, 1));
  int* pfail = nullptr;
  ENMF_TRY(db.get(&pfail, 1));
  int* nsst = nullptr;
  ENMF_TRY(db.get(&nsst, 2));
  double* nsw = nullptr;
  ENMF_TRY(db.get(&nsw, (size_t)3 * r * r + 256));
  CUDA_TRY(cudaMemsetAsync(third, 0, sizeof(unsigned long long), h->st));
  double* W = h->W64;
  // negativity of the unrotated point (info) and max|W| for reading R7
  double neg0u = 0.0, neg0v = 0.0;
  ENMF_TRY(negativity(h, W, mr * r, &neg0u));
  ENMF_TRY(negativity(h, W + mr * r, n * r, &neg0v));
  std::vector<double> hp;
  colabsmax(W, rows, r, 0, h->parts, h->st);
  {
    const int np = colabsmax_parts();
    hp.resize((size_t)np * r * 3);
    CUDA_TRY(cudaMemcpyAsync(hp.data(), h->parts, sizeof(double) * hp.size(),
                             cudaMemcpyDeviceToHost, h->st));
    CUDA_TRY(cudaStreamSynchronize(h->st));
  }
  double wmax = 0.0;
  for (size_t e = 0; e < hp.size(); e += 3) wmax = std::max(wmax, hp[e]);
  if (sh) {
    CUDA_TRY(cudaMemcpyAsync(h->dscal + S_WMAX, &wmax, sizeof(double), cudaMemcpyHostToDevice,
                             h->st));
    ENMF_TRY(ar(h, h->dscal + S_WMAX, 1, CommOp::Max));
    CUDA_TRY(cudaMemcpyAsync(&wmax, h->dscal + S_WMAX, sizeof(double), cudaMemcpyDeviceToHost,
                             h->st));
    CUDA_TRY(cudaStreamSynchronize(h->st));
  }
  const double inv_rho = h->opt.admm_rho > 0.0 ? 1.0 / h->opt.admm_rho
                                                : (wmax > 0.0 ? 1000.0 * wmax : 1.0);
  CUDA_TRY(cudaMemsetAsync(third, 0, sizeof(unsigned long long), h->st));
  std::vector<double> eye((size_t)r * r, 0.0);
  for (int a = 0; a < r; ++a) eye[(size_t)a * r + a] = 1.0;             // R0 = I (R6)
  CUDA_TRY(cudaMemcpyAsync(R, eye.data(), sizeof(double) * r * r, cudaMemcpyHostToDevice, h->st));
  GemmOut o;
  o.ldc = r;
  for (int t = 0; t < h->opt.admm_iters; ++t) {
    o.C = WR;
    gemm<double, double>(false, W, r, R, r, rows, r, r, o, h->work, h->work_elems, h->st);
    admm_z(WR, Yh, Z, B, count, inv_rho, t == 0, h->parts, third, h->st);
    // M = W^T (Z + Y/rho) = W^T B, U rows summed over ranks, V rows counted once
    if (!sh) {
      o.C = M;
      gemm<double, double>(true, W, r, B, r, r, r, rows, o, h->work, h->work_elems, h->st);
    } else {
      o.C = M;
      gemm<double, double>(true, W, r, B, r, r, r, mr, o, h->work, h->work_elems, h->st);
      if (h->prob.rank == 0) {
        o.C = M + r * r;
        gemm<double, double>(true, W + mr * r, r, B + mr * r, r, r, r, n, o, h->work,
                             h->work_elems, h->st);
      } else {
        CUDA_TRY(cudaMemsetAsync(M + r * r, 0, sizeof(double) * r * r, h->st));
      }
      reduce_parts(M, 2, (int64_t)r * r, Cs, h->st);
      CUDA_TRY(cudaMemcpyAsync(M, Cs, sizeof(double) * r * r, cudaMemcpyDeviceToDevice, h->st));
      ENMF_TRY(ar(h, M, (size_t)r * r, CommOp::Sum));
    }
    // R = C D^T from W^T B = C S D^T (orthogonal Procrustes)
    // R = polar factor of M: scaled Newton (polar_newton); if M is numerically singular the
    // device flag `third + 1` gates the Jacobi SVD + basis completion path (rank deficiency)
    if (polar_supported(r)) {
      // Newton-Schulz (multi-CTA, ~20-30 cheap steps) -> scaled Newton if it did not converge
      // -> Jacobi SVD if M is numerically singular; each stage gated by a device flag
      polar_ns(M, r, R, nsst, nsw, 40, h->st);
      polar_newton(M, r, R, pfail, h->st, nullptr, nsst + 1);
      jacobi_svd(M, r, Cs, sv, Ds, jw, h->st, nullptr, pfail);
      procrustes_from_svd(Cs, sv, Ds, r, R, h->st, pfail);
    } else {
      jacobi_svd(M, r, Cs, sv, Ds, jw, h->st, t > 0 ? Ds : nullptr);
      procrustes_from_svd(Cs, sv, Ds, r, R, h->st);
    }
  }
  ENMF_TRY(check_launch());
  unsigned long long third_h = 0;
  CUDA_TRY(cudaMemcpyAsync(&third_h, third, sizeof(third_h), cudaMemcpyDeviceToHost, h->st));
  // (U, V) = (U* R, V* R)   (Alg. 3)
  o.C = WR;
  gemm<double, double>(false, W, r, R, r, rows, r, r, o, h->work, h->work_elems, h->st);
  f64_to_f32(WR, mr, r, nullptr, U, ldu, h->st);
  f64_to_f32(WR + mr * r, n, r, nullptr, V, ldv, h->st);
  double negu = 0.0, negv = 0.0;
  ENMF_TRY(negativity(h, WR, mr * r, &negu));
  ENMF_TRY(negativity(h, WR + mr * r, n * r, &negv));
  std::vector<double> hR((size_t)r * r);
  CUDA_TRY(cudaMemcpyAsync(hR.data(), R, sizeof(double) * r * r, cudaMemcpyDeviceToHost, h->st));
  // lift constants from the rotated point, fixed for the whole ascent stage (R9)
  ENMF_TRY(min_factor(h, U, ldu, mr, S_MINU, sh));
  ENMF_TRY(min_factor(h, V, ldv, n, S_MINV, false));
  double mins[2];
  CUDA_TRY(cudaMemcpyAsync(mins, h->dscal + S_MINU, sizeof(mins), cudaMemcpyDeviceToHost, h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  ENMF_TRY(check_launch());
  const double L = (double)h->opt.lift_steps;
  const double lu = mins[0] < 0 ? (1.0 + 1e-3) * (-mins[0]) / L : 0.0;
  const double lv = mins[1] < 0 ? (1.0 + 1e-3) * (-mins[1]) / L : 0.0;
  ENMF_TRY(enmf_set_stage(h, 0, lu, lv));
  if (info) {
    double orth = 0.0;
    for (int a = 0; a < r; ++a)
      for (int b = 0; b < r; ++b) {
        double s = 0.0;
        for (int c = 0; c < r; ++c) s += hR[(size_t)c * r + a] * hR[(size_t)c * r + b];
        orth = std::max(orth, fabs(s - (a == b ? 1.0 : 0.0)));
      }
    info->orth_residual = orth;
    info->negativity_svd = neg0u + neg0v;
    info->negativity_rot = negu + negv;
    info->admm_third_branch = (int64_t)third_h;
    info->lambda_u = lu;
    info->lambda_v = lv;
  }
  return ENMF_OK;
}

// softImpute-ALS with lambda = 0 (Hastie et al. 2015, Alg. 3.1; the eNMC init of PAPER.md:1017,
// reading R31), on the observed entries only: the completed matrix X* = P_E(X) + P_E-perp(A B^T)
// enters through X*^T U = S^T U + B D and X* V = S V + A D (S = P_E(X - A B^T), U and V
// orthonormal, A = U D, B = V D).  Per iteration:
//   V side: T = X*^T U (n x r); SVD T = V~ D~^2 R^T; V <- V~, D <- D~, U <- U R
//   U side: T = X* V  (m x r); SVD T = U~ D~^2 R^T; U <- U~, D <- D~, V <- V R
// The thin SVD of T comes from the eigen-decomposition of T^T T (one-sided Jacobi, fp64):
// R = its eigenvectors, D~^2 = sqrt of its eigenvalues, the left factor T R D~^-2.  Output:
// A, B (sign rule R5 on A, D descending) into W64 = [A; B] and U, V (fp32) for enmf_rotate.
enmf_status_t softimpute_core(enmf_handle_t h, const float* U0, int64_t ldu0, int iters,
                              float* Uout, int64_t ldu, float* Vout, int64_t ldv,
                              double* d_host) {
  const int64_t m = h->m_loc, n = h->n, big = std::max(m, n);
  const int r = (int)h->r;
  DevBuf db(h);
  double *Ud, *Vd, *A, *B, *T, *Tq, *G, *R, *Rinv, *Ev, *Ee, *sv, *jw, *Dd, *inv, *W;
  int* bad;
  ENMF_TRY(db.get(&Ud, (size_t)(m * r)));
  ENMF_TRY(db.get(&Vd, (size_t)(n * r)));
  ENMF_TRY(db.get(&A, (size_t)(m * r)));
  ENMF_TRY(db.get(&B, (size_t)(n * r)));
  ENMF_TRY(db.get(&T, (size_t)(big * r)));
  ENMF_TRY(db.get(&Tq, (size_t)(big * r)));
  ENMF_TRY(db.get(&W, (size_t)(big * r)));
  ENMF_TRY(db.get(&G, (size_t)r * r));
  ENMF_TRY(db.get(&R, (size_t)r * r));
  ENMF_TRY(db.get(&Rinv, (size_t)r * r));
  ENMF_TRY(db.get(&Ev, (size_t)r * r));
  ENMF_TRY(db.get(&Ee, (size_t)r * r));
  ENMF_TRY(db.get(&sv, (size_t)r));
  ENMF_TRY(db.get(&jw, (size_t)2 * r * r));
  ENMF_TRY(db.get(&Dd, (size_t)r));
  ENMF_TRY(db.get(&inv, (size_t)r));
  ENMF_TRY(db.get(&bad, 1));
  if (!h->W64) ENMF_TRY(dalloc(&h->W64, (size_t)((m + n) * r)));
  // 1. U = orthonormalised U0 (CholeskyQR2: the unique QR with a positive diagonal), D = I,
  //    V = 0: A = U, B = 0
  f32_to_f64(U0, ldu0, m, r, Ud, h->st);
  ENMF_TRY(cholqr(h, Ud, W, m, r, false, G, R, Rinv, bad));
  std::vector<double> ones(r, 1.0);
  CUDA_TRY(cudaMemcpyAsync(Dd, ones.data(), sizeof(double) * r, cudaMemcpyHostToDevice, h->st));
  CUDA_TRY(cudaMemcpyAsync(A, Ud, sizeof(double) * m * r, cudaMemcpyDeviceToDevice, h->st));
  CUDA_TRY(cudaMemsetAsync(B, 0, sizeof(double) * n * r, h->st));
  CUDA_TRY(cudaMemsetAsync(Vd, 0, sizeof(double) * n * r, h->st));
  GemmOut o;
  o.ldc = r;
  // thin SVD of T (rows x r) -> Q (left, into Tq), D~ (Dd), R = Ev; returns after Ev / Dd set
  auto thin_svd = [&](int64_t rows) -> enmf_status_t {
    o.C = G;
    gemm<double, double>(true, T, r, T, r, r, r, rows, o, h->work, h->work_elems, h->st);
    jacobi_svd(G, r, Ee, sv, Ev, jw, h->st);
    nmc_svals(sv, r, Dd, inv, h->st);
    o.C = Tq;
    gemm<double, double>(false, T, r, Ev, r, rows, r, r, o, h->work, h->work_elems, h->st);
    scale_cols_f64(Tq, rows, r, inv, h->st);                       // T R D~^-2
    return ENMF_OK;
  };
  for (int it = 0; it < iters; ++it) {
    // V side: T = S^T U + B D over the CSC lists (rows of T = columns of X)
    nmc_resid_spmm(h->csc_ptr, h->csc_row, h->csc_val, n, r, B, A, Ud, Dd, T, h->st);
    ENMF_TRY(thin_svd(n));
    CUDA_TRY(cudaMemcpyAsync(Vd, Tq, sizeof(double) * n * r, cudaMemcpyDeviceToDevice, h->st));
    o.C = W;
    gemm<double, double>(false, Ud, r, Ev, r, m, r, r, o, h->work, h->work_elems, h->st);
    CUDA_TRY(cudaMemcpyAsync(Ud, W, sizeof(double) * m * r, cudaMemcpyDeviceToDevice, h->st));
    CUDA_TRY(cudaMemcpyAsync(A, Ud, sizeof(double) * m * r, cudaMemcpyDeviceToDevice, h->st));
    scale_cols_f64(A, m, r, Dd, h->st);
    CUDA_TRY(cudaMemcpyAsync(B, Vd, sizeof(double) * n * r, cudaMemcpyDeviceToDevice, h->st));
    scale_cols_f64(B, n, r, Dd, h->st);
    // U side: T = S V + A D over the CSR lists
    nmc_resid_spmm(h->csr_ptr, h->csr_col, h->csr_val, m, r, A, B, Vd, Dd, T, h->st);
    ENMF_TRY(thin_svd(m));
    CUDA_TRY(cudaMemcpyAsync(Ud, Tq, sizeof(double) * m * r, cudaMemcpyDeviceToDevice, h->st));
    o.C = W;
    gemm<double, double>(false, Vd, r, Ev, r, n, r, r, o, h->work, h->work_elems, h->st);
    CUDA_TRY(cudaMemcpyAsync(Vd, W, sizeof(double) * n * r, cudaMemcpyDeviceToDevice, h->st));
    CUDA_TRY(cudaMemcpyAsync(A, Ud, sizeof(double) * m * r, cudaMemcpyDeviceToDevice, h->st));
    scale_cols_f64(A, m, r, Dd, h->st);
    CUDA_TRY(cudaMemcpyAsync(B, Vd, sizeof(double) * n * r, cudaMemcpyDeviceToDevice, h->st));
    scale_cols_f64(B, n, r, Dd, h->st);
  }
  ENMF_TRY(check_launch());
  // sign rule R5 on the columns of A (= U D, D > 0): A and B flipped together
  std::vector<double> sgn;
  ENMF_TRY(column_signs(h, A, m, r, 0, sgn));
  double* dsg = h->work;
  CUDA_TRY(cudaMemcpyAsync(dsg, sgn.data(), sizeof(double) * r, cudaMemcpyHostToDevice, h->st));
  scale_cols_f64(A, m, r, dsg, h->st);
  scale_cols_f64(B, n, r, dsg, h->st);
  CUDA_TRY(cudaMemcpyAsync(h->W64, A, sizeof(double) * m * r, cudaMemcpyDeviceToDevice, h->st));
  CUDA_TRY(cudaMemcpyAsync(h->W64 + m * r, B, sizeof(double) * n * r, cudaMemcpyDeviceToDevice,
                           h->st));
  f64_to_f32(A, m, r, nullptr, Uout, ldu, h->st);
  f64_to_f32(B, n, r, nullptr, Vout, ldv, h->st);
  std::vector<double> dh(r);
  CUDA_TRY(cudaMemcpyAsync(dh.data(), Dd, sizeof(double) * r, cudaMemcpyDeviceToHost, h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  ENMF_TRY(check_launch());
  if (d_host)
    for (int k = 0; k < r; ++k) d_host[k] = dh[k];
  return ENMF_OK;
}

// RSR-ADMM (App. A, Alg. alg:rsr) from W64 = [U*; V*]: T = admm_iters
// iterations of the split (W1 = W_svd R1, W2 = [W11 Lambda; W12 Lambda^-1], W3 = W2 R2) with
// rho = gamma = t = 1e-3 / max|W_svd| (R34), R1 = R2 = Lambda = I, W1 = W2 = W3 = W_svd,
// M = N = P = 0 (R35), last iterate (R36), the lambda root of R37.  Writes U = U* R1 Lambda R2,
// V = V* R1 Lambda^-1 R2 (fp32), fixes the lift constants from them (R9) and enters the
// ascent stage like enmf_rotate; lam_host (r, may be NULL) receives Lambda.  Single rank.
enmf_status_t rsr_core(enmf_handle_t h, float* U, int64_t ldu, float* V, int64_t ldv,
                       enmf_init_info_t* info, double* lam_host) {
  const int64_t mr = h->m_loc, n = h->n, rows = mr + n;
  const int r = (int)h->r;
  const int64_t count = rows * r;
  DevBuf db(h);
  double *W1, *W2, *W3, *M, *N, *P, *WsR1, *W2R2, *B, *G, *R1, *R2, *R2t, *Mr, *lam, *abcd, *cp;
  double *Cs, *Ds, *sv, *jw, *nsw;
  int *pfail, *nsst;
  ENMF_TRY(db.get(&W1, (size_t)count));
  ENMF_TRY(db.get(&W2, (size_t)count));
  ENMF_TRY(db.get(&W3, (size_t)count));
  ENMF_TRY(db.get(&M, (size_t)count));
  ENMF_TRY(db.get(&N, (size_t)count));
  ENMF_TRY(db.get(&P, (size_t)count));
  ENMF_TRY(db.get(&WsR1, (size_t)count));
  ENMF_TRY(db.get(&W2R2, (size_t)count));
  ENMF_TRY(db.get(&B, (size_t)count));
  ENMF_TRY(db.get(&G, (size_t)count));
  ENMF_TRY(db.get(&R1, (size_t)r * r));
  ENMF_TRY(db.get(&R2, (size_t)r * r));
  ENMF_TRY(db.get(&R2t, (size_t)r * r));
  ENMF_TRY(db.get(&Mr, (size_t)r * r));
  ENMF_TRY(db.get(&Cs, (size_t)r * r));
  ENMF_TRY(db.get(&Ds, (size_t)r * r));
  ENMF_TRY(db.get(&sv, (size_t)r));
  ENMF_TRY(db.get(&jw, (size_t)2 * r * r));
  ENMF_TRY(db.get(&nsw, (size_t)3 * r * r + 256));
  ENMF_TRY(db.get(&lam, (size_t)r));
  ENMF_TRY(db.get(&abcd, (size_t)4 * r));
  ENMF_TRY(db.get(&cp, (size_t)rsr_colsum_parts() * 4 * r));
  ENMF_TRY(db.get(&pfail, 1));
  ENMF_TRY(db.get(&nsst, 2));
  const double* Ws = h->W64;
  double neg0u = 0.0, neg0v = 0.0;
  ENMF_TRY(negativity(h, Ws, mr * r, &neg0u));
  ENMF_TRY(negativity(h, Ws + mr * r, n * r, &neg0v));
  // max |W_svd| for R34
  colabsmax(Ws, rows, r, 0, h->parts, h->st);
  std::vector<double> hp((size_t)colabsmax_parts() * r * 3);
  CUDA_TRY(cudaMemcpyAsync(hp.data(), h->parts, sizeof(double) * hp.size(),
                           cudaMemcpyDeviceToHost, h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  double wmax = 0.0;
  for (size_t e = 0; e < hp.size(); e += 3) wmax = std::max(wmax, hp[e]);
  const double pen = h->opt.admm_rho > 0.0 ? h->opt.admm_rho : 1e-3 / (wmax > 0.0 ? wmax : 1.0);
  const double rho = pen, gamma = pen, t = pen;
  // R35: R1 = R2 = I, Lambda = I, W1 = W2 = W3 = W_svd, M = N = P = 0
  std::vector<double> eye((size_t)r * r, 0.0), ones(r, 1.0);
  for (int a = 0; a < r; ++a) eye[(size_t)a * r + a] = 1.0;
  CUDA_TRY(cudaMemcpyAsync(R1, eye.data(), sizeof(double) * r * r, cudaMemcpyHostToDevice, h->st));
  CUDA_TRY(cudaMemcpyAsync(R2, eye.data(), sizeof(double) * r * r, cudaMemcpyHostToDevice, h->st));
  CUDA_TRY(cudaMemcpyAsync(lam, ones.data(), sizeof(double) * r, cudaMemcpyHostToDevice, h->st));
  for (double* A : {W2, WsR1, W2R2})
    CUDA_TRY(cudaMemcpyAsync(A, Ws, sizeof(double) * count, cudaMemcpyDeviceToDevice, h->st));
  for (double* A : {M, N, P}) CUDA_TRY(cudaMemsetAsync(A, 0, sizeof(double) * count, h->st));
  GemmOut o;
  o.ldc = r;
  auto polar = [&](double* R) {      // R = polar(Mr) = C D^T (Procrustes), as rotate_core
    polar_ns(Mr, r, R, nsst, nsw, 40, h->st);
    polar_newton(Mr, r, R, pfail, h->st, nullptr, nsst + 1);
    jacobi_svd(Mr, r, Cs, sv, Ds, jw, h->st, nullptr, pfail);
    procrustes_from_svd(Cs, sv, Ds, r, R, h->st, pfail);
  };
  for (int it = 0; it < h->opt.admm_iters; ++it) {
    // (W1, W3) <- argmin f1 from W_svd R1, W2 R2 of the previous iterate
    rsr_w13(WsR1, W2R2, M, N, W2, P, lam, rows, mr, r, rho, gamma, t, W1, W3, h->st);
    // R1 <- Procrustes(W_svd, W1 + M); W2 <- argmin f2 with G = (W3 + P) R2^T
    rsr_add(W1, M, count, B, h->st);
    o.C = Mr;
    gemm<double, double>(true, Ws, r, B, r, r, r, rows, o, h->work, h->work_elems, h->st);
    if (polar_supported(r)) {
      polar(R1);
    } else {
      jacobi_svd(Mr, r, Cs, sv, Ds, jw, h->st);
      procrustes_from_svd(Cs, sv, Ds, r, R1, h->st);
    }
    rsr_add(W3, P, count, B, h->st);                    // B = W3 + P (f2 and f3)
    rsr_transpose(R2, r, R2t, h->st);
    o.C = G;
    gemm<double, double>(false, B, r, R2t, r, rows, r, r, o, h->work, h->work_elems, h->st);
    rsr_w2(W1, N, G, lam, rows, mr, r, gamma, t, W2, h->st);
    // R2 <- Procrustes(W2, W3 + P); Lambda <- the quartic roots
    o.C = Mr;
    gemm<double, double>(true, W2, r, B, r, r, r, rows, o, h->work, h->work_elems, h->st);
    if (polar_supported(r)) {
      polar(R2);
    } else {
      jacobi_svd(Mr, r, Cs, sv, Ds, jw, h->st);
      procrustes_from_svd(Cs, sv, Ds, r, R2, h->st);
    }
    rsr_lambda(W1, W2, N, rows, mr, r, cp, abcd, lam, h->st);
    // multipliers with the new R1, R2, Lambda
    o.C = WsR1;
    gemm<double, double>(false, Ws, r, R1, r, rows, r, r, o, h->work, h->work_elems, h->st);
    o.C = W2R2;
    gemm<double, double>(false, W2, r, R2, r, rows, r, r, o, h->work, h->work_elems, h->st);
    rsr_dual(W1, WsR1, W2, W3, W2R2, lam, rows, mr, r, M, N, P, h->st);
  }
  ENMF_TRY(check_launch());
  // (U, V) = (U* R1 Lambda R2, V* R1 Lambda^-1 R2)   (Eq. gen_2)
  CUDA_TRY(cudaMemcpyAsync(B, WsR1, sizeof(double) * count, cudaMemcpyDeviceToDevice, h->st));
  rsr_scale(B, lam, rows, mr, r, h->st);
  o.C = G;
  gemm<double, double>(false, B, r, R2, r, rows, r, r, o, h->work, h->work_elems, h->st);
  f64_to_f32(G, mr, r, nullptr, U, ldu, h->st);
  f64_to_f32(G + mr * r, n, r, nullptr, V, ldv, h->st);
  double negu = 0.0, negv = 0.0;
  ENMF_TRY(negativity(h, G, mr * r, &negu));
  ENMF_TRY(negativity(h, G + mr * r, n * r, &negv));
  std::vector<double> hl(r);
  CUDA_TRY(cudaMemcpyAsync(hl.data(), lam, sizeof(double) * r, cudaMemcpyDeviceToHost, h->st));
  ENMF_TRY(min_factor(h, U, ldu, mr, S_MINU, false));
  ENMF_TRY(min_factor(h, V, ldv, n, S_MINV, false));
  double mins[2];
  CUDA_TRY(cudaMemcpyAsync(mins, h->dscal + S_MINU, sizeof(mins), cudaMemcpyDeviceToHost, h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  ENMF_TRY(check_launch());
  const double L = (double)h->opt.lift_steps;
  const double lu = mins[0] < 0 ? (1.0 + 1e-3) * (-mins[0]) / L : 0.0;
  const double lv = mins[1] < 0 ? (1.0 + 1e-3) * (-mins[1]) / L : 0.0;
  ENMF_TRY(enmf_set_stage(h, 0, lu, lv));
  if (lam_host)
    for (int k = 0; k < r; ++k) lam_host[k] = hl[k];
  if (info) {
    info->negativity_svd = neg0u + neg0v;
    info->negativity_rot = negu + negv;
    info->lambda_u = lu;
    info->lambda_v = lv;
  }
  return ENMF_OK;
}

enmf_status_t xnorm2_host(enmf_handle_t h, double* out) {
  CUDA_TRY(cudaMemcpyAsync(out, h->dscal + S_XNORM2, sizeof(double), cudaMemcpyDeviceToHost,
                           h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  return ENMF_OK;
}

}  // namespace

extern "C" {

enmf_status_t enmf_svd(enmf_handle_t h, float* U, int64_t ldu, float* V, int64_t ldv,
                       double* sigma_host) {
  if (!h) return ENMF_ERR_INVALID_ARG;
  if (!h->bound) return ENMF_ERR_STATE;
  ENMF_TRY(validate_ld(U, ldu, h->r));
  ENMF_TRY(validate_ld(V, ldv, h->r));
  LaunchScope ls(h);
  return svd_core(h, U, ldu, V, ldv, sigma_host, nullptr);
}

enmf_status_t enmf_softimpute(enmf_handle_t h, const float* U0, int64_t ldu0, int iters,
                              float* U, int64_t ldu, float* V, int64_t ldv, double* d_host) {
  if (!h || iters < 1) return ENMF_ERR_INVALID_ARG;
  if (!h->bound || !h->nmc) return ENMF_ERR_STATE;
  ENMF_TRY(validate_ld(U0, ldu0, h->r));
  ENMF_TRY(validate_ld(U, ldu, h->r));
  ENMF_TRY(validate_ld(V, ldv, h->r));
  LaunchScope ls(h);
  return softimpute_core(h, U0, ldu0, iters, U, ldu, V, ldv, d_host);
}

enmf_status_t enmf_rotate(enmf_handle_t h, float* U, int64_t ldu, float* V, int64_t ldv,
                          enmf_init_info_t* info) {
  if (!h) return ENMF_ERR_INVALID_ARG;
  if (!h->bound) return ENMF_ERR_STATE;
  ENMF_TRY(validate_ld(U, ldu, h->r));
  ENMF_TRY(validate_ld(V, ldv, h->r));
  LaunchScope ls(h);
  if (!h->W64) ENMF_TRY(dalloc(&h->W64, (size_t)((h->m_loc + h->n) * h->r)));
  f32_to_f64(U, ldu, h->m_loc, h->r, h->W64, h->st);
  f32_to_f64(V, ldv, h->n, h->r, h->W64 + h->m_loc * h->r, h->st);
  ENMF_TRY(rotate_core(h, U, ldu, V, ldv, info));
  if (info) ENMF_TRY(xnorm2_host(h, &info->xnorm2));
  return ENMF_OK;
}

enmf_status_t enmf_rotate_rsr(enmf_handle_t h, float* U, int64_t ldu, float* V, int64_t ldv,
                              enmf_init_info_t* info, double* lambda_host) {
  if (!h) return ENMF_ERR_INVALID_ARG;
  if (!h->bound) return ENMF_ERR_STATE;
  if (h->sharded) return ENMF_ERR_STATE;
  ENMF_TRY(validate_ld(U, ldu, h->r));
  ENMF_TRY(validate_ld(V, ldv, h->r));
  LaunchScope ls(h);
  if (!h->W64) ENMF_TRY(dalloc(&h->W64, (size_t)((h->m_loc + h->n) * h->r)));
  f32_to_f64(U, ldu, h->m_loc, h->r, h->W64, h->st);
  f32_to_f64(V, ldv, h->n, h->r, h->W64 + h->m_loc * h->r, h->st);
  ENMF_TRY(rsr_core(h, U, ldu, V, ldv, info, lambda_host));
  if (info) ENMF_TRY(xnorm2_host(h, &info->xnorm2));
  return ENMF_OK;
}

enmf_status_t enmf_init(enmf_handle_t h, const float* X, int64_t ldx, float* U, int64_t ldu,
                        float* V, int64_t ldv, enmf_init_info_t* info) {
  if (!h) return ENMF_ERR_INVALID_ARG;
  ENMF_TRY(validate_ld(U, ldu, h->r));
  ENMF_TRY(validate_ld(V, ldv, h->r));
  ENMF_TRY(enmf_set_data(h, X, ldx));
  LaunchScope ls(h);
  enmf_init_info_t tmp;
  enmf_init_info_t* inf = info ? info : &tmp;
  memset(inf, 0, sizeof(*inf));
  ENMF_TRY(svd_core(h, U, ldu, V, ldv, nullptr, inf));
  ENMF_TRY(rotate_core(h, U, ldu, V, ldv, inf));   // from the fp64 W64 of svd_core
  ENMF_TRY(xnorm2_host(h, &inf->xnorm2));
  return ENMF_OK;
}

enmf_status_t enmf_solve_host(enmf_handle_t h, const float* X_host, float* U_host,
                              float* V_host, int n_iters, double* f_trace_host,
                              enmf_init_info_t* info) {
  if (!h || !X_host || !U_host || !V_host || n_iters < 0) return ENMF_ERR_INVALID_ARG;
  if (h->sharded) return ENMF_ERR_STATE;
  const int64_t m = h->m_loc, n = h->n, r = h->r;
  if (!h->x_owned) ENMF_TRY(dalloc(&h->x_owned, (size_t)(m * n)));
  // host -> device through two pinned staging buffers, copies overlapped with memcpy
  const size_t chunk = (size_t)64 << 20;
  char* pin[2] = {nullptr, nullptr};
  cudaEvent_t ev[2];
  CUDA_TRY(cudaMallocHost((void**)&pin[0], chunk));
  CUDA_TRY(cudaMallocHost((void**)&pin[1], chunk));
  CUDA_TRY(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  CUDA_TRY(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  const size_t total = sizeof(float) * (size_t)(m * n);
  const char* src = (const char*)X_host;
  char* dst = (char*)h->x_owned;
  int b = 0;
  bool used[2] = {false, false};
  for (size_t off = 0; off < total; off += chunk, b ^= 1) {
    const size_t len = std::min(chunk, total - off);
    if (used[b]) CUDA_TRY(cudaEventSynchronize(ev[b]));
    memcpy(pin[b], src + off, len);
    CUDA_TRY(cudaMemcpyAsync(dst + off, pin[b], len, cudaMemcpyHostToDevice, h->st));
    CUDA_TRY(cudaEventRecord(ev[b], h->st));
    used[b] = true;
  }
  CUDA_TRY(cudaStreamSynchronize(h->st));
  cudaFreeHost(pin[0]);
  cudaFreeHost(pin[1]);
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
  // device factor state: the handle's iterate_host buffers (not the init arena, which
  // enmf_init below reuses)
  if (!h->Ud) ENMF_TRY(dalloc(&h->Ud, (size_t)(m * r)));
  if (!h->Vd) ENMF_TRY(dalloc(&h->Vd, (size_t)(n * r)));
  float* dU = h->Ud;
  float* dV = h->Vd;
  ENMF_TRY(enmf_init(h, h->x_owned, n, dU, r, dV, r, info));
  ENMF_TRY(enmf_iterate(h, dU, r, dV, r, n_iters, f_trace_host, nullptr));
  CUDA_TRY(cudaMemcpyAsync(U_host, dU, sizeof(float) * m * r, cudaMemcpyDeviceToHost, h->st));
  CUDA_TRY(cudaMemcpyAsync(V_host, dV, sizeof(float) * n * r, cudaMemcpyDeviceToHost, h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  return ENMF_OK;
}

}  // extern "C"
