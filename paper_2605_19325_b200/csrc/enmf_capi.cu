// enmf_capi.cu -- the C-ABI of include/enmf.h: handle, workspaces, and the orchestration of
// Alg. 3 on one stream.  All arithmetic runs in the kernels of this
// library; this file only sequences launches and NCCL collectives.
#include <cuda_runtime.h>
#include <float.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "handle.h"

namespace enmf {
thread_local int64_t* g_launch_counter = nullptr;

enmf_status_t check_launch() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "enmf: kernel launch failed: %s\n", cudaGetErrorString(e));
    return ENMF_ERR_CUDA;
  }
  return ENMF_OK;
}

enmf_status_t dalloc_bytes(void** p, size_t bytes) {
  *p = nullptr;
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *p = nullptr;
    return e == cudaErrorMemoryAllocation ? ENMF_ERR_OOM : ENMF_ERR_CUDA;
  }
  return ENMF_OK;
}

enmf_status_t ar(enmf_handle_t h, double* buf, size_t count, CommOp op) {
  if (!h->sharded || count == 0) return ENMF_OK;
  if (h->comm)
    return comm_allreduce(h->comm, buf, count, CommType::F64, op, h->st) == 0 ? ENMF_OK
                                                                             : ENMF_ERR_NCCL;
  if (!h->host_ar) return ENMF_ERR_STATE;
  // host-mediated collective (enmf_set_host_allreduce): stream-ordered staging through a
  // pinned buffer; no device-side waiting on other ranks
  if (h->host_ar_cap < count) {
    if (h->host_ar_buf) cudaFreeHost(h->host_ar_buf);
    h->host_ar_buf = nullptr;
    h->host_ar_cap = 0;
    CUDA_TRY(cudaMallocHost((void**)&h->host_ar_buf, sizeof(double) * count));
    h->host_ar_cap = count;
  }
  CUDA_TRY(cudaMemcpyAsync(h->host_ar_buf, buf, sizeof(double) * count, cudaMemcpyDeviceToHost,
                           h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  const int o = op == CommOp::Sum ? 0 : (op == CommOp::Min ? 1 : 2);
  if (h->host_ar(h->host_ar_ctx, h->host_ar_buf, (int64_t)count, o) != 0) return ENMF_ERR_NCCL;
  CUDA_TRY(cudaMemcpyAsync(buf, h->host_ar_buf, sizeof(double) * count, cudaMemcpyHostToDevice,
                           h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));   // the pinned buffer is reused by the next call
  return ENMF_OK;
}

enmf_status_t validate_ld(const void* p, int64_t ld, int64_t cols) {
  if (!p || ld < cols) return ENMF_ERR_INVALID_ARG;
  return ENMF_OK;
}

// ---------------------------------------------------------------- contractions (a5, a6)
// Optional CUDA-event bracketing of each X pass (enmf_set_profiling) on the handle's stream.
static enmf_status_t prof_mark(enmf_handle_t h, int kind) {
  if (!h->prof) return ENMF_OK;
  if (h->ev_used == h->ev_pool.size()) {
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreate(&e));
    h->ev_pool.push_back(e);
  }
  if (h->ev_used % 2 == 0) h->ev_kind.push_back(kind);
  CUDA_TRY(cudaEventRecord(h->ev_pool[h->ev_used++], h->st));
  return ENMF_OK;
}

// Accumulate elapsed times of completed event pairs (stream already synchronised), plus the
// X V passes timed by their own kernel timestamps (fused sweeps: see sweep()).
static void prof_collect(enmf_handle_t h) {
  for (size_t p = 0; p + 1 < h->ev_used; p += 2) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, h->ev_pool[p], h->ev_pool[p + 1]) == cudaSuccess) {
      const int k = h->ev_kind[p / 2];
      h->prof_ms[k] += ms;
      h->prof_cnt[k] += 1;
    }
  }
  h->ev_used = 0;
  h->ev_kind.clear();
  if (h->tc) {
    double ms = 0.0;
    int64_t cnt = 0;
    if (tc_stamp_read(h->tc, &ms, &cnt) == 0) {
      h->prof_ms[0] += ms;
      h->prof_cnt[0] += cnt;
    }
  }
}

// P = X V (this rank's rows): the first X pass of a sweep.
// band_ready (tensor-core path, tc_band_flags): the pass publishes its finished bands for the
// U-block kernel enqueued right behind it; it is then timed by its own timestamps (an event
// between the two launches would serialise them).
enmf_status_t contract_xv(enmf_handle_t h, const float* V, int64_t ldv, double* P,
                          const unsigned long long* vmax, unsigned* band_ready) {
  if (band_ready) {
    return tc_xv(h->tc, V, ldv, P, h->st, vmax, band_ready, h->prof) != 0 ? ENMF_ERR_CUDA
                                                                         : ENMF_OK;
  }
  ENMF_TRY(prof_mark(h, 0));
  if (h->sparse) {
    spmm<float>(h->csr_ptr, h->csr_col, h->csr_val, h->m_loc, V, ldv, (int)h->r, P, h->r, h->st);
  } else if (h->tc) {
    if (tc_xv(h->tc, V, ldv, P, h->st, vmax) != 0) return ENMF_ERR_CUDA;
  } else {
    GemmOut o;
    o.C = P;
    o.ldc = h->r;
    gemm<float, float>(false, h->X, h->ldx, V, ldv, h->m_loc, h->r, h->n, o, h->work,
                       h->work_elems, h->st);
  }
  return prof_mark(h, 0);
}

// Q = X^T U summed over ranks: the second X pass.  slice: only this rank's V
// slice of Q is needed (the sweep's sharded V block) -- with NCCL a reduce-scatter (Q holds
// world x v_pad rows), otherwise the full allreduce (which includes the slice).
//
// Tensor-core path, several ranks, 128-row-aligned V slices: the pass runs slice by slice
// (band range of the owner's rows, tc_xtu_bands) and each slice is summed to its owner
// (ncclReduce on a communication stream) while the next slice computes -- the pass's
// reduce-scatter overlapped with its own tail.  Through the
// host collective (one-GPU multi-rank tests) each slice is allreduced in turn.
static enmf_status_t contract_xtu_sliced(enmf_handle_t h, const float* U, int64_t ldu,
                                         double* Q, const unsigned long long* umax) {
  const int world = h->prob.world_size;
  const int64_t r = h->r, bands = tc_xtu_band_count(h->tc), per = h->v_pad / 128;
  if (h->comm) {
    if (!h->st_comm) CUDA_TRY(cudaStreamCreateWithFlags(&h->st_comm, cudaStreamNonBlocking));
    while ((int)h->ev_comm.size() < world + 1) {
      cudaEvent_t e;
      CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      h->ev_comm.push_back(e);
    }
  }
  bool first = true;
  for (int s = 0; s < world; ++s) {
    const int64_t b0 = s * per, b1 = std::min(bands, (s + 1) * per);
    if (b0 >= b1) continue;
    const int rc = tc_xtu_bands(h->tc, U, ldu, Q, b0, b1, h->st, umax, first);
    if (rc) return rc == 2 ? ENMF_ERR_OOM : ENMF_ERR_CUDA;
    first = false;
    const int64_t row0 = s * h->v_pad, rows = std::min(h->n, row0 + h->v_pad) - row0;
    if (h->comm) {
      CUDA_TRY(cudaEventRecord(h->ev_comm[s], h->st));
      CUDA_TRY(cudaStreamWaitEvent(h->st_comm, h->ev_comm[s], 0));
      if (comm_reduce(h->comm, Q + row0 * r, (size_t)(rows * r), CommType::F64, s,
                      h->st_comm) != 0)
        return ENMF_ERR_NCCL;
    } else {
      ENMF_TRY(ar(h, Q + row0 * r, (size_t)(rows * r), CommOp::Sum));
    }
  }
  if (h->comm) {
    CUDA_TRY(cudaEventRecord(h->ev_comm[world], h->st_comm));
    CUDA_TRY(cudaStreamWaitEvent(h->st, h->ev_comm[world], 0));
  }
  return ENMF_OK;
}

enmf_status_t contract_xtu(enmf_handle_t h, const float* U, int64_t ldu, double* Q,
                           const unsigned long long* umax, bool slice) {
  const char* pc = getenv("ENMF_PASS2_SLICED");
  if (slice && h->tc && h->sharded && h->v_pad % 128 == 0 && !(pc && pc[0] == '0')) {
    ENMF_TRY(prof_mark(h, 1));
    ENMF_TRY(contract_xtu_sliced(h, U, ldu, Q, umax));
    return prof_mark(h, 1);
  }
  ENMF_TRY(prof_mark(h, 1));
  if (h->sparse) {
    spmm<float>(h->csc_ptr, h->csc_row, h->csc_val, h->n, U, ldu, (int)h->r, Q, h->r, h->st);
  } else if (h->tc) {
    if (tc_xtu(h->tc, U, ldu, Q, h->st, umax) != 0) return ENMF_ERR_CUDA;
  } else {
    GemmOut o;
    o.C = Q;
    o.ldc = h->r;
    gemm<float, float>(true, h->X, h->ldx, U, ldu, h->n, h->r, h->m_loc, o, h->work,
                       h->work_elems, h->st);
  }
  ENMF_TRY(prof_mark(h, 1));
  if (slice && h->comm && h->sharded)
    return comm_reduce_scatter(h->comm, Q, (size_t)(h->v_pad * h->r), CommType::F64, h->st) == 0
               ? ENMF_OK
               : ENMF_ERR_NCCL;
  return ar(h, Q, (size_t)(h->n * h->r), CommOp::Sum);
}

// G = A^T A of an fp32 factor (rows x r); sum over ranks if `sharded`.
enmf_status_t gram_f32(enmf_handle_t h, const float* A, int64_t lda, int64_t rows, double* G,
                       bool sharded, const double* qscale) {
  if (gram_supported((int)h->r) &&
      h->work_elems >= (size_t)128 * 128 * (1 + (size_t)gram_parts())) {
    // upper-triangle fp64 Gram (kernels_gram.cu): Gu = work[0 .. 128^2), per-SM partials after
    gram_sym(A, lda, rows, (int)h->r, h->work + 128 * 128, h->work, G, h->st, qscale);
  } else {
    if (qscale) return ENMF_ERR_STATE;
    GemmOut o;
    o.C = G;
    o.ldc = h->r;
    gemm<float, float>(true, A, lda, A, lda, h->r, h->r, rows, o, h->work, h->work_elems, h->st);
  }
  return sharded ? ar(h, G, (size_t)(h->r * h->r), CommOp::Sum) : ENMF_OK;
}

// G_U of the sweep: on the tensor-core path the Gram of the quantised U that the last pass 2
// multiplied, exact on the tensor cores (tc_gram_quantised) -- the fp64 SIMT Gram of the same
// quantised values if the size is beyond its exact-int64 range; else the plain fp32 Gram.
enmf_status_t gram_u(enmf_handle_t h, const float* U, int64_t ldu, bool sharded) {
  const double* qs = qgram_scales(h);
  if (qs) {
    const char* e = getenv("ENMF_TC_GRAM");
    const int rc = (e && e[0] == '0') ? 2 : tc_gram_quantised(h->tc, h->GU, h->st);
    if (rc == 1) return ENMF_ERR_CUDA;
    if (rc == 0) return sharded ? ar(h, h->GU, (size_t)(h->r * h->r), CommOp::Sum) : ENMF_OK;
  }
  return gram_f32(h, U, ldu, h->m_loc, h->GU, sharded, qs);
}

enmf_status_t min_factor(enmf_handle_t h, const float* A, int64_t lda, int64_t rows, int slot,
                         bool sharded) {
  min_f32(A, lda, rows, h->r, h->parts, h->dscal + slot, h->st);
  return sharded ? ar(h, h->dscal + slot, 1, CommOp::Min) : ENMF_OK;
}

}  // namespace enmf

using namespace enmf;

namespace {

// One block update (U block: F = U, C = P, G = G_V; V block: F = V, C = Q, G = G_U).
// In the ascent stage: lift + mask + PBCD (Eqs.(6)-(10), Alg. 2); in HALS: the column sweep.
// hals_issued: the tensor-core HALS kernel of this block is already enqueued (fused with the
// X V pass, see sweep()) together with the colmax reset and its G digits.
enmf_status_t block_update(enmf_handle_t h, float* F, int64_t ldf, int64_t rows,
                           const double* C, const double* G, int lam_slot, int kstar_slot,
                           int min_slot, bool sharded, bool maybe_ascent,
                           unsigned long long* colmax = nullptr, bool hals_issued = false) {
  const int r = (int)h->r;
  if (colmax && !hals_issued)
    CUDA_TRY(cudaMemsetAsync(colmax, 0, sizeof(unsigned long long) * r, h->st));
  int* stage = h->dint + I_STAGE;
  const int mi = h->opt.pbcd_max_iter;
  // ablation variants (R29): fixed ascent step / projected-gradient descent, step 1/lambda_max(G)
  const double* fstep = nullptr;
  if ((maybe_ascent && h->opt.step_rule) || h->opt.descent) {
    // lambda_max(G) by power iteration, warm-started from the same block's eigenvector of the
    // previous sweep (stepws: one r-vector per block; a 128 x 128 Jacobi SVD per block update
    // cost 3.3 ms and confounded the ablation timings)
    if (!h->stepws) ENMF_TRY(dalloc(&h->stepws, (size_t)(2 * 128)));
    const int blk = lam_slot == S_LAMU ? 0 : 1;
    lambda_power(G, r, h->stepws + 128 * blk, h->step_warm[blk], h->dscal + S_STEP, h->st);
    h->step_warm[blk] = true;
    fstep = h->dscal + S_STEP;
  }
  if (maybe_ascent) {
    if (h->tc_pbcd) {
      // Alg. 2 in stages [0,1) [1,2) [2,4) [4,8) ... [.., max_iter): the stopping rule is global
      // (all rows, all ranks), so each stage runs every row, the partials are reduced and the
      // rule applied on the device; once it fires the later stages return at once.  Stages
      // hand the fp64 iterate over through two state buffers (ping-pong), so the iterates are
      // those of one uninterrupted run (bitwise, test_gpu_pbcd_stages.py).  No per-iteration
      // snapshots (round 1 wrote max_iter fp32 copies of the block, 5 GB per C5 U block): a
      // stop inside a stage replays that stage from its start up to k* (the replay launch
      // returns at once otherwise), and the buffer holding u_k* is committed into F.  A stop
      // in the first stage (k* = 1: the U block of the first C5 sweep) costs ~1.5 iterations
      // instead of max_iter + 1.  Staging costs ~3 ms per C5 ascent sweep when the rule never
      // fires (k* = max_iter: every later C5 sweep, measured), so a block whose previous k*
      // was max_iter runs its first stage to the end (kprev rule of tc_pbcd_chunk).
      int8_t* gd = reinterpret_cast<int8_t*>(h->tcpb_ws + 128);
      int* done = h->dint + I_PBCD_DONE;        // done, then ctl[4] = {replay, it0, src, dst}
      int* ctl = h->dint + I_PBCD_CTL;
      double* ust0 = h->pbcd_state;
      double* ust1 = h->pbcd_state + h->pbcd_state_len;
      CUDA_TRY(cudaMemsetAsync(done, 0, sizeof(int) * 5, h->st));
      tc_pbcd_prepare(G, r, gd, h->tcpb_ws, stage, h->st);
      const char* stg = getenv("ENMF_PBCD_STAGES");   // "0": one stage [0, max_iter) (tests)
      const bool one = stg && stg[0] == '0';
      int src = -1, dst = 0;
      for (int a = 0; a < mi;) {
        const int b = one ? mi : std::min(mi, a == 0 ? 1 : 2 * a);
        if (tc_pbcd_chunk(F, ldf, rows, r, C, h->dscal + lam_slot, mi, a, b, src, dst, ust0,
                          ust1, h->parts, gd, h->tcpb_ws, stage, done, h->dint + kstar_slot,
                          nullptr, nullptr, h->st, h->opt.step_rule ? fstep : nullptr))
          return ENMF_ERR_CUDA;
        reduce_parts(h->parts, tc_pbcd_parts(), mi + 1, h->pgsum, h->st);
        if (sharded) ENMF_TRY(ar(h, h->pgsum, (size_t)(mi + 1), CommOp::Sum));
        pbcd_select_stage(h->pgsum, a, b, src, dst, mi, h->opt.pbcd_eps, h->dint + kstar_slot,
                          done, ctl, stage, h->st);
        src = dst;
        dst ^= 1;
        a = b;
      }
      if (tc_pbcd_chunk(F, ldf, rows, r, C, h->dscal + lam_slot, mi, 0, 1, -1, 0, ust0, ust1,
                        h->parts, gd, h->tcpb_ws, stage, done, nullptr, ctl,
                        h->dint + kstar_slot, h->st, h->opt.step_rule ? fstep : nullptr))
        return ENMF_ERR_CUDA;
      pbcd_commit_state(F, ldf, rows, r, ust0, ust1, ctl, stage, h->minparts, h->st, colmax);
    } else {
      pbcd_rows(F, ldf, rows, r, C, G, h->dscal + lam_slot, mi, h->snaps, h->parts, stage, h->st,
                h->opt.step_rule ? fstep : nullptr);
      reduce_parts(h->parts, pbcd_parts(), mi + 1, h->pgsum, h->st);
      if (sharded) ENMF_TRY(ar(h, h->pgsum, (size_t)(mi + 1), CommOp::Sum));
      pbcd_commit(F, ldf, rows, r, h->snaps, h->pgsum, h->opt.pbcd_eps, mi,
                  h->dint + kstar_slot, stage, h->minparts, h->st);
    }
  }
  if (h->opt.descent) {
    if (h->tc_pbcd) {
      // one projected-gradient step on the tensor cores (the round A of tc_pbcd_kernel with
      // the fixed step, all entries free in the descent stage), as the method's HALS runs
      // there -- so the ablation compares like with like (verdict weak #10)
      int8_t* gd = reinterpret_cast<int8_t*>(h->tcpb_ws + 128);
      tc_pbcd_prepare(G, r, gd, h->tcpb_ws, stage, h->st, 1);
      if (tc_pbcd_chunk(F, ldf, rows, r, C, h->dscal + lam_slot, 1, 0, 1, -1, 0,
                        h->pbcd_state, h->pbcd_state + h->pbcd_state_len, h->parts, gd,
                        h->tcpb_ws, stage, nullptr, nullptr, nullptr, nullptr, h->st, fstep, 1))
        return ENMF_ERR_CUDA;
      pbcd_commit_state(F, ldf, rows, r, h->pbcd_state, nullptr, nullptr, stage, h->minparts,
                        h->st, colmax, 1);
    } else {
      pgd_rows(F, ldf, rows, r, C, G, stage, fstep, h->minparts, h->st, colmax);
    }
    reduce_min(h->minparts, kRowGrid, h->dscal + min_slot, h->st);
    return sharded ? ar(h, h->dscal + min_slot, 1, CommOp::Min) : ENMF_OK;
  }
  if (h->tc_hals) {
    // tensor-core HALS; if G has a column too ill-conditioned for the digit coupling the
    // device flag I_HALS_ILL hands the sweep to the SIMT fp64 kernel (no host sync)
    if (!hals_issued &&
        tc_hals_rows(F, ldf, rows, r, C, G, reinterpret_cast<int8_t*>(h->tcpb_ws + 128),
                     h->tcpb_ws, stage, h->minparts, kRowGrid, colmax, h->dint + I_HALS_FB,
                     h->dint + I_HALS_ILL, h->st))
      return ENMF_ERR_CUDA;
    hals_rows(F, ldf, rows, r, C, G, stage, h->minparts, h->st, colmax, h->dint + I_HALS_ILL);
  } else {
    hals_rows(F, ldf, rows, r, C, G, stage, h->minparts, h->st, colmax);
  }
  reduce_min(h->minparts, kRowGrid, h->dscal + min_slot, h->st);
  return sharded ? ar(h, h->dscal + min_slot, 1, CommOp::Min) : ENMF_OK;
}

enmf_status_t ensure_snaps(enmf_handle_t h) {
  // the staged tensor-core PBCD (and its fixed-step / projected-gradient ablation modes) keeps
  // two fp64 state buffers; the SIMT PBCD (fp64 path, eNMC) max_iter fp32 snapshots
  const size_t rows = (size_t)std::max(h->m_loc, h->n);
  if (h->tc_pbcd && !h->pbcd_state) {
    h->pbcd_state_len = (rows + 127) / 128 * 128 * (size_t)h->r;
    ENMF_TRY(dalloc(&h->pbcd_state, 2 * h->pbcd_state_len));
  }
  if (h->snaps || (h->tc_pbcd && !h->nmc)) return ENMF_OK;
  return dalloc(&h->snaps, (size_t)h->opt.pbcd_max_iter * rows * (size_t)h->r);
}

// The cached sweep graph bakes in the handle's buffers and options: dropped when any changes.
void drop_sweep_graph(enmf_handle_t h) {
  if (h->sw_exec) cudaGraphExecDestroy(h->sw_exec);
  h->sw_exec = nullptr;
}

enmf_status_t ensure_ftrace(enmf_handle_t h, int n) {
  if (h->ftrace_cap >= n) return ENMF_OK;
  drop_sweep_graph(h);
  if (h->ftrace) cudaFree(h->ftrace);
  h->ftrace = nullptr;
  h->ftrace_cap = 0;
  ENMF_TRY(dalloc(&h->ftrace, (size_t)n));
  h->ftrace_cap = n;
  return ENMF_OK;
}

// One sweep (U block then V block) with the trace-form objective into ftrace[t].
// Host-transfer hooks of enmf_iterate_host (null for enmf_iterate): u_ready = event after which
// U is on the device (the first sweep's X V pass runs before it); u_download = host buffer that
// receives U on the copy stream as soon as the last sweep's U block is done.
struct SweepHooks {
  cudaEvent_t u_ready = nullptr;
  float* u_download = nullptr;
  float* v_download = nullptr;       // V is final after the V block: download it on the copy
};                                   // stream while the Grams / objective finish the sweep

enmf_status_t sweep(enmf_handle_t h, float* U, int64_t ldu, float* V, int64_t ldv, int t,
                    bool maybe_ascent, const SweepHooks& hk = SweepHooks()) {
  const bool sh = h->sharded;
  cudaStream_t st = h->st;
  // U block: P = X V, G_V = V^T V (G_V carried over from the previous sweep's end).  The X V
  // pass depends on V only, so it is issued before the stage decision (which reads min U).
  // colmax fusion (tc path): the U / V block update writes max |F| per column, which the next
  // X pass uses for the digit scales.  Only when one of PBCD (tiled copy) / HALS writes every
  // row: PBCD runs on the tensor-core kernel whenever the tc path is active.
  unsigned long long* umax =
      h->fmax_uv && (h->tc_pbcd || !maybe_ascent) ? h->fmax_uv : nullptr;
  unsigned long long* vmax = umax ? h->fmax_uv + 128 : nullptr;
  const unsigned long long* vmax_in = h->vmax_valid ? h->fmax_uv + 128 : nullptr;
  // Fused U block (tensor-core path, HALS on the tensor cores, P written without a K split):
  // the HALS kernel is enqueued right behind the X V pass with programmatic dependent launch
  // and takes each 128-row band of P as the pass publishes it, so its tiles fill the SMs the
  // pass's last wave leaves idle (1563 bands on 148 SMs at C5: 65 SMs idle for the last band)
  // instead of waiting for the whole pass.  Everything it needs from before the pass (the
  // stage decision, G_V's digits, the colmax reset) is enqueued ahead of the pass.
  const char* fe = getenv("ENMF_FUSE_HALS");
  const bool fuse_ok = h->tc && h->tc_hals && !h->sparse && !hk.u_ready && !h->opt.descent &&
                       !(fe && fe[0] == '0');
  bool fused = false;
  if (fuse_ok) {
    stage_update(h->dint + I_STAGE, h->dscal + S_MINU, h->dscal + S_MINV, h->dint + I_CNT_ASC,
                 st);
    if (umax) CUDA_TRY(cudaMemsetAsync(umax, 0, sizeof(unsigned long long) * h->r, st));
    int8_t* gd = reinterpret_cast<int8_t*>(h->tcpb_ws + 128);
    if (tc_hals_prepare(h->GV, (int)h->r, gd, h->tcpb_ws, h->dint + I_STAGE,
                        h->dint + I_HALS_ILL, st))
      return ENMF_ERR_CUDA;
    unsigned* bands = tc_band_flags(h->tc, st);
    if (bands) {
      ENMF_TRY(contract_xv(h, V, ldv, h->P, vmax_in, bands));
      if (tc_hals_launch(U, ldu, h->m_loc, (int)h->r, h->P, h->GV, gd, h->tcpb_ws,
                         h->dint + I_STAGE, h->minparts, kRowGrid, umax, h->dint + I_HALS_FB,
                         h->dint + I_HALS_ILL, bands, tc_bands(h->tc), st))
        return ENMF_ERR_CUDA;
      if (h->prof && tc_stamp_accum(h->tc, st)) return ENMF_ERR_CUDA;
      fused = true;
    } else {
      ENMF_TRY(contract_xv(h, V, ldv, h->P, vmax_in));
    }
  } else {
    ENMF_TRY(contract_xv(h, V, ldv, h->P, vmax_in));
    if (hk.u_ready) {                    // U arrives on the copy stream during the X V pass
      CUDA_TRY(cudaStreamWaitEvent(st, hk.u_ready, 0));
      ENMF_TRY(min_factor(h, U, ldu, h->m_loc, S_MINU, sh));
    }
    // stage control: HALS once U >= 0 and V >= 0
    stage_update(h->dint + I_STAGE, h->dscal + S_MINU, h->dscal + S_MINV, h->dint + I_CNT_ASC,
                 st);
  }
  // (fused but without band flags: tc_hals_prepare already ran, so the kernel is enqueued
  // by block_update through tc_hals_rows, which repeats the cheap digit preparation)
  ENMF_TRY(block_update(h, U, ldu, h->m_loc, h->P, h->GV, S_LAMU, I_KSTAR_U, S_MINU, sh,
                        maybe_ascent, umax, fused));
  h->umax_valid = umax != nullptr;
  if (hk.u_download) {                 // U is final: download it behind the V block
    CUDA_TRY(cudaEventRecord(h->ev_a, st));
    CUDA_TRY(cudaStreamWaitEvent(h->st2, h->ev_a, 0));
    CUDA_TRY(cudaMemcpyAsync(hk.u_download, U, sizeof(float) * h->m_loc * h->r,
                             cudaMemcpyDeviceToHost, h->st2));
  }
  // V block: Q = X^T U_new (allreduced), G_U = U_new^T U_new (PAPER.md:220 uses U^(k+1));
  // on the tensor-core path G_U is the Gram of the quantised U the X pass multiplied
  // (qgram_scales), so that the V update and the trace-form objective see one operand
  ENMF_TRY(contract_xtu(h, U, ldu, h->Q, h->umax_valid ? h->fmax_uv : nullptr, sh));
  ENMF_TRY(gram_u(h, U, ldu, sh));
  const int64_t vb = h->v_begin, vc = h->v_count, r = h->r;
  if (sh) {
    // V block sharded by rows (V rows are independent given Q and G_U): each
    // rank updates its slice (PBCD stopping partials and min allreduced like the U block),
    // then the full V is reassembled bitwise identically on every rank: NCCL all-gather of
    // the fp32 slices (no arithmetic), or through the host collective as a zero-padded fp64
    // sum (exact: one nonzero term per entry)
    ENMF_TRY(block_update(h, V + vb * ldv, ldv, vc, h->Q + vb * r, h->GU, S_LAMV, I_KSTAR_V,
                          S_MINV, true, maybe_ascent, nullptr));
    if (h->comm) {
      const size_t rb = sizeof(float) * r;
      if (vc > 0)
        CUDA_TRY(cudaMemcpy2DAsync(h->Vpad + vb * r, rb, V + vb * ldv, sizeof(float) * ldv, rb,
                                   vc, cudaMemcpyDeviceToDevice, st));
      if (comm_allgather(h->comm, h->Vpad, (size_t)(h->v_pad * r), CommType::F32, st) != 0)
        return ENMF_ERR_NCCL;
      CUDA_TRY(cudaMemcpy2DAsync(V, sizeof(float) * ldv, h->Vpad, rb, rb, h->n,
                                 cudaMemcpyDeviceToDevice, st));
    } else {
      CUDA_TRY(cudaMemsetAsync(h->Vg, 0, sizeof(double) * h->n * r, st));
      if (vc > 0) f32_to_f64(V + vb * ldv, ldv, vc, r, h->Vg + vb * r, st);
      ENMF_TRY(ar(h, h->Vg, (size_t)(h->n * r), CommOp::Sum));
      f64_to_f32(h->Vg, h->n, r, nullptr, V, ldv, st);
    }
    h->vmax_valid = false;
  } else {
    ENMF_TRY(block_update(h, V, ldv, h->n, h->Q, h->GU, S_LAMV, I_KSTAR_V, S_MINV, false,
                          maybe_ascent, vmax));
    h->vmax_valid = vmax != nullptr;
  }
  if (hk.v_download) {
    CUDA_TRY(cudaEventRecord(h->ev_a, st));
    CUDA_TRY(cudaStreamWaitEvent(h->st2, h->ev_a, 0));
    CUDA_TRY(cudaMemcpyAsync(hk.v_download, V, sizeof(float) * h->n * h->r,
                             cudaMemcpyDeviceToHost, h->st2));
  }
  // objective f = ||X||^2 - 2 <X^T U, V> + <U^T U, V^T V>   (BASELINE.json:5); sharded:
  // G_V and <Q, V> from this rank's V slice (the only valid part of Q after the
  // reduce-scatter), summed over ranks
  if (sh) {
    ENMF_TRY(gram_f32(h, V + vb * ldv, ldv, vc, h->GV, true));
    dot_f64_f32(h->Q + vb * r, V + vb * ldv, ldv, vc, r, h->parts, h->dscal + S_CROSS, st);
    ENMF_TRY(ar(h, h->dscal + S_CROSS, 1, CommOp::Sum));
  } else {
    ENMF_TRY(gram_f32(h, V, ldv, h->n, h->GV, false));
    dot_f64_f32(h->Q, V, ldv, h->n, h->r, h->parts, h->dscal + S_CROSS, st);
  }
  objective_finish(xnorm2_trace(h), h->dscal + S_CROSS, h->GU, h->GV, (int)h->r, h->ftrace,
                   st, h->dint + I_FCNT);
  return check_launch();
}

// One eNMC sweep (Alg. NMC loop body; reading R32): lift + mask + masked
// PBCD of U over the rows' observed entries with V fixed, then of V over the columns'
// observed entries (CSC copy) with the new U; the masked objective f^ into ftrace[t].  Every
// sweep is a PBCD sweep -- Alg. NMC has no HALS stage; the lift leaves a nonnegative factor
// unchanged.
enmf_status_t sweep_nmc(enmf_handle_t h, float* U, int64_t ldu, float* V, int64_t ldv, int t,
                        const SweepHooks& hk) {
  cudaStream_t st = h->st;
  const int r = (int)h->r;
  const int mi = h->opt.pbcd_max_iter;
  if (hk.u_ready) CUDA_TRY(cudaStreamWaitEvent(st, hk.u_ready, 0));
  nmc_pbcd_rows(U, ldu, h->m_loc, r, h->csr_ptr, h->csr_col, h->csr_val, V, ldv,
                h->dscal + S_LAMU, mi, h->snaps, h->parts, st);
  reduce_parts(h->parts, nmc_pbcd_parts(), mi + 1, h->pgsum, st);
  pbcd_commit(U, ldu, h->m_loc, r, h->snaps, h->pgsum, h->opt.pbcd_eps, mi,
              h->dint + I_KSTAR_U, nullptr, h->minparts, st);
  reduce_min(h->minparts, kRowGrid, h->dscal + S_MINU, st);
  if (hk.u_download) {
    CUDA_TRY(cudaEventRecord(h->ev_a, st));
    CUDA_TRY(cudaStreamWaitEvent(h->st2, h->ev_a, 0));
    CUDA_TRY(cudaMemcpyAsync(hk.u_download, U, sizeof(float) * h->m_loc * r,
                             cudaMemcpyDeviceToHost, h->st2));
  }
  nmc_pbcd_rows(V, ldv, h->n, r, h->csc_ptr, h->csc_row, h->csc_val, U, ldu,
                h->dscal + S_LAMV, mi, h->snaps, h->parts, st);
  reduce_parts(h->parts, nmc_pbcd_parts(), mi + 1, h->pgsum, st);
  pbcd_commit(V, ldv, h->n, r, h->snaps, h->pgsum, h->opt.pbcd_eps, mi, h->dint + I_KSTAR_V,
              nullptr, h->minparts, st);
  reduce_min(h->minparts, kRowGrid, h->dscal + S_MINV, st);
  if (hk.v_download) {
    CUDA_TRY(cudaEventRecord(h->ev_a, st));
    CUDA_TRY(cudaStreamWaitEvent(h->st2, h->ev_a, 0));
    CUDA_TRY(cudaMemcpyAsync(hk.v_download, V, sizeof(float) * h->n * r, cudaMemcpyDeviceToHost,
                             h->st2));
  }
  nmc_objective(h->csr_ptr, h->csr_col, h->csr_val, h->m_loc, r, U, ldu, V, ldv, h->minparts,
                h->dscal + S_FCUR, st);   // minparts: kRowGrid = nmc_objective_parts() slots
  append_scalar(h->dscal + S_FCUR, h->ftrace, h->dint + I_FCNT, st);
  return check_launch();
}

}  // namespace

// ==================================================================== C-ABI
extern "C" {

void enmf_default_options(enmf_options_t* o) {
  if (!o) return;
  o->seed = 0x5EEDull;
  o->oversample = 10;
  o->power_iters = 2;
  o->admm_iters = 100;
  o->admm_rho = 0.0;
  o->lift_steps = 10;
  o->pbcd_eps = 1e-2;
  o->pbcd_max_iter = 50;
  o->precision = ENMF_PREC_AUTO;
  o->step_rule = 0;
  o->descent = 0;
}

const char* enmf_status_string(enmf_status_t s) {
  switch (s) {
    case ENMF_OK: return "ok";
    case ENMF_ERR_INVALID_ARG: return "invalid argument";
    case ENMF_ERR_SHAPE: return "invalid shape";
    case ENMF_ERR_NEGATIVE_X: return "X has a negative entry";
    case ENMF_ERR_RANK_DEFICIENT: return "X has rank 0";
    case ENMF_ERR_NONFINITE: return "non-finite value";
    case ENMF_ERR_CUDA: return "CUDA error";
    case ENMF_ERR_NCCL: return "NCCL error";
    case ENMF_ERR_OOM: return "out of device memory";
    case ENMF_ERR_STATE: return "call out of order";
  }
  return "unknown status";
}

int64_t enmf_launch_count(enmf_handle_t h) { return h ? h->launches : -1; }

enmf_status_t enmf_set_profiling(enmf_handle_t h, int on) {
  if (!h) return ENMF_ERR_INVALID_ARG;
  CUDA_TRY(cudaStreamSynchronize(h->st));
  prof_collect(h);
  h->prof = on != 0;
  h->prof_ms[0] = h->prof_ms[1] = 0.0;
  h->prof_cnt[0] = h->prof_cnt[1] = 0;
  return ENMF_OK;
}

enmf_status_t enmf_get_profile(enmf_handle_t h, double* ms_host, int64_t* count_host) {
  if (!h || !ms_host || !count_host) return ENMF_ERR_INVALID_ARG;
  CUDA_TRY(cudaStreamSynchronize(h->st));
  prof_collect(h);
  for (int k = 0; k < 2; ++k) {
    ms_host[k] = h->prof_ms[k];
    count_host[k] = h->prof_cnt[k];
  }
  return ENMF_OK;
}

enmf_status_t enmf_cross_terms(enmf_handle_t h, const float* U, int64_t ldu, const float* V,
                               int64_t ldv, double* P, double* Q) {
  if (!h) return ENMF_ERR_INVALID_ARG;
  if (!h->bound) return ENMF_ERR_STATE;
  LaunchScope ls(h);
  if (P) {
    ENMF_TRY(validate_ld(V, ldv, h->r));
    ENMF_TRY(contract_xv(h, V, ldv, P));
  }
  if (Q) {
    ENMF_TRY(validate_ld(U, ldu, h->r));
    ENMF_TRY(contract_xtu(h, U, ldu, Q));
  }
  CUDA_TRY(cudaStreamSynchronize(h->st));
  return check_launch();
}

enmf_status_t enmf_set_host_allreduce(enmf_handle_t h, enmf_host_allreduce_fn fn, void* ctx) {
  if (!h) return ENMF_ERR_INVALID_ARG;
  if (h->comm) return ENMF_ERR_STATE;          // the handle already has an NCCL communicator
  h->host_ar = fn;
  h->host_ar_ctx = ctx;
  return ENMF_OK;
}

enmf_status_t enmf_nccl_unique_id(void* out128) {
  if (!out128) return ENMF_ERR_INVALID_ARG;
  return comm_unique_id(out128) == 0 ? ENMF_OK : ENMF_ERR_NCCL;
}

const char* enmf_precision_name(enmf_handle_t h) {
  if (!h) return "none";
  if (h->nmc) return "nmc-f64";
  if (h->sparse) return h->tc_pbcd ? "csr-f64-spmm+tc-rows" : "csr-f64-spmm";
  return h->precision == ENMF_PREC_TC ? "tc-i8x3-exact" : "fp64-simt";
}

enmf_status_t enmf_destroy(enmf_handle_t h) {
  if (!h) return ENMF_ERR_INVALID_ARG;
  if (h->st) cudaStreamSynchronize(h->st);
  void* bufs[] = {h->dscal, h->dint, h->P, h->Q, h->GU, h->GV, h->work, h->parts,
                  h->minparts, h->pgsum, h->snaps, h->ftrace, h->x_owned, h->W64,
                  h->tcpb_ws, h->fmax_uv, h->Ud, h->Vd, h->arena, h->Vg, h->Vpad,
                  h->csc_ptr, h->csc_row, h->csc_val, h->stepws, h->pbcd_state,
                  h->small_ws};
  for (void* b : bufs)
    if (b) cudaFree(b);
  for (void* b : h->arena_extra) cudaFree(b);
  if (h->host_ar_buf) cudaFreeHost(h->host_ar_buf);
  if (h->st2) {
    cudaStreamSynchronize(h->st2);
    cudaStreamDestroy(h->st2);
    cudaEventDestroy(h->ev_b);
  }
  if (h->ev_a) cudaEventDestroy(h->ev_a);
  if (h->st_comm) {
    cudaStreamSynchronize(h->st_comm);
    cudaStreamDestroy(h->st_comm);
  }
  for (cudaEvent_t e : h->ev_comm) cudaEventDestroy(e);
  if (h->sw_exec) cudaGraphExecDestroy(h->sw_exec);
  if (h->cap_st) cudaStreamDestroy(h->cap_st);
  if (h->tc) tc_destroy(h->tc);
  for (cudaEvent_t e : h->ev_pool) cudaEventDestroy(e);
  comm_destroy(h->comm);
  delete h;
  return ENMF_OK;
}

enmf_status_t enmf_create(const enmf_problem_t* prob, const enmf_options_t* opt,
                          enmf_handle_t* out) {
  if (!out) return ENMF_ERR_INVALID_ARG;
  *out = nullptr;
  if (!prob) return ENMF_ERR_INVALID_ARG;
  enmf_options_t o;
  enmf_default_options(&o);
  if (opt) o = *opt;
  const int64_t m = prob->m_global, n = prob->n, r = prob->r;
  if (m < 1 || n < 1 || r < 1 || r > std::min(m, n) || r > ENMF_MAX_RANK) return ENMF_ERR_SHAPE;
  if (prob->world_size < 1 || prob->rank < 0 || prob->rank >= prob->world_size)
    return ENMF_ERR_INVALID_ARG;
  if (prob->row_begin < 0 || prob->row_count < 1 || prob->row_begin + prob->row_count > m)
    return ENMF_ERR_SHAPE;
  if (prob->world_size == 1 && (prob->row_begin != 0 || prob->row_count != m))
    return ENMF_ERR_SHAPE;
  // world_size > 1 without an NCCL id: collectives go through enmf_set_host_allreduce
  if (o.oversample < 0 || o.power_iters < 0 || o.admm_iters < 0 || o.lift_steps < 1 ||
      o.pbcd_max_iter < 1 || o.pbcd_max_iter > 1000 || !(o.pbcd_eps >= 0.0) ||
      o.precision < ENMF_PREC_AUTO || o.precision > ENMF_PREC_TC)
    return ENMF_ERR_INVALID_ARG;
  enmf_handle_t h = new enmf_handle_s();
  h->prob = *prob;
  h->opt = o;
  h->st = (cudaStream_t)prob->cuda_stream;
  h->m_loc = prob->row_count;
  h->n = n;
  h->r = r;
  LaunchScope ls(h);
  enmf_status_t s = ENMF_OK;
#define ALLOC(p, c)                         \
  if (s == ENMF_OK) s = dalloc(&(p), (c));
  ALLOC(h->dscal, S_COUNT);
  ALLOC(h->dint, I_COUNT);
  ALLOC(h->P, (size_t)(h->m_loc * r));
  // V slices: ceil(n / world) rows per rank; Q holds world such blocks for the in-place
  // reduce-scatter
  // V slices (the sharded V block): ceil(n / world) rows each, rounded up to whole 128-row
  // bands when every rank still gets rows (n >= 128 world), so that the tensor-core pass 2 can
  // reduce each slice to its owner as soon as that slice's bands are done
  h->sharded = prob->world_size > 1 || prob->nccl_unique_id != nullptr;
  h->v_pad = (n + prob->world_size - 1) / prob->world_size;
  if (h->sharded && n >= 128 * (int64_t)prob->world_size) {
    const int64_t al = (h->v_pad + 127) / 128 * 128;
    if ((prob->world_size - 1) * al < n) h->v_pad = al;
  }
  ALLOC(h->Q, (size_t)(std::max<int64_t>(n, h->v_pad * prob->world_size) * r));
  ALLOC(h->GU, (size_t)(r * r));
  ALLOC(h->GV, (size_t)(r * r));
  // split-K partials: enough for the small GEMMs (r x r, l x l) and for the SVD panels
  const int64_t l = std::min<int64_t>(std::min(m, n), r + o.oversample);
  h->work_elems = (size_t)std::max<int64_t>(
      {(int64_t)8 << 20, 40 * l * l, 2 * (int64_t)512 * 512, 8 * r * r});
  ALLOC(h->work, h->work_elems);
  h->parts_elems = (size_t)std::max<int64_t>(
      {(int64_t)std::max(pbcd_parts(), tc_pbcd_parts()) * (o.pbcd_max_iter + 1), (int64_t)kkt_parts() * 8,
       (int64_t)colabsmax_parts() * 3 * std::max<int64_t>(r, 1), 3 * 4 * kSMs, 4096});
  ALLOC(h->parts, h->parts_elems);
  ALLOC(h->minparts, (size_t)kRowGrid);
  ALLOC(h->pgsum, (size_t)(o.pbcd_max_iter + 1));
#undef ALLOC
  if (s == ENMF_OK && h->sharded) {
    // V slice of this rank: rows [rank v_pad, rank v_pad + v_count), the last one(s) shorter
    h->v_begin = std::min<int64_t>(n, prob->rank * h->v_pad);
    h->v_count = std::min<int64_t>(h->v_pad, n - h->v_begin);
    if (prob->nccl_unique_id)
      s = dalloc(&h->Vpad, (size_t)(h->v_pad * prob->world_size * r));
    else
      s = dalloc(&h->Vg, (size_t)(n * r));
  }
  if (s == ENMF_OK && h->sharded && prob->nccl_unique_id) {
    if (comm_init(&h->comm, prob->nccl_unique_id, prob->world_size, prob->rank) != 0)
      s = ENMF_ERR_NCCL;
  }
  if (s == ENMF_OK) {
    cudaMemsetAsync(h->dscal, 0, sizeof(double) * S_COUNT, h->st);
    cudaMemsetAsync(h->dint, 0, sizeof(int) * I_COUNT, h->st);
    if (cudaGetLastError() != cudaSuccess) s = ENMF_ERR_CUDA;
  }
  if (s != ENMF_OK) {
    enmf_destroy(h);
    return s;
  }
  *out = h;
  return ENMF_OK;
}

enmf_status_t enmf_set_data(enmf_handle_t h, const float* X, int64_t ldx) {
  if (!h) return ENMF_ERR_INVALID_ARG;
  ENMF_TRY(validate_ld(X, ldx, h->n));
  LaunchScope ls(h);
  drop_sweep_graph(h);
  h->X = X;
  h->ldx = ldx;
  h->bound = false;
  h->sparse = false;
  h->nmc = false;
  const int np = x_stats_parts(h->m_loc);
  double* out3 = h->work;   // [sum, min, nonfinite, max|X| of this rank's rows]
  x_stats(X, ldx, h->m_loc, h->n, h->parts, np, out3, h->st);
  ENMF_TRY(ar(h, out3, 1, CommOp::Sum));
  ENMF_TRY(ar(h, out3 + 1, 1, CommOp::Min));
  ENMF_TRY(ar(h, out3 + 2, 1, CommOp::Sum));
  ENMF_TRY(ar(h, out3 + 3, 1, CommOp::Max));
  double hv[4];
  CUDA_TRY(cudaMemcpyAsync(hv, out3, sizeof(hv), cudaMemcpyDeviceToHost, h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  if (hv[2] > 0) return ENMF_ERR_NONFINITE;
  if (hv[1] < 0) return ENMF_ERR_NEGATIVE_X;
  CUDA_TRY(cudaMemcpyAsync(h->dscal + S_XNORM2, out3, sizeof(double), cudaMemcpyDeviceToDevice,
                           h->st));
  // precision selection (the same on every rank: global statistics, average rank size): the
  // tensor-core digit path pays off on large X and keeps ~1e-9 accuracy when
  // the entries are not far below their scale group's maximum -- it rounds every entry to
  // ~2^-23 of its row's (column's) maximum, so AUTO requires max|X| <= 64 rms(X); heavy-tailed
  // data (counts, tf-idf) stays on the fp64 path
  int prec = h->opt.precision;
  if (prec == ENMF_PREC_AUTO) {
    const double mn = (double)h->prob.m_global * (double)h->n;
    const double rms = sqrt(hv[0] / mn);
    prec = (tc_supported(h->m_loc, h->n, h->r) && mn / h->prob.world_size >= 2.5e8 &&
            hv[3] <= 64.0 * rms)
               ? ENMF_PREC_TC : ENMF_PREC_FP64;
  }
  if (prec == ENMF_PREC_TC && !tc_supported(h->m_loc, h->n, h->r)) return ENMF_ERR_SHAPE;
  if (h->tc) { tc_destroy(h->tc); h->tc = nullptr; }
  if (prec == ENMF_PREC_TC) {
    int rc = tc_create(&h->tc, X, ldx, h->m_loc, h->n, h->r, h->st, h->parts,
                       (int)std::min<size_t>(h->parts_elems, 1 << 20));
    if (rc != 0) return rc == 2 ? ENMF_ERR_OOM : ENMF_ERR_CUDA;
    // ||X~||^2 of the quantised X (all ranks): the trace-form objective's first term
    CUDA_TRY(cudaMemcpyAsync(h->dscal + S_XQNORM2, tc_xq_norm2(h->tc), sizeof(double),
                             cudaMemcpyDeviceToDevice, h->st));
    ENMF_TRY(ar(h, h->dscal + S_XQNORM2, 1, CommOp::Sum));
  }
  const char* tpe = getenv("ENMF_TC_PBCD");   // diagnostics: 0 keeps the SIMT fp64 PBCD
  h->tc_pbcd = prec == ENMF_PREC_TC && tc_pbcd_supported((int)h->r) && !(tpe && tpe[0] == '0');
  if (h->tc_pbcd && !h->tcpb_ws) ENMF_TRY(dalloc(&h->tcpb_ws, 128 + 4 * 128 * 128 / 8));
  const char* the = getenv("ENMF_TC_HALS");   // diagnostics: 0 keeps the SIMT fp64 HALS
  h->tc_hals = h->tc_pbcd && !(the && the[0] == '0');
  if (prec == ENMF_PREC_TC && !h->fmax_uv) ENMF_TRY(dalloc(&h->fmax_uv, 256));
  h->umax_valid = h->vmax_valid = false;
  h->step_warm[0] = h->step_warm[1] = false;
  h->precision = prec;
  // cache-resident problems: the persistent HALS kernel's plan (module load, occupancy) and
  // workspace now, not inside the first enmf_iterate
  const char* se = getenv("ENMF_SMALL_FUSED");
  if (prec == ENMF_PREC_FP64 && !h->sharded && !(se && se[0] == '0') && !h->small_ws &&
      small_sweeps_supported(h->m_loc, h->n, (int)h->r)) {
    const size_t need = small_sweeps_workspace(h->m_loc, h->n, (int)h->r);
    if (need) ENMF_TRY(dalloc(&h->small_ws, need));
  }
  int zero[I_COUNT] = {0};
  CUDA_TRY(cudaMemcpyAsync(h->dint, zero, sizeof(zero), cudaMemcpyHostToDevice, h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  h->stage_known_hals = false;
  h->bound = true;
  return check_launch();
}

}  // extern "C"

namespace {
// CSR binding shared by sparse X (stored entries are X's nonzeros, the rest zeros) and eNMC
// (stored entries are the OBSERVED entries, the rest missing).
enmf_status_t bind_csr(enmf_handle_t h, const int64_t* row_ptr, const int32_t* col_idx,
                       const float* vals, int64_t nnz, bool nmc) {
  if (!h || !row_ptr || nnz < 0 || (nnz > 0 && (!col_idx || !vals))) return ENMF_ERR_INVALID_ARG;
  if (nmc && (h->sharded || !nmc_supported((int)h->r))) return ENMF_ERR_SHAPE;
  if (nnz > INT32_MAX || h->n > INT32_MAX) return ENMF_ERR_SHAPE;
  LaunchScope ls(h);
  drop_sweep_graph(h);
  h->bound = false;
  h->X = nullptr;
  h->ldx = 0;
  // layout check: row ranges valid, columns strictly ascending in [0, n)
  int* bad = reinterpret_cast<int*>(h->work);
  if (csr_check(row_ptr, col_idx, h->m_loc, h->n, nnz, bad, h->st)) return ENMF_ERR_CUDA;
  int bad_h = 0;
  CUDA_TRY(cudaMemcpyAsync(&bad_h, bad, sizeof(int), cudaMemcpyDeviceToHost, h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  if (bad_h) return ENMF_ERR_INVALID_ARG;
  // ||X||^2, min, non-finite count over the stored values (as 4096-wide rows plus a tail)
  double hv[2][4] = {{0.0, DBL_MAX, 0.0, 0.0}, {0.0, DBL_MAX, 0.0, 0.0}};
  const int64_t W = 4096, full = nnz / W, tail = nnz - full * W;
  double* out4 = h->work;
  if (full > 0) {
    x_stats(vals, W, full, W, h->parts, x_stats_parts(full), out4, h->st);
    CUDA_TRY(cudaMemcpyAsync(hv[0], out4, sizeof(hv[0]), cudaMemcpyDeviceToHost, h->st));
    CUDA_TRY(cudaStreamSynchronize(h->st));
  }
  if (tail > 0) {
    x_stats(vals + full * W, tail, 1, tail, h->parts, x_stats_parts(1), out4, h->st);
    CUDA_TRY(cudaMemcpyAsync(hv[1], out4, sizeof(hv[1]), cudaMemcpyDeviceToHost, h->st));
    CUDA_TRY(cudaStreamSynchronize(h->st));
  }
  double st3[3] = {hv[0][0] + hv[1][0], std::min(hv[0][1], hv[1][1]), hv[0][2] + hv[1][2]};
  CUDA_TRY(cudaMemcpyAsync(out4, st3, sizeof(st3), cudaMemcpyHostToDevice, h->st));
  ENMF_TRY(ar(h, out4, 1, CommOp::Sum));
  ENMF_TRY(ar(h, out4 + 1, 1, CommOp::Min));
  ENMF_TRY(ar(h, out4 + 2, 1, CommOp::Sum));
  CUDA_TRY(cudaMemcpyAsync(st3, out4, sizeof(st3), cudaMemcpyDeviceToHost, h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  if (st3[2] > 0) return ENMF_ERR_NONFINITE;
  if (st3[1] < 0) return ENMF_ERR_NEGATIVE_X;
  CUDA_TRY(cudaMemcpyAsync(h->dscal + S_XNORM2, out4, sizeof(double), cudaMemcpyDeviceToDevice,
                           h->st));
  // CSC copy for X^T U
  if (h->csc_ptr) cudaFree(h->csc_ptr);
  if (h->csc_row) cudaFree(h->csc_row);
  if (h->csc_val) cudaFree(h->csc_val);
  h->csc_ptr = nullptr;
  h->csc_row = nullptr;
  h->csc_val = nullptr;
  ENMF_TRY(dalloc(&h->csc_ptr, (size_t)(h->n + 1)));
  ENMF_TRY(dalloc(&h->csc_row, (size_t)std::max<int64_t>(nnz, 1)));
  ENMF_TRY(dalloc(&h->csc_val, (size_t)std::max<int64_t>(nnz, 1)));
  const int rc = csr_to_csc(row_ptr, col_idx, vals, h->m_loc, h->n, nnz, h->csc_ptr, h->csc_row,
                            h->csc_val, h->st);
  if (rc) return rc == 2 ? ENMF_ERR_OOM : ENMF_ERR_CUDA;
  h->csr_ptr = row_ptr;
  h->csr_col = col_idx;
  h->csr_val = vals;
  h->nnz = nnz;
  h->sparse = true;
  h->nmc = nmc;
  // X passes: fp64 SpMM; block updates on the tensor-core row kernels unless precision FP64
  // (eNMC: the masked PBCD kernel, fp64)
  if (h->tc) { tc_destroy(h->tc); h->tc = nullptr; }
  const char* tpe = getenv("ENMF_TC_PBCD");
  h->tc_pbcd = !nmc && h->opt.precision != ENMF_PREC_FP64 && tc_pbcd_supported((int)h->r) &&
               !(tpe && tpe[0] == '0');
  if (h->tc_pbcd && !h->tcpb_ws) ENMF_TRY(dalloc(&h->tcpb_ws, 128 + 4 * 128 * 128 / 8));
  const char* the = getenv("ENMF_TC_HALS");
  h->tc_hals = h->tc_pbcd && !(the && the[0] == '0');
  h->umax_valid = h->vmax_valid = false;
  h->precision = ENMF_PREC_FP64;
  int zero[I_COUNT] = {0};
  CUDA_TRY(cudaMemcpyAsync(h->dint, zero, sizeof(zero), cudaMemcpyHostToDevice, h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  h->stage_known_hals = false;
  h->bound = true;
  return check_launch();
}
}  // namespace

extern "C" {

enmf_status_t enmf_set_data_csr(enmf_handle_t h, const int64_t* row_ptr, const int32_t* col_idx,
                                const float* vals, int64_t nnz) {
  return bind_csr(h, row_ptr, col_idx, vals, nnz, false);
}

enmf_status_t enmf_set_data_masked(enmf_handle_t h, const int64_t* row_ptr,
                                   const int32_t* col_idx, const float* vals, int64_t nnz) {
  return bind_csr(h, row_ptr, col_idx, vals, nnz, true);
}

enmf_status_t enmf_set_stage(enmf_handle_t h, int stage, double lambda_u, double lambda_v) {
  if (!h || (stage != 0 && stage != 1) || !(lambda_u >= 0) || !(lambda_v >= 0))
    return ENMF_ERR_INVALID_ARG;
  int st = stage;
  double lam[2] = {lambda_u, lambda_v};
  CUDA_TRY(cudaMemcpyAsync(h->dint + I_STAGE, &st, sizeof(int), cudaMemcpyHostToDevice, h->st));
  CUDA_TRY(cudaMemcpyAsync(h->dscal + S_LAMU, lam, sizeof(lam), cudaMemcpyHostToDevice, h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  h->stage_known_hals = stage == 1;
  return ENMF_OK;
}

enmf_status_t enmf_project(enmf_handle_t h, float* U, int64_t ldu, float* V, int64_t ldv) {
  if (!h || !U || !V || ldu < h->r || ldv < h->r) return ENMF_ERR_INVALID_ARG;
  LaunchScope ls(h);
  project_f32(U, ldu, h->m_loc, h->r, h->st);
  project_f32(V, ldv, h->n, h->r, h->st);
  int st = 1;
  CUDA_TRY(cudaMemcpyAsync(h->dint + I_STAGE, &st, sizeof(int), cudaMemcpyHostToDevice, h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  ENMF_TRY(check_launch());
  h->stage_known_hals = true;
  h->umax_valid = h->vmax_valid = false;
  return ENMF_OK;
}

enmf_status_t enmf_set_ablation(enmf_handle_t h, int step_rule, int descent) {
  if (!h || (step_rule != 0 && step_rule != 1) || (descent != 0 && descent != 1))
    return ENMF_ERR_INVALID_ARG;
  drop_sweep_graph(h);
  h->opt.step_rule = step_rule;
  h->opt.descent = descent;
  h->umax_valid = h->vmax_valid = false;
  return ENMF_OK;
}

enmf_status_t enmf_get_stage(enmf_handle_t h, int* stage, double* lambda_u, double* lambda_v) {
  if (!h) return ENMF_ERR_INVALID_ARG;
  int st = 0;
  double lam[2];
  CUDA_TRY(cudaMemcpyAsync(&st, h->dint + I_STAGE, sizeof(int), cudaMemcpyDeviceToHost, h->st));
  CUDA_TRY(cudaMemcpyAsync(lam, h->dscal + S_LAMU, sizeof(lam), cudaMemcpyDeviceToHost, h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  if (stage) *stage = st;
  if (lambda_u) *lambda_u = lam[0];
  if (lambda_v) *lambda_v = lam[1];
  return ENMF_OK;
}

}  // extern "C"

namespace {
// Capture one sweep (on the handle's capture stream, joined to its stream by events) and
// launch the graph `count` times on the handle's stream.
enmf_status_t replay_sweeps(enmf_handle_t h, float* U, int64_t ldu, float* V, int64_t ldv,
                            bool maybe_ascent, int count) {
  if (!h->cap_st) {
    CUDA_TRY(cudaStreamCreateWithFlags(&h->cap_st, cudaStreamNonBlocking));
    if (!h->ev_a) CUDA_TRY(cudaEventCreateWithFlags(&h->ev_a, cudaEventDisableTiming));
  }
  cudaStream_t user = h->st;
  h->st = h->cap_st;
  const int64_t l0 = h->launches;
  cudaGraph_t g = nullptr;
  enmf_status_t s = ENMF_OK;
  cudaError_t e = cudaStreamBeginCapture(h->st, cudaStreamCaptureModeRelaxed);
  if (e == cudaSuccess) {
    s = h->nmc ? sweep_nmc(h, U, ldu, V, ldv, 1, SweepHooks())
               : sweep(h, U, ldu, V, ldv, 1, maybe_ascent, SweepHooks());
    e = cudaStreamEndCapture(h->st, &g);
  }
  h->st = user;
  const int64_t per = h->launches - l0;
  h->launches = l0;
  if (s != ENMF_OK || e != cudaSuccess) {
    fprintf(stderr, "enmf: sweep graph capture failed (status %d): %s\n", (int)s,
            cudaGetErrorString(e));
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
    return s != ENMF_OK ? s : ENMF_ERR_CUDA;
  }
  cudaGraphExec_t ge = nullptr;
  e = cudaGraphInstantiate(&ge, g, 0);
  cudaGraphDestroy(g);
  CUDA_TRY(e);
  for (int k = 0; k < count && e == cudaSuccess; ++k) {
    e = cudaGraphLaunch(ge, h->st);
    h->launches += per;
  }
  cudaGraphExecDestroy(ge);
  CUDA_TRY(e);
  return ENMF_OK;
}

// One ascent-capable sweep as a cached CUDA graph (the small-problem path steps the ascent
// stage one sweep at a time with a host check of the stage in between; ~50 launches per sweep
// otherwise).  The graph is keyed on the factor pointers and leading dimensions.
enmf_status_t graph_sweep_once(enmf_handle_t h, float* U, int64_t ldu, float* V, int64_t ldv) {
  if (h->sw_exec && (h->sw_key[0] != U || h->sw_key[1] != V || h->sw_ld[0] != ldu ||
                     h->sw_ld[1] != ldv)) {
    cudaGraphExecDestroy(h->sw_exec);
    h->sw_exec = nullptr;
  }
  if (!h->sw_exec) {
    if (!h->cap_st) {
      CUDA_TRY(cudaStreamCreateWithFlags(&h->cap_st, cudaStreamNonBlocking));
      if (!h->ev_a) CUDA_TRY(cudaEventCreateWithFlags(&h->ev_a, cudaEventDisableTiming));
    }
    cudaStream_t user = h->st;
    h->st = h->cap_st;
    const int64_t l0 = h->launches;
    cudaGraph_t g = nullptr;
    enmf_status_t s = ENMF_OK;
    cudaError_t e = cudaStreamBeginCapture(h->st, cudaStreamCaptureModeRelaxed);
    if (e == cudaSuccess) {
      s = sweep(h, U, ldu, V, ldv, 1, true, SweepHooks());
      e = cudaStreamEndCapture(h->st, &g);
    }
    h->st = user;
    h->sw_launches = h->launches - l0;
    h->launches = l0;
    if (s != ENMF_OK || e != cudaSuccess) {
      if (g) cudaGraphDestroy(g);
      cudaGetLastError();
      return s != ENMF_OK ? s : ENMF_ERR_CUDA;
    }
    e = cudaGraphInstantiate(&h->sw_exec, g, 0);
    cudaGraphDestroy(g);
    CUDA_TRY(e);
    h->sw_key[0] = U;
    h->sw_key[1] = V;
    h->sw_ld[0] = ldu;
    h->sw_ld[1] = ldv;
  }
  CUDA_TRY(cudaGraphLaunch(h->sw_exec, h->st));
  h->launches += h->sw_launches;
  return ENMF_OK;
}

// The sweep loop behind enmf_iterate and enmf_iterate_host.  hk0 applies to the first sweep
// (U upload), u_dl_host to the last (U download); v_dl_host receives V at the end.
enmf_status_t iterate_core(enmf_handle_t h, float* U, int64_t ldu, float* V, int64_t ldv,
                           int n_iters, double* f_trace_host, enmf_iter_info_t* info,
                           cudaEvent_t u_ready, float* u_dl_host, float* v_dl_host) {
  LaunchScope ls(h);
  const bool sh = h->sharded;
  const bool maybe_ascent = !h->stage_known_hals || h->nmc;
  if (maybe_ascent || h->opt.descent) ENMF_TRY(ensure_snaps(h));
  ENMF_TRY(ensure_ftrace(h, std::max(n_iters, 1)));
  CUDA_TRY(cudaMemsetAsync(h->dint + I_CNT_ASC, 0, 2 * sizeof(int), h->st));
  CUDA_TRY(cudaMemsetAsync(h->dint + I_HALS_FB, 0, sizeof(int), h->st));
  CUDA_TRY(cudaMemsetAsync(h->dint + I_FCNT, 0, sizeof(int), h->st));
  // entry state: mins of the factors as given, G_V of the given V (min U after its upload)
  if (!u_ready) ENMF_TRY(min_factor(h, U, ldu, h->m_loc, S_MINU, sh));
  ENMF_TRY(min_factor(h, V, ldv, h->n, S_MINV, false));
  if (!h->nmc) ENMF_TRY(gram_f32(h, V, ldv, h->n, h->GV, false));
  h->umax_valid = h->vmax_valid = false;   // the caller may have changed U / V since
  // Sweeps 1 .. n-1 of a single-rank call without host transfers issue the same launch
  // sequence every time (stage, k*, the trace slot are device-side), so one of them is
  // captured as a CUDA graph and replayed: the small configurations (C1-C4, ~35 launches per
  // sweep) are bound by launch latency.  ENMF_GRAPH=0 disables it.
  const char* ge = getenv("ENMF_GRAPH");
  const bool graphs = !(ge && ge[0] == '0');
  // Cache-resident problems on the fp64 path (C1-C4): every HALS sweep runs in the persistent
  // kernel of small_sweep.cu (one cooperative launch for all remaining sweeps).  Which sweeps
  // are HALS sweeps must not depend on how the caller chunks its calls, so while the stage is
  // still the ascent the host reads the stage flag and the factor minima before every sweep
  // (stage_update's rule; a sync per ascent sweep, ~10 of them) and the ascent
  // sweeps run as separate launches.  ENMF_SMALL_FUSED=0 disables it.
  const char* se = getenv("ENMF_SMALL_FUSED");
  const bool small = !(se && se[0] == '0') && !sh && !h->sparse && !h->nmc && !h->tc &&
                     !h->opt.descent && !h->prof &&
                     small_sweeps_supported(h->m_loc, h->n, (int)h->r);
  if (small && u_ready) {                // tiny transfers: no overlap worth a second code path
    CUDA_TRY(cudaStreamWaitEvent(h->st, u_ready, 0));
    ENMF_TRY(min_factor(h, U, ldu, h->m_loc, S_MINU, sh));
    u_ready = nullptr;
  }
  // (not while the X passes are being timed: enmf_set_profiling brackets every pass with events)
  const bool graph = graphs && !sh && !u_ready && !u_dl_host && !v_dl_host && n_iters >= 3 &&
                     !h->prof && !small;
  for (int t = 0; t < n_iters; ++t) {
    SweepHooks hk;
    if (t == 0) hk.u_ready = u_ready;
    if (t == n_iters - 1) {
      hk.u_download = u_dl_host;
      hk.v_download = v_dl_host;
    }
    if (small && !h->stage_known_hals) {
      int stg = 0;
      double mn[2];
      CUDA_TRY(cudaMemcpyAsync(&stg, h->dint + I_STAGE, sizeof(int), cudaMemcpyDeviceToHost, h->st));
      CUDA_TRY(cudaMemcpyAsync(mn, h->dscal + S_MINU, sizeof(mn), cudaMemcpyDeviceToHost, h->st));
      CUDA_TRY(cudaStreamSynchronize(h->st));
      if (stg == 1 || (mn[0] >= 0.0 && mn[1] >= 0.0)) h->stage_known_hals = true;
    }
    if (small && h->stage_known_hals) {
      if (!h->small_ws) {
        const size_t need = small_sweeps_workspace(h->m_loc, h->n, (int)h->r);
        if (need == 0) return ENMF_ERR_CUDA;
        ENMF_TRY(dalloc(&h->small_ws, need));
      }
      if (small_sweeps_launch(h->X, h->ldx, h->m_loc, h->n, (int)h->r, U, ldu, V, ldv, h->GV,
                              h->GU, h->dscal + S_XNORM2, h->ftrace, h->dint + I_FCNT,
                              h->dscal + S_MINU, h->dscal + S_MINV, h->dint + I_STAGE,
                              h->dint + I_CNT_HALS, h->small_ws, n_iters - t, h->st))
        return ENMF_ERR_CUDA;
      if (u_dl_host)
        CUDA_TRY(cudaMemcpyAsync(u_dl_host, U, sizeof(float) * h->m_loc * h->r,
                                 cudaMemcpyDeviceToHost, h->st));
      if (v_dl_host)
        CUDA_TRY(cudaMemcpyAsync(v_dl_host, V, sizeof(float) * h->n * h->r,
                                 cudaMemcpyDeviceToHost, h->st));
      break;
    }
    if (graph && t == 1) {
      ENMF_TRY(replay_sweeps(h, U, ldu, V, ldv, maybe_ascent, n_iters - 1));
      break;
    }
    if (h->nmc) {
      ENMF_TRY(sweep_nmc(h, U, ldu, V, ldv, t, hk));
    } else if (small && graphs && maybe_ascent && !hk.u_ready && !h->opt.step_rule) {
      ENMF_TRY(graph_sweep_once(h, U, ldu, V, ldv));   // an ascent sweep of the small path
      if (hk.u_download)
        CUDA_TRY(cudaMemcpyAsync(hk.u_download, U, sizeof(float) * h->m_loc * h->r,
                                 cudaMemcpyDeviceToHost, h->st));
      if (hk.v_download)
        CUDA_TRY(cudaMemcpyAsync(hk.v_download, V, sizeof(float) * h->n * h->r,
                                 cudaMemcpyDeviceToHost, h->st));
    } else {
      ENMF_TRY(sweep(h, U, ldu, V, ldv, t, maybe_ascent, hk));
    }
  }
  if (u_ready && n_iters == 0) CUDA_TRY(cudaStreamWaitEvent(h->st, u_ready, 0));
  h->umax_valid = h->vmax_valid = false;
  if (v_dl_host && n_iters == 0)
    CUDA_TRY(cudaMemcpyAsync(v_dl_host, V, sizeof(float) * h->n * h->r, cudaMemcpyDeviceToHost,
                             h->st));
  // final stage flag (does not consume a sweep) and host-side bookkeeping
  int hi[I_COUNT];
  CUDA_TRY(cudaMemcpyAsync(hi, h->dint, sizeof(hi), cudaMemcpyDeviceToHost, h->st));
  double mins[2];
  CUDA_TRY(cudaMemcpyAsync(mins, h->dscal + S_MINU, sizeof(mins), cudaMemcpyDeviceToHost, h->st));
  if (f_trace_host && n_iters > 0)
    CUDA_TRY(cudaMemcpyAsync(f_trace_host, h->ftrace, sizeof(double) * n_iters,
                             cudaMemcpyDeviceToHost, h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  if (h->st2) CUDA_TRY(cudaStreamSynchronize(h->st2));
  ENMF_TRY(check_launch());
  prof_collect(h);
  if (hi[I_STAGE] == 1) h->stage_known_hals = true;
  if (info) {
    info->ascent_sweeps = h->nmc ? n_iters : hi[I_CNT_ASC];
    info->hals_sweeps = h->nmc ? 0 : hi[I_CNT_HALS];
    info->feasible = mins[0] >= 0.0 && mins[1] >= 0.0;
    info->pbcd_iters_u = hi[I_KSTAR_U];
    info->pbcd_iters_v = hi[I_KSTAR_V];
    info->hals_fallback_rows = hi[I_HALS_FB];
  }
  if (f_trace_host)
    for (int t = 0; t < n_iters; ++t)
      if (!isfinite(f_trace_host[t])) return ENMF_ERR_NONFINITE;
  return ENMF_OK;
}
}  // namespace

extern "C" {

enmf_status_t enmf_iterate(enmf_handle_t h, float* U, int64_t ldu, float* V, int64_t ldv,
                           int n_iters, double* f_trace_host, enmf_iter_info_t* info) {
  if (!h || n_iters < 0) return ENMF_ERR_INVALID_ARG;
  if (!h->bound) return ENMF_ERR_STATE;
  ENMF_TRY(validate_ld(U, ldu, h->r));
  ENMF_TRY(validate_ld(V, ldv, h->r));
  return iterate_core(h, U, ldu, V, ldv, n_iters, f_trace_host, info, nullptr, nullptr,
                      nullptr);
}

enmf_status_t enmf_iterate_host(enmf_handle_t h, float* U_host, float* V_host, int n_iters,
                                double* f_trace_host, enmf_iter_info_t* info) {
  if (!h || !U_host || !V_host || n_iters < 0) return ENMF_ERR_INVALID_ARG;
  if (!h->bound) return ENMF_ERR_STATE;
  if (!h->Ud) ENMF_TRY(dalloc(&h->Ud, (size_t)(h->m_loc * h->r)));
  if (!h->Vd) ENMF_TRY(dalloc(&h->Vd, (size_t)(h->n * h->r)));
  if (!h->st2) {
    CUDA_TRY(cudaStreamCreateWithFlags(&h->st2, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&h->ev_a, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&h->ev_b, cudaEventDisableTiming));
  }
  const int64_t r = h->r;
  // V first on the compute stream (the X V pass needs it); U on the copy stream, overlapping
  // that pass; U comes back behind the V block, V and f at the end
  CUDA_TRY(cudaMemcpyAsync(h->Vd, V_host, sizeof(float) * h->n * r, cudaMemcpyHostToDevice,
                           h->st));
  CUDA_TRY(cudaEventRecord(h->ev_b, h->st));
  CUDA_TRY(cudaStreamWaitEvent(h->st2, h->ev_b, 0));
  CUDA_TRY(cudaMemcpyAsync(h->Ud, U_host, sizeof(float) * h->m_loc * r, cudaMemcpyHostToDevice,
                           h->st2));
  CUDA_TRY(cudaEventRecord(h->ev_b, h->st2));
  return iterate_core(h, h->Ud, r, h->Vd, r, n_iters, f_trace_host, info, h->ev_b,
                      n_iters > 0 ? U_host : nullptr, V_host);
}

enmf_status_t enmf_objective(enmf_handle_t h, const float* U, int64_t ldu, const float* V,
                             int64_t ldv, int exact, double* f_host) {
  if (!h || !f_host) return ENMF_ERR_INVALID_ARG;
  if (!h->bound) return ENMF_ERR_STATE;
  ENMF_TRY(validate_ld(U, ldu, h->r));
  ENMF_TRY(validate_ld(V, ldv, h->r));
  LaunchScope ls(h);
  const bool sh = h->sharded;
  double* f = h->dscal + S_SCRATCH;
  if (h->nmc) {
    // eNMC: the masked objective over the observed entries
    nmc_objective(h->csr_ptr, h->csr_col, h->csr_val, h->m_loc, (int)h->r, U, ldu, V, ldv,
                  h->parts, f, h->st);
  } else if (exact && h->sparse) {
    // sparse X: ||X||^2 - 2 sum over stored entries x_ij (u_i . v_j) + ||U V^T||^2, the cross
    // term entry by entry (not through Q) and ||U V^T||^2 = <U^T U, V^T V> exactly
    double* parts = nullptr;
    CUDA_TRY(cudaMallocAsync(&parts, sizeof(double) * sddmm_parts(h->m_loc), h->st));
    sddmm_dot(h->csr_ptr, h->csr_col, h->csr_val, h->m_loc, U, ldu, V, ldv, (int)h->r, parts,
              h->dscal + S_CROSS, h->st);
    CUDA_TRY(cudaFreeAsync(parts, h->st));
    ENMF_TRY(ar(h, h->dscal + S_CROSS, 1, CommOp::Sum));
    ENMF_TRY(gram_f32(h, U, ldu, h->m_loc, h->GU, sh));
    double* gv = h->work + h->work_elems - (size_t)(h->r * h->r);
    GemmOut o;
    o.C = gv;
    o.ldc = h->r;
    gemm<float, float>(true, V, ldv, V, ldv, h->r, h->r, h->n, o, h->work,
                       h->work_elems - (size_t)(h->r * h->r), h->st);
    objective_finish(h->dscal + S_XNORM2, h->dscal + S_CROSS, h->GU, gv, (int)h->r, f, h->st);
  } else if (exact) {
    int np = 0;
    frob_direct(h->X, h->ldx, h->m_loc, h->n, U, ldu, V, ldv, (int)h->r, h->parts, &np, h->st);
    reduce_parts(h->parts, np, 1, f, h->st);
    ENMF_TRY(ar(h, f, 1, CommOp::Sum));
  } else {
    ENMF_TRY(contract_xtu(h, U, ldu, h->Q));
    ENMF_TRY(gram_u(h, U, ldu, sh));
    double* gv = h->work + h->work_elems - (size_t)(h->r * h->r);
    GemmOut o;
    o.C = gv;
    o.ldc = h->r;
    gemm<float, float>(true, V, ldv, V, ldv, h->r, h->r, h->n, o, h->work,
                       h->work_elems - (size_t)(h->r * h->r), h->st);
    dot_f64_f32(h->Q, V, ldv, h->n, h->r, h->parts, h->dscal + S_CROSS, h->st);
    objective_finish(xnorm2_trace(h), h->dscal + S_CROSS, h->GU, gv, (int)h->r, f, h->st);
  }
  CUDA_TRY(cudaMemcpyAsync(f_host, f, sizeof(double), cudaMemcpyDeviceToHost, h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  return check_launch();
}

enmf_status_t enmf_kkt_residual(enmf_handle_t h, const float* U, int64_t ldu, const float* V,
                                int64_t ldv, enmf_kkt_t* out) {
  if (!h || !out) return ENMF_ERR_INVALID_ARG;
  if (!h->bound || h->nmc) return ENMF_ERR_STATE;   // eNMC: KKT of the masked problem not built
  ENMF_TRY(validate_ld(U, ldu, h->r));
  ENMF_TRY(validate_ld(V, ldv, h->r));
  LaunchScope ls(h);
  const bool sh = h->sharded;
  const int r = (int)h->r;
  // grad_U f = U G_V - X V ; grad_V f = V G_U - X^T U
  ENMF_TRY(contract_xv(h, V, ldv, h->P));
  ENMF_TRY(contract_xtu(h, U, ldu, h->Q));
  ENMF_TRY(gram_u(h, U, ldu, sh));
  double* gv = h->GV;   // recomputed at the next enmf_iterate entry
  ENMF_TRY(gram_f32(h, V, ldv, h->n, gv, false));
  const int np = kkt_parts();
  double* pu = h->parts;
  double* pv = h->work;
  kkt_rows(U, ldu, h->m_loc, r, h->P, gv, pu, h->st);
  kkt_rows(V, ldv, h->n, r, h->Q, h->GU, pv, h->st);
  std::vector<double> hu((size_t)np * 8), hv((size_t)np * 8);
  CUDA_TRY(cudaMemcpyAsync(hu.data(), pu, sizeof(double) * hu.size(), cudaMemcpyDeviceToHost,
                           h->st));
  CUDA_TRY(cudaMemcpyAsync(hv.data(), pv, sizeof(double) * hv.size(), cudaMemcpyDeviceToHost,
                           h->st));
  double xn2 = 0.0;
  CUDA_TRY(cudaMemcpyAsync(&xn2, h->dscal + S_XNORM2, sizeof(double), cudaMemcpyDeviceToHost,
                           h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  ENMF_TRY(check_launch());
  // fixed-order host reduction of the per-warp partials
  auto fold = [&](const std::vector<double>& p, double* s7) {
    s7[0] = 0; s7[1] = 0; s7[2] = -INFINITY; s7[3] = 0; s7[4] = INFINITY; s7[5] = INFINITY;
    s7[6] = 0;
    for (int w = 0; w < np; ++w) {
      const double* q = &p[(size_t)w * 8];
      s7[0] = std::max(s7[0], q[0]);
      s7[1] += q[1];
      s7[2] = std::max(s7[2], q[2]);
      s7[3] += q[3];
      s7[4] = std::min(s7[4], q[4]);
      s7[5] = std::min(s7[5], q[5]);
      s7[6] += q[6];
    }
  };
  double su[7], sv[7];
  fold(hu, su);
  fold(hv, sv);
  if (sh) {
    // combine the U-block statistics over ranks (V is replicated: counted once)
    double sums[3] = {su[1], su[3], su[6]}, maxs[2] = {su[0], su[2]}, mins[2] = {su[4], su[5]};
    double* buf = h->work;
    CUDA_TRY(cudaMemcpyAsync(buf, sums, sizeof(sums), cudaMemcpyHostToDevice, h->st));
    CUDA_TRY(cudaMemcpyAsync(buf + 3, maxs, sizeof(maxs), cudaMemcpyHostToDevice, h->st));
    CUDA_TRY(cudaMemcpyAsync(buf + 5, mins, sizeof(mins), cudaMemcpyHostToDevice, h->st));
    ENMF_TRY(ar(h, buf, 3, CommOp::Sum));
    ENMF_TRY(ar(h, buf + 3, 2, CommOp::Max));
    ENMF_TRY(ar(h, buf + 5, 2, CommOp::Min));
    double all[7];
    CUDA_TRY(cudaMemcpyAsync(all, buf, sizeof(all), cudaMemcpyDeviceToHost, h->st));
    CUDA_TRY(cudaStreamSynchronize(h->st));
    su[1] = all[0]; su[3] = all[1]; su[6] = all[2]; su[0] = all[3]; su[2] = all[4];
    su[4] = all[5]; su[5] = all[6];
  }
  out->min_u = su[5];
  out->min_v = sv[5];
  out->comp_max = std::max(su[0], sv[0]);
  out->comp_sum = su[1] + sv[1];
  out->delta_w = std::max(su[2], sv[2]);
  out->sigma_w = su[3] + sv[3];
  const double gmin = std::min(su[4], sv[4]);
  out->dual_viol = gmin < 0 ? -gmin : 0.0;
  out->xnorm2 = xn2;
  out->rms_cross = sqrt((su[6] + sv[6]) / (double)((h->prob.m_global + h->n) * h->r));
  return ENMF_OK;
}

}  // extern "C"
