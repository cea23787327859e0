// handle.h -- the enmf handle and the orchestration helpers shared by enmf_capi.cu and
// enmf_init.cu (private to libenmf.so).
#pragma once
#include <cuda_runtime.h>
#include <stdio.h>

#include <vector>

#include "comm.h"
#include "enmf.h"
#include "internal.h"
#include "tc.h"

namespace enmf {

// device scalar slots (doubles)
enum {
  S_XNORM2 = 0, S_XMIN, S_XBAD, S_MINU, S_MINV, S_CROSS, S_LAMU, S_LAMV, S_NEG, S_SCRATCH,
  S_WMAX, S_STEP,
  S_XQNORM2,   // ||X~||^2 of the tensor-core path's quantised X (trace-form objective)
  S_FCUR,      // the current sweep's objective before it is appended to the trace
  S_COUNT = 16
};
// device int slots
enum { I_STAGE = 0, I_KSTAR_U, I_KSTAR_V, I_CNT_ASC, I_CNT_HALS, I_BAD, I_HALS_FB, I_HALS_ILL,
       I_FCNT,   // next slot of the objective trace (sweeps append; graph replays share args)
       I_PBCD_DONE,   // staged tensor-core PBCD: the stopping rule has fired in this block
       I_PBCD_CTL,    // 4 slots: replay?, replay it0, replay src, committed state buffer
       I_COUNT = I_PBCD_CTL + 4 };

}  // namespace enmf

struct enmf_handle_s {
  enmf_problem_t prob{};
  enmf_options_t opt{};
  cudaStream_t st = nullptr;
  int64_t m_loc = 0, n = 0, r = 0;
  const float* X = nullptr;
  int64_t ldx = 0;
  bool bound = false;
  bool stage_known_hals = false;   // host mirror: once HALS, always HALS
  enmf::Comm* comm = nullptr;
  int64_t launches = 0;
  int precision = ENMF_PREC_FP64;
  double* dscal = nullptr;
  int* dint = nullptr;
  double* P = nullptr;       // m_loc x r
  double* Q = nullptr;       // n x r
  double* GU = nullptr;      // r x r
  double* GV = nullptr;      // r x r
  double* work = nullptr;    // split-K partials and small dense scratch
  size_t work_elems = 0;
  double* parts = nullptr;   // reduction partials
  size_t parts_elems = 0;
  double* minparts = nullptr;
  double* pgsum = nullptr;   // max_iter + 1
  float* snaps = nullptr;    // max_iter x max(m_loc, n) x r
  double* ftrace = nullptr;
  int ftrace_cap = 0;
  enmf::TcState* tc = nullptr;
  double* tcpb_ws = nullptr;  // tensor-core PBCD: G digits (64 KB) + 128 column scales
  double* pbcd_state = nullptr;  // staged tensor-core PBCD: 2 x fp64 u (tile-major, ping-pong)
  size_t pbcd_state_len = 0;
  double* stepws = nullptr;   // lambda_max workspace of the ablation step rules (R29)
  bool step_warm[2] = {false, false};   // stepws holds a warm start per block (U, V)
  bool tc_pbcd = false;       // ascent PBCD on the tensor cores (precision TC, r <= 128)
  bool tc_hals = false;       // HALS sweep on the tensor cores (tc_hals_rows)
  // tensor-core path: column maxima of |U| / |V| written by the block-update kernels, so the
  // next X pass packs the factor without a separate scan; valid only within one iterate call
  unsigned long long* fmax_uv = nullptr;   // [2][128]: U, V
  bool umax_valid = false, vmax_valid = false;
  // multi-rank V block: this rank updates V rows [v_begin, v_begin + v_count) and the full V
  // is reassembled by a zero-padded fp64 allreduce (exact: adding zeros), SURVEY §8(e)
  int64_t v_begin = 0, v_count = 0;
  // the collective path runs: world_size > 1, or a communicator was requested at one rank
  // (enmf_problem_t.nccl_unique_id set) -- the single-rank NCCL path tests and bench run
  bool sharded = false;
  int64_t v_pad = 0;
  cudaStream_t st_comm = nullptr;          // slice reductions of the sliced pass 2 (NCCL)
  std::vector<cudaEvent_t> ev_comm;
  // sparse X (enmf_set_data_csr): this rank's rows as CSR (caller-owned) and a handle-owned
  // CSC copy for X^T U
  bool sparse = false;
  bool nmc = false;           // eNMC (enmf_set_data_masked): stored entries are the OBSERVED ones
  const int64_t* csr_ptr = nullptr;
  const int32_t* csr_col = nullptr;
  const float* csr_val = nullptr;
  int64_t nnz = 0;
  int64_t* csc_ptr = nullptr;
  int32_t* csc_row = nullptr;
  float* csc_val = nullptr;               // rows per V slice (ceil(n / world)); v_begin = rank v_pad
  float* Vpad = nullptr;           // world x v_pad x r fp32: all-gather of the V slices (NCCL)
  double* Vg = nullptr;            // n x r fp64 staging of the gather
  // host-mediated collectives (enmf_set_host_allreduce) when there is no NCCL communicator
  enmf_host_allreduce_fn host_ar = nullptr;
  void* host_ar_ctx = nullptr;
  double* host_ar_buf = nullptr;   // pinned staging
  size_t host_ar_cap = 0;
  // init workspace arena (enmf_init.cu DevBuf): kept across calls, grown on demand
  uint8_t* arena = nullptr;
  size_t arena_bytes = 0, arena_need = 0;
  std::vector<void*> arena_extra;   // one-off overflow allocations, freed with the handle
  // enmf_iterate_host: device copies of the factor state and a copy stream for the transfers
  float* Ud = nullptr;
  float* Vd = nullptr;
  cudaStream_t st2 = nullptr;
  cudaStream_t cap_st = nullptr;   // non-blocking stream a sweep is captured on (CUDA graph)
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;
  double* small_ws = nullptr;      // workspace of the persistent small-problem HALS kernel
  cudaGraphExec_t sw_exec = nullptr;   // cached graph of one ascent-capable sweep (small path)
  const void* sw_key[2] = {nullptr, nullptr};
  int64_t sw_ld[2] = {0, 0};
  int64_t sw_launches = 0;
  float* x_owned = nullptr;  // device copy of X owned by enmf_solve_host
  double* W64 = nullptr;     // (m_loc + n) x r fp64 [U*; V*] kept from enmf_svd for enmf_rotate
  // profiling of the X passes (enmf_set_profiling): CUDA events around every contraction
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<int> ev_kind;  // 0 = X V, 1 = X^T U, per event pair
  size_t ev_used = 0;
  double prof_ms[2] = {0.0, 0.0};
  int64_t prof_cnt[2] = {0, 0};
};

namespace enmf {

struct LaunchScope {
  explicit LaunchScope(enmf_handle_t h) { g_launch_counter = &h->launches; }
  ~LaunchScope() { g_launch_counter = nullptr; }
};

#define CUDA_TRY(x)                                                                  \
  do {                                                                               \
    cudaError_t _e = (x);                                                            \
    if (_e != cudaSuccess) {                                                         \
      fprintf(stderr, "enmf: CUDA error %s at %s:%d\n", cudaGetErrorString(_e),     \
              __FILE__, __LINE__);                                                   \
      return _e == cudaErrorMemoryAllocation ? ENMF_ERR_OOM : ENMF_ERR_CUDA;         \
    }                                                                                \
  } while (0)

#define ENMF_TRY(x)                        \
  do {                                     \
    enmf_status_t _s = (x);                \
    if (_s != ENMF_OK) return _s;          \
  } while (0)

enmf_status_t check_launch();
enmf_status_t dalloc_bytes(void** p, size_t bytes);
template <typename T>
enmf_status_t dalloc(T** p, size_t count) {
  return dalloc_bytes((void**)p, sizeof(T) * (count ? count : 1));
}
enmf_status_t ar(enmf_handle_t h, double* buf, size_t count, CommOp op);
enmf_status_t contract_xv(enmf_handle_t h, const float* V, int64_t ldv, double* P,
                          const unsigned long long* vmax = nullptr,
                          unsigned* band_ready = nullptr);
enmf_status_t contract_xtu(enmf_handle_t h, const float* U, int64_t ldu, double* Q,
                           const unsigned long long* umax = nullptr, bool slice = false);
enmf_status_t gram_f32(enmf_handle_t h, const float* A, int64_t lda, int64_t rows, double* G,
                       bool sharded, const double* qscale = nullptr);
// Tensor-core path: the digit scales of the factor the last X pass packed (for the Gram of the
// quantised factor), else null.  The trace-form objective's ||X||^2 term: ||X~||^2 of the
// quantised X on the tensor-core path (tc_gemm.cu), else ||X||^2.
inline const double* qgram_scales(enmf_handle_t h) {
  return h->tc && !h->sparse ? tc_factor_scales(h->tc) : nullptr;
}
inline const double* xnorm2_trace(enmf_handle_t h) {
  return h->dscal + (h->tc && !h->sparse ? S_XQNORM2 : S_XNORM2);
}
enmf_status_t min_factor(enmf_handle_t h, const float* A, int64_t lda, int64_t rows, int slot,
                         bool sharded);
enmf_status_t validate_ld(const void* p, int64_t ld, int64_t cols);

}  // namespace enmf
