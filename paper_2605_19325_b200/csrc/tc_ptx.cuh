// tc_ptx.cuh -- inline-PTX wrappers for the tcgen05 / TMA / mbarrier kernels (private header of
// libenmf.so): mbarrier init/arrive/wait (with a trap-on-timeout watchdog), cp.async.bulk,
// tcgen05 fences/commit/mma (kind::i8), UMMA smem descriptors and tcgen05.ld.
#pragma once
#include <stdint.h>
#include <stdio.h>

namespace enmf {
namespace tcp {

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
// mbar_wait with a suspend-time hint: a waiting thread may be suspended in try_wait until the
// phase completes (or ~the hint, in ns) instead of re-polling -- for waits every warp of a CTA
// takes at once (the MMA rounds of tc_pbcd_kernel), where polling warps only steal issue slots
// from the thread that issues the MMAs.
__device__ __forceinline__ void mbar_wait_hint(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  long long t0 = 0;
  int spins = 0;
  while (true) {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity), "r"(20000)
        : "memory");
    if (done) return;
    if (++spins == 64) t0 = clock64();
    if (spins > 64 && (spins & 63) == 0 && clock64() - t0 > 40000000000LL) {
      printf("enmf tc: mbarrier wait timeout (block %d thread %d)\n", blockIdx.x, threadIdx.x);
      __trap();
    }
  }
}
// For barriers a peer CTA arrives on.  CTA-scope polling, as CUTLASS's cluster barriers do:
// try_wait.acquire.cluster invalidates L1 on every poll and a per-stage fence.acq_rel.cluster
// serialises the issuing thread (both measured: 2x slower pair kernel).  The data that matters
// (bulk-copied operands in the peer's shared memory) is read by the tensor core after issue.
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  mbar_wait(bar, parity);
}
// Long waits of otherwise idle warps (epilogue waiting for a whole unit): back off between polls
// so the spinning warps do not steal issue slots from the producer and MMA warps.
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  long long t0 = clock64();
  while (true) {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) return;
    __nanosleep(200);
    if (clock64() - t0 > 40000000000LL) {
      printf("enmf tc: mbarrier wait timeout (block %d thread %d)\n", blockIdx.x, threadIdx.x);
      __trap();
    }
  }
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of the variable at local shared address `a` in CTA `rank`
__device__ __forceinline__ uint32_t mapa_shared(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" :::
                   "memory");
}
__device__ __forceinline__ void tc_commit_pair(uint32_t bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(bar),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tc_mma_i8_pair(uint32_t dtmem, uint64_t adesc, uint64_t bdesc,
                                               uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
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
__device__ __forceinline__ void tc_mma_i8(uint32_t dtmem, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(dtmem),
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

#define TMEM_LD16(taddr, v)                                                                  \
  asm volatile(                                                                              \
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13," \
      "%14,%15}, [%16];"                                                                     \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), \
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),          \
        "=r"(v[13]), "=r"(v[14]), "=r"(v[15])                                                \
      : "r"(taddr))

#define TMEM_ST16_ZERO(taddr)                                                                 \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1," \
               "%1,%1,%1,%1,%1};" ::"r"(taddr), "r"(0u)                                          \
               : "memory")

#define TMEM_LD8(taddr, v)                                                                  \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"      \
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),     \
                 "=r"(v[6]), "=r"(v[7])                                                      \
               : "r"(taddr))

// Balanced base-2^7 digits of t (|t| < 64.5): t = d0 + d1/2^7 + d2/2^14 + d3/2^21 + e,
// |e| <= 2^-22, every digit in [-64, 64].  Exact arithmetic for fp32-derived t (scaling by a
// power of two and subtracting an integer are exact in fp64).
struct Dig4 { int8_t d[4]; };
__device__ __forceinline__ Dig4 digits4(double t) {
  Dig4 out;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double a = rint(t);
    out.d[k] = (int8_t)a;
    t = (t - a) * 128.0;
  }
  return out;
}

// Register-only form of digits4 (no addressable local arrays).  digits_word(t), |t| < 64.5:
// t rounded to the 2^-21 grid (error <= 2^-22, the digits4 bound) split into balanced base-2^7
// digits d0 + d1/2^7 + d2/2^14 + d3/2^21, digit pl in byte pl -- integer arithmetic only.
__device__ __forceinline__ uint32_t digits_n(int n) {
  const int d3 = ((n + 64) & 127) - 64;
  n = (n - d3) >> 7;
  const int d2 = ((n + 64) & 127) - 64;
  n = (n - d2) >> 7;
  const int d1 = ((n + 64) & 127) - 64;
  const int d0 = (n - d1) >> 7;
  return (uint32_t)(d0 & 255) | ((uint32_t)(d1 & 255) << 8) | ((uint32_t)(d2 & 255) << 16) |
         ((uint32_t)(d3 & 255) << 24);
}
__device__ __forceinline__ uint32_t digits_word(double t) {
  return digits_n(__double2int_rn(t * 0x1p21));
}
// X-pass operands (tc_gemm.cu): three digits of t, |t| < 126, in mixed radix (8, 8, 7):
// n = rint(t 2^15) (round half to even) = d0 2^15 + d1 2^7 + d2 with d2 in [-64, 64]
// (balanced base 2^7, a remainder of exactly half a digit goes to +-64 so that the carried
// quotient is even: d2 is symmetric, mean 0), d1 in [-128, 127] (balanced base 2^8) and
// |d0| <= 126.  Every product the X passes drop (d1 d2', d2 d1', d2 d2') has a symmetric
// last digit as a factor, so the truncation is unbiased -- with a base-2^8 last digit (mean
// -1/2) the dropped products carried a bias of ~2e-11 of <X^T U, V>, 2e-6 of the C5 trace-form
// objective (measured).  Digit k in byte k.
__device__ __forceinline__ uint32_t digits3_n(int n) {
  int d2 = ((n + 64) & 127) - 64;
  if (d2 == -64 && ((n + 64) & 128)) d2 = 64;
  n = (n - d2) >> 7;
  const int d1 = ((n + 128) & 255) - 128;
  const int d0 = (n - d1) >> 8;
  return (uint32_t)(d0 & 255) | ((uint32_t)(d1 & 255) << 8) | ((uint32_t)(d2 & 255) << 16);
}
}  // namespace tcp
}  // namespace enmf
