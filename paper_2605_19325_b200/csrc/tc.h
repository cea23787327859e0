// tc.h -- tensor-core (tcgen05) contraction path for large X.
//
// X is repacked once (enmf_set_data) into a handle-owned split copy X = Xhi + Xlo with
// fp16 hi/lo planes (4 bytes per element, the same HBM bytes per pass as fp32 X), laid out
// in pre-swizzled tiles that one bulk copy moves into shared memory.  The two X passes of
// a sweep then run as tcgen05 MMAs
//   P = Xhi Vhi + Xhi Vlo + Xlo Vhi        (and the same for X^T U)
// with fp32 accumulation in TMEM over short K chunks promoted to fp64 in registers.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace enmf {

struct TcState;

// True when the shape is handled by the tensor-core kernels.
bool tc_supported(int64_t rows, int64_t n, int64_t r);
// Build the split copy of X (rows x n, ld).  Returns 0, 1 (CUDA error) or 2 (OOM).
int tc_create(TcState** out, const float* X, int64_t ldx, int64_t rows, int64_t n, int64_t r,
              cudaStream_t st);
void tc_destroy(TcState* s);
// P (rows x r fp64) = X V ; Q (n x r fp64) = X^T U  (this rank's rows only).
int tc_xv(TcState* s, const float* V, int64_t ldv, double* P, cudaStream_t st);
int tc_xtu(TcState* s, const float* U, int64_t ldu, double* Q, cudaStream_t st);

}  // namespace enmf
