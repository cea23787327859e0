// tc.h -- tensor-core (tcgen05) contraction path for large X.
//
// X is repacked once (enmf_set_data) into a handle-owned copy of three balanced base-2^7 int8
// digit planes (3 bytes per element), laid out in UMMA canonical tiles that bulk copies move
// straight into shared memory.  The two X passes of a sweep run as tcgen05.mma kind::i8 with
// exact int32 accumulation in TMEM (6 digit products into 3 weight classes), combined exactly
// in fp64 by the epilogue.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace enmf {

struct TcState;

// True when the shape is handled by the tensor-core kernels.
bool tc_supported(int64_t rows, int64_t n, int64_t r);
// Build the digit-plane copy of X (rows x n, ld).  Returns 0, 1 (CUDA error) or 2 (OOM).
int tc_create(TcState** out, const float* X, int64_t ldx, int64_t rows, int64_t n, int64_t r,
              cudaStream_t st);
void tc_destroy(TcState* s);
// P (rows x r fp64) = X V ; Q (n x r fp64) = X^T U  (this rank's rows only).
int tc_xv(TcState* s, const float* V, int64_t ldv, double* P, cudaStream_t st);
int tc_xtu(TcState* s, const float* U, int64_t ldu, double* Q, cudaStream_t st);

}  // namespace enmf
