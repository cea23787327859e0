// tc_gemm.cu -- tensor-core contraction path (see tc.h).  Not yet enabled: tc_supported()
// returns false until the tcgen05 kernels pass parity, so ENMF_PREC_AUTO selects FP64.
#include "internal.h"
#include "tc.h"

namespace enmf {

struct TcState {
  int dummy;
};

bool tc_supported(int64_t, int64_t, int64_t) { return false; }
int tc_create(TcState** out, const float*, int64_t, int64_t, int64_t, int64_t, cudaStream_t) {
  *out = nullptr;
  return 1;
}
void tc_destroy(TcState* s) { delete s; }
int tc_xv(TcState*, const float*, int64_t, double*, cudaStream_t) { return 1; }
int tc_xtu(TcState*, const float*, int64_t, double*, cudaStream_t) { return 1; }

}  // namespace enmf
