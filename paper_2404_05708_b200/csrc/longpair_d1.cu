// longpair_d1.cu — long-pair kernel instantiations for D = 1 (one TU per
// dimension so the build runs them in parallel).
#include "longpair_kernel.cuh"

namespace ffd {
cudaError_t launch_long_dim1(const LongArgs& a, int sms, cudaStream_t st, const LongWs& w, int G,
                             int64_t* launches) {
  return launch_long_dim<1>(a, sms, st, w, G, launches);
}
}  // namespace ffd
