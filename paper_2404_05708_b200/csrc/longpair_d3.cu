// longpair_d3.cu — long-pair kernel instantiations for D = 3 (one TU per
// dimension so the build runs them in parallel).
#include "longpair_kernel.cuh"

namespace ffd {
cudaError_t launch_long_dim3(const LongArgs& a, int sms, cudaStream_t st, const LongWs& w, int G,
                             int64_t* launches) {
  return launch_long_dim<3>(a, sms, st, w, G, launches);
}
}  // namespace ffd
