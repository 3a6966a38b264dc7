// seg_sq_d3_sqrt.cu — one instantiation of the segmented batch kernel (seg.cuh)
#include "seg.cuh"

namespace ffd {
cudaError_t launch_seg_sq_d3_sqrt(const SegProblem& pb, int sms, cudaStream_t st, bool big) {
  return seg_launch_k<K_SQ, 3, false, F_SQRT>(pb, sms, st, big);
}
}  // namespace ffd
