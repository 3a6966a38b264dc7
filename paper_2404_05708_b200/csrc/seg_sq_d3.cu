// seg_sq_d3.cu — one instantiation of the segmented batch kernel (seg.cuh)
#include "seg.cuh"

namespace ffd {
cudaError_t launch_seg_sq_d3(const SegProblem& pb, int sms, cudaStream_t st, bool big) {
  return seg_launch_k<K_SQ, 3, false, F_NONE>(pb, sms, st, big);
}
}  // namespace ffd
