// seg_ilinf_d2.cu — one instantiation of the segmented batch kernel (seg.cuh)
#include "seg.cuh"

namespace ffd {
cudaError_t launch_seg_ilinf_d2(const SegProblem& pb, int sms, cudaStream_t st, bool big) {
  return seg_launch_k<K_LINF, 2, true, F_NONE>(pb, sms, st, big);
}
}  // namespace ffd
