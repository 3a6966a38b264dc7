// seg.cu — instantiations and launcher of the segmented two-column batch kernel
// (seg.cuh), and the item table its prep builds.
#include <cstdlib>

#include "seg.cuh"

namespace ffd {

namespace {
template <int KIND, int D, bool INT_IN, int FIN>
cudaError_t launch_k(const SegProblem& pb, int sms, cudaStream_t st) {
  auto k = seg_kernel<KIND, D, INT_IN, FIN>;
  const size_t smem = sizeof(SegSmem<KIND, D, INT_IN>) * kWarpsPerCta;
  int dev = 0;
  cudaGetDevice(&dev);
  static int occ_cache[64] = {0};
  int occ = dev < 64 ? occ_cache[dev] : 0;
  if (occ == 0) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kWarp * kWarpsPerCta, smem);
    if (occ < 1) occ = 1;
    if (dev < 64) occ_cache[dev] = occ;
  }
  k<<<sms * occ, kWarp * kWarpsPerCta, smem, st>>>(pb);
  return cudaGetLastError();
}
}  // namespace

// built: the exact-integer 2-D squared-L2 cell (config 2) and the fp32 2-D L2 /
// squared-L2 cells; every other kind stays on the batch kernel
int seg_items_per_segment() {
  static const int L = [] {
    const char* e = getenv("FFD_SEG_L");
    const int v = e ? atoi(e) : kSegL;
    return v < 2 ? 2 : (v > kSegMaxL ? kSegMaxL : v);
  }();
  return L;
}

bool seg_supported(int kind, int dim, int int_in, int fin) {
  static const int off = getenv("FFD_SEG") && atoi(getenv("FFD_SEG")) == 0;
  if (off || dim != 2) return false;
  if (int_in) return kind == K_XSQ && fin == F_NONE;
  return kind == K_SQ && (fin == F_SQRT || fin == F_NONE);
}

cudaError_t launch_seg(const SegProblem& pb, int kind, int dim, int int_in, int fin, int sms, cudaStream_t st) {
  if (dim == 2 && int_in && kind == K_XSQ) return launch_k<K_XSQ, 2, true, F_NONE>(pb, sms, st);
  if (dim == 2 && !int_in && kind == K_SQ && fin == F_SQRT) return launch_k<K_SQ, 2, false, F_SQRT>(pb, sms, st);
  if (dim == 2 && !int_in && kind == K_SQ && fin == F_NONE) return launch_k<K_SQ, 2, false, F_NONE>(pb, sms, st);
  return cudaErrorInvalidValue;
}

}  // namespace ffd
