// seg.cu — instantiations and launcher of the segmented two-column batch kernel
// (seg.cuh), and the item table its prep builds.
#include <cstdlib>

#include "seg.cuh"

namespace ffd {

// one translation unit per built cell (seg_<cell>.cu, compiled in parallel)
cudaError_t launch_seg_xsq_d2(const SegProblem& pb, int sms, cudaStream_t st, bool big);
cudaError_t launch_seg_sq_d2_sqrt(const SegProblem& pb, int sms, cudaStream_t st, bool big);
cudaError_t launch_seg_sq_d2(const SegProblem& pb, int sms, cudaStream_t st, bool big);
cudaError_t launch_seg_l1_d2(const SegProblem& pb, int sms, cudaStream_t st, bool big);
cudaError_t launch_seg_linf_d2(const SegProblem& pb, int sms, cudaStream_t st, bool big);
cudaError_t launch_seg_il1_d2(const SegProblem& pb, int sms, cudaStream_t st, bool big);
cudaError_t launch_seg_ilinf_d2(const SegProblem& pb, int sms, cudaStream_t st, bool big);
cudaError_t launch_seg_sq_d3_sqrt(const SegProblem& pb, int sms, cudaStream_t st, bool big);
cudaError_t launch_seg_sq_d3(const SegProblem& pb, int sms, cudaStream_t st, bool big);

// rows above 256 on two 16-lane segments of up to 32 rows per lane (the big
// kernel, 234 registers: 8 warps/SM).  Measured on config 2: 13 % fewer
// instructions but 51 % issue, 2.69 against 2.65 ms — off unless FFD_SEG_BIG=1
bool seg_big() {
  static const bool on = getenv("FFD_SEG_BIG") && atoi(getenv("FFD_SEG_BIG")) == 1;
  return on;
}

// built: every 2-D Fréchet cell (exact-integer sq-L2 / L1 / L∞, fp32 L2 / sq-L2 /
// L1 / L∞) and the 3-D fp32 L2 / sq-L2 cells; other dimensions stay on the batch kernel
bool seg_supported(int kind, int dim, int int_in, int fin) {
  static const int off = getenv("FFD_SEG") && atoi(getenv("FFD_SEG")) == 0;
  if (off || fin == F_DTW) return false;
  if (dim == 2) {
    if (int_in) return kind == K_XSQ || kind == K_L1 || kind == K_LINF;
    return kind == K_SQ || kind == K_L1 || kind == K_LINF;
  }
  return dim == 3 && !int_in && kind == K_SQ;
}

cudaError_t launch_seg(const SegProblem& pb, int kind, int dim, int int_in, int fin, int sms, cudaStream_t st,
                       int64_t* launches) {
  const bool big = seg_big();
  *launches += big ? 2 : 1;
  if (dim == 2 && int_in && kind == K_XSQ) return launch_seg_xsq_d2(pb, sms, st, big);
  if (dim == 2 && !int_in && kind == K_SQ && fin == F_SQRT) return launch_seg_sq_d2_sqrt(pb, sms, st, big);
  if (dim == 2 && !int_in && kind == K_SQ && fin == F_NONE) return launch_seg_sq_d2(pb, sms, st, big);
  if (dim == 2 && !int_in && kind == K_L1) return launch_seg_l1_d2(pb, sms, st, big);
  if (dim == 2 && !int_in && kind == K_LINF) return launch_seg_linf_d2(pb, sms, st, big);
  if (dim == 2 && int_in && kind == K_L1) return launch_seg_il1_d2(pb, sms, st, big);
  if (dim == 2 && int_in && kind == K_LINF) return launch_seg_ilinf_d2(pb, sms, st, big);
  if (dim == 3 && !int_in && kind == K_SQ && fin == F_SQRT) return launch_seg_sq_d3_sqrt(pb, sms, st, big);
  if (dim == 3 && !int_in && kind == K_SQ && fin == F_NONE) return launch_seg_sq_d3(pb, sms, st, big);
  return cudaErrorInvalidValue;
}

}  // namespace ffd
