// longpair.cuh — pairs too long for the batch kernel's band scratch.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ffd {
struct LongArgs {
  const void* p;
  const void* q;
  const int64_t* offsets;
  const int32_t* lengths;
  int64_t num_pairs;
  int dim, norm, dtype;
  int measure;            // 0: discrete Fréchet (Eq. (1)); 1: DTW (PAPER Appendix B)
  const int* list;        // device list of long pair indices
  const int* list_count;  // device count
  void* out;
  void* wrap;         // device scratch for the multi-pass wrap link (any contents)
  size_t wrap_bytes;  // its size
};
cudaError_t launch_long_pairs(const LongArgs& a, int sms, cudaStream_t st, int64_t* launches);
}  // namespace ffd
