// longpair.cu — placeholder: marks long pairs unsupported (NaN / INT64_MIN).
#include <climits>

#include "ffd.h"
#include "longpair.cuh"

namespace ffd {
__global__ void long_mark_kernel(LongArgs a) {
  const int n = *a.list_count;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int k = a.list[i];
    if (a.dtype == FFD_I32) reinterpret_cast<long long*>(a.out)[k] = LLONG_MIN;
    else reinterpret_cast<float*>(a.out)[k] = __int_as_float(0x7fc00000);
  }
}
cudaError_t launch_long_pairs(const LongArgs& a, int sms, cudaStream_t st, int64_t* launches) {
  long_mark_kernel<<<1, 128, 0, st>>>(a);
  ++*launches;
  return cudaGetLastError();
}
}  // namespace ffd
