// longpair.cu — host dispatch of the long-pair wavefront kernel
// (longpair_kernel.cuh; instantiations in longpair_d<D>.cu).
#include <cstdlib>

#include "ffd.h"
#include "longpair_kernel.cuh"

namespace ffd {

cudaError_t launch_long_pairs(const LongArgs& a, int sms, cudaStream_t st, int64_t* launches) {
  int G = sms;
  if (const char* env = getenv("FFD_LONG_CTAS")) {  // testing: fewer CTAs -> larger R
    const int g = atoi(env);
    if (g > 0 && g < G) G = g;
  }
  if (G > kMaxLongCtas) G = kMaxLongCtas;
  // workspace (stream-ordered, pooled): global link rings + consumer counters +
  // per-pair flags + the abort flag (zeroed by the kernel: tags start at 1, a zero slot is never
  // "ready")
  const size_t ring_b = (size_t)G * kLGlobRing * sizeof(uint2);
  const size_t ctr_b = (size_t)(G + 1) * sizeof(unsigned);
  const size_t bad_b = (size_t)(a.num_pairs > 0 ? a.num_pairs : 1) * sizeof(int);
  const size_t total = ring_b + ctr_b + bad_b + 256;
  char* buf = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&buf), total, st);
  if (e != cudaSuccess) return e;
  LongWs w{reinterpret_cast<uint2*>(buf), reinterpret_cast<unsigned*>(buf + ring_b),
           reinterpret_cast<int*>(buf + ring_b + ctr_b), reinterpret_cast<int*>(buf + total - 256)};
  // (the kernel zeroes the rings, counters and flags itself when it has work)
  {
    switch (a.dim) {
      case 1: e = launch_long_dim1(a, sms, st, w, G, launches); break;
      case 2: e = launch_long_dim2(a, sms, st, w, G, launches); break;
      case 3: e = launch_long_dim3(a, sms, st, w, G, launches); break;
      case 4: e = launch_long_dim4(a, sms, st, w, G, launches); break;
      default: e = cudaErrorInvalidValue;
    }
  }
  cudaFreeAsync(buf, st);
  return e;
}

}  // namespace ffd
