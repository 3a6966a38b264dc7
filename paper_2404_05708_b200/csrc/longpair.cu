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

static size_t pow2_at_least(size_t x) {
  size_t c = 1;
  while (c < x) c <<= 1;
  return c;
}

size_t long_shard_ring_slots(int m) {
  // a whole stream (+64: the producer's flow-control test looks past its end)
  return pow2_at_least((size_t)stream_len<kLCols>(m) + 64);
}

// the one-pair header the long kernel reads (offsets, lengths, list, count)
__global__ void shard_header_kernel(int64_t* offsets, int32_t* lengths, int* list, int* count, int n, int m) {
  offsets[0] = 0;
  offsets[1] = 0;
  lengths[0] = n;
  lengths[1] = m;
  list[0] = 0;
  *count = 1;
}

cudaError_t launch_long_shard(LongArgs a, int n0, int m0, int sms, cudaStream_t st, int64_t* launches) {
  // header + multi-pass wrap buffer (a whole stream of the longer curve) + cons pair
  const size_t wrap_b = long_shard_ring_slots(n0 > m0 ? n0 : m0) * sizeof(uint2);
  const size_t hdr_b = 256;
  char* buf = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&buf), hdr_b + wrap_b, st);
  if (e != cudaSuccess) return e;
  int64_t* offsets = reinterpret_cast<int64_t*>(buf);
  int32_t* lengths = reinterpret_cast<int32_t*>(buf + 16);
  int* list = reinterpret_cast<int*>(buf + 32);
  int* count = reinterpret_cast<int*>(buf + 48);
  a.ext_cons = reinterpret_cast<unsigned*>(buf + 64);
  shard_header_kernel<<<1, 1, 0, st>>>(offsets, lengths, list, count, n0, m0);
  ++*launches;
  a.offsets = offsets;
  a.lengths = lengths;
  a.list = list;
  a.list_count = count;
  a.num_pairs = 1;
  a.wrap = buf + hdr_b;
  a.wrap_bytes = wrap_b;
  a.shard = 1;
  e = cudaGetLastError();
  if (e == cudaSuccess) e = launch_long_pairs(a, sms, st, launches);
  cudaFreeAsync(buf, st);
  return e;
}

}  // namespace ffd
