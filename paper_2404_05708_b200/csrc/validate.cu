// validate.cu — one thread per pair checks the preconditions of include/ffd.h:
// lengths ≥ 1, offsets+lengths inside the point arrays, finite fp32
// coordinates, and for int32 input Σ_k range_k² ≤ 2^63 − 1 over the union of
// the pair's points (which bounds every exact int64 distance).
#include <climits>
#include <type_traits>

#include "ffd.h"
#include "validate.cuh"

namespace ffd {

// priority of a violation: lower = reported first
__device__ __forceinline__ int prio_of(int status) {
  return status == FFD_ERR_EMPTY ? 1 : status == FFD_ERR_RANGE ? 2 : status == FFD_ERR_NONFINITE ? 3 : 4;
}

template <typename In>
__global__ void validate_kernel(const In* p, int64_t np, const In* q, int64_t nq,
                                const int64_t* offsets, const int32_t* lengths, int64_t B, int dim,
                                int* worst) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < B;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t op = offsets[k], oq = offsets[B + k];
    const int32_t n = lengths[k], m = lengths[B + k];
    int bad = 0;
    if (n < 1 || m < 1) bad = FFD_ERR_EMPTY;
    else if (op < 0 || oq < 0 || op + n > np || oq + m > nq) bad = FFD_ERR_RANGE;
    else {
      long long lo[4], hi[4];
      for (int c = 0; c < dim; c++) { lo[c] = LLONG_MAX; hi[c] = LLONG_MIN; }
      for (int side = 0; side < 2 && !bad; side++) {
        const In* base = side ? q + oq * dim : p + op * dim;
        const int32_t len = side ? m : n;
        for (int32_t i = 0; i < len; i++)
          for (int c = 0; c < dim; c++) {
            In v = base[(int64_t)i * dim + c];
            if constexpr (std::is_floating_point<In>::value) {
              if (!isfinite((float)v)) bad = FFD_ERR_NONFINITE;
            } else {
              long long x = (long long)v;
              lo[c] = x < lo[c] ? x : lo[c];
              hi[c] = x > hi[c] ? x : hi[c];
            }
          }
      }
      if constexpr (!std::is_floating_point<In>::value) {
        if (!bad) {
          unsigned long long s = 0;
          for (int c = 0; c < dim && !bad; c++) {
            unsigned long long r = (unsigned long long)(hi[c] - lo[c]);  // < 2^32
            unsigned long long t = r * r;                                 // < 2^64
            if (t > (unsigned long long)LLONG_MAX || s > (unsigned long long)LLONG_MAX - t)
              bad = FFD_ERR_OVERFLOW;
            else
              s += t;
          }
        }
      }
    }
    if (bad) atomicMin(worst, prio_of(bad));
  }
}

int validate_batch(const void* p, int64_t np, const void* q, int64_t nq, const int64_t* offsets,
                   const int32_t* lengths, int64_t B, int dim, int dtype, cudaStream_t st,
                   int64_t* launches) {
  int* d_worst = nullptr;
  if (cudaMallocAsync(&d_worst, sizeof(int), st) != cudaSuccess) return FFD_ERR_CUDA;
  const int init = 100;
  cudaMemcpyAsync(d_worst, &init, sizeof(int), cudaMemcpyHostToDevice, st);
  const int threads = 128;
  int64_t blocks = (B + threads - 1) / threads;
  if (blocks > 4096) blocks = 4096;
  if (dtype == FFD_I32)
    validate_kernel<int32_t><<<(int)blocks, threads, 0, st>>>(
        (const int32_t*)p, np, (const int32_t*)q, nq, offsets, lengths, B, dim, d_worst);
  else
    validate_kernel<float><<<(int)blocks, threads, 0, st>>>(
        (const float*)p, np, (const float*)q, nq, offsets, lengths, B, dim, d_worst);
  ++*launches;
  int worst = 100;
  cudaMemcpyAsync(&worst, d_worst, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(d_worst, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return FFD_ERR_CUDA;
  switch (worst) {
    case 1: return FFD_ERR_EMPTY;
    case 2: return FFD_ERR_RANGE;
    case 3: return FFD_ERR_NONFINITE;
    case 4: return FFD_ERR_OVERFLOW;
    default: return FFD_OK;
  }
}

}  // namespace ffd
