// validate.cu — one block per pair checks the preconditions of include/ffd.h:
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

// one block per pair (grid-stride over pairs): the block's threads stride over
// the pair's points, so one very long pair is checked as fast as many short ones
template <typename In>
__global__ void __launch_bounds__(256) validate_kernel(const In* p, int64_t np, const In* q, int64_t nq,
                                                      const int64_t* offsets, const int32_t* lengths, int64_t B,
                                                      int dim, int* worst) {
  __shared__ int s_lo[4], s_hi[4], s_nonfinite;
  for (int64_t k = blockIdx.x; k < B; k += gridDim.x) {
    const int64_t op = offsets[k], oq = offsets[B + k];
    const int32_t n = lengths[k], m = lengths[B + k];
    int bad = 0;
    if (n < 1 || m < 1) bad = FFD_ERR_EMPTY;
    else if (op < 0 || oq < 0 || op + n > np || oq + m > nq) bad = FFD_ERR_RANGE;
    if (bad) {  // the same for every thread of the block
      if (threadIdx.x == 0) atomicMin(worst, prio_of(bad));
      continue;
    }
    if (threadIdx.x < 4) {
      s_lo[threadIdx.x] = INT_MAX;
      s_hi[threadIdx.x] = INT_MIN;
    }
    if (threadIdx.x == 0) s_nonfinite = 0;
    __syncthreads();
    for (int c = 0; c < dim; c++) {
      int lo = INT_MAX, hi = INT_MIN, nf = 0;
      for (int side = 0; side < 2; side++) {
        const In* base = side ? q + oq * dim : p + op * dim;
        const int32_t len = side ? m : n;
        for (int32_t i = threadIdx.x; i < len; i += blockDim.x) {
          const In v = base[(int64_t)i * dim + c];
          if constexpr (std::is_floating_point<In>::value) {
            nf |= !isfinite((float)v);
          } else {
            lo = min(lo, (int)v);
            hi = max(hi, (int)v);
          }
        }
      }
      if constexpr (std::is_floating_point<In>::value) {
        if (__any_sync(0xffffffffu, nf) && (threadIdx.x & 31) == 0) s_nonfinite = 1;
      } else {
        lo = __reduce_min_sync(0xffffffffu, lo);
        hi = __reduce_max_sync(0xffffffffu, hi);
        if ((threadIdx.x & 31) == 0) {
          atomicMin(&s_lo[c], lo);
          atomicMax(&s_hi[c], hi);
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (s_nonfinite) bad = FFD_ERR_NONFINITE;
      if constexpr (!std::is_floating_point<In>::value) {
        unsigned long long sum = 0;
        for (int c = 0; c < dim && !bad; c++) {
          const unsigned long long r = (unsigned long long)((long long)s_hi[c] - (long long)s_lo[c]);  // < 2^32
          const unsigned long long t = r * r;                                                         // < 2^64
          if (t > (unsigned long long)LLONG_MAX || sum > (unsigned long long)LLONG_MAX - t) bad = FFD_ERR_OVERFLOW;
          else sum += t;
        }
      }
      if (bad) atomicMin(worst, prio_of(bad));
    }
    __syncthreads();  // the shared reductions are reset for the next pair
  }
}

int validate_batch(const void* p, int64_t np, const void* q, int64_t nq, const int64_t* offsets,
                   const int32_t* lengths, int64_t B, int dim, int dtype, cudaStream_t st,
                   int64_t* launches) {
  int* d_worst = nullptr;
  if (cudaMallocAsync(&d_worst, sizeof(int), st) != cudaSuccess) return FFD_ERR_CUDA;
  const int init = 100;
  cudaMemcpyAsync(d_worst, &init, sizeof(int), cudaMemcpyHostToDevice, st);
  const int threads = 256;
  int64_t blocks = B < 148 * 16 ? B : 148 * 16;
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
