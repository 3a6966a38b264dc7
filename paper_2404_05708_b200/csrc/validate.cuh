// validate.cuh — synchronous device-data precondition check (ffd_validate_batch).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ffd {
int validate_batch(const void* p, int64_t np, const void* q, int64_t nq, const int64_t* offsets,
                   const int32_t* lengths, int64_t B, int dim, int dtype, cudaStream_t st,
                   int64_t* launches);
}
