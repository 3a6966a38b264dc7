// distsum.cuh — launcher of the Σ_ij d_ij calibration kernel (distsum.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ffd {

// out[k] = Σ_i Σ_j d(p_i, q_j) of pair k (fp32 coordinates, dim 1..4, norm an
// ffd_norm).  Returns FFD_OK or an ffd_status; counts its launches.
int launch_dist_sum(const float* p, const float* q, const int64_t* offsets, const int32_t* lengths,
                    int64_t B, int dim, int norm, double* out, int sms, cudaStream_t st,
                    int64_t* launches);

}  // namespace ffd
