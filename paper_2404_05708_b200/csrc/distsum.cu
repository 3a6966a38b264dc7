// distsum.cu — Σ_ij d(p_i, q_j) per pair: the B200 analogue of the paper's
// "upper limit" baseline: the DP's distances (L2 with
// a square root per cell, the paper's hypot workload L271) summed, with no
// recurrence.  It calibrates how close the DP kernels come to the cost of the
// distances alone, as the paper's Fig. 1/2 do for SIMD on one core.
//
// Work split: a pair's P×Q cells are cut into tiles of 32 rows × 256 columns.
// A warp takes a tile: lane ℓ holds the 8 columns j0+ℓ+32c (c < 8, coalesced
// loads) in registers, the 32 rows' points arrive by one coalesced load and a
// shuffle broadcast per row, and the lane keeps one fp32 sum per column (8
// independent chains).  A tile's 8 column sums (≤ 32 terms each) are widened
// into the lane's fp64 total.  CTA (k, s) of the grid B×S takes the tiles
// t ≡ s (mod S) of pair k, 8 warps strided; S is chosen so the grid fills the
// SMs even for small B.  Every reduction has a fixed order (shuffle xor tree,
// warps in order, splits in order): results are deterministic.
//
// Rounding: each fp32 column sum of ≤ 32 positive terms is within 31·2⁻²⁴ of
// its exact sum, each term within (2·dim + 4)·2⁻²⁴ of the exact d_ij; the fp64
// steps add nothing visible.  So |out − Σd| ≤ (35 + 2·dim)·2⁻²⁴ · Σd.
#include <algorithm>
#include <climits>
#include <cmath>

#include "distsum.cuh"
#include "ffd.h"

namespace ffd {

constexpr int kDsWarps = 8;   // warps per CTA
constexpr int kDsCols = 8;    // columns per lane per tile
constexpr int kDsTileCols = 32 * kDsCols;

// d_ij in fp32: Δ_k = p_k − q_k; L1 Σ|Δ_k|, L∞ max|Δ_k|, sqL2 Σ Δ_k² (fma
// chain from k = 0), L2 = sqrt(sqL2) by the SFU's approximate square root
// (relative error ≤ 2⁻²³; a subnormal sqL2 flushes to 0, an absolute error
// < 2⁻⁶³ per term) — the cheapest honest distance, as an upper limit should be.
template <int NORM, int D>
__device__ __forceinline__ float ds_dist(const float (&a)[D], const float (&b)[D]) {
  float acc;
  if constexpr (NORM == FFD_L1) {
    acc = fabsf(a[0] - b[0]);
#pragma unroll
    for (int k = 1; k < D; k++) acc += fabsf(a[k] - b[k]);
  } else if constexpr (NORM == FFD_LINF) {
    acc = fabsf(a[0] - b[0]);
#pragma unroll
    for (int k = 1; k < D; k++) acc = fmaxf(acc, fabsf(a[k] - b[k]));
  } else {
    const float d0 = a[0] - b[0];
    acc = d0 * d0;
#pragma unroll
    for (int k = 1; k < D; k++) {
      const float dk = a[k] - b[k];
      acc = fmaf(dk, dk, acc);
    }
    if constexpr (NORM == FFD_L2) asm("sqrt.approx.ftz.f32 %0, %0;" : "+f"(acc));
  }
  return acc;
}

template <int NORM, int D>
__global__ void __launch_bounds__(kDsWarps * 32)
    dist_sum_kernel(const float* __restrict__ p, const float* __restrict__ q,
                    const int64_t* __restrict__ offsets, const int32_t* __restrict__ lengths,
                    int64_t B, int S, double* __restrict__ partial) {
  __shared__ double red[kDsWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t item = blockIdx.x;
  const int64_t k = item / S;
  const int s = (int)(item - k * S);
  const int32_t n = lengths[k], m = lengths[B + k];
  double acc = 0.0;
  if (n >= 1 && m >= 1) {
    const float* pk = p + offsets[k] * D;
    const float* qk = q + offsets[B + k] * D;
    const int64_t tiles_j = (m + kDsTileCols - 1) / kDsTileCols;
    const int64_t tiles = (int64_t)((n + 31) / 32) * tiles_j;
    for (int64_t t = (int64_t)s * kDsWarps + warp; t < tiles; t += (int64_t)S * kDsWarps) {
      const int32_t i0 = (int32_t)(t / tiles_j) * 32;
      const int32_t j0 = (int32_t)(t % tiles_j) * kDsTileCols;
      float qc[kDsCols][D];
#pragma unroll
      for (int c = 0; c < kDsCols; c++) {
        const int32_t j = min(j0 + lane + 32 * c, m - 1);
#pragma unroll
        for (int d = 0; d < D; d++) qc[c][d] = qk[(int64_t)j * D + d];
      }
      float pr[D];
      {
        const int32_t i = min(i0 + lane, n - 1);
#pragma unroll
        for (int d = 0; d < D; d++) pr[d] = pk[(int64_t)i * D + d];
      }
      const int rows = min(32, n - i0);
      float a[kDsCols];
#pragma unroll
      for (int c = 0; c < kDsCols; c++) a[c] = 0.f;
#pragma unroll 4
      for (int r = 0; r < rows; r++) {
        float x[D];
#pragma unroll
        for (int d = 0; d < D; d++) x[d] = __shfl_sync(0xffffffffu, pr[d], r);
#pragma unroll
        for (int c = 0; c < kDsCols; c++) a[c] += ds_dist<NORM, D>(x, qc[c]);
      }
#pragma unroll
      for (int c = 0; c < kDsCols; c++)
        if (j0 + lane + 32 * c < m) acc += (double)a[c];
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
#pragma unroll
    for (int w = 0; w < kDsWarps; w++) tot += red[w];
    partial[item] = (n >= 1 && m >= 1) ? tot : (double)NAN;
  }
}

// out[k] = Σ_s partial[k·S + s], in order
__global__ void dist_sum_reduce_kernel(const double* __restrict__ partial, int64_t B, int S,
                                       double* __restrict__ out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < B;
       k += (int64_t)gridDim.x * blockDim.x) {
    double t = 0.0;
    for (int s = 0; s < S; s++) t += partial[k * S + s];
    out[k] = t;
  }
}

template <int NORM, int D>
static cudaError_t launch_nd(const float* p, const float* q, const int64_t* offsets,
                             const int32_t* lengths, int64_t B, int S, double* partial,
                             cudaStream_t st) {
  dist_sum_kernel<NORM, D><<<(unsigned)(B * S), kDsWarps * 32, 0, st>>>(p, q, offsets, lengths, B,
                                                                       S, partial);
  return cudaGetLastError();
}

template <int NORM>
static cudaError_t launch_n(int dim, const float* p, const float* q, const int64_t* offsets,
                            const int32_t* lengths, int64_t B, int S, double* partial,
                            cudaStream_t st) {
  switch (dim) {
    case 1: return launch_nd<NORM, 1>(p, q, offsets, lengths, B, S, partial, st);
    case 2: return launch_nd<NORM, 2>(p, q, offsets, lengths, B, S, partial, st);
    case 3: return launch_nd<NORM, 3>(p, q, offsets, lengths, B, S, partial, st);
    default: return launch_nd<NORM, 4>(p, q, offsets, lengths, B, S, partial, st);
  }
}

int launch_dist_sum(const float* p, const float* q, const int64_t* offsets, const int32_t* lengths,
                    int64_t B, int dim, int norm, double* out, int sms, cudaStream_t st,
                    int64_t* launches) {
  // enough CTAs for ~8 resident per SM even when B is small
  const int64_t want = (int64_t)sms * 8;
  int S = (int)std::min<int64_t>(1024, std::max<int64_t>(1, (want + B - 1) / B));
  if (B * S > INT_MAX) return FFD_ERR_UNSUPPORTED;
  double* partial = out;
  if (S > 1 && cudaMallocAsync(reinterpret_cast<void**>(&partial), sizeof(double) * B * S, st))
    return FFD_ERR_CUDA;
  cudaError_t e;
  switch (norm) {
    case FFD_L1: e = launch_n<FFD_L1>(dim, p, q, offsets, lengths, B, S, partial, st); break;
    case FFD_L2: e = launch_n<FFD_L2>(dim, p, q, offsets, lengths, B, S, partial, st); break;
    case FFD_LINF: e = launch_n<FFD_LINF>(dim, p, q, offsets, lengths, B, S, partial, st); break;
    default: e = launch_n<FFD_SQL2>(dim, p, q, offsets, lengths, B, S, partial, st); break;
  }
  ++*launches;
  if (e == cudaSuccess && S > 1) {
    const int threads = 256;
    const int64_t blocks = std::min<int64_t>((B + threads - 1) / threads, (int64_t)sms * 8);
    dist_sum_reduce_kernel<<<(unsigned)blocks, threads, 0, st>>>(partial, B, S, out);
    e = cudaGetLastError();
    ++*launches;
  }
  if (S > 1) cudaFreeAsync(partial, st);
  return e == cudaSuccess ? FFD_OK : FFD_ERR_CUDA;
}

}  // namespace ffd
