// common.cuh — shared device definitions of the ffd CUDA library (product path).
//
// Nothing here is shared with oracle/ (the CPU oracle is independent code).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ffd {

// cell kinds: how d_ij is evaluated (PAPER L67 ‖·‖_S)
enum Kind : int {
  K_SQ = 0,    // Σ Δ² (fp32);  L2 = sqrt at the end (hoisted, reading 11)
  K_L1 = 1,    // Σ |Δ|
  K_LINF = 2,  // max |Δ|
  K_XSQ = 3,   // int32 input, Σ Δ² as |p'|² + |q'|² − 2 p'·q' in fp32-exact integer arithmetic
  K_SQRT = 4,  // sqrt(Σ Δ²) per cell (DTW under L2: a sum of distances cannot hoist the sqrt)
};

// output finalisation
// output finalisation / measure: F_DTW selects the dynamic-time-warping cell
// c = min3(up, diag, left) + d (PAPER Appendix B) instead of Fréchet's
// max(min3, d); its result is read from the lane holding row n−1 (no row padding
// is neutral for a sum).
enum Fin : int { F_NONE = 0, F_SQRT = 1, F_DTW = 2 };

constexpr int kWarp = 32;
constexpr int kRing = 128;          // column-stream ring entries per warp (power of two)
constexpr int kRingMask = kRing - 1;
constexpr int kChunkPairs = 8;      // pairs popped per scheduling chunk
constexpr int kMaxR = 16;           // rows per lane, single warp band = 32*kMaxR rows
constexpr int kMaxBands = 16;       // bands per pair in the batch kernel (rows ≤ 8192)
constexpr int kScratchCols = 8260;  // bottom-stream capacity per warp for multi-band chunks
                                    // (columns ≤ 8254: the paper's E2 sweep up to 2^13 stays here;
                                    // the two-column layout needs m + 4 positions)
constexpr int kWarpsPerCta = 4;
#ifndef FFD_TWO_COL
#define FFD_TWO_COL 0
#endif
// batch kernel: two columns per warp step (Fréchet).  Measured and off by default:
// fewer fixed-latency waits, but the larger hot code thrashed the instruction cache.
constexpr bool kTwoCol = FFD_TWO_COL != 0;
#ifndef FFD_MIN_CTAS
#define FFD_MIN_CTAS 4
#endif
constexpr int kMinCtasPerSm = FFD_MIN_CTAS;  // 4 caps registers at 128/thread (16 warps/SM)

// fp32-exact integer window: translated coordinates |x| ≤ lim keep every value
// of the K_XSQ / K_L1 / K_LINF evaluation an integer below 2^24 in magnitude.
__host__ __device__ constexpr int exact_lim(int kind, int D) {
  return kind == K_XSQ ? (D == 1 ? 2047 : D == 2 ? 1448 : D == 3 ? 1182 : 1024)
                       : (1 << 20) / D;
}

// pair descriptor produced by the prep kernels (sorted by band shape)
struct PairDesc {
  int64_t row_off;   // offset (points) of the rows curve (the shorter one)
  int64_t col_off;   // offset (points) of the columns curve
  int32_t n_rows;
  int32_t m_cols;
  int32_t idx;       // original pair index (output slot)
  uint8_t R;         // rows per lane
  uint8_t nb;        // bands
  uint8_t swap;      // 1: rows curve comes from q
  uint8_t pad;
};
static_assert(sizeof(PairDesc) == 32, "PairDesc is 32 bytes");

__device__ __forceinline__ uint64_t pack2(float a, float b) {
  return (uint64_t)__float_as_uint(a) | ((uint64_t)__float_as_uint(b) << 32);
}
__device__ __forceinline__ float lo32(uint64_t v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float hi32(uint64_t v) { return __uint_as_float((uint32_t)(v >> 32)); }

// packed fp32x2 arithmetic (sm_100a FADD2 / FMUL2 / FFMA2), round-to-nearest
__device__ __forceinline__ uint64_t f2_sub_b(uint64_t a, float b) {
  uint64_t r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(pack2(b, b)));
  return r;
}
__device__ __forceinline__ uint64_t f2_add_b(uint64_t a, float b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(pack2(b, b)));
  return r;
}
__device__ __forceinline__ uint64_t f2_mul(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t f2_fma_b(uint64_t a, float b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(pack2(b, b)), "l"(c));
  return r;
}

__device__ __forceinline__ float finf() { return __int_as_float(0x7f800000); }

}  // namespace ffd
