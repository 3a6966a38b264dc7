// prep.cuh — batch preparation (shape keys + counting sort) and the batch
// workspace layout shared by api.cu and the kernels.
#pragma once
#include <climits>
#include <cstddef>

#include "common.cuh"

namespace ffd {

constexpr int kNumKeys = kMaxBands * kMaxR;  // 256 shape bins of the batch kernel
constexpr int kSegBinsP = 24 * 65;          // (shape, period) bins of the segmented kernel (seg.cuh kSegBins)
constexpr int kAllKeys = kNumKeys + kSegBinsP;
constexpr int64_t kPrepSmallMax = 4096;      // batches up to this size: one-block prep

// a valid pair (n, m ≥ 1) too long for the batch kernel's bands / band scratch
__host__ __device__ inline bool pair_too_long(int n, int m) {
  const int rows = n < m ? n : m, cols = n < m ? m : n;
  const int nb = (rows + kWarp * kMaxR - 1) / (kWarp * kMaxR);
  return nb > kMaxBands || (nb > 1 && cols + 6 > kScratchCols);
}

// Fréchet pairs whose shorter curve needs 8 or more bands of 512 rows run on the
// long-pair kernel (a group of CTAs per pair, bands pipelined over its warps)
// instead of one warp walking the bands in sequence: a batch of such pairs
// rarely has enough of them to fill the GPU one warp each (the paper's E2 sweep:
// 1024 pairs of 8192 points ran on 1024 warps at 1.9 T cells/s).
constexpr int kMediumRows = 7 * kWarp * kMaxR;  // 3584
// A batch of at most one pair per SM cannot fill the GPU one warp per pair: there
// every multi-band pair (more than 512 rows) goes to the CTA groups, a CTA or
// more each (the paper's E1 sweep at N ≤ 128 walks of 1024 points ran on N warps).
__host__ __device__ inline int medium_rows_for(int64_t num_pairs, int sms) {
  return num_pairs <= sms ? kWarp * kMaxR : kMediumRows;
}

// the rule of the device prep, shared with host callers that know the lengths:
// the pair goes to the long-pair list (medium_rows = medium_rows_for(B, SMs))
__host__ __device__ inline bool pair_goes_long(int n, int m, int medium_rows) {
  const int rows = n < m ? n : m;
  return pair_too_long(n, m) || rows > medium_rows;
}

// counters block (int32 each), zeroed per call (by the one-block prep, or a
// memset of the counters + histogram block)
enum : int {
  kCtrNumSorted = 0,
  kCtrChunkMain = 1,
  kCtrChunkFb = 2,
  kCtrFb = 3,
  kCtrLong = 4,
  kCtrChunkLong = 5,
  kCtrSegItems = 6,  // groups of the segmented kernel
  kCtrSegChunk = 7,  // (unused: the segmented kernel pops per shape)
  kCtrSegShape = 8,  // [2] group pop counters of the segmented kernels (small, big)
  kNumCtr = 32
};

struct BatchWs {
  PairDesc* tmp;      // [B]
  PairDesc* sorted;   // [B]
  int16_t* keys;      // [B]
  int* hist;          // [kAllKeys]: batch-kernel shape bins, then segmented-kernel bins
  int* cursor;        // [kAllKeys]
  int* counters;      // [kNumCtr]
  int* fb_list;       // [B]
  int* long_list;     // [B]
  float* scratch_main;  // [warps_main][2][kScratchCols] float
  long long* scratch_fb;  // [warps_fb][2][kScratchCols] int64
  PairDesc* seg_sorted;   // [B] pairs of the segmented kernel, by (shape, period) descending
  void* seg_groups;       // [seg_max_groups(B)] SegGroup
  int* seg_off;           // [2 · kSegBinsP + 3 · 24]: first group per bin rank, bin starts, per shape
                          // (first group, end, work as float bits)
  size_t bytes;
};

// long_ok: < 0 = DTW (only pairs too long for the bands go to the long-pair list),
// 0 = no long-pair path (such pairs get NaN / INT64_MIN),
// else the medium-row threshold (medium_rows_for(B, SMs)) of Fréchet
// long_run = false: the long-pair kernel will not run (the caller's length
// bounds rule it out), so a pair that would go long gets NaN / INT64_MIN
// seg: route the Fréchet pairs the segmented kernel takes (seg_bin ≥ 0) to its
// list and item table (general path only: B > kPrepSmallMax)
cudaError_t launch_prep(const int64_t* offsets, const int32_t* lengths, int64_t B, int int_out,
                        int long_ok, void* out, const BatchWs& ws, int num_sms, cudaStream_t st,
                        int64_t* launches, bool seg = false, bool long_run = true);

}  // namespace ffd
