// prep.cuh — batch preparation (shape keys + counting sort) and the batch
// workspace layout shared by api.cu and the kernels.
#pragma once
#include <climits>
#include <cstddef>

#include "common.cuh"

namespace ffd {

constexpr int kNumKeys = kMaxBands * kMaxR;  // 128 shape bins

// counters block (int32 each), zeroed by one memset per call
enum : int {
  kCtrNumSorted = 0,
  kCtrChunkMain = 1,
  kCtrChunkFb = 2,
  kCtrFb = 3,
  kCtrLong = 4,
  kCtrChunkLong = 5,
  kNumCtr = 8
};

struct BatchWs {
  PairDesc* tmp;      // [B]
  PairDesc* sorted;   // [B]
  int16_t* keys;      // [B]
  int* hist;          // [kNumKeys]
  int* cursor;        // [kNumKeys]
  int* counters;      // [kNumCtr]
  int* fb_list;       // [B]
  int* long_list;     // [B]
  float* scratch_main;  // [warps_main][2][kScratchCols] float
  long long* scratch_fb;  // [warps_fb][2][kScratchCols] int64
  size_t bytes;
};

cudaError_t launch_prep(const int64_t* offsets, const int32_t* lengths, int64_t B, int int_out,
                        int long_ok, void* out, const BatchWs& ws, int num_sms, cudaStream_t st,
                        int64_t* launches);

}  // namespace ffd
