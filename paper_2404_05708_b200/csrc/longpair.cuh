// longpair.cuh — pairs too long for the batch kernel's band scratch.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ffd {
struct LongArgs {
  const void* p;
  const void* q;
  const int64_t* offsets;
  const int32_t* lengths;
  int64_t num_pairs;
  int dim, norm, dtype;
  int measure;            // 0: discrete Fréchet (Eq. (1)); 1: DTW (PAPER Appendix B)
  const int* list;        // device list of long pair indices
  const int* list_count;  // device count
  void* out;
  void* wrap;         // device scratch for the multi-pass wrap link (any contents)
  size_t wrap_bytes;  // its size
  // ffd_long_pair_shard: rows [row_begin, row_end) of the single pair, links to the
  // neighbouring GPUs' rings (slots are 8-byte {value, tag}; sizes powers of two)
  int shard;
  int row_begin, row_end;
  void* ext_in;
  size_t ext_in_slots;
  unsigned ext_in_tb;
  void* ext_out;
  size_t ext_out_slots;
  unsigned ext_out_tb;
  unsigned* ext_cons;  // [2] device
};
cudaError_t launch_long_pairs(const LongArgs& a, int sms, cudaStream_t st, int64_t* launches);
// slots of a cross-GPU ring for a pair whose column curve has m points (fp32)
size_t long_shard_ring_slots(int m);
// one pair (n rows after orientation = the shorter curve), rows [row_begin, row_end)
cudaError_t launch_long_shard(LongArgs a, int n0, int m0, int sms, cudaStream_t st, int64_t* launches);
}  // namespace ffd
