// cdist.cuh — all-pairs distances between two dense curve sets (one row shard).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ffd {
struct CdistArgs {
  const void* A;
  const void* B;
  int64_t nA, nB;
  int lenA, lenB, dim, norm, dtype;
  int64_t row_begin, row_end;
  void* out;
  int64_t ld_out;
  void* workspace;
  int self;  // B is A: each unordered pair inside [row_begin, row_end) evaluated once
};
size_t cdist_workspace_bytes();
int launch_cdist(const CdistArgs& a, int sms, cudaStream_t st, int64_t* launches);
}  // namespace ffd
