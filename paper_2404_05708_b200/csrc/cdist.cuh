// cdist.cuh — all-pairs distances between two dense curve sets (one row shard).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ffd {
constexpr int kMaxOuts = 8;  // destinations of one cdist call (this GPU + NVLink peers)

// where the results go: every destination d gets out[d][(row − row_base)·ld + col]
// for (row, col) = (a, col_off + b) — and, with `mirror`, also (col_off + b, a).
struct OutSpec {
  void* out[kMaxOuts];
  int n;
  int64_t row_base, col_off, ld;
  int mirror;
};

struct CdistArgs {
  const void* A;
  const void* B;
  int64_t nA, nB;
  int lenA, lenB, dim, norm, dtype;
  int64_t row_begin, row_end;
  OutSpec dst;
  void* workspace;
  int self;  // B is A (col_off + b indexes A): each unordered pair inside [row_begin, row_end)
             // evaluated once and written to both places
};
size_t cdist_workspace_bytes();
int launch_cdist(const CdistArgs& a, int sms, cudaStream_t st, int64_t* launches);
}  // namespace ffd
