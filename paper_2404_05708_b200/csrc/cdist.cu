// cdist.cu — placeholder
#include "cdist.cuh"
#include "ffd.h"
namespace ffd {
size_t cdist_workspace_bytes() { return 0; }
int launch_cdist(const CdistArgs& a, int sms, cudaStream_t st, int64_t* launches) {
  return FFD_ERR_UNSUPPORTED;
}
}  // namespace ffd
