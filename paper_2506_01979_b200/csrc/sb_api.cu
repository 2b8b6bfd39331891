// sb_api.cu — version, status strings, workspace sizing, device attributes.
#include <cuda_runtime.h>
#include <stdlib.h>

#include "sb_host.h"

namespace sb {
int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}
// queried per call (the driver caches device attributes): a process may drive several GPUs
int num_sms() {
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, current_device());
  return n > 0 ? n : 148;
}
bool tma_disabled() {
  const char* e = getenv("SB_DISABLE_TMA");
  return e && e[0] == '1';
}
}  // namespace sb

extern "C" const char* sb_version(void) { return "specbranch-b200 0.1 (sm_100a)"; }

extern "C" const char* sb_status_string(sb_status s) {
  switch (s) {
    case SB_OK: return "ok";
    case SB_ERR_INVALID_ARG: return "invalid argument";
    case SB_ERR_UNSUPPORTED: return "unsupported";
    case SB_ERR_CUDA: return "CUDA error";
    case SB_ERR_NCCL: return "NCCL error";
    case SB_ERR_WORKSPACE: return "workspace too small";
  }
  return "unknown status";
}

extern "C" size_t sb_workspace_bytes(const sb_dims* d) {
  if (!sb::dims_valid(d)) return 0;
  return sb::carve(*d, nullptr).bytes;
}
