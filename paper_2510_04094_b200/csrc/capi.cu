// C-ABI plumbing: status strings, CUDA error capture, cached device attributes.
#include <atomic>
#include <cstring>

#include "batch_layout.cuh"
#include "common.cuh"

namespace {
thread_local char g_last_err[256] = "";
}

namespace {
std::atomic<unsigned long long> g_launches{0};
}

namespace nys_host {
void count_launches(int k) { g_launches.fetch_add((unsigned long long)k, std::memory_order_relaxed); }

int record_cuda(cudaError_t e) {
  if (e == cudaSuccess) return NYS_OK;
  std::strncpy(g_last_err, cudaGetErrorString(e), sizeof(g_last_err) - 1);
  return NYS_ECUDA;
}
}  // namespace nys_host

namespace nys {
int device_sm_count() {
  static thread_local int cached_dev = -1, cached_sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return cached_sms;
  if (dev != cached_dev) {
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && sms > 0)
      cached_sms = sms;
    cached_dev = dev;
  }
  return cached_sms;
}
}  // namespace nys

extern "C" int nys_abi_version(void) { return NYS_ABI_VERSION; }

extern "C" const char* nys_status_string(int status) {
  switch (status) {
    case NYS_OK: return "ok";
    case NYS_EINVAL: return "invalid argument";
    case NYS_ECUDA: return "CUDA error";
    case NYS_EWORKSPACE: return "workspace too small";
    case NYS_EUNSUPPORTED: return "shape not supported by the compiled kernels";
    default: return "unknown status";
  }
}

extern "C" const char* nys_last_cuda_error(void) { return g_last_err; }

extern "C" unsigned long long nys_launch_count(void) { return g_launches.load(); }
