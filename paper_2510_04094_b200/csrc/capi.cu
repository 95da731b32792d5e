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

// One steady-state pipeline call in a single C call (linear.SingleSolvePipeline):
// graph A (input-independent work) on `stream`, then -- after `in_event`, or
// after everything already on `caller` when in_event is null (recorded into
// caller_event) -- graph B, then `done` on `stream` and a wait on it in `caller`.
// Saves the host the per-operation Python/stream-switch cost of the same five
// CUDA calls.
extern "C" int nys_replay_pair(void* stream, void* exec_a, void* in_event, void* exec_b,
                               void* done, void* caller, void* caller_event) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaGraphLaunch(static_cast<cudaGraphExec_t>(exec_a), st);
  if (e == cudaSuccess) {
    cudaEvent_t w = static_cast<cudaEvent_t>(in_event);
    if (w == nullptr) {
      w = static_cast<cudaEvent_t>(caller_event);
      e = cudaEventRecord(w, static_cast<cudaStream_t>(caller));
    }
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, w, 0);
  }
  if (e == cudaSuccess) e = cudaGraphLaunch(static_cast<cudaGraphExec_t>(exec_b), st);
  if (e == cudaSuccess) e = cudaEventRecord(static_cast<cudaEvent_t>(done), st);
  if (e == cudaSuccess)
    e = cudaStreamWaitEvent(static_cast<cudaStream_t>(caller), static_cast<cudaEvent_t>(done), 0);
  return nys_host::record_cuda(e);
}

// Host staging of one pipeline call (linear.SingleSolvePipeline.run_host), each
// a single C call for the same reason as nys_replay_pair.  Upload: on `copy`,
// after `free_ev` (the solve that last read this device set; may be null), the
// pinned host block -> device, `ready` recorded behind it, and `caller` made to
// wait on it.
extern "C" int nys_stage_upload(void* dst, const void* src, size_t bytes, void* copy,
                                void* free_ev, void* ready, void* caller) {
  if (dst == nullptr || src == nullptr || ready == nullptr) return NYS_EINVAL;
  cudaStream_t cs = static_cast<cudaStream_t>(copy);
  cudaError_t e = cudaSuccess;
  if (free_ev != nullptr) e = cudaStreamWaitEvent(cs, static_cast<cudaEvent_t>(free_ev), 0);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, cs);
  if (e == cudaSuccess) e = cudaEventRecord(static_cast<cudaEvent_t>(ready), cs);
  if (e == cudaSuccess)
    e = cudaStreamWaitEvent(static_cast<cudaStream_t>(caller), static_cast<cudaEvent_t>(ready), 0);
  return nys_host::record_cuda(e);
}

// Download: `free_ev` recorded on `stream` (everything that read the staged
// inputs is ordered before it), then the solution -> pinned host memory.
extern "C" int nys_stage_download(void* dst_host, const void* src, size_t bytes, void* stream,
                                  void* free_ev) {
  if (dst_host == nullptr || src == nullptr) return NYS_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaSuccess;
  if (free_ev != nullptr) e = cudaEventRecord(static_cast<cudaEvent_t>(free_ev), st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dst_host, src, bytes, cudaMemcpyDeviceToHost, st);
  return nys_host::record_cuda(e);
}
