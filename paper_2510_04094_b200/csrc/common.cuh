// Shared device helpers for the nysb200 sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/nysb200.h"

#define NYS_DEV __device__ __forceinline__

namespace nys {

int device_sm_count();   // cached cudaDevAttrMultiProcessorCount (capi.cu)

constexpr int kMaxOrder = 4;   // kernel.py:19 MAX_DERIV_ORDER

// D = A*B + C with A 8x4 (row), B 4x8 (col), C/D 8x8, fp64 -> SASS DMMA.8x8x4.
// Fragments: lane l holds A[l>>2][l&3], B[l&3][l>>2], C[l>>2][2(l&3)+{0,1}].
NYS_DEV void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Coefficients (low degree first) of P_order for bandwidth sigma2, built by the
// same recursion as kernel.py:26-37: P_{a+1} = (2 d / sigma2) P_a - P_a'.
struct Hermite {
  double c[kMaxOrder + 1][kMaxOrder + 1];  // c[a][j]: coefficient of d^j in P_a
  NYS_DEV void init(double sigma2, int pmax) {
    const double s = 2.0 / sigma2;
#pragma unroll
    for (int a = 0; a <= kMaxOrder; ++a)
#pragma unroll
      for (int j = 0; j <= kMaxOrder; ++j) c[a][j] = 0.0;
    c[0][0] = 1.0;
#pragma unroll
    for (int a = 0; a < kMaxOrder; ++a) {
      if (a >= pmax) break;
#pragma unroll
      for (int j = kMaxOrder; j >= 1; --j) c[a + 1][j] = c[a][j - 1] * s;
      c[a + 1][0] = 0.0;
#pragma unroll
      for (int j = 1; j <= kMaxOrder; ++j) c[a + 1][j - 1] -= c[a][j] * (double)j;
    }
  }
  // Horner over degree <= a (kernel.py:62-66)
  NYS_DEV double poly(int a, double d) const {
    double acc = 0.0;
#pragma unroll
    for (int j = kMaxOrder; j >= 0; --j)
      if (j <= a) acc = acc * d + c[a][j];
    return acc;
  }
};

// exp(-(d*d)/sigma2) exactly as kernel.py:78-79 spells it (true division).
NYS_DEV double rbf(double d, double sigma2) { return exp(-(d * d) / sigma2); }

NYS_DEV int lane_id() { return threadIdx.x & 31; }

NYS_DEV double shfl(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }

// ---- async bulk copy (TMA 1-D) + mbarrier -----------------------------------------
NYS_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
NYS_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
NYS_DEV void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
NYS_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
NYS_DEV void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// shared-memory atomic add with acquire-release semantics at CTA scope
NYS_DEV int atomic_add_acq_rel_cta(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], %2;\n"
               : "=r"(old)
               : "r"(smem_u32(p)), "r"(v)
               : "memory");
  return old;
}
// global -> shared bulk copy, completion signalled on `bar` (bytes % 16 == 0).
NYS_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

}  // namespace nys

// host-side helpers shared by the translation units
namespace nys_host {
int record_cuda(cudaError_t e);   // stores the message, returns NYS_ECUDA or NYS_OK
void count_launches(int k);       // process-wide kernel launch counter (nys_launch_count)
inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
}  // namespace nys_host

#define NYS_CHECK_LAUNCH()                                          \
  do {                                                              \
    cudaError_t _e = cudaGetLastError();                            \
    if (_e != cudaSuccess) return nys_host::record_cuda(_e);        \
  } while (0)
