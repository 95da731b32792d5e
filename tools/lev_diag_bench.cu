// Microbenchmark of the leverage diag-tile kernel (includes the product TU).
#include "../paper_2510_04094_b200/csrc/leverage.cu"
#include <cstdio>
#include <vector>

namespace {
__global__ void __launch_bounds__(kThreads) copy_only(const double* At, double* Bt) {
  extern __shared__ __align__(128) double smem[];
  __shared__ uint64_t bar;
  load_tiles(smem, At, nullptr, nullptr, &bar);
  for (int e = threadIdx.x; e < kTT; e += kThreads) Bt[e] = smem[e];
}
__global__ void __launch_bounds__(kThreads) warp_only(const double* At, double* Bt, int* info) {
  extern __shared__ __align__(128) double smem[];
  __shared__ uint64_t bar;
  __shared__ double colv[2][kDB], rowv[2][kDB];
  load_tiles(smem, At, nullptr, nullptr, &bar);
  double* Xm = smem + kTT;
  if (threadIdx.x < 32)
    for (int P = 0; P < 8; ++P)
      if (!warp_chol_inv(smem, Xm, P * 8, colv, rowv)) *info = 1;
  __syncthreads();
  for (int e = threadIdx.x; e < kTT; e += kThreads) Bt[e] = Xm[e];
}
}  // namespace

int main() {
  std::vector<double> h(kTT);
  // SPD tile: exp kernel + ridge, swizzled
  for (int r = 0; r < kT; ++r)
    for (int c = 0; c < kT; ++c) {
      double d = (r - c) / 64.0;
      h[r * kT + (c ^ ((r & 3) << 2))] = exp(-d * d / 0.01) + (r == c ? 1e-3 : 0.0);
    }
  double *A, *B;
  int* info;
  cudaMalloc(&A, kTT * 8);
  cudaMalloc(&B, kTT * 8);
  cudaMalloc(&info, 4);
  cudaMemcpy(A, h.data(), kTT * 8, cudaMemcpyHostToDevice);
  const int smem = 2 * kTT * 8;
  cudaFuncSetAttribute(lev_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(copy_only, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(warp_only, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int v = 0; v < 3; ++v) {
    for (int it = 0; it < 5; ++it) {
      if (v == 0) lev_diag_kernel<<<1, kThreads, smem>>>(A, B, 0, info);
      if (v == 1) copy_only<<<1, kThreads, smem>>>(A, B);
      if (v == 2) warp_only<<<1, kThreads, smem>>>(A, B, info);
    }
    cudaEventRecord(e0);
    const int N = 200;
    for (int it = 0; it < N; ++it) {
      if (v == 0) lev_diag_kernel<<<1, kThreads, smem>>>(A, B, 0, info);
      if (v == 1) copy_only<<<1, kThreads, smem>>>(A, B);
      if (v == 2) warp_only<<<1, kThreads, smem>>>(A, B, info);
    }
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("variant %d: %.2f us/launch (%s)\n", v, ms * 1e3 / N, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
