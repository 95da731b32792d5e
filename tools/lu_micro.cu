// microbenchmark of the persistent kernel's LU (tools only): includes newton.cu
#include "../paper_2510_04094_b200/csrc/newton.cu"
#include <cstdio>
#include <vector>
#include <random>
namespace {
__global__ void lu_bench(const double* Kg, const double* rg, int n, long long* clk, double* out) {
  extern __shared__ double sm[];
  __shared__ int flag;
  double* K = sm; double* ys = K + n * n; int* perm = (int*)(ys + n); double* T = sm + 2 * n * n + 2 * n;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) K[e] = Kg[e];
  for (int e = threadIdx.x; e < n; e += blockDim.x) ys[e] = rg[e];
  __syncthreads();
  long long t0 = clock64();
  int info = persist_lu(K, ys, perm, n, &flag, T);
  long long t1 = clock64();
  if (threadIdx.x == 0) { clk[0] = t1 - t0; clk[1] = info; }
  for (int e = threadIdx.x; e < n; e += blockDim.x) out[e] = ys[e];
}
}
int main() {
  int n = 42;
  std::vector<double> K(n * n), r(n);
  std::mt19937 g(1); std::uniform_real_distribution<double> u(-1, 1);
  for (auto& v : K) v = u(g);
  for (int i = 0; i < n; ++i) K[i * n + i] += 10;
  for (auto& v : r) v = u(g);
  double *dK, *dr, *dout; long long* dc;
  cudaMalloc(&dK, n * n * 8); cudaMalloc(&dr, n * 8); cudaMalloc(&dout, n * 8); cudaMalloc(&dc, 16);
  cudaMemcpy(dK, K.data(), n * n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dr, r.data(), n * 8, cudaMemcpyHostToDevice);
  size_t smem = (3 * n * n + 3 * n) * 8 + 64 * 65 * 8;
  cudaFuncSetAttribute(lu_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int rep = 0; rep < 3; ++rep) {
    lu_bench<<<1, 256, smem>>>(dK, dr, n, dc, dout);
    long long c[2]; cudaMemcpy(c, dc, 16, cudaMemcpyDeviceToHost);
    printf("LU n=%d: %lld clocks info %lld (%s)\n", n, c[0], c[1], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
