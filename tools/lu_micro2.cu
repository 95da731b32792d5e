// phase timing of the persistent LU (tools only)
#include <cstdio>
#include <vector>
#include <random>
#include <cuda_runtime.h>
__global__ void lu_phases(const double* Kg, int n, long long* clk) {
  extern __shared__ double T[];
  __shared__ int perm[64]; __shared__ int flag;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int ld = n | 1;
  for (int e = tid; e < n * n; e += blockDim.x) T[(e / n) * ld + e % n] = Kg[e];
  __syncthreads();
  long long tp = 0, tsync1 = 0, tdiv = 0, tupd = 0, tsync2 = 0;
  for (int k = 0; k < n; ++k) {
    long long t0 = clock64();
    if (warp == 0) {
      double bv = -1.0; int bi = n;
      for (int i = k + lane; i < n; i += 32) { const double a = fabs(T[i * ld + k]); if (a > bv) { bv = a; bi = i; } }
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o); const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; } }
      if (lane == 0) perm[k] = bi;
      if (bi != k) for (int j = lane; j < n; j += 32) { const double a = T[k * ld + j], p = T[bi * ld + j]; T[bi * ld + j] = a; T[k * ld + j] = p; }
    }
    long long t1 = clock64();
    __syncthreads();
    long long t2 = clock64();
    const double inv = 1.0 / T[k * ld + k];
    long long t3 = clock64();
    const double* urow = T + k * ld;
    for (int i = k + 1 + warp; i < n; i += nw) {
      double* r = T + i * ld; const double l = r[k] * inv; __syncwarp(); if (lane == 0) r[k] = l;
      for (int j = k + 1 + lane; j < n; j += 32) r[j] -= l * urow[j];
    }
    long long t4 = clock64();
    __syncthreads();
    long long t5 = clock64();
    tp += t1 - t0; tsync1 += t2 - t1; tdiv += t3 - t2; tupd += t4 - t3; tsync2 += t5 - t4;
  }
  if (tid == 0) { clk[0] = tp; clk[1] = tsync1; clk[2] = tdiv; clk[3] = tupd; clk[4] = tsync2; }
}
int main() {
  int n = 42; std::vector<double> K(n * n); std::mt19937 g(1); std::uniform_real_distribution<double> u(-1, 1);
  for (auto& v : K) v = u(g); for (int i = 0; i < n; ++i) K[i * n + i] += 10;
  double* dK; long long* dc; cudaMalloc(&dK, n * n * 8); cudaMalloc(&dc, 64);
  cudaMemcpy(dK, K.data(), n * n * 8, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 2; ++rep) {
    lu_phases<<<1, 256, 64 * 65 * 8>>>(dK, n, dc);
    long long c[5]; cudaMemcpy(c, dc, 40, cudaMemcpyDeviceToHost);
    printf("pivot %lld sync1 %lld div %lld update %lld sync2 %lld (%s)\n", c[0], c[1], c[2], c[3], c[4], cudaGetErrorString(cudaGetLastError()));
  }
}
