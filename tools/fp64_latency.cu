// FP64 latency probe (one warp): dependent DFMA, dependent DMMA, DMMA issue
// interval with 16 independent accumulators, dependent exp.  Cycles per op.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

__global__ void k(double* out, long long* cyc, int iters, double a, double b) {
  long long t0, t1;
  double x = threadIdx.x * 1e-3;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, a, b);
  t1 = clock64();
  cyc[0] = t1 - t0;
  double c0 = 0, c1 = 0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) dmma(c0, c1, a, b);
  t1 = clock64();
  cyc[1] = t1 - t0;
  double c[16][2] = {};
  t0 = clock64();
  for (int i = 0; i < iters / 16; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) dmma(c[j][0], c[j][1], a, b);
  }
  t1 = clock64();
  cyc[2] = t1 - t0;
  double y = 0.5 + threadIdx.x * 1e-6;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) y = exp(-y * 1e-3) ;
  t1 = clock64();
  cyc[3] = t1 - t0;
  double s = x + c0 + c1 + y;
  for (int j = 0; j < 16; ++j) s += c[j][0] + c[j][1];
  if (s == 1.2345) out[0] = s;
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 8);
  cudaMallocManaged(&cyc, 64);
  int iters = 4096;
  for (int r = 0; r < 2; ++r) {
    k<<<1, 32>>>(out, cyc, iters, 1.0000001, 1e-9);
    cudaDeviceSynchronize();
  }
  printf("dependent DFMA      %.1f cycles/op\n", (double)cyc[0] / iters);
  printf("dependent DMMA      %.1f cycles/op\n", (double)cyc[1] / iters);
  printf("16-indep DMMA       %.1f cycles/op (1 warp)\n", (double)cyc[2] / (iters / 16 * 16));
  printf("dependent exp()     %.1f cycles/op\n", (double)cyc[3] / iters);
  return 0;
}
