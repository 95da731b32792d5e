// FP64 pipe microbenchmark for B200 (sm_100a): DMMA m8n8k4 and DFMA peak.
// Measures the roofline denominator that MEASURED_PEAKS.json lacks (no FP64 entry).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int NACC>
__global__ void k_dmma(double* out, int iters, double a, double b) {
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  double aa = a + threadIdx.x * 1e-9, bb = b - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) dmma(c[i][0], c[i][1], aa, bb);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 123.456) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void k_dfma(double* out, int iters, double a, double b) {
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 123.456) out[threadIdx.x] = s;
}

// mixed: DMMA stream with interleaved DFMA (does DFMA steal DMMA issue slots?)
template <int NACC, int NF>
__global__ void k_mixed(double* out, int iters, double a, double b) {
  double c[NACC][2];
  double f[NF];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
#pragma unroll
  for (int i = 0; i < NF; ++i) f[i] = threadIdx.x + i;
  double aa = a + threadIdx.x * 1e-9, bb = b - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) dmma(c[i][0], c[i][1], aa, bb);
#pragma unroll
    for (int i = 0; i < NF; ++i) f[i] = fma(f[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < NF; ++i) s += f[i];
  if (s == 123.456) out[threadIdx.x] = s;
}

__global__ void k_exp(double* out, int iters, double x0) {
  double x = x0 + threadIdx.x * 1e-7, s = 0;
  for (int it = 0; it < iters; ++it) { s += exp(-x * x); x += 1e-9; }
  if (s == 123.456) out[threadIdx.x] = s;
}

template <typename F>
float timeit(F f) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  f();  // warm
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int sms = p.multiProcessorCount;
  double* out; cudaMalloc(&out, 4096 * sizeof(double));
  int iters = 20000;
  printf("{\"device\": \"%s\", \"sms\": %d", p.name, sms);
  for (int wpb : {4, 8, 16}) {
    int blocks = sms * 2, threads = 32 * wpb;
    float ms = timeit([&] { k_dmma<8><<<blocks, threads>>>(out, iters, 1.0, 1.0); });
    double flops = 2.0 * 256 * 8 * (double)iters * blocks * wpb;
    printf(", \"dmma_m8n8k4_w%d_tflops\": %.3f", wpb, flops / ms / 1e9);
  }
  for (int wpb : {8, 16, 32}) {
    int blocks = sms * 2, threads = 32 * wpb;
    float ms = timeit([&] { k_dfma<16><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); });
    double flops = 2.0 * 16 * (double)iters * blocks * threads;
    printf(", \"dfma_w%d_tflops\": %.3f", wpb, flops / ms / 1e9);
  }
  {
    int blocks = sms * 2, threads = 32 * 8;
    float ms = timeit([&] { k_mixed<8, 8><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); });
    double dm = 2.0 * 256 * 8 * (double)iters * blocks * 8;
    double df = 2.0 * 8 * (double)iters * blocks * threads;
    printf(", \"mixed_8dmma_8dfma_ms\": %.3f, \"mixed_dmma_tflops\": %.3f, \"mixed_total_tflops\": %.3f",
           ms, dm / ms / 1e9, (dm + df) / ms / 1e9);
    float ms2 = timeit([&] { k_dmma<8><<<blocks, threads>>>(out, iters, 1.0, 1.0); });
    printf(", \"dmma_only_same_shape_ms\": %.3f", ms2);
  }
  {
    int blocks = sms * 4, threads = 256; int it2 = 2000;
    float ms = timeit([&] { k_exp<<<blocks, threads>>>(out, it2, 0.1); });
    printf(", \"exp_f64_gops\": %.3f", (double)it2 * blocks * threads / ms / 1e6);
  }
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf(", \"clock_khz_attr\": %d}\n", clk);
  return 0;
}
