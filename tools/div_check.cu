// Checks that the 3-op reciprocal division used by gram_large.cu (neg_div)
// is bit-identical to the IEEE quotient -(x / sigma2) (kernel.py:78-79) over
// many random x (d*d for d spread over many binades) and several bandwidths.
#include <cstdio>
#include <cstdint>
#include <cmath>

__device__ __forceinline__ double neg_div(double x, double s, double inv) {
  double q = x * inv;
  double r = fma(-q, s, x);
  return -fma(r, inv, q);
}

__global__ void check(double s, unsigned long long n, unsigned long long seed,
                      unsigned long long* bad, double* example) {
  const double inv = 1.0 / s;
  unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  unsigned long long local = 0;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += stride) {
    unsigned long long z = (i + seed) * 0x9E3779B97F4A7C15ull;
    z ^= z >> 31; z *= 0xBF58476D1CE4E5B9ull; z ^= z >> 27; z *= 0x94D049BB133111EBull; z ^= z >> 31;
    // d in [-8, 8] with a random binade scale down to 2^-30
    double u = (double)(z >> 11) * 0x1.0p-53;
    int e = (int)((z >> 3) & 31);
    double d = (2.0 * u - 1.0) * 8.0 * ldexp(1.0, -e);
    double x = d * d;
    double a = -(x / s);
    double b = neg_div(x, s, inv);
    if (__double_as_longlong(a) != __double_as_longlong(b)) {
      ++local;
      example[0] = x;
    }
  }
  if (local) atomicAdd(bad, local);
}

int main() {
  const double sig[] = {0.25, 0.01, 0.16, 1e-4, 0.0123456789, 3.7, 0.5 * 0.5, 0.4 * 0.4, 0.1 * 0.1,
                        0.3 * 0.3, 0.7 * 0.7, 2.0, 1.0 / 3.0};
  unsigned long long *bad;
  double* ex;
  cudaMallocManaged(&bad, 8);
  cudaMallocManaged(&ex, 8);
  int total_bad = 0;
  for (double s : sig) {
    *bad = 0;
    check<<<148 * 8, 256>>>(s, 1ull << 32, (unsigned long long)(s * 1e9), bad, ex);
    cudaDeviceSynchronize();
    printf("sigma2=%.17g samples=2^32 mismatches=%llu%s\n", s, *bad, *bad ? "  <-- " : "");
    if (*bad) { printf("  example x=%.17g\n", ex[0]); total_bad++; }
  }
  printf(total_bad ? "DIV_CHECK FAIL\n" : "DIV_CHECK OK\n");
  return total_bad ? 1 : 0;
}
