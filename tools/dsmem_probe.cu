// DSMEM / exchange latency probe: a cluster of 8 CTAs (512 threads) runs K
// rounds of (warp 0: q-loop over shared rows + st.async push of 32 values to
// all 8 CTAs + slot push; exchange wait) and reports cycles per round for
// variants: 0 = full, 1 = no q-loop, 2 = no pushes (local only, no wait),
// 3 = pushes + wait only (no q-loop, no reduce).
#include <cstdio>
#include <cstdint>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, int r) { uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o; }

__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(512, 1) probe(int variant, int K, long long* out) {
  __shared__ double V[128 * 17], W[128 * 17];
  __shared__ double slot[2][8];
  __shared__ uint64_t bar[2];
  cg::cluster_group cl = cg::this_cluster();
  const int rk = cl.block_rank(), tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < 128 * 17; e += 512) { V[e] = 1e-3 * (e % 7); W[e] = 1e-3 * (e % 5); }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cl.sync();
  int xe = 0;
  long long t0 = clock64();
  double acc = 0.0;
  for (int k = 0; k < K; ++k) {
    const int jj = 15, prow = rk * 16;
    const bool local = variant == 2 || variant >= 4;
    const uint32_t bytes = 8u * (256 + 8);
    if (tid == 0 && !local)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(&bar[xe & 1])), "r"(bytes) : "memory");
    if (warp == 0) {
      double c = 1.0 + acc;
      if (variant != 1 && variant != 3 && variant != 4 && variant != 5) {
        const double* Vi = V + (prow + (lane & 15)) * 17; const double* Wi = W + (prow + (lane & 15)) * 17;
        const double* Vj = V + 37 * 17; const double* Wj = W + 37 * 17;
        double c1 = 0, c2 = 0, c3 = 0, c4 = 0;
#pragma unroll
        for (int q = 0; q < 16; q += 2) {
          if (q < jj) { c1 = fma(Vi[q], Wj[q], c1); c2 = fma(Wi[q], Vj[q], c2); }
          if (q + 1 < jj) { c3 = fma(Vi[q + 1], Wj[q + 1], c3); c4 = fma(Wi[q + 1], Vj[q + 1], c4); }
        }
        c = c - ((c1 + c3) + (c2 + c4));
      }
      if (!local) {
        const uint32_t la = su32(V + (prow + (lane & 15)) * 17 + (k & 15)), lb = su32(&bar[xe & 1]);
#pragma unroll
        for (int r = 0; r < 8; ++r)
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" :: "r"(mapa(la, r)), "d"(c), "r"(mapa(lb, r)) : "memory");
      }
      double part = c * c;
      if (variant != 3 && variant != 4 && variant != 6)
        for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      if (lane == 0 && !local) {
        const uint32_t la = su32(&slot[xe & 1][rk]), lb = su32(&bar[xe & 1]);
#pragma unroll
        for (int r = 0; r < 8; ++r)
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" :: "r"(mapa(la, r)), "d"(part), "r"(mapa(lb, r)) : "memory");
      }
      acc += part * 1e-30;
    }
    if (!local) {
      if (tid == 0) {
        const uint32_t b = su32(&bar[xe & 1]), par = (xe >> 1) & 1;
        asm volatile("{ .reg .pred p; W_%=: mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1; @!p bra W_%=; }" :: "r"(b), "r"(par) : "memory");
      }
      ++xe;
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0 && rk == 0) out[variant] = (t1 - t0) / K;
  if (acc == 12345.0) out[15] = 1;
  cl.sync();
}

int main() {
  long long* d; cudaMalloc(&d, 16 * sizeof(long long));
  const char* names[] = {"full (q-loop + push + reduce + wait)", "no q-loop", "no push/wait (local)", "push + wait only",
                         "syncthreads only", "reduce + syncthreads", "q-loop + syncthreads"};
  for (int v = 0; v < 7; ++v) {
    probe<<<8, 512>>>(v, 2000, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[16]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("variant %d %-40s %lld cycles/round  (%s)\n", v, names[v], h[v], cudaGetErrorString(e));
  }
  return 0;
}
