// Small landmark sets (m <= 112, everything in shared memory): two-sided
// cyclic Jacobi for Omega = K(L, L), then the same sort / drop / W epilogue as
// the tridiagonal QL path (eig.cu).
//
// B200's FP64 latency makes the rotation-parameter chain (two divisions, a
// square root and a reciprocal square root) the critical path of every round.
// The ANGLE is therefore computed in FP32 (MUFU-fast), while the rotation
// itself is made orthogonal to FP64 precision (c = rsqrt(1 + t^2), s = t c, in
// FP64): the similarity is exact, only a_pq is not annihilated exactly -- it
// drops by ~1e-7 per rotation instead of to 0, which costs about one extra
// sweep and halves the round latency.  Round-robin ordering: m/2 disjoint
// rotations per round, 8 threads per rotation, two barriers per round.
// Stopping rule: no |a_pq| above eps ||Omega||_F in a sweep (LAPACK-level
// backward error).
#include <cmath>

#include "common.cuh"

namespace {

constexpr int kJThreads = 512;
constexpr int kTPP = 8;          // threads per rotation pair (one quarter warp)
constexpr int kMaxSweeps = 60;
template <int kRows>   // rows (columns) per thread per phase: ceil(m / kTPP)
__global__ void __launch_bounds__(kJThreads, 1)
    jacobi_small_kernel(const double* __restrict__ lm, int m, double sigma2, double drop_tol,
                        double* __restrict__ eigvals, double* __restrict__ eigvecs,
                        double* __restrict__ Wout, int* __restrict__ m_eff_out,
                        int* __restrict__ info) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double diag[128];
  __shared__ int order[128];
  __shared__ double parts[kJThreads / 32];
  __shared__ int degenerate;
  const int lda = m + 1;
  double* A = sm;                        // m x lda
  double* VT = sm + (size_t)m * lda;     // m x m, row p = eigenvector p
  const int tid = threadIdx.x, nt = blockDim.x;

  if (tid == 0) degenerate = 0;
  __syncthreads();
  double fro = 0.0;
  for (int e = tid; e < m * m; e += nt) {
    const int i = e / m, j = e % m;
    const double d = lm[i] - lm[j];
    const double v = nys::rbf(d, sigma2);
    A[(size_t)i * lda + j] = v;
    VT[e] = (i == j) ? 1.0 : 0.0;
    fro = fma(v, v, fro);
    if (i != j && fabs(d) <= 1e-12) degenerate = 1;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) fro += __shfl_xor_sync(0xffffffffu, fro, o);
  if ((tid & 31) == 0) parts[tid >> 5] = fro;
  __syncthreads();
  if (degenerate) {
    if (tid == 0) {
      *info = NYS_INFO_DEGENERATE;
      *m_eff_out = 0;
    }
    return;
  }
  double fro2 = 0.0;
  for (int w = 0; w < nt / 32; ++w) fro2 += parts[w];   // fixed order: deterministic
  const double tol = 2.220446049250313e-16 * sqrt(fro2);

  const int M = (m + 1) & ~1, half = M / 2;
  const int grp = tid / kTPP, gl = tid % kTPP;
  int sweeps = 0;
  for (int sweep = 0; sweep < kMaxSweeps; ++sweep) {
    ++sweeps;
    int rotated = 0;
    for (int r = 0; r < M - 1; ++r) {
      int p = -1, q = -1;
      double c = 1.0, s = 0.0;
      const int k = grp;
      if (k < half) {
        if (k == 0) {
          p = M - 1;
          q = r;
        } else {
          p = r + k;
          if (p >= M - 1) p -= M - 1;
          q = r - k;
          if (q < 0) q += M - 1;
        }
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        if (q < m) {
          const double apq = A[(size_t)p * lda + q];
          if (fabs(apq) > tol) {
            const double app = A[(size_t)p * lda + p], aqq = A[(size_t)q * lda + q];
            // angle in FP32 (tan theta = y / (|x| + hypot(x, y)) sign(x)), scaled so
            // that tiny entries do not underflow
            const double sc = fmax(fabs(aqq - app), fabs(2.0 * apq));
            const float x = (float)((aqq - app) / sc), y = (float)(2.0 * apq / sc);
            const float rr = sqrtf(fmaf(x, x, y * y));
            float tf = __fdividef(y, fabsf(x) + rr);
            if (x < 0.0f) tf = -tf;
            const double t = (double)tf;
            c = rsqrt(fma(t, t, 1.0));   // exact orthogonality in FP64
            s = t * c;
            rotated = 1;
          }
        }
      }
      // all loads of a phase are issued before any store: the compiler cannot
      // prove the rows disjoint, so a load/compute/store loop would serialise on
      // shared-memory + FP64 latency (ncu: short_scoreboard dominated)
      if (s != 0.0) {   // A <- A J (columns p, q)
        double ap[kRows], aq[kRows];
#pragma unroll
        for (int u = 0; u < kRows; ++u) {
          const int i = gl + u * kTPP;
          ap[u] = i < m ? A[(size_t)i * lda + p] : 0.0;
          aq[u] = i < m ? A[(size_t)i * lda + q] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kRows; ++u) {
          const int i = gl + u * kTPP;
          if (i < m) {
            A[(size_t)i * lda + p] = c * ap[u] - s * aq[u];
            A[(size_t)i * lda + q] = s * ap[u] + c * aq[u];
          }
        }
      }
      __syncthreads();
      if (s != 0.0) {   // A <- J^T A, V^T <- J^T V^T (rows p, q)
        double* rp = A + (size_t)p * lda;
        double* rq = A + (size_t)q * lda;
        double* vp = VT + (size_t)p * m;
        double* vq = VT + (size_t)q * m;
        double ap[kRows], aq[kRows], xv[kRows], yv[kRows];
#pragma unroll
        for (int u = 0; u < kRows; ++u) {
          const int j = gl + u * kTPP;
          const bool ok = j < m;
          ap[u] = ok ? rp[j] : 0.0;
          aq[u] = ok ? rq[j] : 0.0;
          xv[u] = ok ? vp[j] : 0.0;
          yv[u] = ok ? vq[j] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kRows; ++u) {
          const int j = gl + u * kTPP;
          if (j < m) {
            rp[j] = c * ap[u] - s * aq[u];
            rq[j] = s * ap[u] + c * aq[u];
            vp[j] = c * xv[u] - s * yv[u];
            vq[j] = s * xv[u] + c * yv[u];
          }
        }
      }
      __syncthreads();
    }
    if (!__syncthreads_or(rotated)) break;
  }

  for (int i = tid; i < m; i += nt) diag[i] = A[(size_t)i * lda + i];
  __syncthreads();
  for (int i = tid; i < m; i += nt) {   // descending; ties: higher index first (nystrom.py:151)
    const double di = diag[i];
    int rank = 0;
    for (int j = 0; j < m; ++j) {
      const double dj = diag[j];
      rank += (dj > di) || (dj == di && j > i);
    }
    order[rank] = i;
  }
  __syncthreads();
  const double s0 = diag[order[0]];
  const double cut = fmax(drop_tol * s0, 0.0);
  for (int k = tid; k < m; k += nt) eigvals[k] = diag[order[k]];
  if (tid == 0) {
    int me = 0;
    while (me < m && diag[order[me]] > cut) ++me;
    *m_eff_out = me;
    *info = NYS_INFO_OK | (sweeps << 8);   // bits 8+: sweeps (diagnostic)
  }
  for (int e = tid; e < m * m; e += nt) {
    const int i = e / m, k = e % m;
    const int src = order[k];
    const double v = VT[(size_t)src * m + i];
    eigvecs[e] = v;
    const double sk = diag[src];
    Wout[e] = (sk > cut) ? v / sqrt(sk) : 0.0;
  }
}

}  // namespace

namespace nys_host {
bool jacobi_small_fits(int m) {
  return m <= 112 && (2 * (size_t)m * (m + 1) * sizeof(double)) <= 200 * 1024;
}

int launch_jacobi_small(const double* lm, int m, double sigma2, double drop_tol, double* eigvals,
                        double* eigvecs, double* W, int* m_eff, int* info, cudaStream_t st) {
  const size_t dyn = 2 * (size_t)m * (m + 1) * sizeof(double);
  const int rows = (m + kTPP - 1) / kTPP;
  auto kern = rows <= 3 ? jacobi_small_kernel<3>
                        : (rows <= 6 ? jacobi_small_kernel<6>
                                     : (rows <= 8 ? jacobi_small_kernel<8> : jacobi_small_kernel<14>));
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  if (e != cudaSuccess) return record_cuda(e);
  int threads = ((m + 1) / 2) * kTPP;
  threads = (threads + 31) / 32 * 32;
  if (threads > kJThreads) threads = kJThreads;
  kern<<<1, threads, dyn, st>>>(lm, m, sigma2, drop_tol, eigvals, eigvecs, W, m_eff, info);
  count_launches(1);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}
}  // namespace nys_host
