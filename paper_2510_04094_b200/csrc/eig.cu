// Landmark eigendecomposition on device: Omega = K(L, L), cyclic parallel
// Jacobi, descending sort, drop rule and W = V / sqrt(s).
// Replaces nystrom.build_feature_map (nystrom.py:136-160) and
// NystromFeatureMap._scaled_vectors (nystrom.py:120-121); LAPACK dsyevd in the
// reference.  Any symmetric eigensolver is parity-safe here (SURVEY.md §0,
// A1: <= 6.5e-8 on y_hat even when m_eff shifts), and the configs use sigma
// where the problem is eigensolver-insensitive (workloads.py).
//
// One CTA per landmark set, two-sided Jacobi (see the kernel comment).  A and
// V^T live in shared memory when they fit (m <= 112), otherwise in the
// caller's workspace (L2-resident).
#include <cmath>

#include "common.cuh"

namespace {

constexpr int kEigThreads = 1024;
constexpr int kMaxSweeps = 60;
constexpr int kTPP = 8;                 // threads per rotation pair
constexpr int kMaxPairsPerGroup = 2;    // m <= 2 * (1024 / kTPP) * 2 = 512


// Two-sided cyclic Jacobi, round-robin ("circle") ordering: m/2 disjoint
// rotations per round, each round = (1) rotation parameters, (2) column update
// of A, (3) row update of A and of V^T (stored row-major, so both row updates
// are contiguous).  A uses an odd row stride (m+1) so the column update is
// bank-conflict free.  Stopping rule: a pair is rotated while |a_pq| exceeds
// eps ||A||_F (LAPACK-level backward error; a relative rule would chase the
// rounding noise of the ~1e-16 s_0 eigenvalues forever).
__global__ void __launch_bounds__(kEigThreads, 1)
    jacobi_eig_kernel(const double* __restrict__ lm, int m, double sigma2, double drop_tol,
                      double* __restrict__ eigvals, double* __restrict__ eigvecs,
                      double* __restrict__ Wout, int* __restrict__ m_eff_out,
                      int* __restrict__ info, double* __restrict__ gA, double* __restrict__ gV,
                      int use_smem) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int degenerate;
  __shared__ double diag[512];
  __shared__ int order[512];
  __shared__ double fro2_s;

  const int lda = m + 1;
  double* A = use_smem ? reinterpret_cast<double*>(smem_raw) : gA;                  // m x lda
  double* VT = use_smem ? reinterpret_cast<double*>(smem_raw) + (size_t)m * lda : gV; // m x m
  const int tid = threadIdx.x, nt = blockDim.x;

  if (tid == 0) {
    degenerate = 0;
    fro2_s = 0.0;
  }
  __syncthreads();
  double fro_local = 0.0;
  for (int e = tid; e < m * m; e += nt) {
    int i = e / m, j = e % m;
    double d = lm[i] - lm[j];
    double v = nys::rbf(d, sigma2);
    A[(size_t)i * lda + j] = v;
    VT[e] = (i == j) ? 1.0 : 0.0;
    fro_local = fma(v, v, fro_local);
    if (i != j && fabs(d) <= 1e-12) degenerate = 1;
  }
  for (int o = 16; o; o >>= 1) fro_local += __shfl_xor_sync(0xffffffffu, fro_local, o);
  __shared__ double fro_parts[kEigThreads / 32];
  if ((tid & 31) == 0) fro_parts[tid >> 5] = fro_local;
  __syncthreads();
  if (tid == 0) {   // fixed-order sum: the tolerance (and so the result) is deterministic
    double acc = 0.0;
    for (int w = 0; w < nt / 32; ++w) acc += fro_parts[w];
    fro2_s = acc;
  }
  __syncthreads();
  if (degenerate) {
    if (tid == 0) {
      *info = NYS_INFO_DEGENERATE;
      *m_eff_out = 0;
    }
    return;
  }
  const double tol = 2.220446049250313e-16 * sqrt(fro2_s);

  const int M = (m + 1) & ~1;
  const int half = M / 2;
  // kTPP threads own one pair: they compute its rotation redundantly (a pair's
  // parameters live in its own two columns, which no other pair of the round
  // touches, so no barrier is needed before the column update) and split its
  // rows/columns.  Two barriers per round.
  const int grp = tid / kTPP, gl = tid % kTPP, ngrp = nt / kTPP;
  int sweeps = 0;
  for (int sweep = 0; sweep < kMaxSweeps; ++sweep) {
    ++sweeps;
    int rotated = 0;
    for (int r = 0; r < M - 1; ++r) {
      int pp[kMaxPairsPerGroup], qq[kMaxPairsPerGroup];
      double cc[kMaxPairsPerGroup], ss[kMaxPairsPerGroup];
#pragma unroll
      for (int u = 0; u < kMaxPairsPerGroup; ++u) {
        const int k = grp + u * ngrp;
        int p = -1, q = -1;
        double c = 1.0, s = 0.0;
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
            int t = p;
            p = q;
            q = t;
          }
          if (q < m) {
            const double apq = A[(size_t)p * lda + q];
            if (fabs(apq) > tol) {
              const double app = A[(size_t)p * lda + p], aqq = A[(size_t)q * lda + q];
              const double tau = (aqq - app) / (2.0 * apq);
              const double t = fabs(tau) > 1e150
                                   ? 0.5 / tau
                                   : copysign(1.0, tau) / (fabs(tau) + sqrt(1.0 + tau * tau));
              c = rsqrt(1.0 + t * t);
              s = t * c;
              rotated = 1;
            }
          }
        }
        pp[u] = p;
        qq[u] = q;
        cc[u] = c;
        ss[u] = s;
      }
      // (2) A <- A J: columns p, q of every row
#pragma unroll
      for (int u = 0; u < kMaxPairsPerGroup; ++u) {
        if (ss[u] == 0.0) continue;
        for (int i = gl; i < m; i += kTPP) {
          double* row = A + (size_t)i * lda;
          const double ap = row[pp[u]], aq = row[qq[u]];
          row[pp[u]] = cc[u] * ap - ss[u] * aq;
          row[qq[u]] = ss[u] * ap + cc[u] * aq;
        }
      }
      __syncthreads();
      // (3) A <- J^T A, V^T <- J^T V^T: rows p, q
#pragma unroll
      for (int u = 0; u < kMaxPairsPerGroup; ++u) {
        if (ss[u] == 0.0) continue;
        double* rp = A + (size_t)pp[u] * lda;
        double* rq = A + (size_t)qq[u] * lda;
        double* vp = VT + (size_t)pp[u] * m;
        double* vq = VT + (size_t)qq[u] * m;
        for (int j = gl; j < m; j += kTPP) {
          const double ap = rp[j], aq = rq[j];
          rp[j] = cc[u] * ap - ss[u] * aq;
          rq[j] = ss[u] * ap + cc[u] * aq;
          const double x = vp[j], y = vq[j];
          vp[j] = cc[u] * x - ss[u] * y;
          vq[j] = ss[u] * x + cc[u] * y;
        }
      }
      __syncwarp();   // the kTPP threads of a group share a warp
#pragma unroll
      for (int u = 0; u < kMaxPairsPerGroup; ++u)
        if (ss[u] != 0.0 && gl == 0) {
          A[(size_t)pp[u] * lda + qq[u]] = 0.0;
          A[(size_t)qq[u] * lda + pp[u]] = 0.0;
        }
      __syncthreads();
    }
    if (!__syncthreads_or(rotated)) break;
  }

  for (int i = tid; i < m; i += nt) diag[i] = A[(size_t)i * lda + i];
  __syncthreads();
  // descending order; ties: higher index first (argsort(...)[::-1], nystrom.py:151)
  for (int i = tid; i < m; i += nt) {
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
    *info = NYS_INFO_OK | (sweeps << 8);   // bits 8+: Jacobi sweeps (diagnostic)
  }
  for (int e = tid; e < m * m; e += nt) {
    const int i = e / m, k = e % m;   // output row-major: row i, column k
    const int src = order[k];
    const double v = VT[(size_t)src * m + i];
    eigvecs[e] = v;
    const double sk = diag[src];
    Wout[e] = (sk > cut) ? v / sqrt(sk) : 0.0;
  }
}

}  // namespace

extern "C" size_t nys_landmark_eig_workspace_bytes(int m) {
  if (m <= 0) return 0;
  size_t need = (2 * (size_t)m * m + m) * sizeof(double);
  return need <= 200 * 1024 ? 0 : need;
}

extern "C" int nys_landmark_eig_f64(const double* landmarks, int m, double sigma2,
                                    double drop_tol, double* eigvals, double* eigvecs,
                                    double* W, int* m_eff, int* info, void* workspace,
                                    size_t workspace_bytes, void* stream) {
  if (m < 1 || m > 512 || !(sigma2 > 0.0) || !(drop_tol >= 0.0 && drop_tol < 1.0))
    return NYS_EINVAL;
  size_t need = (2 * (size_t)m * m + m) * sizeof(double);
  int use_smem = need <= 200 * 1024;
  double *gA = nullptr, *gV = nullptr;
  size_t dyn = 0;
  if (use_smem) {
    dyn = need;
    cudaError_t e = cudaFuncSetAttribute(jacobi_eig_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (e != cudaSuccess) return nys_host::record_cuda(e);
  } else {
    if (workspace == nullptr || workspace_bytes < need) return NYS_EWORKSPACE;
    gA = static_cast<double*>(workspace);
    gV = gA + (size_t)m * (m + 1);
  }
  int pairs = (m + 1) / 2;
  int threads = pairs * kTPP;
  if (threads > kEigThreads) threads = kEigThreads;   // groups then take 2 pairs each
  threads = (threads + 31) / 32 * 32;
  jacobi_eig_kernel<<<1, threads, dyn, static_cast<cudaStream_t>(stream)>>>(
      landmarks, m, sigma2, drop_tol, eigvals, eigvecs, W, m_eff, info, gA, gV, use_smem);
  nys_host::count_launches(1);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}
