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

struct Rot {
  int p, q;
  double c, s;
};

// Two-sided cyclic Jacobi, round-robin ("circle") ordering: m/2 disjoint
// rotations per round, each round = (1) rotation parameters, (2) column update
// of A, (3) row update of A and of V^T (stored row-major, so both row updates
// are contiguous).  A uses an odd row stride (m+1) so the column update is
// bank-conflict free.  Stopping rule: a pair is rotated while |a_pq| exceeds
// eps ||A||_F / m (LAPACK-level backward error; a relative rule would chase the
// rounding noise of the ~1e-16 s_0 eigenvalues forever).
__global__ void __launch_bounds__(kEigThreads, 1)
    jacobi_eig_kernel(const double* __restrict__ lm, int m, double sigma2, double drop_tol,
                      double* __restrict__ eigvals, double* __restrict__ eigvecs,
                      double* __restrict__ Wout, int* __restrict__ m_eff_out,
                      int* __restrict__ info, double* __restrict__ gA, double* __restrict__ gV,
                      int use_smem) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ Rot rots[256];
  __shared__ int changed;
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
  if ((tid & 31) == 0) atomicAdd(&fro2_s, fro_local);
  __syncthreads();
  if (degenerate) {
    if (tid == 0) {
      *info = NYS_INFO_DEGENERATE;
      *m_eff_out = 0;
    }
    return;
  }
  const double tol = 2.220446049250313e-16 * sqrt(fro2_s) / (double)m;

  const int M = (m + 1) & ~1;
  const int half = M / 2;
  int sweeps = 0;
  for (int sweep = 0; sweep < kMaxSweeps; ++sweep) {
    ++sweeps;
    if (tid == 0) changed = 0;
    __syncthreads();
    for (int r = 0; r < M - 1; ++r) {
      for (int k = tid; k < half; k += nt) {
        int p, q;
        if (k == 0) {
          p = M - 1;
          q = r;
        } else {
          p = (r + k) % (M - 1);
          q = (r - k + (M - 1)) % (M - 1);
        }
        if (p > q) {
          int t = p;
          p = q;
          q = t;
        }
        double c = 1.0, s = 0.0;
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
            changed = 1;
          }
        }
        rots[k] = Rot{p, q, c, s};
      }
      __syncthreads();
      // (2) A <- A J  (columns p, q of every row)
      for (int e = tid; e < half * m; e += nt) {
        const int k = e / m, i = e % m;
        const Rot R = rots[k];
        if (R.s == 0.0) continue;
        double* row = A + (size_t)i * lda;
        const double ap = row[R.p], aq = row[R.q];
        row[R.p] = R.c * ap - R.s * aq;
        row[R.q] = R.s * ap + R.c * aq;
      }
      __syncthreads();
      // (3) A <- J^T A and V^T <- J^T V^T  (rows p, q)
      for (int e = tid; e < half * m; e += nt) {
        const int k = e / m, j = e % m;
        const Rot R = rots[k];
        if (R.s == 0.0) continue;
        double* rp = A + (size_t)R.p * lda;
        double* rq = A + (size_t)R.q * lda;
        const double ap = rp[j], aq = rq[j];
        rp[j] = R.c * ap - R.s * aq;
        rq[j] = R.s * ap + R.c * aq;
        double* vp = VT + (size_t)R.p * m;
        double* vq = VT + (size_t)R.q * m;
        const double x = vp[j], y = vq[j];
        vp[j] = R.c * x - R.s * y;
        vq[j] = R.s * x + R.c * y;
      }
      __syncthreads();
      for (int k = tid; k < half; k += nt) {
        const Rot R = rots[k];
        if (R.s != 0.0) {
          A[(size_t)R.p * lda + R.q] = 0.0;
          A[(size_t)R.q * lda + R.p] = 0.0;
        }
      }
      __syncthreads();
    }
    if (!changed) break;
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
  int threads = m <= 64 ? 256 : (m <= 128 ? 512 : kEigThreads);
  jacobi_eig_kernel<<<1, threads, dyn, static_cast<cudaStream_t>(stream)>>>(
      landmarks, m, sigma2, drop_tol, eigvals, eigvecs, W, m_eff, info, gA, gV, use_smem);
  nys_host::count_launches(1);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}
