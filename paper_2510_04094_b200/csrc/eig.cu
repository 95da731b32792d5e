// Landmark eigendecomposition on device: Omega = K(L, L), cyclic parallel
// Jacobi, descending sort, drop rule and W = V / sqrt(s).
// Replaces nystrom.build_feature_map (nystrom.py:136-160) and
// NystromFeatureMap._scaled_vectors (nystrom.py:120-121); LAPACK dsyevd in the
// reference.  Any symmetric eigensolver is parity-safe here (SURVEY.md §0,
// A1: <= 6.5e-8 on y_hat even when m_eff shifts), and the configs use sigma
// where the problem is eigensolver-insensitive (workloads.py).
//
// One CTA per landmark set.  Round-robin ("circle") ordering gives m/2
// disjoint rotations per round; a round is (1) rotation parameters,
// (2) column update of A and V, (3) row update of A.  A and V live in shared
// memory when 2*m^2*8 B fits, otherwise in the caller's workspace (L2-resident).
#include <cmath>

#include "common.cuh"

namespace {

constexpr int kEigThreads = 1024;
constexpr int kMaxSweeps = 40;

struct Rot {
  int p, q;
  double c, s;
};

__global__ void __launch_bounds__(kEigThreads, 1)
    jacobi_eig_kernel(const double* __restrict__ lm, int m, double sigma2, double drop_tol,
                      double* __restrict__ eigvals, double* __restrict__ eigvecs,
                      double* __restrict__ Wout, int* __restrict__ m_eff_out,
                      int* __restrict__ info, double* __restrict__ gA, double* __restrict__ gV,
                      int use_smem) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // small bookkeeping lives in static shared memory
  __shared__ Rot rots[256];
  __shared__ int changed;
  __shared__ int degenerate;
  __shared__ double diag[512];
  __shared__ int order[512];

  const int M = (m + 1) & ~1;   // even player count; index m (if m odd) is a dummy
  double* A = use_smem ? reinterpret_cast<double*>(smem_raw) : gA;
  double* V = use_smem ? reinterpret_cast<double*>(smem_raw) + (size_t)m * m : gV;
  const int tid = threadIdx.x, nt = blockDim.x;

  if (tid == 0) degenerate = 0;
  __syncthreads();
  // Omega and V = I; degenerate-landmark check (nystrom.py:145-146)
  for (int e = tid; e < m * m; e += nt) {
    int i = e / m, j = e % m;
    double d = lm[i] - lm[j];
    A[e] = nys::rbf(d, sigma2);
    V[e] = (i == j) ? 1.0 : 0.0;
    if (i != j && fabs(d) <= 1e-12) degenerate = 1;
  }
  __syncthreads();
  if (degenerate) {
    if (tid == 0) {
      *info = NYS_INFO_DEGENERATE;
      *m_eff_out = 0;
    }
    return;
  }

  const int half = M / 2;
  for (int sweep = 0; sweep < kMaxSweeps; ++sweep) {
    if (tid == 0) changed = 0;
    __syncthreads();
    for (int r = 0; r < M - 1; ++r) {
      // (1) rotation parameters for the m/2 disjoint pairs of round r
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
          double apq = A[p * m + q];
          double app = A[p * m + p], aqq = A[q * m + q];
          if (fabs(apq) > 1e-300 && fabs(apq) > 2.220446049250313e-16 * sqrt(fabs(app * aqq))) {
            double tau = (aqq - app) / (2.0 * apq);
            double t;
            if (fabs(tau) > 1e150)
              t = 0.5 / tau;
            else
              t = copysign(1.0, tau) / (fabs(tau) + sqrt(1.0 + tau * tau));
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
            changed = 1;
          }
        }
        rots[k] = Rot{p, q, c, s};
      }
      __syncthreads();
      // (2) column update A <- A J, V <- V J
      for (int e = tid; e < half * m; e += nt) {
        int k = e / m, i = e % m;
        Rot R = rots[k];
        if (R.s == 0.0) continue;
        double ap = A[i * m + R.p], aq = A[i * m + R.q];
        A[i * m + R.p] = R.c * ap - R.s * aq;
        A[i * m + R.q] = R.s * ap + R.c * aq;
        double vp = V[i * m + R.p], vq = V[i * m + R.q];
        V[i * m + R.p] = R.c * vp - R.s * vq;
        V[i * m + R.q] = R.s * vp + R.c * vq;
      }
      __syncthreads();
      // (3) row update A <- J^T A
      for (int e = tid; e < half * m; e += nt) {
        int k = e / m, j = e % m;
        Rot R = rots[k];
        if (R.s == 0.0) continue;
        double ap = A[R.p * m + j], aq = A[R.q * m + j];
        A[R.p * m + j] = R.c * ap - R.s * aq;
        A[R.q * m + j] = R.s * ap + R.c * aq;
      }
      __syncthreads();
      for (int k = tid; k < half; k += nt) {
        Rot R = rots[k];
        if (R.s != 0.0) {
          A[R.p * m + R.q] = 0.0;
          A[R.q * m + R.p] = 0.0;
        }
      }
      __syncthreads();
    }
    if (!changed) break;
    __syncthreads();
  }

  // sort descending (stable on index, like argsort(...)[::-1] up to ties)
  for (int i = tid; i < m; i += nt) diag[i] = A[i * m + i];
  __syncthreads();
  for (int i = tid; i < m; i += nt) {
    double di = diag[i];
    int rank = 0;
    for (int j = 0; j < m; ++j) {
      double dj = diag[j];
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
    *info = NYS_INFO_OK;
  }
  for (int e = tid; e < m * m; e += nt) {
    int i = e / m, k = e % m;
    int src = order[k];
    double v = V[i * m + src];
    eigvecs[e] = v;
    double sk = diag[src];
    Wout[e] = (sk > cut) ? v / sqrt(sk) : 0.0;
  }
}

}  // namespace

extern "C" size_t nys_landmark_eig_workspace_bytes(int m) {
  if (m <= 0) return 0;
  size_t need = 2 * (size_t)m * m * sizeof(double);
  return need <= 200 * 1024 ? 0 : need;
}

extern "C" int nys_landmark_eig_f64(const double* landmarks, int m, double sigma2,
                                    double drop_tol, double* eigvals, double* eigvecs,
                                    double* W, int* m_eff, int* info, void* workspace,
                                    size_t workspace_bytes, void* stream) {
  if (m < 1 || m > 512 || !(sigma2 > 0.0) || !(drop_tol >= 0.0 && drop_tol < 1.0))
    return NYS_EINVAL;
  size_t need = 2 * (size_t)m * m * sizeof(double);
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
    gV = gA + (size_t)m * m;
  }
  int threads = m <= 32 ? 256 : kEigThreads;
  jacobi_eig_kernel<<<1, threads, dyn, static_cast<cudaStream_t>(stream)>>>(
      landmarks, m, sigma2, drop_tol, eigvals, eigvecs, W, m_eff, info, gA, gV, use_smem);
  nys_host::count_launches(1);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}
