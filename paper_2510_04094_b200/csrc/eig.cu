// Landmark eigendecomposition on device: Omega = K(L, L), cyclic parallel
// Jacobi, descending sort, drop rule and W = V / sqrt(s).
// Replaces nystrom.build_feature_map (nystrom.py:136-160) and
// NystromFeatureMap._scaled_vectors (nystrom.py:120-121); LAPACK dsyevd in the
// reference.  Any symmetric eigensolver is parity-safe here (SURVEY.md §0,
// A1: <= 6.5e-8 on y_hat even when m_eff shifts), and the configs use sigma
// where the problem is eigensolver-insensitive (workloads.py).
//
// One CTA per landmark set, one-sided Jacobi (see the kernel comment).  U and
// V live in shared memory when 2*m^2*8 B fits (m <= 112), otherwise in the
// caller's workspace (L2-resident).
#include <cmath>

#include "common.cuh"

namespace {

constexpr int kEigThreads = 1024;
constexpr int kMaxSweeps = 60;

// One-sided (Hestenes) Jacobi on U = Omega (symmetric): rotate column pairs
// until every pair is orthogonal to 1 ulp; V accumulates the rotations, so
// U = Omega V with orthogonal columns, i.e. u_i = lambda_i v_i.  lambda_i is
// read back as the Rayleigh quotient v_i . u_i (signed, absolute accuracy
// eps ||Omega||, like LAPACK dsyevd).  One warp per column pair, pairs of a
// round are disjoint (round-robin "circle" order), so a round needs a single
// __syncthreads.  U and V are column-major (conflict-free lane-per-row access).
__global__ void __launch_bounds__(kEigThreads, 1)
    hestenes_eig_kernel(const double* __restrict__ lm, int m, double sigma2, double drop_tol,
                        double* __restrict__ eigvals, double* __restrict__ eigvecs,
                        double* __restrict__ Wout, int* __restrict__ m_eff_out,
                        int* __restrict__ info, double* __restrict__ gU, double* __restrict__ gV,
                        int use_smem) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int degenerate;
  __shared__ double lam[512];
  __shared__ int order[512];

  double* U = use_smem ? reinterpret_cast<double*>(smem_raw) : gU;
  double* V = use_smem ? reinterpret_cast<double*>(smem_raw) + (size_t)m * m : gV;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = nt >> 5;

  if (tid == 0) degenerate = 0;
  __syncthreads();
  for (int e = tid; e < m * m; e += nt) {   // Omega symmetric: row- = column-major
    int i = e / m, j = e % m;
    double d = lm[i] - lm[j];
    U[e] = nys::rbf(d, sigma2);
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

  const int M = (m + 1) & ~1;
  const int half = M / 2;
  // ||Omega||_F^2 (warp 0) for the noise floor
  __shared__ double fro2_s;
  if (warp == 0) {
    double acc = 0.0;
    for (int e = lane; e < m * m; e += 32) acc = fma(U[e], U[e], acc);
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) fro2_s = acc;
  }
  __syncthreads();
  const double eps = 2.220446049250313e-16;
  const double tol_rel = sqrt((double)m) * eps;
  // noise floor: columns with |u| < m eps ||Omega||_F carry no direction information
  const double nf = (double)m * eps * sqrt(fro2_s);
  const double noise2 = (nf * nf) * (nf * nf);
  int sweeps = 0;
  for (int sweep = 0; sweep < kMaxSweeps; ++sweep) {
    int rotated = 0;
    ++sweeps;
    for (int r = 0; r < M - 1; ++r) {
      for (int k = warp; k < half; k += nwarps) {
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
        if (q >= m) continue;   // dummy player (odd m)
        double* up = U + (size_t)p * m;
        double* uq = U + (size_t)q * m;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int i = lane; i < m; i += 32) {
          double a = up[i], b = uq[i];
          al = fma(a, a, al);
          be = fma(b, b, be);
          ga = fma(a, b, ga);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        // LAPACK dgesvj-style stopping rule: columns orthogonal to sqrt(m) eps,
        // and pairs of noise-level columns (norm < eps ||Omega||_F) left alone
        if (fabs(ga) > tol_rel * sqrt(al * be) && al * be > noise2) {
          double zeta = (be - al) / (2.0 * ga);
          double t = fabs(zeta) > 1e150 ? 0.5 / zeta
                                        : copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          double c = 1.0 / sqrt(1.0 + t * t), s = t * c;
          double* vp = V + (size_t)p * m;
          double* vq = V + (size_t)q * m;
          for (int i = lane; i < m; i += 32) {
            double a = up[i], b = uq[i];
            up[i] = c * a - s * b;
            uq[i] = s * a + c * b;
            double x = vp[i], y = vq[i];
            vp[i] = c * x - s * y;
            vq[i] = s * x + c * y;
          }
          rotated = 1;
        }
      }
      __syncthreads();
    }
    if (!__syncthreads_or(rotated)) break;
  }

  // lambda_i = v_i . u_i
  for (int i = warp; i < m; i += nwarps) {
    double acc = 0.0;
    for (int r = lane; r < m; r += 32) acc = fma(V[(size_t)i * m + r], U[(size_t)i * m + r], acc);
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) lam[i] = acc;
  }
  __syncthreads();
  // descending order; ties: higher index first (argsort(...)[::-1] in nystrom.py:151)
  for (int i = tid; i < m; i += nt) {
    double di = lam[i];
    int rank = 0;
    for (int j = 0; j < m; ++j) {
      double dj = lam[j];
      rank += (dj > di) || (dj == di && j > i);
    }
    order[rank] = i;
  }
  __syncthreads();
  const double s0 = lam[order[0]];
  const double cut = fmax(drop_tol * s0, 0.0);
  for (int k = tid; k < m; k += nt) eigvals[k] = lam[order[k]];
  if (tid == 0) {
    int me = 0;
    while (me < m && lam[order[me]] > cut) ++me;
    *m_eff_out = me;
    *info = NYS_INFO_OK | (sweeps << 8);   // bits 8+: Jacobi sweeps (diagnostic)
  }
  for (int e = tid; e < m * m; e += nt) {
    int i = e / m, k = e % m;   // output row-major: row i, column k
    int src = order[k];
    double v = V[(size_t)src * m + i];
    eigvecs[e] = v;
    double sk = lam[src];
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
    cudaError_t e = cudaFuncSetAttribute(hestenes_eig_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (e != cudaSuccess) return nys_host::record_cuda(e);
  } else {
    if (workspace == nullptr || workspace_bytes < need) return NYS_EWORKSPACE;
    gA = static_cast<double*>(workspace);
    gV = gA + (size_t)m * m;
  }
  int threads = 32 * ((m + 1) / 2);   // one warp per column pair of a round
  if (threads > kEigThreads) threads = kEigThreads;
  if (threads < 64) threads = 64;
  hestenes_eig_kernel<<<1, threads, dyn, static_cast<cudaStream_t>(stream)>>>(
      landmarks, m, sigma2, drop_tol, eigvals, eigvecs, W, m_eff, info, gA, gV, use_smem);
  nys_host::count_launches(1);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}
