// Landmark eigendecomposition on device: Omega = K(L, L) -> Householder
// tridiagonalisation -> implicit QL with Wilkinson-type shifts -> descending
// sort, drop rule and W = V / sqrt(s).
// Replaces nystrom.build_feature_map (nystrom.py:136-160) and
// NystromFeatureMap._scaled_vectors (nystrom.py:120-121); the reference calls
// LAPACK dsyevd (tridiagonal + divide and conquer).  This is the tridiagonal +
// QL route of LAPACK dsyev: backward error ~eps ||Omega||, like the reference.
// Any accurate symmetric eigensolver is parity-safe.
//
// One CTA per landmark set.
//   phase 1  A <- Q^T A Q, tridiagonal (d, e); Householder vectors kept in A
//   phase 2  Z^T = Q^T accumulated backwards
//   phase 3  QL: one thread generates each sweep's Givens rotations (serial by
//            nature); all threads apply the sweep to their row of Z (column-major
//            Z^T, so a sweep streams down contiguous rows: conflict-free)
//   phase 4  sort, drop, W
// A and Z^T live in shared memory when they fit (m <= 112), otherwise in the
// caller's workspace (L2-resident, config 4: m = 256).
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace nys_host {
size_t dc_buffer_bytes(int n);
bool dc_fits(int n);
bool dc_uses_smem(int n);
int launch_dc_eig(const double* lm, const double* Ain, int n, double sigma2, double drop_tol,
                  double* eigvals, double* eigvecs, double* W, int* m_eff, int* info, void* ws,
                  size_t ws_bytes, cudaStream_t st);
bool jacobi_small_fits(int m);
int launch_jacobi_small(const double* lm, int m, double sigma2, double drop_tol, double* eigvals,
                        double* eigvecs, double* W, int* m_eff, int* info, cudaStream_t st);
}  // namespace nys_host

namespace {

constexpr int kEigThreads = 1024;
constexpr int kMaxM = 512;
constexpr int kMaxQlIters = 60;   // per eigenvalue

struct Shared {
  double d[kMaxM], e[kMaxM], beta[kMaxM], v[kMaxM], p[kMaxM];
  double rc[kMaxM], rs[kMaxM];
  int order[kMaxM];
  double red[kEigThreads / 32];
  int ibcast[4];
  int degenerate;
};

NYS_DEV double block_sum(double x, Shared& S) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  __syncthreads();
  if (lane == 0) S.red[w] = x;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < nw; ++i) s += S.red[i];   // fixed order: deterministic
  return s;
}

__global__ void __launch_bounds__(kEigThreads, 1)
    tql_eig_kernel(const double* __restrict__ lm, int m, double sigma2, double drop_tol,
                   double* __restrict__ eigvals, double* __restrict__ eigvecs,
                   double* __restrict__ Wout, int* __restrict__ m_eff_out, int* __restrict__ info,
                   double* __restrict__ gA, double* __restrict__ gZ, int use_smem, int debug) {
  long long t_start = clock64(), t1 = 0, t2 = 0, t3 = 0;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ Shared S;
  const int ld = m + 1;
  double* A = use_smem ? reinterpret_cast<double*>(smem_raw) : gA;                   // m x ld
  double* ZT = use_smem ? reinterpret_cast<double*>(smem_raw) + (size_t)m * ld : gZ;  // m x ld
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;

  if (tid == 0) S.degenerate = 0;
  __syncthreads();
  for (int e = tid; e < m * m; e += nt) {
    const int i = e / m, j = e % m;
    const double d = lm[i] - lm[j];
    A[(size_t)i * ld + j] = nys::rbf(d, sigma2);   // (Omega + Omega^T)/2 == Omega exactly
    if (i != j && fabs(d) <= 1e-12) S.degenerate = 1;
  }
  __syncthreads();
  if (S.degenerate) {
    if (tid == 0) {
      *info = NYS_INFO_DEGENERATE;
      *m_eff_out = 0;
    }
    return;
  }

  // ---------------- phase 1: Householder tridiagonalisation
  for (int k = 0; k + 2 < m; ++k) {
    const int i0 = k + 1;
    double tail = 0.0;
    for (int i = i0 + tid; i < m; i += nt) {
      const double x = A[(size_t)i * ld + k];
      S.v[i] = x;
      if (i != i0) tail = fma(x, x, tail);
    }
    tail = block_sum(tail, S);
    if (tid == 0) {
      const double x0 = S.v[i0];
      double beta = 0.0, alpha = x0;
      if (tail > 0.0) {
        const double nx = sqrt(fma(x0, x0, tail));
        alpha = -copysign(nx, x0);
        const double v0 = x0 - alpha;
        beta = 2.0 / fma(v0, v0, tail);
        S.v[i0] = v0;
        A[(size_t)i0 * ld + k] = v0;
      }
      S.e[k] = alpha;
      S.beta[k] = beta;
    }
    __syncthreads();
    const double beta = S.beta[k];
    if (beta == 0.0) continue;
    // p = beta S v: thread per row, four independent accumulators (FP64 FMA
    // latency, not throughput, bounds a serial dot product)
    for (int i = i0 + tid; i < m; i += nt) {
      const double* row = A + (size_t)i * ld;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int j = i0;
      for (; j + 3 < m; j += 4) {
        a0 = fma(row[j], S.v[j], a0);
        a1 = fma(row[j + 1], S.v[j + 1], a1);
        a2 = fma(row[j + 2], S.v[j + 2], a2);
        a3 = fma(row[j + 3], S.v[j + 3], a3);
      }
      for (; j < m; ++j) a0 = fma(row[j], S.v[j], a0);
      S.p[i] = beta * ((a0 + a1) + (a2 + a3));
    }
    __syncthreads();
    double vp = 0.0;
    for (int i = i0 + tid; i < m; i += nt) vp = fma(S.v[i], S.p[i], vp);
    vp = block_sum(vp, S);
    const double K = 0.5 * beta * vp;
    for (int i = i0 + tid; i < m; i += nt) S.p[i] = S.p[i] - K * S.v[i];   // w
    __syncthreads();
    for (int i = i0 + warp; i < m; i += nw) {   // A -= v w^T + w v^T (warp per row)
      double* row = A + (size_t)i * ld;
      const double vi = S.v[i], wi = S.p[i];
      for (int j = i0 + lane; j < m; j += 32) row[j] = row[j] - vi * S.p[j] - wi * S.v[j];
    }
    __syncthreads();
  }
  t1 = clock64();
  for (int i = tid; i < m; i += nt) S.d[i] = A[(size_t)i * ld + i];
  if (tid == 0) {
    if (m >= 2) S.e[m - 2] = A[(size_t)(m - 1) * ld + (m - 2)];
    S.e[m - 1] = 0.0;
  }
  // ---------------- phase 2: Z^T = Q^T, Q = H_0 ... H_{m-3}
  for (int e = tid; e < m * m; e += nt) {
    const int i = e / m, j = e % m;
    ZT[(size_t)i * ld + j] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int k = m - 3; k >= 0; --k) {
    const double beta = S.beta[k];
    if (beta == 0.0) continue;
    const int i0 = k + 1;
    for (int i = i0 + tid; i < m; i += nt) S.v[i] = A[(size_t)i * ld + k];
    __syncthreads();
    // u_j = sum_i v_i Z[i][j] = sum_i ZT[j][i] v_i   (thread per j, 4 accumulators)
    for (int j = i0 + tid; j < m; j += nt) {
      const double* zr = ZT + (size_t)j * ld;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int i = i0;
      for (; i + 3 < m; i += 4) {
        a0 = fma(zr[i], S.v[i], a0);
        a1 = fma(zr[i + 1], S.v[i + 1], a1);
        a2 = fma(zr[i + 2], S.v[i + 2], a2);
        a3 = fma(zr[i + 3], S.v[i + 3], a3);
      }
      for (; i < m; ++i) a0 = fma(zr[i], S.v[i], a0);
      S.p[j] = beta * ((a0 + a1) + (a2 + a3));
    }
    __syncthreads();
    for (int j = i0 + warp; j < m; j += nw) {   // warp per row of Z^T
      double* zr = ZT + (size_t)j * ld;
      const double pj = S.p[j];
      for (int i = i0 + lane; i < m; i += 32) zr[i] -= pj * S.v[i];
    }
    __syncthreads();
  }

  t2 = clock64();
  // ---------------- phase 3: implicit QL on (d, e), rotations applied to Z
  const double eps = 2.220446049250313e-16;
  int l = 0, iters = 0, total_iters = 0;   // thread 0's state
  for (;;) {
    if (tid == 0) {
      int lo = -1, hi = -1;
      while (l < m) {
        int mm = l;
        for (; mm < m - 1; ++mm) {
          const double dd = fabs(S.d[mm]) + fabs(S.d[mm + 1]);
          if (fabs(S.e[mm]) <= eps * dd) break;
        }
        if (mm == l || iters >= kMaxQlIters) {
          ++l;
          iters = 0;
          continue;
        }
        ++iters;
        ++total_iters;
        double g = (S.d[l + 1] - S.d[l]) / (2.0 * S.e[l]);
        double r = hypot(g, 1.0);
        g = S.d[mm] - S.d[l] + S.e[l] / (g + copysign(r, g));
        double s = 1.0, c = 1.0, p = 0.0;
        int i = mm - 1;
        bool early = false;
        double ei = S.e[mm - 1], di1 = S.d[mm];
        for (; i >= l; --i) {
          // prefetch the next rotation's operands off the dependency chain
          const double ei_next = i > l ? S.e[i - 1] : 0.0;
          const double di = S.d[i];
          const double f = s * ei, b = c * ei;
          const double rr = fma(f, f, g * g);
          if (rr == 0.0) {
            S.e[i + 1] = 0.0;
            S.d[i + 1] -= p;
            S.e[mm] = 0.0;
            early = true;
            break;
          }
          // r = hypot(f, g), s = f / r, c = g / r with one reciprocal square
          // root instead of hypot + two divisions (shortens the serial chain;
          // |f|, |g| <= ||Omega|| here, so no over/underflow guard is needed)
          const double ir = rsqrt(rr);
          r = rr * ir;
          S.e[i + 1] = r;
          s = f * ir;
          c = g * ir;
          g = di1 - p;
          r = (di - g) * s + 2.0 * c * b;
          p = s * r;
          S.d[i + 1] = g + p;
          g = c * r - b;
          S.rc[i] = c;
          S.rs[i] = s;
          ei = ei_next;
          di1 = di;
        }
        if (!early) {
          S.d[l] -= p;
          S.e[l] = g;
          S.e[mm] = 0.0;
          lo = l;
        } else {
          lo = i + 1;
        }
        hi = mm;
        break;
      }
      S.ibcast[0] = lo;
      S.ibcast[1] = hi;
    }
    __syncthreads();
    const int lo = S.ibcast[0], hi = S.ibcast[1];
    if (lo < 0) break;
    if (lo < hi) {
      for (int k = tid; k < m; k += nt) {   // row k of Z, streamed down the sweep
        double f = ZT[(size_t)hi * ld + k];
        for (int i = hi - 1; i >= lo; --i) {
          const double zi = ZT[(size_t)i * ld + k];
          const double c = S.rc[i], s = S.rs[i];
          ZT[(size_t)(i + 1) * ld + k] = s * zi + c * f;
          f = c * zi - s * f;
        }
        ZT[(size_t)lo * ld + k] = f;
      }
    }
    __syncthreads();
  }

  t3 = clock64();
  if (debug && tid == 0)
    printf("[nys eig] m=%d tridiag=%lld accumQ=%lld ql=%lld cycles, ql_iters=%d\n", m, t1 - t_start,
           t2 - t1, t3 - t2, total_iters);
  // ---------------- phase 4: descending order (ties: higher index first, like
  // argsort(...)[::-1] in nystrom.py:151), drop rule, W
  for (int i = tid; i < m; i += nt) {
    const double di = S.d[i];
    int rank = 0;
    for (int j = 0; j < m; ++j) {
      const double dj = S.d[j];
      rank += (dj > di) || (dj == di && j > i);
    }
    S.order[rank] = i;
  }
  __syncthreads();
  const double s0 = S.d[S.order[0]];
  const double cut = fmax(drop_tol * s0, 0.0);
  for (int k = tid; k < m; k += nt) eigvals[k] = S.d[S.order[k]];
  if (tid == 0) {
    int me = 0;
    while (me < m && S.d[S.order[me]] > cut) ++me;
    *m_eff_out = me;
    if (total_iters > 65535) total_iters = 65535;
    *info = NYS_INFO_OK | (total_iters << 8);   // bits 8+: QL iterations (diagnostic)
  }
  for (int e = tid; e < m * m; e += nt) {
    const int i = e / m, k = e % m;   // row-major: row i, column k
    const int src = S.order[k];
    const double v = ZT[(size_t)src * ld + i];
    eigvecs[e] = v;
    const double sk = S.d[src];
    Wout[e] = (sk > cut) ? v / sqrt(sk) : 0.0;
  }
}

size_t eig_storage_bytes(int m) { return 2 * (size_t)m * (m + 1) * sizeof(double); }
constexpr size_t kEigSmemMax = 160 * 1024;   // + ~30 KB static bookkeeping

}  // namespace

extern "C" size_t nys_landmark_eig_workspace_bytes(int m) {
  if (m <= 0) return 0;
  size_t need = eig_storage_bytes(m);
  size_t ql = need <= kEigSmemMax ? 0 : need;
  size_t dc = nys_host::dc_fits(m) && !nys_host::dc_uses_smem(m) ? nys_host::dc_buffer_bytes(m) : 0;
  return ql > dc ? ql : dc;
}

extern "C" int nys_landmark_eig_f64(const double* landmarks, int m, double sigma2,
                                    double drop_tol, double* eigvals, double* eigvecs,
                                    double* W, int* m_eff, int* info, void* workspace,
                                    size_t workspace_bytes, void* stream) {
  if (m < 1 || m > kMaxM || !(sigma2 > 0.0) || !(drop_tol >= 0.0 && drop_tol < 1.0))
    return NYS_EINVAL;
  // small landmark sets: shared-memory Jacobi with FP32 angles (eig_jacobi.cu);
  // NYS_EIG_ALGO=ql forces the tridiagonal QL path (diagnostics / A-B tests)
  // (measured on B200: Jacobi wins at m = 20, 0.25 vs 0.32 ms; QL wins from
  // m = 50, 0.87 vs 1.05 ms, and at m = 64, 1.27 vs 1.50 ms)
  // default: divide and conquer (eig_dc.cu, m <= 256); NYS_EIG_ALGO = ql | jacobi
  // select the alternatives for diagnostics / A-B tests
  const char* algo = getenv("NYS_EIG_ALGO");
  const bool force_ql = algo && algo[0] == 'q', force_jac = algo && algo[0] == 'j';
  if (force_jac && nys_host::jacobi_small_fits(m))
    return nys_host::launch_jacobi_small(landmarks, m, sigma2, drop_tol, eigvals, eigvecs, W,
                                         m_eff, info, static_cast<cudaStream_t>(stream));
  if (!force_ql && !force_jac && nys_host::dc_fits(m))
    return nys_host::launch_dc_eig(landmarks, nullptr, m, sigma2, drop_tol, eigvals, eigvecs, W, m_eff,
                                   info, workspace, workspace_bytes,
                                   static_cast<cudaStream_t>(stream));
  const size_t need = eig_storage_bytes(m);
  const int use_smem = need <= kEigSmemMax;
  double *gA = nullptr, *gZ = nullptr;
  size_t dyn = 0;
  if (use_smem) {
    dyn = need;
    cudaError_t e = cudaFuncSetAttribute(tql_eig_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)dyn);
    if (e != cudaSuccess) return nys_host::record_cuda(e);
  } else {
    if (workspace == nullptr || workspace_bytes < need) return NYS_EWORKSPACE;
    gA = static_cast<double*>(workspace);
    gZ = gA + (size_t)m * (m + 1);
  }
  const int threads = m <= 64 ? 256 : (m <= 128 ? 512 : kEigThreads);
  tql_eig_kernel<<<1, threads, dyn, static_cast<cudaStream_t>(stream)>>>(
      landmarks, m, sigma2, drop_tol, eigvals, eigvecs, W, m_eff, info, gA, gZ, use_smem,
      getenv("NYS_EIG_DEBUG") != nullptr);
  nys_host::count_launches(1);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" size_t nys_sym_eig_workspace_bytes(int n) {
  if (!nys_host::dc_fits(n)) return 0;
  return nys_host::dc_uses_smem(n) ? 0 : nys_host::dc_buffer_bytes(n);
}

extern "C" int nys_sym_eig_f64(const double* A, int n, double drop_tol, double* eigvals,
                               double* eigvecs, double* W, int* m_eff, int* info, void* workspace,
                               size_t workspace_bytes, void* stream) {
  if (A == nullptr || !(drop_tol >= 0.0 && drop_tol < 1.0)) return NYS_EINVAL;
  if (!nys_host::dc_fits(n)) return NYS_EUNSUPPORTED;
  return nys_host::launch_dc_eig(nullptr, A, n, 1.0, drop_tol, eigvals, eigvecs, W, m_eff, info,
                                 workspace, workspace_bytes, static_cast<cudaStream_t>(stream));
}
