// Batched primal KKT assembly + direct solve.
// Block layout of linear.assemble (linear.py:123-133):
//     [ I/gamma + D^T D   D^T g    A_c^T ] [omega ]   [D^T r]
//     [ g^T D             g^T g    beta^T] [  b   ] = [g^T r]
//     [ A_c               beta     0     ] [lambda]   [  v  ]
// read from the dense extended Gram E = [D g r]^T [D g r], and linear.solve
// (linear.py:140-158): LU with partial pivoting (first maximal |a| wins, like
// LAPACK idamax), solve, one refinement step x += solve(M, rhs - M x), exact
// zero pivot -> SingularSystemError, non-finite x -> SingularSystemError.
//
// Small sides (n <= 96, configs 0-3): one warp per system, LU in shared memory,
// __syncwarp only; the pivot row is held in registers during the trailing
// update, four rows are updated per batch of loads (ILP), and the triangular
// sweeps are column-oriented (no per-row reductions).  The refinement residual
// re-reads M from E (M is symmetric, so lanes read rows of E coalesced).
// Large sides (config 4, n = 259): one CTA per system with an L2-resident
// workspace slice.
#include <cmath>

#include "batch_layout.cuh"
#include <cstdlib>

#include "common.cuh"

namespace nys_host {
int launch_kkt_chol_dense(const double* dense, int m_eff, int n_cond, const double* Ac,
                          const double* beta, const double* values, double gamma, int B,
                          double* x, int* info, cudaStream_t st);
int launch_kkt_big(const double* E, int m_eff, int n_cond, const double* Ac, const double* beta,
                   const double* values, double gamma, double* x, int* info, void* ws,
                   size_t ws_bytes, cudaStream_t st);
}  // namespace nys_host

namespace nys_host {
int launch_batch_unpack(const double* part, int nsplit, int B, int NB, int Pe, double* gram,
                        cudaStream_t st);
}

namespace {

// M[i][j] of linear.py:123-131 from E (row-major Pe x Pe)
NYS_DEV double m_entry(const double* E, int Pe, int i, int j, int me, double inv_gamma,
                       const double* Ac, const double* beta) {
  if (i <= me && j <= me) {
    double v = E[(size_t)i * Pe + j];
    return (i == j && i < me) ? inv_gamma + v : v;
  }
  if (i <= me) return i < me ? Ac[(size_t)(j - me - 1) * me + i] : beta[j - me - 1];
  if (j <= me) return j < me ? Ac[(size_t)(i - me - 1) * me + j] : beta[i - me - 1];
  return 0.0;
}

NYS_DEV double rhs_entry(const double* E, int Pe, int i, int me, const double* vals) {
  return i <= me ? E[(size_t)i * Pe + me + 1] : vals[i - me - 1];
}

constexpr int kWarpKktMaxN = 96;
constexpr int kNC = (kWarpKktMaxN + 31) / 32;

__global__ void __launch_bounds__(32)
    kkt_warp_kernel(const double* __restrict__ gram, int m_eff, int ncond,
                    const double* __restrict__ Ac, const double* __restrict__ beta,
                    const double* __restrict__ values, double gamma, int B,
                    double* __restrict__ xout, int* __restrict__ info, double* __restrict__ Mout,
                    double* __restrict__ rhsout, int only_flagged) {
  extern __shared__ __align__(16) double dsm[];
  const int lane = threadIdx.x;
  const int b = blockIdx.x;
  if (only_flagged && info[b] != 16 /* kNeedsLu */) return;
  const int n = m_eff + 1 + ncond, me = m_eff, Pe = m_eff + 2;
  const double* E = gram + (size_t)b * Pe * Pe;
  const double* vals = values + (size_t)b * ncond;
  double* LU = dsm;                 // n x n
  double* ys = LU + (size_t)n * n;  // n
  double* xs = ys + n;              // n
  int* perm = reinterpret_cast<int*>(xs + n);
  const double inv_gamma = 1.0 / gamma;

  // E block (rows/cols 0..me) in batches of 8 rows so 8 loads per lane are in flight
  for (int i0 = 0; i0 <= me; i0 += 8) {
    double v[8][kNC];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < kNC; ++c) {
        int i = i0 + r, j = lane + 32 * c;
        v[r][c] = (i <= me && j <= me) ? __ldg(E + (size_t)i * Pe + j) : 0.0;
      }
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < kNC; ++c) {
        int i = i0 + r, j = lane + 32 * c;
        if (i <= me && j <= me) LU[(size_t)i * n + j] = (i == j && i < me) ? inv_gamma + v[r][c] : v[r][c];
      }
  }
  // condition rows / columns (linear.py:127-130) and the zero block
  for (int mu = 0; mu < ncond; ++mu) {
    const int row = me + 1 + mu;
    for (int j = lane; j < n; j += 32) {
      double v = j < me ? Ac[(size_t)mu * me + j] : (j == me ? beta[mu] : 0.0);
      LU[(size_t)row * n + j] = v;
      if (j <= me) LU[(size_t)j * n + row] = v;
    }
  }
  __syncwarp();
  if (Mout)
    for (int e = lane; e < n * n; e += 32) Mout[(size_t)b * n * n + e] = LU[e];
  if (rhsout)
    for (int i = lane; i < n; i += 32) rhsout[(size_t)b * n + i] = rhs_entry(E, Pe, i, me, vals);
  __syncwarp();

  // ---------------- LU with partial pivoting
  int bad = 0;
  for (int k = 0; k < n; ++k) {
    double bv = -1.0;
    int bi = n;
#pragma unroll
    for (int c = 0; c < kNC; ++c) {
      int i = k + lane + 32 * c;
      if (i < n) {
        double a = fabs(LU[(size_t)i * n + k]);
        if (a > bv) {
          bv = a;
          bi = i;
        }
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (!(bv > 0.0)) {
      bad = 1;
      break;
    }
    if (lane == 0) perm[k] = bi;
    // swap rows k, bi and keep the (new) pivot row in registers
    double urow[kNC];
#pragma unroll
    for (int c = 0; c < kNC; ++c) {
      int j = lane + 32 * c;
      double u = 0.0;
      if (j < n) {
        double a = LU[(size_t)k * n + j], p = LU[(size_t)bi * n + j];
        if (bi != k) LU[(size_t)bi * n + j] = a;
        LU[(size_t)k * n + j] = p;
        u = p;
      }
      urow[c] = u;
    }
    __syncwarp();
    const double pivot = LU[(size_t)k * n + k];
#pragma unroll
    for (int c = 0; c < kNC; ++c) {
      int i = k + 1 + lane + 32 * c;
      if (i < n) LU[(size_t)i * n + k] /= pivot;
    }
    __syncwarp();
    // trailing update A[i][j] -= l_i u_j, i, j > k; 4 rows per batch of loads
    int i = k + 1;
    for (; i + 3 < n; i += 4) {
      double l[4], a[4][kNC];
#pragma unroll
      for (int r = 0; r < 4; ++r) l[r] = LU[(size_t)(i + r) * n + k];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < kNC; ++c) {
          int j = lane + 32 * c;
          a[r][c] = (j > k && j < n) ? LU[(size_t)(i + r) * n + j] : 0.0;
        }
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < kNC; ++c) {
          int j = lane + 32 * c;
          if (j > k && j < n) LU[(size_t)(i + r) * n + j] = a[r][c] - l[r] * urow[c];
        }
    }
    for (; i < n; ++i) {
      double l = LU[(size_t)i * n + k];
#pragma unroll
      for (int c = 0; c < kNC; ++c) {
        int j = lane + 32 * c;
        if (j > k && j < n) LU[(size_t)i * n + j] -= l * urow[c];
      }
    }
    __syncwarp();
  }
  if (bad) {
    if (lane == 0) info[b] = NYS_INFO_SINGULAR;
    for (int i = lane; i < n; i += 32) xout[(size_t)b * n + i] = NAN;
    return;
  }

  // ---------------- solve + one refinement step (linear.py:144-147)
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 0) {
      for (int i = lane; i < n; i += 32) ys[i] = rhs_entry(E, Pe, i, me, vals);
    } else {
      // ys = rhs - M x ; M symmetric: column i of M = row i of M (coalesced rows of E)
      double acc[kNC];
#pragma unroll
      for (int c = 0; c < kNC; ++c) acc[c] = 0.0;
      for (int j0 = 0; j0 <= me; j0 += 8) {
        double v[8][kNC], xj[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          int j = j0 + r;
          xj[r] = j <= me ? xs[j] : 0.0;
#pragma unroll
          for (int c = 0; c < kNC; ++c) {
            int i = lane + 32 * c;
            v[r][c] = (j <= me && i <= me) ? __ldg(E + (size_t)j * Pe + i) : 0.0;
          }
        }
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int c = 0; c < kNC; ++c) {
            int i = lane + 32 * c, j = j0 + r;
            double mv = (i == j && i < me) ? inv_gamma + v[r][c] : v[r][c];
            acc[c] += mv * xj[r];
          }
      }
      // condition couplings: rows/cols me+1.. of M
#pragma unroll
      for (int c = 0; c < kNC; ++c) {
        int i = lane + 32 * c;
        if (i < n) {
          if (i <= me) {
            for (int mu = 0; mu < ncond; ++mu)
              acc[c] += (i < me ? Ac[(size_t)mu * me + i] : beta[mu]) * xs[me + 1 + mu];
          } else {
            const int mu = i - me - 1;
            double a2 = 0.0;
            for (int j = 0; j < me; ++j) a2 += Ac[(size_t)mu * me + j] * xs[j];
            acc[c] = a2 + beta[mu] * xs[me];
          }
        }
      }
#pragma unroll
      for (int c = 0; c < kNC; ++c) {
        int i = lane + 32 * c;
        if (i < n) ys[i] = rhs_entry(E, Pe, i, me, vals) - acc[c];
      }
    }
    __syncwarp();
    if (lane == 0)
      for (int k = 0; k < n; ++k) {
        int pr = perm[k];
        if (pr != k) {
          double t = ys[k];
          ys[k] = ys[pr];
          ys[pr] = t;
        }
      }
    __syncwarp();
    // L y = P rhs, column-oriented
    for (int j = 0; j < n - 1; ++j) {
      const double yj = ys[j];
#pragma unroll
      for (int c = 0; c < kNC; ++c) {
        int i = j + 1 + lane + 32 * c;
        if (i < n) ys[i] -= LU[(size_t)i * n + j] * yj;
      }
      __syncwarp();
    }
    // U z = y, column-oriented
    for (int j = n - 1; j >= 0; --j) {
      const double zj = ys[j] / LU[(size_t)j * n + j];
      __syncwarp();
      if (lane == 0) ys[j] = zj;
#pragma unroll
      for (int c = 0; c < kNC; ++c) {
        int i = lane + 32 * c;
        if (i < j) ys[i] -= LU[(size_t)i * n + j] * zj;
      }
      __syncwarp();
    }
    for (int i = lane; i < n; i += 32) xs[i] = pass == 0 ? ys[i] : xs[i] + ys[i];
    __syncwarp();
  }
  int nonfinite = 0;
  for (int i = lane; i < n; i += 32) {
    double v = xs[i];
    if (!isfinite(v)) nonfinite = 1;
    xout[(size_t)b * n + i] = v;
  }
  nonfinite = __any_sync(0xffffffffu, nonfinite);
  if (lane == 0) info[b] = nonfinite ? NYS_INFO_NONFINITE : NYS_INFO_OK;
}

// ---------------------------------------------------------------------------
// large sides: one CTA per system, LU in an L2-resident workspace slice
constexpr int kKktThreads = 1024;   // large sides only (config 4: n = 259, B = 1)
constexpr int kCtaMaxN = 512;

__global__ void __launch_bounds__(kKktThreads)
    kkt_cta_kernel(const double* __restrict__ gram, int m_eff, int ncond,
                   const double* __restrict__ Ac, const double* __restrict__ beta,
                   const double* __restrict__ values, double gamma, int B,
                   double* __restrict__ xout, int* __restrict__ info, double* __restrict__ Mout,
                   double* __restrict__ rhsout, double* __restrict__ gws, int only_flagged) {
  if (only_flagged && info[blockIdx.x] != 16 /* kNeedsLu */) return;
  __shared__ int piv_s;
  __shared__ int bad;
  __shared__ double red_v[kKktThreads / 32];
  __shared__ double urow_s[kCtaMaxN], lcol_s[kCtaMaxN];
  __shared__ int red_i[kKktThreads / 32];
  extern __shared__ __align__(16) double vec[];   // ys | xs | perm  (3n)

  const int b = blockIdx.x;
  const int n = m_eff + 1 + ncond, me = m_eff, Pe = m_eff + 2;
  const double* E = gram + (size_t)b * Pe * Pe;
  const double* vals = values + (size_t)b * ncond;
  double* LU = gws + (size_t)b * n * n;
  double* ys = vec;
  double* xs = vec + n;
  int* perm = reinterpret_cast<int*>(vec + 2 * n);
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
  const double inv_gamma = 1.0 / gamma;

  for (int e = tid; e < n * n; e += nt) {
    int i = e / n, j = e % n;
    double v = m_entry(E, Pe, i, j, me, inv_gamma, Ac, beta);
    LU[e] = v;
    if (Mout) Mout[(size_t)b * n * n + e] = v;
  }
  if (rhsout)
    for (int i = tid; i < n; i += nt) rhsout[(size_t)b * n + i] = rhs_entry(E, Pe, i, me, vals);
  if (tid == 0) bad = 0;
  __syncthreads();

  for (int k = 0; k < n; ++k) {
    double bv = -1.0;
    int bi = n;
    for (int i = k + tid; i < n; i += nt) {
      double a = fabs(LU[(size_t)i * n + k]);
      if (a > bv) {
        bv = a;
        bi = i;
      }
    }
    for (int o = 16; o; o >>= 1) {
      double ov = __shfl_down_sync(0xffffffffu, bv, o);
      int oi = __shfl_down_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (lane == 0) {
      red_v[wid] = bv;
      red_i[wid] = bi;
    }
    __syncthreads();
    if (tid == 0) {
      double v = red_v[0];
      int ix = red_i[0];
      for (int w = 1; w < nt / 32; ++w)
        if (red_v[w] > v || (red_v[w] == v && red_i[w] < ix)) {
          v = red_v[w];
          ix = red_i[w];
        }
      piv_s = ix;
      perm[k] = ix;
      if (!(v > 0.0)) bad = 1;
    }
    __syncthreads();
    if (bad) break;
    const int pr = piv_s;
    // swap rows k, pr and stage the pivot row in shared memory
    for (int j = tid; j < n; j += nt) {
      const double a = LU[(size_t)k * n + j], p = LU[(size_t)pr * n + j];
      if (pr != k) LU[(size_t)pr * n + j] = a;
      LU[(size_t)k * n + j] = p;
      urow_s[j] = p;
    }
    __syncthreads();
    const double inv = 1.0 / urow_s[k];
    for (int i = k + 1 + tid; i < n; i += nt) {   // multipliers, staged too
      const double l = LU[(size_t)i * n + k] * inv;
      LU[(size_t)i * n + k] = l;
      lcol_s[i] = l;
    }
    __syncthreads();
    // trailing update: warp per row, lanes over columns (coalesced, one load +
    // one store per element; l and u come from shared memory)
    for (int i = k + 1 + wid; i < n; i += nt / 32) {
      const double l = lcol_s[i];
      double* row = LU + (size_t)i * n;
      for (int j = k + 1 + lane; j < n; j += 32) row[j] -= l * urow_s[j];
    }
    __syncthreads();
  }
  if (bad) {
    if (tid == 0) info[b] = NYS_INFO_SINGULAR;
    for (int i = tid; i < n; i += nt) xout[(size_t)b * n + i] = NAN;
    return;
  }
  for (int pass = 0; pass < 2; ++pass) {
    for (int i = tid; i < n; i += nt) {
      double v = rhs_entry(E, Pe, i, me, vals);
      if (pass == 1) {
        double acc = 0.0;
        for (int j = 0; j < n; ++j) acc += m_entry(E, Pe, j, i, me, inv_gamma, Ac, beta) * xs[j];
        v -= acc;
      }
      ys[i] = v;
    }
    __syncthreads();
    if (tid == 0)
      for (int k = 0; k < n; ++k) {
        int pr = perm[k];
        if (pr != k) {
          double t = ys[k];
          ys[k] = ys[pr];
          ys[pr] = t;
        }
      }
    __syncthreads();
    for (int j = 0; j < n - 1; ++j) {
      const double yj = ys[j];
      for (int i = j + 1 + tid; i < n; i += nt) ys[i] -= LU[(size_t)i * n + j] * yj;
      __syncthreads();
    }
    for (int j = n - 1; j >= 0; --j) {
      const double zj = ys[j] / LU[(size_t)j * n + j];
      __syncthreads();
      if (tid == 0) ys[j] = zj;
      for (int i = tid; i < j; i += nt) ys[i] -= LU[(size_t)i * n + j] * zj;
      __syncthreads();
    }
    for (int i = tid; i < n; i += nt) xs[i] = pass == 0 ? ys[i] : xs[i] + ys[i];
    __syncthreads();
  }
  int nonfinite = 0;
  for (int i = tid; i < n; i += nt) {
    double v = xs[i];
    if (!isfinite(v)) nonfinite = 1;
    xout[(size_t)b * n + i] = v;
  }
  nonfinite = __syncthreads_or(nonfinite);
  if (tid == 0) info[b] = nonfinite ? NYS_INFO_NONFINITE : NYS_INFO_OK;
}

}  // namespace

namespace nys_host {

int launch_kkt(const double* gram, int m_eff, int ncond, const double* Ac, const double* beta,
               const double* values, double gamma, int B, double* x, int* info, double* M,
               double* rhs, void* ws, size_t ws_bytes, cudaStream_t st,
               bool only_flagged = false) {
  const int n = m_eff + 1 + ncond;
  if (B == 1 && M == nullptr && rhs == nullptr && !only_flagged && n <= kWarpKktMaxN &&
      getenv("NYS_KKT_LU") == nullptr) {
    // single solve (SingleSolvePipeline): Cholesky of the SPD omega block + Schur
    // for bias and conditions (kkt_chol.cu, the batched solver's algorithm); the
    // LU below re-solves it only if the Cholesky broke down
    const int rc = launch_kkt_chol_dense(gram, m_eff, ncond, Ac, beta, values, gamma, B, x, info,
                                         st);
    if (rc == NYS_OK)
      return launch_kkt(gram, m_eff, ncond, Ac, beta, values, gamma, B, x, info, M, rhs, ws,
                        ws_bytes, st, true);
    if (rc != NYS_EUNSUPPORTED) return rc;
  }
  if (n <= kWarpKktMaxN) {
    size_t dyn = ((size_t)n * n + 3 * (size_t)n) * sizeof(double);
    if (dyn > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(kkt_warp_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
      if (e != cudaSuccess) return nys_host::record_cuda(e);
    }
    kkt_warp_kernel<<<B, 32, dyn, st>>>(gram, m_eff, ncond, Ac, beta, values, gamma, B, x, info, M,
                                        rhs, only_flagged ? 1 : 0);
    nys_host::count_launches(1);
    NYS_CHECK_LAUNCH();
    return NYS_OK;
  }
  size_t need = (size_t)B * n * n * sizeof(double);
  if (ws == nullptr || ws_bytes < need) return NYS_EWORKSPACE;
  if (B == 1 && M == nullptr && rhs == nullptr && !only_flagged &&
      getenv("NYS_KKT_LU") == nullptr) {
    // blocked Cholesky + Schur (kkt_big.cu); this LU re-solves it on breakdown
    const int rc = launch_kkt_big(gram, m_eff, ncond, Ac, beta, values, gamma, x, info, ws,
                                  ws_bytes, st);
    if (rc == NYS_OK) return launch_kkt(gram, m_eff, ncond, Ac, beta, values, gamma, B, x, info,
                                        M, rhs, ws, ws_bytes, st, true);
    if (rc != NYS_EUNSUPPORTED) return rc;
  }
  kkt_cta_kernel<<<B, kKktThreads, 3 * (size_t)n * sizeof(double), st>>>(
      gram, m_eff, ncond, Ac, beta, values, gamma, B, x, info, M, rhs, static_cast<double*>(ws),
      only_flagged ? 1 : 0);
  nys_host::count_launches(1);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

}  // namespace nys_host

extern "C" size_t nys_kkt_workspace_bytes(int m_eff, int n_cond, int B) {
  int n = m_eff + 1 + n_cond;
  return n <= kWarpKktMaxN ? 0 : (size_t)B * n * n * sizeof(double);
}

extern "C" int nys_kkt_solve_f64(const double* gram_ext, int m_eff, int n_cond, const double* Ac,
                                 const double* beta, const double* values, double gamma, int B,
                                 double* x, int* info, double* M, double* rhs, void* workspace,
                                 size_t workspace_bytes, void* stream) {
  if (m_eff < 1 || n_cond < 0 || B < 0 || !(gamma > 0.0)) return NYS_EINVAL;
  if (B == 0) return NYS_OK;
  return nys_host::launch_kkt(gram_ext, m_eff, n_cond, Ac, beta, values, gamma, B, x, info, M,
                              rhs, workspace, workspace_bytes, static_cast<cudaStream_t>(stream),
                              false);
}

