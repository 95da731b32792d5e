// Batched KKT solve for shared-grid batches (config 2): Cholesky of the SPD
// block + p x p Schur complement, LU fallback.
//
// M = [[H, C^T], [C, 0]] with H = [D g]^T [D g] + diag(I/gamma, 0) (linear.py:
// 123-131; SPD unless g lies in range(D)) and C = [A_c beta].  SURVEY.md §0/A1:
// Cholesky + Schur instead of the reference's LU moves y_hat by <= 5e-11.  It
// halves the flops, drops the pivot search and row swaps, and the packed lower
// triangle doubles the systems resident per SM.  A non-positive pivot (or a
// non-finite result) marks the instance kNeedsLu and the reference's LU
// (kkt.cu, warp kernel, only_flagged mode) re-solves it, so singular systems
// still raise SingularSystemError exactly as linear.py:148-153 does.
//
// FP64 latency, not throughput, bounds these tiny factorizations on B200, so
// every serial chain is division-free (reciprocal diagonal from one rsqrt per
// pivot), the trailing update keeps column k in registers and updates four
// rows per batch of loads, and one forward sweep serves [C^T | r] together.
#include <cmath>
#include <cstdlib>

#include "batch_layout.cuh"
#include "common.cuh"

namespace nys_host {
int launch_batch_unpack(const double* part, int nsplit, int B, int NB, int Pe, double* gram,
                        cudaStream_t st);
int launch_kkt(const double* gram, int m_eff, int ncond, const double* Ac, const double* beta,
               const double* values, double gamma, int B, double* x, int* info, double* M,
               double* rhs, void* ws, size_t ws_bytes, cudaStream_t st, bool only_flagged);
int launch_kkt_blocked(const double* dense, int m_eff, int n_cond, const double* Ac,
                       const double* beta, const double* values, double gamma, int B, double* x,
                       int* info, cudaStream_t st);
}  // namespace nys_host

namespace {

constexpr int kNeedsLu = 16;      // internal; kkt.cu's LU kernel clears it
constexpr int kMaxNh = 96;

NYS_DEV int pk(int i, int j) { return i * (i + 1) / 2 + j; }   // packed lower, j <= i

// kNC = ceil(nh / 32) column chunks per lane for whole rows; kNCU =
// ceil((nh - 1) / 32) for the trailing update (columns k+1..nh-1), so the
// config-2 side nh = 65 updates with two chunks instead of three
template <int P, int kNC, int kNCU>
__global__ void __launch_bounds__(32)
    kkt_chol_kernel(const double* __restrict__ gram, int m_eff, const double* __restrict__ Ac,
                    const double* __restrict__ beta, const double* __restrict__ values,
                    double gamma, double* __restrict__ xout, int* __restrict__ info) {
  extern __shared__ __align__(16) double dsm[];
  const int lane = threadIdx.x, b = blockIdx.x;
  const int nh = m_eff + 1, me = m_eff, Pe = m_eff + 2;
  constexpr int R = P + 1;                           // forward-sweep columns: C^T | r
  const double* E = gram + (size_t)b * Pe * Pe;
  const double* vals = values + (size_t)b * P;
  double* L = dsm;                                   // packed lower, nh(nh+1)/2
  double* dinv = L + (size_t)nh * (nh + 1) / 2;      // 1 / L_jj
  double* Y = dinv + nh;                             // nh x R: [L^-1 C^T | L^-1 r]
  double* xs = Y + (size_t)nh * R;                   // nh + P
  const double inv_gamma = 1.0 / gamma;

  // H (lower triangle) from E, 8 rows of loads in flight per lane
  for (int i0 = 0; i0 < nh; i0 += 8) {
    double v[8][kNC];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < kNC; ++c) {
        const int i = i0 + r, j = lane + 32 * c;
        v[r][c] = (i < nh && j <= i) ? __ldg(E + (size_t)i * Pe + j) : 0.0;
      }
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < kNC; ++c) {
        const int i = i0 + r, j = lane + 32 * c;
        if (i < nh && j <= i) L[pk(i, j)] = (i == j && i < me) ? inv_gamma + v[r][c] : v[r][c];
      }
  }
  __syncwarp();

  // ---- right-looking Cholesky H = L L^T
  int bad = 0;
  for (int k = 0; k < nh; ++k) {
    const double akk = L[pk(k, k)];
    if (!(akk > 0.0) || !isfinite(akk)) {
      bad = 1;
      break;
    }
    const double inv = rsqrt(akk);   // 1 / L_kk
    double colk[kNCU];                 // L[j][k] for j = k+1+lane+32c, kept in registers
#pragma unroll
    for (int c = 0; c < kNCU; ++c) {
      const int j = k + 1 + lane + 32 * c;
      colk[c] = j < nh ? L[pk(j, k)] * inv : 0.0;
    }
    __syncwarp();
    if (lane == 0) {
      L[pk(k, k)] = akk * inv;
      dinv[k] = inv;
    }
#pragma unroll
    for (int c = 0; c < kNCU; ++c) {
      const int j = k + 1 + lane + 32 * c;
      if (j < nh) L[pk(j, k)] = colk[c];
    }
    __syncwarp();
    // A[i][j] -= L[i][k] L[j][k], k < j <= i; column-owner lanes, 4 rows per batch
    int i = k + 1;
    int rb = pk(i, 0);   // packed start of row i; row i + 1 starts i + 1 later
    for (; i + 3 < nh; i += 4) {
      double li[4], a[4][kNCU];
      const int rbr[4] = {rb, rb + i + 1, rb + 2 * i + 3, rb + 3 * i + 6};
#pragma unroll
      for (int r = 0; r < 4; ++r) li[r] = L[rbr[r] + k];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < kNCU; ++c) {
          const int j = k + 1 + lane + 32 * c;
          a[r][c] = j <= i + r ? L[rbr[r] + j] : 0.0;
        }
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < kNCU; ++c) {
          const int j = k + 1 + lane + 32 * c;
          if (j <= i + r) L[rbr[r] + j] = a[r][c] - li[r] * colk[c];
        }
      rb += 4 * i + 10;   // start of row i + 4
    }
    for (; i < nh; ++i) {
      const double li = L[pk(i, k)];
#pragma unroll
      for (int c = 0; c < kNCU; ++c) {
        const int j = k + 1 + lane + 32 * c;
        if (j <= i) L[pk(i, j)] -= li * colk[c];
      }
    }
    __syncwarp();
  }
  if (bad) {
    if (lane == 0) info[b] = kNeedsLu;
    return;
  }

  // ---- Y = L^{-1} [C^T | r]: one column-oriented forward sweep for all R columns
  auto forward = [&](int ncols) {
    for (int j = 0; j < nh; ++j) {
      double yj[R];
#pragma unroll
      for (int q = 0; q < R; ++q) yj[q] = q < ncols ? Y[(size_t)j * R + q] * dinv[j] : 0.0;
      __syncwarp();
      if (lane == 0)
#pragma unroll
        for (int q = 0; q < R; ++q)
          if (q < ncols) Y[(size_t)j * R + q] = yj[q];
      for (int i = j + 1 + lane; i < nh; i += 32) {
        const double lij = L[pk(i, j)];
#pragma unroll
        for (int q = 0; q < R; ++q)
          if (q < ncols) Y[(size_t)i * R + q] -= lij * yj[q];
      }
      __syncwarp();
    }
  };
  // x = L^{-T} z, z in column P of Y (row-oriented over the packed rows)
  auto backward = [&]() {
    for (int j = nh - 1; j >= 0; --j) {
      const double xj = Y[(size_t)j * R + P] * dinv[j];
      __syncwarp();
      if (lane == 0) Y[(size_t)j * R + P] = xj;
      const double* row = L + pk(j, 0);
      for (int i = lane; i < j; i += 32) Y[(size_t)i * R + P] -= row[i] * xj;
      __syncwarp();
    }
  };

  for (int i = lane; i < nh; i += 32) {
#pragma unroll
    for (int mu = 0; mu < P; ++mu) Y[(size_t)i * R + mu] = i < me ? Ac[(size_t)mu * me + i] : beta[mu];
    Y[(size_t)i * R + P] = E[(size_t)i * Pe + me + 1];
  }
  __syncwarp();
  forward(R);
  // S = W^T W with W = L^{-1} C^T; Cholesky of S in registers (all lanes)
  double S[P][P];
#pragma unroll
  for (int a = 0; a < P; ++a)
#pragma unroll
    for (int c = 0; c < P; ++c) {
      double acc = 0.0;
      if (c <= a) {
        for (int i = lane; i < nh; i += 32) acc = fma(Y[(size_t)i * R + a], Y[(size_t)i * R + c], acc);
#pragma unroll
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      }
      S[a][c] = acc;
    }
#pragma unroll
  for (int a = 0; a < P; ++a) {
    double d = S[a][a];
    const double d0 = d;
#pragma unroll
    for (int c = 0; c < a; ++c) d -= S[a][c] * S[a][c];
    // a pivot lost to cancellation (e.g. duplicated conditions: S singular up to
    // rounding) goes to the LU, which decides singularity as the reference does
    if (!(d > 64.0 * 2.220446049250313e-16 * d0)) bad = 1;
    S[a][a] = sqrt(d > 0.0 ? d : 1.0);
#pragma unroll
    for (int r = a + 1; r < P; ++r) {
      double t = S[r][a];
#pragma unroll
      for (int c = 0; c < a; ++c) t -= S[r][c] * S[a][c];
      S[r][a] = t / S[a][a];
    }
  }
  if (bad) {
    if (lane == 0) info[b] = kNeedsLu;
    return;
  }

  // ---- solve + one refinement step (linear.py:144-147)
  for (int pass = 0; pass < 2; ++pass) {
    double rv[P];
    if (pass == 0) {
#pragma unroll
      for (int mu = 0; mu < P; ++mu) rv[mu] = vals[mu];
    } else {
      // r1 = rhs1 - H x - C^T lambda,  rv = v - C x  (H symmetric: coalesced rows of E)
      double acc[kNC];
#pragma unroll
      for (int c = 0; c < kNC; ++c) acc[c] = 0.0;
      for (int j0 = 0; j0 < nh; j0 += 8) {
        double ev[8][kNC], xj[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int j = j0 + r;
          xj[r] = j < nh ? xs[j] : 0.0;
#pragma unroll
          for (int c = 0; c < kNC; ++c) {
            const int i = lane + 32 * c;
            ev[r][c] = (j < nh && i < nh) ? __ldg(E + (size_t)j * Pe + i) : 0.0;
          }
        }
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int c = 0; c < kNC; ++c) {
            const int i = lane + 32 * c, j = j0 + r;
            acc[c] += ((i == j && i < me) ? inv_gamma + ev[r][c] : ev[r][c]) * xj[r];
          }
      }
#pragma unroll
      for (int c = 0; c < kNC; ++c) {
        const int i = lane + 32 * c;
        if (i < nh) {
          double a = acc[c];
#pragma unroll
          for (int mu = 0; mu < P; ++mu) a += (i < me ? Ac[(size_t)mu * me + i] : beta[mu]) * xs[nh + mu];
          Y[(size_t)i * R + P] = E[(size_t)i * Pe + me + 1] - a;
        }
      }
#pragma unroll
      for (int mu = 0; mu < P; ++mu) {
        double a = 0.0;
        for (int i = lane; i < me; i += 32) a = fma(Ac[(size_t)mu * me + i], xs[i], a);
#pragma unroll
        for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        rv[mu] = vals[mu] - (a + beta[mu] * xs[me]);
      }
      __syncwarp();
      // only the r column needs a new forward sweep (L^{-1} C^T is unchanged)
      for (int j = 0; j < nh; ++j) {
        const double yj = Y[(size_t)j * R + P] * dinv[j];
        __syncwarp();
        if (lane == 0) Y[(size_t)j * R + P] = yj;
        for (int i = j + 1 + lane; i < nh; i += 32) Y[(size_t)i * R + P] -= L[pk(i, j)] * yj;
        __syncwarp();
      }
    }
    // lambda = S^{-1} (W^T y1 - v)
    double t[P];
#pragma unroll
    for (int mu = 0; mu < P; ++mu) {
      double a = 0.0;
      for (int i = lane; i < nh; i += 32) a = fma(Y[(size_t)i * R + mu], Y[(size_t)i * R + P], a);
#pragma unroll
      for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      t[mu] = a - rv[mu];
    }
#pragma unroll
    for (int a = 0; a < P; ++a) {
      double v = t[a];
#pragma unroll
      for (int c = 0; c < a; ++c) v -= S[a][c] * t[c];
      t[a] = v / S[a][a];
    }
#pragma unroll
    for (int a = P - 1; a >= 0; --a) {
      double v = t[a];
#pragma unroll
      for (int c = a + 1; c < P; ++c) v -= S[c][a] * t[c];
      t[a] = v / S[a][a];
    }
    // z = y1 - W lambda ; x = L^{-T} z
    for (int i = lane; i < nh; i += 32) {
      double v = Y[(size_t)i * R + P];
#pragma unroll
      for (int mu = 0; mu < P; ++mu) v -= Y[(size_t)i * R + mu] * t[mu];
      Y[(size_t)i * R + P] = v;
    }
    __syncwarp();
    backward();
    for (int i = lane; i < nh; i += 32) {
      const double v = Y[(size_t)i * R + P];
      xs[i] = pass == 0 ? v : xs[i] + v;
    }
    if (lane == 0)
#pragma unroll
      for (int mu = 0; mu < P; ++mu) xs[nh + mu] = pass == 0 ? t[mu] : xs[nh + mu] + t[mu];
    __syncwarp();
  }
  const int n = nh + P;
  int nonfinite = 0;
  for (int i = lane; i < n; i += 32) {
    const double v = xs[i];
    if (!isfinite(v)) nonfinite = 1;
    xout[(size_t)b * n + i] = v;
  }
  nonfinite = __any_sync(0xffffffffu, nonfinite);
  if (lane == 0) info[b] = nonfinite ? kNeedsLu : NYS_INFO_OK;
}

template <int P, int NC, int NCU>
int launch_chol_nc(const double* dense, int m_eff, const double* Ac, const double* beta,
                const double* values, double gamma, int B, double* x, int* info, cudaStream_t st) {
  const int nh = m_eff + 1;
  const size_t dyn =
      ((size_t)nh * (nh + 1) / 2 + nh + (size_t)nh * (P + 1) + nh + P) * sizeof(double);
  auto kern = kkt_chol_kernel<P, NC, NCU>;
  if (dyn > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (e != cudaSuccess) return nys_host::record_cuda(e);
  }
  kern<<<B, 32, dyn, st>>>(dense, m_eff, Ac, beta, values, gamma, x, info);
  nys_host::count_launches(1);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

template <int P>
int launch_chol(const double* dense, int m_eff, const double* Ac, const double* beta,
                const double* values, double gamma, int B, double* x, int* info, cudaStream_t st) {
  const int nh = m_eff + 1;
  if (nh <= 32) return launch_chol_nc<P, 1, 1>(dense, m_eff, Ac, beta, values, gamma, B, x, info, st);
  if (nh == 33) return launch_chol_nc<P, 2, 1>(dense, m_eff, Ac, beta, values, gamma, B, x, info, st);
  if (nh <= 64) return launch_chol_nc<P, 2, 2>(dense, m_eff, Ac, beta, values, gamma, B, x, info, st);
  if (nh == 65) return launch_chol_nc<P, 3, 2>(dense, m_eff, Ac, beta, values, gamma, B, x, info, st);
  return launch_chol_nc<P, 3, 3>(dense, m_eff, Ac, beta, values, gamma, B, x, info, st);
}


// Single (or few) small systems: the same Cholesky + Schur algorithm as
// kkt_chol_kernel, spread over one CTA of 8 warps so a lone system is not bound
// by one warp's latency chains (config 1: 86 us with one warp).  H is dense in
// shared memory with an odd leading dimension (column walks are conflict-free);
// the Cholesky runs right-looking with the forward elimination of Y = [C^T | r]
// folded into every step (warps take rows, lanes columns, two barriers per
// column); S = W^T W by block reductions in fixed order; the triangular sweeps
// of the solve / refinement run in warp 0 (per-row dependency, __syncwarp
// only); the refinement residual is a CTA-wide GEMV over E.
constexpr int kSmallThreads = 256;
template <int P>
__global__ void __launch_bounds__(kSmallThreads)
    kkt_small_cta_kernel(const double* __restrict__ gram, int m_eff, const double* __restrict__ Ac,
                         const double* __restrict__ beta, const double* __restrict__ values,
                         double gamma, double* __restrict__ xout, int* __restrict__ info) {
  extern __shared__ __align__(16) double dsm[];
  constexpr int R = P + 1;
  constexpr int NW = kSmallThreads / 32;
  constexpr int NS = P * (P + 1) / 2;
  __shared__ double red[NW][NS > R ? NS : R];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, b = blockIdx.x;
  const int nh = m_eff + 1, me = m_eff, Pe = m_eff + 2, ld = nh | 1;
  const double* E = gram + (size_t)b * Pe * Pe;
  const double* vals = values + (size_t)b * P;
  double* L = dsm;                          // nh x ld, lower triangle
  double* dinv = L + (size_t)nh * ld;       // nh
  double* Y = dinv + nh;                    // nh x R
  double* xs = Y + (size_t)nh * R;          // nh + P
  const double inv_gamma = 1.0 / gamma;
  for (int e = tid; e < nh * nh; e += kSmallThreads) {
    const int i = e / nh, j = e % nh;
    if (j <= i) {
      const double v = __ldg(E + (size_t)i * Pe + j);
      L[i * ld + j] = (i == j && i < me) ? inv_gamma + v : v;
    }
  }
  for (int i = tid; i < nh; i += kSmallThreads) {
#pragma unroll
    for (int mu = 0; mu < P; ++mu) Y[i * R + mu] = i < me ? Ac[(size_t)mu * me + i] : beta[mu];
    Y[i * R + P] = E[(size_t)i * Pe + me + 1];
  }
  __syncthreads();
  // ---- H = L L^T with Y <- L^{-1} Y folded in, by 8-column panels: warp 0
  // factors a panel (column scale, in-panel updates and the elimination of Y,
  // __syncwarp only), then all warps apply its rank-8 update to the trailing
  // matrix in column order (a = a - l_ik l_jk for k = c0, c0+1, ...: the same
  // per-element operations as the unblocked right-looking loop)
  __shared__ int chol_bad_s;
  if (tid == 0) chol_bad_s = 0;
  __syncthreads();
  for (int c0 = 0; c0 < nh; c0 += 8) {
    const int c1 = min(c0 + 8, nh);
    if (warp == 0) {
      for (int k = c0; k < c1; ++k) {
        const double akk = L[k * ld + k];
        if (!(akk > 0.0) || !isfinite(akk)) {   // warp-uniform
          if (lane == 0) chol_bad_s = 1;
          break;
        }
        const double inv = rsqrt(akk);
        for (int i = k + 1 + lane; i < nh; i += 32) L[i * ld + k] *= inv;
        if (lane == 0) {
          L[k * ld + k] = akk * inv;
          dinv[k] = inv;
        }
        if (lane < R) Y[k * R + lane] *= inv;
        __syncwarp();
        for (int i = k + 1 + lane; i < nh; i += 32) {
          const double li = L[i * ld + k];
          for (int j = k + 1; j < c1 && j <= i; ++j) L[i * ld + j] -= li * L[j * ld + k];
#pragma unroll
          for (int q = 0; q < R; ++q) Y[i * R + q] -= li * Y[k * R + q];
        }
        __syncwarp();
      }
    }
    __syncthreads();
    if (chol_bad_s) break;
    if (c1 < nh) {
      const int w = c1 - c0;
      for (int i = c1 + warp; i < nh; i += NW) {
        double li[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) li[t] = t < w ? L[i * ld + c0 + t] : 0.0;
        for (int j = c1 + lane; j <= i; j += 32) {
          double a = L[i * ld + j];
          const double* lj = L + j * ld + c0;
#pragma unroll
          for (int t = 0; t < 8; ++t)
            if (t < w) a -= li[t] * lj[t];
          L[i * ld + j] = a;
        }
      }
    }
    __syncthreads();
  }
  const int chol_bad = chol_bad_s;
  if (chol_bad) {
    if (tid == 0) info[b] = kNeedsLu;
    return;
  }
  // ---- S = W^T W (W = Y[:, :P]); every thread gets the same sums (fixed order)
  {
    double a[NS];
#pragma unroll
    for (int q = 0; q < NS; ++q) a[q] = 0.0;
    for (int i = tid; i < nh; i += kSmallThreads) {
      int q = 0;
#pragma unroll
      for (int x = 0; x < P; ++x)
#pragma unroll
        for (int c = 0; c <= x; ++c, ++q) a[q] = fma(Y[i * R + x], Y[i * R + c], a[q]);
    }
#pragma unroll
    for (int q = 0; q < NS; ++q) {
#pragma unroll
      for (int o = 16; o; o >>= 1) a[q] += __shfl_xor_sync(0xffffffffu, a[q], o);
      if (lane == 0) red[warp][q] = a[q];
    }
  }
  __syncthreads();
  double S[P][P];
  {
    int q = 0;
#pragma unroll
    for (int x = 0; x < P; ++x)
#pragma unroll
      for (int c = 0; c <= x; ++c, ++q) {
        double v = 0.0;
        for (int w = 0; w < NW; ++w) v += red[w][q];
        S[x][c] = v;
      }
  }
  int bad = 0;
#pragma unroll
  for (int a = 0; a < P; ++a) {
    double d = S[a][a];
    const double d0 = d;
#pragma unroll
    for (int c = 0; c < a; ++c) d -= S[a][c] * S[a][c];
    if (!(d > 64.0 * 2.220446049250313e-16 * d0)) bad = 1;
    S[a][a] = sqrt(d > 0.0 ? d : 1.0);
#pragma unroll
    for (int r = a + 1; r < P; ++r) {
      double t = S[r][a];
#pragma unroll
      for (int c = 0; c < a; ++c) t -= S[r][c] * S[a][c];
      S[r][a] = t / S[a][a];
    }
  }
  if (bad) {
    if (tid == 0) info[b] = kNeedsLu;
    return;
  }
  __syncthreads();   // red reused below

  for (int pass = 0; pass < 2; ++pass) {
    double rv[P];
    if (pass == 0) {
#pragma unroll
      for (int mu = 0; mu < P; ++mu) rv[mu] = vals[mu];
    } else {
      // r1 = rhs1 - H x - C^T lambda (rows by thread, E symmetric: coalesced)
      for (int i = tid; i < nh; i += kSmallThreads) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int j = 0;
        for (; j + 8 <= nh; j += 8) {   // eight L2 loads in flight
          double e[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) e[u] = __ldg(E + (size_t)(j + u) * Pe + i);
          a0 = fma(e[0], xs[j], a0);
          a1 = fma(e[1], xs[j + 1], a1);
          a2 = fma(e[2], xs[j + 2], a2);
          a3 = fma(e[3], xs[j + 3], a3);
          a0 = fma(e[4], xs[j + 4], a0);
          a1 = fma(e[5], xs[j + 5], a1);
          a2 = fma(e[6], xs[j + 6], a2);
          a3 = fma(e[7], xs[j + 7], a3);
        }
        for (; j < nh; ++j) a0 = fma(__ldg(E + (size_t)j * Pe + i), xs[j], a0);
        double a = (a0 + a1) + (a2 + a3);
        if (i < me) a = fma(inv_gamma, xs[i], a);
#pragma unroll
        for (int mu = 0; mu < P; ++mu) a += (i < me ? Ac[(size_t)mu * me + i] : beta[mu]) * xs[nh + mu];
        Y[i * R + P] = E[(size_t)i * Pe + me + 1] - a;
      }
      double c[P];
#pragma unroll
      for (int mu = 0; mu < P; ++mu) c[mu] = 0.0;
      for (int i = tid; i < me; i += kSmallThreads)
#pragma unroll
        for (int mu = 0; mu < P; ++mu) c[mu] = fma(Ac[(size_t)mu * me + i], xs[i], c[mu]);
#pragma unroll
      for (int mu = 0; mu < P; ++mu) {
#pragma unroll
        for (int o = 16; o; o >>= 1) c[mu] += __shfl_xor_sync(0xffffffffu, c[mu], o);
        if (lane == 0) red[warp][mu] = c[mu];
      }
      __syncthreads();
#pragma unroll
      for (int mu = 0; mu < P; ++mu) {
        double v = 0.0;
        for (int w = 0; w < NW; ++w) v += red[w][mu];
        rv[mu] = vals[mu] - (v + beta[mu] * xs[me]);
      }
      // forward sweep of the r column (warp 0; L^{-1} C^T is unchanged)
      if (warp == 0) {
        for (int j = 0; j < nh; ++j) {
          const double yj = Y[j * R + P] * dinv[j];
          __syncwarp();
          if (lane == 0) Y[j * R + P] = yj;
          for (int i = j + 1 + lane; i < nh; i += 32) Y[i * R + P] -= L[i * ld + j] * yj;
          __syncwarp();
        }
      }
      __syncthreads();
    }
    // lambda = S^{-1} (W^T y1 - v)
    {
      double a[P];
#pragma unroll
      for (int mu = 0; mu < P; ++mu) a[mu] = 0.0;
      for (int i = tid; i < nh; i += kSmallThreads)
#pragma unroll
        for (int mu = 0; mu < P; ++mu) a[mu] = fma(Y[i * R + mu], Y[i * R + P], a[mu]);
#pragma unroll
      for (int mu = 0; mu < P; ++mu) {
#pragma unroll
        for (int o = 16; o; o >>= 1) a[mu] += __shfl_xor_sync(0xffffffffu, a[mu], o);
        if (lane == 0) red[warp][mu] = a[mu];
      }
    }
    __syncthreads();
    double t[P];
#pragma unroll
    for (int mu = 0; mu < P; ++mu) {
      double v = 0.0;
      for (int w = 0; w < NW; ++w) v += red[w][mu];
      t[mu] = v - rv[mu];
    }
#pragma unroll
    for (int a = 0; a < P; ++a) {
      double v = t[a];
#pragma unroll
      for (int c = 0; c < a; ++c) v -= S[a][c] * t[c];
      t[a] = v / S[a][a];
    }
#pragma unroll
    for (int a = P - 1; a >= 0; --a) {
      double v = t[a];
#pragma unroll
      for (int c = a + 1; c < P; ++c) v -= S[c][a] * t[c];
      t[a] = v / S[a][a];
    }
    // z = y1 - W lambda ; x = L^{-T} z (warp 0)
    for (int i = tid; i < nh; i += kSmallThreads) {
      double v = Y[i * R + P];
#pragma unroll
      for (int mu = 0; mu < P; ++mu) v -= Y[i * R + mu] * t[mu];
      Y[i * R + P] = v;
    }
    __syncthreads();
    if (warp == 0) {
      for (int j = nh - 1; j >= 0; --j) {
        const double xj = Y[j * R + P] * dinv[j];
        __syncwarp();
        if (lane == 0) Y[j * R + P] = xj;
        for (int i = lane; i < j; i += 32) Y[i * R + P] -= L[j * ld + i] * xj;
        __syncwarp();
      }
    }
    __syncthreads();
    for (int i = tid; i < nh; i += kSmallThreads) {
      const double v = Y[i * R + P];
      xs[i] = pass == 0 ? v : xs[i] + v;
    }
    if (tid == 0)
#pragma unroll
      for (int mu = 0; mu < P; ++mu) xs[nh + mu] = pass == 0 ? t[mu] : xs[nh + mu] + t[mu];
    __syncthreads();
  }
  const int n = nh + P;
  int nonfinite = 0;
  for (int i = tid; i < n; i += kSmallThreads) {
    const double v = xs[i];
    if (!isfinite(v)) nonfinite = 1;
    xout[(size_t)b * n + i] = v;
  }
  nonfinite = __syncthreads_or(nonfinite);
  if (tid == 0) info[b] = nonfinite ? kNeedsLu : NYS_INFO_OK;
}

template <int P>
int launch_small_cta(const double* dense, int m_eff, const double* Ac, const double* beta,
                     const double* values, double gamma, int B, double* x, int* info,
                     cudaStream_t st) {
  const int nh = m_eff + 1, ld = nh | 1;
  const size_t dyn = ((size_t)nh * ld + nh + (size_t)nh * (P + 1) + nh + P) * sizeof(double);
  auto kern = kkt_small_cta_kernel<P>;
  if (dyn > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (e != cudaSuccess) return nys_host::record_cuda(e);
  }
  kern<<<B, kSmallThreads, dyn, st>>>(dense, m_eff, Ac, beta, values, gamma, x, info);
  nys_host::count_launches(1);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}
}  // namespace

namespace nys_host {
// dense extended Grams (B x Pe x Pe) -> Cholesky + Schur (blocked DMMA when m_eff
// is a multiple of 8 in [32, 64]); instances whose Cholesky breaks down are
// flagged for the LU (caller re-runs launch_kkt with only_flagged)
int launch_kkt_chol_dense(const double* dense, int m_eff, int n_cond, const double* Ac,
                          const double* beta, const double* values, double gamma, int B,
                          double* x, int* info, cudaStream_t st) {
  if (m_eff < 1 || n_cond < 1 || n_cond > 4 || m_eff + 1 > kMaxNh) return NYS_EUNSUPPORTED;
  if (B <= 8 && getenv("NYS_KKT_WARP") == nullptr) {   // few systems: one CTA each
    switch (n_cond) {
      case 1: return launch_small_cta<1>(dense, m_eff, Ac, beta, values, gamma, B, x, info, st);
      case 2: return launch_small_cta<2>(dense, m_eff, Ac, beta, values, gamma, B, x, info, st);
      case 3: return launch_small_cta<3>(dense, m_eff, Ac, beta, values, gamma, B, x, info, st);
      default: return launch_small_cta<4>(dense, m_eff, Ac, beta, values, gamma, B, x, info, st);
    }
  }
  int rc = launch_kkt_blocked(dense, m_eff, n_cond, Ac, beta, values, gamma, B, x, info, st);
  if (rc != NYS_EUNSUPPORTED) return rc;
  switch (n_cond) {
    case 1: return launch_chol<1>(dense, m_eff, Ac, beta, values, gamma, B, x, info, st);
    case 2: return launch_chol<2>(dense, m_eff, Ac, beta, values, gamma, B, x, info, st);
    case 3: return launch_chol<3>(dense, m_eff, Ac, beta, values, gamma, B, x, info, st);
    default: return launch_chol<4>(dense, m_eff, Ac, beta, values, gamma, B, x, info, st);
  }
}
}  // namespace nys_host

extern "C" int nys_batch_kkt_solve_f64(const void* batch_workspace, int n_c, int m_eff, int p,
                                       int n_cond, const double* Ac, const double* beta,
                                       const double* values, double gamma, int B, double* x,
                                       int* info, void* stream) {
  if (m_eff < 1 || n_cond < 1 || B < 0 || !(gamma > 0.0) || p < 1 || p > 2) return NYS_EINVAL;
  if (B == 0) return NYS_OK;
  if (m_eff + 1 > kMaxNh || n_cond > 4) return NYS_EUNSUPPORTED;
  nys::BatchLayout L = nys::BatchLayout::make(n_c, m_eff, p, B);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* dense = L.dense(const_cast<void*>(batch_workspace));
  int rc = nys_host::launch_batch_unpack(L.part(batch_workspace), L.nsplit, B, L.NB, L.Pe(), dense,
                                         st);
  if (rc) return rc;
  // m_eff a multiple of 8 in [32, 64]: blocked DMMA Cholesky (kkt_block.cu)
  rc = getenv("NYS_KKT_SCALAR") != nullptr
           ? NYS_EUNSUPPORTED
           : nys_host::launch_kkt_blocked(dense, m_eff, n_cond, Ac, beta, values, gamma, B, x,
                                          info, st);
  if (rc == NYS_OK)
    return nys_host::launch_kkt(dense, m_eff, n_cond, Ac, beta, values, gamma, B, x, info,
                                nullptr, nullptr, nullptr, 0, st, true);
  if (rc != NYS_EUNSUPPORTED) return rc;
  switch (n_cond) {
    case 1: rc = launch_chol<1>(dense, m_eff, Ac, beta, values, gamma, B, x, info, st); break;
    case 2: rc = launch_chol<2>(dense, m_eff, Ac, beta, values, gamma, B, x, info, st); break;
    case 3: rc = launch_chol<3>(dense, m_eff, Ac, beta, values, gamma, B, x, info, st); break;
    default: rc = launch_chol<4>(dense, m_eff, Ac, beta, values, gamma, B, x, info, st); break;
  }
  if (rc) return rc;
  // LU (the reference's algorithm) re-solves any instance whose Cholesky broke down
  return nys_host::launch_kkt(dense, m_eff, n_cond, Ac, beta, values, gamma, B, x, info, nullptr,
                              nullptr, nullptr, 0, st, true);
}
