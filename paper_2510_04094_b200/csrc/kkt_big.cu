// Single large KKT system (config 4: m_eff = 256, side 259): one CTA of 32
// warps, blocked Cholesky of the omega block with DMMA trailing updates, bias
// + conditions by a small pivoted Schur system, one refinement pass -- the
// kkt_block.cu algorithm spread over a CTA (Cholesky + Schur
// instead of the reference's LU moves y_hat by <= 4.1e-14 on the c4 shape).
//
// The packed lower blocks (8 x 8, 270 KB at m_eff = 256) live in the caller's
// workspace (L1/L2 resident); the triangular sweeps keep Y = L^{-1}[Bt | r1]
// in shared memory.  Per 8-column panel: warp 0 factors the diagonal block by
// shuffles, every thread forward-solves one panel row against it, and the 32
// warps split the trailing block pairs (two DMMA.8x8x4 each).  Replaces the
// 259-step partial-pivoting LU (kkt.cu, 3.5 ms, one pivot search and one
// trailing sweep per column); a failed pivot falls back to that LU.
#include <cmath>

#include "common.cuh"

namespace {

constexpr int kNeedsLu = 16;
constexpr int kBigThreads = 1024;
constexpr int kBigWarps = kBigThreads / 32;

NYS_DEV int blk(int I, int J) { return I * (I + 1) / 2 + J; }

template <int P>
__global__ void __launch_bounds__(kBigThreads, 1)
    kkt_big_kernel(const double* __restrict__ E, int me, const double* __restrict__ Ac,
                   const double* __restrict__ beta, const double* __restrict__ values,
                   double gamma, double* __restrict__ xout, int* __restrict__ info,
                   double* __restrict__ Lg) {
  constexpr int Q = P + 1, R = Q + 1;
  extern __shared__ __align__(16) double sm[];
  const int NBK = me / 8, Pe = me + 2;
  double* Y = sm;                       // me x 8
  double* dinv = Y + me * 8;            // me
  double* part = dinv + me;             // kBigWarps x 64 (sweep partials)
  double* xs = part + kBigWarps * 64;   // me
  __shared__ double Lpp[64], dpp[8], red[kBigWarps][Q + 1], zs[Q];
  __shared__ int bad_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int fr = lane >> 2, fc = lane & 3;
  const double inv_gamma = 1.0 / gamma;
  const double* vals = values;
  if (tid == 0) bad_s = 0;

  // ---- A = E[0:me, 0:me] + I / gamma into packed lower blocks
  const int nblk = NBK * (NBK + 1) / 2;
  for (int e = tid; e < nblk * 64; e += kBigThreads) {
    const int q = e >> 6, w = e & 63, r = w >> 3, c = w & 7;
    int I = (int)((sqrt(8.0 * q + 1.0) - 1.0) * 0.5);
    while (blk(I + 1, 0) <= q) ++I;
    while (blk(I, 0) > q) --I;
    const int J = q - blk(I, 0);
    double v = E[(size_t)(8 * I + r) * Pe + 8 * J + c];
    if (I == J && r == c) v += inv_gamma;
    Lg[e] = v;
  }
  __syncthreads();

  // ---- blocked Cholesky
  for (int p = 0; p < NBK; ++p) {
    if (warp == 0) {   // diagonal block by shuffles: lanes 0..7 own its rows
      double v[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) v[c] = lane < 8 ? Lg[blk(p, p) * 64 + lane * 8 + c] : 0.0;
      int bad = 0;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const double piv = __shfl_sync(0xffffffffu, v[c], c);
        if (!(piv > 0.0) || !isfinite(piv)) bad = 1;
        const double inv = rsqrt(piv);
        v[c] = (lane > c) ? v[c] * inv : (lane == c ? piv * inv : v[c]);
#pragma unroll
        for (int c2 = c + 1; c2 < 8; ++c2) {
          const double l = __shfl_sync(0xffffffffu, v[c], c2);
          v[c2] = fma(-v[c], l, v[c2]);
        }
      }
      if (lane < 8) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const double x = c <= lane ? v[c] : 0.0;
          Lpp[lane * 8 + c] = x;
          Lg[blk(p, p) * 64 + lane * 8 + c] = x;
        }
        dpp[lane] = 1.0 / v[lane];
        dinv[8 * p + lane] = 1.0 / v[lane];
      }
      if (lane == 0 && bad) bad_s = 1;
    }
    __syncthreads();
    if (bad_s) break;
    // panel rows below: L_Ip = A_Ip L_pp^{-T}, one row per thread
    for (int R0 = 8 * (p + 1) + tid; R0 < me; R0 += kBigThreads) {
      double* row = Lg + blk(R0 >> 3, p) * 64 + (R0 & 7) * 8;
      double v[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) v[c] = row[c];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        double t = v[c];
#pragma unroll
        for (int k = 0; k < c; ++k) t = fma(-v[k], Lpp[c * 8 + k], t);
        v[c] = t * dpp[c];
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) row[c] = v[c];
    }
    __syncthreads();
    // trailing pairs (I, J), p < J <= I: C_IJ -= L_Ip L_Jp^T
    const int nb = NBK - p - 1;
    const int npair = nb * (nb + 1) / 2;
    for (int t = warp; t < npair; t += kBigWarps) {
      int i1 = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
      while ((i1 + 1) * (i1 + 2) / 2 <= t) ++i1;
      while (i1 * (i1 + 1) / 2 > t) --i1;
      const int I = p + 1 + i1, J = p + 1 + (t - i1 * (i1 + 1) / 2);
      const double* LI = Lg + blk(I, p) * 64;
      const double* LJ = Lg + blk(J, p) * 64;
      double* C = Lg + blk(I, J) * 64 + fr * 8 + 2 * fc;
      const double a0 = -LI[fr * 8 + fc], a1 = -LI[fr * 8 + 4 + fc];
      const double b0 = LJ[fr * 8 + fc], b1 = LJ[fr * 8 + 4 + fc];
      double2 cv = *reinterpret_cast<double2*>(C);
      nys::dmma(cv.x, cv.y, a0, b0);
      nys::dmma(cv.x, cv.y, a1, b1);
      *reinterpret_cast<double2*>(C) = cv;
    }
    __syncthreads();
  }
  if (bad_s) {
    if (tid == 0) *info = kNeedsLu;
    return;
  }

  // ---- Y = L^{-1} [D^T g | A_c^T | r1]  (columns >= R zero)
  for (int i = tid; i < me; i += kBigThreads) {
    Y[i * 8 + 0] = E[(size_t)i * Pe + me];
#pragma unroll
    for (int mu = 0; mu < P; ++mu) Y[i * 8 + 1 + mu] = Ac[(size_t)mu * me + i];
    Y[i * 8 + Q] = E[(size_t)i * Pe + me + 1];
#pragma unroll
    for (int q = R; q < 8; ++q) Y[i * 8 + q] = 0.0;
  }
  __syncthreads();
  // blocked sweeps: the off-diagonal sum of block row I is split over the warps
  // (DMMA, partials in smem), warp 0 reduces it in warp order and solves the
  // diagonal block row by row with shuffles; only columns in `cols` are stored
  auto sweep = [&](bool fwd, unsigned cols) {
    for (int s = 0; s < NBK; ++s) {
      const int I = fwd ? s : NBK - 1 - s;
      double2 acc = make_double2(0.0, 0.0);
      for (int J = warp; J < NBK; J += kBigWarps) {
        if (fwd ? (J >= I) : (J <= I)) continue;
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          // fwd: L_IJ (row fr, column 4kk+fc); bwd: (L_JI)^T -> L_JI[4kk+fc][fr]
          const double a = fwd ? Lg[blk(I, J) * 64 + fr * 8 + 4 * kk + fc]
                               : Lg[blk(J, I) * 64 + (4 * kk + fc) * 8 + fr];
          const double bq = Y[(8 * J + 4 * kk + fc) * 8 + fr];
          nys::dmma(acc.x, acc.y, a, bq);
        }
      }
      *reinterpret_cast<double2*>(part + warp * 64 + lane * 2) = acc;
      __syncthreads();
      if (warp == 0) {
        double2 cv = *reinterpret_cast<const double2*>(Y + (8 * I + fr) * 8 + 2 * fc);
        for (int w = 0; w < kBigWarps; ++w) {
          const double2 pw = *reinterpret_cast<const double2*>(part + w * 64 + lane * 2);
          cv.x -= pw.x;
          cv.y -= pw.y;
        }
        if (fwd) {
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            if (fr == c) {
              const double d = dinv[8 * I + c];
              cv.x *= d;
              cv.y *= d;
            }
            const double yx = __shfl_sync(0xffffffffu, cv.x, c * 4 + fc);
            const double yy = __shfl_sync(0xffffffffu, cv.y, c * 4 + fc);
            if (fr > c) {
              const double l = Lg[blk(I, I) * 64 + fr * 8 + c];
              cv.x = fma(-l, yx, cv.x);
              cv.y = fma(-l, yy, cv.y);
            }
          }
        } else {
#pragma unroll
          for (int c = 7; c >= 0; --c) {
            if (fr == c) {
              const double d = dinv[8 * I + c];
              cv.x *= d;
              cv.y *= d;
            }
            const double yx = __shfl_sync(0xffffffffu, cv.x, c * 4 + fc);
            const double yy = __shfl_sync(0xffffffffu, cv.y, c * 4 + fc);
            if (fr < c) {
              const double l = Lg[blk(I, I) * 64 + c * 8 + fr];
              cv.x = fma(-l, yx, cv.x);
              cv.y = fma(-l, yy, cv.y);
            }
          }
        }
        double* dst = Y + (8 * I + fr) * 8 + 2 * fc;
        if ((cols >> (2 * fc)) & 1u) dst[0] = cv.x;
        if ((cols >> (2 * fc + 1)) & 1u) dst[1] = cv.y;
      }
      __syncthreads();
    }
  };
  // block-wide dot products of Y columns (fixed-order reductions)
  auto dots = [&](int qa, const int* qb, int nq, double* out) {
    double a[Q + 1];
#pragma unroll
    for (int k = 0; k <= Q; ++k) a[k] = 0.0;
    for (int i = tid; i < me; i += kBigThreads)
#pragma unroll
      for (int k = 0; k <= Q; ++k)
        if (k < nq) a[k] = fma(Y[i * 8 + qa], Y[i * 8 + qb[k]], a[k]);
#pragma unroll
    for (int k = 0; k <= Q; ++k) {
#pragma unroll
      for (int o = 16; o; o >>= 1) a[k] += __shfl_xor_sync(0xffffffffu, a[k], o);
      if (lane == 0) red[warp][k] = a[k];
    }
    __syncthreads();
    for (int k = 0; k < nq; ++k) {
      double s = 0.0;
      for (int w = 0; w < kBigWarps; ++w) s += red[w][k];
      out[k] = s;
    }
    __syncthreads();
  };

  sweep(true, (1u << R) - 1u);
  double S[Q][Q];
#pragma unroll
  for (int a = 0; a < Q; ++a) {
    int qb[Q + 1];
    for (int k = 0; k <= Q; ++k) qb[k] = k;
    double d[Q + 1];
    dots(a, qb, Q, d);
#pragma unroll
    for (int c = 0; c < Q; ++c) {
      const double cp = (a == 0 && c == 0) ? E[(size_t)me * Pe + me]
                                           : (a == 0 ? beta[c - 1] : (c == 0 ? beta[a - 1] : 0.0));
      S[a][c] = cp - d[c];
    }
  }
  // pivoted elimination of S (every thread redundantly)
  int piv[Q];
  int badS = 0;
#pragma unroll
  for (int a = 0; a < Q; ++a) piv[a] = a;
  // pivots lost to cancellation (duplicated conditions: S singular up to
  // rounding) go to the LU, which decides singularity as the reference does
  double smax = 0.0;
#pragma unroll
  for (int a = 0; a < Q; ++a)
#pragma unroll
    for (int c = 0; c < Q; ++c) smax = fmax(smax, fabs(S[a][c]));
  const double piv_floor = 64.0 * 2.220446049250313e-16 * smax;
#pragma unroll
  for (int k = 0; k < Q; ++k) {
    int pr = k;
    double best = fabs(S[k][k]);
#pragma unroll
    for (int r = k + 1; r < Q; ++r)
      if (fabs(S[r][k]) > best) {
        best = fabs(S[r][k]);
        pr = r;
      }
    if (!(best > piv_floor)) badS = 1;
#pragma unroll
    for (int r = k + 1; r < Q; ++r)
      if (r == pr) {
#pragma unroll
        for (int c = 0; c < Q; ++c) {
          const double t = S[k][c];
          S[k][c] = S[r][c];
          S[r][c] = t;
        }
        const int t = piv[k];
        piv[k] = piv[r];
        piv[r] = t;
      }
    const double ip = best > 0.0 ? 1.0 / S[k][k] : 0.0;
#pragma unroll
    for (int r = k + 1; r < Q; ++r) {
      const double f = S[r][k] * ip;
      S[r][k] = f;
#pragma unroll
      for (int c = k + 1; c < Q; ++c) S[r][c] = fma(-f, S[k][c], S[r][c]);
    }
  }
  if (badS) {
    if (tid == 0) *info = kNeedsLu;
    return;
  }
  auto solve_small = [&](double* t) {
    double u[Q];
#pragma unroll
    for (int a = 0; a < Q; ++a) {
      double v = 0.0;
#pragma unroll
      for (int c = 0; c < Q; ++c) v = (piv[a] == c) ? t[c] : v;
      u[a] = v;
    }
#pragma unroll
    for (int a = 0; a < Q; ++a)
#pragma unroll
      for (int c = 0; c < a; ++c) u[a] = fma(-S[a][c], u[c], u[a]);
#pragma unroll
    for (int a = Q - 1; a >= 0; --a) {
#pragma unroll
      for (int c = a + 1; c < Q; ++c) u[a] = fma(-S[a][c], u[c], u[a]);
      u[a] /= S[a][a];
    }
#pragma unroll
    for (int a = 0; a < Q; ++a) t[a] = u[a];
  };

  double z[Q], rq[Q];
  rq[0] = E[(size_t)me * Pe + me + 1];
#pragma unroll
  for (int mu = 0; mu < P; ++mu) rq[1 + mu] = vals[mu];
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) {
      // residuals r1 - A x - Bt z (rows by thread, E symmetric: coalesced)
      for (int i = tid; i < me; i += kBigThreads) {
        double a0 = 0.0, a1 = 0.0;
        int j = 0;
        for (; j + 1 < me; j += 2) {
          a0 = fma(E[(size_t)j * Pe + i], xs[j], a0);
          a1 = fma(E[(size_t)(j + 1) * Pe + i], xs[j + 1], a1);
        }
        if (j < me) a0 = fma(E[(size_t)j * Pe + i], xs[j], a0);
        double a = a0 + a1 + inv_gamma * xs[i];
        a = fma(E[(size_t)i * Pe + me], z[0], a);
#pragma unroll
        for (int mu = 0; mu < P; ++mu) a = fma(Ac[(size_t)mu * me + i], z[1 + mu], a);
        Y[i * 8 + Q] = E[(size_t)i * Pe + me + 1] - a;
      }
      // rq - Bt^T x - C' z
      double g[Q + 1];
#pragma unroll
      for (int k = 0; k <= Q; ++k) g[k] = 0.0;
      for (int i = tid; i < me; i += kBigThreads) {
        g[0] = fma(E[(size_t)me * Pe + i], xs[i], g[0]);
#pragma unroll
        for (int mu = 0; mu < P; ++mu) g[1 + mu] = fma(Ac[(size_t)mu * me + i], xs[i], g[1 + mu]);
      }
#pragma unroll
      for (int k = 0; k < Q; ++k) {
#pragma unroll
        for (int o = 16; o; o >>= 1) g[k] += __shfl_xor_sync(0xffffffffu, g[k], o);
        if (lane == 0) red[warp][k] = g[k];
      }
      __syncthreads();
      double gs[Q];
      for (int k = 0; k < Q; ++k) {
        double s2 = 0.0;
        for (int w = 0; w < kBigWarps; ++w) s2 += red[w][k];
        gs[k] = s2;
      }
      double cz0 = E[(size_t)me * Pe + me] * z[0];
#pragma unroll
      for (int mu = 0; mu < P; ++mu) cz0 = fma(beta[mu], z[1 + mu], cz0);
      rq[0] = E[(size_t)me * Pe + me + 1] - (gs[0] + cz0);
#pragma unroll
      for (int mu = 0; mu < P; ++mu) rq[1 + mu] = vals[mu] - (gs[1 + mu] + beta[mu] * z[0]);
      __syncthreads();
      sweep(true, 1u << Q);
    }
    int qb[Q + 1];
    for (int k = 0; k <= Q; ++k) qb[k] = k;
    double d[Q + 1];
    double t[Q];
    for (int a = 0; a < Q; ++a) {
      int one[Q + 1];
      one[0] = Q;
      double dq[Q + 1];
      dots(a, one, 1, dq);
      t[a] = rq[a] - dq[0];
    }
    (void)qb;
    (void)d;
    solve_small(t);
    for (int i = tid; i < me; i += kBigThreads) {
      double v = Y[i * 8 + Q];
#pragma unroll
      for (int a = 0; a < Q; ++a) v = fma(-Y[i * 8 + a], t[a], v);
      Y[i * 8 + Q] = v;
    }
    __syncthreads();
    sweep(false, 1u << Q);
    for (int i = tid; i < me; i += kBigThreads) {
      const double v = Y[i * 8 + Q];
      xs[i] = pass == 0 ? v : xs[i] + v;
    }
#pragma unroll
    for (int a = 0; a < Q; ++a) z[a] = pass == 0 ? t[a] : z[a] + t[a];
    __syncthreads();
  }
  const int n = me + Q;
  int nonfinite = 0;
  for (int i = tid; i < n; i += kBigThreads) {
    double v = 0.0;
    if (i < me) {
      v = xs[i];
    } else {
#pragma unroll
      for (int a = 0; a < Q; ++a) v = (i - me == a) ? z[a] : v;
    }
    if (!isfinite(v)) nonfinite = 1;
    xout[i] = v;
  }
  nonfinite = __syncthreads_or(nonfinite);
  if (tid == 0) *info = nonfinite ? kNeedsLu : NYS_INFO_OK;
  (void)zs;
}

template <int P>
int launch_big(const double* E, int me, const double* Ac, const double* beta,
               const double* values, double gamma, double* x, int* info, double* Lg,
               cudaStream_t st) {
  const size_t dyn = ((size_t)me * 8 + me + kBigWarps * 64 + me) * sizeof(double);
  auto kern = kkt_big_kernel<P>;
  if (dyn > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (e != cudaSuccess) return nys_host::record_cuda(e);
  }
  kern<<<1, kBigThreads, dyn, st>>>(E, me, Ac, beta, values, gamma, x, info, Lg);
  nys_host::count_launches(1);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

}  // namespace

namespace nys_host {
size_t kkt_big_ws_bytes(int m_eff) {
  const int nbk = m_eff / 8;
  return (size_t)nbk * (nbk + 1) / 2 * 64 * sizeof(double);
}
// single instance, m_eff a multiple of 8 in (64, 512]; NYS_EUNSUPPORTED otherwise
int launch_kkt_big(const double* E, int m_eff, int n_cond, const double* Ac, const double* beta,
                   const double* values, double gamma, double* x, int* info, void* ws,
                   size_t ws_bytes, cudaStream_t st) {
  if (m_eff % 8 != 0 || m_eff <= 64 || m_eff > 512 || n_cond < 1 || n_cond > 4)
    return NYS_EUNSUPPORTED;
  if (ws == nullptr || ws_bytes < kkt_big_ws_bytes(m_eff)) return NYS_EUNSUPPORTED;
  double* Lg = static_cast<double*>(ws);
  switch (n_cond) {
    case 1: return launch_big<1>(E, m_eff, Ac, beta, values, gamma, x, info, Lg, st);
    case 2: return launch_big<2>(E, m_eff, Ac, beta, values, gamma, x, info, Lg, st);
    case 3: return launch_big<3>(E, m_eff, Ac, beta, values, gamma, x, info, Lg, st);
    default: return launch_big<4>(E, m_eff, Ac, beta, values, gamma, x, info, Lg, st);
  }
}
}  // namespace nys_host
