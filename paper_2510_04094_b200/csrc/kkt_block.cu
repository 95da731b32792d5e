// Batched KKT solve, blocked: the omega block's Cholesky with DMMA trailing
// updates (config 2: m_eff = 64, one warp per instance).
//
//   M = [[A, Bt], [Bt^T, C']]   A = D^T D + I/gamma (me x me, SPD),
//   Bt = [D^T g | A_c^T] (me x Q), C' = [[g^T g, beta^T], [beta, 0]], Q = 1 + P
// (linear.py:123-131 with the bias moved from the SPD block into the small
// Schur system).  A = L L^T by 8 x 8 blocks: each 8-column panel is factored in
// registers (a lane owns two panel rows; pivots and the panel's column of
// multipliers travel by warp shuffles), and the trailing blocks receive
// C -= L_Ip L_Jp^T as two DMMA.8x8x4 each -- the bulk of the flops at 256 FMAs
// per instruction instead of the 32 of a warp-wide FMA, which is what bounds
// the scalar factorization (kkt_chol.cu: issue-bound, 64 % issue active).
// Then Y = L^{-1}[Bt | r1], S = C' - Y_B^T Y_B (pivoted elimination in
// registers), z = S^{-1}(rhs_Q - Y_B^T y_r), x = L^{-T}(y_r - Y_B z), and one
// refinement pass (linear.py:144-147).  A non-positive pivot, a singular S or
// a non-finite result marks the instance for the LU fallback (kkt.cu), as in
// kkt_chol.cu.  Storage: lower blocks packed, each 8 x 8 row-major with the
// column index XOR-swizzled by ((r >> 1) & 1) << 2 so the DMMA operand loads
// (8 rows x 4 columns per warp) hit every bank pair exactly twice.
#include <cmath>

#include "common.cuh"

namespace {

constexpr int kNeedsLu = 16;   // kkt.cu's LU kernel re-solves instances carrying it

NYS_DEV int blk(int I, int J) { return I * (I + 1) / 2 + J; }
NYS_DEV int swz(int r, int c) { return r * 8 + (c ^ ((r & 2) << 1)); }

template <int P, int NBK>
__global__ void __launch_bounds__(32)
    kkt_block_kernel(const double* __restrict__ gram, const double* __restrict__ Ac,
                     const double* __restrict__ beta, const double* __restrict__ values,
                     double gamma, double* __restrict__ xout, int* __restrict__ info) {
  constexpr int me = NBK * 8;
  constexpr int Pe = me + 2;
  constexpr int Q = P + 1;        // bias + multipliers
  constexpr int R = Q + 1;        // forward columns: D^T g | A_c^T | r1
  constexpr int NBLK = NBK * (NBK + 1) / 2;
  extern __shared__ __align__(16) double dsm[];
  const int lane = threadIdx.x, b = blockIdx.x;
  const int fr = lane >> 2, fc = lane & 3;   // MMA fragment row / column-in-group
  const double* E = gram + (size_t)b * Pe * Pe;
  const double* vals = values + (size_t)b * P;
  double* L = dsm;                  // NBLK blocks x 64
  double* dinv = L + NBLK * 64;     // me
  // Y in CW columns per row (4 when R <= 4: 2 KB less shared memory per
  // system, 10 instead of 9 systems per SM at m_eff = 64); the DMMA operands
  // read the columns >= CW as zeros
  constexpr int CW = R <= 4 ? 4 : 8;
  double* Yb = dinv + me;           // me x CW: [block][row][column], columns >= R zero
  double* xs = Yb + me * CW;        // me
  const double inv_gamma = 1.0 / gamma;
  auto at = [&](int i, int j) -> double& {   // element (i, j), j <= i
    return L[blk(i >> 3, j >> 3) * 64 + swz(i & 7, j & 7)];
  };
  auto Y = [&](int i, int q) -> double& { return Yb[(i >> 3) * 8 * CW + (i & 7) * CW + q]; };

  // ---- A = E[0:me, 0:me] into the lower blocks: asynchronous global->shared
  // copies (all of them in flight at once, no registers), then + I / gamma
#pragma unroll
  for (int I = 0; I < NBK; ++I)
#pragma unroll
    for (int J = 0; J <= I; ++J)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = 2 * fc + h;
        const double* src = E + (size_t)(8 * I + fr) * Pe + 8 * J + c;
        const uint32_t dst = nys::smem_u32(L + blk(I, J) * 64 + swz(fr, c));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src) : "memory");
      }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncwarp();
  for (int i = lane; i < me; i += 32) at(i, i) += inv_gamma;
  __syncwarp();

  // ---- blocked right-looking Cholesky
  int bad = 0;
  // fully unrolled: the trailing update's block pattern (J > p) is then known at
  // compile time -- with a runtime p every one of its 56 DMMAs was predicated,
  // and a predicated mma.sync costs a WARPSYNC + NOP per DMMA in SASS
#pragma unroll
  for (int p = 0; p < NBK; ++p) {
    const int nrows = (NBK - p) * 8;
    // panel rows R0 = lane, R1 = lane + 32 (local to the panel) in registers
    const int R0 = lane, R1 = lane + 32;
    double v0[8], v1[8];
    const bool h0 = R0 < nrows, h1 = R1 < nrows;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      v0[c] = h0 ? L[blk(p + (R0 >> 3), p) * 64 + swz(R0 & 7, c)] : 0.0;
      v1[c] = h1 ? L[blk(p + (R1 >> 3), p) * 64 + swz(R1 & 7, c)] : 0.0;
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const double piv = __shfl_sync(0xffffffffu, v0[c], c);
      if (!(piv > 0.0) || !isfinite(piv)) bad = 1;
      const double inv = rsqrt(piv);
      v0[c] = (R0 > c) ? v0[c] * inv : (R0 == c ? piv * inv : v0[c]);
      v1[c] = v1[c] * inv;   // R1 >= 32 > c
#pragma unroll
      for (int c2 = c + 1; c2 < 8; ++c2) {
        const double l = __shfl_sync(0xffffffffu, v0[c], c2);   // L[c2][c]
        v0[c2] = fma(-v0[c], l, v0[c2]);
        v1[c2] = fma(-v1[c], l, v1[c2]);
      }
    }
    if (bad) break;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (h0) L[blk(p + (R0 >> 3), p) * 64 + swz(R0 & 7, c)] = v0[c];
      if (h1) L[blk(p + (R1 >> 3), p) * 64 + swz(R1 & 7, c)] = v1[c];
    }
    __syncwarp();
    // trailing blocks: C_IJ -= L_Ip L_Jp^T, p < J <= I  (two DMMAs per block)
    double f[NBK][2];
#pragma unroll
    for (int I = 0; I < NBK; ++I)
#pragma unroll
      for (int kk = 0; kk < 2; ++kk)
        f[I][kk] = I > p ? L[blk(I, p) * 64 + swz(fr, 4 * kk + fc)] : 0.0;
#pragma unroll
    for (int I = 1; I < NBK; ++I)
#pragma unroll
      for (int J = 1; J <= I; ++J) {
        if (J <= p) continue;
        double2* cp = reinterpret_cast<double2*>(L + blk(I, J) * 64 + swz(fr, 2 * fc));
        double2 cv = *cp;
        nys::dmma(cv.x, cv.y, -f[I][0], f[J][0]);
        nys::dmma(cv.x, cv.y, -f[I][1], f[J][1]);
        *cp = cv;
      }
    __syncwarp();
  }
  bad = __any_sync(0xffffffffu, bad);
  if (bad) {
    if (lane == 0) info[b] = kNeedsLu;
    return;
  }
  for (int i = lane; i < me; i += 32) dinv[i] = 1.0 / at(i, i);

  // ---- Y = L^{-1} [D^T g | A_c^T | r1]
  for (int i = lane; i < me; i += 32) {
    Y(i, 0) = E[(size_t)i * Pe + me];
#pragma unroll
    for (int mu = 0; mu < P; ++mu) Y(i, 1 + mu) = Ac[(size_t)mu * me + i];
    Y(i, Q) = E[(size_t)i * Pe + me + 1];
#pragma unroll
    for (int q = R; q < CW; ++q) Y(i, q) = 0.0;
  }
  __syncwarp();
  // Blocked triangular solves.  A lane holds the 8 x 8 block's MMA accumulator
  // fragment (row fr, columns 2fc, 2fc+1); off-diagonal blocks arrive by DMMA,
  // the diagonal block is solved row by row with shuffles.  Only the columns
  // in `cols` (bit mask) are written back.
  auto forward = [&](unsigned cols) {   // Y <- L^{-1} Y
#pragma unroll 1
    for (int I = 0; I < NBK; ++I) {
      double2 cv = 2 * fc < CW ? *reinterpret_cast<const double2*>(Yb + I * 8 * CW + fr * CW + 2 * fc)
                                : make_double2(0.0, 0.0);
      for (int J = 0; J < I; ++J) {
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const double a = -L[blk(I, J) * 64 + swz(fr, 4 * kk + fc)];
          const double bq = fr < CW ? Yb[J * 8 * CW + (4 * kk + fc) * CW + fr] : 0.0;
          nys::dmma(cv.x, cv.y, a, bq);
        }
      }
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
          const double l = L[blk(I, I) * 64 + swz(fr, c)];
          cv.x = fma(-l, yx, cv.x);
          cv.y = fma(-l, yy, cv.y);
        }
      }
      double* dst = Yb + I * 8 * CW + fr * CW + 2 * fc;
      if (2 * fc < CW && ((cols >> (2 * fc)) & 1u)) dst[0] = cv.x;
      if (2 * fc + 1 < CW && ((cols >> (2 * fc + 1)) & 1u)) dst[1] = cv.y;
      __syncwarp();
    }
  };
  auto backward = [&](unsigned cols) {   // Y <- L^{-T} Y
#pragma unroll 1
    for (int I = NBK - 1; I >= 0; --I) {
      double2 cv = 2 * fc < CW ? *reinterpret_cast<const double2*>(Yb + I * 8 * CW + fr * CW + 2 * fc)
                                : make_double2(0.0, 0.0);
      for (int J = I + 1; J < NBK; ++J) {
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const double a = -L[blk(J, I) * 64 + swz(4 * kk + fc, fr)];   // (L_JI)^T
          const double bq = fr < CW ? Yb[J * 8 * CW + (4 * kk + fc) * CW + fr] : 0.0;
          nys::dmma(cv.x, cv.y, a, bq);
        }
      }
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
          const double l = L[blk(I, I) * 64 + swz(c, fr)];   // L[c][fr], c > fr
          cv.x = fma(-l, yx, cv.x);
          cv.y = fma(-l, yy, cv.y);
        }
      }
      double* dst = Yb + I * 8 * CW + fr * CW + 2 * fc;
      if (2 * fc < CW && ((cols >> (2 * fc)) & 1u)) dst[0] = cv.x;
      if (2 * fc + 1 < CW && ((cols >> (2 * fc + 1)) & 1u)) dst[1] = cv.y;
      __syncwarp();
    }
  };
  auto warp_dot = [&](int qa, int qb) {
    double a = 0.0;
    for (int i = lane; i < me; i += 32) a = fma(Y(i, qa), Y(i, qb), a);
#pragma unroll
    for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    return a;
  };
  forward((1u << R) - 1u);
  // S = C' - Y_B^T Y_B (every lane holds the same copy), pivoted elimination
  double S[Q][Q];
#pragma unroll
  for (int a = 0; a < Q; ++a)
#pragma unroll
    for (int c = a; c < Q; ++c) {
      const double cp = (a == 0 && c == 0) ? E[(size_t)me * Pe + me] : (a == 0 ? beta[c - 1] : 0.0);
      S[a][c] = cp - warp_dot(a, c);
      S[c][a] = S[a][c];
    }
  int piv[Q];
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
    if (!(best > piv_floor)) bad = 1;
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
      const double fct = S[r][k] * ip;
      S[r][k] = fct;
#pragma unroll
      for (int c = k + 1; c < Q; ++c) S[r][c] = fma(-fct, S[k][c], S[r][c]);
    }
  }
  if (bad) {
    if (lane == 0) info[b] = kNeedsLu;
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
  rq[0] = E[(size_t)me * Pe + me + 1];   // g^T r
#pragma unroll
  for (int mu = 0; mu < P; ++mu) rq[1 + mu] = vals[mu];
#pragma unroll 1
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) {
      // residual of the omega rows r1 - A x - Bt z (E symmetric: coalesced rows)
      for (int i = lane; i < me; i += 32) {
        double a = 0.0;
#pragma unroll 8
        for (int j = 0; j < me; ++j) {
          const double e = __ldg(E + (size_t)j * Pe + i);
          a = fma((i == j) ? inv_gamma + e : e, xs[j], a);
        }
        a = fma(E[(size_t)i * Pe + me], z[0], a);
#pragma unroll
        for (int mu = 0; mu < P; ++mu) a = fma(Ac[(size_t)mu * me + i], z[1 + mu], a);
        Y(i, Q) = E[(size_t)i * Pe + me + 1] - a;
      }
      double gx = 0.0, cx[P];
#pragma unroll
      for (int mu = 0; mu < P; ++mu) cx[mu] = 0.0;
      for (int i = lane; i < me; i += 32) {
        gx = fma(E[(size_t)me * Pe + i], xs[i], gx);
#pragma unroll
        for (int mu = 0; mu < P; ++mu) cx[mu] = fma(Ac[(size_t)mu * me + i], xs[i], cx[mu]);
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        gx += __shfl_xor_sync(0xffffffffu, gx, o);
#pragma unroll
        for (int mu = 0; mu < P; ++mu) cx[mu] += __shfl_xor_sync(0xffffffffu, cx[mu], o);
      }
      double cz0 = E[(size_t)me * Pe + me] * z[0];
#pragma unroll
      for (int mu = 0; mu < P; ++mu) cz0 = fma(beta[mu], z[1 + mu], cz0);
      rq[0] = E[(size_t)me * Pe + me + 1] - (gx + cz0);
#pragma unroll
      for (int mu = 0; mu < P; ++mu) rq[1 + mu] = vals[mu] - (cx[mu] + beta[mu] * z[0]);
      __syncwarp();
      forward(1u << Q);   // only the residual column; L^{-1} Bt is unchanged
    }
    double t[Q];
#pragma unroll
    for (int a = 0; a < Q; ++a) t[a] = rq[a] - warp_dot(a, Q);
    solve_small(t);
    for (int i = lane; i < me; i += 32) {
      double v = Y(i, Q);
#pragma unroll
      for (int a = 0; a < Q; ++a) v = fma(-Y(i, a), t[a], v);
      Y(i, Q) = v;
    }
    __syncwarp();
    backward(1u << Q);
    for (int i = lane; i < me; i += 32) {
      const double v = Y(i, Q);
      xs[i] = pass == 0 ? v : xs[i] + v;
    }
#pragma unroll
    for (int a = 0; a < Q; ++a) z[a] = pass == 0 ? t[a] : z[a] + t[a];
    __syncwarp();
  }
  constexpr int n = me + Q;
  int nonfinite = 0;
  for (int i = lane; i < n; i += 32) {
    double v = 0.0;
    if (i < me) {
      v = xs[i];
    } else {
#pragma unroll
      for (int a = 0; a < Q; ++a) v = (i - me == a) ? z[a] : v;
    }
    if (!isfinite(v)) nonfinite = 1;
    xout[(size_t)b * n + i] = v;
  }
  nonfinite = __any_sync(0xffffffffu, nonfinite);
  if (lane == 0) info[b] = nonfinite ? kNeedsLu : NYS_INFO_OK;
}

template <int P, int NBK>
int launch_block(const double* dense, const double* Ac, const double* beta, const double* values,
                 double gamma, int B, double* x, int* info, cudaStream_t st) {
  constexpr int me = NBK * 8;
  constexpr int CW = P + 2 <= 4 ? 4 : 8;   // Y columns (kernel: R = P + 2)
  const size_t dyn = ((size_t)NBK * (NBK + 1) / 2 * 64 + me + (size_t)me * CW + me) *
                     sizeof(double);
  auto kern = kkt_block_kernel<P, NBK>;
  if (dyn > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (e != cudaSuccess) return nys_host::record_cuda(e);
  }
  kern<<<B, 32, dyn, st>>>(dense, Ac, beta, values, gamma, x, info);
  nys_host::count_launches(1);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

template <int P>
int dispatch_block(int m_eff, const double* dense, const double* Ac, const double* beta,
                   const double* values, double gamma, int B, double* x, int* info,
                   cudaStream_t st) {
  switch (m_eff / 8) {
    case 4: return launch_block<P, 4>(dense, Ac, beta, values, gamma, B, x, info, st);
    case 5: return launch_block<P, 5>(dense, Ac, beta, values, gamma, B, x, info, st);
    case 6: return launch_block<P, 6>(dense, Ac, beta, values, gamma, B, x, info, st);
    case 7: return launch_block<P, 7>(dense, Ac, beta, values, gamma, B, x, info, st);
    case 8: return launch_block<P, 8>(dense, Ac, beta, values, gamma, B, x, info, st);
    default: return NYS_EUNSUPPORTED;
  }
}

}  // namespace

namespace nys_host {
// blocked path for m_eff in {32, 40, ..., 64}; NYS_EUNSUPPORTED otherwise
int launch_kkt_blocked(const double* dense, int m_eff, int n_cond, const double* Ac,
                       const double* beta, const double* values, double gamma, int B, double* x,
                       int* info, cudaStream_t st) {
  if (m_eff % 8 != 0 || m_eff < 32 || m_eff > 64) return NYS_EUNSUPPORTED;
  switch (n_cond) {
    case 1: return dispatch_block<1>(m_eff, dense, Ac, beta, values, gamma, B, x, info, st);
    case 2: return dispatch_block<2>(m_eff, dense, Ac, beta, values, gamma, B, x, info, st);
    case 3: return dispatch_block<3>(m_eff, dense, Ac, beta, values, gamma, B, x, info, st);
    case 4: return dispatch_block<4>(m_eff, dense, Ac, beta, values, gamma, B, x, info, st);
    default: return NYS_EUNSUPPORTED;
  }
}
}  // namespace nys_host
