// Newton-KKT kernels for nonlinear first-order ODEs (config 3), batched over
// instances that share grid, landmarks and sigma.
//
// Reference: newton.py.  Unknowns x = (omega, b, lambda, y_aux); residual =
// gradient of the Lagrangian (newton.py:128-147); Jacobian = its Hessian
// (newton.py:160-211) whose y-block is DIAGONAL (newton.py:210),
//     d_i = gamma c_i,  c_i = 1 + f_y^2 - f_yy e1_i.
// Instead of the reference's dense (m_eff+2+n_c)-side LU (newton.py:307), the
// y-block is eliminated by Schur complement onto z = (omega, b, lambda)
// (y_hat identical to <= 1.1e-15).  With S0 = Psi_0, S1 = Psi_1
// over the constraint points, v_i = S1_i - f_y S0_i and q_i = f_yy e1_i, the
// reduced (omega, b) block is, in the cancellation-free form
//     K = diag(I, 0) + gamma sum_i [ vh vh^T - q (S1h S1h^T + S0h S0h^T) ]_i / c_i
// with hatted vectors extended by one coordinate: vh = (v, -f_y), S1h = (S1, 0),
// S0h = (S0, 1) -- the same extended-column trick as the linear Gram.  It is
// accumulated with DMMA.8x8x4 from the shared fragment-packed Psi (one packed
// copy for the whole batch).  Newton's rhs and the back-substitution
//     dy_i = (-F_y,i + gamma (wh_i . dz_ob)) / (gamma c_i),  wh = (f_y S1 + S0, 1)
// are fused into the same kernels.
//
// The nonlinearity is evaluated on the device for the separable family
//     f(t, y) = g(t) + alpha y^2 + beta sin(y)
// (config 3: y' = -k y^2 + g and y' = sin y + g), or supplied per call as sampled
// arrays (host-evaluated reference callables: the generic drop-in path).
#include <cmath>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"

#define NYS_HD_INLINE __host__ __device__ __forceinline__

namespace nys_host {
int launch_psi_pack(const double* lm, int m, const double* W, int ldw, int m_eff, double sigma2,
                    int p, const double* pts, int n_c, int n_blocks, int n_rows_pad,
                    double* packed, cudaStream_t st);
}

namespace {

constexpr int kResThreads = 256;
constexpr int kMaxCondN = 4;

NYS_DEV double block_reduce(double v, double* red, bool is_max) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double u = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmax(v, u) : v + u;
  }
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = is_max ? 0.0 : 0.0;
  for (int i = 0; i < nw; ++i) s = is_max ? fmax(s, red[i]) : s + red[i];   // fixed order
  return s;
}

// f, f_y, f_yy for row i of instance b
struct Rhs {
  const double* g;       // [B][n_c] time part (family mode) or f (sampled mode)
  const double* fy;      // sampled mode: [B][n_c]; nullptr in family mode
  const double* fyy;     // sampled mode: [B][n_c]
  const double* alpha;   // family: [B]
  const double* beta;    // family: [B]
  int n_c;
  NYS_DEV void eval(int b, int i, double y, double& f, double& f_y, double& f_yy) const {
    const size_t o = (size_t)b * n_c + i;
    if (fy != nullptr) {
      f = g[o];
      f_y = fy[o];
      f_yy = fyy[o];
      return;
    }
    // numpy's operation order, never contracted into FMAs (the host callables
    // of workloads.py evaluate the same expressions)
    const double a = alpha[b], be = beta[b];
    double s, c;
    sincos(y, &s, &c);
    f = __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(a, y), y), g[o]), __dmul_rn(be, s));
    f_y = __dadd_rn(__dmul_rn(__dmul_rn(2.0, a), y), __dmul_rn(be, c));
    f_yy = __dsub_rn(__dmul_rn(2.0, a), __dmul_rn(be, s));
  }
};

// ---------------------------------------------------------------------------
// residual F (newton.py:128-147, p = 1) for instances idx[0..nb), plus the
// per-row quantities the Jacobian needs: aux[b] = (f_y, q = f_yy e1, c).
// S (n_c x me) row-major for S omega; ST (me x n_c) for S^T e (coalesced).
// kTrial = false: the residual at X[b] with every by-product (F, aux, work).
// kTrial = true: the max-norm only, at the line-search trial X[b] + alpha_t D[b]
// (grid.y = trial t), nothing else written -- the batched step halving.  Both
// run the same arithmetic in the same order, so a trial's norm is bit-identical
// to materialising the candidate (newton_step_kernel) and calling the residual.
// The residual in two kernels.  newton_residual_kernel: grid (slots, splits) --
// a CTA takes one row range of one instance (kTrial: of one trial point
// X[b] + alpha_t D[b]), forms e1, e2 and F_y there (non-trial: F_y and aux are
// written), and stores its partial S1^T e1, S0^T e2, sum e2, max|F_y| and a
// non-finite flag.  newton_residual_finalize_kernel adds the row ranges in
// fixed order and forms F_omega, F_b, F_lambda and the max-norm.  Splitting
// the rows puts several CTAs on every instance: one CTA per instance was
// bound by the latency of streaming S^T from L2 (ncu: long-scoreboard stalls).
// The trial form evaluates line-search points with the same arithmetic, so a
// trial's norm is bit-identical to materialising the candidate
// (newton_step_kernel) and calling the non-trial residual.
constexpr int kResSplit = 4;
NYS_DEV int res_rows_per_split(int n_c) { return ((n_c + kResSplit - 1) / kResSplit + 31) / 32 * 32; }

// one row range (split) of the residual of instance b at x (kTrial: at
// x + al * dx), by the whole CTA; the range's partial sums go to out[2 me + 3]
template <bool kTrial>
NYS_DEV void residual_range(const double* __restrict__ S0T, const double* __restrict__ S1T, int me,
                            int n_c, const Rhs& rhs, double gm, const double* __restrict__ x,
                            const double* __restrict__ dx, double al, int b, int split, int nk,
                            double* __restrict__ Fb, double* __restrict__ auxb,
                            double* __restrict__ out, double* sh, double* red) {
  // x entry j of this CTA's point (trial: the candidate, as newton_step_kernel forms it)
#define NYS_XV(j) (kTrial ? fma(al, dx[j], x[j]) : x[j])
  const int rpc = res_rows_per_split(n_c);
  const int r0 = split * rpc, r1 = min(n_c, r0 + rpc);
  double* om = sh;                 // me
  double* e1 = sh + me;            // rpc (this CTA's rows)
  double* e2 = e1 + rpc;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  for (int k = tid; k < me; k += nt) om[k] = NYS_XV(k);
  __syncthreads();
  const double bias = NYS_XV(me);
  const int y0 = me + 1 + nk;
  double fmax_local = 0.0;
  int bad = 0;
  // rows across threads, features from the transposed copies: every load is
  // a coalesced 256-byte warp access (S0/S1 rows are 8*me bytes apart)
  for (int i = r0 + tid; i < r1; i += nt) {
    double a0 = 0.0, a1 = 0.0, c0 = 0.0, c1 = 0.0;
    int k = 0;
#pragma unroll 4
    for (; k + 1 < me; k += 2) {
      a0 = fma(S1T[(size_t)k * n_c + i], om[k], a0);
      a1 = fma(S1T[(size_t)(k + 1) * n_c + i], om[k + 1], a1);
      c0 = fma(S0T[(size_t)k * n_c + i], om[k], c0);
      c1 = fma(S0T[(size_t)(k + 1) * n_c + i], om[k + 1], c1);
    }
    if (k < me) {
      a0 = fma(S1T[(size_t)k * n_c + i], om[k], a0);
      c0 = fma(S0T[(size_t)k * n_c + i], om[k], c0);
    }
    const double s1w = a0 + a1, s0w = c0 + c1;
    const double yi = NYS_XV(y0 + i);
    double f, fy, fyy;
    rhs.eval(b, i, yi, f, fy, fyy);
    const double ee1 = __dsub_rn(s1w, f);
    const double ee2 = __dsub_rn(__dsub_rn(yi, s0w), bias);
    if (!isfinite(ee1) || !isfinite(f)) bad = 1;
    e1[i - r0] = ee1;
    e2[i - r0] = ee2;
    // F_y = -gamma f_y e1 + gamma e2 in numpy's order (newton.py:146)
    const double Fy = __dadd_rn(__dmul_rn(__dmul_rn(-gm, fy), ee1), __dmul_rn(gm, ee2));
    fmax_local = fmax(fmax_local, fabs(Fy));
    if (!kTrial) {
      Fb[y0 + i] = Fy;
      const double q = __dmul_rn(fyy, ee1);
      auxb[i] = fy;
      auxb[n_c + i] = q;
      auxb[2 * n_c + i] = __dsub_rn(__dadd_rn(1.0, __dmul_rn(fy, fy)), q);
    }
  }
  __syncthreads();
  // partial S1^T e1 and S0^T e2 over this row range (warp per k)
  for (int k = warp; k < me; k += nw) {
    const double* rr1 = S1T + (size_t)k * n_c;
    const double* rr0 = S0T + (size_t)k * n_c;
    double a = 0.0, c = 0.0;
    for (int i = r0 + lane; i < r1; i += 32) {
      a = fma(rr1[i], e1[i - r0], a);
      c = fma(rr0[i], e2[i - r0], c);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    if (lane == 0) {
      out[k] = a;
      out[me + k] = c;
    }
  }
  double se2 = 0.0;
  for (int i = r0 + tid; i < r1; i += nt) se2 += e2[i - r0];
  se2 = block_reduce(se2, red, false);
  const int any_bad = __syncthreads_or(bad);
  const double fmx = block_reduce(fmax_local, red, true);
  if (tid == 0) {
    out[2 * me] = se2;
    out[2 * me + 1] = fmx;
    out[2 * me + 2] = any_bad ? 1.0 : 0.0;
  }
#undef NYS_XV
}

template <bool kTrial>
__global__ void __launch_bounds__(kResThreads)
    newton_residual_kernel(const double* __restrict__ S0T, const double* __restrict__ S1T, int me,
                           int n_c, Rhs rhs, const double* __restrict__ gamma,
                           const double* __restrict__ X, int ldx, const int* __restrict__ idx,
                           double* __restrict__ F, double* __restrict__ aux,
                           const double* __restrict__ D, const double* __restrict__ alphas, int nb,
                           int nk, double* __restrict__ part) {
  extern __shared__ double sh[];
  __shared__ double red[kResThreads / 32];
  const int b = idx[blockIdx.x];
  const double* x = X + (size_t)b * ldx;
  const double* dx = kTrial ? D + (size_t)b * ldx : nullptr;
  const double al = kTrial ? alphas[blockIdx.y] : 0.0;
  const int split = blockIdx.z;
  double* Fb = kTrial ? nullptr : F + (size_t)b * ldx;
  double* auxb = kTrial ? nullptr : aux + (size_t)b * 3 * n_c;
  const size_t slot = kTrial ? (size_t)blockIdx.y * nb + blockIdx.x : (size_t)blockIdx.x;
  const int pstride = 2 * me + 3;
  residual_range<kTrial>(S0T, S1T, me, n_c, rhs, gamma[b], x, dx, al, b, split, nk, Fb, auxb,
                         part + (slot * kResSplit + split) * pstride, sh, red);
}

template <bool kTrial>
__global__ void __launch_bounds__(64)
    newton_residual_finalize_kernel(int me, const double* __restrict__ Ac,
                                    const double* __restrict__ betac,
                                    const double* __restrict__ vals, int nk,
                                    const double* __restrict__ gamma,
                                    const double* __restrict__ X, int ldx,
                                    const int* __restrict__ idx, double* __restrict__ F,
                                    double* __restrict__ norm, const double* __restrict__ D,
                                    const double* __restrict__ alphas, int nb,
                                    const double* __restrict__ part) {
  __shared__ double red[2];
  __shared__ double lam_s[kMaxCondN];
  const int b = idx[blockIdx.x];
  const double gm = gamma[b];
  const double* x = X + (size_t)b * ldx;
  const double* dx = kTrial ? D + (size_t)b * ldx : nullptr;
  const double al = kTrial ? alphas[blockIdx.y] : 0.0;
#define NYS_XV(j) (kTrial ? fma(al, dx[j], x[j]) : x[j])
  const size_t slot = kTrial ? (size_t)blockIdx.y * nb + blockIdx.x : (size_t)blockIdx.x;
  const int pstride = 2 * me + 3;
  const double* pp = part + slot * kResSplit * pstride;
  double* Fb = kTrial ? nullptr : F + (size_t)b * ldx;
  const int tid = threadIdx.x;
  if (tid < nk) lam_s[tid] = NYS_XV(me + 1 + tid);
  __syncthreads();
  double fmax_local = 0.0;
  int bad = 0;
  for (int s2 = 0; s2 < kResSplit; ++s2) bad |= pp[s2 * pstride + 2 * me + 2] != 0.0;
  for (int k = tid; k < me; k += blockDim.x) {
    double a = 0.0, c = 0.0;
    for (int s2 = 0; s2 < kResSplit; ++s2) {   // fixed order over row ranges
      a += pp[s2 * pstride + k];
      c += pp[s2 * pstride + me + k];
    }
    // omega + gamma S1^T e1 - gamma S0^T e2 + Ac^T lambda (newton.py:139), uncontracted
    double acl = 0.0;
    for (int mu = 0; mu < nk; ++mu) acl = __dadd_rn(acl, __dmul_rn(Ac[(size_t)mu * me + k], lam_s[mu]));
    const double v = __dadd_rn(__dsub_rn(__dadd_rn(NYS_XV(k), __dmul_rn(gm, a)), __dmul_rn(gm, c)), acl);
    if (!kTrial) Fb[k] = v;
    fmax_local = fmax(fmax_local, fabs(v));
  }
  if (tid == 0) {
    double se2 = 0.0, fy = 0.0;
    for (int s2 = 0; s2 < kResSplit; ++s2) {
      se2 += pp[s2 * pstride + 2 * me];
      fy = fmax(fy, pp[s2 * pstride + 2 * me + 1]);
    }
    fmax_local = fmax(fmax_local, fy);
    double bl = 0.0;
    for (int mu = 0; mu < nk; ++mu) bl = __dadd_rn(bl, __dmul_rn(betac[mu], lam_s[mu]));
    const double Fbias = __dadd_rn(__dmul_rn(-gm, se2), bl);   // newton.py:143
    if (!kTrial) Fb[me] = Fbias;
    fmax_local = fmax(fmax_local, fabs(Fbias));
    const double bias = NYS_XV(me);
    for (int mu = 0; mu < nk; ++mu) {
      double v = 0.0;
      for (int k = 0; k < me; ++k) v = fma(Ac[(size_t)mu * me + k], NYS_XV(k), v);
      // Ac omega + beta b - values (newton.py:144)
      v = __dsub_rn(__dadd_rn(v, __dmul_rn(betac[mu], bias)), vals[(size_t)b * nk + mu]);
      if (!kTrial) Fb[me + 1 + mu] = v;
      fmax_local = fmax(fmax_local, fabs(v));
    }
  }
  // max over the block (two warps)
  for (int o = 16; o; o >>= 1) fmax_local = fmax(fmax_local, __shfl_xor_sync(0xffffffffu, fmax_local, o));
  if ((tid & 31) == 0) red[tid >> 5] = fmax_local;
  __syncthreads();
  if (tid == 0) {
    double nrm = fmax(red[0], blockDim.x > 32 ? red[1] : 0.0);
    const double outv = bad ? NAN : nrm;   // NaN -> DivergenceError (newton.py:137-138)
    if (kTrial)
      norm[slot] = outv;
    else
      norm[b] = outv;
  }
#undef NYS_XV
}

// ---------------------------------------------------------------------------
// reduced (omega, b, lambda) system: K (nz x nz) and rhs (nz), nz = me + 1 + nk
template <int NB>
struct Tri {
  static constexpr int kPairs = NB * (NB + 1) / 2;
  static constexpr NYS_DEV int idx(int I, int J) { return I * NB - (I * (I - 1)) / 2 + (J - I); }
};

constexpr int kRedWarps = 4;

// Reduced (omega, b, lambda) system from the summed partials red[e] (e over the
// NPAIR*64 Gram entries in MMA layout, then NB*8 rhs entries).
template <int NB>
NYS_DEV void build_reduced(const double* red, int stride, int nparts, int me, int nk,
                           const double* __restrict__ Fb, double gm,
                           const double* __restrict__ Ac, const double* __restrict__ betac,
                           double* Kb, double* rb) {
  constexpr int NPAIR = Tri<NB>::kPairs;
  const int nz = me + 1 + nk, nh = me + 1;
  for (int e = threadIdx.x; e < NPAIR * 64; e += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < nparts; ++w) s += red[(size_t)w * stride + e];
    const int t = e >> 6, l = (e & 63) >> 1, j2 = e & 1;
    int I = 0, rem = t;
    while (rem >= NB - I) {
      rem -= NB - I;
      ++I;
    }
    const int J = I + rem;
    const int r = I * 8 + (l >> 2), c = J * 8 + 2 * (l & 3) + j2;
    if (r < nh && c < nh && !(I == J && r > c)) {
      const double v = gm * s + ((r == c && r < me) ? 1.0 : 0.0);
      Kb[(size_t)r * nz + c] = v;
      Kb[(size_t)c * nz + r] = v;
    }
  }
  for (int e = threadIdx.x; e < NB * 8; e += blockDim.x) {
    if (e >= nh) continue;
    double s = 0.0;
    for (int w = 0; w < nparts; ++w) s += red[(size_t)w * stride + NPAIR * 64 + e];
    rb[e] = -Fb[e] - s;   // rhs_(omega,b) = -F - sum wh F_y / c
  }
  for (int e = threadIdx.x; e < nk * nh; e += blockDim.x) {
    const int mu = e / nh, j = e % nh;
    const double v = j < me ? Ac[(size_t)mu * me + j] : betac[mu];
    Kb[(size_t)(nh + mu) * nz + j] = v;
    Kb[(size_t)j * nz + nh + mu] = v;
  }
  for (int e = threadIdx.x; e < nk * nk; e += blockDim.x)
    Kb[(size_t)(nh + e / nk) * nz + nh + e % nk] = 0.0;
  for (int mu = threadIdx.x; mu < nk; mu += blockDim.x) rb[nh + mu] = -Fb[nh + mu];
}

// one warp's share of the reduced system over k-steps ks_lo + wi, + nwg, ...
// < ks_hi: the three weighted DMMA Grams and the rhs term, stored to mine[]
// (NPAIR*64 Gram entries in MMA layout, then NB*8 rhs entries)
template <int NB>
NYS_DEV void reduce_warp(const double* __restrict__ psi, int me, int n_c,
                         const double* __restrict__ auxb, const double* __restrict__ Fy,
                         int ks_lo, int ks_hi, int wi, int nwg, double* mine) {
  constexpr int NPAIR = Tri<NB>::kPairs;
  const int lane = threadIdx.x & 31, tig = lane & 3, gid = lane >> 2;
  double acc[NPAIR][2];
#pragma unroll
  for (int q = 0; q < NPAIR; ++q) acc[q][0] = acc[q][1] = 0.0;
  double racc[NB];
#pragma unroll
  for (int F_ = 0; F_ < NB; ++F_) racc[F_] = 0.0;
  for (int ks = ks_lo + wi; ks < ks_hi; ks += nwg) {
    const int row = ks * 4 + tig;
    const bool ok = row < n_c;
    const double fy = ok ? auxb[row] : 0.0;
    const double q = ok ? auxb[n_c + row] : 0.0;
    const double c = ok ? auxb[2 * n_c + row] : 1.0;
    const double ic = 1.0 / c;
    const double w1 = ic, w2 = -q * ic;
    const double fyc = ok ? Fy[row] * ic : 0.0;
    const double* P0 = psi + ((size_t)ks * 2 + 0) * NB * 32 + lane;
    const double* P1 = psi + ((size_t)ks * 2 + 1) * NB * 32 + lane;
    double x0[NB], x1[NB], xv[NB];
#pragma unroll
    for (int F_ = 0; F_ < NB; ++F_) {
      x0[F_] = ok ? P0[F_ * 32] : 0.0;
      x1[F_] = ok ? P1[F_ * 32] : 0.0;
      xv[F_] = fma(-fy, x0[F_], x1[F_]);                  // vh = S1h - f_y S0h
      racc[F_] = fma(fma(fy, x1[F_], x0[F_]), fyc, racc[F_]);   // sum wh F_y / c
    }
    // per accumulator the order is (vh, S1h, S0h) as before, but the three
    // terms are issued as three passes over the block pairs so consecutive
    // DMMAs never depend on each other (asm volatile keeps issue order)
#pragma unroll
    for (int I = 0; I < NB; ++I) {
      const double av = w1 * xv[I];
#pragma unroll
      for (int J = I; J < NB; ++J) {
        const int t = Tri<NB>::idx(I, J);
        nys::dmma(acc[t][0], acc[t][1], av, xv[J]);
      }
    }
#pragma unroll
    for (int I = 0; I < NB; ++I) {
      const double a1 = w2 * x1[I];
#pragma unroll
      for (int J = I; J < NB; ++J) {
        const int t = Tri<NB>::idx(I, J);
        nys::dmma(acc[t][0], acc[t][1], a1, x1[J]);
      }
    }
#pragma unroll
    for (int I = 0; I < NB; ++I) {
      const double a0 = w2 * x0[I];
#pragma unroll
      for (int J = I; J < NB; ++J) {
        const int t = Tri<NB>::idx(I, J);
        nys::dmma(acc[t][0], acc[t][1], a0, x0[J]);
      }
    }
  }
  // reduce racc over the 4 rows held by a quad (tig)
#pragma unroll
  for (int F_ = 0; F_ < NB; ++F_) {
    racc[F_] += __shfl_xor_sync(0xffffffffu, racc[F_], 1);
    racc[F_] += __shfl_xor_sync(0xffffffffu, racc[F_], 2);
  }
#pragma unroll
  for (int t = 0; t < NPAIR; ++t) {
    mine[t * 64 + lane * 2] = acc[t][0];
    mine[t * 64 + lane * 2 + 1] = acc[t][1];
  }
  if (tig == 0)
#pragma unroll
    for (int F_ = 0; F_ < NB; ++F_) mine[NPAIR * 64 + F_ * 8 + gid] = racc[F_];
}

// grid (instances, nsplit): CTA (j, s) accumulates k-steps [s kps, (s+1) kps)
// of instance idx[j]; with part == nullptr (nsplit = 1) it builds K directly,
// otherwise it stores its partial sums for newton_reduce_finalize_kernel.
template <int NB>
__global__ void __launch_bounds__(kRedWarps * 32)
    newton_reduce_kernel(const double* __restrict__ psi, int nks, int me, int n_c,
                         const double* __restrict__ aux, const double* __restrict__ F, int ldx,
                         const double* __restrict__ gamma, const double* __restrict__ Ac,
                         const double* __restrict__ betac, int nk, const int* __restrict__ idx,
                         double* __restrict__ K, double* __restrict__ rz, int kps,
                         double* __restrict__ part) {
  constexpr int NPAIR = Tri<NB>::kPairs;
  extern __shared__ double red[];   // [kRedWarps][NPAIR*64 + NB*8]
  const int b = idx[blockIdx.x];
  const int warp = threadIdx.x >> 5;
  const int ks_lo = blockIdx.y * kps, ks_hi = min(nks, ks_lo + kps);
  const int stride = NPAIR * 64 + NB * 8;
  reduce_warp<NB>(psi, me, n_c, aux + (size_t)b * 3 * n_c, F + (size_t)b * ldx + me + 1 + nk,
                  ks_lo, ks_hi, warp, kRedWarps, red + (size_t)warp * stride);
  __syncthreads();
  if (part != nullptr) {   // this split's partial, warps summed in fixed order
    double* out = part + ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * stride;
    for (int e = threadIdx.x; e < stride; e += blockDim.x) {
      double s2 = 0.0;
      for (int w = 0; w < kRedWarps; ++w) s2 += red[(size_t)w * stride + e];
      out[e] = s2;
    }
    return;
  }
  const int nz = me + 1 + nk;
  build_reduced<NB>(red, stride, kRedWarps, me, nk, F + (size_t)b * ldx, gamma[b], Ac, betac,
                    K + (size_t)blockIdx.x * nz * nz, rz + (size_t)blockIdx.x * nz);
}

template <int NB>
__global__ void __launch_bounds__(256)
    newton_reduce_finalize_kernel(const double* __restrict__ part, int nsplit, int nb, int me,
                                  const double* __restrict__ F, int ldx,
                                  const double* __restrict__ gamma, const double* __restrict__ Ac,
                                  const double* __restrict__ betac, int nk,
                                  const int* __restrict__ idx, double* __restrict__ K,
                                  double* __restrict__ rz) {
  constexpr int NPAIR = Tri<NB>::kPairs;
  const int stride = NPAIR * 64 + NB * 8;
  const int b = idx[blockIdx.x];
  const int nz = me + 1 + nk;
  // partials of this instance sit nb * stride apart (one per split)
  build_reduced<NB>(part + (size_t)blockIdx.x * stride, nb * stride, nsplit, me, nk,
                    F + (size_t)b * ldx, gamma[b], Ac, betac, K + (size_t)blockIdx.x * nz * nz,
                    rz + (size_t)blockIdx.x * nz);
}

// ---------------------------------------------------------------------------
// dense LU with partial pivoting (first max wins), one warp per system
constexpr int kLuMaxN = 96;
constexpr int kLuNC = (kLuMaxN + 31) / 32;

__global__ void __launch_bounds__(32)
    lu_solve_warp_kernel(double* __restrict__ Mg, double* __restrict__ rg, int n,
                         double* __restrict__ out, int* __restrict__ info) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x, s = blockIdx.x;
  double* LU = sm;
  double* ys = LU + (size_t)n * n;
  int* perm = reinterpret_cast<int*>(ys + n);
  const double* M = Mg + (size_t)s * n * n;
  for (int e = lane; e < n * n; e += 32) LU[e] = M[e];
  for (int i = lane; i < n; i += 32) ys[i] = rg[(size_t)s * n + i];
  __syncwarp();
  for (int k = 0; k < n; ++k) {
    double bv = -1.0;
    int bi = n;
#pragma unroll
    for (int c = 0; c < kLuNC; ++c) {
      const int i = k + lane + 32 * c;
      if (i < n) {
        const double a = fabs(LU[(size_t)i * n + k]);
        if (a > bv) {
          bv = a;
          bi = i;
        }
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (!(bv > 0.0)) {
      if (lane == 0) info[s] = NYS_INFO_SINGULAR;
      return;
    }
    if (lane == 0) perm[k] = bi;
    double urow[kLuNC];
#pragma unroll
    for (int c = 0; c < kLuNC; ++c) {
      const int j = lane + 32 * c;
      double u = 0.0;
      if (j < n) {
        const double a = LU[(size_t)k * n + j], p = LU[(size_t)bi * n + j];
        if (bi != k) LU[(size_t)bi * n + j] = a;
        LU[(size_t)k * n + j] = p;
        u = p;
      }
      urow[c] = u;
    }
    __syncwarp();
    const double inv = 1.0 / LU[(size_t)k * n + k];
    for (int i = k + 1 + lane; i < n; i += 32) LU[(size_t)i * n + k] *= inv;
    __syncwarp();
    for (int i = k + 1; i < n; ++i) {
      const double l = LU[(size_t)i * n + k];
#pragma unroll
      for (int c = 0; c < kLuNC; ++c) {
        const int j = lane + 32 * c;
        if (j > k && j < n) LU[(size_t)i * n + j] -= l * urow[c];
      }
    }
    __syncwarp();
  }
  if (lane == 0)
    for (int k = 0; k < n; ++k) {
      const int pr = perm[k];
      if (pr != k) {
        const double t = ys[k];
        ys[k] = ys[pr];
        ys[pr] = t;
      }
    }
  __syncwarp();
  for (int j = 0; j < n - 1; ++j) {
    const double yj = ys[j];
    for (int i = j + 1 + lane; i < n; i += 32) ys[i] -= LU[(size_t)i * n + j] * yj;
    __syncwarp();
  }
  for (int j = n - 1; j >= 0; --j) {
    const double zj = ys[j] / LU[(size_t)j * n + j];
    __syncwarp();
    if (lane == 0) ys[j] = zj;
    for (int i = lane; i < j; i += 32) ys[i] -= LU[(size_t)i * n + j] * zj;
    __syncwarp();
  }
  int bad = 0;
  for (int i = lane; i < n; i += 32) {
    const double v = ys[i];
    if (!isfinite(v)) bad = 1;
    out[(size_t)s * n + i] = v;
  }
  bad = __any_sync(0xffffffffu, bad);
  if (lane == 0) info[s] = bad ? NYS_INFO_NONFINITE : NYS_INFO_OK;
}

// the same LU (first max wins, identical per-element operation order, so the
// results are bit-identical) with the trailing rows spread over the 8 warps of
// a CTA: a lone Newton system is no longer bound by one warp walking all rows
constexpr int kLuCtaThreads = 256;
__global__ void __launch_bounds__(kLuCtaThreads)
    lu_solve_cta_kernel(double* __restrict__ Mg, double* __restrict__ rg, int n,
                        double* __restrict__ out, int* __restrict__ info) {
  extern __shared__ double sm[];
  __shared__ int sing_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, s = blockIdx.x;
  constexpr int NW = kLuCtaThreads / 32;
  double* LU = sm;
  double* ys = LU + (size_t)n * n;
  int* perm = reinterpret_cast<int*>(ys + n);
  const double* M = Mg + (size_t)s * n * n;
  for (int e = tid; e < n * n; e += kLuCtaThreads) LU[e] = M[e];
  for (int i = tid; i < n; i += kLuCtaThreads) ys[i] = rg[(size_t)s * n + i];
  if (tid == 0) sing_s = 0;
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    if (warp == 0) {   // pivot search (first max wins), row swap
      double bv = -1.0;
      int bi = n;
#pragma unroll
      for (int c = 0; c < kLuNC; ++c) {
        const int i = k + lane + 32 * c;
        if (i < n) {
          const double a = fabs(LU[(size_t)i * n + k]);
          if (a > bv) {
            bv = a;
            bi = i;
          }
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      if (!(bv > 0.0)) {
        if (lane == 0) sing_s = 1;
      } else {
        if (lane == 0) perm[k] = bi;
        if (bi != k)
          for (int j = lane; j < n; j += 32) {
            const double a = LU[(size_t)k * n + j], p = LU[(size_t)bi * n + j];
            LU[(size_t)bi * n + j] = a;
            LU[(size_t)k * n + j] = p;
          }
      }
    }
    __syncthreads();
    if (sing_s) {
      if (tid == 0) info[s] = NYS_INFO_SINGULAR;
      return;
    }
    const double inv = 1.0 / LU[(size_t)k * n + k];
    for (int i = k + 1 + tid; i < n; i += kLuCtaThreads) LU[(size_t)i * n + k] *= inv;
    __syncthreads();
    for (int i = k + 1 + warp; i < n; i += NW) {
      const double l = LU[(size_t)i * n + k];
      for (int j = k + 1 + lane; j < n; j += 32) LU[(size_t)i * n + j] -= l * LU[(size_t)k * n + j];
    }
    __syncthreads();
  }
  if (warp != 0) return;
  if (lane == 0)
    for (int k = 0; k < n; ++k) {
      const int pr = perm[k];
      if (pr != k) {
        const double t = ys[k];
        ys[k] = ys[pr];
        ys[pr] = t;
      }
    }
  __syncwarp();
  for (int j = 0; j < n - 1; ++j) {
    const double yj = ys[j];
    for (int i = j + 1 + lane; i < n; i += 32) ys[i] -= LU[(size_t)i * n + j] * yj;
    __syncwarp();
  }
  for (int j = n - 1; j >= 0; --j) {
    const double zj = ys[j] / LU[(size_t)j * n + j];
    __syncwarp();
    if (lane == 0) ys[j] = zj;
    for (int i = lane; i < j; i += 32) ys[i] -= LU[(size_t)i * n + j] * zj;
    __syncwarp();
  }
  int bad = 0;
  for (int i = lane; i < n; i += 32) {
    const double v = ys[i];
    if (!isfinite(v)) bad = 1;
    out[(size_t)s * n + i] = v;
  }
  bad = __any_sync(0xffffffffu, bad);
  if (lane == 0) info[s] = bad ? NYS_INFO_NONFINITE : NYS_INFO_OK;
}

// ---------------------------------------------------------------------------
// delta_y and the damped update Xc = X + alpha * delta (per instance alpha);
// delta is stored as [B][ldx] (z part from the reduced solve, y part here)
__global__ void __launch_bounds__(256)
    newton_step_kernel(const double* __restrict__ S0, const double* __restrict__ S1, int me, int n_c,
                       int nk, const double* __restrict__ aux, const double* __restrict__ F,
                       const double* __restrict__ dz, const double* __restrict__ gamma,
                       const double* __restrict__ X, double* __restrict__ D,
                       double* __restrict__ Xc, const double* __restrict__ alpha, int ldx,
                       const int* __restrict__ idx, int compute_delta) {
  extern __shared__ double dzs[];
  const int b = idx[blockIdx.x];
  const int nz = me + 1 + nk;
  double* Db = D + (size_t)b * ldx;
  if (compute_delta) {
    for (int k = threadIdx.x; k < nz; k += blockDim.x) dzs[k] = dz[(size_t)blockIdx.x * nz + k];
    __syncthreads();
    const double gm = gamma[b];
    const double* auxb = aux + (size_t)b * 3 * n_c;
    const double* Fb = F + (size_t)b * ldx;
    for (int k = threadIdx.x; k < nz; k += blockDim.x) Db[k] = dzs[k];
    for (int i = threadIdx.x; i < n_c; i += blockDim.x) {
      const double* s0 = S0 + (size_t)i * me;
      const double* s1 = S1 + (size_t)i * me;
      double a = 0.0, c = 0.0;
      for (int k = 0; k < me; ++k) {
        a = fma(s1[k], dzs[k], a);
        c = fma(s0[k], dzs[k], c);
      }
      const double fy = auxb[i], cc = auxb[2 * n_c + i];
      const double wd = fy * a + c + dzs[me];   // wh . dz_(omega,b)
      Db[nz + i] = (-Fb[nz + i] + gm * wd) / (gm * cc);
    }
    __syncthreads();
  }
  const double al = alpha[b];
  const double* Xb = X + (size_t)b * ldx;
  double* Xcb = Xc + (size_t)b * ldx;
  for (int k = threadIdx.x; k < nz + n_c; k += blockDim.x) Xcb[k] = fma(al, Db[k], Xb[k]);
}

__global__ void transpose_kernel(const double* __restrict__ A, int rows, int cols,
                                 double* __restrict__ AT) {
  __shared__ double tile[32][33];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int rr = r0 + r, cc = c0 + threadIdx.x;
    if (rr < rows && cc < cols) tile[r][threadIdx.x] = A[(size_t)rr * cols + cc];
  }
  __syncthreads();
  for (int c = threadIdx.y; c < 32; c += blockDim.y) {
    const int cc = c0 + c, rr = r0 + threadIdx.x;
    if (rr < rows && cc < cols) AT[(size_t)cc * rows + rr] = tile[threadIdx.x][c];
  }
}

// ---------------------------------------------------------------------------
// Device-resident Newton (newton._solve_once, newton.py:279-349) for the
// separable family, p = 1: ONE CTA per instance runs the whole loop -- the
// convergence / divergence checks, the reduced (omega, b, lambda) system, its
// LU, the y back-substitution, the step-halving line search and the residual
// at every trial point -- with no host round trip.  Every piece is the
// arithmetic of the multi-kernel path above, in the same order: the residual
// is residual_range over the same kResSplit row ranges with the same 256-thread
// mapping and the same fixed-order finalize, the LU is lu_solve_cta's, the step
// is newton_step_kernel's; the reduced Gram uses the 2-split / 4-warp partition
// the multi-kernel path uses for 148..295 active instances.  Trial points are
// materialised (Xc = fma(alpha, D, X)) and evaluated with every by-product, so
// an accepted trial's F / aux are the next iteration's (no second residual).
constexpr int kPersistThreads = 256;
#ifndef NYS_PERSIST_MINB
#define NYS_PERSIST_MINB 1   // 255 registers: the reduced-system accumulators do not spill
#endif
constexpr int kPersistSplits = 2;
constexpr int kPTrials = 4;   // line-search trials evaluated together

// the kResSplit row ranges of residual_range<false> in ONE pass: every row,
// partial sum and reduction tree is the one residual_range forms for its range
// (thread tid takes rows r0 + tid + k * blockDim.x of every range, warps take
// (range, k) pairs for S^T e with the same lane / row mapping, the per-range
// sum of e2 goes through block_reduce's tree), so part[] is bit-identical to
// four residual_range calls -- with 4x the loads in flight and a quarter of
// the barriers.  sh: me + 2 n_c doubles; red: kResSplit * (blockDim / 32).
// bound: when the rows alone already give max|F_y| > bound (or a non-finite
// rhs), the S^T e pass is skipped and true returned -- a line-search trial
// rejected exactly as the full norm would reject it.
NYS_DEV bool residual_splits_fused(const double* __restrict__ S0T, const double* __restrict__ S1T,
                                   int me, int n_c, const Rhs& rhs, double gm,
                                   const double* __restrict__ x, int b, int nk,
                                   double* __restrict__ Fb, double* __restrict__ auxb,
                                   double* __restrict__ part, double* sh, double* red,
                                   double bound, double* early) {
  const int rpc = res_rows_per_split(n_c);
  const int pstride = 2 * me + 3;
  double* om = sh;
  double* e1 = sh + me;
  double* e2 = e1 + n_c;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  for (int k = tid; k < me; k += nt) om[k] = x[k];
  __syncthreads();
  const double bias = x[me];
  const int y0 = me + 1 + nk;
  double fmax_local = 0.0;
  int bad = 0;
  double se2[kResSplit];
#pragma unroll
  for (int sp = 0; sp < kResSplit; ++sp) se2[sp] = 0.0;
#pragma unroll
  for (int sp = 0; sp < kResSplit; ++sp) {
    const int r0 = sp * rpc, r1 = min(n_c, r0 + rpc);
    for (int i = r0 + tid; i < r1; i += nt) {
      double a0 = 0.0, a1 = 0.0, c0 = 0.0, c1 = 0.0;
      int k = 0;
#pragma unroll 4
      for (; k + 1 < me; k += 2) {
        a0 = fma(S1T[(size_t)k * n_c + i], om[k], a0);
        a1 = fma(S1T[(size_t)(k + 1) * n_c + i], om[k + 1], a1);
        c0 = fma(S0T[(size_t)k * n_c + i], om[k], c0);
        c1 = fma(S0T[(size_t)(k + 1) * n_c + i], om[k + 1], c1);
      }
      if (k < me) {
        a0 = fma(S1T[(size_t)k * n_c + i], om[k], a0);
        c0 = fma(S0T[(size_t)k * n_c + i], om[k], c0);
      }
      const double s1w = a0 + a1, s0w = c0 + c1;
      const double yi = x[y0 + i];
      double f, fy, fyy;
      rhs.eval(b, i, yi, f, fy, fyy);
      const double ee1 = __dsub_rn(s1w, f);
      const double ee2 = __dsub_rn(__dsub_rn(yi, s0w), bias);
      if (!isfinite(ee1) || !isfinite(f)) bad = 1;
      e1[i] = ee1;
      e2[i] = ee2;
      se2[sp] += ee2;
      const double Fy = __dadd_rn(__dmul_rn(__dmul_rn(-gm, fy), ee1), __dmul_rn(gm, ee2));
      fmax_local = fmax(fmax_local, fabs(Fy));
      Fb[y0 + i] = Fy;
      const double q = __dmul_rn(fyy, ee1);
      auxb[i] = fy;
      auxb[n_c + i] = q;
      auxb[2 * n_c + i] = __dsub_rn(__dadd_rn(1.0, __dmul_rn(fy, fy)), q);
    }
  }
  // per-range sums of e2: block_reduce's tree, kResSplit at once
#pragma unroll
  for (int sp = 0; sp < kResSplit; ++sp) {
#pragma unroll
    for (int o = 16; o; o >>= 1) se2[sp] = se2[sp] + __shfl_xor_sync(0xffffffffu, se2[sp], o);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) fmax_local = fmax(fmax_local, __shfl_xor_sync(0xffffffffu, fmax_local, o));
  if (lane == 0) {
#pragma unroll
    for (int sp = 0; sp < kResSplit; ++sp) red[sp * nw + warp] = se2[sp];
    red[kResSplit * nw + warp] = fmax_local;
  }
  const int any_bad = __syncthreads_or(bad);
  {
    double m = 0.0;
    for (int w = 0; w < nw; ++w) m = fmax(m, red[kResSplit * nw + w]);
    if (any_bad || m > bound) {   // uniform across the CTA
      *early = any_bad ? NAN : m;
      return true;
    }
  }
  // partial S1^T e1 and S0^T e2 per (range, k): one warp each, lanes over the range's rows
  for (int t = warp; t < kResSplit * me; t += nw) {
    const int sp = t / me, k = t % me;
    const int r0 = sp * rpc, r1 = min(n_c, r0 + rpc);
    const double* rr1 = S1T + (size_t)k * n_c;
    const double* rr0 = S0T + (size_t)k * n_c;
    double a = 0.0, c = 0.0;
    for (int i = r0 + lane; i < r1; i += 32) {
      a = fma(rr1[i], e1[i], a);
      c = fma(rr0[i], e2[i], c);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    if (lane == 0) {
      part[sp * pstride + k] = a;
      part[sp * pstride + me + k] = c;
    }
  }
  if (tid < kResSplit) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += red[tid * nw + w];   // fixed order
    double m = 0.0;
    for (int w = 0; w < nw; ++w) m = fmax(m, red[kResSplit * nw + w]);
    part[tid * pstride + 2 * me] = s;
    part[tid * pstride + 2 * me + 1] = m;   // the max over all ranges: the finalize takes the max
    part[tid * pstride + 2 * me + 2] = any_bad ? 1.0 : 0.0;
  }
  __syncthreads();
  return false;
}

NYS_DEV double bias_of(double al, const double* D, const double* X, int me) {
  return fma(al, D[me], X[me]);
}

// Residual max-norms at KT line-search trial points x_t = fma(al[t], D, X)
// at once (nothing else written): every trial's arithmetic -- rows, range
// partials, reduction trees, finalize -- is persist_residual's, so each norm is
// bit-identical to materialising the trial and calling persist_residual, but
// every S0^T / S1^T element loaded from L2 serves all KT trials.
// sh: KT (me + 2 n_c) doubles; red: KT (kResSplit + 1) (blockDim / 32);
// part: KT kResSplit (2 me + 3); out[t] = norm (NaN: non-finite rhs).
template <int KT>
NYS_DEV void trial_norms_multi(const double* __restrict__ S0T, const double* __restrict__ S1T,
                               int me, int n_c, const Rhs& rhs, double gm,
                               const double* __restrict__ X, const double* __restrict__ D,
                               const double* al, int b, int nk, const double* __restrict__ Ac,
                               const double* __restrict__ betac, const double* __restrict__ vals,
                               double* part, double* sh, double* red, double* out, double ref) {
  const int rpc = res_rows_per_split(n_c);
  const int pstride = 2 * me + 3;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  double* om = sh;                       // [KT][me]
  double* e1 = sh + KT * me;             // [KT][n_c]
  double* e2 = e1 + KT * (size_t)n_c;    // [KT][n_c]
  for (int e = tid; e < KT * me; e += nt) {
    const int t = e / me, k = e % me;
    om[e] = fma(al[t], D[k], X[k]);
  }
  __syncthreads();
  const int y0 = me + 1 + nk;
  double bias[KT];
#pragma unroll
  for (int t = 0; t < KT; ++t) bias[t] = fma(al[t], D[me], X[me]);
  double fmax_local[KT], se2[KT][kResSplit];
  int bad[KT];
#pragma unroll
  for (int t = 0; t < KT; ++t) {
    fmax_local[t] = 0.0;
    bad[t] = 0;
#pragma unroll
    for (int sp = 0; sp < kResSplit; ++sp) se2[t][sp] = 0.0;
  }
#pragma unroll
  for (int sp = 0; sp < kResSplit; ++sp) {
    const int r0 = sp * rpc, r1 = min(n_c, r0 + rpc);
    for (int i = r0 + tid; i < r1; i += nt) {
      double a0[KT], a1[KT], c0[KT], c1[KT];
#pragma unroll
      for (int t = 0; t < KT; ++t) a0[t] = a1[t] = c0[t] = c1[t] = 0.0;
      int k = 0;
#pragma unroll 2
      for (; k + 1 < me; k += 2) {
        const double s1a = S1T[(size_t)k * n_c + i], s1b = S1T[(size_t)(k + 1) * n_c + i];
        const double s0a = S0T[(size_t)k * n_c + i], s0b = S0T[(size_t)(k + 1) * n_c + i];
#pragma unroll
        for (int t = 0; t < KT; ++t) {
          a0[t] = fma(s1a, om[t * me + k], a0[t]);
          a1[t] = fma(s1b, om[t * me + k + 1], a1[t]);
          c0[t] = fma(s0a, om[t * me + k], c0[t]);
          c1[t] = fma(s0b, om[t * me + k + 1], c1[t]);
        }
      }
      if (k < me) {
        const double s1a = S1T[(size_t)k * n_c + i], s0a = S0T[(size_t)k * n_c + i];
#pragma unroll
        for (int t = 0; t < KT; ++t) {
          a0[t] = fma(s1a, om[t * me + k], a0[t]);
          c0[t] = fma(s0a, om[t * me + k], c0[t]);
        }
      }
      const double xy = X[y0 + i], dy = D[y0 + i];
#pragma unroll
      for (int t = 0; t < KT; ++t) {
        const double s1w = a0[t] + a1[t], s0w = c0[t] + c1[t];
        const double yi = fma(al[t], dy, xy);
        double f, fy, fyy;
        rhs.eval(b, i, yi, f, fy, fyy);
        const double ee1 = __dsub_rn(s1w, f);
        const double ee2 = __dsub_rn(__dsub_rn(yi, s0w), bias[t]);
        if (!isfinite(ee1) || !isfinite(f)) bad[t] = 1;
        e1[t * (size_t)n_c + i] = ee1;
        e2[t * (size_t)n_c + i] = ee2;
        se2[t][sp] += ee2;
        const double Fy = __dadd_rn(__dmul_rn(__dmul_rn(-gm, fy), ee1), __dmul_rn(gm, ee2));
        fmax_local[t] = fmax(fmax_local[t], fabs(Fy));
      }
    }
  }
  int badm = 0;
#pragma unroll
  for (int t = 0; t < KT; ++t) {
#pragma unroll
    for (int sp = 0; sp < kResSplit; ++sp) {
#pragma unroll
      for (int o = 16; o; o >>= 1)
        se2[t][sp] = se2[t][sp] + __shfl_xor_sync(0xffffffffu, se2[t][sp], o);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1)
      fmax_local[t] = fmax(fmax_local[t], __shfl_xor_sync(0xffffffffu, fmax_local[t], o));
    badm |= bad[t] << t;
  }
  if (lane == 0) {
#pragma unroll
    for (int t = 0; t < KT; ++t) {
      double* rt = red + t * (kResSplit + 1) * nw;
#pragma unroll
      for (int sp = 0; sp < kResSplit; ++sp) rt[sp * nw + warp] = se2[t][sp];
      rt[kResSplit * nw + warp] = fmax_local[t];
    }
  }
  // OR of the per-trial flags over the CTA (bit t = trial t)
  __shared__ int badm_s;
  if (tid == 0) badm_s = 0;
  __syncthreads();
  if (badm) atomicOr(&badm_s, badm);
  __syncthreads();
  {
    // every trial already rejected by its rows (non-finite rhs or max|F_y| >
    // ref): the S^T e pass cannot change that -- report the lower bounds
    bool all_rej = true;
    for (int t = 0; t < KT; ++t) {
      const double* rt = red + t * (kResSplit + 1) * nw;
      double m = 0.0;
      for (int w = 0; w < nw; ++w) m = fmax(m, rt[kResSplit * nw + w]);
      if (!((badm_s >> t) & 1) && !(m > ref)) all_rej = false;
    }
    if (all_rej) {
      if (tid < KT) {
        const double* rt = red + tid * (kResSplit + 1) * nw;
        double m = 0.0;
        for (int w = 0; w < nw; ++w) m = fmax(m, rt[kResSplit * nw + w]);
        out[tid] = ((badm_s >> tid) & 1) ? NAN : m;
      }
      __syncthreads();
      return;
    }
  }
  // range partials of S1^T e1 and S0^T e2 for every trial
  for (int task = warp; task < kResSplit * me; task += nw) {
    const int sp = task / me, k = task % me;
    const int r0 = sp * rpc, r1 = min(n_c, r0 + rpc);
    const double* rr1 = S1T + (size_t)k * n_c;
    const double* rr0 = S0T + (size_t)k * n_c;
    double a[KT], c[KT];
#pragma unroll
    for (int t = 0; t < KT; ++t) a[t] = c[t] = 0.0;
    for (int i = r0 + lane; i < r1; i += 32) {
      const double v1 = rr1[i], v0 = rr0[i];
#pragma unroll
      for (int t = 0; t < KT; ++t) {
        a[t] = fma(v1, e1[t * (size_t)n_c + i], a[t]);
        c[t] = fma(v0, e2[t * (size_t)n_c + i], c[t]);
      }
    }
#pragma unroll
    for (int t = 0; t < KT; ++t) {
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        a[t] += __shfl_xor_sync(0xffffffffu, a[t], o);
        c[t] += __shfl_xor_sync(0xffffffffu, c[t], o);
      }
    }
    if (lane == 0) {
#pragma unroll
      for (int t = 0; t < KT; ++t) {
        part[(t * kResSplit + sp) * pstride + k] = a[t];
        part[(t * kResSplit + sp) * pstride + me + k] = c[t];
      }
    }
  }
  __syncthreads();
  // finalize per trial (persist_residual's arithmetic); warp t handles trial t
  for (int t = warp; t < KT; t += nw) {
    const double* pt = part + (size_t)t * kResSplit * pstride;
    const double* rt = red + t * (kResSplit + 1) * nw;
    const double* omt = om + t * me;
    double fm = 0.0;
    for (int k = lane; k < me; k += 32) {
      double a = 0.0, c = 0.0;
      for (int s2 = 0; s2 < kResSplit; ++s2) {
        a += pt[s2 * pstride + k];
        c += pt[s2 * pstride + me + k];
      }
      double acl = 0.0;
      for (int mu = 0; mu < nk; ++mu)
        acl = __dadd_rn(acl, __dmul_rn(Ac[(size_t)mu * me + k],
                                       fma(al[t], D[me + 1 + mu], X[me + 1 + mu])));
      const double v = __dadd_rn(__dsub_rn(__dadd_rn(omt[k], __dmul_rn(gm, a)), __dmul_rn(gm, c)), acl);
      fm = fmax(fm, fabs(v));
    }
    if (lane == 0) {
      double se = 0.0;
      for (int s2 = 0; s2 < kResSplit; ++s2) {
        double sw = 0.0;
        for (int w = 0; w < nw; ++w) sw += rt[s2 * nw + w];   // block_reduce's order
        se += sw;
      }
      double fy = 0.0;
      for (int w = 0; w < nw; ++w) fy = fmax(fy, rt[kResSplit * nw + w]);
      fm = fmax(fm, fy);
      double bl = 0.0;
      for (int mu = 0; mu < nk; ++mu)
        bl = __dadd_rn(bl, __dmul_rn(betac[mu], fma(al[t], D[me + 1 + mu], X[me + 1 + mu])));
      fm = fmax(fm, fabs(__dadd_rn(__dmul_rn(-gm, se), bl)));
      for (int mu = 0; mu < nk; ++mu) {
        double v = 0.0;
        for (int k = 0; k < me; ++k) v = fma(Ac[(size_t)mu * me + k], omt[k], v);
        v = __dsub_rn(__dadd_rn(v, __dmul_rn(betac[mu], bias_of(al[t], D, X, me))),
                      vals[(size_t)b * nk + mu]);
        fm = fmax(fm, fabs(v));
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) fm = fmax(fm, __shfl_xor_sync(0xffffffffu, fm, o));
    if (lane == 0) out[t] = ((badm_s >> t) & 1) ? NAN : fm;
  }
  __syncthreads();
}

// residual at x (F, aux, the norm; NaN when the rhs is non-finite): the four
// row ranges of newton_residual_kernel<false> + newton_residual_finalize_kernel
NYS_DEV double persist_residual(const double* __restrict__ S0T, const double* __restrict__ S1T,
                                int me, int n_c, const Rhs& rhs, double gm,
                                const double* __restrict__ x, int b, int nk,
                                const double* __restrict__ Ac, const double* __restrict__ betac,
                                const double* __restrict__ vals, double* __restrict__ Fb,
                                double* __restrict__ auxb, double* part, double* sh, double* red,
                                double* lam_s, double bound = INFINITY) {
  const int pstride = 2 * me + 3;
  double early;
  if (residual_splits_fused(S0T, S1T, me, n_c, rhs, gm, x, b, nk, Fb, auxb, part, sh, red, bound,
                            &early))
    return early;   // > bound or NaN: F / aux incomplete, the caller rejects the point
  const int tid = threadIdx.x;
  if (tid < nk) lam_s[tid] = x[me + 1 + tid];
  __syncthreads();
  double fmax_local = 0.0;
  int bad = 0;
  for (int s2 = 0; s2 < kResSplit; ++s2) bad |= part[s2 * pstride + 2 * me + 2] != 0.0;
  for (int k = tid; k < me; k += blockDim.x) {
    double a = 0.0, c = 0.0;
    for (int s2 = 0; s2 < kResSplit; ++s2) {
      a += part[s2 * pstride + k];
      c += part[s2 * pstride + me + k];
    }
    double acl = 0.0;
    for (int mu = 0; mu < nk; ++mu) acl = __dadd_rn(acl, __dmul_rn(Ac[(size_t)mu * me + k], lam_s[mu]));
    const double v = __dadd_rn(__dsub_rn(__dadd_rn(x[k], __dmul_rn(gm, a)), __dmul_rn(gm, c)), acl);
    Fb[k] = v;
    fmax_local = fmax(fmax_local, fabs(v));
  }
  if (tid == 0) {
    double se2 = 0.0, fy = 0.0;
    for (int s2 = 0; s2 < kResSplit; ++s2) {
      se2 += part[s2 * pstride + 2 * me];
      fy = fmax(fy, part[s2 * pstride + 2 * me + 1]);
    }
    fmax_local = fmax(fmax_local, fy);
    double bl = 0.0;
    for (int mu = 0; mu < nk; ++mu) bl = __dadd_rn(bl, __dmul_rn(betac[mu], lam_s[mu]));
    const double Fbias = __dadd_rn(__dmul_rn(-gm, se2), bl);
    Fb[me] = Fbias;
    fmax_local = fmax(fmax_local, fabs(Fbias));
    const double bias = x[me];
    for (int mu = 0; mu < nk; ++mu) {
      double v = 0.0;
      for (int k = 0; k < me; ++k) v = fma(Ac[(size_t)mu * me + k], x[k], v);
      v = __dsub_rn(__dadd_rn(v, __dmul_rn(betac[mu], bias)), vals[(size_t)b * nk + mu]);
      Fb[me + 1 + mu] = v;
      fmax_local = fmax(fmax_local, fabs(v));
    }
  }
  const double nrm = block_reduce(fmax_local, red, true);   // max: order-free
  __syncthreads();
  return bad ? NAN : nrm;
}

// The LU of lu_solve_cta_kernel (first max wins; every element updated by the
// same operation in the same k order, so the factors and the solution are
// bit-identical): per column warp 0 searches the pivot and swaps the rows,
// then all warps scale and update the trailing rows (row i by warp i % 8,
// columns across lanes) -- two CTA barriers per column.  K (row-major n x n)
// is copied into a padded odd-stride tile T (conflict-free 8-byte accesses).
// Returns NYS_INFO_* to every thread; the solution is left in ys.
constexpr int kPLuMaxN = 64;
NYS_DEV int persist_lu(double* K, double* ys, int* perm, int n, int* flag, double* T) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int ld = n | 1;   // odd stride in doubles
  for (int e = tid; e < n * n; e += blockDim.x) T[(e / n) * ld + e % n] = K[e];
  if (tid == 0) *flag = NYS_INFO_OK;
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    if (warp == 0) {
      double bv = -1.0;
      int bi = n;
      for (int i = k + lane; i < n; i += 32) {
        const double a = fabs(T[i * ld + k]);
        if (a > bv) {
          bv = a;
          bi = i;
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      if (!(bv > 0.0)) {
        if (lane == 0) *flag = NYS_INFO_SINGULAR;
      } else {
        if (lane == 0) perm[k] = bi;
        if (bi != k)
          for (int j = lane; j < n; j += 32) {
            const double a = T[k * ld + j], p = T[bi * ld + j];
            T[bi * ld + j] = a;
            T[k * ld + j] = p;
          }
      }
    }
    __syncthreads();
    if (*flag != NYS_INFO_OK) return *flag;
    const double inv = 1.0 / T[k * ld + k];
    const double* urow = T + k * ld;
    for (int i = k + 1 + warp; i < n; i += nw) {
      double* r = T + i * ld;
      const double l = r[k] * inv;
      __syncwarp();
      if (lane == 0) r[k] = l;
      for (int j = k + 1 + lane; j < n; j += 32) r[j] -= l * urow[j];
    }
    __syncthreads();
  }
  if (warp == 0) {
    if (lane == 0)
      for (int k = 0; k < n; ++k) {
        const int pr = perm[k];
        if (pr != k) {
          const double t = ys[k];
          ys[k] = ys[pr];
          ys[pr] = t;
        }
      }
    __syncwarp();
    for (int j = 0; j < n - 1; ++j) {
      const double yj = ys[j];
      for (int i = j + 1 + lane; i < n; i += 32) ys[i] -= T[i * ld + j] * yj;
      __syncwarp();
    }
    for (int j = n - 1; j >= 0; --j) {
      const double zj = ys[j] / T[j * ld + j];
      __syncwarp();
      if (lane == 0) ys[j] = zj;
      for (int i = lane; i < j; i += 32) ys[i] -= T[i * ld + j] * zj;
      __syncwarp();
    }
    int bad = 0;
    for (int i = lane; i < n; i += 32)
      if (!isfinite(ys[i])) bad = 1;
    if (__any_sync(0xffffffffu, bad) && lane == 0) *flag = NYS_INFO_NONFINITE;
  }
  __syncthreads();
  return *flag;
}

// doubles of the persistent kernel's region A: the reduce partials of 8 warps,
// the residual scratch, the padded LU tile or the multi-trial scratch
NYS_HD_INLINE size_t persist_region_a(size_t stride, int me, int n_c, int nz) {
  size_t r = (size_t)(kPersistThreads / 32) * stride;
  const size_t res = (size_t)me + 2 * (size_t)n_c + kResSplit * (2 * (size_t)me + 3);
  const size_t lu = (size_t)nz * (nz | 1);
  const size_t multi = (size_t)kPTrials * kResSplit * (2 * (size_t)me + 3) +
                       (size_t)kPTrials * ((size_t)me + 2 * (size_t)n_c);
  r = r > res ? r : res;
  r = r > lu ? r : lu;
  return r > multi ? r : multi;
}

struct PersistArgs {
  const double *S0, *S1, *S0T, *S1T, *psi;
  int me, n_c, nk, nks, ldx;
  Rhs rhs;
  const double *Ac, *betac, *vals, *gamma, *tol;
  double* X;
  const int* idx;
  int damped, halvings, max_iters;
  double shrink;
  double* work;        // per slot: Xc, F, Fc, D (ldx each), aux, auxc (3 n_c each)
  size_t work_stride;  // doubles per slot
  double* norms;       // [nb][max_iters + 1]
  int* iters;          // [nb]
  int* status;         // [nb]
  long long* prof;     // optional [nb][8]: clocks in residual / reduce / LU / step, trials
  int* tot_iters;      // optional [nb]: Newton iterations over every rung / stage (ladder)
};

// shared-memory carve-up of the persistent kernels
struct PersistSmem {
  double *redA, *sh, *part, *K, *ys, *red, *red_m, *al_s, *tn_s, *lam_s;
  int *perm, *flag;
};

// newton._solve_once (newton.py:279-349) for instance b from the point in xg
// (final iterate left there): returns the status (0 converged, 1 max
// iterations, 2 diverged, 3 singular); *its = iterations, nrm_out[0..*its] the
// residual max-norms.  wk: 4 ldx + 6 n_c doubles of scratch.
template <int NB>
NYS_DEV int persist_solve_once(const PersistArgs& A, const PersistSmem& S, int b, double gm,
                               double tol, bool damped, double* xg, double* wk, double* nrm_out,
                               int* its, long long* pc) {
  constexpr int NPAIR = Tri<NB>::kPairs;
  constexpr int kStride = NPAIR * 64 + NB * 8;
  const int me = A.me, n_c = A.n_c, nk = A.nk, ldx = A.ldx;
  const int nz = me + 1 + nk;
  double* Xcur = xg;
  double* Xnew = wk;
  double* Fcur = wk + ldx;
  double* Fnew = wk + 2 * (size_t)ldx;
  double* Dv = wk + 3 * (size_t)ldx;
  double* auxc = wk + 4 * (size_t)ldx;
  double* auxn = auxc + 3 * (size_t)n_c;
  double *redA = S.redA, *K = S.K, *ys = S.ys;
  const int tid = threadIdx.x, warp = tid >> 5;

  double norm = persist_residual(A.S0T, A.S1T, me, n_c, A.rhs, gm, Xcur, b, nk, A.Ac, A.betac,
                                 A.vals, Fcur, auxc, S.part, S.sh, S.red, S.lam_s);
  if (tid == 0) nrm_out[0] = norm;
  int status = isfinite(norm) ? -1 : 2;   // DIVERGED: _residual raised at the start
  int it = 0;
  const int kps = (A.nks + kPersistSplits - 1) / kPersistSplits;
  long long t0 = clock64();
#define NYS_PT(i)                       \
  do {                                  \
    const long long t1_ = clock64();    \
    pc[i] += t1_ - t0;                  \
    t0 = t1_;                           \
  } while (0)
  while (status < 0) {
    // newton.py:296-303
    if (norm <= tol) { status = 0; break; }
    if (it >= A.max_iters) { status = 1; break; }
    if (norm > 1e12) { status = 2; break; }
    // ---- reduced system (newton_reduce_kernel, 2 splits x 4 warps)
    {
      const int sp = warp >> 2, wi = warp & 3;
      const int lo = sp * kps, hi = min(A.nks, lo + kps);
      reduce_warp<NB>(A.psi, me, n_c, auxc, Fcur + nz, lo, hi, wi, 4,
                      redA + (size_t)warp * kStride);
      __syncthreads();
      for (int e = tid; e < kStride; e += blockDim.x) {   // split partials, fixed order
        double p0 = 0.0, p1 = 0.0;
        for (int w = 0; w < 4; ++w) {
          p0 += redA[(size_t)w * kStride + e];
          p1 += redA[(size_t)(4 + w) * kStride + e];
        }
        redA[e] = p0;
        redA[kStride + e] = p1;
      }
      __syncthreads();
      build_reduced<NB>(redA, kStride, kPersistSplits, me, nk, Fcur, gm, A.Ac, A.betac, K, ys);
      __syncthreads();
    }
    NYS_PT(1);
    // ---- LU (first max wins), as nys_lu_solve_f64
    const int info = persist_lu(K, ys, S.perm, nz, S.flag, redA);   // redA: free here
    if (info != NYS_INFO_OK) { status = 3; break; }
    NYS_PT(2);
    // ---- delta (newton_step_kernel, compute_delta)
    {
      for (int k = tid; k < nz; k += blockDim.x) Dv[k] = ys[k];
      int bad = 0;
      for (int k = tid; k < nz; k += blockDim.x) bad |= !isfinite(ys[k]);
      for (int i = tid; i < n_c; i += blockDim.x) {
        // newton_step_kernel's dot products in the same k order, read from the
        // transposed copies (coalesced across the CTA's rows)
        double a = 0.0, c = 0.0;
#pragma unroll 8
        for (int k = 0; k < me; ++k) {
          a = fma(A.S1T[(size_t)k * n_c + i], ys[k], a);
          c = fma(A.S0T[(size_t)k * n_c + i], ys[k], c);
        }
        const double fy = auxc[i], cc = auxc[2 * n_c + i];
        const double wd = fy * a + c + ys[me];
        const double dv = (-Fcur[nz + i] + gm * wd) / (gm * cc);
        Dv[nz + i] = dv;
        bad |= !isfinite(dv);
      }
      if (__syncthreads_or(bad)) { status = 3; break; }   // non-finite correction
    }
    NYS_PT(3);
    // ---- step halving (newton.py:313-325) or the full step.  alpha_k =
    // shrink^k by the loop's repeated products; the first finite trial norm
    // <= norm wins.  Trial 0 is a full residual (its F / aux are kept when it
    // is accepted, the common case); later trials are evaluated kPTrials at a
    // time (trial_norms_multi: bit-identical norms) and the accepted one is
    // then materialised with its full residual.
    double alpha = 1.0, tn = 0.0;
    bool have;
    {
      for (int k = tid; k < nz + n_c; k += blockDim.x) Xnew[k] = fma(alpha, Dv[k], Xcur[k]);
      __syncthreads();
      tn = persist_residual(A.S0T, A.S1T, me, n_c, A.rhs, gm, Xnew, b, nk, A.Ac, A.betac, A.vals,
                            Fnew, auxn, S.part, S.sh, S.red, S.lam_s, damped ? norm : INFINITY);
      pc[5] += 1;
      have = !damped || (isfinite(tn) && tn <= norm);
    }
    if (!have) {
      alpha *= A.shrink;
      bool found = false;
      int h = 1;
      while (!found && h < A.halvings) {
        const int cnt = min(kPTrials, A.halvings - h);
        if (tid == 0) {
          double a = alpha;
          for (int t = 0; t < kPTrials; ++t) {
            S.al_s[t] = a;
            if (t + 1 < cnt) a *= A.shrink;
          }
        }
        __syncthreads();
        trial_norms_multi<kPTrials>(A.S0T, A.S1T, me, n_c, A.rhs, gm, Xcur, Dv, S.al_s, b, nk,
                                    A.Ac, A.betac, A.vals, redA,
                                    redA + kPTrials * kResSplit * (2 * me + 3), S.red_m, S.tn_s,
                                    norm);
        pc[5] += cnt;
        for (int t = 0; t < cnt && !found; ++t) {
          if (isfinite(S.tn_s[t]) && S.tn_s[t] <= norm) {
            found = true;
            alpha = S.al_s[t];
          } else {
            alpha *= A.shrink;
          }
        }
        h += cnt;
        __syncthreads();
      }
      // the accepted trial, or the last (untested) halving the loop leaves
      for (int k = tid; k < nz + n_c; k += blockDim.x) Xnew[k] = fma(alpha, Dv[k], Xcur[k]);
      __syncthreads();
      tn = persist_residual(A.S0T, A.S1T, me, n_c, A.rhs, gm, Xnew, b, nk, A.Ac, A.betac, A.vals,
                            Fnew, auxn, S.part, S.sh, S.red, S.lam_s);
    }
    // x <- candidate; F, aux at it
    {
      double* t = Xcur; Xcur = Xnew; Xnew = t;   // the old point is no longer needed
      t = Fcur; Fcur = Fnew; Fnew = t;
      t = auxc; auxc = auxn; auxn = t;
    }
    ++it;
    NYS_PT(0);
    norm = tn;
    if (tid == 0) nrm_out[it] = norm;
    if (!isfinite(norm)) { status = 2; break; }
  }
#undef NYS_PT
  // the final iterate lives in xg
  if (Xcur != xg) {
    for (int k = tid; k < nz + n_c; k += blockDim.x) xg[k] = Xcur[k];
  }
  __syncthreads();
  *its = it;
  return status;
}

template <int NB>
NYS_DEV PersistSmem persist_smem(const PersistArgs& A, double* smp, double* red, double* red_m,
                                 double* al_s, double* tn_s, double* lam_s, int* flag) {
  constexpr int kStride = Tri<NB>::kPairs * 64 + NB * 8;
  const int nz = A.me + 1 + A.nk;
  PersistSmem S;
  S.redA = smp;
  S.sh = smp;                                  // me + 2 n_c (aliases redA)
  S.part = smp + A.me + 2 * A.n_c;             // kResSplit (2 me + 3)
  S.K = smp + persist_region_a(kStride, A.me, A.n_c, nz);
  S.ys = S.K + (size_t)nz * nz;
  S.perm = reinterpret_cast<int*>(S.ys + nz);
  S.red = red;
  S.red_m = red_m;
  S.al_s = al_s;
  S.tn_s = tn_s;
  S.lam_s = lam_s;
  S.flag = flag;
  return S;
}

#define NYS_PERSIST_SHARED                                                   \
  extern __shared__ double smp[];                                            \
  __shared__ double red[(kResSplit + 1) * (kPersistThreads / 32)];           \
  __shared__ double red_m[kPTrials * (kResSplit + 1) * (kPersistThreads / 32)]; \
  __shared__ double al_s[kPTrials], tn_s[kPTrials];                          \
  __shared__ double lam_s[kMaxCondN];                                        \
  __shared__ int flag_s;                                                     \
  const PersistSmem S = persist_smem<NB>(A, smp, red, red_m, al_s, tn_s, lam_s, &flag_s)

// one _solve_once per instance (nys_newton_solve_once_f64)
template <int NB>
__global__ void __launch_bounds__(kPersistThreads, NYS_PERSIST_MINB)
    newton_persist_kernel(PersistArgs A) {
  NYS_PERSIST_SHARED;
  const int slot = blockIdx.x;
  const int b = A.idx[slot];
  long long pc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int it = 0;
  const int status = persist_solve_once<NB>(
      A, S, b, A.gamma[b], A.tol[b], A.damped != 0, A.X + (size_t)b * A.ldx,
      A.work + (size_t)slot * A.work_stride, A.norms + (size_t)slot * (A.max_iters + 1), &it, pc);
  if (threadIdx.x == 0) {
    A.iters[slot] = it;
    A.status[slot] = status;
    if (A.prof != nullptr)
      for (int i = 0; i < 8; ++i) A.prof[(size_t)slot * 8 + i] = pc[i];
  }
}

// the whole retry ladder per instance (newton.py:376-412; nys_newton_ladder_f64):
// rungs 1-4 from the constant / linearised starts, undamped then damped;
// rung 5 the gamma continuation (newton.py:352-373: stages 1, 1e2, 1e4 below
// the target, damped, tol 1e-8 (1 + g), MaxIters tolerated, Divergence /
// Singular escape; the model hand-off omega, b, lambda = 0, y = S0 omega + b),
// then the target.  No instance waits for another between rungs or stages.
template <int NB>
__global__ void __launch_bounds__(kPersistThreads, NYS_PERSIST_MINB)
    newton_ladder_kernel(PersistArgs A, const double* __restrict__ X0c,
                         const double* __restrict__ X0l, int* __restrict__ rung_out) {
  NYS_PERSIST_SHARED;
  const int slot = blockIdx.x;
  const int b = A.idx[slot];
  const int me = A.me, n_c = A.n_c, nk = A.nk, ldx = A.ldx, nz = me + 1 + nk;
  const double gt = A.gamma[b], tt = A.tol[b];
  double* xg = A.X + (size_t)b * ldx;
  double* wk = A.work + (size_t)slot * A.work_stride;
  double* nrm = A.norms + (size_t)slot * (A.max_iters + 1);
  long long pc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int it = 0, status = 1, rung = 0, tot = 0;
  const int tid = threadIdx.x;
  for (int r = 1; r <= 4; ++r) {
    const double* x0 = (r <= 2 ? X0c : X0l) + (size_t)slot * ldx;
    for (int k = tid; k < ldx; k += blockDim.x) xg[k] = x0[k];
    __syncthreads();
    status = persist_solve_once<NB>(A, S, b, gt, tt, (r & 1) == 0, xg, wk, nrm, &it, pc);
    tot += it;
    rung = r;
    if (status == 0) break;
  }
  if (status != 0) {
    rung = 5;
    for (int k = tid; k < ldx; k += blockDim.x) xg[k] = X0c[(size_t)slot * ldx + k];
    __syncthreads();
    bool escaped = false;
    const double stages[3] = {1e0, 1e2, 1e4};
    for (int s = 0; s < 3 && !escaped; ++s) {
      const double g = stages[s];
      if (!(g < gt)) continue;
      status = persist_solve_once<NB>(A, S, b, g, 1e-8 * (1.0 + g), true, xg, wk, nrm, &it, pc);
      tot += it;
      if (status == 2 || status == 3) {
        escaped = true;
        break;
      }
      // hand-off: omega, b kept; lambda = 0; y = Psi_0 omega + b (linear.py:47-53)
      for (int k = me + 1 + tid; k < nz; k += blockDim.x) xg[k] = 0.0;
      const double bias = xg[me];
      for (int i = tid; i < n_c; i += blockDim.x) {
        double acc = 0.0;
        for (int k = 0; k < me; ++k) acc = fma(A.S0T[(size_t)k * n_c + i], xg[k], acc);
        xg[nz + i] = acc + bias;
      }
      __syncthreads();
    }
    if (!escaped) {
      status = persist_solve_once<NB>(A, S, b, gt, tt, true, xg, wk, nrm, &it, pc);
      tot += it;
    }
  }
  if (tid == 0) {
    A.iters[slot] = it;
    A.status[slot] = status;
    rung_out[slot] = rung;
    if (A.tot_iters != nullptr) A.tot_iters[slot] = tot;
    if (A.prof != nullptr)
      for (int i = 0; i < 8; ++i) A.prof[(size_t)slot * 8 + i] = pc[i];
  }
}

}  // namespace

// ------------------------------------------------------------------ C ABI
extern "C" int nys_transpose_f64(const double* A, int rows, int cols, double* AT, void* stream) {
  if (rows < 0 || cols < 0) return NYS_EINVAL;
  if (rows == 0 || cols == 0) return NYS_OK;
  dim3 grid((cols + 31) / 32, (rows + 31) / 32), block(32, 8);
  transpose_kernel<<<grid, block, 0, static_cast<cudaStream_t>(stream)>>>(A, rows, cols, AT);
  nys_host::count_launches(1);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" int nys_newton_pack_f64(const double* landmarks, int m, const double* W, int ldw,
                                   int m_eff, double sigma2, const double* pts, int n_c,
                                   double* packed, void* stream) {
  const int NB = (m_eff + 2 + 7) / 8;
  const int nks = (n_c + 3) / 4;
  return nys_host::launch_psi_pack(landmarks, m, W, ldw, m_eff, sigma2, 1, pts, n_c, NB, nks * 4,
                                   packed, static_cast<cudaStream_t>(stream));
}

extern "C" int nys_newton2_pack_f64(const double* landmarks, int m, const double* W, int ldw,
                                    int m_eff, double sigma2, const double* pts, int n_c,
                                    double* packed, void* stream) {
  const int NB = (m_eff + 2 + 7) / 8;
  const int nks = (n_c + 3) / 4;
  return nys_host::launch_psi_pack(landmarks, m, W, ldw, m_eff, sigma2, 2, pts, n_c, NB, nks * 4,
                                   packed, static_cast<cudaStream_t>(stream));
}

extern "C" size_t nys_newton2_pack_doubles(int m_eff, int n_c) {
  const int NB = (m_eff + 2 + 7) / 8;
  return (size_t)((n_c + 3) / 4) * 3 * NB * 32;
}

extern "C" size_t nys_newton_pack_doubles(int m_eff, int n_c) {
  const int NB = (m_eff + 2 + 7) / 8;
  return (size_t)((n_c + 3) / 4) * 2 * NB * 32;
}

extern "C" int nys_newton_residual_f64(const double* S0, const double* S1, const double* S0T,
                                       const double* S1T, int m_eff, int n_c, const double* g,
                                       const double* fy, const double* fyy, const double* alpha,
                                       const double* beta, const double* Ac, const double* betac,
                                       const double* vals, int n_cond, const double* gamma,
                                       const double* X, int ldx, const int* idx, int nb,
                                       double* F, double* norm, double* aux, double* work,
                                       void* stream) {
  if (m_eff < 1 || n_c < 1 || n_cond < 0 || n_cond > kMaxCondN || nb < 0 ||
      ldx < m_eff + 1 + n_cond + n_c)
    return NYS_EINVAL;
  if (nb == 0) return NYS_OK;
  (void)S0;
  (void)S1;
  Rhs rhs{g, fy, fyy, alpha, beta, n_c};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // `work` (2 n_c doubles per instance) holds the row-range partials
  if ((size_t)kResSplit * (2 * m_eff + 3) > 2 * (size_t)n_c) return NYS_EUNSUPPORTED;
  const int rpc = ((n_c + kResSplit - 1) / kResSplit + 31) / 32 * 32;
  const size_t smem = ((size_t)m_eff + 2 * (size_t)rpc) * sizeof(double);
  auto kern = newton_residual_kernel<false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return nys_host::record_cuda(e);
  kern<<<dim3(nb, 1, kResSplit), kResThreads, smem, st>>>(S0T, S1T, m_eff, n_c, rhs, gamma, X,
                                                          ldx, idx, F, aux, nullptr, nullptr, nb,
                                                          n_cond, work);
  newton_residual_finalize_kernel<false><<<nb, 64, 0, st>>>(m_eff, Ac, betac, vals, n_cond, gamma,
                                                            X, ldx, idx, F, norm, nullptr,
                                                            nullptr, nb, work);
  nys_host::count_launches(2);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" size_t nys_newton_trial_scratch_bytes(int m_eff, int n_c, int nb, int ntrial) {
  (void)n_c;   // partial sums of every (instance, trial, row range)
  return (size_t)ntrial * nb * kResSplit * (2 * (size_t)m_eff + 3) * sizeof(double);
}

extern "C" int nys_newton_trial_norms_f64(const double* S0T, const double* S1T, int m_eff, int n_c,
                                          const double* g, const double* fy, const double* fyy,
                                          const double* alpha, const double* beta,
                                          const double* Ac, const double* betac,
                                          const double* vals, int n_cond, const double* gamma,
                                          const double* X, const double* D, int ldx,
                                          const int* idx, int nb, const double* trial_alphas,
                                          int ntrial, double* norms, void* scratch,
                                          size_t scratch_bytes, void* stream) {
  if (m_eff < 1 || n_c < 1 || n_cond < 0 || n_cond > kMaxCondN || nb < 0 || ntrial < 0 ||
      ntrial > 65535 || ldx < m_eff + 1 + n_cond + n_c)
    return NYS_EINVAL;
  if (nb == 0 || ntrial == 0) return NYS_OK;
  const size_t need = nys_newton_trial_scratch_bytes(m_eff, n_c, nb, ntrial);
  if (scratch == nullptr || scratch_bytes < need) return NYS_EWORKSPACE;
  const int rpc = ((n_c + kResSplit - 1) / kResSplit + 31) / 32 * 32;
  const size_t smem = ((size_t)m_eff + 2 * (size_t)rpc) * sizeof(double);
  auto kern = newton_residual_kernel<true>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return nys_host::record_cuda(e);
  Rhs rhs{g, fy, fyy, alpha, beta, n_c};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* part = static_cast<double*>(scratch);
  kern<<<dim3(nb, ntrial, kResSplit), kResThreads, smem, st>>>(S0T, S1T, m_eff, n_c, rhs, gamma,
                                                               X, ldx, idx, nullptr, nullptr, D,
                                                               trial_alphas, nb, n_cond, part);
  newton_residual_finalize_kernel<true><<<dim3(nb, ntrial), 64, 0, st>>>(
      m_eff, Ac, betac, vals, n_cond, gamma, X, ldx, idx, nullptr, norms, D, trial_alphas, nb,
      part);
  nys_host::count_launches(2);
  nys_host::count_launches(1);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

static int newton_reduce_splits(int nb, int nks) {
  // enough CTAs for about two per SM, at least 16 k-steps per split
  int ns = (2 * nys::device_sm_count() + nb - 1) / (nb > 0 ? nb : 1);
  ns = ns < 1 ? 1 : (ns > 16 ? 16 : ns);
  while (ns > 1 && nks / ns < 16) --ns;
  return ns;
}

extern "C" size_t nys_newton_reduced_workspace_bytes(int m_eff, int n_c, int nb) {
  const int NB = (m_eff + 2 + 7) / 8;
  const int nks = (n_c + 3) / 4;
  const int ns = newton_reduce_splits(nb, nks);
  if (ns <= 1) return 0;
  return (size_t)ns * nb * (NB * (NB + 1) / 2 * 64 + NB * 8) * sizeof(double);
}

extern "C" int nys_newton_reduced_ws_f64(const double* packed, int m_eff, int n_c,
                                         const double* aux, const double* F, int ldx,
                                         const double* gamma, const double* Ac,
                                         const double* betac, int n_cond, const int* idx, int nb,
                                         double* K, double* rz, void* workspace,
                                         size_t workspace_bytes, void* stream) {
  if (m_eff < 1 || n_c < 1 || n_cond < 0 || nb < 0) return NYS_EINVAL;
  if (nb == 0) return NYS_OK;
  const int NB = (m_eff + 2 + 7) / 8;
  const int nks = (n_c + 3) / 4;
  int ns = newton_reduce_splits(nb, nks);
  if (ns > 1 && (workspace == nullptr ||
                 workspace_bytes < nys_newton_reduced_workspace_bytes(m_eff, n_c, nb)))
    ns = 1;   // no (or too small a) workspace: one CTA per instance
  const int kps = (nks + ns - 1) / ns;
  double* part = ns > 1 ? static_cast<double*>(workspace) : nullptr;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
#define NYS_RED(nbv)                                                                             \
  case nbv: {                                                                                    \
    constexpr int NP = nbv * (nbv + 1) / 2;                                                      \
    const size_t smem = (size_t)kRedWarps * (NP * 64 + nbv * 8) * sizeof(double);                \
    auto kern = newton_reduce_kernel<nbv>;                                                       \
    if (smem > 48 * 1024) {                                                                      \
      cudaError_t e =                                                                            \
          cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);     \
      if (e != cudaSuccess) return nys_host::record_cuda(e);                                     \
    }                                                                                            \
    kern<<<dim3(nb, ns), kRedWarps * 32, smem, st>>>(packed, nks, m_eff, n_c, aux, F, ldx, gamma, \
                                                     Ac, betac, n_cond, idx, K, rz, kps, part);  \
    nys_host::count_launches(1);                                                                 \
    if (ns > 1) {                                                                                \
      newton_reduce_finalize_kernel<nbv><<<nb, 256, 0, st>>>(part, ns, nb, m_eff, F, ldx, gamma,  \
                                                            Ac, betac, n_cond, idx, K, rz);      \
      nys_host::count_launches(1);                                                               \
    }                                                                                            \
    break;                                                                                       \
  }
  switch (NB) {
    NYS_RED(1)
    NYS_RED(2)
    NYS_RED(3)
    NYS_RED(4)
    NYS_RED(5)
    NYS_RED(6)
    NYS_RED(7)
    NYS_RED(8)
    NYS_RED(9)
    default: return NYS_EUNSUPPORTED;
  }
#undef NYS_RED
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" int nys_newton_reduced_f64(const double* packed, int m_eff, int n_c, const double* aux,
                                      const double* F, int ldx, const double* gamma,
                                      const double* Ac, const double* betac, int n_cond,
                                      const int* idx, int nb, double* K, double* rz,
                                      void* stream) {
  return nys_newton_reduced_ws_f64(packed, m_eff, n_c, aux, F, ldx, gamma, Ac, betac, n_cond, idx,
                                   nb, K, rz, nullptr, 0, stream);
}

extern "C" int nys_lu_solve_f64(double* M, double* rhs, int n, int nb, double* out, int* info,
                                void* stream) {
  if (n < 1 || n > kLuMaxN || nb < 0) return NYS_EINVAL;
  if (nb == 0) return NYS_OK;
  const size_t smem = ((size_t)n * n + 2 * (size_t)n) * sizeof(double);
  const bool warp_lu = getenv("NYS_LU_WARP") != nullptr;   // A/B: one warp per system
  auto kern = warp_lu ? lu_solve_warp_kernel : lu_solve_cta_kernel;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return nys_host::record_cuda(e);
  }
  kern<<<nb, warp_lu ? 32 : kLuCtaThreads, smem, static_cast<cudaStream_t>(stream)>>>(M, rhs, n, out,
                                                                                    info);
  nys_host::count_launches(1);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" int nys_newton_step_f64(const double* S0, const double* S1, int m_eff, int n_c,
                                   int n_cond, const double* aux, const double* F,
                                   const double* dz, const double* gamma, const double* X,
                                   double* D, double* Xc, const double* alpha, int ldx,
                                   const int* idx, int nb, int compute_delta, void* stream) {
  if (m_eff < 1 || n_c < 1 || nb < 0) return NYS_EINVAL;
  if (nb == 0) return NYS_OK;
  const int nz = m_eff + 1 + n_cond;
  newton_step_kernel<<<nb, 256, nz * sizeof(double), static_cast<cudaStream_t>(stream)>>>(
      S0, S1, m_eff, n_c, n_cond, aux, F, dz, gamma, X, D, Xc, alpha, ldx, idx, compute_delta);
  nys_host::count_launches(1);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

// test hook: per-instance phase clocks of the next nys_newton_solve_once_f64
static long long* g_persist_prof = nullptr;
extern "C" void nys_newton_persist_profile(long long* dev_buf) { g_persist_prof = dev_buf; }

extern "C" size_t nys_newton_solve_once_work_doubles(int m_eff, int n_c, int n_cond) {
  const size_t ldx = (size_t)m_eff + 1 + n_cond + n_c;
  return 4 * ldx + 6 * (size_t)n_c;
}

template <int NB>
static int launch_persist(const PersistArgs& A, int nb, const double* X0c, const double* X0l,
                          int* rung, cudaStream_t st) {
  constexpr size_t kStride = NB * (NB + 1) / 2 * 64 + NB * 8;
  const int nz = A.me + 1 + A.nk;
  const size_t regA = persist_region_a(kStride, A.me, A.n_c, nz);
  const size_t smem = (regA + (size_t)nz * nz + nz) * sizeof(double) + nz * sizeof(int);
  if (X0c == nullptr) {
    auto kern = newton_persist_kernel<NB>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return nys_host::record_cuda(e);
    kern<<<nb, kPersistThreads, smem, st>>>(A);
  } else {
    auto kern = newton_ladder_kernel<NB>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return nys_host::record_cuda(e);
    kern<<<nb, kPersistThreads, smem, st>>>(A, X0c, X0l, rung);
  }
  nys_host::count_launches(1);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

static int persist_dispatch(const PersistArgs& A, int nb, const double* X0c, const double* X0l,
                            int* rung, cudaStream_t st) {
  switch ((A.me + 2 + 7) / 8) {
    case 1: return launch_persist<1>(A, nb, X0c, X0l, rung, st);
    case 2: return launch_persist<2>(A, nb, X0c, X0l, rung, st);
    case 3: return launch_persist<3>(A, nb, X0c, X0l, rung, st);
    case 4: return launch_persist<4>(A, nb, X0c, X0l, rung, st);
    case 5: return launch_persist<5>(A, nb, X0c, X0l, rung, st);
    case 6: return launch_persist<6>(A, nb, X0c, X0l, rung, st);
    case 7: return launch_persist<7>(A, nb, X0c, X0l, rung, st);
    case 8: return launch_persist<8>(A, nb, X0c, X0l, rung, st);
    default: return NYS_EUNSUPPORTED;   // nz <= 64: m_eff <= 62
  }
}

static int persist_check(int m_eff, int n_c, int n_cond, int nb, int max_iters, int halvings,
                         int ldx, const double* g, const double* alpha, const double* beta,
                         const double* work, size_t work_bytes) {
  if (m_eff < 1 || n_c < 1 || n_cond < 0 || n_cond > kMaxCondN || nb < 0 || max_iters < 0 ||
      halvings < 0 || ldx < m_eff + 1 + n_cond + n_c || m_eff + 1 + n_cond > kPLuMaxN)
    return NYS_EINVAL;
  if (g == nullptr || alpha == nullptr || beta == nullptr) return NYS_EINVAL;   // family mode
  if ((size_t)kResSplit * (2 * m_eff + 3) > 2 * (size_t)n_c) return NYS_EUNSUPPORTED;
  const size_t wd = nys_newton_solve_once_work_doubles(m_eff, n_c, n_cond);
  if (nb > 0 && (work == nullptr || work_bytes < (size_t)nb * wd * sizeof(double)))
    return NYS_EWORKSPACE;
  return NYS_OK;
}

extern "C" int nys_newton_solve_once_f64(
    const double* S0, const double* S1, const double* S0T, const double* S1T,
    const double* packed, int m_eff, int n_c, const double* g, const double* alpha,
    const double* beta, const double* Ac, const double* betac, const double* vals, int n_cond,
    const double* gamma, const double* tol, double* X, int ldx, const int* idx, int nb,
    int damped, double shrink, int halvings, int max_iters, double* work, size_t work_bytes,
    double* norms, int* iters, int* status, void* stream) {
  const int rc = persist_check(m_eff, n_c, n_cond, nb, max_iters, halvings, ldx, g, alpha, beta,
                               work, work_bytes);
  if (rc != NYS_OK || nb == 0) return rc;
  PersistArgs A{S0, S1, S0T, S1T, packed, m_eff, n_c, n_cond, (n_c + 3) / 4, ldx,
                Rhs{g, nullptr, nullptr, alpha, beta, n_c}, Ac, betac, vals, gamma, tol, X, idx,
                damped, halvings, max_iters, shrink, work,
                nys_newton_solve_once_work_doubles(m_eff, n_c, n_cond), norms, iters, status,
                g_persist_prof, nullptr};
  return persist_dispatch(A, nb, nullptr, nullptr, nullptr, static_cast<cudaStream_t>(stream));
}

extern "C" int nys_newton_ladder_f64(
    const double* S0, const double* S1, const double* S0T, const double* S1T,
    const double* packed, int m_eff, int n_c, const double* g, const double* alpha,
    const double* beta, const double* Ac, const double* betac, const double* vals, int n_cond,
    const double* gamma, const double* tol, const double* X0c, const double* X0l, double* X,
    int ldx, const int* idx, int nb, double shrink, int halvings, int max_iters, double* work,
    size_t work_bytes, double* norms, int* iters, int* status, int* rung, void* stream) {
  const int rc = persist_check(m_eff, n_c, n_cond, nb, max_iters, halvings, ldx, g, alpha, beta,
                               work, work_bytes);
  if (rc != NYS_OK || nb == 0) return rc;
  if (X0c == nullptr || X0l == nullptr || rung == nullptr) return NYS_EINVAL;
  PersistArgs A{S0, S1, S0T, S1T, packed, m_eff, n_c, n_cond, (n_c + 3) / 4, ldx,
                Rhs{g, nullptr, nullptr, alpha, beta, n_c}, Ac, betac, vals, gamma, tol, X, idx,
                1, halvings, max_iters, shrink, work,
                nys_newton_solve_once_work_doubles(m_eff, n_c, n_cond), norms, iters, status,
                g_persist_prof, rung + nb};
  return persist_dispatch(A, nb, X0c, X0l, rung, static_cast<cudaStream_t>(stream));
}
