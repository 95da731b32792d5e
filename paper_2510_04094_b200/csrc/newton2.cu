// Newton-KKT kernels for nonlinear SECOND-order ODEs y'' = f(t, y, y')
// (the catalog's P14 / P15 families), batched over
// instances sharing grid, landmarks and sigma.  Reference: newton.py with p = 2.
//
// Residual (newton.py:128-147): y' = S1 omega enters f, e1 = S2 omega - f,
// e2 = y - S0 omega - b,
//     F_omega = omega + g S2^T e1 - g S0^T e2 + Ac^T lam - g S1^T (f1 e1),
//     F_y = -g f0 e1 + g e2,   (f0 = df/dy, f1 = df/dy', g = gamma).
// Jacobian (newton.py:160-211): with G = S2 - f1 S1 (row-scaled), the y block
// is diag(g c_i), c = 1 + f0^2 - f00 e1, and eliminating it by Schur complement
// onto z = (omega, b) gives, with hatted vectors Gh = (G, 0), S0h = (S0, 1),
// S1h = (S1, 0) and u = f0 Gh + S0h + f01 e1 S1h (u_i = -column i of J_zy / g),
//     K = diag(I, 0) + g sum_i [ Gh Gh^T + S0h S0h^T - f11 e1 S1h S1h^T
//                                 - u u^T / c ]_i,
//     rhs = -F_z - sum_i u_i F_y,i / c_i,
//     dy_i = (-F_y,i + g (u_i . dz)) / (g c_i).
// Four weighted symmetric Grams per 8x8 block pair, accumulated with
// DMMA.8x8x4 from the shared fragment-packed Psi_0..Psi_2 (the p = 1 kernels'
// structure, newton.cu).  f and its partials come per call as host-sampled
// arrays (the reference callables at (t, y, S1 omega)): the generic drop-in path.
#include <cmath>

#include "common.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kSplit = 4;          // row ranges per instance
constexpr int kMaxCond = 4;
constexpr int kRedWarps = 4;

NYS_DEV double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < nw; ++i) s += red[i];
  return s;
}
NYS_DEV double block_max(double v, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < nw; ++i) s = fmax(s, red[i]);
  return s;
}
NYS_DEV int rows_per_split(int n_c) { return ((n_c + kSplit - 1) / kSplit + 31) / 32 * 32; }

// sampled f and partials at the current point, [6][B][n_c]: f, f0, f1, f00, f01, f11
struct Samples {
  const double* s;
  int B, n_c;
  NYS_DEV double at(int q, int b, int i) const { return s[((size_t)q * B + b) * n_c + i]; }
};

// grid (instances, splits): one row range of one instance
__global__ void __launch_bounds__(kThreads)
    newton2_residual_kernel(const double* __restrict__ S0T, const double* __restrict__ S1T,
                            const double* __restrict__ S2T, int me, int n_c, Samples smp,
                            const double* __restrict__ gamma, const double* __restrict__ X,
                            int ldx, const int* __restrict__ idx, int nk, double* __restrict__ F,
                            double* __restrict__ aux, double* __restrict__ part) {
  extern __shared__ double sh[];
  __shared__ double red[kThreads / 32];
  const int b = idx[blockIdx.x], split = blockIdx.y;
  const double gm = gamma[b];
  const double* x = X + (size_t)b * ldx;
  double* Fb = F + (size_t)b * ldx;
  const int rpc = rows_per_split(n_c);
  const int r0 = split * rpc, r1 = min(n_c, r0 + rpc);
  double* om = sh;                 // me
  double* e1 = sh + me;            // rpc
  double* e2 = e1 + rpc;
  double* g1 = e2 + rpc;           // f1 e1
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  for (int k = tid; k < me; k += nt) om[k] = x[k];
  __syncthreads();
  const double bias = x[me];
  const int y0 = me + 1 + nk;
  double* auxb = aux + (size_t)b * 6 * n_c;
  double fmax_local = 0.0;
  int bad = 0;
  for (int i = r0 + tid; i < r1; i += nt) {
    double a0 = 0.0, a1 = 0.0, c0 = 0.0, c1 = 0.0;
    int k = 0;
#pragma unroll 4
    for (; k + 1 < me; k += 2) {
      a0 = fma(S2T[(size_t)k * n_c + i], om[k], a0);
      a1 = fma(S2T[(size_t)(k + 1) * n_c + i], om[k + 1], a1);
      c0 = fma(S0T[(size_t)k * n_c + i], om[k], c0);
      c1 = fma(S0T[(size_t)(k + 1) * n_c + i], om[k + 1], c1);
    }
    if (k < me) {
      a0 = fma(S2T[(size_t)k * n_c + i], om[k], a0);
      c0 = fma(S0T[(size_t)k * n_c + i], om[k], c0);
    }
    const double s2w = a0 + a1, s0w = c0 + c1;
    const double yi = x[y0 + i];
    const double f = smp.at(0, b, i), f0 = smp.at(1, b, i), f1 = smp.at(2, b, i);
    const double f00 = smp.at(3, b, i), f01 = smp.at(4, b, i), f11 = smp.at(5, b, i);
    const double ee1 = __dsub_rn(s2w, f);
    const double ee2 = __dsub_rn(__dsub_rn(yi, s0w), bias);
    if (!isfinite(ee1) || !isfinite(f)) bad = 1;
    e1[i - r0] = ee1;
    e2[i - r0] = ee2;
    g1[i - r0] = __dmul_rn(f1, ee1);
    const double Fy = __dadd_rn(__dmul_rn(__dmul_rn(-gm, f0), ee1), __dmul_rn(gm, ee2));
    fmax_local = fmax(fmax_local, fabs(Fy));
    Fb[y0 + i] = Fy;
    auxb[i] = f0;
    auxb[n_c + i] = f1;
    auxb[2 * n_c + i] = __dmul_rn(f01, ee1);                                    // t
    auxb[3 * n_c + i] = __dmul_rn(f11, ee1);                                    // s
    auxb[4 * n_c + i] = __dsub_rn(__dadd_rn(1.0, __dmul_rn(f0, f0)), __dmul_rn(f00, ee1));   // c
  }
  __syncthreads();
  const int pstride = 3 * me + 3;
  double* out = part + ((size_t)blockIdx.x * kSplit + split) * pstride;
  for (int k = warp; k < me; k += nw) {
    const double* r2 = S2T + (size_t)k * n_c;
    const double* r1p = S1T + (size_t)k * n_c;
    const double* r0p = S0T + (size_t)k * n_c;
    double a = 0.0, a1 = 0.0, c = 0.0;
    for (int i = r0 + lane; i < r1; i += 32) {
      a = fma(r2[i], e1[i - r0], a);
      a1 = fma(r1p[i], g1[i - r0], a1);
      c = fma(r0p[i], e2[i - r0], c);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      a1 += __shfl_xor_sync(0xffffffffu, a1, o);
      c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    if (lane == 0) {
      out[k] = a;
      out[me + k] = a1;
      out[2 * me + k] = c;
    }
  }
  double se2 = 0.0;
  for (int i = r0 + tid; i < r1; i += nt) se2 += e2[i - r0];
  se2 = block_sum(se2, red);
  const int any_bad = __syncthreads_or(bad);
  const double fmx = block_max(fmax_local, red);
  if (tid == 0) {
    out[3 * me] = se2;
    out[3 * me + 1] = fmx;
    out[3 * me + 2] = any_bad ? 1.0 : 0.0;
  }
}

__global__ void __launch_bounds__(64)
    newton2_residual_finalize_kernel(int me, const double* __restrict__ Ac,
                                     const double* __restrict__ betac,
                                     const double* __restrict__ vals, int nk,
                                     const double* __restrict__ gamma,
                                     const double* __restrict__ X, int ldx,
                                     const int* __restrict__ idx, double* __restrict__ F,
                                     double* __restrict__ norm, const double* __restrict__ part) {
  __shared__ double red[2];
  const int b = idx[blockIdx.x];
  const double gm = gamma[b];
  const double* x = X + (size_t)b * ldx;
  const double* lam = x + me + 1;
  const int pstride = 3 * me + 3;
  const double* pp = part + (size_t)blockIdx.x * kSplit * pstride;
  double* Fb = F + (size_t)b * ldx;
  const int tid = threadIdx.x;
  double fmax_local = 0.0;
  int bad = 0;
  for (int s2 = 0; s2 < kSplit; ++s2) bad |= pp[s2 * pstride + 3 * me + 2] != 0.0;
  for (int k = tid; k < me; k += blockDim.x) {
    double a = 0.0, a1 = 0.0, c = 0.0;
    for (int s2 = 0; s2 < kSplit; ++s2) {   // fixed order over row ranges
      a += pp[s2 * pstride + k];
      a1 += pp[s2 * pstride + me + k];
      c += pp[s2 * pstride + 2 * me + k];
    }
    double acl = 0.0;
    for (int mu = 0; mu < nk; ++mu) acl = __dadd_rn(acl, __dmul_rn(Ac[(size_t)mu * me + k], lam[mu]));
    // omega + g S2^T e1 - g S0^T e2 + Ac^T lam, then - g S1^T (f1 e1) (newton.py:139-142)
    double v = __dadd_rn(__dsub_rn(__dadd_rn(x[k], __dmul_rn(gm, a)), __dmul_rn(gm, c)), acl);
    v = __dsub_rn(v, __dmul_rn(gm, a1));
    Fb[k] = v;
    fmax_local = fmax(fmax_local, fabs(v));
  }
  if (tid == 0) {
    double se2 = 0.0, fy = 0.0;
    for (int s2 = 0; s2 < kSplit; ++s2) {
      se2 += pp[s2 * pstride + 3 * me];
      fy = fmax(fy, pp[s2 * pstride + 3 * me + 1]);
    }
    fmax_local = fmax(fmax_local, fy);
    double bl = 0.0;
    for (int mu = 0; mu < nk; ++mu) bl = __dadd_rn(bl, __dmul_rn(betac[mu], lam[mu]));
    const double Fbias = __dadd_rn(__dmul_rn(-gm, se2), bl);
    Fb[me] = Fbias;
    fmax_local = fmax(fmax_local, fabs(Fbias));
    for (int mu = 0; mu < nk; ++mu) {
      double v = 0.0;
      for (int k = 0; k < me; ++k) v = fma(Ac[(size_t)mu * me + k], x[k], v);
      v = __dsub_rn(__dadd_rn(v, __dmul_rn(betac[mu], x[me])), vals[(size_t)b * nk + mu]);
      Fb[me + 1 + mu] = v;
      fmax_local = fmax(fmax_local, fabs(v));
    }
  }
  for (int o = 16; o; o >>= 1) fmax_local = fmax(fmax_local, __shfl_xor_sync(0xffffffffu, fmax_local, o));
  if ((tid & 31) == 0) red[tid >> 5] = fmax_local;
  __syncthreads();
  if (tid == 0) norm[b] = bad ? NAN : fmax(red[0], blockDim.x > 32 ? red[1] : 0.0);
}

template <int NB>
struct Tri {
  static constexpr int kPairs = NB * (NB + 1) / 2;
  static constexpr NYS_DEV int idx(int I, int J) { return I * NB - (I * (I - 1)) / 2 + (J - I); }
};

// grid (instances, splits): weighted DMMA Grams of the reduced (omega, b) block
template <int NB>
__global__ void __launch_bounds__(kRedWarps * 32)
    newton2_reduce_kernel(const double* __restrict__ psi, int nks, int me, int n_c,
                          const double* __restrict__ aux, const double* __restrict__ F, int ldx,
                          int nk, const int* __restrict__ idx, int kps,
                          double* __restrict__ part) {
  constexpr int NPAIR = Tri<NB>::kPairs;
  extern __shared__ double red[];   // [kRedWarps][NPAIR*64 + NB*8]
  const int b = idx[blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tig = lane & 3, gid = lane >> 2;
  const double* auxb = aux + (size_t)b * 6 * n_c;
  const double* Fy = F + (size_t)b * ldx + me + 1 + nk;
  double acc[NPAIR][2];
#pragma unroll
  for (int q = 0; q < NPAIR; ++q) acc[q][0] = acc[q][1] = 0.0;
  double racc[NB];
#pragma unroll
  for (int F_ = 0; F_ < NB; ++F_) racc[F_] = 0.0;
  const int ks_lo = blockIdx.y * kps, ks_hi = min(nks, ks_lo + kps);
  for (int ks = ks_lo + warp; ks < ks_hi; ks += kRedWarps) {
    const int row = ks * 4 + tig;
    const bool ok = row < n_c;
    const double f0 = ok ? auxb[row] : 0.0;
    const double f1 = ok ? auxb[n_c + row] : 0.0;
    const double t = ok ? auxb[2 * n_c + row] : 0.0;
    const double sw = ok ? auxb[3 * n_c + row] : 0.0;
    const double c = ok ? auxb[4 * n_c + row] : 1.0;
    const double ic = 1.0 / c;
    const double fyc = ok ? Fy[row] * ic : 0.0;
    const double* P0 = psi + ((size_t)ks * 3 + 0) * NB * 32 + lane;
    const double* P1 = psi + ((size_t)ks * 3 + 1) * NB * 32 + lane;
    const double* P2 = psi + ((size_t)ks * 3 + 2) * NB * 32 + lane;
    double gh[NB], x0[NB], x1[NB], u[NB];
#pragma unroll
    for (int F_ = 0; F_ < NB; ++F_) {
      x0[F_] = ok ? P0[F_ * 32] : 0.0;
      x1[F_] = ok ? P1[F_ * 32] : 0.0;
      const double x2 = ok ? P2[F_ * 32] : 0.0;
      gh[F_] = fma(-f1, x1[F_], x2);                                 // Gh = S2h - f1 S1h
      u[F_] = fma(t, x1[F_], fma(f0, gh[F_], x0[F_]));             // u = f0 Gh + S0h + t S1h
      racc[F_] = fma(u[F_], fyc, racc[F_]);                          // sum u F_y / c
    }
#pragma unroll
    for (int I = 0; I < NB; ++I) {
      const double a1 = -sw * x1[I], au = -ic * u[I];
#pragma unroll
      for (int J = I; J < NB; ++J) {
        const int q = Tri<NB>::idx(I, J);
        nys::dmma(acc[q][0], acc[q][1], gh[I], gh[J]);
        nys::dmma(acc[q][0], acc[q][1], x0[I], x0[J]);
        nys::dmma(acc[q][0], acc[q][1], a1, x1[J]);
        nys::dmma(acc[q][0], acc[q][1], au, u[J]);
      }
    }
  }
#pragma unroll
  for (int F_ = 0; F_ < NB; ++F_) {
    racc[F_] += __shfl_xor_sync(0xffffffffu, racc[F_], 1);
    racc[F_] += __shfl_xor_sync(0xffffffffu, racc[F_], 2);
  }
  const int stride = NPAIR * 64 + NB * 8;
  double* mine = red + (size_t)warp * stride;
#pragma unroll
  for (int q = 0; q < NPAIR; ++q) {
    mine[q * 64 + lane * 2] = acc[q][0];
    mine[q * 64 + lane * 2 + 1] = acc[q][1];
  }
  if (tig == 0)
#pragma unroll
    for (int F_ = 0; F_ < NB; ++F_) mine[NPAIR * 64 + F_ * 8 + gid] = racc[F_];
  __syncthreads();
  double* out = part + ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * stride;
  for (int e = threadIdx.x; e < stride; e += blockDim.x) {
    double s2 = 0.0;
    for (int w = 0; w < kRedWarps; ++w) s2 += red[(size_t)w * stride + e];
    out[e] = s2;
  }
}

template <int NB>
__global__ void __launch_bounds__(256)
    newton2_reduce_finalize_kernel(const double* __restrict__ part, int nsplit, int nb, int me,
                                   const double* __restrict__ F, int ldx,
                                   const double* __restrict__ gamma,
                                   const double* __restrict__ Ac, const double* __restrict__ betac,
                                   int nk, const int* __restrict__ idx, double* __restrict__ K,
                                   double* __restrict__ rz) {
  constexpr int NPAIR = Tri<NB>::kPairs;
  const int stride = NPAIR * 64 + NB * 8;
  const int b = idx[blockIdx.x];
  const double gm = gamma[b];
  const int nz = me + 1 + nk, nh = me + 1;
  double* Kb = K + (size_t)blockIdx.x * nz * nz;
  double* rb = rz + (size_t)blockIdx.x * nz;
  const double* Fb = F + (size_t)b * ldx;
  const double* pp = part + (size_t)blockIdx.x * stride;
  for (int e = threadIdx.x; e < NPAIR * 64; e += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < nsplit; ++w) s += pp[(size_t)w * nb * stride + e];
    const int q = e >> 6, l = (e & 63) >> 1, j2 = e & 1;
    int I = 0, rem = q;
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
  for (int e = threadIdx.x; e < nh; e += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < nsplit; ++w) s += pp[(size_t)w * nb * stride + NPAIR * 64 + e];
    rb[e] = -Fb[e] - s;
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

// D = (dz, dy) with dy_i = (-F_y,i + g (u_i . dz)) / (g c_i);  Xc = X + alpha D
__global__ void __launch_bounds__(256)
    newton2_step_kernel(const double* __restrict__ S0T, const double* __restrict__ S1T,
                        const double* __restrict__ S2T, int me, int n_c, int nk,
                        const double* __restrict__ aux, const double* __restrict__ F,
                        const double* __restrict__ dz, const double* __restrict__ gamma,
                        const double* __restrict__ X, double* __restrict__ D,
                        double* __restrict__ Xc, const double* __restrict__ alpha, int ldx,
                        const int* __restrict__ idx) {
  extern __shared__ double dzs[];
  const int b = idx[blockIdx.x];
  const int nz = me + 1 + nk;
  double* Db = D + (size_t)b * ldx;
  for (int k = threadIdx.x; k < nz; k += blockDim.x) dzs[k] = dz[(size_t)blockIdx.x * nz + k];
  __syncthreads();
  const double gm = gamma[b];
  const double* auxb = aux + (size_t)b * 6 * n_c;
  const double* Fb = F + (size_t)b * ldx;
  for (int k = threadIdx.x; k < nz; k += blockDim.x) Db[k] = dzs[k];
  for (int i = threadIdx.x; i < n_c; i += blockDim.x) {
    double a2 = 0.0, a1 = 0.0, a0 = 0.0;
    for (int k = 0; k < me; ++k) {
      const double d = dzs[k];
      a2 = fma(S2T[(size_t)k * n_c + i], d, a2);
      a1 = fma(S1T[(size_t)k * n_c + i], d, a1);
      a0 = fma(S0T[(size_t)k * n_c + i], d, a0);
    }
    const double f0 = auxb[i], f1 = auxb[n_c + i], t = auxb[2 * n_c + i], c = auxb[4 * n_c + i];
    const double gd = fma(-f1, a1, a2);                    // G_i . d_omega
    const double ud = fma(t, a1, fma(f0, gd, a0 + dzs[me]));  // u_i . dz
    Db[nz + i] = (-Fb[nz + i] + gm * ud) / (gm * c);
  }
  __syncthreads();
  const double al = alpha[b];
  const double* Xb = X + (size_t)b * ldx;
  double* Xcb = Xc + (size_t)b * ldx;
  for (int k = threadIdx.x; k < nz + n_c; k += blockDim.x) Xcb[k] = fma(al, Db[k], Xb[k]);
}

}  // namespace

// ------------------------------------------------------------------ C ABI
extern "C" size_t nys_newton2_workspace_bytes(int m_eff, int n_c, int nb) {
  const int NB = (m_eff + 2 + 7) / 8;
  const int nks = (n_c + 3) / 4;
  int ns = (2 * nys::device_sm_count() + nb - 1) / (nb > 0 ? nb : 1);
  ns = ns < 1 ? 1 : (ns > 16 ? 16 : ns);
  while (ns > 1 && nks / ns < 16) --ns;
  const size_t red = (size_t)ns * nb * (NB * (NB + 1) / 2 * 64 + NB * 8);
  const size_t res = (size_t)nb * kSplit * (3 * m_eff + 3);
  return (red > res ? red : res) * sizeof(double);
}

extern "C" int nys_newton2_residual_f64(const double* S0T, const double* S1T, const double* S2T,
                                        int m_eff, int n_c, const double* samples, int B,
                                        const double* Ac, const double* betac, const double* vals,
                                        int n_cond, const double* gamma, const double* X, int ldx,
                                        const int* idx, int nb, double* F, double* norm,
                                        double* aux, void* ws, size_t ws_bytes, void* stream) {
  if (m_eff < 1 || n_c < 1 || n_cond < 0 || n_cond > kMaxCond || nb < 0 ||
      ldx < m_eff + 1 + n_cond + n_c)
    return NYS_EINVAL;
  if (nb == 0) return NYS_OK;
  if (ws == nullptr || ws_bytes < (size_t)nb * kSplit * (3 * m_eff + 3) * sizeof(double))
    return NYS_EWORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int rpc = ((n_c + kSplit - 1) / kSplit + 31) / 32 * 32;
  const size_t smem = ((size_t)m_eff + 3 * (size_t)rpc) * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(newton2_residual_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return nys_host::record_cuda(e);
  double* part = static_cast<double*>(ws);
  newton2_residual_kernel<<<dim3(nb, kSplit), kThreads, smem, st>>>(
      S0T, S1T, S2T, m_eff, n_c, Samples{samples, B, n_c}, gamma, X, ldx, idx, n_cond, F, aux,
      part);
  newton2_residual_finalize_kernel<<<nb, 64, 0, st>>>(m_eff, Ac, betac, vals, n_cond, gamma, X, ldx,
                                                      idx, F, norm, part);
  nys_host::count_launches(2);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" int nys_newton2_reduced_f64(const double* packed, int m_eff, int n_c, const double* aux,
                                       const double* F, int ldx, const double* gamma,
                                       const double* Ac, const double* betac, int n_cond,
                                       const int* idx, int nb, double* K, double* rz, void* ws,
                                       size_t ws_bytes, void* stream) {
  if (m_eff < 1 || n_c < 1 || n_cond < 0 || nb < 0) return NYS_EINVAL;
  if (nb == 0) return NYS_OK;
  const int NB = (m_eff + 2 + 7) / 8;
  const int nks = (n_c + 3) / 4;
  int ns = (2 * nys::device_sm_count() + nb - 1) / nb;
  ns = ns < 1 ? 1 : (ns > 16 ? 16 : ns);
  while (ns > 1 && nks / ns < 16) --ns;
  if (ws == nullptr || ws_bytes < nys_newton2_workspace_bytes(m_eff, n_c, nb)) return NYS_EWORKSPACE;
  const int kps = (nks + ns - 1) / ns;
  double* part = static_cast<double*>(ws);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
#define NYS_RED2(nbv)                                                                            \
  case nbv: {                                                                                    \
    constexpr int NP = nbv * (nbv + 1) / 2;                                                      \
    const size_t smem = (size_t)kRedWarps * (NP * 64 + nbv * 8) * sizeof(double);                \
    auto kern = newton2_reduce_kernel<nbv>;                                                      \
    if (smem > 48 * 1024) {                                                                      \
      cudaError_t e =                                                                            \
          cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);     \
      if (e != cudaSuccess) return nys_host::record_cuda(e);                                     \
    }                                                                                            \
    kern<<<dim3(nb, ns), kRedWarps * 32, smem, st>>>(packed, nks, m_eff, n_c, aux, F, ldx,       \
                                                     n_cond, idx, kps, part);                    \
    newton2_reduce_finalize_kernel<nbv><<<nb, 256, 0, st>>>(part, ns, nb, m_eff, F, ldx, gamma,  \
                                                           Ac, betac, n_cond, idx, K, rz);       \
    break;                                                                                       \
  }
  switch (NB) {
    NYS_RED2(1)
    NYS_RED2(2)
    NYS_RED2(3)
    NYS_RED2(4)
    NYS_RED2(5)
    NYS_RED2(6)
    NYS_RED2(7)
    NYS_RED2(8)
    NYS_RED2(9)
    default: return NYS_EUNSUPPORTED;
  }
#undef NYS_RED2
  nys_host::count_launches(2);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" int nys_newton2_step_f64(const double* S0T, const double* S1T, const double* S2T,
                                    int m_eff, int n_c, int n_cond, const double* aux,
                                    const double* F, const double* dz, const double* gamma,
                                    const double* X, double* D, double* Xc, const double* alpha,
                                    int ldx, const int* idx, int nb, void* stream) {
  if (m_eff < 1 || n_c < 1 || nb < 0) return NYS_EINVAL;
  if (nb == 0) return NYS_OK;
  const int nz = m_eff + 1 + n_cond;
  newton2_step_kernel<<<nb, 256, nz * sizeof(double), static_cast<cudaStream_t>(stream)>>>(
      S0T, S1T, S2T, m_eff, n_c, n_cond, aux, F, dz, gamma, X, D, Xc, alpha, ldx, idx);
  nys_host::count_launches(1);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}
