// Fused feature + Gram for ONE linear ODE (configs 0, 1 and any m_eff <= 70).
// Numeric core of linear.assemble (linear.py:103-133) without the n x m
// feature matrices: per 8-row tile a warp
//   1. generates the order-combined kernel row in registers,
//        G_i(s) = [P_p(d) - sum_k f_k(t_i) P_{p-k}(d)] exp(-d^2/sigma2),  d = L_s - t_i
//      (kernel.py:75-82 polynomials; orders combined in kernel space before the
//      single projection -- SURVEY.md A1: <= 1.4e-9, parity-safe), extended by
//      the two columns g_i = -f_p(t_i) and r_i;
//   2. projects through W_ext = diag(W, 1, 1) with DMMA.8x8x4 (W fragments in
//      shared memory) -- the MMA output fragment D^T is laid out exactly as the
//      A/B operand fragment of the Gram MMA, so no shuffle or smem transpose;
//   3. accumulates the upper block triangle of E = [D g r]^T [D g r] in
//      registers with DMMA.8x8x4.
// Warps reduce in shared memory, CTAs in a fixed-order finalize kernel.
#include "common.cuh"

namespace {

template <int NB>
struct Tri {
  static constexpr int kPairs = NB * (NB + 1) / 2;
  static constexpr NYS_DEV int idx(int I, int J) { return I * NB - (I * (I - 1)) / 2 + (J - I); }
};

constexpr int kFusedWarps = 4;

template <int NB, int P>
__global__ void __launch_bounds__(kFusedWarps * 32)
    fused_gram_kernel(const double* __restrict__ lm, int m, const double* __restrict__ W, int ldw,
                      int m_eff, double sigma2, const double* __restrict__ pts,
                      const double* __restrict__ coef, const double* __restrict__ forcing,
                      int n_c, int row_begin, int row_end, int MK, double* __restrict__ part) {
  constexpr int NPAIR = Tri<NB>::kPairs;
  extern __shared__ __align__(16) double sm[];
  double* wf = sm;                              // [MK][NB][32]
  double* lms = wf + (size_t)MK * NB * 32;      // [MK*4]
  double* red = lms + MK * 4;                   // [kFusedWarps][NPAIR][64]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tig = lane & 3, gid = lane >> 2;

  for (int e = threadIdx.x; e < MK * NB * 32; e += blockDim.x) {
    int sk = e / (NB * 32), F = (e / 32) % NB, l = e & 31;
    int s = 4 * sk + (l & 3), c = 8 * F + (l >> 2);
    double v = 0.0;
    if (s < m && c < m_eff)
      v = W[(size_t)s * ldw + c];
    else if ((s == m && c == m_eff) || (s == m + 1 && c == m_eff + 1))
      v = 1.0;
    wf[e] = v;
  }
  for (int s = threadIdx.x; s < MK * 4; s += blockDim.x) lms[s] = s < m ? lm[s] : 0.0;
  __syncthreads();

  nys::Hermite H;
  H.init(sigma2, P);

  double acc[NPAIR][2];
#pragma unroll
  for (int q = 0; q < NPAIR; ++q) acc[q][0] = acc[q][1] = 0.0;

  const int ntiles = (row_end - row_begin + 7) / 8;
  for (int t = blockIdx.x * kFusedWarps + warp; t < ntiles; t += gridDim.x * kFusedWarps) {
    const int i = row_begin + 8 * t + gid;
    const bool valid = i < row_end;
    double ti = 0.0, f[P], r = 0.0;
#pragma unroll
    for (int k = 0; k < P; ++k) f[k] = valid ? coef[(size_t)k * n_c + i] : 0.0;
    if (valid) {
      ti = pts[i];
      r = forcing[i];
    }
    // combined polynomial q(d) = P_p(d) - sum_k f_k P_{p-k}(d)
    double q[P + 1];
#pragma unroll
    for (int j = 0; j <= P; ++j) {
      double v = H.c[P][j];
#pragma unroll
      for (int k = 1; k <= P; ++k) v = fma(-f[k - 1], H.c[P - k][j], v);
      q[j] = v;
    }
    double dacc[NB][2];
#pragma unroll
    for (int F = 0; F < NB; ++F) dacc[F][0] = dacc[F][1] = 0.0;
    const double* wl = wf + lane;
#pragma unroll 2
    for (int sk = 0; sk < MK; ++sk) {
      const int s = 4 * sk + tig;
      double gval = 0.0;
      if (valid) {
        if (s < m) {
          double d = lms[s] - ti;
          double poly = q[P];
#pragma unroll
          for (int j = P - 1; j >= 0; --j) poly = poly * d + q[j];
          gval = poly * nys::rbf(d, sigma2);
        } else if (s == m) {
          gval = -f[P - 1];
        } else if (s == m + 1) {
          gval = r;
        }
      }
#pragma unroll
      for (int F = 0; F < NB; ++F) nys::dmma(dacc[F][0], dacc[F][1], wl[(sk * NB + F) * 32], gval);
    }
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int I = 0; I < NB; ++I)
#pragma unroll
        for (int J = I; J < NB; ++J)
          nys::dmma(acc[Tri<NB>::idx(I, J)][0], acc[Tri<NB>::idx(I, J)][1], dacc[I][j], dacc[J][j]);
  }

  // warp partials -> CTA partial (fixed order)
#pragma unroll
  for (int qq = 0; qq < NPAIR; ++qq) {
    red[((size_t)warp * NPAIR + qq) * 64 + lane * 2] = acc[qq][0];
    red[((size_t)warp * NPAIR + qq) * 64 + lane * 2 + 1] = acc[qq][1];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < NPAIR * 64; e += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < kFusedWarps; ++w) s += red[(size_t)w * NPAIR * 64 + e];
    part[(size_t)blockIdx.x * NPAIR * 64 + e] = s;
  }
}

// CTA partials -> dense E (Pe x Pe), fixed summation order
// partials -> dense E.  Eight lanes per output entry, each summing a fixed
// contiguous range of the CTA partials (8 loads in flight), combined by a
// fixed shuffle tree: deterministic, and 8x the parallelism of one thread per
// entry (config 1: 28 x 64 entries over ~300 partials)
constexpr int kFinSub = 8;
__global__ void fused_finalize_kernel(const double* __restrict__ part, int nparts, int NB, int Pe,
                                      double* __restrict__ gram) {
  const int npair = NB * (NB + 1) / 2;
  const int g = threadIdx.x & (kFinSub - 1);
  const int e = (blockIdx.x * blockDim.x + threadIdx.x) / kFinSub;
  const bool ok = e < npair * 64;
  const int chunk = (nparts + kFinSub - 1) / kFinSub;
  const int p0 = min(nparts, g * chunk), p1 = min(nparts, p0 + chunk);
  const size_t step = (size_t)npair * 64;
  const double* src = part + (ok ? e : 0);
  double s = 0.0;
  int p = p0;
  if (ok) {
    for (; p + 8 <= p1; p += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldg(src + (p + u) * step);
#pragma unroll
      for (int u = 0; u < 8; ++u) s += v[u];
    }
    for (; p < p1; ++p) s += src[p * step];
  }
#pragma unroll
  for (int o = 1; o < kFinSub; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (!ok || g != 0) return;
  const int q = e >> 6, w = e & 63, lane = w >> 1, j = w & 1;
  int I = 0, rem = q;
  while (rem >= NB - I) {
    rem -= NB - I;
    ++I;
  }
  const int J = I + rem;
  const int r = I * 8 + (lane >> 2), c = J * 8 + 2 * (lane & 3) + j;
  if (r < Pe && c < Pe) {
    gram[(size_t)r * Pe + c] = s;
    gram[(size_t)c * Pe + r] = s;
  }
}

struct FusedPlan {
  int NB, MK, npair, nctas;
  size_t smem;
  static FusedPlan make(int n_rows, int m, int m_eff) {
    FusedPlan f{};
    f.NB = (m_eff + 2 + 7) / 8;
    f.MK = (m + 2 + 3) / 4;
    f.npair = f.NB * (f.NB + 1) / 2;
    int ntiles = (n_rows + 7) / 8;
    int want = (ntiles + kFusedWarps - 1) / kFusedWarps;
    int cap = nys::device_sm_count() * 2;
    f.nctas = want < cap ? (want > 0 ? want : 1) : cap;
    f.smem = ((size_t)f.MK * f.NB * 32 + f.MK * 4 + (size_t)kFusedWarps * f.npair * 64) * sizeof(double);
    return f;
  }
  size_t ws_bytes() const { return (size_t)nctas * npair * 64 * sizeof(double); }
};

template <int NB, int P>
int launch_fused(const FusedPlan& F, const double* lm, int m, const double* W, int ldw, int m_eff,
                 double sigma2, const double* pts, const double* coef, const double* forcing,
                 int n_c, int rb, int re, double* part, cudaStream_t st) {
  auto kern = fused_gram_kernel<NB, P>;
  if (F.smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)F.smem);
    if (e != cudaSuccess) return nys_host::record_cuda(e);
  }
  kern<<<F.nctas, kFusedWarps * 32, F.smem, st>>>(lm, m, W, ldw, m_eff, sigma2, pts, coef, forcing,
                                                  n_c, rb, re, F.MK, part);
  nys_host::count_launches(1);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

template <int P>
int dispatch_fused(const FusedPlan& F, const double* lm, int m, const double* W, int ldw,
                   int m_eff, double sigma2, const double* pts, const double* coef,
                   const double* forcing, int n_c, int rb, int re, double* part, cudaStream_t st) {
#define NYS_FUSED_CASE(nb) \
  case nb: return launch_fused<nb, P>(F, lm, m, W, ldw, m_eff, sigma2, pts, coef, forcing, n_c, rb, re, part, st);
  switch (F.NB) {
    NYS_FUSED_CASE(1)
    NYS_FUSED_CASE(2)
    NYS_FUSED_CASE(3)
    NYS_FUSED_CASE(4)
    NYS_FUSED_CASE(5)
    NYS_FUSED_CASE(6)
    NYS_FUSED_CASE(7)
    NYS_FUSED_CASE(8)
    NYS_FUSED_CASE(9)
    default: return NYS_EUNSUPPORTED;
  }
#undef NYS_FUSED_CASE
}

}  // namespace

namespace nys_host {
// the large-m path (gram_large.cu) handles m_eff + 2 > 72
int fused_gram_large(const double* lm, int m, const double* W, int ldw, int m_eff, double sigma2,
                     int p, const double* pts, const double* coef, const double* forcing, int n_c,
                     int row_begin, int row_end, double* gram_ext, void* ws, size_t ws_bytes,
                     cudaStream_t st);
size_t fused_gram_large_ws(int n_rows, int m, int m_eff);
}  // namespace nys_host

extern "C" size_t nys_fused_gram_workspace_bytes(int n_c, int m, int m_eff, int p) {
  (void)p;
  if ((m_eff + 2 + 7) / 8 > 9) return nys_host::fused_gram_large_ws(n_c, m, m_eff);
  return FusedPlan::make(n_c, m, m_eff).ws_bytes() + 256;
}

extern "C" int nys_fused_gram_f64(const double* landmarks, int m, const double* W, int ldw,
                                  int m_eff, double sigma2, int p, const double* pts,
                                  const double* coef, const double* forcing, int n_c,
                                  int row_begin, int row_end, double* gram_ext, void* workspace,
                                  size_t workspace_bytes, void* stream) {
  if (m < 1 || m_eff < 1 || m_eff > m || ldw < m_eff || p < 1 || p > nys::kMaxOrder || n_c < 0 ||
      row_begin < 0 || row_end > n_c || row_begin > row_end || !(sigma2 > 0.0))
    return NYS_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if ((m_eff + 2 + 7) / 8 > 9)
    return nys_host::fused_gram_large(landmarks, m, W, ldw, m_eff, sigma2, p, pts, coef, forcing,
                                      n_c, row_begin, row_end, gram_ext, workspace,
                                      workspace_bytes, st);
  FusedPlan F = FusedPlan::make(row_end - row_begin, m, m_eff);
  if (workspace == nullptr || workspace_bytes < F.ws_bytes()) return NYS_EWORKSPACE;
  double* part = static_cast<double*>(workspace);
  int rc;
  switch (p) {
    case 1: rc = dispatch_fused<1>(F, landmarks, m, W, ldw, m_eff, sigma2, pts, coef, forcing, n_c, row_begin, row_end, part, st); break;
    case 2: rc = dispatch_fused<2>(F, landmarks, m, W, ldw, m_eff, sigma2, pts, coef, forcing, n_c, row_begin, row_end, part, st); break;
    case 3: rc = dispatch_fused<3>(F, landmarks, m, W, ldw, m_eff, sigma2, pts, coef, forcing, n_c, row_begin, row_end, part, st); break;
    default: rc = dispatch_fused<4>(F, landmarks, m, W, ldw, m_eff, sigma2, pts, coef, forcing, n_c, row_begin, row_end, part, st); break;
  }
  if (rc) return rc;
  fused_finalize_kernel<<<(F.npair * 64 * kFinSub + 255) / 256, 256, 0, st>>>(
      part, F.nctas, F.NB, m_eff + 2, gram_ext);
  nys_host::count_launches(1);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}
