// Batched primal KKT assembly + direct solve.
// Block layout of linear.assemble (linear.py:123-133):
//     [ I/gamma + D^T D   D^T g    A_c^T ] [omega ]   [D^T r]
//     [ g^T D             g^T g    beta^T] [  b   ] = [g^T r]
//     [ A_c               beta     0     ] [lambda]   [  v  ]
// and linear.solve (linear.py:140-158): LU with partial pivoting (first
// maximal |a| wins, like LAPACK idamax), solve, one refinement step
// x += solve(M, rhs - M x), non-finite -> SingularSystemError.
// One CTA per instance; M and its LU live in shared memory when they fit
// (side <= ~110: configs 0-3), otherwise in an L2-resident workspace slice
// (config 4, side 259).
#include <cmath>

#include "batch_layout.cuh"
#include "common.cuh"

namespace {

constexpr int kKktThreads = 256;

struct DenseSrc {   // gram_ext[b] is a dense (m_eff+2)^2 matrix
  const double* gram;
  int Pe;
  NYS_DEV double E(int b, int i, int j) const { return gram[(size_t)b * Pe * Pe + (size_t)i * Pe + j]; }
};

struct PartSrc {    // packed block-triangle partials of nys_batch_gram_f64
  const double* part;
  int nsplit, B, NB, npair;
  NYS_DEV double E(int b, int i, int j) const {
    int I = i >> 3, J = j >> 3;
    if (I > J) {
      int t = i;
      i = j;
      j = t;
      t = I;
      I = J;
      J = t;
    }
    int q = I * NB - (I * (I - 1)) / 2 + (J - I);
    int r = i & 7, c = j & 7;
    int off = q * 64 + (r * 4 + (c >> 1)) * 2 + (c & 1);
    double s = 0.0;
    for (int sp = 0; sp < nsplit; ++sp) s += part[((size_t)sp * B + b) * npair * 64 + off];
    return s;
  }
};

template <typename Src>
__global__ void __launch_bounds__(kKktThreads)
    kkt_kernel(Src src, int m_eff, int ncond, const double* __restrict__ Ac,
               const double* __restrict__ beta, const double* __restrict__ values, double gamma,
               int B, double* __restrict__ xout, int* __restrict__ info, double* __restrict__ Mout,
               double* __restrict__ rhsout, double* __restrict__ gws, int use_smem) {
  extern __shared__ __align__(16) double dsm[];
  __shared__ int piv_s;
  __shared__ int bad;
  __shared__ double red_v[kKktThreads / 32];
  __shared__ int red_i[kKktThreads / 32];

  const int b = blockIdx.x;
  const int n = m_eff + 1 + ncond;
  const int me = m_eff;
  double* M0;
  double* LU;
  double* vec;   // rhs0 | x | r | y  (4n)
  if (use_smem) {
    M0 = dsm;
  } else {
    M0 = gws + (size_t)b * (2 * (size_t)n * n + 4 * (size_t)n);
  }
  LU = M0 + (size_t)n * n;
  vec = LU + (size_t)n * n;
  double* rhs0 = vec;
  double* xs = vec + n;
  double* rs = vec + 2 * n;
  int* perm = reinterpret_cast<int*>(vec + 3 * n);   // n ints fit in n doubles
  const int tid = threadIdx.x, nt = blockDim.x;
  const double inv_gamma = 1.0 / gamma;

  // ---- assemble (linear.py:123-133)
  for (int e = tid; e < n * n; e += nt) {
    int i = e / n, j = e % n;
    double v;
    if (i < me && j < me) {
      v = src.E(b, i, j);
      if (i == j) v = inv_gamma + v;
    } else if (i < me && j == me) {
      v = src.E(b, i, me);
    } else if (i == me && j < me) {
      v = src.E(b, j, me);
    } else if (i == me && j == me) {
      v = src.E(b, me, me);
    } else if (i < me) {
      v = Ac[(size_t)(j - me - 1) * me + i];
    } else if (j < me) {
      v = Ac[(size_t)(i - me - 1) * me + j];
    } else if (i == me) {
      v = beta[j - me - 1];
    } else if (j == me) {
      v = beta[i - me - 1];
    } else {
      v = 0.0;
    }
    M0[e] = v;
    LU[e] = v;
    if (Mout) Mout[(size_t)b * n * n + e] = v;
  }
  for (int i = tid; i < n; i += nt) {
    double v;
    if (i < me)
      v = src.E(b, i, me + 1);
    else if (i == me)
      v = src.E(b, me, me + 1);
    else
      v = values[(size_t)b * ncond + (i - me - 1)];
    rhs0[i] = v;
    if (rhsout) rhsout[(size_t)b * n + i] = v;
  }
  if (tid == 0) bad = 0;
  __syncthreads();

  // ---- LU with partial pivoting (dgetrf semantics)
  const int lane = tid & 31, wid = tid >> 5;
  for (int k = 0; k < n; ++k) {
    // pivot: max |LU[i][k]|, i >= k, first index on ties
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
      if (!(v > 0.0)) bad = 1;   // exact zero (or NaN) pivot -> singular
    }
    __syncthreads();
    if (bad) break;
    const int pr = piv_s;
    if (pr != k)
      for (int j = tid; j < n; j += nt) {
        double t = LU[(size_t)k * n + j];
        LU[(size_t)k * n + j] = LU[(size_t)pr * n + j];
        LU[(size_t)pr * n + j] = t;
      }
    __syncthreads();
    const double pivot = LU[(size_t)k * n + k];
    for (int i = k + 1 + tid; i < n; i += nt) LU[(size_t)i * n + k] /= pivot;
    __syncthreads();
    const int w = n - k - 1;
    for (int e = tid; e < w * w; e += nt) {
      int i = k + 1 + e / w, j = k + 1 + e % w;
      LU[(size_t)i * n + j] -= LU[(size_t)i * n + k] * LU[(size_t)k * n + j];
    }
    __syncthreads();
  }
  if (bad) {
    if (tid == 0) info[b] = NYS_INFO_SINGULAR;
    for (int i = tid; i < n; i += nt) xout[(size_t)b * n + i] = NAN;
    return;
  }

  // ---- solve + one refinement step; warp 0 does the triangular sweeps
  for (int pass = 0; pass < 2; ++pass) {
    // rs := rhs (pass 0) or rhs - M0 x (pass 1)
    for (int i = tid; i < n; i += nt) {
      double v = rhs0[i];
      if (pass == 1) {
        double acc = 0.0;
        for (int j = 0; j < n; ++j) acc += M0[(size_t)i * n + j] * xs[j];
        v = v - acc;
      }
      rs[i] = v;
    }
    __syncthreads();
    if (wid == 0) {
      if (lane == 0)
        for (int k = 0; k < n; ++k) {   // row interchanges
          int pr = perm[k];
          if (pr != k) {
            double t = rs[k];
            rs[k] = rs[pr];
            rs[pr] = t;
          }
        }
      __syncwarp();
      for (int i = 1; i < n; ++i) {     // L y = P rhs (unit lower)
        double acc = 0.0;
        for (int j = lane; j < i; j += 32) acc += LU[(size_t)i * n + j] * rs[j];
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) rs[i] -= acc;
        __syncwarp();
      }
      for (int i = n - 1; i >= 0; --i) { // U z = y
        double acc = 0.0;
        for (int j = i + 1 + lane; j < n; j += 32) acc += LU[(size_t)i * n + j] * rs[j];
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) rs[i] = (rs[i] - acc) / LU[(size_t)i * n + i];
        __syncwarp();
      }
    }
    __syncthreads();
    for (int i = tid; i < n; i += nt) xs[i] = pass == 0 ? rs[i] : xs[i] + rs[i];
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

// Warp-per-system variant for small sides (configs 0-3: n <= 96).  The LU lives
// in shared memory (one n x n slice per warp), synchronisation is __syncwarp
// only, and the refinement residual re-reads M's entries from the Gram source
// instead of keeping a second copy (twice the systems per SM).
constexpr int kWarpKktMaxN = 96;
constexpr int kWarpKktWarps = 1;   // 1 warp per CTA: up to 6 systems per SM at n = 67

template <typename Src>
NYS_DEV double kkt_entry(const Src& src, int b, int i, int j, int me, double inv_gamma,
                         const double* Ac, const double* beta) {
  if (i < me && j < me) {
    double v = src.E(b, i, j);
    return i == j ? inv_gamma + v : v;
  }
  if (i < me && j == me) return src.E(b, i, me);
  if (i == me && j < me) return src.E(b, j, me);
  if (i == me && j == me) return src.E(b, me, me);
  if (i < me) return Ac[(size_t)(j - me - 1) * me + i];
  if (j < me) return Ac[(size_t)(i - me - 1) * me + j];
  if (i == me) return beta[j - me - 1];
  if (j == me) return beta[i - me - 1];
  return 0.0;
}

template <typename Src>
__global__ void __launch_bounds__(kWarpKktWarps * 32)
    kkt_warp_kernel(Src src, int m_eff, int ncond, const double* __restrict__ Ac,
                    const double* __restrict__ beta, const double* __restrict__ values,
                    double gamma, int B, double* __restrict__ xout, int* __restrict__ info,
                    double* __restrict__ Mout, double* __restrict__ rhsout) {
  extern __shared__ __align__(16) double dsm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int b = blockIdx.x * kWarpKktWarps + warp;
  if (b >= B) return;
  const int n = m_eff + 1 + ncond, me = m_eff;
  const size_t per = (size_t)n * n + 4 * (size_t)n;
  double* LU = dsm + warp * per;
  double* rhs0 = LU + (size_t)n * n;
  double* xs = rhs0 + n;
  double* rs = xs + n;
  int* perm = reinterpret_cast<int*>(rs + n);
  const double inv_gamma = 1.0 / gamma;

  for (int e = lane; e < n * n; e += 32) {
    int i = e / n, j = e % n;
    double v = kkt_entry(src, b, i, j, me, inv_gamma, Ac, beta);
    LU[e] = v;
    if (Mout) Mout[(size_t)b * n * n + e] = v;
  }
  for (int i = lane; i < n; i += 32) {
    double v = i < me ? src.E(b, i, me + 1)
                      : (i == me ? src.E(b, me, me + 1) : values[(size_t)b * ncond + (i - me - 1)]);
    rhs0[i] = v;
    if (rhsout) rhsout[(size_t)b * n + i] = v;
  }
  __syncwarp();

  int bad = 0;
  for (int k = 0; k < n; ++k) {
    double bv = -1.0;
    int bi = n;
    for (int i = k + lane; i < n; i += 32) {
      double a = fabs(LU[(size_t)i * n + k]);
      if (a > bv) {
        bv = a;
        bi = i;
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
    if (bi != k)
      for (int j = lane; j < n; j += 32) {
        double t = LU[(size_t)k * n + j];
        LU[(size_t)k * n + j] = LU[(size_t)bi * n + j];
        LU[(size_t)bi * n + j] = t;
      }
    __syncwarp();
    const double pivot = LU[(size_t)k * n + k];
    for (int i = k + 1 + lane; i < n; i += 32) LU[(size_t)i * n + k] /= pivot;
    __syncwarp();
    // trailing update, lanes over columns; the pivot row stays in registers
    double urow[(kWarpKktMaxN + 31) / 32];
#pragma unroll
    for (int c = 0; c < (kWarpKktMaxN + 31) / 32; ++c) {
      int j = k + 1 + lane + 32 * c;
      urow[c] = j < n ? LU[(size_t)k * n + j] : 0.0;
    }
    for (int i = k + 1; i < n; ++i) {
      const double l = LU[(size_t)i * n + k];
#pragma unroll
      for (int c = 0; c < (kWarpKktMaxN + 31) / 32; ++c) {
        int j = k + 1 + lane + 32 * c;
        if (j < n) LU[(size_t)i * n + j] -= l * urow[c];
      }
    }
    __syncwarp();
  }
  if (bad) {
    if (lane == 0) info[b] = NYS_INFO_SINGULAR;
    for (int i = lane; i < n; i += 32) xout[(size_t)b * n + i] = NAN;
    return;
  }
  for (int pass = 0; pass < 2; ++pass) {
    for (int i = lane; i < n; i += 32) {
      double v = rhs0[i];
      if (pass == 1) {
        double acc = 0.0;
        for (int j = 0; j < n; ++j) acc += kkt_entry(src, b, i, j, me, inv_gamma, Ac, beta) * xs[j];
        v = v - acc;
      }
      rs[i] = v;
    }
    __syncwarp();
    if (lane == 0)
      for (int k = 0; k < n; ++k) {
        int pr = perm[k];
        if (pr != k) {
          double t = rs[k];
          rs[k] = rs[pr];
          rs[pr] = t;
        }
      }
    __syncwarp();
    for (int i = 1; i < n; ++i) {
      double acc = 0.0;
      for (int j = lane; j < i; j += 32) acc += LU[(size_t)i * n + j] * rs[j];
#pragma unroll
      for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) rs[i] -= acc;
      __syncwarp();
    }
    for (int i = n - 1; i >= 0; --i) {
      double acc = 0.0;
      for (int j = i + 1 + lane; j < n; j += 32) acc += LU[(size_t)i * n + j] * rs[j];
#pragma unroll
      for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) rs[i] = (rs[i] - acc) / LU[(size_t)i * n + i];
      __syncwarp();
    }
    for (int i = lane; i < n; i += 32) xs[i] = pass == 0 ? rs[i] : xs[i] + rs[i];
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

size_t kkt_smem_bytes(int n) { return (2 * (size_t)n * n + 4 * (size_t)n) * sizeof(double); }
constexpr size_t kKktSmemMax = 200 * 1024;

template <typename Src>
int launch_kkt(Src src, int m_eff, int ncond, const double* Ac, const double* beta,
               const double* values, double gamma, int B, double* x, int* info, double* M,
               double* rhs, void* ws, size_t ws_bytes, cudaStream_t st) {
  const int n = m_eff + 1 + ncond;
  if (n <= kWarpKktMaxN) {
    auto wk = kkt_warp_kernel<Src>;
    size_t dyn = kWarpKktWarps * ((size_t)n * n + 4 * (size_t)n) * sizeof(double);
    if (dyn > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(wk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
      if (e != cudaSuccess) return nys_host::record_cuda(e);
    }
    wk<<<(B + kWarpKktWarps - 1) / kWarpKktWarps, kWarpKktWarps * 32, dyn, st>>>(
        src, m_eff, ncond, Ac, beta, values, gamma, B, x, info, M, rhs);
    nys_host::count_launches(1);
    NYS_CHECK_LAUNCH();
    return NYS_OK;
  }
  size_t per = kkt_smem_bytes(n);
  int use_smem = per <= kKktSmemMax;
  size_t dyn = use_smem ? per : 0;
  if (!use_smem && (ws == nullptr || ws_bytes < per * B)) return NYS_EWORKSPACE;
  auto kern = kkt_kernel<Src>;
  if (dyn > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (e != cudaSuccess) return nys_host::record_cuda(e);
  }
  kern<<<B, kKktThreads, dyn, st>>>(src, m_eff, ncond, Ac, beta, values, gamma, B, x, info, M,
                                    rhs, static_cast<double*>(ws), use_smem);
  nys_host::count_launches(1);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

}  // namespace

extern "C" size_t nys_kkt_workspace_bytes(int m_eff, int n_cond, int B) {
  int n = m_eff + 1 + n_cond;
  size_t per = kkt_smem_bytes(n);
  return per <= kKktSmemMax ? 0 : per * (size_t)B;
}

extern "C" int nys_kkt_solve_f64(const double* gram_ext, int m_eff, int n_cond, const double* Ac,
                                 const double* beta, const double* values, double gamma, int B,
                                 double* x, int* info, double* M, double* rhs, void* workspace,
                                 size_t workspace_bytes, void* stream) {
  if (m_eff < 1 || n_cond < 0 || B < 0 || !(gamma > 0.0)) return NYS_EINVAL;
  if (B == 0) return NYS_OK;
  DenseSrc src{gram_ext, m_eff + 2};
  return launch_kkt(src, m_eff, n_cond, Ac, beta, values, gamma, B, x, info, M, rhs, workspace,
                    workspace_bytes, static_cast<cudaStream_t>(stream));
}

extern "C" int nys_batch_kkt_solve_f64(const void* batch_workspace, int n_c, int m_eff, int p,
                                       int n_cond, const double* Ac, const double* beta,
                                       const double* values, double gamma, int B, double* x,
                                       int* info, void* stream) {
  if (m_eff < 1 || n_cond < 0 || B < 0 || !(gamma > 0.0) || p < 1 || p > 2) return NYS_EINVAL;
  if (B == 0) return NYS_OK;
  nys::BatchLayout L = nys::BatchLayout::make(n_c, m_eff, p, B);
  PartSrc src{L.part(batch_workspace), L.nsplit, B, L.NB, L.npair};
  return launch_kkt(src, m_eff, n_cond, Ac, beta, values, gamma, B, x, info, nullptr, nullptr,
                    nullptr, 0, static_cast<cudaStream_t>(stream));
}
