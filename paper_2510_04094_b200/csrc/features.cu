// Feature rows Psi_ell(t) = K_ell(L, t)^T W (nystrom.py:123-127), batched
// prediction (linear.py:47-53), the ODE-residual certificate (linear.py:175-189)
// and the fragment-native packing of Psi_0..Psi_p used by the batched Gram.
//
// These are not the timed hot kernels for the linear configs except
// psi_pack (once per batch); they are small, L2-resident FP64 GEMV/GEMM-like
// loops with the RBF values generated on the fly.
#include "common.cuh"

namespace {

constexpr int kTP = 16;        // points per CTA tile
constexpr int kFeatThreads = 256;

// out(i, k) for points [i0, i0+kTP): K tile in smem, W read from L2.
// mode 0: dense out[i*ldo + k]; mode 1: packed fragment layout for the batch Gram.
__global__ void __launch_bounds__(kFeatThreads)
    feature_tile_kernel(const double* __restrict__ lm, int m, const double* __restrict__ W,
                        int ldw, int m_eff, double sigma2, int ell,
                        const double* __restrict__ pts, int n_pts, double* __restrict__ out,
                        int ldo, int mode, int n_blocks /*packed: NB*/, int n_orders,
                        int n_rows_pad) {
  extern __shared__ double kt[];   // [kTP][m]
  if (mode == 1) ell = blockIdx.y;  // packed: one launch covers orders 0..n_orders-1
  nys::Hermite H;
  H.init(sigma2, ell);
  const int i0 = blockIdx.x * kTP;
  for (int e = threadIdx.x; e < kTP * m; e += blockDim.x) {
    int ii = e / m, s = e % m;
    int i = i0 + ii;
    double v = 0.0;
    if (i < n_pts) {
      double d = lm[s] - pts[i];
      v = H.poly(ell, d) * nys::rbf(d, sigma2);
    }
    kt[e] = v;
  }
  __syncthreads();
  const int ncols = mode == 0 ? m_eff : n_blocks * 8;
  for (int e = threadIdx.x; e < kTP * ncols; e += blockDim.x) {
    int ii = e / ncols, k = e % ncols;
    int i = i0 + ii;
    if (mode == 0 && i >= n_pts) continue;   // partial tile (condition rows: one point)
    double acc = 0.0;
    if (k < m_eff) {   // four independent partial sums (FP64 FMA latency)
      const double* kr = kt + ii * m;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int s = 0;
#pragma unroll 4
      for (; s + 3 < m; s += 4) {
        a0 = fma(kr[s], W[(size_t)s * ldw + k], a0);
        a1 = fma(kr[s + 1], W[(size_t)(s + 1) * ldw + k], a1);
        a2 = fma(kr[s + 2], W[(size_t)(s + 2) * ldw + k], a2);
        a3 = fma(kr[s + 3], W[(size_t)(s + 3) * ldw + k], a3);
      }
      for (; s < m; ++s) a0 = fma(kr[s], W[(size_t)s * ldw + k], a0);
      acc = (a0 + a1) + (a2 + a3);
    }
    if (mode == 0) {
      if (i < n_pts) out[(size_t)i * ldo + k] = acc;
    } else {
      // extended column m_eff: Psi_0 := 1 so that D_ext[:, m_eff] = -f_p = g
      if (k == m_eff && ell == 0 && i < n_pts) acc = 1.0;
      if (i >= n_pts) acc = 0.0;
      if (i < n_rows_pad) {
        int ks = i >> 2, t = i & 3, F = k >> 3, g = k & 7;
        size_t idx = (((size_t)ks * n_orders + ell) * n_blocks + F) * 32 + g * 4 + t;
        out[idx] = acc;
      }
    }
  }
}

// y[b, i] = Psi_ell(pts_i) . x_b (+ bias).  Psi tile for kTP points in smem.
__global__ void __launch_bounds__(kFeatThreads)
    predict_kernel(const double* __restrict__ lm, int m, const double* __restrict__ W, int ldw,
                   int m_eff, double sigma2, int ell, const double* __restrict__ pts, int n_pts,
                   const double* __restrict__ x, int ldx, int B, double* __restrict__ out,
                   int ldo) {
  extern __shared__ double sm[];
  double* kt = sm;                  // [kTP][m]
  double* psi = sm + kTP * m;       // [kTP][m_eff]
  nys::Hermite H;
  H.init(sigma2, ell);
  const int i0 = blockIdx.x * kTP;
  for (int e = threadIdx.x; e < kTP * m; e += blockDim.x) {
    int ii = e / m, s = e % m, i = i0 + ii;
    double v = 0.0;
    if (i < n_pts) {
      double d = lm[s] - pts[i];
      v = H.poly(ell, d) * nys::rbf(d, sigma2);
    }
    kt[e] = v;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < kTP * m_eff; e += blockDim.x) {
    int ii = e / m_eff, k = e % m_eff;
    double acc = 0.0;
    for (int s = 0; s < m; ++s) acc += kt[ii * m + s] * W[(size_t)s * ldw + k];
    psi[e] = acc;
  }
  __syncthreads();
  const int b0 = blockIdx.y * blockDim.x;
  for (int b = b0 + threadIdx.x; b < min(B, b0 + (int)blockDim.x); b += blockDim.x) {
    const double* xb = x + (size_t)b * ldx;
    double bias = ell == 0 ? xb[m_eff] : 0.0;
    for (int ii = 0; ii < kTP; ++ii) {
      int i = i0 + ii;
      if (i >= n_pts) break;
      double acc = 0.0;
      for (int k = 0; k < m_eff; ++k) acc += psi[ii * m_eff + k] * xb[k];
      out[(size_t)b * ldo + i] = acc + bias;
    }
  }
}

// e_i = sum_s [K_p - sum_k f_k K_{p-k}](s, i) v_s + g_i b - r_i,  v = W omega
// (the Psi omega = K^T (W omega) reassociation: SURVEY.md A1 "predict as
// K^T(W omega)" <= 2.3e-8).  v is rebuilt per CTA in shared memory.
constexpr int kResRowsPerThread = 4;
__global__ void __launch_bounds__(256)
    ode_residual_kernel(const double* __restrict__ lm, int m, const double* __restrict__ W,
                        int ldw, int m_eff, double sigma2, int p,
                        const double* __restrict__ pts, const double* __restrict__ coef,
                        const double* __restrict__ forcing, int n_c,
                        const double* __restrict__ x, double* __restrict__ e) {
  extern __shared__ double v[];
  for (int s = threadIdx.x; s < m; s += blockDim.x) {
    double acc = 0.0;
    for (int k = 0; k < m_eff; ++k) acc += W[(size_t)s * ldw + k] * x[k];
    v[s] = acc;
  }
  __syncthreads();
  const double bias = x[m_eff];
  nys::Hermite H;
  H.init(sigma2, p);
  for (int r = 0; r < kResRowsPerThread; ++r) {
    int i = (blockIdx.x * kResRowsPerThread + r) * blockDim.x + threadIdx.x;
    if (i >= n_c) return;
    double f[nys::kMaxOrder + 1];
#pragma unroll
    for (int k = 1; k <= nys::kMaxOrder; ++k)
      f[k] = k <= p ? coef[(size_t)(k - 1) * n_c + i] : 0.0;
    const double t = pts[i];
    double acc = 0.0;
    for (int s = 0; s < m; ++s) {
      double d = lm[s] - t;
      double gk = H.poly(p, d);
      for (int k = 1; k <= p; ++k) gk -= f[k] * H.poly(p - k, d);
      acc += gk * nys::rbf(d, sigma2) * v[s];
    }
    e[i] = acc - f[p] * bias - forcing[i];
  }
}

// Large landmark sets (m = n full-feature maps): the kTP x m kernel tile no
// longer fits shared memory, so the landmarks stream through it in chunks of
// kMC while the Psi tile (kTP x ncols) accumulates in shared memory.  Same
// outputs as feature_tile_kernel (mode 0 dense, mode 1 packed) and
// predict_kernel (mode 2).
constexpr int kMC = 1024;
__global__ void __launch_bounds__(kFeatThreads)
    feature_chunked_kernel(const double* __restrict__ lm, int m, const double* __restrict__ W,
                           int ldw, int m_eff, double sigma2, int ell,
                           const double* __restrict__ pts, int n_pts, double* __restrict__ out,
                           int ldo, int mode, int n_blocks, int n_orders, int n_rows_pad,
                           const double* __restrict__ x, int ldx, int B) {
  extern __shared__ double sm[];
  if (mode == 1) ell = blockIdx.y;
  const int ncols = mode == 1 ? n_blocks * 8 : m_eff;
  double* kt = sm;                   // [kTP][kMC]
  double* psi = sm + kTP * kMC;      // [kTP][ncols]
  nys::Hermite H;
  H.init(sigma2, ell);
  const int i0 = blockIdx.x * kTP;
  for (int e = threadIdx.x; e < kTP * ncols; e += blockDim.x) psi[e] = 0.0;
  for (int c0 = 0; c0 < m; c0 += kMC) {
    const int mc = min(kMC, m - c0);
    __syncthreads();
    for (int e = threadIdx.x; e < kTP * mc; e += blockDim.x) {
      const int ii = e / mc, s = e % mc, i = i0 + ii;
      double v = 0.0;
      if (i < n_pts) {
        const double d = lm[c0 + s] - pts[i];
        v = H.poly(ell, d) * nys::rbf(d, sigma2);
      }
      kt[ii * kMC + s] = v;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < kTP * ncols; e += blockDim.x) {
      const int ii = e / ncols, k = e % ncols;
      if (k >= m_eff) continue;
      const double* kr = kt + ii * kMC;
      const double* wk = W + (size_t)c0 * ldw + k;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int s = 0;
      for (; s + 3 < mc; s += 4) {
        a0 = fma(kr[s], wk[(size_t)s * ldw], a0);
        a1 = fma(kr[s + 1], wk[(size_t)(s + 1) * ldw], a1);
        a2 = fma(kr[s + 2], wk[(size_t)(s + 2) * ldw], a2);
        a3 = fma(kr[s + 3], wk[(size_t)(s + 3) * ldw], a3);
      }
      for (; s < mc; ++s) a0 = fma(kr[s], wk[(size_t)s * ldw], a0);
      psi[e] += (a0 + a1) + (a2 + a3);
    }
  }
  __syncthreads();
  if (mode == 0) {
    for (int e = threadIdx.x; e < kTP * m_eff; e += blockDim.x) {
      const int ii = e / m_eff, k = e % m_eff, i = i0 + ii;
      if (i < n_pts) out[(size_t)i * ldo + k] = psi[e];
    }
  } else if (mode == 1) {
    for (int e = threadIdx.x; e < kTP * ncols; e += blockDim.x) {
      const int ii = e / ncols, k = e % ncols, i = i0 + ii;
      double acc = psi[e];
      if (k == m_eff && ell == 0 && i < n_pts) acc = 1.0;
      if (i >= n_pts) acc = 0.0;
      if (i < n_rows_pad) {
        const int ks = i >> 2, t = i & 3, F = k >> 3, g = k & 7;
        out[(((size_t)ks * n_orders + ell) * n_blocks + F) * 32 + g * 4 + t] = acc;
      }
    }
  } else {
    const int b0 = blockIdx.y * blockDim.x;
    for (int b = b0 + threadIdx.x; b < min(B, b0 + (int)blockDim.x); b += blockDim.x) {
      const double* xb = x + (size_t)b * ldx;
      const double bias = ell == 0 ? xb[m_eff] : 0.0;
      for (int ii = 0; ii < kTP; ++ii) {
        const int i = i0 + ii;
        if (i >= n_pts) break;
        double acc = 0.0;
        for (int k = 0; k < m_eff; ++k) acc += psi[ii * m_eff + k] * xb[k];
        out[(size_t)b * ldo + i] = acc + bias;
      }
    }
  }
}

// kernel tile budget of the single-pass kernels above
constexpr size_t kTileSmemMax = 200 * 1024;

size_t chunked_smem(int ncols) { return ((size_t)kTP * kMC + (size_t)kTP * ncols) * sizeof(double); }

int launch_chunked(dim3 grid, const double* lm, int m, const double* W, int ldw, int m_eff,
                   double sigma2, int ell, const double* pts, int n_pts, double* out, int ldo,
                   int mode, int n_blocks, int n_orders, int n_rows_pad, const double* x, int ldx,
                   int B, cudaStream_t st) {
  const size_t sm = chunked_smem(mode == 1 ? n_blocks * 8 : m_eff);
  cudaError_t e = cudaFuncSetAttribute(feature_chunked_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return nys_host::record_cuda(e);
  feature_chunked_kernel<<<grid, kFeatThreads, sm, st>>>(lm, m, W, ldw, m_eff, sigma2, ell, pts,
                                                         n_pts, out, ldo, mode, n_blocks, n_orders,
                                                         n_rows_pad, x, ldx, B);
  nys_host::count_launches(1);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

// Extended Gram from explicit feature matrices (large landmark sets, where
// the fused kernels cannot hold the landmark tile): D_ext = [D g r] with
// D = Psi_p - sum_k f_k Psi_{p-k} in the reference's order (linear.py:103-112:
// each f_k Psi_{p-k} product rounded, then subtracted), g = -f_p, r = forcing;
// then E = D_ext^T D_ext, one warp per lower entry.
__global__ void explicit_dext_kernel(const double* __restrict__ psi, int n, int me, int p,
                                     const double* __restrict__ coef,
                                     const double* __restrict__ forcing, double* __restrict__ dext) {
  const int i = blockIdx.x;
  const int ld = me + 2;
  for (int k = threadIdx.x; k < ld; k += blockDim.x) {
    double v;
    if (k < me) {
      v = psi[((size_t)p * n + i) * me + k];
      for (int j = 1; j <= p; ++j) {
        const double t = __dmul_rn(coef[(size_t)(j - 1) * n + i], psi[((size_t)(p - j) * n + i) * me + k]);
        v = __dsub_rn(v, t);
      }
    } else if (k == me) {
      v = -coef[(size_t)(p - 1) * n + i];
    } else {
      v = forcing[i];
    }
    dext[(size_t)k * n + i] = v;     // column-major: coalesced pair dots
  }
}

__global__ void explicit_gram_kernel(const double* __restrict__ dext, int n, int ld,
                                     double* __restrict__ E) {
  const int pair = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (pair >= ld * (ld + 1) / 2) return;
  int a = (int)((sqrt(8.0 * pair + 1.0) - 1.0) * 0.5);
  while (a * (a + 1) / 2 > pair) --a;
  while ((a + 1) * (a + 2) / 2 <= pair) ++a;
  const int b = pair - a * (a + 1) / 2;
  const double* pa = dext + (size_t)a * n;
  const double* pb = dext + (size_t)b * n;
  double s0 = 0.0, s1 = 0.0;
  int i = lane;
  for (; i + 32 < n; i += 64) {
    s0 = fma(pa[i], pb[i], s0);
    s1 = fma(pa[i + 32], pb[i + 32], s1);
  }
  if (i < n) s0 = fma(pa[i], pb[i], s0);
  double s = s0 + s1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    E[(size_t)a * ld + b] = s;
    E[(size_t)b * ld + a] = s;
  }
}

}  // namespace

namespace nys_host {
int launch_psi_pack(const double* lm, int m, const double* W, int ldw, int m_eff, double sigma2,
                    int p, const double* pts, int n_c, int n_blocks, int n_rows_pad,
                    double* packed, cudaStream_t st) {
  size_t sm = (size_t)kTP * m * sizeof(double);
  if (sm > kTileSmemMax)
    return launch_chunked(dim3((n_rows_pad + kTP - 1) / kTP, p + 1), lm, m, W, ldw, m_eff, sigma2,
                          0, pts, n_c, packed, 0, 1, n_blocks, p + 1, n_rows_pad, nullptr, 0, 0,
                          st);
  if (sm > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(feature_tile_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return record_cuda(e);
  }
  dim3 grid((n_rows_pad + kTP - 1) / kTP, p + 1);   // grid.y = order
  feature_tile_kernel<<<grid, kFeatThreads, sm, st>>>(lm, m, W, ldw, m_eff, sigma2, 0, pts, n_c,
                                                      packed, 0, 1, n_blocks, p + 1, n_rows_pad);
  nys_host::count_launches(1);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}
}  // namespace nys_host

extern "C" int nys_feature_matrix_f64(const double* landmarks, int m, const double* W, int ldw,
                                      int m_eff, double sigma2, int ell, const double* pts,
                                      int n_pts, double* out, int ldo, void* stream) {
  if (m < 1 || m_eff < 0 || m_eff > m || ldw < m_eff || ldo < m_eff || ell < 0 ||
      ell > nys::kMaxOrder || !(sigma2 > 0.0) || n_pts < 0)
    return NYS_EINVAL;
  if (n_pts == 0 || m_eff == 0) return NYS_OK;
  size_t sm = (size_t)kTP * m * sizeof(double);
  if (sm > kTileSmemMax)
    return launch_chunked(dim3((n_pts + kTP - 1) / kTP), landmarks, m, W, ldw, m_eff, sigma2, ell,
                          pts, n_pts, out, ldo, 0, 0, 0, 0, nullptr, 0, 0,
                          static_cast<cudaStream_t>(stream));
  if (sm > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(feature_tile_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return nys_host::record_cuda(e);
  }
  dim3 grid((n_pts + kTP - 1) / kTP);
  feature_tile_kernel<<<grid, kFeatThreads, sm, static_cast<cudaStream_t>(stream)>>>(
      landmarks, m, W, ldw, m_eff, sigma2, ell, pts, n_pts, out, ldo, 0, 0, 0, 0);
  nys_host::count_launches(1);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" int nys_predict_f64(const double* landmarks, int m, const double* W, int ldw,
                               int m_eff, double sigma2, int ell, const double* pts, int n_pts,
                               const double* x, int ldx, int B, double* out, int ldo,
                               void* stream) {
  if (m < 1 || m_eff < 1 || m_eff > m || ldw < m_eff || ell < 0 || ell > nys::kMaxOrder ||
      !(sigma2 > 0.0) || n_pts < 0 || B < 0 || ldx < m_eff + 1 || ldo < n_pts)
    return NYS_EINVAL;
  if (n_pts == 0 || B == 0) return NYS_OK;
  size_t sm = (size_t)kTP * (m + m_eff) * sizeof(double);
  if (sm > kTileSmemMax)
    return launch_chunked(dim3((n_pts + kTP - 1) / kTP, (B + kFeatThreads - 1) / kFeatThreads),
                          landmarks, m, W, ldw, m_eff, sigma2, ell, pts, n_pts, out, ldo, 2, 0, 0,
                          0, x, ldx, B, static_cast<cudaStream_t>(stream));
  if (sm > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(predict_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return nys_host::record_cuda(e);
  }
  dim3 grid((n_pts + kTP - 1) / kTP, (B + kFeatThreads - 1) / kFeatThreads);
  predict_kernel<<<grid, kFeatThreads, sm, static_cast<cudaStream_t>(stream)>>>(
      landmarks, m, W, ldw, m_eff, sigma2, ell, pts, n_pts, x, ldx, B, out, ldo);
  nys_host::count_launches(1);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" int nys_ode_residual_f64(const double* landmarks, int m, const double* W, int ldw,
                                    int m_eff, double sigma2, int p, const double* pts,
                                    const double* coef, const double* forcing, int n_c,
                                    const double* x, double* e, void* stream) {
  if (m < 1 || m_eff < 1 || m_eff > m || p < 1 || p > nys::kMaxOrder || n_c < 0 ||
      !(sigma2 > 0.0))
    return NYS_EINVAL;
  if (n_c == 0) return NYS_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int rows_per_block = 256 * kResRowsPerThread;
  ode_residual_kernel<<<(n_c + rows_per_block - 1) / rows_per_block, 256, m * sizeof(double), st>>>(
      landmarks, m, W, ldw, m_eff, sigma2, p, pts, coef, forcing, n_c, x, e);
  nys_host::count_launches(1);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" size_t nys_explicit_gram_workspace_bytes(int n, int m_eff) {
  return ((size_t)n * (m_eff + 2)) * sizeof(double) + 256;
}

extern "C" int nys_explicit_gram_f64(const double* psi, int n, int m_eff, int p,
                                     const double* coef, const double* forcing, double* gram_ext,
                                     void* ws, size_t ws_bytes, void* stream) {
  if (n < 0 || m_eff < 1 || p < 1 || p > nys::kMaxOrder) return NYS_EINVAL;
  if (ws == nullptr || ws_bytes < nys_explicit_gram_workspace_bytes(n, m_eff))
    return NYS_EWORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* dext = static_cast<double*>(ws);
  const int ld = m_eff + 2;
  if (n > 0) explicit_dext_kernel<<<n, 128, 0, st>>>(psi, n, m_eff, p, coef, forcing, dext);
  const int npairs = ld * (ld + 1) / 2;
  explicit_gram_kernel<<<(npairs + 7) / 8, 256, 0, st>>>(dext, n, ld, gram_ext);
  nys_host::count_launches(n > 0 ? 2 : 1);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}
