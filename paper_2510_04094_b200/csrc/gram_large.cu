// Fused feature + Gram for ONE linear ODE with many landmarks (m_eff + 2 > 72,
// config 4: m = 256, n_c = 4,194,303).
//
// The 258-wide extended Gram has 561 8x8 block pairs in its upper triangle:
// 287 KB of FP64 accumulators, more than one SM's register file.  The pairs are
// therefore split across a small group of CTAs that work on the same row range
// (grid.y = pair group) and each CTA splits its share across warps.
//
// Operand.  For a well-conditioned landmark matrix (host checks
// s_max / s_min(kept) <= 1e6) the Gram is accumulated in KERNEL space,
//     K = [G g r]^T [G g r],   G_i(s) = [P_p(d) - sum_k f_k P_{p-k}(d)] e^{-d^2/sigma2},
// and projected once at the end, E = W_ext^T K W_ext.  SURVEY.md §0/A1: this
// reassociation costs 1.3e-13 on the config-4 shape (cond(Omega) = 28) but up
// to 2.6e-5 when m_eff < m, hence the host-side gate.  The n x m matrices
// never exist outside a 32-row shared-memory tile.
//
// Work per CTA: a contiguous row range; per 32-row tile the CTA generates the
// G columns its warps need (fragment-native smem layout, conflict-free LDS.64)
// and each warp accumulates a 4 x 4 rectangle of 8x8 blocks (16 pairs, 8
// fragment loads per 16 DMMA.8x8x4).  Partials go to the workspace and are
// reduced in fixed order (deterministic).
#include <cstdint>

#include "common.cuh"

namespace {

constexpr int kRT = 4;             // super-tile edge (blocks)
constexpr int kLargeWarps = 10;    // tasks (super-tiles) per CTA
constexpr int kTileKs = 8;         // 4-row k-steps per row tile (32 rows)

struct LargePlan {
  int Pe, NB, NT, ntasks, ngroups, nrr, ntiles, tiles_per_cta;
  size_t smem;
  static LargePlan make(int n_rows, int m) {
    LargePlan L{};
    L.Pe = m + 2;                                 // kernel-space extended width
    L.NB = (L.Pe + 7) / 8;
    L.NT = (L.NB + kRT - 1) / kRT;                // super-blocks
    L.ntasks = L.NT * (L.NT + 1) / 2;
    L.ngroups = (L.ntasks + kLargeWarps - 1) / kLargeWarps;
    L.ntiles = (n_rows + 4 * kTileKs - 1) / (4 * kTileKs);
    int slots = nys::device_sm_count() * 2;
    int nrr = slots / L.ngroups;
    if (nrr < 1) nrr = 1;
    if (nrr > L.ntiles) nrr = L.ntiles > 0 ? L.ntiles : 1;
    L.nrr = nrr;
    L.tiles_per_cta = (L.ntiles + nrr - 1) / nrr;
    // smem: G tile [kTileKs][NT*kRT][32] + row coefficients
    L.smem = ((size_t)kTileKs * L.NT * kRT * 32 + 32 * 8) * sizeof(double);
    return L;
  }
  size_t part_doubles() const { return (size_t)nrr * ngroups * kLargeWarps * kRT * kRT * 64; }
  size_t ws_bytes(int m_eff) const {
    return (part_doubles() + (size_t)Pe * Pe + (size_t)Pe * (m_eff + 2)) * sizeof(double) + 256;
  }
};

// task t -> super-tile (a, b), a <= b, with rows paired (a, NT-1-a) so groups balance
NYS_DEV void task_ab(int t, int NT, int& a, int& b) {
  // enumerate rows in order 0, NT-1, 1, NT-2, ...
  int idx = t;
  for (int k = 0; k < NT; ++k) {
    int row = (k & 1) ? NT - 1 - (k >> 1) : (k >> 1);
    int len = NT - row;
    if (idx < len) {
      a = row;
      b = row + idx;
      return;
    }
    idx -= len;
  }
  a = b = -1;
}

template <int P>
__global__ void __launch_bounds__(kLargeWarps * 32, 2)
    large_kspace_kernel(const double* __restrict__ lm, int m, double sigma2,
                        const double* __restrict__ pts, const double* __restrict__ coef,
                        const double* __restrict__ forcing, int n_c, int row_begin, int row_end,
                        int NT, int ntasks, int tiles_per_cta, double* __restrict__ part) {
  extern __shared__ __align__(16) double sm[];
  const int NTB = NT * kRT;                     // padded block count
  double* X = sm;                               // [kTileKs][NTB][32]
  double* rowc = X + (size_t)kTileKs * NTB * 32;   // [32][8]: t, q0..qP, g, r

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int group = blockIdx.y;
  const int task = group * kLargeWarps + warp;
  int a = -1, b = -1;
  if (task < ntasks) task_ab(task, NT, a, b);

  // which super-blocks does this CTA need?  (bitmask over NT <= 32)
  __shared__ uint32_t need_mask;
  if (threadIdx.x == 0) need_mask = 0;
  __syncthreads();
  if (lane == 0 && a >= 0) atomicOr(&need_mask, (1u << a) | (1u << b));
  __syncthreads();
  const uint32_t need = need_mask;

  nys::Hermite H;
  H.init(sigma2, P);

  double acc[kRT][kRT][2];
#pragma unroll
  for (int i = 0; i < kRT; ++i)
#pragma unroll
    for (int j = 0; j < kRT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int tile0 = blockIdx.x * tiles_per_cta;
  const int ntiles = (row_end - row_begin + 31) / 32;
  const int tile1 = min(ntiles, tile0 + tiles_per_cta);
  for (int tile = tile0; tile < tile1; ++tile) {
    const int r0 = row_begin + tile * 32;
    // per-row data: combined polynomial coefficients
    if (threadIdx.x < 32) {
      int i = r0 + threadIdx.x;
      bool ok = i < row_end;
      double f[P];
#pragma unroll
      for (int k = 0; k < P; ++k) f[k] = ok ? coef[(size_t)k * n_c + i] : 0.0;
      double* rc = rowc + threadIdx.x * 8;
      rc[0] = ok ? pts[i] : 0.0;
#pragma unroll
      for (int j = 0; j <= P; ++j) {
        double v = H.c[P][j];
#pragma unroll
        for (int k = 1; k <= P; ++k) v = fma(-f[k - 1], H.c[P - k][j], v);
        rc[1 + j] = ok ? v : 0.0;
      }
      rc[6] = ok ? -f[P - 1] : 0.0;
      rc[7] = ok ? forcing[i] : 0.0;
    }
    __syncthreads();
    // generate needed G columns into the fragment layout X[ks][blk][lane]
    const int total = kTileKs * NTB * 32;
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
      int l = e & 31, blk = (e >> 5) % NTB, ks = e / (32 * NTB);
      if (!((need >> (blk / kRT)) & 1u)) continue;
      int row = ks * 4 + (l & 3);
      int s = blk * 8 + (l >> 2);
      const double* rc = rowc + row * 8;
      double v = 0.0;
      if (s < m) {
        double d = lm[s] - rc[0];
        double poly = rc[1 + P];
#pragma unroll
        for (int j = P - 1; j >= 0; --j) poly = poly * d + rc[1 + j];
        v = poly * nys::rbf(d, sigma2);
      } else if (s == m) {
        v = rc[6];
      } else if (s == m + 1) {
        v = rc[7];
      }
      if (r0 + row >= row_end) v = 0.0;
      X[e] = v;
    }
    __syncthreads();
    if (a >= 0) {
      const double* Xl = X + lane;
#pragma unroll 2
      for (int ks = 0; ks < kTileKs; ++ks) {
        double xa[kRT], xb[kRT];
#pragma unroll
        for (int i = 0; i < kRT; ++i) xa[i] = Xl[((size_t)ks * NTB + a * kRT + i) * 32];
#pragma unroll
        for (int j = 0; j < kRT; ++j) xb[j] = Xl[((size_t)ks * NTB + b * kRT + j) * 32];
#pragma unroll
        for (int i = 0; i < kRT; ++i)
#pragma unroll
          for (int j = 0; j < kRT; ++j) nys::dmma(acc[i][j][0], acc[i][j][1], xa[i], xb[j]);
      }
    }
    __syncthreads();
  }
  if (a >= 0) {
    double* out = part + (((size_t)blockIdx.x * gridDim.y + group) * kLargeWarps + warp) *
                             (kRT * kRT * 64) + lane * 2;
#pragma unroll
    for (int i = 0; i < kRT; ++i)
#pragma unroll
      for (int j = 0; j < kRT; ++j) {
        out[(i * kRT + j) * 64] = acc[i][j][0];
        out[(i * kRT + j) * 64 + 1] = acc[i][j][1];
      }
  }
}

// sum partials over row ranges (fixed order) and scatter to dense K (Pe x Pe)
__global__ void large_reduce_kernel(const double* __restrict__ part, int nrr, int ngroups, int NT,
                                    int ntasks, int Pe, double* __restrict__ K) {
  const int per_task = kRT * kRT * 64;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ntasks * per_task;
       e += gridDim.x * blockDim.x) {
    int task = e / per_task, w = e % per_task;
    int a, b;
    task_ab(task, NT, a, b);
    int group = task / kLargeWarps, warp = task % kLargeWarps;
    int ij = w >> 6, lane = (w & 63) >> 1, jj = w & 1;
    int i = ij / kRT, j = ij % kRT;
    double s = 0.0;
    for (int rr = 0; rr < nrr; ++rr)
      s += part[(((size_t)rr * ngroups + group) * kLargeWarps + warp) * per_task + w];
    int I = a * kRT + i, J = b * kRT + j;
    if (a == b && i > j) continue;   // diagonal super-tile: keep the upper part only
    int r = I * 8 + (lane >> 2), c = J * 8 + 2 * (lane & 3) + jj;
    if (I == J && r > c) continue;   // inside a diagonal block write each pair once
    if (r < Pe && c < Pe) {
      K[(size_t)r * Pe + c] = s;
      K[(size_t)c * Pe + r] = s;
    }
  }
}

// T = K W_ext  (Pe x Pw), then E = W_ext^T T (Pw x Pw);  W_ext = diag(W, 1, 1)
__global__ void proj_right_kernel(const double* __restrict__ K, int Pe, const double* __restrict__ W,
                                  int ldw, int m, int m_eff, double* __restrict__ T) {
  const int Pw = m_eff + 2;
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= Pe * Pw) return;
  int r = e / Pw, c = e % Pw;
  double acc = 0.0;
  if (c < m_eff) {
    for (int s = 0; s < m; ++s) acc += K[(size_t)r * Pe + s] * W[(size_t)s * ldw + c];
  } else {
    acc = K[(size_t)r * Pe + m + (c - m_eff)];
  }
  T[e] = acc;
}

__global__ void proj_left_kernel(const double* __restrict__ T, int Pe, const double* __restrict__ W,
                                 int ldw, int m, int m_eff, double* __restrict__ E) {
  const int Pw = m_eff + 2;
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= Pw * Pw) return;
  int r = e / Pw, c = e % Pw;
  if (c < r) return;
  double acc = 0.0;
  if (r < m_eff) {
    for (int s = 0; s < m; ++s) acc += W[(size_t)s * ldw + r] * T[(size_t)s * Pw + c];
  } else {
    acc = T[(size_t)(m + (r - m_eff)) * Pw + c];
  }
  E[(size_t)r * Pw + c] = acc;
  E[(size_t)c * Pw + r] = acc;
}

}  // namespace

namespace nys_host {

size_t fused_gram_large_ws(int n_rows, int m, int m_eff) {
  return LargePlan::make(n_rows, m).ws_bytes(m_eff);
}

int fused_gram_large(const double* lm, int m, const double* W, int ldw, int m_eff, double sigma2,
                     int p, const double* pts, const double* coef, const double* forcing, int n_c,
                     int row_begin, int row_end, double* gram_ext, void* ws, size_t ws_bytes,
                     cudaStream_t st) {
  LargePlan L = LargePlan::make(row_end - row_begin, m);
  if (L.NT > 32) return NYS_EUNSUPPORTED;
  if (ws == nullptr || ws_bytes < L.ws_bytes(m_eff)) return NYS_EWORKSPACE;
  double* part = static_cast<double*>(ws);
  double* K = part + L.part_doubles();
  double* T = K + (size_t)L.Pe * L.Pe;
  dim3 grid(L.nrr, L.ngroups);
  const int nthreads = kLargeWarps * 32;
#define NYS_LARGE(PP)                                                                              \
  do {                                                                                             \
    auto kern = large_kspace_kernel<PP>;                                                           \
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,        \
                                         (int)L.smem);                                             \
    if (e != cudaSuccess) return record_cuda(e);                                                   \
    kern<<<grid, nthreads, L.smem, st>>>(lm, m, sigma2, pts, coef, forcing, n_c, row_begin,        \
                                         row_end, L.NT, L.ntasks, L.tiles_per_cta, part); \
    nys_host::count_launches(1);                                                                   \
  } while (0)
  switch (p) {
    case 1: NYS_LARGE(1); break;
    case 2: NYS_LARGE(2); break;
    case 3: NYS_LARGE(3); break;
    default: NYS_LARGE(4); break;
  }
#undef NYS_LARGE
  NYS_CHECK_LAUNCH();
  int per = L.ntasks * kRT * kRT * 64;
  large_reduce_kernel<<<(per + 255) / 256, 256, 0, st>>>(part, L.nrr, L.ngroups, L.NT, L.ntasks,
                                                         L.Pe, K);
  nys_host::count_launches(1);
  const int Pw = m_eff + 2;
  proj_right_kernel<<<(L.Pe * Pw + 127) / 128, 128, 0, st>>>(K, L.Pe, W, ldw, m, m_eff, T);
  nys_host::count_launches(1);
  proj_left_kernel<<<(Pw * Pw + 127) / 128, 128, 0, st>>>(T, L.Pe, W, ldw, m, m_eff, gram_ext);
  nys_host::count_launches(1);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

}  // namespace nys_host
