// Ridge leverage scores of the grid kernel matrix.
//
// Replaces the exact branch of nystrom.ridge_leverage_scores
// (pkg/src/nysode/nystrom.py:58-70): scores = diag(Omega (Omega + n*ridge*I)^-1)
// over the n <= 4000 grid points.  The reference solves the n x n system for n
// right-hand sides with dgesv; here the identity
//
//     Omega (Omega + c I)^-1 = I - c (Omega + c I)^-1,   c = n * ridge,
//
// turns the problem into diag(A^-1) for the SPD matrix A = Omega + c I, i.e. the
// squared column norms of X = L^-1 where A = L L^T.  Both factors come out of
// one right-looking tile sweep (64 x 64 fp64 tiles, lower triangle only):
//
//   step k:  diag   L_kk = chol(A_kk), X_kk = L_kk^-1             (1 CTA)
//            panel  L_ik = A_ik X_kk^T (i > k);  X_kj = X_kk B_kj (j < k)
//            update A_ij -= L_ik L_jk^T (k < j <= i)
//                   B_ij -= L_ik X_kj   (i > k, j <= k)           (DMMA tiles)
//
// B accumulates the right-looking forward substitution of L X = I, so the
// inverse costs one more n^3/3 of DMMA work beside the n^3/3 Cholesky.  Tiles
// are stored contiguously (32 KB each, packed lower-triangular order) with an
// XOR swizzle so a whole tile moves with one 1-D bulk copy (TMA) into shared
// memory and every DMMA fragment load is bank-conflict free.
#include <cuda_runtime.h>

#include <cmath>

#include "common.cuh"

namespace {

using namespace nys;

constexpr int kT = 64;                 // tile edge
constexpr int kTT = kT * kT;           // doubles per tile
constexpr int kThreads = 256;          // 8 warps: 4 (rows) x 2 (cols) of 16 x 32
constexpr uint32_t kTileBytes = kTT * sizeof(double);

// swizzled position of element (r, c) inside a tile: rows stay contiguous, the
// 4-column groups are permuted by row so fragment loads hit 16 distinct banks
NYS_DEV int sw(int r, int c) { return r * kT + (c ^ ((r & 3) << 2)); }

NYS_DEV size_t tile_off(int i, int j) { return ((size_t)i * (i + 1) / 2 + j) * kTT; }

// acc[rb][cb] (8x8 DMMA blocks of this warp's 16 x 32 sub-tile) += sgn * A * op(B)
// A: row-major tile in smem; op(B) = B^T (kBNormal = false) or B (true).
template <bool kBNormal>
NYS_DEV void tile_mma(double (&acc)[2][4][2], const double* As, const double* Bs, bool negate,
                      int ks_begin, int ks_end) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int r0 = (w >> 1) * 16, c0 = (w & 1) * 32;
  const int lr = lane >> 2, lk = lane & 3;
#pragma unroll 4
  for (int ks = ks_begin; ks < ks_end; ++ks) {
    const int kk = ks * 4 + lk;
    double a[2], b[4];
#pragma unroll
    for (int rb = 0; rb < 2; ++rb) {
      a[rb] = As[sw(r0 + rb * 8 + lr, kk)];
      if (negate) a[rb] = -a[rb];
    }
#pragma unroll
    for (int cb = 0; cb < 4; ++cb)
      b[cb] = kBNormal ? Bs[sw(ks * 4 + lk, c0 + cb * 8 + lr)] : Bs[sw(c0 + cb * 8 + lr, kk)];
#pragma unroll
    for (int rb = 0; rb < 2; ++rb)
#pragma unroll
      for (int cb = 0; cb < 4; ++cb) dmma(acc[rb][cb][0], acc[rb][cb][1], a[rb], b[cb]);
  }
}

NYS_DEV void acc_io(double (&acc)[2][4][2], double* tile, bool load) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int r0 = (w >> 1) * 16, c0 = (w & 1) * 32;
#pragma unroll
  for (int rb = 0; rb < 2; ++rb)
#pragma unroll
    for (int cb = 0; cb < 4; ++cb) {
      const int r = r0 + rb * 8 + (lane >> 2), c = c0 + cb * 8 + 2 * (lane & 3);
      double2* p = reinterpret_cast<double2*>(tile + sw(r, c));
      if (load) {
        const double2 v = *p;
        acc[rb][cb][0] = v.x;
        acc[rb][cb][1] = v.y;
      } else {
        *p = make_double2(acc[rb][cb][0], acc[rb][cb][1]);
      }
    }
}

// one or two tiles global -> shared with a single bulk-copy barrier
NYS_DEV void load_tiles(double* s0, const double* g0, double* s1, const double* g1,
                        uint64_t* bar) {
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(bar, g1 ? 2 * kTileBytes : kTileBytes);
    bulk_g2s(s0, g0, kTileBytes, bar);
    if (g1) bulk_g2s(s1, g1, kTileBytes, bar);
  }
  mbar_wait(bar, 0);
}

// A = Omega + c I on the lower tiles, B = I (padding rows/cols: identity)
__global__ void lev_assemble_kernel(const double* __restrict__ grid, int n, double sigma2,
                                    double c, double* __restrict__ At, double* __restrict__ Bt,
                                    int* info) {
  const int i = blockIdx.y, j = blockIdx.x;
  if (j > i) return;
  if (i == 0 && j == 0 && threadIdx.x == 0) *info = 0;
  double* a = At + tile_off(i, j);
  double* b = Bt + tile_off(i, j);
  for (int e = threadIdx.x; e < kTT; e += blockDim.x) {
    const int r = e >> 6, cc = e & 63;
    const int gr = i * kT + r, gc = j * kT + cc;
    double v;
    if (gr < n && gc < n) {
      // kernel_matrix(k, 0, grid, grid) (kernel.py:75-92) plus n*ridge*eye(n)
      v = rbf(grid[gr] - grid[gc], sigma2);
      if (gr == gc) v = v + c;
    } else {
      v = (gr == gc) ? 1.0 : 0.0;
    }
    a[sw(r, cc)] = v;
    b[sw(r, cc)] = (gr == gc) ? 1.0 : 0.0;
  }
}

// ---- diagonal tile: L_kk = chol(A_kk) and X_kk = L_kk^-1 ------------------------
// Blocked by 16 inside the tile, the same right-looking sweep as the tile level:
// per 16-block P a scalar 16-step Cholesky + inverse of S_PP (one element per
// thread, one barrier per step), then DMMA for the panel (L_IP = S_IP X_PP^T,
// X_PJ = X_PP R_PJ) and the trailing update (S_IJ -= L_IP L_JP^T,
// R_IJ -= L_IP X_PJ).  S (working tile) and Xm (R, then X) are swizzled 64 x 64
// tiles in shared memory.
constexpr int kDB = 8;

// 1/sqrt(x) for a positive finite pivot: the hardware approximation refined by
// two Newton steps (the library rsqrt adds special-case branches on the
// factorisation's critical path)
NYS_DEV double rsqrt_pivot(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  y = y * fma(-hx * y, y, 1.5);
  return y;
}

// 8x8 block (r0, c0) of -/+ A * op(B) over k in [0, 16) of 16-blocks, DMMA
template <bool kBNormal>
NYS_DEV void blk_mma(double& d0, double& d1, const double* A, int ar, int ak, const double* B,
                     int br, int bc, bool negate) {
  const int lane = threadIdx.x & 31;
  const int lr = lane >> 2, lk = lane & 3;
#pragma unroll
  for (int ks = 0; ks < kDB / 4; ++ks) {
    double a = A[sw(ar + lr, ak + ks * 4 + lk)];
    if (negate) a = -a;
    // kBNormal: B[k][c] at (br + k, bc + c); else B^T: B[c][k] at (br + c, bc + k)
    const double b = kBNormal ? B[sw(br + ks * 4 + lk, bc + lr)] : B[sw(br + lr, bc + ks * 4 + lk)];
    dmma(d0, d1, a, b);
  }
}

NYS_DEV void blk_io(double& d0, double& d1, double* T, int r0, int c0, bool load) {
  const int lane = threadIdx.x & 31;
  double2* p = reinterpret_cast<double2*>(T + sw(r0 + (lane >> 2), c0 + 2 * (lane & 3)));
  if (load) {
    const double2 v = *p;
    d0 = v.x;
    d1 = v.y;
  } else {
    *p = make_double2(d0, d1);
  }
}

// Cholesky + inverse of the kDB x kDB block S_PP by warp 0 alone (no block
// barriers): lane l holds rows l / kDB + (32 / kDB) i of column l % kDB of both
// the working block and R; column jj and row jj travel through double-buffered
// shared vectors under __syncwarp.  Writes X_PP into Xm.  Returns false
// (uniformly across the warp) on a pivot that is not positive and finite.
NYS_DEV bool warp_chol_inv(const double* S, double* Xm, int o, double (*col)[kDB],
                           double (*row)[kDB]) {
  constexpr int kRS = 32 / kDB;             // row stride between a lane's rows
  constexpr int kPer = kDB * kDB / 32;      // rows per lane
  const int lane = threadIdx.x & 31;
  const int c = lane % kDB, rh = lane / kDB;
  double sv[kPer], xv[kPer];
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    sv[i] = S[sw(o + rh + kRS * i, o + c)];
    xv[i] = (rh + kRS * i == c) ? 1.0 : 0.0;
  }
#pragma unroll
  for (int jj = 0; jj < kDB; ++jj) {
    double* cb = col[jj & 1];
    double* rb = row[jj & 1];
    // owners publish column jj of S (lanes c == jj) and row jj of R
    if (c == jj) {
#pragma unroll
      for (int i = 0; i < kPer; ++i) cb[rh + kRS * i] = sv[i];
    }
    if (rh == (jj % kRS)) rb[c] = xv[jj / kRS];
    __syncwarp();
    const double ajj = cb[jj];
    if (!(ajj > 0.0) || !(ajj < INFINITY)) return false;
    const double inv = rsqrt_pivot(ajj);
    const double lc = cb[c] * inv;
    const double xj = rb[c] * inv;          // X[jj][c] (meaningful for c <= jj)
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int r = rh + kRS * i;
      if (r > jj) {
        const double lr = cb[r] * inv;
        if (c > jj && r >= c) sv[i] = fma(-lr, lc, sv[i]);
        if (c <= jj) xv[i] = fma(-lr, xj, xv[i]);
      } else if (r == jj && c <= jj) {
        xv[i] = xj;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < kPer; ++i) Xm[sw(o + rh + kRS * i, o + c)] = xv[i];
  return true;
}

// S: working tile (A_kk in, destroyed), Xm: X_kk out (both shared, swizzled).
// Returns false (uniformly) when a pivot is not positive and finite.
NYS_DEV bool diag_factor_inverse(double* S, double* Xm) {
  __shared__ double colv[2][kDB], rowv[2][kDB];
  __shared__ int ok;
  const int t = threadIdx.x, w = t >> 5;
  for (int e = t; e < kTT; e += kThreads) Xm[e] = 0.0;
#pragma unroll 1
  for (int P = 0; P < kT / kDB; ++P) {
    const int o = P * kDB;
    __syncthreads();
    // (1) scalar Cholesky + inverse of S_PP on warp 0
    if (w == 0) {
      const bool good = warp_chol_inv(S, Xm, o, colv, rowv);
      if (t == 0) ok = good;
    }
    __syncthreads();
    if (!ok) return false;
    // (2) panel: L_IP = S_IP X_PP^T (I > P) and X_PJ = X_PP R_PJ (J < P), one
    // 8x8 DMMA block per warp; the results overwrite their own operands, so
    // all products finish before any store
    constexpr int kNB = kT / kDB;
    const int npa = kNB - 1 - P;               // blocks below P
    double d0 = 0.0, d1 = 0.0;
    int sr = -1, sc = -1;
    bool on_s = false;
    if (w < npa) {
      on_s = true;
      sr = (P + 1 + w) * kDB;
      sc = o;
      blk_mma<false>(d0, d1, S, sr, o, Xm, o, o, false);
    } else if (w < npa + P) {
      sr = o;
      sc = (w - npa) * kDB;
      blk_mma<true>(d0, d1, Xm, o, o, Xm, o, sc, false);
    }
    __syncthreads();
    if (sr >= 0) blk_io(d0, d1, on_s ? S : Xm, sr, sc, false);
    __syncthreads();
    // (3) trailing: S_IJ -= L_IP L_JP^T (P < J <= I); R_IJ -= L_IP X_PJ (I > P, J <= P)
    const int nS = npa * (npa + 1) / 2;
    const int ntot = nS + npa * (P + 1);
#pragma unroll 1
    for (int blk = w; blk < ntot; blk += 8) {
      double e0, e1;
      if (blk < nS) {
        int ia = 0;
        while ((ia + 1) * (ia + 2) / 2 <= blk) ++ia;
        const int r0 = (P + 1 + ia) * kDB, c0 = (P + 1 + (blk - ia * (ia + 1) / 2)) * kDB;
        blk_io(e0, e1, S, r0, c0, true);
        blk_mma<false>(e0, e1, S, r0, o, S, c0, o, true);
        blk_io(e0, e1, S, r0, c0, false);
      } else {
        const int bb = blk - nS;
        const int r0 = (P + 1 + bb / (P + 1)) * kDB, c0 = (bb % (P + 1)) * kDB;
        blk_io(e0, e1, Xm, r0, c0, true);
        blk_mma<true>(e0, e1, S, r0, o, Xm, o, c0, true);
        blk_io(e0, e1, Xm, r0, c0, false);
      }
    }
  }
  __syncthreads();
  return true;
}

__global__ void __launch_bounds__(kThreads) lev_diag_kernel(const double* __restrict__ At,
                                                            double* __restrict__ Bt, int k,
                                                            int* info) {
  extern __shared__ __align__(128) double smem[];
  double* S = smem;
  double* Xm = smem + kTT;
  __shared__ uint64_t bar;
  load_tiles(S, At + tile_off(k, k), nullptr, nullptr, &bar);
  if (!diag_factor_inverse(S, Xm)) {
    if (threadIdx.x == 0) atomicExch(info, 1);
    return;
  }
  double* out = Bt + tile_off(k, k);
  for (int e = threadIdx.x; e < kTT; e += kThreads) out[e] = Xm[e];
}

// panel: blocks [0, m): L_ik = A_ik X_kk^T for i = k+1+b;  blocks [m, m+k): X_kj = X_kk B_kj
__global__ void __launch_bounds__(kThreads) lev_panel_kernel(double* __restrict__ At,
                                                             double* __restrict__ Bt, int k,
                                                             int nt) {
  extern __shared__ __align__(128) double smem[];
  double* S0 = smem;
  double* S1 = smem + kTT;
  __shared__ uint64_t bar;
  const int m = nt - k - 1;
  const int b = blockIdx.x;
  double acc[2][4][2] = {};
  const double* Xkk = Bt + tile_off(k, k);
  if (b < m) {
    double* tile = At + tile_off(k + 1 + b, k);
    load_tiles(S0, tile, S1, Xkk, &bar);
    // X_kk is lower triangular: columns c need only kk <= c
    const int c_hi = (threadIdx.x >> 5 & 1) * 32 + 32;
    tile_mma<false>(acc, S0, S1, false, 0, c_hi / 4);
    acc_io(acc, tile, false);
  } else {
    double* tile = Bt + tile_off(k, b - m);
    load_tiles(S0, Xkk, S1, tile, &bar);
    // rows r of X_kk need only kk <= r
    const int r_hi = (threadIdx.x >> 6) * 16 + 16;
    tile_mma<true>(acc, S0, S1, false, 0, r_hi / 4);
    acc_io(acc, tile, false);
  }
}

// trailing update of step k: U1 tiles (k < j <= i) then U2 tiles (i > k, j <= k).
// Block 0 owns tile (k+1, k+1), the next diagonal tile: it finishes its update
// in registers and runs the next step's Cholesky + inverse right away (look-
// ahead), so the diagonal factorisation overlaps this step's bulk update
// instead of serialising between launches.
__global__ void __launch_bounds__(kThreads) lev_update_kernel(double* __restrict__ At,
                                                              double* __restrict__ Bt, int k,
                                                              int nt, int* info) {
  extern __shared__ __align__(128) double smem[];
  double* S0 = smem;
  double* S1 = smem + kTT;
  __shared__ uint64_t bar;
  const int m = nt - k - 1;
  const int t1 = m * (m + 1) / 2;
  const int b = blockIdx.x;
  double acc[2][4][2];
  if (b < t1) {
    int a = (int)((sqrt(8.0 * b + 1.0) - 1.0) * 0.5);
    while (a * (a + 1) / 2 > b) --a;
    while ((a + 1) * (a + 2) / 2 <= b) ++a;
    const int i = k + 1 + a, j = k + 1 + (b - a * (a + 1) / 2);
    double* tile = At + tile_off(i, j);
    load_tiles(S0, At + tile_off(i, k), S1, At + tile_off(j, k), &bar);
    acc_io(acc, tile, true);
    tile_mma<false>(acc, S0, S1, true, 0, kT / 4);
    if (b == 0) {            // tile (k+1, k+1): factor it now
      __syncthreads();       // operands consumed
      acc_io(acc, S0, false);
      __syncthreads();
      if (!diag_factor_inverse(S0, S1)) {
        if (threadIdx.x == 0) atomicExch(info, 1);
        return;
      }
      double* out = Bt + tile_off(k + 1, k + 1);
      for (int e = threadIdx.x; e < kTT; e += kThreads) out[e] = S1[e];
      return;
    }
    acc_io(acc, tile, false);
  } else {
    const int bb = b - t1;
    const int i = k + 1 + bb / (k + 1), j = bb % (k + 1);
    double* tile = Bt + tile_off(i, j);
    load_tiles(S0, At + tile_off(i, k), S1, Bt + tile_off(k, j), &bar);
    acc_io(acc, tile, true);
    tile_mma<true>(acc, S0, S1, true, 0, kT / 4);
    acc_io(acc, tile, false);
  }
}

// squared column norms of X per tile: part[i][j*64 + c] = sum_r X_ij[r][c]^2
__global__ void lev_colnorm_kernel(const double* __restrict__ Bt, int nt,
                                   double* __restrict__ part) {
  const int i = blockIdx.y, j = blockIdx.x;
  if (j > i) return;
  __shared__ double red[4][kT];
  const double* x = Bt + tile_off(i, j);
  const int c = threadIdx.x & 63, rq = threadIdx.x >> 6;
  double s = 0.0;
  for (int q = 0; q < 16; ++q) {
    const double v = x[sw(rq + 4 * q, c)];
    s = fma(v, v, s);
  }
  red[rq][c] = s;
  __syncthreads();
  if (rq == 0)
    part[(size_t)i * nt * kT + j * kT + c] = ((red[0][c] + red[1][c]) + red[2][c]) + red[3][c];
}

// scores = max(1 - c * diag(A^-1), 1e-300)   (np.clip at nystrom.py:81)
__global__ void lev_finalize_kernel(const double* __restrict__ part, int n, int nt, double c,
                                    double* __restrict__ scores) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= n) return;
  const int j = col / kT;
  double d = 0.0;
  for (int i = j; i < nt; ++i) d += part[(size_t)i * nt * kT + col];
  const double s = 1.0 - c * d;
  scores[col] = s > 1e-300 ? s : 1e-300;
}

struct LevLayout {
  int nt;
  size_t ntl;
  static LevLayout make(int n) {
    LevLayout L;
    L.nt = (n + kT - 1) / kT;
    L.ntl = (size_t)L.nt * (L.nt + 1) / 2;
    return L;
  }
  size_t bytes() const {
    return (2 * ntl * kTT + (size_t)nt * nt * kT) * sizeof(double) + 256;
  }
};

}  // namespace

extern "C" size_t nys_leverage_workspace_bytes(int n) {
  if (n < 1) return 0;
  return LevLayout::make(n).bytes();
}

extern "C" int nys_leverage_scores_f64(const double* grid, int n, double sigma2, double ridge,
                                       double* scores, int* info, void* ws, size_t ws_bytes,
                                       void* stream) {
  if (n < 1 || n > NYS_LEVERAGE_MAX_N || !(sigma2 > 0.0) || !(ridge >= 0.0)) return NYS_EINVAL;
  const LevLayout L = LevLayout::make(n);
  if (ws == nullptr || ws_bytes < L.bytes()) return NYS_EWORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t base = (reinterpret_cast<size_t>(ws) + 127) & ~(size_t)127;
  double* At = reinterpret_cast<double*>(base);
  double* Bt = At + L.ntl * kTT;
  double* part = Bt + L.ntl * kTT;
  // n * ridge * np.eye(n) (nystrom.py:66): float(n) * ridge
  const double c = (double)n * ridge;
  const int nt = L.nt;
  static bool attr_done = false;
  const int pair_smem = 2 * kTT * (int)sizeof(double);
  if (!attr_done) {
    cudaFuncSetAttribute(lev_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, pair_smem);
    cudaFuncSetAttribute(lev_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, pair_smem);
    cudaFuncSetAttribute(lev_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, pair_smem);
    attr_done = true;
  }
  int launches = 0;
  lev_assemble_kernel<<<dim3(nt, nt), 256, 0, st>>>(grid, n, sigma2, c, At, Bt, info);
  ++launches;
  NYS_CHECK_LAUNCH();
  // diagonal tile 0 alone; tile k+1 is factored inside the update of step k
  lev_diag_kernel<<<1, kThreads, pair_smem, st>>>(At, Bt, 0, info);
  ++launches;
  for (int k = 0; k < nt; ++k) {
    const int m = nt - k - 1;
    const int npanel = m + k;
    if (npanel > 0) {
      lev_panel_kernel<<<npanel, kThreads, pair_smem, st>>>(At, Bt, k, nt);
      ++launches;
    }
    const int nupd = m * (m + 1) / 2 + m * (k + 1);
    if (nupd > 0) {
      lev_update_kernel<<<nupd, kThreads, pair_smem, st>>>(At, Bt, k, nt, info);
      ++launches;
    }
  }
  NYS_CHECK_LAUNCH();
  lev_colnorm_kernel<<<dim3(nt, nt), 256, 0, st>>>(Bt, nt, part);
  lev_finalize_kernel<<<(n + 127) / 128, 128, 0, st>>>(part, n, nt, c, scores);
  launches += 2;
  nys_host::count_launches(launches);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}
