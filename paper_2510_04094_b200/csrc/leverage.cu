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

// Right-looking tile sweep over the assembled lower tiles At (B = I): leaves
// X = L^-1 in Bt.  Returns the number of launches.
int tile_sweep(double* At, double* Bt, int nt, int* info, cudaStream_t st) {
  static bool attr_done = false;
  const int pair_smem = 2 * kTT * (int)sizeof(double);
  if (!attr_done) {
    cudaFuncSetAttribute(lev_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, pair_smem);
    cudaFuncSetAttribute(lev_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, pair_smem);
    cudaFuncSetAttribute(lev_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, pair_smem);
    attr_done = true;
  }
  int launches = 0;
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
  return launches;
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


// ---- sketch branch (nystrom.py:71-80, n > 4000) -------------------------------
// The reference eigendecomposes the c x c sketch W = K(x, x) (x = grid[idx],
// c = 2000) and keeps vals > 1e-12 vals.max().  The kept spectrum is the
// numerical range of W, so W is compressed first by a pivoted Cholesky
// W ~ G G^T (stopped when the largest remaining diagonal falls below 1e-15,
// far under the 1e-12 relative cut), and the small r x r problem G^T G = U M U^T
// (same nonzero spectrum, eigenvectors v = G u / sqrt(mu)) goes to the
// divide-and-conquer eigensolver.  With T = G U_k M_k^-1:
//   A = C T (n x k, C = K(grid, x)),   scores_i = a_i^T (A^T A + n ridge I)^-1 a_i
// the latter from the same tile Cholesky + inverse sweep: ||L^-1 a_i||^2.
constexpr int kPcThreads = 1024;

__global__ void __launch_bounds__(kPcThreads)
    lev_pchol_kernel(const double* __restrict__ x, int c, double sigma2, double tol, int cap,
                     double* __restrict__ G, int* __restrict__ out) {
  extern __shared__ __align__(16) double sm[];
  double* d = sm;          // remaining diagonal
  double* xs = sm + c;     // sketch points
  __shared__ double rv[32];
  __shared__ int ri[32];
  __shared__ int s_p;
  __shared__ double s_dp;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int i = tid; i < c; i += kPcThreads) {
    d[i] = 1.0;            // rbf(0) = exp(-0) = 1
    xs[i] = x[i];
  }
  __syncthreads();
  int k = 0;
  bool converged = false;
  for (; k < cap; ++k) {
    // argmax of the remaining diagonal, first index on ties
    double bv = -1.0;
    int bi = 0;
    for (int i = tid; i < c; i += kPcThreads)
      if (d[i] > bv) {
        bv = d[i];
        bi = i;
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (lane == 0) {
      rv[w] = bv;
      ri[w] = bi;
    }
    __syncthreads();
    if (w == 0) {
      bv = rv[lane];
      bi = ri[lane];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      if (lane == 0) {
        s_p = bi;
        s_dp = bv;
      }
    }
    __syncthreads();
    const int p = s_p;
    const double dp = s_dp;
    if (!(dp > tol)) {
      converged = true;
      break;
    }
    const double inv = 1.0 / sqrt(dp);
    const double xp = xs[p];
    double* gk = G + (size_t)k * c;
    for (int i = tid; i < c; i += kPcThreads) {
      double g0 = rbf(xs[i] - xp, sigma2), g1 = 0.0;
      int kk = 0;
      for (; kk + 1 < k; kk += 2) {
        g0 = fma(-G[(size_t)kk * c + i], G[(size_t)kk * c + p], g0);
        g1 = fma(-G[(size_t)(kk + 1) * c + i], G[(size_t)(kk + 1) * c + p], g1);
      }
      if (kk < k) g0 = fma(-G[(size_t)kk * c + i], G[(size_t)kk * c + p], g0);
      const double g = (g0 + g1) * inv;
      gk[i] = g;
      d[i] = (i == p) ? 0.0 : d[i] - g * g;
    }
    __syncthreads();
  }
  if (tid == 0) {
    out[0] = k;
    out[1] = converged ? 1 : 0;
  }
}

// H = G^T G (r x r), one warp per lower entry, mirrored
__global__ void lev_gtg_kernel(const double* __restrict__ G, int c, int r, double* __restrict__ H) {
  const int pair = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (pair >= r * (r + 1) / 2) return;
  int a = (int)((sqrt(8.0 * pair + 1.0) - 1.0) * 0.5);
  while (a * (a + 1) / 2 > pair) --a;
  while ((a + 1) * (a + 2) / 2 <= pair) ++a;
  const int b = pair - a * (a + 1) / 2;
  const double* ga = G + (size_t)a * c;
  const double* gb = G + (size_t)b * c;
  double s = 0.0;
  for (int i = lane; i < c; i += 32) s = fma(ga[i], gb[i], s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    H[(size_t)a * r + b] = s;
    H[(size_t)b * r + a] = s;
  }
}

// T[j][l] = (sum_a G[a][j] U[a][l]) / mu[l] for l < k_eff   (T: c x r, row-major)
__global__ void lev_sketch_T_kernel(const double* __restrict__ G, int c, int r,
                                    const double* __restrict__ U, const double* __restrict__ mu,
                                    const int* __restrict__ meta, double* __restrict__ T) {
  const int l = blockIdx.y;
  if (l >= meta[0]) return;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= c) return;
  double s = 0.0;
  for (int a = 0; a < r; ++a) s = fma(G[(size_t)a * c + j], U[(size_t)a * r + l], s);
  T[(size_t)j * r + l] = s / mu[l];
}

// A[l][i] = sum_j rbf(grid_i - x_j) T[j][l]   (A: r x n, l < k_eff)
// block: 64 rows i x 32 columns l, j streamed through shared memory in chunks
__global__ void __launch_bounds__(256)
    lev_sketch_A_kernel(const double* __restrict__ grid, int n, const double* __restrict__ x,
                        int c, double sigma2, const double* __restrict__ T, int r,
                        const int* __restrict__ meta, double* __restrict__ A) {
  constexpr int kI = 64, kL = 32, kJ = 48;
  __shared__ double Cs[kJ][kI + 1];
  __shared__ double Ts[kJ][kL];
  const int keff = meta[0];
  const int i0 = blockIdx.x * kI, l0 = blockIdx.y * kL;
  if (l0 >= keff) return;
  const int t = threadIdx.x;
  const int ii = t & 63, lg = t >> 6;      // row, group of 8 columns
  const double gi = (i0 + ii < n) ? grid[i0 + ii] : 0.0;
  double acc[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) acc[q] = 0.0;
  for (int j0 = 0; j0 < c; j0 += kJ) {
    __syncthreads();
    for (int e = t; e < kJ * kI; e += 256) {
      const int jj = e / kI, iq = e % kI;
      const int j = j0 + jj;
      const double g = (i0 + iq < n) ? grid[i0 + iq] : 0.0;
      Cs[jj][iq] = (j < c) ? rbf(g - x[j], sigma2) : 0.0;
    }
    for (int e = t; e < kJ * kL; e += 256) {
      const int jj = e / kL, lq = e % kL;
      const int j = j0 + jj, l = l0 + lq;
      Ts[jj][lq] = (j < c && l < keff) ? T[(size_t)j * r + l] : 0.0;
    }
    __syncthreads();
    (void)gi;
#pragma unroll 4
    for (int jj = 0; jj < kJ; ++jj) {
      const double cv = Cs[jj][ii];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = fma(cv, Ts[jj][lg * 8 + q], acc[q]);
    }
  }
  if (i0 + ii < n) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int l = l0 + lg * 8 + q;
      if (l < keff) A[(size_t)l * n + i0 + ii] = acc[q];
    }
  }
}

// lower tiles of M = A^T A + cI on the k_eff block, identity padding; B = I
__global__ void lev_sketch_M_kernel(const double* __restrict__ A, int n, double cdiag,
                                    const int* __restrict__ meta, double* __restrict__ At,
                                    double* __restrict__ Bt) {
  const int keff = meta[0];
  const int ti = blockIdx.y, tj = blockIdx.z;
  if (tj > ti) return;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // blockIdx.x covers the 4096 entries of the tile, 8 per block (one per warp)
  const int e = blockIdx.x * 8 + w;
  const int rr = e >> 6, cc = e & 63;
  const int a = ti * kT + rr, b = tj * kT + cc;
  double v;
  if (a < keff && b < keff) {
    const double* pa = A + (size_t)a * n;
    const double* pb = A + (size_t)b * n;
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
    v = (a == b) ? s + cdiag : s;
  } else {
    v = (a == b) ? 1.0 : 0.0;
  }
  if (lane == 0) {
    At[tile_off(ti, tj) + sw(rr, cc)] = v;
    Bt[tile_off(ti, tj) + sw(rr, cc)] = (a == b) ? 1.0 : 0.0;
  }
}

// scores_i = sum_{l < k} (sum_{j <= l} X[l][j] A[j][i])^2, clipped at 1e-300.
// Block: 64 rows i x 4 interleaved l-sets; A rows staged in shared memory.
__global__ void __launch_bounds__(256)
    lev_sketch_scores_kernel(const double* __restrict__ A, int n, const double* __restrict__ Bt,
                             const int* __restrict__ meta, double* __restrict__ scores) {
  extern __shared__ __align__(16) double As[];     // [keff][64]
  __shared__ double red[4][64];
  const int keff = meta[0];
  const int i0 = blockIdx.x * 64;
  const int t = threadIdx.x, ii = t & 63, ls = t >> 6;
  for (int e = t; e < keff * 64; e += 256) {
    const int j = e >> 6, q = e & 63;
    As[e] = (i0 + q < n) ? A[(size_t)j * n + i0 + q] : 0.0;
  }
  __syncthreads();
  double s = 0.0;
  for (int l = ls; l < keff; l += 4) {
    const double* xl = Bt + tile_off(l / kT, 0);
    double y0 = 0.0, y1 = 0.0;
    int j = 0;
    for (; j + 1 <= l; j += 2) {
      y0 = fma(Bt[tile_off(l / kT, j / kT) + sw(l % kT, j % kT)], As[j * 64 + ii], y0);
      y1 = fma(Bt[tile_off(l / kT, (j + 1) / kT) + sw(l % kT, (j + 1) % kT)],
               As[(j + 1) * 64 + ii], y1);
    }
    if (j <= l) y0 = fma(Bt[tile_off(l / kT, j / kT) + sw(l % kT, j % kT)], As[j * 64 + ii], y0);
    (void)xl;
    const double y = y0 + y1;
    s = fma(y, y, s);
  }
  red[ls][ii] = s;
  __syncthreads();
  if (ls == 0 && i0 + ii < n) {
    const double v = ((red[0][ii] + red[1][ii]) + red[2][ii]) + red[3][ii];
    scores[i0 + ii] = v > 1e-300 ? v : 1e-300;
  }
}


// Large landmark sets (m > 512, e.g. the m = n full-feature comparator,
// baselines.py:170-194): Omega = K(L, L) compressed by the pivoted Cholesky
// above, Omega ~ G G^T, and the eigenpairs of G G^T taken from G^T G = U M U^T:
// V[:, k] = G u_k / sqrt(mu_k), W[:, k] = V[:, k] / sqrt(mu_k) = G u_k / mu_k.
__global__ void lev_vw_kernel(const double* __restrict__ G, int m, int r,
                              const double* __restrict__ U, const double* __restrict__ mu,
                              const int* __restrict__ m_eff, int ldv, double* __restrict__ V,
                              double* __restrict__ W) {
  const int k = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  double v = 0.0, w = 0.0;
  if (k < *m_eff) {
    double s0 = 0.0, s1 = 0.0;
    int a = 0;
    for (; a + 1 < r; a += 2) {
      s0 = fma(G[(size_t)a * m + i], U[(size_t)a * r + k], s0);
      s1 = fma(G[(size_t)(a + 1) * m + i], U[(size_t)(a + 1) * r + k], s1);
    }
    if (a < r) s0 = fma(G[(size_t)a * m + i], U[(size_t)a * r + k], s0);
    const double s = s0 + s1;
    v = s / sqrt(mu[k]);
    w = s / mu[k];
  }
  V[(size_t)i * ldv + k] = v;
  W[(size_t)i * ldv + k] = w;
}

struct SketchLayout {
  int r, ntk;
  size_t ntl;
  size_t off_H, off_mu, off_U, off_W, off_meta, off_eig, off_T, off_A, off_At, off_Bt, total;
  static SketchLayout make(int n, int c, int r) {
    SketchLayout L{};
    L.r = r;
    L.ntk = (r + kT - 1) / kT;
    L.ntl = (size_t)L.ntk * (L.ntk + 1) / 2;
    size_t o = 0;
    auto take = [&](size_t doubles) {
      size_t at = o;
      o += (doubles + 15) / 16 * 16;
      return at;
    };
    L.off_H = take((size_t)r * r);
    L.off_mu = take(r);
    L.off_U = take((size_t)r * r);
    L.off_W = take((size_t)r * r);
    L.off_meta = take(2);
    L.off_eig = take(nys_sym_eig_workspace_bytes(r) / sizeof(double) + 1);
    L.off_T = take((size_t)c * r);
    L.off_A = take((size_t)r * n);
    L.off_At = take(L.ntl * kTT);
    L.off_Bt = take(L.ntl * kTT);
    L.total = o * sizeof(double) + 256;
    return L;
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
  int launches = 0;
  lev_assemble_kernel<<<dim3(nt, nt), 256, 0, st>>>(grid, n, sigma2, c, At, Bt, info);
  ++launches;
  NYS_CHECK_LAUNCH();
  launches += tile_sweep(At, Bt, nt, info, st);
  NYS_CHECK_LAUNCH();
  lev_colnorm_kernel<<<dim3(nt, nt), 256, 0, st>>>(Bt, nt, part);
  lev_finalize_kernel<<<(n + 127) / 128, 128, 0, st>>>(part, n, nt, c, scores);
  launches += 2;
  nys_host::count_launches(launches);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" int nys_pchol_rbf_f64(const double* x, int c, double sigma2, double tol, int cap,
                                 double* G, int* out, void* stream) {
  if (c < 1 || c > 8192 || cap < 1 || !(sigma2 > 0.0) || !(tol >= 0.0)) return NYS_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int smem = 2 * c * (int)sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(lev_pchol_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return nys_host::record_cuda(e);
  lev_pchol_kernel<<<1, kPcThreads, smem, st>>>(x, c, sigma2, tol, cap, G, out);
  nys_host::count_launches(1);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" size_t nys_leverage_sketch_workspace_bytes(int n, int c, int r) {
  if (n < 1 || c < 1 || r < 1) return 0;
  return SketchLayout::make(n, c, r).total;
}

extern "C" int nys_leverage_sketch_f64(const double* grid, int n, const double* x, int c,
                                       double sigma2, double ridge, const double* G, int r,
                                       double* scores, int* info, void* ws, size_t ws_bytes,
                                       void* stream) {
  if (n < 1 || c < 1 || r < 1 || !(sigma2 > 0.0) || !(ridge >= 0.0)) return NYS_EINVAL;
  if (r > 256) return NYS_EUNSUPPORTED;
  const SketchLayout L = SketchLayout::make(n, c, r);
  if (ws == nullptr || ws_bytes < L.total) return NYS_EWORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* base = reinterpret_cast<double*>((reinterpret_cast<size_t>(ws) + 127) & ~(size_t)127);
  double* H = base + L.off_H;
  double* mu = base + L.off_mu;
  double* U = base + L.off_U;
  double* Wd = base + L.off_W;
  int* meta = reinterpret_cast<int*>(base + L.off_meta);   // k_eff, eig info
  double* T = base + L.off_T;
  double* A = base + L.off_A;
  double* At = base + L.off_At;
  double* Bt = base + L.off_Bt;
  int launches = 0;
  const int npairs = r * (r + 1) / 2;
  lev_gtg_kernel<<<(npairs + 7) / 8, 256, 0, st>>>(G, c, r, H);
  ++launches;
  NYS_CHECK_LAUNCH();
  // keep = vals > vals.max() * 1e-12 (nystrom.py:76): the eigensolver's drop rule
  int rc = nys_sym_eig_f64(H, r, 1e-12, mu, U, Wd, meta, meta + 1, base + L.off_eig,
                           nys_sym_eig_workspace_bytes(r), stream);
  if (rc != NYS_OK) return rc;
  lev_sketch_T_kernel<<<dim3((c + 127) / 128, r), 128, 0, st>>>(G, c, r, U, mu, meta, T);
  lev_sketch_A_kernel<<<dim3((n + 63) / 64, (r + 31) / 32), 256, 0, st>>>(grid, n, x, c, sigma2, T,
                                                                          r, meta, A);
  // n * ridge * np.eye(A.shape[1]) (nystrom.py:78)
  lev_sketch_M_kernel<<<dim3(kTT / 8, L.ntk, L.ntk), 256, 0, st>>>(A, n, (double)n * ridge, meta,
                                                                   At, Bt);
  launches += 3;
  NYS_CHECK_LAUNCH();
  cudaMemsetAsync(info, 0, sizeof(int), st);
  launches += tile_sweep(At, Bt, L.ntk, info, st);
  const int smem = r * 64 * (int)sizeof(double);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(lev_sketch_scores_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return nys_host::record_cuda(e);
  }
  lev_sketch_scores_kernel<<<(n + 63) / 64, 256, smem, st>>>(A, n, Bt, meta, scores);
  ++launches;
  nys_host::count_launches(launches);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" size_t nys_landmark_eig_compressed_workspace_bytes(int r) {
  if (r < 1) return 0;
  return (2 * (size_t)r * r + 16) * sizeof(double) + nys_sym_eig_workspace_bytes(r) + 256;
}

extern "C" int nys_landmark_eig_compressed_f64(const double* G, int m, int r, double drop_tol,
                                               double* eigvals, double* eigvecs, double* W,
                                               int ldv, int* m_eff, int* info, void* ws,
                                               size_t ws_bytes, void* stream) {
  if (m < 1 || r < 1 || ldv < r || !(drop_tol >= 0.0 && drop_tol < 1.0)) return NYS_EINVAL;
  if (r > 256) return NYS_EUNSUPPORTED;
  if (ws == nullptr || ws_bytes < nys_landmark_eig_compressed_workspace_bytes(r))
    return NYS_EWORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* base = reinterpret_cast<double*>((reinterpret_cast<size_t>(ws) + 127) & ~(size_t)127);
  double* H = base;
  double* U = H + (size_t)r * r;
  double* eig_ws = U + (size_t)r * r + 16;
  const int npairs = r * (r + 1) / 2;
  lev_gtg_kernel<<<(npairs + 7) / 8, 256, 0, st>>>(G, m, r, H);
  nys_host::count_launches(1);
  NYS_CHECK_LAUNCH();
  // eigenvalues (descending) and the drop rule s > max(drop_tol s_0, 0) of
  // nystrom.py:150-154; the r x r W of the small problem goes to H's storage
  int rc = nys_sym_eig_f64(H, r, drop_tol, eigvals, U, H, m_eff, info, eig_ws,
                           nys_sym_eig_workspace_bytes(r), stream);
  if (rc != NYS_OK) return rc;
  lev_vw_kernel<<<dim3((m + 127) / 128, ldv), 128, 0, st>>>(G, m, r, U, eigvals, m_eff, ldv,
                                                           eigvecs, W);
  nys_host::count_launches(1);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}
