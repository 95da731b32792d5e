// Landmark eigendecomposition, divide and conquer (the route of the
// reference's LAPACK dsyevd, nystrom.py:150): Householder tridiagonalisation,
// Cuppen tears at every multiple of kLeaf, leaves by implicit QL (one thread
// each, in parallel), then log2(m / kLeaf) merge levels, each a rank-one
// update diag(D) + rho z z^T solved by
//   * deflation of negligible z_i and of close pairs (Givens rotation),
//   * one thread per secular-equation root (two-pole rational iteration with
//     a bisection bracket, in the coordinates of the nearer pole so d_i - lambda_j
//     is formed without cancellation),
//   * Gu-Eisenstat recomputation of z (Loewner formula) so the eigenvectors are
//     orthogonal to working precision,
//   * one GEMM per block for the new eigenvectors,
// and finally the Householder back-transform.  Everything is parallel except
// the (short) leaf QL chains and the per-block deflation scan -- unlike QL on the
// full tridiagonal, whose ~m^2 dependent Givens rotations are FP64-latency bound
// on B200 (1.2 ms at m = 64, 31 ms at m = 256).
// Epilogue identical to eig.cu: descending order (ties: higher index first,
// nystrom.py:151), drop rule s > max(drop_tol s_0, 0), W = V / sqrt(s).
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace {

constexpr int kLeaf = 8;
constexpr int kDcMaxN = 256;
constexpr int kDcThreads = 1024;
constexpr int kMaxBlocks = kDcMaxN / kLeaf;
constexpr double kEps = 2.220446049250313e-16;

// leading dimension of A: ld = 4 (mod 16) doubles, so the matvec's 8 rows x 4
// column-lanes per warp hit 16 distinct bank pairs twice (2 wavefronts, the
// minimum for 256 bytes) instead of 4-way conflicts with ld = n + 1
__host__ __device__ inline int dc_ld(int n) { return n + (((4 - n) % 16) + 16) % 16; }

struct DcShared {
  double d[kDcMaxN], e[kDcMaxN], beta[kDcMaxN], hv[kDcMaxN], hp[kDcMaxN];
  double lam[kDcMaxN];    // eigenvalues aligned with the columns of Q
  double ds[kDcMaxN];     // per block: sorted (sign-adjusted) D, deflation-modified
  double zs[kDcMaxN];     // per block: sorted z (normalised), deflation-modified
  double zh[kDcMaxN];     // per block: Gu-Eisenstat z over the kept entries
  double rotc[kDcMaxN], rots[kDcMaxN];
  int perm[kDcMaxN];      // per block: sorted index -> global column
  int keep[kDcMaxN];      // per block: kept sorted indices (ascending), then deflated
  int roti[kDcMaxN], rotj[kDcMaxN];
  int col[kDcMaxN];       // per block: Q column of kept / deflated entry c
  double rho[kMaxBlocks], sgn[kMaxBlocks];
  int K[kMaxBlocks], nrot[kMaxBlocks];
  int bs[kMaxBlocks], bmid[kMaxBlocks], be[kMaxBlocks];   // merge: start, boundary, end
  double red[kDcThreads / 32];
  int degenerate;
};


// implicit QL on the leaf [s, s+len) of (d, e), eigenvectors into Q block.
// One warp per leaf: every lane runs the (short) scalar recurrence redundantly
// -- identical values, so the shared d/e writes agree -- and lane k < len
// applies each Givens rotation to row k of the leaf's Z, so no rotation waits
// for a serial len-long row loop.  The arithmetic is the serial version's, op
// for op (results unchanged bit for bit).
NYS_DEV void leaf_ql(DcShared& S, double* Q, int n, int s, int len, int lane) {
  double* d = S.d + s;
  double* e = S.e + s;   // e[i] couples i, i+1 inside the leaf; e[len-1] is unused
  const double ehold = len > 0 ? e[len - 1] : 0.0;
  __syncwarp();
  if (len > 0) e[len - 1] = 0.0;
  double* row = lane < len ? Q + (size_t)(s + lane) * n + s : nullptr;
  if (row)
    for (int c = 0; c < len; ++c) row[c] = (lane == c) ? 1.0 : 0.0;
  for (int l = 0; l < len; ++l) {
    for (int iter = 0; iter < 60; ++iter) {
      int mm = l;
      for (; mm < len - 1; ++mm) {
        const double dd = fabs(d[mm]) + fabs(d[mm + 1]);
        if (fabs(e[mm]) <= kEps * dd) break;
      }
      if (mm == l) break;
      double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
      double r = hypot(g, 1.0);
      g = d[mm] - d[l] + e[l] / (g + copysign(r, g));
      double sn = 1.0, cs = 1.0, p = 0.0;
      bool early = false;
      for (int i = mm - 1; i >= l; --i) {
        const double f = sn * e[i], b = cs * e[i];
        r = hypot(f, g);
        e[i + 1] = r;
        if (r == 0.0) {
          d[i + 1] -= p;
          e[mm] = 0.0;
          early = true;
          break;
        }
        sn = f / r;
        cs = g / r;
        g = d[i + 1] - p;
        r = (d[i] - g) * sn + 2.0 * cs * b;
        p = sn * r;
        d[i + 1] = g + p;
        g = cs * r - b;
        if (row) {   // columns i, i+1 of the leaf's Z, this lane's row
          const double zf = row[i + 1], zi = row[i];
          row[i + 1] = sn * zi + cs * zf;
          row[i] = cs * zi - sn * zf;
        }
      }
      if (early) continue;
      d[l] -= p;
      e[l] = g;
      e[mm] = 0.0;
    }
  }
  __syncwarp();
  if (len > 0) e[len - 1] = ehold;
  if (lane < len) S.lam[s + lane] = d[lane];
}

// secular root j of diag(ds) + rho zz^T over the K kept entries of a block;
// writes DL[i][j] = d_i - lambda_j (i < K) and returns lambda_j
// G adjacent lanes (mask gm, lane index gl within the group) share one root:
// every sum over the K poles is split G ways and butterfly-reduced, the model
// step is computed redundantly (identical in all G lanes)
NYS_DEV double gsum(double v, int G, unsigned gm) {
  for (int o = 1; o < G; o <<= 1) v += __shfl_xor_sync(gm, v, o);
  return v;
}

NYS_DEV double secular_root(const DcShared& S, int s, int j, int K, double rho, double* DL,
                            int n, int gl, int G, unsigned gm) {
  const int* kp = S.keep + s;
  auto dk = [&](int i) { return S.ds[s + kp[i]]; };
  auto z2 = [&](int i) {
    const double z = S.zs[s + kp[i]];
    return z * z;
  };
  int org;
  double lo, hi;
  if (j < K - 1) {
    const double mid = 0.5 * (dk(j) + dk(j + 1));
    double f = 0.0;
    for (int i = gl; i < K; i += G) f += z2(i) / (dk(i) - mid);
    f = 1.0 / rho + gsum(f, G, gm);
    org = f >= 0.0 ? j : j + 1;
    lo = dk(j) - dk(org);
    hi = dk(j + 1) - dk(org);
  } else {
    org = K - 1;
    double zz = 0.0;
    for (int i = gl; i < K; i += G) zz += z2(i);
    zz = gsum(zz, G, gm);
    lo = 0.0;
    hi = rho * zz;
  }
  const double dorg = dk(org);
  double tau = 0.5 * (lo + hi);
  for (int it = 0; it < 80; ++it) {
    double f = 0.0, fabs_sum = 0.0, psi = 0.0, dpsi = 0.0, phi = 0.0, dphi = 0.0;
    for (int i = gl; i < K; i += G) {
      const double dl = (dk(i) - dorg) - tau;
      const double w = 1.0 / dl;
      const double t = z2(i) * w;
      f += t;
      fabs_sum += fabs(t);
      if (j == K - 1 || i <= j) {
        psi += t;
        dpsi += t * w;
      } else {
        phi += t;
        dphi += t * w;
      }
    }
    f = 1.0 / rho + gsum(f, G, gm);
    fabs_sum = 1.0 / rho + gsum(fabs_sum, G, gm);
    psi = gsum(psi, G, gm);
    dpsi = gsum(dpsi, G, gm);
    phi = gsum(phi, G, gm);
    dphi = gsum(dphi, G, gm);
    if (f > 0.0)
      hi = tau;
    else
      lo = tau;
    if (fabs(f) <= 8.0 * kEps * fabs_sum ||
        (hi - lo) <= 2.0 * kEps * fmax(fmax(fabs(lo), fabs(hi)), 1e-300))
      break;
    // two-pole rational model c + s/(dj - x) + S/(dj1 - x) (fixed weight)
    const double dj = (dk(j) - dorg) - tau;
    double x;
    bool ok = false;
    if (j < K - 1) {
      const double dj1 = (dk(j + 1) - dorg) - tau;
      const double sw = dj * dj * dpsi, Sw = dj1 * dj1 * dphi;
      const double c = 1.0 / rho + psi - dj * dpsi + phi - dj1 * dphi;
      const double A = c, B = -(c * (dj + dj1) + sw + Sw), C = c * dj * dj1 + sw * dj1 + Sw * dj;
      if (A != 0.0) {
        const double disc = fmax(B * B - 4.0 * A * C, 0.0);
        const double q = -0.5 * (B + copysign(sqrt(disc), B));
        const double r1 = q / A, r2 = q != 0.0 ? C / q : r1;
        if (r1 > lo - tau && r1 < hi - tau) {
          x = r1;
          ok = true;
        } else if (r2 > lo - tau && r2 < hi - tau) {
          x = r2;
          ok = true;
        }
      } else if (B != 0.0) {
        x = -C / B;
        ok = x > lo - tau && x < hi - tau;
      }
    } else {
      const double sw = dj * dj * dpsi;
      const double c = 1.0 / rho + psi - dj * dpsi;
      if (c != 0.0) {
        x = dj + sw / c;
        ok = x > lo - tau && x < hi - tau;
      }
    }
    const double nt = ok ? tau + x : 0.5 * (lo + hi);
    tau = (nt > lo && nt < hi) ? nt : 0.5 * (lo + hi);
  }
  for (int i = gl; i < K; i += G) DL[(size_t)(s + i) * n + s + j] = (dk(i) - dorg) - tau;
  return dorg + tau;
}

// Blocked Householder tridiagonalisation (LAPACK dsytrd / dlatrd order) for the
// global-memory path (n > 64).  Within a panel of kTNb columns the trailing
// matrix is not touched: each column is corrected on the fly by the panel's
// V W^T + W V^T, the matvec p = A v reads the panel-start matrix once (L2), and
// the panel's rank-2 kTNb update of the trailing block runs as DMMA.8x8x4 GEMM
// tiles at the end.  The unblocked loop re-read and re-wrote the whole trailing
// matrix per reflector.  Same reflectors (alpha, beta, v) as the unblocked
// form, stored the same way (v below the diagonal of A, beta, e, d in S).
constexpr int kTNb = 32;
NYS_DEV double dc_block_sum_all(double x, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  __syncthreads();
  if (lane == 0) red[w] = x;
  __syncthreads();
  double r = 0.0;
  for (int i = 0; i < nw; ++i) r += red[i];
  return r;
}

template <typename SharedT>
NYS_DEV void tridiag_blocked(double* __restrict__ A, int ld, int n, SharedT& S, double* dynsm,
                             int debug) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  constexpr int kLdv = kTNb + 1;      // padded rows: column reads across rows hit
  double* V = dynsm;                  // distinct banks (stride 32 would serialise)
  double* Wm = V + (size_t)n * kLdv;  // n x kLdv
  double* t1 = Wm + (size_t)n * kLdv; // kTNb
  double* t2 = t1 + kTNb;             // kTNb
  double* pacc = t2 + kTNb;           // (nt / 256) x 256 matvec partials
  long long tp = 0, tu = 0, ts[6] = {0, 0, 0, 0, 0, 0};
  for (int k0 = 0; k0 + 2 < n; k0 += kTNb) {
    const int nb = min(kTNb, n - 2 - k0);
    for (int e = tid; e < n * kLdv; e += nt) {
      V[e] = 0.0;
      Wm[e] = 0.0;
    }
    __syncthreads();
    long long ta = clock64();
    for (int jj = 0; jj < nb; ++jj) {
      const int j = k0 + jj;
      long long c0k = clock64();
      // (1) corrected column j, rows i >= j
      for (int i = j + tid; i < n; i += nt) {
        double c = A[(size_t)i * ld + j];
        const double* Vi = V + (size_t)i * kLdv;
        const double* Wi = Wm + (size_t)i * kLdv;
        const double* Vj = V + (size_t)j * kLdv;
        const double* Wj = Wm + (size_t)j * kLdv;
        for (int q = 0; q < jj; ++q) c = c - Vi[q] * Wj[q] - Wi[q] * Vj[q];
        S.hv[i] = c;
      }
      __syncthreads();
      long long c1k = clock64();
      ts[0] += c1k - c0k;
      // (2) reflector of x = c[j+1:]
      double tail = 0.0;
      for (int i = j + 2 + tid; i < n; i += nt) tail = fma(S.hv[i], S.hv[i], tail);
      tail = dc_block_sum_all(tail, S.red);
      if (tid == 0) {
        S.d[j] = S.hv[j];
        const double x0 = S.hv[j + 1];
        double beta = 0.0, alpha = x0;
        if (tail > 0.0) {
          const double nx = sqrt(fma(x0, x0, tail));
          alpha = -copysign(nx, x0);
          const double v0 = x0 - alpha;
          beta = 2.0 / fma(v0, v0, tail);
          S.hv[j + 1] = v0;
        }
        S.e[j] = alpha;
        S.beta[j] = beta;
      }
      __syncthreads();
      long long c2k = clock64();
      ts[1] += c2k - c1k;
      const double beta = S.beta[j];
      if (beta == 0.0) continue;   // identity reflector: V, W columns stay zero
      for (int i = j + 1 + tid; i < n; i += nt) {
        const double v = S.hv[i];
        A[(size_t)i * ld + j] = v;   // Householder vector for the back-transform
        V[(size_t)i * kLdv + jj] = v;
      }
      // (3) p = A v over rows i > j (panel-start matrix).  A is symmetric, so
      // p_i = sum_c A[c][i] v_c: a warp reads 32 consecutive doubles of row c
      // (one 256-byte line) and each thread owns one p_i; the c range is split
      // over nt / 256 groups whose partial sums meet in shared memory.
      {
        const int ng = nt >> 8, g = tid >> 8, ii = tid & 255;
        const int i = j + 1 + ii;
        const int len = n - j - 1;
        const int chunk = (len + ng - 1) / ng;
        const int cb = j + 1 + g * chunk, ce = min(n, cb + chunk);
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        if (i < n) {
          int c = cb;
          for (; c + 7 < ce; c += 8) {   // eight L2 loads in flight per thread
            double x[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) x[t] = A[(size_t)(c + t) * ld + i];
            a0 = fma(x[0], S.hv[c], a0);
            a1 = fma(x[1], S.hv[c + 1], a1);
            a2 = fma(x[2], S.hv[c + 2], a2);
            a3 = fma(x[3], S.hv[c + 3], a3);
            a0 = fma(x[4], S.hv[c + 4], a0);
            a1 = fma(x[5], S.hv[c + 5], a1);
            a2 = fma(x[6], S.hv[c + 6], a2);
            a3 = fma(x[7], S.hv[c + 7], a3);
          }
          for (; c < ce; ++c) a0 = fma(A[(size_t)c * ld + i], S.hv[c], a0);
        }
        pacc[g * 256 + ii] = (a0 + a1) + (a2 + a3);
        __syncthreads();
        if (g == 0 && i < n) {
          double s2 = 0.0;
          for (int q = 0; q < ng; ++q) s2 += pacc[q * 256 + ii];
          S.hp[i] = s2;
        }
      }
      long long c3k = clock64();
      ts[2] += c3k - c2k;
      // (4) t1 = W^T v, t2 = V^T v (warp q for column q < jj)
      for (int q = warp; q < jj; q += nw) {
        double a1 = 0.0, a2 = 0.0;
        for (int i = j + 1 + lane; i < n; i += 32) {
          const double v = S.hv[i];
          a1 = fma(Wm[(size_t)i * kLdv + q], v, a1);
          a2 = fma(V[(size_t)i * kLdv + q], v, a2);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          a1 += __shfl_xor_sync(0xffffffffu, a1, o);
          a2 += __shfl_xor_sync(0xffffffffu, a2, o);
        }
        if (lane == 0) {
          t1[q] = a1;
          t2[q] = a2;
        }
      }
      __syncthreads();
      long long c4k = clock64();
      ts[3] += c4k - c3k;
      // (5) p <- beta (A v - V t1 - W t2);  w = p - (beta/2)(v.p) v
      double vp = 0.0;
      for (int i = j + 1 + tid; i < n; i += nt) {
        double pi = S.hp[i];
        const double* Vi = V + (size_t)i * kLdv;
        const double* Wi = Wm + (size_t)i * kLdv;
        for (int q = 0; q < jj; ++q) pi = pi - Vi[q] * t1[q] - Wi[q] * t2[q];
        pi *= beta;
        S.hp[i] = pi;
        vp = fma(S.hv[i], pi, vp);
      }
      vp = dc_block_sum_all(vp, S.red);
      const double Kc = 0.5 * beta * vp;
      for (int i = j + 1 + tid; i < n; i += nt)
        Wm[(size_t)i * kLdv + jj] = S.hp[i] - Kc * S.hv[i];
      __syncthreads();
      ts[4] += clock64() - c4k;
    }
    long long tb = clock64();
    tp += tb - ta;
    // trailing update A[r][c] -= (V W^T + W V^T)[r][c], r, c >= k0 + nb
    {
      const int t0 = k0 + nb, nn = n - t0;
      const int fr = lane >> 2, fc = lane & 3;
      const int trows = (nn + 15) / 16, tcols = (nn + 31) / 32;
      for (int tt = warp; tt < trows * tcols; tt += nw) {
        const int r0 = t0 + (tt / tcols) * 16, c0 = t0 + (tt % tcols) * 32;
        double acc[2][4][2];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int jb = 0; jb < 4; ++jb) {
            const int r = r0 + 8 * i + fr;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int c = c0 + 8 * jb + 2 * fc + h;
              acc[i][jb][h] = (r < n && c < n) ? A[(size_t)r * ld + c] : 0.0;
            }
          }
        for (int k4 = 0; k4 < 2 * kTNb; k4 += 4) {
          const int kq = k4 + fc;   // 0..2kTNb: [V | W] against [W | V]
          double a[2], bq[4];
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int r = r0 + 8 * i + fr;
            a[i] = r < n ? -(kq < kTNb ? V[(size_t)r * kLdv + kq] : Wm[(size_t)r * kLdv + kq - kTNb])
                         : 0.0;
          }
#pragma unroll
          for (int jb = 0; jb < 4; ++jb) {
            const int c = c0 + 8 * jb + fr;
            bq[jb] = c < n ? (kq < kTNb ? Wm[(size_t)c * kLdv + kq] : V[(size_t)c * kLdv + kq - kTNb])
                           : 0.0;
          }
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int jb = 0; jb < 4; ++jb) nys::dmma(acc[i][jb][0], acc[i][jb][1], a[i], bq[jb]);
        }
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int jb = 0; jb < 4; ++jb) {
            const int r = r0 + 8 * i + fr;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int c = c0 + 8 * jb + 2 * fc + h;
              if (r < n && c < n) A[(size_t)r * ld + c] = acc[i][jb][h];
            }
          }
      }
    }
    __syncthreads();
    tu += clock64() - tb;
  }
  if (debug && tid == 0)
    printf("[nys dc] blocked tridiag: panels %lld (col %lld refl %lld matvec %lld t12 %lld w %lld) trailing %lld\n",
           tp, ts[0], ts[1], ts[2], ts[3], ts[4], tu);
}

// kSmem: the working matrices live in dynamic shared memory (n <= 64) -- a
// compile-time address space, so the compiler emits LDS/STS; kT: columns per
// lane in the rank-2 update (ceil(n / 32) bound)
template <bool kSmem, int kT>
__global__ void __launch_bounds__(kT <= 2 ? 256 : kDcThreads, 1)
    dc_eig_kernel(const double* __restrict__ lm, const double* __restrict__ Ain, int n,
                  double sigma2, double drop_tol,
                  double* __restrict__ eigvals, double* __restrict__ eigvecs,
                  double* __restrict__ Wout, int* __restrict__ m_eff_out, int* __restrict__ info,
                  double* __restrict__ gbuf, int use_smem, int debug) {
  extern __shared__ __align__(16) double dyn[];
  __shared__ DcShared S;
  const int ld = dc_ld(n);
  (void)use_smem;
  double* base = kSmem ? dyn : gbuf;
  double* A = base;                           // n x ld (Householder vectors below diagonal)
  double* Q = A + (size_t)n * ld;             // n x n
  double* Qn = Q + (size_t)n * n;             // n x n
  double* DL = Qn + (size_t)n * n;            // n x n
  const int tid = threadIdx.x, nt = blockDim.x;
  long long tc0 = clock64(), tc1 = 0, tc2 = 0, tc3 = 0, tc4 = 0;

  if (tid == 0) S.degenerate = 0;
  __syncthreads();
  for (int e = tid; e < n * n; e += nt) {
    const int i = e / n, j = e % n;
    if (Ain != nullptr) {          // explicit symmetric input (nys_sym_eig_f64)
      A[(size_t)i * ld + j] = Ain[e];
      continue;
    }
    const double d = lm[i] - lm[j];
    A[(size_t)i * ld + j] = nys::rbf(d, sigma2);
    if (i != j && fabs(d) <= 1e-12) S.degenerate = 1;
  }
  __syncthreads();
  if (S.degenerate) {
    if (tid == 0) {
      *info = NYS_INFO_DEGENERATE;
      *m_eff_out = 0;
      if (!kSmem)   // the split epilogue reads the verdict from the buffer tail
        reinterpret_cast<int*>(gbuf + (size_t)n * ld + 3 * (size_t)n * n + 2 * n)[1] = 1;
    }
    return;
  }

  // ---------------- Householder tridiagonalisation (as eig.cu phase 1)
  // Three barriers per reflector: warp 0 forms the reflector (norm by warp
  // shuffles), the matvec splits every row over tpr lanes, and each warp
  // recomputes v.p itself so the rank-2 update needs no extra barrier.
  long long tq[4] = {0, 0, 0, 0};
  const long long tsetup = clock64() - tc0;
  if constexpr (!kSmem) {
    tridiag_blocked(A, ld, n, S, dyn, debug);
  } else {
    const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
    for (int k = 0; k + 2 < n; ++k) {
      const int i0 = k + 1;
      long long tt = clock64();
      if (warp == 0) {
        double tail = 0.0;
        for (int i = i0 + 1 + lane; i < n; i += 32) {
          const double x = A[(size_t)i * ld + k];
          S.hv[i] = x;
          tail = fma(x, x, tail);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) tail += __shfl_xor_sync(0xffffffffu, tail, o);
        if (lane == 0) {
          const double x0 = A[(size_t)i0 * ld + k];
          double beta = 0.0, alpha = x0;
          S.hv[i0] = x0;
          if (tail > 0.0) {
            const double nx = sqrt(fma(x0, x0, tail));
            alpha = -copysign(nx, x0);
            const double v0 = x0 - alpha;
            beta = 2.0 / fma(v0, v0, tail);
            S.hv[i0] = v0;
            A[(size_t)i0 * ld + k] = v0;
          }
          S.e[k] = alpha;
          S.beta[k] = beta;
        }
      }
      __syncthreads();
      if (debug) { long long t2 = clock64(); tq[0] += t2 - tt; tt = t2; }
      const double beta = S.beta[k];
      if (beta == 0.0) continue;
      const int len = n - i0;
      const int tpr = (nt >= 8 * len) ? 8 : (nt >= 4 * len) ? 4 : (nt >= 2 * len) ? 2 : 1;
      const int rows_per_pass = nt / tpr;
      const int npass = (len + rows_per_pass - 1) / rows_per_pass;
      for (int ps = 0; ps < npass; ++ps) {   // whole passes: the shuffles need full warps
        const int r = ps * rows_per_pass + tid / tpr, sub = tid % tpr;
        const int i = i0 + r;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        if (r < len) {
          const double* __restrict__ row = A + (size_t)i * ld;
          const double* __restrict__ hv = S.hv;
          int j = i0 + sub;
          for (; j + 3 * tpr < n; j += 4 * tpr) {   // four independent loads per trip
            a0 = fma(row[j], hv[j], a0);
            a1 = fma(row[j + tpr], hv[j + tpr], a1);
            a2 = fma(row[j + 2 * tpr], hv[j + 2 * tpr], a2);
            a3 = fma(row[j + 3 * tpr], hv[j + 3 * tpr], a3);
          }
          for (; j < n; j += tpr) a0 = fma(row[j], hv[j], a0);
        }
        double acc = (a0 + a1) + (a2 + a3);
        for (int o = 1; o < tpr; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (sub == 0 && r < len) S.hp[i] = beta * acc;
      }
      __syncthreads();
      if (debug) { long long t2 = clock64(); tq[1] += t2 - tt; tt = t2; }
      double vp = 0.0;
      for (int i = i0 + lane; i < n; i += 32) vp = fma(S.hv[i], S.hp[i], vp);
#pragma unroll
      for (int o = 16; o; o >>= 1) vp += __shfl_xor_sync(0xffffffffu, vp, o);
      const double Kc = 0.5 * beta * vp;
      // this lane's columns j = i0 + lane + 32 t: v_j and w_j in registers; rows
      // in groups of kG whose loads are all issued before any store (the
      // compiler cannot prove different rows do not alias)
      double hvj[kT], wj[kT];
#pragma unroll
      for (int t = 0; t < kT; ++t) {
        const int j = i0 + lane + 32 * t;
        hvj[t] = j < n ? S.hv[j] : 0.0;
        wj[t] = j < n ? S.hp[j] - Kc * S.hv[j] : 0.0;
      }
      constexpr int kG = kT <= 2 ? 4 : 1;
      for (int ib = i0 + warp; ib < n; ib += nw * kG) {
        double val[kG][kT];
#pragma unroll
        for (int g = 0; g < kG; ++g) {
          const int i = ib + g * nw;
#pragma unroll
          for (int t = 0; t < kT; ++t) {
            const int j = i0 + lane + 32 * t;
            val[g][t] = (i < n && j < n) ? A[(size_t)i * ld + j] : 0.0;
          }
        }
#pragma unroll
        for (int g = 0; g < kG; ++g) {
          const int i = ib + g * nw;
          if (i >= n) break;
          const double vi = S.hv[i], wi = S.hp[i] - Kc * vi;
#pragma unroll
          for (int t = 0; t < kT; ++t) {
            const int j = i0 + lane + 32 * t;
            if (j < n) A[(size_t)i * ld + j] = val[g][t] - vi * wj[t] - wi * hvj[t];
          }
        }
      }
      __syncthreads();
      if (debug) { long long t2 = clock64(); tq[2] += t2 - tt; tt = t2; }
    }
  }
  if (debug && tid == 0) printf("[nys dc] tridiag phases: setup %lld reflector %lld matvec %lld update %lld\n", tsetup, tq[0], tq[1], tq[2]);
  if constexpr (kSmem) {
    for (int i = tid; i < n; i += nt) S.d[i] = A[(size_t)i * ld + i];
  } else {   // tridiag_blocked set d[0..n-3] from the corrected panel columns
    for (int i = max(n - 2, 0) + tid; i < n; i += nt) S.d[i] = A[(size_t)i * ld + i];
  }
  if (tid == 0) {
    if (n >= 2) S.e[n - 2] = A[(size_t)(n - 1) * ld + (n - 2)];
    S.e[n - 1] = 0.0;
  }
  __syncthreads();

  tc1 = clock64();
  // ---------------- tears at every multiple of kLeaf, then leaves by QL
  if (tid == 0)
    for (int b = kLeaf; b < n; b += kLeaf) {
      const double rho = S.e[b - 1];
      S.d[b - 1] -= rho;
      S.d[b] -= rho;
    }
  for (int e = tid; e < n * n; e += nt) Q[e] = 0.0;
  __syncthreads();
  const int nleaf = (n + kLeaf - 1) / kLeaf;
  for (int t = tid >> 5; t < nleaf; t += nt >> 5) {   // one warp per leaf
    const int s = t * kLeaf, len = min(kLeaf, n - s);
    leaf_ql(S, Q, n, s, len, tid & 31);
  }
  __syncthreads();

  tc2 = clock64();
  // ---------------- merge levels
  long long tm[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tlast = clock64();
  for (int width = kLeaf; width < n; width *= 2) {
    const int nmerge = (n + 2 * width - 1) / (2 * width);
    // block geometry; a block without a right partner is carried unchanged
    for (int b = tid; b < nmerge; b += nt) {
      const int s = b * 2 * width;
      S.bs[b] = s;
      S.bmid[b] = min(s + width, n);
      S.be[b] = min(s + 2 * width, n);
      const double rho = S.bmid[b] < S.be[b] ? S.e[S.bmid[b] - 1] : 0.0;
      S.sgn[b] = rho < 0.0 ? -1.0 : 1.0;
    }
    __syncthreads();
    // the next Q is block diagonal: clear it so the off-diagonal child blocks
    // that the GEMM of the next level reads are exact zeros
    for (int e = tid; e < n * n; e += nt) Qn[e] = 0.0;
    if (debug) { long long tn = clock64(); tm[0] += tn - tlast; tlast = tn; }
    // M1: rank-sort the (sign-adjusted) eigenvalues of both children, gather z
    for (int b = 0; b < nmerge; ++b) {
      const int s = S.bs[b], mid = S.bmid[b], end = S.be[b], N = end - s;
      if (mid >= end) continue;
      const double sg = S.sgn[b];
      for (int c = tid; c < N; c += nt) {
        const double lc = sg * S.lam[s + c];
        int rank = 0;
        for (int c2 = 0; c2 < N; ++c2) {
          const double l2 = sg * S.lam[s + c2];
          rank += (l2 < lc) || (l2 == lc && c2 < c);
        }
        S.perm[s + rank] = s + c;
        S.ds[s + rank] = lc;
        S.zs[s + rank] = (s + c < mid) ? Q[(size_t)(mid - 1) * n + s + c] : Q[(size_t)mid * n + s + c];
      }
    }
    __syncthreads();
    if (debug) { long long tn = clock64(); tm[1] += tn - tlast; tlast = tn; }
    // M2: normalise, deflate (the serial dlaed2-style scan's decisions).
    // One warp per block: the norms and the type-1 tests (|rho z_i| <= tol) are
    // lane-parallel, the close-pair Givens test is evaluated speculatively for
    // every pair of consecutive surviving entries with their original values, and
    // lane 0 walks the entries in order, recomputing a pair only when its left
    // entry was itself just rotated (the sequential dependence of dlaed2).
    for (int b = (tid >> 5); b < nmerge; b += (nt >> 5)) {
      const int lane = tid & 31;
      const int s = S.bs[b], mid = S.bmid[b], end = S.be[b], N = end - s;
      if (mid >= end) continue;
      // ||z||^2 in index order by one lane (the serial scan's rounding, so the
      // one-CTA eigensolver's results are unchanged), max |d| by the warp
      double zn2 = 0.0, dmax = 0.0;
      if (lane == 0)
        for (int i = 0; i < N; ++i) zn2 += S.zs[s + i] * S.zs[s + i];
      zn2 = __shfl_sync(0xffffffffu, zn2, 0);
      for (int i = lane; i < N; i += 32) dmax = fmax(dmax, fabs(S.ds[s + i]));
#pragma unroll
      for (int o = 16; o; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
      const double rho = fabs(S.e[mid - 1]) * zn2;
      const double inv = zn2 > 0.0 ? 1.0 / sqrt(zn2) : 0.0;
      const double tol = 8.0 * kEps * fmax(dmax, rho);
      int* keep = S.keep + s;
      int* srot = S.col + s;                       // scratch: speculative verdicts
      double *sc = S.hv + s, *ssn = S.hp + s, *sr = S.zh + s;
      // surviving (not type-1) entries as a bit mask, 8 words for N <= 256
      unsigned surv[kDcMaxN / 32];
#pragma unroll
      for (int wd = 0; wd < kDcMaxN / 32; ++wd) {
        const int i = 32 * wd + lane;
        bool sv = false;
        if (i < N) {
          const double z = S.zs[s + i] * inv;
          S.zs[s + i] = z;
          sv = !(fabs(rho * z) <= tol);
        }
        surv[wd] = __ballot_sync(0xffffffffu, sv);
      }
      __syncwarp();
      if (!(rho <= tol)) {
        for (int i = lane; i < N; i += 32) {
          srot[i] = 0;
          if (!((surv[i >> 5] >> (i & 31)) & 1u)) continue;
          int p = -1;   // previous surviving entry
          for (int wd = i >> 5; wd >= 0 && p < 0; --wd) {
            unsigned m = surv[wd];
            if (wd == (i >> 5)) m &= (i & 31) ? (0xffffffffu >> (32 - (i & 31))) : 0u;
            if (m) p = 32 * wd + 31 - __clz(m);
          }
          if (p < 0) continue;
          const double zi = S.zs[s + i], zp = S.zs[s + p];
          const double r = hypot(zi, zp);
          const double c = zi / r, sn = -zp / r;
          const double t = S.ds[s + i] - S.ds[s + p];
          srot[i] = fabs(t * c * sn) <= tol ? 1 : 0;
          sc[i] = c;
          ssn[i] = sn;
          sr[i] = r;
        }
      }
      __syncwarp();
      if (lane == 0) {
        S.rho[b] = rho;
        int K = 0, nd = 0, nrot = 0, prev = -1;
        bool prev_mod = false;
        if (rho <= tol) {
          for (int i = 0; i < N; ++i) keep[N - 1 - i] = i;
        } else {
          for (int i = 0; i < N; ++i) {
            if (!((surv[i >> 5] >> (i & 31)) & 1u)) {
              keep[N - 1 - nd++] = i;
              continue;
            }
            bool mod = false;
            if (prev >= 0) {
              double c, sn, r;
              bool rot;
              if (!prev_mod) {
                rot = srot[i] != 0;
                c = sc[i];
                sn = ssn[i];
                r = sr[i];
              } else {
                const double zi = S.zs[s + i], zp = S.zs[s + prev];
                r = hypot(zi, zp);
                c = zi / r;
                sn = -zp / r;
                const double t = S.ds[s + i] - S.ds[s + prev];
                rot = fabs(t * c * sn) <= tol;
              }
              if (rot) {
                const double dp = S.ds[s + prev] * c * c + S.ds[s + i] * sn * sn;
                const double di = S.ds[s + prev] * sn * sn + S.ds[s + i] * c * c;
                S.ds[s + prev] = dp;
                S.ds[s + i] = di;
                S.zs[s + i] = r;
                S.zs[s + prev] = 0.0;
                S.roti[s + nrot] = prev;
                S.rotj[s + nrot] = i;
                S.rotc[s + nrot] = c;
                S.rots[s + nrot] = sn;
                ++nrot;
                --K;
                keep[N - 1 - nd++] = prev;
                mod = true;
              }
            }
            keep[K++] = i;
            prev = i;
            prev_mod = mod;
          }
        }
        S.K[b] = K;
        S.nrot[b] = nrot;
      }
      __syncwarp();
    }
    __syncthreads();
    if (debug) { long long tn = clock64(); tm[2] += tn - tlast; tlast = tn; }
    // M3: secular roots, one thread per (block, root)
    {
      int total = 0;
      for (int b = 0; b < nmerge; ++b) total += (S.bmid[b] < S.be[b]) ? S.K[b] : 0;
      constexpr int G = 4;
      const int gl = tid % G;
      const unsigned gm = 0xFu << ((tid & 31) & ~(G - 1));
      for (int w = tid / G; w < total; w += nt / G) {
        int b = 0, j = w;
        while (j >= ((S.bmid[b] < S.be[b]) ? S.K[b] : 0)) {
          j -= (S.bmid[b] < S.be[b]) ? S.K[b] : 0;
          ++b;
        }
        const int s = S.bs[b];
        const double lj = secular_root(S, s, j, S.K[b], S.rho[b], DL, n, gl, G, gm);
        if (gl == 0) S.zh[s + j] = lj;   // park lambda_j (zh is rebuilt in M4 from DL)
      }
    }
    __syncthreads();
    if (debug) { long long tn = clock64(); tm[3] += tn - tlast; tlast = tn; }
    // M4: Gu-Eisenstat z over kept entries; lambda moves to lam after M6
    for (int b = 0; b < nmerge; ++b) {
      const int s = S.bs[b], mid = S.bmid[b], end = S.be[b];
      if (mid >= end) continue;
      const int K = S.K[b];
      const double rho = S.rho[b];
      // four lanes per entry, each a strided partial product (the ratios are
      // independent; only the running products are dependency chains)
      constexpr int G = 4;
      const int gl = tid % G;
      const unsigned gm = 0xFu << ((tid & 31) & ~(G - 1));
      const int Kr = (K + G - 1) / G * G;   // whole groups
      for (int w = tid / G; w < Kr; w += nt / G) {
        const int i = w < K ? w : K - 1;
        const double di = S.ds[s + S.keep[s + i]];
        double v0 = gl == 0 ? -DL[(size_t)(s + i) * n + s + K - 1] / rho : 1.0, v1 = 1.0;
        int t = 0;
        for (int jj = gl; jj < K - 1; jj += G, ++t) {
          const double dj = jj < i ? S.ds[s + S.keep[s + jj]] : S.ds[s + S.keep[s + jj + 1]];
          const double ratio = (-DL[(size_t)(s + i) * n + s + jj]) / (dj - di);
          if (t & 1)
            v1 *= ratio;
          else
            v0 *= ratio;
        }
        double vv = v0 * v1;
        for (int o = 1; o < G; o <<= 1) vv *= __shfl_xor_sync(gm, vv, o);
        if (gl == 0 && w < K) S.hv[s + i] = copysign(sqrt(fmax(vv, 0.0)), S.zs[s + S.keep[s + i]]);
      }
    }
    __syncthreads();
    if (debug) { long long tn = clock64(); tm[4] += tn - tlast; tlast = tn; }
    // M5: U[i][j] = zhat_i / (d_i - lambda_j), then unit columns
    for (int b = 0; b < nmerge; ++b) {
      const int s = S.bs[b], mid = S.bmid[b], end = S.be[b];
      if (mid >= end) continue;
      const int K = S.K[b];
      for (int e = tid; e < K * K; e += nt) {
        const int i = e / K, j = e % K;
        double* u = DL + (size_t)(s + i) * n + s + j;
        *u = S.hv[s + i] / *u;
      }
    }
    __syncthreads();
    for (int b = 0; b < nmerge; ++b) {
      const int s = S.bs[b], mid = S.bmid[b], end = S.be[b];
      if (mid >= end) continue;
      const int K = S.K[b];
      for (int j = tid; j < K; j += nt) {
        double nrm = 0.0;
        for (int i = 0; i < K; ++i) {
          const double u = DL[(size_t)(s + i) * n + s + j];
          nrm = fma(u, u, nrm);
        }
        S.hp[s + j] = rsqrt(nrm);
      }
    }
    __syncthreads();
    if (debug) { long long tn = clock64(); tm[5] += tn - tlast; tlast = tn; }
    // M6: deflation rotations on the columns of Q (order matters: serial over
    // rotations, parallel over rows)
    for (int b = 0; b < nmerge; ++b) {
      const int s = S.bs[b], mid = S.bmid[b], end = S.be[b];
      if (mid >= end) continue;
      const int N = end - s;
      for (int c = tid; c < N; c += nt) S.col[s + c] = S.perm[s + S.keep[s + c]];
      for (int r = tid; r < N; r += nt) {
        double* row = Q + (size_t)(s + r) * n;
        for (int q = 0; q < S.nrot[b]; ++q) {
          const int cp = S.perm[s + S.roti[s + q]], ci = S.perm[s + S.rotj[s + q]];
          const double c = S.rotc[s + q], sn = S.rots[s + q];
          const double gp = row[cp], gi = row[ci];
          row[cp] = c * gp + sn * gi;
          row[ci] = -sn * gp + c * gi;
        }
      }
    }
    __syncthreads();
    if (debug) { long long tn = clock64(); tm[6] += tn - tlast; tlast = tn; }
    // M7: new eigenvectors: kept columns Q[:, perm[keep]] U, deflated columns copied;
    // carried blocks copied unchanged
    for (int b = 0; b < nmerge; ++b) {
      const int s = S.bs[b], mid = S.bmid[b], end = S.be[b], N = end - s;
      if (mid >= end) {
        for (int e = tid; e < N * N; e += nt) {
          const int r = e / N, c = e % N;
          Qn[(size_t)(s + r) * n + s + c] = Q[(size_t)(s + r) * n + s + c];
        }
        continue;
      }
      const int K = S.K[b];
      if (N >= 64 && K >= 16) {
        // kept columns by DMMA.8x8x4: warp tiles of 16 rows x 32 columns
        // (2 x 4 accumulator blocks), A = Q[:, col[k]] gathered, B = U
        const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
        const int fr = lane >> 2, fc = lane & 3;
        const int trows = (N + 15) / 16, tcols = (K + 31) / 32;
        for (int tt = warp; tt < trows * tcols; tt += nw) {
          const int r0 = (tt / tcols) * 16, c0 = (tt % tcols) * 32;
          double acc[2][4][2];
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
          for (int k0 = 0; k0 < K; k0 += 4) {
            const int k = k0 + fc;
            const bool kok = k < K;
            const int qc = kok ? S.col[s + k] : 0;
            double a[2], bb[4];
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int r = r0 + 8 * i + fr;
              a[i] = (kok && r < N) ? Q[(size_t)(s + r) * n + qc] : 0.0;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int c = c0 + 8 * j + fr;
              bb[j] = (kok && c < K) ? DL[(size_t)(s + k) * n + s + c] : 0.0;
            }
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
              for (int j = 0; j < 4; ++j) nys::dmma(acc[i][j][0], acc[i][j][1], a[i], bb[j]);
          }
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int r = r0 + 8 * i + fr, c = c0 + 8 * j + 2 * fc + h;
                if (r < N && c < K) Qn[(size_t)(s + r) * n + s + c] = acc[i][j][h] * S.hp[s + c];
              }
        }
      } else {
      // kept columns: 4 outputs per thread (independent FMA chains share the
      // Q-row loads); deflated columns: gathered copies
      // adjacent lanes take adjacent output columns (conflict-free U reads); each
      // thread owns 4 rows, whose Q entries are warp-broadcast loads
      const int NQ = (N + 3) / 4;
      for (int e = tid; e < NQ * K; e += nt) {
        const int c = e % K, r0 = 4 * (e / K);
        double a[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 4
        for (int i = 0; i < K; ++i) {
          const double u = DL[(size_t)(s + i) * n + s + c];
          const int qc = S.col[s + i];
#pragma unroll
          for (int t = 0; t < 4; ++t)
            if (r0 + t < N) a[t] = fma(Q[(size_t)(s + r0 + t) * n + qc], u, a[t]);
        }
        const double h = S.hp[s + c];
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (r0 + t < N) Qn[(size_t)(s + r0 + t) * n + s + c] = a[t] * h;
      }
      }
      for (int e = tid; e < N * (N - K); e += nt) {
        const int r = e / (N - K), c = K + e % (N - K);
        Qn[(size_t)(s + r) * n + s + c] = Q[(size_t)(s + r) * n + S.perm[s + S.keep[s + c]]];
      }
    }
    __syncthreads();
    for (int b = 0; b < nmerge; ++b) {
      const int s = S.bs[b], mid = S.bmid[b], end = S.be[b], N = end - s;
      if (mid >= end) continue;
      const int K = S.K[b];
      const double sg = S.sgn[b];
      for (int c = tid; c < N; c += nt) {
        const double l = c < K ? S.zh[s + c] : S.ds[s + S.keep[s + c]];
        S.lam[s + c] = sg * l;
      }
    }
    if (debug) { long long tn = clock64(); tm[7] += tn - tlast; tlast = tn; }
    // swap Q <-> Qn (all threads hold the same pointers)
    double* t = Q;
    Q = Qn;
    Qn = t;
    __syncthreads();
  }

  tc3 = clock64();
  if (!kSmem) {
    // large n: the back-transform and the epilogue run as separate kernels
    // (dc_backT_out_kernel: columns of Q in registers, reflectors staged in smem)
    double* tail = gbuf + (size_t)n * ld + 3 * (size_t)n * n;   // lam | beta | qsel
    for (int i = tid; i < n; i += nt) {
      tail[i] = S.lam[i];
      tail[n + i] = S.beta[i];
    }
    if (tid == 0) {
      reinterpret_cast<int*>(tail + 2 * n)[0] = (Q == base + (size_t)n * ld) ? 0 : 1;
      reinterpret_cast<int*>(tail + 2 * n)[1] = 0;
    }
    if (debug && tid == 0) {
      printf("[nys dc] merge phases: pre %lld M1 %lld M2 %lld M3 %lld M4 %lld M5 %lld M6 %lld M7+ %lld\n",
             tm[0], tm[1], tm[2], tm[3], tm[4], tm[5], tm[6], tm[7]);
      printf("[nys dc] n=%d tridiag=%lld leaves=%lld merges=%lld (backT split)\n", n, tc1 - tc0, tc2 - tc1, tc3 - tc2);
    }
    return;
  }
  // ---------------- back-transform Z = H_0 ... H_{n-3} Q (reflectors in A)
  // tpc threads (adjacent lanes) share one column's dot product: FP64 FMA
  // latency, not bandwidth, bounds a serial n-term chain on B200
  const int tpc = (nt / n) >= 8 ? 8 : ((nt / n) >= 4 ? 4 : ((nt / n) >= 2 ? 2 : 1));
  for (int k = n - 3; k >= 0; --k) {
    const double beta = S.beta[k];
    if (beta == 0.0) continue;
    const int i0 = k + 1;
    for (int i = i0 + tid; i < n; i += nt) S.hv[i] = A[(size_t)i * ld + k];
    __syncthreads();
    const int work = (n * tpc + 31) / 32 * 32;   // whole warps: the shuffles need all lanes
    for (int t = tid; t < work; t += nt) {
      const int c = t / tpc, sub = t % tpc;
      double a0 = 0.0, a1 = 0.0;
      if (c < n) {
        int i = i0 + sub;
        for (; i + tpc < n; i += 2 * tpc) {
          a0 = fma(S.hv[i], Q[(size_t)i * n + c], a0);
          a1 = fma(S.hv[i + tpc], Q[(size_t)(i + tpc) * n + c], a1);
        }
        if (i < n) a0 = fma(S.hv[i], Q[(size_t)i * n + c], a0);
      }
      double acc = a0 + a1;
      for (int o = 1; o < tpc; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (sub == 0 && c < n) S.hp[c] = beta * acc;
    }
    __syncthreads();
    const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
    // this lane's columns c = lane + 32 t; rows in groups of kG, loads first
    double hpc[kT];
#pragma unroll
    for (int t = 0; t < kT; ++t) hpc[t] = lane + 32 * t < n ? S.hp[lane + 32 * t] : 0.0;
    constexpr int kG = kT <= 2 ? 4 : 1;
    for (int ib = i0 + warp; ib < n; ib += nw * kG) {
      double val[kG][kT];
#pragma unroll
      for (int g = 0; g < kG; ++g) {
        const int i = ib + g * nw;
#pragma unroll
        for (int t = 0; t < kT; ++t) {
          const int c = lane + 32 * t;
          val[g][t] = (i < n && c < n) ? Q[(size_t)i * n + c] : 0.0;
        }
      }
#pragma unroll
      for (int g = 0; g < kG; ++g) {
        const int i = ib + g * nw;
        if (i >= n) break;
        const double vi = S.hv[i];
#pragma unroll
        for (int t = 0; t < kT; ++t) {
          const int c = lane + 32 * t;
          if (c < n) Q[(size_t)i * n + c] = val[g][t] - vi * hpc[t];
        }
      }
    }
    __syncthreads();
  }

  tc4 = clock64();
  if (debug && tid == 0)
    printf("[nys dc] merge phases: pre %lld M1 %lld M2 %lld M3 %lld M4 %lld M5 %lld M6 %lld M7+ %lld\n",
           tm[0], tm[1], tm[2], tm[3], tm[4], tm[5], tm[6], tm[7]);
  if (debug && tid == 0) printf("[nys dc] n=%d tridiag=%lld leaves=%lld merges=%lld backT=%lld\n", n, tc1 - tc0, tc2 - tc1, tc3 - tc2, tc4 - tc3);
  // ---------------- epilogue: descending order, drop rule, W
  for (int i = tid; i < n; i += nt) {
    const double di = S.lam[i];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const double dj = S.lam[j];
      rank += (dj > di) || (dj == di && j > i);
    }
    S.perm[rank] = i;
  }
  __syncthreads();
  const double s0 = S.lam[S.perm[0]];
  const double cut = fmax(drop_tol * s0, 0.0);
  for (int k = tid; k < n; k += nt) eigvals[k] = S.lam[S.perm[k]];
  if (tid == 0) {
    int me = 0;
    while (me < n && S.lam[S.perm[me]] > cut) ++me;
    *m_eff_out = me;
    *info = NYS_INFO_OK;
  }
  for (int e = tid; e < n * n; e += nt) {
    const int i = e / n, k = e % n;
    const int src = S.perm[k];
    const double v = Q[(size_t)i * n + src];
    eigvecs[e] = v;
    const double sk = S.lam[src];
    Wout[e] = (sk > cut) ? v / sqrt(sk) : 0.0;
  }
}

// Back-transform Z = H_0 H_1 ... H_{n-3} Q fused with the epilogue (descending
// order, ties: higher index first, nystrom.py:151; drop rule; W = V / sqrt(s)).
// Each warp owns kCpw columns of Q in registers (kRows rows per lane); the CTA
// stages the Householder vectors through shared memory kRefl at a time (zeros
// above the diagonal written explicitly), the next chunk prefetched into
// registers while this one is applied, so every reflector costs shared-memory
// loads and one warp reduction instead of an L2 round trip.  A column's rank in
// the sorted spectrum is counted by its own warp, which then writes its
// eigenvector and W column straight to their final place.
constexpr int kRefl = 8, kBtWarps = 8, kCpw = 2;
template <int kRows>
__global__ void __launch_bounds__(kBtWarps * 32)
    dc_backT_out_kernel(const double* __restrict__ gbuf, int n, double drop_tol,
                        double* __restrict__ eigvals, double* __restrict__ eigvecs,
                        double* __restrict__ Wout, int* __restrict__ m_eff_out,
                        int* __restrict__ info) {
  __shared__ double vs[2][kRefl][kDcMaxN];
  __shared__ double bs[kDcMaxN];
  const int ld = dc_ld(n);
  const double* A = gbuf;
  const double* tail = gbuf + (size_t)n * ld + 3 * (size_t)n * n;
  const double* lam = tail;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (reinterpret_cast<const int*>(tail + 2 * n)[1] != 0) {   // degenerate landmarks
    if (blockIdx.x == 0 && tid == 0) {
      *m_eff_out = 0;
      *info = NYS_INFO_DEGENERATE;
    }
    return;
  }
  const int qsel = reinterpret_cast<const int*>(tail + 2 * n)[0];
  const double* Q = gbuf + (size_t)n * ld + (qsel ? (size_t)n * n : 0);
  for (int i = tid; i < n; i += blockDim.x) bs[i] = tail[n + i];
  int col[kCpw];
  double z[kCpw][kRows];
#pragma unroll
  for (int w = 0; w < kCpw; ++w) {
    col[w] = (blockIdx.x * kBtWarps + warp) * kCpw + w;
#pragma unroll
    for (int t = 0; t < kRows; ++t) {
      const int i = lane + 32 * t;
      z[w][t] = (col[w] < n && i < n) ? Q[(size_t)i * n + col[w]] : 0.0;
    }
  }
  // chunks of reflectors [k_lo, k_lo + kRefl), applied from the last one down
  const int nk = n - 2;                          // reflectors 0 .. n-3
  const int nchunk = (nk + kRefl - 1) / kRefl;
  constexpr int kPer = (kRefl * kDcMaxN) / (kBtWarps * 32);   // staged entries per thread
  double pre[kPer];
  auto fetch = [&](int c) {   // chunk c into registers: entry e = kk * n + i
    const int k_lo = c * kRefl;
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = tid + u * kBtWarps * 32, kk = e / kDcMaxN, i = e % kDcMaxN, k = k_lo + kk;
      pre[u] = (k < nk && i > k && i < n) ? A[(size_t)i * ld + k] : 0.0;
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = tid + u * kBtWarps * 32;
      vs[buf][e / kDcMaxN][e % kDcMaxN] = pre[u];
    }
  };
  if (nchunk > 0) {
    fetch(nchunk - 1);
    stash(0);
  }
  __syncthreads();
  for (int c = nchunk - 1, buf = 0; c >= 0; --c, buf ^= 1) {
    if (c > 0) fetch(c - 1);
    const int k_lo = c * kRefl;
    for (int kk = min(kRefl, nk - k_lo) - 1; kk >= 0; --kk) {
      const double bk = bs[k_lo + kk];
      if (bk == 0.0) continue;
      double v[kRows];
#pragma unroll
      for (int t = 0; t < kRows; ++t) v[t] = vs[buf][kk][lane + 32 * t];
      double d[kCpw];
#pragma unroll
      for (int w = 0; w < kCpw; ++w) {
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int t = 0; t < kRows; t += 2) {
          a0 = fma(v[t], z[w][t], a0);
          if (t + 1 < kRows) a1 = fma(v[t + 1], z[w][t + 1], a1);
        }
        d[w] = a0 + a1;
      }
#pragma unroll
      for (int o = 16; o; o >>= 1)
#pragma unroll
        for (int w = 0; w < kCpw; ++w) d[w] += __shfl_xor_sync(0xffffffffu, d[w], o);
#pragma unroll
      for (int w = 0; w < kCpw; ++w) {
        const double wk = bk * d[w];
#pragma unroll
        for (int t = 0; t < kRows; ++t) z[w][t] = fma(-v[t], wk, z[w][t]);
      }
    }
    if (c > 0) stash(buf ^ 1);
    __syncthreads();
  }
  // epilogue: s_0, the cut, this column's rank; m_eff and the eigenvalues
  double smax = -INFINITY;
  for (int j = lane; j < n; j += 32) smax = fmax(smax, lam[j]);
#pragma unroll
  for (int o = 16; o; o >>= 1) smax = fmax(smax, __shfl_xor_sync(0xffffffffu, smax, o));
  const double cut = fmax(drop_tol * smax, 0.0);
  if (blockIdx.x == 0 && warp == 0) {
    int cnt = 0;
    for (int j = lane; j < n; j += 32) cnt += lam[j] > cut;
#pragma unroll
    for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) {
      *m_eff_out = cnt;
      *info = NYS_INFO_OK;
    }
  }
#pragma unroll
  for (int w = 0; w < kCpw; ++w) {
    if (col[w] >= n) continue;
    const double lc = lam[col[w]];
    int rank = 0;
    for (int j = lane; j < n; j += 32) {
      const double lj = lam[j];
      rank += (lj > lc) || (lj == lc && j > col[w]);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
    if (lane == 0) eigvals[rank] = lc;
    const bool keep = lc > cut;
    const double rs = keep ? 1.0 / sqrt(lc) : 0.0;
#pragma unroll
    for (int t = 0; t < kRows; ++t) {
      const int i = lane + 32 * t;
      if (i < n) {
        eigvecs[(size_t)i * n + rank] = z[w][t];
        Wout[(size_t)i * n + rank] = keep ? z[w][t] * rs : 0.0;
      }
    }
  }
}

}  // namespace

namespace nys_host {
bool dcc_fits(int n);
int launch_dcc_eig(const double* lm, const double* Ain, int n, double sigma2, double* gbuf,
                   int debug, cudaStream_t st);
size_t dc_buffer_bytes(int n) {
  // A (n x ld) | Q | Qn | DL (n x n each) | lam, beta (n each) | qsel
  return ((size_t)n * dc_ld(n) + 3 * (size_t)n * n + 2 * (size_t)n + 2) * sizeof(double);
}
bool dc_fits(int n) { return n >= 1 && n <= kDcMaxN; }
bool dc_uses_smem(int n) { return dc_buffer_bytes(n) <= 150 * 1024; }

int launch_dc_eig(const double* lm, const double* Ain, int n, double sigma2, double drop_tol,
                  double* eigvals, double* eigvecs, double* W, int* m_eff, int* info, void* ws,
                  size_t ws_bytes, cudaStream_t st) {
  const size_t need = dc_buffer_bytes(n);
  const int use_smem = dc_uses_smem(n);
  size_t dyn = 0;
  if (!use_smem && (ws == nullptr || ws_bytes < need)) return NYS_EWORKSPACE;
  const int threads = n <= 64 ? 256 : kDcThreads;
  const int dbg = getenv("NYS_EIG_DEBUG") != nullptr;
  auto launch = [&](auto kern) -> int {
    // smem path: the matrices; global path: the panel's V and W (tridiag_blocked)
    dyn = use_smem ? need
                   : (2 * (size_t)n * (kTNb + 1) + 2 * kTNb + 4 * 256) * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)dyn);
    if (e != cudaSuccess) return record_cuda(e);
    kern<<<1, threads, dyn, st>>>(lm, Ain, n, sigma2, drop_tol, eigvals, eigvecs, W, m_eff, info,
                                  static_cast<double*>(ws), use_smem, dbg);
    return NYS_OK;
  };
  int rc;
  // 64 < n <= 256: the cluster kernel (eig_cluster.cu); NYS_EIG_ALGO=dc1 keeps the
  // one-CTA kernel (A/B tests)
  const char* algo = getenv("NYS_EIG_ALGO");
  const bool one_cta = algo && algo[0] == 'd' && algo[1] == 'c' && algo[2] == '1';
  if (!use_smem && !one_cta && dcc_fits(n))
    rc = launch_dcc_eig(lm, Ain, n, sigma2, static_cast<double*>(ws), dbg, st);
  else if (use_smem)
    rc = n <= 64 ? launch(dc_eig_kernel<true, 2>) : launch(dc_eig_kernel<true, kDcMaxN / 32>);
  else
    rc = n <= 64 ? launch(dc_eig_kernel<false, 2>) : launch(dc_eig_kernel<false, kDcMaxN / 32>);
  if (rc) return rc;
  if (use_smem || one_cta || !dcc_fits(n)) count_launches(1);
  NYS_CHECK_LAUNCH();
  if (!use_smem) {
    double* g = static_cast<double*>(ws);
    const int grid = (n + kBtWarps * kCpw - 1) / (kBtWarps * kCpw);
    if (n <= 128)
      dc_backT_out_kernel<4><<<grid, 32 * kBtWarps, 0, st>>>(g, n, drop_tol, eigvals, eigvecs, W,
                                                             m_eff, info);
    else
      dc_backT_out_kernel<kDcMaxN / 32><<<grid, 32 * kBtWarps, 0, st>>>(g, n, drop_tol, eigvals,
                                                                        eigvecs, W, m_eff, info);
    count_launches(1);
    NYS_CHECK_LAUNCH();
  }
  return NYS_OK;
}
}  // namespace nys_host
