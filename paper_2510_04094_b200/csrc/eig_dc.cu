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

NYS_DEV double dc_block_sum(double x, DcShared& S) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  __syncthreads();
  if (lane == 0) S.red[w] = x;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < nw; ++i) s += S.red[i];
  return s;
}

// implicit QL on the leaf [s, s+len) of (d, e), eigenvectors into Q block
NYS_DEV void leaf_ql(DcShared& S, double* Q, int n, int s, int len) {
  double* d = S.d + s;
  double* e = S.e + s;   // e[i] couples i, i+1 inside the leaf; e[len-1] is unused
  double ehold = len > 0 ? e[len - 1] : 0.0;
  if (len > 0) e[len - 1] = 0.0;
  for (int r = 0; r < len; ++r)
    for (int c = 0; c < len; ++c) Q[(size_t)(s + r) * n + s + c] = (r == c) ? 1.0 : 0.0;
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
      int i = mm - 1;
      bool early = false;
      for (; i >= l; --i) {
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
        for (int k = 0; k < len; ++k) {   // columns i, i+1 of the leaf's Z
          double* row = Q + (size_t)(s + k) * n + s;
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
  if (len > 0) e[len - 1] = ehold;
  for (int c = 0; c < len; ++c) S.lam[s + c] = d[c];
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

// kSmem: the working matrices live in dynamic shared memory (n <= 64) -- a
// compile-time address space, so the compiler emits LDS/STS; kT: columns per
// lane in the rank-2 update (ceil(n / 32) bound)
template <bool kSmem, int kT>
__global__ void __launch_bounds__(kT <= 2 ? 256 : kDcThreads, 1)
    dc_eig_kernel(const double* __restrict__ lm, int n, double sigma2, double drop_tol,
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
    const double d = lm[i] - lm[j];
    A[(size_t)i * ld + j] = nys::rbf(d, sigma2);
    if (i != j && fabs(d) <= 1e-12) S.degenerate = 1;
  }
  __syncthreads();
  if (S.degenerate) {
    if (tid == 0) {
      *info = NYS_INFO_DEGENERATE;
      *m_eff_out = 0;
    }
    return;
  }

  // ---------------- Householder tridiagonalisation (as eig.cu phase 1)
  // Three barriers per reflector: warp 0 forms the reflector (norm by warp
  // shuffles), the matvec splits every row over tpr lanes, and each warp
  // recomputes v.p itself so the rank-2 update needs no extra barrier.
  long long tq[4] = {0, 0, 0, 0};
  const long long tsetup = clock64() - tc0;
  {
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
  for (int i = tid; i < n; i += nt) S.d[i] = A[(size_t)i * ld + i];
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
  for (int t = tid; t < nleaf; t += nt) {
    const int s = t * kLeaf, len = min(kLeaf, n - s);
    leaf_ql(S, Q, n, s, len);
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
    // M2: normalise, deflate (serial scan per block)
    for (int b = tid; b < nmerge; b += nt) {
      const int s = S.bs[b], mid = S.bmid[b], end = S.be[b], N = end - s;
      if (mid >= end) continue;
      double zn2 = 0.0, dmax = 0.0;
      for (int i = 0; i < N; ++i) {
        zn2 += S.zs[s + i] * S.zs[s + i];
        dmax = fmax(dmax, fabs(S.ds[s + i]));
      }
      const double rho = fabs(S.e[mid - 1]) * zn2;
      const double inv = zn2 > 0.0 ? 1.0 / sqrt(zn2) : 0.0;
      for (int i = 0; i < N; ++i) S.zs[s + i] *= inv;
      S.rho[b] = rho;
      const double tol = 8.0 * kEps * fmax(dmax, rho);
      int K = 0, nd = 0, nrot = 0, prev = -1;
      int* keep = S.keep + s;
      // keep[] collects kept indices from the front and deflated ones from the back
      if (rho <= tol) {
        for (int i = 0; i < N; ++i) keep[N - 1 - i] = i;   // all deflated
        nd = N;
      } else {
        for (int i = 0; i < N; ++i) {
          if (fabs(rho * S.zs[s + i]) <= tol) {
            keep[N - 1 - nd++] = i;
            continue;
          }
          if (prev >= 0) {
            const double zi = S.zs[s + i], zp = S.zs[s + prev];
            const double r = hypot(zi, zp);
            const double c = zi / r, sn = -zp / r;
            const double t = S.ds[s + i] - S.ds[s + prev];
            if (fabs(t * c * sn) <= tol) {
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
              // prev becomes deflated: remove it from the kept list
              --K;
              keep[N - 1 - nd++] = prev;
            }
          }
          keep[K++] = i;
          prev = i;
        }
      }
      S.K[b] = K;
      S.nrot[b] = nrot;
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

}  // namespace

namespace nys_host {
size_t dc_buffer_bytes(int n) {
  return ((size_t)n * dc_ld(n) + 3 * (size_t)n * n) * sizeof(double);
}
bool dc_fits(int n) { return n >= 1 && n <= kDcMaxN; }
bool dc_uses_smem(int n) { return dc_buffer_bytes(n) <= 150 * 1024; }

int launch_dc_eig(const double* lm, int n, double sigma2, double drop_tol, double* eigvals,
                  double* eigvecs, double* W, int* m_eff, int* info, void* ws, size_t ws_bytes,
                  cudaStream_t st) {
  const size_t need = dc_buffer_bytes(n);
  const int use_smem = dc_uses_smem(n);
  size_t dyn = 0;
  if (!use_smem && (ws == nullptr || ws_bytes < need)) return NYS_EWORKSPACE;
  const int threads = n <= 64 ? 256 : kDcThreads;
  const int dbg = getenv("NYS_EIG_DEBUG") != nullptr;
  auto launch = [&](auto kern) -> int {
    if (use_smem) {
      dyn = need;
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)dyn);
      if (e != cudaSuccess) return record_cuda(e);
    }
    kern<<<1, threads, dyn, st>>>(lm, n, sigma2, drop_tol, eigvals, eigvecs, W, m_eff, info,
                                  static_cast<double*>(ws), use_smem, dbg);
    return NYS_OK;
  };
  int rc;
  if (use_smem)
    rc = n <= 64 ? launch(dc_eig_kernel<true, 2>) : launch(dc_eig_kernel<true, kDcMaxN / 32>);
  else
    rc = n <= 64 ? launch(dc_eig_kernel<false, 2>) : launch(dc_eig_kernel<false, kDcMaxN / 32>);
  if (rc) return rc;
  count_launches(1);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}
}  // namespace nys_host
