// Landmark eigendecomposition for 64 < m <= 256 on ONE THREAD-BLOCK CLUSTER of
// 8 CTAs (8 SMs), the route of the reference's LAPACK dsyevd
// (nystrom.py:150): Householder tridiagonalisation, Cuppen divide and conquer,
// back-transform.  The one-CTA kernel (eig_dc.cu) keeps the m x m matrices in
// L2 at this size (512 KB each does not fit one SM's shared memory): every
// reflector's matvec then streams the trailing matrix from L2 on one SM and the
// merge GEMMs read their operands from L2 -- 3.7 ms at m = 256.  Here the
// matrices are split over the cluster's shared memories and the CTAs exchange
// only vectors through DSMEM (distributed shared memory):
//
//  * tridiagonalisation (dsytrd / dlatrd order, panels of kPb columns): CTA r
//    owns rows i = r + 8t of A in shared memory; the panel's V and W are
//    REPLICATED in every CTA (each new column pushed to all eight), so t1 =
//    W^T v and t2 = V^T v are local.  Per reflector: corrected column + tail
//    norm partial (push, cluster barrier), reflector formed redundantly in every
//    CTA, local matvec of the CTA's rows, v.p partial (push, barrier), w column
//    (push, barrier).  The panel's rank-2 update of the trailing rows runs as
//    DMMA.8x8x4 tiles on each CTA's own rows.
//  * divide and conquer: tears every kLeaf rows, leaves by QL (each CTA its own
//    rows' leaves), then log2(m / kLeaf) merge levels.  The eigenvector matrix Q
//    is split by contiguous row slabs; every O(m) vector step (sort, deflation,
//    eigenvalue bookkeeping) runs redundantly in all CTAs on replicated vectors
//    (identical inputs, identical code: identical results), the O(K^2) steps
//    (secular roots, Gu-Eisenstat z, column norms of U) are split over the
//    eight CTAs and their results pushed to all, and the merge GEMM
//    Q_new = Q[:, kept] U runs on each CTA's own rows with U generated in
//    registers from the replicated vectors: U_ij = zhat_i / ((d_i - d_org(j)) -
//    tau_j) (the root stored as pole + offset, as the one-CTA kernel forms
//    d_i - lambda_j), so the K x K matrix never exists anywhere.
//
// The back-transform and the epilogue (descending order, drop rule, W) are the
// multi-SM kernels of eig_dc.cu; the buffer layout is the same.
#include <cooperative_groups.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int kNC = 8;             // CTAs per cluster
constexpr int kCThreads = 512;     // 16 warps per CTA
constexpr int kCWarps = kCThreads / 32;
constexpr int kCMaxN = 256;
constexpr int kCLeaf = 8;
constexpr int kCBlocks = kCMaxN / kCLeaf;
constexpr int kPb = 16;            // panel width (V, W replicated: 2 n (kPb+1) doubles)
constexpr int kLdv = kPb + 1;
constexpr int kMaxOwn = kCMaxN / kNC;   // tridiagonal rows per CTA
constexpr double kEpsC = 2.220446049250313e-16;
#ifndef DCC_SKIP_T12
#define DCC_SKIP_T12 0   // timing experiments only (wrong results when set)
#endif
#ifndef DCC_SKIP_MV
#define DCC_SKIP_MV 0
#endif
#ifndef DCC_SKIP_Q
#define DCC_SKIP_Q 0
#endif

// permuted index space of the tridiagonalisation: row / column i <-> position
NYS_DEV int dcc_pos(int i) { return (i % kNC) * kMaxOwn + i / kNC; }
NYS_DEV int dcc_ipos(int p) { return (p % kMaxOwn) * kNC + p / kMaxOwn; }

// must match eig_dc.cu (shared global buffer layout)
__host__ __device__ inline int dcc_ld(int n) { return n + (((4 - n) % 16) + 16) % 16; }

struct DccShared {
  double d[kCMaxN], e[kCMaxN], beta[kCMaxN], lam[kCMaxN];
  double ds[kCMaxN], zs[kCMaxN], zraw[kCMaxN], tau[kCMaxN];
  double hv[kCMaxN], hp[kCMaxN], rotc[kCMaxN], rots[kCMaxN];
  int perm[kCMaxN], keep[kCMaxN], roti[kCMaxN], rotj[kCMaxN], col[kCMaxN], org[kCMaxN];
  double t1[kPb], t2[kPb];
  double slotA[2][kNC], slotB[2][kNC], slotP[2], slotD[kNC];
  uint64_t xbar[2];
  double colA[kMaxOwn], ploc[kMaxOwn], mvp[kNC][kMaxOwn];
  double rho[kCBlocks], sgn[kCBlocks];
  int K[kCBlocks], nrot[kCBlocks], bs[kCBlocks], bmid[kCBlocks], be[kCBlocks];
  int degenerate;
};

// ---- DSMEM exchanges: every push is an st.async into the destination CTA's
// shared memory that completes bytes on that CTA's exchange mbarrier; each CTA
// announces the bytes it expects (identical everywhere: every CTA receives
// every pushed value) and waits on its own barrier.  No cluster-wide barrier
// (barrier.cluster = MEMBAR.ALL.GPU + ERRBAR + CGA barrier, ~1 us) on the
// per-reflector path.  Two barriers alternate; exchange x uses barrier x & 1
// in phase x >> 1.  A CTA can run at most one exchange ahead of another (its
// next exchange needs the other's pushes), so early bytes land in the right
// phase (a phase cannot complete before its own expect_tx arrival).
struct Xch {
  uint64_t* bar;
  int xe;
};
NYS_DEV uint32_t mapa_u32(uint32_t local, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
NYS_DEV void xpush(const Xch& X, double* p, double v) {
  const uint32_t la = nys::smem_u32(p), lb = nys::smem_u32(X.bar + (X.xe & 1));
#pragma unroll
  for (int r = 0; r < kNC; ++r)
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];\n" ::"r"(
            mapa_u32(la, r)),
        "d"(v), "r"(mapa_u32(lb, r))
        : "memory");
}
NYS_DEV void xpush(const Xch& X, int* p, int v) {
  const uint32_t la = nys::smem_u32(p), lb = nys::smem_u32(X.bar + (X.xe & 1));
#pragma unroll
  for (int r = 0; r < kNC; ++r)
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.s32 [%0], %1, [%2];\n" ::"r"(
            mapa_u32(la, r)),
        "r"(v), "r"(mapa_u32(lb, r))
        : "memory");
}
// thread 0 of every CTA, once per exchange: the bytes this CTA will receive
NYS_DEV void xbegin(const Xch& X, uint32_t bytes) {
  if (threadIdx.x == 0)
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                     nys::smem_u32(X.bar + (X.xe & 1))),
                 "r"(bytes)
                 : "memory");
}
// one thread polls the barrier (a CTA full of try_wait loops would contend for
// the shared-memory port with the warp doing the critical-path work), then a
// CTA barrier releases the rest (the acquire is cumulative through bar.sync)
NYS_DEV void xwait(Xch& X) {
  if (threadIdx.x == 0) {
    const uint32_t b = nys::smem_u32(X.bar + (X.xe & 1)), par = (X.xe >> 1) & 1;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "XW_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra XW_%=;\n"
        "}\n" ::"r"(b),
        "r"(par)
        : "memory");
  }
  __syncthreads();
  ++X.xe;
}

NYS_DEV double gsum_c(double v, int G, unsigned gm) {
  for (int o = 1; o < G; o <<= 1) v += __shfl_xor_sync(gm, v, o);
  return v;
}

// implicit QL on the leaf [s, s+len) of (d, e) (one warp; every lane runs the
// scalar recurrence redundantly, lane k rotates row k of the leaf).  Q rows are
// the CTA's own (row 0 of `Qrow` is global row s), columns global.  Same
// arithmetic as eig_dc.cu's leaf_ql.
NYS_DEV void leaf_ql_c(DccShared& S, double* Qrow, int ldq, int s, int len, int lane) {
  double* d = S.d + s;
  double* e = S.e + s;
  const double ehold = len > 0 ? e[len - 1] : 0.0;
  __syncwarp();
  if (len > 0) e[len - 1] = 0.0;
  double* row = lane < len ? Qrow + (size_t)lane * ldq + s : nullptr;
  if (row)
    for (int c = 0; c < len; ++c) row[c] = (lane == c) ? 1.0 : 0.0;
  for (int l = 0; l < len; ++l) {
    for (int iter = 0; iter < 60; ++iter) {
      int mm = l;
      for (; mm < len - 1; ++mm) {
        const double dd = fabs(d[mm]) + fabs(d[mm + 1]);
        if (fabs(e[mm]) <= kEpsC * dd) break;
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
        if (row) {
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
  __syncwarp();
}

// d_i - lambda_j in the coordinates of root j's pole (as eig_dc.cu forms DL)
NYS_DEV double dl_of(const DccShared& S, int s, int i, int j) {
  const int* kp = S.keep + s;
  return (S.ds[s + kp[i]] - S.ds[s + kp[S.org[s + j]]]) - S.tau[s + j];
}

// secular root j of diag(ds) + rho zz^T over the K kept entries of a block
// (eig_dc.cu's secular_root); returns the pole index and the offset tau
NYS_DEV void secular_root_c(const DccShared& S, int s, int j, int K, double rho, int gl, int G,
                            unsigned gm, int& org_out, double& tau_out) {
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
    f = 1.0 / rho + gsum_c(f, G, gm);
    org = f >= 0.0 ? j : j + 1;
    lo = dk(j) - dk(org);
    hi = dk(j + 1) - dk(org);
  } else {
    org = K - 1;
    double zz = 0.0;
    for (int i = gl; i < K; i += G) zz += z2(i);
    zz = gsum_c(zz, G, gm);
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
    f = 1.0 / rho + gsum_c(f, G, gm);
    fabs_sum = 1.0 / rho + gsum_c(fabs_sum, G, gm);
    psi = gsum_c(psi, G, gm);
    dpsi = gsum_c(dpsi, G, gm);
    phi = gsum_c(phi, G, gm);
    dphi = gsum_c(dphi, G, gm);
    if (f > 0.0)
      hi = tau;
    else
      lo = tau;
    if (fabs(f) <= 8.0 * kEpsC * fabs_sum ||
        (hi - lo) <= 2.0 * kEpsC * fmax(fmax(fabs(lo), fabs(hi)), 1e-300))
      break;
    const double dj = (dk(j) - dorg) - tau;
    double x = 0.0;
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
  org_out = org;
  tau_out = tau;
}

// flattened (block, index) -> block; j becomes the index inside the block
NYS_DEV int find_block(const DccShared& S, int nmerge, int& j) {
  int b = 0;
  while (b < nmerge) {
    const int Kb = (S.bmid[b] < S.be[b]) ? S.K[b] : 0;
    if (j < Kb) break;
    j -= Kb;
    ++b;
  }
  return b;
}

__global__ void __cluster_dims__(kNC, 1, 1) __launch_bounds__(kCThreads, 1)
    dcc_eig_kernel(const double* __restrict__ lm, const double* __restrict__ Ain, int n,
                   double sigma2, double* __restrict__ gbuf, int debug) {
  extern __shared__ __align__(16) double dyn[];
  __shared__ DccShared S;
  cg::cluster_group cl = cg::this_cluster();
  const int rk = (int)cl.block_rank();
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int ld = dcc_ld(n);
  const int nloc = (n - rk + kNC - 1) / kNC;   // own tridiagonal rows i = rk + kNC t
  double* Vr = dyn;                            // positions x kLdv, replicated
  double* Wr = Vr + (size_t)kCMaxN * kLdv;
  double* tail = gbuf + (size_t)n * ld + 3 * (size_t)n * n;   // lam | beta | flags
  long long tc0 = clock64(), tc1 = 0, tc2 = 0, tc3 = 0;

  // ---------------- Omega = K(L, L), own rows (kernel.py:78-79 via nys::rbf)
  // Column / replicated-row index space is PERMUTED: position p = (i % 8) * 32 +
  // i / 8, so a CTA's own rows are 32 consecutive positions (warp lane t ->
  // position rk * 32 + t: V, W rows at stride kLdv, conflict-free).  The own
  // rows of A live in REGISTERS, in DMMA accumulator layout: warp w holds the
  // 16-row x 32-position tile (w / 8, w % 8) -- the panel's rank-2 update is
  // one DMMA tile per warp, the matvec reads only v from shared memory.
  if (tid == 0) {
    S.degenerate = 0;
    nys::mbar_init(&S.xbar[0], 1);
    nys::mbar_init(&S.xbar[1], 1);
    nys::fence_mbar_init();
  }
  Xch X{S.xbar, 0};
  const int fr = lane >> 2, fc = lane & 3;
  const int rt = warp >> 3, ct = warp & 7;   // this warp's tile of A (own rows x positions)
  double acc[2][4][2];
#pragma unroll
  for (int i2 = 0; i2 < 2; ++i2)
#pragma unroll
    for (int jb = 0; jb < 4; ++jb)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int lr = 16 * rt + 8 * i2 + fr, i = rk + kNC * lr;
        const int c = dcc_ipos(32 * ct + 8 * jb + 2 * fc + h);
        double a = 0.0;
        if (lr < nloc && c < n) a = Ain ? Ain[(size_t)i * n + c] : nys::rbf(lm[i] - lm[c], sigma2);
        acc[i2][jb][h] = a;
      }
  for (int e = tid; e < 2 * kCMaxN * kLdv; e += nt) Vr[e] = 0.0;   // Vr, Wr contiguous
  if (Ain == nullptr)   // every CTA checks every pair: the verdict needs no exchange
    for (int e = tid; e < n * n; e += nt) {
      const int i = e / n, j = e % n;
      if (i != j && fabs(lm[i] - lm[j]) <= 1e-12) S.degenerate = 1;
    }
  cl.sync();   // all CTAs resident (and their barriers initialised) before any push
  if (S.degenerate) {
    if (rk == 0 && tid == 0) reinterpret_cast<int*>(tail + 2 * n)[1] = 1;
    return;
  }
  // own rows' entries of column position pc -> S.colA (for the corrected column)
  auto emit_col = [&](int pc) {
    if ((pc >> 5) != ct) return;
    const int jb = (pc & 31) >> 3, f = (pc & 7) >> 1, h = pc & 1;
    if (fc != f) return;
#pragma unroll
    for (int i2 = 0; i2 < 2; ++i2) {
      double a = 0.0;
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh)
          if (b == jb && hh == h) a = acc[i2][b][hh];
      S.colA[16 * rt + 8 * i2 + fr] = a;
    }
  };

  // ---------------- Householder tridiagonalisation (dlatrd order, as eig_dc.cu)
  // Two exchanges per reflector: (A) the corrected column and the tail-norm
  // partials, (B) the v.p partials.  The w column is pushed without an exchange
  // of its own: its first remote reader (t1 of the next column) waits on the
  // next exchange (A); the one entry the next column's correction needs at
  // once, w_{j+1}, every CTA forms itself from p_{j+1} (pushed in B by its owner).
  long long tt_[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tl_ = clock64();
#define DCC_TT(k)                                                                  \
  if (debug) {                                                                     \
    const long long tn = clock64();                                                \
    tt_[k] += tn - tl_;                                                            \
    tl_ = tn;                                                                      \
  }
  const int prow = rk * kMaxOwn;   // position of own row t = prow + t
  int wprev = 0;                   // w entries pushed by the previous column
  emit_col(dcc_pos(0));
  __syncthreads();
  for (int k0 = 0; k0 + 2 < n; k0 += kPb) {
    const int nb = min(kPb, n - 2 - k0);
    for (int jj = 0; jj < nb; ++jj) {
      const int j = k0 + jj, pj = dcc_pos(j), pj1 = dcc_pos(j + 1), jp = j & 1;
      // exchange A: this column's V entries (rows >= j), the tail partials, and
      // the previous column's w entries (rows > j)
      xbegin(X, 8u * (uint32_t)((n - j) + kNC + wprev));
      // (1) corrected column j on the own rows i >= j, pushed into every V copy
      if (warp == 0) {
        const int t = lane, i = rk + kNC * t;
        double part = 0.0;
        if (t < nloc && i >= j) {
          double c = S.colA[t];
          const double* Vi = Vr + (size_t)(prow + t) * kLdv;
          const double* Wi = Wr + (size_t)(prow + t) * kLdv;
          const double* Vj = Vr + (size_t)pj * kLdv;
          const double* Wj = Wr + (size_t)pj * kLdv;
          double c1 = 0.0, c2 = 0.0, c3 = 0.0, c4 = 0.0;
#pragma unroll
          for (int q = 0; q < kPb; q += 2) {
            if (DCC_SKIP_Q) break;
            if (q < jj) {
              c1 = fma(Vi[q], Wj[q], c1);
              c2 = fma(Wi[q], Vj[q], c2);
            }
            if (q + 1 < jj) {
              c3 = fma(Vi[q + 1], Wj[q + 1], c3);
              c4 = fma(Wi[q + 1], Vj[q + 1], c4);
            }
          }
          c = c - ((c1 + c3) + (c2 + c4));
          if (i >= j + 2) part = c * c;
          xpush(X, Vr + (size_t)(prow + t) * kLdv + jj, c);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        if (lane == 0) xpush(X, &S.slotA[jp][rk], part);
      }
      DCC_TT(0);
      xwait(X);
      DCC_TT(1);
      // (2) the reflector, formed redundantly in every CTA (identical inputs)
      double tail2 = 0.0;
#pragma unroll
      for (int r = 0; r < kNC; ++r) tail2 += S.slotA[jp][r];
      const double x0 = Vr[(size_t)pj1 * kLdv + jj];
      double beta = 0.0, alpha = x0, v0 = x0;
      if (tail2 > 0.0) {
        const double nx = sqrt(fma(x0, x0, tail2));
        alpha = -copysign(nx, x0);
        v0 = x0 - alpha;
        beta = 2.0 / fma(v0, v0, tail2);
      }
      if (tid == 0) {
        S.d[j] = Vr[(size_t)pj * kLdv + jj];
        S.e[j] = alpha;
        S.beta[j] = beta;
      }
      if (beta == 0.0) {   // identity reflector: V, W columns stay zero
        __syncthreads();
        for (int p = tid; p < kCMaxN; p += nt) {
          const int c = dcc_ipos(p);
          if (c > j && c < n) {
            Vr[(size_t)p * kLdv + jj] = 0.0;
            Wr[(size_t)p * kLdv + jj] = 0.0;
          }
        }
        if (jj + 1 < nb) emit_col(pj1);
        __syncthreads();
        wprev = 0;
        continue;
      }
      DCC_TT(2);
      // (3) p = A v on the own rows i > j (panel-start matrix) from the register
      //     tiles: 8 entries per lane and row, reduced over the 4 lanes of a row
      //     and then (step 4) over the 8 column tiles; t1 = W^T v, t2 = V^T v
      //     redundantly (V, W are replicated).  v_{j+1} = v0 is substituted (the
      //     shared copy still holds x0 until the patch below).
      {
        double vv[4][2];
#pragma unroll
        for (int jb = 0; jb < 4; ++jb)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int p = 32 * ct + 8 * jb + 2 * fc + h, c = dcc_ipos(p);
            vv[jb][h] = (c > j && c < n) ? (c == j + 1 ? v0 : Vr[(size_t)p * kLdv + jj]) : 0.0;
          }
#pragma unroll
        for (int i2 = 0; i2 < 2; ++i2) {
          double a = 0.0;
#pragma unroll
          for (int jb = 0; jb < 4; ++jb)
#pragma unroll
            for (int h = 0; h < 2; ++h) if (!DCC_SKIP_MV) a = fma(acc[i2][jb][h], vv[jb][h], a);
          a += __shfl_xor_sync(0xffffffffu, a, 1);
          a += __shfl_xor_sync(0xffffffffu, a, 2);
          if (fc == 0) S.mvp[ct][16 * rt + 8 * i2 + fr] = a;
        }
        if (jj + 1 < nb) emit_col(pj1);   // next column's entries (panel-start matrix)
      }
      if (!DCC_SKIP_T12 && warp < jj) {   // lane owns positions lane + 32 u (column 8 lane + u)
        const int q = warp;
        double a1 = 0.0, a2 = 0.0;
#pragma unroll
        for (int u = 0; u < kCMaxN / 32; ++u) {
          const int p = lane + 32 * u, c = 8 * lane + u;
          if (c > j && c < n) {
            const double v = c == j + 1 ? v0 : Vr[(size_t)p * kLdv + jj];
            a1 = fma(Wr[(size_t)p * kLdv + q], v, a1);
            a2 = fma(Vr[(size_t)p * kLdv + q], v, a2);
          }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          a1 += __shfl_xor_sync(0xffffffffu, a1, o);
          a2 += __shfl_xor_sync(0xffffffffu, a2, o);
        }
        if (lane == 0) {
          S.t1[q] = a1;
          S.t2[q] = a2;
        }
      }
      __syncthreads();
      if (tid == 0) Vr[(size_t)pj1 * kLdv + jj] = v0;   // read again after exchange B
      xbegin(X, 8u * (kNC + 1));   // exchange B: v.p partials + p_{j+1}
      // (4) p <- beta (A v - V t1 - W t2) on the own rows; v.p partial; the owner
      //     of row j+1 also pushes p_{j+1}
      if (warp == 0) {
        const int t = lane, i = rk + kNC * t;
        double part = 0.0;
        if (t < nloc && i > j) {
          double pi = 0.0;
#pragma unroll
          for (int c8 = 0; c8 < 8; ++c8) pi += S.mvp[c8][t];
          const double* Vi = Vr + (size_t)(prow + t) * kLdv;
          const double* Wi = Wr + (size_t)(prow + t) * kLdv;
          double c1 = 0.0, c2 = 0.0, c3 = 0.0, c4 = 0.0;
#pragma unroll
          for (int q = 0; q < kPb; q += 2) {
            if (DCC_SKIP_Q) break;
            if (q < jj) {
              c1 = fma(Vi[q], S.t1[q], c1);
              c2 = fma(Wi[q], S.t2[q], c2);
            }
            if (q + 1 < jj) {
              c3 = fma(Vi[q + 1], S.t1[q + 1], c3);
              c4 = fma(Wi[q + 1], S.t2[q + 1], c4);
            }
          }
          pi = pi - ((c1 + c3) + (c2 + c4));
          pi *= beta;
          S.ploc[t] = pi;
          part = (i == j + 1 ? v0 : Vi[jj]) * pi;
          if (i == j + 1) xpush(X, &S.slotP[jp], pi);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        if (lane == 0) xpush(X, &S.slotB[jp][rk], part);
      }
      DCC_TT(3);
      xwait(X);
      DCC_TT(4);
      // (5) w = p - (beta/2)(v.p) v on the own rows, pushed into every W copy
      //     (row j+1: formed locally in every CTA); v to the global buffer below
      //     the diagonal (the back-transform's Householder vectors)
      if (warp == 0) {
        double vp = 0.0;
#pragma unroll
        for (int r = 0; r < kNC; ++r) vp += S.slotB[jp][r];
        const double Kc = 0.5 * beta * vp;
        const int t = lane, i = rk + kNC * t;
        if (t < nloc && i > j + 1) {
          const double v = Vr[(size_t)(prow + t) * kLdv + jj];
          const double w = S.ploc[t] - Kc * v;
          // the own copy by a plain store as well: the next column's correction
          // reads it before the exchange that completes the st.async
          Wr[(size_t)(prow + t) * kLdv + jj] = w;
          xpush(X, Wr + (size_t)(prow + t) * kLdv + jj, w);
          gbuf[(size_t)i * ld + j] = v;
        }
        if (t < nloc && i == j + 1) gbuf[(size_t)i * ld + j] = v0;
        if (lane == 0) Wr[(size_t)pj1 * kLdv + jj] = S.slotP[jp] - Kc * v0;
        __syncwarp();
      }
      wprev = n - j - 2;   // w rows > j + 1, counted by the next exchange
      DCC_TT(5);
    }
    xbegin(X, 8u * (uint32_t)wprev);   // the last column's w entries
    xwait(X);
    wprev = 0;
    __syncthreads();
    DCC_TT(6);
    // rank-2 update of the own rows: A -= V W^T + W V^T, one DMMA tile per warp.
    // Entries of rows or columns < t0 are never read again, so the tile is
    // updated whole; the k slots beyond 2 nb are masked.
    {
#pragma unroll 1
      for (int k4 = 0; k4 < 2 * nb; k4 += 4) {
        const int kq = k4 + fc;
        const bool kok = kq < 2 * nb;
        double a[2], bq[4];
#pragma unroll
        for (int i2 = 0; i2 < 2; ++i2) {
          const int pr = prow + 16 * rt + 8 * i2 + fr;
          a[i2] = kok ? -(kq < nb ? Vr[(size_t)pr * kLdv + kq] : Wr[(size_t)pr * kLdv + kq - nb])
                      : 0.0;
        }
#pragma unroll
        for (int jb = 0; jb < 4; ++jb) {
          const int p = 32 * ct + 8 * jb + fr;
          bq[jb] = kok ? (kq < nb ? Wr[(size_t)p * kLdv + kq] : Vr[(size_t)p * kLdv + kq - nb]) : 0.0;
        }
#pragma unroll
        for (int i2 = 0; i2 < 2; ++i2)
#pragma unroll
          for (int jb = 0; jb < 4; ++jb) nys::dmma(acc[i2][jb][0], acc[i2][jb][1], a[i2], bq[jb]);
      }
    }
    if (k0 + nb + 2 < n) emit_col(dcc_pos(k0 + nb));   // the next panel's first column
    // every CTA is done with this panel's V, W before the next panel's pushes
    __syncthreads();
    xbegin(X, 8u * kNC);
    if (tid == 0) xpush(X, &S.slotD[rk], 0.0);
    xwait(X);
    DCC_TT(7);
  }
#undef DCC_TT
  if (debug && rk == 0 && tid == 0)
    printf("[nys dcc] tridiag: col %lld xA %lld refl %lld mv+p %lld xB %lld w %lld xP %lld trail+xD %lld\n",
           tt_[0], tt_[1], tt_[2], tt_[3], tt_[4], tt_[5], tt_[6], tt_[7]);
  // last 2 x 2 block from the register tiles
  xbegin(X, 3 * 8);
#pragma unroll
  for (int i2 = 0; i2 < 2; ++i2)
#pragma unroll
    for (int jb = 0; jb < 4; ++jb)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int lr = 16 * rt + 8 * i2 + fr, i = rk + kNC * lr;
        const int c = dcc_ipos(32 * ct + 8 * jb + 2 * fc + h);
        if (lr >= nloc) continue;
        if (i == n - 2 && c == n - 2) xpush(X, &S.d[n - 2], acc[i2][jb][h]);
        if (i == n - 1 && c == n - 1) xpush(X, &S.d[n - 1], acc[i2][jb][h]);
        if (i == n - 1 && c == n - 2) xpush(X, &S.e[n - 2], acc[i2][jb][h]);
      }
  if (tid == 0) S.e[n - 1] = 0.0;
  xwait(X);
  __syncthreads();
  tc1 = clock64();

  // ---------------- divide and conquer; Q by row slabs [r0, r1)
  const int R = ((n + kNC - 1) / kNC + kCLeaf - 1) / kCLeaf * kCLeaf;
  const int r0 = rk * R, r1 = min(n, r0 + R), nr = max(0, r1 - r0);
  const int ldq = n + 1;
  double* Qs = dyn;                     // R x ldq (aliases A, V, W: done with them)
  double* Qn = dyn + (size_t)R * ldq;
  if (tid == 0)
    for (int b = kCLeaf; b < n; b += kCLeaf) {
      const double rho = S.e[b - 1];
      S.d[b - 1] -= rho;
      S.d[b] -= rho;
    }
  for (int e = tid; e < R * ldq; e += nt) Qs[e] = 0.0;
  __syncthreads();
  xbegin(X, 8u * (uint32_t)n);   // every row's leaf eigenvalue
  for (int lf = warp; lf * kCLeaf < nr; lf += kCWarps) {
    const int s = r0 + lf * kCLeaf;
    leaf_ql_c(S, Qs + (size_t)(s - r0) * ldq, ldq, s, min(kCLeaf, n - s), lane);
  }
  __syncthreads();
  for (int i = r0 + tid; i < r1; i += nt) xpush(X, &S.lam[i], S.lam[i]);
  xwait(X);
  __syncthreads();
  tc2 = clock64();

  long long tm[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tlast = clock64();
#define DCC_T(k)                                                                   \
  if (debug) {                                                                     \
    const long long tn = clock64();                                                \
    tm[k] += tn - tlast;                                                           \
    tlast = tn;                                                                    \
  }
  constexpr int G = 16;   // lanes per root / entry / column in the split steps
  const int gl = tid % G;
  const unsigned gm = 0xFFFFu << ((tid & 31) & ~(G - 1));
  for (int width = kCLeaf; width < n; width *= 2) {
    const int nmerge = (n + 2 * width - 1) / (2 * width);
    for (int b = tid; b < nmerge; b += nt) {
      const int s = b * 2 * width;
      S.bs[b] = s;
      S.bmid[b] = min(s + width, n);
      S.be[b] = min(s + 2 * width, n);
      const double rho = S.bmid[b] < S.be[b] ? S.e[S.bmid[b] - 1] : 0.0;
      S.sgn[b] = rho < 0.0 ? -1.0 : 1.0;
    }
    for (int e = tid; e < R * ldq; e += nt) Qn[e] = 0.0;
    __syncthreads();
    {
      int zb = 0;
      for (int b = 0; b < nmerge; ++b) zb += S.bmid[b] < S.be[b] ? S.be[b] - S.bs[b] : 0;
      xbegin(X, 8u * (uint32_t)zb);
    }
    // z = (last row of Q1, first row of Q2), pushed by the owners of those rows
    for (int c = tid; c < n; c += nt) {
      const int b = c / (2 * width);
      const int mid = S.bmid[b], end = S.be[b];
      if (mid >= end) continue;
      const int row = c < mid ? mid - 1 : mid;
      if (row >= r0 && row < r1) xpush(X, &S.zraw[c], Qs[(size_t)(row - r0) * ldq + c]);
    }
    xwait(X);
    __syncthreads();
    DCC_T(0);
    // M1: rank-sort the (sign-adjusted) eigenvalues of both children (redundant)
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
        S.zs[s + rank] = S.zraw[s + c];
      }
    }
    __syncthreads();
    DCC_T(1);
    // M2: normalise, deflate (redundant in every CTA; eig_dc.cu M2's decisions).
    // One warp per block: the norms and the type-1 tests (|rho z_i| <= tol) are
    // lane-parallel, the close-pair Givens test is evaluated speculatively for
    // every pair of consecutive surviving entries with their original values, and
    // lane 0 walks the entries in order, recomputing a pair only when its left
    // entry was itself just rotated (the sequential dependence of dlaed2).
    for (int b = warp; b < nmerge; b += kCWarps) {
      const int s = S.bs[b], mid = S.bmid[b], end = S.be[b], N = end - s;
      if (mid >= end) continue;
      double zn2 = 0.0, dmax = 0.0;
      for (int i = lane; i < N; i += 32) {
        zn2 = fma(S.zs[s + i], S.zs[s + i], zn2);
        dmax = fmax(dmax, fabs(S.ds[s + i]));
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        zn2 += __shfl_xor_sync(0xffffffffu, zn2, o);
        dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
      }
      const double rho = fabs(S.e[mid - 1]) * zn2;
      const double inv = zn2 > 0.0 ? 1.0 / sqrt(zn2) : 0.0;
      const double tol = 8.0 * kEpsC * fmax(dmax, rho);
      int* keep = S.keep + s;
      int* srot = S.col + s;                       // scratch: speculative verdicts
      double *sc = S.hv + s, *ssn = S.hp + s, *sr = S.zraw + s;
      // surviving (not type-1) entries as a bit mask, 8 words for N <= 256
      unsigned surv[kCMaxN / 32];
#pragma unroll
      for (int wd = 0; wd < kCMaxN / 32; ++wd) {
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
    DCC_T(2);
    int total = 0;
    for (int b = 0; b < nmerge; ++b) total += (S.bmid[b] < S.be[b]) ? S.K[b] : 0;
    const int gstride = kNC * (nt / G);
    xbegin(X, 12u * (uint32_t)total);
    // M3: secular roots, split over the cluster, (pole, offset) pushed to all
    for (int w = rk + kNC * (tid / G); w < total; w += gstride) {
      int j = w;
      const int b = find_block(S, nmerge, j);
      const int s = S.bs[b];
      int org;
      double tau;
      secular_root_c(S, s, j, S.K[b], S.rho[b], gl, G, gm, org, tau);
      if (gl == 0) {
        xpush(X, &S.org[s + j], org);
        xpush(X, &S.tau[s + j], tau);
      }
    }
    xwait(X);
    __syncthreads();
    xbegin(X, 8u * (uint32_t)total);
    DCC_T(3);
    // M4: Gu-Eisenstat z over the kept entries, split over the cluster
    for (int w = rk + kNC * (tid / G); w < total; w += gstride) {
      int i = w;
      const int b = find_block(S, nmerge, i);
      const int s = S.bs[b], K = S.K[b];
      const double rho = S.rho[b];
      const double di = S.ds[s + S.keep[s + i]];
      double v0 = gl == 0 ? -dl_of(S, s, i, K - 1) / rho : 1.0, v1 = 1.0;
      int t = 0;
      for (int jj = gl; jj < K - 1; jj += G, ++t) {
        const double dj = jj < i ? S.ds[s + S.keep[s + jj]] : S.ds[s + S.keep[s + jj + 1]];
        const double ratio = (-dl_of(S, s, i, jj)) / (dj - di);
        if (t & 1)
          v1 *= ratio;
        else
          v0 *= ratio;
      }
      double vv = v0 * v1;
      for (int o = 1; o < G; o <<= 1) vv *= __shfl_xor_sync(gm, vv, o);
      if (gl == 0) xpush(X, &S.hv[s + i], copysign(sqrt(fmax(vv, 0.0)), S.zs[s + S.keep[s + i]]));
    }
    xwait(X);
    __syncthreads();
    xbegin(X, 8u * (uint32_t)total);
    DCC_T(4);
    // M5: 1 / ||U[:, j]||, U_ij = zhat_i / (d_i - lambda_j), split over the cluster
    for (int w = rk + kNC * (tid / G); w < total; w += gstride) {
      int j = w;
      const int b = find_block(S, nmerge, j);
      const int s = S.bs[b], K = S.K[b];
      double nrm = 0.0;
      for (int i = gl; i < K; i += G) {
        const double u = S.hv[s + i] / dl_of(S, s, i, j);
        nrm = fma(u, u, nrm);
      }
      nrm = gsum_c(nrm, G, gm);
      if (gl == 0) xpush(X, &S.hp[s + j], rsqrt(nrm));
    }
    xwait(X);
    __syncthreads();
    DCC_T(5);
    // M6: deflation rotations on the own rows' columns (serial over rotations)
    for (int b = 0; b < nmerge; ++b) {
      const int s = S.bs[b], mid = S.bmid[b], end = S.be[b], N = end - s;
      if (mid >= end) continue;
      for (int c = tid; c < N; c += nt) S.col[s + c] = S.perm[s + S.keep[s + c]];
      const int ra = max(s, r0), rb = min(end, r1);
      for (int r = ra + tid; r < rb; r += nt) {
        double* row = Qs + (size_t)(r - r0) * ldq;
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
    DCC_T(6);
    // M7: own rows of the new eigenvectors: kept columns Q[:, col] U (U from
    // the replicated vectors), deflated columns copied, carried blocks copied
    for (int b = 0; b < nmerge; ++b) {
      const int s = S.bs[b], mid = S.bmid[b], end = S.be[b], N = end - s;
      const int ra = max(s, r0), rb = min(end, r1);
      if (ra >= rb) continue;
      const int nrw = rb - ra;
      if (mid >= end) {
        for (int e = tid; e < nrw * N; e += nt) {
          const int r = ra + e / N, c = s + e % N;
          Qn[(size_t)(r - r0) * ldq + c] = Qs[(size_t)(r - r0) * ldq + c];
        }
        continue;
      }
      const int K = S.K[b];
      if (N >= 64) {
        // warp tile: all own rows of the block (<= 32: 4 fragments) x 8 columns
        const int fr = lane >> 2, fc = lane & 3;
        const int tcols = (K + 7) / 8;
        for (int ct = warp; ct < tcols; ct += kCWarps) {
          const int c0 = ct * 8;
          double acc[4][2];
#pragma unroll
          for (int i2 = 0; i2 < 4; ++i2) acc[i2][0] = acc[i2][1] = 0.0;
          const int cb = c0 + fr;
          for (int k0 = 0; k0 < K; k0 += 4) {
            const int k = k0 + fc;
            const bool kok = k < K;
            const int qc = kok ? S.col[s + k] : 0;
            const double bv = (kok && cb < K) ? S.hv[s + k] / dl_of(S, s, k, cb) : 0.0;
#pragma unroll
            for (int i2 = 0; i2 < 4; ++i2) {
              const int r = ra + 8 * i2 + fr;
              const double av = (kok && r < rb) ? Qs[(size_t)(r - r0) * ldq + qc] : 0.0;
              nys::dmma(acc[i2][0], acc[i2][1], av, bv);
            }
          }
#pragma unroll
          for (int i2 = 0; i2 < 4; ++i2)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int r = ra + 8 * i2 + fr, c = c0 + 2 * fc + h;
              if (r < rb && c < K) Qn[(size_t)(r - r0) * ldq + s + c] = acc[i2][h] * S.hp[s + c];
            }
        }
      } else {
        for (int e = tid; e < nrw * K; e += nt) {
          const int r = ra + e / K, c = e % K;
          const double* qrow = Qs + (size_t)(r - r0) * ldq;
          double a = 0.0;
          for (int k = 0; k < K; ++k) a = fma(qrow[S.col[s + k]], S.hv[s + k] / dl_of(S, s, k, c), a);
          Qn[(size_t)(r - r0) * ldq + s + c] = a * S.hp[s + c];
        }
      }
      for (int e = tid; e < nrw * (N - K); e += nt) {
        const int r = ra + e / (N - K), c = K + e % (N - K);
        Qn[(size_t)(r - r0) * ldq + s + c] = Qs[(size_t)(r - r0) * ldq + S.perm[s + S.keep[s + c]]];
      }
    }
    __syncthreads();
    for (int b = 0; b < nmerge; ++b) {
      const int s = S.bs[b], mid = S.bmid[b], end = S.be[b], N = end - s;
      if (mid >= end) continue;
      const int K = S.K[b];
      const double sg = S.sgn[b];
      for (int c = tid; c < N; c += nt) {
        const double l = c < K ? S.ds[s + S.keep[s + S.org[s + c]]] + S.tau[s + c]
                               : S.ds[s + S.keep[s + c]];
        S.lam[s + c] = sg * l;
      }
    }
    double* tq = Qs;
    Qs = Qn;
    Qn = tq;
    __syncthreads();
    DCC_T(7);
  }
#undef DCC_T
  tc3 = clock64();
  // Q (own rows) to the first Q slot of the global buffer; lam, beta, flags
  double* gQ = gbuf + (size_t)n * ld;
  for (int e = tid; e < nr * n; e += nt) {
    const int r = r0 + e / n, c = e % n;
    gQ[(size_t)r * n + c] = Qs[(size_t)(r - r0) * ldq + c];
  }
  if (rk == 0) {
    for (int i = tid; i < n; i += nt) {
      tail[i] = S.lam[i];
      tail[n + i] = S.beta[i];
    }
    if (tid == 0) {
      reinterpret_cast<int*>(tail + 2 * n)[0] = 0;
      reinterpret_cast<int*>(tail + 2 * n)[1] = 0;
    }
  }
  if (debug && rk == 0 && tid == 0) {
    printf("[nys dcc] merge phases: z %lld M1 %lld M2 %lld M3 %lld M4 %lld M5 %lld M6 %lld M7+ %lld\n",
           tm[0], tm[1], tm[2], tm[3], tm[4], tm[5], tm[6], tm[7]);
    printf("[nys dcc] n=%d tridiag=%lld leaves=%lld merges=%lld\n", n, tc1 - tc0, tc2 - tc1,
           tc3 - tc2);
  }
  cl.sync();
}

}  // namespace

namespace nys_host {
bool dcc_fits(int n) { return n > 2 * kCLeaf && n <= kCMaxN; }

int launch_dcc_eig(const double* lm, const double* Ain, int n, double sigma2, double* gbuf,
                   int debug, cudaStream_t st) {
  const int ld = dcc_ld(n);
  const int R = ((n + kNC - 1) / kNC + kCLeaf - 1) / kCLeaf * kCLeaf;
  const size_t tri = 2 * (size_t)kCMaxN * kLdv;
  const size_t dc = 2 * (size_t)R * (n + 1);
  const size_t dyn = (tri > dc ? tri : dc) * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(dcc_eig_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)dyn);
  if (e != cudaSuccess) return record_cuda(e);
  dcc_eig_kernel<<<kNC, kCThreads, dyn, st>>>(lm, Ain, n, sigma2, gbuf, debug);
  count_launches(1);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}
}  // namespace nys_host
