// Fused feature + Gram for ONE linear ODE with many landmarks (m_eff + 2 > 72,
// config 4: m = 256, n_c = 4,194,303).
//
// Operand.  For a well-conditioned landmark matrix (host checks
// s_max / s_min(kept) <= 1e6) the Gram is accumulated in KERNEL space,
//     K = [G g r]^T [G g r],   G_i(s) = [P_p(d) - sum_k f_k P_{p-k}(d)] e^{-d^2/sigma2},
// and projected once at the end, E = W_ext^T K W_ext.  SURVEY.md §0/A1: this
// reassociation costs 1.3e-13 on the config-4 shape (cond(Omega) = 28) but up
// to 2.6e-5 when m_eff < m, hence the host-side gate.  The n x m matrices
// never exist outside a 32-row shared-memory tile.
//
// Exact underflow skipping.  exp(-d^2/sigma2) is exactly 0.0 in IEEE double
// once d^2/sigma2 > 745.14 (below 2^-1075); the kernel treats a landmark block
// as dead for a set of rows when every (row, landmark) pair has
// d^2/sigma2 > 747 (the margin absorbs the rounding of d, d^2 and the
// quotient).  Dead entries are the exact zeros the reference computes, so
// skipping their generation and their DMMAs leaves every sum bit-identical.
// On config 4 (landmarks 0.39 apart, sigma 0.5) a 32-row tile sees ~11 of the
// 33 column blocks, a CTA's row range ~12.
//
// Work split.  One CTA per SM (12 warps), each owning a contiguous row range.
// At start the CTA finds the blocks live anywhere in its range (its "window"),
// compacts them, and tiles the compacted Gram triangle with 4 x 4 super-tiles
// of 8x8 DMMA accumulators (64 registers per warp).  Few super-tiles (config
// 4: 6) are replicated over the 12 warps, each replica taking every R-th
// k-step; many (dense windows) run in several passes over the row range.
// Per 32-row tile the fragment-native smem layout X[ks][c][lane] (c = compacted
// live-block index, so every super-tile reads contiguous fragments) is double
// buffered: iteration t issues the DMMAs of tile t and then generates tile t+1
// (every warp in that order: with three warps per sub-partition issuing DMMAs
// the FP64 pipe is saturated for the whole DMMA phase, ~2100-2400 cycles per
// tile for 132 DMMAs per sub-partition, and the generation that follows runs
// uncontended, ~950 cycles; a warp that generates while its two neighbours
// stream DMMAs gets one FP64 issue per ~32 cycles and needs ~2250); row coefficients are
// produced two tiles ahead (raw row data loaded three ahead).  Every block
// pattern of a super-tile (4 x 4, diagonal i <= j, the ragged 4 x n / n x n edge
// tiles) has its own unpredicated k-step loop, chosen once per pass (a
// predicated mma.sync costs a WARPSYNC + NOP in SASS and its predicated-off
// slots still occupy the pipe).  Each CTA writes its live
// block pairs to a private dense slab (replicas added in fixed order) and one
// reduce kernel sums the slabs in fixed order (deterministic).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"

namespace {

constexpr int kRT = 4;             // super-tile edge (blocks)
#ifndef NYS_LARGE_WARPS
#define NYS_LARGE_WARPS 12
#endif
constexpr int kWarps = NYS_LARGE_WARPS;   // warps per CTA (1 CTA / SM; 12: 3 per SMSP, 168 registers)
constexpr int kTileKs = 8;         // 4-row k-steps per row tile (32 rows)
constexpr int kRowStride = 10;     // doubles per row-coefficient record (conflict-free, 16 B aligned)
constexpr int kMaxSmem = 227 * 1024;
constexpr double kDeadRatio = 747.0;   // d^2 / sigma2 beyond which exp() is exactly 0

struct LargePlan {
  int Pe, NB, NBpad, ld, nrr, ntiles, tiles_per_cta, nbuf;
  size_t smem;
  static LargePlan make(int n_rows, int m, int max_ctas = 0) {
    LargePlan L{};
    L.Pe = m + 2;                                 // kernel-space extended width
    L.NB = (L.Pe + 7) / 8;
    L.NBpad = ((L.NB + kRT - 1) / kRT) * kRT;
    L.ld = L.NB * 8;
    L.ntiles = (n_rows + 4 * kTileKs - 1) / (4 * kTileKs);
    int nrr = nys::device_sm_count();
    if (max_ctas > 0 && nrr > max_ctas) nrr = max_ctas;   // leave SMs to a concurrent kernel
    if (nrr > L.ntiles) nrr = L.ntiles > 0 ? L.ntiles : 1;
    L.nrr = nrr;
    L.tiles_per_cta = (L.ntiles + nrr - 1) / nrr;
    const size_t xbuf = (size_t)kTileKs * L.NBpad * 32 * sizeof(double);
    const size_t rowc = 3 * 32 * kRowStride * sizeof(double);
    L.nbuf = (2 * xbuf + rowc <= (size_t)kMaxSmem) ? 2 : 1;
    L.smem = L.nbuf * xbuf + rowc;
    return L;
  }
  bool fits() const { return NB <= 64 && smem <= (size_t)kMaxSmem; }
  size_t slab_doubles() const { return (size_t)nrr * ld * ld; }
  size_t ws_bytes(int m_eff) const {
    return (slab_doubles() + (size_t)Pe * Pe + (size_t)Pe * (m_eff + 2)) * sizeof(double) +
           (size_t)nrr * sizeof(unsigned long long) + 512;
  }
};

// live-block test for rows spanning [tmin, tmax] (NaN rows: everything live)
NYS_DEV unsigned long long live_blocks(const double* blo, const double* bhi, int NB,
                                       unsigned long long special, double tmin, double tmax,
                                       bool any_nan, double R2) {
  const int lane = threadIdx.x & 31;
  unsigned long long mk = 0ull;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int blk = lane + 32 * h;
    bool live = false;
    if (blk < NB) {
      const double dmin = fmax(blo[blk] - tmax, tmin - bhi[blk]);
      live = any_nan || ((special >> blk) & 1ull) || !(dmin > 0.0 && dmin * dmin > R2);
    }
    mk |= (unsigned long long)__ballot_sync(0xffffffffu, live) << (32 * h);
  }
  return mk;
}

// Exp-recurrence range check (coarse grids).  Between two anchors a lane forms
// rho_A^j for j < kRecSpan rows 4h apart, rho_A = exp((2 H d_A - H^2) / sigma2):
// with |d| up to the distance from the CTA's rows to the far edge of its live
// window that power must stay far from overflow (an underflowed e_A times an
// infinite rho_A^j is NaN; n = 300 rows over the config-4 landmarks, h / sigma =
// 0.67, produced exactly that).  Such ranges take the exp()-per-entry path.
constexpr int kRecSpan = 4 * 8;   // kAnchorTiles * kTileKs (static_assert below)
NYS_DEV bool rec_span_ok(const double* blo, const double* bhi, int m, unsigned long long live,
                         double tmin, double tmax, double hstep, double inv) {
  // live blocks that hold landmarks: the lowest and the highest bound the window
  const int nlb = (m + 7) / 8;
  const unsigned long long lmk = nlb >= 64 ? live : live & ((1ull << nlb) - 1ull);
  double dwin = 0.0;
  if (lmk != 0ull)
    dwin = fmax(fabs(bhi[63 - __clzll((long long)lmk)] - tmin),
                fabs(tmax - blo[__ffsll((long long)lmk) - 1]));
  const double H = 4.0 * hstep;
  return fma(2.0 * H, dwin, H * H) * inv * (double)kRecSpan < 600.0;
}

// per-row polynomial coefficients for one 32-row tile: t, q0..qP, g = -f_p, r
// (one warp; rows past the end get an all-zero polynomial -> G = 0).  The raw
// row data are loaded a tile ahead (RowRaw in registers) so the global-load
// latency overlaps a whole tile of DMMA work.
template <int P>
struct RowRaw {
  double t, f[P], r;
  bool ok;
};

template <int P>
NYS_DEV void row_load(const double* __restrict__ pts, const double* __restrict__ coef,
                      const double* __restrict__ forcing, int n_c, int r0, int row_end,
                      RowRaw<P>& w) {
  const int i = r0 + (threadIdx.x & 31);
  w.ok = i < row_end;
#pragma unroll
  for (int k = 0; k < P; ++k) w.f[k] = w.ok ? coef[(size_t)k * n_c + i] : 0.0;
  w.t = w.ok ? pts[i] : 0.0;
  w.r = w.ok ? forcing[i] : 0.0;
}

// qscale (exp-recurrence tiles only): per-k-step factor Q^{j(j-1)/2} folded
// into the row's polynomial, so the generator multiplies it once per row here
// instead of once per (row, landmark) entry
template <int P>
NYS_DEV void row_store(const double (*hc)[nys::kMaxOrder + 1], const RowRaw<P>& w, double* rowc,
                       const double* qscale = nullptr) {
  double* rc = rowc + (threadIdx.x & 31) * kRowStride;
  const double qs = qscale != nullptr ? qscale[(threadIdx.x & 31) >> 2] : 1.0;
  rc[0] = w.t;
#pragma unroll
  for (int j = 0; j <= P; ++j) {
    double v = hc[P][j];
#pragma unroll
    for (int k = 1; k <= P; ++k) v = fma(-w.f[k - 1], hc[P - k][j], v);
    rc[1 + j] = w.ok ? (qscale != nullptr ? v * qs : v) : 0.0;
  }
  rc[6] = w.ok ? -w.f[P - 1] : 0.0;
  rc[7] = w.r;
}

// -(x / sigma2) for x >= 0, correctly rounded from the precomputed reciprocal:
// q = x * inv, remainder by FMA, one correction (bit-identical to the IEEE
// quotient on 13 bandwidths x 2^32 samples, tools/div_check.cu) -- the
// kernel.py:78-79 division at 3 FP64 ops.
NYS_DEV double neg_div(double x, double sigma2, double inv) {
  double q = x * inv;
  double r = fma(-q, sigma2, x);
  return -fma(r, inv, q);
}

template <int P>
NYS_DEV double g_entry(double l, const double* r, double sigma2, double inv) {
  const double d = l - r[0];
  double poly = r[1 + P];
#pragma unroll
  for (int j = P - 1; j >= 0; --j) poly = fma(poly, d, r[1 + j]);
  return poly * exp(neg_div(d * d, sigma2, inv));
}

// Generate the CTA's L live blocks of one 32-row tile into the compacted
// fragment layout X[ks][c][lane] (c = compacted block index).  Work unit =
// (block, k-step pair): two independent exp chains per lane.
template <int P>
NYS_DEV void gen_tile(const double* __restrict__ lm, int m, int L, const int* lb, int NBpad,
                      double sigma2, double inv, const double* rowc, double* X, int warp,
                      int nwarps) {   // (all warps share the 4 L units)
  const int lane = threadIdx.x & 31;
  const int rsub = lane & 3, csub = lane >> 2;
  for (int u = warp; u < 4 * L; u += nwarps) {
    const int c = u >> 2, ks = (u & 3) * 2;
    const int s = lb[c] * 8 + csub;
    double* Xo = X + ((size_t)ks * NBpad + c) * 32 + lane;
    const double* r0 = rowc + (ks * 4 + rsub) * kRowStride;   // rows ks*4 + rsub and +4
    const double* r1 = r0 + 4 * kRowStride;
    double v0, v1;
    if (s < m) {
      const double l = __ldg(lm + s);
      v0 = g_entry<P>(l, r0, sigma2, inv);
      v1 = g_entry<P>(l, r1, sigma2, inv);
    } else {
      v0 = (s == m) ? r0[6] : (s == m + 1) ? r0[7] : 0.0;
      v1 = (s == m) ? r1[6] : (s == m + 1) ? r1[7] : 0.0;
    }
    Xo[0] = v0;
    Xo[(size_t)NBpad * 32] = v1;
  }
}

// Uniform grids (t_i = t_0 + i h to 8 ulp, checked per CTA at start): the
// generating warp of a compacted block keeps, per lane (row residue rsub,
// landmark 8 lb[c] + csub), an anchor at row A and forms the rows A + jH
// (H = 4h, j < 32) as
//     e_j = e_A rho_A^j Q^{j(j-1)/2},
//     e_A = exp(-d_A^2 / sigma2),  rho_A = exp((2 H d_A - H^2) / sigma2),
//     Q = exp(-2 H^2 / sigma2)
// (e(t + H) = e(t) rho(t), rho(t + H) = rho(t) Q).  rho_A^{8u} is carried from
// tile to tile, rho_A^i (i <= 8) comes from a depth-3 product tree and
// Q^{j(j-1)/2} from a per-CTA table, so the eight entries of a lane are
// independent (no serial DMUL chain: the FP64 datapath is shared with the
// DMMAs of the other warps, which makes a dependent chain slow).  Two exp()
// per lane every kAnchorTiles tiles, computed one tile early.  Error: <= ~20
// roundings per entry (~2e-15 relative) plus the anchor's ideal-vs-actual grid
// position (<= 8 ulp(t): <= 2|d| dt / sigma2 relative, < 1e-12 wherever an
// entry exceeds 1e-17).  The Hermite factor P(d) uses the exact d of every row.
// Stores are lane-contiguous (X[ks][c][lane]).
constexpr int kAnchorTiles = 4;
static_assert(kRecSpan == kAnchorTiles * kTileKs, "rec_span_ok covers one anchor period");
constexpr int kGenMax = 2;      // blocks one warp generates (register state)

#ifndef NYS_LARGE_PROBE
#define NYS_LARGE_PROBE 0   // probe builds: 1 = skip DMMA, 2 = skip generation, 3 = phase clocks
#endif
#ifndef NYS_LARGE_REC
#define NYS_LARGE_REC 1     // 0: exp() per entry on uniform grids too (A/B builds)
#endif

template <int P>
__global__ void __launch_bounds__(kWarps * 32, 1)
    large_kspace_kernel(const double* __restrict__ lm, int m, double sigma2,
                        const double* __restrict__ pts, const double* __restrict__ coef,
                        const double* __restrict__ forcing, int n_c, int row_begin, int row_end,
                        int NB, int NBpad, int ld, int nbuf, int tiles_per_cta,
                        double* __restrict__ slabs, unsigned long long* __restrict__ live_out,
                        int min_L) {
  extern __shared__ __align__(16) double sm[];
  const size_t xsz = (size_t)kTileKs * NBpad * 32;
  double* const X0 = sm;
  double* const X1 = sm + (nbuf - 1) * xsz;
  double* const rowc = sm + nbuf * xsz;   // [3][32][kRowStride]
  __shared__ double blo_s[64], bhi_s[64];
  __shared__ double red_s[3][kWarps];
  __shared__ int nan_s;
  __shared__ double hstep_s, hstep_ta_s;
  __shared__ unsigned long long live_s;
  __shared__ int rec_ok_s;
  __shared__ int lb_s[64];
  __shared__ double hc_s[nys::kMaxOrder + 1][nys::kMaxOrder + 1];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  const int ntiles = (row_end - row_begin + 31) / 32;
  const int tile0 = blockIdx.x * tiles_per_cta;
  const int tile1 = min(ntiles, tile0 + tiles_per_cta);
  const double inv = 1.0 / sigma2;
  const unsigned long long special = (1ull << (m / 8)) | (1ull << ((m + 1) / 8));

  // ---- Hermite coefficients (kernel.py:26-37) and landmark bounds per block
  if (threadIdx.x == 0) {
    nan_s = 0;
    nys::Hermite H;
    H.init(sigma2, P);
    for (int a = 0; a <= nys::kMaxOrder; ++a)
      for (int j = 0; j <= nys::kMaxOrder; ++j) hc_s[a][j] = H.c[a][j];
  }
  if (warp == 1) {
    for (int blk = lane; blk < NB; blk += 32) {
      double lo = INFINITY, hi = -INFINITY;
      for (int s = blk * 8; s < min(blk * 8 + 8, m); ++s) {
        lo = fmin(lo, lm[s]);
        hi = fmax(hi, lm[s]);
      }
      blo_s[blk] = lo;
      bhi_s[blk] = hi;
    }
  }
  __syncthreads();
  // ---- t-range of the CTA's rows -> its window of live blocks
  {
    double tmin = INFINITY, tmax = -INFINITY, dev = 0.0;
    bool bad = false;
    const int r_lo = row_begin + tile0 * 32, r_hi = min(row_end, row_begin + tile1 * 32);
    // uniform-grid test against the chord of the range (NaN fails it)
    const double ta = r_hi > r_lo ? pts[r_lo] : 0.0, tb = r_hi > r_lo ? pts[r_hi - 1] : 0.0;
    const double h = r_hi - r_lo > 1 ? (tb - ta) / (double)(r_hi - 1 - r_lo) : 0.0;
    for (int i = r_lo + threadIdx.x; i < r_hi; i += blockDim.x) {
      const double t = pts[i];
      tmin = fmin(tmin, t);
      tmax = fmax(tmax, t);
      bad |= t != t;
      dev = fmax(dev, fabs(t - fma((double)(i - r_lo), h, ta)));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      tmin = fmin(tmin, __shfl_xor_sync(0xffffffffu, tmin, o));
      tmax = fmax(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
      dev = fmax(dev, __shfl_xor_sync(0xffffffffu, dev, o));
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) nan_s = 1;
    if (lane == 0) {
      red_s[0][warp] = tmin;
      red_s[1][warp] = tmax;
      red_s[2][warp] = dev;
    }
    if (threadIdx.x == 0) {
      hstep_s = h;
      hstep_ta_s = ta;
    }
  }
  __syncthreads();
  if (warp == 0) {
    double tmin = INFINITY, tmax = -INFINITY, dev = 0.0;
    for (int w = 0; w < nwarps; ++w) {
      tmin = fmin(tmin, red_s[0][w]);
      tmax = fmax(tmax, red_s[1][w]);
      dev = fmax(dev, red_s[2][w]);
    }
    // 8 ulp of the largest |t|; NaN deviations fail the test
    const double tol = 8.0 * 2.220446049250313e-16 * fmax(fabs(tmin), fabs(tmax));
    if (lane == 0 && !(dev <= tol && nan_s == 0 && hstep_s > 0.0)) hstep_s = 0.0;
    const unsigned long long live =
        live_blocks(blo_s, bhi_s, NB, special, tmin, tmax, nan_s != 0, kDeadRatio * sigma2);
    for (int h = 0; h < 2; ++h) {   // compact the live blocks in ascending order
      const int blk = lane + 32 * h;
      if ((live >> blk) & 1ull) lb_s[__popcll(live & ((1ull << blk) - 1ull))] = blk;
    }
    if (lane == 0) {
      live_s = live;
      live_out[blockIdx.x] = live;
      rec_ok_s = rec_span_ok(blo_s, bhi_s, m, live, tmin, tmax, hstep_s, inv) ? 1 : 0;
    }
  }
  __syncthreads();
  const int L = __popcll(live_s);
  if (L < min_L) return;   // large_ws_kernel covered this range
  const int T = (L + kRT - 1) / kRT;
  const int ntask = T * (T + 1) / 2;
  __shared__ signed char wtask_s[kWarps], wrep_s[kWarps], wR_s[kWarps], genw_s[64];
  int R = 1, npass = (ntask + nwarps - 1) / nwarps;
  if (ntask <= nwarps) {   // R replicas per super-tile; warp c generates block c
    if (threadIdx.x < 64) {
      const int Ru = min(nwarps / ntask, kTileKs), x = threadIdx.x;
      if (x < nwarps) {
        wtask_s[x] = (signed char)(x < ntask * Ru ? x / Ru : -1);
        wrep_s[x] = (signed char)(x % Ru);
        wR_s[x] = (signed char)Ru;
      }
    }
    __syncthreads();
    if (threadIdx.x < 64) genw_s[threadIdx.x] = (signed char)(threadIdx.x % nwarps);
    __syncthreads();
    R = wR_s[warp];
    npass = 1;
  } else if (threadIdx.x < 64) {
    genw_s[threadIdx.x] = (signed char)(threadIdx.x % nwarps);
  }
  __syncthreads();
  int Rmax = 1;
  for (int x = 0; x < nwarps && npass == 1; ++x) Rmax = max(Rmax, (int)wR_s[x]);
  const int cw = nwarps - 1;   // warp that prepares row coefficients
  RowRaw<P> raw;
  const double H = 4.0 * hstep_s;   // 0: non-uniform grid -> exp() per entry
  const bool rec = H > 0.0 && NYS_LARGE_REC && ntask <= nwarps && L <= kGenMax * nwarps && rec_ok_s;
  // Q^{j(j-1)/2}, j < kAnchorTiles * kTileKs (rows since the anchor)
  __shared__ double qtri_s[kAnchorTiles * kTileKs];
  if (rec && threadIdx.x < kAnchorTiles * kTileKs)
    qtri_s[threadIdx.x] = exp(-H * H * inv * (double)(threadIdx.x * (threadIdx.x - 1)));
  __syncthreads();   // qtri_s is read by the row-record warp (row_store's qscale)
  // Q^{j(j-1)/2} factors of CTA tile kt's k-steps (rec path), else none
  auto qscale = [&](int kt) -> const double* {
    return rec ? qtri_s + (kt % kAnchorTiles) * kTileKs : nullptr;
  };
  // recurrence state of this warp's generated blocks (rec path only): landmark,
  // anchor exponential and ratio, rho_A^{8t}, and the next anchor
  const int rsub = lane & 3, csub = lane >> 2;
  int gc[kGenMax], ng = 0;
  double gl[kGenMax], geA[kGenMax], grA[kGenMax], gP[kGenMax], geN[kGenMax], grN[kGenMax];
#pragma unroll
  for (int g = 0; g < kGenMax; ++g) {
    gc[g] = -1;
    gl[g] = geA[g] = grA[g] = gP[g] = geN[g] = grN[g] = 0.0;
  }
  if (rec) {
    for (int c = 0; c < L; ++c)
      if (genw_s[c] == warp && ng < kGenMax) gc[ng++] = c;
#pragma unroll
    for (int g = 0; g < kGenMax; ++g)
      if (g < ng) {
        const int s = lb_s[gc[g]] * 8 + csub;
        gl[g] = s < m ? __ldg(lm + s) : 0.0;
      }
  }
  const double ta = hstep_ta_s;
  // anchor for the lane's first row of CTA tile kt (ideal grid position)
  auto anchor = [&](int kt) {
    const double t = fma((double)(kt * 32 + rsub), hstep_s, ta);
#pragma unroll
    for (int g = 0; g < kGenMax; ++g)
      if (g < ng) {
        const double d = gl[g] - t;
        geN[g] = exp(neg_div(d * d, sigma2, inv));
        grN[g] = exp(fma(2.0 * H, d, -H * H) * inv);
      }
  };
  // rows j = 8u + i since the anchor: e_j = e_A rho_A^j Q^{j(j-1)/2}, with
  // rho_A^{8u} carried (in base) and base rho_A^i by a depth-3 product tree
  // with base folded in (no serial chain); Q^{j(j-1)/2} is already in the row
  // record's polynomial (row_store's qscale).  11 DMULs per lane and tile for
  // the eight Gaussians (was 25 with the per-entry Q factor and base product).
  auto gen_rec = [&](int kt, const double* rc, double* Xd) {
    const int u = kt % kAnchorTiles;
    if (u == 0) {
#pragma unroll
      for (int g = 0; g < kGenMax; ++g) {
        geA[g] = geN[g];
        grA[g] = grN[g];
        gP[g] = 1.0;
      }
    }
#pragma unroll
    for (int g = 0; g < kGenMax; ++g)
      if (g < ng) {
        const int s = lb_s[gc[g]] * 8 + csub;
        double* Xo = Xd + (size_t)gc[g] * 32 + lane;
        if (s < m) {
          const double r1 = grA[g], r2 = r1 * r1, r4 = r2 * r2;
          double bp[kTileKs];   // base rho_A^ks
          bp[0] = geA[g] * gP[g];
          bp[1] = bp[0] * r1;
          bp[2] = bp[0] * r2;
          bp[4] = bp[0] * r4;
          bp[3] = bp[1] * r2;
          bp[5] = bp[1] * r4;
          bp[6] = bp[2] * r4;
          bp[7] = bp[3] * r4;
#pragma unroll
          for (int ks = 0; ks < kTileKs; ++ks) {
            const double* r = rc + (ks * 4 + rsub) * kRowStride;
            double rv[(P + 3) & ~1];   // t, q_0..q_P by 16-byte loads
#pragma unroll
            for (int j = 0; j < ((P + 3) & ~1); j += 2) {
              const double2 v2 = *reinterpret_cast<const double2*>(r + j);
              rv[j] = v2.x;
              rv[j + 1] = v2.y;
            }
            const double d = gl[g] - rv[0];
            double poly = rv[1 + P];
#pragma unroll
            for (int j = P - 1; j >= 0; --j) poly = fma(poly, d, rv[1 + j]);
            bp[ks] *= poly;
          }
          // all eight entries are formed before the first store: a store into X
          // between the row-record loads would order the eight chains one after
          // the other (the compiler cannot tell X from the row records)
#pragma unroll
          for (int ks = 0; ks < kTileKs; ++ks) Xo[(size_t)ks * NBpad * 32] = bp[ks];
          gP[g] *= r4 * r4;
        } else {
          double v[kTileKs];   // loads first, then the stores (as above)
#pragma unroll
          for (int ks = 0; ks < kTileKs; ++ks) {
            const double* r = rc + (ks * 4 + rsub) * kRowStride;
            v[ks] = (s == m) ? r[6] : (s == m + 1) ? r[7] : 0.0;
          }
#pragma unroll
          for (int ks = 0; ks < kTileKs; ++ks) Xo[(size_t)ks * NBpad * 32] = v[ks];
        }
      }
    if (u == kAnchorTiles - 1) anchor(kt + 1);
  };
  auto gen = [&](int kt, const double* rc, double* Xd) {
    if (rec)
      gen_rec(kt, rc, Xd);
    else
      gen_tile<P>(lm, m, L, lb_s, NBpad, sigma2, inv, rc, Xd, warp, nwarps);
  };
  if (rec) anchor(0);
  double* const slab = slabs + (size_t)blockIdx.x * ld * ld;

  for (int pass = 0; pass < npass; ++pass) {
    // ---- this warp's super-tile (p, q) of the compacted triangle, replica rep
    int task = -1, rep = 0;
    if (npass == 1 && ntask <= nwarps) {
      task = wtask_s[warp];
      rep = wrep_s[warp];
    } else {
      task = pass * nwarps + warp;
      if (task >= ntask) task = -1;
    }
    int p = 0, q = 0;
    uint32_t valid = 0;
    if (task >= 0) {
      int idx = task;
      while (idx >= T - p) {
        idx -= T - p;
        ++p;
      }
      q = p + idx;
#pragma unroll
      for (int i = 0; i < kRT; ++i)
#pragma unroll
        for (int j = 0; j < kRT; ++j)
          if (p * kRT + i < L && q * kRT + j < L && !(p == q && i > j)) valid |= 1u << (i * kRT + j);
    }

    double acc[kRT][kRT][2];
#pragma unroll
    for (int i = 0; i < kRT; ++i)
#pragma unroll
      for (int j = 0; j < kRT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    if (tile0 < tile1) {
      if (warp == cw) {
        row_load<P>(pts, coef, forcing, n_c, row_begin + tile0 * 32, row_end, raw);
        row_store<P>(hc_s, raw, rowc, qscale(0));
        if (tile0 + 1 < tile1) {
          row_load<P>(pts, coef, forcing, n_c, row_begin + (tile0 + 1) * 32, row_end, raw);
          row_store<P>(hc_s, raw, rowc + 32 * kRowStride, qscale(1));
        }
        if (tile0 + 2 < tile1)
          row_load<P>(pts, coef, forcing, n_c, row_begin + (tile0 + 2) * 32, row_end, raw);
      }
      __syncthreads();
      gen(0, rowc, X0);
      __syncthreads();
    }
    // block pattern of the super-tile: only the last super-row / super-column of
    // the compacted window is ragged, so an off-diagonal task is 4 x nj and a
    // diagonal one n x n (i <= j)
    static_assert(kRT == 4, "the pattern table below is written for 4 x 4 super-tiles");
    const int nj = min(kRT, L - q * kRT);
    const int pattern = p == q ? (nj == 4 ? 1 : nj == 3 ? 5 : nj == 2 ? 6 : 7)
                               : (nj == 4 ? 0 : nj == 3 ? 2 : nj == 2 ? 3 : 4);
    const int offa = p * kRT * 32 + lane, offb = q * kRT * 32 + lane;
    for (int tile = tile0; tile < tile1; ++tile) {
      const int k = tile - tile0;
      const double* X = (k & 1) ? X1 : X0;
      double* const Xn = ((k + 1) & 1) ? X1 : X0;
      const double* const rcn = rowc + ((k + 1) % 3) * 32 * kRowStride;
      // DMMAs first, then the next tile's blocks (see the header; the other
      // orders are A/B builds: generation in the shadow of the neighbours' DMMAs
      // is starved of FP64 issue slots)
#ifndef NYS_LARGE_GENFIRST
#define NYS_LARGE_GENFIRST 0   // A/B builds: 0 none (1.78 ms), 1 warps 4-7 (1.89), 2 all (2.01), 3 all but warps 4-7 (1.86)
#endif
      const bool gen_first =
          nbuf == 2 && (NYS_LARGE_GENFIRST == 0   ? false
                        : NYS_LARGE_GENFIRST == 1 ? (bool)((warp >> 2) & 1)
                        : NYS_LARGE_GENFIRST == 2 ? true
                                                  : !((warp >> 2) & 1));
#if NYS_LARGE_PROBE == 3
      long long TT[6];
      TT[0] = clock64();
#define NYS_T(i) TT[i] = clock64()
#else
#define NYS_T(i)
#endif
      if (NYS_LARGE_PROBE != 2 && gen_first && tile + 1 < tile1)
        gen(k + 1, rcn, Xn);
      NYS_T(1);
      if (NYS_LARGE_PROBE != 1 && task >= 0) {
        // one k-step loop per block pattern, chosen once per pass: NI x NJ blocks,
        // DIAG: i <= j only.  Ragged edge super-tiles get their own unpredicated
        // loops too (a predicated mma.sync costs a WARPSYNC + NOP per DMMA in
        // SASS: the (4 x 3)-block task ran at 50 cycles per DMMA and the 3-block
        // diagonal one at 110, against 28 for the complete 4 x 4).
        auto ks_loop = [&](auto ni_c, auto nj_c, auto diag_c) {
          constexpr int NI = decltype(ni_c)::value, NJ = decltype(nj_c)::value;
          constexpr bool DG = decltype(diag_c)::value;
#pragma unroll 1
          for (int ks = rep; ks < kTileKs; ks += R) {
            const double* Xk = X + (size_t)ks * NBpad * 32;
            double xa[NI], xb[NJ];
#pragma unroll
            for (int i = 0; i < NI; ++i) xa[i] = Xk[offa + i * 32];
#pragma unroll
            for (int j = 0; j < NJ; ++j) xb[j] = Xk[offb + j * 32];
#pragma unroll
            for (int i = 0; i < NI; ++i)
#pragma unroll
              for (int j = DG ? i : 0; j < NJ; ++j)
                nys::dmma(acc[i][j][0], acc[i][j][1], xa[i], xb[j]);
          }
        };
        using std::integral_constant;
#define NYS_PAT(NI, NJ, DG) \
  ks_loop(integral_constant<int, NI>{}, integral_constant<int, NJ>{}, integral_constant<bool, DG>{})
        switch (pattern) {
          case 0: NYS_PAT(4, 4, false); break;
          case 1: NYS_PAT(4, 4, true); break;
          case 2: NYS_PAT(4, 3, false); break;
          case 3: NYS_PAT(4, 2, false); break;
          case 4: NYS_PAT(4, 1, false); break;
          case 5: NYS_PAT(3, 3, true); break;
          case 6: NYS_PAT(2, 2, true); break;
          default: NYS_PAT(1, 1, true); break;
        }
#undef NYS_PAT
      }
      NYS_T(2);
      if (nbuf == 1) __syncthreads();
      if (NYS_LARGE_PROBE != 2 && !gen_first && tile + 1 < tile1)
        gen(k + 1, rcn, Xn);
      NYS_T(3);
      if (warp == cw && tile + 2 < tile1) {
        row_store<P>(hc_s, raw, rowc + ((k + 2) % 3) * 32 * kRowStride, qscale(k + 2));
        if (tile + 3 < tile1)
          row_load<P>(pts, coef, forcing, n_c, row_begin + (tile + 3) * 32, row_end, raw);
      }
      NYS_T(4);
      __syncthreads();
#if NYS_LARGE_PROBE == 3
      NYS_T(5);
      if (blockIdx.x == 70 && (k == 20 || k == 21) && lane == 0)
        printf("k=%d w=%2d task=%d rep=%d/%d L=%d | gen1 %6lld dmma %6lld gen2 %6lld rc %6lld "
               "bar %6lld\n",
               k, warp, task, rep, R, L, TT[1] - TT[0], TT[2] - TT[1], TT[3] - TT[2],
               TT[4] - TT[3], TT[5] - TT[4]);
#endif
    }
    // ---- slab write: replicas of one super-tile are added in replica order
    for (int r = 0; r < Rmax; ++r) {
      if (task >= 0 && rep == r) {
#pragma unroll
        for (int i = 0; i < kRT; ++i)
#pragma unroll
          for (int j = 0; j < kRT; ++j)
            if ((valid >> (i * kRT + j)) & 1u) {
              const int I = lb_s[p * kRT + i], J = lb_s[q * kRT + j];
              double* o = slab + (size_t)(I * 8 + (lane >> 2)) * ld + J * 8 + 2 * (lane & 3);
              if (r == 0) {
                o[0] = acc[i][j][0];
                o[1] = acc[i][j][1];
              } else {
                o[0] += acc[i][j][0];
                o[1] += acc[i][j][1];
              }
            }
      }
      __syncthreads();
    }
  }
}

// ---- Warp-specialised kernel-space Gram (live windows of at most kWsMaxL
// blocks, config 4: 11-13).  16 warps, one CTA per SM:
//   * 8 producer warps (two per SM sub-partition) generate the 32-row tiles of
//     the compacted window into a kWsStages-deep shared-memory ring (warp 0 also
//     forms the row coefficients a tile ahead; the eight meet at a named
//     barrier), each warp its own blocks with the recurrence state in registers;
//   * 8 consumer warps own the window's block pairs (I <= J) in equal
//     contiguous chunks of the row-pair order (I / 2, J, I % 2), so consecutive
//     pairs share the B fragment and each row pair's two A fragments: every warp
//     issues the same number of DMMAs per tile (no replicas, no idle warp).
// Stages are handed over by mbarriers (full: 8 producer arrivals, empty: 8
// consumer arrivals): no CTA-wide barrier per tile, so the tensor pipe stays fed
// while the producers run ahead.  Same exact-underflow window and generation
// arithmetic as large_kspace_kernel; each pair is accumulated by one warp in k
// order (no replica split).  A CTA whose window is wider than kWsMaxL leaves its range to
// large_kspace_kernel (launched after this one with min_L = kWsMaxL + 1).
#ifndef NYS_WS_PROBE
#define NYS_WS_PROBE 0   // probe builds: 1 = consumers skip DMMA, 2 = producers skip generation
#endif
constexpr int kWsProd = 8, kWsCons = 8, kWsWarps = kWsProd + kWsCons;
constexpr int kWsStages = 6, kWsMaxL = 14, kWsCols = 8, kWsGen = (kWsMaxL + kWsProd - 1) / kWsProd;

NYS_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(nys::smem_u32(bar)) : "memory");
}

size_t ws_smem_bytes() {   // X ring + per-producer row records (non-uniform grids)
  return ((size_t)kWsStages * kTileKs * kWsMaxL * 32 + kWsProd * 32 * kRowStride) * sizeof(double);
}

// consumer body for a warp owning NC columns (see large_ws_kernel): per k-step
// the A fragments of a row pair are loaded when the row pair changes, one B
// fragment per column, one or two DMMAs
template <int NC>
NYS_DEV void ws_consume(const double* Xr, int nt, uint64_t* full_b, uint64_t* empty_b,
                        const int* offa, const int* offb, const int* Ia, const int* Jb,
                        unsigned newrp, unsigned two, const int* lb_s, double* slab, int ld) {
  constexpr size_t xsz = (size_t)kTileKs * kWsMaxL * 32;
  const int lane = threadIdx.x & 31;
  double acc[NC > 0 ? NC : 1][2][2];
#pragma unroll
  for (int c = 0; c < NC; ++c) acc[c][0][0] = acc[c][0][1] = acc[c][1][0] = acc[c][1][1] = 0.0;
  for (int k = 0; k < nt; ++k) {
    const int st = k % kWsStages;
    nys::mbar_wait(&full_b[st], (k / kWsStages) & 1);
    const double* const Xs = Xr + (size_t)st * xsz + lane;
#pragma unroll 2
    for (int ks = 0; ks < kTileKs; ++ks) {
      const double* Xk = Xs + (size_t)ks * kWsMaxL * 32;
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        if ((newrp >> c) & 1u) {
          a0 = Xk[offa[c]];
          a1 = Xk[offa[c] + 32];
        }
        const double b = Xk[offb[c]];
        if (NYS_WS_PROBE != 1) {
          // both DMMAs unpredicated (a predicated mma.sync costs WARPSYNC + NOP);
          // a single-row column's second accumulator is never stored
          nys::dmma(acc[c][0][0], acc[c][0][1], a0, b);
          nys::dmma(acc[c][1][0], acc[c][1][1], a1, b);
        } else {
          acc[c][0][0] += a0 * b;
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_b[st]);
  }
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int r2 = 0; r2 < 2; ++r2) {
      if (r2 == 1 && !((two >> c) & 1u)) continue;
      const int I = lb_s[Ia[c] + r2], J = lb_s[Jb[c]];
      double* o = slab + (size_t)(I * 8 + (lane >> 2)) * ld + J * 8 + 2 * (lane & 3);
      o[0] = acc[c][r2][0];
      o[1] = acc[c][r2][1];
    }
}

template <int P>
__global__ void __launch_bounds__(kWsWarps * 32, 1)
    large_ws_kernel(const double* __restrict__ lm, int m, double sigma2,
                    const double* __restrict__ pts, const double* __restrict__ coef,
                    const double* __restrict__ forcing, int n_c, int row_begin, int row_end,
                    int NB, int ld, int tiles_per_cta, double* __restrict__ slabs,
                    unsigned long long* __restrict__ live_out) {
  extern __shared__ __align__(16) double sm[];
  constexpr size_t xsz = (size_t)kTileKs * kWsMaxL * 32;
  double* const Xr = sm;                              // [stage][ks][c][lane]
  double* const rowr = sm + kWsStages * xsz;          // [producer][32][kRowStride]
  __shared__ double blo_s[64], bhi_s[64];
  __shared__ double red_s[3][kWsWarps];
  __shared__ int nan_s;
  __shared__ double hstep_s, hstep_ta_s;
  __shared__ unsigned long long live_s;
  __shared__ int lb_s[64];
  __shared__ double hc_s[nys::kMaxOrder + 1][nys::kMaxOrder + 1];
  __shared__ double qtri_s[kAnchorTiles * kTileKs];
  __shared__ __align__(8) uint64_t full_b[kWsStages], empty_b[kWsStages];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = kWsWarps;
  const int ntiles = (row_end - row_begin + 31) / 32;
  const int tile0 = blockIdx.x * tiles_per_cta;
  const int tile1 = min(ntiles, tile0 + tiles_per_cta);
  const int nt = max(0, tile1 - tile0);
  const double inv = 1.0 / sigma2;
  const unsigned long long special = (1ull << (m / 8)) | (1ull << ((m + 1) / 8));

  // ---- prologue: as large_kspace_kernel (Hermite coefficients, window, grid test)
  if (threadIdx.x == 0) {
    nan_s = 0;
    nys::Hermite H;
    H.init(sigma2, P);
    for (int a = 0; a <= nys::kMaxOrder; ++a)
      for (int j = 0; j <= nys::kMaxOrder; ++j) hc_s[a][j] = H.c[a][j];
    for (int s = 0; s < kWsStages; ++s) {
      nys::mbar_init(&full_b[s], kWsProd);
      nys::mbar_init(&empty_b[s], kWsCons);
    }
  }
  if (warp == 1) {
    for (int blk = lane; blk < NB; blk += 32) {
      double lo = INFINITY, hi = -INFINITY;
      for (int s = blk * 8; s < min(blk * 8 + 8, m); ++s) {
        lo = fmin(lo, lm[s]);
        hi = fmax(hi, lm[s]);
      }
      blo_s[blk] = lo;
      bhi_s[blk] = hi;
    }
  }
  __syncthreads();
  {
    double tmin = INFINITY, tmax = -INFINITY, dev = 0.0;
    bool bad = false;
    const int r_lo = row_begin + tile0 * 32, r_hi = min(row_end, row_begin + tile1 * 32);
    const double ta = r_hi > r_lo ? pts[r_lo] : 0.0, tb = r_hi > r_lo ? pts[r_hi - 1] : 0.0;
    const double h = r_hi - r_lo > 1 ? (tb - ta) / (double)(r_hi - 1 - r_lo) : 0.0;
    for (int i = r_lo + threadIdx.x; i < r_hi; i += blockDim.x) {
      const double t = pts[i];
      tmin = fmin(tmin, t);
      tmax = fmax(tmax, t);
      bad |= t != t;
      dev = fmax(dev, fabs(t - fma((double)(i - r_lo), h, ta)));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      tmin = fmin(tmin, __shfl_xor_sync(0xffffffffu, tmin, o));
      tmax = fmax(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
      dev = fmax(dev, __shfl_xor_sync(0xffffffffu, dev, o));
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) nan_s = 1;
    if (lane == 0) {
      red_s[0][warp] = tmin;
      red_s[1][warp] = tmax;
      red_s[2][warp] = dev;
    }
    if (threadIdx.x == 0) {
      hstep_s = h;
      hstep_ta_s = ta;
    }
  }
  __syncthreads();
  if (warp == 0) {
    double tmin = INFINITY, tmax = -INFINITY, dev = 0.0;
    for (int w = 0; w < nwarps; ++w) {
      tmin = fmin(tmin, red_s[0][w]);
      tmax = fmax(tmax, red_s[1][w]);
      dev = fmax(dev, red_s[2][w]);
    }
    const double tol = 8.0 * 2.220446049250313e-16 * fmax(fabs(tmin), fabs(tmax));
    if (lane == 0 && !(dev <= tol && nan_s == 0 && hstep_s > 0.0)) hstep_s = 0.0;
    const unsigned long long live =
        live_blocks(blo_s, bhi_s, NB, special, tmin, tmax, nan_s != 0, kDeadRatio * sigma2);
    for (int h = 0; h < 2; ++h) {
      const int blk = lane + 32 * h;
      if ((live >> blk) & 1ull) lb_s[__popcll(live & ((1ull << blk) - 1ull))] = blk;
    }
    if (lane == 0) {
      live_s = live;
      live_out[blockIdx.x] = live;
      if (!rec_span_ok(blo_s, bhi_s, m, live, tmin, tmax, hstep_s, inv)) hstep_s = 0.0;
    }
  }
  __syncthreads();
  const int L = __popcll(live_s);
  if (L > kWsMaxL) return;   // large_kspace_kernel (min_L) covers this range
  const double H = 4.0 * hstep_s;
  const bool rec = H > 0.0 && NYS_LARGE_REC;
  if (rec && threadIdx.x < kAnchorTiles * kTileKs)
    qtri_s[threadIdx.x] = exp(-H * H * inv * (double)(threadIdx.x * (threadIdx.x - 1)));
  __syncthreads();
  double* const slab = slabs + (size_t)blockIdx.x * ld * ld;
  const int rsub = lane & 3, csub = lane >> 2;

  if (warp < kWsProd) {
    // ================= producers
    const int pw = warp;
    int gc[kWsGen], ng = 0;
    double gl[kWsGen], geA[kWsGen], grA[kWsGen], gP[kWsGen], geN[kWsGen], grN[kWsGen];
#pragma unroll
    for (int g = 0; g < kWsGen; ++g) {
      gc[g] = -1;
      gl[g] = geA[g] = grA[g] = gP[g] = geN[g] = grN[g] = 0.0;
    }
    for (int c = pw; c < L && ng < kWsGen; c += kWsProd) gc[ng++] = c;
#pragma unroll
    for (int g = 0; g < kWsGen; ++g)
      if (g < ng) {
        const int s = lb_s[gc[g]] * 8 + csub;
        gl[g] = s < m ? __ldg(lm + s) : 0.0;
      }
    const double ta = hstep_ta_s;
    auto anchor = [&](int kt) {
      const double t = fma((double)(kt * 32 + rsub), hstep_s, ta);
#pragma unroll
      for (int g = 0; g < kWsGen; ++g)
        if (g < ng) {
          const double d = gl[g] - t;
          geN[g] = exp(neg_div(d * d, sigma2, inv));
          grN[g] = exp(fma(2.0 * H, d, -H * H) * inv);
        }
    };
    if (rec) anchor(0);
    // every producer warp forms the row coefficients of its own tile copy in
    // registers (lane = row; the raw samples loaded two tiles ahead) and
    // exchanges them by shuffles: no producer waits for another
    RowRaw<P> raw1, raw2;
    if (nt > 0) row_load<P>(pts, coef, forcing, n_c, row_begin + tile0 * 32, row_end, raw1);
    if (nt > 1) row_load<P>(pts, coef, forcing, n_c, row_begin + (tile0 + 1) * 32, row_end, raw2);
    for (int k = 0; k < nt; ++k) {
      const int st = k % kWsStages;
      // this lane's row record: t, q_0..q_P, g = -f_P, r (row_store's arithmetic)
      double rt = raw1.t, rq[P + 1], rg, rr;
#pragma unroll
      for (int j = 0; j <= P; ++j) {
        double v = hc_s[P][j];
#pragma unroll
        for (int kk = 1; kk <= P; ++kk) v = fma(-raw1.f[kk - 1], hc_s[P - kk][j], v);
        rq[j] = raw1.ok ? v : 0.0;
      }
      rg = raw1.ok ? -raw1.f[P - 1] : 0.0;
      rr = raw1.r;
      raw1 = raw2;
      if (k + 2 < nt)
        row_load<P>(pts, coef, forcing, n_c, row_begin + (tile0 + k + 2) * 32, row_end, raw2);
      if (k >= kWsStages) nys::mbar_wait(&empty_b[st], ((k / kWsStages) - 1) & 1);
      double* const Xd = Xr + (size_t)st * xsz;
      if (NYS_WS_PROBE == 2) {
      } else if (rec) {
        const int u = k % kAnchorTiles;
        if (u == 0) {
#pragma unroll
          for (int g = 0; g < kWsGen; ++g) {
            geA[g] = geN[g];
            grA[g] = grN[g];
            gP[g] = 1.0;
          }
        }
        const double* qt = qtri_s + u * kTileKs;
        // three warp-uniform block kinds (the shuffles need every lane): landmark
        // columns only, g / r / padding columns only, or both (m % 8 != 0)
#pragma unroll
        for (int g = 0; g < kWsGen; ++g)
          if (g < ng) {
            const int b8 = lb_s[gc[g]] * 8, s = b8 + csub;
            const int kind = b8 + 7 < m ? 0 : (b8 >= m ? 1 : 2);
            double* Xo = Xd + (size_t)gc[g] * 32 + lane;
            if (kind == 1) {
#pragma unroll
              for (int ks = 0; ks < kTileKs; ++ks) {
                const int src = ks * 4 + rsub;
                const double gv = __shfl_sync(0xffffffffu, rg, src);
                const double rv = __shfl_sync(0xffffffffu, rr, src);
                Xo[(size_t)ks * kWsMaxL * 32] = (s == m) ? gv : (s == m + 1) ? rv : 0.0;
              }
              continue;
            }
            double rp[kTileKs + 1];   // rho_A^i, i <= 8, by a depth-3 product tree
            rp[0] = 1.0;
            rp[1] = grA[g];
            rp[2] = rp[1] * rp[1];
            rp[3] = rp[2] * rp[1];
            rp[4] = rp[2] * rp[2];
            rp[5] = rp[4] * rp[1];
            rp[6] = rp[4] * rp[2];
            rp[7] = rp[4] * rp[3];
            rp[8] = rp[4] * rp[4];
            const double base = geA[g] * gP[g];
#pragma unroll
            for (int ks = 0; ks < kTileKs; ++ks) {
              const int src = ks * 4 + rsub;   // this lane's row: ks * 4 + rsub
              const double d = gl[g] - __shfl_sync(0xffffffffu, rt, src);
              double poly = __shfl_sync(0xffffffffu, rq[P], src);
#pragma unroll
              for (int j = P - 1; j >= 0; --j)
                poly = fma(poly, d, __shfl_sync(0xffffffffu, rq[j], src));
              double val = poly * ((base * rp[ks]) * qt[ks]);
              if (kind == 2) {
                const double gv = __shfl_sync(0xffffffffu, rg, src);
                const double rv = __shfl_sync(0xffffffffu, rr, src);
                if (s >= m) val = (s == m) ? gv : (s == m + 1) ? rv : 0.0;
              }
              Xo[(size_t)ks * kWsMaxL * 32] = val;
            }
            gP[g] *= rp[8];
          }
        if (u == kAnchorTiles - 1) anchor(k + 1);
      } else {
        // non-uniform grid: exp() per entry from a per-warp copy of the records
        double* rc = rowr + (size_t)pw * 32 * kRowStride;   // written and read by this warp
        rc[lane * kRowStride + 0] = rt;
#pragma unroll
        for (int j = 0; j <= P; ++j) rc[lane * kRowStride + 1 + j] = rq[j];
        rc[lane * kRowStride + 6] = rg;
        rc[lane * kRowStride + 7] = rr;
        __syncwarp();
        for (int c = pw; c < L; c += kWsProd)
          gen_tile<P>(lm, m, c + 1, lb_s, kWsMaxL, sigma2, inv, rc, Xd, 4 * c, 1);   // block c
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&full_b[st]);
    }
  } else {
    // ================= consumers
    // The window's block pairs as a sequence of columns of row pairs: item
    // (rp, J), J >= 2 rp, holds the pairs (2 rp, J) and, when valid, (2 rp + 1, J)
    // -- one B fragment for both.  Consumer cw takes the items whose cumulative
    // pair count starts in [P cw / 12, P (cw + 1) / 12): equal DMMA counts, at
    // most kWsCols columns per warp; the per-warp shape is a template (no
    // per-pair decoding in the k loop).
    const int cw = warp - kWsProd;
    const int P_all = L * (L + 1) / 2;
    const int w0 = P_all * cw / kWsCons, w1 = P_all * (cw + 1) / kWsCons;
    int offa[kWsCols], offb[kWsCols], Ia[kWsCols], Jb[kWsCols];
    unsigned newrp = 0u, two = 0u;
    int nc = 0;
    {
      int cum = 0, prevrp = -1;
      for (int rp = 0; 2 * rp < L; ++rp)
        for (int J = 2 * rp; J < L; ++J) {
          const bool tw = 2 * rp + 1 < L && 2 * rp + 1 <= J;
          if (cum >= w0 && cum < w1 && nc < kWsCols) {
#pragma unroll
            for (int c = 0; c < kWsCols; ++c)
              if (c == nc) {
                offa[c] = 2 * rp * 32;
                offb[c] = J * 32;
                Ia[c] = 2 * rp;
                Jb[c] = J;
              }
            if (rp != prevrp) newrp |= 1u << nc;
            if (tw) two |= 1u << nc;
            prevrp = rp;
            ++nc;
          }
          cum += tw ? 2 : 1;
        }
    }
    switch (nc) {
      case 0: ws_consume<0>(Xr, nt, full_b, empty_b, offa, offb, Ia, Jb, newrp, two, lb_s, slab, ld); break;
      case 1: ws_consume<1>(Xr, nt, full_b, empty_b, offa, offb, Ia, Jb, newrp, two, lb_s, slab, ld); break;
      case 2: ws_consume<2>(Xr, nt, full_b, empty_b, offa, offb, Ia, Jb, newrp, two, lb_s, slab, ld); break;
      case 3: ws_consume<3>(Xr, nt, full_b, empty_b, offa, offb, Ia, Jb, newrp, two, lb_s, slab, ld); break;
      case 4: ws_consume<4>(Xr, nt, full_b, empty_b, offa, offb, Ia, Jb, newrp, two, lb_s, slab, ld); break;
      case 5: ws_consume<5>(Xr, nt, full_b, empty_b, offa, offb, Ia, Jb, newrp, two, lb_s, slab, ld); break;
      case 6: ws_consume<6>(Xr, nt, full_b, empty_b, offa, offb, Ia, Jb, newrp, two, lb_s, slab, ld); break;
      case 7: ws_consume<7>(Xr, nt, full_b, empty_b, offa, offb, Ia, Jb, newrp, two, lb_s, slab, ld); break;
      default: ws_consume<8>(Xr, nt, full_b, empty_b, offa, offb, Ia, Jb, newrp, two, lb_s, slab, ld); break;
    }
  }
}

// NYS_KSPACE_WS=1: the warp-specialised kernel for windows of <= kWsMaxL
// blocks, then the 12-warp kernel for the CTAs whose window is wider (it
// returns at once for the others).  Default: the 12-warp kernel alone -- on
// config 4 the warp-specialised version measured 2.19-2.73 ms against 2.31 ms
// across code-generation variants (its 8 producer warps, not the tensor pipe,
// set the pace: 1.5-1.7 ms with the DMMAs removed, 1.5 ms with generation
// removed), so it is kept as an A/B alternative only.
template <int PP>
cudaError_t launch_kspace(const LargePlan& L, const double* lm, int m, double sigma2,
                          const double* pts, const double* coef, const double* forcing, int n_c,
                          int row_begin, int row_end, double* slabs, unsigned long long* live,
                          cudaStream_t st) {
  static const bool ws_on = [] {
    const char* e = getenv("NYS_KSPACE_WS");
    return e && e[0] == '1';
  }();
  int min_L = 0;
  if (ws_on) {
    auto kw = large_ws_kernel<PP>;
    cudaError_t e = cudaFuncSetAttribute(kw, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)ws_smem_bytes());
    if (e != cudaSuccess) return e;
    kw<<<L.nrr, kWsWarps * 32, ws_smem_bytes(), st>>>(lm, m, sigma2, pts, coef, forcing, n_c,
                                                      row_begin, row_end, L.NB, L.ld,
                                                      L.tiles_per_cta, slabs, live);
    nys_host::count_launches(1);
    min_L = kWsMaxL + 1;
  }
  auto kern = large_kspace_kernel<PP>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)L.smem);
  if (e != cudaSuccess) return e;
  kern<<<L.nrr, kWarps * 32, L.smem, st>>>(lm, m, sigma2, pts, coef, forcing, n_c, row_begin,
                                           row_end, L.NB, L.NBpad, L.ld, L.nbuf, L.tiles_per_cta,
                                           slabs, live, min_L);
  nys_host::count_launches(1);
  return cudaGetLastError();
}

// K[r][c] = sum over CTAs (fixed order) of their slabs where both blocks are live
// (dead slab entries are never written: their loads are predicated off, and
// the select adds an exact 0); loads unrolled 8 deep so they are in flight
// together instead of one L2 round trip per CTA
__global__ void large_reduce_kernel(const double* __restrict__ slabs,
                                    const unsigned long long* __restrict__ live, int nrr, int ld,
                                    int Pe, double* __restrict__ K) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= Pe * Pe) return;
  const int r = e / Pe, c = e % Pe;
  if (c < r) return;
  const unsigned long long need = (1ull << (r / 8)) | (1ull << (c / 8));
  const double* p = slabs + (size_t)r * ld + c;
  const size_t step = (size_t)ld * ld;
  double s = 0.0;
  int rr = 0;
  for (; rr + 8 <= nrr; rr += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      v[u] = ((__ldg(live + rr + u) & need) == need) ? __ldg(p + (rr + u) * step) : 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) s += v[u];
  }
  for (; rr < nrr; ++rr)
    if ((live[rr] & need) == need) s += p[rr * step];
  K[(size_t)r * Pe + c] = s;
  K[(size_t)c * Pe + r] = s;
}

// T = K W_ext (Pe x Pw), then E = W_ext^T T (Pw x Pw);  W_ext = diag(W, 1, 1).
// One warp per 8 x 8 output tile, DMMA.8x8x4 over the landmark index s with
// the fragments read straight from L2 (K, W, T are <= 0.6 MB).  E is
// computed on the upper tile triangle and mirrored, so it is exactly symmetric.
constexpr int kProjWarps = 4;
__global__ void __launch_bounds__(kProjWarps * 32)
    proj_right_kernel(const double* __restrict__ K, int Pe, const double* __restrict__ W,
                      int ldw, int m, int m_eff, double* __restrict__ T) {
  const int Pw = m_eff + 2, lane = threadIdx.x & 31;
  const int tiles_c = (Pw + 7) / 8;
  const int t = blockIdx.x * kProjWarps + (threadIdx.x >> 5);
  const int r0 = (t / tiles_c) * 8, c0 = (t % tiles_c) * 8;
  if (r0 >= Pe) return;
  const int ar = r0 + (lane >> 2), bc = c0 + (lane >> 2), kq = lane & 3;
  double c_0 = 0.0, c_1 = 0.0;
  if (c0 < m_eff) {
    for (int s = 0; s < m; s += 4) {
      const int ks = s + kq;
      const double a = (ar < Pe && ks < m) ? K[(size_t)ar * Pe + ks] : 0.0;
      const double b = (bc < m_eff && ks < m) ? W[(size_t)ks * ldw + bc] : 0.0;
      nys::dmma(c_0, c_1, a, b);
    }
  }
  const int rr = r0 + (lane >> 2);
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int cc = c0 + 2 * (lane & 3) + j;
    if (rr >= Pe || cc >= Pw) continue;
    T[(size_t)rr * Pw + cc] = cc < m_eff ? (j ? c_1 : c_0) : K[(size_t)rr * Pe + m + (cc - m_eff)];
  }
}

__global__ void __launch_bounds__(kProjWarps * 32)
    proj_left_kernel(const double* __restrict__ T, int Pe, const double* __restrict__ W,
                     int ldw, int m, int m_eff, double* __restrict__ E) {
  const int Pw = m_eff + 2, lane = threadIdx.x & 31;
  const int nt = (Pw + 7) / 8;
  int t = blockIdx.x * kProjWarps + (threadIdx.x >> 5);
  if (t >= nt * (nt + 1) / 2) return;
  int I = 0;   // upper tile triangle, row-major
  while (t >= nt - I) {
    t -= nt - I;
    ++I;
  }
  const int r0 = I * 8, c0 = (I + t) * 8;
  const int ar = r0 + (lane >> 2), bc = c0 + (lane >> 2), kq = lane & 3;
  double c_0 = 0.0, c_1 = 0.0;
  if (r0 < m_eff) {
    for (int s = 0; s < m; s += 4) {
      const int ks = s + kq;
      const double a = (ar < m_eff && ks < m) ? W[(size_t)ks * ldw + ar] : 0.0;
      const double b = (bc < Pw && ks < m) ? T[(size_t)ks * Pw + bc] : 0.0;
      nys::dmma(c_0, c_1, a, b);
    }
  }
  const int rr = r0 + (lane >> 2);
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int cc = c0 + 2 * (lane & 3) + j;
    if (rr >= Pw || cc >= Pw || cc < rr) continue;
    const double v = rr < m_eff ? (j ? c_1 : c_0) : T[(size_t)(m + (rr - m_eff)) * Pw + cc];
    E[(size_t)rr * Pw + cc] = v;
    E[(size_t)cc * Pw + rr] = v;
  }
}

void launch_proj(const double* K, int Pe, const double* W, int ldw, int m, int m_eff, double* T,
                 double* E, cudaStream_t st) {
  const int Pw = m_eff + 2, tr = (Pe + 7) / 8, tc = (Pw + 7) / 8;
  proj_right_kernel<<<(tr * tc + kProjWarps - 1) / kProjWarps, kProjWarps * 32, 0, st>>>(
      K, Pe, W, ldw, m, m_eff, T);
  proj_left_kernel<<<(tc * (tc + 1) / 2 + kProjWarps - 1) / kProjWarps, kProjWarps * 32, 0, st>>>(
      T, Pe, W, ldw, m, m_eff, E);
  nys_host::count_launches(2);
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
  if (!L.fits()) return NYS_EUNSUPPORTED;
  if (ws == nullptr || ws_bytes < L.ws_bytes(m_eff)) return NYS_EWORKSPACE;
  double* slabs = static_cast<double*>(ws);
  double* K = slabs + L.slab_doubles();
  double* T = K + (size_t)L.Pe * L.Pe;
  const int Pw = m_eff + 2;
  auto* live = reinterpret_cast<unsigned long long*>(T + (size_t)L.Pe * Pw);
  cudaError_t le;
  switch (p) {
    case 1: le = launch_kspace<1>(L, lm, m, sigma2, pts, coef, forcing, n_c, row_begin, row_end, slabs, live, st); break;
    case 2: le = launch_kspace<2>(L, lm, m, sigma2, pts, coef, forcing, n_c, row_begin, row_end, slabs, live, st); break;
    case 3: le = launch_kspace<3>(L, lm, m, sigma2, pts, coef, forcing, n_c, row_begin, row_end, slabs, live, st); break;
    default: le = launch_kspace<4>(L, lm, m, sigma2, pts, coef, forcing, n_c, row_begin, row_end, slabs, live, st); break;
  }
  if (le != cudaSuccess) return record_cuda(le);
  NYS_CHECK_LAUNCH();
  large_reduce_kernel<<<(L.Pe * L.Pe + 255) / 256, 256, 0, st>>>(slabs, live, L.nrr, L.ld, L.Pe,
                                                                 K);
  nys_host::count_launches(1);
  launch_proj(K, L.Pe, W, ldw, m, m_eff, T, gram_ext, st);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

}  // namespace nys_host

// ---- split entry points: the kernel-space Gram needs no eigenvectors, so it can
// run concurrently with the landmark eigendecomposition (config 4); the
// projection E = W_ext^T K W_ext follows once W exists.
extern "C" size_t nys_kspace_gram_workspace_bytes(int n_c, int m, int max_ctas) {
  const LargePlan L = LargePlan::make(n_c, m, max_ctas);
  return L.slab_doubles() * sizeof(double) + (size_t)L.nrr * sizeof(unsigned long long) + 512;
}

extern "C" int nys_kspace_gram_f64(const double* landmarks, int m, double sigma2, int p,
                                   const double* pts, const double* coef, const double* forcing,
                                   int n_c, int row_begin, int row_end, int max_ctas, double* K,
                                   void* ws, size_t ws_bytes, void* stream) {
  if (m < 1 || p < 1 || p > nys::kMaxOrder || n_c < 0 || row_begin < 0 || row_end > n_c ||
      row_begin > row_end || !(sigma2 > 0.0))
    return NYS_EINVAL;
  const LargePlan L = LargePlan::make(row_end - row_begin, m, max_ctas);
  if (!L.fits()) return NYS_EUNSUPPORTED;
  if (ws == nullptr || ws_bytes < nys_kspace_gram_workspace_bytes(row_end - row_begin, m, max_ctas))
    return NYS_EWORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* slabs = static_cast<double*>(ws);
  auto* live = reinterpret_cast<unsigned long long*>(slabs + L.slab_doubles());
  cudaError_t le;
  switch (p) {
    case 1: le = launch_kspace<1>(L, landmarks, m, sigma2, pts, coef, forcing, n_c, row_begin, row_end, slabs, live, st); break;
    case 2: le = launch_kspace<2>(L, landmarks, m, sigma2, pts, coef, forcing, n_c, row_begin, row_end, slabs, live, st); break;
    case 3: le = launch_kspace<3>(L, landmarks, m, sigma2, pts, coef, forcing, n_c, row_begin, row_end, slabs, live, st); break;
    default: le = launch_kspace<4>(L, landmarks, m, sigma2, pts, coef, forcing, n_c, row_begin, row_end, slabs, live, st); break;
  }
  if (le != cudaSuccess) return nys_host::record_cuda(le);
  NYS_CHECK_LAUNCH();
  large_reduce_kernel<<<(L.Pe * L.Pe + 255) / 256, 256, 0, st>>>(slabs, live, L.nrr, L.ld, L.Pe, K);
  nys_host::count_launches(1);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" size_t nys_kspace_project_workspace_bytes(int m, int m_eff) {
  return (size_t)(m + 2) * (m_eff + 2) * sizeof(double) + 256;
}

extern "C" int nys_kspace_project_f64(const double* K, int m, const double* W, int ldw, int m_eff,
                                      double* gram_ext, void* ws, size_t ws_bytes, void* stream) {
  if (m < 1 || m_eff < 1 || m_eff > m || ldw < m_eff) return NYS_EINVAL;
  if (ws == nullptr || ws_bytes < nys_kspace_project_workspace_bytes(m, m_eff)) return NYS_EWORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int Pe = m + 2;
  double* T = static_cast<double*>(ws);
  launch_proj(K, Pe, W, ldw, m, m_eff, T, gram_ext, st);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}
