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
// Layout.  The Pe = m + 2 columns form NB 8-wide blocks grouped in 4-block
// super-blocks; the Gram's upper triangle is a set of super-tiles (a <= b),
// each a 4 x 4 rectangle of 8x8 DMMA accumulators held by one warp (64
// registers).  The 258-wide config-4 Gram (561 block pairs, 287 KB of FP64
// accumulators) does not fit one SM's register file, so the super-tiles are
// split over `ngroups` CTAs (one per SM, up to 18 warps each) that walk the
// same row range; when the last super-block holds a single block (NB % 4 == 1,
// config 4) the diagonal super-tile a and its stub (a, last) share one warp
// (10 + 4 pairs in the 16 accumulator slots) and the corner (last, last) rides
// along, so every DMMA issued is a block pair of the Gram.
//
// Pipeline per CTA: 32-row tiles, double-buffered in shared memory in the
// fragment-native layout X[ks][blk][lane] (conflict-free LDS.64).  Iteration t
// issues the DMMAs of tile t and generates tile t+1 (exp + Hermite polynomial
// per element) into the other buffer; the DMMA pipe and the generation
// arithmetic overlap across warps, one __syncthreads per tile.  The per-row
// polynomial coefficients are produced two tiles ahead.  Partials go to the
// workspace and are reduced in fixed order (deterministic).
#include <cstdint>
#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace {

constexpr int kRT = 4;             // super-tile edge (blocks)
constexpr int kMaxWarps = 18;      // warps per CTA (576 threads, 1 CTA / SM)
constexpr int kTileKs = 8;         // 4-row k-steps per row tile (32 rows)
constexpr int kMaxTasks = 384;
constexpr int kMaxSmem = 227 * 1024;

// task word: a | b << 8 | mode << 16 | corner << 17   (mode 1 = diag a + stub (a, last))
struct TaskTable {
  int word[kMaxTasks];
};

NYS_DEV void task_decode(int w, int& a, int& b, int& stub, int& corner) {
  a = w & 255;
  b = (w >> 8) & 255;
  stub = (w >> 16) & 1;
  corner = (w >> 17) & 1;
}

struct LargePlan {
  int Pe, NB, NSB, NBpad, ntasks, ngroups, wpc, nrr, ntiles, tiles_per_cta, nbuf;
  bool stub;
  size_t smem;
  TaskTable tasks;

  static LargePlan make(int n_rows, int m) {
    LargePlan L;
    std::memset(&L, 0, sizeof(L));
    L.Pe = m + 2;                                 // kernel-space extended width
    L.NB = (L.Pe + 7) / 8;
    L.NSB = (L.NB + kRT - 1) / kRT;
    L.NBpad = L.NSB * kRT;
    L.stub = (L.NB % kRT == 1) && L.NSB >= 2;
    // task list with DMMA weights
    std::vector<std::pair<int, int>> t;   // (word, weight)
    const int full = L.stub ? L.NSB - 1 : L.NSB;
    for (int a = 0; a < full; ++a)
      for (int b = a; b < L.NSB; ++b) {
        if (L.stub && b == L.NSB - 1) continue;   // stub folded into the diagonal task
        int w = a | (b << 8);
        int weight = 0;
        for (int i = 0; i < kRT; ++i)
          for (int j = 0; j < kRT; ++j)
            if (a * kRT + i < L.NB && b * kRT + j < L.NB && !(a == b && i > j)) ++weight;
        if (L.stub && a == b) {
          w |= 1 << 16;
          weight += kRT;
          if (a == L.NSB - 2) {
            w |= 1 << 17;
            weight += 1;
          }
        }
        t.push_back({w, weight});
      }
    L.ntasks = (int)t.size();
    L.ngroups = (L.ntasks + kMaxWarps - 1) / kMaxWarps;
    L.wpc = (L.ntasks + L.ngroups - 1) / L.ngroups;
    // deal tasks heaviest-first: round-robin over groups, then within a group
    // over the 4 SM sub-partitions (warp w runs on SMSP w % 4) by least load
    std::sort(t.begin(), t.end(), [](auto& x, auto& y) { return x.second > y.second; });
    std::vector<std::vector<std::pair<int, int>>> grp(L.ngroups);
    std::vector<int> gload(L.ngroups, 0);
    for (auto& e : t) {
      int best = -1;
      for (int g = 0; g < L.ngroups; ++g)
        if ((int)grp[g].size() < L.wpc && (best < 0 || gload[g] < gload[best])) best = g;
      grp[best].push_back(e);
      gload[best] += e.second;
    }
    for (int g = 0; g < L.ngroups; ++g) {
      int cap[4], load[4] = {0, 0, 0, 0};
      for (int s = 0; s < 4; ++s) cap[s] = (L.wpc - s + 3) / 4;
      std::vector<int> slot_words[4];
      for (auto& e : grp[g]) {
        int best = -1;
        for (int s = 0; s < 4; ++s)
          if ((int)slot_words[s].size() < cap[s] && (best < 0 || load[s] < load[best])) best = s;
        slot_words[best].push_back(e.first);
        load[best] += e.second;
      }
      for (int w = 0; w < L.wpc; ++w) {
        auto& v = slot_words[w % 4];
        size_t k = (size_t)(w / 4);
        L.tasks.word[g * L.wpc + w] = k < v.size() ? v[k] : -1;
      }
    }
    L.ntiles = (n_rows + 4 * kTileKs - 1) / (4 * kTileKs);
    int nrr = nys::device_sm_count() / L.ngroups;
    if (nrr < 1) nrr = 1;
    if (nrr > L.ntiles) nrr = L.ntiles > 0 ? L.ntiles : 1;
    L.nrr = nrr;
    L.tiles_per_cta = (L.ntiles + nrr - 1) / nrr;
    const size_t xbuf = (size_t)kTileKs * L.NBpad * 32 * sizeof(double);
    const size_t rowc = 3 * 32 * 8 * sizeof(double);
    L.nbuf = (2 * xbuf + rowc <= (size_t)kMaxSmem) ? 2 : 1;
    L.smem = L.nbuf * xbuf + rowc;
    return L;
  }
  bool fits() const {
    return ntasks <= kMaxTasks && ngroups * wpc <= kMaxTasks && smem <= (size_t)kMaxSmem;
  }
  size_t part_doubles() const { return (size_t)nrr * ngroups * wpc * kRT * kRT * 64; }
  size_t ws_bytes(int m_eff) const {
    return (part_doubles() + (size_t)Pe * Pe + (size_t)Pe * (m_eff + 2)) * sizeof(double) + 256;
  }
};

// per-row polynomial coefficients for one 32-row tile: t, q0..qP, g = -f_p, r
template <int P>
NYS_DEV void row_coeffs(const nys::Hermite& H, const double* __restrict__ pts,
                        const double* __restrict__ coef, const double* __restrict__ forcing,
                        int n_c, int r0, int row_end, double* rowc) {
  const int lane = threadIdx.x & 31;
  const int i = r0 + lane;
  const bool ok = i < row_end;
  double f[P];
#pragma unroll
  for (int k = 0; k < P; ++k) f[k] = ok ? coef[(size_t)k * n_c + i] : 0.0;
  double* rc = rowc + lane * 8;
  rc[0] = ok ? pts[i] : 0.0;
#pragma unroll
  for (int j = 0; j <= P; ++j) {
    double v = H.c[P][j];
#pragma unroll
    for (int k = 1; k <= P; ++k) v = fma(-f[k - 1], H.c[P - k][j], v);
    rc[1 + j] = ok ? v : 0.0;   // rows past the end: all-zero polynomial -> G = 0
  }
  rc[6] = ok ? -f[P - 1] : 0.0;
  rc[7] = ok ? forcing[i] : 0.0;
}

// -(x / sigma2) for x >= 0, correctly rounded from the precomputed reciprocal:
// q = x * inv, remainder by FMA, one correction (checked bit-exact against the
// IEEE quotient by tools/div_check.cu) -- the kernel.py:78-79 division at 3 FP64 ops.
NYS_DEV double neg_div(double x, double sigma2, double inv) {
  double q = x * inv;
  double r = fma(-q, sigma2, x);
  return -fma(r, inv, q);
}

template <int P>
NYS_DEV void gen_tile(const double* __restrict__ lm, int m, int NB, int NBpad, double sigma2,
                      double inv, uint64_t need, const double* rowc, double* X, int warp,
                      int nwarps) {
  const int lane = threadIdx.x & 31;
  const int rsub = lane & 3, csub = lane >> 2;
  int blk = warp, ks = 0;
  while (blk >= NB) { blk -= NB; ++ks; }
  for (; ks < kTileKs;) {
    if ((need >> blk) & 1ull) {
      const int s = blk * 8 + csub;
      const double* rc = rowc + (ks * 4 + rsub) * 8;
      double v = 0.0;
      if (s < m) {
        const double d = __ldg(lm + s) - rc[0];
        double poly = rc[1 + P];
#pragma unroll
        for (int j = P - 1; j >= 0; --j) poly = fma(poly, d, rc[1 + j]);
        v = poly * exp(neg_div(d * d, sigma2, inv));
      } else if (s == m) {
        v = rc[6];
      } else if (s == m + 1) {
        v = rc[7];
      }
      X[((size_t)ks * NBpad + blk) * 32 + lane] = v;
    }
    blk += nwarps;
    while (blk >= NB) { blk -= NB; ++ks; }
  }
}

template <int P>
__global__ void __launch_bounds__(kMaxWarps * 32, 1)
    large_kspace_kernel(const double* __restrict__ lm, int m, double sigma2,
                        const double* __restrict__ pts, const double* __restrict__ coef,
                        const double* __restrict__ forcing, int n_c, int row_begin, int row_end,
                        int NB, int NBpad, int wpc, int nbuf, int tiles_per_cta,
                        const __grid_constant__ TaskTable tasks, double* __restrict__ part) {
  extern __shared__ __align__(16) double sm[];
  const size_t xsz = (size_t)kTileKs * NBpad * 32;
  double* const X0 = sm;
  double* const X1 = sm + (nbuf - 1) * xsz;
  double* rowc = sm + nbuf * xsz;   // [3][32][8]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  const int group = blockIdx.y;
  const int word = warp < wpc ? tasks.word[group * wpc + warp] : -1;
  int a = -1, b = -1, stub = 0, corner = 0;
  if (word >= 0) task_decode(word, a, b, stub, corner);
  const int last = NB - 1;

  // blocks this CTA's warps read (NB <= 64)
  __shared__ unsigned long long need_s;
  if (threadIdx.x == 0) need_s = 0ull;
  __syncthreads();
  if (lane == 0 && a >= 0) {
    unsigned long long mk = 0ull;
    for (int i = 0; i < kRT; ++i) {
      if (a * kRT + i < NB) mk |= 1ull << (a * kRT + i);
      if (b * kRT + i < NB) mk |= 1ull << (b * kRT + i);
    }
    if (stub) mk |= 1ull << last;
    atomicOr(&need_s, mk);
  }
  // DMMA predicate mask for the generic (non-stub) tasks
  uint32_t valid = 0;
  if (a >= 0 && !stub)
    for (int i = 0; i < kRT; ++i)
      for (int j = 0; j < kRT; ++j)
        if (a * kRT + i < NB && b * kRT + j < NB && !(a == b && i > j)) valid |= 1u << (i * kRT + j);

  nys::Hermite H;
  H.init(sigma2, P);
  const double inv = 1.0 / sigma2;

  double acc[kRT][kRT][2];
#pragma unroll
  for (int i = 0; i < kRT; ++i)
#pragma unroll
    for (int j = 0; j < kRT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int ntiles = (row_end - row_begin + 31) / 32;
  const int tile0 = blockIdx.x * tiles_per_cta;
  const int tile1 = min(ntiles, tile0 + tiles_per_cta);
  const int cw = nwarps - 1;   // warp that prepares row coefficients

  if (tile0 < tile1) {
    if (warp == cw) {
      row_coeffs<P>(H, pts, coef, forcing, n_c, row_begin + tile0 * 32, row_end, rowc);
      if (tile0 + 1 < tile1)
        row_coeffs<P>(H, pts, coef, forcing, n_c, row_begin + (tile0 + 1) * 32, row_end,
                      rowc + 256);
    }
    __syncthreads();
    gen_tile<P>(lm, m, NB, NBpad, sigma2, inv, need_s, rowc, X0, warp, nwarps);
    __syncthreads();
  }
  const uint64_t need = need_s;
  for (int tile = tile0; tile < tile1; ++tile) {
    const int k = tile - tile0;
    const double* X = (k & 1) ? X1 : X0;
    if (a >= 0) {
      const double* Xl = X + lane;
      if (stub) {
#pragma unroll 1
        for (int ks = 0; ks < kTileKs; ++ks) {
          const double* Xk = Xl + (size_t)ks * NBpad * 32;
          double xa[kRT];
#pragma unroll
          for (int i = 0; i < kRT; ++i) xa[i] = Xk[(a * kRT + i) * 32];
          const double xl = Xk[last * 32];
#pragma unroll
          for (int i = 0; i < kRT; ++i)
#pragma unroll
            for (int j = i; j < kRT; ++j) nys::dmma(acc[i][j][0], acc[i][j][1], xa[i], xa[j]);
          // stub (a-block i, last) in the lower slots (1,0) (2,0) (3,0) (2,1)
          nys::dmma(acc[1][0][0], acc[1][0][1], xa[0], xl);
          nys::dmma(acc[2][0][0], acc[2][0][1], xa[1], xl);
          nys::dmma(acc[3][0][0], acc[3][0][1], xa[2], xl);
          nys::dmma(acc[2][1][0], acc[2][1][1], xa[3], xl);
          if (corner) nys::dmma(acc[3][1][0], acc[3][1][1], xl, xl);
        }
      } else {
#pragma unroll 1
        for (int ks = 0; ks < kTileKs; ++ks) {
          const double* Xk = Xl + (size_t)ks * NBpad * 32;
          double xa[kRT], xb[kRT];
#pragma unroll
          for (int i = 0; i < kRT; ++i) xa[i] = Xk[(a * kRT + i) * 32];
#pragma unroll
          for (int j = 0; j < kRT; ++j) xb[j] = Xk[(b * kRT + j) * 32];
#pragma unroll
          for (int i = 0; i < kRT; ++i)
#pragma unroll
            for (int j = 0; j < kRT; ++j)
              if ((valid >> (i * kRT + j)) & 1u)
                nys::dmma(acc[i][j][0], acc[i][j][1], xa[i], xb[j]);
        }
      }
    }
    if (nbuf == 1) __syncthreads();
    if (tile + 1 < tile1)
      gen_tile<P>(lm, m, NB, NBpad, sigma2, inv, need, rowc + ((k + 1) % 3) * 256,
                  ((k + 1) & 1) ? X1 : X0, warp, nwarps);
    if (warp == cw && tile + 2 < tile1)
      row_coeffs<P>(H, pts, coef, forcing, n_c, row_begin + (tile + 2) * 32, row_end,
                    rowc + ((k + 2) % 3) * 256);
    __syncthreads();
  }
  if (a >= 0) {
    double* out = part + (((size_t)blockIdx.x * gridDim.y + group) * wpc + warp) *
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
__global__ void large_reduce_kernel(const double* __restrict__ part, int nrr, int nslots, int NB,
                                    int Pe, const __grid_constant__ TaskTable tasks,
                                    double* __restrict__ K) {
  const int per = kRT * kRT * 64;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nslots * per;
       e += gridDim.x * blockDim.x) {
    const int slot = e / per, w = e % per;
    const int word = tasks.word[slot];
    if (word < 0) continue;
    int a, b, stub, corner;
    task_decode(word, a, b, stub, corner);
    const int ij = w >> 6, lane = (w & 63) >> 1, jj = w & 1;
    const int i = ij / kRT, j = ij % kRT;
    int I, J;   // block row / column of this accumulator
    if (stub && i > j) {
      if (i == 3 && j == 1) {
        if (!corner) continue;
        I = J = NB - 1;
      } else {
        const int src = (i == 1) ? 0 : (i == 2 && j == 0) ? 1 : (i == 3) ? 2 : 3;
        I = a * kRT + src;
        J = NB - 1;
        if (i == 3 && j == 2) continue;   // unused slot
      }
    } else {
      if (a == b && i > j) continue;
      I = a * kRT + i;
      J = b * kRT + j;
      if (I >= NB || J >= NB) continue;
    }
    double s = 0.0;
    for (int rr = 0; rr < nrr; ++rr) s += part[((size_t)rr * nslots + slot) * per + w];
    const int r = I * 8 + (lane >> 2), c = J * 8 + 2 * (lane & 3) + jj;
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
  static_assert(sizeof(TaskTable) <= 4000, "task table must fit the kernel parameter space");
  LargePlan L = LargePlan::make(row_end - row_begin, m);
  if (L.NB > 64 || !L.fits()) return NYS_EUNSUPPORTED;
  if (ws == nullptr || ws_bytes < L.ws_bytes(m_eff)) return NYS_EWORKSPACE;
  double* part = static_cast<double*>(ws);
  double* K = part + L.part_doubles();
  double* T = K + (size_t)L.Pe * L.Pe;
  dim3 grid(L.nrr, L.ngroups);
  const int nthreads = L.wpc * 32;
#define NYS_LARGE(PP)                                                                              \
  do {                                                                                             \
    auto kern = large_kspace_kernel<PP>;                                                           \
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,        \
                                         (int)L.smem);                                             \
    if (e != cudaSuccess) return record_cuda(e);                                                   \
    kern<<<grid, nthreads, L.smem, st>>>(lm, m, sigma2, pts, coef, forcing, n_c, row_begin,        \
                                         row_end, L.NB, L.NBpad, L.wpc, L.nbuf, L.tiles_per_cta,   \
                                         L.tasks, part);                                           \
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
  const int nslots = L.ngroups * L.wpc;
  int per = nslots * kRT * kRT * 64;
  large_reduce_kernel<<<(per + 255) / 256, 256, 0, st>>>(part, L.nrr, nslots, L.NB, L.Pe, L.tasks,
                                                         K);
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
