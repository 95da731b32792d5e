// Batched extended Gram for B linear ODEs that share grid, landmarks and sigma
// (config 2).  Numeric core of linear.assemble (linear.py:103-133) per
// instance:
//     D_b = Psi_p - sum_k f_{b,k} (.) Psi_{p-k},  g_b = -f_{b,p},  r_b
//     E_b = [D_b g_b r_b]^T [D_b g_b r_b]
// Psi_0..Psi_p are formed once per batch (the reference's own per-order
// projection, linear.py:103-112) in a fragment-native packed layout; the CTA
// streams them through shared memory (1-D TMA bulk copies, double buffered on
// mbarriers).  Each instance is owned by SPLIT warps (SPLIT = 2 for wide Grams:
// each warp holds half of the upper block triangle, so a CTA of 16 warps keeps
// 4 warps per scheduler to hide FP64 latency).  A warp combines its rows in
// registers (FP64 FMA) and feeds the SAME register fragment to both operands of
// DMMA.8x8x4.  Gram and rhs come from one rounding of D (mixing
// roundings costs up to 5.9e-5).  Row splits (grid.y) give whole waves on 148
// SMs; their partials are summed in a fixed order (deterministic, no FP64
// atomics).
#include <algorithm>

#include "batch_layout.cuh"
#include "common.cuh"

namespace nys_host {
int launch_psi_pack(const double* lm, int m, const double* W, int ldw, int m_eff, double sigma2,
                    int p, const double* pts, int n_c, int n_blocks, int n_rows_pad,
                    double* packed, cudaStream_t st);
}

namespace {

using nys::BatchLayout;

constexpr int kStages = 4;   // Psi chunks in flight (55 KB each at NB = 9, p = 2)
#ifndef NYS_GB_UNROLL
#define NYS_GB_UNROLL 2   // k-steps per loop trip in gram_body: 2 lets the next k-step's combine fill DMMA throttle stalls (2.84 -> 2.79 ms; 4 spills)
#endif
constexpr int kGbUnroll = NYS_GB_UNROLL;

template <int NB>
struct Tri {
  static constexpr int kPairs = NB * (NB + 1) / 2;
  static constexpr NYS_DEV int idx(int I, int J) { return I * NB - (I * (I - 1)) / 2 + (J - I); }
};

// pairs [Lo, Hi) of the I-major upper block triangle
template <int NB, int Lo, int Hi>
struct Role {
  static constexpr int kCount = Hi - Lo;
  static constexpr NYS_DEV bool has(int I, int J) {
    return Tri<NB>::idx(I, J) >= Lo && Tri<NB>::idx(I, J) < Hi;
  }
  static constexpr NYS_DEV bool needs(int F) {
    for (int I = 0; I < NB; ++I)
      for (int J = I; J < NB; ++J)
        if (has(I, J) && (I == F || J == F)) return true;
    return false;
  }
};

// NB = blocks in the packed Psi chunk; EXT: block NB-1 holds only (g, r) and
// is accumulated with FMAs (DMMA over blocks 0..NB-2 only)
template <int NB, int NO, int WARPS, int SPLIT, int Lo, int Hi, bool EXT>
NYS_DEV void gram_body(const double* __restrict__ psi, const double* __restrict__ coef,
                       const double* __restrict__ forcing, int n_c, int B, int b, int ks0,
                       int nchunks, int rcol, double* sm, uint64_t* bar, int* cnt,
                       double* __restrict__ part) {
  constexpr int P = NO - 1;
  constexpr int CH = nys::kBatchChunkKs;
  constexpr int kChunkDoubles = CH * NO * NB * 32;
  constexpr uint32_t kChunkBytes = kChunkDoubles * sizeof(double);
  constexpr int NBD = EXT ? NB - 1 : NB;        // blocks that go through DMMA
  constexpr int SLOT = EXT ? NBD * (NBD + 1) / 2 * 64 + NBD * 64 + 96 : NB * (NB + 1) / 2 * 64;
  using R = Role<NBD, Lo, Hi>;

  const int lane = threadIdx.x & 31, tig = lane & 3, gid = lane >> 2;
  const bool active = b < B;
  double acc[R::kCount][2];
#pragma unroll
  for (int q = 0; q < R::kCount; ++q) acc[q][0] = acc[q][1] = 0.0;
  double accg[EXT ? NBD : 1], accr[EXT ? NBD : 1], accgg = 0.0, accgr = 0.0, accrr = 0.0;
#pragma unroll
  for (int F = 0; F < (EXT ? NBD : 1); ++F) accg[F] = accr[F] = 0.0;

  const double* cb = coef + (size_t)(active ? b : 0) * P * n_c;
  const double* rb = forcing + (size_t)(active ? b : 0) * n_c;
  double fk[P], rr, fk_n[P], rr_n;
  auto load_rows = [&](int c, double* f, double& r) {
    const int row = (ks0 + c * CH) * 4 + lane;
    const bool ok = active && row < n_c;
#pragma unroll
    for (int k = 0; k < P; ++k) f[k] = ok ? __ldg(cb + (size_t)k * n_c + row) : 0.0;
    r = ok ? __ldg(rb + row) : 0.0;
  };
  load_rows(0, fk, rr);

  constexpr int NS = kStages;
  for (int c = 0; c < nchunks; ++c) {
    const int stage = c % NS;
    const uint32_t phase = (c / NS) & 1;
    if (c + 1 < nchunks) load_rows(c + 1, fk_n, rr_n);
    nys::mbar_wait(&bar[stage], phase);
    const double* Q = sm + stage * kChunkDoubles + lane;
    if (active) {
#pragma unroll kGbUnroll
      for (int kk = 0; kk < CH; ++kk) {
        const int src = kk * 4 + tig;
        double f[P];
#pragma unroll
        for (int k = 0; k < P; ++k) f[k] = nys::shfl(fk[k], src);
        const double r = nys::shfl(rr, src);
        double x[NBD];
#pragma unroll
        for (int F = 0; F < NBD; ++F) {
          if (!R::needs(F)) {
            x[F] = 0.0;
            continue;
          }
          // Q layout per k-step: [order][block][lane]
          double v = Q[((kk * NO + P) * NB + F) * 32];
#pragma unroll
          for (int k = 1; k <= P; ++k)
            v = fma(-f[k - 1], Q[((kk * NO + (P - k)) * NB + F) * 32], v);
          x[F] = (!EXT && F * 8 + gid == rcol) ? r : v;
        }
#pragma unroll
        for (int I = 0; I < NBD; ++I)
#pragma unroll
          for (int J = I; J < NBD; ++J)
            if (R::has(I, J)) {
              const int q = Tri<NBD>::idx(I, J) - Lo;
              nys::dmma(acc[q][0], acc[q][1], x[I], x[J]);
            }
        if constexpr (EXT) {
          // extended columns of this lane's row: g = -f_p (what Psi_0's unit
          // column makes of the combine), r = forcing
          const double gq = -f[P - 1];
#pragma unroll
          for (int F = 0; F < NBD; ++F) {
            accg[F] = fma(x[F], gq, accg[F]);
            accr[F] = fma(x[F], r, accr[F]);
          }
          accgg = fma(gq, gq, accgg);
          accgr = fma(gq, r, accgr);
          accrr = fma(r, r, accrr);
        }
      }
    }
    if (c + 1 < nchunks) {
#pragma unroll
      for (int k = 0; k < P; ++k) fk[k] = fk_n[k];
      rr = rr_n;
    }
    // release the stage without a CTA barrier: the last warp to finish it
    // refills it with chunk c + NS (warps drift up to NS - 1 chunks apart).
    // Ordering: __syncwarp orders the warp's shared-memory reads of the stage
    // before lane 0's release (acq_rel atomic); the last arriver's acquire
    // sees every warp's reads complete, then fence.proxy.async orders them
    // before the async-proxy refill.  The counter only grows (one WARPS-sized
    // round per use of the stage), so no reset store races the next round.
    __syncwarp();
    if (lane == 0) {
      const int done = nys::atomic_add_acq_rel_cta(&cnt[stage], 1);
      if (done % WARPS == WARPS - 1) {
        if (c + NS < nchunks) {
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          nys::mbar_expect_tx(&bar[stage], kChunkBytes);
          nys::bulk_g2s(sm + stage * kChunkDoubles,
                        psi + (size_t)(ks0 + (c + NS) * CH) * NO * NB * 32, kChunkBytes,
                        &bar[stage]);
        }
      }
    }
  }
  if (active) {
    double* slot = part + ((size_t)blockIdx.y * B + b) * SLOT;
    double* out = slot + (size_t)Lo * 64 + lane * 2;
#pragma unroll
    for (int q = 0; q < R::kCount; ++q) {
      out[q * 64] = acc[q][0];
      out[q * 64 + 1] = acc[q][1];
    }
    if constexpr (EXT) {
      double* ex = slot + NBD * (NBD + 1) / 2 * 64;
#pragma unroll
      for (int F = 0; F < NBD; ++F) {
        ex[(F * 32 + lane) * 2] = accg[F];
        ex[(F * 32 + lane) * 2 + 1] = accr[F];
      }
      double* sc = ex + NBD * 64 + lane * 3;
      sc[0] = accgg;
      sc[1] = accgr;
      sc[2] = accrr;
    }
  }
}

template <int NB, int NO, int WARPS, int SPLIT, bool EXT>
__global__ void __launch_bounds__(WARPS * 32, 1)
    batch_gram_kernel(const double* __restrict__ psi, const double* __restrict__ coef,
                      const double* __restrict__ forcing, int n_c, int B, int ks_per_split,
                      int rcol, double* __restrict__ part) {
  constexpr int CH = nys::kBatchChunkKs;
  constexpr int kChunkDoubles = CH * NO * NB * 32;
  constexpr uint32_t kChunkBytes = kChunkDoubles * sizeof(double);
  constexpr int NPAIR = Tri<EXT ? NB - 1 : NB>::kPairs;
  constexpr int H = (NPAIR + 1) / 2;

  extern __shared__ __align__(128) double sm[];   // [kStages][kChunkDoubles]
  __shared__ __align__(8) uint64_t bar[kStages];
  __shared__ int cnt[kStages];

  const int warp = threadIdx.x >> 5;
  const int b = blockIdx.x * (WARPS / SPLIT) + warp / SPLIT;
  const int ks0 = blockIdx.y * ks_per_split;
  const int nchunks = ks_per_split / CH;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      nys::mbar_init(&bar[s], 1);
      cnt[s] = 0;
    }
    nys::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages && s < nchunks; ++s) {
      nys::mbar_expect_tx(&bar[s], kChunkBytes);
      nys::bulk_g2s(sm + s * kChunkDoubles, psi + (size_t)(ks0 + s * CH) * NO * NB * 32,
                    kChunkBytes, &bar[s]);
    }
  }
  if constexpr (SPLIT == 1) {
    gram_body<NB, NO, WARPS, SPLIT, 0, NPAIR, EXT>(psi, coef, forcing, n_c, B, b, ks0, nchunks,
                                                   rcol, sm, bar, cnt, part);
  } else {
    if ((warp & 1) == 0)
      gram_body<NB, NO, WARPS, SPLIT, 0, H, EXT>(psi, coef, forcing, n_c, B, b, ks0, nchunks,
                                                 rcol, sm, bar, cnt, part);
    else
      gram_body<NB, NO, WARPS, SPLIT, H, NPAIR, EXT>(psi, coef, forcing, n_c, B, b, ks0, nchunks,
                                                     rcol, sm, bar, cnt, part);
  }
}

// partials -> dense E (Pe x Pe) per instance, summing splits (and, for the
// FMA-accumulated extended columns, the lanes that share a column) in fixed order
__global__ void batch_unpack_kernel(const double* __restrict__ part, int nsplit, int B, int NB,
                                    int Pe, int ext, double* __restrict__ gram) {
  const int b = blockIdx.x;
  const int NBD = ext ? NB - 1 : NB;
  const int npair = NBD * (NBD + 1) / 2;
  const size_t slot = nys::BatchLayout::slot_doubles_for(ext != 0, NB, NBD);
  double* E = gram + (size_t)b * Pe * Pe;
  for (int e = threadIdx.x; e < npair * 64; e += blockDim.x) {
    const int q = e >> 6, w = e & 63, lane = w >> 1, j = w & 1;
    int I = 0, rem = q;
    while (rem >= NBD - I) {
      rem -= NBD - I;
      ++I;
    }
    const int J = I + rem;
    double s = 0.0;
    for (int sp = 0; sp < nsplit; ++sp) s += part[((size_t)sp * B + b) * slot + e];
    const int r = I * 8 + (lane >> 2), c = J * 8 + 2 * (lane & 3) + j;
    if (r < Pe && c < Pe) {
      if (I == J && r > c) continue;   // diagonal block: each pair once
      E[(size_t)r * Pe + c] = s;
      E[(size_t)c * Pe + r] = s;
    }
  }
  if (!ext) return;
  const int me = Pe - 2;
  const size_t xo = (size_t)npair * 64;
  // D^T g (column me) and D^T r (column me + 1): row 8F + gid, lanes gid*4 + tig
  for (int t = threadIdx.x; t < 2 * me; t += blockDim.x) {
    const int row = t >> 1, which = t & 1, F = row >> 3, gid = row & 7;
    double s = 0.0;
    for (int sp = 0; sp < nsplit; ++sp) {
      const double* ex = part + ((size_t)sp * B + b) * slot + xo;
      for (int tig = 0; tig < 4; ++tig) s += ex[(F * 32 + gid * 4 + tig) * 2 + which];
    }
    E[(size_t)row * Pe + me + which] = s;
    E[(size_t)(me + which) * Pe + row] = s;
  }
  if (threadIdx.x < 3) {
    const int k = threadIdx.x;   // gg, gr, rr: rows are lanes 0..3 (gid 0)
    double s = 0.0;
    for (int sp = 0; sp < nsplit; ++sp) {
      const double* sc = part + ((size_t)sp * B + b) * slot + xo + (size_t)NBD * 64;
      for (int tig = 0; tig < 4; ++tig) s += sc[tig * 3 + k];
    }
    const int r = k == 2 ? me + 1 : me, c = k == 0 ? me : me + 1;
    E[(size_t)r * Pe + c] = s;
    E[(size_t)c * Pe + r] = s;
  }
}

template <int NB, int NO, bool EXT>
int launch_gram(const double* psi, const double* coef, const double* forcing, int n_c, int B,
                const BatchLayout& L, double* part, cudaStream_t st) {
  // SPLIT = 2 (two warps per instance, 128 registers each) measured slower on
  // B200 for NB = 9: 4.15 ms vs 3.33 ms (doubled combine + Psi reads, spills)
  constexpr int SPLIT = 1;
  constexpr int WARPS = nys::kBatchWarps * SPLIT;
  auto kern = batch_gram_kernel<NB, NO, WARPS, SPLIT, EXT>;
  const size_t smem = (size_t)kStages * nys::kBatchChunkKs * NO * NB * 32 * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return nys_host::record_cuda(e);
  dim3 grid((B + nys::kBatchWarps - 1) / nys::kBatchWarps, L.nsplit);
  kern<<<grid, WARPS * 32, smem, st>>>(psi, coef, forcing, n_c, B, L.ks_per_split, L.m_eff + 1,
                                       part);
  nys_host::count_launches(1);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

template <int NO>
int dispatch_nb(int NB, bool ext, const double* psi, const double* coef, const double* forcing,
                int n_c, int B, const BatchLayout& L, double* part, cudaStream_t st) {
#define NYS_NB(N)                                                                \
  case N:                                                                        \
    return ext ? launch_gram<N, NO, true>(psi, coef, forcing, n_c, B, L, part, st) \
               : launch_gram<N, NO, false>(psi, coef, forcing, n_c, B, L, part, st);
  switch (NB) {
    case 1: return launch_gram<1, NO, false>(psi, coef, forcing, n_c, B, L, part, st);
    NYS_NB(2)
    NYS_NB(3)
    NYS_NB(4)
    NYS_NB(5)
    NYS_NB(6)
    NYS_NB(7)
    NYS_NB(8)
    NYS_NB(9)
    default: return NYS_EUNSUPPORTED;
  }
#undef NYS_NB
}

}  // namespace

namespace nys_host {
int launch_batch_unpack(const double* part, int nsplit, int B, int NB, int Pe, double* gram,
                        cudaStream_t st) {
  const int ext = ((Pe - 2) % 8 == 0) && NB >= 2;   // BatchLayout::ext
  batch_unpack_kernel<<<B, 256, 0, st>>>(part, nsplit, B, NB, Pe, ext, gram);
  count_launches(1);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}
}  // namespace nys_host

extern "C" size_t nys_batch_gram_workspace_bytes(int n_c, int m_eff, int p, int B) {
  BatchLayout L = BatchLayout::make(n_c, m_eff, p, B);
  return L.ws_bytes();
}

extern "C" int nys_batch_gram_f64(const double* landmarks, int m, const double* W, int ldw,
                                  int m_eff, double sigma2, int p, const double* pts, int n_c,
                                  const double* coef, const double* forcing, int B,
                                  double* gram_ext, void* workspace, size_t workspace_bytes,
                                  void* stream) {
  if (m < 1 || m_eff < 1 || m_eff > m || ldw < m_eff || p < 1 || p > 2 || n_c < 1 || B < 0 ||
      !(sigma2 > 0.0))
    return NYS_EINVAL;
  if (B == 0) return NYS_OK;
  BatchLayout L = BatchLayout::make(n_c, m_eff, p, B);
  if (L.NB > nys::kBatchMaxNB) return NYS_EUNSUPPORTED;
  if (workspace == nullptr || workspace_bytes < L.ws_bytes()) return NYS_EWORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* psi = L.psi(workspace);
  double* part = L.part(workspace);
  int rc = nys_host::launch_psi_pack(landmarks, m, W, ldw, m_eff, sigma2, p, pts, n_c, L.NB,
                                     L.rows_pad(), psi, st);
  if (rc) return rc;
  rc = (p == 1) ? dispatch_nb<2>(L.NB, L.ext, psi, coef, forcing, n_c, B, L, part, st)
                : dispatch_nb<3>(L.NB, L.ext, psi, coef, forcing, n_c, B, L, part, st);
  if (rc) return rc;
  if (gram_ext != nullptr) return nys_host::launch_batch_unpack(part, L.nsplit, B, L.NB, m_eff + 2,
                                                                gram_ext, st);
  return NYS_OK;
}
