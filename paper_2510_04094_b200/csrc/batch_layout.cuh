// Workspace layout shared by nys_batch_gram_f64 and nys_batch_kkt_solve_f64.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

namespace nys {

constexpr int kBatchWarps = 8;      // instances per CTA (one warp each)
constexpr int kBatchChunkKs = 8;    // k-steps (4 rows each) per TMA chunk = 32 rows
constexpr int kBatchMaxNB = 9;      // extended width m_eff + 2 <= 72

int device_sm_count();              // cached cudaDevAttrMultiProcessorCount

struct BatchLayout {
  int n_c, m_eff, p, B;
  int NB, NO, npair;
  // ext: m_eff % 8 == 0, so the last 8-column block holds only the two extended
  // columns (g, r); the kernel then accumulates D^T g, D^T r, g.g, g.r, r.r with
  // FP64 FMAs instead of 9 mostly-empty DMMA blocks
  bool ext;
  int NBD;
  int nsplit, ks_per_split, nks_pad;

  static BatchLayout make(int n_c, int m_eff, int p, int B) {
    BatchLayout L{};
    L.n_c = n_c;
    L.m_eff = m_eff;
    L.p = p;
    L.B = B;
    L.NB = (m_eff + 2 + 7) / 8;
    L.NO = p + 1;
    L.npair = L.NB * (L.NB + 1) / 2;
    L.ext = (m_eff % 8 == 0) && L.NB >= 2;
    L.NBD = L.ext ? L.NB - 1 : L.NB;
    const int nks = (n_c + 3) / 4;
    const int nchunks = (nks + kBatchChunkKs - 1) / kBatchChunkKs;
    // row splits: fill whole waves of one CTA per SM (the kernel is register
    // bound to 1 CTA/SM); prefer fewer splits when equally good.
    const int sms = device_sm_count();
    const int ctas = (B + kBatchWarps - 1) / kBatchWarps;
    int best = 1;
    double best_eff = 0.0;
    for (int s = 1; s <= 8 && s <= nchunks; ++s) {
      int cps = (nchunks + s - 1) / s;
      double work = (double)ctas * s * cps;            // chunk-units incl. padding
      double waves = (double)((ctas * s + sms - 1) / sms);
      double eff = ((double)ctas * nchunks) / (waves * sms * cps);
      (void)work;
      if (eff > best_eff * 1.02) {
        best_eff = eff;
        best = s;
      }
    }
    L.nsplit = best;
    L.ks_per_split = ((nchunks + best - 1) / best) * kBatchChunkKs;
    L.nks_pad = L.ks_per_split * best;
    return L;
  }
  int rows_pad() const { return nks_pad * 4; }
  size_t psi_doubles() const { return (size_t)nks_pad * NO * NB * 32; }
  // per-instance partial: upper block triangle of the DMMA blocks (MMA layout),
  // then in ext mode [NBD][32 lanes][g, r] and [32 lanes][gg, gr, rr]
  __host__ __device__ static size_t slot_doubles_for(bool ext, int NB, int NBD) {
    return ext ? (size_t)NBD * (NBD + 1) / 2 * 64 + (size_t)NBD * 64 + 96
               : (size_t)NB * (NB + 1) / 2 * 64;
  }
  size_t slot_doubles() const { return slot_doubles_for(ext, NB, NBD); }
  size_t part_doubles() const { return (size_t)nsplit * B * slot_doubles(); }
  int Pe() const { return m_eff + 2; }
  size_t e_doubles() const { return (size_t)B * Pe() * Pe(); }
  size_t ws_bytes() const {
    return (psi_doubles() + part_doubles() + e_doubles()) * sizeof(double) + 256;
  }
  double* psi(void* ws) const {
    size_t a = (reinterpret_cast<size_t>(ws) + 127) & ~(size_t)127;
    return reinterpret_cast<double*>(a);
  }
  double* part(void* ws) const { return psi(ws) + psi_doubles(); }
  const double* part(const void* ws) const { return psi(const_cast<void*>(ws)) + psi_doubles(); }
  // dense extended Grams (B x Pe x Pe), filled by the unpack kernel
  double* dense(void* ws) const { return part(ws) + part_doubles(); }
};

}  // namespace nys
