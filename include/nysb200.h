/*
 * nysb200 -- C ABI of the B200 (sm_100a) Nystrom LS-SVM ODE hot path.
 *
 * Drop-in boundary for the reference package `nysode` (arXiv 2510.04094,
 * /root/reference/pkg/src/nysode).  The reference has no FFI layer: its seam is
 * the Python solver API, so each entry point below replaces the numeric core
 * of one reference function (cited per entry).  The Python host mirror
 * (paper_2510_04094_b200/{nystrom,linear,newton}.py) keeps the reference's
 * signatures, callables and exceptions and binds this ABI through ctypes
 * (INTEGRATION.md shows the binding).
 *
 * Conventions (all entry points):
 *   - every pointer argument is CUDA device memory owned by the caller
 *     (torch tensors on the host side), row-major, fp64 unless stated;
 *   - work is enqueued on `stream` (a cudaStream_t passed as void*; NULL =
 *     legacy default stream); nothing synchronises the host;
 *   - return value is an nys_status (NYS_OK = 0); per-instance numerical
 *     outcomes go to `info` arrays (NYS_INFO_*), mirroring the reference's
 *     exceptions (SingularSystemError, FloatingPointError, Newton errors);
 *   - no allocation: scratch comes from a caller workspace sized by the
 *     matching *_workspace_bytes() query;
 *   - re-entrant; no global state beyond cached device attributes.
 */
#ifndef NYSB200_H
#define NYSB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NYS_ABI_VERSION 1

enum nys_status {
  NYS_OK = 0,
  NYS_EINVAL = 1,      /* argument out of range (reference: ValueError)        */
  NYS_ECUDA = 2,       /* CUDA launch / runtime error                           */
  NYS_EWORKSPACE = 3,  /* workspace too small                                   */
  NYS_EUNSUPPORTED = 4 /* shape outside the compiled kernel variants            */
};

enum nys_info {
  NYS_INFO_OK = 0,
  NYS_INFO_SINGULAR = 1,   /* exact zero pivot   (linear.py:148-151 LinAlgError)  */
  NYS_INFO_NONFINITE = 2,  /* non-finite result  (linear.py:152-153)              */
  NYS_INFO_DIVERGED = 3,   /* Newton ||F|| > 1e12 (newton.py:298-299)             */
  NYS_INFO_MAXITERS = 4,   /* Newton budget hit  (newton.py:345-348)              */
  NYS_INFO_DEGENERATE = 5  /* landmarks within 1e-12 (nystrom.py:145-146)         */
};

int nys_abi_version(void);
const char* nys_status_string(int status);
/* last CUDA error string seen by this thread (diagnostics only) */
const char* nys_last_cuda_error(void);
/* number of kernels this library has launched in the process (evidence for
 * benchmark launch counts) */
unsigned long long nys_launch_count(void);
/* Pipeline plumbing (no reference equivalent): replay CUDA graph A on `stream`,
 * wait for `in_event` (or, if NULL, for the work already on `caller`, recorded
 * into `caller_event`), replay graph B, record `done` and make `caller` wait on
 * it.  Graph arguments are cudaGraphExec_t handles, the others cudaStream_t /
 * cudaEvent_t. */
int nys_replay_pair(void* stream, void* exec_a, void* in_event, void* exec_b, void* done,
                    void* caller, void* caller_event);

/* Host staging of one SingleSolvePipeline call (the reference's callers hold
 * NumPy arrays: linear.py:90-137 samples the spec on the host).  Upload: on
 * stream `copy`, after `free_ev` (null: no wait), bytes from pinned host `src`
 * to device `dst`; `ready` is recorded behind the copy and `caller` waits on it.
 * Download: `free_ev` (null: none) is recorded on `stream`, then bytes from
 * device `src` to pinned host `dst_host`.  Streams / events are cudaStream_t /
 * cudaEvent_t handles; nothing synchronises the host. */
int nys_stage_upload(void* dst, const void* src, size_t bytes, void* copy, void* free_ev,
                     void* ready, void* caller);
int nys_stage_download(void* dst_host, const void* src, size_t bytes, void* stream, void* free_ev);

/* ------------------------------------------------------------------------
 * (i) Landmark eigendecomposition.  Replaces nystrom.build_feature_map
 * (nystrom.py:136-160) + NystromFeatureMap._scaled_vectors (nystrom.py:120-121).
 * Omega = K(L, L); Householder tridiagonalisation + Cuppen divide and conquer
 * (one CTA for m <= 68; one 8-CTA thread-block cluster exchanging through
 * DSMEM for 68 < m <= 256, then a multi-SM back-transform; implicit QL above
 * 256); eigenpairs sorted descending; keep s > max(drop_tol * s_0, 0).
 *   eigvals  [m]     descending (entries >= m_eff are the dropped ones)
 *   eigvecs  [m*m]   column k = eigenvector k (row-major m x m)
 *   W        [m*m]   W[:, k] = eigvecs[:, k] / sqrt(s_k) for k < m_eff, 0 else
 *   m_eff    [1]     int32, device
 *   info     [1]     int32, NYS_INFO_DEGENERATE if two landmarks coincide
 * ------------------------------------------------------------------------ */
size_t nys_landmark_eig_workspace_bytes(int m);
int nys_landmark_eig_f64(const double* landmarks, int m, double sigma2, double drop_tol,
                         double* eigvals, double* eigvecs, double* W, int* m_eff,
                         int* info, void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------
 * Feature rows.  Replaces NystromFeatureMap.feature_matrix (nystrom.py:123-127):
 *   out[i*ldo + k] = sum_s dK^ell(L_s, pts_i)/dt^ell * W[s*ldw + k],  k < m_eff
 * ------------------------------------------------------------------------ */
int nys_feature_matrix_f64(const double* landmarks, int m, const double* W, int ldw,
                           int m_eff, double sigma2, int ell, const double* pts, int n_pts,
                           double* out, int ldo, void* stream);

/* ------------------------------------------------------------------------
 * Batched prediction.  Replaces PrimalModel.predict (linear.py:47-53) for B
 * models sharing one feature map:
 *   out[b*ldo + i] = Psi_ell(pts_i) . x[b*ldx + 0 : m_eff]  (+ x[b*ldx+m_eff] if ell == 0)
 * ------------------------------------------------------------------------ */
int nys_predict_f64(const double* landmarks, int m, const double* W, int ldw, int m_eff,
                    double sigma2, int ell, const double* pts, int n_pts,
                    const double* x, int ldx, int B, double* out, int ldo, void* stream);

/* ------------------------------------------------------------------------
 * (ii-a) Fused feature + Gram, one ODE.  Replaces the numeric core of
 * linear.assemble (linear.py:103-133): for constraint rows i in
 * [row_begin, row_end) forms, in registers only,
 *   D_i = phi^(p)(t_i) - sum_k f_k(t_i) phi^(p-k)(t_i),  g_i = -f_p(t_i),  r_i
 * and writes the extended Gram  E = [D g r]^T [D g r]  ((m_eff+2)^2, row-major)
 * so E[:m_eff,:m_eff] = D^T D, E[:m_eff, m_eff] = D^T g, E[:m_eff, m_eff+1] = D^T r,
 * E[m_eff, m_eff] = g^T g, E[m_eff, m_eff+1] = g^T r.  The n x m feature
 * matrices never reach memory.  Row ranges make row sharding possible (the
 * partial E of disjoint ranges sum to the full E).
 *   coef    [p * n_c]   coef[(k-1)*n_c + i] = f_k(pts_i)
 *   forcing [n_c]
 * ------------------------------------------------------------------------ */
size_t nys_fused_gram_workspace_bytes(int n_c, int m, int m_eff, int p);
int nys_fused_gram_f64(const double* landmarks, int m, const double* W, int ldw, int m_eff,
                       double sigma2, int p, const double* pts, const double* coef,
                       const double* forcing, int n_c, int row_begin, int row_end,
                       double* gram_ext, void* workspace, size_t workspace_bytes,
                       void* stream);

/* ------------------------------------------------------------------------
 * (ii-b) Batched extended Gram for B ODEs sharing grid, landmarks and sigma
 * (config 2).  Same output as (ii-a) per instance, but the per-order features
 * Psi_0..Psi_p are formed once (the reference's own per-order order,
 * linear.py:103-112) and each instance only pays its row combine + Gram.
 *   coef    [B * p * n_c],  forcing [B * n_c],  gram_ext [B * (m_eff+2)^2]
 * gram_ext may be NULL when only the packed partials are wanted by
 * nys_batch_kkt_solve_f64 (they live in the workspace).
 * ------------------------------------------------------------------------ */
size_t nys_batch_gram_workspace_bytes(int n_c, int m_eff, int p, int B);
int nys_batch_gram_f64(const double* landmarks, int m, const double* W, int ldw, int m_eff,
                       double sigma2, int p, const double* pts, int n_c,
                       const double* coef, const double* forcing, int B,
                       double* gram_ext, void* workspace, size_t workspace_bytes,
                       void* stream);

/* ------------------------------------------------------------------------
 * (iii) KKT assembly + solve, batched.  Replaces linear.assemble's block
 * layout (linear.py:123-133) and linear.solve (linear.py:140-158): LU with
 * partial pivoting + one refinement step, per instance.
 *   gram_ext [B * (m_eff+2)^2]  (from ii-a / ii-b)
 *   Ac       [n_cond * m_eff]    condition rows (shared), beta [n_cond]
 *   values   [B * n_cond]
 *   x        [B * side], side = m_eff + 1 + n_cond: (omega, b, lambda)
 *   M, rhs   optional outputs (NULL to skip): [B * side^2], [B * side]
 *   info     [B] int32
 * ------------------------------------------------------------------------ */
int nys_kkt_solve_f64(const double* gram_ext, int m_eff, int n_cond, const double* Ac,
                      const double* beta, const double* values, double gamma, int B,
                      double* x, int* info, double* M, double* rhs, void* workspace,
                      size_t workspace_bytes, void* stream);
size_t nys_kkt_workspace_bytes(int m_eff, int n_cond, int B);

/* (iii-b) Same, reading the packed Gram partials that nys_batch_gram_f64 left
 * in `batch_workspace` (saves the dense gram_ext round trip). */
int nys_batch_kkt_solve_f64(const void* batch_workspace, int n_c, int m_eff, int p,
                            int n_cond, const double* Ac, const double* beta,
                            const double* values, double gamma, int B, double* x,
                            int* info, void* stream);

/* ------------------------------------------------------------------------
 * KKT certificate pieces (linear.check_kkt, linear.py:161-189) without
 * materialising D:  e_i = D_i . omega + g_i b - r_i  over rows [0, n_c).
 * ------------------------------------------------------------------------ */
int nys_ode_residual_f64(const double* landmarks, int m, const double* W, int ldw, int m_eff,
                         double sigma2, int p, const double* pts, const double* coef,
                         const double* forcing, int n_c, const double* x, double* e,
                         void* stream);

/* ------------------------------------------------------------------------
 * (v) Newton-KKT for nonlinear first-order ODEs, batched over instances that
 * share grid / landmarks (config 3).  Replaces newton._residual
 * (newton.py:128-147), _jacobian_analytic + np.linalg.solve(J, -F)
 * (newton.py:160-211, 307) by a Schur complement onto (omega, b, lambda): the
 * Jacobian's y-block is diagonal (newton.py:210).  The driver loop, damping,
 * gamma continuation and retry ladder (newton.py:279-412) run on the host
 * (paper_2510_04094_b200/newton.py) around these stream-ordered calls.
 * Unknown layout per instance: X[b*ldx + (omega[m_eff], b, lambda[n_cond], y[n_c])].
 * idx[nb] lists the instances to process (device int32).
 * Nonlinearity: family mode f = g + alpha y^2 + beta sin y (g [B*n_c],
 * alpha/beta [B], fy = fyy = NULL) or sampled mode (g = f, fy, fyy [B*n_c]
 * evaluated by the caller at the current y).
 * ------------------------------------------------------------------------ */
int nys_transpose_f64(const double* A, int rows, int cols, double* AT, void* stream);
size_t nys_newton_pack_doubles(int m_eff, int n_c);
int nys_newton_pack_f64(const double* landmarks, int m, const double* W, int ldw, int m_eff,
                        double sigma2, const double* pts, int n_c, double* packed, void* stream);
/* F [B*ldx], norm [B] (= max|F|, NaN when f or e1 is non-finite), aux [B*3*n_c]
 * (f_y, f_yy e1, 1 + f_y^2 - f_yy e1), work [B*2*n_c] */
int nys_newton_residual_f64(const double* S0, const double* S1, const double* S0T,
                            const double* S1T, int m_eff, int n_c, const double* g,
                            const double* fy, const double* fyy, const double* alpha,
                            const double* beta, const double* Ac, const double* betac,
                            const double* vals, int n_cond, const double* gamma,
                            const double* X, int ldx, const int* idx, int nb, double* F,
                            double* norm, double* aux, double* work, void* stream);
/* Batched step halving (newton.py:305-318): norms[t * nb + j] = max|F| at the
 * trial X[idx[j]] + trial_alphas[t] * D[idx[j]] for t < ntrial, bit-identical to
 * forming the candidate with nys_newton_step_f64 and calling nys_newton_residual_f64;
 * nothing else is written.  scratch: nys_newton_trial_scratch_bytes (row-range
 * partial sums of every instance and trial). */
size_t nys_newton_trial_scratch_bytes(int m_eff, int n_c, int nb, int ntrial);
int nys_newton_trial_norms_f64(const double* S0T, const double* S1T, int m_eff, int n_c,
                               const double* g, const double* fy, const double* fyy,
                               const double* alpha, const double* beta, const double* Ac,
                               const double* betac, const double* vals, int n_cond,
                               const double* gamma, const double* X, const double* D, int ldx,
                               const int* idx, int nb, const double* trial_alphas, int ntrial,
                               double* norms, void* scratch, size_t scratch_bytes, void* stream);
/* reduced system K [nb * nz^2], rz [nb * nz], nz = m_eff + 1 + n_cond (DMMA weighted Grams) */
int nys_newton_reduced_f64(const double* packed, int m_eff, int n_c, const double* aux,
                           const double* F, int ldx, const double* gamma, const double* Ac,
                           const double* betac, int n_cond, const int* idx, int nb, double* K,
                           double* rz, void* stream);
/* Same, with the row range of every instance split over several CTAs (about two
 * per SM) whose partial sums are added in fixed order: workspace of
 * nys_newton_reduced_workspace_bytes(m_eff, n_c, nb) bytes (0 = one CTA per instance). */
size_t nys_newton_reduced_workspace_bytes(int m_eff, int n_c, int nb);
int nys_newton_reduced_ws_f64(const double* packed, int m_eff, int n_c, const double* aux,
                              const double* F, int ldx, const double* gamma, const double* Ac,
                              const double* betac, int n_cond, const int* idx, int nb, double* K,
                              double* rz, void* workspace, size_t workspace_bytes, void* stream);
/* ---- second-order nonlinear ODEs y'' = f(t, y, y') (newton2.cu) ------------------
 * samples [6][B][n_c]: f, f_y, f_y', f_yy, f_yy', f_y'y' at (t, y, S1 omega) of
 * instance b (host-evaluated reference callables).  aux [B][6][n_c]; workspace of
 * nys_newton2_workspace_bytes(m_eff, n_c, nb) bytes for both calls.  The packed
 * Psi_0..Psi_2 come from nys_newton2_pack_f64. */
size_t nys_newton2_workspace_bytes(int m_eff, int n_c, int nb);
size_t nys_newton2_pack_doubles(int m_eff, int n_c);
int nys_newton2_pack_f64(const double* landmarks, int m, const double* W, int ldw, int m_eff,
                         double sigma2, const double* pts, int n_c, double* packed, void* stream);
int nys_newton2_residual_f64(const double* S0T, const double* S1T, const double* S2T, int m_eff,
                             int n_c, const double* samples, int B, const double* Ac,
                             const double* betac, const double* vals, int n_cond,
                             const double* gamma, const double* X, int ldx, const int* idx,
                             int nb, double* F, double* norm, double* aux, void* workspace,
                             size_t workspace_bytes, void* stream);
int nys_newton2_reduced_f64(const double* packed, int m_eff, int n_c, const double* aux,
                            const double* F, int ldx, const double* gamma, const double* Ac,
                            const double* betac, int n_cond, const int* idx, int nb, double* K,
                            double* rz, void* workspace, size_t workspace_bytes, void* stream);
int nys_newton2_step_f64(const double* S0T, const double* S1T, const double* S2T, int m_eff,
                         int n_c, int n_cond, const double* aux, const double* F,
                         const double* dz, const double* gamma, const double* X, double* D,
                         double* Xc, const double* alpha, int ldx, const int* idx, int nb,
                         void* stream);
/* batched dense LU (partial pivoting) solve, one system of side n <= 96 per slot */
int nys_lu_solve_f64(double* M, double* rhs, int n, int nb, double* out, int* info, void* stream);
/* D[b] = (dz, dy) (compute_delta = 1) and Xc[b] = X[b] + alpha[b] * D[b] */
int nys_newton_step_f64(const double* S0, const double* S1, int m_eff, int n_c, int n_cond,
                        const double* aux, const double* F, const double* dz,
                        const double* gamma, const double* X, double* D, double* Xc,
                        const double* alpha, int ldx, const int* idx, int nb, int compute_delta,
                        void* stream);

/* Device-resident Newton loop (replaces newton._solve_once, newton.py:279-349,
 * for the separable family f = g + alpha y^2 + beta sin y, p = 1): one CTA per
 * instance idx[j] runs the convergence / divergence checks, the Schur-reduced
 * system, its LU, the y back-substitution, the step-halving line search
 * (damped != 0: alpha = shrink^k, k < halvings, accept the first finite trial
 * norm <= the current one, else shrink^halvings) and the residual at every
 * trial with no host round trip.  X[idx[j]] holds the start point on entry
 * and the final iterate on exit; norms[j][0..iters[j]] the residual max-norms
 * (the trace); status[j] 0 converged / 1 max iterations / 2 diverged /
 * 3 singular.  work: nb * nys_newton_solve_once_work_doubles doubles. */
size_t nys_newton_solve_once_work_doubles(int m_eff, int n_c, int n_cond);
/* diagnostics: when dev_buf != NULL, later persistent Newton launches write
 * per-instance phase clocks there ([nb][8]: residual + line search, reduced
 * system, LU, step, -, trials); NULL turns it off */
void nys_newton_persist_profile(long long* dev_buf);
int nys_newton_solve_once_f64(const double* S0, const double* S1, const double* S0T,
                              const double* S1T, const double* packed, int m_eff, int n_c,
                              const double* g, const double* alpha, const double* beta,
                              const double* Ac, const double* betac, const double* vals,
                              int n_cond, const double* gamma, const double* tol, double* X,
                              int ldx, const int* idx, int nb, int damped, double shrink,
                              int halvings, int max_iters, double* work, size_t work_bytes,
                              double* norms, int* iters, int* status, void* stream);

/* The whole retry ladder on the device (replaces newton.solve_nonlinear's
 * ladder, newton.py:376-412, and _solve_with_continuation, newton.py:352-373):
 * per instance, one CTA runs rung 1 (X0c, undamped), 2 (X0c, damped), 3 (X0l,
 * undamped), 4 (X0l, damped) until one converges, else rung 5: damped stages
 * at gamma = 1, 1e2, 1e4 below gamma[idx] with tol 1e-8 (1 + g) (MaxIters
 * tolerated, divergence / singularity ends the instance), each handing
 * (omega, b, lambda = 0, y = Psi_0 omega + b) on, then gamma[idx] itself.
 * X0c / X0l [nb][ldx] (indexed by slot j): the constant and linearised
 * starts; X[idx[j]] the final iterate; rung[2 nb]: rung[j] 1..5 the rung that
 * produced status[j] / norms[j][0..iters[j]] (the trace of that last
 * _solve_once), rung[nb + j] the Newton iterations over every rung and stage. */
int nys_newton_ladder_f64(const double* S0, const double* S1, const double* S0T,
                          const double* S1T, const double* packed, int m_eff, int n_c,
                          const double* g, const double* alpha, const double* beta,
                          const double* Ac, const double* betac, const double* vals, int n_cond,
                          const double* gamma, const double* tol, const double* X0c,
                          const double* X0l, double* X, int ldx, const int* idx, int nb,
                          double shrink, int halvings, int max_iters, double* work,
                          size_t work_bytes, double* norms, int* iters, int* status, int* rung,
                          void* stream);

/* ---- ridge leverage scores -------------------------
 * Replaces the exact branch of nystrom.ridge_leverage_scores (nystrom.py:58-70,
 * n <= _LEVERAGE_EXACT_LIMIT = 4000): scores[i] = diag(Omega (Omega + n*ridge*I)^-1)_i,
 * Omega = kernel_matrix(RBF(sigma2), 0, grid, grid), clipped below at 1e-300
 * (nystrom.py:81).  Computed as 1 - n*ridge*diag(A^-1) from a tiled DMMA Cholesky
 * A = L L^T fused with X = L^-1.  info[0] = NYS_INFO_SINGULAR when A is not
 * numerically positive definite (the reference's dgesv would still return; the
 * host mirror raises np.linalg.LinAlgError).  The sketch branch for n > 4000
 * (nystrom.py:71-80) is not served by this entry. */
#define NYS_LEVERAGE_MAX_N 8192
size_t nys_leverage_workspace_bytes(int n);
int nys_leverage_scores_f64(const double* grid, int n, double sigma2, double ridge, double* scores,
                            int* info, void* ws, size_t ws_bytes, void* stream);

/* Sketch branch of ridge_leverage_scores (nystrom.py:71-80, n > 4000), in two
 * calls so the host can size the second from the rank of the first:
 *   nys_pchol_rbf_f64: pivoted Cholesky W ~ G G^T of the c x c sketch kernel
 *     matrix W = K(x, x) (x = grid[idx] from the host, nystrom.py:72-74), stopped
 *     when the largest remaining diagonal is <= tol or after cap columns;
 *     G is cap x c (row k = column k of the factor); out[0] = rank r,
 *     out[1] = 1 if it converged before cap.
 *   nys_leverage_sketch_f64: eigh of G^T G (r <= 256) with the reference's
 *     keep rule vals > 1e-12 vals.max() (:75-76), A = C V_k / sqrt(vals_k)
 *     (:77), scores = diag(A (A^T A + n ridge I)^-1 A^T) (:78-79) clipped at
 *     1e-300; info[0] = NYS_INFO_SINGULAR if the r x r system is not SPD. */
int nys_pchol_rbf_f64(const double* x, int c, double sigma2, double tol, int cap, double* G,
                      int* out, void* stream);
size_t nys_leverage_sketch_workspace_bytes(int n, int c, int r);
int nys_leverage_sketch_f64(const double* grid, int n, const double* x, int c, double sigma2,
                            double ridge, const double* G, int r, double* scores, int* info,
                            void* ws, size_t ws_bytes, void* stream);

/* Kernel-space Gram split in two (config 4, m_eff + 2 > 72): the first part
 * needs no eigenvectors, so it can run concurrently with nys_landmark_eig_f64
 * (max_ctas < #SMs leaves SMs for it); the second projects with W.
 *   K [(m+2)^2]: kernel-space extended Gram [G g r]^T [G g r], G the
 *                order-combined kernel rows (same sums as nys_fused_gram_f64)
 *   gram_ext [(m_eff+2)^2] = W_ext^T K W_ext */
size_t nys_kspace_gram_workspace_bytes(int n_c, int m, int max_ctas);
int nys_kspace_gram_f64(const double* landmarks, int m, double sigma2, int p, const double* pts,
                        const double* coef, const double* forcing, int n_c, int row_begin,
                        int row_end, int max_ctas, double* K, void* ws, size_t ws_bytes,
                        void* stream);
size_t nys_kspace_project_workspace_bytes(int m, int m_eff);
int nys_kspace_project_f64(const double* K, int m, const double* W, int ldw, int m_eff,
                           double* gram_ext, void* ws, size_t ws_bytes, void* stream);

/* Large landmark sets (m > 512; the m = n full-feature comparator,
 * baselines.py:170-194): after nys_pchol_rbf_f64 on the landmarks (Omega ~ G G^T,
 * rank r <= 256), the kept eigenpairs of G G^T from the r x r problem G^T G:
 * eigvals [r] descending, eigvecs / W [m x ldv] (columns >= m_eff zero),
 * drop rule s > max(drop_tol s_0, 0) as nystrom.py:150-154. */
size_t nys_landmark_eig_compressed_workspace_bytes(int r);
int nys_landmark_eig_compressed_f64(const double* G, int m, int r, double drop_tol,
                                    double* eigvals, double* eigvecs, double* W, int ldv,
                                    int* m_eff, int* info, void* ws, size_t ws_bytes,
                                    void* stream);

/* Extended Gram E = [D g r]^T [D g r] from explicit feature matrices
 * psi[(ell * n + i) * m_eff + k] = Psi_ell(pts_i)[k], ell = 0..p (the large-m
 * path of linear.assemble, linear.py:103-133). */
size_t nys_explicit_gram_workspace_bytes(int n, int m_eff);
int nys_explicit_gram_f64(const double* psi, int n, int m_eff, int p, const double* coef,
                          const double* forcing, double* gram_ext, void* ws, size_t ws_bytes,
                          void* stream);

/* Dense symmetric eigendecomposition of an explicit n x n matrix (n <= 256,
 * divide and conquer as nys_landmark_eig_f64): eigenvalues descending,
 * eigvecs[i*n + k] = V[i][k], W[:, k] = V[:, k] / sqrt(s_k) for the kept
 * s_k > drop_tol * s_0, m_eff = number kept. */
size_t nys_sym_eig_workspace_bytes(int n);
int nys_sym_eig_f64(const double* A, int n, double drop_tol, double* eigvals, double* eigvecs,
                    double* W, int* m_eff, int* info, void* workspace, size_t workspace_bytes,
                    void* stream);

#ifdef __cplusplus
}
#endif
#endif /* NYSB200_H */
