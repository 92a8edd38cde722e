/*
 * rsvd_b200.h -- C ABI of the B200-native randomized SVD hot path
 * (arXiv 1608.02148, the `rsvd` package).  sm_100a only.
 *
 * Everything here is plain C: pointers (host or device, as stated per
 * argument) and sizes.  No torch types.  The Python binding
 * (paper_1608_02148_b200/__init__.py) marshals arguments only.
 *
 * Conventions common to every entry point
 * ---------------------------------------
 *  * Matrices are ROW-MAJOR with an explicit leading dimension (elements, not
 *    bytes): element (i, j) of X lives at X[i*ldx + j], ldx >= #columns.
 *  * "device" = memory of the context's CUDA device (cudaMalloc / torch).
 *    The library never frees caller memory; it owns only its workspace.
 *  * All work is enqueued on the context's stream (the one given to
 *    rsvd_create) and the calls return as soon as it is enqueued: no host
 *    synchronisation, so a call can be captured into a CUDA graph.  Outputs
 *    are valid once the stream has reached the end of the call.  Numerical
 *    failures found on the device (non-finite values, the Jacobi sweep cap,
 *    a rank-deficient pivoted QR in rid/rcur) are recorded in the context's
 *    status word and reported by rsvd_sync().  The CholeskyQR breakdown of
 *    a rank-deficient sketch is handled on the device (Householder TSQR
 *    fallback), never reported as an error.  Exceptions:
 *    rsvd_rrpca (its IALM loop decides on the host, one read per iteration)
 *    and rsvd_run_host (host buffers) return after a stream synchronisation
 *    with the numerical status of the call.
 *  * Validation errors (RSVD_EINVAL / RSVD_EUNSUPPORTED) are returned BEFORE
 *    any launch and write nothing.  rsvd_last_error() gives the message for
 *    the last non-OK status, or a warning (e.g. nu > k clamped).
 *  * dtype RSVD_F64: A, u, d, v are double.  RSVD_F32: A, u, d, v are float;
 *    the power-scheme panels, the small SVD and the orthonormalisations run
 *    in FP64 (reading R12).
 *  * Distributed mode (after rsvd_comm_init with nranks > 1): A is row-sharded,
 *    this rank holds rows [row_offset, row_offset + m_local) of the m_global x n
 *    matrix; u returns this rank's rows, d and v are replicated.  Requires
 *    m_global >= n.  Collectives: NCCL allreduce(sum) of the n x l partials
 *    (Z = A^T Q, B^T = A^T Q), of l x l Gram matrices and of column sums.
 */
#ifndef RSVD_B200_H
#define RSVD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RSVD_OK = 0,
  RSVD_EINVAL = 1,        /* bad argument (nothing launched, nothing written) */
  RSVD_ENOMEM = 2,        /* workspace allocation failed                      */
  RSVD_ECUDA = 3,         /* CUDA runtime error (message in rsvd_last_error)  */
  RSVD_ENCCL = 4,         /* NCCL error                                       */
  RSVD_ENUMERIC = 5,      /* non-finite intermediate or Jacobi sweep cap hit  */
  RSVD_EUNSUPPORTED = 6   /* valid request outside this build's envelope      */
} rsvd_status;

/* Random test matrix distributions, PAPER.md:417-430 (§2.3) and the
 * `sdist = c("normal", "unif", "rademacher")` argument. */
typedef enum { RSVD_NORMAL = 0, RSVD_UNIF = 1, RSVD_RADEMACHER = 2 } rsvd_sdist;
typedef enum { RSVD_F64 = 0, RSVD_F32 = 1 } rsvd_dtype;

typedef struct rsvd_ctx rsvd_ctx;   /* opaque: device, stream, workspace, comm */

/* Create a context bound to `device` and `cuda_stream` (a cudaStream_t; NULL
 * = legacy default stream).  The stream must outlive the context. */
rsvd_status rsvd_create(rsvd_ctx** ctx, int device, void* cuda_stream);
rsvd_status rsvd_destroy(rsvd_ctx* ctx);
const char* rsvd_last_error(const rsvd_ctx* ctx);
const char* rsvd_version(void);

/* Wait for the context's stream, then return (and clear) the numerical status
 * accumulated by the calls completed since the last rsvd_sync: RSVD_OK, or
 * RSVD_ENUMERIC with the reason in rsvd_last_error (non-finite input or
 * intermediate, Jacobi sweep cap, numerical rank < k in rid / rcur). */
rsvd_status rsvd_sync(rsvd_ctx* ctx);

/* NCCL plumbing (multi-GPU, one process per GPU).  rank 0 calls
 * rsvd_nccl_unique_id (writes 128 bytes to host memory `out`), the caller
 * broadcasts them (e.g. torch.distributed), and every rank calls
 * rsvd_comm_init.  nranks == 1 is accepted and means single-GPU. */
rsvd_status rsvd_nccl_unique_id(void* out128);
rsvd_status rsvd_comm_init(rsvd_ctx* ctx, const void* nccl_unique_id128, int nranks, int rank);

/* In-process rank groups: `nranks` contexts (2 <= nranks <= 16, on the same
 * device or on devices with peer access), one host thread each, run the
 * row-sharded path together with the collectives replaced by fixed-rank-order
 * device reductions over the group's staging buffers (every rank gets
 * bitwise the same sums).  Same semantics as rsvd_comm_init; used to run the
 * distributed algorithm on one GPU (tests) and for multi-GPU without NCCL.
 * rsvd_group_destroy after every member context is destroyed.  A member that
 * fails inside a call aborts the group: the others return RSVD_ENCCL. */
typedef struct rsvd_group rsvd_group;
rsvd_status rsvd_group_create(rsvd_group** group, int nranks);
rsvd_status rsvd_group_destroy(rsvd_group* group);
rsvd_status rsvd_comm_init_group(rsvd_ctx* ctx, rsvd_group* group, int rank);

/* Input matrix descriptor.  `A` is caller-owned DEVICE memory, read-only,
 * row-major m_local x n with leading dimension lda >= n; it must stay valid
 * until the call returns.  Single GPU: m_global == m_local, row_offset == 0. */
typedef struct {
  int32_t dtype;          /* rsvd_dtype */
  const void* A;
  int64_t m_local, n, lda;
  int64_t m_global, row_offset;
} rsvd_matrix;

/* rsvd parameters: rsvd(A, k, nu = NULL, nv = NULL, p = 10, q = 2,
 * sdist = "normal") (§3.6).
 *   k      target rank, 1 <= k <= min(m, n) (reading R10)
 *   nu,nv  number of left/right singular vectors to return; values
 *          > k are clamped to k with a warning; 0 = not formed
 *   p      oversampling, l = min(k + p, min(m, n)) (Alg. 4 step 1);
 *          l <= 4096 (RSVD_EUNSUPPORTED above).  l <= 120 runs the tcgen05
 *          Ozaki / TF32 passes and the shared-memory panels and Jacobi;
 *          120 < l <= 4096 runs a "wide plan" (reading R34): DMMA passes over
 *          column blocks of 128, shifted CholeskyQR3 panels, a grid-wide
 *          Jacobi.  A sketch rank-deficient to working precision (k + p >
 *          rank(A)) takes a device-side Householder fallback on one GPU; a
 *          row-sharded wide plan reports it as RSVD_ENUMERIC at rsvd_sync
 *   q      subspace iterations (Alg. 2)
 *   seed, stream  counter-based Omega (reading R1)
 *   center  1 = implicit column centring of A (rpca, Alg. 6)
 *   scale   1 = implicit column scaling by the (centred) column s.d.
 *   power   power scheme between the sketch and the final QR: 0 = subspace
 *           iterations with QR (Alg. 2, default), 1 = the direct
 *           scheme Y = (A A^T)^q A Omega without normalisation (Alg. 1,
 *           P:343-362; "not recommended in practice"), 2 = normalized
 *           power iterations with pivoted LU (Alg. 3; single GPU, l <= 128);
 *           RSVD_EINVAL otherwise */
typedef struct {
  int32_t k, nu, nv, p, q;
  int32_t sdist;          /* rsvd_sdist */
  uint64_t seed, stream;
  int32_t center, scale;
  int32_t power;
} rsvd_params;

/* Fill the defaults of P:708: nu = nv = k, p = 10, q = 2, normal, seed 0,
 * stream 0, no centring/scaling. */
void rsvd_params_default(rsvd_params* prm, int32_t k);

/* Randomized SVD, Alg. 5 on top of Alg. 4 rqb.
 *   u  DEVICE, m_local x nu, row-major, ldu >= nu (NULL iff nu == 0): this
 *      rank's rows of U(:, 1:nu)
 *   d  DEVICE, k values of the dtype of A, descending (replicated)
 *   v  DEVICE, n x nv, row-major, ldv >= nv (NULL iff nv == 0); V is NOT
 *      transposed (replicated)
 * Sign convention (reading R9): the largest-|.| entry of each V column is
 * positive; the same flip is applied to U. */
rsvd_status rsvd_run(rsvd_ctx* ctx, const rsvd_matrix* A, const rsvd_params* prm,
                     void* u, int64_t ldu, void* d, void* v, int64_t ldv);

/* Device workspace (bytes) the library will own for rsvd_run on this matrix
 * and these parameters (panels, Ozaki slices of A, TSQR fallback scratch);
 * HOST out-param.  Validation as rsvd_run; nothing is allocated. */
rsvd_status rsvd_workspace_bytes(rsvd_ctx* ctx, const rsvd_matrix* A, const rsvd_params* prm, size_t* bytes);

/* rsvd_run on HOST buffers (end to end): A is read from host memory (pinned
 * or pageable; m x n row-major, lda), copied to a device staging buffer the
 * context owns, factored, and u, d, v are copied back to HOST memory
 * (layouts as rsvd_run).  With a communicator A holds this rank's m_local
 * rows (m_global / row_offset as rsvd_run; u gets the same rows).  Blocks until the results are in
 * host memory; returns the numerical status of the call (as rsvd_sync). */
rsvd_status rsvd_run_host(rsvd_ctx* ctx, const rsvd_matrix* A, const rsvd_params* prm,
                          void* u, int64_t ldu, void* d, void* v, int64_t ldv);

/* Randomized QB decomposition, Alg. 4, with the final QR
 * of reading R3.  Q: DEVICE m_local x l (ldq >= l), this rank's rows;
 * Bt: DEVICE n x l (ldb >= l), B^T = A^T Q, replicated.  l = min(k+p, min(m,n)).
 * Results in the dtype of A. */
rsvd_status rsvd_rqb(rsvd_ctx* ctx, const rsvd_matrix* A, const rsvd_params* prm,
                     void* Q, int64_t ldq, void* Bt, int64_t ldb);

/* Randomized column interpolative decomposition, Alg. rid
 * with Alg. id applied to B = Q^T A of rqb (reading R31):
 * A ~ C Z with C = A(:, J), Z(:, J) = I_k.  Pivots: Businger-Golub pivoted QR
 * of B stopped after k steps.  FP64, m >= n; rows may be
 * distributed (C holds this rank's rows, Z and J are replicated).
 *   C  DEVICE m_local x k (ldc >= k)   skeleton columns
 *   Z  DEVICE k x n (ldz >= n)         interpolation matrix
 *   J  DEVICE int64 k                  column indices, in pivot order
 * RSVD_ENUMERIC if the numerical rank of B is < k (S(1:k,1:k) singular). */
rsvd_status rsvd_rid(rsvd_ctx* ctx, const rsvd_matrix* A, const rsvd_params* prm,
                     void* C, int64_t ldc, void* Z, int64_t ldz, int64_t* J);

/* Randomized CUR decomposition, Alg. rcur: rid, then the
 * pivoted QR of C^T gives the row indices I = P(1:k); R = A(I, :) and
 * U = Z pinv(R) with pinv(R) = Q_R S_R^-T from the Householder QR R^T =
 * Q_R S_R (reading R31).  A ~ C U R.  FP64, single GPU, m >= n.
 *   C  DEVICE m x k (ldc >= k);  U  DEVICE k x k (ldu >= k);
 *   R  DEVICE k x n (ldr >= n);  J, I  DEVICE int64 k (column / row indices) */
rsvd_status rsvd_rcur(rsvd_ctx* ctx, const rsvd_matrix* A, const rsvd_params* prm,
                      void* C, int64_t ldc, void* U, int64_t ldu, void* R, int64_t ldr,
                      int64_t* J, int64_t* I);

/* Randomized PCA, Alg. 6, interface
 * rpca(A, k, center = TRUE, scale = TRUE, retx = TRUE, p = 10, q = 2)
 * (P:1381-1398): rsvd on X = (A - 1 c^T) diag(1/s) (centring / scaling never
 * materialised; prm->center, prm->scale select them, rsvd_rpca_params_default
 * sets both as the paper does).  Every output is DEVICE memory in the dtype
 * of A, caller-owned, and NULL = not computed:
 *   rotation  n x k (ldr >= k)        W = V, the principal directions
 *   eigvals   k                       Lambda = d^2 / (m - 1)          (Eq. P:1322)
 *   sdev      k                       sqrt(eigvals)
 *   x         m_local x k (ldx >= k)  scores Z = X W = U diag(d)      (Eq. PCs; retx)
 *   center    n                       column means c
 *   scale     n                       column s.d. s (1 for constant columns)
 *   loadings  n x k (ldl >= k)        L = W Lambda^{1/2}
 *   x_white   m_local x k (ldw >= k)  whitened PCs z_i / sqrt(lambda_i) (
 *                                     reading R32: the text's X L is taken as Z Lambda^{-1/2})
 *   var_ratio k                       lambda_i / sum_{all} lambda
 *   var_cum   k                       cumulative proportion of variance (summary())
 *   total_var 1                       sum of all eigenvalues = trace of the
 *                                     covariance (correlation) matrix, from the
 *                                     column sums of squares (one extra pass over
 *                                     A when scale is FALSE) */
typedef struct {
  void* rotation; int64_t ldr;
  void* eigvals;
  void* sdev;
  void* x; int64_t ldx;
  void* center;
  void* scale;
  void* loadings; int64_t ldl;
  void* x_white; int64_t ldw;
  void* var_ratio;
  void* var_cum;
  void* total_var;
} rsvd_pca_out;
void rsvd_rpca_params_default(rsvd_params* prm, int32_t k);   /* rsvd defaults + center = scale = 1 */
rsvd_status rsvd_rpca(rsvd_ctx* ctx, const rsvd_matrix* A, const rsvd_params* prm, const rsvd_pca_out* out);

/* rsvd_rpca on HOST buffers (end to end; with a communicator A holds this rank's rows and m_global / row_offset place them): A and every non-NULL
 * output of `out` are HOST memory (layouts as rsvd_rpca); A is staged into a
 * device buffer the context owns and the outputs are copied back.  Blocks;
 * returns the numerical status of the call (as rsvd_sync). */
rsvd_status rsvd_rpca_host(rsvd_ctx* ctx, const rsvd_matrix* A, const rsvd_params* prm, const rsvd_pca_out* out);

/* Out-of-sample projection, predict() of the rpca object: the
 * scores of new rows, out = ((Anew - 1 c^T) diag(1/s)) W, computed by the same
 * pass kernels as the sketch.  Anew: rsvd_matrix (DEVICE, m_new x n, dtype of
 * the outputs); rotation DEVICE n x k (ldr); center, scale DEVICE n (nullable
 * = no centring / scaling; scale entries must be nonzero); out DEVICE
 * m_new x k (ldo >= k).  1 <= k <= 128. */
rsvd_status rsvd_rpca_predict(rsvd_ctx* ctx, const rsvd_matrix* Anew, int32_t k, const void* rotation, int64_t ldr,
                              const void* center, const void* scale, void* out, int64_t ldo);

/* Randomized robust PCA by inexact ALM, Alg. 7, with the
 * readings R17-R23, R30 of DESIGN.md (mu_0 = 1.25/||A||_2, fresh Omega stream t per
 * iteration, mu <- min(1.5 mu, 1e7 mu_0)).
 *   lambda  <= 0 selects max(m, n)^-1/2
 *   tol     stop when ||A - L - S||_F / ||A||_F < tol
 *   k       > 0: fixed target rank k (R22), needs k <= min(m, n), k + p <= 4096;
 *           0: adaptive target rank -- k = 2 at step (1), then step (7)
 *           predict_rank (Remark 1): l = max(1, #{sigma_i > 1/mu}),
 *           k <- l + 1 if l < k else min(l + ceil(0.05 min(m, n)), min(m, n)),
 *           capped at min(m, n) (at 4096 - p when min(m, n) > 4096); the
 *           deterministic SVD of Remark 2 is used while k > min(m, n)/4 if
 *           min(m, n) <= 4096, else the randomized SVD is kept with a warning (R30)
 * FP64 only.  L, S: DEVICE m_local x n (ld == n), caller-owned; A contiguous.
 *   iters, final_residual: HOST out-params (nullable)
 *   trace: HOST, nullable, 4*maxiter doubles per iteration: (residual, l, mu,
 *          target rank k used by that iteration's rsvd)
 * Errors: RSVD_EINVAL (null, k < 0, maxiter < 1, tol <= 0), RSVD_EUNSUPPORTED
 * (FP32, strided A/L/S, k beyond the envelope), RSVD_ENUMERIC (||A||_2 = 0). */
typedef struct {
  double lambda, tol;
  int32_t maxiter;
  int32_t k, p, q;
  int32_t sdist;
  uint64_t seed;
  int32_t rand;   /* 1 (default): randomized SVD in step (6); 0: the deterministic
                     truncated SVD (P:1743-1744 rand = FALSE), computed as rsvd with
                     l = min(m, n), q = 0 (Q spans the whole column space, so the
                     SVD of B is the exact SVD; a wide plan when min(m, n) > 120); needs
                     min(m, n) <= 4096.  With k = 0
                     the same switch happens whenever the predicted k > min(m, n)/4
                     (Remark 2). */
} rsvd_rrpca_params;
void rsvd_rrpca_params_default(rsvd_rrpca_params* prm);
rsvd_status rsvd_rrpca(rsvd_ctx* ctx, const rsvd_matrix* A, const rsvd_rrpca_params* prm,
                       void* L, void* S, int64_t ld, int32_t* iters, double* final_residual,
                       double* trace);

/* rsvd_rrpca on HOST buffers (end to end; with a communicator A holds this rank's rows and m_global / row_offset place them): A, L, S HOST memory
 * (m x n, ld == n); staged through device buffers the context owns. */
rsvd_status rsvd_rrpca_host(rsvd_ctx* ctx, const rsvd_matrix* A, const rsvd_rrpca_params* prm,
                            void* L, void* S, int64_t ld, int32_t* iters, double* final_residual,
                            double* trace);

/* Random test matrix alone (K1): writes the n x l matrix
 * Omega to DEVICE `out` (row-major, ldo >= l) in `dtype` (FP32 = round to
 * nearest of the FP64 value).  Exposed for bit-exact parity tests. */
rsvd_status rsvd_omega(rsvd_ctx* ctx, int64_t n, int64_t l, int32_t sdist, uint64_t seed,
                       uint64_t stream, int32_t dtype, void* out, int64_t ldo);

/* Per-kernel timing of the last calls (CUDA events on the context stream,
 * enabled by rsvd_set_profiling(ctx, 1); 2 = only the pass kernels, kind 0
 * on one call and kind 1 on the next, for the least event overhead).  kind: 0 = sketch/power pass A.X,
 * 1 = transposed pass A^T.X (incl. its split reduction), 2 = panel
 * orthonormalisation, 3 = small SVD, 4 = other, 5 = Ozaki slicing of A
 * (FP64 inputs on the tensor-core path, once per call), 6 = Ozaki slicing of
 * the panel X before each pass (kinds 0 / 1 then time the pass kernels
 * alone).  Returns accumulated
 * milliseconds and launch count since the last reset (HOST out-params). */
rsvd_status rsvd_set_profiling(rsvd_ctx* ctx, int enable);
rsvd_status rsvd_profile(rsvd_ctx* ctx, int kind, double* total_ms, int64_t* count,
                         double* bytes);
rsvd_status rsvd_profile_reset(rsvd_ctx* ctx);
/* Number of kernels this library launched since the last reset. */
int64_t rsvd_launch_count(const rsvd_ctx* ctx);

/* Diagnostics of the last rsvd-family call (HOST out-param, n <= 4 slots):
 * out[0] = one-sided Jacobi sweeps, out[1] = 1 if the Householder TSQR
 * fallback after a CholeskyQR breakdown ran (as of the last rsvd_sync), out[2] = kernel
 * launches since the last rsvd_profile_reset, out[3] = passes run on the
 * FP64 Ozaki tensor-core path since the context was created (RSVD_FP64_PATH=dmma
 * in the environment at rsvd_create selects the FP64 DMMA path instead). */
rsvd_status rsvd_stats(const rsvd_ctx* ctx, int64_t* out, int n);

#ifdef __cplusplus
}
#endif
#endif /* RSVD_B200_H */
