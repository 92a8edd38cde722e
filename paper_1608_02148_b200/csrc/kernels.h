// kernels.h -- internal launchers of the B200 rsvd library (host-callable).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <atomic>

#include "common.cuh"

namespace rsvd {

// Kernels launched by this library (all launchers add to it; rank-group threads share it).
extern std::atomic<int64_t> g_kernel_launches;

// Stream-K bookkeeping in the context's 4096-word flag array: [0, grid) the
// DMMA / TF32 passes' "partial published" flags, [2048, 2048 + 4 grid) the
// Ozaki passes' arrival counters, kEpochSlot the device-side launch epoch
// (advanced by the kernel that precedes each pass, so CUDA-graph replays of a
// captured call see a new epoch every time).
constexpr int kEpochSlot = 4095;

// ---- K2/K3 streaming passes (gemm_pass.cu)
struct GemmCall {
  const void* A; int64_t lda; bool a_f32; bool trans;
  const double* B; int64_t ldb;          // K x N, N % 16 == 0, zero-padded columns
  double* C; int64_t ldc;                // output M x Nout
  double* P;                             // split partials (>= gemm_partial_bytes)
  unsigned* flags; unsigned epoch;       // >= 4096 flag words, zero-initialised once (epoch: unused, see kEpochSlot)
  const double* center;                  // per A-column mean (nullable)
  const double* rscale;                  // per A-column 1/s.d. (nullable)
  int64_t M, K; int N, Nout;
  int grid;                              // persistent stream-K grid (<= #SMs)
};
int gemm_choose_grid(int64_t M, int64_t K, int num_sms);
size_t gemm_partial_bytes(int N, int grid);
cudaError_t gemm_pass(const GemmCall& c, cudaStream_t st);


// ---- FP32 A on tcgen05 (pass_tf32.cu): 3-term TF32 split, TMEM accumulators
struct Tf32Call {
  const float* A; int64_t lda; bool trans;   // A row-major FP32 (16-byte aligned rows)
  const double* B; int64_t ldb;              // K x N panel, FP64 (split to TF32 hi/lo inside)
  double* C; int64_t ldc;                    // M x Nout output, FP64
  double* P;                                 // stream-K partials + FP64 drain sums (tf32_partial_bytes)
  unsigned* flags; unsigned epoch;           // as GemmCall
  float* split;                              // 2 * K * tf32_n(N) floats scratch
  int64_t M, K; int N, Nout; int grid;
};
bool tf32_pass_supported(const void* A, int64_t lda);
int tf32_n(int Np);
size_t tf32_partial_bytes(int Np, int num_sms);   // 2 x grid x 128 x tf32_n(Np) doubles
size_t tf32_split_bytes(int64_t K, int Np);
cudaError_t tf32_pass(const Tf32Call& c, cudaStream_t st);

// ---- CholeskyQR panel path (cholqr.cu)
// G (Np x Np, ld ldg) = S^T S for S (rows x Np, ld lds): gram_partial over
// gram_ctas() row chunks into `partial` (>= gram_partial_bytes) + fixed-order reduce.
int gram_ctas(int64_t rows, int num_sms);
size_t gram_partial_bytes(int Np, int num_sms);
cudaError_t launch_gram(const double* S, int64_t lds, int64_t rows, int Np, double* partial, double* G, int ldg,
                        int num_sms, cudaStream_t st, Pred pr = Pred{});
// G = R^T R (l x l leading block of G, ld ldg) and R^-1, by symmetric elimination
// on [G | I]; R, Rinv npad x npad (ld npad, zero padded; R nullable); flag |= flag_bit
// on breakdown (pivot <= 1e-13 of its original diagonal, or non-finite).
cudaError_t launch_chol_aug(const double* G, int ldg, int l, int npad, double* R, double* Rinv, int* flag,
                            int flag_bit, cudaStream_t st, Pred pr = Pred{});
// C (rows x Nout, ld ldc) = S (rows x Np, ld lds) * T (Np x Np, ld ldt); C may alias S.
// upper: T is upper triangular (skips the zero blocks).
cudaError_t launch_panel_apply(const double* S, int64_t lds, int64_t rows, int Np, const double* T, int64_t ldt,
                               double* C, int64_t ldc, int Nout, bool upper, int num_sms, cudaStream_t st,
                               Pred pr = Pred{});

// ---- passes by Ozaki-scheme int8 slices on tcgen05 (pass_ozaki.cu)
#define OZ_S 7                                   // FP64 A: 8-bit digits per element (A: 56-bit two's complement, X: 54-bit balanced)
#define OZ_S32 3                                 // FP32 A: 3 digits (A: 24-bit two's complement, X: 22-bit balanced)
struct OzakiA {                                  // A sliced once per call: m x (ldn/128) x s x 128 int8 + exponents
  int8_t* slices;
  int* erow;                                     // E_r: max_j |f(a_rj)| < 2^{E_r}, one per row
  unsigned* emax;                                // max_r E_r + 4096 (biased, atomicMax)
  int64_t m, n, ldn;
  int s;                                         // digits per element: OZ_S (FP64 A) or OZ_S32 (FP32 A)
};
size_t ozaki_a_bytes(int64_t m, int64_t n, int s);
OzakiA ozaki_layout_a(void* buf, int64_t m, int64_t n, int s);
// slices of f(A) = (A - 1 c^T) diag(rs) (c, rs nullable; A FP64, or FP32 when f32);
// flag |= 4 on non-finite A
cudaError_t ozaki_slice_a(const OzakiA& a, const void* A, bool f32, int64_t lda, const double* c, const double* rs,
                          int* flag, cudaStream_t st);
struct OzakiCall {
  const OzakiA* a; bool trans;                   // trans: C = f(A)^T B (M = n, K = m), else C = f(A) B
  const double* B; int64_t ldb;                  // K x N panel (FP64), N = Np <= 128 (two 64-column halves above 64)
  double* C; int64_t ldc; int Nout;
  double* P; unsigned* flags; unsigned epoch;    // stream-K partials / flags as GemmCall
  unsigned epoch2;                               // second column block (N > 64)
  void* xscratch;                                // >= ozaki_x_bytes(K, min(N, 64))
  void* xscratch2;                               // second column block (N > 64), same size
  int64_t M, K; int N; int grid;
  cudaEvent_t mark, mark2;                       // nullable: both recorded after X slicing, before the pass kernel(s)
};
bool ozaki_supported(int Np);
// stream-K partials of the pass kernels: 2 slots (first / last segment) per CTA
size_t ozaki_partial_bytes(int Np, int grid);
size_t ozaki_x_bytes(int64_t K, int Np, int s);
int ozaki_x_cols(int s, int Np);                 // columns per X slice scratch (64, or 128 for FP32 A at Np = 128)
cudaError_t ozaki_pass(const OzakiCall& c, cudaStream_t st);

// ---- K1 Omega (omega.cu)
cudaError_t launch_omega(int64_t n, int64_t l, int64_t ldo, int64_t ncols_zero, int sdist,
                         uint64_t seed, uint64_t stream, bool f32_round, bool out_f32, void* out,
                         cudaStream_t st);

// ---- small / panel kernels (panel.cu)
// Column sums of A (m x n): out[j] = sum_i f(A[i][j]) with f = identity (mode 0)
// or (a - c_j)^2 (mode 1).  Deterministic two-level reduction.
cudaError_t launch_colsum(const void* A, int64_t lda, bool a_f32, int64_t m, int64_t n, int mode,
                          const double* c, double* partial, double* out, cudaStream_t st, int* launches);
size_t colsum_partial_bytes(int64_t m, int64_t n);
// c = sum / m  (mode 0); rs = 1/sqrt(sumsq/(m-1)) and s (mode 1)
cudaError_t launch_colstat_finish(double* v, int64_t n, double m_global, int mode, double* s_out,
                                  cudaStream_t st);

// Cholesky of the l x l Gram G (ld ldg): R upper with G = R^T R, Rinv = R^-1 into
// ldr x ldr buffers (zero padded to npad); flag |= 1 on breakdown.
cudaError_t launch_chol_inv(const double* G, int ldg, int l, int npad, double* R, double* Rinv,
                            int* flag, int flag_bit, cudaStream_t st);
// C (l x l) = A (l x l) * B (l x l), all ld = lda; single CTA.
cudaError_t launch_small_matmul(const double* A, const double* B, double* C, int l, int ld,
                                cudaStream_t st);
// Householder leaves: rows [leaf*rows_base + min(leaf, rem) ...] of Y (ld ldy, l
// columns).  Explicit Q overwrites the leaf rows; R (l x l, diag >= 0) goes to
// Rstack + leaf*l*l (ld l).
int leaf_rows_cap(int l);
// Register-column Householder QR of one small panel (M <= 1024 rows, l <= 32):
// Q in place, R (diag >= 0, row-major l x l); cudaErrorNotSupported if it does not fit.
cudaError_t launch_hqr_small(double* Y, int64_t ldy, int64_t M, int l, double* R, cudaStream_t st);
cudaError_t launch_hqr_leaves(double* Y, int64_t ldy, int64_t M, int l, int64_t nleaves,
                              double* Rstack, cudaStream_t st, Pred pr = Pred{});
// Q rows of each leaf <- Q rows * S_leaf, S_leaf = rows [leaf*l, leaf*l+l) of S (ld lds).
cudaError_t launch_tsqr_combine(double* Y, int64_t ldy, int64_t M, int l, int64_t nleaves,
                                const double* S, int64_t lds, cudaStream_t st, Pred pr = Pred{});

// The whole local TSQR of an M x l panel in one cooperative launch (panel.cu):
// level i reduces lev[i].buf (lev[i].M rows, ld lev[i].ld) in lev[i].P leaves,
// stacking their R factors in lev[i+1].buf (cur for the last level, ld l);
// the final leaf factors cur (Mc rows, ld ldc) into R (l x l, ld l), copied to
// Rout (ld ldro) if non-null; then Q is formed downwards in every level's buf.
// bar: 2 kTsqrMaxLev + 2 device words, zero before the first launch; the
// kernel leaves them zero (ticket + per-phase completion counters).
constexpr int kTsqrMaxLev = 24;
struct TsqrLevel { double* buf; int64_t ld, M, P; };
struct TsqrArgs {
  TsqrLevel lev[kTsqrMaxLev];
  int nlev, l;
  double* cur; int64_t ldc, Mc;
  double* R; double* Rout; int64_t ldro;
  unsigned* bar;
};
cudaError_t launch_tsqr_fused(const TsqrArgs& a, int num_sms, cudaStream_t st, Pred pr = Pred{});

// One-sided Jacobi SVD of X = R^T (R upper l x l, ld ldr): X J = W Sigma (jacobi.cu).
// Outputs: sigma (l, descending), W (ldo x ldo) = U~, J (ldo x ldo), zero outside
// their leading l x l blocks (l <= ldo <= 128).
// flag |= 2 if the sweep cap was hit, 4 on non-finite input.  scratch: device
// buffer of jacobi_scratch_bytes(l) (rotation log + ranks).
size_t jacobi_scratch_bytes(int l);
cudaError_t launch_jacobi(const double* R, int ldr, int l, double* sigma, double* W, double* J,
                          int ldo, int* flag, int* sweeps, void* scratch, cudaStream_t st);

// Sign convention (reading R9): sgn[i] = -1 iff the largest-|.| entry of V(:,i)
// (lowest index on ties) is negative.
cudaError_t launch_sign_from_v(const double* V, int64_t ldv, int64_t n, int l, double* sgn,
                               cudaStream_t st);
// X(:, j) *= sgn[j] for j < l (rows r, ld ldx)
cudaError_t launch_scale_cols(double* X, int64_t ldx, int64_t rows, int l, const double* sgn,
                              cudaStream_t st);
// dst (rows x cols, ldd, f32 or f64) = src (ld lds) ; optional per-column factor
cudaError_t launch_copy_out(const double* src, int64_t lds, int64_t rows, int cols, void* dst,
                            int64_t ldd, bool dst_f32, const double* colfac, cudaStream_t st,
                            Pred pr = Pred{});
cudaError_t launch_fill(double* p, int64_t count, double v, cudaStream_t st);
// Y (rows x ld) columns [l, npad) set to zero
cudaError_t launch_zero_cols(double* Y, int64_t ld, int64_t rows, int l, int npad, cudaStream_t st);
// rpca: eig[i] = d[i]^2 / (m-1)
cudaError_t launch_pca_eig(const double* d, int k, double m, void* eig, bool f32, cudaStream_t st);
// rpca outputs (Alg. 6; reading R32 of DESIGN.md)
cudaError_t launch_colstat_scale(const double* ss, int64_t n, double m_global, double* rs, double* s, cudaStream_t st);
cudaError_t launch_total_var(const double* ss, const double* rs, int64_t n, double m_global, double* out,
                             cudaStream_t st);
cudaError_t launch_pca_stats(const double* d, int k, double m_global, const double* total, void* eig, void* sdev,
                             void* ratio, void* cum, bool f32, cudaStream_t st);
// dst[j] = src[j] (mode 0), 1/src[j] (1), src[j]/sqrt(v-1) (2), v (3)
cudaError_t launch_vec_map(const void* src, bool src_f32, int64_t n, int mode, double v, double* dst, cudaStream_t st);
// X (rows x npad, FP64, zero padded) = src (rows x cols)
cudaError_t launch_copy_in(const void* src, bool src_f32, int64_t lds, int64_t rows, int cols, int npad, double* X,
                           int64_t ldx, cudaStream_t st);
// status words: *flag |= bits (predicated); end-of-call sticky status
cudaError_t launch_flag_or(int* flag, int bits, cudaStream_t st, Pred pr);
cudaError_t launch_status_finish(const int* flag, int* sticky, int fallback_bit, cudaStream_t st);
// plain-launched helpers that order later PDL kernels behind non-kernel stream work
cudaError_t launch_zero_words(int* p, int n, cudaStream_t st);
cudaError_t launch_stream_fence(cudaStream_t st);
// in-process rank groups: out = in[0] op in[1] ... (fixed rank order)
constexpr int kMaxGroup = 16;
struct GroupPtrs { const double* p[kMaxGroup]; };
cudaError_t launch_group_reduce(const GroupPtrs& in, int nranks, int64_t n, int op_max, double* out, cudaStream_t st);
// Finite check of flags: flag |= 4 if any non-finite among v[0..n)
cudaError_t launch_check_finite(const double* v, int64_t n, int* flag, cudaStream_t st);

// ---- pivoted QR / interpolative decomposition (qrcp.cu), Alg. id / rid / rcur, reading R31
// Column-contiguous W (column c = rows doubles at W + c*ld), `steps` Businger-Golub
// pivots into perm; W is overwritten.  Z != null: Z (steps x ncols, ld ldz) = the
// ID interpolation matrix (Z(:, P) = [I, S_kk^-1 S_12]); flag |= flag_bit if S_kk
// is singular (rank < steps).  Cooperative launch, one CTA per SM.
size_t qrcp_scratch_bytes(int64_t ncols, int steps, int num_sms);
cudaError_t launch_qrcp(double* W, int64_t ld, int rows, int64_t ncols, int steps, int64_t* perm, double* Z,
                        int64_t ldz, void* scratch, int* flag, int flag_bit, int num_sms, cudaStream_t st);
cudaError_t launch_gather_cols(const double* A, int64_t lda, int64_t m, const int64_t* J, int k, double* C,
                               int64_t ldc, cudaStream_t st);
cudaError_t launch_gather_rows(const double* A, int64_t lda, int64_t n, const int64_t* I, int k, double* R,
                               int64_t ldr, double* Rt, int64_t ldt, cudaStream_t st);
// In-place GEPP of a tall row-contiguous panel (m x l, ld): Y <- the permuted unit
// lower factor L of Y = L U (Alg. 3 "[L, ~] = lu(Y)"); flag |= flag_bit on a zero pivot.
size_t lu_scratch_bytes(int64_t m, int num_sms);
cudaError_t launch_lu_rows(double* Y, int64_t ld, int64_t m, int l, void* scratch, int* flag, int flag_bit,
                           int num_sms, cudaStream_t st);
size_t zq_partial_bytes(int k, int num_sms);
cudaError_t launch_zq(const double* Z, int64_t ldz, const double* Q, int64_t ldq, int64_t n, int k, double* partial,
                      double* W, int ldw, int num_sms, cudaStream_t st);
cudaError_t launch_rtsolve(const double* W, int ldw, const double* S, int lds, int k, double* U, int64_t ldu,
                           cudaStream_t st);

// ---- wide plans, l > 120 (wide.cu; reading R34): cooperative launches, one CTA per SM
// G + s I = R^T R (l x l leading block of G; s = shift_c trace(G), 0 when shift_c <= 0) and
// R^-1 into npad x npad (ld npad, zero padded); breakdown as launch_chol_aug (flag |= flag_bit;
// the column is dropped).
size_t chol_wide_scratch_bytes(int npad);
cudaError_t launch_chol_wide(const double* G, int ldg, int l, int npad, double* R, double* Rinv, void* scratch,
                             int* flag, int flag_bit, double shift_c, int num_sms, cudaStream_t st);
// One-sided Jacobi SVD of X = R^T, X J = W Sigma, for any l (outputs as launch_jacobi, ldo >= l).
size_t jacobi_wide_scratch_bytes(int l);
cudaError_t launch_jacobi_wide(const double* R, int ldr, int l, double* sigma, double* W, double* J, int ldo,
                               int* flag, int* sweeps, void* scratch, int num_sms, cudaStream_t st);
// Householder QR of the saved rows x l panel (ld npad; overwritten) into Q (ld npad) and R
// (npad x npad upper, diag >= 0, nullable), only when (*flag & bit); clears the bit, sets ran_bit.
// part: >= num_sms x npad doubles; scratch: >= 3 npad doubles.  Cooperative launch.
cudaError_t launch_hqr_wide(double* Wsaved, int64_t rows, int l, int npad, double* Q, double* R, double* part,
                            void* scratch, int* flag, int bit, int ran_bit, int num_sms, cudaStream_t st);
// Bt (r x ldb) = diag(dl) V^T (V n x r, ld ldv), columns >= n zero
cudaError_t launch_scale_transpose(const double* V, int64_t ldv, int64_t n, int r, const double* dl, double* Bt,
                                   int64_t ldb, cudaStream_t st);
// IALM steps (10)-(11) with L materialised (contiguous m x n, total = m n); partial[b], b < nblocks
cudaError_t launch_ialm_update_dense(const double* A, double* S, double* Z, double* Mnext, const double* L,
                                     int64_t total, double inv_mu, double mu, double lam, double inv_mu_next,
                                     double* partial, int nblocks, cudaStream_t st);

// ---- IALM (ialm.cu), FP64, reading R17-R23 of DESIGN.md
// M = A - S + Z * inv_mu ;  optional: norms of A (||A||_F^2 partials, max|A|)
cudaError_t launch_ialm_form_m(const double* A, const double* S, const double* Z, int64_t ld,
                               int64_t m, int64_t n, double inv_mu, double* M, cudaStream_t st);
// Fused update with L = U diag(dl) V^T (rank r <= 128, never materialised):
//   S = shrink(A - L + Z inv_mu, lam inv_mu);  E = A - L - S;  Z += mu E;
//   M_next = A - S + Z * inv_mu_next;  partial[b] = sum E^2 (per block).
cudaError_t launch_ialm_update(const double* A, double* S, double* Z, double* Mnext, int64_t ld,
                               int64_t m, int64_t n, const double* U, int64_t ldu,
                               const double* V, int64_t ldv, const double* dl, int r,
                               double inv_mu, double mu, double lam, double inv_mu_next,
                               double* partial, int nblocks, cudaStream_t st);
// L = U diag(dl) V^T materialised (final output)
cudaError_t launch_lowrank_materialise(const double* U, int64_t ldu, const double* V, int64_t ldv,
                                       const double* dl, int r, int64_t m, int64_t n, double* L,
                                       int64_t ldl, cudaStream_t st);
// Z = A / dual ; partials of ||A||_F^2 and max|A| (per block)
cudaError_t launch_ialm_init(const double* A, int64_t ld, int64_t m, int64_t n, double* sumsq_part,
                             double* max_part, int nblocks, cudaStream_t st);
cudaError_t launch_scale_copy(const double* A, int64_t ld, int64_t m, int64_t n, double f,
                              double* Z, cudaStream_t st);
cudaError_t launch_reduce_blocks(const double* part, int nb, int op_max, double* out, cudaStream_t st);
int ialm_blocks();
// number of partials launch_ialm_update writes for n columns and nblocks (<= nblocks)
int ialm_partials(int64_t n, int nblocks);
// dl_t = max(d_t - inv_mu, 0) for t < k (d descending); *l_out = #{d_t > inv_mu}
cudaError_t launch_ialm_threshold(const double* d, int k, double inv_mu, double* dl, double* l_out,
                                  cudaStream_t st);

}  // namespace rsvd
