// panel.cu -- panel orthonormalisation and the small (l x l) factorisations.
//
//  * chol_inv:   Cholesky of an l x l Gram and the explicit inverse of its
//                factor, for CholeskyQR2 ("[Q,~] = qr(Y)", Alg. 2 steps 2-3,
//                PAPER.md:377-378; Alg. 4 step 9).  Breakdown (pivot
//                <= 1e-13 of the original diagonal, or non-finite) sets a flag;
//                the orchestrator then re-runs with the Householder path.
//  * hqr_leaves: Householder QR of row blocks that fit in one CTA's shared
//                memory (explicit thin Q in place, R with diag >= 0): the
//                single-CTA panel QR for small panels and the leaves of TSQR.
//                Robust for exactly rank-deficient panels (config 1).
//  * tsqr_combine: Q_leaf <- Q_leaf * S_leaf, the downward sweep of TSQR.
//  * jacobi:     one-sided (Hestenes) Jacobi SVD of R_B^T in shared memory,
//                parallel round-robin ordering, one warp per column pair with
//                warp-shuffle dot products; economic SVD of B (Alg. 5 step 2,
//                P:628) via B^T = Q_B R_B.
//  * sign / copy / column statistics helpers.
#include <math.h>

#include "common.cuh"
#include "kernels.h"

namespace rsvd {

constexpr int SMEM_OPTIN = 232448;   // B200 per-block opt-in shared memory (profiles/peaks_box.json)

static cudaError_t set_smem(const void* fn, size_t bytes) {
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

// ------------------------------------------------------------------ column statistics
template <typename TA>
__global__ void colsum_kernel(const TA* __restrict__ A, int64_t lda, int64_t m, int64_t n, int mode,
                              const double* __restrict__ c, double* __restrict__ partial,
                              int64_t rows_per_chunk) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t r0 = blockIdx.y * rows_per_chunk;
  int64_t r1 = r0 + rows_per_chunk;
  if (r1 > m) r1 = m;
  if (j >= n) return;
  const double cj = (mode == 1) ? c[j] : 0.0;
  double s = 0.0;
  for (int64_t i = r0; i < r1; ++i) {
    const double a = (double)A[i * lda + j];
    s += (mode == 1) ? (a - cj) * (a - cj) : a;
  }
  partial[blockIdx.y * n + j] = s;
}

__global__ void colsum_finish_kernel(const double* __restrict__ partial, int chunks, int64_t n,
                                     double* __restrict__ out) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  double s = 0.0;
  for (int t = 0; t < chunks; ++t) s += partial[t * n + j];
  out[j] = s;
}

static int colsum_chunks(int64_t m) {
  int64_t ch = ceil_div(m, 512);
  if (ch > 256) ch = 256;
  if (ch < 1) ch = 1;
  return (int)ch;
}

size_t colsum_partial_bytes(int64_t m, int64_t n) { return (size_t)colsum_chunks(m) * n * sizeof(double); }

cudaError_t launch_colsum(const void* A, int64_t lda, bool a_f32, int64_t m, int64_t n, int mode,
                          const double* c, double* partial, double* out, cudaStream_t st, int* launches) {
  const int chunks = colsum_chunks(m);
  const int64_t rpc = ceil_div(m, chunks);
  dim3 grid((unsigned)ceil_div(n, 128), (unsigned)chunks);
  if (a_f32)
    colsum_kernel<float><<<grid, 128, 0, st>>>((const float*)A, lda, m, n, mode, c, partial, rpc);
  else
    colsum_kernel<double><<<grid, 128, 0, st>>>((const double*)A, lda, m, n, mode, c, partial, rpc); ++g_kernel_launches;
  colsum_finish_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(partial, chunks, n, out); ++g_kernel_launches;
  return cudaGetLastError();
}

__global__ void colstat_finish_kernel(double* v, int64_t n, double mg, int mode, double* s_out) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  if (mode == 0) {
    v[j] = v[j] / mg;
  } else {
    double sd = sqrt(v[j] / (mg - 1.0));
    if (!(sd > 0.0)) sd = 1.0;
    if (s_out) s_out[j] = sd;
    v[j] = 1.0 / sd;
  }
}

cudaError_t launch_colstat_finish(double* v, int64_t n, double m_global, int mode, double* s_out,
                                  cudaStream_t st) {
  colstat_finish_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(v, n, m_global, mode, s_out); ++g_kernel_launches;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ Cholesky + inverse
__global__ void __launch_bounds__(1024) chol_inv_kernel(const double* __restrict__ G, int ldg, int l,
                                                        int npad, double* __restrict__ R,
                                                        double* __restrict__ Rinv, int* flag,
                                                        int flag_bit) {
  extern __shared__ double sm[];
  double* Gs = sm;                 // l x l (ld l), becomes R (upper) in place
  double* d0 = Gs + l * l;         // original diagonal
  __shared__ int bad;
  const int tid = threadIdx.x, nt = blockDim.x;
  if (tid == 0) bad = 0;
  for (int e = tid; e < l * l; e += nt) Gs[e] = G[(e / l) * ldg + (e % l)];
  __syncthreads();
  for (int j = tid; j < l; j += nt) d0[j] = Gs[j * l + j];
  __syncthreads();
  for (int j = 0; j < l; ++j) {
    const double d = Gs[j * l + j];
    const bool brk = !(d > 1e-13 * d0[j]) || !isfinite(d);
    const double r = brk ? 1.0 : sqrt(d);
    __syncthreads();
    if (tid == 0) {
      if (brk) bad = 1;
      Gs[j * l + j] = r;
    }
    for (int c = j + 1 + tid; c < l; c += nt) Gs[j * l + c] = brk ? 0.0 : Gs[j * l + c] / r;
    __syncthreads();
    const int rem = l - j - 1;
    for (int e = tid; e < rem * rem; e += nt) {
      const int a = j + 1 + e / rem, b = j + 1 + e % rem;
      if (b >= a) Gs[a * l + b] -= Gs[j * l + a] * Gs[j * l + b];
    }
    __syncthreads();
  }
  // R (upper, zero-padded to npad) and its inverse by column back-substitution:
  // one warp per column c of X = R^-1: X[i][c] = (delta_ic - sum_{k>i} R[i][k] X[k][c]) / R[i][i]
  const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  for (int e = tid; e < npad * npad; e += nt) {
    const int a = e / npad, b = e % npad;
    if (R) R[e] = (a < l && b < l && b >= a) ? Gs[a * l + b] : 0.0;
    Rinv[e] = 0.0;
  }
  __syncthreads();
  for (int c = warp; c < l; c += nw) {
    for (int i = c; i >= 0; --i) {
      double s = 0.0;
      for (int k = i + 1 + lane; k <= c; k += 32) s += Gs[i * l + k] * Rinv[k * npad + c];
      s = warp_sum(s);
      if (lane == 0) Rinv[i * npad + c] = ((i == c ? 1.0 : 0.0) - s) / Gs[i * l + i];
      __syncwarp();
    }
  }
  __syncthreads();
  if (tid == 0 && bad) atomicOr(flag, flag_bit);
}

cudaError_t launch_chol_inv(const double* G, int ldg, int l, int npad, double* R, double* Rinv, int* flag,
                            int flag_bit, cudaStream_t st) {
  const size_t smem = ((size_t)l * l + l) * sizeof(double);
  if (smem > (size_t)SMEM_OPTIN - 1024) return cudaErrorInvalidValue;
  cudaError_t e = set_smem((const void*)chol_inv_kernel, smem);
  if (e != cudaSuccess) return e;
  chol_inv_kernel<<<1, 1024, smem, st>>>(G, ldg, l, npad, R, Rinv, flag, flag_bit); ++g_kernel_launches;
  return cudaGetLastError();
}

__global__ void small_matmul_kernel(const double* A, const double* B, double* C, int l, int ld) {
  for (int e = threadIdx.x; e < l * l; e += blockDim.x) {
    const int i = e / l, j = e % l;
    double s = 0.0;
    for (int k = 0; k < l; ++k) s += A[i * ld + k] * B[k * ld + j];
    C[i * ld + j] = s;
  }
}

cudaError_t launch_small_matmul(const double* A, const double* B, double* C, int l, int ld,
                                cudaStream_t st) {
  small_matmul_kernel<<<1, 1024, 0, st>>>(A, B, C, l, ld); ++g_kernel_launches;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ Householder leaves
constexpr int HQR_THREADS = 512;

int leaf_rows_cap(int l) {
  const int64_t avail = (SMEM_OPTIN - 1024) / (int64_t)sizeof(double) - 2 * l - 32;
  return (int)(avail / l);
}

__global__ void __launch_bounds__(HQR_THREADS) hqr_leaves_kernel(double* __restrict__ Y, int64_t ldy,
                                                                 int64_t M, int l, int64_t nleaves,
                                                                 double* __restrict__ Rstack) {
  extern __shared__ double sm[];
  const int64_t leaf = blockIdx.x;
  const int64_t rb = M / nleaves, rem = M % nleaves;
  const int b = (int)(rb + (leaf < rem ? 1 : 0));
  const int64_t r0 = leaf * rb + (leaf < rem ? leaf : rem);
  double* Ys = sm;                 // column-major, ld = b
  double* tau = Ys + (int64_t)l * b;
  double* w = tau + l;
  double* red = w + l;             // 32
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;

  for (int64_t e = tid; e < (int64_t)b * l; e += nt) {
    const int r = (int)(e / l), c = (int)(e % l);
    Ys[(int64_t)c * b + r] = Y[(r0 + r) * ldy + c];
  }
  __syncthreads();

  // ---- factorisation (LAPACK dgeqr2 / dlarfg convention, v_j = 1 implicit)
  for (int j = 0; j < l; ++j) {
    double* x = Ys + (int64_t)j * b;
    double part = 0.0;
    for (int r = j + 1 + tid; r < b; r += nt) part += x[r] * x[r];
    const double sig2 = block_sum(part, red);
    const double x0 = x[j];
    double t = 0.0, beta = x0, scal = 0.0;
    if (sig2 != 0.0) {
      const double nrm = sqrt(x0 * x0 + sig2);
      beta = -copysign(nrm, x0);                 // sign(0) = +1 => beta = -||x||
      t = (beta - x0) / beta;
      scal = 1.0 / (x0 - beta);
    }
    __syncthreads();
    for (int r = j + 1 + tid; r < b; r += nt) x[r] *= scal;
    if (tid == 0) { tau[j] = t; x[j] = beta; }
    __syncthreads();
    if (t != 0.0) {
      // apply H_j to the trailing columns; each column is owned by one warp
      for (int c = j + 1 + warp; c < l; c += nw) {
        double* y = Ys + (int64_t)c * b;
        double sdot = 0.0;
        for (int r = j + 1 + lane; r < b; r += 32) sdot += x[r] * y[r];
        sdot = warp_sum(sdot) + y[j];
        const double f = t * sdot;
        for (int r = j + 1 + lane; r < b; r += 32) y[r] -= f * x[r];
        if (lane == 0) y[j] -= f;
      }
      __syncthreads();
    }
  }

  // ---- R (upper l x l) with diag >= 0 to the stack; remember the signs in w
  for (int j = tid; j < l; j += nt) w[j] = (Ys[(int64_t)j * b + j] < 0.0) ? -1.0 : 1.0;
  __syncthreads();
  double* Rl = Rstack + leaf * (int64_t)l * l;
  for (int e = tid; e < l * l; e += nt) {
    const int i = e / l, c = e % l;
    Rl[e] = (c >= i) ? w[i] * Ys[(int64_t)c * b + i] : 0.0;
  }
  __syncthreads();

  // ---- explicit Q in place (LAPACK dorg2r), then column signs
  for (int i = l - 1; i >= 0; --i) {
    double* x = Ys + (int64_t)i * b;
    const double t = tau[i];
    if (i < l - 1 && t != 0.0) {
      if (tid == 0) x[i] = 1.0;
      __syncthreads();
      for (int c = i + 1 + warp; c < l; c += nw) {
        double* y = Ys + (int64_t)c * b;
        double sdot = 0.0;
        for (int r = i + lane; r < b; r += 32) sdot += x[r] * y[r];
        const double f = t * warp_sum(sdot);
        for (int r = i + lane; r < b; r += 32) y[r] -= f * x[r];
      }
    }
    __syncthreads();
    for (int r = i + 1 + tid; r < b; r += nt) x[r] *= -t;
    if (tid == 0) x[i] = 1.0 - t;
    for (int r = tid; r < i; r += nt) x[r] = 0.0;
    __syncthreads();
  }
  for (int64_t e = tid; e < (int64_t)b * l; e += nt) {
    const int r = (int)(e / l), c = (int)(e % l);
    Y[(r0 + r) * ldy + c] = w[c] * Ys[(int64_t)c * b + r];
  }
}

cudaError_t launch_hqr_leaves(double* Y, int64_t ldy, int64_t M, int l, int64_t nleaves, double* Rstack,
                              cudaStream_t st) {
  const int64_t bmax = ceil_div(M, nleaves);
  const size_t smem = ((size_t)bmax * l + 2 * l + 32) * sizeof(double);
  if (smem > (size_t)SMEM_OPTIN - 1024 || bmax < l) return cudaErrorInvalidValue;
  cudaError_t e = set_smem((const void*)hqr_leaves_kernel, smem);
  if (e != cudaSuccess) return e;
  hqr_leaves_kernel<<<(unsigned)nleaves, HQR_THREADS, smem, st>>>(Y, ldy, M, l, nleaves, Rstack); ++g_kernel_launches;
  return cudaGetLastError();
}

__global__ void tsqr_combine_kernel(double* __restrict__ Y, int64_t ldy, int64_t M, int l, int64_t nleaves,
                                    const double* __restrict__ S, int64_t lds) {
  extern __shared__ double sm[];
  double* Ss = sm;                 // l x l
  double* rows = Ss + l * l;       // 16 x l
  const int64_t leaf = blockIdx.x;
  const int64_t rb = M / nleaves, rem = M % nleaves;
  const int b = (int)(rb + (leaf < rem ? 1 : 0));
  const int64_t r0 = leaf * rb + (leaf < rem ? leaf : rem);
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < l * l; e += nt) Ss[e] = S[(leaf * l + e / l) * lds + (e % l)];
  for (int rc = 0; rc < b; rc += 16) {
    const int nr = (b - rc) < 16 ? (b - rc) : 16;
    __syncthreads();
    for (int e = tid; e < nr * l; e += nt) rows[e] = Y[(r0 + rc + e / l) * ldy + (e % l)];
    __syncthreads();
    for (int e = tid; e < nr * l; e += nt) {
      const int r = e / l, c = e % l;
      double s = 0.0;
      for (int k = 0; k < l; ++k) s += rows[r * l + k] * Ss[k * l + c];
      Y[(r0 + rc + r) * ldy + c] = s;
    }
  }
}

cudaError_t launch_tsqr_combine(double* Y, int64_t ldy, int64_t M, int l, int64_t nleaves, const double* S,
                                int64_t lds, cudaStream_t st) {
  const size_t smem = ((size_t)l * l + 16 * (size_t)l) * sizeof(double);
  cudaError_t e = set_smem((const void*)tsqr_combine_kernel, smem);
  if (e != cudaSuccess) return e;
  tsqr_combine_kernel<<<(unsigned)nleaves, 512, smem, st>>>(Y, ldy, M, l, nleaves, S, lds); ++g_kernel_launches;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ one-sided Jacobi
__global__ void __launch_bounds__(1024) jacobi_kernel(const double* __restrict__ R, int ldr, int l,
                                                      double* __restrict__ sigma, double* __restrict__ Wo,
                                                      double* __restrict__ Jo, int ldo, int* flag,
                                                      int* sweeps_out) {
  extern __shared__ double sm[];
  double* X = sm;                  // X[p*l + i] = column p of X = R^T  (= row p of R)
  double* J = X + l * l;           // J[p*l + i] = column p of J
  __shared__ int rotated, bad;
  __shared__ double sg[128];
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  if (tid == 0) { rotated = 0; bad = 0; }
  for (int e = tid; e < l * l; e += nt) {
    const int p = e / l, i = e % l;
    const double v = (i >= p) ? R[p * ldr + i] : 0.0;   // R upper: row p, col i
    if (!isfinite(v)) bad = 1;
    X[e] = v;
    J[e] = (p == i) ? 1.0 : 0.0;
  }
  __syncthreads();
  const double tol = (double)l * 0x1.0p-52;
  const int L = l + (l & 1);
  int sweeps = 0;
  bool converged = (bad != 0);
  for (int sweep = 0; sweep <= 30 && !converged; ++sweep) {
    __syncthreads();
    if (tid == 0) rotated = 0;
    __syncthreads();
    for (int s = 0; s < L - 1; ++s) {
      for (int pi = warp; pi < L / 2; pi += nw) {
        // round-robin (circle) pairing: index 0 fixed, others rotate
        const int a = (pi == 0) ? 0 : ((pi - 1 + s) % (L - 1)) + 1;
        const int bq = ((L - 2 - pi + s) % (L - 1)) + 1;
        const int p = a < bq ? a : bq, q = a < bq ? bq : a;
        if (q >= l) continue;
        double* xp = X + p * l;
        double* xq = X + q * l;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int i = lane; i < l; i += 32) {
          const double u = xp[i], v = xq[i];
          al += u * u; be += v * v; ga += u * v;
        }
        al = warp_sum(al); be = warp_sum(be); ga = warp_sum(ga);
        if (fabs(ga) > tol * sqrt(al * be)) {
          const double zeta = (be - al) / (2.0 * ga);
          const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double c = 1.0 / sqrt(1.0 + t * t), sn = c * t;
          for (int i = lane; i < l; i += 32) {
            const double u = xp[i], v = xq[i];
            xp[i] = c * u - sn * v;
            xq[i] = sn * u + c * v;
          }
          double* jp = J + p * l;
          double* jq = J + q * l;
          for (int i = lane; i < l; i += 32) {
            const double u = jp[i], v = jq[i];
            jp[i] = c * u - sn * v;
            jq[i] = sn * u + c * v;
          }
          if (lane == 0) rotated = 1;
        }
      }
      __syncthreads();
    }
    if (!rotated) converged = true;
    else ++sweeps;
  }
  __syncthreads();
  // sigma, stable descending order
  for (int p = warp; p < l; p += nw) {
    double s = 0.0;
    for (int i = lane; i < l; i += 32) s += X[p * l + i] * X[p * l + i];
    s = warp_sum(s);
    if (lane == 0) sg[p] = sqrt(s);
  }
  __syncthreads();
  for (int p = tid; p < l; p += nt) {
    int rank = 0;
    const double sp = sg[p];
    for (int q = 0; q < l; ++q) rank += (sg[q] > sp) || (sg[q] == sp && q < p);
    sigma[rank] = sp;
    const double inv = sp > 0.0 ? 1.0 / sp : 1.0;
    for (int i = 0; i < l; ++i) {
      Wo[i * ldo + rank] = X[p * l + i] * inv;
      Jo[i * ldo + rank] = J[p * l + i];
    }
  }
  if (tid == 0) {
    if (sweeps > 30 || (!converged)) atomicOr(flag, 2);
    if (bad) atomicOr(flag, 4);
    if (sweeps_out) *sweeps_out = sweeps;
  }
}

cudaError_t launch_jacobi(const double* R, int ldr, int l, double* sigma, double* W, double* J, int ldo,
                          int* flag, int* sweeps, cudaStream_t st) {
  const size_t smem = 2 * (size_t)l * l * sizeof(double);
  if (l > 120 || smem > (size_t)SMEM_OPTIN - 2048) return cudaErrorInvalidValue;
  cudaError_t e = set_smem((const void*)jacobi_kernel, smem);
  if (e != cudaSuccess) return e;
  jacobi_kernel<<<1, 1024, smem, st>>>(R, ldr, l, sigma, W, J, ldo, flag, sweeps); ++g_kernel_launches;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ signs / copies
__global__ void sign_from_v_kernel(const double* __restrict__ V, int64_t ldv, int64_t n, double* sgn) {
  const int col = blockIdx.x;
  __shared__ double bv[256];
  __shared__ int64_t bi[256];
  double best = -1.0;
  int64_t bidx = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double a = fabs(V[i * ldv + col]);
    if (a > best) { best = a; bidx = i; }       // ascending i per thread => lowest index kept on ties
  }
  bv[threadIdx.x] = best;
  bi[threadIdx.x] = bidx;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double o = bv[threadIdx.x + s];
      const int64_t oi = bi[threadIdx.x + s];
      if (o > bv[threadIdx.x] || (o == bv[threadIdx.x] && oi < bi[threadIdx.x])) {
        bv[threadIdx.x] = o;
        bi[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) sgn[col] = (V[bi[0] * ldv + col] < 0.0) ? -1.0 : 1.0;
}

cudaError_t launch_sign_from_v(const double* V, int64_t ldv, int64_t n, int l, double* sgn, cudaStream_t st) {
  sign_from_v_kernel<<<l, 256, 0, st>>>(V, ldv, n, sgn); ++g_kernel_launches;
  return cudaGetLastError();
}

__global__ void scale_cols_kernel(double* X, int64_t ldx, int64_t rows, int l, const double* sgn) {
  const int64_t total = rows * l;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / l;
    const int c = (int)(e % l);
    X[r * ldx + c] *= sgn[c];
  }
}

static int grid_for(int64_t total) {
  int64_t b = ceil_div(total, 256);
  if (b > 148 * 16) b = 148 * 16;
  if (b < 1) b = 1;
  return (int)b;
}

cudaError_t launch_scale_cols(double* X, int64_t ldx, int64_t rows, int l, const double* sgn, cudaStream_t st) {
  scale_cols_kernel<<<grid_for(rows * l), 256, 0, st>>>(X, ldx, rows, l, sgn); ++g_kernel_launches;
  return cudaGetLastError();
}

template <typename TO>
__global__ void copy_out_kernel(const double* __restrict__ src, int64_t lds, int64_t rows, int cols,
                                TO* __restrict__ dst, int64_t ldd, const double* colfac) {
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / cols;
    const int c = (int)(e % cols);
    double v = src[r * lds + c];
    if (colfac) v *= colfac[c];
    dst[r * ldd + c] = (TO)v;
  }
}

cudaError_t launch_copy_out(const double* src, int64_t lds, int64_t rows, int cols, void* dst, int64_t ldd,
                            bool dst_f32, const double* colfac, cudaStream_t st) {
  if (rows * cols == 0) return cudaSuccess;
  if (dst_f32)
    copy_out_kernel<float><<<grid_for(rows * cols), 256, 0, st>>>(src, lds, rows, cols, (float*)dst, ldd, colfac);
  else
    copy_out_kernel<double><<<grid_for(rows * cols), 256, 0, st>>>(src, lds, rows, cols, (double*)dst, ldd, colfac); ++g_kernel_launches;
  return cudaGetLastError();
}

__global__ void fill_kernel(double* p, int64_t n, double v) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) p[e] = v;
}

cudaError_t launch_fill(double* p, int64_t count, double v, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  fill_kernel<<<grid_for(count), 256, 0, st>>>(p, count, v); ++g_kernel_launches;
  return cudaGetLastError();
}

__global__ void zero_cols_kernel(double* Y, int64_t ld, int64_t rows, int l, int npad) {
  const int w = npad - l;
  const int64_t total = rows * w;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x)
    Y[(e / w) * ld + l + (e % w)] = 0.0;
}

cudaError_t launch_zero_cols(double* Y, int64_t ld, int64_t rows, int l, int npad, cudaStream_t st) {
  if (npad <= l || rows == 0) return cudaSuccess;
  zero_cols_kernel<<<grid_for(rows * (npad - l)), 256, 0, st>>>(Y, ld, rows, l, npad); ++g_kernel_launches;
  return cudaGetLastError();
}

template <typename TO>
__global__ void pca_eig_kernel(const double* d, int k, double m, TO* eig) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < k) eig[i] = (TO)(d[i] * d[i] / (m - 1.0));
}

cudaError_t launch_pca_eig(const double* d, int k, double m, void* eig, bool f32, cudaStream_t st) {
  if (f32) pca_eig_kernel<float><<<(k + 255) / 256, 256, 0, st>>>(d, k, m, (float*)eig);
  else pca_eig_kernel<double><<<(k + 255) / 256, 256, 0, st>>>(d, k, m, (double*)eig);
  ++g_kernel_launches;
  return cudaGetLastError();
}

__global__ void check_finite_kernel(const double* v, int64_t n, int* flag) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(v[e])) { atomicOr(flag, 4); return; }
}

cudaError_t launch_check_finite(const double* v, int64_t n, int* flag, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  check_finite_kernel<<<grid_for(n), 256, 0, st>>>(v, n, flag); ++g_kernel_launches;
  return cudaGetLastError();
}

}  // namespace rsvd
