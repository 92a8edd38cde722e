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
//  * sign / copy / column statistics helpers.
#include <math.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace rsvd {

constexpr int SMEM_OPTIN = 232448;   // B200 per-block opt-in shared memory (profiles/peaks_box.json)

// cudaFuncSetAttribute is a slow host call: raise each kernel's dynamic
// shared-memory limit to the opt-in maximum once per device (smem_optin_fn).
static cudaError_t set_smem(const void* fn, size_t bytes) {
  (void)bytes;
  return smem_optin_fn(fn);
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
  // loads in batches of 8 (in flight together), summed in the same ascending order
  double s = 0.0;
  for (int t0 = 0; t0 < chunks; t0 += 8) {
    double v[8];
#pragma unroll
    for (int b = 0; b < 8; ++b) v[b] = (t0 + b < chunks) ? partial[(int64_t)(t0 + b) * n + j] : 0.0;
#pragma unroll
    for (int b = 0; b < 8; ++b)
      if (t0 + b < chunks) s += v[b];
  }
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
// Blocked Cholesky + triangular inverse, NB x NB blocks, 256 threads.
// Only the NB-column diagonal factorisations and the NB x NB diagonal-block
// inverses are sequential, and they run warp-synchronously (no CTA barrier);
// the block-row solves, trailing updates and off-diagonal inverse blocks are
// CTA-parallel with 3 (Cholesky) / 2 (inverse) barriers per block.
constexpr int CHOL_NB = 16, CHOL_THREADS = 256;
#ifndef CPROBE
#define CPROBE(k)
#endif

__global__ void __launch_bounds__(CHOL_THREADS, 1) chol_inv_kernel(const double* __restrict__ G, int ldg, int l,
                                                                   int npad, double* __restrict__ R,
                                                                   double* __restrict__ Rinv, int* flag,
                                                                   int flag_bit) {
  constexpr int NB = CHOL_NB;
  extern __shared__ double sm[];
  double* Gs = sm;                 // l x l, becomes R (upper)
  double* Xs = Gs + l * l;         // l x l, R^-1 (upper)
  __shared__ double d0[120], rdiag[120];
  __shared__ int bad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nthr = blockDim.x;
  CPROBE(0)
  if (tid == 0) bad = 0;
  for (int e = tid; e < l * l; e += nthr) {
    const int a = e / l, b = e - (e / l) * l;
    const double g = G[a * ldg + b];
    Gs[e] = g;
    Xs[e] = 0.0;
    if (a == b) d0[a] = g;
  }
  __syncthreads();
  CPROBE(1)
  // ---------------- Cholesky G = R^T R, right-looking by NB-column blocks
  for (int k0 = 0; k0 < l; k0 += NB) {
    const int kb = min(NB, l - k0), ke = k0 + kb;
    if (warp == 0) {                                   // (1) diagonal block, warp-synchronous
      for (int c = k0; c < ke; ++c) {
        const double d = Gs[c * l + c];
        const bool brk = !(d > 1e-13 * d0[c]) || !isfinite(d);
        const double ir = brk ? 1.0 : rsqrt(d);       // one long-latency op per pivot
        const double r = brk ? 1.0 : d * ir;
        __syncwarp();
        if (lane == 0) { Gs[c * l + c] = r; rdiag[c] = ir; if (brk) bad = 1; }
        const int b = c + 1 + (lane & 15);
        if (lane < 16 && b < ke) Gs[c * l + b] = brk ? 0.0 : Gs[c * l + b] * ir;
        __syncwarp();
        // in-block trailing update, lane = (row parity, column); all operands are
        // loaded into registers before the stores (no load-after-store chains)
        if (b < ke) {
          const double rcb = Gs[c * l + b];
          double rca[NB / 2], gg[NB / 2];
#pragma unroll
          for (int t = 0; t < NB / 2; ++t) {
            const int a = c + 1 + (lane >> 4) + 2 * t;
            rca[t] = (a <= b) ? Gs[c * l + a] : 0.0;
            gg[t] = (a <= b) ? Gs[a * l + b] : 0.0;
          }
#pragma unroll
          for (int t = 0; t < NB / 2; ++t) {
            const int a = c + 1 + (lane >> 4) + 2 * t;
            if (a <= b) Gs[a * l + b] = fma(-rca[t], rcb, gg[t]);
          }
        }
        __syncwarp();
      }
    }
    __syncthreads();
    CPROBE(2)
    // (2) block row: R[k0:ke][j] = R_kk^-T G[k0:ke][j]  (forward substitution per column j)
    for (int j = ke + tid; j < l; j += nthr) {
      double x[NB];
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        if (i < kb) {
          double s = Gs[(k0 + i) * l + j];
#pragma unroll
          for (int p = 0; p < NB; ++p)
            if (p < i) s -= Gs[(k0 + p) * l + k0 + i] * x[p];
          x[i] = s * rdiag[k0 + i];
          Gs[(k0 + i) * l + j] = x[i];
        }
      }
    }
    __syncthreads();
    CPROBE(3)
    // (3) trailing update: G[i][j] -= sum_p R[p][i] R[p][j], ke <= i <= j
    const int tr = l - ke;
    for (int i = ke + (tid >> 4); i < l; i += (nthr >> 4)) {
      double ri[NB];
#pragma unroll
      for (int p = 0; p < NB; ++p) ri[p] = (p < kb) ? Gs[(k0 + p) * l + i] : 0.0;
      for (int j = i + (tid & 15); j < l; j += 16) {
        double s = 0.0;
#pragma unroll
        for (int p = 0; p < NB; ++p) if (p < kb) s = fma(ri[p], Gs[(k0 + p) * l + j], s);
        Gs[i * l + j] -= s;
      }
    }
    (void)tr;
    __syncthreads();
    CPROBE(4)
  }
  // ---------------- X = R^-1
  const int nblk = (l + NB - 1) / NB;
  // (1) diagonal blocks, one warp per block, one lane per column (back substitution)
  for (int kbk = warp; kbk < nblk; kbk += nthr / 32) {
    const int k0 = kbk * NB, kb = min(NB, l - k0);
    if (lane < kb) {
      const int c = lane;
      double x[NB];
#pragma unroll
      for (int ii = NB - 1; ii >= 0; --ii) {
        if (ii <= c) {
          double s = 0.0;
#pragma unroll
          for (int p = 0; p < NB; ++p)
            if (p > ii && p <= c) s = fma(Gs[(k0 + ii) * l + k0 + p], x[p], s);
          x[ii] = (ii == c) ? rdiag[k0 + c] : -s * rdiag[k0 + ii];
          Xs[(k0 + ii) * l + k0 + c] = x[ii];
        } else {
          x[ii] = 0.0;
        }
      }
    }
  }
  __syncthreads();
  CPROBE(5)
  // (2) off-diagonal blocks, block rows bottom-up:
  //     T[I][j] = sum_{p >= i0+kb} R[I][p] X[p][j];  X[I][j] = -X_II T[I][j]
  for (int ib = nblk - 2; ib >= 0; --ib) {
    const int i0 = ib * NB, kb = min(NB, l - i0), je = i0 + kb;
    const int ncols = l - je;
    for (int e = tid; e < kb * ncols; e += nthr) {
      const int ii = e / ncols, j = je + e % ncols;
      double s0 = 0.0, s1 = 0.0;
      int p = je;
      for (; p + 1 <= j; p += 2) {
        s0 = fma(Gs[(i0 + ii) * l + p], Xs[p * l + j], s0);
        s1 = fma(Gs[(i0 + ii) * l + p + 1], Xs[(p + 1) * l + j], s1);
      }
      if (p <= j) s0 = fma(Gs[(i0 + ii) * l + p], Xs[p * l + j], s0);
      Xs[(i0 + ii) * l + j] = s0 + s1;                 // T, in place (rows i0..je of column j)
    }
    __syncthreads();
    for (int j = je + tid; j < l; j += nthr) {
      double t[NB];
#pragma unroll
      for (int q = 0; q < NB; ++q) t[q] = (q < kb) ? Xs[(i0 + q) * l + j] : 0.0;
#pragma unroll
      for (int ii = 0; ii < NB; ++ii) {
        if (ii < kb) {
          double s = 0.0;
#pragma unroll
          for (int q = 0; q < NB; ++q) if (q >= ii && q < kb) s = fma(Xs[(i0 + ii) * l + i0 + q], t[q], s);
          Xs[(i0 + ii) * l + j] = -s;
        }
      }
    }
    __syncthreads();
  }
  CPROBE(6)
  for (int e = tid; e < npad * npad; e += nthr) {
    const int r2 = e / npad, c = e - r2 * npad;
    const bool in = r2 < l && c < l && c >= r2;
    if (R) R[e] = in ? Gs[r2 * l + c] : 0.0;
    Rinv[e] = in ? Xs[r2 * l + c] : 0.0;
  }
  if (tid == 0 && bad) atomicOr(flag, flag_bit);
  CPROBE(7)
}

int g_chol_ny = 16;  // (unused; kept for tools/bench_small)

cudaError_t launch_chol_inv(const double* G, int ldg, int l, int npad, double* R, double* Rinv, int* flag,
                            int flag_bit, cudaStream_t st) {
  const size_t smem = 2 * (size_t)l * l * sizeof(double);   // + ~2 KB static: fits up to l = 120
  if (l > 120 || smem > (size_t)SMEM_OPTIN - 2048) return cudaErrorInvalidValue;
  cudaError_t e = set_smem((const void*)chol_inv_kernel, smem);
  if (e != cudaSuccess) return e;
  chol_inv_kernel<<<1, CHOL_THREADS, smem, st>>>(G, ldg, l, npad, R, Rinv, flag, flag_bit);
  ++g_kernel_launches;
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
constexpr int HQR_THREADS = 1024;

// rows of one leaf held in shared memory: b l + l (tau) + 32 (reduction / sign
// bits) doubles; at l = 120 this is 240 = 2 l, so two R factors always combine
int leaf_rows_cap(int l) {
  const int64_t avail = SMEM_OPTIN / (int64_t)sizeof(double) - l - 32;
  return (int)(avail / l);
}

// Householder QR of leaf `leaf` of the M x l panel Y (nleaves near-equal row
// blocks): R (diag >= 0) to Rstack + leaf l^2, the explicit Q over the leaf's rows.
__device__ void hqr_leaf(double* __restrict__ Y, int64_t ldy, int64_t M, int l, int64_t nleaves, int64_t leaf,
                         double* __restrict__ Rstack) {
  extern __shared__ double sm[];
  const int64_t rb = M / nleaves, rem = M % nleaves;
  const int b = (int)(rb + (leaf < rem ? 1 : 0));
  const int64_t r0 = leaf * rb + (leaf < rem ? leaf : rem);
  double* Ys = sm;                 // column-major, ld = b
  double* tau = Ys + (int64_t)l * b;
  double* red = tau + l;           // 32 (block sums; then the R-diagonal sign bits)
  unsigned* sgn = reinterpret_cast<unsigned*>(red);
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;

  // eight independent loads in flight per thread before the shared stores
  const int bl = b * l;                               // <= SMEM_OPTIN / 8
  for (int e0 = tid; e0 < bl; e0 += 8 * nt) {
    double v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = e0 + q * nt, r = e / l, c = e - r * l;
      v[q] = e < bl ? Y[(r0 + r) * ldy + c] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = e0 + q * nt, r = e / l, c = e - r * l;
      if (e < bl) Ys[c * b + r] = v[q];
    }
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

  // ---- R (upper l x l) with diag >= 0 to the stack; remember the signs as bits
  __syncthreads();
  if (tid < 8) sgn[tid] = 0u;
  __syncthreads();
  for (int j = tid; j < l; j += nt)
    if (Ys[(int64_t)j * b + j] < 0.0) atomicOr(&sgn[j >> 5], 1u << (j & 31));
  __syncthreads();
  auto w = [&](int c) { return ((sgn[c >> 5] >> (c & 31)) & 1u) ? -1.0 : 1.0; };
  double* Rl = Rstack + leaf * (int64_t)l * l;
  for (int e = tid; e < l * l; e += nt) {
    const int i = e / l, c = e % l;
    Rl[e] = (c >= i) ? w(i) * Ys[(int64_t)c * b + i] : 0.0;
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
    Y[(r0 + r) * ldy + c] = w(c) * Ys[(int64_t)c * b + r];
  }
  __syncthreads();   // the shared buffers are reused by the caller's next leaf
}

__global__ void __launch_bounds__(HQR_THREADS) hqr_leaves_kernel(double* __restrict__ Y, int64_t ldy,
                                                                 int64_t M, int l, int64_t nleaves,
                                                                 double* __restrict__ Rstack, Pred pr) {
  pdl_wait();
  pdl_trigger();
  if (pred_skip(pr)) return;
  hqr_leaf(Y, ldy, M, l, nleaves, blockIdx.x, Rstack);
}

cudaError_t launch_hqr_leaves(double* Y, int64_t ldy, int64_t M, int l, int64_t nleaves, double* Rstack,
                              cudaStream_t st, Pred pr) {
  const int64_t bmax = ceil_div(M, nleaves);
  const size_t smem = ((size_t)bmax * l + l + 32) * sizeof(double);
  if (smem > (size_t)SMEM_OPTIN || bmax < l) return cudaErrorInvalidValue;
  cudaError_t e = set_smem((const void*)hqr_leaves_kernel, smem);
  if (e != cudaSuccess) return e;
  e = launch_pdl(hqr_leaves_kernel, dim3((unsigned)nleaves), dim3(HQR_THREADS), smem, st, Y, ldy, M, l, nleaves, Rstack, pr);
  if (e != cudaSuccess) return e;
  ++g_kernel_launches;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ register-column Householder
// The single-CTA panel QR of hqr_leaf for small panels (b <= 32 RPL rows, l <= 32
// columns) with the panel held in REGISTERS: warp c owns column c (row r = lane +
// 32 i in element i), so the trailing update of a column step reads only the
// Householder vector from shared memory (hqr_leaf re-reads the vector and every
// trailing column from shared memory twice per step: ~760 KB per step at 1000 x
// 20, bound by shared-memory bandwidth).  Same LAPACK dgeqr2 /
// dorg2r arithmetic and conventions (v_j = 1 implicit, sign(0) = +1, tau = 0 for a
// zero column: R_jj = 0, reading R6), same outputs: Q in place, R (diag >= 0)
// row-major l x l.  The explicit Q needs no barrier: warp c applies H_c .. H_0 to
// e_c on its own (the vectors are read-only by then).
// VREG: the vector is read once into registers per step (RPL <= 16, l <= 20:
// 2 x RPL doubles per lane fit 640 threads' registers), else re-read (volatile).
template <int RPL, bool VREG>
__global__ void __launch_bounds__((RPL >= 32 || VREG) ? 640 : 1024, 1)
hqr_cols_kernel(double* __restrict__ Y, int64_t ldy, int b, int l, double* __restrict__ Rout) {
  pdl_wait();
  pdl_trigger();
  constexpr int B = 32 * RPL;
  extern __shared__ double sv[];
  double* V = sv;                      // l x B, column j = v_j (zeros above row j)
  double* tau = V + (int64_t)l * B;    // l
  double* Rs = tau + l;                // l x l row-major (upper part)
  const int lane = threadIdx.x & 31, c = threadIdx.x >> 5;
  double y[RPL];
#pragma unroll
  for (int i = 0; i < RPL; ++i) {
    const int r = lane + 32 * i;
    y[i] = r < b ? Y[(int64_t)r * ldy + c] : 0.0;
  }
  for (int j = 0; j < l; ++j) {
    if (c == j) {
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
        const int r = lane + 32 * i;
        if (r > j) s += y[i] * y[i];
      }
      s = warp_sum(s);
      double x0 = 0.0;
#pragma unroll
      for (int i = 0; i < RPL; ++i)
        if (i == (j >> 5)) x0 = y[i];
      x0 = __shfl_sync(0xffffffffu, x0, j & 31);
      double t = 0.0, beta = x0, scal = 0.0;
      if (s != 0.0) {
        const double nrm = sqrt(x0 * x0 + s);
        beta = -copysign(nrm, x0);                 // sign(0) = +1 => beta = -||x||
        t = (beta - x0) / beta;
        scal = 1.0 / (x0 - beta);
      }
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
        const int r = lane + 32 * i;
        if (r < j) Rs[r * l + j] = y[i];
        V[(int64_t)j * B + r] = r > j ? y[i] * scal : (r == j ? 1.0 : 0.0);
      }
      if (lane == 0) { tau[j] = t; Rs[j * l + j] = beta; }
    }
    __syncthreads();
    if (c > j) {
      const double t = tau[j];
      if (t != 0.0) {
        const double* v = V + (int64_t)j * B + lane;
        double w = 0.0;
#pragma unroll
        for (int i = 0; i < RPL; ++i) w += v[32 * i] * y[i];
        const double f = t * warp_sum(w);
        if constexpr (VREG) {
#pragma unroll
          for (int i = 0; i < RPL; ++i) y[i] -= f * v[32 * i];
        } else {
          // re-read v (volatile): holding it across the reduction would double the registers
          const volatile double* vv = v;
#pragma unroll
          for (int i = 0; i < RPL; ++i) y[i] -= f * vv[32 * i];
        }
      }
    }
  }
  __syncthreads();
  // explicit Q column c = H_0 ... H_c e_c (H_i e_c = e_c for i > c), diag(R) >= 0
  const double sg = Rs[c * l + c] < 0.0 ? -1.0 : 1.0;
#pragma unroll
  for (int i = 0; i < RPL; ++i) y[i] = (lane + 32 * i == c) ? 1.0 : 0.0;
  for (int i = c; i >= 0; --i) {
    const double t = tau[i];
    if (t == 0.0) continue;
    const double* v = V + (int64_t)i * B + lane;
    double w = 0.0;
#pragma unroll
    for (int e = 0; e < RPL; ++e) w += v[32 * e] * y[e];
    const double f = t * warp_sum(w);
    if constexpr (VREG) {
#pragma unroll
      for (int e = 0; e < RPL; ++e) y[e] -= f * v[32 * e];
    } else {
      const volatile double* vv = v;
#pragma unroll
      for (int e = 0; e < RPL; ++e) y[e] -= f * vv[32 * e];
    }
  }
#pragma unroll
  for (int i = 0; i < RPL; ++i) {
    const int r = lane + 32 * i;
    if (r < b) Y[(int64_t)r * ldy + c] = sg * y[i];
  }
  // R row c: (diag sign of row c) x upper part; zeros below the diagonal
  for (int e = lane; e < l; e += 32) Rout[c * l + e] = e >= c ? sg * Rs[c * l + e] : 0.0;
}

// Register-column Householder for a b x l panel if it fits (l <= 32, b <= 1024 and
// the registers of 32 l threads); cudaErrorNotSupported otherwise (the caller
// uses launch_hqr_leaves).
cudaError_t launch_hqr_small(double* Y, int64_t ldy, int64_t M, int l, double* R, cudaStream_t st) {
  if (l < 1 || l > 32 || M < l || M > 1024) return cudaErrorNotSupported;
  int rpl = 4;
  while (32 * rpl < M) rpl *= 2;
  // registers: ~2 RPL + 32 per thread within 65536 / (32 l); RPL = 32 needs l <= 20
  if ((rpl == 32 && l > 20) || 64 * rpl + 1024 > 65536 / l) return cudaErrorNotSupported;
  const size_t smem = ((size_t)l * 32 * rpl + l + (size_t)l * l) * sizeof(double);
  cudaError_t e = cudaSuccess;
#define RSVD_HQC(RP, VR)                                                                              \
  {                                                                                                  \
    e = set_smem((const void*)hqr_cols_kernel<RP, VR>, smem);                                        \
    if (e != cudaSuccess) return e;                                                                  \
    e = launch_pdl(hqr_cols_kernel<RP, VR>, dim3(1), dim3(32 * l), smem, st, Y, ldy, (int)M, l, R);  \
  }
  const bool vreg = rpl <= 16 && l <= 20;
  switch (rpl) {
    case 4: if (vreg) RSVD_HQC(4, true) else RSVD_HQC(4, false) break;
    case 8: if (vreg) RSVD_HQC(8, true) else RSVD_HQC(8, false) break;
    case 16: if (vreg) RSVD_HQC(16, true) else RSVD_HQC(16, false) break;
    default: RSVD_HQC(32, false) break;
  }
#undef RSVD_HQC
  if (e != cudaSuccess) return e;
  ++g_kernel_launches;
  return cudaGetLastError();
}

// Q rows of leaf `leaf` <- Q rows * S_leaf (S_leaf = rows [leaf l, leaf l + l) of S)
__device__ void tsqr_combine_leaf(double* __restrict__ Y, int64_t ldy, int64_t M, int l, int64_t nleaves,
                                  int64_t leaf, const double* __restrict__ S, int64_t lds) {
  extern __shared__ double sm[];
  double* Ss = sm;                 // l x l
  double* rows = Ss + l * l;       // 16 x l
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
  __syncthreads();
}

__global__ void tsqr_combine_kernel(double* __restrict__ Y, int64_t ldy, int64_t M, int l, int64_t nleaves,
                                    const double* __restrict__ S, int64_t lds, Pred pr) {
  pdl_wait();
  pdl_trigger();
  if (pred_skip(pr)) return;
  tsqr_combine_leaf(Y, ldy, M, l, nleaves, blockIdx.x, S, lds);
}

cudaError_t launch_tsqr_combine(double* Y, int64_t ldy, int64_t M, int l, int64_t nleaves, const double* S,
                                int64_t lds, cudaStream_t st, Pred pr) {
  const size_t smem = ((size_t)l * l + 16 * (size_t)l) * sizeof(double);
  cudaError_t e = set_smem((const void*)tsqr_combine_kernel, smem);
  if (e != cudaSuccess) return e;
  e = launch_pdl(tsqr_combine_kernel, dim3((unsigned)nleaves), dim3(512), smem, st, Y, ldy, M, l, nleaves, S, lds, pr);
  if (e != cudaSuccess) return e;
  ++g_kernel_launches;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ whole TSQR, one launch
// The complete local TSQR of launch_hqr_leaves / launch_tsqr_combine as ONE
// persistent launch: the upward levels (Householder leaves, their R factors
// stacked), the final leaf (R, also copied to Rout), the downward combines.  It
// is the CholeskyQR breakdown fallback, so on the happy path it is enqueued
// predicated and exits at once: one launch per orthonormalisation instead of
// one per level.
//
// Scheduling without a co-residency assumption (no cooperative launch, which
// serialises the stream): CTAs take work items from an atomic ticket in
// dependency order -- level 0 leaves, level 1 leaves, ..., the final leaf, the
// combines of level nlev-1 down to 0.  An item waits only for the completion
// counter of the phase before it, whose items hold lower tickets and so are
// owned by CTAs already running: progress never depends on a CTA that has not
// started.  Every CTA ends with one failed fetch; the last of those (all work
// done, nobody waiting) returns the ticket and counters to zero.
// Words: bar[0] ticket, bar[1 + ph] completion count of phase ph.
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(HQR_THREADS, 1) tsqr_fused_kernel(TsqrArgs a, Pred pr) {
  pdl_wait();
  if (pred_skip(pr)) return;
  __shared__ int64_t s_item;
  const int l = a.l, L = a.nlev;
  // phases: 0..L-1 leaves of level i; L the final leaf; L+1+j combines of level L-1-j
  int64_t total = 1;
  for (int i = 0; i < L; ++i) total += 2 * a.lev[i].P;
  unsigned* ticket = a.bar;
  unsigned* done = a.bar + 1;
  for (;;) {
    if (threadIdx.x == 0) s_item = (int64_t)atomicAdd(ticket, 1u);
    __syncthreads();
    int64_t t = s_item;
    __syncthreads();
    if (t >= total) {
      if (threadIdx.x == 0 && t == total + gridDim.x - 1) {   // the last CTA to leave
        for (int ph = 0; ph < 2 * L + 1; ++ph) done[ph] = 0u;
        *ticket = 0u;
        __threadfence();
      }
      return;
    }
    int ph = 0;
    int64_t idx = t;
    for (; ph < L && idx >= a.lev[ph].P; ++ph) idx -= a.lev[ph].P;
    if (ph == L && idx >= 1) {
      idx -= 1;
      ph = L + 1;
      while (idx >= a.lev[2 * L - ph].P) { idx -= a.lev[2 * L - ph].P; ++ph; }
    }
    // wait for the phase this one reads
    if (ph > 0 && threadIdx.x == 0) {
      const unsigned need = (ph <= L) ? (unsigned)a.lev[ph - 1].P                    // leaves / final leaf
                                      : (ph == L + 1 ? 1u : (unsigned)a.lev[2 * L - ph + 1].P);   // combines
      while (ld_acquire_u32(done + ph - 1) < need) __nanosleep(128);
    }
    __syncthreads();
    if (ph < L) {
      const TsqrLevel& V = a.lev[ph];
      hqr_leaf(V.buf, V.ld, V.M, l, V.P, idx, (ph + 1 < L) ? a.lev[ph + 1].buf : a.cur);
    } else if (ph == L) {
      hqr_leaf(a.cur, a.ldc, a.Mc, l, 1, 0, a.R);
      if (a.Rout)
        for (int e = threadIdx.x; e < l * l; e += blockDim.x) a.Rout[(int64_t)(e / l) * a.ldro + e % l] = a.R[e];
      __syncthreads();
    } else {
      const int i = 2 * L - ph;
      const TsqrLevel& V = a.lev[i];
      tsqr_combine_leaf(V.buf, V.ld, V.M, l, V.P, idx, (i + 1 < L) ? a.lev[i + 1].buf : a.cur, l);
    }
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(done + ph, 1u);
    }
  }
}

cudaError_t launch_tsqr_fused(const TsqrArgs& a, int num_sms, cudaStream_t st, Pred pr) {
  const int l = a.l;
  size_t smem = ((size_t)a.Mc * l + l + 32) * sizeof(double);
  int64_t pmax = 1;
  for (int i = 0; i < a.nlev; ++i) {
    const int64_t bmax = ceil_div(a.lev[i].M, a.lev[i].P);
    if (bmax < l) return cudaErrorInvalidValue;
    smem = std::max(smem, ((size_t)bmax * l + l + 32) * sizeof(double));
    pmax = std::max(pmax, a.lev[i].P);
  }
  smem = std::max(smem, ((size_t)l * l + 16 * (size_t)l) * sizeof(double));
  if (smem > (size_t)SMEM_OPTIN || a.nlev > kTsqrMaxLev || a.Mc < l || pmax >= (int64_t)1 << 30)
    return cudaErrorInvalidValue;
  CUDA_TRY(set_smem((const void*)tsqr_fused_kernel, smem));
  const int grid = (int)std::min<int64_t>(pmax, num_sms);
  CUDA_TRY(launch_pdl(tsqr_fused_kernel, dim3((unsigned)grid), dim3(HQR_THREADS), smem, st, a, pr));
  ++g_kernel_launches;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ signs / copies
__global__ void sign_from_v_kernel(const double* __restrict__ V, int64_t ldv, int64_t n, double* sgn) {
  pdl_wait();
  pdl_trigger();
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
  CUDA_TRY(launch_pdl(sign_from_v_kernel, dim3(l), dim3(256), 0, st, V, ldv, n, sgn)); ++g_kernel_launches;
  return cudaGetLastError();
}

__global__ void scale_cols_kernel(double* X, int64_t ldx, int64_t rows, int l, const double* sgn) {
  pdl_wait();
  pdl_trigger();
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
  CUDA_TRY(launch_pdl(scale_cols_kernel, dim3(grid_for(rows * l)), dim3(256), 0, st, X, ldx, rows, l, sgn)); ++g_kernel_launches;
  return cudaGetLastError();
}

template <typename TO>
__global__ void copy_out_kernel(const double* __restrict__ src, int64_t lds, int64_t rows, int cols,
                                TO* __restrict__ dst, int64_t ldd, const double* colfac, Pred pr) {
  pdl_wait();
  pdl_trigger();
  if (pred_skip(pr)) return;
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
                            bool dst_f32, const double* colfac, cudaStream_t st, Pred pr) {
  if (rows * cols == 0) return cudaSuccess;
  if (dst_f32)
    CUDA_TRY(launch_pdl(copy_out_kernel<float>, dim3(grid_for(rows * cols)), dim3(256), 0, st, src, lds, rows, cols, (float*)dst, ldd, colfac, pr));
  else
    CUDA_TRY(launch_pdl(copy_out_kernel<double>, dim3(grid_for(rows * cols)), dim3(256), 0, st, src, lds, rows, cols, (double*)dst, ldd, colfac, pr));
  ++g_kernel_launches;
  return cudaGetLastError();
}

__global__ void fill_kernel(double* p, int64_t n, double v) {
  pdl_wait();
  pdl_trigger();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) p[e] = v;
}

cudaError_t launch_fill(double* p, int64_t count, double v, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  CUDA_TRY(launch_pdl(fill_kernel, dim3(grid_for(count)), dim3(256), 0, st, p, count, v)); ++g_kernel_launches;
  return cudaGetLastError();
}

__global__ void zero_cols_kernel(double* Y, int64_t ld, int64_t rows, int l, int npad) {
  pdl_wait();
  pdl_trigger();
  const int w = npad - l;
  const int64_t total = rows * w;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x)
    Y[(e / w) * ld + l + (e % w)] = 0.0;
}

cudaError_t launch_zero_cols(double* Y, int64_t ld, int64_t rows, int l, int npad, cudaStream_t st) {
  if (npad <= l || rows == 0) return cudaSuccess;
  CUDA_TRY(launch_pdl(zero_cols_kernel, dim3(grid_for(rows * (npad - l))), dim3(256), 0, st, Y, ld, rows, l, npad)); ++g_kernel_launches;
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
  pdl_wait();
  pdl_trigger();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(v[e])) { atomicOr(flag, 4); return; }
}

cudaError_t launch_check_finite(const double* v, int64_t n, int* flag, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  CUDA_TRY(launch_pdl(check_finite_kernel, dim3(grid_for(n)), dim3(256), 0, st, v, n, flag)); ++g_kernel_launches;
  return cudaGetLastError();
}

}  // namespace rsvd

namespace rsvd {

// ------------------------------------------------------------------ rpca outputs (Alg. 6)
// rs = 1 / s.d. and s = s.d. from the column sums of squares ss of the centred
// data (non-destructive: ss stays for the total variance); constant columns
// get s = 1 (no scaling)
__global__ void colstat_scale_kernel(const double* ss, int64_t n, double mg, double* rs, double* s) {
  pdl_wait();
  pdl_trigger();
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  double sd = sqrt(ss[j] / (mg - 1.0));
  if (!(sd > 0.0)) sd = 1.0;
  s[j] = sd;
  rs[j] = 1.0 / sd;
}

cudaError_t launch_colstat_scale(const double* ss, int64_t n, double m_global, double* rs, double* s, cudaStream_t st) {
  CUDA_TRY(launch_pdl(colstat_scale_kernel, dim3((unsigned)ceil_div(n, 256)), dim3(256), 0, st, ss, n, m_global, rs, s));
  ++g_kernel_launches;
  return cudaGetLastError();
}

// total variance sum_j var(X_j) = sum_j ss_j rs_j^2 / (m - 1) (the trace of the
// covariance / correlation matrix = sum of ALL its eigenvalues);
// one CTA, fixed-order partial sums then a fixed tree (deterministic)
__global__ void total_var_kernel(const double* ss, const double* rs, int64_t n, double mg, double* out) {
  pdl_wait();
  pdl_trigger();
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    const double f = rs ? rs[j] : 1.0;
    s += ss[j] * f * f;
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s / (mg - 1.0);
}

cudaError_t launch_total_var(const double* ss, const double* rs, int64_t n, double m_global, double* out, cudaStream_t st) {
  CUDA_TRY(launch_pdl(total_var_kernel, dim3(1), dim3(256), 0, st, ss, rs, n, m_global, out));
  ++g_kernel_launches;
  return cudaGetLastError();
}

// eigvals = d^2 / (m-1), sdev = sqrt(eigvals), the proportion of
// variance eigvals / total and its cumulative sum (summary());
// every output nullable; one thread per value, the cumulative sum in index order
template <typename TO>
__global__ void pca_stats_kernel(const double* d, int k, double mg, const double* total, TO* eig, TO* sdev, TO* ratio,
                                 TO* cum) {
  pdl_wait();
  pdl_trigger();
  const int i = threadIdx.x;
  if (i < k) {
    const double e = d[i] * d[i] / (mg - 1.0);
    if (eig) eig[i] = (TO)e;
    if (sdev) sdev[i] = (TO)sqrt(e);
    if (ratio && total) ratio[i] = (TO)(e / *total);
  }
  if (cum && total && i == 0) {
    double c = 0.0;
    for (int t = 0; t < k; ++t) {
      c += d[t] * d[t] / (mg - 1.0);
      cum[t] = (TO)(c / *total);
    }
  }
}

cudaError_t launch_pca_stats(const double* d, int k, double m_global, const double* total, void* eig, void* sdev,
                             void* ratio, void* cum, bool f32, cudaStream_t st) {
  if (k > 1024) return cudaErrorInvalidValue;
  if (f32)
    CUDA_TRY(launch_pdl(pca_stats_kernel<float>, dim3(1), dim3(1024), 0, st, d, k, m_global, total, (float*)eig,
                        (float*)sdev, (float*)ratio, (float*)cum));
  else
    CUDA_TRY(launch_pdl(pca_stats_kernel<double>, dim3(1), dim3(1024), 0, st, d, k, m_global, total, (double*)eig,
                        (double*)sdev, (double*)ratio, (double*)cum));
  ++g_kernel_launches;
  return cudaGetLastError();
}

// dst[j] = f(src[j]) for a small vector: mode 0 copy, 1 reciprocal, 2 sqrt(src / (m - 1)) (= sdev from d), 3 = constant v
template <typename TI>
__global__ void vec_map_kernel(const TI* src, int64_t n, int mode, double v, double* dst) {
  pdl_wait();
  pdl_trigger();
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  const double x = src ? (double)src[j] : 0.0;
  dst[j] = mode == 0 ? x : mode == 1 ? 1.0 / x : mode == 2 ? x / sqrt(v - 1.0) : v;
}

cudaError_t launch_vec_map(const void* src, bool src_f32, int64_t n, int mode, double v, double* dst, cudaStream_t st) {
  const dim3 g((unsigned)ceil_div(n, 256));
  if (src_f32) CUDA_TRY(launch_pdl(vec_map_kernel<float>, g, dim3(256), 0, st, (const float*)src, n, mode, v, dst));
  else CUDA_TRY(launch_pdl(vec_map_kernel<double>, g, dim3(256), 0, st, (const double*)src, n, mode, v, dst));
  ++g_kernel_launches;
  return cudaGetLastError();
}

// X (rows x npad, ld ldx, FP64) = src (rows x cols, ld lds, f32 or f64), columns [cols, npad) zero
template <typename TI>
__global__ void copy_in_kernel(const TI* __restrict__ src, int64_t lds, int64_t rows, int cols, int npad,
                               double* __restrict__ X, int64_t ldx) {
  pdl_wait();
  pdl_trigger();
  const int64_t total = rows * npad;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / npad;
    const int c = (int)(e % npad);
    X[r * ldx + c] = c < cols ? (double)src[r * lds + c] : 0.0;
  }
}

cudaError_t launch_copy_in(const void* src, bool src_f32, int64_t lds, int64_t rows, int cols, int npad, double* X,
                           int64_t ldx, cudaStream_t st) {
  const int64_t total = rows * npad;
  const unsigned g = (unsigned)std::min<int64_t>(ceil_div(total, 256), 148 * 16);
  if (src_f32) CUDA_TRY(launch_pdl(copy_in_kernel<float>, dim3(g), dim3(256), 0, st, (const float*)src, lds, rows, cols, npad, X, ldx));
  else CUDA_TRY(launch_pdl(copy_in_kernel<double>, dim3(g), dim3(256), 0, st, (const double*)src, lds, rows, cols, npad, X, ldx));
  ++g_kernel_launches;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ status words
__global__ void flag_or_kernel(int* flag, int bits, Pred pr) {
  pdl_wait();
  pdl_trigger();
  if (pred_skip(pr)) return;
  atomicOr(flag, bits);
}

cudaError_t launch_flag_or(int* flag, int bits, cudaStream_t st, Pred pr) {
  CUDA_TRY(launch_pdl(flag_or_kernel, dim3(1), dim3(1), 0, st, flag, bits, pr));
  ++g_kernel_launches;
  return cudaGetLastError();
}

// end of a call: the call's flags (flag[0]) are OR-ed into the context's sticky
// status (read and cleared by rsvd_sync); sticky[1] = Jacobi sweeps, sticky[2] =
// 1 if the TSQR fallback ran in this call
__global__ void status_finish_kernel(const int* flag, int* sticky, int fallback_bit) {
  pdl_wait();
  pdl_trigger();
  atomicOr(sticky, flag[0]);
  sticky[1] = flag[8];
  sticky[2] = (flag[0] & fallback_bit) ? 1 : 0;
}

cudaError_t launch_status_finish(const int* flag, int* sticky, int fallback_bit, cudaStream_t st) {
  CUDA_TRY(launch_plain(status_finish_kernel, dim3(1), dim3(1), 0, st, flag, sticky, fallback_bit));
  ++g_kernel_launches;
  return cudaGetLastError();
}

// p[0..n) = 0 by a plain launch (instead of cudaMemsetAsync, so that the
// following PDL kernels are ordered behind it), then nothing else
__global__ void zero_words_kernel(int* p, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] = 0;
}

cudaError_t launch_zero_words(int* p, int n, cudaStream_t st) {
  CUDA_TRY(launch_plain(zero_words_kernel, dim3(1), dim3(64), 0, st, p, n));
  ++g_kernel_launches;
  return cudaGetLastError();
}

// an empty plain kernel: orders the following PDL kernels behind preceding
// non-kernel stream work (collective copies, NCCL)
__global__ void stream_fence_kernel() {}

cudaError_t launch_stream_fence(cudaStream_t st) {
  CUDA_TRY(launch_plain(stream_fence_kernel, dim3(1), dim3(1), 0, st));
  ++g_kernel_launches;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ in-process rank groups
// out[i] = stage[0][i] (+ / max) stage[1][i] ... stage[R-1][i], ranks in order
// (every rank computes the identical result: the stand-in for ncclAllReduce)
__global__ void group_reduce_kernel(GroupPtrs in, int nranks, int64_t n, int op_max, double* out) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double s = in.p[0][i];
    for (int r = 1; r < nranks; ++r) s = op_max ? fmax(s, in.p[r][i]) : s + in.p[r][i];
    out[i] = s;
  }
}

cudaError_t launch_group_reduce(const GroupPtrs& in, int nranks, int64_t n, int op_max, double* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const unsigned g = (unsigned)std::min<int64_t>(ceil_div(n, 256), 148 * 8);
  // plain launch: it follows the staging copies and the cross-stream event waits
  CUDA_TRY(launch_plain(group_reduce_kernel, dim3(g), dim3(256), 0, st, in, nranks, n, op_max, out));
  ++g_kernel_launches;
  return cudaGetLastError();
}

}  // namespace rsvd
