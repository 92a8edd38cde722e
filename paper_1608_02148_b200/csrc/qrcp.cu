// qrcp.cu -- column-pivoted Householder QR of a short-wide matrix, stopped
// after `steps` pivots, and the interpolative-decomposition solve of Alg. id
// (used by rid P:2100-2127 and rcur P:1975-2010; reading
// R31 of DESIGN.md: Businger-Golub pivot = largest remaining column norm,
// ties to the lowest index).
//
// B200 design.  The matrix is "column-contiguous": column c is `rows` doubles
// at W + c * ld -- exactly B^T (n x Np, row-major) for rid and C (m x k,
// row-major) for rcur's pivoted QR of C^T, so no transpose is formed.  One
// cooperative grid (one CTA per SM) owns contiguous column ranges; per pivot
// step:
//   (1) every CTA takes the largest remaining norm of its unpivoted columns
//       (recomputed exactly from rows j.., no downdating);
//   (2) grid barrier; every CTA reduces the per-CTA candidates in the same
//       fixed order, so all agree on the pivot without atomics;
//   (3) every CTA reads the pivot column and forms the same Householder
//       reflector (fixed-order block reductions: bit-identical in all CTAs);
//   (4) every CTA reflects its own unpivoted columns (warp per column).
// The pivot column itself is never written (its S entries above row j are
// final; S_jj = alpha_j is kept apart), so step j+1 can read it without a
// second barrier; the candidate array is double-buffered.  After the last
// step each CTA back-substitutes T = S_kk^-1 S_12 for its columns and writes
// Z(:, c) (Z(:, P) = [I_k, T]).
#include <cooperative_groups.h>
#include <math.h>

#include "common.cuh"
#include "kernels.h"

namespace rsvd {

namespace cg = cooperative_groups;

namespace {
constexpr int QC_THREADS = 256, QC_WARPS = QC_THREADS / 32, QC_RMAX = 128;

struct QrcpArgs {
  double* W; int64_t ld; int rows; int64_t ncols; int steps;
  double* cval; int64_t* cidx;             // [2][grid] per-CTA candidates
  double* alpha;                           // [steps] S_jj
  unsigned char* done;                     // [ncols] pivoted flags (owner CTA only)
  int64_t* perm;                           // [steps] pivots, output
  double* Z; int64_t ldz;                  // k x ncols interpolation matrix (nullable)
  int* flag; int flag_bit;
};

__device__ __forceinline__ bool better(double v, int64_t i, double bv, int64_t bi) {
  return v > bv || (v == bv && i < bi);
}

// fixed-order block sum (all threads get the result)
__device__ __forceinline__ double qc_block_sum(double v, double* red) {
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < QC_WARPS; ++w) s += red[w];
  return s;
}

__global__ void __launch_bounds__(QC_THREADS, 1) qrcp_kernel(QrcpArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double x[QC_RMAX];
  __shared__ double red[QC_WARPS];
  __shared__ double wv[QC_WARPS];
  __shared__ int64_t wi[QC_WARPS];
  __shared__ int64_t s_piv;
  __shared__ double s_alpha, s_tau;
  extern __shared__ double skk[];          // steps x steps (solve phase)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x;
  const int64_t c0 = a.ncols * blockIdx.x / G, c1 = a.ncols * (blockIdx.x + 1) / G;
  const int rows = a.rows;
  for (int j = 0; j < a.steps; ++j) {
    // (1) local candidate
    double bv = -1.0;
    int64_t bi = INT64_MAX;
    for (int64_t c = c0 + warp; c < c1; c += QC_WARPS) {
      if (a.done[c]) continue;
      const double* col = a.W + c * a.ld;
      double s = 0.0;
      for (int i = j + lane; i < rows; i += 32) s = fma(col[i], col[i], s);
      s = warp_sum(s);
      if (better(s, c, bv, bi)) { bv = s; bi = c; }
    }
    if (lane == 0) { wv[warp] = bv; wi[warp] = bi; }
    __syncthreads();
    if (tid == 0) {
      double v = wv[0];
      int64_t i = wi[0];
      for (int w = 1; w < QC_WARPS; ++w)
        if (better(wv[w], wi[w], v, i)) { v = wv[w]; i = wi[w]; }
      a.cval[(j & 1) * G + blockIdx.x] = v;
      a.cidx[(j & 1) * G + blockIdx.x] = i;
    }
    grid.sync();
    // (2) global pivot, same fixed order in every CTA
    if (warp == 0) {
      double v = -1.0;
      int64_t i = INT64_MAX;
      for (int b = lane; b < G; b += 32) {
        const double vb = __ldcg(a.cval + (j & 1) * G + b);
        const int64_t ib = __ldcg(a.cidx + (j & 1) * G + b);
        if (better(vb, ib, v, i)) { v = vb; i = ib; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double vo = __shfl_xor_sync(0xffffffffu, v, o);
        const int64_t io = __shfl_xor_sync(0xffffffffu, i, o);
        if (better(vo, io, v, i)) { v = vo; i = io; }
      }
      if (lane == 0) s_piv = i;
    }
    __syncthreads();
    const int64_t piv = s_piv;
    if (blockIdx.x == 0 && tid == 0) a.perm[j] = piv;
    if (piv >= c0 && piv < c1 && tid == 0) a.done[piv] = 1;
    // (3) reflector from the pivot column (rows j..)
    const double* pc = a.W + piv * a.ld;
    const int len = rows - j;
    for (int i = tid; i < len; i += QC_THREADS) x[i] = __ldcg(pc + j + i);
    __syncthreads();
    double sq = 0.0;
    for (int i = tid; i < len; i += QC_THREADS) sq = fma(x[i], x[i], sq);
    const double nx = sqrt(qc_block_sum(sq, red));
    if (tid == 0) {
      const double x0 = x[0];
      const double al = nx == 0.0 ? 0.0 : (x0 >= 0.0 ? -nx : nx);
      s_alpha = al;
      x[0] = x0 - al;                                   // v = x - alpha e_1 (in place)
      if (blockIdx.x == 0) a.alpha[j] = al;
    }
    __syncthreads();
    double vv = 0.0;
    for (int i = tid; i < len; i += QC_THREADS) vv = fma(x[i], x[i], vv);
    vv = qc_block_sum(vv, red);
    if (tid == 0) s_tau = vv > 0.0 ? 2.0 / vv : 0.0;
    __syncthreads();
    const double tau = s_tau;
    // (4) reflect the CTA's unpivoted columns
    if (tau != 0.0) {
      for (int64_t c = c0 + warp; c < c1; c += QC_WARPS) {
        if (a.done[c]) continue;
        double* col = a.W + c * a.ld + j;
        double w = 0.0;
        for (int i = lane; i < len; i += 32) w = fma(x[i], col[i], w);
        w = warp_sum(w) * tau;
        for (int i = lane; i < len; i += 32) col[i] = fma(-w, x[i], col[i]);
      }
    }
    __syncthreads();
  }
  grid.sync();
  if (!a.Z) return;
  // ID solve: S_kk (upper, k x k) from the pivot columns, T = S_kk^-1 S_12 per column
  const int k = a.steps;
  for (int e = tid; e < k * k; e += QC_THREADS) {
    const int i = e / k, jj = e - i * k;
    double v = 0.0;
    if (i < jj) v = __ldcg(a.W + __ldcg(a.perm + jj) * a.ld + i);
    else if (i == jj) v = __ldcg(a.alpha + jj);
    skk[e] = v;
  }
  __syncthreads();
  if (blockIdx.x == 0 && tid == 0) {
    // numerical rank < k: |S_jj| <= rows 2^-52 |S_11| (reading R31)
    const double thr = (double)rows * 0x1.0p-52 * fabs(skk[0]);
    bool sing = !(fabs(skk[0]) > 0.0);
    for (int i = 1; i < k; ++i) sing |= !(fabs(skk[i * k + i]) > thr);
    if (sing) atomicOr(a.flag, a.flag_bit);
  }
  for (int64_t c = c0 + warp; c < c1; c += QC_WARPS) {
    if (a.done[c]) {
      // pivot column: Z(:, c) = e_p for its position p in the pivot order
      int pos = -1;
      for (int i = lane; i < k; i += 32)
        if (__ldcg(a.perm + i) == c) pos = i;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) pos = max(pos, __shfl_xor_sync(0xffffffffu, pos, o));
      for (int i = lane; i < k; i += 32) a.Z[(int64_t)i * a.ldz + c] = (i == pos) ? 1.0 : 0.0;
      continue;
    }
    // back substitution, lane r holds t_r for r = lane + 32 q (k <= 128)
    const double* col = a.W + c * a.ld;
    double t[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) t[q] = (lane + 32 * q < k) ? col[lane + 32 * q] : 0.0;
    for (int i = k - 1; i >= 0; --i) {
      const int qi = i >> 5, li = i & 31;
      double ti = 0.0;
#pragma unroll
      for (int q = 0; q < 4; ++q) if (q == qi) ti = t[q];
      ti = __shfl_sync(0xffffffffu, ti, li) / skk[i * k + i];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int r = lane + 32 * q;
        if (r == i) t[q] = ti;
        else if (r < i) t[q] = fma(-skk[r * k + i], ti, t[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = lane + 32 * q;
      if (r < k) a.Z[(int64_t)r * a.ldz + c] = t[q];
    }
  }
}

// ---------------------------------------------------------------- pivoted LU
// "[L, ~] = lu(Y)  pivoted LU" of Alg. 3 (norm_iterations):
// Gaussian elimination with partial pivoting of a tall row-contiguous panel
// (row i = l doubles at Y + i * ld), in place, overwritten by the permuted
// unit lower factor L (L[p_j][j] = 1, L[p_j][c > j] = 0, multipliers
// elsewhere).  Same cooperative structure as qrcp_kernel with rows in place
// of columns: per step a per-CTA largest |y_ij| among unpivoted rows, one
// grid barrier, the same fixed-order pivot choice in every CTA, then each CTA
// eliminates its own rows against the (never again written) pivot row.
struct LuArgs {
  double* Y; int64_t ld; int64_t m; int l;
  double* cval; int64_t* cidx;             // [2][grid]
  int* stepof;                             // [m] step at which a row was pivoted, -1 before
  int* flag; int flag_bit;
};

__global__ void __launch_bounds__(QC_THREADS, 1) lu_rows_kernel(LuArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double u[QC_RMAX];
  __shared__ double wv[QC_WARPS];
  __shared__ int64_t wi[QC_WARPS];
  __shared__ int64_t s_piv;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x;
  const int64_t r0 = a.m * blockIdx.x / G, r1 = a.m * (blockIdx.x + 1) / G;
  const int l = a.l;
  for (int64_t i = r0 + tid; i < r1; i += QC_THREADS) a.stepof[i] = -1;
  __syncthreads();
  for (int j = 0; j < l; ++j) {
    double bv = -1.0;
    int64_t bi = INT64_MAX;
    for (int64_t i = r0 + tid; i < r1; i += QC_THREADS) {
      if (a.stepof[i] >= 0) continue;
      const double v = fabs(a.Y[i * a.ld + j]);
      if (better(v, i, bv, bi)) { bv = v; bi = i; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double vo = __shfl_xor_sync(0xffffffffu, bv, o);
      const int64_t io = __shfl_xor_sync(0xffffffffu, bi, o);
      if (better(vo, io, bv, bi)) { bv = vo; bi = io; }
    }
    if (lane == 0) { wv[warp] = bv; wi[warp] = bi; }
    __syncthreads();
    if (tid == 0) {
      double v = wv[0];
      int64_t i = wi[0];
      for (int w = 1; w < QC_WARPS; ++w)
        if (better(wv[w], wi[w], v, i)) { v = wv[w]; i = wi[w]; }
      a.cval[(j & 1) * G + blockIdx.x] = v;
      a.cidx[(j & 1) * G + blockIdx.x] = i;
    }
    grid.sync();
    if (warp == 0) {
      double v = -1.0;
      int64_t i = INT64_MAX;
      for (int b = lane; b < G; b += 32) {
        const double vb = __ldcg(a.cval + (j & 1) * G + b);
        const int64_t ib = __ldcg(a.cidx + (j & 1) * G + b);
        if (better(vb, ib, v, i)) { v = vb; i = ib; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double vo = __shfl_xor_sync(0xffffffffu, v, o);
        const int64_t io = __shfl_xor_sync(0xffffffffu, i, o);
        if (better(vo, io, v, i)) { v = vo; i = io; }
      }
      if (lane == 0) s_piv = i;
    }
    __syncthreads();
    const int64_t p = s_piv;
    for (int c = j + tid; c < l; c += QC_THREADS) u[c - j] = __ldcg(a.Y + p * a.ld + c);
    if (p >= r0 && p < r1 && tid == 0) a.stepof[p] = j;
    __syncthreads();
    const double u0 = u[0];
    if (blockIdx.x == 0 && tid == 0 && !(u0 != 0.0)) atomicOr(a.flag, a.flag_bit);
    const double inv = u0 != 0.0 ? 1.0 / u0 : 0.0;
    for (int64_t i = r0 + warp; i < r1; i += QC_WARPS) {
      if (i == p || a.stepof[i] >= 0) continue;
      double* y = a.Y + i * a.ld;
      const double lij = y[j] * inv;
      for (int c = j + 1 + lane; c < l; c += 32) y[c] = fma(-lij, u[c - j], y[c]);
      if (lane == 0) y[j] = lij;
    }
    __syncthreads();
  }
  // pivot rows: unit diagonal, zeros to the right
  for (int64_t i = r0 + warp; i < r1; i += QC_WARPS) {
    const int s = a.stepof[i];
    if (s < 0) continue;
    double* y = a.Y + i * a.ld;
    for (int c = s + lane; c < l; c += 32) y[c] = (c == s) ? 1.0 : 0.0;
  }
}

// C[r][i] = A[r][J[i]] (column gather, m x k) / R[i][c] = A[I[i]][c] (row gather, k x n)
// Rt[c][i] = A[I[i]][c] (row gather, transposed into an n x ldt panel)
__global__ void gather_cols_kernel(const double* __restrict__ A, int64_t lda, int64_t m, const int64_t* __restrict__ J,
                                   int k, double* __restrict__ C, int64_t ldc) {
  const int64_t total = m * k;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / k;
    const int i = (int)(e - r * k);
    C[r * ldc + i] = A[r * lda + J[i]];
  }
}

__global__ void gather_rows_kernel(const double* __restrict__ A, int64_t lda, int64_t n, const int64_t* __restrict__ I,
                                   int k, double* __restrict__ R, int64_t ldr, double* __restrict__ Rt, int64_t ldt) {
  const int64_t total = (int64_t)k * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / n);
    const int64_t c = e - (int64_t)i * n;
    const double v = A[I[i] * lda + c];
    if (R) R[i * ldr + c] = v;
    if (Rt) Rt[c * ldt + i] = v;
  }
}

// W (k x k, ld ldw) = Z (k x n, ld ldz) Q (n x k, ld ldq): per-CTA partial over a
// column range (partial[b] is k x k), then a fixed-order reduce.
__global__ void __launch_bounds__(256) zq_partial_kernel(const double* __restrict__ Z, int64_t ldz,
                                                          const double* __restrict__ Q, int64_t ldq, int64_t n,
                                                          int k, double* __restrict__ partial) {
  const int64_t b0 = n * blockIdx.x / gridDim.x, b1 = n * (blockIdx.x + 1) / gridDim.x;
  double* out = partial + (int64_t)blockIdx.x * k * k;
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
    const int i = e / k, j = e - i * k;
    double s = 0.0;
    for (int64_t c = b0; c < b1; ++c) s = fma(Z[i * ldz + c], Q[c * ldq + j], s);
    out[e] = s;
  }
}

__global__ void zq_reduce_kernel(const double* __restrict__ partial, int P, int k, double* __restrict__ W, int ldw) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < k * k; e += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < P; ++b) s += partial[(int64_t)b * k * k + e];
    W[(e / k) * ldw + (e % k)] = s;
  }
}

// U = W S^-T: row r of U solves S x = W(r, :)^T (S upper k x k, ld lds)
__global__ void rtsolve_kernel(const double* __restrict__ W, int ldw, const double* __restrict__ S, int lds, int k,
                               double* __restrict__ U, int64_t ldu) {
  const int r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= k) return;
  double t[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) t[q] = (lane + 32 * q < k) ? W[r * ldw + lane + 32 * q] : 0.0;
  for (int i = k - 1; i >= 0; --i) {
    const int qi = i >> 5, li = i & 31;
    double ti = 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) if (q == qi) ti = t[q];
    ti = __shfl_sync(0xffffffffu, ti, li) / S[i * lds + i];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int rr = lane + 32 * q;
      if (rr == i) t[q] = ti;
      else if (rr < i) t[q] = fma(-S[rr * lds + i], ti, t[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (lane + 32 * q < k) U[r * ldu + lane + 32 * q] = t[q];
}
}  // namespace

size_t qrcp_scratch_bytes(int64_t ncols, int steps, int num_sms) {
  return (size_t)2 * num_sms * (sizeof(double) + sizeof(int64_t)) + (size_t)steps * sizeof(double) + 256 +
         (size_t)round_up(ncols, 256);
}

cudaError_t launch_qrcp(double* W, int64_t ld, int rows, int64_t ncols, int steps, int64_t* perm, double* Z,
                        int64_t ldz, void* scratch, int* flag, int flag_bit, int num_sms, cudaStream_t st) {
  if (rows < 1 || rows > QC_RMAX || steps < 1 || steps > rows || steps > ncols) return cudaErrorInvalidValue;
  QrcpArgs a{};
  a.W = W; a.ld = ld; a.rows = rows; a.ncols = ncols; a.steps = steps;
  char* p = reinterpret_cast<char*>(scratch);
  a.cval = reinterpret_cast<double*>(p); p += 2 * num_sms * sizeof(double);
  a.cidx = reinterpret_cast<int64_t*>(p); p += 2 * num_sms * sizeof(int64_t);
  a.alpha = reinterpret_cast<double*>(p); p += round_up((int64_t)steps * sizeof(double), 256);
  a.done = reinterpret_cast<unsigned char*>(p);
  a.perm = perm; a.Z = Z; a.ldz = ldz; a.flag = flag; a.flag_bit = flag_bit;
  cudaError_t e = cudaMemsetAsync(a.done, 0, (size_t)ncols, st);
  if (e != cudaSuccess) return e;
  const size_t smem = Z ? (size_t)steps * steps * sizeof(double) : 0;
  if (smem > 48 * 1024) {
    e = smem_optin(qrcp_kernel);
    if (e != cudaSuccess) return e;
  }
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, qrcp_kernel, QC_THREADS, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorCooperativeLaunchTooLarge;
  int grid = num_sms;
  if ((int64_t)grid > ncols) grid = (int)ncols;
  void* args[] = {&a};
  // the candidate arrays are sized for num_sms CTAs
  e = cudaLaunchCooperativeKernel((void*)qrcp_kernel, dim3(grid), dim3(QC_THREADS), args, smem, st);
  ++g_kernel_launches;
  return e;
}

cudaError_t launch_gather_cols(const double* A, int64_t lda, int64_t m, const int64_t* J, int k, double* C,
                               int64_t ldc, cudaStream_t st) {
  gather_cols_kernel<<<148 * 4, 256, 0, st>>>(A, lda, m, J, k, C, ldc); ++g_kernel_launches;
  return cudaGetLastError();
}

cudaError_t launch_gather_rows(const double* A, int64_t lda, int64_t n, const int64_t* I, int k, double* R,
                               int64_t ldr, double* Rt, int64_t ldt, cudaStream_t st) {
  gather_rows_kernel<<<148 * 4, 256, 0, st>>>(A, lda, n, I, k, R, ldr, Rt, ldt); ++g_kernel_launches;
  return cudaGetLastError();
}

size_t zq_partial_bytes(int k, int num_sms) { return (size_t)num_sms * k * k * sizeof(double); }

cudaError_t launch_zq(const double* Z, int64_t ldz, const double* Q, int64_t ldq, int64_t n, int k, double* partial,
                      double* W, int ldw, int num_sms, cudaStream_t st) {
  int P = num_sms;
  if ((int64_t)P > n) P = (int)n;
  zq_partial_kernel<<<P, 256, 0, st>>>(Z, ldz, Q, ldq, n, k, partial); ++g_kernel_launches;
  zq_reduce_kernel<<<(unsigned)ceil_div((int64_t)k * k, 256), 256, 0, st>>>(partial, P, k, W, ldw); ++g_kernel_launches;
  return cudaGetLastError();
}

cudaError_t launch_rtsolve(const double* W, int ldw, const double* S, int lds, int k, double* U, int64_t ldu,
                           cudaStream_t st) {
  if (k > 128) return cudaErrorInvalidValue;
  rtsolve_kernel<<<(unsigned)ceil_div(k, 4), 128, 0, st>>>(W, ldw, S, lds, k, U, ldu); ++g_kernel_launches;
  return cudaGetLastError();
}

size_t lu_scratch_bytes(int64_t m, int num_sms) {
  return (size_t)2 * num_sms * (sizeof(double) + sizeof(int64_t)) + 256 + (size_t)round_up(m, 64) * sizeof(int);
}

cudaError_t launch_lu_rows(double* Y, int64_t ld, int64_t m, int l, void* scratch, int* flag, int flag_bit,
                           int num_sms, cudaStream_t st) {
  if (l < 1 || l > QC_RMAX || m < l) return cudaErrorInvalidValue;
  LuArgs a{};
  a.Y = Y; a.ld = ld; a.m = m; a.l = l;
  char* p = reinterpret_cast<char*>(scratch);
  a.cval = reinterpret_cast<double*>(p); p += 2 * num_sms * sizeof(double);
  a.cidx = reinterpret_cast<int64_t*>(p); p += 2 * num_sms * sizeof(int64_t);
  p = reinterpret_cast<char*>(round_up((int64_t)(uintptr_t)p, 256));
  a.stepof = reinterpret_cast<int*>(p);
  a.flag = flag; a.flag_bit = flag_bit;
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lu_rows_kernel, QC_THREADS, 0);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorCooperativeLaunchTooLarge;
  int grid = num_sms;
  if ((int64_t)grid > m) grid = (int)m;
  void* args[] = {&a};
  e = cudaLaunchCooperativeKernel((void*)lu_rows_kernel, dim3(grid), dim3(QC_THREADS), args, 0, st);
  ++g_kernel_launches;
  return e;
}

}  // namespace rsvd
