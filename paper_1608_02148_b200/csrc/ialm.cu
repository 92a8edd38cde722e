// ialm.cu -- the elementwise part of the randomized robust PCA loop
// (Alg. 7 rrpca; readings R17-R23 in DESIGN.md).
//
// One fused, HBM-bound pass per IALM iteration: with the rank-r
// factors of step (9) (L = U_l diag(d_l) V_l^T, never materialised: r <= 32
// FMAs per entry recompute it in registers) it does steps (10)-(11), the
// residual partials and the next rsvd input of step (6):
//   S = shrink(A - L + Z/mu, lambda/mu)       step (10)
//   E = A - L - S ;  Z = Z + E mu             step (11)
//   partial += E^2                            convergence test (R21)
//   M = A - S + Z/mu_next                     step (6) of the next iteration
// Reads A, S, Z (24 B/entry), writes S, Z, M (24 B/entry).  Block layout: one
// CTA per row chunk, threads over columns (coalesced), V diag(d) row of the
// thread's column held in registers, the U row broadcast from shared memory.
// Deterministic: fixed grid, fixed per-thread order, fixed-order block sums.
#include <math.h>

#include "common.cuh"
#include "kernels.h"

namespace rsvd {

constexpr int IALM_THREADS = 256;
constexpr int RMAX = 32;
int ialm_blocks() { return 148 * 4; }

__device__ __forceinline__ double shrink(double x, double t) {
  const double a = fabs(x) - t;
  return a > 0.0 ? copysign(a, x) : 0.0;
}

__global__ void __launch_bounds__(IALM_THREADS) ialm_update_kernel(
    const double* __restrict__ A, double* __restrict__ S, double* __restrict__ Z, double* __restrict__ Mn,
    int64_t ld, int64_t m, int64_t n, const double* __restrict__ U, int64_t ldu, const double* __restrict__ V,
    int64_t ldv, const double* __restrict__ dl, int r, double mu, double lam, double mu_next,
    double* __restrict__ partial) {
  __shared__ double us[RMAX];
  __shared__ double red[32];
  const int64_t rows_per = ceil_div(m, gridDim.x);
  const int64_t r0 = blockIdx.x * rows_per;
  const int64_t r1 = (r0 + rows_per) < m ? (r0 + rows_per) : m;
  double acc = 0.0;
  const double tshr = lam / mu;
  for (int64_t j0 = 0; j0 < n; j0 += IALM_THREADS) {
    const int64_t j = j0 + threadIdx.x;
    double vd[RMAX];
#pragma unroll
    for (int t = 0; t < RMAX; ++t) vd[t] = (t < r && j < n) ? V[j * ldv + t] * dl[t] : 0.0;
    for (int64_t i = r0; i < r1; ++i) {
      __syncthreads();
      if (threadIdx.x < r) us[threadIdx.x] = U[i * ldu + threadIdx.x];
      __syncthreads();
      if (j < n) {
        double L = 0.0;
#pragma unroll
        for (int t = 0; t < RMAX; ++t)
          if (t < r) L += us[t] * vd[t];
        const int64_t e = i * ld + j;
        const double a = A[e], z = Z[e];
        const double s = shrink(a - L + z / mu, tshr);
        const double E = a - L - s;
        const double zn = z + E * mu;
        S[e] = s;
        Z[e] = zn;
        if (Mn) Mn[e] = a - s + zn / mu_next;
        acc += E * E;
      }
    }
  }
  const double tot = block_sum(acc, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

cudaError_t launch_ialm_update(const double* A, double* S, double* Z, double* Mnext, int64_t ld, int64_t m,
                               int64_t n, const double* U, int64_t ldu, const double* V, int64_t ldv,
                               const double* dl, int r, double inv_mu, double mu, double lam, double inv_mu_next,
                               double* partial, int nblocks, cudaStream_t st) {
  (void)inv_mu;
  if (r > RMAX) return cudaErrorInvalidValue;
  ialm_update_kernel<<<nblocks, IALM_THREADS, 0, st>>>(A, S, Z, Mnext, ld, m, n, U, ldu, V, ldv, dl, r, mu, lam,
                                                       1.0 / inv_mu_next, partial); ++g_kernel_launches;
  return cudaGetLastError();
}

__global__ void form_m_kernel(const double* __restrict__ A, const double* __restrict__ S,
                              const double* __restrict__ Z, int64_t ld, int64_t m, int64_t n, double mu,
                              double* __restrict__ M) {
  const int64_t total = m * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e % n, x = i * ld + j;
    M[x] = A[x] - S[x] + Z[x] / mu;
  }
}

cudaError_t launch_ialm_form_m(const double* A, const double* S, const double* Z, int64_t ld, int64_t m,
                               int64_t n, double inv_mu, double* M, cudaStream_t st) {
  form_m_kernel<<<148 * 8, 256, 0, st>>>(A, S, Z, ld, m, n, 1.0 / inv_mu, M); ++g_kernel_launches;
  return cudaGetLastError();
}

__global__ void lowrank_kernel(const double* __restrict__ U, int64_t ldu, const double* __restrict__ V,
                               int64_t ldv, const double* __restrict__ dl, int r, int64_t m, int64_t n,
                               double* __restrict__ L, int64_t ldl) {
  const int64_t total = m * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e % n;
    double s = 0.0;
    for (int t = 0; t < r; ++t) s += U[i * ldu + t] * dl[t] * V[j * ldv + t];
    L[i * ldl + j] = s;
  }
}

cudaError_t launch_lowrank_materialise(const double* U, int64_t ldu, const double* V, int64_t ldv,
                                       const double* dl, int r, int64_t m, int64_t n, double* L, int64_t ldl,
                                       cudaStream_t st) {
  lowrank_kernel<<<148 * 8, 256, 0, st>>>(U, ldu, V, ldv, dl, r, m, n, L, ldl); ++g_kernel_launches;
  return cudaGetLastError();
}

__global__ void ialm_init_kernel(const double* __restrict__ A, int64_t ld, int64_t m, int64_t n,
                                 double* __restrict__ sumsq, double* __restrict__ mx) {
  __shared__ double red[32];
  const int64_t total = m * n;
  double s = 0.0, x = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const double a = A[(e / n) * ld + (e % n)];
    s += a * a;
    x = fmax(x, fabs(a));
  }
  const double ts = block_sum(s, red);
  // block max
  for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
  __shared__ double redm[32];
  if ((threadIdx.x & 31) == 0) redm[threadIdx.x >> 5] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    double mm = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) mm = fmax(mm, redm[w]);
    sumsq[blockIdx.x] = ts;
    mx[blockIdx.x] = mm;
  }
}

cudaError_t launch_ialm_init(const double* A, int64_t ld, int64_t m, int64_t n, double* sumsq_part,
                             double* max_part, int nblocks, cudaStream_t st) {
  ialm_init_kernel<<<nblocks, 256, 0, st>>>(A, ld, m, n, sumsq_part, max_part); ++g_kernel_launches;
  return cudaGetLastError();
}

__global__ void scale_copy_kernel(const double* __restrict__ A, int64_t ld, int64_t m, int64_t n, double f,
                                  double* __restrict__ Z) {
  const int64_t total = m * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = (e / n) * ld + (e % n);
    Z[x] = A[x] / f;
  }
}

cudaError_t launch_scale_copy(const double* A, int64_t ld, int64_t m, int64_t n, double f, double* Z,
                              cudaStream_t st) {
  scale_copy_kernel<<<148 * 8, 256, 0, st>>>(A, ld, m, n, f, Z); ++g_kernel_launches;
  return cudaGetLastError();
}

__global__ void reduce_blocks_kernel(const double* part, int nb, int op_max, double* out) {
  if (threadIdx.x != 0) return;
  double s = 0.0;
  for (int i = 0; i < nb; ++i) s = op_max ? fmax(s, part[i]) : s + part[i];
  *out = s;
}

cudaError_t launch_reduce_blocks(const double* part, int nb, int op_max, double* out, cudaStream_t st) {
  reduce_blocks_kernel<<<1, 32, 0, st>>>(part, nb, op_max, out); ++g_kernel_launches;
  return cudaGetLastError();
}

}  // namespace rsvd
