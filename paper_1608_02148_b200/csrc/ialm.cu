// ialm.cu -- the elementwise part of the randomized robust PCA loop
// (Alg. 7 rrpca; readings R17-R23 in DESIGN.md).
//
// One fused, HBM-bound pass per IALM iteration: with the rank-r
// factors of step (9) (L = U_l diag(d_l) V_l^T, never materialised: r <= 128
// FMAs per entry recompute it in registers) it does steps (10)-(11), the
// residual partials and the next rsvd input of step (6):
//   S = shrink(A - L + Z/mu, lambda/mu)       step (10)
//   E = A - L - S ;  Z = Z + E mu             step (11)
//   partial += E^2                            convergence test (R21)
//   M = A - S + Z/mu_next                     step (6) of the next iteration
// Reads A, S, Z (24 B/entry), writes S, Z, M (24 B/entry).  Block layout: one
// CTA per (row range, 256-column chunk), threads over columns (coalesced),
// V diag(d) row of the thread's column held in registers, 8-row tiles of U
// broadcast from shared memory.  The divisions by mu of Alg. 7 are
// multiplications by the host-computed 1/mu (a last-bit difference, inside the
// parity tolerance).  Deterministic: fixed grid, fixed per-thread order,
// fixed-order block sums.
#include <math.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace rsvd {

constexpr int IALM_THREADS = 256;
int ialm_blocks() { return 148 * 4; }

__device__ __forceinline__ double shrink(double x, double t) {
  const double a = fabs(x) - t;
  return a > 0.0 ? copysign(a, x) : 0.0;
}

// Tile = IALM_TR (8; 4 for R > 64, register budget) rows x 256 columns (one column per thread, coalesced rows).
// blockIdx.y selects the 256-column chunk, blockIdx.x a contiguous row range.
// The thread's V diag(dl) row (R >= r, zero padded) lives in shared memory for
// R <= 32 ([t/2][column] double2, conflict-free; keeps registers for 3 CTAs
// per SM) and in registers above; the tile's U rows are broadcast from shared
// memory (one barrier pair per tile, not per row).
// L(i, j) = sum_t U(i, t) (dl_t V(j, t)), t ascending.
// UPDATE: steps (10)-(11) + residual partial + next M (see header);
// else: write L (the returned low-rank component, step (9)).
template <int R, bool UPDATE>
__global__ void __launch_bounds__(IALM_THREADS, R <= 32 ? (UPDATE ? 2 : 3) : 1) ialm_tile_kernel(
    const double* __restrict__ A, double* __restrict__ S, double* __restrict__ Z, double* __restrict__ Mn,
    int64_t ld, int64_t m, int64_t n, const double* __restrict__ U, int64_t ldu, const double* __restrict__ V,
    int64_t ldv, const double* __restrict__ dl, int r, double inv_mu, double tshr, double mu,
    double inv_mu_next, int64_t rows_per, double* __restrict__ partial) {
  constexpr int IALM_TR = R > 64 ? 4 : 8;   // rows per tile: 2*TR loads in flight per thread
  __shared__ __align__(16) double us[IALM_TR][R];
  __shared__ double red[32];
  const int64_t j = (int64_t)blockIdx.y * IALM_THREADS + threadIdx.x;
  const bool jv = j < n;
  constexpr bool VS = R <= 32;
  extern __shared__ double2 vds[];   // VS: [R/2][IALM_THREADS]
  double vd[VS ? 2 : R];
  if constexpr (VS) {
#pragma unroll 4
    for (int t = 0; t < R; t += 2) {
      vd[0] = (t < r && jv) ? V[j * ldv + t] * dl[t] : 0.0;
      vd[1] = (t + 1 < r && jv) ? V[j * ldv + t + 1] * dl[t + 1] : 0.0;
      vds[(t / 2) * IALM_THREADS + threadIdx.x] = make_double2(vd[0], vd[1]);
    }
  } else {
#pragma unroll
    for (int t = 0; t < R; ++t) vd[t] = (t < r && jv) ? V[j * ldv + t] * dl[t] : 0.0;
  }
  const int64_t r0 = (int64_t)blockIdx.x * rows_per;
  const int64_t r1 = (r0 + rows_per) < m ? (r0 + rows_per) : m;
  double acc = 0.0;
  // U tiles are prefetched into registers one tile ahead (UPT values per
  // thread) and the tile's A, Z loads are issued before the barrier pair, so
  // neither latency sits on the per-tile critical path.
  constexpr int UPT = (IALM_TR * R + IALM_THREADS - 1) / IALM_THREADS;
  double un[UPT];
  auto load_u = [&](int64_t i0) {
#pragma unroll
    for (int c = 0; c < UPT; ++c) {
      const int e = threadIdx.x + c * IALM_THREADS;
      const int q = e / R, t = e % R;
      un[c] = (e < IALM_TR * R && t < r && i0 + q < r1) ? U[(i0 + q) * ldu + t] : 0.0;
    }
  };
  if (r0 < r1) load_u(r0);
#pragma unroll 1
  for (int64_t i0 = r0; i0 < r1; i0 += IALM_TR) {
    const int nq = (int)((r1 - i0) < IALM_TR ? (r1 - i0) : IALM_TR);
    // ld laundered per tile: stops the compiler from keeping 8 row pointers per
    // array live across the loop (register blow-up and spills)
    int64_t ldt;
    asm volatile("mov.b64 %0, %1;" : "=l"(ldt) : "l"(ld));
    const int64_t e0 = i0 * ldt + j;
    double a[IALM_TR], z[IALM_TR];
    if constexpr (UPDATE) {
#pragma unroll
      for (int q = 0; q < IALM_TR; ++q) {
        a[q] = (jv && q < nq) ? A[e0 + q * ldt] : 0.0;
        z[q] = (jv && q < nq) ? Z[e0 + q * ldt] : 0.0;
      }
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < UPT; ++c) {
      const int e = threadIdx.x + c * IALM_THREADS;
      if (e < IALM_TR * R) us[e / R][e % R] = un[c];
    }
    __syncthreads();
    if (i0 + IALM_TR < r1) load_u(i0 + IALM_TR);
    if (!jv) continue;
    double L[IALM_TR];
#pragma unroll
    for (int q = 0; q < IALM_TR; ++q) L[q] = 0.0;
#pragma unroll
    for (int t = 0; t < R; t += 2) {
      double v0, v1;
      if constexpr (VS) {
        const double2 w = vds[(t / 2) * IALM_THREADS + threadIdx.x];
        v0 = w.x; v1 = w.y;
      } else {
        v0 = vd[t]; v1 = vd[t + 1];
      }
#pragma unroll
      for (int q = 0; q < IALM_TR; ++q) {
        const double2 u = *reinterpret_cast<const double2*>(&us[q][t]);
        L[q] = fma(u.x, v0, L[q]);
        L[q] = fma(u.y, v1, L[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < IALM_TR; ++q) {
      if (q >= nq) continue;
      const int64_t e = e0 + q * ldt;
      if constexpr (UPDATE) {
        const double s = shrink(a[q] - L[q] + z[q] * inv_mu, tshr);
        const double E = a[q] - L[q] - s;
        const double zn = z[q] + E * mu;
        S[e] = s;
        Z[e] = zn;
        if (Mn) Mn[e] = a[q] - s + zn * inv_mu_next;
        acc += E * E;
      } else {
        Mn[e] = L[q];
      }
    }
  }
  if constexpr (UPDATE) {
    const double tot = block_sum(acc, red);
    if (threadIdx.x == 0) partial[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = tot;
  }
}

template <bool UPDATE>
static cudaError_t launch_tile(const double* A, double* S, double* Z, double* Mn, int64_t ld, int64_t m, int64_t n,
                               const double* U, int64_t ldu, const double* V, int64_t ldv, const double* dl, int r,
                               double inv_mu, double tshr, double mu, double inv_mu_next, double* partial,
                               int nblocks, cudaStream_t st) {
  // grid: ceil(n / 256) column chunks x (nblocks / chunks) row ranges, so that
  // the partial count gx * gy <= nblocks (the caller's partial buffer)
  const int gy = (int)ceil_div(n, (int64_t)IALM_THREADS);
  if (gy > nblocks) return cudaErrorInvalidValue;
  const int gx = std::max(1, nblocks / gy);
  const dim3 grid(gx, gy);
  const int TR = r > 64 ? 4 : 8;
  const int64_t rows_per = ceil_div(ceil_div(m, (int64_t)gx), (int64_t)TR) * TR;
#define IALM_CASE(RR)                                                                                         \
  if (r <= RR) {                                                                                              \
    const int dsm = RR <= 32 ? RR * IALM_THREADS * 8 : 0;                                                     \
    if (dsm > 48 * 1024) {                                                                                    \
      const cudaError_t ea = smem_optin(ialm_tile_kernel<RR, UPDATE>);                                        \
      if (ea != cudaSuccess) return ea;                                                                       \
    }                                                                                                         \
    ialm_tile_kernel<RR, UPDATE><<<grid, IALM_THREADS, dsm, st>>>(A, S, Z, Mn, ld, m, n, U, ldu, V, ldv, dl, r, \
                                                                inv_mu, tshr, mu, inv_mu_next, rows_per,      \
                                                                partial);                                     \
    ++g_kernel_launches;                                                                                      \
    return cudaGetLastError();                                                                                \
  }
  IALM_CASE(8) IALM_CASE(16) IALM_CASE(32) IALM_CASE(64) IALM_CASE(128)
#undef IALM_CASE
  return cudaErrorInvalidValue;
}

int ialm_partials(int64_t n, int nblocks) {
  const int gy = (int)ceil_div(n, (int64_t)IALM_THREADS);
  return std::max(1, nblocks / gy) * gy;
}

cudaError_t launch_ialm_update(const double* A, double* S, double* Z, double* Mnext, int64_t ld, int64_t m,
                               int64_t n, const double* U, int64_t ldu, const double* V, int64_t ldv,
                               const double* dl, int r, double inv_mu, double mu, double lam, double inv_mu_next,
                               double* partial, int nblocks, cudaStream_t st) {
  return launch_tile<true>(A, S, Z, Mnext, ld, m, n, U, ldu, V, ldv, dl, r, inv_mu, lam * inv_mu, mu, inv_mu_next,
                           partial, nblocks, st);
}

// M = A - S + Z / mu (contiguous, ld == n): vectorised grid-stride
__global__ void form_m_kernel(const double* __restrict__ A, const double* __restrict__ S,
                              const double* __restrict__ Z, int64_t total, double inv_mu, double* __restrict__ M) {
  const int64_t h = total / 2;
  const double2* A2 = reinterpret_cast<const double2*>(A);
  const double2* S2 = reinterpret_cast<const double2*>(S);
  const double2* Z2 = reinterpret_cast<const double2*>(Z);
  double2* M2 = reinterpret_cast<double2*>(M);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < h; e += (int64_t)gridDim.x * blockDim.x) {
    const double2 a = A2[e], s = S2[e], z = Z2[e];
    M2[e] = make_double2(a.x - s.x + z.x * inv_mu, a.y - s.y + z.y * inv_mu);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (total & 1)) {
    const int64_t e = total - 1;
    M[e] = A[e] - S[e] + Z[e] * inv_mu;
  }
}

cudaError_t launch_ialm_form_m(const double* A, const double* S, const double* Z, int64_t ld, int64_t m,
                               int64_t n, double inv_mu, double* M, cudaStream_t st) {
  if (ld != n) return cudaErrorInvalidValue;
  form_m_kernel<<<148 * 8, 256, 0, st>>>(A, S, Z, m * n, inv_mu, M); ++g_kernel_launches;
  return cudaGetLastError();
}

cudaError_t launch_lowrank_materialise(const double* U, int64_t ldu, const double* V, int64_t ldv,
                                       const double* dl, int r, int64_t m, int64_t n, double* L, int64_t ldl,
                                       cudaStream_t st) {
  if (r < 1) return cudaMemset2DAsync(L, ldl * 8, 0, n * 8, m, st);
  return launch_tile<false>(nullptr, nullptr, nullptr, L, ldl, m, n, U, ldu, V, ldv, dl, r, 0.0, 0.0, 0.0, 0.0,
                            nullptr, ialm_blocks(), st);
}

// dl_t = d_t - 1/mu for d_t > 1/mu, else 0 (steps (7)-(8), d descending);
// out[0] = l = #{d_t > 1/mu} as a double
__global__ void ialm_threshold_kernel(const double* __restrict__ d, int k, double inv_mu, double* __restrict__ dl,
                                      double* __restrict__ out) {
  if (threadIdx.x != 0) return;
  int l = 0;
  for (int t = 0; t < k; ++t) {
    const bool keep = d[t] > inv_mu;
    l += keep ? 1 : 0;
    dl[t] = keep ? d[t] - inv_mu : 0.0;
  }
  out[0] = (double)l;
}

cudaError_t launch_ialm_threshold(const double* d, int k, double inv_mu, double* dl, double* l_out,
                                  cudaStream_t st) {
  ialm_threshold_kernel<<<1, 32, 0, st>>>(d, k, inv_mu, dl, l_out); ++g_kernel_launches;
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

__global__ void scale_copy_kernel(const double* __restrict__ A, int64_t total, double f, double* __restrict__ Z) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x)
    Z[e] = A[e] / f;
}

cudaError_t launch_scale_copy(const double* A, int64_t ld, int64_t m, int64_t n, double f, double* Z,
                              cudaStream_t st) {
  if (ld != n) return cudaErrorInvalidValue;
  scale_copy_kernel<<<148 * 8, 256, 0, st>>>(A, m * n, f, Z); ++g_kernel_launches;
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
