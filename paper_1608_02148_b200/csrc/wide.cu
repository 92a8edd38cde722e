// wide.cu -- sketch widths l > 120 ("wide plans"; reading R34).
//
// The single-CTA panel, Cholesky and Jacobi kernels keep the l x l factors
// and the panel rows of a leaf in shared memory, which bounds them at l <= 120.
// A wide plan runs the same steps of Alg. 4 / Alg. 5 with
//  * every pass and every small-K product as DMMA gemm_pass launches over
//    column blocks of <= 128 (api.cu gemm_blocks; A is read ceil(l/128) times
//    per pass: the price of more than 128 accumulators per row);
//  * the panels by shifted CholeskyQR3 (api.cu orth_wide): the Gram from
//    gemm_pass (TN form), the Cholesky factor of G (+ s I) and its inverse
//    from chol_wide_kernel below;
//  * the SVD of R_B^T by jacobi_wide_kernel below (Alg. 5 step 2);
//  * for rrpca at a rank above 128 (Remark 2's deterministic SVD):
//    L = U diag(d_l) V^T materialised by gemm_pass and the IALM update of
//    steps (10)-(11) as a plain elementwise pass (ialm_dense_kernel).
// The two factor kernels are cooperative launches (one CTA per SM, grid
// barriers): the l x l factors (<= 128 MB at l = 4096) live in global memory
// and L2, every cross-CTA read goes through L2 (__ldcg: no stale L1 lines).
// The rotation rule is the oracle's (reading R8): rotate iff
// |gamma| > tau sqrt(alpha beta), tau = l 2^-52; zeta = (beta - alpha) / (2 gamma),
// t = sgn(zeta) / (|zeta| + sqrt(1 + zeta^2)), c = 1/sqrt(1 + t^2), s = c t;
// stop after a sweep without rotation, cap 30 sweeps.  Pairs meet in the
// circle-method round robin (every pair once per sweep of Lp - 1 rounds, Lp =
// l rounded up to even), one warp per pair; each round's pairs are disjoint,
// so the result does not depend on the scheduling (deterministic).
#include <cooperative_groups.h>
#include <math.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace rsvd {

namespace cg = cooperative_groups;

namespace {

constexpr int WT = 256;            // threads per CTA of the cooperative kernels
constexpr int kWideCap = 30;       // Jacobi sweep cap (R8)

struct CholWideArgs {
  const double* G; int ldg; int l; int np;
  double* Wk;                      // l x np working copy of the upper triangle, then the x vectors
  double* d0;                      // original diagonal
  double* R; double* Rinv;         // np x np, ld np, zero padded
  int* flag; int flag_bit;
  double shift_c;                  // > 0: factor G + s I, s = shift_c trace(G) (shifted CholeskyQR)
};

// G (+ s I) = R^T R (right-looking, one grid barrier per column), then R^-1 by
// back substitution (one warp per column of R^-1).  Breakdown (pivot <= 1e-13
// of its original diagonal, or non-finite; as launch_chol_aug): flag |= bit,
// the column is treated as dropped (r_jj = 1, rest of row j zero).
__global__ void __launch_bounds__(WT) chol_wide_kernel(CholWideArgs a) {
  cg::grid_group grid = cg::this_grid();
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int l = a.l, np = a.np;
  double shift = 0.0;
  if (a.shift_c > 0.0) {            // every CTA sums the diagonal in the same order
    __shared__ double red[32];
    double t = 0.0;
    for (int i = threadIdx.x; i < l; i += blockDim.x) t += a.G[(int64_t)i * a.ldg + i];
    shift = a.shift_c * block_sum(t, red);
  }
  for (int64_t e = gt; e < (int64_t)np * np; e += nth) {
    const int i = (int)(e / np), c = (int)(e - (int64_t)i * np);
    a.R[e] = 0.0;
    a.Rinv[e] = 0.0;
    if (i < l && c < l) a.Wk[e] = c >= i ? a.G[(int64_t)i * a.ldg + c] + (i == c ? shift : 0.0) : 0.0;
    if (i == c && i < l) a.d0[i] = a.G[(int64_t)i * a.ldg + i] + shift;
  }
  grid.sync();
  bool broke = false;
  for (int j = 0; j < l; ++j) {
    const double* wj = a.Wk + (int64_t)j * np;
    const double d = __ldcg(wj + j);
    const bool bad = !(d > 1e-13 * __ldcg(a.d0 + j)) || !isfinite(d);
    broke |= bad;
    const double rjj = bad ? 1.0 : sqrt(d), inv_r = 1.0 / rjj, inv_d = bad ? 0.0 : 1.0 / d;
    for (int64_t c = j + gt; c < l; c += nth)
      a.R[(int64_t)j * np + c] = c == j ? rjj : (bad ? 0.0 : __ldcg(wj + c) * inv_r);
    const int64_t t = l - j - 1;
    if (!bad) {
      for (int64_t e = gt; e < t * t; e += nth) {
        const int64_t i = j + 1 + e / t, c = j + 1 + e % t;
        if (c < i) continue;
        double* w = a.Wk + i * np + c;
        *w = __ldcg(w) - __ldcg(wj + i) * __ldcg(wj + c) * inv_d;
      }
    }
    grid.sync();
  }
  if (broke && gt == 0) atomicOr(a.flag, a.flag_bit);
  // R^-1 column c: x_c = 1 / r_cc, x_i = -(sum_{t=i+1..c} r_it x_t) / r_ii, i descending;
  // x kept in row c of Wk (contiguous, owned by this warp)
  const int lane = threadIdx.x & 31;
  const int64_t nw = nth >> 5, gw = gt >> 5;
  for (int64_t c = gw; c < l; c += nw) {
    double* x = a.Wk + c * np;
    if (lane == 0) x[c] = 1.0 / __ldcg(a.R + c * np + c);
    __syncwarp();
    for (int64_t i = c - 1; i >= 0; --i) {
      const double* ri = a.R + i * np;
      double s = 0.0;
      for (int64_t t = i + 1 + lane; t <= c; t += 32) s = fma(__ldcg(ri + t), x[t], s);
      s = warp_sum(s);
      if (lane == 0) x[i] = -s / __ldcg(ri + i);
      __syncwarp();
    }
    for (int64_t i = lane; i <= c; i += 32) a.Rinv[i * np + c] = x[i];
    __syncwarp();
  }
}

struct JacWideArgs {
  const double* R; int ldr; int l; int Lp;
  double* Xc; double* Jc;          // Lp columns of l rows each (column j at + j l)
  double* sg; int* cnt;            // column norms; per-sweep rotation counters
  double* sigma; double* W; double* J; int ldo;
  int* flag; int* sweeps;
  unsigned long long* gmax;        // bits of max |x| (zeroed by the launcher)
};

// pair i of round r of the circle method over n (even) players: the last is
// fixed, the others rotate (m = n - 1 is odd, so every pair meets once in m rounds)
__device__ __forceinline__ void rr_pair(int n, int r, int i, int& a, int& b) {
  const int m = n - 1;
  if (i == 0) { a = r % m; b = n - 1; return; }
  a = (r + i) % m;
  b = (r - i + m) % m;
}

// One-sided Jacobi on X = R^T (column j of X = row j of R): X J = W Sigma.
__global__ void __launch_bounds__(WT) jacobi_wide_kernel(JacWideArgs a) {
  cg::grid_group grid = cg::this_grid();
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int l = a.l, Lp = a.Lp, lane = threadIdx.x & 31;
  const int nw = (int)(nth >> 5), gw = (int)(gt >> 5);
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  double mx = 0.0;
  for (int64_t e = gt; e < (int64_t)l * l; e += nth) {
    const int j = (int)(e / l), i = (int)(e - (int64_t)j * l);
    const double v = i >= j ? a.R[(int64_t)j * a.ldr + i] : 0.0;
    if (!isfinite(v)) bad = 1;
    mx = fmax(mx, fabs(v));
    a.Xc[e] = v;
    a.Jc[e] = i == j ? 1.0 : 0.0;
  }
  // max |x| over the grid (non-negative doubles order as their bit patterns;
  // the slot is zeroed by the launcher) for the power-of-two prescaling (R35)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0 && mx > 0.0 && isfinite(mx))
    atomicMax(a.gmax, (unsigned long long)__double_as_longlong(mx));
  for (int64_t e = gt; e < (int64_t)a.ldo * a.ldo; e += nth) { a.W[e] = 0.0; a.J[e] = 0.0; }
  if (gt < 32) a.cnt[gt] = 0;
  __syncthreads();
  if (threadIdx.x == 0 && bad) atomicOr(a.flag, 4);
  grid.sync();
  // X <- 2^-E X (exact), sigma <- 2^E sigma at the end: the squared norms of the
  // rotation test stay in range whatever the scale of A (as jac_prescale, R35)
  double jscale = 1.0;
  {
    const double gm = __longlong_as_double((long long)__ldcg(a.gmax));
    if (gm > 0.0) {
      int ex;
      frexp(gm, &ex);
      const double sc = ldexp(1.0, -ex);
      jscale = ldexp(1.0, ex);
      for (int64_t e = gt; e < (int64_t)l * l; e += nth) a.Xc[e] *= sc;
    }
  }
  grid.sync();
  const double tol = (double)l * 0x1.0p-52;
  int sweeps = 0;
  bool conv = false;
  for (int sw = 0; sw <= kWideCap; ++sw) {
    int rot = 0;
    for (int r = 0; r < Lp - 1; ++r) {
      for (int pi = gw; pi < Lp / 2; pi += nw) {
        int pa, pb;
        rr_pair(Lp, r, pi, pa, pb);
        const int p = min(pa, pb), q = max(pa, pb);
        if (q >= l) continue;
        double* xp = a.Xc + (int64_t)p * l;
        double* xq = a.Xc + (int64_t)q * l;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int i = lane; i < l; i += 32) {
          const double u = __ldcg(xp + i), v = __ldcg(xq + i);
          al = fma(u, u, al);
          be = fma(v, v, be);
          ga = fma(u, v, ga);
        }
        al = warp_sum(al);
        be = warp_sum(be);
        ga = warp_sum(ga);
        if (!(fabs(ga) > tol * sqrt(al * be))) continue;
        const double zeta = (be - al) / (2.0 * ga);
        const double az = fabs(zeta);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (az > 1e150 ? 2.0 * az : az + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        for (int i = lane; i < l; i += 32) {
          const double u = __ldcg(xp + i), v = __ldcg(xq + i);
          xp[i] = c * u - s * v;
          xq[i] = s * u + c * v;
        }
        double* jp = a.Jc + (int64_t)p * l;
        double* jq = a.Jc + (int64_t)q * l;
        for (int i = lane; i < l; i += 32) {
          const double u = __ldcg(jp + i), v = __ldcg(jq + i);
          jp[i] = c * u - s * v;
          jq[i] = s * u + c * v;
        }
        ++rot;
      }
      if (r == Lp - 2 && lane == 0 && rot) atomicAdd(a.cnt + sw, rot);
      grid.sync();
    }
    if (__ldcg(a.cnt + sw) == 0) { conv = true; break; }
    ++sweeps;
  }
  // sigma_j = ||x_j||, stable descending ranks, W(:, rank) = x_j / sigma_j, J(:, rank) = J_j
  for (int j = gw; j < l; j += nw) {
    const double* xj = a.Xc + (int64_t)j * l;
    double s2 = 0.0;
    for (int i = lane; i < l; i += 32) { const double u = __ldcg(xj + i); s2 = fma(u, u, s2); }
    s2 = warp_sum(s2);
    if (lane == 0) a.sg[j] = sqrt(s2);
  }
  grid.sync();
  for (int j = gw; j < l; j += nw) {
    const double sj = __ldcg(a.sg + j);
    int rk = 0;
    for (int i = lane; i < l; i += 32) {
      const double si = __ldcg(a.sg + i);
      rk += (si > sj) || (si == sj && i < j);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rk += __shfl_xor_sync(0xffffffffu, rk, o);
    if (lane == 0) a.sigma[rk] = sj * jscale;
    const double inv = sj > 0.0 ? 1.0 / sj : 1.0;
    const double* xj = a.Xc + (int64_t)j * l;
    const double* jj = a.Jc + (int64_t)j * l;
    for (int i = lane; i < l; i += 32) {
      a.W[(int64_t)i * a.ldo + rk] = __ldcg(xj + i) * inv;
      a.J[(int64_t)i * a.ldo + rk] = __ldcg(jj + i);
    }
  }
  if (gt == 0) {
    if (!conv) atomicOr(a.flag, 2);
    if (a.sweeps) *a.sweeps = sweeps;
  }
}

struct HqrWideArgs {
  double* W; int64_t rows; int l; int np;   // saved panel (rows x np), overwritten by the reflectors
  double* Q;                                // output Q (rows x np, first l columns)
  double* R;                                // output R (np x np, upper, zero padded), nullable
  double* part;                             // grid x np partial sums
  double* al; double* vt; double* vj;       // per column: alpha, v^T v, v_j
  int* flag; int bit;                       // runs only if (*flag & bit); clears the bit
  int ran_bit;                              // set when it ran (informational)
};

// CTA b's rows: [b rows / G, (b + 1) rows / G)
__device__ __forceinline__ int64_t hw_row(int64_t rows, int G, int b) { return rows * b / G; }

// Partial sums over this CTA's rows of f(i, c) for columns c in [c0, c1), one
// warp per column, written to part[blockIdx.x * np + c]; then a grid barrier.
template <typename F>
__device__ __forceinline__ void hw_col_sums(const HqrWideArgs& a, int64_t r0, int64_t r1, int c0, int c1, F f,
                                            cg::grid_group& grid) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int c = c0 + warp; c < c1; c += nw) {
    double s = 0.0;
    for (int64_t i = r0 + lane; i < r1; i += 32) s += f(i, c);
    s = warp_sum(s);
    if (lane == 0) a.part[(int64_t)blockIdx.x * a.np + c] = s;
  }
  grid.sync();
}

// The grid's sums of columns [c0, c1) into tot (shared), fixed CTA order:
// identical in every CTA
__device__ __forceinline__ void hw_totals(const HqrWideArgs& a, int c0, int c1, double* tot) {
  for (int c = c0 + threadIdx.x; c < c1; c += blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < (int)gridDim.x; ++b) s += __ldcg(a.part + (int64_t)b * a.np + c);
    tot[c] = s;
  }
  __syncthreads();
}

// Householder QR of a wide panel in global memory (the fallback of a wide
// plan's CholeskyQR, reading R34): column j -- ||x||, alpha = -sgn(x_0)||x||,
// v = x - alpha e_0 (skipped when ||x|| = 0, R_jj = 0); H = I - 2 v v^T / v^T v
// applied to the trailing columns; then the explicit Q = H_0 ... H_{l-1} [I; 0]
// by backward accumulation and diag(R) >= 0 (sign flips of R's rows and Q's
// columns), as the oracle's hqr.  Grid sums in fixed CTA order
// (deterministic).  Runs only when the call's breakdown bit is set.
__global__ void __launch_bounds__(WT) hqr_wide_kernel(HqrWideArgs a) {
  if ((*(volatile int*)a.flag & a.bit) == 0) return;   // uniform: read before any barrier
  cg::grid_group grid = cg::this_grid();
  const int G = gridDim.x, l = a.l, np = a.np;
  const int64_t r0 = hw_row(a.rows, G, blockIdx.x), r1 = hw_row(a.rows, G, blockIdx.x + 1);
  double* W = a.W;
  extern __shared__ double tot[];                        // np doubles
  for (int j = 0; j < l; ++j) {
    // ||x||^2 over rows >= j
    hw_col_sums(a, r0 > j ? r0 : j, r1, j, j + 1, [&](int64_t i, int c) { const double w = W[i * np + c]; return w * w; }, grid);
    hw_totals(a, j, j + 1, tot);
    const double nx2 = tot[j];
    const double x0 = __ldcg(W + (int64_t)j * np + j);
    const double nx = sqrt(nx2);
    const double alpha = nx == 0.0 ? 0.0 : (x0 >= 0.0 ? -nx : nx);
    const double v0 = x0 - alpha;
    const double vtv = nx2 - x0 * x0 + v0 * v0;
    if (blockIdx.x == 0 && threadIdx.x == 0) { a.al[j] = alpha; a.vt[j] = vtv; a.vj[j] = v0; }
    __syncthreads();                                     // tot[j] read by every thread
    if (nx == 0.0 || !(vtv > 0.0)) { grid.sync(); continue; }
    // d_c = v^T W[:, c] for c > j (v_j = v0, v_i = W[i][j] below)
    hw_col_sums(a, r0 > j ? r0 : j, r1, j + 1, l, [&](int64_t i, int c) {
      const double vi = i == j ? v0 : W[i * np + j];
      return vi * W[i * np + c];
    }, grid);
    const double f = 2.0 / vtv;
    hw_totals(a, j + 1, l, tot);
    for (int c = j + 1; c < l; ++c) {
      const double dc = tot[c] * f;
      for (int64_t i = (r0 > j ? r0 : j) + threadIdx.x; i < r1; i += blockDim.x) {
        const double vi = i == j ? v0 : W[i * np + j];
        W[i * np + c] -= dc * vi;
      }
    }
    grid.sync();
  }
  // R (upper): R_jj = alpha_j, R_jc = W[j][c] (c > j); signs so that diag(R) >= 0
  if (a.R) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)np * np; e += (int64_t)G * blockDim.x) {
      const int i = (int)(e / np), c = (int)(e % np);
      double v = 0.0;
      if (i < l && c < l && c >= i) {
        const double sg = __ldcg(a.al + i) < 0.0 ? -1.0 : 1.0;
        v = sg * (c == i ? __ldcg(a.al + i) : __ldcg(W + (int64_t)i * np + c));
      }
      a.R[e] = v;
    }
  }
  // Q = [I; 0], then for j = l-1 .. 0: Q[:, j:] -= (2 / v^T v) v (v^T Q[:, j:])
  for (int64_t i = r0; i < r1; ++i)
    for (int c = threadIdx.x; c < l; c += blockDim.x) a.Q[i * np + c] = i == c ? 1.0 : 0.0;
  grid.sync();
  for (int j = l - 1; j >= 0; --j) {
    const double vtv = __ldcg(a.vt + j), v0 = __ldcg(a.vj + j);
    if (__ldcg(a.al + j) == 0.0 && v0 == 0.0) continue;      // skipped column (H = I)
    if (!(vtv > 0.0)) continue;
    hw_col_sums(a, r0 > j ? r0 : j, r1, j, l, [&](int64_t i, int c) {
      const double vi = i == j ? v0 : W[i * np + j];
      return vi * a.Q[i * np + c];
    }, grid);
    const double f = 2.0 / vtv;
    hw_totals(a, j, l, tot);
    for (int c = j; c < l; ++c) {
      const double dc = tot[c] * f;
      for (int64_t i = (r0 > j ? r0 : j) + threadIdx.x; i < r1; i += blockDim.x) {
        const double vi = i == j ? v0 : W[i * np + j];
        a.Q[i * np + c] -= dc * vi;
      }
    }
    grid.sync();
  }
  // diag(R) >= 0: Q(:, j) *= sgn(alpha_j) where alpha_j < 0
  for (int64_t i = r0; i < r1; ++i)
    for (int c = threadIdx.x; c < l; c += blockDim.x)
      if (__ldcg(a.al + c) < 0.0) a.Q[i * np + c] = -a.Q[i * np + c];
  grid.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    atomicAnd(a.flag, ~a.bit);
    atomicOr(a.flag, a.ran_bit);
  }
}

template <typename K>
cudaError_t coop_launch(K kernel, void* arg, int num_sms, cudaStream_t st) {
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, WT, 0);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorCooperativeLaunchTooLarge;
  void* args[] = {arg};
  e = cudaLaunchCooperativeKernel((void*)kernel, dim3(num_sms), dim3(WT), args, 0, st);
  ++g_kernel_launches;
  return e;
}

// Bt (r x ldb) = diag(dl) V^T for V (n x r, ld ldv); columns n..ldb-1 zero
__global__ void scale_transpose_kernel(const double* __restrict__ V, int64_t ldv, int64_t n, int r,
                                       const double* __restrict__ dl, double* __restrict__ Bt, int64_t ldb) {
  pdl_wait();
  pdl_trigger();
  const int64_t total = (int64_t)r * ldb;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = e / ldb, j = e - t * ldb;
    Bt[e] = j < n ? dl[t] * V[j * ldv + t] : 0.0;
  }
}

__device__ __forceinline__ double shrink_w(double x, double t) {
  const double a = fabs(x) - t;
  return a > 0.0 ? copysign(a, x) : 0.0;
}

// Steps (10)-(11) of Alg. 7 with L materialised (as ialm_tile_kernel, UPDATE):
// S = shrink(A - L + Z inv_mu, tshr); E = A - L - S; Z += mu E;
// M = A - S + Z inv_mu_next; partial[block] = sum E^2 (fixed grid: deterministic)
__global__ void ialm_dense_kernel(const double* __restrict__ A, double* __restrict__ S, double* __restrict__ Z,
                                  double* __restrict__ Mn, const double* __restrict__ L, int64_t total, double inv_mu,
                                  double tshr, double mu, double inv_mu_next, double* __restrict__ partial) {
  pdl_wait();
  pdl_trigger();
  __shared__ double red[32];
  double acc = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const double a = A[e], l = L[e], z = Z[e];
    const double s = shrink_w(a - l + z * inv_mu, tshr);
    const double E = a - l - s;
    const double zn = z + E * mu;
    S[e] = s;
    Z[e] = zn;
    Mn[e] = a - s + zn * inv_mu_next;
    acc += E * E;
  }
  const double tot = block_sum(acc, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

}  // namespace

size_t chol_wide_scratch_bytes(int npad) { return ((size_t)npad * npad + npad) * sizeof(double) + 256; }

cudaError_t launch_chol_wide(const double* G, int ldg, int l, int npad, double* R, double* Rinv, void* scratch,
                             int* flag, int flag_bit, double shift_c, int num_sms, cudaStream_t st) {
  if (l < 1 || npad < l || ldg < l) return cudaErrorInvalidValue;
  CholWideArgs a;
  a.G = G; a.ldg = ldg; a.l = l; a.np = npad;
  a.Wk = reinterpret_cast<double*>(scratch);
  a.d0 = a.Wk + (size_t)npad * npad;
  a.R = R; a.Rinv = Rinv; a.flag = flag; a.flag_bit = flag_bit; a.shift_c = shift_c;
  return coop_launch(chol_wide_kernel, &a, num_sms, st);
}

cudaError_t launch_hqr_wide(double* Wsaved, int64_t rows, int l, int npad, double* Q, double* R, double* part,
                            void* scratch, int* flag, int bit, int ran_bit, int num_sms, cudaStream_t st) {
  if (l < 1 || npad < l || rows < l) return cudaErrorInvalidValue;
  HqrWideArgs a;
  a.W = Wsaved; a.rows = rows; a.l = l; a.np = npad; a.Q = Q; a.R = R; a.part = part;
  a.al = reinterpret_cast<double*>(scratch);
  a.vt = a.al + npad;
  a.vj = a.vt + npad;
  a.flag = flag; a.bit = bit; a.ran_bit = ran_bit;
  const int grid = (int)std::min<int64_t>(num_sms, std::max<int64_t>(1, rows / 32));
  const size_t smem = (size_t)npad * sizeof(double);
  cudaError_t e = cudaSuccess;
  if (smem > 48 * 1024 && (e = smem_optin(hqr_wide_kernel)) != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, hqr_wide_kernel, WT, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorCooperativeLaunchTooLarge;
  void* args[] = {&a};
  e = cudaLaunchCooperativeKernel((void*)hqr_wide_kernel, dim3(grid), dim3(WT), args, smem, st);
  ++g_kernel_launches;
  return e;
}

size_t jacobi_wide_scratch_bytes(int l) {
  const size_t Lp = (size_t)(l + (l & 1));
  return (2 * Lp * l + Lp) * sizeof(double) + 64 * sizeof(int) + 256;
}

cudaError_t launch_jacobi_wide(const double* R, int ldr, int l, double* sigma, double* W, double* J, int ldo,
                               int* flag, int* sweeps, void* scratch, int num_sms, cudaStream_t st) {
  if (l < 1 || ldo < l || ldr < l) return cudaErrorInvalidValue;
  JacWideArgs a;
  a.R = R; a.ldr = ldr; a.l = l; a.Lp = l + (l & 1);
  a.Xc = reinterpret_cast<double*>(scratch);
  a.Jc = a.Xc + (size_t)a.Lp * l;
  a.sg = a.Jc + (size_t)a.Lp * l;
  a.cnt = reinterpret_cast<int*>(a.sg + a.Lp);
  a.sigma = sigma; a.W = W; a.J = J; a.ldo = ldo; a.flag = flag; a.sweeps = sweeps;
  a.gmax = reinterpret_cast<unsigned long long*>(a.cnt + 32);
  const cudaError_t e = cudaMemsetAsync(a.gmax, 0, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  return coop_launch(jacobi_wide_kernel, &a, num_sms, st);
}

cudaError_t launch_scale_transpose(const double* V, int64_t ldv, int64_t n, int r, const double* dl, double* Bt,
                                   int64_t ldb, cudaStream_t st) {
  if (r < 1 || ldb < n) return cudaErrorInvalidValue;
  CUDA_TRY(launch_pdl(scale_transpose_kernel, dim3(148 * 4), dim3(256), 0, st, V, ldv, n, r, dl, Bt, ldb));
  ++g_kernel_launches;
  return cudaGetLastError();
}

cudaError_t launch_ialm_update_dense(const double* A, double* S, double* Z, double* Mnext, const double* L,
                                     int64_t total, double inv_mu, double mu, double lam, double inv_mu_next,
                                     double* partial, int nblocks, cudaStream_t st) {
  CUDA_TRY(launch_pdl(ialm_dense_kernel, dim3(nblocks), dim3(256), 0, st, A, S, Z, Mnext, L, total, inv_mu,
                      lam * inv_mu, mu, inv_mu_next, partial));
  ++g_kernel_launches;
  return cudaGetLastError();
}

}  // namespace rsvd
