// cholqr.cu -- the CholeskyQR panel path: "[Q, ~] = qr(Y)" of Alg. 2 steps
// 2-3 and Alg. 4 step 9 for a tall panel S
// (rows x Np, row-major, columns l..Np-1 exact zeros):
//
//   gram_partial   P CTAs, each G_p = S_p^T S_p over its row chunk (DMMA m8n8k4)
//   gram_reduce    G = sum_p G_p in fixed order (deterministic)
//   chol_aug       one CTA: G = R^T R and R^-1 together, by blocked symmetric
//                  elimination on [G | I] (the right block becomes R^-T)
//   panel_apply    C = S T for a small T (Np x Np): Q = S R^-1, U = Q U~, V = Q_B J
//
// Breakdown (pivot <= 1e-13 of its original diagonal, or non-finite) sets a
// flag bit; the orchestrator re-runs the call with Householder TSQR.
#include <math.h>

#include "common.cuh"
#include "kernels.h"

namespace rsvd {

namespace {
constexpr int CQ_THREADS = 256;
constexpr int GR_BK = 32;                  // rows of S per pipeline stage
constexpr int GR_STAGES = 3;

__host__ __device__ inline int ldpad(int n) { return n + ((4 - n) & 15); }   // stride = 4 (mod 16) doubles
}  // namespace

int cq_ng(int Np) { return (int)round_up(Np, 32); }

// ------------------------------------------------------------------ Gram partials
// Warps 2 (M) x 4 (N) over the Ng x Ng output; warp tile (Ng/2) x (Ng/4) =
// TI x TJ m8n8 tiles with TI = 2 TJ, TJ = Ng / 32.
template <int TJ>
__global__ void __launch_bounds__(CQ_THREADS, 1)
gram_partial_kernel(const double* __restrict__ S, int64_t lds, int64_t rows, int Np, int64_t rows_per_cta,
                    double* __restrict__ partial, Pred pr) {
  pdl_wait();
  pdl_trigger();
  if (pred_skip(pr)) return;
  constexpr int TI = 2 * TJ, NG = 32 * TJ;
  constexpr int LDT = NG + ((4 - NG) & 15);
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
  const int gq = lane >> 2, tq = lane & 3;
  const int64_t r0 = blockIdx.x * rows_per_cta;
  int64_t r1 = r0 + rows_per_cta;
  if (r1 > rows) r1 = rows;
  const int nst = (int)ceil_div(r1 > r0 ? r1 - r0 : 0, GR_BK);
  const int cpr = Np / 2;                                    // 16-byte chunks per row
  const bool lower_warp = (wm == 1 && wn < 2);               // G is symmetric: upper blocks only

  auto load = [&](int s, int it) {
    double* t = sm + s * GR_BK * LDT;
    const int64_t base = r0 + (int64_t)it * GR_BK;
    for (int ch = tid; ch < GR_BK * cpr; ch += CQ_THREADS) {
      const int r = ch / cpr, c = (ch - r * cpr) * 2;
      const int64_t g = base + r;
      const bool ok = g < r1;
      cp_async16(t + r * LDT + c, ok ? S + g * lds + c : S, ok ? 16 : 0);
    }
    if (NG > Np)                                             // zero the Ng - Np padding columns
      for (int e = tid; e < GR_BK * (NG - Np); e += CQ_THREADS) {
        const int r = e / (NG - Np), c = Np + e % (NG - Np);
        t[r * LDT + c] = 0.0;
      }
  };

  double acc[TI][TJ][2];
#pragma unroll
  for (int i = 0; i < TI; ++i)
#pragma unroll
    for (int j = 0; j < TJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < GR_STAGES - 1; ++s) {
    if (s < nst) load(s, s);
    cp_async_commit();
  }
  for (int it = 0; it < nst; ++it) {
    cp_async_wait<GR_STAGES - 2>();
    __syncthreads();
    if (it + GR_STAGES - 1 < nst) load((it + GR_STAGES - 1) % GR_STAGES, it + GR_STAGES - 1);
    cp_async_commit();
    const double* t = sm + (it % GR_STAGES) * GR_BK * LDT;
    if (lower_warp) continue;                                // strictly below the diagonal: mirrored
#pragma unroll
    for (int kk = 0; kk < GR_BK; kk += 4) {
      double af[TI], bf[TJ];
#pragma unroll
      for (int i = 0; i < TI; ++i) af[i] = t[(kk + tq) * LDT + wm * (NG / 2) + i * 8 + gq];
#pragma unroll
      for (int j = 0; j < TJ; ++j) bf[j] = t[(kk + tq) * LDT + wn * (NG / 4) + j * 8 + gq];
#pragma unroll
      for (int i = 0; i < TI; ++i)
#pragma unroll
        for (int j = 0; j < TJ; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();
  if (lower_warp) return;
  double* out = partial + (int64_t)blockIdx.x * NG * NG;
#pragma unroll
  for (int i = 0; i < TI; ++i)
#pragma unroll
    for (int j = 0; j < TJ; ++j) {
      const int r = wm * (NG / 2) + i * 8 + gq, c = wn * (NG / 4) + j * 8 + 2 * tq;
      *reinterpret_cast<double2*>(out + r * NG + c) = make_double2(acc[i][j][0], acc[i][j][1]);
    }
}

// Ng = 128 (configs 3 and 4): the upper triangle only, as the 36 upper 16 x 16
// blocks (I <= J) of the 8 x 8 block grid dealt round-robin to the 8 warps (warps w
// and w + 4 share an SM sub-partition: 5 + 4 blocks each), i.e. 9 of the 16
// blocks' DMMAs per sub-partition instead of 16 (gram_partial_kernel<4> skips
// only the two lower 64 x 32 warp tiles, so its busiest sub-partitions still do
// 4 of 4 tiles).  Same 3-stage cp.async ring; partial p holds the upper blocks.
constexpr int GS_MAXB = 5;
__global__ void __launch_bounds__(CQ_THREADS, 1)
gram_sym128_kernel(const double* __restrict__ S, int64_t lds, int64_t rows, int Np, int64_t rows_per_cta,
                   double* __restrict__ partial, Pred pr) {
  pdl_wait();
  pdl_trigger();
  if (pred_skip(pr)) return;
  constexpr int NG = 128, LDT = NG + ((4 - NG) & 15);
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int64_t r0 = blockIdx.x * rows_per_cta;
  int64_t r1 = r0 + rows_per_cta;
  if (r1 > rows) r1 = rows;
  const int nst = (int)ceil_div(r1 > r0 ? r1 - r0 : 0, GR_BK);
  const int cpr = Np / 2;
  // this warp's blocks b = warp + 8 q (b enumerates I <= J row by row; 36 blocks)
  int bI[GS_MAXB], bJ[GS_MAXB];
  const int nb = warp < 4 ? 5 : 4;
#pragma unroll
  for (int q = 0; q < GS_MAXB; ++q) {
    int b = warp + 8 * q, I = 0;
    if (b > 35) b = 35;
    while (b >= 8 - I) { b -= 8 - I; ++I; }
    bI[q] = I;
    bJ[q] = I + b;
  }
  auto load = [&](int st, int it) {
    double* t = sm + st * GR_BK * LDT;
    const int64_t base = r0 + (int64_t)it * GR_BK;
    for (int ch = tid; ch < GR_BK * cpr; ch += CQ_THREADS) {
      const int r = ch / cpr, c = (ch - r * cpr) * 2;
      const int64_t g = base + r;
      const bool ok = g < r1;
      cp_async16(t + r * LDT + c, ok ? S + g * lds + c : S, ok ? 16 : 0);
    }
    if (NG > Np)
      for (int e = tid; e < GR_BK * (NG - Np); e += CQ_THREADS) {
        const int r = e / (NG - Np), c = Np + e % (NG - Np);
        t[r * LDT + c] = 0.0;
      }
  };
  double acc[GS_MAXB][2][2][2];
#pragma unroll
  for (int q = 0; q < GS_MAXB; ++q)
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) acc[q][i][j][0] = acc[q][i][j][1] = 0.0;
#pragma unroll
  for (int st = 0; st < GR_STAGES - 1; ++st) {
    if (st < nst) load(st, st);
    cp_async_commit();
  }
  for (int it = 0; it < nst; ++it) {
    cp_async_wait<GR_STAGES - 2>();
    __syncthreads();
    if (it + GR_STAGES - 1 < nst) load((it + GR_STAGES - 1) % GR_STAGES, it + GR_STAGES - 1);
    cp_async_commit();
    const double* t = sm + (it % GR_STAGES) * GR_BK * LDT;
#pragma unroll
    for (int kk = 0; kk < GR_BK; kk += 4) {
      const double* tr = t + (kk + tq) * LDT + gq;
#pragma unroll
      for (int q = 0; q < GS_MAXB; ++q) {
        if (q >= nb) break;
        const double a0 = tr[bI[q] * 16], a1 = tr[bI[q] * 16 + 8];
        const double b0 = tr[bJ[q] * 16], b1 = tr[bJ[q] * 16 + 8];
        dmma884(acc[q][0][0][0], acc[q][0][0][1], a0, b0);
        dmma884(acc[q][0][1][0], acc[q][0][1][1], a0, b1);
        dmma884(acc[q][1][0][0], acc[q][1][0][1], a1, b0);
        dmma884(acc[q][1][1][0], acc[q][1][1][1], a1, b1);
      }
    }
  }
  cp_async_wait<0>();
  double* out = partial + (int64_t)blockIdx.x * NG * NG;
#pragma unroll
  for (int q = 0; q < GS_MAXB; ++q) {
    if (q >= nb) break;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int r = bI[q] * 16 + i * 8 + gq, c = bJ[q] * 16 + j * 8 + 2 * tq;
        *reinterpret_cast<double2*>(out + r * NG + c) = make_double2(acc[q][i][j][0], acc[q][i][j][1]);
      }
  }
}

// upper triangle of G (Np x Np, ld ldg) = sum_{p < P} partial_p (Ng x Ng), fixed order: T lanes per
// element each sum p = t, t+T, ... ascending (loads issued in batches of 8 so
// they are in flight together), then a fixed xor tree.
__global__ void gram_reduce_kernel(const double* __restrict__ partial, int P, int Ng, int Np,
                                   double* __restrict__ G, int ldg, Pred pr) {
  pdl_wait();
  pdl_trigger();
  if (pred_skip(pr)) return;
  constexpr int T = 8, B = 8;
  const int e = blockIdx.x * (blockDim.x / T) + threadIdx.x / T;
  const int t = threadIdx.x % T;
  const int r = e / Np, c = e - (e / Np) * Np;
  const bool ok = e < Np * Np && r <= c;                  // upper triangle (all chol_aug reads)
  double s = 0.0;
  if (ok) {
    const double* p = partial + r * Ng + c;                          // upper blocks hold G
    const int64_t step = (int64_t)Ng * Ng;
    for (int q0 = t; q0 < P; q0 += T * B) {
      double v[B];
#pragma unroll
      for (int b = 0; b < B; ++b) v[b] = (q0 + b * T < P) ? __ldcg(p + (q0 + b * T) * step) : 0.0;
#pragma unroll
      for (int b = 0; b < B; ++b) s += v[b];
    }
  }
#pragma unroll
  for (int o = T / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (ok && t == 0) G[r * ldg + c] = s;
}

int gram_ctas(int64_t rows, int num_sms) {
  int64_t p = ceil_div(rows, 64);
  if (p > num_sms) p = num_sms;
  if (p < 1) p = 1;
  return (int)p;
}

size_t gram_partial_bytes(int Np, int num_sms) {
  const int ng = cq_ng(Np);
  return (size_t)num_sms * ng * ng * sizeof(double);
}

cudaError_t launch_gram(const double* S, int64_t lds, int64_t rows, int Np, double* partial, double* G, int ldg,
                        int num_sms, cudaStream_t st, Pred pr) {
  if (Np % 2 || Np > 128 || rows < 1) return cudaErrorInvalidValue;
  const int ng = cq_ng(Np);
  const int P = gram_ctas(rows, num_sms);
  const int64_t rpc = ceil_div(rows, P);
  const size_t smem = (size_t)GR_STAGES * GR_BK * ldpad(ng) * sizeof(double);
  cudaError_t e = cudaSuccess;
#define RSVD_GRAM(TJ)                                                                                     \
  {                                                                                                      \
    e = smem_optin(gram_partial_kernel<TJ>); if (e != cudaSuccess) return e;                                                                                                     \
    e = launch_pdl(gram_partial_kernel<TJ>, dim3(P), dim3(CQ_THREADS), smem, st, S, lds, rows, Np, rpc, partial, pr); \
    if (e != cudaSuccess) return e;                                                                      \
  }
  const size_t smem_max = (size_t)GR_STAGES * GR_BK * ldpad(128) * sizeof(double);
  static const bool sym = [] { const char* v = getenv("RSVD_GRAM_SYM"); return !v || atoi(v) != 0; }();
  if (ng == 128 && sym) {
    e = smem_optin(gram_sym128_kernel);
    if (e != cudaSuccess) return e;
    e = launch_pdl(gram_sym128_kernel, dim3(P), dim3(CQ_THREADS), smem, st, S, lds, rows, Np, rpc, partial, pr);
    if (e != cudaSuccess) return e;
  } else {
    switch (ng / 32) {
      case 1: RSVD_GRAM(1) break;
      case 2: RSVD_GRAM(2) break;
      case 3: RSVD_GRAM(3) break;
      default: RSVD_GRAM(4) break;
    }
  }
#undef RSVD_GRAM
  ++g_kernel_launches;
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int per_block = 256 / 8;
  e = launch_pdl(gram_reduce_kernel, dim3((unsigned)ceil_div((int64_t)Np * Np, per_block)), dim3(256), 0, st,
                 (const double*)partial, P, ng, Np, G, ldg, pr);
  if (e != cudaSuccess) return e;
  ++g_kernel_launches;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ Cholesky + inverse
#ifndef CB_PROBE
#define CB_PROBE(slot)
#define CB_PROBE_DECL
#define CB_PROBE_OUT
#endif

__device__ __forceinline__ double rsqrt_nr(double p) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(p));
  const double h = 0.5 * p;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return y;
}

// G = R^T R and R^-1 by blocked symmetric elimination on [G | I] (the right
// block becomes R^-T): 16 x 16 blocks, 8 warps.  Diagonal blocks are factored
// by one warp (register columns, augmented with the identity so R_kk^-T comes
// out of the same 16 steps); panels and trailing updates are 16x16x16 DMMA
// block products.  The Ng x Ng shared array holds R in its upper blocks and
// the off-diagonal blocks of R^-T in its strictly lower blocks; the diagonal
// blocks of R^-T live in Ld.
constexpr int CB_LDB = 20;                  // 16 + 4: conflict-free fragment loads

// C (16x16, acc) += op(A) B, op(A) = A or A^T (A, B 16x16 row-major in smem)
template <bool TA>
__device__ __forceinline__ void blk_mma(double (&acc)[2][2][2], const double* A, int lda, const double* B, int ldb,
                                        int g, int t) {
#pragma unroll
  for (int kk = 0; kk < 16; kk += 4) {
    double a[2], b[2];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) a[mi] = TA ? A[(kk + t) * lda + mi * 8 + g] : A[(mi * 8 + g) * lda + kk + t];
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) b[ni] = B[(kk + t) * ldb + ni * 8 + g];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) dmma884(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
  }
}

// Diagonal block factorisation by one warp: lanes 0..15 hold the columns of
// the 16x16 block D (upper part), lanes 16..31 the columns of I; 16 column
// steps produce R_kk (left lanes) and R_kk^-T (right lanes).  Row c of the
// factor is broadcast by shuffles, the element needed by the next pivot first.
__device__ __forceinline__ void chol_diag16(double* D, int ldd, double* Lk, int ldl, const double* d0k, int lane,
                                            int* bad) {
  const int jc = lane & 15;
  const bool left = lane < 16;
  double col[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) col[i] = left ? (i <= jc ? D[i * ldd + jc] : 0.0) : (i == jc ? 1.0 : 0.0);
  double thr[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) thr[i] = 1e-13 * d0k[i];
  bool brk_any = false;
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    const double pv = __shfl_sync(0xffffffffu, col[c], c);
    const bool brk = !(pv > thr[c]) || !isfinite(pv);
    brk_any |= brk;
    const double ir = brk ? 0.0 : rsqrt_nr(pv);
    const double sv = (lane == c) ? (brk ? 1.0 : pv * ir) : col[c] * ir;
    col[c] = sv;
#pragma unroll
    for (int i = c + 1; i < 16; ++i) col[i] = fma(-__shfl_sync(0xffffffffu, sv, i), sv, col[i]);
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    if (left) D[i * ldd + jc] = (i <= jc) ? col[i] : 0.0;
    else Lk[i * ldl + jc] = (i >= jc) ? col[i] : 0.0;
  }
  if (brk_any && lane == 0) *bad = 1;
}

template <int NBLK>
__global__ void __launch_bounds__(256, 1)
chol_blk_kernel(const double* __restrict__ G, int ldg, int l, int npad, double* __restrict__ R,
                double* __restrict__ Rinv, int* flag, int flag_bit, Pred pr) {
  pdl_wait();
  pdl_trigger();
  if (pred_skip(pr)) return;
  constexpr int NG = 16 * NBLK, LDM = NG + 4;
  extern __shared__ __align__(16) double smc[];
  double* M = smc;                          // NG x LDM
  double* Ld = M + NG * LDM;                // NBLK x 16 x CB_LDB
  __shared__ double d0[NG];
  __shared__ int bad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  CB_PROBE_DECL
  if (tid == 0) bad = 0;
  // load: upper blocks of G (mirrored from the upper triangle), identity padding;
  // two consecutive columns per thread.  All of a thread's loads are issued
  // before its first shared store (one L2 round trip, not one per element pair).
  constexpr int NLD = (NG * NG / 2 + 255) / 256;
  double v0[NLD], v1[NLD];
#pragma unroll
  for (int r = 0; r < NLD; ++r) {
    const int e = tid + 256 * r;
    const int i = e / (NG / 2), j = 2 * (e - i * (NG / 2));
    v0[r] = 0.0; v1[r] = 0.0;
    if (e < NG * NG / 2 && (i >> 4) <= (j >> 4)) {
      if (i < l) {
        if (j < l) v0[r] = (j >= i) ? G[i * ldg + j] : G[j * ldg + i];
        if (j + 1 < l) v1[r] = (j + 1 >= i) ? G[i * ldg + j + 1] : G[(j + 1) * ldg + i];
      }
      if (i >= l && i == j) v0[r] = 1.0;
      if (i >= l && i == j + 1) v1[r] = 1.0;
    }
  }
#pragma unroll
  for (int r = 0; r < NLD; ++r) {
    const int e = tid + 256 * r;
    if (e >= NG * NG / 2) break;
    const int i = e / (NG / 2), j = 2 * (e - i * (NG / 2));
    *reinterpret_cast<double2*>(M + i * LDM + j) = make_double2(v0[r], v1[r]);
    if (i == j) d0[i] = (i < l) ? v0[r] : 1.0;
    if (i == j + 1) d0[i] = (i < l) ? v1[r] : 1.0;
  }
  __syncthreads();
  if (warp == 0) chol_diag16(M, LDM, Ld, CB_LDB, d0, lane, &bad);
  __syncthreads();
  CB_PROBE(0)
  for (int kb = 0; kb < NBLK; ++kb) {
    // (2) block row kb: R[kb][j] = L_kk G[kb][j] (j > kb); R^-T[kb][m] = L_kk R^-T[kb][m] (m < kb)
    {
      const double* Lk = Ld + kb * 16 * CB_LDB;
      for (int task = warp; task < NBLK - 1; task += 8) {
        const int j = task < kb ? task : task + 1;
        double* B = M + (kb * 16) * LDM + j * 16;
        double acc[2][2][2] = {};
        blk_mma<false>(acc, Lk, CB_LDB, B, LDM, g, t);
        __syncwarp();
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int ni = 0; ni < 2; ++ni)
            *reinterpret_cast<double2*>(B + (mi * 8 + g) * LDM + ni * 8 + 2 * t) = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
      }
    }
    __syncthreads();
    CB_PROBE(1)
    if (kb + 1 == NBLK) break;
    // (3) rows bi > kb: left M[bi][bj] -= R[kb][bi]^T R[kb][bj] (bj >= bi);
    //     right M[bi][m] -= R[kb][bi]^T R^-T[kb][m] (m <= kb; m == kb uses L_kk).
    // Look-ahead: warp 0 updates block (kb+1, kb+1) and factors it while warps
    // 1..7 do the rest.
    {
      auto do_task = [&](int bi, int bj) {
        const double* A = M + (kb * 16) * LDM + bi * 16;              // R[kb][bi] (used transposed)
        const double* B = (bj == kb) ? Ld + kb * 16 * CB_LDB : M + (kb * 16) * LDM + bj * 16;
        const int ldb = (bj == kb) ? CB_LDB : LDM;
        double* C = M + (bi * 16) * LDM + bj * 16;
        double acc[2][2][2] = {};
        blk_mma<true>(acc, A, LDM, B, ldb, g, t);
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int ni = 0; ni < 2; ++ni) {
            double2* cp = reinterpret_cast<double2*>(C + (mi * 8 + g) * LDM + ni * 8 + 2 * t);
            double2 v = *cp;
            v.x -= acc[mi][ni][0];
            v.y -= acc[mi][ni][1];
            *cp = v;
          }
      };
      if (warp == 0) {
        const int d = kb + 1;
        do_task(d, d);
        __syncwarp();
        chol_diag16(M + (d * 16) * LDM + d * 16, LDM, Ld + d * 16 * CB_LDB, CB_LDB, d0 + d * 16, lane, &bad);
      } else {
        const int per_row_right = kb + 1;
        int ntask = 0;
        for (int bi = kb + 1; bi < NBLK; ++bi) ntask += per_row_right + (NBLK - bi);
        for (int task = warp - 1; task < ntask; task += 7) {
          int bi = kb + 1, rem = task;
          while (rem >= per_row_right + (NBLK - bi)) { rem -= per_row_right + (NBLK - bi); ++bi; }
          const int bj = rem < per_row_right ? rem : bi + (rem - per_row_right);
          if (bi == kb + 1 && bj == kb + 1) continue;
          do_task(bi, bj);
        }
      }
    }
    __syncthreads();
    CB_PROBE(2)
  }
  CB_PROBE(3)
  // outputs: R (upper), R^-1 = (R^-T)^T, zero outside the leading l x l
  for (int e = tid; e < npad * npad; e += 256) {
    const int i = e / npad, j = e - (e / npad) * npad;
    const bool in = i < l && j < l;
    double rv = 0.0, wv = 0.0;
    if (in && j >= i) {
      rv = M[i * LDM + j];
      // Rinv[i][j] = R^-T[j][i]
      if ((j >> 4) == (i >> 4)) wv = Ld[(j >> 4) * 16 * CB_LDB + (j & 15) * CB_LDB + (i & 15)];
      else wv = M[j * LDM + i];
    }
    if (R) R[e] = rv;
    Rinv[e] = wv;
  }
  CB_PROBE(4)
  CB_PROBE_OUT
  if (tid == 0 && bad) atomicOr(flag, flag_bit);
}

cudaError_t launch_chol_aug(const double* G, int ldg, int l, int npad, double* R, double* Rinv, int* flag,
                            int flag_bit, cudaStream_t st, Pred pr) {
  if (l < 1 || l > 128 || npad > 128 || npad < l) return cudaErrorInvalidValue;
  const int nblk = (npad + 15) / 16;
  const size_t smem = ((size_t)16 * nblk * (16 * nblk + 4) + (size_t)nblk * 16 * CB_LDB) * sizeof(double);
  cudaError_t e = cudaSuccess;
#define RSVD_CB(NBK)                                                                                      \
  {                                                                                                      \
    e = smem_optin(chol_blk_kernel<NBK>); if (e != cudaSuccess) return e;                                                                                                     \
    e = launch_pdl(chol_blk_kernel<NBK>, dim3(1), dim3(256), smem, st, G, ldg, l, npad, R, Rinv, flag, flag_bit, pr); \
    if (e != cudaSuccess) return e;                                                                      \
  }
  switch (nblk) {
    case 1: RSVD_CB(1) break;
    case 2: RSVD_CB(2) break;
    case 3: RSVD_CB(3) break;
    case 4: RSVD_CB(4) break;
    case 5: RSVD_CB(5) break;
    case 6: RSVD_CB(6) break;
    case 7: RSVD_CB(7) break;
    default: RSVD_CB(8) break;
  }
#undef RSVD_CB
  ++g_kernel_launches;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ C = S T (small K)
// Persistent CTAs over 64-row blocks; warps 2 (M, 32 rows) x 4 (N, Ng/4
// columns).  T (Np x Np, ld ldt) is staged in shared memory once per CTA; the
// next row block of S is prefetched (cp.async) while the current one is
// multiplied.  A row block is fully read into shared memory before its output
// rows are written, so C may alias S.  upper: T is upper triangular (R^-1), the
// k loop of a warp stops at its last column.
constexpr int AP_BM = 64;

template <int TJ, int NBUF>
__global__ void __launch_bounds__(CQ_THREADS)
panel_apply_kernel(const double* S, int64_t lds, int64_t rows, int Np, const double* __restrict__ T, int64_t ldt,
                   double* C, int64_t ldc, int Nout, int upper, Pred pr) {
  pdl_wait();
  pdl_trigger();
  if (pred_skip(pr)) return;
  constexpr int NG = 32 * TJ;
  constexpr int LDX = NG + ((4 - NG) & 15);
  extern __shared__ __align__(16) double sm[];
  const int LDSS = Np + ((4 - Np) & 15);
  double* Ts = sm;                        // Np x LDX
  double* Ss = sm + Np * LDX;             // NBUF x AP_BM x LDSS
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
  const int gq = lane >> 2, tq = lane & 3;
  const int cpr = Np / 2;
  const int64_t nblk = ceil_div(rows, AP_BM);
  int kmax = Np;
  if (upper) kmax = min(Np, (wn + 1) * (NG / 4));
  for (int ch = tid; ch < Np * cpr; ch += CQ_THREADS) {
    const int r = ch / cpr, c = (ch - r * cpr) * 2;
    cp_async16(Ts + r * LDX + c, T + r * ldt + c, 16);
  }
  for (int e = tid; e < Np * (NG - Np); e += CQ_THREADS) {
    const int r = e / (NG - Np), c = Np + e % (NG - Np);
    Ts[r * LDX + c] = 0.0;
  }
  auto load = [&](int buf, int64_t rb) {
    double* ss = Ss + buf * AP_BM * LDSS;
    const int64_t m0 = rb * AP_BM;
    for (int ch = tid; ch < AP_BM * cpr; ch += CQ_THREADS) {
      const int r = ch / cpr, c = (ch - r * cpr) * 2;
      const bool ok = m0 + r < rows;
      cp_async16(ss + r * LDSS + c, ok ? S + (m0 + r) * lds + c : S, ok ? 16 : 0);
    }
  };
  int64_t rb = blockIdx.x;
  if (rb < nblk) load(0, rb);
  cp_async_commit();
  for (int it = 0; rb < nblk; ++it, rb += gridDim.x) {
    const int buf = NBUF == 2 ? (it & 1) : 0;
    if (NBUF == 2 && rb + gridDim.x < nblk) load(buf ^ 1, rb + gridDim.x);
    cp_async_commit();
    if (NBUF == 2) cp_async_wait<1>();
    else cp_async_wait<0>();
    __syncthreads();
    const double* ss = Ss + buf * AP_BM * LDSS;
    double acc[4][TJ][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < TJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int kk = 0; kk < kmax; kk += 4) {
      double af[4], bf[TJ];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = ss[(wm * 32 + i * 8 + gq) * LDSS + kk + tq];
#pragma unroll
      for (int j = 0; j < TJ; ++j) bf[j] = Ts[(kk + tq) * LDX + wn * (NG / 4) + j * 8 + gq];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < TJ; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    const int64_t m0 = rb * AP_BM;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t r = m0 + wm * 32 + i * 8 + gq;
      if (r >= rows) continue;
#pragma unroll
      for (int j = 0; j < TJ; ++j) {
        const int c = wn * (NG / 4) + j * 8 + 2 * tq;
        if (c < Nout) C[r * ldc + c] = acc[i][j][0];
        if (c + 1 < Nout) C[r * ldc + c + 1] = acc[i][j][1];
      }
    }
    __syncthreads();                      // buffer `buf` is refilled in iteration it + NBUF
    if (NBUF == 1 && rb + gridDim.x < nblk) load(0, rb + gridDim.x);
  }
  cp_async_wait<0>();
}

// Np in (96, 128] (configs 3 and 4): 32-row blocks, double-buffered (T takes 135
// KB of shared memory, so 64-row blocks fit only once: the load of the next block
// was exposed), and warps over column PAIRS of 8-column tiles (w, 15 - w): with
// an upper-triangular T (R^-1) tile j needs k < 8 j + 8, so every warp does the
// same 17 x 8 k-steps instead of 32 .. 128 (the slowest warp set the pace).
constexpr int AP2_BM = 32;
__global__ void __launch_bounds__(CQ_THREADS, 1)
panel_apply128_kernel(const double* S, int64_t lds, int64_t rows, int Np, const double* __restrict__ T,
                      int64_t ldt, double* C, int64_t ldc, int Nout, int upper, Pred pr) {
  pdl_wait();
  pdl_trigger();
  if (pred_skip(pr)) return;
  constexpr int NG = 128, LDX = NG + ((4 - NG) & 15);
  extern __shared__ __align__(16) double sm[];
  const int LDSS = Np + ((4 - Np) & 15);
  double* Ts = sm;                        // Np x LDX
  double* Ss = sm + Np * LDX;             // 2 x AP2_BM x LDSS
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int cpr = Np / 2;
  const int64_t nblk = ceil_div(rows, AP2_BM);
  const int jt[2] = {warp, 15 - warp};                 // the warp's two 8-column tiles
  const int kend0 = upper ? min(Np, 8 * jt[0] + 8) : Np;
  const int kend1 = upper ? min(Np, 8 * jt[1] + 8) : Np;   // >= kend0
  for (int ch = tid; ch < Np * cpr; ch += CQ_THREADS) {
    const int r = ch / cpr, c = (ch - r * cpr) * 2;
    cp_async16(Ts + r * LDX + c, T + r * ldt + c, 16);
  }
  for (int e = tid; e < Np * (NG - Np); e += CQ_THREADS) {
    const int r = e / (NG - Np), c = Np + e % (NG - Np);
    Ts[r * LDX + c] = 0.0;
  }
  auto load = [&](int buf, int64_t rb) {
    double* ss = Ss + buf * AP2_BM * LDSS;
    const int64_t m0 = rb * AP2_BM;
    for (int ch = tid; ch < AP2_BM * cpr; ch += CQ_THREADS) {
      const int r = ch / cpr, c = (ch - r * cpr) * 2;
      const bool ok = m0 + r < rows;
      cp_async16(ss + r * LDSS + c, ok ? S + (m0 + r) * lds + c : S, ok ? 16 : 0);
    }
  };
  int64_t rb = blockIdx.x;
  if (rb < nblk) load(0, rb);
  cp_async_commit();
  for (int it = 0; rb < nblk; ++it, rb += gridDim.x) {
    const int buf = it & 1;
    if (rb + gridDim.x < nblk) load(buf ^ 1, rb + gridDim.x);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double* ss = Ss + buf * AP2_BM * LDSS;
    double acc[4][2][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    int kk = 0;
    for (; kk < kend0; kk += 4) {
      double af[4], bf[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = ss[(i * 8 + gq) * LDSS + kk + tq];
#pragma unroll
      for (int j = 0; j < 2; ++j) bf[j] = Ts[(kk + tq) * LDX + jt[j] * 8 + gq];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    for (; kk < kend1; kk += 4) {
      double af[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = ss[(i * 8 + gq) * LDSS + kk + tq];
      const double bf = Ts[(kk + tq) * LDX + jt[1] * 8 + gq];
#pragma unroll
      for (int i = 0; i < 4; ++i) dmma884(acc[i][1][0], acc[i][1][1], af[i], bf);
    }
    const int64_t m0 = rb * AP2_BM;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t r = m0 + i * 8 + gq;
      if (r >= rows) continue;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int c = jt[j] * 8 + 2 * tq;
        if (c < Nout) C[r * ldc + c] = acc[i][j][0];
        if (c + 1 < Nout) C[r * ldc + c + 1] = acc[i][j][1];
      }
    }
    __syncthreads();                      // buffer `buf` is refilled in iteration it + 2
  }
  cp_async_wait<0>();
}

cudaError_t launch_panel_apply(const double* S, int64_t lds, int64_t rows, int Np, const double* T, int64_t ldt,
                               double* C, int64_t ldc, int Nout, bool upper, int num_sms, cudaStream_t st, Pred pr) {
  if (Np % 4 || Np > 128 || (lds & 1) || (ldt & 1) || rows < 1) return cudaErrorInvalidValue;
  const int ng = cq_ng(Np);
  const int ldx = ldpad(ng), ldss = Np + ((4 - Np) & 15);
  const int nbuf = ng == 128 ? 1 : 2;     // Np <= 96: double-buffered S blocks
  const size_t smem = ((size_t)Np * ldx + nbuf * (size_t)AP_BM * ldss) * sizeof(double);
  const size_t smem_max = ((size_t)ng * ldpad(ng) + nbuf * (size_t)AP_BM * ldpad(ng)) * sizeof(double);
  const int64_t nblk = ceil_div(rows, AP_BM);
  int per_sm = (int)(220 * 1024 / smem);
  if (per_sm < 1) per_sm = 1;
  if (per_sm > 4) per_sm = 4;
  int64_t grid = (int64_t)num_sms * per_sm;
  if (grid > nblk) grid = nblk;
  cudaError_t e = cudaSuccess;
#define RSVD_APPLY(TJ)                                                                                    \
  {                                                                                                      \
    e = smem_optin(panel_apply_kernel<TJ, (TJ == 4 ? 1 : 2)>); if (e != cudaSuccess) return e;                                                                                                     \
    e = launch_pdl(panel_apply_kernel<TJ, (TJ == 4 ? 1 : 2)>, dim3((unsigned)grid), dim3(CQ_THREADS), smem, st, S, lds, rows, Np, T, ldt, C, ldc, Nout, upper ? 1 : 0, pr); \
    if (e != cudaSuccess) return e; \
  }
  static const bool bal = [] { const char* v = getenv("RSVD_APPLY128"); return !v || atoi(v) != 0; }();
  if (ng == 128 && bal) {
    const size_t sm2 = ((size_t)Np * ldx + 2 * (size_t)AP2_BM * ldss) * sizeof(double);
    int64_t g2 = ceil_div(rows, AP2_BM);
    if (g2 > num_sms) g2 = num_sms;
    e = smem_optin(panel_apply128_kernel);
    if (e != cudaSuccess) return e;
    e = launch_pdl(panel_apply128_kernel, dim3((unsigned)g2), dim3(CQ_THREADS), sm2, st, S, lds, rows, Np, T, ldt, C, ldc,
                   Nout, upper ? 1 : 0, pr);
    if (e != cudaSuccess) return e;
    ++g_kernel_launches;
    return cudaGetLastError();
  }
  switch (ng / 32) {
    case 1: RSVD_APPLY(1) break;
    case 2: RSVD_APPLY(2) break;
    case 3: RSVD_APPLY(3) break;
    default: RSVD_APPLY(4) break;
  }
#undef RSVD_APPLY
  ++g_kernel_launches;
  return cudaGetLastError();
}

}  // namespace rsvd
