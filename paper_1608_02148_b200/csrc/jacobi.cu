// jacobi.cu -- economic SVD of the l x l factor (Alg. 5 step 2):
// one-sided (Hestenes) Jacobi on X = R_B^T, X J = W Sigma (reading R7/R8 of
// rotate iff |gamma| > tau sqrt(alpha beta), tau = l 2^-52, stop
// after a sweep without rotation, cap 30 sweeps).
//
// B200 design.  The columns are padded to L = 2^ceil(log2 l) (zero columns
// never rotate).  A sweep is L - 1 parallel steps of L/2 disjoint pairs in a
// recursive "stationary / travelling" order: at level d the columns form
// blocks of B = L / 2^d; in step s the k-th column of a block's first half
// (stationary, kept in registers for the whole level) meets column (k + s) mod
// B/2 of its second half (travelling, read from and written back to shared
// memory).  Every pair meets exactly once per sweep (at the level of their
// highest differing index bit), and only half of X crosses shared memory per
// step.  Four lanes own a pair.
//
// J is not accumulated by the sweeping CTA: each step's rotations (c, s) go to
// a log in global memory, and the other CTAs of the same launch replay the log
// on the rows of J (rows are independent: the rotations act on columns) while
// the sweeps run -- the log is published in chunks of JA_CH steps with
// release/acquire counters tagged by a per-launch epoch -- so the replay adds
// only its last chunk to the critical path.
#include <math.h>

#include <algorithm>
#include <cstdlib>

#include <atomic>

#include "common.cuh"
#include "kernels.h"

#ifndef JB_PROBE
#define JB_PROBE(slot)                              // probe builds: per-phase cycles of a block round (tools/bench_jacobi)
#endif
#ifndef JAC_PROBE
#define JAC_PROBE_DECL
#define JAC_PROBE(slot)
#define JAC_PROBE_OUT
#endif

namespace rsvd {

namespace {

__host__ __device__ inline int jac_L(int l) {
  int L = 2;
  while (L < l) L <<= 1;
  return L;
}

// (stationary p, travelling q) of pair k at a level with half-block h = 2^lh, step s
__device__ __forceinline__ void jac_pair(int lh, int s, int k, int& p, int& q) {
  const int h = 1 << lh;
  const int kk = k & (h - 1), base = (k >> lh) << (lh + 1);
  p = base + kk;
  q = base + h + ((kk + s) & (h - 1));
}

// Rotation (c, s) annihilating gamma for column norms alpha, beta:
// t = 2 ga sgn(be - al) / (|be - al| + sqrt((be - al)^2 + 4 ga^2)) (the oracle's zeta
// formula rewritten).  The angle only steers convergence (orthogonality of the
// rotation comes from c^2 + s^2 = 1), so t is formed from the hardware FP64
// reciprocal / rsqrt approximations (one Newton step each, ~2^-40) on operands
// scaled by a power of two to O(1), and c = (1 + t^2)^-1/2 is refined to FP64
// by Newton.  No FP32 round trips (each F2F conversion sits on the per-step
// critical path).
__device__ __forceinline__ double rcp_nr1(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y * fma(-x, y, 2.0);
}
__device__ __forceinline__ double rsqrt_approx(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}
__device__ __forceinline__ void jac_rot(double al, double be, double ga, double& c, double& sn) {
  const double dlt = be - al, g2 = 2.0 * ga;
  const double mx = fmax(fabs(dlt), fabs(g2));
  const long long ex = (__double_as_longlong(mx) >> 52) & 0x7ff;          // biased exponent
  const double scale = __longlong_as_double((2046 - ex) << 52);           // ~ 1 / mx (power of two)
  const double df = dlt * scale, gf = g2 * scale;                          // exact
  const double h = fma(df, df, gf * gf);
  double r = rsqrt_approx(h);
  r = r * fma(-0.5 * h * r, r, 1.5);
  const double t = (df >= 0.0 ? gf : -gf) * rcp_nr1(fabs(df) + h * r);
  const double x = fma(t, t, 1.0);
  double c0 = rsqrt_approx(x);
  c0 = c0 * fma(-0.5 * x * c0, c0, 1.5);
  c0 = c0 * fma(-0.5 * x * c0, c0, 1.5);
  c = c0;
  sn = c0 * t;
}
}  // namespace

// Scale X (count doubles in shared memory) by 2^-E, E the exponent of max |x|
// (exact: a power of two), so that the squared norms and products of the
// rotation test stay inside the FP64 range whatever the scale of A (reading
// R35); every rotation is unchanged (the test and the angle are homogeneous).
// Returns 2^E, the factor of the singular values (1 for a zero / non-finite X).
// All threads of the block call it; red: >= 32 doubles of shared scratch.
__device__ double jac_prescale(double* Xs, int count, double* red, int bad) {
  double mx = 0.0;
  for (int e = threadIdx.x; e < count; e += blockDim.x) mx = fmax(mx, fabs(Xs[e]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  mx = 0.0;
  for (int w = 0; w < nw; ++w) mx = fmax(mx, red[w]);
  __syncthreads();
  if (bad || !(mx > 0.0) || !isfinite(mx)) return 1.0;
  int ex;
  frexp(mx, &ex);
  const double sc = ldexp(1.0, -ex);
  for (int e = threadIdx.x; e < count; e += blockDim.x) Xs[e] *= sc;
  __syncthreads();
  return ldexp(1.0, ex);
}

size_t jacobi_log_bytes(int l) {
  const int L = jac_L(l);
  return (size_t)31 * (L - 1) * (L / 2) * 2 * sizeof(double);
}

constexpr int JA_CH = 16;   // rotation-log chunk (steps) published / replayed at once

__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Replay of the rotation log on rows [row0, row0 + nw) of J (one warp per row,
// identity start): chunk c of JA_CH steps is read once prog (epoch-tagged step
// count) covers it; after `done` (epoch-tagged final step count) the rest.
// Jo(i, rank[p]) = J(i, p).
__device__ void jacobi_replay(const double2* __restrict__ rlog, const int* __restrict__ rank, int l,
                              double* __restrict__ Jo, int ldo, int row0, const unsigned long long* prog,
                              const unsigned long long* done, unsigned epoch, unsigned char* sm) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5, nt = blockDim.x;
  const int i = row0 + warp;
  const int L = jac_L(l), npairs = L / 2;
  double2* buf = reinterpret_cast<double2*>(sm);                       // [JA_CH * 64]
  double* row = reinterpret_cast<double*>(sm + JA_CH * 64 * sizeof(double2)) + warp * 129;
  for (int p = lane; p < L; p += 32) row[p] = (p == i) ? 1.0 : 0.0;
  int levels = 0;
  while ((1 << levels) < L) ++levels;
  __shared__ long long s_avail;
  __shared__ int s_fin;
  int lh = levels - 1, s = 0;
  for (int64_t ch = 0;; ++ch) {
    if (threadIdx.x == 0) {
      long long avail = -1;
      int fin = 0;
      for (;;) {
        const unsigned long long d = ld_acquire_u64(done);
        if ((unsigned)(d >> 32) == epoch) { avail = (long long)(d & 0xffffffffu); fin = 1; break; }
        const unsigned long long pg = ld_acquire_u64(prog);
        if ((unsigned)(pg >> 32) == epoch && (long long)(pg & 0xffffffffu) >= (ch + 1) * JA_CH) {
          avail = (long long)(pg & 0xffffffffu);
          break;
        }
        __nanosleep(256);
      }
      s_avail = avail;
      s_fin = fin;
    }
    __syncthreads();
    const long long avail = s_avail;
    const int fin = s_fin;
    const int64_t s0 = ch * JA_CH;
    if (s0 >= avail) {
      if (fin) break;
      continue;                                        // (not reached: prog covered the chunk)
    }
    const int nst = (int)min((int64_t)JA_CH, (int64_t)avail - s0);
    for (int e = threadIdx.x; e < nst * npairs; e += nt) buf[e] = __ldcg(rlog + s0 * npairs + e);
    __syncthreads();
    for (int st = 0; st < nst; ++st) {
      for (int k = lane; k < npairs; k += 32) {
        int p, q;
        jac_pair(lh, s, k, p, q);
        const double2 cs = buf[st * npairs + k];
        const double u = row[p], v = row[q];
        row[p] = cs.x * u - cs.y * v;
        row[q] = cs.y * u + cs.x * v;
      }
      __syncwarp();
      if (++s == (1 << lh)) {
        s = 0;
        if (--lh < 0) lh = levels - 1;
      }
    }
    __syncthreads();                                   // buf reused by the next chunk
  }
  if (i < l) {
    for (int p = lane; p < l; p += 32) Jo[i * ldo + __ldcg(rank + p)] = row[p];
    for (int c = l + lane; c < ldo; c += 32) Jo[i * ldo + c] = 0.0;      // padded columns
  } else if (i < ldo) {
    for (int c = lane; c < ldo; c += 32) Jo[i * ldo + c] = 0.0;          // padded rows
  }
}

// JG lanes own a column pair; EPL = elements of a column per lane (l <= JG * EPL)
template <int JG, int EPL>
__global__ void __launch_bounds__(512, 1)
jacobi_x_kernel(const double* __restrict__ R, int ldr, int l, double* __restrict__ sigma, double* __restrict__ Wo,
                int ldo, double2* __restrict__ rlog, int* __restrict__ rank_out, int* flag, int* sweeps_out,
                double* __restrict__ Jo, unsigned long long* prog, unsigned long long* done, unsigned epoch) {
  pdl_wait();
  pdl_trigger();
  if (blockIdx.x > 0) {                                  // J-replay CTAs
    extern __shared__ __align__(16) unsigned char jsm[];
    jacobi_replay(rlog, rank_out, l, Jo, ldo, (blockIdx.x - 1) * (int)(blockDim.x >> 5), prog, done, epoch, jsm);
    return;
  }
  extern __shared__ __align__(16) double Xs[];           // L columns x LDX (column p: Xs + p * LDX)
  const int L = jac_L(l);
  constexpr int LDX = JG * EPL + 4;                      // consecutive columns 4 doubles apart mod 32 banks
  __shared__ int rotated, bad;
  __shared__ double sg[128];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int npairs = L / 2;
  const bool act = tid / JG < npairs;                    // lanes beyond the last pair mirror it
  const int k = act ? tid / JG : npairs - 1, gs = tid % JG;   // pair slot, lane within the pair
  if (tid == 0) { rotated = 0; bad = 0; }
  __syncthreads();
  // X = R^T: column p of X = row p of R (upper: entries i >= p); rows/columns >= l are zero
  // (eight independent loads in flight per thread before the shared stores)
  for (int e0 = tid; e0 < L * LDX; e0 += 8 * nt) {
    double v[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int e = e0 + r * nt, p = e / LDX, i = e - p * LDX;
      v[r] = (e < L * LDX && p < l && i < l && i >= p) ? R[p * ldr + i] : 0.0;
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int e = e0 + r * nt;
      if (e < L * LDX) {
        if (!isfinite(v[r])) bad = 1;
        Xs[e] = v[r];
      }
    }
  }
  __syncthreads();
  const double jscale = jac_prescale(Xs, L * LDX, sg, bad);
  const double tol = (double)l * 0x1.0p-52, tol2 = tol * tol;
  int levels = 0;
  while ((1 << levels) < L) ++levels;
  int sweeps = 0;
  bool converged = bad != 0;
  int64_t gstep = 0;                                     // global step index into the log
  JAC_PROBE_DECL
  for (int sweep = 0; sweep <= 30 && !converged; ++sweep) {
    for (int d = 0; d < levels; ++d) {
      const int lh = levels - 1 - d, h = 1 << lh;
      int p = 0, q = 0;
      double xs[EPL], xt[EPL];
      {
        jac_pair(lh, 0, k, p, q);
#pragma unroll
        for (int e = 0; e < EPL; ++e) xs[e] = Xs[p * LDX + gs + JG * e];
      }
      for (int s = 0; s < h; ++s, ++gstep) {
        double c = 1.0, sn = 0.0;
        {
          jac_pair(lh, s, k, p, q);
          JAC_PROBE(0)
#pragma unroll
          for (int e = 0; e < EPL; ++e) xt[e] = Xs[q * LDX + gs + JG * e];
          constexpr int NCH = EPL >= 4 ? 4 : EPL;        // independent accumulation chains
          double a[NCH], b[NCH], g[NCH];
#pragma unroll
          for (int w = 0; w < NCH; ++w) a[w] = b[w] = g[w] = 0.0;
#pragma unroll
          for (int e = 0; e < EPL; ++e) {
            a[e % NCH] = fma(xs[e], xs[e], a[e % NCH]);
            b[e % NCH] = fma(xt[e], xt[e], b[e % NCH]);
            g[e % NCH] = fma(xs[e], xt[e], g[e % NCH]);
          }
#pragma unroll
          for (int w = 1; w < NCH; ++w) { a[0] += a[w]; b[0] += b[w]; g[0] += g[w]; }
          double al = a[0], be = b[0], ga = g[0];
#pragma unroll
          for (int o = JG / 2; o > 0; o >>= 1) {
            al += __shfl_xor_sync(0xffffffffu, al, o);
            be += __shfl_xor_sync(0xffffffffu, be, o);
            ga += __shfl_xor_sync(0xffffffffu, ga, o);
          }
          JAC_PROBE(1)
          if (ga * ga > tol2 * (al * be)) {
            jac_rot(al, be, ga, c, sn);
            JAC_PROBE(2)
#pragma unroll
            for (int e = 0; e < EPL; ++e) {
              const double u = xs[e], v = xt[e];
              xs[e] = c * u - sn * v;
              xt[e] = sn * u + c * v;
            }
            if (gs == 0 && act) rotated = 1;
          }
          if (act) {
#pragma unroll
            for (int e = 0; e < EPL; ++e) Xs[q * LDX + gs + JG * e] = xt[e];
            if (gs == 0) rlog[gstep * npairs + k] = make_double2(c, sn);
          }
          JAC_PROBE(3)
        }
        __syncthreads();                                 // travelling columns published
        if (tid == 0 && ((gstep + 1) % JA_CH) == 0) {
          __threadfence();
          st_release_u64(prog, ((unsigned long long)epoch << 32) | (unsigned long long)(gstep + 1));
        }
        JAC_PROBE(4)
      }
      if (act) {
#pragma unroll
        for (int e = 0; e < EPL; ++e) Xs[p * LDX + gs + JG * e] = xs[e];
      }
      __syncthreads();
    }
    const bool any = rotated != 0;
    __syncthreads();
    if (tid == 0) rotated = 0;
    if (!any) converged = true;
    else ++sweeps;
    __syncthreads();
  }
  JAC_PROBE_OUT
  // sigma_p = ||x_p||, stable descending ranks, W(:, rank) = x_p / sigma_p
  const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  for (int p = warp; p < l; p += nw) {
    double s = 0.0;
    for (int i = lane; i < l; i += 32) s = fma(Xs[p * LDX + i], Xs[p * LDX + i], s);
    s = warp_sum(s);
    if (lane == 0) sg[p] = sqrt(s);
  }
  __syncthreads();
  for (int p = warp; p < l; p += nw) {
    int rk = 0;
    const double sp = sg[p];
    for (int q = lane; q < l; q += 32) rk += (sg[q] > sp) || (sg[q] == sp && q < p);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rk += __shfl_xor_sync(0xffffffffu, rk, o);
    if (lane == 0) { sigma[rk] = sp * jscale; rank_out[p] = rk; }
    const double inv = sp > 0.0 ? 1.0 / sp : 1.0;
    for (int i = lane; i < l; i += 32) Wo[i * ldo + rk] = Xs[p * LDX + i] * inv;
  }
  // padding of the ldo x ldo W outside its leading l x l block: exact zeros
  for (int e = tid; e < ldo * ldo; e += nt) {
    const int i = e / ldo, c = e - (e / ldo) * ldo;
    if (i >= l || c >= l) Wo[e] = 0.0;
  }
  __syncthreads();                                     // rank_out complete
  if (tid == 0) {
    if (!converged) atomicOr(flag, 2);
    if (bad) atomicOr(flag, 4);
    if (sweeps_out) *sweeps_out = sweeps;
    rank_out[128] = sweeps;
    __threadfence();
    st_release_u64(done, ((unsigned long long)epoch << 32) | (unsigned long long)gstep);   // every logged step
  }
}

// ------------------------------------------------------------------ block ordering
// The same one-sided Jacobi (rotation formula, threshold, stopping rule, sweep
// cap) in a block-cyclic order built for one SM's register file.  Columns form
// NB blocks of B (B = 8 for l > 64, else 4; NB even, padding columns are zero
// and never rotate).  A sweep is NB block steps: step 0 pairs blocks (2w,
// 2w+1) and rotates the pairs inside each block (B - 1 round-robin rounds, the
// B-th round logs identities); step s >= 1 pairs the blocks by a closed-form
// round-robin tournament (block 0 fixed) and rotates the B^2 cross pairs in B
// rounds of B disjoint pairs.  Warp w holds its two blocks (2B columns, rows
// lane + 32e) in registers for the whole step: a round's B dot-product triples
// are reduce-scattered by shuffles so that lanes 4j.. (B = 8) own pair j's
// (alpha, beta, gamma), compute its rotation, and broadcast (c, s) to the warp.
// Shared memory is touched once per block step (load / store of the blocks)
// and the CTA synchronises once per block step (NB per sweep, not L - 1).
// Every pair of columns meets once per sweep, as in the cyclic order.
namespace {
int blk_B(int l) {
  static const int force = getenv("RSVD_JACOBI_B") ? atoi(getenv("RSVD_JACOBI_B")) : 0;   // A/B probes
  if (force == 8 || (force == 4 && l <= 64)) return force;
  return l > 64 ? 8 : 4;
}
__host__ __device__ inline int blk_NB(int l, int B) {
  int nb = (l + B - 1) / B;
  if (nb < 2) nb = 2;
  return nb + (nb & 1);
}
// blocks (I, J) of warp w at block step s of a sweep
__host__ __device__ inline void blk_blocks(int NB, int s, int w, int& I, int& J) {
  if (s == 0) { I = 2 * w; J = 2 * w + 1; return; }
  const int m = NB - 1, r = s - 1;
  if (w == 0) { I = 0; J = r + 1; }
  else { I = (r + w) % m + 1; J = (r - w + m) % m + 1; }
}
// local columns (0..2B-1) of pair j in round rho: cross steps (j, B + (j + rho) % B);
// the intra step pairs within each block by round robin (block 0 fixed), its
// last round repeats round 0 (identity rotations)
__host__ __device__ constexpr int blk_lp(int B, bool intra, int rho, int j) {
  return !intra ? j
                : ((j < B / 2 ? 0 : B) + ((j % (B / 2)) == 0 ? 0 : ((rho % (B - 1)) + (j % (B / 2))) % (B - 1) + 1));
}
__host__ __device__ constexpr int blk_lq(int B, bool intra, int rho, int j) {
  return !intra ? B + (j + rho) % B
                : ((j < B / 2 ? 0 : B) +
                   ((j % (B / 2)) == 0 ? (rho % (B - 1)) + 1
                                       : ((rho % (B - 1)) - (j % (B / 2)) + (B - 1)) % (B - 1) + 1));
}
}  // namespace

size_t jacobi_blk_log_bytes(int l) {   // either block size
  size_t mx = 0;
  for (int B : {4, 8}) {
    const int NB = blk_NB(l, B);
    mx = std::max(mx, (size_t)31 * NB * B * (NB / 2) * B * sizeof(double2));
  }
  return mx;
}

constexpr int JB_CHS = 2;   // block steps per published / replayed chunk

// J replay for the block order: one warp per row of J, the log applied chunk by chunk
template <int B>
__device__ void jacobi_blk_replay(const double2* __restrict__ rlog, const int* __restrict__ rank, int l, int NB,
                                  double* __restrict__ Jo, int ldo, int row0, const unsigned long long* prog,
                                  const unsigned long long* done, unsigned epoch, unsigned char* sm) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nt = blockDim.x;
  const int i = row0 + warp;
  const int W = NB / 2, NC = NB * B, per_step = B * W * B;
  double2* buf = reinterpret_cast<double2*>(sm);                         // [JB_CHS * per_step]
  double* row = reinterpret_cast<double*>(sm + (size_t)JB_CHS * per_step * sizeof(double2)) + warp * (NC + 1);
  for (int p = lane; p < NC; p += 32) row[p] = (p == i) ? 1.0 : 0.0;
  __shared__ long long s_avail;
  __shared__ int s_fin;
  for (int64_t ch = 0;; ++ch) {
    if (threadIdx.x == 0) {
      long long avail = -1;
      int fin = 0;
      for (;;) {
        const unsigned long long d = ld_acquire_u64(done);
        if ((unsigned)(d >> 32) == epoch) { avail = (long long)(d & 0xffffffffu); fin = 1; break; }
        const unsigned long long pg = ld_acquire_u64(prog);
        if ((unsigned)(pg >> 32) == epoch && (long long)(pg & 0xffffffffu) >= (ch + 1) * JB_CHS) {
          avail = (long long)(pg & 0xffffffffu);
          break;
        }
        __nanosleep(256);
      }
      s_avail = avail;
      s_fin = fin;
    }
    __syncthreads();
    const long long avail = s_avail;
    const int fin = s_fin;
    const int64_t g0 = ch * JB_CHS;
    if (g0 >= avail) {
      if (fin) break;
      continue;
    }
    const int nst = (int)min((int64_t)JB_CHS, (int64_t)avail - g0);
    for (int e = threadIdx.x; e < nst * per_step; e += nt) buf[e] = __ldcg(rlog + g0 * per_step + e);
    __syncthreads();
    for (int st = 0; st < nst; ++st) {
      const int s = (int)((g0 + st) % NB);
      for (int rho = 0; rho < B; ++rho) {
        for (int k = lane; k < W * B; k += 32) {
          const int w = k / B, j = k - w * B;
          int I, J;
          blk_blocks(NB, s, w, I, J);
          const int lp = blk_lp(B, s == 0, rho, j), lq = blk_lq(B, s == 0, rho, j);
          const int p = lp < B ? I * B + lp : J * B + lp - B;
          const int q = lq < B ? I * B + lq : J * B + lq - B;
          const double2 cs = buf[(st * B + rho) * W * B + k];
          const double u = row[p], v = row[q];
          row[p] = cs.x * u - cs.y * v;
          row[q] = cs.y * u + cs.x * v;
        }
        __syncwarp();
      }
    }
    __syncthreads();                                   // buf reused by the next chunk
  }
  if (i < l) {
    for (int p = lane; p < l; p += 32) Jo[i * ldo + __ldcg(rank + p)] = row[p];
    for (int c = l + lane; c < ldo; c += 32) Jo[i * ldo + c] = 0.0;
  } else if (i < ldo) {
    for (int c = lane; c < ldo; c += 32) Jo[i * ldo + c] = 0.0;
  }
}

// one round of B disjoint pairs on the warp's registers x[2B][RPL]: the B
// dot-product triples are reduce-scattered by shuffles so that lane group j
// (lanes j G .. j G + G - 1, G = 32 / B) holds pair j's (alpha, beta, gamma),
// computes its rotation and broadcasts (c, s) to the warp.  (A shared-memory
// reduction / broadcast was measured slower: tools/bench_jacobi.)
template <int B, int RPL, bool INTRA, int RHO>
__device__ __forceinline__ void blk_round(double (&x)[2 * B][RPL], int lane, double tol2, bool& rot,
                                          double2* __restrict__ logp) {
  constexpr int LB = B == 8 ? 3 : 2;
  JB_PROBE(0)
  double v[3][B];
#pragma unroll
  for (int j = 0; j < B; ++j) {
    const int p = blk_lp(B, INTRA, RHO, j), q = blk_lq(B, INTRA, RHO, j);
    double a = 0.0, b = 0.0, g = 0.0;
#pragma unroll
    for (int e = 0; e < RPL; ++e) {
      a = fma(x[p][e], x[p][e], a);
      b = fma(x[q][e], x[q][e], b);
      g = fma(x[p][e], x[q][e], g);
    }
    v[0][j] = a; v[1][j] = b; v[2][j] = g;
  }
  JB_PROBE(1)
  // reduce-scatter over lane bits 4 .. 5 - LB: lane keeps the pair j = lane >> (5 - LB)
#pragma unroll
  for (int k = 0; k < LB; ++k) {
    const int h = (B >> k) / 2;
    const bool up = (lane >> (4 - k)) & 1;
#pragma unroll
    for (int qv = 0; qv < 3; ++qv)
#pragma unroll
      for (int i2 = 0; i2 < h; ++i2) {
        const double send = up ? v[qv][i2] : v[qv][i2 + h];
        const double keep = up ? v[qv][i2 + h] : v[qv][i2];
        v[qv][i2] = keep + __shfl_xor_sync(0xffffffffu, send, 16 >> k);
      }
  }
#pragma unroll
  for (int o = 16 >> LB; o > 0; o >>= 1) {
    v[0][0] += __shfl_xor_sync(0xffffffffu, v[0][0], o);
    v[1][0] += __shfl_xor_sync(0xffffffffu, v[1][0], o);
    v[2][0] += __shfl_xor_sync(0xffffffffu, v[2][0], o);
  }
  JB_PROBE(2)
  double c = 1.0, sn = 0.0;
  const double al = v[0][0], be = v[1][0], ga = v[2][0];
  const bool doit = !(INTRA && RHO == B - 1) && ga * ga > tol2 * (al * be);
  if (doit) jac_rot(al, be, ga, c, sn);
  JB_PROBE(3)
  rot |= __any_sync(0xffffffffu, doit);
  if ((lane & ((32 >> LB) - 1)) == 0) logp[lane >> (5 - LB)] = make_double2(c, sn);
#pragma unroll
  for (int j = 0; j < B; ++j) {
    const int p = blk_lp(B, INTRA, RHO, j), q = blk_lq(B, INTRA, RHO, j);
    const double cj = __shfl_sync(0xffffffffu, c, j << (5 - LB));
    const double sj = __shfl_sync(0xffffffffu, sn, j << (5 - LB));
#pragma unroll
    for (int e = 0; e < RPL; ++e) {
      const double u = x[p][e], w = x[q][e];
      x[p][e] = cj * u - sj * w;
      x[q][e] = sj * u + cj * w;
    }
  }
  JB_PROBE(4)
}

template <int B, int RPL, bool INTRA, int RHO>
struct BlkRounds {
  __device__ __forceinline__ static void run(double (&x)[2 * B][RPL], int lane, double tol2, bool& rot,
                                             double2* logp, int stride) {
    blk_round<B, RPL, INTRA, RHO>(x, lane, tol2, rot, logp);
    BlkRounds<B, RPL, INTRA, RHO + 1>::run(x, lane, tol2, rot, logp + stride, stride);
  }
};
template <int B, int RPL, bool INTRA>
struct BlkRounds<B, RPL, INTRA, B> {
  __device__ __forceinline__ static void run(double (&)[2 * B][RPL], int, double, bool&, double2*, int) {}
};

template <int B, int RPL>
__global__ void __launch_bounds__(256, 1)
jacobi_blk_kernel(const double* __restrict__ R, int ldr, int l, int NB, double* __restrict__ sigma,
                  double* __restrict__ Wo, int ldo, double2* __restrict__ rlog, int* __restrict__ rank_out, int* flag,
                  int* sweeps_out, double* __restrict__ Jo, unsigned long long* prog, unsigned long long* done,
                  unsigned epoch) {
  pdl_wait();
  pdl_trigger();
  if (blockIdx.x > 0) {                                  // J-replay CTAs
    extern __shared__ __align__(16) unsigned char jsm[];
    jacobi_blk_replay<B>(rlog, rank_out, l, NB, Jo, ldo, (blockIdx.x - 1) * (int)(blockDim.x >> 5), prog, done,
                         epoch, jsm);
    return;
  }
  extern __shared__ __align__(16) double Xs[];           // NC columns x LDX rows (column p: Xs + p * LDX)
  constexpr int LDX = 32 * RPL;
  const int NC = NB * B, W = NB / 2;
  __shared__ int rotated, bad;
  __shared__ double sg[128];
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) { rotated = 0; bad = 0; }
  __syncthreads();
  // X = R^T: column p of X = row p of R (entries i >= p); rows / columns >= l are zero
  for (int e0 = tid; e0 < NC * LDX; e0 += 8 * nt) {
    double v[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int e = e0 + r * nt, p = e / LDX, i = e - p * LDX;
      v[r] = (e < NC * LDX && p < l && i < l && i >= p) ? R[p * ldr + i] : 0.0;
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int e = e0 + r * nt;
      if (e < NC * LDX) {
        if (!isfinite(v[r])) bad = 1;
        Xs[e] = v[r];
      }
    }
  }
  __syncthreads();
  const double jscale = jac_prescale(Xs, NC * LDX, sg, bad);
  const double tol = (double)l * 0x1.0p-52, tol2 = tol * tol;
  const int per_step = B * W * B;
  int sweeps = 0;
  bool converged = bad != 0;
  int64_t gstep = 0;
  for (int sweep = 0; sweep <= 30 && !converged; ++sweep) {
    bool rot = false;
    for (int s = 0; s < NB; ++s, ++gstep) {
      int I, J;
      blk_blocks(NB, s, warp, I, J);
      double x[2 * B][RPL];
#pragma unroll
      for (int c = 0; c < 2 * B; ++c)
#pragma unroll
        for (int e = 0; e < RPL; ++e) x[c][e] = Xs[((c < B ? I * B + c : J * B + c - B)) * LDX + lane + 32 * e];
      double2* logp = rlog + gstep * per_step + warp * B;
      if (s == 0) BlkRounds<B, RPL, true, 0>::run(x, lane, tol2, rot, logp, W * B);
      else BlkRounds<B, RPL, false, 0>::run(x, lane, tol2, rot, logp, W * B);
#pragma unroll
      for (int c = 0; c < 2 * B; ++c)
#pragma unroll
        for (int e = 0; e < RPL; ++e) Xs[((c < B ? I * B + c : J * B + c - B)) * LDX + lane + 32 * e] = x[c][e];
      __syncthreads();                                   // blocks published for the next step
      if (tid == 0 && ((gstep + 1) % JB_CHS) == 0) {
        __threadfence();
        st_release_u64(prog, ((unsigned long long)epoch << 32) | (unsigned long long)(gstep + 1));
      }
    }
    if (rot && lane == 0) rotated = 1;
    __syncthreads();
    const bool any = rotated != 0;
    __syncthreads();
    if (tid == 0) rotated = 0;
    if (!any) converged = true;
    else ++sweeps;
  }
  // sigma_p = ||x_p||, stable descending ranks, W(:, rank) = x_p / sigma_p
  const int nw = nt >> 5;
  for (int p = warp; p < l; p += nw) {
    double s2 = 0.0;
    for (int i = lane; i < l; i += 32) s2 = fma(Xs[p * LDX + i], Xs[p * LDX + i], s2);
    s2 = warp_sum(s2);
    if (lane == 0) sg[p] = sqrt(s2);
  }
  __syncthreads();
  for (int p = warp; p < l; p += nw) {
    int rk = 0;
    const double sp = sg[p];
    for (int q = lane; q < l; q += 32) rk += (sg[q] > sp) || (sg[q] == sp && q < p);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rk += __shfl_xor_sync(0xffffffffu, rk, o);
    if (lane == 0) { sigma[rk] = sp * jscale; rank_out[p] = rk; }
    const double inv = sp > 0.0 ? 1.0 / sp : 1.0;
    for (int i = lane; i < l; i += 32) Wo[i * ldo + rk] = Xs[p * LDX + i] * inv;
  }
  for (int e = tid; e < ldo * ldo; e += nt) {
    const int i = e / ldo, c = e - (e / ldo) * ldo;
    if (i >= l || c >= l) Wo[e] = 0.0;
  }
  __syncthreads();                                     // rank_out complete
  if (tid == 0) {
    if (!converged) atomicOr(flag, 2);
    if (bad) atomicOr(flag, 4);
    if (sweeps_out) *sweeps_out = sweeps;
    rank_out[128] = sweeps;
    __threadfence();
    st_release_u64(done, ((unsigned long long)epoch << 32) | (unsigned long long)gstep);
  }
}

int g_jacobi_lanes = 0;   // lanes per column pair (4, 8, 16; 0: 4 for L <= 64, else 8; tools/bench_jacobi)

cudaError_t launch_jacobi(const double* R, int ldr, int l, double* sigma, double* W, double* J, int ldo,
                          int* flag, int* sweeps, void* scratch, cudaStream_t st) {
  if (l < 1 || l > 128 || ldo < l || ldo > 128) return cudaErrorInvalidValue;
  const int L = jac_L(l);
  double2* rlog = reinterpret_cast<double2*>(scratch);
  int* rank = reinterpret_cast<int*>(reinterpret_cast<char*>(scratch) + std::max(jacobi_log_bytes(l), jacobi_blk_log_bytes(l)));
  unsigned long long* prog = reinterpret_cast<unsigned long long*>(rank + 192);   // 8-byte aligned, after rank[0..128]
  unsigned long long* done = prog + 1;
  static std::atomic<unsigned> epoch_ctr{0};   // unique per launch (the scratch is per context; threads may share the counter)
  const unsigned epoch = ++epoch_ctr;
  // block order for l <= 32 and l > 64; the cyclic order (measured 2 % faster
  // at l = 60 on config 2) in between.  RSVD_JACOBI_CYCLIC / _BLOCK force one (A/B).
  static const bool force_cyc = getenv("RSVD_JACOBI_CYCLIC") != nullptr;
  static const bool force_blk = getenv("RSVD_JACOBI_BLOCK") != nullptr;
  const bool use_blk = force_blk || (!force_cyc && (l <= 32 || l > 64));
  if (use_blk && g_jacobi_lanes == 0) {
    const int B = blk_B(l), NB = blk_NB(l, B), nwp = NB / 2, NC = NB * B;
    const int rpl = (l + 31) / 32;
    const int threads = nwp * 32;
    const size_t smem = std::max((size_t)NC * 32 * (rpl <= 1 ? 1 : rpl <= 2 ? 2 : 4) * sizeof(double),
                                 (size_t)JB_CHS * B * nwp * B * sizeof(double2) + (size_t)nwp * (NC + 1) * sizeof(double));
    const dim3 grid(1 + (unsigned)ceil_div(ldo, nwp));
    cudaError_t e = cudaSuccess;
#define RSVD_JB(BB, RP)                                                                                     \
  {                                                                                                         \
    e = smem_optin(jacobi_blk_kernel<BB, RP>);                                                              \
    if (e != cudaSuccess) return e;                                                                         \
    e = launch_pdl(jacobi_blk_kernel<BB, RP>, grid, dim3(threads), smem, st, R, ldr, l, NB, sigma, W, ldo, \
                   rlog, rank, flag, sweeps, J, prog, done, epoch);                                         \
  }
    if (B == 8) {
      if (rpl <= 2) RSVD_JB(8, 2) else RSVD_JB(8, 4)
    } else {
      if (rpl <= 1) RSVD_JB(4, 1) else RSVD_JB(4, 2)
    }
#undef RSVD_JB
    if (e != cudaSuccess) return e;
    ++g_kernel_launches;
    return cudaGetLastError();
  }
  const int JGv = g_jacobi_lanes ? g_jacobi_lanes : (L <= 64 ? 4 : 8);
  const int threads = (int)round_up((int64_t)(L / 2) * JGv, 32);
  const int epl_need = (l + JGv - 1) / JGv;
  cudaError_t e = cudaSuccess;
#define RSVD_JX(JG, EPL)                                                                                   \
  {                                                                                                       \
    const int ldx = JG * EPL + 4;                                                                         \
    const size_t smem = std::max((size_t)L * ldx * sizeof(double),                                        \
                                 (size_t)JA_CH * 64 * sizeof(double2) + (size_t)(threads / 32) * 129 * sizeof(double)); \
    e = smem_optin(jacobi_x_kernel<JG, EPL>); if (e != cudaSuccess) return e;                                                                                                      \
    e = launch_pdl(jacobi_x_kernel<JG, EPL>, dim3(1 + (unsigned)ceil_div(ldo, threads / 32)), dim3(threads), smem, st, \
                   R, ldr, l, sigma, W, ldo, rlog, rank, flag, sweeps, J, prog, done, epoch);               \
    if (e != cudaSuccess) return e; \
  }
#define RSVD_JX_EPL(JG)                  \
  if (epl_need <= 1) RSVD_JX(JG, 1)      \
  else if (epl_need <= 2) RSVD_JX(JG, 2) \
  else if (epl_need <= 4) RSVD_JX(JG, 4) \
  else if (epl_need <= 8) RSVD_JX(JG, 8) \
  else if (epl_need <= 16) RSVD_JX(JG, 16) \
  else RSVD_JX(JG, 32)
  if (JGv == 4) { RSVD_JX_EPL(4) }
  else if (JGv == 16) { RSVD_JX_EPL(16) }
  else { RSVD_JX_EPL(8) }
#undef RSVD_JX_EPL
#undef RSVD_JX
  ++g_kernel_launches;
  return cudaGetLastError();
}

size_t jacobi_scratch_bytes(int l) {   // rotation log (either order), rank[129], prog, done
  return std::max(jacobi_log_bytes(l), jacobi_blk_log_bytes(l)) + 256 * sizeof(int);
}

}  // namespace rsvd
