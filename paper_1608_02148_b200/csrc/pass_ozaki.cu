// pass_ozaki.cu -- the FP64 passes over A on the 5th-generation tensor cores:
// Ozaki-scheme emulation of the FP64 products Y = A X (sketch / power pass,
// Eq. YAQ, Alg. 2 step 4) and Z = A^T Q (Alg. 2 step 3, Eq. BQA
// P:220) with tcgen05.mma kind::i8 (int8 x int8 -> int32 in TMEM).
//
// Why: tcgen05 has no f64 kind; the warp-level DMMA pipe (37 TFLOP/s measured)
// bounds a pass at l/4 flop per A byte to ~20-40% of the HBM roof.
// int8 tensor throughput is ~60x higher, so an exact slice decomposition
// moves the pass to the HBM roof.
//
// Representation: every row r of A gets one exponent E_r with max_j |a_rj| <
// 2^{E_r}; a is rounded to the 56-bit integer N = rn(a 2^{55-E_r}) (exact for
// every a >= 2^{E_r-3}; error <= 2^{E_r-56} otherwise) and N is stored as S = 7
// two's-complement bytes: digit 0 signed (s8), digits 1..6 unsigned (u8),
// weight of digit t = 2^{E_r-7-8t}.  The row exponents are found and applied
// in ONE read of A (ozaki_slice_rows_kernel: a warp per row, the row re-read
// from L1/L2 for the digits).  X (the panel, K x Np) is cut per (1024-row
// block, column) with exponent F into S balanced signed digits (s8, N =
// rn(x 2^{54-F}) < 2^54 in magnitude, weight of digit u = 2^{F-6-8u}).  The
// NN pass applies 2^{E_r} to output row r at write-out; the TN pass (A^T X,
// reducing over rows) slices X' = X diag(2^{E_k - E_max}) instead (exact
// power-of-two row scaling) and applies 2^{E_max} at write-out.  Then
//   (A X)_ij = 2^{E_i} sum_sb 2^{F} sum_{t,u} 2^{-13-8(t+u)} (D_t X_u)_ij
// where D_t X_u over one super-block is an exact int32 dot product
// (|.| <= 1024 * 255 * 128 < 2^25).  Products with t + u > S - 1 are dropped
// (weight <= 2^{-69} relative to 2^{E+F}: below FP64 rounding of the sum).
// Terms of equal weight g = t + u share one TMEM accumulator: S groups x N
// columns (N <= 64: 448 of 512 TMEM columns); the t = 0 MMAs run as s8 x s8,
// the others as u8 x s8 (kind::i8 takes the operand signedness per
// instruction).  After each super-block the epilogue converts the groups to
// FP64 and accumulates the scaled sum in registers.
//
// A is sliced once per rsvd call (ozaki_slice_a) and read by every pass (S
// bytes per element instead of 8); X is sliced before each pass.
//
// Roles (384 threads): warp 0 = TMA producer, warp 1 = MMA issuer, warp 2 =
// TMEM allocator, warps 4..11 = epilogue (TMEM lanes = output rows, two warps
// per lane quadrant splitting the columns, so the FP64 accumulators stay in
// registers).  Stream-K over (row block, k-block) units with an in-kernel
// fix-up (column-major partials; the last segment of a CTA stages its rows
// through the idle unit buffers for coalesced stores).
#include <cuda.h>

#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace rsvd {
namespace oz {
using namespace tc;

// 384 threads: warp 0 TMA producer, warp 1 MMA issuer, warp 2 TMEM allocator,
// warps 4..11 epilogue (two per TMEM lane quadrant, each owning half of the N
// columns, so the FP64 accumulators stay in registers: <= 168 per thread)
constexpr int BM = 128, BKO = 128, THREADS = 384, EPI_WARPS = 8, EPI_THREADS = 32 * EPI_WARPS;
// N = 128 (FP32 A at Np = 128, one CTA per row block): 16 epilogue warps, 32 columns each
__host__ __device__ constexpr int oz_epi_warps(int N) { return N > 64 ? 16 : EPI_WARPS; }
__host__ __device__ constexpr int oz_threads(int N) { return 128 + 32 * oz_epi_warps(N); }
constexpr int A_TILE = BM * BKO;                    // bytes of one slice tile
constexpr int ET = 1024;                            // exponent blocks of X: 1024 rows x 1 column;
// the drain interval / X exponent block: 4096 k for both digit counts (int32
// headroom: 7 pairs x 4096 x 255 x 128 < 2^30): a quarter of the TMEM drains that
// stall the MMA issuer (probes: FP32 pass 2232 -> 2098 us, config-3 FP64 pass 2235
// -> 2179 us; config-3 step 21.2 -> 20.3 ms; 8192 at S = 3 gained nothing more).
// The X slicer reduces a block's column maxima over a cluster of 4 CTAs.
__host__ __device__ constexpr int oz_et(int S) { return S > 0 ? 4096 : ET; }
                                                    // int32 accumulation over 1024 k: <= 7 pairs * 1024 * 255 * 128 < 2^28

__host__ __device__ inline int64_t unit_lo(int64_t units, int grid, int c) { return (units * (int64_t)c) / grid; }

// first k-block of row block mb (Args::krot)
__device__ __forceinline__ int oz_phi(int64_t krot, int64_t KB, int mb) {
  return krot > 0 ? (int)((((int64_t)mb * KB) % krot) % KB) : 0;
}
#ifndef OZ_PROBE
#define OZ_PROBE_DECL
#define OZ_PROBE(slot)
#define OZ_PROBE_OUT
#define OZ_PROBE2_DECL
#define OZ_PROBE2(slot)
#define OZ_PROBE2_OUT
#define OZ_PROBE3_DECL
#define OZ_PROBE3(slot)
#define OZ_PROBE3_OUT
#endif
#ifndef OZ_TL
#define OZ_TL(slot) {}                              // probe builds: per-CTA timeline (tools/test_ozaki.cu)
#endif

// L2 policies of the loads (the CUTLASS CacheHintSm90 encodings): A's slices
// are read once per pass (evict first, so the stream does not push X out),
// X's slices by every row block (evict last).
constexpr uint64_t kL2EvictFirst = 0x12F0000000000000ull, kL2EvictLast = 0x14F0000000000000ull;

__device__ __forceinline__ void tma_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4, %5}], [%6], %7;"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar)),
        "l"(kL2EvictFirst)
      : "memory");
}
__device__ __forceinline__ void tma_2d_keep(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(kL2EvictLast)
      : "memory");
}
// A-slice tile multicast into both CTAs of a 2-CTA cluster (same smem offset;
// each CTA's mbarrier at the same offset receives the bytes)
__device__ __forceinline__ void tma_4d_mc(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3, uint64_t* bar,
                                          uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster.L2::cache_hint [%0], [%1, {%2, %3, %4, %5}], [%6], %7, %8;"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar)), "h"(mask),
        "l"(kL2EvictFirst)
      : "memory");
}
// MODE 3 (row pair, cta_group::2): each CTA loads its own tiles into its own shared
// memory and signals the LEADER's (rank 0) barrier: the peer bit of the barrier's
// shared::cluster address cleared (the CUTLASS 2-SM TMA convention)
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;
__device__ __forceinline__ void tma_4d_2sm(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4, %5}], [%6], %7;"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
        "r"(smem_u32(bar) & kPeerMask), "l"(kL2EvictFirst)
      : "memory");
}
__device__ __forceinline__ void tma_2d_2sm_keep(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar) & kPeerMask),
        "l"(kL2EvictLast)
      : "memory");
}
__device__ __forceinline__ void tma_4d_2sm_keep(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4, %5}], [%6], %7;"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
        "r"(smem_u32(bar) & kPeerMask), "l"(kL2EvictLast)
      : "memory");
}
__device__ __forceinline__ void mma_i8_2sm(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(tmem), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit_2sm_mc(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               ::"r"(smem_u32(bar)), "h"((uint16_t)3) : "memory");
}
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(smem_u32(bar) & kPeerMask) : "memory");
}
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               ::"r"(smem_u32(bar)), "h"(mask) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mma_i8(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(tmem), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// ---------------------------------------------------------------- slicing
// exponent E with max |a| < 2^E (0 for an all-zero block)
__device__ __forceinline__ int block_exp(double mx) { return mx > 0.0 ? ilogb(mx) + 1 : 0; }

// A digits: N = rn(v 2^{8S-1-E}) (|N| < 2^{8S-1}) as S two's-complement bytes,
// most significant first (byte 0 read as s8, the others as u8); packed 4
// elements per word
template <int S>
__device__ __forceinline__ void digits_a4(const double (&v)[4], double s1, double s2, uint32_t (&w)[S]) {
#pragma unroll
  for (int t = 0; t < S; ++t) w[t] = 0u;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    // exact power-of-two scaling in two steps (2^{55-E} alone over/underflows
    // at the ends of the exponent range), then round
    long long q = __double2ll_rn(v[e] * s1 * s2);
    if constexpr (S < 7) {
      // fewer digits than a double's significand: rounding may reach 2^{8S-1}; clamp
      // (an error of one unit in the last digit, as the rounding itself)
      constexpr long long lim = (1ll << (8 * S - 1)) - 1;
      q = q > lim ? lim : (q < -lim ? -lim : q);
    }
#pragma unroll
    for (int t = 0; t < S; ++t) w[t] |= ((uint32_t)(q >> (8 * (S - 1 - t))) & 0xffu) << (8 * e);
  }
}

// f(a) = (a - c_j) * rs_j when c / rs are given (rpca centring / scaling, Alg. 6)
__device__ __forceinline__ double fval(const double* A, int64_t lda, const double* c, const double* rs, int64_t r,
                                       int64_t cc) {
  double a = A[r * lda + cc];
  if (c) a -= c[cc];
  if (rs) a *= rs[cc];
  return a;
}

// 2^e as two exactly representable factors (e in about [-2200, 2200])
__device__ __forceinline__ void pow2_split(int e, double& p1, double& p2) {
  const int h = e / 2;
  p1 = ldexp(1.0, h);
  p2 = ldexp(1.0, e - h);
}

// four consecutive f(a) of one row starting at column j0 (zeros beyond n);
// 16-byte loads when the row is 16-byte aligned (T = double or float)
template <bool LAST, typename T>
__device__ __forceinline__ void load_f4(const T* row, int64_t j0, int64_t n, bool vec, const double* c,
                                        const double* rs, double (&v)[4]) {
  if (vec && j0 + 3 < n) {
    // first read: default caching (the row is read again right after); second: evict-first
    if constexpr (sizeof(T) == 8) {
      const double2 a = LAST ? __ldcs(reinterpret_cast<const double2*>(row + j0)) : *reinterpret_cast<const double2*>(row + j0);
      const double2 b = LAST ? __ldcs(reinterpret_cast<const double2*>(row + j0 + 2)) : *reinterpret_cast<const double2*>(row + j0 + 2);
      v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
    } else {
      const float4 a = LAST ? __ldcs(reinterpret_cast<const float4*>(row + j0)) : *reinterpret_cast<const float4*>(row + j0);
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = j0 + q < n ? (double)row[j0 + q] : 0.0;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (j0 + q >= n) { v[q] = 0.0; continue; }
    if (c) v[q] -= c[j0 + q];
    if (rs) v[q] *= rs[j0 + q];
  }
}

// Slices of f(A) = (A - 1 c^T) diag(rs) with one exponent per row, in one HBM
// read of A: a warp per row finds max_j |f(a_rj)| (pass 1, the row streamed
// from HBM), then writes the S digit bytes of every 128-column block (pass 2,
// the row re-read from L1 / L2); layout [row][col block][t][128 B] (one
// unit's S slice boxes = one contiguous S x 128 B run per row).  erow[r] =
// E_r; *emax = max_r E_r + kEBias (atomicMax, zeroed by the launcher); flag
// |= 4 on a non-finite f(a).
constexpr int kEBias = 4096;
template <int S, typename T>
__global__ void __launch_bounds__(256)
ozaki_slice_rows_kernel(const T* __restrict__ A, int64_t lda, int64_t m, int64_t n, const double* __restrict__ c,
                        const double* __restrict__ rs, int8_t* __restrict__ slices, int64_t ldn, int* __restrict__ erow,
                        unsigned* emax, int* flag) {
  pdl_wait();
  pdl_trigger();
  __shared__ unsigned wm[8];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t nblk = ldn / BKO;
  const bool vec = ((lda * (int64_t)sizeof(T)) % 16 == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
  unsigned mymax = 0;
  bool nf = false;
  for (int64_t r = (int64_t)blockIdx.x * 8 + wid; r < m; r += (int64_t)gridDim.x * 8) {
    const T* row = A + r * lda;
    double mx = 0.0;
#pragma unroll 4
    for (int64_t j0 = 4 * lane; j0 < n; j0 += 128) {
      double v[4];
      load_f4<false>(row, j0, n, vec, c, rs, v);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (!isfinite(v[q])) nf = true;
        mx = fmax(mx, fabs(v[q]));
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const int E = isfinite(mx) ? block_exp(mx) : 0;
    if (lane == 0) erow[r] = E;
    mymax = max(mymax, (unsigned)(E + kEBias));
    double s1, s2;
    pow2_split(8 * S - 1 - E, s1, s2);
    for (int64_t b = 0; b < nblk; ++b) {
      const int64_t j0 = b * BKO + 4 * lane;
      double v[4];
      load_f4<true>(row, j0, n, vec, c, rs, v);
      uint32_t w[S];
      digits_a4<S>(v, s1, s2, w);
      int8_t* dst = slices + ((r * nblk + b) * S) * BKO + 4 * lane;
#pragma unroll
      for (int t = 0; t < S; ++t) *reinterpret_cast<uint32_t*>(dst + t * BKO) = w[t];
    }
  }
  if (nf) atomicOr(flag, 4);
  if (lane == 0) wm[wid] = mymax;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = 0;
    for (int q = 0; q < 8; ++q) t = max(t, wm[q]);
    if (t) atomicMax(emax, t);
  }
}

// The same slices with the rows staged in shared memory: one CTA per SM made
// of G groups of SR_W warps, each group owning one row buffer; the group's
// first thread bulk-copies the group's next row (cp.async.bulk, one
// transaction, the group's mbarrier), the group reduces max |f(a)| (shuffles +
// a named barrier of the group only) and writes the digits from shared memory.
// Groups never wait for each other, so copies and arithmetic overlap with up
// to 32 warps per SM.  One HBM read of A.  The centring / scaling vectors (rpca)
// are staged in shared memory too, in place of row buffers.  Needs 16-byte
// aligned rows (16-byte row pitch and row length) and room for two row buffers.
// T = double (FP64 A) or float (FP32 A: the digits of the exactly upcast value).
constexpr int SR_SMEM = 200 * 1024, SR_W = 4, SR_MAX_G = 8;
template <int S, typename T>
__global__ void __launch_bounds__(32 * SR_W * SR_MAX_G, 1)
ozaki_slice_rows_smem_kernel(const T* __restrict__ A, int64_t lda, int64_t m, int64_t n,
                             const double* __restrict__ c, const double* __restrict__ rs, int8_t* __restrict__ slices,
                             int64_t ldn, int* __restrict__ erow, unsigned* emax, int* flag) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(128) unsigned char srow_raw[];
  __shared__ uint64_t full[SR_MAX_G];
  __shared__ double redm[SR_MAX_G][SR_W];
  __shared__ unsigned wmx[SR_MAX_G * SR_W];
  constexpr int GT = 32 * SR_W;                     // threads per group
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int grp = wid / SR_W, gw = wid % SR_W, gt = threadIdx.x % GT;
  const int ng = blockDim.x / GT;
  const int64_t nblk = ldn / BKO;
  const uint32_t row_bytes = (uint32_t)(n * sizeof(T));
  const int64_t rbuf = (row_bytes + 127) / 128 * 128;          // bytes per group buffer (128-byte aligned)
  const int64_t vstride = (n * 8 + 127) / 128 * 16;            // doubles per staged vector
  T* row = reinterpret_cast<T*>(srow_raw + grp * rbuf);
  // the centring / scaling vectors staged once behind the row buffers: with most
  // of the SM's L1 given to shared memory they would otherwise come from L2 for
  // every element (measured: the dominant stall of the centred config-3 slicing)
  double* cs = reinterpret_cast<double*>(srow_raw + ng * rbuf);
  double* rss = cs + (c ? vstride : 0);
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    if (c) cs[j] = c[j];
    if (rs) rss[j] = rs[j];
  }
  if (gt == 0) mbar_init(&full[grp], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  unsigned mymax = 0;
  bool nf = false;
  uint32_t phase = 0;
  const int64_t gstride = (int64_t)gridDim.x * ng;
  for (int64_t r = (int64_t)blockIdx.x * ng + grp; r < m; r += gstride, phase ^= 1u) {
    if (gt == 0) {
      mbar_expect_tx(&full[grp], row_bytes);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(row)), "l"(A + r * lda), "r"(row_bytes), "r"(smem_u32(&full[grp])) : "memory");
    }
    mbar_wait(&full[grp], phase);
    // FP32 A without centring / scaling: the row in float arithmetic (exact: |a|,
    // max, and below the power-of-two scaling), 16-byte reads, four chains
    constexpr bool F32 = sizeof(T) == 4;
    const bool fast = F32 && !c && !rs;
    double mx = 0.0;
    if (fast) {
      float m4[4] = {0.f, 0.f, 0.f, 0.f};
      bool bad = false;
      for (int64_t j = 4 * gt; j < n; j += 4 * GT) {
        const float4 a = *reinterpret_cast<const float4*>(row + j);
        const float e[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          bad |= !isfinite(e[q]);
          m4[q] = fmaxf(m4[q], fabsf(e[q]));
        }
      }
      if (bad) nf = true;
      mx = bad ? (double)INFINITY : (double)fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
    } else {
      for (int64_t j = gt; j < n; j += GT) {
        double v = (double)row[j];
        if (c) v -= cs[j];
        if (rs) v *= rss[j];
        if (!isfinite(v)) nf = true;
        mx = fmax(mx, fabs(v));
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) redm[grp][gw] = mx;
    asm volatile("bar.sync %0, %1;" ::"r"(grp + 1), "n"(GT) : "memory");
#pragma unroll
    for (int w = 0; w < SR_W; ++w) mx = fmax(mx, redm[grp][w]);
    const int E = isfinite(mx) ? block_exp(mx) : 0;
    if (gt == 0) erow[r] = E;
    mymax = max(mymax, (unsigned)(E + kEBias));
    double s1, s2;
    pow2_split(8 * S - 1 - E, s1, s2);
    if constexpr (F32) {
      // 2^{8S-1-E} as a normal float: N = rn(a 2^{8S-1-E}) in float arithmetic
      // (the scaling is exact, |N| < 2^{8S-1} <= 2^31)
      const int se = 8 * S - 1 - E;
      if (fast && se >= -126 && se <= 127) {
        const float sf = __int_as_float((se + 127) << 23);
        for (int64_t q = gt; q < nblk * 32; q += GT) {
          const int64_t blk = q >> 5;
          const int64_t j0 = blk * BKO + 4 * (q & 31);
          uint32_t w[S];
#pragma unroll
          for (int t = 0; t < S; ++t) w[t] = 0u;
          if (j0 < n) {
            const float4 a = *reinterpret_cast<const float4*>(row + j0);
            // rounding may reach 2^{8S-1} (a within half a unit below 2^E): clamp
            constexpr int lim = (int)((1ll << (8 * S - 1)) - 1);
            const float4 b = make_float4(a.x * sf, a.y * sf, a.z * sf, a.w * sf);
            const int nq[4] = {max(-lim, min(lim, __float2int_rn(b.x))), max(-lim, min(lim, __float2int_rn(b.y))),
                               max(-lim, min(lim, __float2int_rn(b.z))), max(-lim, min(lim, __float2int_rn(b.w)))};
#pragma unroll
            for (int e = 0; e < 4; ++e)
#pragma unroll
              for (int t = 0; t < S; ++t) w[t] |= ((uint32_t)(nq[e] >> (8 * (S - 1 - t))) & 0xffu) << (8 * e);
          }
          int8_t* dst = slices + ((r * nblk + blk) * S) * BKO + 4 * (q & 31);
#pragma unroll
          for (int t = 0; t < S; ++t) *reinterpret_cast<uint32_t*>(dst + t * BKO) = w[t];
        }
        asm volatile("bar.sync %0, %1;" ::"r"(grp + 1), "n"(GT) : "memory");   // the buffer and redm are reused
        continue;
      }
    }
    // 32 threads per 128-column block, 4 consecutive columns per thread
    for (int64_t q = gt; q < nblk * 32; q += GT) {
      const int64_t blk = q >> 5;
      const int64_t j0 = blk * BKO + 4 * (q & 31);
      double v[4];
      if constexpr (sizeof(T) == 8) {
        // two 16-byte reads per thread (n even: a pair is wholly inside or outside
        // the row); lanes with bit 2 set read their second half first, so each
        // read instruction of the warp touches every bank group equally
        const bool h0 = (q >> 2) & 1;
        double2 a[2];
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int64_t jj = j0 + 2 * (hh ^ (int)h0);
          a[hh] = make_double2(0.0, 0.0);
          if (jj < n) {
            a[hh] = *reinterpret_cast<const double2*>(row + jj);
            if (c) { const double2 cc = *reinterpret_cast<const double2*>(cs + jj); a[hh].x -= cc.x; a[hh].y -= cc.y; }
            if (rs) { const double2 rr = *reinterpret_cast<const double2*>(rss + jj); a[hh].x *= rr.x; a[hh].y *= rr.y; }
          }
        }
        const double2 lo = h0 ? a[1] : a[0], hi = h0 ? a[0] : a[1];
        v[0] = lo.x; v[1] = lo.y; v[2] = hi.x; v[3] = hi.y;
      } else {
        // one 16-byte read per thread (n % 4 == 0: a quad is wholly inside or outside the row)
        v[0] = v[1] = v[2] = v[3] = 0.0;
        if (j0 < n) {
          const float4 a = *reinterpret_cast<const float4*>(row + j0);
          v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (c) v[e] -= cs[j0 + e];
            if (rs) v[e] *= rss[j0 + e];
          }
        }
      }
      uint32_t w[S];
      digits_a4<S>(v, s1, s2, w);
      int8_t* dst = slices + ((r * nblk + blk) * S) * BKO + 4 * (q & 31);
#pragma unroll
      for (int t = 0; t < S; ++t) *reinterpret_cast<uint32_t*>(dst + t * BKO) = w[t];
    }
    asm volatile("bar.sync %0, %1;" ::"r"(grp + 1), "n"(GT) : "memory");   // the buffer and redm are reused
  }
  if (nf) atomicOr(flag, 4);
  if (lane == 0) wmx[wid] = mymax;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = max(t, wmx[w]);
    if (t) atomicMax(emax, t);
  }
}

// X (K x Np, ldx) -> xs[u][j][k] (u < S, j < Np, ld ldk bytes) and
// xf[sb * Np + j] = 2^E(sb, j) for 1024-row super-blocks sb, in one kernel:
// a CTA (512 threads) owns one super-block x 8 columns, 16 values per thread
// kept in registers; (1) column maxima by a fixed-order reduction, (2) the
// digits into a shared tile [u][column][row] (row stride XT_LD bytes), (3)
// the tile written out as 1024-byte rows (16-byte stores).  Rows >= K are
// zero digits.
constexpr int XT_COLS = 8, XT_THREADS = 512, XT_G = XT_THREADS / XT_COLS, XT_V = ET / XT_G, XT_LD = ET + 16;
__host__ __device__ constexpr int xt_smem(int S) { return S * XT_COLS * XT_LD; }

template <int S>
__global__ void __launch_bounds__(XT_THREADS)
ozaki_slice_x_kernel(const double* __restrict__ X, int64_t ldx, int64_t K, int Np, int8_t* __restrict__ xs,
                     int64_t ldk, double* __restrict__ xf, unsigned* epoch_ctr, const int* __restrict__ erow,
                     const unsigned* __restrict__ emax) {
  pdl_wait();
  pdl_trigger();
  // the next pass kernel's stream-K epoch (read by it after its griddepcontrol.wait):
  // advanced on the device so that CUDA-graph replays get fresh epochs too
  if (epoch_ctr && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) ++*epoch_ctr;
  extern __shared__ __align__(16) unsigned char xt[];      // S x XT_COLS x XT_LD
  __shared__ double red[XT_G][XT_COLS];
  __shared__ double escale[XT_COLS][2];
  const int tid = threadIdx.x, c = tid & (XT_COLS - 1), g = tid / XT_COLS;
  // grid: x = column group (fastest), y = super-block, so the CTAs reading the
  // column groups of the same rows run together (whole rows from DRAM, not
  // 64-byte pieces of rows read at different times)
  // oz_et(S) > 1024: the CX = oz_et(S) / 1024 CTAs of a cluster (along y) slice one
  // exponent block together; their column maxima meet in shared memory (DSMEM)
  constexpr int CX = oz_et(S) / ET;
  const int64_t sb = blockIdx.y, k0 = sb * ET;
  const int j = blockIdx.x * XT_COLS + c;
  const bool jv = j < Np;
  double v[XT_V];
  int ev[XT_V];
  double mx = 0.0;
  // all loads first (X values and, for TN passes, the row exponents), then the
  // arithmetic: the exponent-dependent scaling otherwise serialised the loads
  // (ncu: long-scoreboard stalls on the exponent subtraction dominated)
#pragma unroll
  for (int i = 0; i < XT_V; ++i) {
    const int64_t k = k0 + g + XT_G * i;
    v[i] = (jv && k < K) ? X[k * ldx + j] : 0.0;
    ev[i] = (erow && k < K) ? __ldg(erow + k) : 0;
  }
  const int eoff = erow ? (int)*emax - kEBias : 0;
#pragma unroll
  for (int i = 0; i < XT_V; ++i) {
    // TN passes: X' = diag(2^{E_k - E_max}) X folds A's row exponents into the panel
    if (erow) {
      const int d = ev[i] - eoff;                             // <= 0 (rows beyond K: v = 0)
      v[i] *= d >= -1022 ? __hiloint2double((d + 1023) << 20, 0) : ldexp(1.0, d);
    }
    mx = fmax(mx, fabs(v[i]));
  }
  // column maxima: the 4 row groups of a warp by shuffles (lane bits 3, 4), then
  // the 16 warp maxima of a column by one thread (fixed order: deterministic)
  mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
  mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
  if ((threadIdx.x & 31) < XT_COLS) red[threadIdx.x >> 5][c] = mx;
  __syncthreads();
  if constexpr (CX > 1) {
    __shared__ double cmax[CX][XT_COLS];
    const int crk = (int)(blockIdx.y % CX);
    // every CTA of the cluster must be running before its shared memory is written
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
    if (g == 0) {
      double m2 = red[0][c];
      for (int r = 1; r < XT_THREADS / 32; ++r) m2 = fmax(m2, red[r][c]);
      const uint32_t local = (uint32_t)__cvta_generic_to_shared(&cmax[crk][c]);
      for (int pr = 0; pr < CX; ++pr) {
        uint32_t remote;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(pr));
        asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(remote), "d"(m2) : "memory");
      }
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (g == 0) {
      double m2 = cmax[0][c];
      for (int pr = 1; pr < CX; ++pr) m2 = fmax(m2, cmax[pr][c]);
      const int E = block_exp(m2);
      if (jv && crk == 0) xf[(sb / CX) * Np + j] = ldexp(1.0, E);
      pow2_split(8 * S - 2 - E, escale[c][0], escale[c][1]);
    }
  } else if (g == 0) {
    double m2 = red[0][c];
    for (int r = 1; r < XT_THREADS / 32; ++r) m2 = fmax(m2, red[r][c]);
    const int E = block_exp(m2);
    if (jv) xf[sb * Np + j] = ldexp(1.0, E);
    pow2_split(8 * S - 2 - E, escale[c][0], escale[c][1]);
  }
  __syncthreads();
  const double sc1 = escale[c][0], sc2 = escale[c][1];
#pragma unroll
  for (int i = 0; i < XT_V; ++i) {
    const int r = g + XT_G * i;
    long long q = __double2ll_rn(v[i] * sc1 * sc2);
#pragma unroll
    for (int t = S - 1; t >= 1; --t) {
      const int d = (int)(signed char)(q & 0xff);
      q = (q - d) >> 8;                                      // exact
      xt[(t * XT_COLS + c) * XT_LD + r] = (unsigned char)d;
    }
    xt[c * XT_LD + r] = (unsigned char)q;
  }
  __syncthreads();
  const int64_t kend = min((int64_t)ET, ldk - k0);          // multiple of 16
  const int chunks = (int)(kend / 16);
  for (int e = tid; e < S * XT_COLS * chunks; e += XT_THREADS) {
    const int row = e / chunks, ch = e - row * chunks;
    const int t = row / XT_COLS, cc = row - t * XT_COLS;
    const int jj = blockIdx.x * XT_COLS + cc;
    if (jj >= Np) continue;
    *reinterpret_cast<uint4*>(xs + ((int64_t)t * Np + jj) * ldk + k0 + 16 * ch) =
        *reinterpret_cast<const uint4*>(xt + row * XT_LD + 16 * ch);
  }
}

// ---------------------------------------------------------------- pass kernel
struct Args {
  double* C; int64_t ldc;
  double* P; unsigned* flags; unsigned epoch;
  const int* erow; const unsigned* emax;            // A's row exponents E_r, max_r E_r + kEBias
  const double* xf;                                 // 2^E per (k-block, column) of X
  int64_t M, K; int N, Nout, Np;
  int64_t KB, units; int grid;
  // k rotation of the Aᵀ·X passes (0 = off): the units of row block mb visit the
  // k-blocks from phi(mb) = ((mb KB) mod krot) mod KB on (cyclically), krot = the
  // units per CTA (pair).  Every CTA (pair) then starts its range at one of ~3
  // k offsets instead of one per CTA, so the CTAs stream the same X-slice rows
  // at the same time and X (Q's slices, > L2 at config 3) is read ~once from HBM.
  int64_t krot;
  // CL = 2 (Np = 128): the second CTA of each pair computes columns [64, 128)
  double* C2; const double* xf2; int Nout2;
};

// One unit = (128-row output block, BK-k block): S A-slice tiles (128 x BK B)
// + the S X-slice tiles (N x BK B), loaded as one transaction into one of NB
// unit buffers (as many as fit in 219 KB, at most 6).  BK = 64 (default: 2
// buffers at N = 64); BK = 32 (RSVD_OZ_BK=32) fits 5 buffers but its 32-byte
// box rows stream slower (measured: DESIGN.md §9).
constexpr int kMaxBuf = 6;
__host__ __device__ constexpr int oz_ubuf(int S, int N, int BK) { return (S * BM * BK + S * N * BK + 1023) / 1024 * 1024; }
__host__ __device__ constexpr int oz_nbuf(int S, int N, int BK) {
  return (219 * 1024 - 1024) / oz_ubuf(S, N, BK) < kMaxBuf ? (219 * 1024 - 1024) / oz_ubuf(S, N, BK) : kMaxBuf;
}

// CL = 2 (Np = 128 as two 64-column halves in one launch): the CTAs of a
// 2-CTA cluster take the same units in lock step, CTA r computing columns
// [64 r, 64 r + 64) from its own X slices; each loads half of the unit's A
// slice tiles and multicasts them to both, so A's slices are read once per
// pass instead of once per column half.  Stream-K runs over the pairs.
//
// MODE 3 (row pair, FP32 A at Np = 128): the two CTAs of a cluster own two
// adjacent 128-row blocks of the SAME unit (256 rows) and one tcgen05.mma
// .cta_group::2 (M = 256, N = 128) covers both: each CTA streams only its own A
// rows and HALF of the X tile (64 of the 128 columns; the pair's MMA reads the
// other half from the peer), so a CTA ingests 1.5 bytes per byte of its A slices
// instead of 3 (column pair) or 2 (one CTA, N = 128) -- the SM's L2 -> shared
// ingest (~10 TB/s chip-wide) is what bounds the pass (tools/test_ozaki.cu
// probes: the kernel with its MMAs removed runs as fast as with them).  The
// leader (rank 0) arms the stage barriers and issues the MMAs; both CTAs' TMA
// loads complete on the leader's barriers; commits are multicast to both.
template <bool TRANS, int S, int N, int MODE, int BK>
__global__ void __launch_bounds__(oz_threads(N), 1)
ozaki_pass_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapX,
                  const __grid_constant__ CUtensorMap mapX2, Args g) {
  constexpr int CL = MODE == 1 ? 1 : 2;             // cluster size
  constexpr bool RP = MODE == 3;                    // row pair (cta_group::2)
  constexpr int NX = RP ? N / 2 : N;                // X columns (B rows) held per CTA
  pdl_wait();
  if (threadIdx.x == 0) OZ_TL(0)
  pdl_trigger();
  const unsigned epoch = *reinterpret_cast<const volatile unsigned*>(g.flags + kEpochSlot);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int BKU = BK;                           // k per unit
#ifdef OZ_KSU_OVERRIDE                               // probe builds only: drain interval in units (wrong numerics)
  constexpr int KSU = OZ_KSU_OVERRIDE;
#else
  constexpr int KSU = oz_et(S) / BKU;               // units per exponent super-block
#endif
  constexpr int A_UT = BM * BKU;                    // bytes of one A-slice tile of a unit
  constexpr int XSL = NX * BKU;                     // bytes of one X slice tile (NX rows x BK k)
  constexpr int UBUF = oz_ubuf(S, NX, BK);
  constexpr int NB = oz_nbuf(S, NX, BK);            // unit buffers
  constexpr int KPB = BKO / BKU;                    // units per 128-column slice block
  // NN: K-major tiles with BK-byte rows (SW64 / SW32); TN: MN-major 128 B rows (SW128)
  constexpr uint32_t LAY_K = BK == 64 ? LAYOUT_SW64 : LAYOUT_SW32;
  constexpr uint32_t SBO_K = BK == 64 ? 512 : 256;
  // accumulator sets in TMEM: two (at column 0 and 256) when S x N <= 256, so the
  // MMAs of the next exponent super-block never wait for the epilogue's drain
  constexpr int NACC = 2 * S * N <= 512 ? 2 : 1;
  static_assert(!RP || (CL == 2 && N == 128), "row pairs: N = 128");
  __shared__ uint64_t ufull[kMaxBuf], uempty[kMaxBuf], accf[2], acce[2];
  __shared__ uint32_t tmem_base;
  constexpr int EPI_WARPS = oz_epi_warps(N), EPI_THREADS = 32 * EPI_WARPS;
  constexpr int XFW = N / (EPI_WARPS / 4) > 32 ? N / (EPI_WARPS / 4) : 32;   // column factors per epilogue warp
  __shared__ double xfsm[EPI_WARPS * XFW + 1];    // + 1: last-arriver broadcast slot

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t KB = g.KB;                          // 64-k blocks
  const int crank = CL == 2 ? (int)(blockIdx.x & 1) : 0;   // rank in the cluster = column half (MODE 2) / row block (MODE 3)
  const int pid = (int)blockIdx.x / CL, npair = g.grid / CL;
  const int64_t u_lo = unit_lo(g.units, npair, pid);
  const int64_t u_hi = unit_lo(g.units, npair, pid + 1);
  const int nun = (int)(u_hi - u_lo);
  // (row block, unit index j within it, k-block) of the first unit; the loops
  // advance them incrementally (no 64-bit division per unit on the single-thread
  // producer / MMA paths).  kb = (j + phi(mb)) mod KB (Args::krot).
  const int mb0 = (int)(u_lo / KB), j0 = (int)(u_lo - (int64_t)mb0 * KB);
  const int KBi = (int)KB;
  const int kb0 = (int)((j0 + oz_phi(g.krot, KB, mb0)) % KBi);
  // next unit: j wraps into the next row block (kb restarts at its phi), kb wraps at KB
  auto adv = [&](int& mb, int& j, int& kb) {
    if (++kb == KBi) kb = 0;
    if (++j == KBi) { j = 0; ++mb; kb = oz_phi(g.krot, KB, mb); }
  };
  double* const Cout = (crank && !RP) ? g.C2 : g.C;
  const double* const xfh = (crank && !RP) ? g.xf2 : g.xf;
  const int Nout = (crank && !RP) ? g.Nout2 : g.Nout;

  if (tid == 0) {
    for (int s = 0; s < NB; ++s) { mbar_init(&ufull[s], 1); mbar_init(&uempty[s], RP ? 1 : CL); }
    for (int s = 0; s < 2; ++s) { mbar_init(&accf[s], 1); mbar_init(&acce[s], RP ? 2 * EPI_WARPS : EPI_WARPS); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    if constexpr (RP) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "n"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "n"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  if (CL == 2) cluster_sync_all(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    // ---------------- TMA producer: one transaction per unit
    if (lane == 0) {
      OZ_PROBE2_DECL
      int mb = mb0, j = j0, kb = kb0, ub = 0;
      uint32_t ph = 0;
      for (int it = 0; it < nun; ++it, adv(mb, j, kb), (++ub == NB ? (ub = 0, ph ^= 1u) : 0u)) {
        unsigned char* ubuf = base + ub * UBUF;
        OZ_PROBE2(0)
        mbar_wait(&uempty[ub], ph ^ 1u);
        OZ_PROBE2(1)
        if constexpr (RP) {
          // own 128 rows of A (row block 2 mb + crank) and own half of the X columns;
          // the bytes of both CTAs complete on the leader's barrier, which the leader arms
          if (crank == 0) mbar_expect_tx(&ufull[ub], (uint32_t)(2 * (S * A_UT + S * XSL)));
          // ONE box per operand and unit: all S digit tiles of A (tensor map dims
          // {byte, row, digit, column block}: box -> [digit][row][BK]) and all S digit
          // tiles of this CTA's X half (dims {k, column, half, digit}) -- the TMA
          // engine streams large boxes faster than many 4-8 KB ones
          const int orb = 2 * mb + crank;
          if (!TRANS) tma_4d_2sm(ubuf, &mapA, (int)((kb % KPB) * BKU), (int)((int64_t)orb * BM), 0, (int)(kb / KPB), &ufull[ub]);
          else tma_4d_2sm(ubuf, &mapA, 0, (int)(kb * BKU), 0, orb, &ufull[ub]);
          tma_4d_2sm_keep(ubuf + S * A_UT, &mapX, (int)(kb * BKU), 0, crank, 0, &ufull[ub]);
        } else {
#if defined(OZ_NO_A_TMA)            // probe builds only (tools/test_ozaki.cu): no A-slice loads
        mbar_expect_tx(&ufull[ub], (uint32_t)(S * XSL));
        if (false) {
#elif defined(OZ_NO_X_TMA)          // probe builds only: no X-slice loads
        mbar_expect_tx(&ufull[ub], (uint32_t)(S * A_UT));
        if (CL == 1) {
#else
        mbar_expect_tx(&ufull[ub], (uint32_t)(S * A_UT + S * XSL));
        if (CL == 1) {
#endif
          for (int t = 0; t < S; ++t) {
            if (!TRANS) tma_4d(ubuf + t * A_UT, &mapA, (int)((kb % KPB) * BKU), t, (int)(kb / KPB), (int)((int64_t)mb * BM), &ufull[ub]);
            else tma_4d(ubuf + t * A_UT, &mapA, 0, t, (int)mb, (int)(kb * BKU), &ufull[ub]);
          }
        } else {
          for (int t = crank; t < S; t += 2) {
            if (!TRANS)
              tma_4d_mc(ubuf + t * A_UT, &mapA, (int)((kb % KPB) * BKU), t, (int)(kb / KPB), (int)((int64_t)mb * BM), &ufull[ub], (uint16_t)3);
            else tma_4d_mc(ubuf + t * A_UT, &mapA, 0, t, (int)mb, (int)(kb * BKU), &ufull[ub], (uint16_t)3);
          }
        }
        const CUtensorMap* mx = crank ? &mapX2 : &mapX;
#ifndef OZ_NO_X_TMA
        for (int t = 0; t < S; ++t) tma_2d_keep(ubuf + S * A_UT + t * XSL, mx, (int)(kb * BKU), t * g.Np, &ufull[ub]);
#endif
        }
        OZ_PROBE2(2)
      }
      if (CL == 2) {
        // the peer's commits for the last units must have landed before this CTA exits
        for (int it = nun > NB ? nun - NB : 0; it < nun; ++it) mbar_wait(&uempty[it % NB], (uint32_t)((it / NB) & 1));
      }
      OZ_PROBE2(0)
      OZ_PROBE2_OUT
      OZ_TL(1)
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (MODE 3: the leader only, one MMA for both CTAs)
    if (lane == 0 && (!RP || crank == 0)) {
      // X slices u0..u0+c-1 are consecutive N-row tiles and their groups t+u0..t+u0+c-1
      // consecutive N-column blocks of TMEM: one MMA with N_mma = c N covers them (<= 256)
      // D s32; B s8; A s8 for digit 0, u8 for the others (bits 7-9, set per t)
      const uint32_t idesc0 = (2u << 4) | (1u << 10) | ((TRANS ? 1u : 0u) << 15) | (0u << 16) |
                              ((uint32_t)((RP ? 2 * BM : BM) >> 4) << 24);
      // MODE 3: one digit per MMA (the pair's B operand is split by columns: digit
      // batches would put different digits in the two CTAs)
      constexpr int CMAX = RP ? 1 : 256 / N;
      const uint32_t ub0 = smem_u32(base);
      const uint64_t dA0 = TRANS ? sdesc(ub0, 16, 1024, LAYOUT_SW128) : sdesc(ub0, 16, SBO_K, LAY_K);
      const uint64_t dX0 = sdesc(ub0 + S * A_UT, 16, SBO_K, LAY_K);
      OZ_PROBE_DECL
      int ndrain = 0;
      bool fresh = true;
      int mb = mb0, j = j0, kb = kb0, ub = 0;
      uint32_t ph = 0;
      for (int it = 0; it < nun; ++it, adv(mb, j, kb), (++ub == NB ? (ub = 0, ph ^= 1u) : 0u)) {
        // drain at the end of an X exponent super-block, of K, and of the row block
        const bool drain = (kb % KSU == KSU - 1) || kb == KBi - 1 || j == KBi - 1 || it == nun - 1;
        OZ_PROBE(0)
        mbar_wait(&ufull[ub], ph);
        OZ_PROBE(3)
#ifndef OZ_NO_EPI
        // a fresh super-block reuses accumulator set ndrain % NACC: drain ndrain - NACC must be done
        if (fresh && ndrain >= NACC) mbar_wait(&acce[ndrain % NACC], (uint32_t)((ndrain / NACC - 1) & 1));
#endif
        OZ_PROBE(2)
        tc_fence_after();
        // descriptors = the buffer-0 descriptors + the 16-byte offset of this unit's
        // buffer (the start-address field is the low 14 bits, addr >> 4 < 2^14: no
        // carry) -- no descriptor rebuilt per unit on the single issuing thread
        const uint64_t uo = (uint64_t)((ub * UBUF) >> 4);
        const uint64_t dx0 = dX0 + uo;
        const uint32_t acc0 = fresh ? 0u : 1u;
        const uint32_t tacc = tmem + (uint32_t)((ndrain % NACC) * 256);
#pragma unroll
        for (int t = 0; t < S; ++t) {
          // NN: A tile K-major, 64 B rows (SW64, k-step +32 B); TN: MN-major, 128 B rows (SW128, k-step +32 rows)
          const uint64_t da0 = dA0 + uo + (uint64_t)((t * A_UT) >> 4);
#pragma unroll
          for (int kk = 0; kk < BKU / 32; ++kk) {
            const uint64_t da = da0 + (uint64_t)(TRANS ? kk * 256 : kk * 2);
#pragma unroll
            for (int u0 = 0; u0 < S - t; u0 += CMAX) {
              const int cnt = (S - t - u0) < CMAX ? (S - t - u0) : CMAX;
              const uint64_t db = dx0 + (uint64_t)((u0 * XSL + kk * 32) >> 4);
              const uint32_t idesc = idesc0 | ((t == 0 ? 1u : 0u) << 7) | ((uint32_t)((cnt * N) >> 3) << 17);
#ifndef OZ_SKIP_MMA
              if constexpr (RP) mma_i8_2sm(tacc + (uint32_t)((t + u0) * N), da, db, idesc, (t > 0 || kk > 0) ? 1u : acc0);
              else mma_i8(tacc + (uint32_t)((t + u0) * N), da, db, idesc, (t > 0 || kk > 0) ? 1u : acc0);
#endif
            }
          }
        }
        OZ_PROBE(4)
        if constexpr (RP) {
          mma_commit_2sm_mc(&uempty[ub]);
          if (drain) { mma_commit_2sm_mc(&accf[ndrain % NACC]); ++ndrain; }
        } else {
          if (CL == 1) mma_commit(&uempty[ub]);
          else mma_commit_mc(&uempty[ub], (uint16_t)3);
          if (drain) { mma_commit(&accf[ndrain % NACC]); ++ndrain; }
        }
        fresh = drain;
      }
      OZ_PROBE_OUT
      OZ_TL(2)
    }
  } else if (warp >= 4) {
#ifdef OZ_NO_EPI                    // probe builds only: no epilogue at all
    if (true) {} else
#endif
    {
    // ---------------- epilogue: TMEM groups -> FP64, scale, accumulate; segment write-out
    // thread (row, hf) owns columns [hf * NC, hf * NC + NC) of output row `row`
    constexpr int NC = N / (EPI_WARPS / 4);           // columns per thread (32, or 8..24 at N < 64)
    const int et = tid - 128;                         // 0 .. EPI_THREADS - 1
    const int row = 32 * (warp & 3) + lane;
    const int hf = (warp - 4) >> 2;                   // column part
    const int c0 = hf * NC;
    const uint32_t tlane = (uint32_t)(32 * (warp & 3)) << 16;
    double acc[NC];
#pragma unroll
    for (int j = 0; j < NC; ++j) acc[j] = 0.0;
    double* xfs = xfsm + (warp - 4) * XFW;            // per-warp copy of this super-block's column factors
    int64_t ndrain = 0;
    OZ_PROBE3_DECL
    int mb = mb0, j = j0, kb = kb0;
    for (int it = 0; it < nun; ++it, adv(mb, j, kb)) {
      const int64_t u = u_lo + it;
      if (!((kb % KSU == KSU - 1) || kb == KBi - 1 || j == KBi - 1 || it == nun - 1)) continue;
      const int64_t sb = kb / KSU;                          // super-block along k (X exponent block)
      for (int j = lane; j < NC; j += 32) xfs[j] = xfh[sb * g.Np + c0 + j];
      __syncwarp();
      OZ_PROBE3(0)
      // one thread waits (sleeping), the other epilogue warps block on a named barrier
      const int abuf = (int)(ndrain % NACC);
      const uint32_t aoff = (uint32_t)(abuf * 256);
      if (et == 0) mbar_wait_sleep(&accf[abuf], (uint32_t)((ndrain / NACC) & 1));
      asm volatile("bar.sync 2, %0;" ::"n"(EPI_THREADS) : "memory");
      OZ_PROBE3(1)
      ++ndrain;
      tc_fence_after();
      // 8 columns at a time: the S group loads are issued back to back, one wait
#pragma unroll
      for (int c = 0; c < NC / 8; ++c) {
        uint32_t v[S][8];
#pragma unroll
#if defined(OZ_EPI_V) && (OZ_EPI_V & 1)   // probe builds only: no TMEM loads
        for (int gg = 0; gg < S; ++gg) for (int i = 0; i < 8; ++i) v[gg][i] = (uint32_t)(gg + i + c) * (uint32_t)row;
#else
        for (int gg = 0; gg < S; ++gg) TMEM_LD8(tmem + tlane + aoff + (uint32_t)(gg * N + c0 + 8 * c), v[gg]);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#endif
        // group g = t + u weighs 2^{-13-8g} (for every S); |v_g| < S * 1024 * 255 * 128 < 2^28
        static_assert(S == 7 || S == 3, "group combination for 7 (FP64) or 3 (FP32) digit groups");
        if constexpr (S == 7) {
          // groups 0..3 and 4..6 combine in int64 (exactly: < 2^55 and < 2^47), then two
          // int -> FP64 conversions (one rounding of the 55-bit group-0..3 sum, at
          // FP64 unit roundoff) instead of seven conversions
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const long long s0 = (((long long)(int)v[0][i] * 256 + (int)v[1][i]) * 256 + (int)v[2][i]) * 256 + (int)v[3][i];
            const long long s1 = ((long long)(int)v[4][i] * 256 + (int)v[5][i]) * 256 + (int)v[6][i];
            const double part = fma((double)s0, 0x1.0p-37, (double)s1 * 0x1.0p-61);
            acc[8 * c + i] = fma(part, xfs[8 * c + i], acc[8 * c + i]);
          }
        } else {
          // groups 0..2 combine exactly in int64 (< 2^45): one conversion per column
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const long long s0 = ((long long)(int)v[0][i] * 256 + (int)v[1][i]) * 256 + (int)v[2][i];
            acc[8 * c + i] = fma((double)s0 * 0x1.0p-29, xfs[8 * c + i], acc[8 * c + i]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (RP) mbar_arrive_leader(&acce[abuf]);
        else mbar_arrive(&acce[abuf]);
      }
      if (et == 0 && it == nun - 1) OZ_TL(5)
      OZ_PROBE3(2)
#if defined(OZ_EPI_V) && (OZ_EPI_V & 4)   // probe builds only: one store of the row sum, no fix-up
      if (j == KBi - 1 || it == nun - 1) {
        double sacc = 0.0;
#pragma unroll
        for (int j = 0; j < NC; ++j) sacc += acc[j];
        g.P[(int64_t)blockIdx.x * BM + row] = sacc;
#pragma unroll
        for (int j = 0; j < NC; ++j) acc[j] = 0.0;
      }
      if (false) {
#elif defined(OZ_EPI_V) && (OZ_EPI_V & 2)   // probe builds only: no write-out / fix-up
      if (false) {
#else
      if (j == KBi - 1 || it == nun - 1) {
#endif
        // stream-K fix-up, wait-free: a row block split over several CTAs (pairs)
        // gets one column-major partial per segment (slot 0 = the CTA's first
        // segment, 1 = its last) and an epoch-tagged arrival counter; the last
        // arriver sums the partials in CTA order (the same order whoever arrives
        // last, so results are bitwise reproducible) and writes the rows.
        const int64_t rb_lo = (int64_t)mb * KB, rb_hi = rb_lo + KB;
        const int64_t seg_start = (rb_lo > u_lo) ? rb_lo : u_lo;
        const bool full = seg_start == rb_lo && u + 1 == rb_hi;
        bool write = full;
        if (!full) {
          int pf = pid, pl = pid;                    // pairs covering this row block
          while (pf > 0 && unit_lo(g.units, npair, pf) > rb_lo) --pf;
          while (pl + 1 < npair && unit_lo(g.units, npair, pl + 1) < rb_hi) ++pl;
          const int slot = seg_start == u_lo ? 0 : 1;
          double* dst = g.P + (((int64_t)blockIdx.x * 2 + slot) * N + c0) * BM + row;
#pragma unroll
          for (int j = 0; j < NC; ++j) dst[(int64_t)j * BM] = acc[j];
          asm volatile("bar.sync 1, %0;" ::"n"(EPI_THREADS) : "memory");
          if (et == 0) {
            unsigned long long* cnt = reinterpret_cast<unsigned long long*>(g.flags + 2048) + (pf * CL + crank);
            __threadfence();                         // this CTA's partial before its arrival
            unsigned long long old = *reinterpret_cast<volatile unsigned long long*>(cnt), nw;
            for (;;) {
              nw = ((old >> 32) == epoch) ? old + 1 : (((unsigned long long)epoch << 32) | 1ull);
              const unsigned long long seen = atomicCAS(cnt, old, nw);
              if (seen == old) break;
              old = seen;
            }
            const bool last = (int)(nw & 0xffffffffu) == pl - pf + 1;
            if (last) {
              __threadfence();                       // the other partials are visible after the last arrival
              atomicExch(cnt, 0ull);                 // back to zero: a later launch with the same epoch starts clean
            }
            xfsm[EPI_WARPS * XFW] = last ? 1.0 : 0.0;  // broadcast to the epilogue warps
          }
          asm volatile("bar.sync 1, %0;" ::"n"(EPI_THREADS) : "memory");
          write = xfsm[EPI_WARPS * XFW] != 0.0;
          if (write) {
#pragma unroll
            for (int j = 0; j < NC; ++j) acc[j] = 0.0;
            for (int pc = pf; pc <= pl; ++pc) {
              const int cc = pc * CL + crank;
              const int64_t ps = (rb_lo > unit_lo(g.units, npair, pc)) ? rb_lo : unit_lo(g.units, npair, pc);
              const int sl = ps == unit_lo(g.units, npair, pc) ? 0 : 1;
              const double* src = g.P + (((int64_t)cc * 2 + sl) * N + c0) * BM + row;
#pragma unroll
              for (int j = 0; j < NC; ++j) acc[j] += __ldcg(src + (int64_t)j * BM);
            }
            if (et == 0) OZ_TL(6)
          }
        }
        if (write) {
          // A's exponent: 2^{E_row} for NN, 2^{E_max} for TN (exact, two factors)
          {
            const int64_t gmr = (int64_t)(RP ? 2 * mb + crank : mb) * BM + row;
            const int e = TRANS ? (int)*g.emax - kEBias : (gmr < g.M ? g.erow[gmr] : 0);
            double p1, p2;
            pow2_split(e, p1, p2);
#pragma unroll
            for (int j = 0; j < NC; ++j) acc[j] = acc[j] * p1 * p2;
          }
          if (it == nun - 1) {
            // the CTA's last segment: every MMA and TMA load is complete, so the unit
            // buffers stage the 128 x N block for row-contiguous (coalesced) stores
            constexpr int LDS = N + 1;
            double* stg = reinterpret_cast<double*>(base);
#pragma unroll
            for (int j = 0; j < NC; ++j) stg[row * LDS + c0 + j] = acc[j];
            asm volatile("bar.sync 1, %0;" ::"n"(EPI_THREADS) : "memory");
            for (int r = warp - 4; r < BM; r += EPI_WARPS) {
              const int64_t grow = (int64_t)(RP ? 2 * mb + crank : mb) * BM + r;
              if (grow >= g.M) break;
              for (int j = lane; j < Nout; j += 32) Cout[grow * g.ldc + j] = stg[r * LDS + j];
            }
          } else {
            const int64_t gm = (int64_t)(RP ? 2 * mb + crank : mb) * BM + row;
            if (gm < g.M) {
              double* dsto = Cout + gm * g.ldc + c0;
#pragma unroll
              for (int j = 0; j < NC; ++j)
                if (c0 + j < Nout) dsto[j] = acc[j];
            }
          }
        }
#pragma unroll
        for (int j = 0; j < NC; ++j) acc[j] = 0.0;
      }
      OZ_PROBE3(3)
    }
    OZ_PROBE3(0)
    OZ_PROBE3_OUT
    if (et == 0) OZ_TL(3)
    }
  }
  tc_fence_before();
  if (CL == 2) cluster_sync_all(); else __syncthreads();
  if (threadIdx.x == 0) OZ_TL(4)
  if (warp == 2) {
    tc_fence_after();
    if constexpr (RP) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
  }
}

// ---------------------------------------------------------------- host side
// slices as a 4-D tensor (byte j < 128, slice t, column block, row) over the
// interleaved layout.  NN unit tile: 128 rows x 64 B (box {64, 1, 1, 128},
// SW64, K-major); TN unit tile: 64 rows x 128 B (box {128, 1, 1, 64}, SW128,
// MN-major operand).
static bool map_slices(CUtensorMap* mp, const int8_t* p, int64_t rows, int64_t nblk, int S, bool trans, int bk) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[4] = {128, (cuuint64_t)S, (cuuint64_t)nblk, (cuuint64_t)rows};
  cuuint64_t strides[3] = {128, (cuuint64_t)(128 * S), (cuuint64_t)(128 * S * nblk)};
  cuuint32_t box[4] = {trans ? 128u : (cuuint32_t)bk, 1, 1, trans ? (cuuint32_t)bk : 128u};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(mp, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<int8_t*>(p), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE,
             trans ? CU_TENSOR_MAP_SWIZZLE_128B : (bk == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B),
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// All S digit tiles of a unit in one box: dims {byte j < 128, row, digit, column
// block} (strides not increasing: the row stride is the largest) so the box lands
// as [digit][row][bytes] -- the per-digit tiles the MMA descriptors address.
// NN: box {bk, 128 rows, S, 1} (K-major, SW64 / SW32); TN: box {128, bk rows, S, 1}
// (MN-major, SW128).
static bool map_slices_all(CUtensorMap* mp, const int8_t* p, int64_t rows, int64_t nblk, int S, bool trans, int bk) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[4] = {128, (cuuint64_t)rows, (cuuint64_t)S, (cuuint64_t)nblk};
  cuuint64_t strides[3] = {(cuuint64_t)(128 * S * nblk), 128, (cuuint64_t)(128 * S)};
  cuuint32_t box[4] = {trans ? 128u : (cuuint32_t)bk, trans ? (cuuint32_t)bk : 128u, (cuuint32_t)S, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(mp, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<int8_t*>(p), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE,
             trans ? CU_TENSOR_MAP_SWIZZLE_128B : (bk == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B),
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// X slices xs[(t Np + j) ldk + k] viewed as {k, j < Np / 2, half, digit}: box
// {bk, Np / 2, 1, S} = one CTA's column half of all S digit tiles, [digit][column][k]
static bool map_x_halves(CUtensorMap* mp, const int8_t* p, int64_t K, int Np, int64_t ldk, int S, int bk) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[4] = {(cuuint64_t)K, (cuuint64_t)(Np / 2), 2, (cuuint64_t)S};
  cuuint64_t strides[3] = {(cuuint64_t)ldk, (cuuint64_t)(ldk * (Np / 2)), (cuuint64_t)(ldk * Np)};
  cuuint32_t box[4] = {(cuuint32_t)bk, (cuuint32_t)(Np / 2), 1, (cuuint32_t)S};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(mp, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<int8_t*>(p), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, bk == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
static bool map_i8_2d(CUtensorMap* mp, const int8_t* p, int64_t cols, int64_t rows, int64_t ld, int box_rows, int bk) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld};
  cuuint32_t box[2] = {(cuuint32_t)bk, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  return enc(mp, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(p), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, bk == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace oz

int ozaki_slices() { return OZ_S; }

// Np <= 64 in one launch; 64 < Np <= 128 as two column blocks (64, Np - 64):
// at Np = 128 one launch of CTA pairs (ozaki_pass_pair), else two launches over the same A slices (TMEM holds S groups x 64 columns)
bool ozaki_supported(int Np) { return Np <= 128 && Np % 16 == 0 && tc::get_encode() != nullptr; }

// FP32 A (3 digits) at Np = 128: all 128 columns per CTA (3 groups x 128 TMEM
// columns) -- MODE 3 row pairs (cta_group::2, default) or MODE 1 one CTA per
// row block (RSVD_OZ_MODE128=1); RSVD_OZ_MODE128=2: the column-pair launch
static int oz_mode128_env() {
  static const int env = [] { const char* v = getenv("RSVD_OZ_MODE128"); return v ? atoi(v) : 3; }();
  return env;
}
static bool oz_single128(int s, int Np) { return oz_mode128_env() != 2 && s == OZ_S32 && Np == 128; }
int ozaki_x_cols(int s, int Np) { return oz_single128(s, Np) ? 128 : (Np < 64 ? Np : 64); }

size_t ozaki_partial_bytes(int Np, int grid) {
  return (size_t)grid * 2 * oz::BM * (size_t)(Np < 128 ? Np : 128) * sizeof(double);
}

size_t ozaki_a_bytes(int64_t m, int64_t n, int s) {
  const int64_t ldn = round_up(n, oz::BKO);
  return (size_t)s * m * ldn + 256 + (size_t)round_up(m, 64) * sizeof(int) + 512;
}

size_t ozaki_x_bytes(int64_t K, int Np, int s) {
  const int64_t ldk = round_up(K, 16);
  return (size_t)s * Np * ldk + 256 + (size_t)round_up(ceil_div(K, (int64_t)oz::oz_et(s)) * Np, 32) * sizeof(double) + 256;
}

template <int S, typename T>
static cudaError_t ozaki_slice_a_t(const OzakiA& a, const T* A, int64_t lda, const double* c, const double* rs,
                                   int* flag, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(a.emax, 0, sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  // shared-memory staged rows (one buffer per group, bulk copies) when 16-byte aligned rows fit
  const int64_t rbuf = (a.n * (int64_t)sizeof(T) + 127) / 128 * 128;
  const int64_t vbuf = (a.n * 8 + 127) / 128 * 128;
  const int64_t vecs = (int64_t)(c != nullptr) + (rs != nullptr);          // staged c / rs, vbuf bytes each
  const int ngroups = (int)std::max<int64_t>(0, std::min<int64_t>(oz::SR_MAX_G, (oz::SR_SMEM - vecs * vbuf) / rbuf));
  const int64_t qa = 16 / (int64_t)sizeof(T);                            // elements per 16 bytes
  if (ngroups >= 2 && (a.n % qa == 0) && (lda % qa == 0) && (reinterpret_cast<uintptr_t>(A) % 16 == 0)) {
    e = smem_optin(oz::ozaki_slice_rows_smem_kernel<S, T>);
    if (e != cudaSuccess) return e;
    e = launch_plain(oz::ozaki_slice_rows_smem_kernel<S, T>,
                     dim3((unsigned)std::min<int64_t>(ceil_div(a.m, (int64_t)ngroups), 148)),
                     dim3(32 * oz::SR_W * ngroups), (size_t)(ngroups * rbuf + vecs * vbuf), st, A, lda, a.m, a.n, c, rs,
                     a.slices, a.ldn, a.erow, a.emax, flag);
    if (e != cudaSuccess) return e;
    ++g_kernel_launches;
    return cudaGetLastError();
  }
  // otherwise one warp per row, rows in flight bounded so that the second read of
  // each row hits L1 / L2: at most ~256 KB of rows per SM
  const int64_t row_bytes = std::max<int64_t>(a.n * (int64_t)sizeof(T), 1);
  const int64_t per_sm = std::max<int64_t>(1, std::min<int64_t>(8, (256 << 10) / (8 * row_bytes)));
  const int64_t grid = std::min<int64_t>(ceil_div(a.m, 8), 148 * per_sm);
  // plain launch: it follows the memset of emax
  e = launch_plain(oz::ozaki_slice_rows_kernel<S, T>, dim3((unsigned)grid), dim3(256), 0, st, A, lda, a.m, a.n, c, rs,
                   a.slices, a.ldn, a.erow, a.emax, flag);
  if (e != cudaSuccess) return e;
  ++g_kernel_launches;
  return cudaGetLastError();
}

cudaError_t ozaki_slice_a(const OzakiA& a, const void* A, bool f32, int64_t lda, const double* c, const double* rs,
                          int* flag, cudaStream_t st) {
  if (f32 && a.s == OZ_S32) return ozaki_slice_a_t<OZ_S32>(a, (const float*)A, lda, c, rs, flag, st);
  if (!f32 && a.s == OZ_S) return ozaki_slice_a_t<OZ_S>(a, (const double*)A, lda, c, rs, flag, st);
  return cudaErrorInvalidValue;
}

OzakiA ozaki_layout_a(void* buf, int64_t m, int64_t n, int s) {
  OzakiA a{};
  a.m = m; a.n = n; a.ldn = round_up(n, oz::BKO); a.s = s;
  a.slices = reinterpret_cast<int8_t*>(buf);
  a.erow = reinterpret_cast<int*>(reinterpret_cast<char*>(buf) + round_up((int64_t)s * m * a.ldn, 256));
  a.emax = reinterpret_cast<unsigned*>(a.erow + round_up(m, 64));
  return a;
}

// k per unit of the pass kernels: 64 (default) or 32 (RSVD_OZ_BK=32)
static int oz_bk() {
  static const int v = [] { const char* e = getenv("RSVD_OZ_BK"); return (e && atoi(e) == 32) ? 32 : 64; }();
  return v;
}
template <int S> static cudaError_t ozaki_slice_cols(const OzakiCall& c, cudaStream_t st);
template <int S> static cudaError_t ozaki_pass_cols(const OzakiCall& c, cudaStream_t st);
template <int S> static cudaError_t ozaki_pass_pair(const OzakiCall& h0, const OzakiCall& h1, cudaStream_t st);
template <int S> static cudaError_t ozaki_pass_rowpair(const OzakiCall& c, cudaStream_t st);

// X slicing of every column block first, then the pass kernel(s): c.mark (if
// set) separates the two in time for the per-kernel profile.
template <int S>
static cudaError_t ozaki_pass_t(const OzakiCall& c, cudaStream_t st) {
  if (oz_single128(S, c.N)) {
    cudaError_t e = ozaki_slice_cols<S>(c, st);
    if (e != cudaSuccess) return e;
    if (c.mark) cudaEventRecord(c.mark, st);
    if (c.mark2) cudaEventRecord(c.mark2, st);
    if (oz_mode128_env() == 3 && c.grid >= 2) return ozaki_pass_rowpair<S>(c, st);
    return ozaki_pass_cols<S>(c, st);
  }
  OzakiCall h0 = c, h1 = c;
  const bool two = c.N > 64;
  if (two) {
    h0.N = 64; h0.Nout = c.Nout < 64 ? c.Nout : 64;   // columns [0, 64): B, C with their own leading dimensions
    h1.B = c.B + 64; h1.C = c.C + 64; h1.N = c.N - 64; h1.Nout = c.Nout - 64; h1.epoch = c.epoch2;
    h1.xscratch = c.xscratch2;
    if (!c.xscratch2) return cudaErrorInvalidValue;
  }
  cudaError_t e = ozaki_slice_cols<S>(h0, st);
  if (e == cudaSuccess && two) e = ozaki_slice_cols<S>(h1, st);
  if (e != cudaSuccess) return e;
  if (c.mark) cudaEventRecord(c.mark, st);
  if (c.mark2) cudaEventRecord(c.mark2, st);
  // Np = 128: both halves in one launch of CTA pairs sharing A (RSVD_OZ_PAIR=0: two launches)
  static const int env_pair = [] { const char* v = getenv("RSVD_OZ_PAIR"); return v ? atoi(v) : 1; }();
  if (two && c.N == 128 && h1.Nout > 0 && env_pair != 0 && c.grid >= 2) return ozaki_pass_pair<S>(h0, h1, st);
  e = ozaki_pass_cols<S>(h0, st);
  if (e == cudaSuccess && two && h1.Nout > 0) e = ozaki_pass_cols<S>(h1, st);
  return e;
}

cudaError_t ozaki_pass(const OzakiCall& c, cudaStream_t st) {
  if (!ozaki_supported(c.N) || c.M <= 0 || c.K <= 0) return cudaErrorInvalidValue;
  if (c.a->s == OZ_S) return ozaki_pass_t<OZ_S>(c, st);
  if (c.a->s == OZ_S32) return ozaki_pass_t<OZ_S32>(c, st);
  return cudaErrorInvalidValue;
}

template <int S>
static cudaError_t ozaki_slice_cols(const OzakiCall& c, cudaStream_t st) {
  using namespace oz;
  const int N = c.N;
  const int64_t ldk = round_up(c.K, 16);
  int8_t* xs = reinterpret_cast<int8_t*>(c.xscratch);
  double* xf = reinterpret_cast<double*>(reinterpret_cast<char*>(c.xscratch) + round_up((int64_t)S * N * ldk, 256));
  const cudaError_t ea = smem_optin(ozaki_slice_x_kernel<S>);
  if (ea != cudaSuccess) return ea;
  constexpr int CX = oz_et(S) / ET;
  const dim3 gs((unsigned)ceil_div(N, XT_COLS), (unsigned)(ceil_div(ceil_div(ldk, (int64_t)ET), (int64_t)CX) * CX));
  cudaError_t el;
  if constexpr (CX == 1) {
    el = launch_pdl(ozaki_slice_x_kernel<S>, gs, dim3(XT_THREADS), (size_t)xt_smem(S), st, c.B, c.ldb, c.K, N, xs, ldk, xf,
                    c.flags ? c.flags + kEpochSlot : nullptr,
                    c.trans ? (const int*)c.a->erow : nullptr, (const unsigned*)c.a->emax);
  } else {
    // clusters of CX CTAs along y: one exponent block of oz_et(S) rows
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = gs;
    cfg.blockDim = dim3(XT_THREADS);
    cfg.dynamicSmemBytes = (size_t)xt_smem(S);
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = 1;
    at[1].val.clusterDim.y = CX;
    at[1].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    el = cudaLaunchKernelEx(&cfg, ozaki_slice_x_kernel<S>, c.B, c.ldb, c.K, N, xs, ldk, xf,
                            c.flags ? c.flags + kEpochSlot : nullptr,
                            c.trans ? (const int*)c.a->erow : nullptr, (const unsigned*)c.a->emax);
  }
  if (el != cudaSuccess) return el;
  ++g_kernel_launches;
  return cudaGetLastError();
}

// k rotation of the TN passes (Args::krot): the units per CTA (pair), or 0 (NN
// passes: X is L2-resident; RSVD_OZ_KROT=0 disables it for A/B runs)
static int64_t oz_krot(bool trans, int64_t units, int nctas) {
  static const bool off = [] { const char* v = getenv("RSVD_OZ_KROT"); return v && atoi(v) == 0; }();
  if (!trans || off || nctas < 1) return 0;
  const int64_t u = units / nctas;
  return u > 0 ? u : 1;
}

template <int S>
static cudaError_t ozaki_pass_cols(const OzakiCall& c, cudaStream_t st) {
  using namespace oz;
  const OzakiA& a = *c.a;
  const int N = c.N;
  // X slices (ozaki_slice_cols) are in c.xscratch
  const int64_t ldk = round_up(c.K, 16);
  int8_t* xs = reinterpret_cast<int8_t*>(c.xscratch);
  double* xf = reinterpret_cast<double*>(reinterpret_cast<char*>(c.xscratch) + round_up((int64_t)S * N * ldk, 256));
  // 2) tensor maps: A slices as (cols = n, rows = m, S); X slices as (cols = K, rows = S * N)
  const int bk = oz_bk();
  CUtensorMap mA, mX;
  if (!map_slices(&mA, a.slices, a.m, a.ldn / BKO, S, c.trans, bk)) return cudaErrorInvalidValue;
  if (!map_i8_2d(&mX, xs, c.K, (int64_t)S * N, ldk, N, bk)) return cudaErrorInvalidValue;
  Args g{};
  g.C = c.C; g.ldc = c.ldc; g.P = c.P; g.flags = c.flags; g.epoch = c.epoch;
  g.erow = a.erow; g.emax = a.emax; g.xf = xf;
  g.M = c.M; g.K = c.K; g.N = N; g.Nout = c.Nout; g.Np = N;
  g.KB = ceil_div(c.K, bk);
  const int64_t mblocks = ceil_div(c.M, BM);
  g.units = mblocks * g.KB;
  int64_t grid = g.units / (256 / bk);
  if (grid < mblocks) grid = mblocks;
  if (grid > c.grid) grid = c.grid;
  if (grid < 1) grid = 1;
  g.grid = (int)grid;
  g.krot = oz_krot(c.trans, g.units, g.grid);
  const int Nt = N <= 16 ? 16 : N <= 32 ? 32 : N <= 48 ? 48 : N <= 64 ? 64 : 128;
  const size_t smem = (size_t)oz_nbuf(S, Nt, bk) * oz_ubuf(S, Nt, bk) + 1024;
  cudaError_t e = cudaSuccess;
#define RSVD_OZ(TR, NN)                                                                                   \
  if (bk == 64) RSVD_OZB(TR, NN, 64) else RSVD_OZB(TR, NN, 32)
#define RSVD_OZB(TR, NN, BK)                                                                              \
  {                                                                                                      \
    e = smem_optin(ozaki_pass_kernel<TR, S, NN, 1, BK>); if (e != cudaSuccess) return e;                \
    e = launch_pdl(ozaki_pass_kernel<TR, S, NN, 1, BK>, dim3(g.grid), dim3(oz_threads(NN)), smem, st, mA, mX, mX, g); \
    if (e != cudaSuccess) return e;                                                                      \
  }
  if constexpr (S == OZ_S32) {
    if (N == 128) {
      if (!c.trans) RSVD_OZ(false, 128) else RSVD_OZ(true, 128)
      ++g_kernel_launches;
      return cudaGetLastError();
    }
  }
  if (!c.trans) {
    switch (N) { case 16: RSVD_OZ(false, 16) break; case 32: RSVD_OZ(false, 32) break;
                 case 48: RSVD_OZ(false, 48) break; default: RSVD_OZ(false, 64) break; }
  } else {
    switch (N) { case 16: RSVD_OZ(true, 16) break; case 32: RSVD_OZ(true, 32) break;
                 case 48: RSVD_OZ(true, 48) break; default: RSVD_OZ(true, 64) break; }
  }
#undef RSVD_OZ
#undef RSVD_OZB
  ++g_kernel_launches;
  return cudaGetLastError();
}

// Np = 128: one launch of 2-CTA clusters, CTA r of a pair computing column
// half r (h0 / h1, each sliced into its own X scratch) over the same units.
template <int S>
static cudaError_t ozaki_pass_pair(const OzakiCall& h0, const OzakiCall& h1, cudaStream_t st) {
  using namespace oz;
  const OzakiA& a = *h0.a;
  constexpr int N = 64;
  const int64_t ldk = round_up(h0.K, 16);
  int8_t* xs0 = reinterpret_cast<int8_t*>(h0.xscratch);
  int8_t* xs1 = reinterpret_cast<int8_t*>(h1.xscratch);
  const double* xf0 = reinterpret_cast<const double*>(reinterpret_cast<char*>(h0.xscratch) + round_up((int64_t)S * N * ldk, 256));
  const double* xf1 = reinterpret_cast<const double*>(reinterpret_cast<char*>(h1.xscratch) + round_up((int64_t)S * N * ldk, 256));
  const int bk = oz_bk();
  CUtensorMap mA, mX0, mX1;
  if (!map_slices(&mA, a.slices, a.m, a.ldn / BKO, S, h0.trans, bk)) return cudaErrorInvalidValue;
  if (!map_i8_2d(&mX0, xs0, h0.K, (int64_t)S * N, ldk, N, bk) || !map_i8_2d(&mX1, xs1, h1.K, (int64_t)S * N, ldk, N, bk))
    return cudaErrorInvalidValue;
  Args g{};
  g.C = h0.C; g.ldc = h0.ldc; g.P = h0.P; g.flags = h0.flags; g.epoch = h0.epoch;
  g.erow = a.erow; g.emax = a.emax; g.xf = xf0;
  g.C2 = h1.C; g.xf2 = xf1; g.Nout2 = h1.Nout;
  g.M = h0.M; g.K = h0.K; g.N = N; g.Nout = h0.Nout; g.Np = N;
  g.KB = ceil_div(h0.K, bk);
  const int64_t mblocks = ceil_div(h0.M, BM);
  g.units = mblocks * g.KB;
  int64_t npair = g.units / (256 / bk);
  if (npair < mblocks) npair = mblocks;
  if (npair > h0.grid / 2) npair = h0.grid / 2;
  if (npair < 1) npair = 1;
  g.grid = (int)(2 * npair);
  g.krot = oz_krot(h0.trans, g.units, (int)npair);
  const size_t smem = (size_t)oz_nbuf(S, N, bk) * oz_ubuf(S, N, bk) + 1024;
  cudaError_t e = cudaSuccess;
#define RSVD_OZP(TR)                                                                                      \
  if (bk == 64) RSVD_OZPB(TR, 64) else RSVD_OZPB(TR, 32)
#define RSVD_OZPB(TR, BK)                                                                                 \
  {                                                                                                      \
    e = smem_optin(ozaki_pass_kernel<TR, S, N, 2, BK>); if (e != cudaSuccess) return e;                 \
    e = launch_pdl_cluster(ozaki_pass_kernel<TR, S, N, 2, BK>, dim3(g.grid), dim3(THREADS), smem, st, 2u, mA, mX0, mX1, g); \
    if (e != cudaSuccess) return e;                                                                      \
  }
  if (!h0.trans) RSVD_OZP(false) else RSVD_OZP(true)
#undef RSVD_OZP
#undef RSVD_OZPB
  ++g_kernel_launches;
  return cudaGetLastError();
}

// MODE 3 (FP32 A at Np = 128): clusters of two CTAs over pairs of 128-row
// blocks, one cta_group::2 MMA (M = 256, N = 128) per digit product.
template <int S>
static cudaError_t ozaki_pass_rowpair(const OzakiCall& c, cudaStream_t st) {
  using namespace oz;
  if constexpr (S != OZ_S32) {
    return cudaErrorInvalidValue;
  } else {
    const OzakiA& a = *c.a;
    constexpr int N = 128;
    const int64_t ldk = round_up(c.K, 16);
    int8_t* xs = reinterpret_cast<int8_t*>(c.xscratch);
    const double* xf = reinterpret_cast<const double*>(reinterpret_cast<char*>(c.xscratch) + round_up((int64_t)S * N * ldk, 256));
    const int bk = oz_bk();
    CUtensorMap mA, mX;
    if (!map_slices_all(&mA, a.slices, a.m, a.ldn / BKO, S, c.trans, bk)) return cudaErrorInvalidValue;
    if (!map_x_halves(&mX, xs, c.K, N, ldk, S, bk)) return cudaErrorInvalidValue;   // half the columns per CTA
    Args g{};
    g.C = c.C; g.ldc = c.ldc; g.P = c.P; g.flags = c.flags; g.epoch = c.epoch;
    g.erow = a.erow; g.emax = a.emax; g.xf = xf;
    g.C2 = c.C; g.xf2 = xf; g.Nout2 = c.Nout;
    g.M = c.M; g.K = c.K; g.N = N; g.Nout = c.Nout; g.Np = N;
    g.KB = ceil_div(c.K, bk);
    const int64_t mpairs = ceil_div(c.M, 2 * BM);                    // 256-row unit blocks
    g.units = mpairs * g.KB;
    int64_t npair = g.units / (256 / bk);
    if (npair < mpairs) npair = mpairs;
    if (npair > c.grid / 2) npair = c.grid / 2;
    if (npair < 1) npair = 1;
    g.grid = (int)(2 * npair);
    g.krot = oz_krot(c.trans, g.units, (int)npair);
    const size_t smem = (size_t)oz_nbuf(S, N / 2, bk) * oz_ubuf(S, N / 2, bk) + 1024;
    cudaError_t e = cudaSuccess;
#define RSVD_OZR(TR, BK)                                                                                  \
    {                                                                                                    \
      e = smem_optin(ozaki_pass_kernel<TR, S, N, 3, BK>); if (e != cudaSuccess) return e;               \
      e = launch_pdl_cluster(ozaki_pass_kernel<TR, S, N, 3, BK>, dim3(g.grid), dim3(oz_threads(N)), smem, st, 2u, mA, mX, mX, g); \
      if (e != cudaSuccess) return e;                                                                    \
    }
    if (bk == 64) { if (!c.trans) RSVD_OZR(false, 64) else RSVD_OZR(true, 64) }
    else { if (!c.trans) RSVD_OZR(false, 32) else RSVD_OZR(true, 32) }
#undef RSVD_OZR
    ++g_kernel_launches;
    return cudaGetLastError();
  }
}

}  // namespace rsvd
