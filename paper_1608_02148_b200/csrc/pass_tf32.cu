// pass_tf32.cu -- the passes over an FP32 A (config 4) on the 5th-generation
// tensor cores: tcgen05.mma kind::tf32 with a 3-term split, TMEM accumulators,
// TMA-fed shared-memory ring, warp-specialised roles, stream-K partition.
//
//   NN:  C (M x N) = A (M x K) X (K x N)      (sketch / power pass, Alg. 4 step 3, Alg. 2 step 4)
//   TN:  C (M x N) = A^T (M x K) Q (K x N)    (A^T Q passes, Alg. 2 step 3, Alg. 4 step 10)
//
// Precision (reading R12): every FP32 operand x is
// split as x = hi + lo with hi = x truncated to TF32 (the bits kind::tf32
// consumes) and lo = rna_tf32(x - hi) (x - hi is exact in FP32); the product is
// A_hi B_hi + A_lo B_hi + A_hi B_lo, accumulated in FP32 in TMEM for at most
// TF_DRAIN units (2048 k) and then summed in FP64: the tensor core's FP32
// accumulation truncates, and over the 10^6-row reductions of config 4 an
// undrained TMEM accumulator drifted by ~2e-3 relative (full-size property
// test); two TMEM accumulator buffers alternate so the MMAs never wait for a
// drain.  Drains inside a row-block segment add into a per-CTA FP64 buffer.  The panel (X or
// Q) is split once per pass into global hi/lo FP32 copies by prep_split_b;
// the A tile is split in shared memory by the 4 epilogue warps.
//
// Roles (384 threads): warp 0 = TMA producer, warp 1 = MMA issuer (one
// thread), warp 2 = TMEM allocator, warps 4..7 = A-tile split, warps 8..11 =
// drains / epilogue (warp w reads TMEM lanes 32*(w%4)..+32), so a drain never
// delays the split of the next units.  Shared memory per stage:
// A (16 KB, SWIZZLE_128B; K-major for NN, MN-major for TN), A_lo (16 KB),
// B_hi, B_lo (N/32 boxes of 4 KB, MN-major).  3 stages.
#include <cuda.h>
#include <stdlib.h>

#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace rsvd {
namespace tf32 {
using namespace tc;

constexpr int BM = 128, BK = 32, STAGES = 3, THREADS = 384;
constexpr int TF_DRAIN = 64;                  // units (of BK = 32 k) per TMEM accumulation run
constexpr int A_BYTES = BM * BK * 4;          // 16 KB
constexpr int B_BOX_BYTES = 32 * BK * 4;      // 4 KB per 32-column box

struct Args {
  double* C; int64_t ldc;
  double* P;                                  // [grid][BM][N] partial of a CTA's leading segment
  double* Pacc;                               // [grid][BM][N] FP64 running sum between drains
  unsigned* flags; unsigned epoch;
  int64_t M, K; int N, Nout;
  int64_t KT, units;
  int grid;
};

__host__ __device__ inline int64_t unit_lo(int64_t units, int grid, int c) { return (units * (int64_t)c) / grid; }

#ifndef TF32_DEBUG_SPLIT
#define TF32_DEBUG_SPLIT
#endif
template <bool TRANS>
__global__ void __launch_bounds__(THREADS, 1)
pass_tf32_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapBhi,
                 const __grid_constant__ CUtensorMap mapBlo, Args g) {
  const unsigned epoch = *reinterpret_cast<const volatile unsigned*>(g.flags + kEpochSlot);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte aligned carve-up (SWIZZLE_128B atoms)
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int nbox = g.N / 32;
  const int b_bytes = nbox * B_BOX_BYTES;
  const int stage_bytes = 2 * A_BYTES + 2 * b_bytes;
  __shared__ uint64_t full[STAGES], splitd[STAGES], empty_[STAGES], accf[2], acce[2];
  __shared__ uint32_t tmem_base;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t KT = g.KT;
  const int64_t u_lo = unit_lo(g.units, g.grid, blockIdx.x);
  const int64_t u_hi = unit_lo(g.units, g.grid, blockIdx.x + 1);
  const int64_t nun = u_hi - u_lo;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&splitd[s], 4); mbar_init(&empty_[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&accf[b], 1); mbar_init(&acce[b], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "n"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;

  auto stageA = [&](int s) { return base + (size_t)s * stage_bytes; };
  auto stageAlo = [&](int s) { return base + (size_t)s * stage_bytes + A_BYTES; };
  auto stageBhi = [&](int s) { return base + (size_t)s * stage_bytes + 2 * A_BYTES; };
  auto stageBlo = [&](int s) { return base + (size_t)s * stage_bytes + 2 * A_BYTES + b_bytes; };

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      for (int64_t it = 0; it < nun; ++it) {
        const int s = (int)(it % STAGES);
        const uint32_t ph = (uint32_t)((it / STAGES) & 1);
        mbar_wait(&empty_[s], ph ^ 1);
        const int64_t u = u_lo + it, mb = u / KT, kt = u - mb * KT;
        const int m0 = (int)(mb * BM), k0 = (int)(kt * BK);
        mbar_expect_tx(&full[s], (uint32_t)(A_BYTES + 2 * b_bytes));
        if (!TRANS) {
          tma_2d(stageA(s), &mapA, k0, m0, &full[s]);                       // box {32 k, 128 rows}
        } else {
          for (int j = 0; j < 4; ++j) tma_2d(stageA(s) + j * B_BOX_BYTES, &mapA, m0 + 32 * j, k0, &full[s]);
        }
        for (int j = 0; j < nbox; ++j) {
          tma_2d(stageBhi(s) + j * B_BOX_BYTES, &mapBhi, 32 * j, k0, &full[s]);
          tma_2d(stageBlo(s) + j * B_BOX_BYTES, &mapBlo, 32 * j, k0, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (lane == 0) {
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((TRANS ? 1u : 0u) << 15) | (1u << 16) |
                             ((uint32_t)(g.N >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
      int64_t run = 0;                                // accumulation runs (drains) so far
      bool first = true;
      int in_run = 0;
      uint32_t acc_t = tmem;
      for (int64_t it = 0; it < nun; ++it) {
        const int s = (int)(it % STAGES);
        const uint32_t ph = (uint32_t)((it / STAGES) & 1);
        const int64_t u = u_lo + it, kt = u % KT;
        const bool run_end = (kt == KT - 1) || (it == nun - 1) || (in_run == TF_DRAIN - 1);
        if (first) {
          const int b = (int)(run & 1);
          if (run >= 2) { mbar_wait(&acce[b], (uint32_t)(((run - 2) >> 1) & 1)); }
          acc_t = tmem + (uint32_t)(b * g.N);
        }
        mbar_wait(&splitd[s], ph);
        tc_fence_after();
        const uint32_t aH = smem_u32(stageA(s)), aL = smem_u32(stageAlo(s));
        const uint32_t bH = smem_u32(stageBhi(s)), bL = smem_u32(stageBlo(s));
#pragma unroll
        for (int kk = 0; kk < BK / 8; ++kk) {
          uint64_t dAh, dAl;
          if (!TRANS) {   // K-major A: advance 32 B per 8-wide k step inside the 128 B swizzle row
            dAh = sdesc(aH + kk * 32, 16, 1024);
            dAl = sdesc(aL + kk * 32, 16, 1024);
          } else {        // MN-major A: 8 k rows (1 KB) per k step; 512 B k atoms; 32-column boxes 4 KB apart
            dAh = sdesc(aH + kk * 1024, B_BOX_BYTES, 512, LAYOUT_SW128_BASE32B);
            dAl = sdesc(aL + kk * 1024, B_BOX_BYTES, 512, LAYOUT_SW128_BASE32B);
          }
          const uint64_t dBh = sdesc(bH + kk * 1024, B_BOX_BYTES, 512, LAYOUT_SW128_BASE32B);
          const uint64_t dBl = sdesc(bL + kk * 1024, B_BOX_BYTES, 512, LAYOUT_SW128_BASE32B);
          const uint32_t acc0 = (first && kk == 0) ? 0u : 1u;
          mma_tf32(acc_t, dAh, dBh, idesc, acc0);
          mma_tf32(acc_t, dAl, dBh, idesc, 1u);
          mma_tf32(acc_t, dAh, dBl, idesc, 1u);
        }
        mma_commit(&empty_[s]);                       // smem stage free when these MMAs complete
        first = false;
        ++in_run;
        if (run_end) {
          mma_commit(&accf[run & 1]);                 // this accumulation run complete
          ++run;
          first = true;
          in_run = 0;
        }
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ---------------- A-tile split (warps 4..7)
    const int et = tid - 128;                         // 0..127
    for (int64_t it = 0; it < nun; ++it) {
      const int s = (int)(it % STAGES);
      const uint32_t ph = (uint32_t)((it / STAGES) & 1);
      if (et == 0) mbar_wait_sleep(&full[s], ph);    // one thread sleeps; the split warps block on a named barrier
      asm volatile("bar.sync 3, 128;" ::: "memory");
      float4* a4 = reinterpret_cast<float4*>(stageA(s));
      float4* l4 = reinterpret_cast<float4*>(stageAlo(s));
#pragma unroll 4
      for (int q = et; q < A_BYTES / 16; q += 128) {
        float4 a = a4[q], hi, lo;
        hi.x = tf32_trunc(a.x); lo.x = tf32_rna(a.x - hi.x);
        hi.y = tf32_trunc(a.y); lo.y = tf32_rna(a.y - hi.y);
        hi.z = tf32_trunc(a.z); lo.z = tf32_rna(a.z - hi.z);
        hi.w = tf32_trunc(a.w); lo.w = tf32_rna(a.w - hi.w);
#ifdef TF32_STORE_HI
        a4[q] = hi;                                   // (kind::tf32 ignores the low 13 bits anyway)
#endif
        l4[q] = lo;
      }
      TF32_DEBUG_SPLIT
      fence_proxy_async();                            // generic-proxy writes -> async proxy (MMA)
      __syncwarp();
      if (lane == 0) mbar_arrive(&splitd[s]);
    }
  } else if (warp >= 8) {
    // ---------------- drains + epilogue (warps 8..11)
    const int et = tid - 256;                         // 0..127
    int64_t run = 0;
    int in_run = 0, sub = 0;                          // sub: drains so far in this row-block segment
    const int row = 32 * (warp & 3) + lane;
    double* pacc = g.Pacc + ((int64_t)blockIdx.x * BM + row) * g.N;
    for (int64_t it = 0; it < nun; ++it) {
      const int64_t u = u_lo + it, mb = u / KT, kt = u - mb * KT;
      const bool seg_end = (kt == KT - 1) || (it == nun - 1);
      const bool run_end = seg_end || (in_run == TF_DRAIN - 1);
      ++in_run;
      if (!run_end) continue;
      in_run = 0;
      const int b = (int)(run & 1);
      if (et == 0) mbar_wait_sleep(&accf[b], (uint32_t)((run >> 1) & 1));
      asm volatile("bar.sync 2, 128;" ::: "memory");
      tc_fence_after();
      const uint32_t tbase = tmem + (uint32_t)(b * g.N) + ((uint32_t)(32 * (warp & 3)) << 16);
      if (!seg_end) {
        // intermediate drain: FP64 running sum of this row-block segment
        for (int c0 = 0; c0 < g.N; c0 += 32) {
          uint32_t v[32];
          TMEM_LD32(tbase + (uint32_t)c0, v);
          TMEM_WAIT_LD(v);
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            double2* pp = reinterpret_cast<double2*>(pacc + c0 + j);
            const double2 o = sub ? *pp : make_double2(0.0, 0.0);
            *pp = make_double2(o.x + (double)__uint_as_float(v[j]), o.y + (double)__uint_as_float(v[j + 1]));
          }
        }
        ++sub;
      } else {
        // in-kernel stream-K fix-up (see gemm_pass.cu): continuation -> partial +
        // release flag; head of a spanning row block -> acquire later partials
        const int64_t rb_lo = mb * KT, rb_hi = rb_lo + KT;
        const int64_t seg_start = (rb_lo > u_lo) ? rb_lo : u_lo;
        const bool cont = seg_start > rb_lo;
        const bool head = !cont && (u + 1 < rb_hi);
        const int64_t gm = mb * BM + row;
        for (int c0 = 0; c0 < g.N; c0 += 32) {
          uint32_t v[32];
          TMEM_LD32(tbase + (uint32_t)c0, v);
          TMEM_WAIT_LD(v);    // the registers are defined only after wait::ld
          double a[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) a[j] = (double)__uint_as_float(v[j]);
          if (sub) {
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
              const double2 o = *reinterpret_cast<const double2*>(pacc + c0 + j);
              a[j] += o.x;
              a[j + 1] += o.y;
            }
          }
          if (cont) {
            double* dst = g.P + ((int64_t)blockIdx.x * BM + row) * g.N + c0;
#pragma unroll
            for (int j = 0; j < 32; j += 2) *reinterpret_cast<double2*>(dst + j) = make_double2(a[j], a[j + 1]);
          } else {
            if (head) {
              for (int c = blockIdx.x + 1; c < g.grid && unit_lo(g.units, g.grid, c) < rb_hi; ++c) {
                unsigned f;
                do {
                  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(g.flags + c) : "memory");
                } while (f != epoch);
                const double* src = g.P + ((int64_t)c * BM + row) * g.N + c0;
#pragma unroll
                for (int j = 0; j < 32; j += 2) {
                  const double2 pv = *reinterpret_cast<const double2*>(src + j);
                  a[j] += pv.x;
                  a[j + 1] += pv.y;
                }
              }
            }
            if (gm < g.M) {
              double* dst = g.C + gm * g.ldc + c0;
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (c0 + j < g.Nout) dst[j] = a[j];
            }
          }
        }
        if (cont) {
          __threadfence();
          asm volatile("bar.sync 1, 128;" ::: "memory");     // the four epilogue warps
          if (et == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(g.flags + blockIdx.x), "r"(epoch) : "memory");
        }
        sub = 0;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acce[b]);
      ++run;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(256));
  }
}

// ---------------------------------------------------------------- TN as Q^T A
// C^T (N x M) = Q^T (N x K) A (K x M): the panel Q is the M-side operand (its
// hi / lo FP32 copies, 128 columns, zero-filled beyond N) and 256-column
// chunks of A are the N side, so the panel is re-read once per 256 columns of
// A instead of once per 128 (ncu, config 4: 136 GB of DRAM reads per launch
// for 40 GB of A with the A^T Q form).  Same roles, drains and stream-K
// fix-up as pass_tf32_kernel; D (128 x 256) double-buffered in all 512 TMEM
// columns; TMEM lane i = output column i, TMEM column j = output row c0 + j.
constexpr int TN_BN = 256, TN_STAGES = 2;
constexpr int TN_Q_BYTES = 128 * BK * 4;             // 16 KB: 4 boxes of 32 columns x 32 k
constexpr int TN_A_BYTES = TN_BN * BK * 4;           // 32 KB: 8 boxes
constexpr int TN_STAGE = 2 * TN_Q_BYTES + 2 * TN_A_BYTES;

// NN = true: the same with C^T = X^T A^T -- 256-row chunks of A (K-major, one
// TMA box) as the N-side operand, so the panel tile is shared by 256 rows.
template <bool NN>
__global__ void __launch_bounds__(THREADS, 1)
pass_tf32_tn_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapQhi,
                    const __grid_constant__ CUtensorMap mapQlo, Args g) {
  const unsigned epoch = *reinterpret_cast<const volatile unsigned*>(g.flags + kEpochSlot);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[TN_STAGES], splitd[TN_STAGES], empty_[TN_STAGES], accf[2], acce[2];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t KT = g.KT;
  const int64_t u_lo = unit_lo(g.units, g.grid, blockIdx.x);
  const int64_t u_hi = unit_lo(g.units, g.grid, blockIdx.x + 1);
  const int64_t nun = u_hi - u_lo;
  if (tid == 0) {
    for (int s = 0; s < TN_STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&splitd[s], 4); mbar_init(&empty_[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&accf[b], 1); mbar_init(&acce[b], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  auto stQh = [&](int s) { return base + (size_t)s * TN_STAGE; };
  auto stQl = [&](int s) { return base + (size_t)s * TN_STAGE + TN_Q_BYTES; };
  auto stA = [&](int s) { return base + (size_t)s * TN_STAGE + 2 * TN_Q_BYTES; };
  auto stAl = [&](int s) { return base + (size_t)s * TN_STAGE + 2 * TN_Q_BYTES + TN_A_BYTES; };

  if (warp == 0) {
    if (lane == 0) {
      for (int64_t it = 0; it < nun; ++it) {
        const int s = (int)(it % TN_STAGES);
        const uint32_t ph = (uint32_t)((it / TN_STAGES) & 1);
        mbar_wait(&empty_[s], ph ^ 1);
        const int64_t u = u_lo + it, ct = u / KT, kt = u - ct * KT;
        const int c0 = (int)(ct * TN_BN), k0 = (int)(kt * BK);
        mbar_expect_tx(&full[s], (uint32_t)(2 * TN_Q_BYTES + TN_A_BYTES));
        if (NN) tma_2d(stA(s), &mapA, k0, c0, &full[s]);                      // box {32 k, 256 rows}, K-major
        else
          for (int j = 0; j < 8; ++j) tma_2d(stA(s) + j * B_BOX_BYTES, &mapA, c0 + 32 * j, k0, &full[s]);
        for (int j = 0; j < 4; ++j) {
          tma_2d(stQh(s) + j * B_BOX_BYTES, &mapQhi, 32 * j, k0, &full[s]);
          tma_2d(stQl(s) + j * B_BOX_BYTES, &mapQlo, 32 * j, k0, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // D f32, A (= Q^T) tf32 MN-major, B (= A chunk) tf32 MN-major, N = 256, M = 128
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | ((NN ? 0u : 1u) << 16) |
                             ((uint32_t)(TN_BN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      int64_t run = 0;
      bool first = true;
      int in_run = 0;
      uint32_t acc_t = tmem;
      for (int64_t it = 0; it < nun; ++it) {
        const int s = (int)(it % TN_STAGES);
        const uint32_t ph = (uint32_t)((it / TN_STAGES) & 1);
        const int64_t u = u_lo + it, kt = u % KT;
        const bool run_end = (kt == KT - 1) || (it == nun - 1) || (in_run == TF_DRAIN - 1);
        if (first) {
          const int b = (int)(run & 1);
          if (run >= 2) mbar_wait(&acce[b], (uint32_t)(((run - 2) >> 1) & 1));
          acc_t = tmem + (uint32_t)(b * TN_BN);
        }
        mbar_wait(&splitd[s], ph);
        tc_fence_after();
        const uint32_t qH = smem_u32(stQh(s)), qL = smem_u32(stQl(s));
        const uint32_t aH = smem_u32(stA(s)), aL = smem_u32(stAl(s));
#pragma unroll
        for (int kk = 0; kk < BK / 8; ++kk) {
          const uint64_t dQh = sdesc(qH + kk * 1024, B_BOX_BYTES, 512, LAYOUT_SW128_BASE32B);
          const uint64_t dQl = sdesc(qL + kk * 1024, B_BOX_BYTES, 512, LAYOUT_SW128_BASE32B);
          uint64_t dAh, dAl;
          if (NN) {   // K-major chunk: 32 B per 8-wide k step inside the 128 B swizzle row
            dAh = sdesc(aH + kk * 32, 16, 1024);
            dAl = sdesc(aL + kk * 32, 16, 1024);
          } else {
            dAh = sdesc(aH + kk * 1024, B_BOX_BYTES, 512, LAYOUT_SW128_BASE32B);
            dAl = sdesc(aL + kk * 1024, B_BOX_BYTES, 512, LAYOUT_SW128_BASE32B);
          }
          const uint32_t acc0 = (first && kk == 0) ? 0u : 1u;
          mma_tf32(acc_t, dQh, dAh, idesc, acc0);
          mma_tf32(acc_t, dQl, dAh, idesc, 1u);
          mma_tf32(acc_t, dQh, dAl, idesc, 1u);
        }
        mma_commit(&empty_[s]);
        first = false;
        ++in_run;
        if (run_end) {
          mma_commit(&accf[run & 1]);
          ++run;
          first = true;
          in_run = 0;
        }
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // A-chunk split (32 KB per unit) into hi (in place) / lo
    const int et = tid - 128;
    for (int64_t it = 0; it < nun; ++it) {
      const int s = (int)(it % TN_STAGES);
      const uint32_t ph = (uint32_t)((it / TN_STAGES) & 1);
      if (et == 0) mbar_wait_sleep(&full[s], ph);    // one thread sleeps; the split warps block on a named barrier
      asm volatile("bar.sync 3, 128;" ::: "memory");
      float4* a4 = reinterpret_cast<float4*>(stA(s));
      float4* l4 = reinterpret_cast<float4*>(stAl(s));
#pragma unroll 4
      for (int q = et; q < TN_A_BYTES / 16; q += 128) {
        float4 a = a4[q], hi, lo;
        hi.x = tf32_trunc(a.x); lo.x = tf32_rna(a.x - hi.x);
        hi.y = tf32_trunc(a.y); lo.y = tf32_rna(a.y - hi.y);
        hi.z = tf32_trunc(a.z); lo.z = tf32_rna(a.z - hi.z);
        hi.w = tf32_trunc(a.w); lo.w = tf32_rna(a.w - hi.w);
#ifdef TF32_STORE_HI
        a4[q] = hi;                                   // (kind::tf32 ignores the low 13 bits anyway)
#endif
        l4[q] = lo;
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&splitd[s]);
    }
  } else if (warp >= 8) {
    // drains + epilogue: lane i of the TMEM quadrant = output column i
    const int et = tid - 256;
    int64_t run = 0;
    int in_run = 0, sub = 0;
    const int col = 32 * (warp & 3) + lane;            // output column (< 128)
    double* pacc = g.Pacc + ((int64_t)blockIdx.x * 128 + col) * TN_BN;
    for (int64_t it = 0; it < nun; ++it) {
      const int64_t u = u_lo + it, ct = u / KT, kt = u - ct * KT;
      const bool seg_end = (kt == KT - 1) || (it == nun - 1);
      const bool run_end = seg_end || (in_run == TF_DRAIN - 1);
      ++in_run;
      if (!run_end) continue;
      in_run = 0;
      const int b = (int)(run & 1);
      if (et == 0) mbar_wait_sleep(&accf[b], (uint32_t)((run >> 1) & 1));
      asm volatile("bar.sync 2, 128;" ::: "memory");
      tc_fence_after();
      const uint32_t tbase = tmem + (uint32_t)(b * TN_BN) + ((uint32_t)(32 * (warp & 3)) << 16);
      if (!seg_end) {
        for (int j0 = 0; j0 < TN_BN; j0 += 32) {
          uint32_t v[32];
          TMEM_LD32(tbase + (uint32_t)j0, v);
          TMEM_WAIT_LD(v);
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            double2* pp = reinterpret_cast<double2*>(pacc + j0 + j);
            const double2 o = sub ? *pp : make_double2(0.0, 0.0);
            *pp = make_double2(o.x + (double)__uint_as_float(v[j]), o.y + (double)__uint_as_float(v[j + 1]));
          }
        }
        ++sub;
      } else {
        const int64_t rb_lo = ct * KT, rb_hi = rb_lo + KT;
        const int64_t seg_start = (rb_lo > u_lo) ? rb_lo : u_lo;
        const bool cont = seg_start > rb_lo;
        const bool head = !cont && (u + 1 < rb_hi);
        for (int j0 = 0; j0 < TN_BN; j0 += 32) {
          uint32_t v[32];
          TMEM_LD32(tbase + (uint32_t)j0, v);
          TMEM_WAIT_LD(v);
          double a[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) a[j] = (double)__uint_as_float(v[j]);
          if (sub) {
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
              const double2 o = *reinterpret_cast<const double2*>(pacc + j0 + j);
              a[j] += o.x;
              a[j + 1] += o.y;
            }
          }
          if (cont) {
            double* dst = g.P + ((int64_t)blockIdx.x * 128 + col) * TN_BN + j0;
#pragma unroll
            for (int j = 0; j < 32; j += 2) *reinterpret_cast<double2*>(dst + j) = make_double2(a[j], a[j + 1]);
          } else {
            if (head) {
              for (int c = blockIdx.x + 1; c < g.grid && unit_lo(g.units, g.grid, c) < rb_hi; ++c) {
                unsigned f;
                do {
                  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(g.flags + c) : "memory");
                } while (f != epoch);
                const double* src = g.P + ((int64_t)c * 128 + col) * TN_BN + j0;
#pragma unroll
                for (int j = 0; j < 32; j += 2) {
                  const double2 pv = *reinterpret_cast<const double2*>(src + j);
                  a[j] += pv.x;
                  a[j + 1] += pv.y;
                }
              }
            }
            if (col < g.Nout) {
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                const int64_t r = ct * TN_BN + j0 + j;
                if (r < g.M) g.C[r * g.ldc + col] = a[j];
              }
            }
          }
        }
        if (cont) {
          __threadfence();
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (et == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(g.flags + blockIdx.x), "r"(epoch) : "memory");
        }
        sub = 0;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acce[b]);
      ++run;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
  }
}

// X (K x Np, FP64, ld ldx) -> Xhi, Xlo (K x N, FP32, row-major, zero-padded columns)
__global__ void prep_split_b(const double* __restrict__ X, int64_t ldx, int64_t K, int Np, int N,
                             float* __restrict__ hi, float* __restrict__ lo, unsigned* epoch_ctr) {
  if (blockIdx.x == 0 && threadIdx.x == 0) ++*epoch_ctr;   // the pass kernel's stream-K epoch (kernels.h)
  const int64_t total = K * N;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e / N;
    const int n = (int)(e - k * N);
    const float x = (n < Np) ? (float)X[k * ldx + n] : 0.0f;
    const float h = tf32_trunc(x);
    hi[e] = h;
    lo[e] = tf32_rna(x - h);
  }
}

// ------------------------------------------------------------------ host side
// 2-D FP32 row-major tensor (rows x cols, ld elements), box {box_cols, box_rows};
// SWIZZLE_128B for K-major use, SWIZZLE_128B_ATOM_32B for MN-major use
static bool make_map(CUtensorMap* m, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_cols,
                     int box_rows, bool mn_major) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                   mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace tf32

namespace tc {
EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}
}  // namespace tc

bool tf32_pass_supported(const void* A, int64_t lda) {
  return ((uintptr_t)A % 16 == 0) && ((lda * 4) % 16 == 0) && tc::get_encode() != nullptr;
}

int tf32_n(int Np) { return (int)round_up(Np, 32); }

size_t tf32_partial_bytes(int Np, int num_sms) {
  // NN: [grid][128][N] partials + drain sums; TN (Q^T A form): [grid][128][256] each
  return 2 * (size_t)num_sms * 128 * (tf32_n(Np) > 256 ? tf32_n(Np) : 256) * sizeof(double);
}

size_t tf32_split_bytes(int64_t K, int Np) { return 2 * (size_t)K * tf32_n(Np) * sizeof(float); }

cudaError_t tf32_pass(const Tf32Call& c, cudaStream_t st) {
  using namespace tf32;
  const int N = tf32_n(c.N);
  if (N > 128 || c.M <= 0 || c.K <= 0) return cudaErrorInvalidValue;
  // 1) panel split into FP32 hi / lo (K x N, row-major)
  float* hi = c.split;
  float* lo = c.split + (size_t)c.K * N;
  {
    int64_t total = c.K * N;
    int blocks = (int)ceil_div(total, 256);
    if (blocks > 148 * 8) blocks = 148 * 8;
    prep_split_b<<<blocks, 256, 0, st>>>(c.B, c.ldb, c.K, c.N, N, hi, lo, c.flags + kEpochSlot);
    ++g_kernel_launches;
  }
  // 2) tensor maps
  CUtensorMap mA, mBh, mBl;
  bool ok;
  if (!c.trans) ok = make_map(&mA, c.A, c.M, c.K, c.lda, 32, BM, false);     // A: M rows x K cols (K-major)
  else ok = make_map(&mA, c.A, c.K, c.M, c.lda, 32, BK, true);               // A: K rows x M cols (MN-major)
  ok = ok && make_map(&mBh, hi, c.K, N, N, 32, BK, true) && make_map(&mBl, lo, c.K, N, N, 32, BK, true);
  if (!ok) return cudaErrorInvalidValue;
  Args g;
  g.C = c.C; g.ldc = c.ldc; g.P = c.P; g.M = c.M; g.K = c.K; g.N = N; g.Nout = c.Nout;
  g.flags = c.flags;
  if (c.flags == nullptr) return cudaErrorInvalidValue;
  g.KT = ceil_div(c.K, BK);
  static const bool tn_qta = [] { const char* e = getenv("RSVD_TF32_TN"); return !(e && e[0] == '0'); }();
  static const bool nn_xta = [] { const char* e = getenv("RSVD_TF32_NN"); return !(e && e[0] == '0'); }();
  if ((c.trans && tn_qta) || (!c.trans && nn_xta)) {
    // C^T = Q^T A (TN) / X^T A^T (NN) with 256-column (row) chunks of A (pass_tf32_tn_kernel)
    if (!c.trans && !make_map(&mA, c.A, c.M, c.K, c.lda, 32, TN_BN, false)) return cudaErrorInvalidValue;
    const int64_t ctiles = ceil_div(c.M, (int64_t)TN_BN);
    g.units = ctiles * g.KT;
    int64_t grid = g.units / 8;
    if (grid < ctiles) grid = ctiles;
    if (grid > c.grid) grid = c.grid;
    if (grid < 1) grid = 1;
    g.grid = (int)grid;
    g.Pacc = c.P + (size_t)c.grid * 128 * TN_BN;
    const size_t smem = (size_t)TN_STAGES * TN_STAGE + 1024;
    cudaError_t e;
    if (c.trans) {
      e = smem_optin(pass_tf32_tn_kernel<false>);
      if (e != cudaSuccess) return e;
      pass_tf32_tn_kernel<false><<<g.grid, THREADS, smem, st>>>(mA, mBh, mBl, g);
    } else {
      e = smem_optin(pass_tf32_tn_kernel<true>);
      if (e != cudaSuccess) return e;
      pass_tf32_tn_kernel<true><<<g.grid, THREADS, smem, st>>>(mA, mBh, mBl, g);
    }
    ++g_kernel_launches;
    return cudaGetLastError();
  }
  const int64_t mblocks = ceil_div(c.M, BM);
  g.units = mblocks * g.KT;
  int64_t grid = g.units / 8;
  if (grid < mblocks) grid = mblocks;
  if (grid > c.grid) grid = c.grid;
  if (grid < 1) grid = 1;
  g.grid = (int)grid;
  g.Pacc = c.P + (size_t)c.grid * BM * N;            // second half of the partial buffer (tf32_partial_bytes)
  const size_t smem = (size_t)STAGES * (2 * A_BYTES + 2 * (N / 32) * B_BOX_BYTES) + 1024;
  cudaError_t e;
  if (!c.trans) {
    e = smem_optin(pass_tf32_kernel<false>);
    if (e != cudaSuccess) return e;
    pass_tf32_kernel<false><<<g.grid, THREADS, smem, st>>>(mA, mBh, mBl, g);
  } else {
    e = smem_optin(pass_tf32_kernel<true>);
    if (e != cudaSuccess) return e;
    pass_tf32_kernel<true><<<g.grid, THREADS, smem, st>>>(mA, mBh, mBl, g);
  }
  ++g_kernel_launches;
  return cudaGetLastError();
}

}  // namespace rsvd
