// tcgen05.mma kind::i8 throughput, cta_group::1 (M = 128, one CTA per SM) vs
// cta_group::2 (M = 256 over a CTA pair in a 2-CTA cluster): back-to-back MMAs
// from shared memory into TMEM; reports MACs/clk/SM.  Not product code.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma_rate2 tools/mma_rate2.cu
#include <cstdio>
#include <cstdint>
#include "../paper_1608_02148_b200/csrc/tc_common.cuh"
using namespace rsvd::tc;

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int G>
__global__ void probe(long long* out, int N, int iters, int mode) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = (unsigned char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 196608 / 4; i += blockDim.x) ((uint32_t*)base)[i] = 0x01010101u * (1 + (i % 7));
  if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  if (warp == 0) {
    if (G == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tb)), "n"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tb)), "n"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  fence_proxy_async();
  tc_fence_before();
  if (G == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tb;
  const bool leader = G == 1 || cta_rank() == 0;
  if (tid == 0 && leader) {
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(G * 128 >> 4) << 24);
    const uint32_t a = smem_u32(base), b = smem_u32(base + 65536);   // A slots 16 KB apart, B slots 32 KB (N <= 128 for 4 slots)
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      // mode 0: both fixed; 1: A and B rotate over 4 slots; 2: only A rotates; 3: only B rotates;
      // 4: GEMM-like, 4 k-steps of 32 B inside each 128 B swizzle row, then the next slot
      const int s = (mode == 4 ? i >> 2 : i) & 3, kk = mode == 4 ? (i & 3) : 0;
      const uint64_t da = sdesc(a + ((mode == 1 || mode == 2 || mode == 4) ? s * 16384 : 0), 16, 1024) + 2 * kk;
      const uint64_t db = sdesc(b + ((mode == 1 || mode == 3 || mode == 4) ? s * 32768 : 0), 16, 1024) + 2 * kk;
      const uint32_t d = tmem + (uint32_t)((i & 1) * N);
      if (G == 1) asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 1;" ::"r"(d), "l"(da), "l"(db), "r"(idesc));
      else asm volatile("tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, 1;" ::"r"(d), "l"(da), "l"(db), "r"(idesc));
    }
    if (G == 1) mma_commit(&bar);
    else
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(smem_u32(&bar)),
                   "h"((uint16_t)3));
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  if (G == 2 && tid == 0 && !leader) mbar_wait(&bar, 0);
  tc_fence_before();
  if (G == 2) cluster_sync(); else __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    if (G == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
    else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
  }
}

int main() {
  long long* out;
  cudaMalloc(&out, 148 * 8);
  cudaMemset(out, 0, 148 * 8);
  cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int G = 1; G <= 2; ++G)
    for (int mode = 0; mode < 5; ++mode)
      for (int N : {64, 128, 256}) {
        const int iters = 4000;
        for (int rep = 0; rep < 2; ++rep) {
          if (G == 1) probe<1><<<148, 128, 200 * 1024>>>(out, N, iters, mode);
          else {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(148);
            cfg.blockDim = dim3(128);
            cfg.dynamicSmemBytes = 200 * 1024;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = 2;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, probe<2>, out, N, iters, mode);
          }
        }
        cudaError_t e = cudaDeviceSynchronize();
        long long c[148];
        cudaMemcpy(c, out, sizeof c, cudaMemcpyDeviceToHost);
        const double macs_sm = 128.0 * N * 32 * iters;   // per SM (a pair does 2x over 2 SMs)
        printf("cta_group::%d mode %d N %3d: %8.1f cyc/mma  %7.0f MACs/clk/SM  (%s)\n", G, mode, N, (double)c[0] / iters, macs_sm / c[0],
               cudaGetErrorString(e));
      }
  return 0;
}
