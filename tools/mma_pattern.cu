// Replays the Ozaki pass MMA pattern (S = 8 slices, Np = 64: per k-step the 36
// (t, u) products batched along N) from shared memory without any loads, to
// time the tensor work per k-step in isolation.  Not product code.
#include <cstdio>
#include <cstdint>
#include "../paper_1608_02148_b200/csrc/tc_common.cuh"
using namespace rsvd::tc;
__global__ void probe(long long* out, int iters) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = (unsigned char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 200 * 1024 / 4; i += blockDim.x) ((uint32_t*)base)[i] = 0x01010101u * (1 + (i % 5));
  if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tb)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tb;
  constexpr int S = 8, N = 64, CMAX = 4, XSL = N * 128;
  if (tid == 0) {
    const uint32_t idesc0 = (2u << 4) | (1u << 7) | (1u << 10) | (8u << 24);
    const uint64_t dx0 = sdesc(smem_u32(base + 5 * 16384), 16, 1024);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int t = 0; t < S; ++t) {
        const uint64_t da0 = sdesc(smem_u32(base + (t % 5) * 16384), 16, 1024);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t da = da0 + (uint64_t)(kk * 2);
#pragma unroll
          for (int u0 = 0; u0 < S - t; u0 += CMAX) {
            const int cnt = (S - t - u0) < CMAX ? (S - t - u0) : CMAX;
            const uint64_t db = dx0 + (uint64_t)((u0 * XSL + kk * 32) >> 4);
            const uint32_t idesc = idesc0 | ((uint32_t)((cnt * N) >> 3) << 17);
            asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 1;" ::"r"(tmem + (uint32_t)((t + u0) * N)), "l"(da), "l"(db), "r"(idesc));
          }
        }
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
  }
}
int main() {
  long long* out; cudaMalloc(&out, 148 * 8);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  const int iters = 200;
  for (int rep = 0; rep < 2; ++rep) probe<<<148, 128, 210 * 1024>>>(out, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long c; cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
  printf("per unit (4 k-steps x 36 products, 48 MMAs): %.0f cycles (%s); 21.4 units/CTA -> %.1f us at 1.965 GHz\n",
         (double)c / iters, cudaGetErrorString(e), (double)c / iters * 21.4 / 1965.0);
  return 0;
}
