// Replays the Ozaki pass MMA pattern (S = 7 slices, Np = 64: per 32-k step the 28
// (t, u) products batched along N into 10 MMAs) from shared memory without any loads, to
// time the tensor work per k-step in isolation.  Not product code.
#include <cstdio>
#include <cstdint>
#include "../paper_1608_02148_b200/csrc/tc_common.cuh"
using namespace rsvd::tc;
__global__ void probe(long long* out, int iters, int mode) {
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
  // mode 0: NN (A K-major SW64, 64 B rows); 1: TN (A MN-major SW128); 2: A K-major SW128 (128 B rows, first 64 B used)
  constexpr int S = 7, N = 64, CMAX = 4, BKU = 64, XSL = N * BKU, A_UT = 128 * BKU;
  if (tid == 0) {
    const uint32_t idesc0 = (2u << 4) | (1u << 10) | ((mode == 1 ? 1u : 0u) << 15) | (8u << 24);
    const uint32_t ua = smem_u32(base);
    const uint64_t dx0 = sdesc(ua + S * A_UT, 16, 512, LAYOUT_SW64);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t ub = ua + (i & 1) * 0;   // same buffer
#pragma unroll
      for (int t = 0; t < S; ++t) {
        const uint64_t da0 = mode == 1 ? sdesc(ub + t * A_UT, 16, 1024, LAYOUT_SW128)
                           : mode == 0 ? sdesc(ub + t * A_UT, 16, 512, LAYOUT_SW64) : sdesc(ub + (t & 3) * 16384, 16, 1024, LAYOUT_SW128);
#pragma unroll
        for (int kk = 0; kk < BKU / 32; ++kk) {
          const uint64_t da = da0 + (uint64_t)(mode == 1 ? kk * 256 : kk * 2);
#pragma unroll
          for (int u0 = 0; u0 < S - t; u0 += CMAX) {
            const int cnt = (S - t - u0) < CMAX ? (S - t - u0) : CMAX;
            const uint64_t db = dx0 + (uint64_t)((u0 * XSL + kk * 32) >> 4);
            const uint32_t idesc = idesc0 | ((t == 0 ? 1u : 0u) << 7) | ((uint32_t)((cnt * N) >> 3) << 17);
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
  const int iters = 400;
  const char* names[] = {"NN  A K-major SW64 ", "TN  A MN-major SW128", "A K-major SW128    "};
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) probe<<<148, 128, 210 * 1024>>>(out, iters, mode);
    cudaError_t e = cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
    printf("%s per 64-k unit (2 k-steps x 28 products, 20 MMAs): %.0f cycles (%s); model max(79, N/2) = 2040\n", names[mode],
           (double)c / iters, cudaGetErrorString(e));
  }
  return 0;
}
