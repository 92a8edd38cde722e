// tcgen05.mma throughput probe: one CTA per SM issues back-to-back MMAs from
// shared memory (SS mode, K-major SW128) into TMEM; reports MACs/clk/SM.
// kinds: 0 = i8 (s8 x s8 -> s32), 1 = f16 (bf16 -> f32), 2 = tf32, 3 = f8f6f4 (e4m3 -> f32).
#include <cstdio>
#include <cstdint>
#include "../paper_1608_02148_b200/csrc/tc_common.cuh"
using namespace rsvd::tc;
template <int KIND>
__global__ void probe(long long* out, int N, int iters, int a_major, int rot) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = (unsigned char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 196608 / 4; i += blockDim.x) ((uint32_t*)base)[i] = 0x01010101u * (1 + (i % 7));
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
  if (tid == 0) {
    uint32_t cf = KIND == 0 ? 2u : 1u, af = KIND == 0 ? 1u : (KIND == 1 ? 1u : (KIND == 2 ? 2u : 0u));
    const uint32_t idesc = (cf << 4) | (af << 7) | (af << 10) | ((uint32_t)a_major << 15) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
    const uint32_t a = smem_u32(base), b = smem_u32(base + 16384);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint64_t da = rot ? sdesc(a + (i % 6) * 16384, 16, 1024) : sdesc(a, 16, 1024);
      const uint64_t db = rot ? sdesc(b + 81920 + (i % 7) * 8192, 16, 1024) : sdesc(b, 16, 1024);
      if (KIND == 0) asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 1;" ::"r"(tmem), "l"(da), "l"(db), "r"(idesc));
      if (KIND == 1) asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;" ::"r"(tmem), "l"(da), "l"(db), "r"(idesc));
      if (KIND == 2) asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;" ::"r"(tmem), "l"(da), "l"(db), "r"(idesc));
      if (KIND == 3) asm volatile("tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, 1;" ::"r"(tmem), "l"(da), "l"(db), "r"(idesc));
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
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
  const char* names[] = {"i8", "bf16", "tf32", "e4m3"};
  const int kbytes = 32;
  for (int rot = 0; rot < 2; ++rot)
  for (int kind = 0; kind < 1; ++kind)
    for (int am = 0; am < 2; ++am)
      for (int N : {64, 128, 256}) {
        if (kind == 3 && am == 1) continue;
        const int iters = 2000;
        cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(probe<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        for (int rep = 0; rep < 2; ++rep) {
          if (kind == 0) probe<0><<<148, 128, 200 * 1024>>>(out, N, iters, am, rot);
          if (kind == 1) probe<1><<<148, 128, 200 * 1024>>>(out, N, iters, am, rot);
          if (kind == 2) probe<2><<<148, 128, 200 * 1024>>>(out, N, iters, am, rot);
          if (kind == 3) probe<3><<<148, 128, 200 * 1024>>>(out, N, iters, am, rot);
        }
        cudaError_t e = cudaDeviceSynchronize();
        long long c[148]; cudaMemcpy(c, out, sizeof c, cudaMemcpyDeviceToHost);
        const int K = kind == 0 || kind == 3 ? 32 : (kind == 1 ? 16 : 8);
        const double macs = 128.0 * N * K * iters;
        printf("rot %d %-5s a_major %d N %3d: %8.1f cyc/mma  %7.0f MACs/clk/SM  (%s)\n", rot, names[kind], am, N, (double)c[0] / iters,
               macs / c[0], cudaGetErrorString(e));
      }
  return 0;
}
