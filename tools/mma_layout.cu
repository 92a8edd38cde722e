// tcgen05 kind::i8 issue rate by operand smem layout (K-major SW128 / SW64 /
// SW32, A MN-major SW128 as in the TN pass) and N, back-to-back M = 128, K =
// 32 MMAs, one CTA per SM; two k-steps per 64-byte row as in the Ozaki pass.
// Decides whether the pass's SW64 operand tiles slow the tensor pipe.  Not product code.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma_layout tools/mma_layout.cu
#include <cstdint>
#include <cstdio>
#include "../paper_1608_02148_b200/csrc/tc_common.cuh"
using namespace rsvd::tc;

// LA / LB: 0 = K-major SW128, 1 = K-major SW64, 2 = K-major SW32, 3 = MN-major SW128 (A only)
template <int LA, int LB, int N>
__global__ void __launch_bounds__(128, 1) burst(int iters, unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = (unsigned char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 98304 / 4; i += blockDim.x) ((uint32_t*)base)[i] = 0x01010101u;
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
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((LA == 3 ? 1u : 0u) << 15) |
                           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    auto lay = [](int L) { return L == 1 ? LAYOUT_SW64 : L == 2 ? LAYOUT_SW32 : LAYOUT_SW128; };
    auto sbo = [](int L) { return L == 1 ? 512u : L == 2 ? 256u : 1024u; };
    const uint64_t da0 = sdesc(smem_u32(base), 16, sbo(LA), lay(LA));
    const uint64_t db0 = sdesc(smem_u32(base + 32768), 16, sbo(LB), lay(LB));
    for (int i = 0; i < iters; ++i) {
      const int kk = i & 1;                                        // two k-steps of 32 in a 64-byte row
      const uint64_t da = da0 + (uint64_t)(LA == 3 ? kk * 256 : kk * 2);
      const uint64_t db = db0 + (uint64_t)(kk * 2);
      const uint32_t d = tmem + (uint32_t)(((i >> 1) % (N <= 64 ? 7 : (N <= 128 ? 3 : 1))) * N);
      asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 1;" ::"r"(d), "l"(da), "l"(db), "r"(idesc));
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    if (blockIdx.x == 0) *sink = (unsigned long long)iters;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
  }
}

template <int LA, int LB, int N>
static void run(int nsm, int iters) {
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  cudaFuncSetAttribute(burst<LA, LB, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  burst<LA, LB, N><<<nsm, 128, 100 * 1024>>>(iters / 10, sink);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    burst<LA, LB, N><<<nsm, 128, 100 * 1024>>>(iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaFree(sink);
  const char* nm[] = {"K-SW128", "K-SW64", "K-SW32", "MN-SW128"};
  const double cyc = best * 1e-3 * 1.965e9 / iters;
  printf("A %-8s B %-8s N %3d: %.1f cycles per MMA (at 1965 MHz)  %s\n", nm[LA], nm[LB], N, cyc,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 200000;
  run<0, 0, 64>(nsm, iters); run<0, 0, 128>(nsm, iters); run<0, 0, 192>(nsm, iters); run<0, 0, 256>(nsm, iters);
  run<1, 1, 64>(nsm, iters); run<1, 1, 128>(nsm, iters); run<1, 1, 192>(nsm, iters); run<1, 1, 256>(nsm, iters);
  run<3, 1, 64>(nsm, iters); run<3, 1, 128>(nsm, iters); run<3, 1, 192>(nsm, iters); run<3, 1, 256>(nsm, iters);
  run<2, 2, 64>(nsm, iters); run<2, 2, 128>(nsm, iters); run<2, 2, 256>(nsm, iters);
  run<3, 0, 128>(nsm, iters); run<3, 0, 256>(nsm, iters);
  return 0;
}
