// tcgen05 kind::i8 issue rates by operand source and N: back-to-back
// cta_group::1 MMAs (M = 128, K = 32) with both operands in shared memory (SS)
// or A in TMEM (TS), one CTA per SM, CUDA-event timed.  Decides whether the
// Ozaki pass's N = 64 MMAs are limited by shared-memory operand reads.  Not product code.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma_ts tools/mma_ts.cu
#include <cstdint>
#include <cstdio>
#include "../paper_1608_02148_b200/csrc/tc_common.cuh"
using namespace rsvd::tc;

template <int TS, int N, int M = 128>
__global__ void __launch_bounds__(128, 1) burst(int iters, unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = (unsigned char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 65536 / 4; i += blockDim.x) ((uint32_t*)base)[i] = 0x01010101u;
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
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const uint64_t da = sdesc(smem_u32(base), 16, 1024), db = sdesc(smem_u32(base + 16384), 16, 1024);
    const uint32_t ta = tmem + 448;                 // A operand columns (8 x 32 bit = 32 int8 per lane)
    for (int i = 0; i < iters; ++i) {
      const uint32_t d = tmem + (uint32_t)((i % (N <= 64 ? 7 : (N <= 128 ? 3 : 1))) * N);
      if (TS) asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, 1;" ::"r"(d), "r"(ta), "l"(db), "r"(idesc));
      else asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 1;" ::"r"(d), "l"(da), "l"(db), "r"(idesc));
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

template <int TS, int N, int M = 128>
static void run(int nsm, int iters) {
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  cudaFuncSetAttribute(burst<TS, N, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  burst<TS, N, M><<<nsm, 128, 100 * 1024>>>(iters / 10, sink);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    burst<TS, N, M><<<nsm, 128, 100 * 1024>>>(iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaFree(sink);
  const double tops = 2.0 * M * N * 32 * (double)iters * nsm / (best * 1e-3) / 1e12;
  const double cyc = best * 1e-3 * 1.965e9 / iters;
  printf("{\"operands\": \"%s\", \"M\": %d, \"N\": %d, \"K\": 32, \"tops\": %.1f, \"cycles_per_mma\": %.2f, \"err\": \"%s\"}\n",
         TS ? "TS (A in TMEM)" : "SS", M, N, tops, cyc, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 200000;
  run<0, 64>(nsm, iters);
  run<0, 128>(nsm, iters);
  run<0, 256>(nsm, iters);
  run<1, 64>(nsm, iters);
  run<1, 128>(nsm, iters);
  run<0, 64, 64>(nsm, iters);
  run<0, 128, 64>(nsm, iters);
  run<0, 256, 64>(nsm, iters);
  return 0;
}
