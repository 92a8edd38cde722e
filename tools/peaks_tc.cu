// Whole-chip tcgen05 tensor peaks for the roofline denominators of bench.py:
// one CTA per SM issues back-to-back cta_group::1 MMAs (M = 128, N = 256, SS
// operands, K-major SW128, data irrelevant) into TMEM for `iters` MMAs; the
// launch is timed with CUDA events (wall clock, all 148 SMs, clocks as the
// driver left them).  kind::i8 (K = 32), kind::tf32 (K = 8), kind::f16 (bf16,
// K = 16).  Prints one JSON object.  Not product code.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/peaks_tc tools/peaks_tc.cu
#include <cstdint>
#include <cstdio>
#include "../paper_1608_02148_b200/csrc/tc_common.cuh"
using namespace rsvd::tc;

// RND: operands are pseudo-random bytes (two different tiles alternating), the
// switching activity of real data: the power-capped sustained rate
template <int KIND, bool RND = false>
__global__ void __launch_bounds__(128, 1) burst(int iters, unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = (unsigned char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 98304 / 4; i += blockDim.x) {
    uint32_t h = 0x3c003c00u;
    if (RND) {
      h = (uint32_t)i * 2654435761u + blockIdx.x * 40503u + 0x9e3779b9u;
      h ^= h >> 15; h *= 2246822519u; h ^= h >> 13; h *= 3266489917u; h ^= h >> 16;
    }
    ((uint32_t*)base)[i] = h;
  }
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
    // D: s32 (i8) or f32; A/B formats: s8 / tf32 (2) / bf16 (1); N = 256, M = 128
    const uint32_t cf = KIND == 0 ? 2u : 1u;
    const uint32_t af = KIND == 0 ? 1u : (KIND == 1 ? 2u : 1u);
    const uint32_t idesc = (cf << 4) | (af << 7) | (af << 10) | ((uint32_t)(256 >> 3) << 17) | (8u << 24);
    const uint64_t da = sdesc(smem_u32(base), 16, 1024), db = sdesc(smem_u32(base + 32768), 16, 1024);
    for (int i = 0; i < iters; ++i) {
      const uint32_t d = tmem + (uint32_t)((i & 1) * 256);
      // RND: alternate between two operand tiles (16 KB further) so consecutive MMAs differ
      const uint64_t off = RND ? (uint64_t)((i & 1) * (16384 >> 4)) : 0;
      if (KIND == 0) asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 1;" ::"r"(d), "l"(da + off), "l"(db + off), "r"(idesc));
      if (KIND == 1) asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;" ::"r"(d), "l"(da), "l"(db), "r"(idesc));
      if (KIND == 2) asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;" ::"r"(d), "l"(da), "l"(db), "r"(idesc));
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

// back-to-back launches for ~secs seconds (clocks settle under the power
// limit): the sustained figure for kernels timed inside long steps
template <int KIND, bool RND = false>
static double run_sustained(int nsm, int iters, double secs) {
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  cudaFuncSetAttribute(burst<KIND, RND>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  burst<KIND, RND><<<nsm, 128, 100 * 1024>>>(iters, sink);
  cudaEventRecord(e0);
  cudaEventSynchronize(e0);
  long long launches = 0;
  float ms = 0.f;
  while (ms < secs * 1e3) {
    for (int r = 0; r < 20; ++r) burst<KIND, RND><<<nsm, 128, 100 * 1024>>>(iters, sink);
    launches += 20;
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  cudaFree(sink);
  const int K = KIND == 0 ? 32 : (KIND == 1 ? 8 : 16);
  return 2.0 * 128 * 256 * K * (double)iters * nsm * launches / (ms * 1e-3) / 1e12;
}

template <int KIND>
static double run(int nsm, int iters) {
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  cudaFuncSetAttribute(burst<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  burst<KIND><<<nsm, 128, 100 * 1024>>>(iters / 10, sink);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best = 1e30;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    burst<KIND><<<nsm, 128, 100 * 1024>>>(iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaFree(sink);
  const int K = KIND == 0 ? 32 : (KIND == 1 ? 8 : 16);
  return 2.0 * 128 * 256 * K * (double)iters * nsm / (best * 1e-3) / 1e12;   // T(FL)OPS
}

int main() {
  int nsm = 0, clk = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 200000;
  const double i8 = run<0>(nsm, iters), tf32 = run<1>(nsm, iters), bf16 = run<2>(nsm, iters);
  const double i8s = run_sustained<0>(nsm, iters / 4, 4.0), tf32s = run_sustained<1>(nsm, iters / 4, 4.0);
  const double i8r = run_sustained<0, true>(nsm, iters / 4, 6.0);
  printf("{\"tcgen05_i8_tops_sustained\": %.1f, \"tcgen05_tf32_tflops_sustained\": %.1f, "
         "\"sustained_how\": \"back-to-back launches for 4 s\", ", i8s, tf32s);
  printf("\"tcgen05_i8_tops_sustained_random\": %.1f, \"sustained_random_how\": \"the same loop on pseudo-random "
         "operand bytes (two tiles alternating), back to back for 6 s: the power-capped rate of real data\", ", i8r);
  printf("\"tcgen05_i8_tops\": %.1f, \"tcgen05_tf32_tflops\": %.1f, \"tcgen05_bf16_tflops\": %.1f, "
         "\"tc_peaks_how\": \"tools/peaks_tc.cu: %d CTAs x back-to-back cta_group::1 M=128 N=256 SS MMAs (%d each), "
         "best of 5 CUDA-event timings, dense\", \"sms\": %d, \"clock_khz_attr\": %d, \"cudaError\": \"%s\"}\n",
         i8, tf32, bf16, nsm, iters, nsm, clk, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
