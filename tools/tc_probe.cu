// Minimal tcgen05 probes: TMEM st/ld roundtrip; one kind::tf32 / kind::f16 MMA on constant operands.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include "../paper_1608_02148_b200/csrc/common.cuh"
#include "../paper_1608_02148_b200/csrc/kernels.h"
namespace rsvd { int64_t g_kernel_launches = 0; cudaError_t gemm_streamk_fixup_launch(double*, int64_t, double*, int64_t, int, int, int64_t, int64_t, int, cudaStream_t) { return cudaSuccess; } }
#include "../paper_1608_02148_b200/csrc/pass_tf32.cu"
using namespace rsvd::tf32;
__device__ __forceinline__ uint64_t sdesc2(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}
// mode: 0 = st/ld roundtrip, 1 = tf32 MMA, 2 = f16(bf16) MMA
__global__ void probe(float* out, int mode, uint32_t layout, uint32_t lbo, uint32_t sbo, int bmaj, int n) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = (unsigned char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  float* A = (float*)base;
  float* B = (float*)(base + 16384);
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (mode == 2) {
    __nv_bfloat16* Ab = (__nv_bfloat16*)A; __nv_bfloat16* Bb = (__nv_bfloat16*)B;
    for (int i = tid; i < 8192; i += blockDim.x) { Ab[i] = __float2bfloat16(1.0f); Bb[i] = __float2bfloat16(1.0f); }
  } else {
    for (int i = tid; i < 4096; i += blockDim.x) { A[i] = 1.0f; B[i] = 1.0f; }
  }
  if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tb)), "n"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tb;
  if (mode == 0) {
    if (warp < 4) {
      uint32_t v[32];
      for (int j = 0; j < 32; ++j) v[j] = __float_as_uint((float)(1000 * (32 * warp + lane) + j));
      asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%32], {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                   "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31};"
                   :: "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
                      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
                      "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
                      "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]),
                      "r"(tmem + ((uint32_t)(32 * warp) << 16)));
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
  } else if (tid == 32) {
    uint32_t idesc;
    if (mode == 1) idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)bmaj << 16) | ((uint32_t)(n >> 3) << 17) | (8u << 24);
    else idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)bmaj << 16) | ((uint32_t)(n >> 3) << 17) | (8u << 24);
    uint64_t da = sdesc2(smem_u32(A), lbo, sbo, layout), db = sdesc2(smem_u32(B), lbo, sbo, layout);
    if (mode == 1) {
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                   ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(0));
    } else {
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                   ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(0));
    }
    mma_commit(&bar);
  }
  if (mode != 0) mbar_wait(&bar, 0);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp < 4) {
    uint32_t v[32];
    TMEM_LD32(tmem + ((uint32_t)(32 * warp) << 16), v);
    TMEM_WAIT_LD(v);
    for (int j = 0; j < 32; ++j) out[(32 * warp + lane) * 32 + j] = __uint_as_float(v[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(128)); }
}
int main() {
  float* out; cudaMalloc(&out, 128 * 32 * 4);
  static float h[128 * 32];
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  struct Cfg { int mode; uint32_t layout, lbo, sbo; int bmaj; const char* name; };
  Cfg cfgs[] = {{0, 0, 0, 0, 0, "st/ld roundtrip"},
                {1, 2, 16, 1024, 0, "tf32 K-major SW128 both"},
                {1, 0, 128, 256, 0, "tf32 K-major no-swizzle"},
                {1, 1, 4096, 512, 1, "tf32 B MN-major BASE32B"},
                {2, 2, 16, 1024, 0, "bf16 K-major SW128 both"}};
  for (auto& c : cfgs) {
    cudaMemset(out, 0, sizeof h);
    probe<<<1, 256, 40000>>>(out, c.mode, c.layout, c.lbo, c.sbo, c.bmaj, 64);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
    printf("%-30s err=%s D[0][0..3] %g %g %g %g  D[37][5] %g D[127][31] %g\n", c.name, cudaGetErrorString(e), h[0], h[1], h[2], h[3], h[37 * 32 + 5], h[127 * 32 + 31]);
  }
  return 0;
}
