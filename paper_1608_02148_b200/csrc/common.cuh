// common.cuh -- internal helpers of the B200 rsvd library (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace rsvd {

constexpr int kWarp = 32;

// Programmatic dependent launch: a kernel launched with launch_pdl may start
// while its predecessor on the stream finishes; it waits for the predecessor's
// completion (and memory) before touching any global data, and lets its own
// successor launch early.  Both are no-ops for a normal launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#define CUDA_TRY(x) do { const cudaError_t _e = (x); if (_e != cudaSuccess) return _e; } while (0)
extern int g_pdl;   // 1: launch_pdl sets programmatic stream serialization (RSVD_PDL=0 disables)

// Raise `fn`'s dynamic shared-memory limit to the device's opt-in maximum
// (minus its static shared memory) on the CURRENT device, once per (kernel,
// device); thread-safe (omega.cu).
cudaError_t smem_optin_fn(const void* fn);
template <typename... KArgs>
inline cudaError_t smem_optin(void (*kernel)(KArgs...)) { return smem_optin_fn(reinterpret_cast<const void*>(kernel)); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<Args&&>(args)...);
}

// A launch WITHOUT programmatic stream serialization: for a kernel that
// follows non-kernel stream work (memcpy / memset / cross-stream event waits),
// which griddepcontrol.wait does not cover.  Later PDL kernels then depend on
// this kernel, i.e. on everything before it.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_plain(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = nullptr;
  cfg.numAttrs = 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<Args&&>(args)...);
}

// launch_pdl with a thread-block cluster of cx CTAs along x
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_cluster(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                      unsigned cx, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = cx;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<Args&&>(args)...);
}

// Device-side predicate on a status word (the call's flags): a predicated
// kernel returns at entry (after releasing its dependents) unless
// ((*flag & mask) != 0) == want.  flag == nullptr: always run.  Used for the
// CholeskyQR -> TSQR breakdown fallback, decided on the device so that a call
// never waits on the host (api.cu orth()).
struct Pred { const int* flag; int mask; int want; };
__device__ __forceinline__ bool pred_skip(const Pred p) {
  return p.flag != nullptr && (((*reinterpret_cast<const volatile int*>(p.flag) & p.mask) != 0) != (p.want != 0));
}

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum for blockDim.x == nthreads (multiple of 32); `scratch` holds
// >= 32 doubles.  All threads receive the result.
__device__ __forceinline__ double block_sum(double v, double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  double t = (lane < nw) ? scratch[lane] : 0.0;
  t = warp_sum(t);
  return t;
}

// cp.async with zero-fill: copies `src_bytes` (0..16) from global, fills the
// rest of the 16-byte (or 8-byte) destination with zeros.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, int src_bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// FP64 tensor-core MMA, D(8x8) += A(8x4, row) * B(4x8, col); lowers to SASS
// DMMA.8x8x4 on sm_100a (tcgen05 has no f64 kind).
// Fragments: a = A[g][t], b = B[t][g], c = {C[g][2t], C[g][2t+1]},
// g = lane/4, t = lane%4.
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

}  // namespace rsvd
