// omega.cu -- K1: the random test matrix Omega (n x l) on the device.
//
// Paper: Gaussian N(0,1), uniform U(-1,1) or Rademacher +-1 entries
// (§2.3; Alg. 4 step 2 "Omega = rnorm(n, l)").
// Counter spec (reading R1, shared with the oracle by specification
// only): entry (i, j) -> e = j*n + i; Philox4x32-10 with counter
// (lo e, hi e, lo stream, hi stream) and key (lo seed, hi seed);
// a = w1:w0, b = w3:w2; U01(x) = (2 (x >> 12) + 1) 2^-53;
// normal = sqrt(-2 ln U01(a)) cos(2 pi U01(b)); unif = 2 U01(a) - 1;
// rademacher = +1 if a >> 63 == 0 else -1.
// Integer work only (one Philox per entry); <= 1.2 M entries for the configs,
// so this is a few microseconds and L2-resident.  Output row-major, ldo >= l;
// columns [l, ncols_zero) are zero-filled (the GEMM N padding).
#include <mutex>
#include <set>
#include <utility>

#include "common.cuh"
#include "kernels.h"

namespace rsvd {

std::atomic<int64_t> g_kernel_launches{0};

cudaError_t smem_optin_fn(const void* fn) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({fn, dev})) return cudaSuccess;
  cudaFuncAttributes fa;
  e = cudaFuncGetAttributes(&fa, fn);
  if (e != cudaSuccess) return e;
  int optin = 0;
  e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes);
  if (e == cudaSuccess) done.insert({fn, dev});
  return e;
}
int g_pdl = [] { const char* e = getenv("RSVD_PDL"); return (e && e[0] == '0') ? 0 : 1; }();

__device__ __forceinline__ uint4 philox_round(uint4 c, uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
  const uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
  return make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
}

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    c = philox_round(c, k0, k1);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

__device__ __forceinline__ double u01(uint64_t x) {
  return ((double)(x >> 12) * 2.0 + 1.0) * 0x1.0p-53;
}

template <typename TO>
__global__ void omega_kernel(int64_t n, int64_t l, int64_t ldo, int64_t ncz, int sdist, uint64_t seed,
                             uint64_t stream, bool f32_round, TO* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int64_t total = n * ncz;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / ncz, j = t % ncz;
    double v = 0.0;
    if (j < l) {
      const uint64_t e = (uint64_t)j * (uint64_t)n + (uint64_t)i;
      const uint4 w = philox4x32_10(
          make_uint4((uint32_t)e, (uint32_t)(e >> 32), (uint32_t)stream, (uint32_t)(stream >> 32)),
          (uint32_t)seed, (uint32_t)(seed >> 32));
      const uint64_t a = ((uint64_t)w.y << 32) | w.x;
      const uint64_t b = ((uint64_t)w.w << 32) | w.z;
      if (sdist == 0) v = sqrt(-2.0 * log(u01(a))) * cos(6.283185307179586 * u01(b));
      else if (sdist == 1) v = 2.0 * u01(a) - 1.0;
      else v = (a >> 63) == 0 ? 1.0 : -1.0;
      if (f32_round) v = (double)(float)v;
    }
    out[i * ldo + j] = (TO)v;
  }
}

cudaError_t launch_omega(int64_t n, int64_t l, int64_t ldo, int64_t ncols_zero, int sdist, uint64_t seed,
                         uint64_t stream, bool f32_round, bool out_f32, void* out, cudaStream_t st) {
  if (ncols_zero < l) ncols_zero = l;
  const int64_t total = n * ncols_zero;
  int blocks = (int)ceil_div(total, 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  cudaError_t e;
  if (out_f32)
    e = launch_pdl(omega_kernel<float>, dim3(blocks), dim3(256), 0, st, n, l, ldo, ncols_zero, sdist, seed, stream,
                   f32_round, static_cast<float*>(out));
  else
    e = launch_pdl(omega_kernel<double>, dim3(blocks), dim3(256), 0, st, n, l, ldo, ncols_zero, sdist, seed, stream,
                   f32_round, static_cast<double*>(out));
  ++g_kernel_launches;
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace rsvd
