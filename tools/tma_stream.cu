// Microbenchmark: how fast can one persistent CTA per SM stream the Ozaki
// pass operands (A slices + X slices) into shared memory, without any MMA?
// Compares the tensor-map boxes the pass uses (64 B / 128 B box rows) with
// plain bulk copies of pre-arranged contiguous unit images.  Not product code.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lcuda -o tools/tma_stream tools/tma_stream.cu
#include <cuda.h>
#include <cstdio>
#include <cstdlib>
#include "../paper_1608_02148_b200/csrc/tc_common.cuh"
namespace rsvd { namespace tc {
EncodeTiledFn get_encode() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess) return reinterpret_cast<EncodeTiledFn>(p);
  return nullptr;
}
} }
using namespace rsvd::tc;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ void tma_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

struct P {
  const int8_t* A; const int8_t* X; int64_t KB, units; int mode, nbuf, piece;
  uint32_t abytes, xbytes;   // per unit
  int hold;                  // consumer cycles per unit (emulated MMA time)
};

__global__ void __launch_bounds__(64, 1) stream_kernel(const __grid_constant__ CUtensorMap mA,
                                                       const __grid_constant__ CUtensorMap mX, P p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[8], empty[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t per = (p.units + gridDim.x - 1) / gridDim.x;
  const int64_t u_lo = blockIdx.x * per, u_hi = min(p.units, u_lo + per);
  const uint32_t ub_bytes = (p.abytes + p.xbytes + 1023) / 1024 * 1024;
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.nbuf; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0 && lane == 0) {
    for (int64_t it = 0; it < u_hi - u_lo; ++it) {
      const int64_t u = u_lo + it, mb = u / p.KB, kb = u - mb * p.KB;
      const int s = (int)(it % p.nbuf);
      unsigned char* buf = base + s * ub_bytes;
      mbar_wait(&empty[s], (uint32_t)(((it / p.nbuf) & 1) ^ 1));
      mbar_expect_tx(&full[s], p.abytes + p.xbytes);
      if (p.mode == 0) {          // NN tensor boxes: 8 x {64 B x 128 rows} + 8 x {64 B x 64 rows}
        for (int t = 0; t < 8; ++t) tma_4d(buf + t * 8192, &mA, (int)((kb & 1) * 64), t, (int)(kb >> 1), (int)(mb * 128), &full[s]);
        for (int t = 0; t < 8; ++t) tma_2d(buf + 65536 + t * 4096, &mX, (int)(kb * 64), t * 64, &full[s]);
      } else if (p.mode == 1) {   // TN tensor boxes: 8 x {128 B x 64 rows} + X
        for (int t = 0; t < 8; ++t) tma_4d(buf + t * 8192, &mA, 0, t, (int)mb, (int)(kb * 64), &full[s]);
        for (int t = 0; t < 8; ++t) tma_2d(buf + 65536 + t * 4096, &mX, (int)((kb % 80) * 64), t * 64, &full[s]);
      } else {                    // bulk copies of the contiguous unit image, in `piece`-byte chunks
        const int8_t* a = p.A + u * (int64_t)p.abytes;
        for (uint32_t o = 0; o < p.abytes; o += p.piece) bulk(buf + o, a + o, p.piece, &full[s]);
        const int8_t* x = p.X + kb * (int64_t)p.xbytes;
        for (uint32_t o = 0; o < p.xbytes; o += p.piece) bulk(buf + p.abytes + o, x + o, min((uint32_t)p.piece, p.xbytes - o), &full[s]);
      }
    }
  } else if (warp == 1 && lane == 0) {
    for (int64_t it = 0; it < u_hi - u_lo; ++it) {
      const int s = (int)(it % p.nbuf);
      mbar_wait(&full[s], (uint32_t)((it / p.nbuf) & 1));
      const long long t0 = clock64();
      while (clock64() - t0 < p.hold) {}
      mbar_arrive(&empty[s]);
    }
  }
  __syncthreads();
}

int main(int argc, char** argv) {
  const int64_t rows = argc > 1 ? atol(argv[1]) : 10000, nblk = argc > 2 ? atol(argv[2]) : 40, S = 8;   // cfg2 default
  const int only = argc > 3 ? atoi(argv[3]) : -1;
  const int64_t abytes_total = rows * nblk * S * 128;         // 410 MB
  int8_t *A, *X;
  CK(cudaMalloc(&A, abytes_total + (1 << 20)));
  CK(cudaMalloc(&X, 8 * 64 * 5120 + (1 << 20)));
  CK(cudaMemset(A, 1, abytes_total)); CK(cudaMemset(X, 1, 8 * 64 * 5120));
  EncodeTiledFn enc = get_encode();
  CUtensorMap mA_nn, mA_tn, mX;
  {
    cuuint64_t dims[4] = {128, (cuuint64_t)S, (cuuint64_t)nblk, (cuuint64_t)rows};
    cuuint64_t strides[3] = {128, (cuuint64_t)(128 * S), (cuuint64_t)(128 * S * nblk)};
    cuuint32_t es[4] = {1, 1, 1, 1};
    cuuint32_t bnn[4] = {64, 1, 1, 128}, btn[4] = {128, 1, 1, 64};
    if (enc(&mA_nn, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, A, dims, strides, bnn, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ||
        enc(&mA_tn, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, A, dims, strides, btn, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)) { printf("enc A\n"); return 1; }
    cuuint64_t xd[2] = {5120, 8 * 64}; cuuint64_t xs[1] = {5120}; cuuint32_t xb[2] = {64, 64}; cuuint32_t xe[2] = {1, 1};
    if (enc(&mX, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, X, xd, xs, xb, xe, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)) { printf("enc X\n"); return 1; }
  }
  CK(cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  struct Cfg { const char* name; int mode, nbuf, piece; uint32_t ab, xb; int hold; };
  const Cfg cfgs[] = {
      {"NN boxes 2 x 96 KB hold 2368", 0, 2, 0, 65536, 32768, 2368},
      {"NN boxes 2 x 96 KB hold 1800", 0, 2, 0, 65536, 32768, 1800},
      {"bulk16K 2 x 96 KB hold 2368", 2, 2, 16384, 65536, 32768, 2368},
      {"bulk16K 4 x 48 KB hold 1184", 2, 4, 16384, 32768, 16384, 1184},
      {"bulk8K 4 x 48 KB hold 1184", 2, 4, 8192, 32768, 16384, 1184},
      {"bulk16K 4 x 48 KB hold 1000", 2, 4, 16384, 32768, 16384, 1000},
      {"bulk8K 8 x 24 KB hold 592", 2, 8, 8192, 16384, 8192, 592},
      {"bulk14K 2 x 84 KB hold 1842 (7 slices u8)", 2, 2, 14336, 57344, 28672, 1842},
      {"bulk7K 4 x 42 KB hold 921 (7 slices u8)", 2, 4, 7168, 28672, 14336, 921},
      {"NN tensor boxes, 2 x 96 KB", 0, 2, 0, 65536, 32768, 0},
      {"TN tensor boxes, 2 x 96 KB", 1, 2, 0, 65536, 32768, 0},
      {"bulk 64K+32K pieces, 2 x 96 KB", 2, 2, 65536, 65536, 32768, 0},
      {"bulk 16K pieces, 2 x 96 KB", 2, 2, 16384, 65536, 32768, 0},
      {"bulk 4K pieces, 2 x 96 KB", 2, 2, 4096, 65536, 32768, 0},
      {"bulk 4K pieces, 4 x 48 KB", 2, 4, 4096, 32768, 16384, 0},
      {"bulk 16K pieces, 4 x 48 KB", 2, 4, 16384, 32768, 16384, 0},
      {"bulk 2K pieces, 4 x 48 KB", 2, 4, 2048, 32768, 16384, 0},
      {"bulk 4K pieces, 3 x 64 KB (A 48K + X 16K)", 2, 3, 4096, 49152, 16384, 0},
  };
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int ci = -1;
  for (const Cfg& c : cfgs) {
    ++ci;
    if (only >= 0 && (only & (1 << ci)) == 0) continue;
    P p{};
    p.A = A; p.X = X; p.mode = c.mode; p.nbuf = c.nbuf; p.piece = c.piece; p.abytes = c.ab; p.xbytes = c.xb; p.hold = c.hold;
    const int64_t units = abytes_total / c.ab;
    p.KB = c.mode == 0 ? 2 * nblk : c.mode == 1 ? rows / 64 : (8 * 64 * 5120) / c.xb;   // k-blocks per output block
    p.units = c.mode == 1 ? nblk * (rows / 64) : units;
    const uint32_t ub = (c.ab + c.xb + 1023) / 1024 * 1024;
    const size_t smem = (size_t)c.nbuf * ub + 1024;
    const CUtensorMap* ma = c.mode == 1 ? &mA_tn : &mA_nn;
    stream_kernel<<<148, 64, smem>>>(*ma, mX, p);
    CK(cudaDeviceSynchronize());
    const int reps = 20;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) stream_kernel<<<148, 64, smem>>>(*ma, mX, p);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
    printf("%-44s units %6lld  %7.1f us  A %6.0f GB/s  A+X %6.0f GB/s\n", c.name, (long long)p.units, ms * 1e3,
           p.units * (double)c.ab / ms / 1e6, p.units * (double)(c.ab + c.xb) / ms / 1e6);
  }
  return 0;
}
