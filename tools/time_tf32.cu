// Timing harness for the tcgen05 3xTF32 pass (pass_tf32.cu) at config-4-like
// sizes: A (M x K FP32) filled on device, C = A X and C = A^T X.  Not product code.
#include <cstdio>
#include <cstdlib>
#include "../paper_1608_02148_b200/csrc/pass_tf32.cu"
namespace rsvd { int64_t g_kernel_launches = 0; }
using namespace rsvd;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)
__global__ void fill(float* a, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = (float)((i * 2654435761ull) % 2001) / 1000.0f - 1.0f;
}
__global__ void filld(double* a, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = (double)((i * 40503ull) % 2001) / 1000.0 - 1.0;
}
int main(int argc, char** argv) {
  const int64_t M = argc > 1 ? atol(argv[1]) : 250000, K = argc > 2 ? atol(argv[2]) : 10000;
  const int Np = argc > 3 ? atoi(argv[3]) : 128, reps = argc > 4 ? atoi(argv[4]) : 5;
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float *dA, *split; double *dB, *dC, *dP; unsigned* flags;
  CK(cudaMalloc(&dA, M * K * 4)); fill<<<4096, 256>>>(dA, M * K);
  const int64_t big = M > K ? M : K;
  CK(cudaMalloc(&dB, big * Np * 8)); filld<<<1024, 256>>>(dB, big * Np);
  CK(cudaMalloc(&dC, big * Np * 8)); CK(cudaMalloc(&dP, tf32_partial_bytes(128, nsm)));
  CK(cudaMalloc(&split, tf32_split_bytes(big, Np))); CK(cudaMalloc(&flags, 4096 * 4)); CK(cudaMemset(flags, 0, 4096 * 4));
  unsigned epoch = 0;
  for (int trans = 0; trans < 2; ++trans) {
    Tf32Call t{};
    t.A = dA; t.lda = K; t.trans = trans; t.B = dB; t.ldb = Np; t.C = dC; t.ldc = Np; t.P = dP; t.split = split;
    t.M = trans ? K : M; t.K = trans ? M : K; t.N = Np; t.Nout = Np; t.grid = nsm; t.flags = flags;
    t.epoch = ++epoch; CK(tf32_pass(t, 0)); CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) { t.epoch = ++epoch; tf32_pass(t, 0); }
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
    printf("trans %d: %.3f ms per pass, A %.2f GB -> %.0f GB/s\n", trans, ms, M * K * 4e-9, M * K * 4e-6 / ms);
  }
  return 0;
}
