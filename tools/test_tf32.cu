// Standalone check of the tcgen05 3xTF32 pass kernel against a CPU FP64 reference.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
__device__ double g_dbg[16];
#define TF32_DEBUG_SPLIT if (blockIdx.x == 0 && it == 0) { double sA = 0, sL = 0, sB = 0; \
  for (int q2 = et; q2 < A_BYTES / 4; q2 += 128) { sA += fabs(((float*)stageA(s))[q2]); sL += fabs(((float*)stageAlo(s))[q2]); } \
  for (int q2 = et; q2 < b_bytes / 4; q2 += 128) sB += fabs(((float*)stageBhi(s))[q2]); \
  atomicAdd(&g_dbg[0], sA); atomicAdd(&g_dbg[1], sL); atomicAdd(&g_dbg[2], sB); if (et == 0) g_dbg[3] = (double)tmem; }
#include "../paper_1608_02148_b200/csrc/pass_tf32.cu"
#include "../paper_1608_02148_b200/csrc/gemm_pass.cu"
namespace rsvd { int64_t g_kernel_launches = 0; }
using namespace rsvd;
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); exit(1);}}while(0)
int main(int argc, char** argv) {
  for (int trans = 0; trans < 2; ++trans) {
    const int64_t M = 300, K = 200; const int Np = 48;    // C = op(A) B
    const int64_t arows = trans ? K : M, acols = trans ? M : K;
    std::vector<float> A(arows * acols);
    std::vector<double> B(K * Np), C(M * Np, -7.0), R(M * Np, 0.0);
    srand(1 + trans);
    for (auto& v : A) v = (rand() % 20001) / 10000.0f - 1.0f;
    for (auto& v : B) v = (rand() % 20001) / 10000.0 - 1.0;
    for (int64_t i = 0; i < M; ++i) for (int j = 0; j < Np; ++j) {
      double s = 0; for (int64_t k = 0; k < K; ++k) s += (double)(trans ? A[k * acols + i] : A[i * acols + k]) * (double)(float)B[k * Np + j];
      R[i * Np + j] = s;
    }
    float *dA, *split; double *dB, *dC, *dP;
    CK(cudaMalloc(&dA, A.size() * 4)); CK(cudaMalloc(&dB, B.size() * 8)); CK(cudaMalloc(&dC, C.size() * 8));
    CK(cudaMalloc(&dP, 148 * 2 * 128 * 128 * 8)); CK(cudaMalloc(&split, tf32_split_bytes(K, Np)));
    CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dC, C.data(), C.size() * 8, cudaMemcpyHostToDevice));
    Tf32Call t{};
    t.A = dA; t.lda = acols; t.trans = trans; t.B = dB; t.ldb = Np; t.C = dC; t.ldc = Np; t.P = dP; t.split = split;
    t.M = M; t.K = K; t.N = Np; t.Nout = Np; t.grid = argc > 1 ? atoi(argv[1]) : 148;
    printf("supported %d\n", (int)tf32_pass_supported(dA, acols));
    CK(tf32_pass(t, 0));
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(C.data(), dC, C.size() * 8, cudaMemcpyDeviceToHost));
    { double dbg[16]; cudaMemcpyFromSymbol(dbg, g_dbg, sizeof dbg); printf("debug: |A_hi| %.3f |A_lo| %.3e |B_hi| %.3f tmem %.0f\n", dbg[0], dbg[1], dbg[2], dbg[3]);
      double z[16] = {0}; cudaMemcpyToSymbol(g_dbg, z, sizeof z); }
    { std::vector<float> h(K * 64); CK(cudaMemcpy(h.data(), split, K * 64 * 4, cudaMemcpyDeviceToHost)); double sh = 0; for (auto v : h) sh += fabs(v); printf("debug: |Bhi global| %.3f\n", sh); }
    double emax = 0, rmax = 0; int bad = 0;
    for (int64_t i = 0; i < M * Np; ++i) { emax = fmax(emax, fabs(C[i] - R[i])); rmax = fmax(rmax, fabs(R[i])); if (fabs(C[i]-R[i]) > 1e-3*rmax) ++bad; }
    printf("trans %d: max|C-R| %.3e (max|R| %.3e), bad %d, C[0..3] %f %f %f %f  R[0..3] %f %f %f %f\n", trans, emax, rmax, bad,
           C[0], C[1], C[2], C[3], R[0], R[1], R[2], R[3]);
  }
  return 0;
}
