// Microbenchmark + self-check of the CholeskyQR panel kernels (cholqr.cu):
// gram (partial + reduce), chol_aug, panel_apply.  Not product code.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude -o tools/bench_cholqr tools/bench_cholqr.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
__device__ long long g_cq[8];
__device__ long long g_cq_last;
#define CQ_PROBE_OFF(slot) if ((threadIdx.x & 31) == 0) { long long _t = clock64(); atomicAdd((unsigned long long*)&g_cq[slot], (unsigned long long)(_t - g_cq_last)); g_cq_last = _t; }
__device__ long long g_cb[8];
#define CB_PROBE_DECL long long _cbt[6] = {0, 0, 0, 0, 0, 0}; long long _cbl = clock64(); long long _cb0 = _cbl;
#define CB_PROBE(slot) if (threadIdx.x == 0) { long long _t = clock64(); _cbt[slot] += _t - _cbl; _cbl = _t; }
#define CB_PROBE_OUT if (threadIdx.x == 0) { for (int q = 0; q < 5; ++q) atomicAdd((unsigned long long*)&g_cb[q], (unsigned long long)_cbt[q]); atomicAdd((unsigned long long*)&g_cb[5], (unsigned long long)(clock64() - _cb0)); }
#include "../paper_1608_02148_b200/csrc/cholqr.cu"
namespace rsvd { std::atomic<int64_t> g_kernel_launches{0}; int g_pdl = 1; cudaError_t smem_optin_fn(const void* fn) { cudaFuncAttributes a; cudaError_t e = cudaFuncGetAttributes(&a, fn); if (e != cudaSuccess) return e; int o = 0; cudaDeviceGetAttribute(&o, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0); return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, o - (int)a.sharedSizeBytes); } }
using namespace rsvd;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__global__ void clk_probe(long long* out) {
  long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  long long c0 = clock64();
  while (clock64() - c0 < 2000000) {}
  long long c1 = clock64();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  out[0] = c1 - c0; out[1] = t1 - t0;
}
// cycles per chol_aug step: clock64 around the kernel body is not available from
// outside, so time one launch of a 1-CTA kernel in cycles via clk_probe's MHz.
template <typename F> float timeit(F f, int reps) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); CK(cudaDeviceSynchronize());
  cudaEventRecord(a); for (int r = 0; r < reps; ++r) f(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); CK(cudaGetLastError()); return ms * 1000.f / reps;
}

int main(int argc, char** argv) {
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  const int reps = argc > 2 ? atoi(argv[2]) : 20;
  int ci = -1;
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int* flag; CK(cudaMalloc(&flag, 64));
  struct C { int64_t rows; int l; };
  for (C c : {C{1000, 20}, C{10000, 60}, C{5000, 60}, C{100000, 30}, C{200000, 120}, C{1000000, 120}}) {
    ++ci;
    if (only >= 0 && ci != only) continue;
    const int l = c.l, Np = (l + 15) / 16 * 16;
    const int64_t rows = c.rows;
    std::vector<double> S(rows * Np, 0.0);
    srand(7);
    for (int64_t r = 0; r < rows; ++r)
      for (int j = 0; j < l; ++j) S[r * Np + j] = ((rand() % 20001) / 10000.0 - 1.0) * std::exp(-j / 20.0) + (j == 0 ? 0.5 : 0.0);
    double *dS, *dQ, *part, *G, *R, *Ri;
    CK(cudaMalloc(&dS, rows * Np * 8)); CK(cudaMalloc(&dQ, rows * Np * 8));
    CK(cudaMalloc(&part, gram_partial_bytes(Np, nsm))); CK(cudaMalloc(&G, Np * Np * 8));
    CK(cudaMalloc(&R, Np * Np * 8)); CK(cudaMalloc(&Ri, Np * Np * 8));
    CK(cudaMemcpy(dS, S.data(), rows * Np * 8, cudaMemcpyHostToDevice));
    CK(cudaMemset(flag, 0, 64));
    float tg = timeit([&] { launch_gram(dS, Np, rows, Np, part, G, Np, nsm, 0); }, reps);
    {
      long long* d; cudaMalloc(&d, 16); long long h[2];
      clk_probe<<<1, 32>>>(d); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("  [clock during probe: %.0f MHz]\n", 1000.0 * h[0] / h[1]); cudaFree(d);
    }
    {
      long long z[8] = {0}; cudaMemcpyToSymbol(g_cb, z, sizeof z);
      timeit([&] { launch_chol_aug(G, Np, l, Np, R, Ri, flag, 1, 0); }, reps);
      long long pr[8]; cudaMemcpyFromSymbol(pr, g_cb, sizeof pr);
      const double n = reps + 1;
      printf("    blocked cycles: init+diag0 %.0f panel %.0f trailing+diag %.0f (tail %.0f) out %.0f | total in-kernel %.0f\n", pr[0] / n, pr[1] / n, pr[2] / n, pr[3] / n, pr[4] / n, pr[5] / n);
    }
    float tc = timeit([&] { launch_chol_aug(G, Np, l, Np, R, Ri, flag, 1, 0); }, reps);
    {
      long long pr[8]; cudaMemcpyFromSymbol(pr, g_cq, sizeof pr); long long z[8] = {0}; cudaMemcpyToSymbol(g_cq, z, sizeof z);
      const double st = (double)(reps + 1) * l;
      printf("  chol_aug cycles/step (look-ahead warp): barrier->row k+1 updated %.0f  pivot+publish %.0f  rest of update %.0f  -> barrier %.0f\n", pr[0] / st, pr[1] / st, pr[2] / st, pr[3] / st);
    }
    float ta = timeit([&] { launch_panel_apply(dS, Np, rows, Np, Ri, Np, dQ, Np, Np, true, nsm, 0); }, reps);
    CK(cudaDeviceSynchronize());
    int fl; CK(cudaMemcpy(&fl, flag, 4, cudaMemcpyDeviceToHost));
    // checks: G vs host Gram (sampled), R R^-1 = I, Q^T Q = I, Q R = S (sampled rows)
    std::vector<double> hG(Np * Np), hR(Np * Np), hRi(Np * Np), hQ(rows * Np);
    CK(cudaMemcpy(hG.data(), G, Np * Np * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hR.data(), R, Np * Np * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hRi.data(), Ri, Np * Np * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hQ.data(), dQ, rows * Np * 8, cudaMemcpyDeviceToHost));
    double eg = 0, gmax = 0;
    for (int i = 0; i < l; i += 7) for (int j = 0; j < l; j += 5) {
      double s = 0; for (int64_t r = 0; r < rows; ++r) s += S[r * Np + i] * S[r * Np + j];
      eg = std::fmax(eg, std::fabs(s - hG[i * Np + j])); gmax = std::fmax(gmax, std::fabs(s));
    }
    double ei = 0;
    for (int i = 0; i < Np; ++i) for (int j = 0; j < Np; ++j) {
      double s = 0; for (int k = 0; k < Np; ++k) s += hR[i * Np + k] * hRi[k * Np + j];
      ei = std::fmax(ei, std::fabs(s - ((i == j && i < l) ? 1.0 : 0.0)));
    }
    double eo = 0;
    for (int i = 0; i < l; ++i) for (int j = i; j < l; ++j) {
      double s = 0; for (int64_t r = 0; r < rows; ++r) s += hQ[r * Np + i] * hQ[r * Np + j];
      eo = std::fmax(eo, std::fabs(s - (i == j ? 1.0 : 0.0)));
    }
    double er = 0;
    for (int64_t r = 0; r < rows; r += rows / 97 + 1) for (int j = 0; j < l; ++j) {
      double s = 0; for (int k = 0; k <= j; ++k) s += hQ[r * Np + k] * hR[k * Np + j];
      er = std::fmax(er, std::fabs(s - S[r * Np + j]));
    }
    double pad = 0;
    for (int64_t r = 0; r < rows; ++r) for (int j = l; j < Np; ++j) pad = std::fmax(pad, std::fabs(hQ[r * Np + j]));
    printf("rows %7lld l %3d Np %3d: gram %7.2f us  chol_aug %7.2f us  apply %7.2f us | flag %d |G err| %.1e (rel %.1e) |RRi-I| %.1e |QtQ-I| %.1e |QR-S| %.1e pad %.1e\n",
           (long long)rows, l, Np, tg, tc, ta, fl, eg, eg / gmax, ei, eo, er, pad);
    cudaFree(dS); cudaFree(dQ); cudaFree(part); cudaFree(G); cudaFree(R); cudaFree(Ri);
  }
  return 0;
}
