// Microbenchmark + self-check of the one-sided Jacobi SVD (jacobi.cu):
// X = R^T, X J = W Sigma.  Checks W^T W = I, J^T J = I, X J = W Sigma, sorted
// sigma.  Not product code.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude -o tools/bench_jacobi tools/bench_jacobi.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
__device__ unsigned long long g_jp[6];
#define JAC_PROBE
#define JAC_PROBE_DECL long long _jt[5] = {0, 0, 0, 0, 0}; long long _jl = clock64();
#define JAC_PROBE(slot) if (threadIdx.x == 0) { long long _t = clock64(); _jt[slot] += _t - _jl; _jl = _t; }
#define JAC_PROBE_OUT if (threadIdx.x == 0) { for (int q = 0; q < 5; ++q) atomicAdd(&g_jp[q], (unsigned long long)_jt[q]); atomicAdd(&g_jp[5], (unsigned long long)gstep); }
__device__ unsigned long long g_jb[8];
__shared__ long long g_jbl;
#define JB_PROBE(slot) if (blockIdx.x == 0 && threadIdx.x == 0) { const long long _t = clock64(); if (slot > 0) atomicAdd(&g_jb[slot - 1], (unsigned long long)(_t - g_jbl)); else atomicAdd(&g_jb[5], 1ull); g_jbl = _t; }
#include "../paper_1608_02148_b200/csrc/jacobi.cu"
namespace rsvd { std::atomic<int64_t> g_kernel_launches{0}; int g_pdl = 1; cudaError_t smem_optin_fn(const void* fn) { cudaFuncAttributes a; cudaError_t e = cudaFuncGetAttributes(&a, fn); if (e != cudaSuccess) return e; int o = 0; cudaDeviceGetAttribute(&o, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0); return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, o - (int)a.sharedSizeBytes); } }
using namespace rsvd;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

template <typename F> float timeit(F f, int reps) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); CK(cudaDeviceSynchronize());
  cudaEventRecord(a); for (int r = 0; r < reps; ++r) f(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); CK(cudaGetLastError()); return ms * 1000.f / reps;
}

// host check of the block order: per sweep every column pair meets exactly
// once (the intra step's last round is the identity round) and the pairs of a
// round (over all warps) are disjoint
static bool check_block_order() {
  bool ok = true;
  for (int B : {4, 8})
    for (int NB = 2; NB <= 16; NB += 2) {
      const int NC = NB * B, W = NB / 2;
      std::vector<int> met(NC * NC, 0);
      for (int s = 0; s < NB; ++s)
        for (int rho = 0; rho < B; ++rho) {
          if (s == 0 && rho == B - 1) continue;
          std::vector<int> used(NC, 0);
          for (int w = 0; w < W; ++w) {
            int I, J;
            blk_blocks(NB, s, w, I, J);
            for (int j = 0; j < B; ++j) {
              const int lp = blk_lp(B, s == 0, rho, j), lq = blk_lq(B, s == 0, rho, j);
              const int p = lp < B ? I * B + lp : J * B + lp - B, q = lq < B ? I * B + lq : J * B + lq - B;
              if (p == q || used[p]++ || used[q]++) ok = false;
              met[std::min(p, q) * NC + std::max(p, q)]++;
            }
          }
        }
      for (int p = 0; p < NC; ++p)
        for (int q = p + 1; q < NC; ++q)
          if (met[p * NC + q] != 1) ok = false;
      if (!ok) { printf("block order FAILED at B %d NB %d\n", B, NB); return false; }
    }
  printf("block order: every pair once per sweep, rounds disjoint (B 4/8, NB 2..16)\n");
  return ok;
}

int main(int argc, char** argv) {
  if (!check_block_order()) return 1;
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  int* flag; CK(cudaMalloc(&flag, 64));
  int* sw; CK(cudaMalloc(&sw, 64));
  for (int l : {1, 2, 7, 20, 30, 60, 64, 100, 120, 128}) {
    if (only > 0 && l != only) continue;
    const int ld = (l + 15) / 16 * 16;
    std::vector<double> R(ld * ld, 0.0);
    srand(l);
    for (int i = 0; i < l; ++i)
      for (int j = i; j < l; ++j)
        R[i * ld + j] = (i == j) ? std::exp(-i / 20.0) : 0.3 * ((rand() % 2001) / 1000.0 - 1.0) * std::exp(-i / 20.0);
    double *dR, *sig, *W, *J; void* scr;
    CK(cudaMalloc(&dR, ld * ld * 8)); CK(cudaMalloc(&sig, ld * 8)); CK(cudaMalloc(&W, ld * ld * 8));
    CK(cudaMalloc(&J, ld * ld * 8)); CK(cudaMalloc(&scr, jacobi_scratch_bytes(l)));
    CK(cudaMemcpy(dR, R.data(), ld * ld * 8, cudaMemcpyHostToDevice));
    CK(cudaMemset(flag, 0, 64));
    for (int jg : {4, 8}) {
      g_jacobi_lanes = jg;
      float tj = timeit([&] { launch_jacobi(dR, ld, l, sig, W, J, ld, flag, sw, scr, 0); }, 10);
      unsigned long long pr[6]; cudaMemcpyFromSymbol(pr, g_jp, sizeof pr); unsigned long long z[6] = {0}; cudaMemcpyToSymbol(g_jp, z, sizeof z);
      const double st = pr[5] > 0 ? (double)pr[5] : 1.0;
      printf("    lanes/pair %2d: %8.2f us | cycles/step (thread 0): ld->reduced %.0f  rot %.0f  apply+store %.0f  barrier %.0f  (other %.0f)\n", jg, tj,
             pr[1] / st, pr[2] / st, pr[3] / st, pr[4] / st, pr[0] / st);
    }
    g_jacobi_lanes = 0;
    {
      unsigned long long z[8] = {0}; cudaMemcpyToSymbol(g_jb, z, sizeof z);
      timeit([&] { launch_jacobi(dR, ld, l, sig, W, J, ld, flag, sw, scr, 0); }, 3);
      unsigned long long pr[8]; cudaMemcpyFromSymbol(pr, g_jb, sizeof pr);
      const double n = pr[5] ? (double)pr[5] : 1.0;
      printf("    block order, cycles per round (warp 0): dots %.0f  reduce %.0f  rot %.0f  bcast+apply %.0f  | rounds %.0f\n",
             pr[0] / n, pr[1] / n, pr[2] / n, pr[3] / n, n / 4);
    }
    float t = timeit([&] { launch_jacobi(dR, ld, l, sig, W, J, ld, flag, sw, scr, 0); }, 10);
    int sweeps, fl;
    CK(cudaMemcpy(&sweeps, sw, 4, cudaMemcpyDeviceToHost)); CK(cudaMemcpy(&fl, flag, 4, cudaMemcpyDeviceToHost));
    std::vector<double> hs(ld), hW(ld * ld), hJ(ld * ld);
    CK(cudaMemcpy(hs.data(), sig, ld * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hW.data(), W, ld * ld * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hJ.data(), J, ld * ld * 8, cudaMemcpyDeviceToHost));
    double ew = 0, ej = 0, er = 0, srt = 0;
    for (int a = 0; a < l; ++a)
      for (int b = 0; b < l; ++b) {
        double sw_ = 0, sj = 0;
        for (int i = 0; i < l; ++i) { sw_ += hW[i * ld + a] * hW[i * ld + b]; sj += hJ[i * ld + a] * hJ[i * ld + b]; }
        ew = std::fmax(ew, std::fabs(sw_ - (a == b))); ej = std::fmax(ej, std::fabs(sj - (a == b)));
      }
    for (int i = 0; i < l; ++i)            // X J = W Sigma, X = R^T: X[i][p] = R[p][i]
      for (int c = 0; c < l; ++c) {
        double s = 0; for (int p = 0; p < l; ++p) s += R[p * ld + i] * hJ[p * ld + c];
        er = std::fmax(er, std::fabs(s - hW[i * ld + c] * hs[c]));
      }
    for (int i = 1; i < l; ++i) if (hs[i] > hs[i - 1]) srt = 1;
    printf("l %3d: jacobi %8.2f us  sweeps %d flag %d | |WtW-I| %.1e |JtJ-I| %.1e |XJ-WS| %.1e unsorted %d s0 %.6f s_l %.3e\n",
           l, t, sweeps, fl, ew, ej, er, (int)srt, hs[0], hs[l - 1]);
    cudaFree(dR); cudaFree(sig); cudaFree(W); cudaFree(J); cudaFree(scr);
  }
  return 0;
}
