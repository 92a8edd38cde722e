// Microbenchmark of the single-CTA kernels (chol_inv, jacobi, hqr leaves)
// on synthetic well-conditioned inputs.  Not product code.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
__device__ long long g_probe[8];
__device__ long long g_probe_last;
__device__ long long c_probe[8];
__device__ long long c_probe_last;
#define CPROBE(k) if (threadIdx.x == 0) { long long _t = clock64(); if (k > 0) c_probe[k] += _t - c_probe_last; c_probe_last = _t; }
#define JPROBE(k) if (threadIdx.x == 0) { long long _t = clock64(); if (k > 0) g_probe[k] += _t - g_probe_last; g_probe_last = _t; }
#include "../paper_1608_02148_b200/csrc/panel.cu"
namespace rsvd { int64_t g_kernel_launches = 0; }
using namespace rsvd;
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); exit(1);}}while(0)
template<typename F> float timeit(F f, int reps) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); CK(cudaDeviceSynchronize());
  cudaEventRecord(a); for (int r = 0; r < reps; ++r) f(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); CK(cudaGetLastError()); return ms * 1000.f / reps;
}
int main() {
  int* flag; CK(cudaMalloc(&flag, 64)); CK(cudaMemset(flag, 0, 64));
  int* sw; CK(cudaMalloc(&sw, 64));
  for (int l : {20, 32, 60, 64, 120}) {
    // R upper with a decaying spectrum-ish diagonal, Gram G = R^T R
    std::vector<double> R(l * l, 0.0), G(l * l, 0.0);
    srand(l);
    for (int i = 0; i < l; ++i) for (int j = i; j < l; ++j)
      R[i * l + j] = (i == j) ? std::exp(-i / 20.0) : 0.1 * ((rand() % 2001) / 1000.0 - 1.0) * std::exp(-i / 20.0);
    for (int i = 0; i < l; ++i) for (int j = 0; j < l; ++j) { double s = 0; for (int k = 0; k < l; ++k) s += R[k*l+i]*R[k*l+j]; G[i*l+j] = s; }
    int np = (l + 15) / 16 * 16;
    double *dR, *dG, *dR1, *dRi, *sig, *W, *Jm;
    CK(cudaMalloc(&dR, l*l*8)); CK(cudaMalloc(&dG, l*l*8)); CK(cudaMalloc(&dR1, np*np*8)); CK(cudaMalloc(&dRi, np*np*8));
    CK(cudaMalloc(&sig, np*8)); CK(cudaMalloc(&W, np*np*8)); CK(cudaMalloc(&Jm, np*np*8));
    CK(cudaMemcpy(dR, R.data(), l*l*8, cudaMemcpyHostToDevice)); CK(cudaMemcpy(dG, G.data(), l*l*8, cudaMemcpyHostToDevice));
    for (int ny : {16}) {
      rsvd::g_chol_ny = ny;
      float t1 = timeit([&]{ launch_chol_inv(dG, l, l, np, dR1, dRi, flag, 1, 0); }, 20);
      printf("      chol_inv ny=%2d: %8.2f us\n", ny, t1);
    }
    rsvd::g_chol_ny = 16;
    float tc = timeit([&]{ launch_chol_inv(dG, l, l, np, dR1, dRi, flag, 1, 0); }, 20);
    // check: R1 ~ R, R1 * Rinv ~ I
    std::vector<double> R1(np*np), Ri(np*np);
    CK(cudaMemcpy(R1.data(), dR1, np*np*8, cudaMemcpyDeviceToHost)); CK(cudaMemcpy(Ri.data(), dRi, np*np*8, cudaMemcpyDeviceToHost));
    double e1 = 0, e2 = 0;
    for (int i = 0; i < l; ++i) for (int j = 0; j < l; ++j) {
      e1 = std::fmax(e1, std::fabs(R1[i*np+j] - R[i*l+j]));
      double s = 0; for (int k = 0; k < l; ++k) s += R1[i*np+k]*Ri[k*np+j];
      e2 = std::fmax(e2, std::fabs(s - (i == j)));
    }
    { long long pr[8]; cudaMemcpyFromSymbol(pr, c_probe, sizeof pr); long long z[8] = {0}; cudaMemcpyToSymbol(c_probe, z, sizeof z);
      printf("      chol probe (all runs): load %lld diag %lld rowsolve %lld trail %lld invdiag %lld invoff %lld store %lld\n", pr[1], pr[2], pr[3], pr[4], pr[5], pr[6], pr[7]); }
    printf("l=%3d chol_inv %8.2f us (|R1-R| %.1e, |R R^-1 - I| %.1e)\n", l, tc, e1, e2);
    for (int cfg = 0; cfg < 8; ++cfg) {
      const int gls[4] = {4, 8, 16, 32};
      int gl = gls[cfg % 4];
      rsvd::g_jacobi_fastt = cfg >= 4;
      rsvd::g_jacobi_lanes = gl;
      float tj = timeit([&]{ launch_jacobi(dR, l, l, sig, W, Jm, np, flag, sw, 0); }, 10);
      int sweeps; CK(cudaMemcpy(&sweeps, sw, 4, cudaMemcpyDeviceToHost));
      int fl; CK(cudaMemcpy(&fl, flag, 4, cudaMemcpyDeviceToHost));
      std::vector<double> sv(l); CK(cudaMemcpy(sv.data(), sig, l * 8, cudaMemcpyDeviceToHost));
      long long pr[8]; cudaMemcpyFromSymbol(pr, g_probe, sizeof pr); long long z[8] = {0}; cudaMemcpyToSymbol(g_probe, z, sizeof z);
      printf("      probe cycles (11 runs): dot+red %lld math %lld rot %lld barrier %lld\n", pr[1], pr[2], pr[3], pr[4]);
      printf("      jacobi fastt %d lanes/pair %2d: %8.2f us sweeps %d flag %d sigma0 %.15f sigma_l %.3e\n", (int)rsvd::g_jacobi_fastt, gl, tj, sweeps, fl, sv[0], sv[l-1]);
    }
    cudaFree(dR); cudaFree(dG); cudaFree(dR1); cudaFree(dRi); cudaFree(sig); cudaFree(W); cudaFree(Jm);
  }
  // Householder single leaf
  for (auto ml : std::vector<std::pair<int,int>>{{1000, 20}, {1400, 20}, {460, 60}, {240, 120}}) {
    int m = ml.first, l = ml.second; std::vector<double> Y(m * l);
    for (auto& v : Y) v = (rand() % 2001) / 1000.0 - 1.0;
    double *dY, *dYs, *Rs; CK(cudaMalloc(&dY, m*l*8)); CK(cudaMalloc(&dYs, m*l*8)); CK(cudaMalloc(&Rs, l*l*8));
    CK(cudaMemcpy(dYs, Y.data(), m*l*8, cudaMemcpyHostToDevice));
    float th = timeit([&]{ cudaMemcpyAsync(dY, dYs, m*l*8, cudaMemcpyDeviceToDevice); launch_hqr_leaves(dY, l, m, l, 1, Rs, 0); }, 10);
    printf("hqr leaf %dx%d: %.2f us (incl. copy)\n", m, l, th);
    cudaFree(dY); cudaFree(dYs); cudaFree(Rs);
  }
  return 0;
}
