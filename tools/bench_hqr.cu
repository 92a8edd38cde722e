// Microbenchmark of the single-CTA Householder panel QR (panel.cu hqr_leaves). Not product code.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_1608_02148_b200/csrc/panel.cu"
namespace rsvd { int64_t g_kernel_launches = 0; }
using namespace rsvd;
int main() {
  for (auto ml : std::vector<std::pair<int, int>>{{1000, 20}, {500, 20}, {1400, 20}, {460, 60}}) {
    const int m = ml.first, l = ml.second, ld = (l + 15) / 16 * 16;
    std::vector<double> Y(m * ld, 0.0);
    for (int r = 0; r < m; ++r) for (int c = 0; c < l; ++c) Y[r * ld + c] = (rand() % 2001) / 1000.0 - 1.0;
    double *dY, *dYs, *Rs; cudaMalloc(&dY, m * ld * 8); cudaMalloc(&dYs, m * ld * 8); cudaMalloc(&Rs, l * l * 8);
    cudaMemcpy(dYs, Y.data(), m * ld * 8, cudaMemcpyHostToDevice);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaMemcpy(dY, dYs, m * ld * 8, cudaMemcpyDeviceToDevice); launch_hqr_leaves(dY, ld, m, l, 1, Rs, 0);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int r = 0; r < 10; ++r) launch_hqr_leaves(dY, ld, m, l, 1, Rs, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    // orthonormality of the result (of the first factorisation applied repeatedly: Q of Q = Q up to signs)
    std::vector<double> Q(m * ld); cudaMemcpy(Q.data(), dY, m * ld * 8, cudaMemcpyDeviceToHost);
    double eo = 0;
    for (int i = 0; i < l; ++i) for (int j = 0; j < l; ++j) { double s = 0; for (int r = 0; r < m; ++r) s += Q[r * ld + i] * Q[r * ld + j]; eo = fmax(eo, fabs(s - (i == j))); }
    printf("hqr %5d x %3d: %8.2f us  |QtQ-I| %.1e (%s)\n", m, l, ms * 100, eo, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
