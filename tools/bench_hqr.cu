// Microbenchmark of the small-panel Householder QR (panel.cu): the single-CTA
// hqr_leaves kernel against the one-launch TSQR (tsqr_fused_kernel) over
// small leaves of about `leaf` rows.  Checks Q^T Q = I and Q R = Y.  Not product code.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Iinclude -o tools/bench_hqr tools/bench_hqr.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_1608_02148_b200/csrc/panel.cu"
namespace rsvd {
std::atomic<int64_t> g_kernel_launches{0};
int g_pdl = 1;
cudaError_t smem_optin_fn(const void* fn) {
  cudaFuncAttributes a;
  cudaError_t e = cudaFuncGetAttributes(&a, fn);
  if (e != cudaSuccess) return e;
  int o = 0;
  cudaDeviceGetAttribute(&o, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, o - (int)a.sharedSizeBytes);
}
}  // namespace rsvd
using namespace rsvd;

// the level structure of tsqr_levels with a leaf-row target instead of the shared-memory cap
static bool plan(int64_t rows, int l, int cap, std::vector<int64_t>& leaves) {
  int64_t Mc = rows;
  while (Mc > cap) {
    int64_t P = (Mc + cap - 1) / cap;
    if (Mc / P < l) P = Mc / l;
    if (P < 1 || P * l >= Mc) return false;
    leaves.push_back(P);
    Mc = P * l;
  }
  return true;
}

static void check(const char* what, int m, int l, int ld, const std::vector<double>& Y, double* dQ, double* dR, float us) {
  std::vector<double> Q(m * ld), R(l * l);
  cudaMemcpy(Q.data(), dQ, m * ld * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(R.data(), dR, l * l * 8, cudaMemcpyDeviceToHost);
  double eo = 0, er = 0;
  for (int i = 0; i < l; ++i)
    for (int j = 0; j < l; ++j) {
      double s = 0;
      for (int r = 0; r < m; ++r) s += Q[r * ld + i] * Q[r * ld + j];
      eo = fmax(eo, fabs(s - (i == j)));
    }
  for (int r = 0; r < m; r += 7)
    for (int j = 0; j < l; ++j) {
      double s = 0;
      for (int k = 0; k <= j; ++k) s += Q[r * ld + k] * R[k * l + j];
      er = fmax(er, fabs(s - Y[r * ld + j]));
    }
  printf("%-22s %5d x %3d: %8.2f us  |QtQ-I| %.1e  |QR-Y| %.1e (%s)\n", what, m, l, us, eo, er,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  void* ws;
  cudaMalloc(&ws, 64 << 20);
  unsigned* bar;
  cudaMalloc(&bar, 256 * sizeof(unsigned));
  cudaMemset(bar, 0, 256 * sizeof(unsigned));
  for (auto ml : std::vector<std::pair<int, int>>{{1000, 20}, {500, 20}, {1400, 20}, {460, 60}, {5000, 60}}) {
    const int m = ml.first, l = ml.second, ld = (l + 15) / 16 * 16;
    std::vector<double> Y(m * ld, 0.0);
    for (int r = 0; r < m; ++r)
      for (int c = 0; c < l; ++c) Y[r * ld + c] = (rand() % 2001) / 1000.0 - 1.0;
    double *dY, *dYs, *Rs;
    cudaMalloc(&dY, m * ld * 8);
    cudaMalloc(&dYs, m * ld * 8);
    cudaMalloc(&Rs, l * l * 8);
    cudaMemcpy(dYs, Y.data(), m * ld * 8, cudaMemcpyHostToDevice);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timed = [&](auto f) {
      float best = 1e30f;
      for (int rep = 0; rep < 5; ++rep) {
        cudaMemcpy(dY, dYs, m * ld * 8, cudaMemcpyDeviceToDevice);
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        f();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = fmin(best, ms * 1000.f);
      }
      return best;
    };
    if ((size_t)m * l + l + 32 <= (size_t)SMEM_OPTIN / 8) {
      const float t = timed([&] { launch_hqr_leaves(dY, ld, m, l, 1, Rs, 0); });
      check("hqr (one CTA)", m, l, ld, Y, dY, Rs, t);
    }
    for (int cap : {64, 128, 256, 512}) {
      std::vector<int64_t> leaves;
      if (cap < 2 * l || !plan(m, l, cap, leaves)) continue;
      TsqrArgs ta = {};
      char* wp = (char*)ws;
      double* cur = dY;
      int64_t ldc = ld, Mc = m;
      for (int64_t P : leaves) {
        double* stack = (double*)wp;
        wp += ((size_t)P * l * l * 8 + 255) / 256 * 256;
        ta.lev[ta.nlev++] = TsqrLevel{cur, ldc, Mc, P};
        cur = stack; ldc = l; Mc = P * l;
      }
      ta.l = l; ta.cur = cur; ta.ldc = ldc; ta.Mc = Mc; ta.R = Rs; ta.Rout = nullptr; ta.ldro = 0; ta.bar = bar;
      const float t = timed([&] { launch_tsqr_fused(ta, nsm, 0); });
      char name[64];
      snprintf(name, sizeof name, "tsqr leaves<=%d (%d lv)", cap, ta.nlev);
      check(name, m, l, ld, Y, dY, Rs, t);
    }
    cudaFree(dY); cudaFree(dYs); cudaFree(Rs);
  }
  return 0;
}
