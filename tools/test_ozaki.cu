// Standalone check of the Ozaki int8 tcgen05 pass (pass_ozaki.cu) against a
// host long-double reference, NN (C = A X) and TN (C = A^T Q).  Not product code.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude -lcuda -o tools/test_ozaki tools/test_ozaki.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
__device__ unsigned long long g_oz[8];
#define OZ_PROBE_DECL long long _ozt[5] = {0, 0, 0, 0, 0}; long long _ozl = clock64();
#define OZ_PROBE(slot) { long long _t = clock64(); _ozt[slot] += _t - _ozl; _ozl = _t; }
#define OZ_PROBE_OUT for (int q = 0; q < 5; ++q) atomicAdd(&g_oz[q], (unsigned long long)_ozt[q]);
__device__ unsigned long long g_oz2[4], g_oz3[4];
#define OZ_PROBE2_DECL long long _p2[3] = {0, 0, 0}; long long _p2l = clock64();
#define OZ_PROBE2(slot) { long long _t = clock64(); _p2[slot] += _t - _p2l; _p2l = _t; }
#define OZ_PROBE2_OUT for (int q = 0; q < 3; ++q) atomicAdd(&g_oz2[q], (unsigned long long)_p2[q]);
#define OZ_PROBE3_DECL long long _p3[4] = {0, 0, 0, 0}; long long _p3l = clock64();
#define OZ_PROBE3(slot) if (lane == 0) { long long _t = clock64(); _p3[slot] += _t - _p3l; _p3l = _t; }
#define OZ_PROBE3_OUT if (lane == 0) for (int q = 0; q < 4; ++q) atomicAdd(&g_oz3[q], (unsigned long long)_p3[q]);
__device__ unsigned long long g_tl[1024][8];
#define OZ_TL(slot) { unsigned long long _g; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_g)); g_tl[blockIdx.x][slot] = _g; }
#include "../paper_1608_02148_b200/csrc/pass_tf32.cu"
#include "../paper_1608_02148_b200/csrc/pass_ozaki.cu"
namespace rsvd {
std::atomic<int64_t> g_kernel_launches{0}; int g_pdl = getenv("RSVD_PDL") ? atoi(getenv("RSVD_PDL")) : 1;
cudaError_t smem_optin_fn(const void* fn) {
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, fn);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448 - (int)fa.sharedSizeBytes);
}
}
using namespace rsvd;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

int main(int argc, char** argv) {
  const int64_t m = argc > 1 ? atol(argv[1]) : 1000, n = argc > 2 ? atol(argv[2]) : 700;
  const int reps = argc > 3 ? atoi(argv[3]) : 0;
  const int mode = argc > 4 ? atoi(argv[4]) : 0;   // 1: one-digit data (A, X = small integers / 128)
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  std::vector<double> A(m * n);
  srand(5);
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double v = (rand() % 200001) / 100000.0 - 1.0;
      if (i % 7 == 3) v *= 1e-6;                 // rows of very different scale
      if (j % 11 == 5) v *= 37.5;
      if (mode == 1) v = ((i * 7 + j * 3) % 255 - 127) / 128.0;
      if (mode == 2) v = (i == j) ? 1.0 / 128 : 0.0;
      A[i * n + j] = v;
    }
  // OZ_F32=1: FP32 A (3-digit slices); OZ_NOCHECK=1: timing only
  const bool f32 = getenv("OZ_F32") && atoi(getenv("OZ_F32"));
  const bool nocheck = getenv("OZ_NOCHECK") && atoi(getenv("OZ_NOCHECK"));
  const int S = f32 ? OZ_S32 : OZ_S;
  if (f32) for (auto& v : A) v = (double)(float)v;
  std::vector<float> Af(f32 ? m * n : 0);
  for (size_t i = 0; i < Af.size(); ++i) Af[i] = (float)A[i];
  double *dA, *dC, *dB, *dP; int* flag; unsigned* flags; void *abuf, *xbuf, *xbuf2;
  CK(cudaMalloc(&dA, m * n * 8));
  if (f32) CK(cudaMemcpy(dA, Af.data(), m * n * 4, cudaMemcpyHostToDevice));
  else CK(cudaMemcpy(dA, A.data(), m * n * 8, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&abuf, ozaki_a_bytes(m, n, S))); CK(cudaMalloc(&flag, 64)); CK(cudaMemset(flag, 0, 64));
  CK(cudaMalloc(&flags, 4096 * 4)); CK(cudaMemset(flags, 0, 4096 * 4));
  const int64_t big = m > n ? m : n;
  CK(cudaMalloc(&dB, big * 128 * 8)); CK(cudaMalloc(&dC, big * 128 * 8)); CK(cudaMalloc(&dP, (size_t)nsm * 2 * 128 * 128 * 8));
  CK(cudaMalloc(&xbuf, ozaki_x_bytes(big, 128, S))); CK(cudaMalloc(&xbuf2, ozaki_x_bytes(big, 128, S)));
  OzakiA oa = ozaki_layout_a(abuf, m, n, S);
  CK(ozaki_slice_a(oa, dA, f32, n, nullptr, nullptr, flag, 0));
  CK(cudaDeviceSynchronize());
  if (!f32 && !nocheck) {
    std::vector<int8_t> sl((size_t)OZ_S * m * oa.ldn);
    std::vector<int> er(m);
    CK(cudaMemcpy(sl.data(), oa.slices, sl.size(), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(er.data(), oa.erow, m * sizeof(int), cudaMemcpyDeviceToHost));
    double e = 0;
    for (int64_t i = 0; i < m; ++i) for (int64_t j = 0; j < n; ++j) {
      long double v = 0, w = 1.0L / 128;      // digit 0 s8 (weight 2^-7), digits t >= 1 u8 (weight 2^{-7-8t})
      for (int t = 0; t < OZ_S; ++t) {
        const int8_t d = sl[((i * (oa.ldn / 128) + j / 128) * OZ_S + t) * 128 + j % 128];
        v += (t == 0 ? (long double)d : (long double)(uint8_t)d) * w;
        w /= 256;
      }
      const double row_max = ldexp(1.0, er[i]);
      v *= row_max;
      e = fmax(e, fabs((double)(v - A[i * n + j])) / row_max);
    }
    printf("A slice reconstruction: max |err| / 2^E_row = %.3e (expect <= 2^-56 = %.1e)\n", e, ldexp(1.0, -56));
  }
  unsigned epoch = 0;
  for (int trans = 0; trans < 2; ++trans)
    for (int N : {16, 32, 48, 64, 80, 96, 112, 128}) {
      if (argc > 5 && N != atoi(argv[5])) continue;
      const int64_t M = trans ? n : m, K = trans ? m : n;
      std::vector<double> B(K * N), C(M * N, -7.0);
      for (int64_t k = 0; k < K; ++k) for (int j = 0; j < N; ++j) {
        B[k * N + j] = ((rand() % 200001) / 100000.0 - 1.0) * (j % 3 == 1 ? 1e3 : 1.0);
        if (mode >= 1) B[k * N + j] = ((k * 5 + j * 11) % 255 - 127) / 128.0;
      }
      CK(cudaMemcpy(dB, B.data(), K * N * 8, cudaMemcpyHostToDevice));
      OzakiCall c{};
      c.a = &oa; c.trans = trans; c.B = dB; c.ldb = N; c.C = dC; c.ldc = N; c.Nout = N; c.P = dP; c.flags = flags;
      c.epoch = ++epoch; c.epoch2 = ++epoch; c.xscratch = xbuf; c.xscratch2 = xbuf2; c.M = M; c.K = K; c.N = N; c.grid = nsm;
      { cudaError_t e0 = ozaki_pass(c, 0); cudaError_t e1 = cudaDeviceSynchronize(); if (e0 || e1) { printf("ozaki_pass N=%d trans=%d: ret %s sync %s\n", N, trans, cudaGetErrorString(e0), cudaGetErrorString(e1)); continue; } }
      CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(C.data(), dC, M * N * 8, cudaMemcpyDeviceToHost));
      double emax_abs = 0, emax_rel = 0, rmax = 0;
      const int64_t istep = M > 2000 ? M / 499 : 1;   // sampled rows for large problems
      for (int64_t i = 0; i < (nocheck ? 0 : M); i += istep)
        for (int j = 0; j < N; ++j) {
          long double s = 0, sa = 0;
          for (int64_t k = 0; k < K; ++k) {
            const double a = trans ? A[k * n + i] : A[i * n + k];
            s += (long double)a * B[k * N + j];
            sa += fabsl((long double)a * B[k * N + j]);
          }
          const double e = fabs((double)(C[i * N + j] - s));
          emax_abs = fmax(emax_abs, e);
          if (sa > 0) emax_rel = fmax(emax_rel, e / (double)sa);
          rmax = fmax(rmax, fabs((double)s));
        }
      {
        unsigned long long pr[8]; cudaMemcpyFromSymbol(pr, g_oz, sizeof pr); unsigned long long z[8] = {0}; cudaMemcpyToSymbol(g_oz, z, sizeof z);
        const double tot = pr[0] + pr[1] + pr[2] + pr[3] + pr[4];
        printf("  MMA thread time: issue %.1f%%  wait xfull %.1f%%  wait acce %.1f%%  wait afull %.1f%%  mma-issue %.1f%%\n",
               100 * pr[0] / tot, 100 * pr[1] / tot, 100 * pr[2] / tot, 100 * pr[3] / tot, 100 * pr[4] / tot);
        unsigned long long p2[4], p3[4]; cudaMemcpyFromSymbol(p2, g_oz2, sizeof p2); cudaMemcpyFromSymbol(p3, g_oz3, sizeof p3);
        cudaMemcpyToSymbol(g_oz2, z, sizeof(g_oz2)); cudaMemcpyToSymbol(g_oz3, z, sizeof(g_oz3));
        const double t2 = p2[0] + p2[1] + p2[2], t3 = p3[0] + p3[1] + p3[2] + p3[3];
        printf("  producer: issue %.1f%%  wait xempty %.1f%%  wait aempty %.1f%% | epilogue: other %.1f%%  wait accf %.1f%%  drain %.1f%%  write-out %.1f%%\n",
               100 * p2[0] / t2, 100 * p2[1] / t2, 100 * p2[2] / t2, 100 * p3[0] / t3, 100 * p3[1] / t3, 100 * p3[2] / t3, 100 * p3[3] / t3);
      }
      if (getenv("OZ_TIMELINE")) {
        static unsigned long long tl[1024][8];
        cudaMemcpyFromSymbol(tl, g_tl, sizeof tl);
        unsigned long long t0 = ~0ull; int nc = 0;
        for (int b = 0; b < 1024; ++b) if (tl[b][0]) { t0 = tl[b][0] < t0 ? tl[b][0] : t0; ++nc; }
        std::vector<double> col[8];
        for (int b = 0; b < nc; ++b) for (int q = 0; q < 8; ++q) if (tl[b][q]) col[q].push_back((tl[b][q] - t0) * 1e-3);
        const char* nm[8] = {"start", "producer-end", "mma-end", "epi-end", "cta-end", "last-drain", "head-added", "-"};
        for (int q = 0; q < 7; ++q) {
          if (col[q].empty()) continue;
          const int nc = (int)col[q].size();
          std::sort(col[q].begin(), col[q].end());
          printf("  %-13s us: min %.1f p10 %.1f med %.1f p90 %.1f max %.1f\n", nm[q], col[q][0], col[q][nc / 10], col[q][nc / 2],
                 col[q][nc * 9 / 10], col[q][nc - 1]);
        }
        cudaMemset(g_tl, 0, 0);
        static unsigned long long z[1024][8] = {}; cudaMemcpyToSymbol(g_tl, z, sizeof z);
      }
      float us = 0;
      if (reps > 0) {
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        for (int r = 0; r < reps; ++r) { c.epoch = ++epoch; c.epoch2 = ++epoch; ozaki_pass(c, 0); }
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&us, e0, e1); us = us * 1000 / reps;
      }
      if (mode >= 1 && N == 16) {
        printf("  C[0][0..7]:"); for (int j = 0; j < 8; ++j) printf(" %.6f", C[j]); printf("\n");
        printf("  R[0][0..7]:");
        for (int j = 0; j < 8; ++j) { long double s2 = 0; for (int64_t k = 0; k < K; ++k) s2 += (long double)(trans ? A[k * n] : A[k]) * B[k * N + j]; printf(" %.6f", (double)s2); }
        printf("\n  C[1][0..7]:"); for (int j = 0; j < 8; ++j) printf(" %.6f", C[N + j]); printf("\n");
      }
      printf("trans %d N %2d: max|C-R| %.3e (max|R| %.3e)  max |C-R|/sum|a x| %.3e  %s  %.1f us\n", trans, N, emax_abs, rmax,
             emax_rel, emax_rel < (f32 ? 2e-6 : 1e-13) ? "OK" : "FAIL", us);
    }
  int fl; CK(cudaMemcpy(&fl, flag, 4, cudaMemcpyDeviceToHost));
  printf("flag %d\n", fl);
  return 0;
}
