// Dependent-chain latencies (cycles per iteration) of the primitives on the
// critical path of the single-warp factorisations.  Not product code.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rsqrt_nr(double p) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(p));
  const double h = 0.5 * p;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return y;
}
__device__ __forceinline__ double rsqrt_approx(double p) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(p));
  return y;
}
template <int MODE>
__global__ void k(double* out, long long* cyc, int iters) {
  __shared__ double sm[64];
  const int lane = threadIdx.x & 31;
  sm[lane] = 1.0 + lane; __syncwarp();
  double x = 1.0 + lane * 1e-3;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) x = fma(x, 0.999999, 1e-7);                          // DFMA
    if (MODE == 1) x = x * 0.99999999;                                  // DMUL
    if (MODE == 2) x = rsqrt_approx(x) + 0.5;                           // MUFU.RSQ64H + DADD
    if (MODE == 3) x = rsqrt_nr(x) + 0.5;                               // full rsqrt
    if (MODE == 4) x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31) * 1.0000001;  // SHFL double + DMUL
    if (MODE == 5) { sm[lane] = x; __syncwarp(); x = sm[(lane + 1) & 31] * 1.0000001; __syncwarp(); }  // STS+LDS
    if (MODE == 6) x = sqrt(x) + 0.5;                                   // IEEE sqrt
    if (MODE == 7) x = 1.0 / x + 0.5;                                   // IEEE div
    if (MODE == 8) { float f = rsqrtf((float)x); x = (double)f + 0.5; } // FP32 MUFU path
  }
  long long t1 = clock64();
  if (lane == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = x;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 8192); cudaMalloc(&cyc, 8);
  const char* names[] = {"DFMA", "DMUL", "rsqrt.approx.f64+DADD", "rsqrt_nr (2 NR)+DADD", "SHFL.f64+DMUL",
                         "STS+syncwarp+LDS+DMUL", "sqrt(double)+DADD", "1.0/x+DADD", "f32 rsqrt+cvt"};
  for (int m = 0; m < 9; ++m) {
    long long c = 0;
    for (int rep = 0; rep < 2; ++rep) {
      switch (m) {
        case 0: k<0><<<1, 32>>>(out, cyc, 4096); break; case 1: k<1><<<1, 32>>>(out, cyc, 4096); break;
        case 2: k<2><<<1, 32>>>(out, cyc, 4096); break; case 3: k<3><<<1, 32>>>(out, cyc, 4096); break;
        case 4: k<4><<<1, 32>>>(out, cyc, 4096); break; case 5: k<5><<<1, 32>>>(out, cyc, 4096); break;
        case 6: k<6><<<1, 32>>>(out, cyc, 4096); break; case 7: k<7><<<1, 32>>>(out, cyc, 4096); break;
        case 8: k<8><<<1, 32>>>(out, cyc, 4096); break;
      }
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    }
    printf("%-26s %7.1f cycles/iter\n", names[m], (double)c / 4096);
  }
  return 0;
}
