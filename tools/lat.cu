// Latency probes for the single-CTA kernels (cycles per loop iteration).
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void probe(double* out, long long* cyc, int iters, int nthreads_active) {
  __shared__ double sm[4096];
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < 4096; i += blockDim.x) sm[i] = 1.0 + i * 1e-6;
  __syncthreads();
  double acc = 0.0, x = sm[tid];
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) { __syncthreads(); }                                  // barrier only
    if (MODE == 1) { acc += sm[(it * 37 + tid) & 4095]; __syncthreads(); }  // LDS + barrier
    if (MODE == 2) { double v = sm[(it * 37 + tid) & 4095];             // LDS + 5-level double shuffle + barrier
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      acc += v; __syncthreads(); }
    if (MODE == 3) { x = sqrt(x * 1.0000001 + 1e-3); x = 1.0 / (x + 1.0); x = rsqrt(x + 2.0); acc += x; }  // fp64 math chain
    if (MODE == 4) { x = fma(x, 1.0000001, 1e-9); }                          // dfma chain
    if (MODE == 5) { double v = sm[(it * 37 + tid) & 4095]; sm[(it * 53 + tid) & 4095] = v * 1.0000001; __syncthreads(); }
  }
  long long t1 = clock64();
  if (tid == 0) cyc[0] = (t1 - t0);
  out[tid] = acc + x;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 8192 * 8); cudaMalloc(&cyc, 8);
  const char* names[] = {"barrier", "lds+barrier", "lds+shfl5+barrier", "sqrt+div+rsqrt chain", "dfma chain", "lds+sts+barrier"};
  for (int threads : {32, 128, 512, 1024}) {
    for (int mode = 0; mode < 6; ++mode) {
      const int iters = 2000;
      long long c = 0;
      for (int rep = 0; rep < 2; ++rep) {
        switch (mode) {
          case 0: probe<0><<<1, threads>>>(out, cyc, iters, threads); break;
          case 1: probe<1><<<1, threads>>>(out, cyc, iters, threads); break;
          case 2: probe<2><<<1, threads>>>(out, cyc, iters, threads); break;
          case 3: probe<3><<<1, threads>>>(out, cyc, iters, threads); break;
          case 4: probe<4><<<1, threads>>>(out, cyc, iters, threads); break;
          case 5: probe<5><<<1, threads>>>(out, cyc, iters, threads); break;
        }
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      }
      printf("threads %4d  %-24s %8.1f cycles/iter\n", threads, names[mode], (double)c / iters);
    }
  }
  return 0;
}
