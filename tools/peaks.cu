// Box-measurement microbenchmarks: FP64 DMMA vs DFMA
// peak, read-only HBM streaming bandwidth, device properties.  Not product
// code; results land in profiles/peaks_box.json.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); exit(1);}}while(0)

template<int NACC>
__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[NACC][2];
  #pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  #pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

template<int NACC>
__global__ void dmma16_loop(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4=a0+4,a5=a0+5,a6=a0+6,a7=a0+7;
  double b0 = 1.0 + threadIdx.x * 1e-4, b1 = b0 + 1, b2=b0+2, b3=b0+3;
  double c[NACC][4];
  #pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0; }
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a0),"d"(a1),"d"(a2),"d"(a3),"d"(a4),"d"(a5),"d"(a6),"d"(a7),"d"(b0),"d"(b1),"d"(b2),"d"(b3));
  }
  double s = 0;
  #pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.0) out[0] = s;
}

template<int NACC>
__global__ void dfma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[NACC];
  #pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0;
  #pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 12345.0) out[0] = s;
}

__global__ void read_bw(const double4* __restrict__ p, size_t n, double* out) {
  double s = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride * 4) {
    double4 v[4];
    #pragma unroll
    for (int u = 0; u < 4; ++u) { size_t j = i + u * stride; if (j < n) { const double2* q = (const double2*)(p + j); double2 x = __ldcs(q), y = __ldcs(q + 1); v[u] = make_double4(x.x, x.y, y.x, y.y); } else v[u] = make_double4(0,0,0,0); }
    #pragma unroll
    for (int u = 0; u < 4; ++u) s += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (s == 12345.0) out[0] = s;
}

template<typename F> float timeit(F f, int reps) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  return best;
}

int main() {
  cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, 0));
  int smemOptin = 0; cudaDeviceGetAttribute(&smemOptin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"name\":\"%s\",\"sms\":%d,\"l2_bytes\":%d,\"smem_optin\":%d,\"smem_per_sm\":%zu,\"clock_khz\":%d,\"mem_bytes\":%zu",
         pr.name, pr.multiProcessorCount, pr.l2CacheSize, smemOptin, pr.sharedMemPerMultiprocessor, clk, pr.totalGlobalMem);
  double* out; CK(cudaMalloc(&out, 64));
  int sms = pr.multiProcessorCount;
  const int iters = 20000;
  for (int wpb : {4, 8, 16}) {
    int threads = wpb * 32, blocks = sms * 4;
    float ms = timeit([&]{ dmma_loop<8><<<blocks, threads>>>(out, iters); }, 5);
    double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (blocks * wpb);
    printf(",\"dmma_m8n8k4_tflops_w%d\":%.2f", wpb, flops / ms / 1e9);
    ms = timeit([&]{ dmma16_loop<4><<<blocks, threads>>>(out, iters / 4); }, 5);
    flops = 2.0 * 16 * 8 * 16 * 4.0 * (iters / 4) * (blocks * wpb);
    printf(",\"dmma_m16n8k16_tflops_w%d\":%.2f", wpb, flops / ms / 1e9);
    ms = timeit([&]{ dfma_loop<8><<<blocks, threads>>>(out, iters); }, 5);
    flops = 2.0 * 8.0 * iters * (blocks * (double)threads);
    printf(",\"dfma_tflops_w%d\":%.2f", wpb, flops / ms / 1e9);
  }
  size_t bytes = (size_t)8 << 30;
  double4* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 0, bytes));
  size_t n = bytes / sizeof(double4);
  for (int bpsm : {2, 4, 8}) {
    float ms = timeit([&]{ read_bw<<<sms * bpsm, 512>>>(buf, n, out); }, 10);
    printf(",\"read_gbs_b%d\":%.1f", bpsm, bytes / ms / 1e6);
  }
  float ms = timeit([&]{ cudaMemcpyAsync((char*)buf + bytes / 2, buf, bytes / 2, cudaMemcpyDeviceToDevice); }, 10);
  printf(",\"copy_gbs\":%.1f}\n", bytes / ms / 1e6);
  return 0;
}
