// Test-only known-answer source: cuRAND's curand_Philox4x32_10, compiled for
// the HOST (its mulhilo32 has a host branch).  Independent of both the oracle
// (oracle/philox.py) and the product generator (csrc/omega.cu).
// stdin: lines "c0 c1 c2 c3 k0 k1" (hex); stdout: "w0 w1 w2 w3" (hex).
#include <cstdio>
#include <vector_types.h>
#define QUALIFIERS static inline __host__ __device__
#include <curand_philox4x32_x.h>
int main() {
  unsigned c0, c1, c2, c3, k0, k1;
  while (scanf("%x %x %x %x %x %x", &c0, &c1, &c2, &c3, &k0, &k1) == 6) {
    uint4 c = make_uint4(c0, c1, c2, c3);
    uint2 k = make_uint2(k0, k1);
    uint4 w = curand_Philox4x32_10(c, k);
    printf("%08x %08x %08x %08x\n", w.x, w.y, w.z, w.w);
  }
  return 0;
}
