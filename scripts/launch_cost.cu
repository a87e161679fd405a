// Launch cost of an empty persistent-style grid on the B200 (params size, smem):
// CUDA events around each launch on one stream, as bench.py times K1.
#include <cstdio>
#include <cuda_runtime.h>
struct Big { char b[1300]; };
struct Small { int x; };
__global__ void k_big(const Big p) { if (p.b[threadIdx.x & 1023] == 123 && threadIdx.x == 9999) printf("x"); }
__global__ void k_small(const Small p) { if (p.x == 123 && threadIdx.x == 9999) printf("x"); }
template <typename F, typename P>
float run(F f, P p, int grid, int smem) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  if (smem > 48 * 1024) cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  float tot = 0; int n = 0;
  for (int i = 0; i < 60; ++i) {
    cudaEventRecord(a); f<<<grid, 128, smem>>>(p); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (i >= 10) { tot += ms; ++n; }
  }
  return tot / n * 1000.f;
}
int main() {
  Big big{}; Small small{};
  for (int smem : {0, 36 * 1024})
    for (int grid : {148, 740}) {
      printf("grid %4d smem %6d: big params %.2f us, small params %.2f us\n", grid, smem,
             run(k_big, big, grid, smem), run(k_small, small, grid, smem));
    }
  return 0;
}
