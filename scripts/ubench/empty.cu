// Diagnostic: device time of near-empty kernels (launch + CTA ramp/drain) for several grids,
// measured back to back with CUDA events (the floor under any per-call kernel time).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void empty_kernel(int* sink) { if (threadIdx.x == 1023) sink[blockIdx.x] = 1; }
int main() {
  int* sink; cudaMalloc(&sink, 4096 * sizeof(int));
  int grids[] = {1, 148, 296, 592, 1184};
  int blocks[] = {256, 1024};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int b : blocks) for (int g : grids) {
    for (int i = 0; i < 10; ++i) empty_kernel<<<g, b>>>(sink);
    cudaEventRecord(e0);
    for (int i = 0; i < 1000; ++i) empty_kernel<<<g, b>>>(sink);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("grid %5d x %4d threads: %.2f us per launch (back to back)\n", g, b, ms);
  }
  return 0;
}
