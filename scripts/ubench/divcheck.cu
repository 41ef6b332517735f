// Exhaustive check (diagnostic, not part of libgpuar) of the reciprocal division used by the
// argmin rule (kernels_argmin.cu div_by_recip, R23): for EVERY pair of binary32
// significands (t in [0.5, 1), d in [1, 2): 2^46 pairs), q0 = RN(t*y), q = RN(q0 + RN(t - d*q0)*y)
// with y = RN(1/d) must equal the IEEE quotient RN(t/d).  Away from underflow and overflow
// every quantity scales exactly with powers of two, so this covers every exponent pair the
// kernel admits.  Prints the number of mismatches (expected 0).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void check(uint32_t d_lo, uint32_t d_count, unsigned long long* bad, uint32_t* first) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d_count) return;
  const float d = __uint_as_float(0x3f800000u | (d_lo + i));  // [1, 2)
  const float y = __frcp_rn(d);
  unsigned long long nbad = 0;
  for (uint32_t m = 0; m < (1u << 23); ++m) {
    const float t = __uint_as_float(0x3f000000u | m);  // [0.5, 1)
    const float q0 = __fmul_rn(t, y);
    const float q = __fmaf_rn(__fmaf_rn(-q0, d, t), y, q0);
    const float ref = __fdiv_rn(t, d);
    if (__float_as_uint(q) != __float_as_uint(ref)) {
      ++nbad;
      atomicCAS(first, 0xffffffffu, (d_lo + i));
    }
  }
  if (nbad) atomicAdd(bad, nbad);
}

int main() {
  unsigned long long* bad;
  uint32_t* first;
  cudaMalloc(&bad, 8);
  cudaMalloc(&first, 4);
  cudaMemset(bad, 0, 8);
  cudaMemset(first, 0xff, 4);
  const uint32_t total = 1u << 23, per = 1u << 19;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (uint32_t lo = 0; lo < total; lo += per) check<<<per / 256, 256>>>(lo, per, bad, first);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h = 0; uint32_t f = 0;
  cudaMemcpy(&h, bad, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(&f, first, 4, cudaMemcpyDeviceToHost);
  printf("pairs checked: %llu  mismatches: %llu  first bad d-significand: 0x%x  (%.1f s) %s\n",
         (unsigned long long)total * total, h, f, ms / 1e3, cudaGetErrorString(cudaGetLastError()));
  return h != 0;
}
