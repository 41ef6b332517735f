// synth_rows.cu -- libsynth: the per-realization matrix recipe of synth/__init__.py
// (`rows`) as a CUDA kernel, so bench.py can fill a 4 GiB K x M matrix in HBM in
// milliseconds.  Input generation only: no Philox, no acceptance test, no reductions.
// Cell (k, j) = rates[j] if bit 63 of mix64(gen_seed, k*M + j) else 0; padding columns
// j in [M, ld) are 0.  Integer-only, so it is bit-identical to the numpy recipe
// (checked by tests/test_synth.py).
#include <cstdint>
#include <cuda_runtime.h>

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t seed, uint64_t counter) {
  uint64_t z = seed + (counter + 1ull) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void synth_rows_kernel(float* __restrict__ out, const float* __restrict__ rates, uint64_t M, uint64_t ld,
                                  uint64_t k0, uint64_t nrows, uint64_t gen_seed) {
  const uint64_t total = nrows * ld;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = e / ld, j = e - r * ld;
    float v = 0.f;
    if (j < M && (mix64(gen_seed, (k0 + r) * M + j) >> 63)) v = rates[j];
    out[e] = v;
  }
}

}  // namespace

extern "C" int synth_rows(float* d_out, const float* d_rates, int64_t M, int64_t ld, int64_t k0, int64_t nrows,
                          uint64_t gen_seed, void* stream) {
  if (!d_out || !d_rates || M < 1 || ld < M || k0 < 0 || nrows < 0) return -1;
  if (nrows == 0) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  synth_rows_kernel<<<sms * 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      d_out, d_rates, (uint64_t)M, (uint64_t)ld, (uint64_t)k0, (uint64_t)nrows, gen_seed);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}
