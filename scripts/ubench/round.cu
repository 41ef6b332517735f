// Microbenchmark (diagnostic, not part of libgpuar): throughput of the trial-round
// instruction mix on B200, to separate the round's own cost from selection bookkeeping.
//   mode 0: Philox4x32-10 only (one call per iteration, dependent loop)
//   mode 1: + umulhi index, u scaling, two LDS gathers, compare, ballot, uniform branch
//   mode 2: mode 1 with two independent calls per iteration
//   mode 3: mode 1 with the acceptance as an integer threshold compare (x >> 8) < T_j
//   mode 4: mode 0 with each 32x32->64 multiply written as mul.hi.u32 + mul.lo.u32 (inline
//           PTX; SASS IMAD.HI.U32 + IMAD instead of one IMAD.WIDE.U32)
//   mode 5: mode 3 with the split multiplies of mode 4
// (modes 4/5: does the split dual-issue better than the register-pair-writing IMAD.WIDE?)
// Usage: round <mode> <warps_per_block> <blocks_per_sm> <iters>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void round1(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3, uint32_t k0, uint32_t k1) {
  const uint64_t p0 = 0xD2511F53ull * c0, p1 = 0xCD9E8D57ull * c2;
  const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0, n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
  c1 = (uint32_t)p1; c3 = (uint32_t)p0; c0 = n0; c2 = n2;
}
__device__ __forceinline__ uint32_t mulhi_ptx(uint32_t a, uint32_t b) {
  uint32_t r;
  asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t mullo_ptx(uint32_t a, uint32_t b) {
  uint32_t r;
  asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
// the low halves multiply by copies of the constants held in the constant bank (g_m): ptxas
// cannot prove them equal to the immediates, so it cannot re-fuse hi/lo into IMAD.WIDE
__constant__ uint32_t g_m[2];
__device__ __forceinline__ void round_split(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3, uint32_t k0, uint32_t k1) {
  const uint32_t h0 = mulhi_ptx(0xD2511F53u, c0), l0 = mullo_ptx(g_m[0], c0);
  const uint32_t h1 = mulhi_ptx(0xCD9E8D57u, c2), l1 = mullo_ptx(g_m[1], c2);
  const uint32_t n0 = h1 ^ c1 ^ k0, n2 = h0 ^ c3 ^ k1;
  c1 = l1; c3 = l0; c0 = n0; c2 = n2;
}
template <bool SPLIT = false>
__device__ __forceinline__ uint4 philox(uint32_t a, uint32_t b, uint32_t k0, uint32_t k1) {
  uint32_t c0 = a, c1 = b, c2 = 0x1234u, c3 = 0u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (SPLIT) round_split(c0, c1, c2, c3, k0 + r * 0x9E3779B9u, k1 + r * 0xBB67AE85u);
    else round1(c0, c1, c2, c3, k0 + r * 0x9E3779B9u, k1 + r * 0xBB67AE85u);
  }
  return make_uint4(c0, c1, c2, c3);
}

template <int MODE>
__global__ void kern(uint32_t iters, uint32_t k0, uint32_t k1, uint32_t M, float amax, uint32_t* sink) {
  extern __shared__ float sv[];
  uint32_t* st = reinterpret_cast<uint32_t*>(sv);
  for (uint32_t i = threadIdx.x; i < M; i += blockDim.x) sv[i] = (float)((i * 2654435761u) >> 8) * 0x1p-24f;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t acc = 0, c = lane, sel = blockIdx.x * blockDim.x + threadIdx.x;
  const float as = amax * 0x1p-24f;
  for (uint32_t it = 0; it < iters; ++it) {
    if (MODE == 3 || MODE == 5) {
      const uint4 x = philox<MODE == 5>(c, sel, k0, k1);
      const uint32_t j0 = __umulhi(x.x, M), j1 = __umulhi(x.z, M);
      const bool a0 = (x.y >> 8) < st[j0];
      const bool a1 = (x.w >> 8) < st[j1];
      const uint32_t b = __ballot_sync(0xffffffffu, a0 || a1);
      if (b == 0xdeadbeefu) acc += 1u;
      acc += b;
      c += 32u;
    } else if (MODE == 0 || MODE == 4) {
      const uint4 x = philox<MODE == 4>(c, sel, k0, k1);
      acc += x.x ^ x.y ^ x.z ^ x.w;
      c += 32u;
    } else {
#pragma unroll
      for (int q = 0; q < (MODE == 2 ? 2 : 1); ++q) {
        const uint4 x = philox(c + q * 7u, sel, k0, k1);
        const uint32_t j0 = __umulhi(x.x, M), j1 = __umulhi(x.z, M);
        const bool a0 = __fmul_rn(__uint2float_rn(x.y >> 8), as) < sv[j0];
        const bool a1 = __fmul_rn(__uint2float_rn(x.w >> 8), as) < sv[j1];
        const uint32_t b = __ballot_sync(0xffffffffu, a0 || a1);
        if (b == 0xdeadbeefu) acc += 1u;  // practically never: keeps the vote live
        acc += b;
      }
      c += 32u;
    }
  }
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main(int argc, char** argv) {
  const int mode = atoi(argv[1]), wpb = atoi(argv[2]), bps = atoi(argv[3]);
  const uint32_t iters = (uint32_t)atoi(argv[4]);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * bps, threads = wpb * 32;
  const uint32_t M = 1029;
  const uint32_t hm[2] = {0xD2511F53u, 0xCD9E8D57u};
  cudaMemcpyToSymbol(g_m, hm, sizeof(hm));
  uint32_t* sink;
  cudaMalloc(&sink, sizeof(uint32_t) * blocks * threads);
  auto launch = [&]() {
    if (mode == 0) kern<0><<<blocks, threads, M * 4>>>(iters, 1u, 2u, M, 1.0f, sink);
    else if (mode == 1) kern<1><<<blocks, threads, M * 4>>>(iters, 1u, 2u, M, 1.0f, sink);
    else if (mode == 2) kern<2><<<blocks, threads, M * 4>>>(iters, 1u, 2u, M, 1.0f, sink);
    else if (mode == 3) kern<3><<<blocks, threads, M * 4>>>(iters, 1u, 2u, M, 1.0f, sink);
    else if (mode == 4) kern<4><<<blocks, threads, M * 4>>>(iters, 1u, 2u, M, 1.0f, sink);
    else kern<5><<<blocks, threads, M * 4>>>(iters, 1u, 2u, M, 1.0f, sink);
  };
  launch();
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
  const double calls = (double)blocks * threads * iters * (mode == 2 ? 2 : 1);
  printf("mode %d warps/SM %d : %.3e calls/s (%.1f%% of 4.65e11)  %s\n", mode, wpb * bps, calls / (ms * 1e-3),
         100.0 * calls / (ms * 1e-3) / 4.65e11, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
