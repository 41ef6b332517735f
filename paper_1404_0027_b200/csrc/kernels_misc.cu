// kernels_misc.cu -- shared-vector statistics (alpha_max, alpha_0, validity), the exact
// shared-memory prefilter for large M, the validation histogram and the Philox roofline
// microkernel.
//
// alpha_0 = sum_j alpha_j and the threshold T = max_j alpha_j
// (PAPER.md:361-365 with w = 1, R2) are computed once per registered vector.
// alpha_max is the maximum of the uint32 bit patterns: for +0 and positive finite floats
// that order is the numeric order, and any negative / -0.0 / NaN / Inf pattern is >=
// 0x7f800000, so one max both finds alpha_max exactly and validates the input.
// alpha_0 is summed in binary64 in a fixed tree (deterministic: same bits on every run
// and every rank, because the launch shape depends only on M).
#include <algorithm>

#include "gpuar_internal.cuh"
#include "philox.cuh"

namespace gpuar {

namespace {

constexpr int kStatsThreads = 256;

__device__ __forceinline__ void block_reduce(double& acc, uint32_t& mx, double* sh_sum, uint32_t* sh_max) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
  mx = __reduce_max_sync(kFull, mx);
  if (lane == 0) {
    sh_sum[warp] = acc;
    sh_max[warp] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    uint32_t m = 0;
    for (int w = 0; w < kStatsThreads / 32; ++w) {
      a += sh_sum[w];
      m = max(m, sh_max[w]);
    }
    acc = a;
    mx = m;
  }
}

__global__ void __launch_bounds__(kStatsThreads) stats_pass1(const float* __restrict__ alpha, uint32_t M,
                                                             double* part_sum, uint32_t* part_max) {
  __shared__ double sh_sum[kStatsThreads / 32];
  __shared__ uint32_t sh_max[kStatsThreads / 32];
  const uint32_t chunk = (M + gridDim.x - 1) / gridDim.x;
  const uint32_t lo = blockIdx.x * chunk;
  const uint32_t hi = min(M, lo + chunk);
  double acc = 0.0;
  uint32_t mx = 0;
  for (uint32_t j = lo + threadIdx.x; j < hi; j += kStatsThreads) {
    const float a = __ldg(alpha + j);
    mx = max(mx, __float_as_uint(a));
    acc += (double)a;
  }
  block_reduce(acc, mx, sh_sum, sh_max);
  if (threadIdx.x == 0) {
    part_sum[blockIdx.x] = acc;
    part_max[blockIdx.x] = mx;
  }
}

__global__ void __launch_bounds__(kStatsThreads) stats_pass2(const double* part_sum, const uint32_t* part_max,
                                                             int nparts, uint32_t M, DevStats* stats,
                                                             DevCounters* ctr) {
  __shared__ double sh_sum[kStatsThreads / 32];
  __shared__ uint32_t sh_max[kStatsThreads / 32];
  double acc = 0.0;
  uint32_t mx = 0;
  for (int i = threadIdx.x; i < nparts; i += kStatsThreads) {
    acc += part_sum[i];
    mx = max(mx, part_max[i]);
  }
  block_reduce(acc, mx, sh_sum, sh_max);
  if (threadIdx.x == 0) {
    DevStats s;
    s.amax_bits = mx;
    s.valid = mx < kInfBits ? 1u : 0u;
    s.a0d = acc;
    s.a0f = __double2float_rn(acc);
    double p = 0.0;
    if (s.valid && mx != 0) p = acc / ((double)M * (double)__uint_as_float(mx));
    s.p = (float)p;
    // ~8192 expected trials per atomic grab, 1 .. 2048 selections (the select kernel raises
    // it to at least one selection per team of the warp).
    double g = 8192.0 * p;
    uint32_t grab = g < 1.0 ? 1u : (g > 2048.0 ? 2048u : (uint32_t)g);
    s.grab = grab;
    s.pad = 0;
    *stats = s;
    for (uint32_t i = 0; i < kStripes; ++i) ctr->next[0][i] = ctr->next[1][i] = 0ull;
    if (!s.valid) atomicOr(&ctr->err, 1u);
  }
}

// Path 2: per-element bf16 truncation t_j = bits(alpha_j) >> 16, so that
// bf16(t_j) <= alpha_j < bf16(t_j + 1).  Path 3: per-group bf16 round-up of the group
// maximum, an upper bound of every alpha_j in the group.
__global__ void prefilter_kernel(const float* __restrict__ alpha, uint32_t M, uint16_t* pref, uint32_t n_pref,
                                 uint32_t group_shift, int path) {
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < n_pref; g += gridDim.x * blockDim.x) {
    if (path == kPathSmemBf16) {
      pref[g] = (uint16_t)(__float_as_uint(__ldg(alpha + g)) >> 16);
    } else {
      const uint32_t lo = g << group_shift;
      const uint32_t hi = min(M, lo + (1u << group_shift));
      uint32_t mx = 0;
      for (uint32_t j = lo; j < hi; ++j) mx = max(mx, __float_as_uint(__ldg(alpha + j)));
      // round up to bf16; saturates to +inf (0x7f80), still an upper bound
      const uint32_t up = mx >= 0x7f7f0001u ? 0x7f80u : ((mx + 0xffffu) >> 16);
      pref[g] = (uint16_t)up;
    }
  }
}

// Validation histogram (untimed): hist[M+1] (bin M = idx -1), totals = {sum trials, #rejected}.
__global__ void histogram_kernel(const int32_t* __restrict__ idx, const uint32_t* __restrict__ trials, uint32_t K,
                                 uint32_t M, unsigned long long* hist, unsigned long long* totals, int use_smem) {
  extern __shared__ uint32_t sh_hist[];
  if (use_smem) {
    for (uint32_t b = threadIdx.x; b <= M; b += blockDim.x) sh_hist[b] = 0;
    __syncthreads();
  }
  unsigned long long tsum = 0, rej = 0;
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < K; s += gridDim.x * blockDim.x) {
    const int32_t j = idx[s];
    const uint32_t bin = (j >= 0 && (uint32_t)j < M) ? (uint32_t)j : M;
    rej += (bin == M);
    if (trials) tsum += trials[s];
    if (use_smem)
      atomicAdd(&sh_hist[bin], 1u);
    else
      atomicAdd(&hist[bin], 1ull);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    tsum += __shfl_xor_sync(kFull, tsum, o);
    rej += __shfl_xor_sync(kFull, rej, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (tsum) atomicAdd(&totals[0], tsum);
    if (rej) atomicAdd(&totals[1], rej);
  }
  if (use_smem) {
    __syncthreads();
    for (uint32_t b = threadIdx.x; b <= M; b += blockDim.x)
      if (sh_hist[b]) atomicAdd(&hist[b], (unsigned long long)sh_hist[b]);
  }
}

// Philox generate-and-fold: `calls` Philox4x32-10 calls per thread, outputs folded into
// one word so the work cannot be eliminated.  Counter {c, tid, 0, 0} as in the trials.
__global__ void __launch_bounds__(256) bench_philox_kernel(uint32_t n_threads, uint32_t calls, uint32_t k0,
                                                           uint32_t k1, uint32_t* sink) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= n_threads) return;
  uint32_t acc = 0;
  for (uint32_t c = 0; c < calls; ++c) {
    const Philox4 x = philox4x32_10(c, tid, 0u, 0u, k0, k1);
    acc += (x.x ^ x.y) + (x.z ^ x.w);
  }
  sink[tid] = acc;
}

}  // namespace

cudaError_t launch_stats(const float* alpha, uint32_t M, double* part_sum, uint32_t* part_max, DevStats* stats,
                         DevCounters* ctr, int stats_blocks, cudaStream_t st) {
  stats_pass1<<<stats_blocks, kStatsThreads, 0, st>>>(alpha, M, part_sum, part_max);
  stats_pass2<<<1, kStatsThreads, 0, st>>>(part_sum, part_max, stats_blocks, M, stats, ctr);
  return cudaGetLastError();
}

cudaError_t launch_prefilter(const float* alpha, uint32_t M, uint16_t* pref, uint32_t n_pref, uint32_t group_shift,
                             int path, cudaStream_t st) {
  const int block = 256;
  const int grid = (int)std::min<uint32_t>((n_pref + block - 1) / block, 4096u);
  prefilter_kernel<<<grid, block, 0, st>>>(alpha, M, pref, n_pref, group_shift, path);
  return cudaGetLastError();
}

cudaError_t launch_histogram(const int32_t* idx, const uint32_t* trials, uint32_t K, uint32_t M,
                             unsigned long long* hist, unsigned long long* totals, int grid, cudaStream_t st) {
  const int block = 512;
  const size_t sh = (size_t)(M + 1) * sizeof(uint32_t);
  const int use_smem = sh <= 48 * 1024 ? 1 : 0;
  const int g = (int)std::min<uint32_t>((K + block - 1) / block, (uint32_t)grid);
  histogram_kernel<<<g > 0 ? g : 1, block, use_smem ? sh : 0, st>>>(idx, trials, K, M, hist, totals, use_smem);
  return cudaGetLastError();
}

cudaError_t launch_bench_philox(uint32_t n_threads, uint32_t calls, uint32_t seed_lo, uint32_t seed_hi,
                                uint32_t* sink, cudaStream_t st) {
  const int block = 256;
  bench_philox_kernel<<<(n_threads + block - 1) / block, block, 0, st>>>(n_threads, calls, seed_lo, seed_hi, sink);
  return cudaGetLastError();
}

}  // namespace gpuar
