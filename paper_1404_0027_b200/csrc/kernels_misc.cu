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
  // programmatic dependent launch (gpuar_internal.cuh).  The statistics and threshold
  // kernels do NOT trigger their dependents early: a shared-vector select reads their
  // outputs before its own wait (kernels_select.cu), so it must start only after they complete.
  pdl_wait();
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
  pdl_wait();  // no early trigger (see stats_pass1)
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

// Acceptance threshold (R22).  The classic test on candidate j accepts the 24-bit
// uniform v = x >> 8 iff fl32(fl32(v 2^-24) alpha_max) < alpha_j (with
// u = v 2^-24 exact).  v -> fl32(v 2^-24 alpha_max) is non-decreasing (an exact scaling
// followed by one round-to-nearest multiply by alpha_max >= 0), so the accepted v form a
// prefix [0, T_j): T_j = min{v in [0, 2^24] : v = 2^24 or fl32(fl32(v 2^-24) alpha_max) >=
// alpha_j}, found by bisection on exactly that expression.  The trial then tests the
// integer v < T_j: bit-identical decisions, no int->float conversion or multiply per trial.
__device__ __forceinline__ uint32_t accept_threshold(float alpha_j, float amax) {
  uint32_t lo = 0u, hi = 1u << 24;  // answer in [lo, hi]
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (__fmul_rn(__fmul_rn(__uint2float_rn(mid), 0x1p-24f), amax) >= alpha_j)
      hi = mid;
    else
      lo = mid + 1u;
  }
  return lo;
}

// T_j for every reaction, plus the shared-memory prefilter of paths 2 and 3:
//  path 2: B_j = min(T_j >> 8, 65535), so that (x >> 16) < B_j accepts, (x >> 16) > B_j
//          rejects, and only (x >> 16) == B_j (probability 2^-16) needs the exact T_j;
//  path 3: per group of 2^group_shift reactions G_g = min(ceil(max T_j / 256), 65535), so that
//          (x >> 16) > G_g rejects every j of the group; otherwise the exact T_j decides.
__global__ void thresholds_kernel(const float* __restrict__ alpha, uint32_t M, const DevStats* __restrict__ stats,
                                  uint32_t* thr, uint16_t* pref, uint32_t n_pref, uint32_t group_shift, int path) {
  pdl_wait();  // no early trigger (see stats_pass1): the select kernels read thr before their wait
  const DevStats st = *stats;
  if (!st.valid) return;  // the select kernels stop on invalid statistics
  const float amax = __uint_as_float(st.amax_bits);
  const uint32_t stride = gridDim.x * blockDim.x;
  if (path != kPathSmemGroup) {
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < M; j += stride) {
      const uint32_t t = accept_threshold(__ldg(alpha + j), amax);
      thr[j] = t;
      if (path == kPathSmemBf16) pref[j] = (uint16_t)min(t >> 8, 65535u);
    }
  } else {
    for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < n_pref; g += stride) {
      const uint32_t lo = g << group_shift;
      const uint32_t hi = min(M, lo + (1u << group_shift));
      uint32_t mx = 0;
      for (uint32_t j = lo; j < hi; ++j) {
        const uint32_t t = accept_threshold(__ldg(alpha + j), amax);
        thr[j] = t;
        mx = max(mx, t);
      }
      pref[g] = (uint16_t)min((mx + 255u) >> 8, 65535u);
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
                         DevCounters* ctr, int stats_blocks, cudaStream_t st, bool pdl) {
  cudaError_t e = launch_pdl(stats_pass1, stats_blocks, kStatsThreads, 0, st, pdl, alpha, M, part_sum, part_max);
  if (e == cudaSuccess)
    e = launch_pdl(stats_pass2, 1, kStatsThreads, 0, st, pdl, (const double*)part_sum, (const uint32_t*)part_max,
                   stats_blocks, M, stats, ctr);
  return e;
}

cudaError_t launch_thresholds(const float* alpha, uint32_t M, const DevStats* stats, uint32_t* thr, uint16_t* pref,
                              uint32_t n_pref, uint32_t group_shift, int path, cudaStream_t st, bool pdl) {
  const int block = 256;
  const uint32_t n = path == kPathSmemGroup ? n_pref : M;
  const int grid = (int)std::min<uint32_t>((n + block - 1) / block, 4096u);
  return launch_pdl(thresholds_kernel, grid, block, 0, st, pdl, alpha, M, stats, thr, pref, n_pref, group_shift, path);
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
