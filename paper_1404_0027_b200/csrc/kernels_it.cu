// kernels_it.cu -- NEXT-3: the classic inverse-transform ("direct method") selection of
// PAPER.md:270-275 on the GPU, for a shared propensity vector: the smallest j with
// C_j = sum_{j' <= j} alpha_j' > u2 * alpha_0, u2 = (x >> 8) 2^-24 from Philox counter
// {0, s, epoch, 2} (R12).  This is the method the paper argues against; it is
// built so AR and IT can be compared on identical inputs on B200.
//
// C_j is the SEQUENTIAL binary64 prefix sum (the oracle's order), computed once per
// registered vector by one 1024-thread CTA.  No partial sum rounds when every alpha_j is a
// multiple of 2^q (q = the ulp exponent of the smallest non-zero alpha_j) and alpha_0 <
// 2^(q+53) (R24): then every partial sum in any order is exact, C_j = S_j, and the
// CTA computes them in parallel (per-thread contiguous blocks, a block scan, a second pass
// writing C).  A vector that fails the test (partial sums that round) gets the sequential
// chain on one thread: O(M) dependent binary64 adds, ~4 ms at M = 10^6.  Either way C is
// bit-identical to the oracle, so the selected index is too.  Each selection is then one
// Philox call and a binary search (upper bound) over C: log2(M) dependent loads from shared
// memory (M <= 27 K) or L2.
#include <algorithm>

#include "gpuar_internal.cuh"
#include "philox.cuh"

namespace gpuar {

namespace {

constexpr uint32_t kPrefixThreads = 1024;

__global__ void __launch_bounds__(kPrefixThreads) it_prefix_kernel(const float* __restrict__ alpha, uint32_t M,
                                                                   double* __restrict__ C) {
  __shared__ double s_part[kPrefixThreads / 32];
  __shared__ uint32_t s_mx[kPrefixThreads / 32], s_mn[kPrefixThreads / 32];
  __shared__ uint32_t s_exact;
  const uint32_t t = threadIdx.x, lane = t & 31u, warp = t >> 5;
  const uint32_t B = (M + kPrefixThreads - 1u) / kPrefixThreads;
  const uint32_t j0 = min(t * B, M), j1 = min(j0 + B, M);
  // pass 1: this thread's contiguous block -- sum, max and min non-zero bit pattern
  double s = 0.0;
  uint32_t mx = 0, mn = 0xffffffffu;
  for (uint32_t j = j0; j < j1; ++j) {
    const float v = __ldg(alpha + j);
    mx = max(mx, __float_as_uint(v));
    mn = min(mn, __float_as_uint(v) - 1u);
    s = __dadd_rn(s, (double)v);
  }
  // block-exclusive prefix of the thread sums: warp scans, then a scan of the warp totals
  double incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(kFull, incl, o);
    if (lane >= (uint32_t)o) incl = __dadd_rn(incl, y);
  }
  mx = __reduce_max_sync(kFull, mx);
  mn = __reduce_min_sync(kFull, mn);
  if (lane == 31u) s_part[warp] = incl;
  if (lane == 0u) s_mx[warp] = mx, s_mn[warp] = mn;
  __syncthreads();
  if (warp == 0) {
    double w = s_part[lane];
    uint32_t wm = s_mx[lane], wn = s_mn[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(kFull, w, o);
      if (lane >= (uint32_t)o) w = __dadd_rn(w, y);
    }
    wm = __reduce_max_sync(kFull, wm);
    wn = __reduce_min_sync(kFull, wn) + 1u;  // the smallest non-zero bit pattern
    s_part[lane] = w;  // inclusive over warps
    if (lane == 31u) {
      // exact iff a0 < 2^(q + 52) (then the exact sum < 2^(q + 53)); q = max(E_min, 1) - 150
      const int q = (int)max(wn >> 23, 1u) - 150;
      const int ea = (int)(uint32_t)(__double_as_longlong(w) >> 52) - 1023;
      s_exact = (wm != 0u && wm < kInfBits && ea <= q + 51) ? 1u : 0u;
    }
  }
  __syncthreads();
  if (s_exact) {
    // pass 2: C_j = (prefix before this thread's block) + the running sum -- exact
    double c = __dsub_rn(incl, s);
    if (warp > 0) c = __dadd_rn(c, s_part[warp - 1]);
    for (uint32_t j = j0; j < j1; ++j) {
      c = __dadd_rn(c, (double)__ldg(alpha + j));
      C[j] = c;
    }
  } else if (t == 0) {
    // partial sums that round (or a degenerate / invalid vector): the oracle's order
    double acc = 0.0;
    for (uint32_t j = 0; j < M; ++j) {
      acc = __dadd_rn(acc, (double)__ldg(alpha + j));
      C[j] = acc;
    }
  }
}

template <bool SMEM>
__global__ void __launch_bounds__(256) it_select_kernel(const SharedParams P, const double* __restrict__ Cg) {
  extern __shared__ __align__(16) unsigned char smem[];
  pdl_wait();  // programmatic dependent launch: nothing before the previous grids complete
  pdl_launch_dependents();
  const double* C = Cg;
  if constexpr (SMEM) {
    __shared__ uint64_t stage_bar;
    stage_to_smem(smem, Cg, 8u * P.M, &stage_bar);  // d_prefix is 256-byte aligned: no offset
    C = reinterpret_cast<const double*>(smem);
  }
  const DevStats st = *P.stats;
  const bool invalid = st.valid == 0u;
  const bool zero = st.amax_bits == 0u;
  const double a0 = C[P.M - 1];  // == the sequential alpha_0 of the oracle
  const uint32_t nthreads = gridDim.x * blockDim.x;
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < P.K; s += nthreads) {
    int32_t id = -1;
    float tau;
    if (invalid) {
      tau = __uint_as_float(0x7fc00000u);
    } else if (zero) {
      tau = __uint_as_float(kInfBits);
    } else {
      const Philox4 x = philox4x32_10(0u, P.s0 + s, P.epoch, kTagIT, P.seed_lo, P.seed_hi);
      const double target = (double)unit24(x.x) * a0;
      uint32_t lo = 0, hi = P.M - 1;  // C[M-1] = a0 > target always (u2 <= 1 - 2^-24)
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (C[mid] > target)
          hi = mid;
        else
          lo = mid + 1;
      }
      id = (int32_t)lo;
      tau = __fdiv_rn(neg_log_u1(P.seed_lo, P.seed_hi, P.s0 + s, P.epoch), st.a0f);
    }
    P.idx[s] = id;
    if (P.tau) P.tau[s] = tau;
    if (P.trials) P.trials[s] = (invalid || zero) ? 0u : 1u;  // one uniform per selection
  }
}

}  // namespace

cudaError_t launch_it_prefix(const float* alpha, uint32_t M, double* C, cudaStream_t st) {
  it_prefix_kernel<<<1, kPrefixThreads, 0, st>>>(alpha, M, C);
  return cudaGetLastError();
}

cudaError_t launch_it_select(const SharedParams& p, const double* C, bool smem, int grid, cudaStream_t st, bool pdl) {
  if (smem) return launch_pdl(it_select_kernel<true>, grid, 256, ((size_t)p.M * 8u + 15u) & ~(size_t)15, st, pdl, p, C);
  return launch_pdl(it_select_kernel<false>, grid, 256, 0, st, pdl, p, C);
}

void set_it_limits(int bytes) {
  set_max_dynamic_smem(it_select_kernel<true>, bytes);
}

}  // namespace gpuar
