// kernels_argmin.cu -- the paper's PRINTED GPU/AR rule (NEXT-1), fused into one kernel:
// election (pseudo-code electionStep PAPER.md:498-513) and selection
// (SelectionStep PAPER.md:528-560) for a shared propensity vector.
//
// For selection s every reaction j draws v_j (Philox counter {j >> 2, s, epoch, 3}, word
// j & 3), u_j = fl32(v_j T) with T = fl32(w alpha_max) (T_w); j is
// eligible iff u_j < D_j and is rated R_j = fl32(u_j / D_j); otherwise R_j = 1.0.  The
// selection is the lexicographic minimum of (R_j, j) -- ties to the lowest index -- and a
// minimum >= 1 is a rejection (idx -1; the paper's M+1).  DESIGN.md R16-R19.
//
// B200 mapping (vs the paper's K blocks x M threads, an RNG array and a ratings array in
// global memory): a team of g lanes per selection, each lane makes Philox calls c = rank,
// rank + g, ... and rates the 4 reactions 4c..4c+3 of each call from the shared-memory
// copy of the vector (LDS.128); the team's (rating bits, index) minimum is a shuffle
// butterfly on one 64-bit key.  No rating or random number ever touches memory.  The work
// per selection is fixed (M draws), so selections are assigned statically.
#include <algorithm>

#include "gpuar_internal.cuh"
#include "philox.cuh"

namespace gpuar {

namespace {

// election: eligible iff t < d (d = 0 is never eligible since t >= 0), rating t / d; a
// lane sees its reactions in increasing j, so a strict `<` keeps the lowest index on ties.
template <bool FASTDIV>
__device__ __forceinline__ void elect(float t, float d, float y, uint32_t j, float& bestR, uint32_t& bestJ) {
  float R = 1.0f;
  if (t < d) R = FASTDIV ? div_by_recip(t, d, y) : __fdiv_rn(t, d);
  if (R < bestR) {
    bestR = R;
    bestJ = j;
  }
}

template <bool SMEM, bool FOLD, bool FASTDIV>
__device__ __forceinline__ void argmin_teams(const SharedParams& P, uint32_t sbase, uint32_t rbase, float T,
                                             uint32_t g) {
  const float T_s = __fmul_rn(T, 0x1p-24f);
  const uint32_t M = P.M, K = P.K;
  const uint32_t calls = (M + 3u) >> 2;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t rank = lane & (g - 1u);
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t nteams = (gridDim.x * blockDim.x) / g;
  const TrialStream ts(P.seed_lo, P.seed_hi, P.epoch, kTagElection);
  // every lane of a warp runs the same number of iterations (K rounded up per warp)
  const uint32_t team0 = tid / g;
  const uint32_t warp_teams = 32u / g;
  const uint32_t team_in_warp = team0 % warp_teams;
  const uint32_t warp_first = team0 - team_in_warp;
  for (uint32_t base = warp_first; base < K; base += nteams) {
    const uint32_t s = base + team_in_warp;
    const bool live = s < K;
    const uint32_t sel = ts.sel_word(P.s0 + s);
    float bestR = 1.0f;  // sentinel: nothing eligible yet
    uint32_t bestJ = 0xffffffffu;
    auto rate = [&](uint32_t c, const Philox4& x) {
      const uint32_t j = 4u * c;
      float4 d, y = make_float4(0.f, 0.f, 0.f, 0.f);
      if constexpr (SMEM) {
        d = lds_f32x4(sbase + 16u * c);  // zero-padded to a multiple of 4 in smem
        if constexpr (FASTDIV) y = lds_f32x4(rbase + 16u * c);
      } else {
        d.x = __ldg(P.alpha + j);
        d.y = j + 1u < M ? __ldg(P.alpha + j + 1u) : 0.f;
        d.z = j + 2u < M ? __ldg(P.alpha + j + 2u) : 0.f;
        d.w = j + 3u < M ? __ldg(P.alpha + j + 3u) : 0.f;
      }
      elect<FASTDIV>(scaled_u<FOLD>(x.x, T, T_s), d.x, y.x, j, bestR, bestJ);
      elect<FASTDIV>(scaled_u<FOLD>(x.y, T, T_s), d.y, y.y, j + 1u, bestR, bestJ);
      elect<FASTDIV>(scaled_u<FOLD>(x.z, T, T_s), d.z, y.z, j + 2u, bestR, bestJ);
      elect<FASTDIV>(scaled_u<FOLD>(x.w, T, T_s), d.w, y.w, j + 3u, bestR, bestJ);
    };
    // two calls per iteration: independent IMAD.WIDE chains interleave; rated in call order
    uint32_t c = rank;
    for (; c + g < calls; c += 2u * g) {
      const Philox4 xa = ts(c, sel);
      const Philox4 xb = ts(c + g, sel);
      rate(c, xa);
      rate(c + g, xb);
    }
    if (c < calls) rate(c, ts(c, sel));
    // team minimum of the lexicographic (rating bits, index) key
    unsigned long long best = ((unsigned long long)__float_as_uint(bestR) << 32) | bestJ;
    for (uint32_t o = g >> 1; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(kFull, best, o));
    if (live && rank == 0u) {
      const bool ok = (uint32_t)(best >> 32) < 0x3f800000u;  // some rating < 1
      P.idx[s] = ok ? (int32_t)(uint32_t)best : -1;
      if (P.trials) P.trials[s] = M;  // election draws consumed
    }
  }
}

template <bool SMEM>
__global__ void __launch_bounds__(256) argmin_shared_kernel(const SharedParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  pdl_wait();  // programmatic dependent launch: nothing before the previous grids complete
  pdl_launch_dependents();
  const DevStats st = *P.stats;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t nthreads = gridDim.x * blockDim.x;
  const bool invalid = st.valid == 0u;
  const bool zero = st.amax_bits == 0u;
  // tau for every selection; degenerate / invalid outputs
  for (uint32_t s = tid; s < P.K; s += nthreads) {
    if (invalid || zero) {
      P.idx[s] = -1;
      if (P.trials) P.trials[s] = 0u;
      if (P.tau) P.tau[s] = invalid ? __uint_as_float(0x7fc00000u) : __uint_as_float(kInfBits);
    } else if (P.tau) {
      P.tau[s] = __fdiv_rn(neg_log_u1(P.seed_lo, P.seed_hi, P.s0 + s, P.epoch), st.a0f);
    }
  }
  if (invalid || zero) return;
  const uint32_t padded = (P.M + 3u) & ~3u;
  if constexpr (SMEM) {  // alpha and RN(1/alpha), zero-padded to a multiple of 4 (LDS.128 per call)
    float* sv = reinterpret_cast<float*>(smem);
    float* sr = sv + padded;
    for (uint32_t j = threadIdx.x; j < padded; j += blockDim.x) {
      const float a = j < P.M ? __ldg(P.alpha + j) : 0.f;
      sv[j] = a;
      // (a reaction with alpha < 2^-100 is eligible only for t = 0, where q = 0 for y = 0)
      sr[j] = a >= 0x1p-100f ? __frcp_rn(a) : 0.f;
    }
    __syncthreads();
  }
  const float T = __fmul_rn(P.w, __uint_as_float(st.amax_bits));
  const uint32_t calls = (P.M + 3u) >> 2;
  uint32_t g = 1u;
  while (g < 32u && g < calls) g <<= 1;  // one or a few calls per lane
  const uint32_t sb = smem_u32(smem), rb = sb + 4u * padded;
  // R23: with 2^-40 <= T <= 2^60 every eligible t > 0 is >= 2^-64 and every quotient is 0 or
  // >= 2^-24, so the reciprocal division stays clear of underflow and overflow
  const bool fastdiv = SMEM && T >= 0x1p-40f && T <= 0x1p60f;
  const bool fold = can_fold(__float_as_uint(T));
  if (fastdiv) {
    if (fold)
      argmin_teams<SMEM, true, true>(P, sb, rb, T, g);
    else
      argmin_teams<SMEM, false, true>(P, sb, rb, T, g);
  } else {
    if (fold)
      argmin_teams<SMEM, true, false>(P, sb, rb, T, g);
    else
      argmin_teams<SMEM, false, false>(P, sb, rb, T, g);
  }
}

}  // namespace

cudaError_t launch_argmin_shared(const SharedParams& p, bool smem, int grid, int block, cudaStream_t st, bool pdl) {
  if (smem) {
    const size_t sh = (size_t)((p.M + 3u) & ~3u) * 8u;  // alpha and its reciprocals
    return launch_pdl(argmin_shared_kernel<true>, grid, block, sh, st, pdl, p);
  }
  return launch_pdl(argmin_shared_kernel<false>, grid, block, 0, st, pdl, p);
}

int argmin_blocks_per_sm(bool smem, size_t bytes) {
  int n = 0;
  const cudaError_t e =
      smem ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, argmin_shared_kernel<true>, 256, bytes)
           : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, argmin_shared_kernel<false>, 256, 0);
  return e == cudaSuccess ? n : 0;
}

void set_argmin_limits(int bytes) {
  set_max_dynamic_smem(argmin_shared_kernel<true>, bytes);
}

}  // namespace gpuar
