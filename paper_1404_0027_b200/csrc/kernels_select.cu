// kernels_select.cu -- GPU-AR selection from ONE shared propensity vector (configs c1, c2,
// c3, c5): classic acceptance-rejection with T = alpha_max
// (PAPER.md:361-365), the first accepted trial winning (north_star; R6).
//
// Design (B200-first, not the paper's election/argmin kernels of PAPER.md:498-555):
//  * one persistent launch; the vector (or an exact prefilter of it) is staged once per
//    CTA in shared memory;
//  * a selection is worked by a TEAM of g lanes (g = 1..32, a power of two picked on the
//    device from K and p): in round q lane `rank` makes Philox call c = q*g + rank, i.e.
//    trials 2c and 2c+1, so a round covers the contiguous trial block [2qg, 2(q+1)g).
//    The team's ballot + __ffs picks the lowest accepting lane, and within it the even
//    trial first -> the globally smallest accepted trial index, independent of g;
//  * teams that finish take the next selection from a warp-local pool refilled by one
//    64-bit atomic per `grab` selections (work stealing: no tail from geometric trial
//    counts);
//  * tau is a separate, fully coalesced grid-stride phase.
#include <algorithm>

#include "gpuar_internal.cuh"
#include "philox.cuh"

namespace gpuar {

namespace {

template <int PATH>
__device__ __forceinline__ bool accept(float t, uint32_t j, const void* sm, const float* __restrict__ alpha,
                                       uint32_t group_shift) {
  if constexpr (PATH == kPathSmemF32) {
    return t < static_cast<const float*>(sm)[j];
  } else if constexpr (PATH == kPathSmemBf16) {
    // bf16(code) <= alpha_j < bf16(code + 1): decide without the exact value unless t
    // falls inside that bracket (exact: DESIGN.md "prefilter").
    const uint32_t code = static_cast<const uint16_t*>(sm)[j];
    const float lo = __uint_as_float(code << 16);
    const float hi = __uint_as_float((code + 1u) << 16);
    if (t < lo) return true;
    if (t >= hi) return false;
    return t < __ldg(alpha + j);
  } else {
    // group maximum rounded up to bf16 is an upper bound of alpha_j
    const float ub = __uint_as_float(static_cast<uint32_t>(static_cast<const uint16_t*>(sm)[j >> group_shift]) << 16);
    if (t >= ub) return false;
    return t < __ldg(alpha + j);
  }
}

template <int PATH>
__global__ void __launch_bounds__(1024, 1) select_shared_kernel(const SharedParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  const DevStats st = *P.stats;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t nthreads = gridDim.x * blockDim.x;
  const bool invalid = st.valid == 0u;
  const bool zero = st.amax_bits == 0u;

  // ---- phase A: tau for every selection; degenerate / invalid outputs
  for (uint32_t s = tid; s < P.K; s += nthreads) {
    if (invalid || zero) {
      P.idx[s] = -1;
      if (P.trials) P.trials[s] = 0u;
      if (P.tau) P.tau[s] = invalid ? __uint_as_float(0x7fc00000u) : __uint_as_float(kInfBits);
    } else if (P.tau) {
      P.tau[s] = __fdiv_rn(neg_log_u1(P.seed_lo, P.seed_hi, P.s0 + s, P.epoch), st.a0f);
    }
  }
  if (invalid || zero) return;  // uniform over the grid; the pool counter is untouched

  // ---- phase B: stage the vector (path 1) or its prefilter (paths 2, 3) in smem
  if constexpr (PATH == kPathSmemF32) {
    float* sv = reinterpret_cast<float*>(smem);
    for (uint32_t j = threadIdx.x; j < P.M; j += blockDim.x) sv[j] = __ldg(P.alpha + j);
  } else {
    uint16_t* pf = reinterpret_cast<uint16_t*>(smem);
    for (uint32_t g = threadIdx.x; g < P.n_pref; g += blockDim.x) pf[g] = __ldg(P.prefilter + g);
  }
  __syncthreads();

  // ---- phase C: trials
  const float amax = __uint_as_float(st.amax_bits);
  const uint32_t M = P.M, K = P.K;
  const uint32_t half = P.max_trials >> 1;                 // calls whose odd trial is < max_trials
  const uint32_t calls = half + (P.max_trials & 1u);       // calls whose even trial is < max_trials
  // team size: enough teams to cover K, and g*p <= ~1/4 so the last round wastes little
  uint32_t g = 32u;
  {
    const uint32_t ratio = max(1u, nthreads / max(K, 1u));
    g = min(g, 1u << (31 - __clz(ratio)));
    const float lim = st.p > 0.f ? 0.25f / st.p : 32.f;
    const uint32_t gl = lim >= 32.f ? 32u : (lim < 1.f ? 1u : (uint32_t)lim);
    g = min(g, 1u << (31 - __clz(gl)));
  }
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t tbase = lane & ~(g - 1u);
  const uint32_t rank = lane & (g - 1u);
  const uint32_t tmask = (g == 32u) ? kFull : (((1u << g) - 1u) << tbase);
  const bool leader = rank == 0u;
  const unsigned long long grab = st.grab;

  uint32_t my = kNone;  // local selection index of this lane's team
  uint32_t q = 0;       // round within the selection
  unsigned long long pool_next = 0, pool_end = 0;
  bool exhausted = false;

  while (true) {
    uint32_t need = __ballot_sync(kFull, leader && my == kNone);
    while (need != 0u && !exhausted) {
      if (pool_next >= pool_end) {
        unsigned long long base = 0;
        if (lane == 0u) base = atomicAdd(&P.ctr->next, grab);
        base = __shfl_sync(kFull, base, 0);
        if (base >= K) {
          exhausted = true;
          break;
        }
        pool_next = base;
        pool_end = min(base + grab, (unsigned long long)K);
      }
      const uint32_t avail = (uint32_t)(pool_end - pool_next);
      const uint32_t r = __popc(need & lanemask_lt());
      uint32_t mine = kNone;
      if (((need >> lane) & 1u) && r < avail) mine = (uint32_t)pool_next + r;
      const uint32_t got = __shfl_sync(kFull, mine, tbase);
      if (got != kNone) {
        my = got;
        q = 0;
      }
      pool_next += min((uint32_t)__popc(need), avail);
      need = __ballot_sync(kFull, leader && my == kNone);
    }
    if (exhausted && __all_sync(kFull, my == kNone)) break;

    const bool active = my != kNone;
    const uint32_t c = q * g + rank;
    const Philox4 x = philox4x32_10(c, P.s0 + my, P.epoch, kTagTrials, P.seed_lo, P.seed_hi);
    const uint32_t j0 = __umulhi(x.x, M);
    const uint32_t j1 = __umulhi(x.z, M);
    const float t0 = __fmul_rn(unit24(x.y), amax);
    const float t1 = __fmul_rn(unit24(x.w), amax);
    const bool a0 = active && c < calls && accept<PATH>(t0, j0, smem, P.alpha, P.group_shift);
    const bool a1 = active && !a0 && c < half && accept<PATH>(t1, j1, smem, P.alpha, P.group_shift);
    const uint32_t b = __ballot_sync(kFull, a0 || a1) & tmask;
    const uint32_t src = b ? (uint32_t)(__ffs(b) - 1) : lane;
    const uint32_t pick_j = a0 ? j0 : j1;
    const uint32_t pick_t = a0 ? 2u * c + 1u : 2u * c + 2u;
    const uint32_t wj = __shfl_sync(kFull, pick_j, src);
    const uint32_t wt = __shfl_sync(kFull, pick_t, src);
    const bool out_of_calls = (q + 1u) * g >= calls;
    if (active) {
      if (b != 0u || out_of_calls) {
        if (leader) {
          P.idx[my] = b ? (int32_t)wj : -1;
          if (P.trials) P.trials[my] = b ? wt : P.max_trials;
        }
        my = kNone;
      } else {
        ++q;
      }
    }
  }

  // ---- the last CTA out resets the work-stealing ticket for the next launch
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int prev = atomicAdd(&P.ctr->done, 1u);
    if (prev == gridDim.x - 1u) {
      P.ctr->next = 0ull;
      P.ctr->done = 0u;
      __threadfence();
    }
  }
}

template <int PATH>
void set_limit(int bytes) {
  cudaFuncSetAttribute(select_shared_kernel<PATH>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

}  // namespace

cudaError_t launch_select_shared(const SharedParams& p, int path, int grid, int block, cudaStream_t st) {
  const size_t sh = p.smem_bytes;
  switch (path) {
    case kPathSmemF32:
      select_shared_kernel<kPathSmemF32><<<grid, block, sh, st>>>(p);
      break;
    case kPathSmemBf16:
      select_shared_kernel<kPathSmemBf16><<<grid, block, sh, st>>>(p);
      break;
    case kPathSmemGroup:
      select_shared_kernel<kPathSmemGroup><<<grid, block, sh, st>>>(p);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

int select_shared_blocks_per_sm(int path, int block, size_t smem) {
  int n = 0;
  cudaError_t e = cudaErrorInvalidValue;
  if (path == kPathSmemF32)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, select_shared_kernel<kPathSmemF32>, block, smem);
  else if (path == kPathSmemBf16)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, select_shared_kernel<kPathSmemBf16>, block, smem);
  else if (path == kPathSmemGroup)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, select_shared_kernel<kPathSmemGroup>, block, smem);
  return e == cudaSuccess ? n : 0;
}

void set_select_shared_limits(int bytes) {
  set_limit<kPathSmemF32>(bytes);
  set_limit<kPathSmemBf16>(bytes);
  set_limit<kPathSmemGroup>(bytes);
}

}  // namespace gpuar
