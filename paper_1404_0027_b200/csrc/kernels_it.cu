// kernels_it.cu -- NEXT-3: the classic inverse-transform ("direct method") selection of
// PAPER.md:270-275 on the GPU, for a shared propensity vector: the smallest j with
// C_j = sum_{j' <= j} alpha_j' > u2 * alpha_0, u2 = (x >> 8) 2^-24 from Philox counter
// {0, s, epoch, 2} (R12).  This is the method the paper argues against; it is
// built so AR and IT can be compared on identical inputs on B200.
//
// C_j is the SEQUENTIAL binary64 prefix sum (the oracle's order), computed once per
// registered vector by one thread -- O(M) and latency-bound (~4 ms at M = 10^6), but
// bit-identical to the oracle, so the selected index is too.  Each selection is then one
// Philox call and a binary search (upper bound) over C: log2(M) dependent loads from shared
// memory (M <= 27 K) or L2.
#include <algorithm>

#include "gpuar_internal.cuh"
#include "philox.cuh"

namespace gpuar {

namespace {

__global__ void it_prefix_kernel(const float* __restrict__ alpha, uint32_t M, double* __restrict__ C) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double acc = 0.0;
  for (uint32_t j = 0; j < M; ++j) {
    acc += (double)__ldg(alpha + j);
    C[j] = acc;
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
  it_prefix_kernel<<<1, 32, 0, st>>>(alpha, M, C);
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
