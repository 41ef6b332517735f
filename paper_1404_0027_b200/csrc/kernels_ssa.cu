// kernels_ssa.cu -- NEXT-2: the full SSA loop around the selector:
// "two uniform random numbers u1 and u2 ... tau = (1/a0) ln(1/u1) ... the index j of the
// next reaction ... Then the system is updated using v_j, t <- t + tau", with the next
// reaction chosen by the classic AR hot path.
//
// One warp owns one realization at a time; its state X (N int32) and its propensity row
// (M binary32) live in the warp's shared-memory slice, the reaction network (reactants,
// rate constants, sparse change vectors) is staged once per CTA.  Per step: mass-action
// propensities (R20) in the row, alpha_max / alpha_0 by row_reduce (the matrix
// kernel's code and order), tau, the first-accept trials of kernels_rows.cu,
// then X += v_j and t += tau -- nothing leaves the SM until the run ends.  Realization
// k is selection s0 + k and step i uses epoch epoch0 + i, so every step is bit-identical
// to a gpuar_select on the same row.
#include <algorithm>

#include "gpuar_internal.cuh"
#include "philox.cuh"

namespace gpuar {

namespace {

// Mass-action propensity, branch-free.  Per reaction a 16-byte descriptor {i0, i1, c, h}:
// i0 = r0 (or N, a dummy species pinned at 1 in shared memory), i1 = r1 (or N for none and
// for dimerisation), c = rate, h = 0.5 for dimerisation else 1.  Then
//   a = ((c * x0) * x1) * h,  x1 = max(x0 - 1, 0) for dimerisation, X[i1] otherwise.
// Multiplying by exactly 1.0 is the identity and c * 0 = +0, so this is bit-identical to
// the oracle's branchy left-to-right definition (R20): order 0 -> c, order 1 ->
// c x0, two species -> (c x0) x1, dimer -> ((c x)(x-1)) / 2 with +0 for x < 2.
__device__ __forceinline__ float propensity(uint32_t xs, const int4 d) {
  const int32_t x0 = (int32_t)lds_u32(xs + 4u * (uint32_t)d.x);
  const int32_t xb = (int32_t)lds_u32(xs + 4u * (uint32_t)d.y);
  const float h = __int_as_float(d.w);
  const int32_t x1 = (h == 0.5f) ? max(x0 - 1, 0) : xb;
  return __fmul_rn(__fmul_rn(__fmul_rn(__int_as_float(d.z), (float)x0), (float)x1), h);
}

template <bool FOLD, bool CAP>
__device__ __forceinline__ bool ssa_round(const TrialStream& ts, uint32_t c0, uint32_t sel, uint32_t row_s, uint32_t M,
                                          float amax, float amax_s, uint32_t half, uint32_t calls, uint32_t lane,
                                          int32_t& id) {
  const uint32_t c = c0 + lane;
  const Philox4 x = ts(c, sel);
  const uint32_t j0 = __umulhi(x.x, M);
  const uint32_t j1 = __umulhi(x.z, M);
  const float v0 = lds_f32(row_s + 4u * j0);
  const float v1 = lds_f32(row_s + 4u * j1);
  const bool a0 = (!CAP || c < calls) & (scaled_u<FOLD>(x.y, amax, amax_s) < v0);
  const bool a1 = (!CAP || c < half) & (scaled_u<FOLD>(x.w, amax, amax_s) < v1);
  const uint32_t b = __ballot_sync(kFull, a0 || a1);
  if (b != 0u) {
    id = (int32_t)__shfl_sync(kFull, a0 ? j0 : j1, __ffs(b) - 1);
    return true;
  }
  return false;
}

template <bool FOLD>
__device__ __forceinline__ void ssa_trials(const TrialStream& ts, uint32_t sel, uint32_t row_s, uint32_t M,
                                           float amax, uint32_t half, uint32_t calls, uint32_t lane, int32_t& id) {
  const float amax_s = __fmul_rn(amax, 0x1p-24f);
  // rounds entirely below max_trials skip the cap tests (c0 + 31 < half), as in row_trials
  const uint32_t free_end = half & ~31u;
  uint32_t c0 = 0;
  for (; c0 < free_end; c0 += 32u)
    if (ssa_round<FOLD, false>(ts, c0, sel, row_s, M, amax, amax_s, half, calls, lane, id)) return;
  for (; c0 < calls; c0 += 32u)
    if (ssa_round<FOLD, true>(ts, c0, sel, row_s, M, amax, amax_s, half, calls, lane, id)) return;
}

__global__ void __launch_bounds__(768, 1) ssa_kernel(const SsaParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t warps = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  const uint32_t M = P.M, N = P.N, D = P.D;
  // ---- stage the network: descriptors (M x int4), didx / dval (M x D)
  int4* s_desc = reinterpret_cast<int4*>(smem);
  int32_t* s_didx = reinterpret_cast<int32_t*>(s_desc + M);
  int32_t* s_dval = s_didx + D * M;
  for (uint32_t j = threadIdx.x; j < M; j += blockDim.x) {
    const int32_t r0 = P.reac[2u * j], r1 = P.reac[2u * j + 1u];
    const bool dimer = r0 >= 0 && r1 == r0;
    s_desc[j] = make_int4(r0 >= 0 ? r0 : (int32_t)N, (r1 >= 0 && !dimer) ? r1 : (int32_t)N,
                          __float_as_int(P.rate[j]), __float_as_int(dimer ? 0.5f : 1.0f));
  }
  for (uint32_t i = threadIdx.x; i < D * M; i += blockDim.x) {
    s_didx[i] = P.didx[i];
    s_dval[i] = P.dval[i];
  }
  // dependency lists (CSR): after reaction j fires only its dependents' propensities change
  int32_t* s_dptr = s_dval + D * M;
  int32_t* s_didxs = s_dptr + (M + 1u);
  const bool deps = P.dep_ptr != nullptr;
  if (deps) {
    for (uint32_t i = threadIdx.x; i <= M; i += blockDim.x) s_dptr[i] = P.dep_ptr[i];
    for (uint32_t i = threadIdx.x; i < P.dep_total; i += blockDim.x) s_didxs[i] = P.dep_idx[i];
  }
  __syncthreads();
  const uint32_t desc_s = smem_u32(s_desc);
  unsigned char* mine = smem + P.net_bytes + (size_t)warp * P.warp_bytes;
  const uint32_t row_s = smem_u32(mine);
  const uint32_t xs = row_s + ((4u * M + 15u) & ~15u);
  int32_t* Xs = reinterpret_cast<int32_t*>(mine + ((4u * M + 15u) & ~15u));
  float* row = reinterpret_cast<float*>(mine);

  const uint32_t half = P.max_trials >> 1;
  const uint32_t calls = half + (P.max_trials & 1u);
  TrialStream ts(P.seed_lo, P.seed_hi, P.epoch0);
  const uint32_t WT = gridDim.x * warps;

  for (uint32_t k = blockIdx.x * warps + warp; k < P.K; k += WT) {
    int32_t* Xg = P.X + (size_t)k * N;
    for (uint32_t i = lane; i < N; i += 32u) Xs[i] = Xg[i];
    if (lane == 0) Xs[N] = 1;  // dummy species: absent reactant
    double t = P.t[k];
    uint32_t fired = 0;
    const uint32_t s = P.s0 + k;
    __syncwarp();
    float nlog = 0.f;  // -ln(u1) of step (step & ~31) + lane: tau draws 32 steps at a time
    for (int32_t step = 0; step < P.n_steps; ++step) {
      if ((step & 31) == 0) nlog = neg_log_u1(P.seed_lo, P.seed_hi, s, P.epoch0 + (uint32_t)(step + (int32_t)lane));
      // ---- propensities -> row: all of them on the first step of the call (else only the
      // dependents of the last fired reaction, already updated below), then alpha_max (bits)
      // and alpha_0 over the whole row in the fixed order of the matrix kernel (row_reduce)
      if (step == 0 || !deps) {
        for (uint32_t j = lane; j < M; j += 32u) row[j] = propensity(xs, lds_i4(desc_s + 16u * j));
        __syncwarp();
      }
      uint32_t mx;
      double acc;
      row_reduce_counted(row_s, M, lane, mx, acc);
      __syncwarp();  // row complete before the gathers
      if (mx >= kInfBits) {  // invalid propensity: sticky EPROPENSITY, stop this realization
        if (lane == 0) atomicOr(&P.ctr->err, 1u);
        break;
      }
      if (mx == 0u) break;  // nothing can fire: halted
      const uint32_t epoch = P.epoch0 + (uint32_t)step;
      const float tau = __fdiv_rn(__shfl_sync(kFull, nlog, step & 31), __double2float_rn(acc));
      if (t + (double)tau > P.t_end) break;  // the next event is past t_end
      ts.set_epoch(epoch);
      int32_t id = -1;
      const float amax = __uint_as_float(mx);
      if (can_fold(mx))
        ssa_trials<true>(ts, ts.sel_word(s), row_s, M, amax, half, calls, lane, id);
      else
        ssa_trials<false>(ts, ts.sel_word(s), row_s, M, amax, half, calls, lane, id);
      if (id >= 0) {  // X += v_id, t += tau  (rejected: no event this step, R21)
        if (lane < D) {
          const int32_t sp = s_didx[(uint32_t)id * D + lane];
          if (sp >= 0) atomicAdd(&Xs[sp], s_dval[(uint32_t)id * D + lane]);
        }
        t += (double)tau;
        ++fired;
        if (deps) {  // refresh the propensities that read a changed species
          __syncwarp();
          const int32_t d0 = s_dptr[id], d1 = s_dptr[id + 1];
          for (int32_t d = d0 + (int32_t)lane; d < d1; d += 32) {
            const uint32_t j = (uint32_t)s_didxs[d];
            row[j] = propensity(xs, lds_i4(desc_s + 16u * j));
          }
        }
      }
      __syncwarp();
    }
    __syncwarp();
    for (uint32_t i = lane; i < N; i += 32u) Xg[i] = Xs[i];
    if (lane == 0) {
      P.t[k] = t;
      if (P.steps) P.steps[k] = fired;
    }
    __syncwarp();
  }
}

}  // namespace

cudaError_t launch_ssa(const SsaParams& p, int grid, int warps, cudaStream_t st) {
  const size_t sh = (size_t)p.net_bytes + (size_t)warps * p.warp_bytes;
  ssa_kernel<<<grid, warps * 32, sh, st>>>(p);
  return cudaGetLastError();
}

int ssa_blocks_per_sm(int warps, size_t smem) {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, ssa_kernel, warps * 32, smem) != cudaSuccess) return 0;
  return n;
}

void set_ssa_limits(int bytes) {
  set_max_dynamic_smem(ssa_kernel, bytes);
}

}  // namespace gpuar
