// gpuar_internal.cuh -- device-side structures, PTX helpers and kernel launchers shared
// by libgpuar's translation units.  Not part of the ABI (include/gpuar.h is).
#pragma once
#include <cstdint>
#include <utility>
#include <cuda_runtime.h>

namespace gpuar {

constexpr uint32_t kFull = 0xffffffffu;
constexpr uint32_t kNone = 0xffffffffu;
constexpr uint32_t kInfBits = 0x7f800000u;   // a valid propensity's bits are < this

// Shared-vector statistics (written by the stats kernel, read by the select kernels).
struct DevStats {
  uint32_t amax_bits;  // bits of alpha_max = max over uint bits (order-free, exact)
  uint32_t valid;      // 1 iff every bit pattern < 0x7f800000 (+0 or positive finite)
  float a0f;           // fl32(alpha_0)
  float p;             // alpha_0 / (M alpha_max), 0 if alpha_max == 0
  double a0d;          // alpha_0 in binary64, fixed reduction tree
  uint32_t grab;       // work-stealing chunk (selections per atomic grab)
  uint32_t pad;
};

// Per-handle device counters.
constexpr uint32_t kStripes = 64;  // work-stealing tickets, one per stripe of selections
struct DevCounters {
  // Tickets, double-buffered: launch n of the shared-vector kernel uses set n & 1 and zeroes
  // set (n + 1) & 1 for the next launch (the launch before it, which used that set, has
  // completed in stream order) -- no end-of-launch counter or fence.
  unsigned long long next[2][kStripes];
  unsigned int err;                   // sticky EPROPENSITY flag (cleared by the host)
  unsigned int team;                  // team size of the last shared-vector classic launch
};

enum Path : int {
  kPathNone = 0,
  kPathSmemF32 = 1,    // shared vector: its acceptance thresholds T_j (32-bit) all in shared memory
  kPathSmemBf16 = 2,   // shared vector: 16-bit threshold brackets in smem, exact T_j in L2
  kPathSmemGroup = 3,  // shared vector: 16-bit group bounds of T_j in smem, exact T_j in L2
  kPathRows = 4,       // per-realization K x M matrix, bulk-async staged rows
};

enum Rule : int {
  kRuleClassic = 0,  // classic AR, first accept (the north_star hot path)
  kRuleArgmin = 1,   // the paper's printed election + argmin selection
  kRuleIT = 2,       // inverse transform, the classic direct method
  kRuleITScan = 3,   // the same, per-realization matrix as a linear scan from j = 0
};

struct SharedParams {
  const float* alpha;        // M floats (device)
  const uint32_t* thr;       // classic rule: acceptance thresholds T_j (device, M words)
  const uint16_t* prefilter; // paths 2/3: 16-bit threshold brackets / group bounds (device)
  const DevStats* stats;
  DevCounters* ctr;
  int32_t* idx;
  float* tau;
  uint32_t* trials;
  uint32_t M;
  uint32_t K;
  uint32_t s0;
  uint32_t epoch;
  uint32_t seed_lo, seed_hi;
  uint32_t max_trials;
  uint32_t n_pref;           // number of prefilter entries (paths 2/3)
  uint32_t group_shift;      // path 3: log2(group size)
  uint32_t smem_bytes;       // bytes of the staged vector / prefilter
  float w;                   // argmin rule: T = fl32(w * alpha_max)
  uint32_t grab_override;    // tuning: fixed selections per ticket grab (0 = model)
  uint32_t team_override;    // tuning: fixed team size g (power of two 1..32; 0 = model)
  uint32_t fair;             // work stealing: max(1, K / warps of the grid)
  uint32_t first_base;       // static first chunk before the team minimum: 3 fair / 4, or, with
                             // fair <= 4, ceil(ceil(K / kStripes) / max(1, warps / kStripes))
                             // (static chunks that cover each stripe: no tickets at all)
  uint32_t no_prefetch;      // tuning: 1 = fetch tickets on demand
  uint32_t no_endgame;       // tuning: 1 = the lane loop never hands its last selections to the whole warp
  uint32_t phase;            // ticket set of this launch (DevCounters::next)
  // multi-epoch launches (gpuar_select_epochs): K above is the number of work items
  // n_epochs * Ksel; item q is selection q mod Ksel at epoch + q / Ksel, output slot q
  uint32_t Ksel;             // selections per epoch
  uint32_t n_epochs;         // epochs in this launch (1: a plain gpuar_select)
  float kinv;                // fl32(1 / Ksel): q / Ksel to within one, then corrected
};

// Item q of a multi-epoch launch -> (epoch offset e, selection s): q = e * Ksel + s.  The
// binary32 estimate is within one of q / Ksel for e < 2^16 (relative error < 2^-22); one
// exact correction step in 64-bit arithmetic.
__device__ __forceinline__ void split_item(uint32_t q, uint32_t Ksel, float kinv, uint32_t& e, uint32_t& s) {
  e = __float2uint_rz(__fmul_rn(__uint2float_rn(q), kinv));
  long long r = (long long)q - (long long)e * Ksel;
  if (r < 0) {
    --e;
    r += Ksel;
  } else if (r >= (long long)Ksel) {
    ++e;
    r -= Ksel;
  }
  s = (uint32_t)r;
}

struct RowsParams {
  const float* alpha;        // K rows, pitch ld floats, 16-byte aligned base
  DevCounters* ctr;
  int32_t* idx;
  float* tau;
  uint32_t* trials;
  float* amax_out;           // gpuar_row_stats only
  double* a0_out;            // gpuar_row_stats only
  uint64_t ld;
  uint32_t M;
  uint32_t K;
  uint32_t s0;
  uint32_t epoch;
  uint32_t seed_lo, seed_hi;
  uint32_t max_trials;
  uint32_t log2_stages;      // ring depth per warp = 2^log2_stages (1, 2 or 4)
  uint32_t stage_bytes;      // bytes per ring slot (multiple of 16)
  uint32_t stats_only;       // 1: gpuar_row_stats (no trials)
  int rule;                  // kRuleClassic / kRuleArgmin / kRuleIT / kRuleITScan
  float w;                   // argmin rule: T = fl32(w * alpha_max)
  uint32_t log2_block;       // rows per warp block = 2^log2_block (<= 32)
};

struct SsaParams {
  const int32_t* reac;   // M x 2 reactant species (-1 = none)
  const float* rate;     // M mass-action constants
  const int32_t* didx;   // M x D state-change species (-1 = unused)
  const int32_t* dval;   // M x D state-change values
  int32_t* X;            // K x N copy numbers (in/out)
  double* t;             // K times (in/out)
  uint32_t* steps;       // K events fired (out, may be null)
  DevCounters* ctr;
  double t_end;
  uint32_t N, M, D, K;
  uint32_t s0, epoch0, seed_lo, seed_hi, max_trials;
  int32_t n_steps;
  uint32_t net_bytes;    // staged network (smem), including the dependency lists
  uint32_t warp_bytes;   // per-warp row + state (smem)
  const int32_t* dep_ptr;  // M+1 CSR offsets: reactions whose propensity reads a species
  const int32_t* dep_idx;  // that reaction j changes (null: recompute every propensity)
  uint32_t dep_total;
};

// ---------------------------------------------------------------- PTX helpers
// Shared-memory loads by 32-bit shared-window address (no generic->shared conversion per
// access).  volatile: never deleted, duplicated or merged (ring slots and SSA rows are
// rewritten in place) and never reordered against the other side-effecting operations that
// produce the data -- __syncthreads / __syncwarp, the mbarrier wait, the bulk-copy issue.
// No "memory" clobber: it would force every kernel parameter to be re-read from the
// constant bank after each load (LDCU traffic seen in r01_c4_select_rows_v6).

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}

// The same three operations on 32-bit shared-window addresses computed once by the caller
// (no generic->shared conversion per use).
__device__ __forceinline__ void mbar_arrive_expect_tx_s(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait_s(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s_s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                           uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(policy)
      : "memory");
}

// 1-D bulk async copy global -> shared (SASS UBLKCP), completion counted on `bar`.
// dst, src 16-byte aligned; bytes a multiple of 16.  L2 policy evict_first: every
// propensity row is read exactly once.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// 1-D bulk async copy without an L2 policy (data re-read by every CTA: keep it in L2).
__device__ __forceinline__ void bulk_g2s_plain(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// Stage `nbytes` at global `src` into this CTA's shared memory at `dst` (16-byte aligned)
// with bulk async copies of the 16-byte-aligned hull, in two halves so that the copy
// overlaps other work: stage_issue (thread 0 initialises the mbarrier and issues the
// copies; every thread gets the shared address of the first byte of src), then, after a
// __syncthreads that publishes the barrier's initialisation, stage_wait by every thread.
__device__ __forceinline__ uint32_t stage_issue(unsigned char* dst, const void* src, uint32_t nbytes, uint64_t* bar) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(src);
  const uintptr_t lo = a & ~(uintptr_t)15;
  const uint32_t total = (uint32_t)(((a + nbytes + 15u) & ~(uintptr_t)15) - lo);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1u);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_arrive_expect_tx(bar, total);
    for (uint32_t off = 0; off < total; off += 32768u)
      bulk_g2s_plain(dst + off, reinterpret_cast<const unsigned char*>(lo) + off, min(32768u, total - off), bar);
  }
  return smem_u32(dst) + (uint32_t)(a - lo);
}

__device__ __forceinline__ void stage_wait(uint64_t* bar) { mbar_wait(bar, 0u); }

// Both halves at once.  Every thread of the CTA must call it (it synchronises the CTA).
__device__ __forceinline__ uint32_t stage_to_smem(unsigned char* dst, const void* src, uint32_t nbytes, uint64_t* bar) {
  const uint32_t s = stage_issue(dst, src, nbytes, bar);
  __syncthreads();
  stage_wait(bar);
  return s;
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ float lds_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ void sts_f32(uint32_t addr, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v));
}

__device__ __forceinline__ float4 lds_f32x4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}

__device__ __forceinline__ int4 lds_i4(uint32_t addr) {
  int4 v;
  asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ uint32_t lds_u16(uint32_t addr) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
  return v;
}

// Packed binary32 pair add (SASS FADD2, sm_100+): each half is one IEEE round-to-nearest add,
// bit-identical to two __fadd_rn.
__device__ __forceinline__ float2 fadd2_rn(float2 a, float2 b) {
  unsigned long long ra, rb, rd;
  asm("mov.b64 %0, {%1, %2};" : "=l"(ra) : "f"(a.x), "f"(a.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(rb) : "f"(b.x), "f"(b.y));
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(rd) : "l"(ra), "l"(rb));
  float2 d;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(d.x), "=f"(d.y) : "l"(rd));
  return d;
}

// RN(t / d) from the correctly rounded reciprocal y = RN(1/d): q0 = RN(t y), r = t - d q0
// (exact with an FMA), q = RN(q0 + r y) -- the final correction of IEEE division by
// Newton-Raphson with an FMA (Markstein), which returns the correctly rounded quotient when
// nothing underflows or overflows (checked exhaustively over all 2^46 significand pairs,
// DESIGN.md R23); the caller guarantees the exponent range, so this is bit-identical to
// __fdiv_rn(t, d) at 3 instead of ~8 instructions (no MUFU.RCP, no reciprocal refinement,
// no FCHK slow-path test).  Used by the argmin rule's ratings and the shared-vector tau.
__device__ __forceinline__ float div_by_recip(float t, float d, float y) {
  const float q0 = __fmul_rn(t, y);
  return __fmaf_rn(__fmaf_rn(-q0, d, t), y, q0);
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---------------------------------------------------------------- row reduction
// alpha_max (max of bit patterns: exact, and >= 0x7f800000 flags an invalid value) and
// alpha_0 of one M-element row in shared memory at `row_s`, by one warp, in a FIXED order
// (R11), shared by the matrix kernel and the SSA kernel so that an SSA step and
// gpuar_select on the same row see the same bits.  Each lane takes 16 elements per
// 512-chunk (conflict-free scalar LDS, consecutive lanes), sums them pairwise in binary32
// (depth 4, packed FADD2) and adds the chunk sum in binary64; a last 256-chunk likewise with
// 8; the < 256 tail in warp-wide steps of 32 (<= 8 per lane, sequential); then a 5-level
// xor butterfly in binary64.  Relative error of alpha_0 <= 8u before the final rounding.
// (A 16-byte-vector variant measured slower: profiles/r01_c4_select_rows_v3.md.)
__device__ __forceinline__ void row_reduce(uint32_t row_s, uint32_t M, uint32_t lane, uint32_t& mx_out,
                                           double& acc_out) {
  uint32_t mx = 0;
  double acc = 0.0;
  uint32_t b0 = 0;
  for (; b0 + 512u <= M; b0 += 512u) {
    const uint32_t p = row_s + 4u * (b0 + lane);
    float v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      v[k] = lds_f32(p + 128u * k);
      mx = max(mx, __float_as_uint(v[k]));
    }
    float2 q[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) q[k] = make_float2(v[2 * k], v[2 * k + 1]);
    const float2 rr = fadd2_rn(fadd2_rn(fadd2_rn(q[0], q[1]), fadd2_rn(q[2], q[3])),
                               fadd2_rn(fadd2_rn(q[4], q[5]), fadd2_rn(q[6], q[7])));
    acc += (double)__fadd_rn(rr.x, rr.y);
  }
  if (b0 + 256u <= M) {
    const uint32_t p = row_s + 4u * (b0 + lane);
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      v[k] = lds_f32(p + 128u * k);
      mx = max(mx, __float_as_uint(v[k]));
    }
    const float2 rr = fadd2_rn(fadd2_rn(make_float2(v[0], v[1]), make_float2(v[2], v[3])),
                               fadd2_rn(make_float2(v[4], v[5]), make_float2(v[6], v[7])));
    acc += (double)__fadd_rn(rr.x, rr.y);
    b0 += 256u;
  }
  if (b0 < M) {  // tail: warp-uniform trip count, one predicated load per lane per step
    float sum = 0.f;
#pragma unroll 1
    for (uint32_t j = b0; j < M; j += 32u) {
      const float v = (j + lane < M) ? lds_f32(row_s + 4u * (j + lane)) : 0.f;
      mx = max(mx, __float_as_uint(v));
      sum = __fadd_rn(sum, v);  // + 0.0 leaves a sum of non-negative values unchanged
    }
    acc += (double)sum;
  }
  mx_out = __reduce_max_sync(kFull, mx);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
  acc_out = acc;
}

// The same reduction, bit for bit (same chunks, same pairwise sums, same binary64 order), with
// counted loops over a running shared address: per row the loop control is a compare and an
// add per two 512-chunks instead of the ~30 instructions of the generic `b0 + 512 <= M` loop
// the compiler unrolls by two.  Used where the trials are ALU-heavy (the SSA kernel: s1 +3.2 %;
// the argmin rule on rows: +1.3 %, A/B on one box); the classic matrix kernel keeps
// row_reduce, under which its burst read rate measured 1 % higher (sustained 2 % lower).
__device__ __forceinline__ void row_reduce_counted(uint32_t row_s, uint32_t M, uint32_t lane, uint32_t& mx_out,
                                                   double& acc_out) {
  uint32_t mx = 0;
  double acc = 0.0;
  uint32_t p = row_s + 4u * lane;
  const uint32_t n512 = M >> 9;
  // one 512-chunk: 16 conflict-free loads per lane, pairwise binary32 sum of them (FADD2)
  auto chunk = [&](uint32_t q) -> float {
    float v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      v[k] = lds_f32(q + 128u * k);
      mx = max(mx, __float_as_uint(v[k]));
    }
    float2 w[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) w[k] = make_float2(v[2 * k], v[2 * k + 1]);
    const float2 rr = fadd2_rn(fadd2_rn(fadd2_rn(w[0], w[1]), fadd2_rn(w[2], w[3])),
                               fadd2_rn(fadd2_rn(w[4], w[5]), fadd2_rn(w[6], w[7])));
    return __fadd_rn(rr.x, rr.y);
  };
  uint32_t i = 0;
#pragma unroll 1
  for (; i + 2u <= n512; i += 2u, p += 4096u) {  // two chunks per step: 32 loads in flight
    const float s0 = chunk(p), s1 = chunk(p + 2048u);
    acc += (double)s0;
    acc += (double)s1;
  }
  if (i < n512) {
    acc += (double)chunk(p);
    p += 2048u;
  }
  if (M & 256u) {
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      v[k] = lds_f32(p + 128u * k);
      mx = max(mx, __float_as_uint(v[k]));
    }
    const float2 rr = fadd2_rn(fadd2_rn(make_float2(v[0], v[1]), make_float2(v[2], v[3])),
                               fadd2_rn(make_float2(v[4], v[5]), make_float2(v[6], v[7])));
    acc += (double)__fadd_rn(rr.x, rr.y);
    p += 1024u;
  }
  const uint32_t b0 = M & ~255u;
  if (b0 < M) {  // tail: warp-uniform trip count, one predicated load per lane per step
    float sum = 0.f;
#pragma unroll 1
    for (uint32_t j = b0 + lane; j < M + lane; j += 32u, p += 128u) {
      const float v = (j < M) ? lds_f32(p) : 0.f;
      mx = max(mx, __float_as_uint(v));
      sum = __fadd_rn(sum, v);  // + 0.0 leaves a sum of non-negative values unchanged
    }
    acc += (double)sum;
  }
  mx_out = __reduce_max_sync(kFull, mx);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
  acc_out = acc;
}

// Programmatic dependent launch (PDL, sm_90+): griddepcontrol.wait blocks until every
// prerequisite grid of the stream has completed and its memory is visible; launch_dependents
// lets the next PDL-launched grid be scheduled before this one finishes.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// Launch with (pdl) or without the programmatic-stream-serialization attribute.
template <class... KArgs, class... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), int grid, int block, size_t smem, cudaStream_t st, bool pdl,
                       Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------- launchers (host)

cudaError_t launch_stats(const float* alpha, uint32_t M, double* part_sum, uint32_t* part_max,
                         DevStats* stats, DevCounters* ctr, int stats_blocks, cudaStream_t st, bool pdl);
cudaError_t launch_thresholds(const float* alpha, uint32_t M, const DevStats* stats, uint32_t* thr, uint16_t* pref,
                              uint32_t n_pref, uint32_t group_shift, int path, cudaStream_t st, bool pdl);
cudaError_t launch_select_shared(const SharedParams& p, int path, int grid, int block, cudaStream_t st, bool pdl);
cudaError_t launch_argmin_shared(const SharedParams& p, bool smem, int grid, int block, cudaStream_t st, bool pdl);
void set_argmin_limits(int bytes);
int argmin_blocks_per_sm(bool smem, size_t bytes);
cudaError_t launch_it_prefix(const float* alpha, uint32_t M, double* C, cudaStream_t st);
cudaError_t launch_it_select(const SharedParams& p, const double* C, bool smem, int grid, cudaStream_t st, bool pdl);
void set_it_limits(int bytes);
cudaError_t launch_ssa(const SsaParams& p, int grid, int warps, cudaStream_t st);
int ssa_blocks_per_sm(int warps, size_t smem);
void set_ssa_limits(int bytes);
cudaError_t launch_select_rows(const RowsParams& p, int grid, int warps, cudaStream_t st, bool pdl);
cudaError_t launch_histogram(const int32_t* idx, const uint32_t* trials, uint32_t K, uint32_t M,
                             unsigned long long* hist, unsigned long long* totals, int grid,
                             cudaStream_t st);
cudaError_t launch_bench_philox(uint32_t n_threads, uint32_t calls, uint32_t seed_lo, uint32_t seed_hi,
                                uint32_t* sink, cudaStream_t st);

// Allow `fn` the opt-in dynamic shared memory `optin` minus its own static shared memory
// (asking for more than that is an error and would leave the 48 KB default in place).
template <typename F>
inline void set_max_dynamic_smem(F fn, int optin) {
  cudaFuncAttributes a{};
  if (cudaFuncGetAttributes(&a, fn) != cudaSuccess) return;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)a.sharedSizeBytes);
}

// Occupancy helpers (filled by the TU owning each kernel).
int select_shared_blocks_per_sm(int path, int block, size_t smem);
int select_rows_blocks_per_sm(int warps, size_t smem);
void set_select_shared_limits(int bytes);
void set_select_rows_limits(int bytes);

}  // namespace gpuar
