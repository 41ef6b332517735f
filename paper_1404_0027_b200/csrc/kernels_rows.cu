// kernels_rows.cu -- GPU-AR selection over a per-realization K x M propensity matrix
// (config c4: M = 1029, K = 2^20, 4.02 GiB): row k = D[k*ld + j] is
// realization k's propensity vector, so each row needs its own alpha_max / alpha_0
// before its trials.
//
// The row must be read once in full (alpha_0 needs every alpha_j), so the kernel is
// HBM-bound: 4M bytes per selection is the algorithmic minimum.  Design:
//  * persistent CTAs, W warps each; every warp owns a private ring of S row slots in
//    shared memory and its own mbarriers -- it is its own producer (lane 0 issues a 1-D
//    bulk async copy, cp.async.bulk -> SASS UBLKCP, of the row's 16-byte-aligned cover)
//    and consumer, so a slow row (geometric trial count) never stalls another warp;
//  * rows are streamed with an L2 evict_first policy (read exactly once);
//  * per row: warp-wide max of the bit patterns (exact alpha_max + validity) and alpha_0
//    by row_reduce (binary32 pairwise sums of 16 per lane promoted to binary64, error <= 8u
//    relative, R11), then trials in rounds of 32 Philox calls = 64 trials per
//    warp with a ballot/__ffs first-accept; -ln(u1) is drawn 32 rows at a time and tau is
//    formed once per block of rows at the output flush.
// The same pipeline serves the paper's printed argmin rule (NEXT-1), the inverse transform
// (NEXT-3: prefix + search, and the linear scan, bit-identical to the oracle's sequential
// binary64 sums, R24) and gpuar_row_stats, as template modes.
// Row 4116 bytes is not a multiple of 16, so no 2-D tensor map can describe the matrix;
// each row's copy covers [floor16(start), ceil16(end)) -- at most 15 extra bytes on
// each side, always inside 16-byte chunks that hold row data -- EXCEPT where ceil16(end)
// passes the end of the caller's buffer (the last row's last element, for the last 1-3
// rows of the matrix): those rows' copies stop at floor16(buffer end) and the <= 3 words
// after it are loaded by lanes 0-2 into the slot, so nothing outside [base, base +
// ((K-1) ld + M) * 4) is ever read (include/gpuar.h).
#include <algorithm>

#include "gpuar_internal.cuh"
#include "philox.cuh"

namespace gpuar {

namespace {

// Trials of one row by one warp: round t = Philox calls [32t, 32t+32), lane l -> call
// 32t + l -> trials 2c, 2c+1; the ballot's lowest lane (even trial first) is the first
// accept in canonical order (R6).  Rounds whose 64 trials all lie below max_trials
// (every round a selection reaches at the default cap) skip the cap tests: c0 + 31 < half.
template <bool FOLD, bool CAP, class Stream>
__device__ __forceinline__ bool row_round(const Stream& ts, uint32_t c0, uint32_t sel, uint32_t row_s, uint32_t M,
                                          float amax, float amax_s, uint32_t half, uint32_t calls, uint32_t lane,
                                          int32_t& id, uint32_t& tr) {
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
    const uint32_t w = __ffs(b) - 1;
    id = (int32_t)__shfl_sync(kFull, a0 ? j0 : j1, w);
    tr = __shfl_sync(kFull, a0 ? 2u * c + 1u : 2u * c + 2u, w);
    return true;
  }
  return false;
}

template <bool FOLD, class Stream>
__device__ __forceinline__ void row_trials(const Stream& ts, uint32_t sel, uint32_t row_s, uint32_t M,
                                           float amax, uint32_t half, uint32_t calls, uint32_t lane, int32_t& id,
                                           uint32_t& tr) {
  const float amax_s = __fmul_rn(amax, 0x1p-24f);
  const uint32_t free_end = half & ~31u;  // c0 < free_end (c0 a multiple of 32) <=> c0 + 31 < half
  uint32_t c0 = 0;
  for (; c0 < free_end; c0 += 32u)
    if (row_round<FOLD, false>(ts, c0, sel, row_s, M, amax, amax_s, half, calls, lane, id, tr)) return;
  for (; c0 < calls; c0 += 32u)
    if (row_round<FOLD, true>(ts, c0, sel, row_s, M, amax, amax_s, half, calls, lane, id, tr)) return;
}

// N Philox calls' reactions 4c_i..4c_i+3 (FULL: all < M, else bounds-tested), calls in
// increasing order.  The common case -- none of the 4N eligible (probability (1 - p)^4N) --
// costs the loads, uniforms and compares and ONE branch, and with N = 2 the two calls'
// independent IMAD.WIDE chains interleave (24 warps per SM do not hide one chain's
// latency); the division and the minimum update run only for an eligible reaction (an
// ineligible one rates 1.0, which never beats bestR).
template <int N, bool FOLD, bool FULL>
__device__ __forceinline__ void rate_calls(const Philox4 (&x)[N], const uint32_t (&c)[N], uint32_t row_s, uint32_t M,
                                           float T, float T_s, float& bestR, uint32_t& bestJ) {
  float d[4 * N], t[4 * N];
  bool e[4 * N];
  bool any = false;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const uint32_t a = row_s + 16u * c[i];
    const uint32_t xs[4] = {x[i].x, x[i].y, x[i].z, x[i].w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      d[4 * i + q] = lds_f32(a + 4u * q);
      // a leftover call may be the row's partial one: reactions >= M do not exist
      if (!FULL && q > 0) d[4 * i + q] = 4u * c[i] + q < M ? d[4 * i + q] : 0.f;
      t[4 * i + q] = scaled_u<FOLD>(xs[q], T, T_s);
      e[4 * i + q] = t[4 * i + q] < d[4 * i + q];
      any |= e[4 * i + q];
    }
  }
  if (any) {
#pragma unroll
    for (int k = 0; k < 4 * N; ++k) {
      if (e[k]) {  // increasing j with a strict `<`: the lowest index keeps a tied rating
        const float R = __fdiv_rn(t[k], d[k]);
        if (R < bestR) bestR = R, bestJ = 4u * c[k >> 2] + (k & 3);
      }
    }
  }
}

// The paper's printed rule on one row (R16-R19): lane l rates reactions 4c..4c+3
// of its calls c = l, l+32, ...; warp butterfly on the (rating bits, index) key.
// Leftover calls precomputed for a batch of rows (see the kernel): when every lane runs the
// same number of pair iterations and 1 or 2 calls are left per row, the Philox words of the
// leftovers of the next kLeftRows rows are drawn in one warp-wide step (lane l: row
// l / L, call 64 nP + l % L) and each row takes its words by shuffle -- one Philox latency
// per 16 rows instead of per row.
constexpr uint32_t kLeftRows = 16;
struct Leftover {
  bool batched;    // the batched path applies to this launch's M
  uint32_t src;    // lane holding this row's first leftover call
  Philox4 x;       // this lane's precomputed words
};

template <bool FOLD, class Stream>
__device__ __forceinline__ void row_argmin(const Stream& ts, uint32_t sel, uint32_t row_s, uint32_t M, float T,
                                           uint32_t lane, int32_t& id, const Leftover& lo) {
  const float T_s = __fmul_rn(T, 0x1p-24f);
  const uint32_t k1t = ts.rk1[0] ^ kTagElection;
  const uint32_t full = M >> 2;  // calls whose four reactions all exist
  const uint32_t calls = (M + 3u) >> 2;
  float bestR = 1.0f;  // lane-local minimum; a lane sees its j in increasing order
  uint32_t bestJ = 0xffffffffu;
  // two full calls per iteration
  uint32_t c = lane;
  for (; c + 32u < full; c += 64u) {
    const Philox4 x[2] = {ts.with_tag(c, sel, k1t), ts.with_tag(c + 32u, sel, k1t)};
    const uint32_t cc[2] = {c, c + 32u};
    rate_calls<2, FOLD, true>(x, cc, row_s, M, T, T_s, bestR, bestJ);
  }
  if (lo.batched) {  // c = lane + 64 nP for every lane; lanes < L rate their call
    Philox4 xb;
    xb.x = __shfl_sync(kFull, lo.x.x, lo.src + lane);
    xb.y = __shfl_sync(kFull, lo.x.y, lo.src + lane);
    xb.z = __shfl_sync(kFull, lo.x.z, lo.src + lane);
    xb.w = __shfl_sync(kFull, lo.x.w, lo.src + lane);
    if (c < calls) {
      const Philox4 x[1] = {xb};
      const uint32_t cc[1] = {c};
      rate_calls<1, FOLD, false>(x, cc, row_s, M, T, T_s, bestR, bestJ);
    }
  } else {
    // the leftover calls (at most two per lane) in ONE predicated step, so the warp pays
    // one Philox latency
    for (; c < calls; c += 32u) {
      const Philox4 x[1] = {ts.with_tag(c, sel, k1t)};
      const uint32_t cc[1] = {c};
      rate_calls<1, FOLD, false>(x, cc, row_s, M, T, T_s, bestR, bestJ);
    }
  }
  unsigned long long best = ((unsigned long long)__float_as_uint(bestR) << 32) | bestJ;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(kFull, best, o));
  id = (uint32_t)(best >> 32) < 0x3f800000u ? (int32_t)(uint32_t)best : -1;
}

// ---------------------------------------------------------------- inverse transform (NEXT-3)
// The classic direct method on one row (oracle_it_one): idx = the smallest
// j with C_j > u2 * alpha_0, C_j = fl64(C_{j-1} + alpha_j) the SEQUENTIAL binary64 prefix sum
// and alpha_0 = C_{M-1} (R24).  A warp reaches the sequential values without the
// M-long dependent chain when no partial sum rounds: every alpha_j is a multiple of 2^q
// (q = the ulp exponent of the smallest non-zero alpha_j), so every partial sum in ANY order
// is a multiple of 2^q, and if alpha_0 < 2^(q+53) each is exact in binary64 -- then
// C_j = S_j, the exact prefix, which a warp scan computes in any order.  The test uses the
// warp's own binary64 sum a (a < 2^(q+52) implies the exact sum < 2^(q+53), the sum's
// relative error being far below 1/2).  Rows failing it (a dynamic range above ~2^(52 -
// log2 M)) run the oracle's two sequential passes on lane 0.  The yeast-like rows (0.1 ..
// 953, M = 1029) pass with 2^5 to spare.

// inclusive warp scan in binary64 (exact on rows that pass the test)
__device__ __forceinline__ double warp_incl_scan(double x, uint32_t lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double t = __shfl_up_sync(kFull, x, o);
    if (lane >= (uint32_t)o) x = __dadd_rn(x, t);
  }
  return x;
}

// Linear scan of elements [j, end) in warp-wide steps of 32 with carry C = C_{j-1}: the first
// k with C_k > target, or -1.  The number of steps is the row's random crossing position / 32.
__device__ __forceinline__ int32_t it_scan_from(uint32_t row_s, uint32_t j, uint32_t end, double C, double target,
                                                uint32_t lane) {
  for (; j < end; j += 32u) {
    const uint32_t k = j + lane;
    const double v = k < end ? (double)lds_f32(row_s + 4u * k) : 0.0;
    const double Ck = __dadd_rn(C, warp_incl_scan(v, lane));
    const uint32_t b = __ballot_sync(kFull, k < end && Ck > target);
    if (b != 0u) return (int32_t)(j + (uint32_t)__ffs(b) - 1u);
    C = __shfl_sync(kFull, Ck, 31);
  }
  return -1;
}

// The same linear scan in warp-wide steps of 64 (lane l holds elements j + 2l, j + 2l + 1):
// one warp scan of the pair sums per 64 elements, then the crossing lane resolves its pair.
// Half the scan steps of it_scan_from for the same result (all partial sums exact).
__device__ __forceinline__ int32_t it_scan_pairs(uint32_t row_s, uint32_t M, double target, uint32_t lane) {
  double C = 0.0;
  for (uint32_t j = 0; j < M; j += 64u) {
    const uint32_t k = j + 2u * lane;
    const double v0 = k < M ? (double)lds_f32(row_s + 4u * k) : 0.0;
    const double v1 = k + 1u < M ? (double)lds_f32(row_s + 4u * k + 4u) : 0.0;
    const double pair = __dadd_rn(v0, v1);
    const double incl = __dadd_rn(C, warp_incl_scan(pair, lane));  // C_{k+1}
    const uint32_t b = __ballot_sync(kFull, k < M && incl > target);
    if (b != 0u) {
      const uint32_t w = (uint32_t)__ffs(b) - 1u;
      const double first = __dsub_rn(incl, v1);                    // C_k (exact)
      const bool at0 = __shfl_sync(kFull, first > target ? 1u : 0u, w) != 0u;
      return (int32_t)(j + 2u * w + (at0 ? 0u : 1u));
    }
    C = __shfl_sync(kFull, incl, 31);
  }
  return -1;
}

// The oracle's algorithm verbatim on one lane (rows whose partial sums round): alpha_0 by the
// sequential sum, then the sequential scan; the last positive j if rounding exhausts it.
__device__ __noinline__ int32_t it_sequential(uint32_t row_s, uint32_t M, float u2, double& a0) {
  double C = 0.0;
  for (uint32_t j = 0; j < M; ++j) C = __dadd_rn(C, (double)lds_f32(row_s + 4u * j));
  a0 = C;
  const double target = __dmul_rn((double)u2, a0);
  C = 0.0;
  int32_t last = -1;
  for (uint32_t j = 0; j < M; ++j) {
    const float a = lds_f32(row_s + 4u * j);
    C = __dadd_rn(C, (double)a);
    if (a > 0.0f) last = (int32_t)j;
    if (C > target) return (int32_t)j;
  }
  return last;
}

// One row by one warp.  SCAN: the paper's "iterate in the cumulative distribution" -- a
// linear scan from j = 0 (its step count is random).  Otherwise prefix +
// search: lane l sums the contiguous block [l B, l B + B) (B odd: conflict-free LDS), a warp
// scan gives the block prefixes, a ballot finds the block holding the crossing and one
// linear scan of that block (<= ceil(B / 32) steps) the element.  mx: max of the bit patterns
// (alpha_max, validity).  Outputs id and a0 (= C_{M-1}); nothing when mx flags the row.
template <bool SCAN>
__device__ __forceinline__ void row_it(uint32_t row_s, uint32_t M, uint32_t B, uint32_t lane, float u2,
                                       uint32_t& mx_out, int32_t& id, double& a0) {
  uint32_t mx = 0, mn = 0xffffffffu;  // mn: min over (bits - 1), i.e. the smallest non-zero - 1
  double s = 0.0;
  const uint32_t j0 = lane * B;
  const uint32_t n = j0 < M ? min(B, M - j0) : 0u;
  const uint32_t p = row_s + 4u * j0;
#pragma unroll 4
  for (uint32_t k = 0; k < n; ++k) {
    const float v = lds_f32(p + 4u * k);
    const uint32_t b = __float_as_uint(v);
    mx = max(mx, b);
    mn = min(mn, b - 1u);
    s = __dadd_rn(s, (double)v);
  }
  mx = __reduce_max_sync(kFull, mx);
  mx_out = mx;
  if (mx >= kInfBits || mx == 0u) return;
  mn = __reduce_min_sync(kFull, mn) + 1u;  // the smallest non-zero bit pattern
  const double P = warp_incl_scan(s, lane);
  a0 = __shfl_sync(kFull, P, 31);
  // exact iff a0 < 2^(q + 52), q = max(E_min, 1) - 150 the ulp exponent of the smallest value
  const int q = (int)max(mn >> 23, 1u) - 150;
  const int ea = (int)(uint32_t)(__double_as_longlong(a0) >> 52) - 1023;  // a0 > 0: floor(log2 a0)
  id = -1;
  if (ea <= q + 51) {  // warp-uniform
    const double target = __dmul_rn((double)u2, a0);
    if constexpr (SCAN) {
      id = it_scan_pairs(row_s, M, target, lane);
    } else {
      const uint32_t bl = __ballot_sync(kFull, P > target);  // P_31 = a0 > target always
      if (bl != 0u) {
        const uint32_t w = (uint32_t)__ffs(bl) - 1u;
        const double Ew = __shfl_sync(kFull, __dsub_rn(P, s), w);  // C before block w (exact)
        id = it_scan_from(row_s, w * B, min(w * B + B, M), Ew, target, lane);
      }
    }
  }
  if (id < 0) {  // rounding partial sums (or no crossing found): the oracle's passes
    double a = 0.0;
    int32_t i = -1;
    if (lane == 0) i = it_sequential(row_s, M, u2, a);
    id = __shfl_sync(kFull, i, 0);
    a0 = __shfl_sync(kFull, a, 0);
  }
}

// MODE: kRuleClassic / kRuleArgmin / kRuleIT / kRuleITScan (selection), or kModeStats
// (gpuar_row_stats)
constexpr int kModeStats = 8;

template <int MAXW, int MODE>
__global__ void __launch_bounds__(MAXW * 32, 1) select_rows_kernel(const RowsParams P) {
  extern __shared__ __align__(128) unsigned char smem[];
  pdl_wait();  // programmatic dependent launch: the rows may come from the previous grid
  pdl_launch_dependents();
  const uint32_t warps = blockDim.x >> 5;
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t lS = P.log2_stages;  // ring depth S = 2^lS (1, 2 or 4): slot/parity by shifts
  const uint32_t S = 1u << lS;
  const uint32_t SB = P.stage_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + warp * S;
  unsigned char* ring = smem + ((warps * S * 8u + 127u) & ~127u) + (size_t)warp * S * SB;
  // shared-window addresses, computed once (no generic->shared conversion per row)
  const uint32_t bars_s = smem_u32(bars);
  const uint32_t ring_s = smem_u32(ring);

  if (lane < S) mbar_init(&bars[lane], 1u);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();

  const uint64_t policy = policy_evict_first();
  const uint32_t K = P.K;
  const uint32_t M = P.M;
  const uint32_t row_bytes = (uint32_t)(P.ld * 4ull);
  const unsigned char* base = reinterpret_cast<const unsigned char*>(P.alpha);
  // Rows of this warp: warps take turns on blocks of B = 2^lb consecutive rows (block
  // b = wg, wg + WT, ...), so the rows in flight over the whole GPU stay within a window of
  // B*WT rows (B = 8: ~117 MB, inside the 256 MB TLB reach) while a warp's outputs for a
  // block go out as one store per output array from B lanes.  The warp's row count is fixed
  // up front, so the walk below never compares row indices against K.
  const uint32_t WT = gridDim.x * warps;
  const uint32_t wg = blockIdx.x * warps + warp;
  const uint32_t lb = P.log2_block;
  const uint32_t bm = (1u << lb) - 1u;
  const uint32_t nfull = K >> lb, rem = K & bm;  // full blocks, rows of the partial block
  const uint32_t n_rows = ((nfull > wg) ? ((nfull - wg - 1u) / WT + 1u) << lb : 0u) +
                          ((rem != 0u && nfull % WT == wg) ? rem : 0u);
  auto row_of = [&](uint32_t n) -> uint32_t { return (((n >> lb) * WT + wg) << lb) + (n & bm); };
  // Incremental walk (row index, position in its block): a few 32-bit ops per row; the byte
  // offset is one wide multiply.
  const uint32_t jump = (WT - 1u) * (bm + 1u) + 1u;  // from the last row of a block to the next block
  struct Walk {
    uint32_t r, pos;
  };
  auto advance = [&](Walk& w) {
    const bool last = w.pos == bm;
    w.r += last ? jump : 1u;
    w.pos = last ? 0u : w.pos + 1u;
  };
  // The caller's buffer ends after the last row's M-th element; rows >= r_tail have a
  // 16-byte hull that passes that end (at most 3 rows; monotone in r).
  const uint64_t buf_end = (uint64_t)(K - 1u) * row_bytes + 4ull * M;
  const uint64_t buf_end16 = buf_end & ~15ull;
  uint32_t r_tail = K;
  while (r_tail > 0u && ((((uint64_t)(r_tail - 1u) * row_bytes + 4ull * M + 15ull) & ~15ull) > buf_end)) --r_tail;
  auto issue = [&](uint32_t r, uint32_t slot) {
    const uint64_t off = (uint64_t)r * row_bytes;
    const uint64_t a = off & ~15ull;
    const uint64_t e = r < r_tail ? (off + 4ull * M + 15ull) & ~15ull : buf_end16;  // >= a
    const uint32_t bytes = (uint32_t)(e - a);
    mbar_arrive_expect_tx_s(bars_s + 8u * slot, bytes);  // 0 bytes: a plain arrive
    if (bytes != 0u) bulk_g2s_s(ring_s + slot * SB, base + a, bytes, bars_s + 8u * slot, policy);
  };
  Walk cur{wg << lb, 0u};
  Walk pre = cur;  // row n + S: the next row to prefetch into the slot row n frees
  for (uint32_t i = 0; i < S; ++i) {
    if (lane == 0 && i < n_rows) issue(pre.r, i);
    advance(pre);
  }

  const uint32_t half = P.max_trials >> 1;
  const uint32_t calls = half + (P.max_trials & 1u);
  const TrialStream ts(P.seed_lo, P.seed_hi, P.epoch);
  // argmin rule: batched leftover calls when every lane runs floor(full / 64) pair
  // iterations ((full mod 64) <= 32) and 1 or 2 calls remain (M = 1029: calls 256, 257)
  const uint32_t full4 = M >> 2, ncalls4 = (M + 3u) >> 2;
  const uint32_t left_c0 = full4 & ~63u, nleft = ncalls4 - left_c0;
  Leftover left;
  left.batched = MODE == kRuleArgmin && (full4 & 63u) <= 32u && nleft >= 1u && nleft <= 2u;
  left.src = 0;
  left.x = Philox4{0u, 0u, 0u, 0u};
  float nlog = 0.f;  // -ln(u1) of row_of(n0 + lane)
  constexpr bool kIT = MODE == kRuleIT || MODE == kRuleITScan;
  float u2v = 0.f;   // inverse transform: u2 of row_of(n0 + lane) (Philox tag 2)
  const uint32_t itB = ((M + 31u) >> 5) | 1u;  // IT prefix blocks: odd, >= M / 32
  // this lane's buffered outputs for row (block base + lane); tau is formed at the flush,
  // one division per block: tau = -ln(u1) / fl32(alpha_0), with fl32(alpha_0) = 0 for an
  // all-zero row (tau = +inf) and NaN for an invalid one (tau = NaN)
  int32_t o_id = -1;
  uint32_t o_tr = 0;
  float o_a0f = 0.f;
  double o_a0 = 0.0;

  for (uint32_t n = 0; n < n_rows; ++n) {
    const uint32_t r = cur.r;
    const uint32_t slot = n & (S - 1u);
    const uint32_t parity = (n >> lS) & 1u;
    if ((n & 31u) == 0u && MODE != kModeStats) {
      const uint32_t nn = n + lane;
      nlog = nn < n_rows ? neg_log_u1(P.seed_lo, P.seed_hi, P.s0 + row_of(nn), P.epoch) : 0.f;
      if constexpr (kIT)
        u2v = nn < n_rows ? unit24(philox4x32_10(0u, P.s0 + row_of(nn), P.epoch, kTagIT, P.seed_lo, P.seed_hi).x)
                          : 0.f;
    }
    if constexpr (MODE == kRuleArgmin) {
      if (left.batched && (n & (kLeftRows - 1u)) == 0u) {  // leftovers of rows n .. n+15
        const uint32_t nn = n + lane / nleft;
        if (lane < kLeftRows * nleft && nn < n_rows)
          left.x = ts.with_tag(left_c0 + lane % nleft, ts.sel_word(P.s0 + row_of(nn)), ts.rk1[0] ^ kTagElection);
      }
      left.src = (n & (kLeftRows - 1u)) * nleft;
    }
    mbar_wait_s(bars_s + 8u * slot, parity);
    // The slot holds the row's 16-byte hull: element j sits at word lead + j.
    const uint32_t lead = (r * row_bytes & 15u) >> 2;
    const uint32_t row_s = ring_s + slot * SB + 4u * lead;
    if (r >= r_tail) {  // (warp-uniform) the words past floor16(buffer end): plain loads
      const uint64_t off = (uint64_t)r * row_bytes;
      const uint64_t t0 = max(off, buf_end16);
      const uint32_t nt = (uint32_t)((off + 4ull * M - t0) >> 2);  // <= 3
      if (lane < nt)
        sts_f32(ring_s + slot * SB + (uint32_t)(t0 - (off & ~15ull)) + 4u * lane,
                __ldg(reinterpret_cast<const float*>(base + t0) + lane));
      __syncwarp();
    }

    const uint32_t nl32 = cur.pos;  // this row's slot in the block's output buffer
    if constexpr (kIT) {
      // ---- inverse transform: alpha_0 = C_{M-1} and the crossing in one routine
      const float u2 = __shfl_sync(kFull, u2v, n & 31u);
      uint32_t mx;
      int32_t id = -1;
      double a0 = 0.0;
      row_it<MODE == kRuleITScan>(row_s, M, itB, lane, u2, mx, id, a0);
      float a0f = 0.f;
      if (mx >= kInfBits) {  // invalid row: sticky EPROPENSITY
        a0f = __uint_as_float(0x7fc00000u);
        id = -1;
        if (lane == 0) atomicOr(&P.ctr->err, 1u);
      } else if (mx != 0u) {
        a0f = __double2float_rn(a0);
      }
      if (lane == nl32) {
        o_id = id;
        o_a0f = a0f;
        o_tr = mx != 0u && mx < kInfBits ? 1u : 0u;  // one uniform per selection
      }
    } else {
    // ---- alpha_max (max of bit patterns) and alpha_0 in the fixed order of row_reduce
    uint32_t mx;
    double acc;
    if constexpr (MODE == kRuleArgmin)
      row_reduce_counted(row_s, M, lane, mx, acc);
    else
      row_reduce(row_s, M, lane, mx, acc);

    if constexpr (MODE == kModeStats) {
      if (lane == nl32) {
        o_a0f = mx < kInfBits ? __uint_as_float(mx) : __uint_as_float(0x7fc00000u);
        o_a0 = mx < kInfBits ? acc : __longlong_as_double(0x7ff8000000000000ll);
      }
    } else {
      int32_t id = -1;
      uint32_t tr = 0;
      float a0f;
      if (mx >= kInfBits) {  // invalid row: sticky EPROPENSITY
        a0f = __uint_as_float(0x7fc00000u);
        if (lane == 0) atomicOr(&P.ctr->err, 1u);
      } else if (mx == 0u) {  // all-zero row: nothing can fire
        a0f = 0.f;
      } else {
        const float amax = __uint_as_float(mx);
        a0f = __double2float_rn(acc);
        const uint32_t sel = ts.sel_word(P.s0 + r);
        if constexpr (MODE == kRuleArgmin) {
          // the paper's printed rule on this row: election + argmin selection
          const float T = __fmul_rn(P.w, amax);
          if (can_fold(__float_as_uint(T)))
            row_argmin<true>(ts, sel, row_s, M, T, lane, id, left);
          else
            row_argmin<false>(ts, sel, row_s, M, T, lane, id, left);
          tr = M;
        } else {
          // (two Philox calls per lane per round -- 128 trials -- measured +7 % instructions
          // and 5 % slower in r01: the extra ILP does not pay for the larger last round)
          if (can_fold(mx))
            row_trials<true>(ts, sel, row_s, M, amax, half, calls, lane, id, tr);
          else
            row_trials<false>(ts, sel, row_s, M, amax, half, calls, lane, id, tr);
          if (id < 0) tr = P.max_trials;
        }
      }
      if (lane == nl32) {
        o_id = id;
        o_a0f = a0f;
        o_tr = tr;
      }
    }
    }
    if (nl32 == bm || n + 1u == n_rows) {  // flush the block: one coalesced store per output
      const uint32_t rl = r - nl32 + lane;
      if constexpr (MODE == kModeStats) {
        if (lane <= nl32) {
          P.amax_out[rl] = o_a0f;
          P.a0_out[rl] = o_a0;
        }
      } else {
        // -ln(u1) of this lane's row sits in lane (n - nl32 + lane) & 31 of the batch (a
        // block never straddles a batch: 32 is a multiple of B)
        const float nl = __shfl_sync(kFull, nlog, (n - nl32 + lane) & 31u);
        if (lane <= nl32) {
          P.idx[rl] = o_id;
          if (P.tau) P.tau[rl] = __fdiv_rn(nl, o_a0f);
          if (P.trials) P.trials[rl] = o_tr;
        }
      }
    }
    __syncwarp();
    if (lane == 0 && n + S < n_rows) {
      fence_proxy_async_smem();  // generic-proxy reads of the slot precede the async refill
      issue(pre.r, slot);
    }
    advance(cur);
    advance(pre);
  }
}

template <int MAXW>
cudaError_t launch_w(const RowsParams& p, int grid, int warps, size_t sh, cudaStream_t st, bool pdl) {
  if (p.stats_only) return launch_pdl(select_rows_kernel<MAXW, kModeStats>, grid, warps * 32, sh, st, pdl, p);
  if (p.rule == kRuleArgmin) return launch_pdl(select_rows_kernel<MAXW, kRuleArgmin>, grid, warps * 32, sh, st, pdl, p);
  if (p.rule == kRuleIT) return launch_pdl(select_rows_kernel<MAXW, kRuleIT>, grid, warps * 32, sh, st, pdl, p);
  if (p.rule == kRuleITScan) return launch_pdl(select_rows_kernel<MAXW, kRuleITScan>, grid, warps * 32, sh, st, pdl, p);
  return launch_pdl(select_rows_kernel<MAXW, kRuleClassic>, grid, warps * 32, sh, st, pdl, p);
}

template <int MAXW>
void set_limits_w(int bytes) {
  set_max_dynamic_smem(select_rows_kernel<MAXW, kRuleClassic>, bytes);
  set_max_dynamic_smem(select_rows_kernel<MAXW, kRuleArgmin>, bytes);
  set_max_dynamic_smem(select_rows_kernel<MAXW, kModeStats>, bytes);
  set_max_dynamic_smem(select_rows_kernel<MAXW, kRuleIT>, bytes);
  set_max_dynamic_smem(select_rows_kernel<MAXW, kRuleITScan>, bytes);
}

}  // namespace

cudaError_t launch_select_rows(const RowsParams& p, int grid, int warps, cudaStream_t st, bool pdl) {
  const size_t S = (size_t)1 << p.log2_stages;
  const size_t sh = (((size_t)warps * S * 8u + 127u) & ~(size_t)127u) + (size_t)warps * S * p.stage_bytes;
  if (warps <= 16) return launch_w<16>(p, grid, warps, sh, st, pdl);
  if (warps <= 20) return launch_w<20>(p, grid, warps, sh, st, pdl);
  if (warps <= 24) return launch_w<24>(p, grid, warps, sh, st, pdl);
  return launch_w<32>(p, grid, warps, sh, st, pdl);
}

int select_rows_blocks_per_sm(int warps, size_t smem) {
  int n = 0;
  cudaError_t e;
  if (warps <= 16)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, select_rows_kernel<16, kRuleClassic>, warps * 32, smem);
  else if (warps <= 20)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, select_rows_kernel<20, kRuleClassic>, warps * 32, smem);
  else if (warps <= 24)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, select_rows_kernel<24, kRuleClassic>, warps * 32, smem);
  else
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, select_rows_kernel<32, kRuleClassic>, warps * 32, smem);
  return e == cudaSuccess ? n : 0;
}

void set_select_rows_limits(int bytes) {
  set_limits_w<16>(bytes);
  set_limits_w<20>(bytes);
  set_limits_w<24>(bytes);
  set_limits_w<32>(bytes);
}

}  // namespace gpuar
