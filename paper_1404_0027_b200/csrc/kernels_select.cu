// kernels_select.cu -- GPU-AR selection from ONE shared propensity vector (configs c1, c2,
// c3, c5): classic acceptance-rejection with T = alpha_max
// (PAPER.md:361-365), the first accepted trial winning (north_star; R6).
//
// Design (B200-first, not the paper's election/argmin kernels of PAPER.md:498-555):
//  * one persistent launch; the vector's acceptance thresholds T_j (or a 16-bit prefilter of
//    them) are staged once per CTA in shared memory by one bulk async copy, so a trial is
//    an integer compare (x >> 8) < T_j (R22);
//  * a selection is worked by a TEAM of g lanes (g = 1..32, a power of two picked once per
//    CTA from K and p by an instruction-count model): in round q lane `rank` makes Philox
//    call c = q*g + rank, i.e. trials 2c and 2c+1, so a round covers the contiguous trial
//    block [2qg, 2(q+1)g).  The team's ballot + __ffs picks the lowest accepting lane, and
//    within it the even trial first -> the globally smallest accepted trial index,
//    independent of g.  g = 32 runs warp_loop, g = 1 lane_loop, others trial_loop;
//  * teams that finish take the next selection from a warp-local pool refilled from one of
//    64 striped tickets (one 64-bit atomic per `grab` selections, prefetched one chunk
//    ahead): work stealing, so geometric trial counts leave no long tail;
//  * when a lane-loop warp's pool is dry, the whole warp finishes its last selections one at
//    a time (warp_rounds, the endgame);
//  * tau is a separate, fully coalesced grid-stride phase, drawn on the
//    trial stream's round keys, partly before the programmatic-dependent-launch wait;
//  * with fewer work items than threads, select_shared_pre_kernel lets whole-warp teams work
//    their static chunk before that wait instead;
//  * MULTI: one launch works n consecutive selects (gpuar_select_epochs): the work items are
//    the n*K (epoch, selection) pairs, item q -> selection q mod K at epoch + q / K, output
//    slot q.
#include <algorithm>
#include <type_traits>

#include "gpuar_internal.cuh"
#include "philox.cuh"

namespace gpuar {

namespace {

// The classic acceptance test fl32(u alpha_max) < alpha_j on the 24-bit
// uniform v = x >> 8, as the integer test v < T_j with the thresholds of
// kernels_misc.cu (R22).  Path 1: T_j from the shared-memory copy of the
// threshold table.  Path 2: the 16-bit bracket B_j = min(T_j >> 8, 65535) decides unless
// x >> 16 == B_j.  Path 3: x >> 16 above the group bound rejects; otherwise T_j from L2.
// `sbase` is the shared-state-space address of the staged array.
template <int PATH>
__device__ __forceinline__ bool accept(uint32_t x, uint32_t j, uint32_t sbase, const uint32_t* __restrict__ thr,
                                       uint32_t group_shift) {
  if constexpr (PATH == kPathSmemF32) {
    return (x >> 8) < lds_u32(sbase + 4u * j);
  } else if constexpr (PATH == kPathSmemBf16) {
    const uint32_t b = lds_u16(sbase + 2u * j);
    const uint32_t h = x >> 16;
    if (h != b) return h < b;
    return (x >> 8) < __ldg(thr + j);
  } else {
    if ((x >> 16) > lds_u16(sbase + 2u * (j >> group_shift))) return false;
    return (x >> 8) < __ldg(thr + j);
  }
}

// Both trials of a Philox call (words (x.y, j0) and (x.w, j1)) for the whole warp.  On the
// prefilter paths the 16-bit test decides all but a rare few trials (a bracket tie, 2^-16 per
// trial on path 2; h <= the group bound on path 3); those read the exact T_j from L2 under one
// warp vote instead of as predicated instructions every trial (~10 issue slots per round).
// Every lane of the warp must call it (it votes).
template <int PATH>
__device__ __forceinline__ void accept2(uint32_t xy, uint32_t j0, uint32_t xw, uint32_t j1, uint32_t sbase,
                                        const uint32_t* __restrict__ thr, uint32_t group_shift, bool& r0, bool& r1) {
  if constexpr (PATH == kPathSmemF32) {
    r0 = accept<PATH>(xy, j0, sbase, thr, group_shift);
    r1 = accept<PATH>(xw, j1, sbase, thr, group_shift);
  } else {
    const uint32_t h0 = xy >> 16, h1 = xw >> 16;
    bool u0, u1;
    if constexpr (PATH == kPathSmemBf16) {
      const uint32_t b0 = lds_u16(sbase + 2u * j0), b1 = lds_u16(sbase + 2u * j1);
      r0 = h0 < b0;
      r1 = h1 < b1;
      u0 = h0 == b0;
      u1 = h1 == b1;
    } else {
      u0 = h0 <= lds_u16(sbase + 2u * (j0 >> group_shift));
      u1 = h1 <= lds_u16(sbase + 2u * (j1 >> group_shift));
      r0 = false;
      r1 = false;
    }
    if (__any_sync(kFull, u0 | u1)) {
      if (u0) r0 = (xy >> 8) < __ldg(thr + j0);
      if (u1) r1 = (xw >> 8) < __ldg(thr + j1);
    }
  }
}

// Round-1 words of work item q: selection s0 + q at the launch's epoch, or (multi-epoch
// launch) selection s0 + q mod Ksel at epoch + q / Ksel.  elo is lo(M1 * epoch).
template <bool MULTI>
__device__ __forceinline__ void item_words(const SharedParams& P, const TrialStream& ts, uint32_t q, uint32_t& sel,
                                           uint32_t& elo) {
  if constexpr (MULTI) {
    uint32_t e, s;
    split_item(q, P.Ksel, P.kinv, e, s);
    ts.words(P.epoch + e, P.s0 + s, sel, elo);
  } else {
    sel = ts.sel_word(P.s0 + q);
    elo = ts.e_lo;
  }
}

// tau = -ln(u1) / fl32(alpha_0) (R10) in binary32, IEEE division:
// by the staged reciprocal (div_by_recip, bit-identical) when 2^-60 <= fl32(alpha_0) <= 2^60
// -- then -ln(u1) in [2^-24, 16.7] keeps every quotient and residual normal -- else __fdiv_rn.
struct TauDiv {
  float a0f, ra0;
  bool fast;
  __device__ __forceinline__ float operator()(float nl) const {
    return fast ? div_by_recip(nl, a0f, ra0) : __fdiv_rn(nl, a0f);
  }
};
__device__ __forceinline__ TauDiv tau_div(float a0f) {
  return TauDiv{a0f, __frcp_rn(a0f), a0f >= 0x1p-60f && a0f <= 0x1p60f};
}

// -ln(u1) of work item q's tau (R10) from the trial stream's keys
template <bool MULTI>
__device__ __forceinline__ float item_neg_log_u1(const SharedParams& P, const TrialStream& ts, uint32_t q) {
  uint32_t sel, elo;
  if constexpr (MULTI) {
    uint32_t e, sl;
    split_item(q, P.Ksel, P.kinv, e, sl);
    ts.words(P.epoch + e, P.s0 + sl, sel, elo);
  } else {
    sel = ts.sel_word(P.s0 + q);
    elo = ts.e_lo;
  }
  return neg_log_u1_ts(ts, sel, elo);
}

template <bool MULTI>
__device__ __forceinline__ Philox4 item_call(const TrialStream& ts, uint32_t c, uint32_t sel, uint32_t elo) {
  if constexpr (MULTI)
    return ts.call(c, sel, elo);
  else
    return ts(c, sel);  // e_lo from the (uniform) stream
}

#ifdef GPUAR_TIMELINE
// Diagnostic build only (scripts/diag_timeline.py; never in libgpuar.so): %globaltimer stamps
// of the last two launches (slot = epoch & 1): per CTA [entry, after the PDL wait, trials
// start, %smid], per warp its exit and (at kTlCta + 16384 + warp) when its pool ran dry.
constexpr uint32_t kTlCta = 4u * 1024u, kTlN = kTlCta + 32u * 1024u;
__device__ unsigned long long g_tl[2][kTlN];
__device__ __forceinline__ unsigned long long tl_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TL_CTA(k, v) \
  if (threadIdx.x == 0) g_tl[P.epoch & 1u][4u * blockIdx.x + (k)] = (v)
#endif

// Work distribution: the K selections are cut into kStripes contiguous stripes; warp w
// belongs to stripe w % kStripes, takes a static first chunk of it, then grabs `grab`
// selections at a time from the stripe's ticket until the stripe is exhausted.  kStripes
// tickets keep same-address atomic contention low; a warp never leaves its stripe (a
// stripe holds K/kStripes selections, so stripes finish within ~1/sqrt(K/kStripes) of
// each other), so each warp makes at most one failing atomic.
struct Pool {
  uint32_t next, end;            // current chunk [next, end) (selections < K < 2^32)
  uint32_t hi;                   // end of this warp's stripe
  uint32_t grab;                 // selections per ticket grab
  unsigned long long dbase;      // start of the stripe's dynamic part (after the static chunks)
  unsigned long long pending;    // lane 0: ticket of the NEXT chunk, fetched one chunk ahead
  unsigned long long* tickets;   // this launch's ticket set (DevCounters::next[phase])
  uint32_t stripe;
  bool exhausted;
#ifdef GPUAR_TIMELINE
  uint32_t tl_slot;
#endif

  // Lane 0 issues the atomic for the chunk after the current one; its latency (~1 us under
  // contention) overlaps the current chunk's work instead of stalling the warp.
  bool ahead;                    // prefetch one chunk ahead (else fetch on demand)
  __device__ __forceinline__ void prefetch(uint32_t lane) {
    if (lane == 0u) pending = dbase + atomicAdd(&tickets[stripe], (unsigned long long)grab);
  }
  // Move to the prefetched chunk (and prefetch the one after); false when the stripe is done.
  __device__ __forceinline__ bool refill(uint32_t lane) {
    if (!ahead) prefetch(lane);
    const unsigned long long b = __shfl_sync(kFull, pending, 0);
    if (b >= hi) {
      exhausted = true;
#ifdef GPUAR_TIMELINE
      if (lane == 0u) g_tl[tl_slot][kTlCta + 16384u + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5)] = tl_now();
#endif
      return false;
    }
    next = (uint32_t)b;
    end = next + min(grab, hi - next);
    if (ahead) prefetch(lane);
    return true;
  }
};

__device__ __forceinline__ unsigned long long stripe_lo(uint32_t K, uint32_t s) {
  const unsigned long long sz = ((unsigned long long)K + kStripes - 1) / kStripes;
  return min((unsigned long long)s * sz, (unsigned long long)K);
}

__device__ __forceinline__ void pool_init(Pool& pl, uint32_t K, uint32_t nwarps, uint32_t warp_global,
                                          unsigned long long first, unsigned long long grab,
                                          unsigned long long* tickets, bool ahead) {
  pl.ahead = ahead;
  pl.tickets = tickets;
  pl.grab = (uint32_t)min(grab, (unsigned long long)K);
  pl.stripe = warp_global % kStripes;
  const unsigned long long hi = stripe_lo(K, pl.stripe + 1);
  const unsigned long long lo = stripe_lo(K, pl.stripe) + (unsigned long long)(warp_global / kStripes) * first;
  // start of the dynamic part of the stripe: after all its warps' static chunks
  const unsigned long long nw = (nwarps > pl.stripe) ? (nwarps - pl.stripe + kStripes - 1) / kStripes : 0;
  pl.dbase = stripe_lo(K, pl.stripe) + nw * first;
  pl.hi = (uint32_t)hi;
  pl.next = (uint32_t)min(lo, hi);
  pl.end = (uint32_t)min(lo + first, hi);
  // nothing static and no dynamic part left in the stripe: done without touching the ticket
  pl.exhausted = pl.next >= pl.end && pl.dbase >= hi;
  pl.pending = ~0ull;
}

// The first ticket prefetch (after the PDL wait: the launch's ticket set is only known to be
// zeroed once the previous launch has completed).
__device__ __forceinline__ void pool_start(Pool& pl, uint32_t lane) {
  if (pl.ahead && pl.dbase < pl.hi) pl.prefetch(lane);
}

// Hand idle teams (leader lanes in `need`) the next selections of the warp's pool.
// Returns the new selection of this lane's team (broadcast from its leader) or kNone.
__device__ __forceinline__ uint32_t pool_take(Pool& pl, uint32_t need, uint32_t lane, uint32_t tbase) {
  uint32_t got = kNone;
  while (need != 0u && !pl.exhausted) {
    if (pl.next >= pl.end && !pl.refill(lane)) break;
    const uint32_t avail = pl.end - pl.next;
    const uint32_t r = __popc(need & lanemask_lt());
    uint32_t mine = kNone;
    if (((need >> lane) & 1u) && r < avail) mine = pl.next + r;
    mine = __shfl_sync(kFull, mine, tbase);
    if (mine != kNone) got = mine;
    pl.next += min((uint32_t)__popc(need), avail);
    // leaders that got work drop out of `need`
    const uint32_t served = __ballot_sync(kFull, ((need >> lane) & 1u) && r < avail);
    need &= ~served;
  }
  return got;
}

// Trial phase of one warp with sub-warp teams (1 < g < 32 lanes per selection).
// Fast path: one Philox call + two gathers + one vote per round; team bookkeeping only
// when some team of the warp finished a selection.
template <int PATH, bool MULTI>
__device__ __forceinline__ void trial_loop(const SharedParams& P, const TrialStream& ts, uint32_t sbase, uint32_t g,
                                           Pool pl) {
  const uint32_t M = P.M;
  const uint32_t half = P.max_trials >> 1;            // calls whose odd trial is < max_trials
  const uint32_t calls = half + (P.max_trials & 1u);  // calls whose even trial is < max_trials
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t tbase = lane & ~(g - 1u);
  const uint32_t rank = lane & (g - 1u);
  const uint32_t tmask = (g == 32u) ? kFull : (((1u << g) - 1u) << tbase);
  const bool leader = rank == 0u;

  uint32_t my = kNone;  // local selection of this lane's team
  uint32_t sel = 0;     // its round-1 Philox word
  uint32_t elo = 0;     // (multi-epoch) its epoch word
  uint32_t c = 0;       // this lane's Philox call within the selection

  while (true) {
    const uint32_t need = __ballot_sync(kFull, leader && my == kNone);
    if (need != 0u) {
      const uint32_t got = pool_take(pl, need, lane, tbase);
      if (got != kNone) {
        my = got;
        item_words<MULTI>(P, ts, got, sel, elo);
        c = rank;
      }
    }
    if (pl.exhausted && __all_sync(kFull, my == kNone)) break;
    const bool active = my != kNone;

    bool a0, a1, out;
    uint32_t j0, j1, ball;
    while (true) {
      const Philox4 x = item_call<MULTI>(ts, c, sel, elo);
      j0 = __umulhi(x.x, M);
      j1 = __umulhi(x.z, M);
      // branch-free: both gathers always issue (j < M is always a valid index)
      bool r0, r1;
      accept2<PATH>(x.y, j0, x.w, j1, sbase, P.thr, P.group_shift, r0, r1);
      a0 = active & (c < calls) & r0;
      a1 = active & (c < half) & r1;
      ball = __ballot_sync(kFull, a0 || a1);
      out = active && c - rank + g >= calls;   // the team's next round would start past max_trials
      if (ball != 0u || __any_sync(kFull, out)) break;
      c += g;
    }
    // slow path: resolve finished selections
    const uint32_t b = ball & tmask;
    uint32_t wj = 0, wt = 0;
    if (ball != 0u) {
      const uint32_t src = b ? (uint32_t)(__ffs(b) - 1) : lane;
      wj = __shfl_sync(kFull, a0 ? j0 : j1, src);
      wt = __shfl_sync(kFull, a0 ? 2u * c + 1u : 2u * c + 2u, src);
    }
    if (active) {
      if (b != 0u || out) {
        if (leader) {
          P.idx[my] = b ? (int32_t)wj : -1;
          if (P.trials) P.trials[my] = b ? wt : P.max_trials;
        }
        my = kNone;
      } else {
        c += g;
      }
    }
  }
}

// The endgame of the lane loop: the warp's pool is empty and few lanes still hold a selection
// (each at its own next call c).  Every lane then works one of them at a time, rounds of calls
// [c0, c0 + 32) from c0 = c: the lowest accepting lane (even trial first) is the first accept at
// or after call c, so the result is the one the lane itself would have reached (R6),
// in ~1 / (1 - (1 - p)^64) warp rounds instead of the geometric tail of the slowest lane.
template <int PATH, bool MULTI>
__device__ __forceinline__ void warp_rounds(const SharedParams& P, const TrialStream& ts, uint32_t sbase,
                                            uint32_t sel, uint32_t elo, uint32_t c0, uint32_t lane, int32_t& id,
                                            uint32_t& tr) {
  const uint32_t M = P.M;
  const uint32_t half = P.max_trials >> 1;
  const uint32_t calls = half + (P.max_trials & 1u);
  id = -1;
  tr = P.max_trials;
#pragma unroll 1
  for (; c0 < calls; c0 += 32u) {
    const uint32_t c = c0 + lane;
    const Philox4 x = item_call<MULTI>(ts, c, sel, elo);
    const uint32_t j0 = __umulhi(x.x, M);
    const uint32_t j1 = __umulhi(x.z, M);
    bool r0, r1;
    accept2<PATH>(x.y, j0, x.w, j1, sbase, P.thr, P.group_shift, r0, r1);
    const bool a0 = (c < calls) & r0;
    const bool a1 = (c < half) & r1;
    const uint32_t b = __ballot_sync(kFull, a0 || a1);
    if (b != 0u) {
      const uint32_t w = __ffs(b) - 1;
      id = (int32_t)__shfl_sync(kFull, a0 ? j0 : j1, w);
      tr = __shfl_sync(kFull, a0 ? 2u * c + 1u : 2u * c + 2u, w);
      return;
    }
  }
}

// Largest number of still-busy lanes k for which the endgame above issues fewer warp
// instructions than letting the lane loop run on: k selections x 1 / (1 - (1 - p)^64) warp
// rounds of ~77 instructions against the expected maximum of k geometric lane-round counts
// (H_k / -ln(1 - q) + 1/2, q = 1 - (1 - p)^(2 nc), H_k ~ ln k + 0.5772 + 1 / 2k) of ~117
// (nc = 1) / ~162 (nc = 2) instructions (the SASS counts of choose_team).  Lane l tests
// k = l + 1 (the warp cost is linear in k, the lane-loop cost concave: the test holds for
// k <= T); evaluated by a warp once, when its pool first runs dry.
__device__ __forceinline__ uint32_t endgame_lanes(float p, uint32_t nc, uint32_t lane) {
  const float l1 = __logf(fmaxf(1.0f - p, 1e-30f));
  const float rw = 1.0f / fmaxf(1.0f - __expf(64.0f * l1), 1e-30f);
  const float L = fmaxf(-2.0f * (float)nc * l1, 1e-30f);
  const float k = (float)(lane + 1u);
  const float H = __logf(k) + 0.5772157f + 0.5f / k;
  return __popc(__ballot_sync(kFull, k * rw * 77.0f < (H / L + 0.5f) * (nc == 2u ? 162.0f : 117.0f)));
}

// One lane per selection (g = 1, high p): every round each lane makes NC Philox calls (1, or
// 2 for p <= 1/4) for its own selection; a lane that finishes stores its result and takes the next selection of
// the warp's pool (one ballot + popc), with no cross-lane data exchange.  At high p most
// rounds finish some lane, so the hand-out has a fast path: the current chunk covers every
// idle lane -> one popc and a 32-bit add (selection indices are < K < 2^32); only a chunk
// boundary takes the general loop (refill / prefetch).
template <int PATH, int NC, bool MULTI, bool WANT_TR>
__device__ __forceinline__ void lane_loop(const SharedParams& P, const TrialStream& ts, uint32_t sbase, Pool pl,
                                          float p_acc) {
  const uint32_t M = P.M;
  const uint32_t half = P.max_trials >> 1;
  const uint32_t calls = half + (P.max_trials & 1u);
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t lt = lanemask_lt();
  int32_t* const idx_out = P.idx;
  uint32_t* const tr_out = P.trials;  // non-null iff WANT_TR (a compile-time branch per round)
  uint32_t my = kNone, sel = 0, elo = 0, c = 0;
  bool active = false;
  uint32_t need = kFull;  // lanes without a selection
  uint32_t endgame = kNone;  // endgame_lanes, once the pool has run dry
  while (true) {
    if (need != 0u) {  // warp-uniform: hand out selections
      const uint32_t n = __popc(need);
      const uint32_t nx = pl.next;
      if (pl.end - nx >= n) {  // fast path: the chunk covers all (next <= end always)
        if (!active) {
          my = nx + __popc(need & lt);
          item_words<MULTI>(P, ts, my, sel, elo);
          c = 0;
          active = true;
        }
        pl.next = nx + n;
      } else {
        while (need != 0u && !pl.exhausted) {
          if (pl.next >= pl.end && !pl.refill(lane)) break;
          const uint32_t avail = pl.end - pl.next;
          const uint32_t r = __popc(need & lt);
          const bool mine = ((need >> lane) & 1u) && r < avail;
          if (mine) {
            my = pl.next + r;
            item_words<MULTI>(P, ts, my, sel, elo);
            c = 0;
            active = true;
          }
          pl.next += min((uint32_t)__popc(need), avail);
          need &= ~__ballot_sync(kFull, mine);
        }
        if constexpr (NC == 1) {
          if (pl.exhausted && !__any_sync(kFull, active)) break;
        } else if (pl.exhausted) {
          // (the two-call loop only: at p > 1/4 the warp takes over at most two lanes and the
          // extra code cost the one-call loop 5 % on c3 uniform)
          const uint32_t busy = __ballot_sync(kFull, active);
          if (busy == 0u) break;
          if (endgame == kNone) endgame = P.no_endgame ? 0u : endgame_lanes(p_acc, (uint32_t)NC, lane);
          if ((uint32_t)__popc(busy) <= endgame) {  // the warp finishes the rest one by one
            for (uint32_t b = busy; b != 0u; b &= b - 1u) {
              const uint32_t src = __ffs(b) - 1;
              const uint32_t m = __shfl_sync(kFull, my, src);
              int32_t id;
              uint32_t tr;
              warp_rounds<PATH, MULTI>(P, ts, sbase, __shfl_sync(kFull, sel, src), __shfl_sync(kFull, elo, src),
                                       __shfl_sync(kFull, c, src), lane, id, tr);
              if (lane == 0u) {
                idx_out[m] = id;
                if constexpr (WANT_TR) tr_out[m] = tr;
              }
            }
            break;
          }
        }
      }
    }
    // NC = 1: call c (trials 2c, 2c+1); NC = 2: calls c and c+1 (trials 2c .. 2c+3), decided
    // in canonical order -- half the per-round bookkeeping per call at the price of the
    // second call when the first accepts (used for p <= 1/4, kernel dispatch below)
    const Philox4 x = item_call<MULTI>(ts, c, sel, elo);
    const uint32_t j0 = __umulhi(x.x, M);
    const uint32_t j1 = __umulhi(x.z, M);
    bool r0, r1;
    accept2<PATH>(x.y, j0, x.w, j1, sbase, P.thr, P.group_shift, r0, r1);
    const bool a0 = (c < calls) & r0;
    const bool a1 = (c < half) & r1;
    bool a2 = false, a3 = false;
    uint32_t j2 = 0, j3 = 0;
    if constexpr (NC == 2) {
      const Philox4 y = item_call<MULTI>(ts, c + 1u, sel, elo);
      j2 = __umulhi(y.x, M);
      j3 = __umulhi(y.z, M);
      bool r2, r3;
      accept2<PATH>(y.y, j2, y.w, j3, sbase, P.thr, P.group_shift, r2, r3);
      a2 = (c + 1u < calls) & r2;
      a3 = (c + 1u < half) & r3;
    }
    const bool acc = a0 | a1 | a2 | a3;
    const bool done = active & (acc | (c + (uint32_t)NC >= calls));
    if (done) {
      // branch-free: the first accepting trial k of the round (a0 first) -> j_k, trials 2c + 1 + k
      uint32_t k, jk;
      if constexpr (NC == 1) {
        k = a0 ? 0u : 1u;
        jk = a0 ? j0 : j1;
      } else {
        k = a0 ? 0u : a1 ? 1u : a2 ? 2u : 3u;
        jk = a0 ? j0 : a1 ? j1 : a2 ? j2 : j3;
      }
      idx_out[my] = acc ? (int32_t)jk : -1;
      if constexpr (WANT_TR) tr_out[my] = acc ? 2u * c + 1u + k : P.max_trials;
      active = false;
    }
    c += NC;
    need = __ballot_sync(kFull, !active);
  }
}

// Whole-warp teams (g = 32): the warp works its selections one after another, 64 trials
// per round, like the matrix kernel -- no per-round team bookkeeping, ~15 instructions of
// overhead per selection (pool refill by lane 0 once per `grab` selections).
// warp_select: work item `my` by the whole warp; id / tr on every lane.
template <int PATH, bool MULTI>
__device__ __forceinline__ void warp_select(const SharedParams& P, const TrialStream& ts, uint32_t sbase, uint32_t my,
                                            uint32_t lane, int32_t& id, uint32_t& tr) {
  const uint32_t M = P.M;
  const uint32_t half = P.max_trials >> 1;
  const uint32_t calls = half + (P.max_trials & 1u);
  const uint32_t free_end = half & ~31u;  // rounds starting below it need no cap test
  uint32_t sel, elo;
  item_words<MULTI>(P, ts, my, sel, elo);
  id = -1;
  tr = P.max_trials;
  // one round: calls [c0, c0 + 32); CAP: test the trials against max_trials (only rounds
  // reaching past half = floor(max_trials / 2) need it)
  auto round = [&](uint32_t c0, auto cap) -> bool {
    const uint32_t c = c0 + lane;
    const Philox4 x = item_call<MULTI>(ts, c, sel, elo);
    const uint32_t j0 = __umulhi(x.x, M);
    const uint32_t j1 = __umulhi(x.z, M);
    bool r0, r1;
    accept2<PATH>(x.y, j0, x.w, j1, sbase, P.thr, P.group_shift, r0, r1);
    const bool a0 = (!decltype(cap)::value || c < calls) & r0;
    const bool a1 = (!decltype(cap)::value || c < half) & r1;
    const uint32_t b = __ballot_sync(kFull, a0 || a1);
    if (b != 0u) {
      const uint32_t w = __ffs(b) - 1;
      id = (int32_t)__shfl_sync(kFull, a0 ? j0 : j1, w);
      tr = __shfl_sync(kFull, a0 ? 2u * c + 1u : 2u * c + 2u, w);
      return true;
    }
    return false;
  };
  uint32_t c0 = 0;
  bool hit = false;
  for (; c0 < free_end; c0 += 32u)
    if ((hit = round(c0, std::false_type{}))) break;
  if (!hit)
    for (; c0 < calls; c0 += 32u)
      if (round(c0, std::true_type{})) break;
}

template <int PATH, bool MULTI>
__device__ __forceinline__ void warp_loop(const SharedParams& P, const TrialStream& ts, uint32_t sbase, Pool pl) {
  const uint32_t lane = threadIdx.x & 31u;
  while (!pl.exhausted) {
    if (pl.next >= pl.end && !pl.refill(lane)) break;
    const uint32_t my = pl.next++;
    int32_t id;
    uint32_t tr;
    warp_select<PATH, MULTI>(P, ts, sbase, my, lane, id, tr);
    if (lane == 0u) {
      P.idx[my] = id;
      if (P.trials) P.trials[my] = tr;
    }
  }
}

// Team size g (power of two, 1..32) minimising the estimated warp instructions per
// selection (E = 1/p expected trials; SASS counts of the r01 build):
//   g = 32 (warp_loop): (E/64 + 1/2) rounds x 62 + 15 per selection;
//   g = 1 (lane_loop): (E + 1)/64 warp-rounds x (72 + 45 P(any lane of the warp finished)),
//     or with two calls per round (1/320 <= p <= 1/4) (E + 2)/128 warp-rounds x (117 + 45 P(any));
//   1 < g < 32 (trial_loop): (E + g)/64 warp-rounds x (67 + 45 P(any lane finished));
// (finish costs recalibrated in session 2: ncu counts ~125 warp instructions per lane-loop
// round when a lane finishes almost every round (c3 exponential, M = 10^4), and the
// GPUAR_TEAM sweep has g = 4 fastest at E ~ 73 (c3 Pareto, M = 10^3));
// times (1 + drain tail), tail = 0.1 T ln(T+1) * warps / K with T = 32/g teams per warp.
// (The 0.1 is the session-2 team sweep, GPUAR_TEAM: at K = 10^4 the unscaled tail chose
// g = 32 where g = 4 runs 5 % faster; at K >= 2^16 the tail is too small to move a choice.)
#ifndef GPUAR_TWO_CALL_MIN_P
#define GPUAR_TWO_CALL_MIN_P (1.0f / 320.0f)
#endif
constexpr float kTwoCallMinP = GPUAR_TWO_CALL_MIN_P;  // the two-call lane loop's lower bound on p

__device__ __forceinline__ uint32_t choose_team(float p, uint32_t K, uint32_t nwarps) {
  const float wk = (float)nwarps / (float)max(K, 1u);
  const float E = 1.0f / fmaxf(p, 1e-30f);
  const float any = 1.0f - __expf(64.0f * __logf(fmaxf(1.0f - p, 1e-30f)));
  uint32_t best = 32u;
  float best_cost = (E / 64.0f + 0.5f) * 62.0f + 15.0f;
  best_cost *= 1.0f + 0.06931f * wk;
  // lane loop with two calls per round (p <= 1/4): 128 trials per warp-round at ~117
  // instructions plus the finish handling.  Considered only up to E = 320: before the lane
  // loop's endgame (the warp takes over its last selections, warp_rounds) it measured +16-20 %
  // at E = 14 and 73 but -29 % at E = 292 and -31 % at E ~ 10^5, where the last selection of
  // each lane left most of the warp idle; with the endgame (A/B on one box) +20 % at E = 73
  // (c3 Pareto M = 10^3), +8 % at E = 188 (M = 10^4), +4 % at E = 266, -2 % at E = 391,
  // -10 % at E = 1561 and -6 % at E ~ 10^5 (c5): whole-warp teams beyond E = 320
  const float any2 = 1.0f - __expf(128.0f * __logf(fmaxf(1.0f - p, 1e-30f)));
  for (uint32_t g = 1u; g < 32u; g <<= 1) {
    const float T = (float)(32u / g);
    float rounds, round;
    if (g == 1u && p <= 0.25f && p >= kTwoCallMinP) {
      rounds = (E + 2.0f) / 128.0f;
      round = 117.0f + 45.0f * any2;
    } else {
      rounds = (E + (float)g) / 64.0f;
      round = (g == 1u) ? 72.0f + 45.0f * any : 67.0f + 45.0f * any;
    }
    const float cost = rounds * round * (1.0f + 0.1f * T * __logf(T + 1.0f) * wk);
    if (cost < best_cost) {
      best_cost = cost;
      best = g;
    }
  }
  return best;
}

// The warp's work-stealing pool: static first chunk of half a warp's fair share, then grabs
// of ~8192 expected trials (st.grab), at most an eighth of the fair share (but two teams'
// worth), at least one selection per team; tickets are prefetched one chunk ahead (the first
// by pool_start, after the PDL wait).  (fair = max(1, K / warps) and the static chunk come
// from the host, launch_select: two 64-bit divisions per warp were ~100 of the ~170 set-up
// instructions of every warp.)
__device__ __forceinline__ void pool_setup(const SharedParams& P, const DevStats& st, uint32_t g, uint32_t nwarps,
                                           uint32_t warp_global, Pool& pl) {
  const unsigned long long teams = 32u / g;
  const unsigned long long fair = P.fair;
  // p > 1/4: a selection takes ~1-2 rounds with little variance, so a warp's fair share
  // hardly varies and 15/16 of it static balances as well with fewer tickets (c3 uniform
  // +2 % over 3/4; at heavy tails 15/16 lost 3-8 %)
  const unsigned long long fb = (st.p > 0.25f && fair > 4u) ? fair - fair / 16u : P.first_base;
  const unsigned long long first = max(teams, fb);
  // (r01 sweep, GPUAR_GRAB: c2 best at 2 with prefetch; heavy tails (st.grab = 1) at 1;
  // session 4: the two-call lane loop best at one selection per lane, c3 Pareto +2.6-2.9 %)
  const unsigned long long two_min = (g == 1u && st.p <= 0.25f) ? 1ull : 2ull;
  unsigned long long grab = max(teams, min((unsigned long long)st.grab, max(two_min * teams, fair / 8ull)));
  if (P.grab_override) grab = P.grab_override;
#ifdef GPUAR_TIMELINE
  pl.tl_slot = P.epoch & 1u;
#endif
  pool_init(pl, P.K, nwarps, warp_global, first, grab, P.ctr->next[P.phase], P.no_prefetch == 0u);
}

// The trial loop of the CTA's team size g.
template <int PATH, bool MULTI>
__device__ __forceinline__ void run_trials(const SharedParams& P, const DevStats& st, const TrialStream& ts,
                                           uint32_t sbase, uint32_t g, const Pool& pl) {
  if (g == 1u) {
    // two calls per round exactly where choose_team priced them (1/128 <= p <= 1/4); a
    // forced g = 1 (GPUAR_TEAM) outside that range runs the one-call loop
    const bool two = st.p <= 0.25f && st.p >= kTwoCallMinP;
    if (P.trials) {
      if (two)
        lane_loop<PATH, 2, MULTI, true>(P, ts, sbase, pl, st.p);
      else
        lane_loop<PATH, 1, MULTI, true>(P, ts, sbase, pl, st.p);
    } else {
      if (two)
        lane_loop<PATH, 2, MULTI, false>(P, ts, sbase, pl, st.p);
      else
        lane_loop<PATH, 1, MULTI, false>(P, ts, sbase, pl, st.p);
    }
  } else if (g == 32u) {
    warp_loop<PATH, MULTI>(P, ts, sbase, pl);
  } else {
    trial_loop<PATH, MULTI>(P, ts, sbase, g, pl);
  }
}

constexpr uint32_t kPreTau = 8;  // tau values per thread computed before the PDL wait


template <int PATH, bool MULTI>
__global__ void __launch_bounds__(1024, 1) select_shared_kernel(const SharedParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint64_t stage_bar;
  __shared__ uint32_t s_g;
#ifdef GPUAR_TIMELINE
  TL_CTA(0, tl_now());
  {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    TL_CTA(3, smid);
  }
#endif
  // Programmatic dependent launch: this grid may be resident before the previous kernel of
  // the stream has finished (its CTAs fill the SM slots freed by that kernel's tail).  Before
  // the wait below it touches only what this handle's set_propensities kernels produced --
  // the thresholds / prefilter and the statistics: those kernels never trigger their
  // dependents early (kernels_misc.cu), and every other grid of the stream either triggers
  // only after its own wait (so everything before it has completed) or is a plain launch, so
  // when this grid starts they have completed and their writes are visible.  Outputs,
  // tickets and alpha are touched only after the wait.
  // ---- stage the thresholds (path 1) or their prefilter (paths 2, 3) in smem with one bulk async
  // copy per CTA (16-byte hull; the data starts `sbase` bytes into it), issued first so that
  // it overlaps the statistics load, the wait and the tau phase
  const uint32_t sbase = (PATH == kPathSmemF32) ? stage_issue(smem, P.thr, 4u * P.M, &stage_bar)
                                                : stage_issue(smem, P.prefilter, 2u * P.n_pref, &stage_bar);
  const DevStats st = *P.stats;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t nthreads = gridDim.x * blockDim.x;
  const bool invalid = st.valid == 0u;
  const bool zero = st.amax_bits == 0u;
  const uint32_t K = P.K;
  const uint32_t nwarps = nthreads >> 5;
  const TrialStream ts(P.seed_lo, P.seed_hi, P.epoch);  // (also tau's round keys)
  const TauDiv tdiv = tau_div(st.a0f);
  if (threadIdx.x == 0) s_g = P.team_override ? P.team_override : choose_team(st.p, K, nwarps);  // once per CTA
  // tau of this thread's first kPreTau selections, computed before the wait (pure arithmetic
  // on the statistics) and stored after it: on an SM the previous call left early this work
  // overlaps that call's drain
  // (only when every thread has at least one: c2's 65 536 selections over 151 552 threads gain
  // nothing and measured -1.5 %)
  const bool want_tau = P.tau != nullptr && !invalid && !zero && K >= nthreads;
  float pre_tau[kPreTau];
#pragma unroll
  for (uint32_t i = 0; i < kPreTau; ++i) {
    const uint32_t s = tid + i * nthreads;
    pre_tau[i] = 0.f;
    if (want_tau && s < K) pre_tau[i] = tdiv(item_neg_log_u1<MULTI>(P, ts, s));
  }
  // every prerequisite grid complete; then let the next launch be scheduled early
  pdl_wait();
  pdl_launch_dependents();
#ifdef GPUAR_TIMELINE
  TL_CTA(1, tl_now());
#endif
  // the next launch's ticket set (its previous user, launch n - 1, has completed)
  if (blockIdx.x == 0 && threadIdx.x < kStripes) P.ctr->next[P.phase ^ 1u][threadIdx.x] = 0ull;

  // ---- phase A: tau for every selection (the first kPreTau per thread already computed);
  // degenerate / invalid outputs
  if (want_tau) {
#pragma unroll
    for (uint32_t i = 0; i < kPreTau; ++i) {
      const uint32_t s = tid + i * nthreads;
      if (s < K) P.tau[s] = pre_tau[i];
    }
  }
  for (uint32_t s = tid + (want_tau ? kPreTau * nthreads : 0u); s < K; s += nthreads) {
    if (invalid || zero) {
      P.idx[s] = -1;
      if (P.trials) P.trials[s] = 0u;
      if (P.tau) P.tau[s] = invalid ? __uint_as_float(0x7fc00000u) : __uint_as_float(kInfBits);
    } else if (P.tau) {
      P.tau[s] = tdiv(item_neg_log_u1<MULTI>(P, ts, s));
    }
  }
  __syncthreads();        // publishes the barrier's initialisation and s_g
  stage_wait(&stage_bar);  // (also before an early exit: no copy may outlive the CTA)
  if (invalid || zero) return;  // uniform over the grid; the tickets are untouched
#ifdef GPUAR_TIMELINE
  TL_CTA(2, tl_now());
#endif

  // ---- phase C: trials
  const uint32_t warp_global = tid >> 5;
  const uint32_t g = s_g;
  if (tid == 0) P.ctr->team = g;
  Pool pl;
  pool_setup(P, st, g, nwarps, warp_global, pl);
  pool_start(pl, threadIdx.x & 31u);
  run_trials<PATH, MULTI>(P, st, ts, sbase, g, pl);
#ifdef GPUAR_TIMELINE
  if ((threadIdx.x & 31u) == 0u) g_tl[P.epoch & 1u][kTlCta + warp_global] = tl_now();
#endif
}

// Fewer work items than threads (c1, c2): at most one tau per thread, so there is no tau to
// compute before the PDL wait (it gained nothing there); instead whole-warp
// teams (g = 32) work the first <= 32 items of their static chunk before the wait -- pure
// arithmetic on the staged thresholds and the statistics, lane k holding item k's result
// until the stores after the wait.  On an SM the previous call left early this overlaps that
// call's end, which otherwise idles ~2.7 us of a 28 us c2 call (scripts/diag_timeline.py).
// The same outputs as select_shared_kernel; a separate kernel so that the K >= threads
// configurations keep their code (the pre-wait loop costs registers: 46 -> ~60).
template <int PATH>
__global__ void __launch_bounds__(1024, 1) select_shared_pre_kernel(const SharedParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint64_t stage_bar;
  __shared__ uint32_t s_g;
#ifdef GPUAR_TIMELINE
  TL_CTA(0, tl_now());
  {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    TL_CTA(3, smid);
  }
#endif
  // before the wait: only the thresholds / prefilter and the statistics (see select_shared_kernel)
  const uint32_t sbase = (PATH == kPathSmemF32) ? stage_issue(smem, P.thr, 4u * P.M, &stage_bar)
                                                : stage_issue(smem, P.prefilter, 2u * P.n_pref, &stage_bar);
  const DevStats st = *P.stats;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t nthreads = gridDim.x * blockDim.x;
  const bool invalid = st.valid == 0u;
  const bool zero = st.amax_bits == 0u;
  const uint32_t K = P.K;
  const uint32_t nwarps = nthreads >> 5;
  if (threadIdx.x == 0) s_g = P.team_override ? P.team_override : choose_team(st.p, K, nwarps);  // once per CTA
  __syncthreads();         // publishes the barrier's initialisation and s_g
  stage_wait(&stage_bar);  // (also before an early exit: no copy may outlive the CTA)
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t warp_global = tid >> 5;
  const uint32_t g = s_g;
  Pool pl;
  pool_setup(P, st, g, nwarps, warp_global, pl);
  const TrialStream ts(P.seed_lo, P.seed_hi, P.epoch);
  const TauDiv tdiv = tau_div(st.a0f);
  uint32_t pre_n = 0;
  const uint32_t pre_base = pl.next;
  int32_t pre_id = -1;
  uint32_t pre_tr = 0;
  if (g == 32u && !invalid && !zero) {
    pre_n = min(32u, pl.end - pl.next);
    for (uint32_t k = 0; k < pre_n; ++k) {
      int32_t id;
      uint32_t tr;
      warp_select<PATH, false>(P, ts, sbase, pre_base + k, lane, id, tr);
      if (lane == k) {
        pre_id = id;
        pre_tr = tr;
      }
    }
    pl.next += pre_n;
  }
  // every prerequisite grid complete; then let the next launch be scheduled early
  pdl_wait();
  pdl_launch_dependents();
#ifdef GPUAR_TIMELINE
  TL_CTA(1, tl_now());
#endif
  // the next launch's ticket set (its previous user, launch n - 1, has completed)
  if (blockIdx.x == 0 && threadIdx.x < kStripes) P.ctr->next[P.phase ^ 1u][threadIdx.x] = 0ull;
  // tau (at most one per thread); degenerate / invalid outputs
  for (uint32_t s = tid; s < K; s += nthreads) {
    if (invalid || zero) {
      P.idx[s] = -1;
      if (P.trials) P.trials[s] = 0u;
      if (P.tau) P.tau[s] = invalid ? __uint_as_float(0x7fc00000u) : __uint_as_float(kInfBits);
    } else if (P.tau) {
      P.tau[s] = tdiv(item_neg_log_u1<false>(P, ts, s));
    }
  }
  if (invalid || zero) return;  // uniform over the grid; the tickets are untouched
#ifdef GPUAR_TIMELINE
  TL_CTA(2, tl_now());
#endif
  if (lane < pre_n) {
    P.idx[pre_base + lane] = pre_id;
    if (P.trials) P.trials[pre_base + lane] = pre_tr;
  }
  if (tid == 0) P.ctr->team = g;
  pool_start(pl, lane);
  run_trials<PATH, false>(P, st, ts, sbase, g, pl);
#ifdef GPUAR_TIMELINE
  if (lane == 0u) g_tl[P.epoch & 1u][kTlCta + warp_global] = tl_now();
#endif
}

template <int PATH>
void set_limit(int bytes) {
  set_max_dynamic_smem(select_shared_kernel<PATH, false>, bytes);
  set_max_dynamic_smem(select_shared_kernel<PATH, true>, bytes);
  set_max_dynamic_smem(select_shared_pre_kernel<PATH>, bytes);
}

}  // namespace

#ifdef GPUAR_TIMELINE
extern "C" int gpuar_dbg_timeline(void* host, size_t bytes) {
  return (int)cudaMemcpyFromSymbol(host, g_tl, bytes < sizeof(g_tl) ? bytes : sizeof(g_tl));
}
#endif

cudaError_t launch_select_shared(const SharedParams& p, int path, int grid, int block, cudaStream_t st, bool pdl) {
  const size_t sh = p.smem_bytes;
  const bool multi = p.n_epochs > 1u;
  // fewer work items than threads: the variant that works trials before the PDL wait
  const bool pre = !multi && (uint64_t)p.K < (uint64_t)grid * (uint64_t)block;
  switch (path) {
    case kPathSmemF32:
      return multi ? launch_pdl(select_shared_kernel<kPathSmemF32, true>, grid, block, sh, st, pdl, p)
             : pre ? launch_pdl(select_shared_pre_kernel<kPathSmemF32>, grid, block, sh, st, pdl, p)
                   : launch_pdl(select_shared_kernel<kPathSmemF32, false>, grid, block, sh, st, pdl, p);
    case kPathSmemBf16:
      return multi ? launch_pdl(select_shared_kernel<kPathSmemBf16, true>, grid, block, sh, st, pdl, p)
             : pre ? launch_pdl(select_shared_pre_kernel<kPathSmemBf16>, grid, block, sh, st, pdl, p)
                   : launch_pdl(select_shared_kernel<kPathSmemBf16, false>, grid, block, sh, st, pdl, p);
    case kPathSmemGroup:
      return multi ? launch_pdl(select_shared_kernel<kPathSmemGroup, true>, grid, block, sh, st, pdl, p)
             : pre ? launch_pdl(select_shared_pre_kernel<kPathSmemGroup>, grid, block, sh, st, pdl, p)
                   : launch_pdl(select_shared_kernel<kPathSmemGroup, false>, grid, block, sh, st, pdl, p);
    default:
      return cudaErrorInvalidValue;
  }
}

int select_shared_blocks_per_sm(int path, int block, size_t smem) {
  int n = 0;
  cudaError_t e = cudaErrorInvalidValue;
  if (path == kPathSmemF32)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, select_shared_kernel<kPathSmemF32, false>, block, smem);
  else if (path == kPathSmemBf16)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, select_shared_kernel<kPathSmemBf16, false>, block, smem);
  else if (path == kPathSmemGroup)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, select_shared_kernel<kPathSmemGroup, false>, block, smem);
  return e == cudaSuccess ? n : 0;
}

void set_select_shared_limits(int bytes) {
  set_limit<kPathSmemF32>(bytes);
  set_limit<kPathSmemBf16>(bytes);
  set_limit<kPathSmemGroup>(bytes);
}

}  // namespace gpuar
