// philox.cuh -- Philox4x32-10 in registers (Salmon et al., SC'11), the counter-based
// stream BASELINE.json's north_star fixes for GPU-AR.  The paper instead filled a K x M
// array of uniforms in global memory with a third-party generator (PAPER.md:455-459,
// 713-714); a counter-based generator needs no storage and makes every selection's
// draws a pure function of (seed, selection, epoch, call).
#pragma once
#include <cstdint>

namespace gpuar {

constexpr uint32_t kPhiloxM0 = 0xD2511F53u;
constexpr uint32_t kPhiloxM1 = 0xCD9E8D57u;
constexpr uint32_t kPhiloxW0 = 0x9E3779B9u;
constexpr uint32_t kPhiloxW1 = 0xBB67AE85u;

// Stream tags (counter word 3), R12.
constexpr uint32_t kTagTrials = 0u;
constexpr uint32_t kTagTau = 1u;
constexpr uint32_t kTagIT = 2u;       // inverse transform: u2 = word x0 of call 0
constexpr uint32_t kTagElection = 3u;  // the paper's argmin rule: call j >> 2, word j & 3

struct Philox4 {
  uint32_t x, y, z, w;
};

// One round: (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2, c = (hi1^c1^k0, lo1, hi0^c3^k1, lo0).
// mul.wide.u32 gives hi and lo in one IMAD.WIDE.U32.
__device__ __forceinline__ void philox_round(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3, uint32_t k0,
                                             uint32_t k1) {
  const uint64_t p0 = (uint64_t)kPhiloxM0 * c0;
  const uint64_t p1 = (uint64_t)kPhiloxM1 * c2;
  const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
  const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
  c0 = hi1 ^ c1 ^ k0;
  c1 = lo1;
  c2 = hi0 ^ c3 ^ k1;
  c3 = lo0;
}

// Ten rounds; key += Weyl constants between rounds.
__device__ __forceinline__ Philox4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                                 uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    philox_round(c0, c1, c2, c3, k0, k1);
    k0 += kPhiloxW0;
    k1 += kPhiloxW1;
  }
  return Philox4{c0, c1, c2, c3};
}

// The trial stream with everything that is invariant hoisted: counter = {c, s, epoch, tag}.
// Round 1 of M1*c2 involves only the epoch (warp-uniform), and c1 = s, c3 = tag, so round 1
// collapses to one IMAD.WIDE: c0' = hi(M1*epoch) ^ s ^ k0, c1' = lo(M1*epoch),
// c2' = hi(M0*c) ^ tag ^ k1, c3' = lo(M0*c).  Rounds 2..10 use precomputed round keys.  The
// output is bit-identical to philox4x32_10(c, s, epoch, tag, k0, k1) (same arithmetic).
struct TrialStream {
  uint32_t rk0[10], rk1[10];  // round keys (warp-uniform)
  uint32_t e_hi_k0;           // hi(M1*epoch) ^ k0
  uint32_t e_lo;              // lo(M1*epoch)
  uint32_t k1_tag;            // k1 ^ tag (counter word 3 enters round 1 only)

  __device__ __forceinline__ TrialStream(uint32_t seed_lo, uint32_t seed_hi, uint32_t epoch,
                                         uint32_t tag = kTagTrials) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      rk0[r] = seed_lo + (uint32_t)r * kPhiloxW0;
      rk1[r] = seed_hi + (uint32_t)r * kPhiloxW1;
    }
    const uint64_t p1 = (uint64_t)kPhiloxM1 * epoch;
    e_hi_k0 = (uint32_t)(p1 >> 32) ^ seed_lo;
    e_lo = (uint32_t)p1;
    k1_tag = seed_hi ^ tag;
  }

  // switch to another epoch (counter word 2) keeping the round keys
  __device__ __forceinline__ void set_epoch(uint32_t epoch) {
    const uint64_t p1 = (uint64_t)kPhiloxM1 * epoch;
    e_hi_k0 = (uint32_t)(p1 >> 32) ^ rk0[0];
    e_lo = (uint32_t)p1;
  }

  // per-selection constant of round 1
  __device__ __forceinline__ uint32_t sel_word(uint32_t s) const { return e_hi_k0 ^ s; }

  // both round-1 constants of selection s at another epoch (multi-epoch launches): the
  // per-selection word and lo(M1*epoch), which call() takes instead of the member e_lo
  __device__ __forceinline__ void words(uint32_t epoch, uint32_t s, uint32_t& sel, uint32_t& elo) const {
    const uint64_t p1 = (uint64_t)kPhiloxM1 * epoch;
    sel = (uint32_t)(p1 >> 32) ^ rk0[0] ^ s;
    elo = (uint32_t)p1;
  }
  __device__ __forceinline__ Philox4 call(uint32_t c, uint32_t sel, uint32_t elo) const {
    const uint64_t p0 = (uint64_t)kPhiloxM0 * c;
    uint32_t c0 = sel, c1 = elo, c2 = (uint32_t)(p0 >> 32) ^ k1_tag, c3 = (uint32_t)p0;
#pragma unroll
    for (int r = 1; r < 10; ++r) philox_round(c0, c1, c2, c3, rk0[r], rk1[r]);
    return Philox4{c0, c1, c2, c3};
  }

  // call() with another stream tag: k1t = seed_hi ^ tag
  __device__ __forceinline__ Philox4 call_tag(uint32_t c, uint32_t sel, uint32_t elo, uint32_t k1t) const {
    const uint64_t p0 = (uint64_t)kPhiloxM0 * c;
    uint32_t c0 = sel, c1 = elo, c2 = (uint32_t)(p0 >> 32) ^ k1t, c3 = (uint32_t)p0;
#pragma unroll
    for (int r = 1; r < 10; ++r) philox_round(c0, c1, c2, c3, rk0[r], rk1[r]);
    return Philox4{c0, c1, c2, c3};
  }

  __device__ __forceinline__ Philox4 operator()(uint32_t c, uint32_t sel) const { return with_tag(c, sel, k1_tag); }

  // same stream family with another tag: k1t = seed_hi ^ tag
  __device__ __forceinline__ Philox4 with_tag(uint32_t c, uint32_t sel, uint32_t k1t) const {
    const uint64_t p0 = (uint64_t)kPhiloxM0 * c;
    uint32_t c0 = sel, c1 = e_lo, c2 = (uint32_t)(p0 >> 32) ^ k1t, c3 = (uint32_t)p0;
#pragma unroll
    for (int r = 1; r < 10; ++r) philox_round(c0, c1, c2, c3, rk0[r], rk1[r]);
    return Philox4{c0, c1, c2, c3};
  }
};

// u = (x >> 8) * 2^-24 in [0,1): 24 random bits, exact in binary32 (R3).
__device__ __forceinline__ float unit24(uint32_t x) {
  return __fmul_rn(__uint2float_rn(x >> 8), 0x1p-24f);
}

// fl32(u * amax) for u = (x >> 8) 2^-24.  With amax_s = amax * 2^-24 exact (amax >=
// 2^-102, so no underflow), (x>>8) * amax_s is the same real product, hence the same
// round-to-nearest result, with one multiply instead of two.
template <bool FOLD>
__device__ __forceinline__ float scaled_u(uint32_t x, float amax, float amax_s) {
  if constexpr (FOLD)
    return __fmul_rn(__uint2float_rn(x >> 8), amax_s);
  else
    return __fmul_rn(unit24(x), amax);
}

// u1 = (2 (x >> 9) + 1) * 2^-24 in (0,1) (R10).
__device__ __forceinline__ float unit24_open(uint32_t x) {
  return __fmul_rn(__uint2float_rn(((x >> 9) << 1) | 1u), 0x1p-24f);
}

// tau = ln(1/u1) / alpha_0 in binary32: -logf(u1) / a0f.
__device__ __forceinline__ float neg_log_u1(uint32_t seed_lo, uint32_t seed_hi, uint32_t s, uint32_t epoch) {
  const Philox4 t = philox4x32_10(0u, s, epoch, kTagTau, seed_lo, seed_hi);
  return -logf(unit24_open(t.x));
}

// The same -ln(u1) from a TrialStream of the same seed (any tag; its round keys are already
// in registers, so the call skips the key schedule -- ~16 instructions per tau): counter
// {0, s, epoch, kTagTau} with sel / elo the stream's round-1 words of (s, epoch).
__device__ __forceinline__ float neg_log_u1_ts(const TrialStream& ts, uint32_t sel, uint32_t elo) {
  return -logf(unit24_open(ts.call_tag(0u, sel, elo, ts.rk1[0] ^ kTagTau).x));
}

// amax >= 2^-102  <=>  amax * 2^-24 is a normal binary32 (exact scaling)
__device__ __forceinline__ bool can_fold(uint32_t amax_bits) { return amax_bits >= 0x0C800000u; }

}  // namespace gpuar
