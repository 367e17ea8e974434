// ising_kernels.cu — sm_100a kernels of the multi-spin checkerboard Metropolis path.
//
//   k_halfsweep  one colour phase of one slab: nibble
//                SWAR neighbour sums, inline Philox4x32-10, integer acceptance,
//                XOR flip, 128-bit store, fused halo store.  PAPER.md:212-218 §3.3.
//   k_init       random / cold start (row a3), halo rows included.
//   k_observables popcount up-spins and antiparallel bonds (row a8), Eq. 1.
//   k_pack / k_unpack  +-1 byte full lattice <-> packed planes (row a9).
//
// All arithmetic is integer.  Nothing here is shared with oracle/.
#include <algorithm>
#include <cstdio>
#include <type_traits>
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "ising_kernels.cuh"

namespace ising {

// ------------------------------------------------------------------ Philox
// Philox4x32-10 (Salmon et al., SC'11), the generator the paper uses through
// cuRAND.  Counter {c0, c1, c2, c3}; the key schedule is
// precomputed per launch (PhiloxKeys) so each round is 2 IMAD.WIDE.U32 + 2 LOP3.
// With the site counter {t, j/4, c, i} (reading R6) only word 1 varies across a warp, so
// round 1's two products and one product each of rounds 2 and 3 are warp-uniform:
// 16 of the 20 multiplies per block are per-thread work.
__device__ __forceinline__ uint4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                               const PhiloxKeys& K) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)c0 * kPhiloxM0;
    const uint64_t p1 = (uint64_t)c2 * kPhiloxM1;
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ K.k0[r];
    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ K.k1[r];
    c1 = (uint32_t)p1;
    c3 = (uint32_t)p0;
    c0 = n0;
    c2 = n2;
  }
  return make_uint4(c0, c1, c2, c3);
}

constexpr uint32_t kLane0 = 0x11111111u;  // bit 0 of every nibble of a 32-bit half

// Side-word splices (reading R10) as funnel shifts on the 32-bit halves (two
// SHF per word, no IMAD.SHL on the FMA pipe): west = (C << 4) | (L >> 60) with L the word to
// the left, east = (C >> 4) | (R << 60) with R the word to the right.
__device__ __forceinline__ uint64_t splice_west(uint64_t c, uint64_t l) {
  const uint32_t lo = __funnelshift_l((uint32_t)(l >> 32), (uint32_t)c, 4);
  const uint32_t hi = __funnelshift_l((uint32_t)c, (uint32_t)(c >> 32), 4);
  return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ uint64_t splice_east(uint64_t c, uint64_t r) {
  const uint32_t lo = __funnelshift_r((uint32_t)c, (uint32_t)(c >> 32), 4);
  const uint32_t hi = __funnelshift_r((uint32_t)(c >> 32), (uint32_t)r, 4);
  return ((uint64_t)hi << 32) | lo;
}

// One 64-bit target word: 16 spins of plane row `row` (global), plane columns
// 4*ctr0 .. 4*ctr0 + 15.  n, c, s: source words above / same / below; side: the
// spliced side word.  Metropolis acceptance:
// flip iff a <= 2 (e <= 0) or r < T[e].
template <int RULE>
__device__ __forceinline__ uint64_t update_word(uint64_t tgt, uint64_t n, uint64_t c, uint64_t s,
                                                uint64_t side, uint32_t ctr0, uint32_t row, uint32_t t,
                                                const HalfSweepParams& p);

// Acceptance test of one lane against both thresholds, on the carry chain: the
// borrow-free carry of r - T is [r >= T] ("no flip for this class"), and madc shifts it
// into the accumulator's next nibble, acc = 16 acc + carry (sub.cc -> IADD3 on the ALU
// pipe, madc -> IMAD.X on the FMA pipe), so lanes arrive in descending order.  Measured
// alternatives (profiles/r01_ncu_halfsweep.md): ISETP + predicated OR for one threshold —
// 1 % slower; an ALU-only insert (3-input LOP3) — 11 % slower.
__device__ __forceinline__ void nc_step(uint32_t& a3, uint32_t& a4, uint32_t r, uint32_t t3,
                                        uint32_t t4) {
  asm("{\n\t.reg .u32 d;\n\t"
      "sub.cc.u32 d, %2, %3;\n\t"
      "madc.lo.u32 %0, %0, 16, 0;\n\t"
      "sub.cc.u32 d, %2, %4;\n\t"
      "madc.lo.u32 %1, %1, 16, 0;\n\t}"
      : "+r"(a3), "+r"(a4)
      : "r"(r), "r"(t3), "r"(t4));
}

// Flip decision for 8 lanes (one 32-bit half).  With b = number of neighbours anti-aligned
// with the spin, cnt = [r < T_3] + [r < T_4] and T_4 <= T_3, Metropolis flips iff
// a - 2 <= cnt (a = 4 - b aligned), i.e. iff b - nc >= 0 with nc = 2 - cnt = a3 + a4 (the
// Horner accumulators).  Per lane x = b + 8 - nc lies in [6, 12]; bit 3 of x is the flip bit.
// b per lane is the sum of the four XORs of the spin with its neighbours (lanes hold 0/1 in
// bit 0, sums <= 4: no carries) — four LOP3 and two adds on the ALU pipe, where the
// s ? 4 - n : n form of the up-neighbour count took two IMADs on the FMA pipe.
#ifndef ISING_ANTI_XOR
#define ISING_ANTI_XOR 0
#endif
__device__ __forceinline__ uint32_t anti8(uint32_t t, uint32_t n, uint32_t c, uint32_t s,
                                          uint32_t side) {
  return (t ^ n) + (t ^ c) + (t ^ s) + (t ^ side);
}

__device__ __forceinline__ uint32_t flip8(uint32_t t, uint32_t b, uint32_t nc) {
  const uint32_t x = b + 0x88888888u - nc;
  return t ^ ((x >> 3) & kLane0);
}

// (the up-count form, kept for the heat-bath kernels)
__device__ __forceinline__ uint32_t accept8(uint32_t s, uint32_t n, uint32_t nc) {
  const uint32_t x = (n ^ (s * 15u)) + (s * (uint32_t)-11 + 0x88888888u) - nc;
  return s ^ ((x >> 3) & kLane0);
}

// RULE 0: Metropolis, both thresholds < 2^32.
// RULE 2: Metropolis, generic (a threshold may be 2^32: the accumulators are masked).
template <int RULE>
__device__ __forceinline__ uint64_t update_word_metropolis(uint64_t tgt, uint64_t n, uint64_t c,
                                                           uint64_t s, uint64_t side, uint32_t ctr0,
                                                           uint32_t row, uint32_t t, const HalfSweepParams& p) {
  constexpr bool kSingle = RULE == 0;
  // "three additions are sufficient to compute the neighbors sums": here the
  // sums of the XORs with the target (anti-aligned neighbours); lanes hold 0/1 and sums <= 4,
  // so the 64-bit adds split into independent 32-bit halves.
#if ISING_ANTI_XOR
  const uint32_t b_lo = anti8((uint32_t)tgt, (uint32_t)n, (uint32_t)c, (uint32_t)s, (uint32_t)side);
  const uint32_t b_hi = anti8((uint32_t)(tgt >> 32), (uint32_t)(n >> 32), (uint32_t)(c >> 32),
                              (uint32_t)(s >> 32), (uint32_t)(side >> 32));
#else
  const uint32_t sum_lo = (uint32_t)n + (uint32_t)c + (uint32_t)s + (uint32_t)side;
  const uint32_t sum_hi =
      (uint32_t)(n >> 32) + (uint32_t)(c >> 32) + (uint32_t)(s >> 32) + (uint32_t)(side >> 32);
#endif
  const uint32_t t3 = p.acc.thr[3], t4 = p.acc.thr[4];
  // lanes k = 4b + q; Horner order is lane 7 .. 0 (lo half) and 15 .. 8 (hi half)
  uint32_t a3lo = 0, a4lo = 0, a3hi = 0, a4hi = 0;
  {
    const uint4 r1 = philox4x32_10(t, ctr0 + 1, p.colour, row, p.keys);
    nc_step(a3lo, a4lo, r1.w, t3, t4);
    nc_step(a3lo, a4lo, r1.z, t3, t4);
    nc_step(a3lo, a4lo, r1.y, t3, t4);
    nc_step(a3lo, a4lo, r1.x, t3, t4);
    const uint4 r0 = philox4x32_10(t, ctr0 + 0, p.colour, row, p.keys);
    nc_step(a3lo, a4lo, r0.w, t3, t4);
    nc_step(a3lo, a4lo, r0.z, t3, t4);
    nc_step(a3lo, a4lo, r0.y, t3, t4);
    nc_step(a3lo, a4lo, r0.x, t3, t4);
  }
  {
    const uint4 r3 = philox4x32_10(t, ctr0 + 3, p.colour, row, p.keys);
    nc_step(a3hi, a4hi, r3.w, t3, t4);
    nc_step(a3hi, a4hi, r3.z, t3, t4);
    nc_step(a3hi, a4hi, r3.y, t3, t4);
    nc_step(a3hi, a4hi, r3.x, t3, t4);
    const uint4 r2 = philox4x32_10(t, ctr0 + 2, p.colour, row, p.keys);
    nc_step(a3hi, a4hi, r2.w, t3, t4);
    nc_step(a3hi, a4hi, r2.z, t3, t4);
    nc_step(a3hi, a4hi, r2.y, t3, t4);
    nc_step(a3hi, a4hi, r2.x, t3, t4);
  }
  uint32_t nclo, nchi;
  if (kSingle) {
    nclo = a3lo + a4lo;
    nchi = a3hi + a4hi;
  } else {
    // a class whose threshold is 2^32 ("always", tiny beta) never blocks a flip
    const uint32_t k3 = p.acc.keep3, k4 = p.acc.keep4;
    nclo = (a3lo & k3) + (a4lo & k4);
    nchi = (a3hi & k3) + (a4hi & k4);
  }
#if ISING_ANTI_XOR
  const uint32_t lo = flip8((uint32_t)tgt, b_lo, nclo);
  const uint32_t hi = flip8((uint32_t)(tgt >> 32), b_hi, nchi);
#else
  const uint32_t lo = accept8((uint32_t)tgt, sum_lo, nclo);
  const uint32_t hi = accept8((uint32_t)(tgt >> 32), sum_hi, nchi);
#endif
  return ((uint64_t)hi << 32) | lo;
}

template <>
__device__ __forceinline__ uint64_t update_word<0>(uint64_t tgt, uint64_t n, uint64_t c, uint64_t s,
                                                   uint64_t side, uint32_t ctr0, uint32_t row, uint32_t t,
                                                   const HalfSweepParams& p) {
  return update_word_metropolis<0>(tgt, n, c, s, side, ctr0, row, t, p);
}

template <>
__device__ __forceinline__ uint64_t update_word<2>(uint64_t tgt, uint64_t n, uint64_t c, uint64_t s,
                                                   uint64_t side, uint32_t ctr0, uint32_t row, uint32_t t,
                                                   const HalfSweepParams& p) {
  return update_word_metropolis<2>(tgt, n, c, s, side, ctr0, row, t, p);
}

// RULE 4: Metropolis with both thresholds in {0, 2^32} (beta = inf: zero-temperature
// quench; beta = 0): the acceptance no longer depends on the draw, and with a counter-
// based generator skipping a draw changes nothing else, so no Philox is evaluated.
// nc = [r >= T3] + [r >= T4] is the per-launch constant p.acc.nc_const.
template <>
__device__ __forceinline__ uint64_t update_word<4>(uint64_t tgt, uint64_t n, uint64_t c, uint64_t s,
                                                   uint64_t side, uint32_t ctr0, uint32_t row, uint32_t t,
                                                   const HalfSweepParams& p) {
  const uint32_t sum_lo = (uint32_t)n + (uint32_t)c + (uint32_t)s + (uint32_t)side;
  const uint32_t sum_hi =
      (uint32_t)(n >> 32) + (uint32_t)(c >> 32) + (uint32_t)(s >> 32) + (uint32_t)(side >> 32);
  const uint32_t lo = accept8((uint32_t)tgt, sum_lo, p.acc.nc_const);
  const uint32_t hi = accept8((uint32_t)(tgt >> 32), sum_hi, p.acc.nc_const);
  return ((uint64_t)hi << 32) | lo;
}

// Heat bath, fast path.  The Horner accumulator counts nc = #{m : r >= T[m]} per lane on
// the carry chain (one madc and an addc per further class), and since T is non-increasing
// in a, r < T[a] <=> a + nc <= 4.  With B = a + 3 from classify's SWAR form, x = B + nc <= 12
// and flip <=> bit 3 of x clear.  NA = number of "always" classes (T = 2^32, a prefix of the
// non-increasing T: none for beta < ~2.77, a = 0 up to ~5.5, a = 0, 1 beyond; T[2] = 2^31
// always): [r >= 2^32] = 0 for those, so their compares are simply left out.
template <int NA>
__device__ __forceinline__ void hb_step(uint32_t& acc, uint32_t r, const uint32_t* T) {
  static_assert(NA >= 0 && NA <= 2, "T[2] = 2^31 is never 'always'");
  if constexpr (NA == 0)
    asm("{\n\t.reg .u32 d;\n\t"
        "sub.cc.u32 d, %1, %2;\n\t"
        "madc.lo.u32 %0, %0, 16, 0;\n\t"
        "sub.cc.u32 d, %1, %3;\n\t"
        "addc.u32 %0, %0, 0;\n\t"
        "sub.cc.u32 d, %1, %4;\n\t"
        "addc.u32 %0, %0, 0;\n\t"
        "sub.cc.u32 d, %1, %5;\n\t"
        "addc.u32 %0, %0, 0;\n\t"
        "sub.cc.u32 d, %1, %6;\n\t"
        "addc.u32 %0, %0, 0;\n\t}"
        : "+r"(acc)
        : "r"(r), "r"(T[0]), "r"(T[1]), "r"(T[2]), "r"(T[3]), "r"(T[4]));
  else if constexpr (NA == 1)
    asm("{\n\t.reg .u32 d;\n\t"
        "sub.cc.u32 d, %1, %2;\n\t"
        "madc.lo.u32 %0, %0, 16, 0;\n\t"
        "sub.cc.u32 d, %1, %3;\n\t"
        "addc.u32 %0, %0, 0;\n\t"
        "sub.cc.u32 d, %1, %4;\n\t"
        "addc.u32 %0, %0, 0;\n\t"
        "sub.cc.u32 d, %1, %5;\n\t"
        "addc.u32 %0, %0, 0;\n\t}"
        : "+r"(acc)
        : "r"(r), "r"(T[1]), "r"(T[2]), "r"(T[3]), "r"(T[4]));
  else
    asm("{\n\t.reg .u32 d;\n\t"
        "sub.cc.u32 d, %1, %2;\n\t"
        "madc.lo.u32 %0, %0, 16, 0;\n\t"
        "sub.cc.u32 d, %1, %3;\n\t"
        "addc.u32 %0, %0, 0;\n\t"
        "sub.cc.u32 d, %1, %4;\n\t"
        "addc.u32 %0, %0, 0;\n\t}"
        : "+r"(acc)
        : "r"(r), "r"(T[2]), "r"(T[3]), "r"(T[4]));
}

__device__ __forceinline__ uint32_t hb_accept8(uint32_t s, uint32_t n, uint32_t nc) {
  // a + 3 per lane (a = s ? n : 4 - n): s = 1 -> n + 3; s = 0 -> n ^ 7 = 7 - n
  const uint32_t B = (n + 3u * s) ^ (7u * s) ^ 0x77777777u;
  const uint32_t x = B + nc;
  return s ^ ((~x >> 3) & kLane0);
}

template <int NA>
__device__ __forceinline__ uint64_t update_word_heatbath(uint64_t tgt, uint64_t n, uint64_t c,
                                                         uint64_t s, uint64_t side, uint32_t ctr0,
                                                         uint32_t row, uint32_t t,
                                                         const HalfSweepParams& p) {
  const uint32_t sum_lo = (uint32_t)n + (uint32_t)c + (uint32_t)s + (uint32_t)side;
  const uint32_t sum_hi =
      (uint32_t)(n >> 32) + (uint32_t)(c >> 32) + (uint32_t)(s >> 32) + (uint32_t)(side >> 32);
  const uint32_t* T = p.acc.thr;
  uint32_t lo = 0, hi = 0;
  {
    const uint4 r1 = philox4x32_10(t, ctr0 + 1, p.colour, row, p.keys);
    hb_step<NA>(lo, r1.w, T);
    hb_step<NA>(lo, r1.z, T);
    hb_step<NA>(lo, r1.y, T);
    hb_step<NA>(lo, r1.x, T);
    const uint4 r0 = philox4x32_10(t, ctr0 + 0, p.colour, row, p.keys);
    hb_step<NA>(lo, r0.w, T);
    hb_step<NA>(lo, r0.z, T);
    hb_step<NA>(lo, r0.y, T);
    hb_step<NA>(lo, r0.x, T);
  }
  {
    const uint4 r3 = philox4x32_10(t, ctr0 + 3, p.colour, row, p.keys);
    hb_step<NA>(hi, r3.w, T);
    hb_step<NA>(hi, r3.z, T);
    hb_step<NA>(hi, r3.y, T);
    hb_step<NA>(hi, r3.x, T);
    const uint4 r2 = philox4x32_10(t, ctr0 + 2, p.colour, row, p.keys);
    hb_step<NA>(hi, r2.w, T);
    hb_step<NA>(hi, r2.z, T);
    hb_step<NA>(hi, r2.y, T);
    hb_step<NA>(hi, r2.x, T);
  }
  const uint32_t flo = hb_accept8((uint32_t)tgt, sum_lo, lo);
  const uint32_t fhi = hb_accept8((uint32_t)(tgt >> 32), sum_hi, hi);
  return ((uint64_t)fhi << 32) | flo;
}

#define ISING_HB_RULE(RULE, NA)                                                                  \
  template <>                                                                                   \
  __device__ __forceinline__ uint64_t update_word<RULE>(                                        \
      uint64_t tgt, uint64_t n, uint64_t c, uint64_t s, uint64_t side, uint32_t ctr0,           \
      uint32_t row, uint32_t t, const HalfSweepParams& p) {                                     \
    return update_word_heatbath<NA>(tgt, n, c, s, side, ctr0, row, t, p);                       \
  }
ISING_HB_RULE(3, 0)  // RULE 3: every T < 2^32
ISING_HB_RULE(5, 1)  // RULE 5: T[0] = 2^32
ISING_HB_RULE(6, 2)  // RULE 6: T[0] = T[1] = 2^32
#undef ISING_HB_RULE

// Heat bath, symmetric fast path (RULE 7).  Applies when the host has verified T[2] = 2^31 and
// T[0] + T[4] = T[1] + T[3] = 2^32 + 1 — what ceil(2^32 P) gives for P(e) + P(-e) = 1
// unless 2^32 P(e) lands within rounding of an integer, in which case RULE 3 / 5 / 6 run.
// With nc = #{m : r >= T[m]} and T non-increasing:
//   r <  2^31: T[0] >= T[1] > 2^31 > r and r < T[2], so nc = [r >= T3] + [r >= T4];
//   r >= 2^31: r >= T[2] >= T[3] >= T[4], and with v = 2^32 - r (|r| as int32, in [1, 2^31]),
//              r >= T[0] <=> v <= 2^32 - T[0] <=> v < T[4] (likewise T[1] / T[3]), so
//              nc = 3 + (1 - [v >= T4]) + (1 - [v >= T3]) = 5 - ([v >= T3] + [v >= T4]).
// So every lane needs the Metropolis compare pair on v = |r| plus the msb of r: 6 integer
// operations per lane instead of 5 compares and 5 inserts.
__device__ __forceinline__ void hbs_step(uint32_t& a3, uint32_t& a4, uint32_t& am, uint32_t r,
                                         uint32_t t3, uint32_t t4) {
  nc_step(a3, a4, (uint32_t)abs((int32_t)r), t3, t4);
  am = __funnelshift_l(r, am, 4);  // (am << 4) | (r >> 28): r's msb is bit 3 of the new nibble
}

// nc per lane from the compare pair count c (0..2) and the msb bit of the lane's nibble in am
__device__ __forceinline__ uint32_t hbs_nc(uint32_t c, uint32_t am) {
  const uint32_t m = (am >> 3) & kLane0;
  const uint32_t m15 = (m << 4) - m;  // 0xF in lanes with r >= 2^31
  return (c ^ m15) - (m15 & 0xAAAAAAAAu);  // m: (15 - c) - 10 = 5 - c; else c (no borrows)
}

template <>
__device__ __forceinline__ uint64_t update_word<7>(uint64_t tgt, uint64_t n, uint64_t c, uint64_t s,
                                                   uint64_t side, uint32_t ctr0, uint32_t row, uint32_t t,
                                                   const HalfSweepParams& p) {
  const uint32_t sum_lo = (uint32_t)n + (uint32_t)c + (uint32_t)s + (uint32_t)side;
  const uint32_t sum_hi =
      (uint32_t)(n >> 32) + (uint32_t)(c >> 32) + (uint32_t)(s >> 32) + (uint32_t)(side >> 32);
  const uint32_t t3 = p.acc.thr[3], t4 = p.acc.thr[4];
  uint32_t a3lo = 0, a4lo = 0, amlo = 0, a3hi = 0, a4hi = 0, amhi = 0;
  {
    const uint4 r1 = philox4x32_10(t, ctr0 + 1, p.colour, row, p.keys);
    hbs_step(a3lo, a4lo, amlo, r1.w, t3, t4);
    hbs_step(a3lo, a4lo, amlo, r1.z, t3, t4);
    hbs_step(a3lo, a4lo, amlo, r1.y, t3, t4);
    hbs_step(a3lo, a4lo, amlo, r1.x, t3, t4);
    const uint4 r0 = philox4x32_10(t, ctr0 + 0, p.colour, row, p.keys);
    hbs_step(a3lo, a4lo, amlo, r0.w, t3, t4);
    hbs_step(a3lo, a4lo, amlo, r0.z, t3, t4);
    hbs_step(a3lo, a4lo, amlo, r0.y, t3, t4);
    hbs_step(a3lo, a4lo, amlo, r0.x, t3, t4);
  }
  {
    const uint4 r3 = philox4x32_10(t, ctr0 + 3, p.colour, row, p.keys);
    hbs_step(a3hi, a4hi, amhi, r3.w, t3, t4);
    hbs_step(a3hi, a4hi, amhi, r3.z, t3, t4);
    hbs_step(a3hi, a4hi, amhi, r3.y, t3, t4);
    hbs_step(a3hi, a4hi, amhi, r3.x, t3, t4);
    const uint4 r2 = philox4x32_10(t, ctr0 + 2, p.colour, row, p.keys);
    hbs_step(a3hi, a4hi, amhi, r2.w, t3, t4);
    hbs_step(a3hi, a4hi, amhi, r2.z, t3, t4);
    hbs_step(a3hi, a4hi, amhi, r2.y, t3, t4);
    hbs_step(a3hi, a4hi, amhi, r2.x, t3, t4);
  }
  const uint32_t flo = hb_accept8((uint32_t)tgt, sum_lo, hbs_nc(a3lo + a4lo, amlo));
  const uint32_t fhi = hb_accept8((uint32_t)(tgt >> 32), sum_hi, hbs_nc(a3hi + a4hi, amhi));
  return ((uint64_t)fhi << 32) | flo;
}

// Heat bath, generic (some threshold is 2^32): flip iff r < T[a] for every class.
// T is non-increasing in a, so "r < T[a]" <=> a < #{m : r < T[m]}.
template <>
__device__ __forceinline__ uint64_t update_word<1>(uint64_t tgt, uint64_t n, uint64_t c, uint64_t s,
                                                   uint64_t side, uint32_t ctr0, uint32_t row, uint32_t t,
                                                   const HalfSweepParams& p) {
  const uint64_t sum = n + c + s + side;  // no inter-lane carries (sums <= 4)
  // a = s ? n : 4 - n per lane
  const uint64_t S = tgt & 0x1111111111111111ull;
  const uint64_t mask = (S << 4) - S;  // 0xF in lanes with s = 1
  const uint64_t a = (sum & mask) | ((0x4444444444444444ull - sum) & ~mask);
  uint64_t flip = 0;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const uint4 r = philox4x32_10(t, ctr0 + b, p.colour, row, p.keys);
    const uint32_t rr[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int k = 4 * b + q;
      const uint32_t ak = (uint32_t)(a >> (4 * k)) & 7u;
      uint32_t cnt = 0;
#pragma unroll
      for (int m = 0; m < 5; ++m)
        cnt += ((p.acc.always_mask >> m) & 1u) | (rr[q] < p.acc.thr[m] ? 1u : 0u);
      // always-classes form a prefix of the non-increasing T, so cnt is still
      // "number of classes m with r < T[m]" with T[m] = 2^32 counted.
      if (ak < cnt) flip |= 1ull << (4 * k);
    }
  }
  return tgt ^ flip;
}

// Eight Philox blocks (counter words 1 = c1base + b, b = 0..7) advanced round by round in
// lockstep — the two words of a thread's 128-bit chunk.  Written this way (rather than block by
// block inside update_word) ptxas schedules the staged kernel's row better: Metropolis
// 1541 -> 1551, symmetric heat bath 1276 -> 1303 flips/ns on C3 (ISING_PHILOX8=0: old form).
#ifndef ISING_PHILOX8
#define ISING_PHILOX8 1
#endif
#ifndef ISING_PROBE8
// 1: the probe advances eight blocks per thread in lockstep, like the kernels (1899 -> 2005
// draws/ns); 2: and walks rows with a fixed column chunk per thread, as the half-sweeps do —
// the products that do not depend on the row (round 2's per-block c0 * M0) leave the loop
// there too, so the probe does the same per-draw multiply work as the kernels
#define ISING_PROBE8 2
#endif
__device__ __forceinline__ void philox8(uint32_t t, uint32_t c1base, uint32_t colour, uint32_t row,
                                        const PhiloxKeys& K, uint4 (&out)[8]) {
  uint32_t c0[8], c1[8], c2[8], c3[8];
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    c0[b] = t;
    c1[b] = c1base + b;
    c2[b] = colour;
    c3[b] = row;
  }
#pragma unroll
  for (int r = 0; r < 10; ++r) {
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const uint64_t p0 = (uint64_t)c0[b] * kPhiloxM0;
      const uint64_t p1 = (uint64_t)c2[b] * kPhiloxM1;
      const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1[b] ^ K.k0[r];
      const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3[b] ^ K.k1[r];
      c1[b] = (uint32_t)p1;
      c3[b] = (uint32_t)p0;
      c0[b] = n0;
      c2[b] = n2;
    }
  }
#pragma unroll
  for (int b = 0; b < 8; ++b) out[b] = make_uint4(c0[b], c1[b], c2[b], c3[b]);
}

// philox8 with round 1's per-block product given: for colour <= 1, round 0 leaves block b's
// counter word 0 at (c1base + b) ^ k0[0] (hi(colour * M1) = 0), so round 1's c0 * M0 depends on
// the column only — a thread that keeps its column for many rows / sweeps computes
// P1[b] = ((c1base + b) ^ k0[0]) * M0 once (philox8_round1) and saves 8 multiplies per call.
__device__ __forceinline__ void philox8_round1(uint32_t c1base, const PhiloxKeys& K, uint64_t (&P1)[8]) {
#pragma unroll
  for (int b = 0; b < 8; ++b) P1[b] = (uint64_t)((c1base + b) ^ K.k0[0]) * kPhiloxM0;
}
__device__ __forceinline__ void philox8_pre(uint32_t t, uint32_t colour, uint32_t row,
                                            const PhiloxKeys& K, const uint64_t (&P1)[8],
                                            uint4 (&out)[8]) {
  const uint64_t q0 = (uint64_t)t * kPhiloxM0;  // round 0, warp-uniform
  const uint32_t c1r0 = colour * kPhiloxM1;      // lo(colour * M1); hi = 0
  const uint32_t n2 = (uint32_t)(q0 >> 32) ^ row ^ K.k1[0];
  const uint32_t c3r0 = (uint32_t)q0;
  const uint64_t q1 = (uint64_t)n2 * kPhiloxM1;  // round 1, warp-uniform half
  uint32_t c0[8], c1[8], c2[8], c3[8];
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    c0[b] = (uint32_t)(q1 >> 32) ^ c1r0 ^ K.k0[1];
    c1[b] = (uint32_t)q1;
    c2[b] = (uint32_t)(P1[b] >> 32) ^ c3r0 ^ K.k1[1];
    c3[b] = (uint32_t)P1[b];
  }
#pragma unroll
  for (int r = 2; r < 10; ++r) {
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const uint64_t p0 = (uint64_t)c0[b] * kPhiloxM0;
      const uint64_t p1 = (uint64_t)c2[b] * kPhiloxM1;
      const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1[b] ^ K.k0[r];
      const uint32_t n2b = (uint32_t)(p0 >> 32) ^ c3[b] ^ K.k1[r];
      c1[b] = (uint32_t)p1;
      c3[b] = (uint32_t)p0;
      c0[b] = n0;
      c2[b] = n2b;
    }
  }
#pragma unroll
  for (int b = 0; b < 8; ++b) out[b] = make_uint4(c0[b], c1[b], c2[b], c3[b]);
}

// Metropolis (RULE 0) acceptance of one word from its four precomputed blocks rb[0..3]
// (block q serves lanes 4q .. 4q + 3), same Horner order as update_word_metropolis.
template <int RULE>
__device__ __forceinline__ uint64_t metropolis_from_draws(uint64_t tgt, uint64_t n, uint64_t c,
                                                          uint64_t s, uint64_t side,
                                                          const uint4* rb, const HalfSweepParams& p) {
  const uint32_t sum_lo = (uint32_t)n + (uint32_t)c + (uint32_t)s + (uint32_t)side;
  const uint32_t sum_hi =
      (uint32_t)(n >> 32) + (uint32_t)(c >> 32) + (uint32_t)(s >> 32) + (uint32_t)(side >> 32);
  const uint32_t t3 = p.acc.thr[3], t4 = p.acc.thr[4];
  uint32_t a3lo = 0, a4lo = 0, a3hi = 0, a4hi = 0;
  const uint32_t dl[8] = {rb[1].w, rb[1].z, rb[1].y, rb[1].x, rb[0].w, rb[0].z, rb[0].y, rb[0].x};
  const uint32_t dh[8] = {rb[3].w, rb[3].z, rb[3].y, rb[3].x, rb[2].w, rb[2].z, rb[2].y, rb[2].x};
#pragma unroll
  for (int q = 0; q < 8; ++q) nc_step(a3lo, a4lo, dl[q], t3, t4);
#pragma unroll
  for (int q = 0; q < 8; ++q) nc_step(a3hi, a4hi, dh[q], t3, t4);
  uint32_t nclo = a3lo + a4lo, nchi = a3hi + a4hi;
  if constexpr (RULE == 2) {  // a class whose threshold is 2^32 never blocks a flip
    const uint32_t k3 = p.acc.keep3, k4 = p.acc.keep4;
    nclo = (a3lo & k3) + (a4lo & k4);
    nchi = (a3hi & k3) + (a4hi & k4);
  }
  const uint32_t lo = accept8((uint32_t)tgt, sum_lo, nclo);
  const uint32_t hi = accept8((uint32_t)(tgt >> 32), sum_hi, nchi);
  return ((uint64_t)hi << 32) | lo;
}

// Five-compare heat bath (RULE 3 / 5 / 6: NA leading "always" classes) from precomputed draws.
template <int NA>
__device__ __forceinline__ uint64_t hb_from_draws(uint64_t tgt, uint64_t n, uint64_t c, uint64_t s,
                                                  uint64_t side, const uint4* rb,
                                                  const HalfSweepParams& p) {
  const uint32_t sum_lo = (uint32_t)n + (uint32_t)c + (uint32_t)s + (uint32_t)side;
  const uint32_t sum_hi =
      (uint32_t)(n >> 32) + (uint32_t)(c >> 32) + (uint32_t)(s >> 32) + (uint32_t)(side >> 32);
  const uint32_t* T = p.acc.thr;
  uint32_t lo = 0, hi = 0;
  const uint32_t dl[8] = {rb[1].w, rb[1].z, rb[1].y, rb[1].x, rb[0].w, rb[0].z, rb[0].y, rb[0].x};
  const uint32_t dh[8] = {rb[3].w, rb[3].z, rb[3].y, rb[3].x, rb[2].w, rb[2].z, rb[2].y, rb[2].x};
#pragma unroll
  for (int q = 0; q < 8; ++q) hb_step<NA>(lo, dl[q], T);
#pragma unroll
  for (int q = 0; q < 8; ++q) hb_step<NA>(hi, dh[q], T);
  const uint32_t flo = hb_accept8((uint32_t)tgt, sum_lo, lo);
  const uint32_t fhi = hb_accept8((uint32_t)(tgt >> 32), sum_hi, hi);
  return ((uint64_t)fhi << 32) | flo;
}

// Symmetric heat bath (RULE 7) of one word from its four precomputed blocks.
__device__ __forceinline__ uint64_t hbs_from_draws(uint64_t tgt, uint64_t n, uint64_t c, uint64_t s,
                                                   uint64_t side, const uint4* rb,
                                                   const HalfSweepParams& p) {
  const uint32_t sum_lo = (uint32_t)n + (uint32_t)c + (uint32_t)s + (uint32_t)side;
  const uint32_t sum_hi =
      (uint32_t)(n >> 32) + (uint32_t)(c >> 32) + (uint32_t)(s >> 32) + (uint32_t)(side >> 32);
  const uint32_t t3 = p.acc.thr[3], t4 = p.acc.thr[4];
  uint32_t a3lo = 0, a4lo = 0, amlo = 0, a3hi = 0, a4hi = 0, amhi = 0;
  const uint32_t lo_draws[8] = {rb[1].w, rb[1].z, rb[1].y, rb[1].x, rb[0].w, rb[0].z, rb[0].y, rb[0].x};
  const uint32_t hi_draws[8] = {rb[3].w, rb[3].z, rb[3].y, rb[3].x, rb[2].w, rb[2].z, rb[2].y, rb[2].x};
#pragma unroll
  for (int q = 0; q < 8; ++q) hbs_step(a3lo, a4lo, amlo, lo_draws[q], t3, t4);
#pragma unroll
  for (int q = 0; q < 8; ++q) hbs_step(a3hi, a4hi, amhi, hi_draws[q], t3, t4);
  const uint32_t flo = hb_accept8((uint32_t)tgt, sum_lo, hbs_nc(a3lo + a4lo, amlo));
  const uint32_t fhi = hb_accept8((uint32_t)(tgt >> 32), sum_hi, hbs_nc(a3hi + a4hi, amhi));
  return ((uint64_t)fhi << 32) | flo;
}

// One word of RULE from its four precomputed Philox blocks (every rule that draws, except the
// unreachable generic heat bath RULE 1, which keeps update_word).
template <int RULE>
__device__ __forceinline__ uint64_t word_from_draws(uint64_t tgt, uint64_t n, uint64_t c, uint64_t s,
                                                    uint64_t side, const uint4* rb,
                                                    const HalfSweepParams& p) {
  if constexpr (RULE == 0 || RULE == 2) return metropolis_from_draws<RULE>(tgt, n, c, s, side, rb, p);
  else if constexpr (RULE == 7) return hbs_from_draws(tgt, n, c, s, side, rb, p);
  else return hb_from_draws<RULE == 3 ? 0 : RULE == 5 ? 1 : 2>(tgt, n, c, s, side, rb, p);
}
__host__ __device__ constexpr bool lockstep_rule(int rule) {
  return rule == 0 || rule == 2 || rule == 3 || rule == 5 || rule == 6 || rule == 7;
}

// Host-side rule dispatch shared by every launcher: f(integral_constant<int, RULE>,
// bool_constant<OBS>).  An unknown rule is an error, never a silent fallback.
template <typename F>
static cudaError_t dispatch_rule(int rule, bool obs, F&& f) {
#define ISING_RULE_CASE(R)                                                       \
  case R:                                                                        \
    return obs ? f(std::integral_constant<int, R>{}, std::true_type{})           \
               : f(std::integral_constant<int, R>{}, std::false_type{});
  switch (rule) {
    ISING_RULE_CASE(0)
    ISING_RULE_CASE(1)
    ISING_RULE_CASE(2)
    ISING_RULE_CASE(3)
    ISING_RULE_CASE(4)
    ISING_RULE_CASE(5)
    ISING_RULE_CASE(6)
    ISING_RULE_CASE(7)
  }
#undef ISING_RULE_CASE
  return cudaErrorInvalidValue;
}

// Observables of one target word t after its update (row a8, Eq. 1): up spins in t and in
// the centre source word c, and bonds from t's 16 sites to their four neighbours that are
// antiparallel.  Lanes use bit 0 of each nibble only, so the four neighbour XORs are packed
// into the four bits of each nibble — X = (t * 15) ^ (n | c << 1 | s << 2 | side << 3) — and
// one popcount counts all of them (likewise t | c << 1 for the up count): 2 popcounts per
// word instead of 6.
// Acc: 32-bit in the half-sweep kernels (per-thread counts stay far below 2^32 and 64-bit
// adds would put an IMAD.X on the FMA pipe per add), 64-bit in k_observables.
template <typename Acc>
__device__ __forceinline__ void obs_word(uint64_t t, uint64_t n, uint64_t c, uint64_t s,
                                         uint64_t side, Acc& up, Acc& anti) {
  const uint64_t t15 = (t << 4) - t;
  up += __popcll(t | (c << 1));
  anti += __popcll(t15 ^ (n | (c << 1) | (s << 2) | (side << 3)));
}

// Launch with programmatic stream serialisation (the kernel itself calls
// griddepcontrol.launch_dependents / griddepcontrol.wait before touching global memory).
template <typename K>
static cudaError_t launch_pdl(K kernel, unsigned grid, cudaStream_t st, const HalfSweepParams& p,
                              unsigned threads = 128) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, p);
}

// One colour phase of one slab.  Work item = (band of H rows, 128-bit chunk
// column q); the thread walks down the band keeping the N/C/S source chunks in
// registers, so each source word is read from memory once per band (plus one halo
// row per band).  Grid-stride over items; the grid is a multiple of the SM count.
#ifndef ISING_VPT
#define ISING_VPT 1  // 128-bit vectors (2 words, 32 spins) per thread and row
#endif
constexpr int kWords = 2 * ISING_VPT;
#ifndef ISING_MINB
#define ISING_MINB 4  // 116 registers, 4 blocks/SM: measured best of 1..8 (r01)
#endif
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Spin until every flag >= v.  A peer that never arrives (crashed rank) must not hang the
// GPU: after ~2^36 SM cycles (tens of seconds) the kernel traps, so the host call returns
// a CUDA error instead.
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// (%globaltimer, not clock64: a spinning block may be preempted and resumed on another SM,
// whose cycle counter is unrelated)
__device__ __noinline__ void spin_timeout(const unsigned long long* flags, int k,
                                          unsigned long long v) {
  printf("ising: peer flag wait timed out (block %d, flag %d = %llu, want %llu)\n",
         (int)blockIdx.x, k, ld_acquire_sys(flags + k), v);
  __trap();
}

__device__ __forceinline__ void spin_until(const unsigned long long* flags, int n,
                                           unsigned long long v) {
  unsigned long long t0 = 0;
  for (int k = 0; k < n; ++k)
    while (ld_acquire_sys(flags + k) < v) {
      __nanosleep(64);
      const unsigned long long now = global_ns();
      if (t0 == 0) t0 = now;
      if (now - t0 > 30000000000ull) spin_timeout(flags, k, v);
    }
}

// Loads of the source plane: L2-coherent ld.global.cg everywhere.  The persistent kernel
// reads in one phase what other SMs wrote in the previous phase of the same launch, and with
// programmatic dependent launch a half-sweep grid is resident (its launch-time L1
// invalidation behind it) while older grids may still run, so the non-coherent read-only path
// (ld.global.nc, "read-only for the lifetime of the kernel") is not used for plane data.
template <bool COHERENT>
__device__ __forceinline__ ulonglong2 ld_v2(const uint64_t* p) {
  return __ldcg(reinterpret_cast<const ulonglong2*>(p));
}
template <bool COHERENT>
__device__ __forceinline__ uint64_t ld_1(const uint64_t* p) {
  return __ldcg(reinterpret_cast<const unsigned long long*>(p));
}
template <bool COHERENT>
__device__ __forceinline__ ulonglong2 ld_tgt(const uint64_t* p) {  // streaming: no L1 reuse
  return __ldcg(reinterpret_cast<const ulonglong2*>(p));
}

// All work items of one colour phase (the half-sweep proper).  OBS: also reduce the
// observables of the state this (white) phase produces — every bond has exactly one white
// end, whose four black neighbours are the N, C, S and side words loaded here, and every
// black word is the C word of exactly one white word — so a measured chain needs no
// separate pass over the lattice (Eq. 1; row a8).
template <int RULE, bool OBS, bool COHERENT>
__device__ __forceinline__ void halfsweep_items(const HalfSweepParams& p, const uint32_t t,
                                                uint32_t& obs_up, uint32_t& obs_anti) {
  const int64_t W = p.W;
  const int64_t chunks = W / kWords;
  const uint64_t* src = p.src + W;  // local row r (r = -1 .. R) at src + r * W
  uint64_t* tgt = p.tgt + W;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t item = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; item < p.items;
       item += stride) {
    const int64_t q = item % chunks;
    const int band = (int)(item / chunks);
    const int ra = p.r_begin + band * p.H;
    const int rb = min(ra + p.H, p.r_end);
    const int64_t wc = kWords * q;
    const int64_t wwest = (wc == 0) ? W - 1 : wc - 1;     // periodic wrap
    const int64_t weast = (wc + kWords == W) ? 0 : wc + kWords;
    uint64_t nv[kWords], cv[kWords];
#pragma unroll
    for (int v = 0; v < kWords / 2; ++v) {
      const ulonglong2 a = ld_v2<COHERENT>(src + (int64_t)(ra - 1) * W + wc + 2 * v);
      const ulonglong2 b = ld_v2<COHERENT>(src + (int64_t)ra * W + wc + 2 * v);
      nv[2 * v] = a.x;
      nv[2 * v + 1] = a.y;
      cv[2 * v] = b.x;
      cv[2 * v + 1] = b.y;
    }
    // row pointers advanced by W per row (no per-row 64-bit index arithmetic)
    const uint64_t* sp = src + (int64_t)(ra + 1) * W + wc;  // source row r + 1
    const uint64_t* swp = src + (int64_t)ra * W;             // source row r (side words)
    uint64_t* tp = tgt + (int64_t)ra * W + wc;               // target row r
    for (int r = ra; r < rb; ++r, sp += W, swp += W, tp += W) {
      uint64_t sv[kWords], tv[kWords];
#pragma unroll
      for (int v = 0; v < kWords / 2; ++v) {
        const ulonglong2 a = ld_v2<COHERENT>(sp + 2 * v);
        const ulonglong2 b = ld_tgt<COHERENT>(tp + 2 * v);
        sv[2 * v] = a.x;
        sv[2 * v + 1] = a.y;
        tv[2 * v] = b.x;
        tv[2 * v + 1] = b.y;
      }
      const int64_t gi = p.row0 + r;
      // side word: the left word if (black and i even) or (white and i odd), else the
      // right one (Fig. 3 caption PAPER.md:208; reading R2)
      const bool west = ((gi & 1) == 0) == (p.colour == 0);
      const uint64_t sw = ld_1<COHERENT>(swp + (west ? wwest : weast));
      uint64_t side[kWords];
#pragma unroll
      for (int k = 0; k < kWords; ++k) {
        if (west)
          side[k] = splice_west(cv[k], k == 0 ? sw : cv[k - 1]);
        else
          side[k] = splice_east(cv[k], k == kWords - 1 ? sw : cv[k + 1]);
      }
#if ISING_PHILOX8
      if constexpr (kWords == 2 && lockstep_rule(RULE)) {  // lockstep Philox, as staged
        uint4 rb[8];
        philox8(t, (uint32_t)(4 * wc), p.colour, (uint32_t)gi, p.keys, rb);
#pragma unroll
        for (int k = 0; k < 2; ++k)
          tv[k] = word_from_draws<RULE>(tv[k], nv[k], cv[k], sv[k], side[k], rb + 4 * k, p);
      } else
#endif
      {
#pragma unroll
        for (int k = 0; k < kWords; ++k) {
          const uint32_t ctr0 = (uint32_t)(4 * (wc + k));  // Philox counter word 1 = j / 4 (R6)
          tv[k] = update_word<RULE>(tv[k], nv[k], cv[k], sv[k], side[k], ctr0, (uint32_t)gi, t, p);
        }
      }
      if (OBS) {
#pragma unroll
        for (int k = 0; k < kWords; ++k) obs_word(tv[k], nv[k], cv[k], sv[k], side[k], obs_up, obs_anti);
      }
#pragma unroll
      for (int v = 0; v < kWords / 2; ++v) {
        const ulonglong2 o = make_ulonglong2(tv[2 * v], tv[2 * v + 1]);
        *reinterpret_cast<ulonglong2*>(tp + 2 * v) = o;
        if (r == 0 && p.halo_up) *reinterpret_cast<ulonglong2*>(p.halo_up + wc + 2 * v) = o;
        if (r == p.R - 1 && p.halo_dn) *reinterpret_cast<ulonglong2*>(p.halo_dn + wc + 2 * v) = o;
      }
#pragma unroll
      for (int k = 0; k < kWords; ++k) {
        nv[k] = cv[k];
        cv[k] = sv[k];
      }
    }
  }
}

template <int RULE, bool OBS = false>
__global__ void __launch_bounds__(128, ISING_MINB) k_halfsweep(const HalfSweepParams p) {
  if (p.pdl) {  // programmatic dependent launch, as in k_halfsweep_staged
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  if (p.obs_clear && blockIdx.x == 0 && threadIdx.x == 0) {  // after the grid dependency
    p.obs_clear[0] = 0;
    p.obs_clear[1] = 0;
  }
  if (p.wait_flags) {  // rank-p2p: neighbours done with the previous phase
    if (threadIdx.x == 0) spin_until(p.wait_flags, 2, p.wait_value);
    __syncthreads();
  }
  // sweep index: absolute, or (CUDA graph replays) a device-resident base + the offset
  const uint32_t t = p.t_dev ? *p.t_dev + p.t : p.t;
  uint32_t obs_up = 0, obs_anti = 0;
  halfsweep_items<RULE, OBS, false>(p, t, obs_up, obs_anti);
  if (OBS) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      obs_up += __shfl_xor_sync(0xffffffffu, obs_up, off);
      obs_anti += __shfl_xor_sync(0xffffffffu, obs_anti, off);
    }
    if ((threadIdx.x & 31) == 0 && (obs_up | obs_anti)) {
      unsigned long long* o = p.obs_out + (p.slot_dev ? 2 * (size_t)*p.slot_dev : 0);
      atomicAdd(&o[0], obs_up);
      atomicAdd(&o[1], obs_anti);
    }
  }
  if (p.signal_up) {  // rank-p2p: the last block publishes "phase done" to both neighbours
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned int prev = atomicAdd(p.done_counter, 1u);
      if (prev == gridDim.x - 1) {
        *p.done_counter = 0;  // re-armed for the next launch (stream-ordered)
        __threadfence_system();
        st_release_sys(p.signal_up, p.signal_value);
        st_release_sys(p.signal_dn, p.signal_value);
      }
    }
  }
}

__global__ void k_sync(const SyncParams p) {
  if (p.wait_flags) spin_until(p.wait_flags, p.wait_count, p.wait_value);
  __threadfence_system();
  for (int k = 0; k < 2; ++k)
    if (p.signal[k]) st_release_sys(p.signal[k], p.signal_value);
}

// Observable all-reduce over peer memory.  The slots are double-buffered by epoch parity: a
// rank can start gather e + 1 (writing the other parity) while a slower rank still reads
// epoch e, but it cannot finish e + 1 — and so cannot start e + 2, which reuses e's slots —
// before every rank has published e + 1, i.e. has finished reading e.
__global__ void k_gather(const GatherParams p) {
  const unsigned long long up = p.local[0], anti = p.local[1];
  const int base = 3 * kMaxRanks * (int)(p.epoch & 1);
  for (int r = 0; r < p.world; ++r) {
    unsigned long long* s = p.slots[r] + base + 3 * p.rank;
    s[0] = up;
    s[1] = anti;
  }
  __threadfence_system();
  for (int r = 0; r < p.world; ++r) st_release_sys(p.slots[r] + base + 3 * p.rank + 2, p.epoch);
  unsigned long long su = 0, sa = 0;
  for (int r = 0; r < p.world; ++r) {
    const unsigned long long* m = p.mine + base + 3 * r;
    spin_until(m + 2, 1, p.epoch);
    su += __ldcg(m);
    sa += __ldcg(m + 1);
  }
  p.out[0] = su;
  p.out[1] = sa;
}

__global__ void k_set_u32(uint32_t* dst, uint32_t v, int add) { *dst = add ? *dst + v : v; }

__global__ void k_zero_u64(unsigned long long* dst, int n) {
  for (int k = threadIdx.x; k < n; k += blockDim.x) dst[k] = 0;
}

// Small zero fills as a kernel rather than cudaMemsetAsync: in one process driving several
// rank-p2p handles on one device (ising_p2p_connect_local), a memset queued behind another
// rank's phase that spins on this rank's flags was observed never to run (a deadlock the
// flag timeout turned into a trap); kernels on independent streams do not have that problem.
cudaError_t launch_zero_u64(cudaStream_t st, unsigned long long* dst, int n) {
  k_zero_u64<<<1, 32, 0, st>>>(dst, n);
  return cudaGetLastError();
}

__global__ void k_copy_u64(uint64_t* __restrict__ dst, const uint64_t* __restrict__ src, int64_t n) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    dst[k] = src[k];
}

// Row copies into a neighbour's halo (possibly peer memory) as a kernel, for the same reason.
cudaError_t launch_copy_u64(cudaStream_t st, uint64_t* dst, const uint64_t* src, int64_t n) {
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 1024);
  k_copy_u64<<<grid, 256, 0, st>>>(dst, src, n);
  return cudaGetLastError();
}

cudaError_t launch_set_u32(cudaStream_t st, uint32_t* dst, uint32_t v, int add) {
  k_set_u32<<<1, 1, 0, st>>>(dst, v, add);
  return cudaGetLastError();
}

cudaError_t launch_sync(cudaStream_t st, const SyncParams& p) {
  k_sync<<<1, 1, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_gather(cudaStream_t st, const GatherParams& p) {
  k_gather<<<1, 1, 0, st>>>(p);
  return cudaGetLastError();
}

// ------------------------------------------------------- TMA-staged variant
// The north_star's "shared-memory or TMA staging of the neighbour-colour rows": a block
// owns 128 chunks (256 words) of a band of up to kStageRows rows; one elected thread
// issues one cp.async.bulk (TMA bulk copy, completes on an mbarrier) per source row of
// the band plus its two halo rows, the two words beyond the block's span come from plain
// loads, and the threads read N / C / S / side words from shared memory.  Measured
// against the register-rolling kernel in profiles/r01_ncu_halfsweep.md (371.6 vs 394.6 us
// per C3 half-sweep: the shared-memory reads replace the per-row global loads and their
// address arithmetic); used whenever W is a multiple of 256 words (ISING_STAGED=0 opts out).
#ifndef ISING_STAGE_ROWS
#define ISING_STAGE_ROWS 20  // 44 KB of source rows per block, 4 blocks per SM
#endif
// __launch_bounds__ minimum blocks per SM of the staged kernel.  All of 2, 3, 4 give 118
// registers (4 resident blocks), but ptxas schedules the Philox / carry-chain stream
// differently: 3 measured 1524-1531 flips/ns on C3 against 1498 for 4 (profiles/
// r01_ncu_halfsweep.md); the draw-free variant (RULE 4, memory-bound) keeps 4.
#ifndef ISING_ROW_UNROLL
#define ISING_ROW_UNROLL 1
#endif
constexpr int kRowUnroll = ISING_ROW_UNROLL;  // staged row loop unroll factor
#ifndef ISING_STAGED_MINB
#define ISING_STAGED_MINB 3
#endif
#ifndef ISING_STAGED_MINB_DRAWFREE
#define ISING_STAGED_MINB_DRAWFREE 4
#endif
__host__ __device__ constexpr int staged_minb(int rule) {
  return rule == 4 ? ISING_STAGED_MINB_DRAWFREE : ISING_STAGED_MINB;
}
#ifndef ISING_STAGE_ROWS_DRAWFREE
#define ISING_STAGE_ROWS_DRAWFREE 16  // memory-bound variant: 3341 vs 3027 flips/ns at 20 rows
#endif
__host__ __device__ constexpr int stage_rows(int rule) {
  return rule == 4 ? ISING_STAGE_ROWS_DRAWFREE : ISING_STAGE_ROWS;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int RULE, bool OBS = false>
__global__ void __launch_bounds__(kStageThreads, staged_minb(RULE)) k_halfsweep_staged(const HalfSweepParams p) {
  constexpr int kRows = stage_rows(RULE);
  // Programmatic dependent launch (p.pdl: launched with programmatic stream serialisation):
  // let the next kernel in the stream be scheduled as soon as every block of this one is
  // resident, and wait here until the previous kernel has completed and its writes are
  // visible — nothing before this line touches global memory.
  if (p.pdl) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  if (p.obs_clear && blockIdx.x == 0 && threadIdx.x == 0) {  // after the grid dependency
    p.obs_clear[0] = 0;
    p.obs_clear[1] = 0;
  }
  __shared__ alignas(128) uint64_t tile[kRows + 2][kStageWords];
  __shared__ uint64_t edge[kRows + 2][2];
  __shared__ alignas(8) uint64_t mbar;
  const int64_t W = p.W;
  const int64_t bpr = W / kStageWords;  // blocks per band
  const int pband = (int)(blockIdx.x / bpr);
  const int64_t w0 = (int64_t)(blockIdx.x - (int64_t)pband * bpr) * kStageWords;
  // rank-p2p: the two edge bands (the only ones that wait for / signal the neighbours) take
  // the first two slots of the grid, so their system fences and the phase signal happen while
  // the interior bands still run instead of at the end of the kernel
  const int64_t bands = gridDim.x / bpr;
  const int band = (p.wait_flags && bands > 1)
                       ? (pband == 0 ? 0 : (pband == 1 ? (int)(bands - 1) : pband - 1))
                       : pband;
  // bands of kRows rows; with a guided tail (tail_band8 > 0) the last bands are 8 and
  // then 4 rows tall, so the partial last wave idles for a short block lifetime only
  int ra, rb;
  if (band < p.tail_band8 || p.tail_band8 == 0) {
    ra = p.r_begin + band * kRows;
    rb = min(ra + kRows, p.r_end);
  } else if (band < p.tail_band4) {
    ra = p.r_begin + p.tail_band8 * kRows + (band - p.tail_band8) * p.tail_h1;
    rb = min(ra + p.tail_h1, p.r_begin + p.tail_row4);
  } else {
    ra = p.r_begin + p.tail_row4 + (band - p.tail_band4) * p.tail_h2;
    rb = min(ra + p.tail_h2, p.r_end);
  }
  if (p.mirror) {  // same band heights, rows mirrored within [r_begin, r_end)
    const int a = ra;
    ra = p.r_begin + p.r_end - rb;
    rb = p.r_begin + p.r_end - a;
  }
  const int nrows = rb - ra;
  // rank-p2p: only the bands at the slab edges depend on the neighbours — they read the halo
  // rows the neighbours stored in the previous phase and store rows 0 / R - 1 into halo rows
  // the neighbours read in it — so only their blocks wait for both neighbours to finish that
  // phase; interior blocks touch this slab's own rows only (ordered by the stream)
  // the first and the last band of the slab (the only bands of a rank-p2p launch that read
  // halo rows or store into the neighbours' halo rows: it always updates rows 0 .. R - 1)
  const bool edge_band = band == 0 || band == bands - 1;
  if (p.wait_flags && edge_band) {
    if (threadIdx.x == 0) {
      spin_until(p.wait_flags, 2, p.wait_value);
      // The neighbours stored the halo rows with generic-proxy stores, made visible to this
      // thread by its acquire; the bulk copies below read them through the async proxy, so
      // order the two proxies before issuing them.
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    __syncthreads();
  }
  const uint64_t* src = p.src + W;  // local row r at src + r * W
  uint64_t* tgt = p.tgt + W;
  const uint32_t bar = smem_u32(&mbar);
  // One block barrier for the start-up: thread 0 initialises the mbarrier (the init fence
  // orders it before the TMA's complete_tx) and issues the copies; warps 1-2 load the edge
  // words meanwhile; the barrier below then orders the init before every thread's wait.
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint32_t bytes = (uint32_t)(nrows + 2) * kStageWords * 8;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
    for (int rr = 0; rr < nrows + 2; ++rr) {
      const uint64_t* g = src + (int64_t)(ra - 1 + rr) * W + w0;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
          ::"r"(smem_u32(&tile[rr][0])), "l"(g), "r"((uint32_t)(kStageWords * 8)), "r"(bar)
          : "memory");
    }
  }
  // the word left of the span (west side of the first thread) and right of it (east side
  // of the last thread) for the band's rows, with the periodic wrap
  if (threadIdx.x >= 32 && threadIdx.x < 32 + 2 * nrows) {
    const int e = threadIdx.x - 32;
    const int rr = e >> 1;
    const int64_t col = (e & 1) ? ((w0 + kStageWords == W) ? 0 : w0 + kStageWords)
                                : ((w0 == 0) ? W - 1 : w0 - 1);
    edge[rr + 1][e & 1] = __ldcg(reinterpret_cast<const unsigned long long*>(src + (int64_t)(ra + rr) * W + col));
  }
  __syncthreads();
  {
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{\n\t.reg .pred q;\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 q, [%1], 0;\n\t"
          "selp.u32 %0, 1, 0, q;\n\t}"
          : "=r"(done)
          : "r"(bar)
          : "memory");
  }
  const uint32_t t = p.t_dev ? *p.t_dev + p.t : p.t;
  const int tid = threadIdx.x;
  const int64_t wc = w0 + 2 * tid;
  uint32_t obs_up = 0, obs_anti = 0;
  uint64_t* tp = tgt + (int64_t)ra * W + wc;  // target chunk of row r, advanced by W per row
#pragma unroll kRowUnroll
  for (int rr = 0; rr < nrows; ++rr, tp += W) {
    const int r = ra + rr;
    const int64_t gi = p.row0 + r;
    const bool west = ((gi & 1) == 0) == (p.colour == 0);
    const uint64_t n0 = tile[rr][2 * tid], n1 = tile[rr][2 * tid + 1];
    const uint64_t c0 = tile[rr + 1][2 * tid], c1 = tile[rr + 1][2 * tid + 1];
    const uint64_t s0 = tile[rr + 2][2 * tid], s1 = tile[rr + 2][2 * tid + 1];
    uint64_t side0, side1;
    if (west) {
      const uint64_t wl = tid == 0 ? edge[rr + 1][0] : tile[rr + 1][2 * tid - 1];
      side0 = splice_west(c0, wl);
      side1 = splice_west(c1, c0);
    } else {
      const uint64_t er = tid == kStageThreads - 1 ? edge[rr + 1][1] : tile[rr + 1][2 * tid + 2];
      side0 = splice_east(c0, c1);
      side1 = splice_east(c1, er);
    }
    ulonglong2 tv = __ldcg(reinterpret_cast<const ulonglong2*>(tp));  // L2: see ld_v2
    const uint32_t ctr0 = (uint32_t)(4 * wc);
#if ISING_PHILOX8
    if constexpr (lockstep_rule(RULE)) {
      uint4 rb[8];
      philox8(t, ctr0, p.colour, (uint32_t)gi, p.keys, rb);
      tv.x = word_from_draws<RULE>(tv.x, n0, c0, s0, side0, rb, p);
      tv.y = word_from_draws<RULE>(tv.y, n1, c1, s1, side1, rb + 4, p);
    } else
#endif
    {
      tv.x = update_word<RULE>(tv.x, n0, c0, s0, side0, ctr0, (uint32_t)gi, t, p);
      tv.y = update_word<RULE>(tv.y, n1, c1, s1, side1, ctr0 + 4, (uint32_t)gi, t, p);
    }
    *reinterpret_cast<ulonglong2*>(tp) = tv;
    if (r == 0 && p.halo_up) *reinterpret_cast<ulonglong2*>(p.halo_up + wc) = tv;
    if (r == p.R - 1 && p.halo_dn) *reinterpret_cast<ulonglong2*>(p.halo_dn + wc) = tv;
    if (OBS) {  // same fused observables as k_halfsweep (white phase of a measured sweep)
      obs_word(tv.x, n0, c0, s0, side0, obs_up, obs_anti);
      obs_word(tv.y, n1, c1, s1, side1, obs_up, obs_anti);
    }
  }
  if (OBS) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      obs_up += __shfl_xor_sync(0xffffffffu, obs_up, off);
      obs_anti += __shfl_xor_sync(0xffffffffu, obs_anti, off);
    }
    if ((threadIdx.x & 31) == 0 && (obs_up | obs_anti)) {
      unsigned long long* o = p.obs_out + (p.slot_dev ? 2 * (size_t)*p.slot_dev : 0);
      atomicAdd(&o[0], obs_up);
      atomicAdd(&o[1], obs_anti);
    }
  }
  // rank-p2p: the last edge-band block publishes "phase done" to both neighbours.  Only the
  // edge bands touch memory the neighbours use (they read this slab's halo rows, which the
  // neighbours overwrite next phase, and store rows 0 / R - 1 into the neighbours' halo
  // rows, which they read next phase), so interior blocks neither fence nor count.
  if (p.signal_up && edge_band) {
    const unsigned int n_edge = (unsigned int)(bpr * (bands == 1 ? 1 : 2));
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned int prev = atomicAdd(p.done_counter, 1u);
      if (prev == n_edge - 1) {
        *p.done_counter = 0;  // re-armed for the next launch (stream-ordered)
        __threadfence_system();
        st_release_sys(p.signal_up, p.signal_value);
        st_release_sys(p.signal_dn, p.signal_value);
      }
    }
  }
}

// slots = resident blocks (SMs x blocks per SM), 0: no guided tail.  The tail is one wave of
// 8-row bands then one of 4-row bands, used when the 16-row grid is 3 to 64 waves long (a
// partial last wave costs about half a block lifetime per slot: 3.6 % on C3).
cudaError_t launch_halfsweep_staged(int rule, int64_t slots, cudaStream_t st, HalfSweepParams p) {
  const int64_t rows = p.r_end - p.r_begin;
  const int kStageRows = stage_rows(rule);  // band height of this rule's kernel
  const int64_t spans = p.W / kStageWords;
  int64_t bands = (rows + kStageRows - 1) / kStageRows;
  p.tail_band8 = p.tail_band4 = p.tail_row4 = 0;
  const int64_t per_wave = slots / spans;  // bands per wave
  // measured on C3 (profiles/r01_ncu_halfsweep.md): heights 8/4, 8/2, 4/2, 12/6 and one or
  // two waves each all land within 0.3 % of each other
#ifndef ISING_TAIL_H1
#define ISING_TAIL_H1 8
#endif
#ifndef ISING_TAIL_H2
#define ISING_TAIL_H2 4
#endif
  constexpr int h1 = ISING_TAIL_H1, h2 = ISING_TAIL_H2, w1 = 1, w2 = 1;
  if (per_wave > 0 && bands * spans >= 3 * slots && bands * spans < 64 * slots) {
    const int64_t row4 = rows - (int64_t)h2 * w2 * per_wave;
    const int64_t row8 = ((row4 - (int64_t)h1 * w1 * per_wave) / kStageRows) * kStageRows;
    const int64_t n8 = (row4 - row8 + h1 - 1) / h1;
    p.tail_band8 = (int32_t)(row8 / kStageRows);
    p.tail_band4 = (int32_t)(p.tail_band8 + n8);
    p.tail_row4 = (int32_t)row4;
    p.tail_h1 = h1;
    p.tail_h2 = h2;
    bands = p.tail_band4 + (rows - row4 + h2 - 1) / h2;
  }
  const unsigned grid = (unsigned)(spans * bands);
  return dispatch_rule(rule, p.obs_out != nullptr, [&](auto R, auto O) {
    if (!p.pdl) {
      k_halfsweep_staged<decltype(R)::value, decltype(O)::value><<<grid, kStageThreads, 0, st>>>(p);
      return cudaGetLastError();
    }
    return launch_pdl(k_halfsweep_staged<decltype(R)::value, decltype(O)::value>, grid, st, p,
                      kStageThreads);
  });
}

cudaError_t staged_occupancy(int* blocks_per_sm) {
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_halfsweep_staged<0>,
                                                       kStageThreads, 0);
}

// ------------------------------------------------------- persistent sweeps
// Small lattices are launch-bound (a 2048^2 half-sweep is ~1.5 us of work).  One
// cooperative launch runs n whole sweeps: every block of the (co-resident) grid walks its
// items of the black phase, meets the others at a grid barrier, walks the white phase, and
// meets them again.  Loads are L2-coherent (a plane written in one phase is read by other
// SMs in the next).  With obs_base, the white phase of every `every`-th sweep also reduces
// the observables of the state it produces into slot (s / every - 1).
__device__ __forceinline__ unsigned int ld_acquire_gpu(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void grid_barrier(unsigned int* count, unsigned int* gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int g = ld_acquire_gpu(gen);
    __threadfence();
    if (atomicAdd(count, 1u) == gridDim.x - 1) {
      atomicExch(count, 0u);
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      while (ld_acquire_gpu(gen) == g) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

constexpr int kPersistThreads = 512;  // one CTA per SM: fewer barrier arrivals
template <int RULE, bool OBS>
__global__ void __launch_bounds__(kPersistThreads, 1) k_sweeps_persistent(const PersistentParams P) {
  for (uint32_t s = 1; s <= P.n; ++s) {
    const uint32_t t = P.t0 + s;
    uint32_t up = 0, anti = 0;
    halfsweep_items<RULE, false, true>(P.ph[0], t, up, anti);
    grid_barrier(P.bar_count, P.bar_gen);
    if (OBS && s % P.every == 0) {
      halfsweep_items<RULE, true, true>(P.ph[1], t, up, anti);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        up += __shfl_xor_sync(0xffffffffu, up, off);
        anti += __shfl_xor_sync(0xffffffffu, anti, off);
      }
      if ((threadIdx.x & 31) == 0 && (up | anti)) {
        unsigned long long* slot = P.obs_base + 2 * (size_t)(s / P.every - 1);
        atomicAdd(&slot[0], up);
        atomicAdd(&slot[1], anti);
      }
    } else {
      halfsweep_items<RULE, false, true>(P.ph[1], t, up, anti);
    }
    grid_barrier(P.bar_count, P.bar_gen);
  }
}

template <int RULE, bool OBS>
static cudaError_t coop_launch(int grid, cudaStream_t st, const PersistentParams& P) {
  void* args[] = {const_cast<PersistentParams*>(&P)};
  return cudaLaunchCooperativeKernel((const void*)k_sweeps_persistent<RULE, OBS>, dim3(grid),
                                     dim3(kPersistThreads), args, 0, st);
}

cudaError_t launch_persistent(int rule, int grid, cudaStream_t st, const PersistentParams& P) {
  return dispatch_rule(rule, P.obs_base != nullptr, [&](auto R, auto O) {
    return coop_launch<decltype(R)::value, decltype(O)::value>(grid, st, P);
  });
}

cudaError_t persistent_occupancy(int* blocks_per_sm) {
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_sweeps_persistent<0, true>,
                                                       kPersistThreads, 0);
}

// Philox-only throughput probe (ALU roofline denominator):
// the same philox4x32_10 as the half-sweep, counter {x, row, t, colour} with the
// same warp-uniform words, outputs XOR-folded so nothing but the fold is stored.
__global__ void __launch_bounds__(128) k_philox_probe(PhiloxKeys K, uint32_t blocks_per_thread,
                                                      uint32_t t, unsigned int* sink) {
  uint32_t acc = 0;
  const uint32_t row = blockIdx.x;
#if ISING_PROBE8 == 2
  // a thread owns one 128-bit column chunk (counter word 1 = c1base + 0..7) and walks
  // blocks_per_thread / 8 rows down it
  const uint32_t c1base = 8 * (blockIdx.x * blockDim.x + threadIdx.x);
  for (uint32_t b = 0; b < blocks_per_thread; b += 8) {
    uint4 r[8];
    philox8(t, c1base, 1u, row + b / 8, K, r);
#pragma unroll
    for (int q = 0; q < 8; ++q) acc ^= r[q].x ^ r[q].y ^ r[q].z ^ r[q].w;
  }
#elif ISING_PROBE8
  for (uint32_t b = 0; b < blocks_per_thread; b += 8) {  // eight blocks in lockstep
    uint4 r[8];
    philox8(t, 8 * (b * blockDim.x / 8 + threadIdx.x), 1u, row, K, r);
#pragma unroll
    for (int q = 0; q < 8; ++q) acc ^= r[q].x ^ r[q].y ^ r[q].z ^ r[q].w;
  }
#else
  for (uint32_t b = 0; b < blocks_per_thread; ++b) {
    const uint4 r = philox4x32_10(t, b * blockDim.x + threadIdx.x, 1u, row, K);
    acc ^= r.x ^ r.y ^ r.z ^ r.w;
  }
#endif
  if (acc == 0x9E3779B9u) atomicAdd(sink, 1u);  // practically never; keeps the work live
}

cudaError_t launch_philox_probe(int grid, cudaStream_t st, const PhiloxKeys& K,
                                uint32_t blocks_per_thread, unsigned int* sink) {
  k_philox_probe<<<grid, 128, 0, st>>>(K, blocks_per_thread, 1u, sink);
  return cudaGetLastError();
}

cudaError_t launch_halfsweep(int rule, int grid, cudaStream_t st, const HalfSweepParams& p) {
  return dispatch_rule(rule, p.obs_out != nullptr, [&](auto R, auto O) {
    if (!p.pdl) {
      k_halfsweep<decltype(R)::value, decltype(O)::value><<<grid, 128, 0, st>>>(p);
      return cudaGetLastError();
    }
    return launch_pdl(k_halfsweep<decltype(R)::value, decltype(O)::value>, grid, st, p);
  });
}

cudaError_t halfsweep_occupancy(int* blocks_per_sm) {
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_halfsweep<0>, 128, 0);
}

// ------------------------------------------------------------------- init
// Random start: spin +1 iff r(seed, 0, c, i, j) < 2^31 (reading R8); cold: all +1.
// Covers padded rows -1..R (global rows wrap mod N), so no exchange is needed.
__global__ void k_init(const InitParams p) {
  const int64_t total = 2 * (int64_t)(p.R + 2) * p.W;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += stride) {
    const int c = (int)(idx / ((int64_t)(p.R + 2) * p.W));
    const int64_t rem = idx - (int64_t)c * (p.R + 2) * p.W;
    const int64_t pr = rem / p.W;  // padded row 0 .. R+1
    const int64_t w = rem - pr * p.W;
    uint64_t word;
    if (p.cold) {
      word = 0x1111111111111111ull;
    } else {
      int64_t gi = (p.row0 + pr - 1) % p.N;
      if (gi < 0) gi += p.N;
      word = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const uint4 r = philox4x32_10(0u, (uint32_t)(4 * w + b), (uint32_t)c, (uint32_t)gi, p.keys);
        const uint32_t rr[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (rr[q] < 0x80000000u) word |= 1ull << (4 * (4 * b + q));
      }
    }
    p.plane[c][pr * p.W + w] = word;
  }
}

// ------------------------------------------------------------- observables
// Every bond has exactly one black end, and a black word's 4 neighbour words are the
// white N, C, S and side words of the black stencil, so
//   antiparallel bonds U = sum_black popc(b^N) + popc(b^C) + popc(b^S) + popc(b^side),
//   E = -(2NM - U) + U = 2U - 2NM (Eq. 1; reading R11).
__global__ void __launch_bounds__(256) k_observables(const ObsParams p) {
  const int64_t total = (int64_t)p.R * p.W;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint64_t* wh = p.white + p.W;
  const uint64_t* bl = p.black + p.W;
  unsigned long long up = 0, anti = 0;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += stride) {
    const int64_t r = idx / p.W;
    const int64_t w = idx - r * p.W;
    const uint64_t b = bl[r * p.W + w];
    const uint64_t cw = wh[r * p.W + w];
    const uint64_t nw = wh[(r - 1) * p.W + w];
    const uint64_t sw = wh[(r + 1) * p.W + w];
    const bool west = ((p.row0 + r) & 1) == 0;  // black target: west iff row even
    uint64_t side;
    if (west) {
      const uint64_t ww = wh[r * p.W + (w == 0 ? p.W - 1 : w - 1)];
      side = (cw << 4) | (ww >> 60);
    } else {
      const uint64_t ew = wh[r * p.W + (w + 1 == p.W ? 0 : w + 1)];
      side = (cw >> 4) | (ew << 60);
    }
    obs_word(b, nw, cw, sw, side, up, anti);
  }
  // warp reduction by shuffles, then one atomic per warp
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    up += __shfl_xor_sync(0xffffffffu, up, off);
    anti += __shfl_xor_sync(0xffffffffu, anti, off);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&p.out[0], up);
    atomicAdd(&p.out[1], anti);
  }
}

// ------------------------------------------------------------ pack / unpack
// Full lattice (row-major +-1 bytes) <-> planes.  Site (i, J) has colour c = (i + J) & 1 and
// plane column J / 2 (reading R1), so full columns J0 .. J0 + 15 (J0 = 16 u) of row i are
// plane columns 8u .. 8u + 7 — the 32-bit half-word u of each plane row — with byte 2j' + x
// from colour (i + x) & 1.  One thread per 16 bytes: 128-bit full-row accesses and 32-bit
// plane accesses, both coalesced across the warp.
__device__ __forceinline__ void bytes_to_lanes(const uint4 v, uint32_t& even, uint32_t& odd,
                                               unsigned int& bad) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  even = odd = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const uint32_t byte = (w[q] >> (8 * b)) & 0xFFu;  // full column J0 + 4q + b
      bad |= (byte != 0x01u && byte != 0xFFu);
      const int jj = 2 * q + (b >> 1);                  // plane column 8u + jj
      const uint32_t up = byte == 0x01u ? 1u : 0u;
      if (b & 1) odd |= up << (4 * jj);
      else even |= up << (4 * jj);
    }
}

__device__ __forceinline__ uint4 lanes_to_bytes(uint32_t even, uint32_t odd) {
  uint32_t w[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    // bytes: (2q, even), (2q, odd), (2q + 1, even), (2q + 1, odd); 0/1 bits at 0, 8, 16, 24
    const uint32_t f = ((even >> (8 * q)) & 1u) | (((odd >> (8 * q)) & 1u) << 8) |
                       (((even >> (8 * q + 4)) & 1u) << 16) | (((odd >> (8 * q + 4)) & 1u) << 24);
    w[q] = ~((f << 8) - (f << 1));  // per byte: f ? 0x01 : 0xFF (0xFE f = (f << 8) - 2 f)
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

__global__ void k_pack(const PackParams p) {
  const int64_t rows = p.rb - p.ra;
  const int64_t halves = 2 * p.W;  // 32-bit half-words per plane row
  const int64_t total = rows * halves;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  uint32_t* pl0 = reinterpret_cast<uint32_t*>(p.plane[0]);
  uint32_t* pl1 = reinterpret_cast<uint32_t*>(p.plane[1]);
  unsigned int bad = 0;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += stride) {
    const int64_t lr = idx / halves;  // row within staging
    const int64_t u = idx - lr * halves;
    const int64_t r = p.ra + lr;      // padded local row (-1 .. R)
    int64_t gi = (p.row0 + r) % p.N;
    if (gi < 0) gi += p.N;
    uint32_t even, odd;
    bytes_to_lanes(*reinterpret_cast<const uint4*>(p.full + lr * p.M + 16 * u), even, odd, bad);
    const int64_t o = (r + 1) * halves + u;
    // even full columns have colour i & 1, odd ones the other
    if (gi & 1) {
      pl1[o] = even;
      pl0[o] = odd;
    } else {
      pl0[o] = even;
      pl1[o] = odd;
    }
  }
  if (bad) atomicOr(p.bad, 1u);
}

__global__ void k_unpack(const UnpackParams p) {
  const int64_t rows = p.rb - p.ra;
  const int64_t halves = 2 * p.W;
  const int64_t total = rows * halves;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint32_t* pl0 = reinterpret_cast<const uint32_t*>(p.plane[0]);
  const uint32_t* pl1 = reinterpret_cast<const uint32_t*>(p.plane[1]);
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += stride) {
    const int64_t lr = idx / halves;
    const int64_t u = idx - lr * halves;
    const int64_t r = p.ra + lr;
    const int64_t o = (r + 1) * halves + u;
    const uint32_t a = pl0[o], b = pl1[o];
    const bool odd_row = ((p.row0 + r) & 1) != 0;
    *reinterpret_cast<uint4*>(p.full + lr * p.M + 16 * u) =
        odd_row ? lanes_to_bytes(b, a) : lanes_to_bytes(a, b);
  }
}

// ------------------------------------------------------ bit-packed host format
// 32 full columns J0 .. J0 + 31 (J0 = 32 w) of row i are plane columns 16 w .. 16 w + 15 of
// both colours — exactly word w of each plane row; even columns have colour i & 1 (R1).
// part1by1 moves bit p to bit 2p, compact1by1 is its inverse: the even-column bits (at 2k)
// land on nibble lane k (bit 4k) and back.
__device__ __forceinline__ uint64_t part1by1(uint64_t x) {
  x &= 0x00000000FFFFFFFFull;
  x = (x | (x << 16)) & 0x0000FFFF0000FFFFull;
  x = (x | (x << 8)) & 0x00FF00FF00FF00FFull;
  x = (x | (x << 4)) & 0x0F0F0F0F0F0F0F0Full;
  x = (x | (x << 2)) & 0x3333333333333333ull;
  x = (x | (x << 1)) & 0x5555555555555555ull;
  return x;
}
__device__ __forceinline__ uint64_t compact1by1(uint64_t x) {
  x &= 0x5555555555555555ull;
  x = (x | (x >> 1)) & 0x3333333333333333ull;
  x = (x | (x >> 2)) & 0x0F0F0F0F0F0F0F0Full;
  x = (x | (x >> 4)) & 0x00FF00FF00FF00FFull;
  x = (x | (x >> 8)) & 0x0000FFFF0000FFFFull;
  x = (x | (x >> 16)) & 0x00000000FFFFFFFFull;
  return x;
}

__global__ void k_pack_bits(const PackBitsParams p) {
  const int64_t total = (int64_t)(p.rb - p.ra) * p.W;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lr = idx / p.W, w = idx - lr * p.W;
    const int64_t r = p.ra + lr;  // padded local row (-1 .. R)
    int64_t gi = (p.row0 + r) % p.N;
    if (gi < 0) gi += p.N;
    const uint64_t x = p.bits[idx];
    const uint64_t even = part1by1(x & 0x55555555u), odd = part1by1((x >> 1) & 0x55555555u);
    const int ce = (int)(gi & 1);  // colour of the even columns
    p.plane[ce][(r + 1) * p.W + w] = even;
    p.plane[1 - ce][(r + 1) * p.W + w] = odd;
  }
}

__global__ void k_unpack_bits(const UnpackBitsParams p) {
  const int64_t total = (int64_t)(p.rb - p.ra) * p.W;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lr = idx / p.W, w = idx - lr * p.W;
    const int64_t r = p.ra + lr;
    const int ce = (int)((p.row0 + r) & 1);
    const uint64_t even = p.plane[ce][(r + 1) * p.W + w] & 0x1111111111111111ull;
    const uint64_t odd = p.plane[1 - ce][(r + 1) * p.W + w] & 0x1111111111111111ull;
    p.bits[idx] = (uint32_t)(compact1by1(even) | (compact1by1(odd) << 1));
  }
}

cudaError_t launch_pack_bits(int grid, cudaStream_t st, const PackBitsParams& p) {
  k_pack_bits<<<grid, 256, 0, st>>>(p);
  return cudaGetLastError();
}
cudaError_t launch_unpack_bits(int grid, cudaStream_t st, const UnpackBitsParams& p) {
  k_unpack_bits<<<grid, 256, 0, st>>>(p);
  return cudaGetLastError();
}

}  // namespace ising

namespace ising {

// Load every kernel the multi-slab / rank paths can launch, on the current device, before
// any of them runs.  With CUDA's lazy module loading (the default), the first launch of a
// kernel loads it, and loading can wait for kernels already running in the context; when
// several ranks share one process (ising_p2p_connect_local), a rank whose half-sweep spins on
// another rank's flags then blocks that other rank's first launch of a kernel — a deadlock
// (observed: the flag-wait timeout fired).  cudaFuncGetAttributes forces the load.
// ------------------------------------------------------------- lattice batches
// One CTA per lattice, the lattice in shared memory for the whole chunk of sweeps (row f2).
// The update is the same as the half-sweep kernels' — the same counter-based draws (reading
// R6 with this lattice's seed), side-word splices and acceptance — so every lattice of a
// batch is bit-identical to a one-lattice handle and to the oracle.  Metropolis runs the
// generic lockstep form (RULE 2: any beta, thresholds at 2^32 masked), heat bath the generic
// per-lane form (RULE 1).
// MR: the lockstep acceptance variant all lattices share (0 / 2 Metropolis, 3 / 5 / 6 / 7 heat
// bath); HB: the generic per-lane heat bath instead (lattices of different heat-bath classes).
template <bool HB, int MR = 2>
__global__ void __launch_bounds__(kBatchMaxThreads) k_batch_sweeps(const BatchParams P) {
  extern __shared__ uint4 batch_smem[];
  uint64_t* sm = reinterpret_cast<uint64_t*>(batch_smem);
  __shared__ BatchLattice L;
  __shared__ unsigned long long red[2];
  const int k = blockIdx.x;
  const int N = P.N, W = P.W;
  const int plane_words = N * W;
  uint64_t* g = P.planes + (size_t)k * 2 * plane_words;
  for (int i = threadIdx.x; i < plane_words; i += blockDim.x) {  // both planes, 128-bit
    reinterpret_cast<uint4*>(sm)[i] = __ldcg(reinterpret_cast<const uint4*>(g) + i);
  }
  if (threadIdx.x == 0) {
    L = P.lat[k];
    red[0] = red[1] = 0;
  }
  __syncthreads();
  HalfSweepParams p{};
  p.acc = L.acc;
  if constexpr (HB) p.keys = L.keys;
  const int half = W / 2;  // a thread updates two words (one 128-bit chunk) per row
  const int bands = batch_bands(N, W);
  const int H = (N + bands - 1) / bands;
  const int band = (int)threadIdx.x / half;
  const int w = 2 * ((int)threadIdx.x - band * half);
  const int i0 = band < bands ? band * H : N, i1 = min(i0 + H, N);
  const int wwest = w == 0 ? W - 1 : w - 1, weast = w + 2 == W ? 0 : w + 2;
  uint64_t P1[8];  // round 1's column-only Philox products (philox8_pre)
  philox8_round1((uint32_t)(4 * w), L.keys, P1);
  const uint32_t total = P.measure_only ? 1u : P.sweeps;
  for (uint32_t s = 1; s <= total; ++s) {
    const uint32_t t = P.t0 + s;
    const bool measure = P.obs && (P.measure_only || (P.every && (P.s_base + s) % P.every == 0));
    uint32_t up = 0, anti = 0;
    for (int c = 0; c < 2; ++c) {
      uint64_t* tgt = sm + c * plane_words;
      const uint64_t* src = sm + (1 - c) * plane_words;
      if (P.measure_only && c == 0) continue;
      // a thread owns column pair `w` of a band of consecutive rows [i0, i1) and rolls the
      // north / centre source words down it (one 128-bit load of the south pair per row, as
      // the staged kernel does)
      if (i0 < i1) {
        const ulonglong2 nn = *reinterpret_cast<const ulonglong2*>(src + (i0 == 0 ? N - 1 : i0 - 1) * W + w);
        const ulonglong2 cc = *reinterpret_cast<const ulonglong2*>(src + i0 * W + w);
        uint64_t n0 = nn.x, n1 = nn.y, c0 = cc.x, c1 = cc.y;
        int ro = i0 * W;
        for (int i = i0; i < i1; ++i, ro += W) {
          const ulonglong2 ss = *reinterpret_cast<const ulonglong2*>(src + (i == N - 1 ? 0 : ro + W) + w);
          const uint64_t s0 = ss.x, s1 = ss.y;
          const bool west = ((i & 1) == 0) == (c == 0);  // reading R2
          uint64_t side0, side1;
          if (west) {
            side0 = splice_west(c0, src[ro + wwest]);
            side1 = splice_west(c1, c0);
          } else {
            side0 = splice_east(c0, c1);
            side1 = splice_east(c1, src[ro + weast]);
          }
          const ulonglong2 tv = *reinterpret_cast<const ulonglong2*>(tgt + ro + w);
          uint64_t t0w = tv.x, t1w = tv.y;
          if (!P.measure_only) {
            if constexpr (HB) {
              const uint32_t ctr0 = (uint32_t)(4 * w);
              p.colour = (uint32_t)c;
              t0w = update_word<1>(t0w, n0, c0, s0, side0, ctr0, (uint32_t)i, t, p);
              t1w = update_word<1>(t1w, n1, c1, s1, side1, ctr0 + 4, (uint32_t)i, t, p);
            } else {
              uint4 rb[8];
              philox8_pre(t, (uint32_t)c, (uint32_t)i, L.keys, P1, rb);
              t0w = word_from_draws<MR>(t0w, n0, c0, s0, side0, rb, p);
              t1w = word_from_draws<MR>(t1w, n1, c1, s1, side1, rb + 4, p);
            }
            *reinterpret_cast<ulonglong2*>(tgt + ro + w) = make_ulonglong2(t0w, t1w);
          }
          if (c == 1 && measure) {  // every bond has exactly one white end (row a8)
            obs_word(t0w, n0, c0, s0, side0, up, anti);
            obs_word(t1w, n1, c1, s1, side1, up, anti);
          }
          n0 = c0;
          n1 = c1;
          c0 = s0;
          c1 = s1;
        }
      }
      __syncthreads();
    }
    if (measure) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        up += __shfl_xor_sync(0xffffffffu, up, off);
        anti += __shfl_xor_sync(0xffffffffu, anti, off);
      }
      if ((threadIdx.x & 31) == 0) {
        atomicAdd(&red[0], (unsigned long long)up);
        atomicAdd(&red[1], (unsigned long long)anti);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        const uint32_t slot = P.measure_only ? 0u : (P.s_base + s) / P.every - 1;
        unsigned long long* o = P.obs + 2 * ((size_t)k * P.n_samples + slot);
        o[0] = red[0];
        o[1] = red[1];
        red[0] = red[1] = 0;
      }
      __syncthreads();
    }
  }
  if (!P.measure_only)
    for (int i = threadIdx.x; i < plane_words; i += blockDim.x)
      __stcg(reinterpret_cast<uint4*>(g) + i, reinterpret_cast<const uint4*>(sm)[i]);
}

template <bool HB, int MR>
static cudaError_t batch_launch(int n_lattices, int threads, size_t smem, cudaStream_t st,
                                const BatchParams& p) {
  cudaError_t e = cudaFuncSetAttribute((const void*)k_batch_sweeps<HB, MR>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)kBatchMaxSmem);  // one value for every handle:
                                                              // no race between threads
  if (e != cudaSuccess) return e;
  k_batch_sweeps<HB, MR><<<n_lattices, threads, smem, st>>>(p);
  return cudaGetLastError();
}

// variant: the kernel variant every lattice of the batch shares (kernel_variant's numbering:
// 0 / 2 Metropolis, 3 / 5 / 6 / 7 heat bath, lockstep draws), 1 = generic heat bath (lattices
// of different heat-bath classes)
cudaError_t launch_batch_sweeps(int variant, int n_lattices, int threads, size_t smem,
                                cudaStream_t st, const BatchParams& p) {
  switch (variant) {
    case 0: return batch_launch<false, 0>(n_lattices, threads, smem, st, p);
    case 2: return batch_launch<false, 2>(n_lattices, threads, smem, st, p);
    case 3: return batch_launch<false, 3>(n_lattices, threads, smem, st, p);
    case 5: return batch_launch<false, 5>(n_lattices, threads, smem, st, p);
    case 6: return batch_launch<false, 6>(n_lattices, threads, smem, st, p);
    case 7: return batch_launch<false, 7>(n_lattices, threads, smem, st, p);
    case 1: return batch_launch<true, 2>(n_lattices, threads, smem, st, p);
  }
  return cudaErrorInvalidValue;
}

// Lattices too large for one CTA's shared memory (up to 2048^2): a thread-block cluster of
// P.cluster CTAs per lattice, CTA r holding rows [r R, (r + 1) R) of both planes plus one halo
// row above and below (R = N / cluster).  Each phase starts by pulling the source plane's two
// halo rows from the neighbouring CTAs' shared memory (distributed shared memory, the torus
// wrap across the cluster), updates the band like k_batch_sweeps, and ends with a cluster
// barrier — the neighbours' edge rows are final before anyone pulls them, and nobody
// overwrites a row a neighbour is still pulling.  Observables reduce per CTA, then into CTA 0's
// counters through DSMEM atomics.
template <bool HB, int MR>
__global__ void __launch_bounds__(kBatchMaxThreads) k_batch_cluster_sweeps(const BatchParams P) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ uint4 batch_smem[];
  uint64_t* sm = reinterpret_cast<uint64_t*>(batch_smem);  // plane c: (R + 2) x W, padded
  __shared__ BatchLattice L;
  __shared__ unsigned long long red[2];
  const int C = (int)cluster.num_blocks();
  const int r = (int)cluster.block_rank();
  const int k = blockIdx.x / C;
  const int N = P.N, W = P.W;
  const int R = N / C;
  const int pw = (R + 2) * W;  // padded plane words
  uint64_t* g = P.planes + (size_t)k * 2 * N * W;
  for (int c = 0; c < 2; ++c)
    for (int i = threadIdx.x; i < R * W / 2; i += blockDim.x)  // own rows, 128-bit
      reinterpret_cast<uint4*>(sm + c * pw + W)[i] =
          __ldcg(reinterpret_cast<const uint4*>(g + (size_t)c * N * W + (size_t)r * R * W) + i);
  if (threadIdx.x == 0) {
    L = P.lat[k];
    red[0] = red[1] = 0;
  }
  HalfSweepParams p{};
  const int up_rank = (r + C - 1) % C, dn_rank = (r + 1) % C;
  uint64_t* up_sm = cluster.map_shared_rank(sm, up_rank);
  uint64_t* dn_sm = cluster.map_shared_rank(sm, dn_rank);
  unsigned long long* red0 = cluster.map_shared_rank(red, 0);
  cluster.sync();  // every CTA loaded before anyone pulls halos
  p.acc = L.acc;
  if constexpr (HB) p.keys = L.keys;
  const int half = W / 2;
  const int bands = batch_bands(R, W);
  const int H = (R + bands - 1) / bands;
  const int band = (int)threadIdx.x / half;
  const int w = 2 * ((int)threadIdx.x - band * half);
  const int i0 = band < bands ? band * H : R, i1 = min(i0 + H, R);
  const int wwest = w == 0 ? W - 1 : w - 1, weast = w + 2 == W ? 0 : w + 2;
  const int grow0 = r * R;  // global row of local row 0
  uint64_t P1[8];  // round 1's column-only Philox products (philox8_pre)
  philox8_round1((uint32_t)(4 * w), L.keys, P1);
  const uint32_t total = P.measure_only ? 1u : P.sweeps;
  for (uint32_t s = 1; s <= total; ++s) {
    const uint32_t t = P.t0 + s;
    const bool measure = P.obs && (P.measure_only || (P.every && (P.s_base + s) % P.every == 0));
    uint32_t up = 0, anti = 0;
    for (int c = 0; c < 2; ++c) {
      if (P.measure_only && c == 0) continue;
      uint64_t* tgt = sm + c * pw + W;  // local row 0
      uint64_t* src = sm + (1 - c) * pw + W;
      // halo rows of the source plane: the upper neighbour's last row, the lower one's first
      for (int q = threadIdx.x; q < 2 * W; q += blockDim.x) {
        if (q < W)
          src[-W + q] = up_sm[(1 - c) * pw + W + (R - 1) * W + q];
        else
          src[R * W + q - W] = dn_sm[(1 - c) * pw + W + q - W];
      }
      __syncthreads();
      if (i0 < i1) {
        const ulonglong2 nn = *reinterpret_cast<const ulonglong2*>(src + (i0 - 1) * W + w);
        const ulonglong2 cc = *reinterpret_cast<const ulonglong2*>(src + i0 * W + w);
        uint64_t n0 = nn.x, n1 = nn.y, c0 = cc.x, c1 = cc.y;
        int ro = i0 * W;
        for (int i = i0; i < i1; ++i, ro += W) {
          const ulonglong2 ss = *reinterpret_cast<const ulonglong2*>(src + ro + W + w);
          const uint64_t s0 = ss.x, s1 = ss.y;
          const int gi = grow0 + i;
          const bool west = ((gi & 1) == 0) == (c == 0);  // reading R2
          uint64_t side0, side1;
          if (west) {
            side0 = splice_west(c0, src[ro + wwest]);
            side1 = splice_west(c1, c0);
          } else {
            side0 = splice_east(c0, c1);
            side1 = splice_east(c1, src[ro + weast]);
          }
          const ulonglong2 tv = *reinterpret_cast<const ulonglong2*>(tgt + ro + w);
          uint64_t t0w = tv.x, t1w = tv.y;
          if (!P.measure_only) {
            if constexpr (HB) {
              p.colour = (uint32_t)c;
              t0w = update_word<1>(t0w, n0, c0, s0, side0, (uint32_t)(4 * w), (uint32_t)gi, t, p);
              t1w = update_word<1>(t1w, n1, c1, s1, side1, (uint32_t)(4 * w + 4), (uint32_t)gi, t, p);
            } else {
              uint4 rb[8];
              philox8_pre(t, (uint32_t)c, (uint32_t)gi, L.keys, P1, rb);
              t0w = word_from_draws<MR>(t0w, n0, c0, s0, side0, rb, p);
              t1w = word_from_draws<MR>(t1w, n1, c1, s1, side1, rb + 4, p);
            }
            *reinterpret_cast<ulonglong2*>(tgt + ro + w) = make_ulonglong2(t0w, t1w);
          }
          if (c == 1 && measure) {
            obs_word(t0w, n0, c0, s0, side0, up, anti);
            obs_word(t1w, n1, c1, s1, side1, up, anti);
          }
          n0 = c0;
          n1 = c1;
          c0 = s0;
          c1 = s1;
        }
      }
      cluster.sync();  // this plane final everywhere before the next phase pulls its halos
    }
    if (measure) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        up += __shfl_xor_sync(0xffffffffu, up, off);
        anti += __shfl_xor_sync(0xffffffffu, anti, off);
      }
      if ((threadIdx.x & 31) == 0 && (up | anti)) {
        atomicAdd(&red0[0], (unsigned long long)up);
        atomicAdd(&red0[1], (unsigned long long)anti);
      }
      cluster.sync();
      if (r == 0 && threadIdx.x == 0) {
        const uint32_t slot = P.measure_only ? 0u : (P.s_base + s) / P.every - 1;
        unsigned long long* o = P.obs + 2 * ((size_t)k * P.n_samples + slot);
        o[0] = red[0];
        o[1] = red[1];
        red[0] = red[1] = 0;  // before CTA 0 reaches the next cluster barrier
      }
    }
  }
  if (!P.measure_only)
    for (int c = 0; c < 2; ++c)
      for (int i = threadIdx.x; i < R * W / 2; i += blockDim.x)
        __stcg(reinterpret_cast<uint4*>(g + (size_t)c * N * W + (size_t)r * R * W) + i,
               reinterpret_cast<const uint4*>(sm + c * pw + W)[i]);
  cluster.sync();  // no CTA exits while a neighbour may still read its shared memory
}

template <bool HB, int MR>
static cudaError_t cluster_launch(int n_lattices, int cluster, int threads, size_t smem,
                                  cudaStream_t st, const BatchParams& p) {
  const void* f = (const void*)k_batch_cluster_sweeps<HB, MR>;
  cudaError_t e =
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBatchMaxSmem);
  if (e == cudaSuccess && cluster > 8)
    e = cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(n_lattices * cluster));
  cfg.blockDim = dim3((unsigned)threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_batch_cluster_sweeps<HB, MR>, p);
}

cudaError_t launch_batch_cluster_sweeps(int variant, int n_lattices, int cluster, int threads,
                                        size_t smem, cudaStream_t st, const BatchParams& p) {
  switch (variant) {
    case 0: return cluster_launch<false, 0>(n_lattices, cluster, threads, smem, st, p);
    case 2: return cluster_launch<false, 2>(n_lattices, cluster, threads, smem, st, p);
    case 3: return cluster_launch<false, 3>(n_lattices, cluster, threads, smem, st, p);
    case 5: return cluster_launch<false, 5>(n_lattices, cluster, threads, smem, st, p);
    case 6: return cluster_launch<false, 6>(n_lattices, cluster, threads, smem, st, p);
    case 7: return cluster_launch<false, 7>(n_lattices, cluster, threads, smem, st, p);
    case 1: return cluster_launch<true, 2>(n_lattices, cluster, threads, smem, st, p);
  }
  return cudaErrorInvalidValue;
}

// Random / cold start of every lattice of a batch (row a3 with each lattice's seed): spin +1
// iff r(seed_k, 0, c, i, j) < 2^31 — the same draws k_init takes for a one-lattice handle.
__global__ void k_batch_init(const BatchParams P, int cold) {
  const int64_t plane_words = (int64_t)P.N * P.W;
  const int64_t total = 2 * plane_words;
  const int k = blockIdx.y;
  const BatchLattice& L = P.lat[k];
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(idx / plane_words);
    const int64_t rem = idx - c * plane_words;
    const int i = (int)(rem / P.W);
    const int w = (int)(rem - (int64_t)i * P.W);
    uint64_t word = 0x1111111111111111ull;
    if (!cold) {
      word = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const uint4 r = philox4x32_10(0u, (uint32_t)(4 * w + b), (uint32_t)c, (uint32_t)i, L.keys);
        const uint32_t rr[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (rr[q] < 0x80000000u) word |= 1ull << (4 * (4 * b + q));
      }
    }
    P.planes[(size_t)k * total + idx] = word;
  }
}

cudaError_t launch_batch_init(int n_lattices, int cold, cudaStream_t st, const BatchParams& p) {
  const int64_t total = 2 * (int64_t)p.N * p.W;
  const int gx = (int)std::min<int64_t>((total + 255) / 256, 1024);
  k_batch_init<<<dim3(gx, n_lattices), 256, 0, st>>>(p, cold);
  return cudaGetLastError();
}

// Lattice k as the +-1 byte full lattice (row a9): site (i, J) is plane (i + J) & 1, plane
// column J / 2 = lane (J / 2) % 16 of word J / 32.
__global__ void k_batch_unpack(const BatchParams P, int k, int8_t* full) {
  const int64_t M = (int64_t)P.W * 32;
  const int64_t total = (int64_t)P.N * M;
  const uint64_t* g = P.planes + (size_t)k * 2 * P.N * P.W;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / M, J = idx - i * M;
    const int c = (int)((i + J) & 1);
    const int64_t j = J >> 1;
    const uint64_t word = g[(size_t)c * P.N * P.W + i * P.W + (j >> 4)];
    full[idx] = ((word >> (4 * (j & 15))) & 1) ? 1 : -1;
  }
}

// Lattice k from the +-1 byte full lattice (the inverse of k_batch_unpack); *bad := 1 if a
// value is not -1 / +1.
__global__ void k_batch_pack(const BatchParams P, int k, const int8_t* full, unsigned int* bad) {
  const int64_t plane_words = (int64_t)P.N * P.W;
  const int64_t M = (int64_t)P.W * 32;
  uint64_t* g = P.planes + (size_t)k * 2 * plane_words;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < 2 * plane_words;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(idx / plane_words);
    const int64_t rem = idx - c * plane_words;
    const int64_t i = rem / P.W, w = rem - i * P.W;
    const int8_t* row = full + i * M;
    uint64_t word = 0;
    bool ok = true;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int64_t J = 2 * (16 * w + q) + ((i + c) & 1);  // reading R1
      const int8_t v = row[J];
      ok = ok && (v == 1 || v == -1);
      word |= (uint64_t)(v == 1) << (4 * q);
    }
    if (!ok) atomicExch(bad, 1u);
    g[idx] = word;
  }
}

cudaError_t launch_batch_pack(int lattice, cudaStream_t st, const BatchParams& p, const int8_t* full,
                              unsigned int* bad) {
  const int64_t total = 2 * (int64_t)p.N * p.W;
  const int grid = (int)std::min<int64_t>((total + 255) / 256, 4096);
  k_batch_pack<<<grid, 256, 0, st>>>(p, lattice, full, bad);
  return cudaGetLastError();
}

cudaError_t launch_batch_unpack(int lattice, cudaStream_t st, const BatchParams& p, int8_t* full) {
  const int64_t total = (int64_t)p.N * p.W * 32;
  const int grid = (int)std::min<int64_t>((total + 255) / 256, 4096);
  k_batch_unpack<<<grid, 256, 0, st>>>(p, lattice, full);
  return cudaGetLastError();
}

template <int R>
static cudaError_t preload_rule() {
  cudaFuncAttributes a;
  cudaError_t e;
  if ((e = cudaFuncGetAttributes(&a, k_halfsweep<R, false>)) != cudaSuccess) return e;
  if ((e = cudaFuncGetAttributes(&a, k_halfsweep<R, true>)) != cudaSuccess) return e;
  if ((e = cudaFuncGetAttributes(&a, k_halfsweep_staged<R, false>)) != cudaSuccess) return e;
  return cudaFuncGetAttributes(&a, k_halfsweep_staged<R, true>);
}

cudaError_t preload_kernels() {
  cudaError_t e;
  if ((e = preload_rule<0>()) != cudaSuccess) return e;
  if ((e = preload_rule<1>()) != cudaSuccess) return e;
  if ((e = preload_rule<2>()) != cudaSuccess) return e;
  if ((e = preload_rule<3>()) != cudaSuccess) return e;
  if ((e = preload_rule<4>()) != cudaSuccess) return e;
  if ((e = preload_rule<5>()) != cudaSuccess) return e;
  if ((e = preload_rule<6>()) != cudaSuccess) return e;
  if ((e = preload_rule<7>()) != cudaSuccess) return e;
  cudaFuncAttributes a;
  const void* others[] = {(const void*)k_sync,      (const void*)k_gather, (const void*)k_set_u32,
                          (const void*)k_zero_u64,  (const void*)k_copy_u64, (const void*)k_init,
                          (const void*)k_observables, (const void*)k_pack,  (const void*)k_unpack,
                          (const void*)k_pack_bits, (const void*)k_unpack_bits};
  for (const void* f : others)
    if ((e = cudaFuncGetAttributes(&a, f)) != cudaSuccess) return e;
  return cudaSuccess;
}

}  // namespace ising
