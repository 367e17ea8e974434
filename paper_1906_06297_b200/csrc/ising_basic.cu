// ising_basic.cu — the paper's *basic* implementation (§3.1, the Fig. 2 CUDA C
// listing `update_lattice<is_black>`) rebuilt for sm_100a as a second
// workload: one signed byte per spin, two colour planes of
// N x M/2 "compacted along the rows", the listing's stencil with periodic
// wrap, and the same draw contract / integer thresholds as the multi-spin path, so both
// layouts are bit-identical to each other and to the oracle.
//
// B200 choices (default kernel): a thread owns 16 consecutive plane sites (four Philox4x32-10
// blocks, 128-bit loads / stores) of a band of rows, keeps the source rows above / at /
// below in registers as it walks down, and evaluates the listing's stencil and acceptance
// on four byte lanes per 32-bit word (SWAR) instead of site by site; no random-number array
// in HBM (the paper pre-generates one): 3 algorithmic bytes per attempted
// flip.  The listing-shaped kernel (a thread per four sites, per-site selects) is kept for
// the layout / kernel-style comparison (ISING_BASIC_LISTING=1) and for widths whose plane
// rows are not a whole number of 16-byte chunks (L_cols % 32 != 0).
#include <cuda_runtime.h>

#include <algorithm>

#include "ising_kernels.cuh"

namespace ising {

__device__ __forceinline__ uint4 philox_basic(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
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

// ---- listing form (ISING_BASIC_LISTING=1): the Fig. 2 kernel site by site ----
// One colour phase: lattice (target colour c) and op_lattice (the other colour), both
// nx x ny int8.  Thread = plane sites (i, 4q .. 4q+3); x covers the quads of a row, y
// strides over rows (no 64-bit division in the index math).  rule 0 = Metropolis, else
// heat bath.
template <int RULE>
__global__ void __launch_bounds__(256) k_basic_listing(const BasicParams p) {
  const int64_t quads = p.ny >> 2;
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= quads) return;
  const int64_t j0 = 4 * q;
  const int8_t* op = p.op_lattice;
  for (int64_t i = blockIdx.y; i < p.nx; i += gridDim.y) {
    // "Set stencil indices with periodicity"
    const int64_t ipp = (i + 1 < p.nx) ? i + 1 : 0;
    const int64_t inn = (i - 1 >= 0) ? i - 1 : p.nx - 1;
    const char4 up = *reinterpret_cast<const char4*>(op + inn * p.ny + j0);
    const char4 mid = *reinterpret_cast<const char4*>(op + i * p.ny + j0);
    const char4 dn = *reinterpret_cast<const char4*>(op + ipp * p.ny + j0);
    // "Select off-column index based on color and row index parity":
    // black: joff = (i % 2) ? jpp : jnn; white: joff = (i % 2) ? jnn : jpp
    const bool east = (p.colour == 0) == ((i & 1) == 1);
    const int64_t jside = east ? ((j0 + 4 < p.ny) ? j0 + 4 : 0) : ((j0 - 1 >= 0) ? j0 - 1 : p.ny - 1);
    const int8_t side_edge = op[i * p.ny + jside];
    const int8_t o[4] = {mid.x, mid.y, mid.z, mid.w};
    const int8_t u[4] = {up.x, up.y, up.z, up.w};
    const int8_t d[4] = {dn.x, dn.y, dn.z, dn.w};
    char4 tv = *reinterpret_cast<const char4*>(p.lattice + i * p.ny + j0);
    int8_t s[4] = {tv.x, tv.y, tv.z, tv.w};
    const uint4 r4 = philox_basic(p.t, (uint32_t)q, p.colour, (uint32_t)i, p.keys);
    const uint32_t rr[4] = {r4.x, r4.y, r4.z, r4.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int8_t joff = east ? (k < 3 ? o[k + 1] : side_edge) : (k > 0 ? o[k - 1] : side_edge);
      const int nn_sum = u[k] + o[k] + d[k] + joff;
      const int a = (nn_sum * s[k] + 4) >> 1;       // e = nn_sum * s = 2a - 4, dE = 2 J e
      uint32_t thr;
      bool always;
      if (RULE == 0) {
        // Metropolis (PAPER.md:40-41, :155-156 with the integer compare of reading R5)
        thr = (a == 4) ? p.acc.thr[4] : p.acc.thr[3];
        always = (a <= 2) || ((p.acc.always_mask >> a) & 1u);
      } else {
        // heat bath
        thr = p.acc.thr[a];
        always = (p.acc.always_mask >> a) & 1u;
      }
      if (always || rr[k] < thr) s[k] = (int8_t)-s[k];
    }
    tv.x = s[0];
    tv.y = s[1];
    tv.z = s[2];
    tv.w = s[3];
    *reinterpret_cast<char4*>(p.lattice + i * p.ny + j0) = tv;
  }
}

// ---- B200 form (default): byte-lane SWAR, 16 sites per thread, rows rolled in registers ----
// Per 32-bit word = 4 byte lanes (plane sites j .. j+3, one Philox block, word k = j & 3 ->
// byte k).  A +-1 byte has bit 1 set iff the spin is -1, so with t the target word,
//   b2 = sum over the 4 neighbour words of ((nb ^ t) & 0x02020202)
// is twice the number of anti-aligned neighbours b per lane (<= 8, no carries).  Both rules
// reduce to "flip iff b >= nc", nc = #{compared classes m : r >= T[m]}: Metropolis compares
// classes a = 3, 4 (a <= 2 flips), heat bath every class whose T is below 2^32 (r < T[a] <=>
// a + nc <= 4 for the non-increasing T, a = 4 - b).  x = b2 + 16 - 2 nc lies in [6, 24] per
// lane and bit 4 of x is the flip bit.  A flip negates the byte: t ^= 0xFE per flipped lane,
// 0xFE f = (f << 8) - 2 f exactly (mod 2^32) for 0/1 lanes f.
constexpr uint32_t kByte0 = 0x01010101u;
constexpr uint32_t kByteDown = 0x02020202u;

__device__ __forceinline__ void horner8(uint32_t& acc, uint32_t r, uint32_t T) {
  asm("{\n\t.reg .u32 d;\n\t"
      "sub.cc.u32 d, %1, %2;\n\t"
      "madc.lo.u32 %0, %0, 256, 0;\n\t}"
      : "+r"(acc)
      : "r"(r), "r"(T));
}

__device__ __forceinline__ void add_carry(uint32_t& acc, uint32_t r, uint32_t T) {
  asm("{\n\t.reg .u32 d;\n\t"
      "sub.cc.u32 d, %1, %2;\n\t"
      "addc.u32 %0, %0, 0;\n\t}"
      : "+r"(acc)
      : "r"(r), "r"(T));
}

// nc per byte lane for one Philox block (lanes 3 .. 0 in Horner order).
template <int RULE>
__device__ __forceinline__ uint32_t basic_nc(const uint4 r, const Accept& A) {
  const uint32_t rr[4] = {r.w, r.z, r.y, r.x};
  if constexpr (RULE == 4) {
    return (A.nc_const & 0xFu) * kByte0;  // draw-free (T3, T4 in {0, 2^32})
  } else if constexpr (RULE == 0 || RULE == 2) {
    uint32_t a3 = 0, a4 = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      horner8(a3, rr[k], A.thr[3]);
      horner8(a4, rr[k], A.thr[4]);
    }
    if constexpr (RULE == 0) return a3 + a4;
    return (a3 & A.keep3) + (a4 & A.keep4);  // a class at 2^32 never blocks a flip
  } else if constexpr (RULE == 3 || RULE == 5 || RULE == 6) {
    constexpr int NA = RULE == 3 ? 0 : RULE == 5 ? 1 : 2;  // "always" prefix, left out
    uint32_t acc = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      horner8(acc, rr[k], A.thr[NA]);
#pragma unroll
      for (int m = NA + 1; m < 5; ++m) add_carry(acc, rr[k], A.thr[m]);
    }
    return acc;
  } else if constexpr (RULE == 7) {
    // symmetric heat bath (ising_kernels.cu, update_word<7>): the Metropolis compare pair on
    // v = |r| (as int32), and nc = 5 - that count in lanes with r >= 2^31
    uint32_t a3 = 0, a4 = 0, am = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t v = (uint32_t)abs((int32_t)rr[k]);
      horner8(a3, v, A.thr[3]);
      horner8(a4, v, A.thr[4]);
      am = __funnelshift_l(rr[k], am, 8);  // r's msb -> bit 7 of the new byte
    }
    const uint32_t m = (am >> 7) & kByte0;
    const uint32_t m255 = (m << 8) - m;
    return ((a3 + a4) ^ m255) - (m255 & 0xFAFAFAFAu);  // m: (255 - c) - 250 = 5 - c
  } else {  // RULE 1: heat bath with an arbitrary always-mask (not produced by the host)
    uint32_t nc = 0;
#pragma unroll
    for (int m = 0; m < 5; ++m) {
      uint32_t acc = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) horner8(acc, rr[k], A.thr[m]);
      nc += ((A.always_mask >> m) & 1u) ? 0u : acc;
    }
    return nc;
  }
}

__device__ __forceinline__ uint32_t basic_update(uint32_t t, uint32_t n, uint32_t c, uint32_t s,
                                                 uint32_t side, uint32_t nc) {
  const uint32_t b2 = ((n ^ t) & kByteDown) + ((c ^ t) & kByteDown) + ((s ^ t) & kByteDown) +
                      ((side ^ t) & kByteDown);
  const uint32_t x = b2 + 0x10101010u - (nc << 1);
  const uint32_t f = (x >> 4) & kByte0;
  return t ^ ((f << 8) - (f << 1));
}

__device__ __forceinline__ uint4 ld_u4_nc(const int8_t* p) {
  return __ldg(reinterpret_cast<const uint4*>(p));
}

constexpr int kBasicRows = 16;  // rows per work item (source rows reused in registers)

// OBS (white phase of a measured sweep): also add the observables of the resulting state —
// every bond has exactly one white end, whose four black neighbours are the N / C / S / side
// words here, and every black site is the C word of exactly one white site.
template <int RULE, bool OBS = false>
__global__ void __launch_bounds__(128, 4) k_basic_halfsweep(const BasicParams p) {
  const int64_t chunks = p.ny >> 4;  // 16-byte chunks per plane row
  uint32_t obs_up = 0, obs_anti = 0;
  const int64_t bands = (p.nx + kBasicRows - 1) / kBasicRows;
  const int64_t items = chunks * bands;
  const int8_t* op = p.op_lattice;
  for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < items;
       it += (int64_t)gridDim.x * blockDim.x) {
    const int64_t band = it / chunks;
    const int64_t q = it - band * chunks;
    const int64_t j0 = 16 * q;
    const int64_t i0 = band * kBasicRows;
    const int64_t i1 = (i0 + kBasicRows < p.nx) ? i0 + kBasicRows : p.nx;
    // "Set stencil indices with periodicity": rows wrap mod nx
    uint4 up = ld_u4_nc(op + ((i0 > 0) ? i0 - 1 : p.nx - 1) * p.ny + j0);
    uint4 mid = ld_u4_nc(op + i0 * p.ny + j0);
    const int64_t je = (j0 + 16 < p.ny) ? j0 + 16 : 0;  // east edge byte's column
    const int64_t jw = (j0 > 0) ? j0 - 1 : p.ny - 1;    // west edge byte's column
    for (int64_t i = i0; i < i1; ++i) {
      const uint4 dn = ld_u4_nc(op + ((i + 1 < p.nx) ? i + 1 : 0) * p.ny + j0);
      // off-column neighbour: black odd rows and white even rows
      // look east (j + 1), the others west (j - 1)
      const bool east = (p.colour == 0) == ((i & 1) == 1);
      const uint32_t edge = (uint8_t)__ldg(op + i * p.ny + (east ? je : jw));
      uint4 side;
      if (east) {
        side.x = __funnelshift_r(mid.x, mid.y, 8);
        side.y = __funnelshift_r(mid.y, mid.z, 8);
        side.z = __funnelshift_r(mid.z, mid.w, 8);
        side.w = __funnelshift_r(mid.w, edge, 8);
      } else {
        side.x = __funnelshift_l(edge << 24, mid.x, 8);
        side.y = __funnelshift_l(mid.x, mid.y, 8);
        side.z = __funnelshift_l(mid.y, mid.z, 8);
        side.w = __funnelshift_l(mid.z, mid.w, 8);
      }
      int8_t* tp = p.lattice + i * p.ny + j0;
      uint4 t = *reinterpret_cast<const uint4*>(tp);
      const uint32_t ctr = (uint32_t)(j0 >> 2);  // Philox block of plane site j: j >> 2
      const uint32_t row = (uint32_t)i;
      t.x = basic_update(t.x, up.x, mid.x, dn.x, side.x,
                         basic_nc<RULE>(philox_basic(p.t, ctr + 0, p.colour, row, p.keys), p.acc));
      t.y = basic_update(t.y, up.y, mid.y, dn.y, side.y,
                         basic_nc<RULE>(philox_basic(p.t, ctr + 1, p.colour, row, p.keys), p.acc));
      t.z = basic_update(t.z, up.z, mid.z, dn.z, side.z,
                         basic_nc<RULE>(philox_basic(p.t, ctr + 2, p.colour, row, p.keys), p.acc));
      t.w = basic_update(t.w, up.w, mid.w, dn.w, side.w,
                         basic_nc<RULE>(philox_basic(p.t, ctr + 3, p.colour, row, p.keys), p.acc));
      *reinterpret_cast<uint4*>(tp) = t;
      if (OBS) {  // +-1 bytes differ iff bit 1 differs; +1 has bit 1 clear
        const uint32_t tw[4] = {t.x, t.y, t.z, t.w}, nw[4] = {up.x, up.y, up.z, up.w};
        const uint32_t cw[4] = {mid.x, mid.y, mid.z, mid.w}, sw[4] = {dn.x, dn.y, dn.z, dn.w};
        const uint32_t dw[4] = {side.x, side.y, side.z, side.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          obs_up += __popc(~tw[k] & kByteDown) + __popc(~cw[k] & kByteDown);
          obs_anti += __popc((tw[k] ^ nw[k]) & kByteDown) + __popc((tw[k] ^ cw[k]) & kByteDown) +
                      __popc((tw[k] ^ sw[k]) & kByteDown) + __popc((tw[k] ^ dw[k]) & kByteDown);
        }
      }
      up = mid;
      mid = dn;
    }
  }
  if (OBS) {
    unsigned long long u = obs_up, a = obs_anti;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      u += __shfl_xor_sync(0xffffffffu, u, off);
      a += __shfl_xor_sync(0xffffffffu, a, off);
    }
    if ((threadIdx.x & 31) == 0 && (u | a)) {
      atomicAdd(&p.obs_out[0], u);
      atomicAdd(&p.obs_out[1], a);
    }
  }
}

// Random / cold start on the byte planes (reading R8).
__global__ void k_basic_init(int8_t* black, int8_t* white, int64_t nx, int64_t ny, int cold,
                             PhiloxKeys keys) {
  const int64_t quads = ny >> 2;
  const int64_t total = 2 * nx * quads;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += stride) {
    const int c = (int)(idx / (nx * quads));
    const int64_t rem = idx - (int64_t)c * nx * quads;
    const int64_t i = rem / quads;
    const int64_t j0 = 4 * (rem - i * quads);
    char4 v = make_char4(1, 1, 1, 1);
    if (!cold) {
      const uint4 r = philox_basic(0u, (uint32_t)(j0 >> 2), (uint32_t)c, (uint32_t)i, keys);
      v = make_char4(r.x < 0x80000000u ? 1 : -1, r.y < 0x80000000u ? 1 : -1,
                     r.z < 0x80000000u ? 1 : -1, r.w < 0x80000000u ? 1 : -1);
    }
    *reinterpret_cast<char4*>((c == 0 ? black : white) + i * ny + j0) = v;
  }
}

// Up count and antiparallel bonds (every bond has one black end: its 4 white neighbours).
// Vectorised observables (ny % 16 == 0): one thread per 16 black sites of a row, loaded as
// uint4 together with the white N / C / S words; the side neighbours (j - 1 for even rows, j + 1
// for odd, Fig. 2 listing) are byte funnel shifts of the C words with the word beyond
// the chunk.  +-1 bytes differ iff bit 1 differs, so popcounts of (x ^ y) & 0x02020202 count
// antiparallel bonds; up spins are bytes with bit 1 clear.  Rows are walked with a 2D
// grid-stride (no 64-bit divisions).
__global__ void __launch_bounds__(256) k_basic_observables16(const int8_t* black,
                                                             const int8_t* white, int64_t nx,
                                                             int64_t ny, unsigned long long* out) {
  const int64_t chunks = ny >> 4;
  uint32_t up = 0, anti = 0;  // per thread: <= 4 bonds + 2 spins per site, few chunks
  unsigned long long up64 = 0, anti64 = 0;
  for (int64_t i = blockIdx.y; i < nx; i += gridDim.y) {
    const int64_t inn = i == 0 ? nx - 1 : i - 1, ipp = i + 1 == nx ? 0 : i + 1;
    const int8_t* wrow = white + i * ny;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < chunks;
         q += (int64_t)gridDim.x * blockDim.x) {
      const int64_t j0 = 16 * q;
      const uint4 b = *reinterpret_cast<const uint4*>(black + i * ny + j0);
      const uint4 wn = *reinterpret_cast<const uint4*>(white + inn * ny + j0);
      const uint4 wc = *reinterpret_cast<const uint4*>(wrow + j0);
      const uint4 ws = *reinterpret_cast<const uint4*>(white + ipp * ny + j0);
      const uint32_t bb[4] = {b.x, b.y, b.z, b.w}, n[4] = {wn.x, wn.y, wn.z, wn.w};
      const uint32_t c[4] = {wc.x, wc.y, wc.z, wc.w}, sd[4] = {ws.x, ws.y, ws.z, ws.w};
      uint32_t side[4];
      if (i & 1) {  // east: bytes j + 1 .. j + 16
        const uint32_t e = *reinterpret_cast<const uint32_t*>(wrow + (j0 + 16 == ny ? 0 : j0 + 16));
        side[0] = __funnelshift_r(c[0], c[1], 8);
        side[1] = __funnelshift_r(c[1], c[2], 8);
        side[2] = __funnelshift_r(c[2], c[3], 8);
        side[3] = __funnelshift_r(c[3], e, 8);
      } else {  // west: bytes j - 1 .. j + 14
        const uint32_t w = *reinterpret_cast<const uint32_t*>(wrow + (j0 == 0 ? ny - 4 : j0 - 4));
        side[0] = __funnelshift_l(w, c[0], 8);
        side[1] = __funnelshift_l(c[0], c[1], 8);
        side[2] = __funnelshift_l(c[1], c[2], 8);
        side[3] = __funnelshift_l(c[2], c[3], 8);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        up += __popc(~bb[k] & kByteDown) + __popc(~c[k] & kByteDown);
        anti += __popc((bb[k] ^ n[k]) & kByteDown) + __popc((bb[k] ^ c[k]) & kByteDown) +
                __popc((bb[k] ^ sd[k]) & kByteDown) + __popc((bb[k] ^ side[k]) & kByteDown);
      }
    }
    up64 += up;
    anti64 += anti;
    up = anti = 0;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    up64 += __shfl_xor_sync(0xffffffffu, up64, off);
    anti64 += __shfl_xor_sync(0xffffffffu, anti64, off);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&out[0], up64);
    atomicAdd(&out[1], anti64);
  }
}

// Vectorised conversion (ny % 8 == 0): one thread per 16 bytes of a full row = 8 sites of each
// plane; full byte J = 2 j + x comes from colour (i + x) & 1, so the row is a byte interleave
// of the two planes' 8-byte segments (PRMT both ways).
__global__ void __launch_bounds__(256) k_basic_convert16(int8_t* black, int8_t* white, int8_t* full,
                                                         int64_t ny, int64_t r0, int64_t rows,
                                                         int to_full, unsigned int* bad) {
  const int64_t M = 2 * ny;
  const int64_t segs = M >> 4;
  unsigned int badv = 0;
  for (int64_t li = blockIdx.y; li < rows; li += gridDim.y) {
    const int64_t i = r0 + li;
    int8_t* pa = ((i & 1) ? white : black) + i * ny;  // even full columns
    int8_t* pb = ((i & 1) ? black : white) + i * ny;  // odd full columns
    for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < segs;
         u += (int64_t)gridDim.x * blockDim.x) {
      uint4* f = reinterpret_cast<uint4*>(full + li * M + 16 * u);
      uint2* a = reinterpret_cast<uint2*>(pa + 8 * u);
      uint2* b = reinterpret_cast<uint2*>(pb + 8 * u);
      if (to_full) {
        const uint2 A = *a, B = *b;
        *f = make_uint4(__byte_perm(A.x, B.x, 0x5140), __byte_perm(A.x, B.x, 0x7362),
                        __byte_perm(A.y, B.y, 0x5140), __byte_perm(A.y, B.y, 0x7362));
      } else {
        const uint4 o = *f;
        const uint32_t w[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {  // every byte must be 0x01 or 0xFF
          const uint32_t y = w[k] ^ 0x01010101u;
          badv |= (y & 0x01010101u) | (((y >> 1) ^ y) & 0x7E7E7E7Eu);
        }
        *a = make_uint2(__byte_perm(o.x, o.y, 0x6420), __byte_perm(o.z, o.w, 0x6420));
        *b = make_uint2(__byte_perm(o.x, o.y, 0x7531), __byte_perm(o.z, o.w, 0x7531));
      }
    }
  }
  if (badv) atomicOr(bad, 1u);
}

__global__ void __launch_bounds__(256) k_basic_observables(const int8_t* black, const int8_t* white,
                                                           int64_t nx, int64_t ny,
                                                           unsigned long long* out) {
  const int64_t total = nx * ny;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned long long up = 0, anti = 0;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += stride) {
    const int64_t i = idx / ny;
    const int64_t j = idx - i * ny;
    const int64_t ipp = (i + 1 < nx) ? i + 1 : 0;
    const int64_t inn = (i - 1 >= 0) ? i - 1 : nx - 1;
    const int64_t joff = (i & 1) ? ((j + 1 < ny) ? j + 1 : 0) : ((j - 1 >= 0) ? j - 1 : ny - 1);
    const int b = black[idx];
    up += (b > 0) + (white[idx] > 0);
    anti += (b != white[inn * ny + j]) + (b != white[idx]) + (b != white[ipp * ny + j]) +
            (b != white[i * ny + joff]);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    up += __shfl_xor_sync(0xffffffffu, up, off);
    anti += __shfl_xor_sync(0xffffffffu, anti, off);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&out[0], up);
    atomicAdd(&out[1], anti);
  }
}

// Full lattice (row-major +-1 bytes, rows [r0, r0 + rows)) <-> planes.  to_full = 1 unpacks.
__global__ void k_basic_convert(int8_t* black, int8_t* white, int8_t* full, int64_t ny, int64_t r0,
                                int64_t rows, int to_full, unsigned int* bad) {
  const int64_t M = 2 * ny;
  const int64_t total = rows * M;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += stride) {
    const int64_t li = idx / M;
    const int64_t J = idx - li * M;
    const int64_t i = r0 + li;
    int8_t* plane = ((i + J) & 1) ? white : black;
    if (to_full) {
      full[idx] = plane[i * ny + (J >> 1)];
    } else {
      const int8_t v = full[idx];
      if (v != 1 && v != -1) atomicOr(bad, 1u);
      plane[i * ny + (J >> 1)] = v;
    }
  }
}

cudaError_t launch_basic_halfsweep(int rule, int listing, int sms, cudaStream_t st,
                                   const BasicParams& p) {
  if (listing || (p.ny & 15) != 0) {  // the SWAR kernel needs whole 16-byte chunks
    if (p.obs_out) return cudaErrorInvalidValue;  // fused observables: SWAR kernel only
    const int64_t quads = p.ny >> 2;
    const dim3 g((unsigned)((quads + 255) / 256), (unsigned)(p.nx < 65535 ? p.nx : 65535));
    const bool metropolis = rule == 0 || rule == 2 || rule == 4;
    if (metropolis)
      k_basic_listing<0><<<g, 256, 0, st>>>(p);
    else
      k_basic_listing<1><<<g, 256, 0, st>>>(p);
    return cudaGetLastError();
  }
  const int64_t items = (p.ny >> 4) * ((p.nx + kBasicRows - 1) / kBasicRows);
  const int64_t cap = (int64_t)sms * 4 * 64;  // grid-stride beyond 64 waves
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((items + 127) / 128, cap));
#define ISING_BASIC_CASE(R)                                                     \
  case R:                                                                       \
    if (p.obs_out)                                                              \
      k_basic_halfsweep<R, true><<<grid, 128, 0, st>>>(p);                      \
    else                                                                        \
      k_basic_halfsweep<R><<<grid, 128, 0, st>>>(p);                            \
    break;
  switch (rule) {
    ISING_BASIC_CASE(0)
    ISING_BASIC_CASE(1)
    ISING_BASIC_CASE(2)
    ISING_BASIC_CASE(3)
    ISING_BASIC_CASE(4)
    ISING_BASIC_CASE(5)
    ISING_BASIC_CASE(6)
    ISING_BASIC_CASE(7)
    default: return cudaErrorInvalidValue;
  }
#undef ISING_BASIC_CASE
  return cudaGetLastError();
}

cudaError_t launch_basic_init(int grid, cudaStream_t st, int8_t* black, int8_t* white, int64_t nx,
                              int64_t ny, int cold, const PhiloxKeys& keys) {
  k_basic_init<<<grid, 256, 0, st>>>(black, white, nx, ny, cold, keys);
  return cudaGetLastError();
}

cudaError_t launch_basic_observables(int grid, cudaStream_t st, const int8_t* black,
                                     const int8_t* white, int64_t nx, int64_t ny,
                                     unsigned long long* out) {
  if ((ny & 15) == 0) {
    const int64_t chunks = ny >> 4;
    const unsigned gx = (unsigned)std::min<int64_t>((chunks + 255) / 256, 65535);
    const unsigned gy = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nx, std::max(1, grid / (int)gx)));
    k_basic_observables16<<<dim3(gx, gy), 256, 0, st>>>(black, white, nx, ny, out);
  } else {
    k_basic_observables<<<grid, 256, 0, st>>>(black, white, nx, ny, out);
  }
  return cudaGetLastError();
}

cudaError_t launch_basic_convert(int grid, cudaStream_t st, int8_t* black, int8_t* white,
                                 int8_t* full, int64_t ny, int64_t r0, int64_t rows, int to_full,
                                 unsigned int* bad) {
  if ((ny & 7) == 0) {
    const int64_t segs = ny >> 3;  // 16-byte segments of a full row
    const unsigned gx = (unsigned)std::min<int64_t>((segs + 255) / 256, 65535);
    const unsigned gy = (unsigned)std::max<int64_t>(1, std::min<int64_t>(rows, std::max(1, grid / (int)gx)));
    k_basic_convert16<<<dim3(gx, gy), 256, 0, st>>>(black, white, full, ny, r0, rows, to_full, bad);
  } else {
    k_basic_convert<<<grid, 256, 0, st>>>(black, white, full, ny, r0, rows, to_full, bad);
  }
  return cudaGetLastError();
}

}  // namespace ising
