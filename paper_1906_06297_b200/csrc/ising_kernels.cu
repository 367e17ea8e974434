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
#include <cuda_runtime.h>

#include "ising_kernels.cuh"

namespace ising {

// ------------------------------------------------------------------ Philox
// Philox4x32-10 (Salmon et al., SC'11), the generator the paper uses through
// cuRAND.  Counter {c0, c1, c2, c3}; the key schedule is
// precomputed per launch (PhiloxKeys) so each round is 2 IMAD.WIDE.U32 + 2 LOP3.
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

__device__ __forceinline__ ulonglong2 ld_nc_v2(const uint64_t* p) {
  ulonglong2 v;
  asm("ld.global.nc.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p));
  return v;
}

__device__ __forceinline__ uint64_t ld_nc(const uint64_t* p) {
  uint64_t v;
  asm("ld.global.nc.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

constexpr uint32_t kLane0 = 0x11111111u;  // bit 0 of every nibble of a 32-bit half

// Per-half (8 lanes) classification of the aligned-neighbour count a = s ? n : 4 - n
// (s = spin bit, n = neighbour sum).  B = a + 3 in 3..7 per lane:
//   s = 1: B = n + 3;  s = 0: B = n ^ 7 = 7 - n.
// ge3 (a >= 3) <=> B in {6, 7} <=> bits 1 and 2 set; is4 (a = 4) <=> B = 7.
struct Class8 {
  uint32_t ge3, is4;  // lane bit at 4k
};

__device__ __forceinline__ Class8 classify8(uint32_t s, uint32_t n) {
  const uint32_t B = (n + 3u * s) ^ (7u * s) ^ 0x77777777u;
  const uint32_t g = B & (B << 1) & 0x44444444u;
  Class8 c;
  c.ge3 = g >> 2;
  c.is4 = (g & (B << 2)) >> 2;
  return c;
}

// One 64-bit target word: 16 spins of plane row `row` (global), plane columns
// 4*ctr0 .. 4*ctr0 + 15.  n, c, s: source words above / same / below; side: the
// spliced side word.  Metropolis acceptance:
// flip iff a <= 2 (e <= 0) or r < T[e].
template <int RULE>
__device__ __forceinline__ uint64_t update_word(uint64_t tgt, uint64_t n, uint64_t c, uint64_t s,
                                                uint64_t side, uint32_t ctr0, uint32_t row,
                                                const HalfSweepParams& p);

template <>
__device__ __forceinline__ uint64_t update_word<0>(uint64_t tgt, uint64_t n, uint64_t c, uint64_t s,
                                                   uint64_t side, uint32_t ctr0, uint32_t row,
                                                   const HalfSweepParams& p) {
  // "three additions are sufficient to compute the neighbors sums":
  // lanes hold 0/1 and sums <= 4, so the 64-bit adds split into independent halves.
  const uint32_t sum_lo = (uint32_t)n + (uint32_t)c + (uint32_t)s + (uint32_t)side;
  const uint32_t sum_hi =
      (uint32_t)(n >> 32) + (uint32_t)(c >> 32) + (uint32_t)(s >> 32) + (uint32_t)(side >> 32);
  const uint32_t t_lo = (uint32_t)tgt, t_hi = (uint32_t)(tgt >> 32);
  const Class8 cl = classify8(t_lo, sum_lo);
  const Class8 ch = classify8(t_hi, sum_hi);

  const uint32_t thr3 = p.acc.thr[3], thr4 = p.acc.thr[4];
  uint32_t c3lo = 0, c3hi = 0, c4lo = 0, c4hi = 0;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const uint4 r = philox4x32_10(ctr0 + b, row, p.t, p.colour, p.keys);
    const uint32_t rr[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int k = 4 * b + q;
      const uint32_t bit = 1u << (4 * (k & 7));
      if (k < 8) {
        if (rr[q] < thr3) c3lo |= bit;
        if (rr[q] < thr4) c4lo |= bit;
      } else {
        if (rr[q] < thr3) c3hi |= bit;
        if (rr[q] < thr4) c4hi |= bit;
      }
    }
  }
  // classes whose threshold is 2^32 ("always") need no draw
  const uint32_t need3 = (p.acc.always_mask & 8u) ? 0u : kLane0;
  const uint32_t need4 = (p.acc.always_mask & 16u) ? 0u : kLane0;
  const uint32_t is3lo = cl.ge3 & ~cl.is4, is3hi = ch.ge3 & ~ch.is4;
  const uint32_t needlo = (is3lo & need3) | (cl.is4 & need4);
  const uint32_t needhi = (is3hi & need3) | (ch.is4 & need4);
  const uint32_t flo = (~needlo | (c3lo & is3lo) | (c4lo & cl.is4)) & kLane0;
  const uint32_t fhi = (~needhi | (c3hi & is3hi) | (c4hi & ch.is4)) & kLane0;
  return tgt ^ (((uint64_t)fhi << 32) | flo);
}

// Heat bath: flip iff r < T[a] for every class.
// T is non-increasing in a, so "r < T[a]" <=> a < #{m : r < T[m]}.
template <>
__device__ __forceinline__ uint64_t update_word<1>(uint64_t tgt, uint64_t n, uint64_t c, uint64_t s,
                                                   uint64_t side, uint32_t ctr0, uint32_t row,
                                                   const HalfSweepParams& p) {
  const uint64_t sum = n + c + s + side;  // no inter-lane carries (sums <= 4)
  // a = s ? n : 4 - n per lane
  const uint64_t S = tgt & 0x1111111111111111ull;
  const uint64_t mask = (S << 4) - S;  // 0xF in lanes with s = 1
  const uint64_t a = (sum & mask) | ((0x4444444444444444ull - sum) & ~mask);
  uint64_t flip = 0;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const uint4 r = philox4x32_10(ctr0 + b, row, p.t, p.colour, p.keys);
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

// One colour phase of one slab.  Work item = (band of H rows, 128-bit chunk
// column q); the thread walks down the band keeping the N/C/S source chunks in
// registers, so each source word is read from memory once per band (plus one halo
// row per band).  Grid-stride over items; the grid is a multiple of the SM count.
template <int RULE>
__global__ void __launch_bounds__(128) k_halfsweep(const HalfSweepParams p) {
  const int64_t W = p.W;
  const int64_t chunks = W >> 1;
  const uint64_t* src = p.src + W;  // local row r (r = -1 .. R) at src + r * W
  uint64_t* tgt = p.tgt + W;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t item = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; item < p.items;
       item += stride) {
    const int64_t q = item % chunks;
    const int band = (int)(item / chunks);
    const int ra = p.r_begin + band * p.H;
    const int rb = min(ra + p.H, p.r_end);
    const int64_t wc = 2 * q;
    const int64_t wwest = (wc == 0) ? W - 1 : wc - 1;     // periodic wrap
    const int64_t weast = (wc + 2 == W) ? 0 : wc + 2;
    ulonglong2 nv = ld_nc_v2(src + (int64_t)(ra - 1) * W + wc);
    ulonglong2 cv = ld_nc_v2(src + (int64_t)ra * W + wc);
    for (int r = ra; r < rb; ++r) {
      const ulonglong2 sv = ld_nc_v2(src + (int64_t)(r + 1) * W + wc);
      const int64_t gi = p.row0 + r;
      // side word: the left word if (black and i even) or (white and i odd), else the
      // right one (Fig. 3 caption PAPER.md:208; reading R2)
      const bool west = ((gi & 1) == 0) == (p.colour == 0);
      const uint64_t sw = ld_nc(src + (int64_t)r * W + (west ? wwest : weast));
      ulonglong2 tv = *reinterpret_cast<const ulonglong2*>(tgt + (int64_t)r * W + wc);
      uint64_t side0, side1;
      if (west) {
        side0 = (cv.x << 4) | (sw >> 60);
        side1 = (cv.y << 4) | (cv.x >> 60);
      } else {
        side0 = (cv.x >> 4) | (cv.y << 60);
        side1 = (cv.y >> 4) | (sw << 60);
      }
      const uint32_t ctr0 = (uint32_t)(4 * wc);  // Philox counter word 0 = j / 4 (reading R6)
      tv.x = update_word<RULE>(tv.x, nv.x, cv.x, sv.x, side0, ctr0, (uint32_t)gi, p);
      tv.y = update_word<RULE>(tv.y, nv.y, cv.y, sv.y, side1, ctr0 + 4, (uint32_t)gi, p);
      *reinterpret_cast<ulonglong2*>(tgt + (int64_t)r * W + wc) = tv;
      if (r == 0 && p.halo_up) *reinterpret_cast<ulonglong2*>(p.halo_up + wc) = tv;
      if (r == p.R - 1 && p.halo_dn) *reinterpret_cast<ulonglong2*>(p.halo_dn + wc) = tv;
      nv = cv;
      cv = sv;
    }
  }
}

// Philox-only throughput probe (ALU roofline denominator):
// the same philox4x32_10 as the half-sweep, counter {x, row, t, colour} with the
// same warp-uniform words, outputs XOR-folded so nothing but the fold is stored.
__global__ void __launch_bounds__(128) k_philox_probe(PhiloxKeys K, uint32_t blocks_per_thread,
                                                      uint32_t t, unsigned int* sink) {
  uint32_t acc = 0;
  const uint32_t row = blockIdx.x;
  for (uint32_t b = 0; b < blocks_per_thread; ++b) {
    const uint4 r = philox4x32_10(b * blockDim.x + threadIdx.x, row, t, 1u, K);
    acc ^= r.x ^ r.y ^ r.z ^ r.w;
  }
  if (acc == 0x9E3779B9u) atomicAdd(sink, 1u);  // practically never; keeps the work live
}

cudaError_t launch_philox_probe(int grid, cudaStream_t st, const PhiloxKeys& K,
                                uint32_t blocks_per_thread, unsigned int* sink) {
  k_philox_probe<<<grid, 128, 0, st>>>(K, blocks_per_thread, 1u, sink);
  return cudaGetLastError();
}

cudaError_t launch_halfsweep(int rule, int grid, cudaStream_t st, const HalfSweepParams& p) {
  if (rule == 0)
    k_halfsweep<0><<<grid, 128, 0, st>>>(p);
  else
    k_halfsweep<1><<<grid, 128, 0, st>>>(p);
  return cudaGetLastError();
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
        const uint4 r = philox4x32_10((uint32_t)(4 * w + b), (uint32_t)gi, 0u, (uint32_t)c, p.keys);
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
    up += __popcll(b) + __popcll(cw);
    anti += __popcll(b ^ nw) + __popcll(b ^ cw) + __popcll(b ^ sw) + __popcll(b ^ side);
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
// Full lattice (row-major +-1 bytes) <-> planes.  Site (i, J) has colour
// c = (i + J) & 1 and plane column J / 2, i.e. J = 2 j + ((i + c) & 1).
__global__ void k_pack(const PackParams p) {
  const int64_t rows = p.rb - p.ra;
  const int64_t total = 2 * rows * p.W;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += stride) {
    const int c = (int)(idx / (rows * p.W));
    const int64_t rem = idx - (int64_t)c * rows * p.W;
    const int64_t lr = rem / p.W;  // row within staging
    const int64_t w = rem - lr * p.W;
    const int64_t r = p.ra + lr;   // padded local row (-1 .. R)
    int64_t gi = (p.row0 + r) % p.N;
    if (gi < 0) gi += p.N;
    const int x = (int)((gi + c) & 1);
    const int8_t* rowp = p.full + lr * p.M;
    uint64_t word = 0;
    unsigned int bad = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int8_t v = rowp[2 * (16 * w + k) + x];
      bad |= (v != 1 && v != -1);
      if (v == 1) word |= 1ull << (4 * k);
    }
    if (bad) atomicOr(p.bad, 1u);
    p.plane[c][(r + 1) * p.W + w] = word;
  }
}

__global__ void k_unpack(const UnpackParams p) {
  const int64_t rows = p.rb - p.ra;
  const int64_t total = 2 * rows * p.W;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += stride) {
    const int c = (int)(idx / (rows * p.W));
    const int64_t rem = idx - (int64_t)c * rows * p.W;
    const int64_t lr = rem / p.W;
    const int64_t w = rem - lr * p.W;
    const int64_t r = p.ra + lr;
    const int64_t gi = p.row0 + r;
    const int x = (int)((gi + c) & 1);
    const uint64_t word = p.plane[c][(r + 1) * p.W + w];
    int8_t* rowp = p.full + lr * p.M;
#pragma unroll
    for (int k = 0; k < 16; ++k) rowp[2 * (16 * w + k) + x] = ((word >> (4 * k)) & 1) ? 1 : -1;
  }
}

}  // namespace ising
