// ising_kernels.cuh — device-side layout, Philox and kernel parameter blocks.
//
// Layout (DESIGN.md §Data layout; §3.3): each colour plane of a slab
// is a row-major array of (R + 2) rows x W uint64 words, W = L_cols / 32.  Array
// row 0 is the top halo (global row row0 - 1 mod N), rows 1..R the slab's rows,
// row R + 1 the bottom halo (global row row0 + R mod N).  Lane k of word w (bits
// [4k, 4k+4)) holds plane column j = 16 w + k; nibble value 1 = spin +1,
// 0 = spin -1 ("-1/1 are mapped to 0/1").  Site (i, J) is black iff
// i + J is even and sits in plane column J / 2 (reading R1).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace ising {

constexpr uint32_t kPhiloxM0 = 0xD2511F53u;
constexpr uint32_t kPhiloxM1 = 0xCD9E8D57u;
constexpr uint32_t kPhiloxW0 = 0x9E3779B9u;
constexpr uint32_t kPhiloxW1 = 0xBB67AE85u;

// Per-launch Philox key schedule (k0, k1 for each of the 10 rounds), computed on
// the host once per seed so the kernels read it from the constant bank.
struct PhiloxKeys {
  uint32_t k0[10];
  uint32_t k1[10];
};

// Acceptance parameters for one half-sweep.  Class a = number of neighbours
// aligned with the spin (0..4), e = s*h = 2a - 4.  thr[a] is the low 32 bits of
// the threshold T[e] (flip iff r < T[e]); bit a of always_mask marks T[e] = 2^32.
struct Accept {
  uint32_t thr[5];
  uint32_t always_mask;
  uint32_t keep3, keep4;  // Metropolis: 0 if T[a=3] / T[a=4] is 2^32, else ~0
};

struct HalfSweepParams {
  uint64_t* tgt;          // target plane (colour c), padded (R + 2) x W
  const uint64_t* src;    // source plane (colour 1 - c), padded (R + 2) x W
  uint64_t* halo_up;      // destination row for local row 0 (upper slab's bottom halo) or null
  uint64_t* halo_dn;      // destination row for local row R - 1 (lower slab's top halo) or null
  int64_t W;              // words per plane row (multiple of 2)
  int64_t row0;           // global row of local row 0
  int32_t R;              // rows in the slab
  int32_t r_begin;        // first local row to update
  int32_t r_end;          // one past the last local row to update
  int32_t H;              // rows per work item (register-rolling band)
  int64_t items;          // number of work items = (W / 2) * ceil((r_end - r_begin) / H)
  uint32_t t;             // sweep index (>= 1)
  uint32_t colour;        // 0 black, 1 white
  PhiloxKeys keys;
  Accept acc;
};

struct InitParams {
  uint64_t* plane[2];
  int64_t W;
  int64_t row0;           // global row of local row 0
  int64_t N;              // total rows (for the halo wrap)
  int32_t R;
  int32_t cold;
  PhiloxKeys keys;
};

struct ObsParams {
  const uint64_t* black;
  const uint64_t* white;
  int64_t W;
  int64_t row0;
  int32_t R;
  unsigned long long* out;  // [0] = up count, [1] = antiparallel bonds
};

struct PackParams {
  uint64_t* plane[2];
  const int8_t* full;     // staging: rows [ra, rb) of the slab's padded row range, M bytes each
  int64_t W;
  int64_t M;
  int64_t row0;
  int64_t N;
  int32_t ra;             // first padded local row in staging (may be -1)
  int32_t rb;
  unsigned int* bad;      // set to 1 if a value is not -1/+1
};

struct UnpackParams {
  const uint64_t* plane[2];
  int8_t* full;           // staging: rows [ra, rb) of the slab (interior rows only)
  int64_t W;
  int64_t M;
  int64_t row0;
  int32_t ra;
  int32_t rb;
};

// Host-side launchers (defined in ising_kernels.cu).
cudaError_t launch_halfsweep(int rule, int grid, cudaStream_t st, const HalfSweepParams& p);
cudaError_t halfsweep_occupancy(int* blocks_per_sm);
cudaError_t launch_philox_probe(int grid, cudaStream_t st, const PhiloxKeys& K,
                                uint32_t blocks_per_thread, unsigned int* sink);

}  // namespace ising
